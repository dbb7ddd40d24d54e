#!/bin/bash
# Round-2 heterogeneity runs at the survey's own C2 / C4 configs, both K4 emulations
# (DESIGN.md §3 #46), virtual mode (all ranks on one GPU, timed one after another), with the affine-cost
# min-max bound beside the linear Σspeed bound.  Output: gpurun_out/hetero_r2.jsonl, gpurun_out/hetero_r2.csv
out=${1:-gpurun_out/hetero_r2.jsonl}
csv=${out%.jsonl}.csv
: > "$out"; rm -f "$csv"
for spin in t1 sample; do
  for sc in c2 c2-equal c2-adapt c4 c4-static; do
    extra=""
    name=$sc
    if [ "$sc" = "c4-static" ]; then name=c4; extra="--static"; fi
    echo "== $sc spin=$spin" >&2
    python experiments.py --virtual --scenario "$name" --epochs 6 --spin "$spin" $extra --metrics-csv "$csv" \
      | sed "s/^{/{\"run\": \"$sc\", \"spin_mode\": \"$spin\", /" >> "$out"
  done
done
