#!/bin/bash
# Repeatability of the heterogeneity results: 3 repetitions of C4 / C2-adapt / C4-replace (sample emulation,
# stop rule as specified) with the paper's Eq. 10 and with the affine controller.
out=${1:-gpurun_out/hetero_reps.jsonl}
: > "$out"
for rep in 1 2 3; do
  for sc in c4 c2-adapt c4-replace; do
    for model in proportional affine; do
      echo "== rep $rep $sc $model" >&2
      timeout 900 python experiments.py --virtual --scenario $sc --epochs 6 --spin sample --model $model \
        | sed "s/^{/{\"rep\": $rep, \"run\": \"$sc-$model\", \"spin_mode\": \"sample\", /" >> "$out"
    done
  done
done
