#!/bin/bash
# Round-2 follow-ups: (1) the stop rule's effect — the same C2-adapt / C4 runs with --never-freeze, so Eq. 10
# keeps iterating towards its fixed point (equal step times); (2) C3 (VGG-16, ImageNet-shaped) with the
# measured-cost bound.  Output: gpurun_out/hetero_r2c.jsonl
out=${1:-gpurun_out/hetero_r2c.jsonl}
: > "$out"
for spin in sample t1; do
  for sc in c2-adapt c4; do
    echo "== $sc spin=$spin never-freeze" >&2
    python experiments.py --virtual --scenario "$sc" --epochs 10 --spin "$spin" --never-freeze \
      | sed "s/^{/{\"run\": \"$sc-nf\", \"spin_mode\": \"$spin\", /" >> "$out"
  done
done
echo "== c3 t1" >&2
python experiments.py --virtual --scenario c3 --epochs 4 --spin t1 | sed "s/^{/{\"run\": \"c3\", \"spin_mode\": \"t1\", /" >> "$out"
