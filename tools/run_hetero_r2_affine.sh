#!/bin/bash
# The affine step-cost controller (DESIGN.md §3 #49) at the survey's C2 (batch, adaptive) and C4 configs,
# both K4 emulations, stop rule as specified (window 2, tol 1).  Output: gpurun_out/hetero_r2_affine.jsonl
out=${1:-gpurun_out/hetero_r2_affine.jsonl}
: > "$out"
for spin in sample t1; do
  for sc in c4 c2-adapt c4-replace; do
    echo "== $sc spin=$spin model=affine" >&2
    python experiments.py --virtual --scenario "$sc" --epochs 8 --spin "$spin" --model affine \
      | sed "s/^{/{\"run\": \"$sc-affine\", \"spin_mode\": \"$spin\", /" >> "$out"
  done
done
