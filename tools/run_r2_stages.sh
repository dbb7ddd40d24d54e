#!/bin/bash
# Per-channel throughput at P = 8 (few CTAs, HBM idle) vs pipeline depth / tile size: is a channel bound by
# bytes in flight (Little's law over the stage round trip) or by per-tile serial work?
mkdir -p gpurun_out
: > gpurun_out/stages.jsonl
for rep in 1 2; do
for c in "6 16384 512" "3 32768 512" "12 8192 512" "4 16384 512" "2 32768 512" "6 16384 256" "3 32768 256"; do
  set -- $c
  CFG="{\"stages\": $1, \"tile_bytes\": $2, \"slot_bytes\": 1048576, \"threads\": $3, \"slots\": 8}"
  timeout 300 python tools/sweep_cta.py --P 8 --channels 4 --mib 128 --sys --cfg "$CFG" >> gpurun_out/stages.jsonl 2>&1
done
done
cat gpurun_out/stages.jsonl
