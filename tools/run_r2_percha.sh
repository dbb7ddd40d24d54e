#!/bin/bash
# Per-channel bus throughput vs P with HBM far from saturated (few CTAs in total): the store-path analysis
# predicts ≈ 1.4× more per channel at P = 8 than at P = 2 (stores per bus byte 1.07 vs 1.5).
mkdir -p gpurun_out
CFG='{"stages": 6, "tile_bytes": 16384, "slot_bytes": 1048576, "threads": 512, "slots": 8}'
: > gpurun_out/percha.jsonl
for rep in 1 2; do
for pc in "2 8" "2 16" "4 4" "4 8" "8 2" "8 4"; do
  set -- $pc
  timeout 300 python tools/sweep_cta.py --P $1 --channels $2 --mib 128 --sys --cfg "$CFG" >> gpurun_out/percha.jsonl 2>&1
done
done
cat gpurun_out/percha.jsonl
