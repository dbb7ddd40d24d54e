#!/bin/bash
# K1 refill: warps-per-SM sweep (A/B vs the direct kernel, bit-exact check) + ncu of the default.
mkdir -p gpurun_out
timeout 600 python tools/ab_k1.py > gpurun_out/k1b_ab.jsonl 2> gpurun_out/k1b_ab.err
timeout 600 ncu --clock-control none --set full --import-source on -k regex:walk_refill -s 1 -c 1 -f -o gpurun_out/k1b_refill \
    python tools/profile_kernels.py shard 2 > gpurun_out/k1b_ncu_refill.log 2>&1
ncu -i gpurun_out/k1b_refill.ncu-rep --page raw --csv > gpurun_out/k1b_refill_raw.csv 2>/dev/null
cat gpurun_out/k1b_ab.jsonl; tail -3 gpurun_out/k1b_ab.err
