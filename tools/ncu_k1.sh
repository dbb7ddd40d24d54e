#!/bin/bash
# K1 (permutation) --set full capture at N = 1,281,167 for its integer-ALU roofline (issue slots, pipes).
mkdir -p gpurun_out
ncu --clock-control none --set full --import-source on -k regex:walk_ -s 1 -c 1 -f -o gpurun_out/prof5_permute \
    python tools/profile_kernels.py shard 2 > gpurun_out/ncu5_permute.log 2>&1
ncu -i gpurun_out/prof5_permute.ncu-rep --page raw --csv > gpurun_out/prof5_permute_raw.csv 2>/dev/null
ls -la gpurun_out/prof5_permute*
