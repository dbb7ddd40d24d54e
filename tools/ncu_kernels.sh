#!/bin/bash
# Full ncu captures of the library kernels exactly as the bench launches them (one GPU).
mkdir -p gpurun_out
NCU="ncu --clock-control none --set full --import-source on"
$NCU -k regex:gather_kernel -s 1 -c 1 -f -o gpurun_out/prof_gather_hwc python tools/profile_kernels.py gather_epoch_hwc_lsu 3 > gpurun_out/ncu_gather.log 2>&1
$NCU -k regex:ring_kernel -s 2 -c 1 -f -o gpurun_out/prof_ring python tools/profile_kernels.py ring 3 > gpurun_out/ncu_ring.log 2>&1
$NCU -k regex:walk_ -s 1 -c 1 -f -o gpurun_out/prof_permute python tools/profile_kernels.py shard 2 > gpurun_out/ncu_permute.log 2>&1
ls -la gpurun_out/*.ncu-rep
