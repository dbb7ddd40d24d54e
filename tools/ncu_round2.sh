#!/bin/bash
# Round-2 ncu evidence (one GPU): full captures of every library kernel at the bench's sizes, and the launch
# list of the bench's headline command.  Summarise here with
#   python tools/summarize_ncu.py round2 gpurun_out/prof2_*.ncu-rep --launches gpurun_out/launches2.csv
mkdir -p gpurun_out
NCU="ncu --clock-control none --set full --import-source on"
$NCU -k regex:sgd_kernel -s 2 -c 1 -f -o gpurun_out/prof2_sgd python tools/profile_kernels.py sgd 3 > gpurun_out/ncu2_sgd.log 2>&1
$NCU -k regex:sgd_kernel -s 2 -c 1 -f -o gpurun_out/prof2_sgd_vgg16 python tools/profile_kernels.py sgd_vgg16 3 > gpurun_out/ncu2_sgdv.log 2>&1
$NCU -k regex:gather_kernel -s 2 -c 1 -f -o gpurun_out/prof2_gather_hwc python tools/profile_kernels.py gather_epoch_hwc_lsu 3 > gpurun_out/ncu2_gather.log 2>&1
$NCU -k regex:gather_kernel -s 2 -c 1 -f -o gpurun_out/prof2_gather_imagenet python tools/profile_kernels.py gather_imagenet_epoch_hwc_lsu 3 > gpurun_out/ncu2_gatheri.log 2>&1
$NCU -k regex:ring_kernel -s 2 -c 1 -f -o gpurun_out/prof2_ring python tools/profile_kernels.py ring 3 > gpurun_out/ncu2_ring.log 2>&1
$NCU -k regex:ring_kernel -s 2 -c 1 -f -o gpurun_out/prof2_ring_fused python tools/profile_kernels.py ring_fused_only 3 > gpurun_out/ncu2_ringf.log 2>&1
$NCU -k regex:walk_ -s 1 -c 1 -f -o gpurun_out/prof2_permute python tools/profile_kernels.py shard 2 > gpurun_out/ncu2_permute.log 2>&1
BENCH="bench.py --steps 1 --warmup 1 --e2e-epochs 0 --no-cpu-baseline --no-colocated --no-vgg"
timeout 1500 ncu --clock-control none --metrics gpu__time_duration.sum --csv --log-file gpurun_out/launches2.csv python $BENCH > gpurun_out/ncu2_bench.log 2>&1
ls -la gpurun_out/prof2_*.ncu-rep
