#!/bin/bash
# ncu evidence for the current kernels: full captures in isolation at bench sizes + the launch list of
# the bench command (full data set, 1 warm-up + 1 timed epoch) with its live-event shares.
mkdir -p gpurun_out
NCU="ncu --clock-control none"
$NCU --set full --import-source on -k regex:'gather_kernel' -s 2 -c 1 -f -o gpurun_out/prof_gather_hwc python tools/profile_kernels.py gather_epoch_hwc_lsu 3 > gpurun_out/ncu_gather.log 2>&1
$NCU --set full --import-source on -k regex:ring_kernel -s 2 -c 1 -f -o gpurun_out/prof_ring python tools/profile_kernels.py ring 3 > gpurun_out/ncu_ring.log 2>&1
$NCU --set full --import-source on -k regex:ring_kernel -s 2 -c 1 -f -o gpurun_out/prof_ring_fused python tools/profile_kernels.py ring_fused_only 3 > gpurun_out/ncu_ring_fused.log 2>&1
$NCU --set full --import-source on -k regex:sgd_kernel -s 2 -c 1 -f -o gpurun_out/prof_sgd python tools/profile_kernels.py sgd 3 > gpurun_out/ncu_sgd.log 2>&1
$NCU --set full --import-source on -k regex:walk_ -s 1 -c 1 -f -o gpurun_out/prof_permute python tools/profile_kernels.py shard 2 > gpurun_out/ncu_permute.log 2>&1
BENCH="bench.py --steps 1 --warmup 1 --e2e-epochs 0 --no-cpu-baseline --no-colocated"
python $BENCH > gpurun_out/bench_profiling_variant.json 2> gpurun_out/bench_profiling_variant.err
timeout 1500 $NCU --metrics gpu__time_duration.sum --csv --log-file gpurun_out/launches.csv python $BENCH > gpurun_out/ncu_bench.log 2>&1
ls -la gpurun_out | tail -12
