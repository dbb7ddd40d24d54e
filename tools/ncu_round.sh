#!/bin/bash
# ncu evidence for the current kernels: full captures in isolation at bench sizes + the bench launch list.
mkdir -p gpurun_out
NCU="ncu --clock-control none"
$NCU --set full --import-source on -k regex:gather_tma_kernel -s 2 -c 1 -f -o gpurun_out/prof_gather_epoch python tools/profile_kernels.py gather_epoch 3 > gpurun_out/ncu_gather.log 2>&1
$NCU --set full --import-source on -k regex:ring_kernel -s 2 -c 1 -f -o gpurun_out/prof_ring python tools/profile_kernels.py ring 3 > gpurun_out/ncu_ring.log 2>&1
$NCU --set full --import-source on -k regex:permute_kernel -s 1 -c 1 -f -o gpurun_out/prof_permute python tools/profile_kernels.py shard 2 > gpurun_out/ncu_permute.log 2>&1
timeout 1500 $NCU --metrics gpu__time_duration.sum --csv --log-file gpurun_out/launches.csv python bench.py --steps 1 --warmup 0 --e2e-epochs 0 --no-cpu-baseline --no-colocated > gpurun_out/ncu_bench.log 2>&1
ls -la gpurun_out
