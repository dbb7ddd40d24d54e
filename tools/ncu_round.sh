#!/bin/bash
# ncu evidence: full captures of the library kernels in isolation + the bench launch list.
mkdir -p gpurun_out
NCU="ncu --clock-control none"
$NCU --set full --import-source on -k regex:gather_kernel -s 2 -c 2 -f -o gpurun_out/prof_gather python tools/profile_kernels.py gather 4 > gpurun_out/ncu_gather.log 2>&1
$NCU --set full --import-source on -k regex:gather_kernel -s 2 -c 1 -f -o gpurun_out/prof_gather_imagenet python tools/profile_kernels.py gather_imagenet 4 > gpurun_out/ncu_gather_in.log 2>&1
$NCU --set full --import-source on -k regex:ring_kernel -s 1 -c 1 -f -o gpurun_out/prof_ring python tools/profile_kernels.py ring 2 > gpurun_out/ncu_ring.log 2>&1
$NCU --set full --import-source on -k regex:permute_kernel -s 1 -c 1 -f -o gpurun_out/prof_permute python tools/profile_kernels.py shard 2 > gpurun_out/ncu_permute.log 2>&1
timeout 1200 $NCU --metrics gpu__time_duration.sum --csv --log-file gpurun_out/launches.csv python bench.py --steps 1 --warmup 1 --e2e-epochs 0 --no-cpu-baseline --no-colocated > gpurun_out/ncu_bench.log 2>&1
ls -la gpurun_out
