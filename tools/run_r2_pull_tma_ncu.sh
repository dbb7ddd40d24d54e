#!/bin/bash
# ncu --set full: register-queued vs TMA-staged pull at C3's VGG-16 size (P = 4 co-located).
mkdir -p gpurun_out
NCU="ncu --clock-control none --set full --import-source on"
timeout 600 $NCU -k regex:twoshot_pull -s 1 -c 1 -f -o gpurun_out/pull_vgg python tools/profile_kernels.py pull_vgg 8 > gpurun_out/pull_vgg_ncu.log 2>&1
timeout 600 $NCU -k regex:twoshot_pull_tma -s 1 -c 1 -f -o gpurun_out/pull_tma_vgg python tools/profile_kernels.py pull_tma_vgg 8 > gpurun_out/pull_tma_vgg_ncu.log 2>&1
for k in pull_vgg pull_tma_vgg; do ncu -i gpurun_out/$k.ncu-rep --page raw --csv > gpurun_out/${k}_raw.csv 2>/dev/null; done
python tools/profile_kernels.py pull_vgg 8; python tools/profile_kernels.py pull_tma_vgg 8
