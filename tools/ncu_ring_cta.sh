#!/bin/bash
# ncu --set full of K3 in the per-channel (CTA-bound) regime: 2 ranks co-located, cross-GPU config.
mkdir -p gpurun_out
ncu --clock-control none --set full --import-source on -k regex:ring_kernel -s 2 -c 1 -f -o gpurun_out/prof4_ring_cta \
    python tools/profile_kernels.py ring_cta 3 > gpurun_out/ncu4_ring_cta.log 2>&1
ncu -i gpurun_out/prof4_ring_cta.ncu-rep --page source --csv > gpurun_out/prof4_ring_cta_source.csv 2>/dev/null
ls -la gpurun_out/prof4_ring_cta*
