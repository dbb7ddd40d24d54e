#!/bin/bash
# K2 mix ceiling at the ImageNet size (store flavours, clean vs dirty L2), then the stop-rule follow-ups.
mkdir -p gpurun_out
nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o /tmp/mix_probe tools/probes/mix_probe.cu
timeout 300 /tmp/mix_probe > gpurun_out/mix_probe.txt 2>&1
timeout 300 python tools/profile_kernels.py gather_imagenet_epoch_hwc_lsu 10 > gpurun_out/k2_imagenet_iso.txt 2>&1
timeout 3000 bash tools/run_hetero_r2_extra.sh gpurun_out/hetero_r2c.jsonl 2> gpurun_out/hetero_r2c.err
tail -5 gpurun_out/hetero_r2c.err; cat gpurun_out/mix_probe.txt
