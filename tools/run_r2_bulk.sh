#!/bin/bash
# K2 bulk-store kernel: parity, then A/B against the LSU kernel at the bench's launch sizes (CTAs per SM
# swept through PR_GATHER_BULK_CTAS), then the K7 variants probe.
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_kernels.py -q -x -k "gather" -p no:cacheprovider > gpurun_out/bulk_pytest.log 2>&1
tail -3 gpurun_out/bulk_pytest.log
: > gpurun_out/bulk_ab.txt
for ctas in 2 3 4; do
  echo "== PR_GATHER_BULK_CTAS=$ctas" >> gpurun_out/bulk_ab.txt
  PR_GATHER_BULK_CTAS=$ctas timeout 300 python tools/profile_kernels.py gather_bulk_ab 10 >> gpurun_out/bulk_ab.txt 2>&1
done
nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o /tmp/sgd_probe tools/probes/sgd_probe.cu
timeout 300 /tmp/sgd_probe > gpurun_out/sgd_probe.txt 2>&1
cat gpurun_out/bulk_ab.txt
