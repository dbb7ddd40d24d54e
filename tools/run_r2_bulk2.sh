#!/bin/bash
# K2 bulk-store kernel: unit size (groups per thread) x CTAs per SM sweep, parity of each unit size.
mkdir -p gpurun_out
: > gpurun_out/bulk_ab2.txt
for g in 1 2 4; do
  PR_GATHER_BULK_GROUPS=$g timeout 600 python -m pytest tests/test_gpu_kernels.py -q -x -k "hwc" -p no:cacheprovider 2>&1 | tail -1 >> gpurun_out/bulk_ab2.txt
  for ctas in 4 6 8; do
    echo "== PR_GATHER_BULK_GROUPS=$g PR_GATHER_BULK_CTAS=$ctas" >> gpurun_out/bulk_ab2.txt
    PR_GATHER_BULK_GROUPS=$g PR_GATHER_BULK_CTAS=$ctas timeout 300 python tools/profile_kernels.py gather_bulk_ab 10 2>&1 | grep BULK >> gpurun_out/bulk_ab2.txt
  done
done
cat gpurun_out/bulk_ab2.txt
