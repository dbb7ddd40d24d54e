#!/bin/bash
# Co-located channel default 128/P: parity of every allreduce path + IPC, ring timings at P = 2/4/8;
# then the ncu capture of K3 in the per-channel regime.
mkdir -p gpurun_out
timeout 1500 python -m pytest tests/test_gpu_allreduce.py tests/test_multiproc.py -q -x -p no:cacheprovider > gpurun_out/b9_pytest.log 2>&1
tail -2 gpurun_out/b9_pytest.log
timeout 600 python tools/profile_kernels.py ring_sizes 20 > gpurun_out/b9_ring_sizes.txt 2>&1
cat gpurun_out/b9_ring_sizes.txt
bash tools/ncu_ring_cta.sh
