#!/bin/bash
# K1 default (refill, 16 warps/SM): K1 parity tests, timing, ncu --set full.
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_kernels.py tests/test_gpu_end_to_end.py -q -x -p no:cacheprovider > gpurun_out/k1c_pytest.log 2>&1
echo "pytest exit $?" >> gpurun_out/k1c_pytest.log
PR_K1_KERNEL=refill timeout 300 python tools/ab_k1.py --child > gpurun_out/k1c_default.jsonl 2>&1
timeout 600 ncu --clock-control none --set full --import-source on -k regex:walk_refill -s 1 -c 1 -f -o gpurun_out/k1c_refill \
    python tools/profile_kernels.py shard 2 > gpurun_out/k1c_ncu_refill.log 2>&1
ncu -i gpurun_out/k1c_refill.ncu-rep --page raw --csv > gpurun_out/k1c_refill_raw.csv 2>/dev/null
tail -2 gpurun_out/k1c_pytest.log; cat gpurun_out/k1c_default.jsonl
