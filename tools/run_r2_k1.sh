#!/bin/bash
# K1 lane-refill walk: parity (K1 tests), A/B against the one-thread-per-index kernel, ncu --set full of both.
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_kernels.py -q -x -p no:cacheprovider -k "permute or shard or philox" > gpurun_out/k1_pytest.log 2>&1
echo "pytest exit $?" >> gpurun_out/k1_pytest.log
timeout 600 python tools/ab_k1.py > gpurun_out/k1_ab.jsonl 2> gpurun_out/k1_ab.err
timeout 600 ncu --clock-control none --set full --import-source on -k regex:walk_refill -s 1 -c 1 -f -o gpurun_out/k1_refill \
    python tools/profile_kernels.py shard 2 > gpurun_out/k1_ncu_refill.log 2>&1
PR_K1_KERNEL=direct timeout 600 ncu --clock-control none --set full --import-source on -k regex:walk_direct -s 1 -c 1 -f -o gpurun_out/k1_direct \
    python tools/profile_kernels.py shard 2 > gpurun_out/k1_ncu_direct.log 2>&1
for k in refill direct; do ncu -i gpurun_out/k1_$k.ncu-rep --page raw --csv > gpurun_out/k1_${k}_raw.csv 2>/dev/null; done
tail -2 gpurun_out/k1_pytest.log; cat gpurun_out/k1_ab.jsonl; tail -3 gpurun_out/k1_ab.err
