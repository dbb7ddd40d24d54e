#!/bin/bash
# Pull two-shot: the whole allreduce parity file, timings, ncu --set full in both regimes (+ the ring's
# per-channel regime for the same store-path metrics).
mkdir -p gpurun_out
timeout 1800 python -m pytest tests/test_gpu_allreduce.py -q -x -p no:cacheprovider > gpurun_out/pull2_pytest.log 2>&1
echo "pytest exit $?" >> gpurun_out/pull2_pytest.log
for m in pull pull_cta ring_cta; do timeout 300 python tools/profile_kernels.py $m 8 >> gpurun_out/pull2_times.txt 2>&1; done
NCU="ncu --clock-control none --set full --import-source on"
timeout 600 $NCU -k regex:twoshot_pull -s 1 -c 1 -f -o gpurun_out/pull2_colocated python tools/profile_kernels.py pull 2 > gpurun_out/pull2_ncu1.log 2>&1
timeout 600 $NCU -k regex:twoshot_pull -s 1 -c 1 -f -o gpurun_out/pull2_cta python tools/profile_kernels.py pull_cta 2 > gpurun_out/pull2_ncu2.log 2>&1
timeout 600 $NCU -k regex:ring_kernel -s 1 -c 1 -f -o gpurun_out/pull2_ring_cta python tools/profile_kernels.py ring_cta 2 > gpurun_out/pull2_ncu3.log 2>&1
for k in colocated cta ring_cta; do ncu -i gpurun_out/pull2_$k.ncu-rep --page raw --csv > gpurun_out/pull2_${k}_raw.csv 2>/dev/null; done
tail -n 3 gpurun_out/pull2_pytest.log; cat gpurun_out/pull2_times.txt
