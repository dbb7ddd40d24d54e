#!/bin/bash
# Final: full GPU suite, smoke, bench line, ncu of the fused pull kernel.
mkdir -p gpurun_out
timeout 2700 python -m pytest tests -m gpu -q -x -p no:cacheprovider > gpurun_out/pytest_gpu_final2.log 2>&1
echo "pytest exit $?" >> gpurun_out/pytest_gpu_final2.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke(); print('smoke ok')" > gpurun_out/smoke_final2.log 2>&1
timeout 1500 python bench.py > gpurun_out/bench_final2.json 2> gpurun_out/bench_final2.err
timeout 600 ncu --clock-control none --set full --import-source on -k regex:twoshot_pull -s 1 -c 1 -f -o gpurun_out/pull_fused \
    python tools/profile_kernels.py pull_fused 2 > gpurun_out/pull_fused_ncu.log 2>&1
ncu -i gpurun_out/pull_fused.ncu-rep --page raw --csv > gpurun_out/pull_fused_raw.csv 2>/dev/null
tail -n 3 gpurun_out/pytest_gpu_final2.log; tail -n 2 gpurun_out/smoke_final2.log; tail -n 2 gpurun_out/bench_final2.err
head -c 300 gpurun_out/bench_final2.json
