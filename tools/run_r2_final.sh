#!/bin/bash
# Final verification of the round: full GPU parity suite, smoke(), the default bench line.
mkdir -p gpurun_out
timeout 2700 python -m pytest tests -m gpu -q -x -p no:cacheprovider > gpurun_out/pytest_gpu_final.log 2>&1
echo "pytest exit $?" >> gpurun_out/pytest_gpu_final.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke(); print('smoke ok')" > gpurun_out/smoke_final.log 2>&1
timeout 1500 python bench.py > gpurun_out/bench_final.json 2> gpurun_out/bench_final.err
tail -3 gpurun_out/pytest_gpu_final.log; tail -2 gpurun_out/smoke_final.log; tail -2 gpurun_out/bench_final.err
head -c 300 gpurun_out/bench_final.json
