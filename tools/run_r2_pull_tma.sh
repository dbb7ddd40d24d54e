#!/bin/bash
# TMA-staged pull: parity (all pull tests incl. the TMA ones), then the A/B of every K3 data path.
mkdir -p gpurun_out
timeout 1500 python -m pytest tests/test_gpu_allreduce.py -q -x -p no:cacheprovider -k "pull" > gpurun_out/ptma_pytest.log 2>&1
echo "pytest exit $?" >> gpurun_out/ptma_pytest.log
tail -n 3 gpurun_out/ptma_pytest.log
timeout 900 python tools/ab_pull.py > gpurun_out/ptma_ab.jsonl 2> gpurun_out/ptma_ab.err
grep -E 'pull' gpurun_out/ptma_ab.jsonl; tail -n 4 gpurun_out/ptma_ab.err
