#!/bin/bash
# Pull two-shot: parity (new tests + the randomized all-algorithm sweep), A/B against ring / push two-shot.
mkdir -p gpurun_out
timeout 1200 python -m pytest tests/test_gpu_allreduce.py -q -x -p no:cacheprovider -k "pull or randomized" > gpurun_out/pull_pytest.log 2>&1
echo "pytest exit $?" >> gpurun_out/pull_pytest.log
tail -n 3 gpurun_out/pull_pytest.log
timeout 900 python tools/ab_pull.py > gpurun_out/pull_ab.jsonl 2> gpurun_out/pull_ab.err
cat gpurun_out/pull_ab.jsonl; tail -n 5 gpurun_out/pull_ab.err
