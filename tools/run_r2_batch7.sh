#!/bin/bash
# L2-prefetch ring option: parity + A/B; sanitizers (bulk gather added); e2e host-gather CTA A/B.
mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_gpu_allreduce.py -q -x -k "l2_prefetch or c5_maximum" -p no:cacheprovider > gpurun_out/pf_pytest.log 2>&1
tail -2 gpurun_out/pf_pytest.log
timeout 600 python tools/ab_bulk.py l2_prefetch > gpurun_out/ab_l2pf.jsonl 2>&1
cat gpurun_out/ab_l2pf.jsonl
bash tools/run_sanitizers.sh
bash tools/run_r2_e2e_ab.sh
