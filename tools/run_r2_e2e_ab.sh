#!/bin/bash
# e2e leg: CTAs of the host-source (PCIe) gather that runs beside the compute on a side stream.
mkdir -p gpurun_out
: > gpurun_out/e2e_ab.jsonl
for rep in 1 2; do
for hg in 16 32 64 128; do
  PR_GATHER_HOST_GRID=$hg timeout 600 python bench.py --steps 5 --warmup 3 --e2e-epochs 3 --no-vgg --no-cpu-baseline --no-colocated 2>/dev/null \
    | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(json.dumps({'host_grid': $hg, 'rep': $rep, 'value': d['value'], 'e2e': d['e2e']['value']}))" >> gpurun_out/e2e_ab.jsonl
done
done
cat gpurun_out/e2e_ab.jsonl
