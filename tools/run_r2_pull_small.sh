#!/bin/bash
# Small buffers: one-shot LL vs LL ring vs pull two-shot (co-located, in CUDA graphs, both scopes).
mkdir -p gpurun_out
for P in 2 8; do
  for sc in "" "--sys"; do
    timeout 600 python tools/ar_latency.py --P $P $sc --graph --reps 20 --algos oneshot,ll,pull \
      --sizes 4096,16384,65536,262144,1048576 --os-max 1048576 --ll-max 1048576 >> gpurun_out/pull_small.jsonl 2>> gpurun_out/pull_small.err
  done
done
python - <<'PY'
import json
rows=[json.loads(l) for l in open("gpurun_out/pull_small.jsonl")]
for P in (2,8):
    for sysf in (False,True):
        print(f"P={P} sys={sysf}")
        for Z in sorted({r["bytes"] for r in rows}):
            d={r["algo"]:r["us"] for r in rows if r["P"]==P and r["sys"]==sysf and r["bytes"]==Z}
            print(f"   {Z:>9}  " + "  ".join(f"{k}={v:8.1f}" for k,v in d.items()))
PY
tail -n 3 gpurun_out/pull_small.err
