#!/bin/bash
# Pull two-shot vs push two-shot vs ring across sizes (co-located, .sys scope and .gpu scope, in CUDA graphs):
# is the pull a better AUTO choice than the push two-shot?
mkdir -p gpurun_out
for P in 2 4 8; do
  for sc in "" "--sys"; do
    timeout 600 python tools/ar_latency.py --P $P $sc --graph --reps 20 --algos ring,two_shot,pull \
      --sizes 65536,262144,1048576,4194304,16777216,67108864 >> gpurun_out/pull_lat.jsonl 2>> gpurun_out/pull_lat.err
  done
done
python - <<'PY'
import json
rows=[json.loads(l) for l in open("gpurun_out/pull_lat.jsonl")]
for P in (2,4,8):
    for sysf in (False,True):
        print(f"P={P} sys={sysf}")
        for Z in sorted({r["bytes"] for r in rows}):
            d={r["algo"]:r["us"] for r in rows if r["P"]==P and r["sys"]==sysf and r["bytes"]==Z}
            print(f"   {Z:>9}  " + "  ".join(f"{k}={v:8.1f}" for k,v in d.items()))
PY
tail -n 3 gpurun_out/pull_lat.err
