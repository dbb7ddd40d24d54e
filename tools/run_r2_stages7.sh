#!/bin/bash
# 7 stages of 16 KiB (224 KiB of shared memory) vs the 6-stage default: per-channel rate at P = 2 / 8 and the
# co-located P = 8 ResNet-18 ring, plus the parity of a 7-stage group.
mkdir -p gpurun_out
: > gpurun_out/stages7.jsonl
for rep in 1 2; do
for pc in "2 16" "8 4"; do
  set -- $pc
  for st in 6 7; do
    timeout 300 python tools/sweep_cta.py --P $1 --channels $2 --mib 128 --sys --cfg "{\"stages\": $st, \"tile_bytes\": 16384, \"slot_bytes\": 1048576, \"threads\": 512, \"slots\": 8}" >> gpurun_out/stages7.jsonl 2>&1
  done
done
done
cat gpurun_out/stages7.jsonl | cut -c1-200
python - <<'PY'
import torch, paper_2111_08272_b200 as pr, time
L = 11_689_512
for st in (6, 7):
    cs = pr.comm_init_local(8, 0, pr.comm_config(stages=st))
    b = [torch.randn(L, device="cuda") for _ in range(8)]
    n = [64, 64, 64, 64, 128, 128, 256, 256]
    for _ in range(3): pr.weighted_allreduce_local(cs, b, n)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(20): pr.weighted_allreduce_local(cs, b, n)
    e1.record(); torch.cuda.synchronize()
    print("P8 resnet18 ring stages", st, round(e0.elapsed_time(e1) / 20 * 1e3, 1), "us")
    for c in cs: c.destroy()
PY
