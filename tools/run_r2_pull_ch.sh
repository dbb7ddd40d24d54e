#!/bin/bash
# Pull two-shot co-located channel sweep (full sizes): does filling all 148 SMs pay?
mkdir -p gpurun_out
python - > gpurun_out/pull_ch.jsonl 2> gpurun_out/pull_ch.err <<'PY'
import json, torch, sys
sys.path.insert(0, ".")
import paper_2111_08272_b200 as pr
def t(P, L, ch, threads=512, k=10):
    comms = pr.comm_init_local(P, 0, pr.comm_config(algo=pr.ALGO_TWO_SHOT_PULL, channels=ch, threads=threads))
    bufs = [torch.randn(L, device="cuda") for _ in range(P)]
    n = [1 + r for r in range(P)]
    for _ in range(3): pr.weighted_allreduce_local(comms, bufs, n)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(k): pr.weighted_allreduce_local(comms, bufs, n)
    e1.record(); torch.cuda.synchronize()
    us = e0.elapsed_time(e1) / k * 1e3
    for c in comms: c.destroy()
    return us
for P, L, chs in ((8, 11_689_512, (8, 16, 18, 24, 32, 37)), (4, 138_357_544, (16, 32, 37, 48, 64)), (2, 138_357_544, (32, 64, 74, 96))):
    for ch in chs:
        for th in (256, 512):
            us = t(P, L, ch, th, 10 if L < 5e7 else 4)
            print(json.dumps({"P": P, "L": L, "channels": ch, "threads": th, "us": round(us, 1),
                              "hbm_frac": round(2 * P * L * 4 / (us * 1e-6) / 6.551e12, 3)}), flush=True)
PY
cat gpurun_out/pull_ch.jsonl; tail -n 3 gpurun_out/pull_ch.err
