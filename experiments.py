#!/usr/bin/env python
"""Heterogeneous-cluster scenarios of BASELINE.json configs[1..3], one rank per GPU.

    python -m torch.distributed.run --nproc-per-node P --master-addr 127.0.0.1 experiments.py --scenario c4

Heterogeneity is emulated (the box is homogeneous): rank r is slowed by σ_r through a K4 spin of
(σ_r − 1)·c0·n_r ns per aggregation, c0 = its calibrated compute seconds per sample.
Each epoch rank 0 prints one JSON line: w (units), t_s per rank, t_w per rank (barrier wait,
from the allreduce time above the fastest rank's), epoch time T, and the Σspeed-balanced bound
T_ideal = S·(B/Σv + t_c) with v_r = S·n_r/t_s^r measured under the slowdown and t_c the measured
allreduce + update time per step.  The paper's claims being reproduced: the ratio
stabilises after 4-5 epochs and the epoch time falls 20-40% below equal allocation.

PR_BENCH_SHARED_GPU=1 runs every rank on cuda:0 (functional check on a one-GPU box; times meaningless).
"""

from __future__ import annotations

import argparse
import json
import os
import statistics
import sys

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

SCENARIOS = {
    # name: (model, N, shape, P, ratios, C, g, sigma, adaptive)
    "c2": ("resnet18", 50_000, (3, 32, 32), 2, [1, 2], 3, 128, [2.0, 1.0], False),
    "c2-equal": ("resnet18", 50_000, (3, 32, 32), 2, [1, 1], 2, 192, [2.0, 1.0], False),
    "c2-5x": ("resnet18", 50_000, (3, 32, 32), 2, [1, 1], 12, 32, [5.0, 1.0], True),
    "c3": ("vgg16", 51_200, (3, 224, 224), 4, [1, 1, 1, 1], 64, 16, [2.0, 2.0, 1.0, 1.0], True),
    "c4": ("resnet18", 50_000, (3, 32, 32), 8, [1] * 8, 64, 16, [4, 4, 4, 4, 2, 2, 1, 1], True),
    "c4-replace": ("resnet18", 50_000, (3, 32, 32), 8, [1] * 8, 64, 16, [1, 4, 4, 4, 2, 2, 1, 1], True),
    "c4-add-base": ("resnet18", 50_000, (3, 32, 32), 7, [1] * 7, 256, 4, [4, 4, 4, 2, 2, 1, 1], True),
    "c4-add": ("resnet18", 50_000, (3, 32, 32), 8, [1] * 8, 256, 4, [4, 4, 4, 2, 2, 1, 1, 4], True),
}


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--scenario", default="c2", choices=sorted(SCENARIOS))
    ap.add_argument("--epochs", type=int, default=8)
    ap.add_argument("--N", type=int, default=0, help="override the data set size (shorter epochs)")
    ap.add_argument("--static", action="store_true", help="disable the self-adaptive controller")
    args = ap.parse_args()

    import torch
    import torch.distributed as dist

    import paper_2111_08272_b200 as pr
    from paper_2111_08272_b200.trainer import RunConfig, Worker

    model, N, shape, P, ratios, C, g, sigma, adaptive = SCENARIOS[args.scenario]
    if args.N:
        N = args.N
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    assert world == P, f"scenario {args.scenario} needs {P} ranks, got WORLD_SIZE={world}"
    shared = os.environ.get("PR_BENCH_SHARED_GPU") == "1"
    if shared:
        local = 0
    torch.cuda.set_device(local)
    dist.init_process_group("gloo" if shared else "nccl", **({} if shared else {"device_id": torch.device("cuda", local)}))
    tdev = "cpu" if shared else "cuda"
    comm = pr.comm_init(rank, world, local)
    cfg = RunConfig(N=N, shape=shape, model=model, ratios=ratios, C=C, g=g, slowdown=sigma,
                    adaptive=adaptive and not args.static, micro=256 if model == "vgg16" else 1024)
    wk = Worker(cfg, rank, world, local, comm)
    wk.calibrate()
    c0 = torch.tensor([wk.c0_ns], dtype=torch.float64, device=tdev)
    dist.all_reduce(c0, op=dist.ReduceOp.MAX)          # one common per-sample cost => σ ratios are exact
    wk.c0_ns = float(c0)

    for e in range(args.epochs):
        changed = wk.boundary()
        dist.barrier()
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        wk.ar_events.clear()
        a.record()
        rec = wk.run_epoch(record=True)
        b.record()
        torch.cuda.synchronize()
        T = a.elapsed_time(b) / 1e3
        ar = sum(x.elapsed_time(y) for x, y in wk.ar_events) / 1e3
        row = torch.tensor([rec["t_s"], ar, T, float(rec["n_r"])], dtype=torch.float64, device=tdev)
        rows = [torch.zeros_like(row) for _ in range(world)]
        dist.all_gather(rows, row)
        if rank == 0:
            ts = [float(r[0]) for r in rows]
            ars = [float(r[1]) for r in rows]
            n = [float(r[3]) for r in rows]
            S = rec["S"]
            B = sum(n)
            v = [S * nr / t for nr, t in zip(n, ts)]                   # samples/s under the slowdown
            t_c = min(ars) / S + 0.0                                  # pure transfer: the fastest rank's AR
            Tmax = max(float(r[2]) for r in rows)
            bound = S * (B / sum(v) + t_c)
            print(json.dumps({"scenario": args.scenario, "epoch": e, "w": rec["w"], "changed": changed,
                              "frozen": wk.alloc.view()["frozen"], "t_s": ts,
                              "t_w": [x - min(ars) for x in ars], "T": Tmax, "bound": bound,
                              "T_over_bound": Tmax / bound, "loss": rec["loss"]}), flush=True)
    comm.destroy()
    dist.destroy_process_group()


if __name__ == "__main__":
    main()
