"""Per-CTA throughput of the K3 TMA ring: P = 2 ranks co-located with few channels, so HBM is far from
saturated and each channel CTA's own data path is the limit — the regime of a real multi-GPU run, where a
rank has only its `channels` CTAs (a co-located P = 8 run saturates HBM and hides it).

    python tools/sweep_cta.py [--sys] [--mib 256] [--channels 16]
Prints per config: per-rank bus-bandwidth equivalent Z·2(P−1)/P / t_c (GB/s) and GB/s per channel.
"""

import argparse
import itertools
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import paper_2111_08272_b200 as pr  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--sys", action="store_true")
    ap.add_argument("--mib", type=int, default=256)
    ap.add_argument("--channels", type=int, default=16)
    ap.add_argument("--P", type=int, default=2)
    ap.add_argument("--quick", action="store_true", help="four reference configurations only")
    ap.add_argument("--bulk", action="store_true", help="TMA bulk-store data path (PR_COMM_FLAG_BULK_STORE)")
    ap.add_argument("--cfg", default="", help="one configuration as JSON (overrides the grid)")
    a = ap.parse_args()
    P, L = a.P, (a.mib << 20) // 4
    store = [torch.randn(L, device="cuda") for _ in range(P)]
    n = [1 + r for r in range(P)]
    grid = {"stages": [2, 3, 4, 6, 8, 12], "tile_bytes": [4096, 8192, 16384, 32768],
            "slot_bytes": [262144, 1048576], "threads": [256, 512], "slots": [4, 8]}
    keys = list(grid)
    cfgs = [dict(zip(keys, vals)) for vals in itertools.product(*[grid[k] for k in keys])]
    if a.quick:
        cfgs = [dict(stages=6, tile_bytes=16384, slot_bytes=262144, threads=512, slots=8),
                dict(stages=3, tile_bytes=32768, slot_bytes=1048576, threads=512, slots=8),
                dict(stages=6, tile_bytes=16384, slot_bytes=1048576, threads=512, slots=8),
                dict(stages=12, tile_bytes=8192, slot_bytes=1048576, threads=512, slots=8)]
    if a.cfg:
        cfgs = [json.loads(a.cfg)]
    for cfg in cfgs:
        if cfg["stages"] * 2 * cfg["tile_bytes"] > 224 * 1024 or cfg["stages"] * cfg["tile_bytes"] < 32768:
            continue
        try:
            comms = pr.comm_init_local(P, 0, pr.comm_config(channels=a.channels, sys_scope=a.sys, bulk_store=a.bulk,
                                                            **cfg))
        except pr.PropringError as e:
            print(json.dumps({**cfg, "err": str(e)[:80]}), flush=True)
            continue
        for _ in range(2):
            pr.weighted_allreduce_local(comms, store, n)
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        for _ in range(3):
            pr.weighted_allreduce_local(comms, store, n)
        e1.record()
        torch.cuda.synchronize()
        us = e0.elapsed_time(e1) / 3 * 1e3
        bus = L * 4 * 2 * (P - 1) / P / (us * 1e-6) / 1e9
        print(json.dumps({**cfg, "P": P, "channels": a.channels, "sys": a.sys, "bulk": a.bulk, "us": round(us, 1),
                          "busbw_equiv_GBs": round(bus),
                          "per_channel_GBs": round(bus / a.channels, 1)}), flush=True)
        for c in comms:
            c.destroy()


if __name__ == "__main__":
    main()
