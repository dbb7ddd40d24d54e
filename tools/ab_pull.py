"""K3 A/B: the TMA ring vs the push two-shot vs the pull two-shot (PR_ALGO_TWO_SHOT_PULL), co-located ranks.

    python tools/ab_pull.py [--quick]

Two regimes:
  * per channel — few channels per rank, HBM far from saturated: each channel CTA's own data path is
    the limit, as on a real multi-GPU run where a rank has only its `channels` CTAs.  Reported as the
    per-rank bus-bandwidth equivalent Z·2(P−1)/P / t and per channel;
  * co-located full size — the ResNet-18 gradient at P = 8 and the VGG-16 gradient at P = 4 with the
    default channel count: an HBM proxy (all ranks' traffic in one GPU's HBM).
Every pull result is compared bit for bit with the ring's on the same inputs (`same_bits_as_ring`).
Device time: CUDA events over 3 back-to-back calls after 2 warm-up calls, median of 3 repetitions.
"""

import argparse
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import paper_2111_08272_b200 as pr  # noqa: E402

ALGOS = {"ring": pr.ALGO_RING, "twoshot_push": pr.ALGO_TWO_SHOT, "twoshot_pull": pr.ALGO_TWO_SHOT_PULL,
         "twoshot_pull_tma": pr.ALGO_TWO_SHOT_PULL}


def time_case(P, L, channels, algo, sys_scope=False, check=None):
    g = torch.Generator(device="cuda").manual_seed(P * 1000 + L % 997)
    src = [torch.randn(L, device="cuda", generator=g) for _ in range(P)]
    bufs = [s.clone() for s in src]
    n = [1 + r for r in range(P)]
    comms = pr.comm_init_local(P, 0, pr.comm_config(channels=channels, algo=ALGOS[algo], sys_scope=sys_scope,
                                                    watchdog_ns=20_000_000_000, pull_tma=algo.endswith("_tma")))
    try:
        pr.weighted_allreduce_local(comms, bufs, n)
        torch.cuda.synchronize()
        result = bufs[0].clone()
        for _ in range(2):
            pr.weighted_allreduce_local(comms, bufs, n)
        torch.cuda.synchronize()
        reps = []
        for _ in range(3):
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record()
            for _ in range(3):
                pr.weighted_allreduce_local(comms, bufs, n)
            e1.record()
            torch.cuda.synchronize()
            reps.append(e0.elapsed_time(e1) / 3 * 1e3)
        assert all(c.status() == 0 for c in comms)
    finally:
        for c in comms:
            c.destroy()
    us = sorted(reps)[1]
    return us, result


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--quick", action="store_true")
    a = ap.parse_args()
    # per-channel regime
    for P, mib in ((2, 256), (4, 128), (8, 64)):
        L = (mib << 20) // 4
        for ch in ((4, 8) if a.quick else (2, 4, 8, 16)):
            ring_out = None
            for name in ALGOS:
                us, out = time_case(P, L, ch, name)
                if name == "ring":
                    ring_out = out
                bus = L * 4 * 2 * (P - 1) / P / (us * 1e-6) / 1e9
                row = {"regime": "per_channel", "P": P, "MiB": mib, "channels": ch, "algo": name, "us": round(us, 1),
                       "busbw_equiv_GBs": round(bus, 1), "per_channel_GBs": round(bus / ch, 1)}
                if name != "ring":
                    row["same_bits_as_ring"] = bool(torch.equal(out, ring_out))
                print(json.dumps(row), flush=True)
    # co-located full size (HBM proxy), default channels
    for P, L, model in ((8, 11_689_512, "resnet18"), (4, 138_357_544, "vgg16"), (2, 138_357_544, "vgg16")):
        ring_out = None
        for name in ALGOS:
            us, out = time_case(P, L, 0, name)
            if name == "ring":
                ring_out = out
            bus = L * 4 * 2 * (P - 1) / P / (us * 1e-6) / 1e9
            row = {"regime": "colocated_full", "P": P, "model": model, "bytes_per_rank": L * 4, "algo": name,
                   "us": round(us, 1), "busbw_equiv_GBs": round(bus, 1)}
            if name != "ring":
                row["same_bits_as_ring"] = bool(torch.equal(out, ring_out))
            print(json.dumps(row), flush=True)


if __name__ == "__main__":
    main()
