#!/usr/bin/env python
"""K3 small-buffer latency breakdown (co-located ranks on one GPU).

    python tools/ar_latency.py [--P 8] [--reps 50]

Per size/algorithm: mean event time per call and the rank-0 %globaltimer stamps of the last call
(entry -> handshake complete = t_w, handshake -> exit = t_c), so the fixed cost (launch + barrier) and the
per-phase cost of the ring can be told apart.  Buffers come from pr_comm_alloc (registered: direct
all-gather) unless --staged.
"""

import argparse
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import torch  # noqa: E402

import paper_2111_08272_b200 as pr  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--P", type=int, default=8)
    ap.add_argument("--reps", type=int, default=50)
    ap.add_argument("--staged", action="store_true")
    ap.add_argument("--sys", action="store_true")
    ap.add_argument("--graph", action="store_true", help="time the calls inside one captured CUDA graph")
    ap.add_argument("--sizes", default="16384,65536,262144,1048576,4194304,16777216")
    ap.add_argument("--algos", default="ring,two_shot,ll")
    ap.add_argument("--channels", type=int, default=16)
    ap.add_argument("--ll-max", type=int, default=16 << 20)
    ap.add_argument("--os-max", type=int, default=4 << 20)
    ap.add_argument("--slots", type=int, default=8)
    ap.add_argument("--slot-bytes", type=int, default=256 * 1024)
    a = ap.parse_args()
    P = a.P
    n = [64 * (1 + (r % 4)) for r in range(P)]
    sizes = [int(s) for s in a.sizes.split(",")]
    for algo_name in a.algos.split(","):
        algo = {"ring": pr.ALGO_RING, "two_shot": pr.ALGO_TWO_SHOT, "ll": pr.ALGO_LL, "oneshot": pr.ALGO_ONESHOT,
                "auto": pr.ALGO_AUTO, "pull": pr.ALGO_TWO_SHOT_PULL}[algo_name]
        comms = pr.comm_init_local(P, 0, pr.comm_config(algo=algo, sys_scope=a.sys, channels=a.channels,
                                                         ll_max_bytes=a.ll_max, os_max_bytes=a.os_max,
                                                         slots=a.slots,
                                                         slot_bytes=a.slot_bytes))
        zmax = max(sizes)
        if a.staged:
            raws = [torch.empty(zmax, dtype=torch.uint8, device="cuda") for _ in range(P)]
        else:
            raws = [c.alloc(zmax) for c in comms]
        for Z in sizes:
            bufs = [raws[r][:Z].view(torch.float32) for r in range(P)]
            for r in range(P):
                bufs[r].normal_()
            for _ in range(5):
                pr.weighted_allreduce_local(comms, bufs, n)
            torch.cuda.synchronize()
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            if a.graph:   # reps calls captured in one CUDA graph: device time per call, no host launch gaps
                st = torch.cuda.Stream()
                g = torch.cuda.CUDAGraph()
                with torch.cuda.stream(st):
                    with torch.cuda.graph(g, stream=st):
                        for _ in range(a.reps):
                            pr.weighted_allreduce_local(comms, bufs, n, stream=st)
                g.replay()
                torch.cuda.synchronize()
                e0.record()
                g.replay()
                e1.record()
            else:
                e0.record()
                for _ in range(a.reps):
                    pr.weighted_allreduce_local(comms, bufs, n)
                e1.record()
            torch.cuda.synchronize()
            us = e0.elapsed_time(e1) / a.reps * 1e3
            st = comms[0].timestamps()
            ok = all(c.status() == 0 for c in comms)
            print(json.dumps({"algo": algo_name, "P": P, "bytes": Z, "us": round(us, 2),
                              "t_w_us": (st[1] - st[0]) / 1e3, "t_c_us": (st[2] - st[1]) / 1e3,
                              "staged": a.staged, "sys": a.sys, "graph": a.graph, "channels": a.channels, "slots": a.slots,
                              "slot_bytes": a.slot_bytes, "ok": ok}), flush=True)
        del raws
        for c in comms:
            c.destroy()


if __name__ == "__main__":
    main()
