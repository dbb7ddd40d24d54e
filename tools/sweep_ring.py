"""Sweep K3 configurations with all ranks co-located on one GPU (HBM-bound proxy).

    python tools/sweep_ring.py [P] [L]
Prints one line per config: channels slots slot_KB threads stages tile_KB -> us, algorithmic GB/s.
"""

import itertools
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import paper_2111_08272_b200 as pr  # noqa: E402

P = int(sys.argv[1]) if len(sys.argv) > 1 else 8
L = int(sys.argv[2]) if len(sys.argv) > 2 else 11_689_512
bufs = [torch.randn(L, device="cuda") for _ in range(P)]
n = [64, 64, 64, 64, 128, 128, 256, 256][:P] if P <= 8 else [64] * P
byts = (6 + 5 * (P - 2)) * L * 4 if P > 1 else 0


def run(cfg, reps=10):
    try:
        comms = pr.comm_init_local(P, 0, pr.comm_config(**cfg))
    except pr.PropringError as e:
        return None, str(e)
    try:
        for _ in range(3):
            pr.weighted_allreduce_local(comms, bufs, n)
        torch.cuda.synchronize()
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record()
        for _ in range(reps):
            pr.weighted_allreduce_local(comms, bufs, n)
        b.record()
        torch.cuda.synchronize()
        return a.elapsed_time(b) / reps * 1e3, ""
    except pr.PropringError as e:
        return None, str(e)
    finally:
        for c in comms:
            c.destroy()


grid = {
    "channels": [16, 32],
    "slots": [4, 8],
    "slot_bytes": [131072, 262144, 524288],
    "threads": [256, 512],
    "stages": [4, 6],
    "tile_bytes": [8192, 16384],
}
keys = list(grid)
best = None
for vals in itertools.product(*[grid[k] for k in keys]):
    cfg = dict(zip(keys, vals))
    if cfg["stages"] * 2 * cfg["tile_bytes"] > 200 * 1024:
        continue
    us, err = run(cfg)
    if us is None:
        print(cfg, "ERR", err, flush=True)
        continue
    gbs = byts / us / 1e3
    print(" ".join(f"{k}={v}" for k, v in cfg.items()), f"-> {us:.1f} us {gbs:.0f} GB/s", flush=True)
    if best is None or us < best[0]:
        best = (us, cfg)
print("BEST", best)
