#!/usr/bin/env python
"""Heterogeneous-cluster scenarios of BASELINE.json configs[1..3], one rank per GPU.

    python -m torch.distributed.run --nproc-per-node P --master-addr 127.0.0.1 experiments.py --scenario c4

Heterogeneity is emulated (the box is homogeneous): rank r is slowed by σ_r through a K4 spin of
(σ_r − 1)·t1(n_r) per aggregation, t1(n_r) = its own measured step time for its n_r rows.
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
    # C2's batch (B = 384) in units of g = 16, so the controller can place it (equal start, self-adaptive)
    "c2-adapt": ("resnet18", 50_000, (3, 32, 32), 2, [1, 1], 24, 16, [2.0, 1.0], True),
    "c2-5x": ("resnet18", 50_000, (3, 32, 32), 2, [1, 1], 12, 32, [5.0, 1.0], True),
    "c3": ("vgg16", 51_200, (3, 224, 224), 4, [1, 1, 1, 1], 64, 16, [2.0, 2.0, 1.0, 1.0], True),
    "c4": ("resnet18", 50_000, (3, 32, 32), 8, [1] * 8, 64, 16, [4, 4, 4, 4, 2, 2, 1, 1], True),
    "c4-replace": ("resnet18", 50_000, (3, 32, 32), 8, [1] * 8, 64, 16, [1, 4, 4, 4, 2, 2, 1, 1], True),
    "c4-add-base": ("resnet18", 50_000, (3, 32, 32), 7, [1] * 7, 256, 4, [4, 4, 4, 2, 2, 1, 1], True),
    "c4-add": ("resnet18", 50_000, (3, 32, 32), 8, [1] * 8, 256, 4, [4, 4, 4, 2, 2, 1, 1, 4], True),
    # Large-batch variants: on a B200 a ResNet-18/CIFAR step costs ~1.3 ms + 1.5 us/row (tools/
    # model_scaling.py), so the paper's linear-speed model (t_s ∝ samples) holds only from ~2k
    # rows per rank; these keep every rank in that regime (the survey's batch sizes are kept above).
    "c2-lin": ("resnet18", 50_000, (3, 32, 32), 2, [1, 1], 24, 256, [2.0, 1.0], True),
    "c2-5x-lin": ("resnet18", 50_000, (3, 32, 32), 2, [1, 1], 24, 256, [5.0, 1.0], True),
    "c4-lin": ("resnet18", 50_000, (3, 32, 32), 8, [1] * 8, 64, 256, [4, 4, 4, 4, 2, 2, 1, 1], True),
    "c4-replace-lin": ("resnet18", 50_000, (3, 32, 32), 8, [1] * 8, 64, 256, [1, 4, 4, 4, 2, 2, 1, 1], True),
    # add-slow-worker pair in the same regime: 7 ranks (speeds 1:1:1:2:2:4:4), then an 8th speed-1 rank
    # joins (separate runs); C = 256, g = 64: B = 16,384, S = 12 (rounding excess 1.1% / 0%)
    "c4-add-base-lin": ("resnet18", 204_800, (3, 32, 32), 7, [1] * 7, 256, 64, [4, 4, 4, 2, 2, 1, 1], True),
    "c4-add-lin": ("resnet18", 204_800, (3, 32, 32), 8, [1] * 8, 256, 64, [4, 4, 4, 2, 2, 1, 1, 4], True),
    # N4: convergence invariance under static ratios (Fig. 6, caption P:291):
    # minibatch 100, total batch 1000 (C = 10), lr 1e-2, wd 1e-4, ratios 5:5, 6:4, 3:7, 7:3
    "n4-55": ("resnet18", 50_000, (3, 32, 32), 2, [5, 5], 10, 100, [1.0, 1.0], False),
    "n4-64": ("resnet18", 50_000, (3, 32, 32), 2, [6, 4], 10, 100, [1.0, 1.0], False),
    "n4-37": ("resnet18", 50_000, (3, 32, 32), 2, [3, 7], 10, 100, [1.0, 1.0], False),
    "n4-73": ("resnet18", 50_000, (3, 32, 32), 2, [7, 3], 10, 100, [1.0, 1.0], False),
    # N3: time-varying stragglers ("Load and network bandwidth during training will change",
    # P:98).  Two pairs of ranks swap a 3x slowdown every 150 aggregation steps (1.5 epochs of S = 100).
    "n3-swap": ("resnet18", 409_600, (3, 32, 32), 4, [1] * 4, 64, 64, [3, 3, 1, 1], True),
}

# σ schedules of the drift scenarios: [(global step, σ per rank), ...]
SCHEDULES = {
    "n3-swap": [(0, [3, 3, 1, 1]), (150, [1, 1, 3, 3]), (300, [3, 3, 1, 1]), (450, [1, 1, 3, 3])],
}


def make_policy(args):
    """Alloc.set_policy kwargs from the command line (None = the library defaults: Eq. 10, stop rule on)."""
    policy = {}
    if args.never_freeze or args.scenario in SCHEDULES:
        policy["never_freeze"] = True
    if args.ema < 1.0:
        policy["ema_alpha"] = args.ema
    if args.model == "affine":
        import paper_2111_08272_b200 as pr

        policy["model"] = pr.ALLOC_MODEL_AFFINE
    return policy or None


def step_cost(t1, n, sigma, spin, c0):
    """Step time (s) of a rank σ× slower that processes n rows, from its σ = 1 step time t1 = t1(n): "t1"
    emulation σ·t1(n); "sample" emulation t1(n) + (σ−1)·c0·n (DESIGN.md §3 #46)."""
    if n <= 0:
        return 0.0
    return sigma * t1 if spin == "t1" else t1 + (sigma - 1.0) * c0 * n


def minmax_alloc(cost, P, C, floor=1):
    """The best integer allocation for measured per-rank step costs: min over w (Σw = C, w_r >= floor) of
    max_r cost(r, w_r).  Costs need not be monotone in w (cuDNN picks a different algorithm per batch size,
    so a measured t1(n) table has dips): for a candidate T, rank r may take any u with cost(r, u) <= T, and
    a subset-sum DP over the ranks decides whether the units can total exactly C; a binary search over the
    sorted achievable step times finds the smallest feasible T.  Among the allocations meeting it, the DP
    keeps the one whose costs sum lowest.  Returns (T_step, w)."""
    table = [[cost(r, u) for u in range(floor, C + 1)] for r in range(P)]
    cands = sorted({t for row in table for t in row})

    def solve(T):
        # best[k] = (sum of costs, choice list) reaching k units with the ranks so far
        best = {0: (0.0, [])}
        for r in range(P):
            nxt = {}
            for k, (sc, ch) in best.items():
                for j, t in enumerate(table[r]):
                    u = floor + j
                    if t > T or k + u > C:
                        continue
                    cand = (sc + t, ch + [u])
                    if k + u not in nxt or cand[0] < nxt[k + u][0]:
                        nxt[k + u] = cand
            best = nxt
        return best.get(C)

    lo, hi = 0, len(cands) - 1
    if solve(cands[hi]) is None:
        raise ValueError("no feasible allocation")
    while lo < hi:
        mid = (lo + hi) // 2
        if solve(cands[mid]) is not None:
            hi = mid
        else:
            lo = mid + 1
    return cands[lo], solve(cands[lo])[1]


def affine_minmax(a, b, sigma, g, C, floor=1, spin="t1", c0=0.0):
    """minmax_alloc for the affine σ = 1 step cost t1(n) = a + b·n."""
    return minmax_alloc(lambda r, u: step_cost(a + b * g * u, g * u, sigma[r], spin, c0), len(sigma), C, floor)


def fit_affine(ns, ts):
    """Least-squares t1(n) = a + b·n over the measured (n, t1) points (b = 0 if only one n)."""
    if len(ns) == 1:
        return ts[0], 0.0
    mn, mt = sum(ns) / len(ns), sum(ts) / len(ts)
    b = sum((x - mn) * (y - mt) for x, y in zip(ns, ts)) / sum((x - mn) ** 2 for x in ns)
    return mt - b * mn, b


METRICS_HEADER = "scenario,epoch,rank,w,n,len,t_s_ns,t_w_ns,t_c_ns,T_ns,loss\n"


def write_metrics_rows(path, scenario, epoch, w, n, lens, t_s, t_w, t_c, T, loss):
    """SURVEY §5 per-(epoch, rank) metrics CSV: epoch,rank,w,n,len,t_s_ns,t_w_ns,t_c_ns,T_ns,loss (times summed
    over the epoch; t_w = barrier wait, t_c = the exchange itself, T = the epoch's wall time on the device)."""
    new = not os.path.exists(path) or os.path.getsize(path) == 0
    with open(path, "a") as f:
        if new:
            f.write(METRICS_HEADER)
        for r in range(len(w)):
            ln = "" if lens is None else str(int(lens[r]))
            f.write(f"{scenario},{epoch},{r},{int(w[r])},{int(n[r])},{ln},{t_s[r] * 1e9:.0f},{t_w[r] * 1e9:.0f},"
                    f"{t_c * 1e9:.0f},{T * 1e9:.0f},{loss:.6g}\n")


def run_virtual(args):
    """All P ranks of a scenario on ONE GPU, one after another (--virtual).

    Each aggregation step: for every rank r, its own rows (K1 shard, K2 gather) go through the shared
    model's forward/backward with rank r's emulated slowdown (K4), timed alone by CUDA events (t_{r,s},
    the rank's gradient-computing time); its local mean gradient is copied into buffer r; then K3
    reduces the P buffers (local group) and SGD updates the model once.  At each controller boundary
    (every epoch — Algorithm 1 — or every k steps with --adapt-every k, N3) the controller gets
    t_s^r = Σ_s t_{r,s} over the steps since the last boundary.  Because ranks run serially, the
    *emulated parallel* time is T = Σ_s max_r t_{r,s} + S·t_c (what P GPUs would take, each rank's
    compute measured alone on a full B200), compared with the bound Σ_s B/Σ_r v_{r,s} + S·t_c, where
    v_{r,s} = n_r/t_{r,s} is rank r's measured speed at step s (= S·(B/Σv + t_c) when speeds are constant).
    """
    import torch

    import paper_2111_08272_b200 as pr
    from paper_2111_08272_b200.trainer import RunConfig, Worker

    model, N, shape, P, ratios, C, g, sigma, adaptive = SCENARIOS[args.scenario]
    if args.N:
        N = args.N
    k = args.adapt_every
    policy = make_policy(args)
    cfg = RunConfig(N=N, shape=shape, model=model, ratios=ratios, C=C, g=g, slowdown=sigma,
                    adaptive=adaptive and not args.static, micro=args.micro or (256 if model == "vgg16" else 1024),
                    adapt_every=k, policy=policy, slowdown_schedule=SCHEDULES.get(args.scenario), spin=args.spin)
    w = Worker(cfg, 0, 1, 0, None)
    comms = pr.comm_init_local(P, 0, pr.comm_config())
    bufs = [torch.zeros(w.L, dtype=torch.float32, device="cuda") for _ in range(P)]
    idx = [torch.empty(N, dtype=torch.int64, device="cuda") for _ in range(P)]
    totals = {"T": 0.0, "bound": 0.0}
    last_T = last_bound = last_tc = None
    for e in range(args.epochs):
        S = w.alloc.view()["S"]
        seg = k if k > 0 else S
        rows, losses, ws = [], [], []
        for s0 in range(0, S, seg):
            v = w.alloc.view()
            n, ns = v["n"], min(seg, S - s0)
            ws.append(v["w"])
            if s0 == 0:
                lens0 = v["len"]
            xs, ys = [], []
            for r in range(P):                            # a2 + a3 for every rank
                if k > 0:
                    pr.shard_steps(w.alloc, r, e, cfg.seed, s0, ns, idx[r])
                else:
                    pr.shard_indices(w.alloc, r, e, cfg.seed, idx[r])
                x = torch.empty((max(1, ns * n[r]), w.row_elems), dtype=w.xdt, device="cuda")
                y = torch.empty(max(1, ns * n[r]), dtype=torch.int64, device="cuda")
                pr.gather_rows(w.X.data_ptr(), N, w.row_bytes, idx[r], ns * n[r], x, w.gop, w.Y, y)
                xs.append(x)
                ys.append(y)
            for r in range(P):                            # graphs + t1(n_r) outside the timed region
                w.rank = r
                w.prepare(n[r])
            ev = [[(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(ns)]
                  for _ in range(P)]
            ar = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(ns)]
            for j in range(ns):
                for r in range(P):
                    w.rank = r
                    ev[r][j][0].record()
                    if n[r] > 0:
                        losses.append(w.compute_graphed(xs[r][j * n[r]:], ys[r][j * n[r]:], n[r]))
                    ev[r][j][1].record()
                    bufs[r].copy_(w.flat)
                    w.flat.zero_()
                ar[j][0].record()
                pr.weighted_allreduce_local(comms, bufs, n)                              # K3
                w.flat.copy_(bufs[0])
                if w.pflat is not None:                   # a9: K7 (SGD + gradient reset)
                    pr.sgd_update(w.pflat, w.flat, cfg.lr, cfg.wd, zero_grad=True)
                else:
                    w.opt.step()
                    w.flat.zero_()
                ar[j][1].record()
                w.gstep += 1
            torch.cuda.synchronize()
            t = [[ev[r][j][0].elapsed_time(ev[r][j][1]) / 1e3 for j in range(ns)] for r in range(P)]
            t_c = [a.elapsed_time(b) / 1e3 for a, b in ar]
            rows.append((n, t, t_c))
            if cfg.adaptive:
                w.alloc.update([sum(x) for x in t])       # a10: Eq. 10 + rounding + stop rule
        # emulated parallel time and the speed-balanced bound over the epoch's steps
        T = sum(sum(max(t[r][j] for r in range(P)) + tc[j] for j in range(len(tc))) for _, t, tc in rows)
        bound = sum(sum(sum(n) / sum(n[r] / t[r][j] for r in range(P) if n[r] > 0) + tc[j] for j in range(len(tc)))
                    for n, t, tc in rows)
        ts = [sum(sum(t[r]) for _, t, _ in rows) for r in range(P)]
        totals["T"] += T
        totals["bound"] += bound
        last_T, last_bound, last_tc = T, bound, sum(sum(tc) for _, _, tc in rows) / S
        if args.metrics_csv:
            tw = [sum(sum(max(t[q][j] for q in range(P)) - t[r][j] for j in range(len(tc))) for _, t, tc in rows)
                  for r in range(P)]
            write_metrics_rows(args.metrics_csv, args.scenario, e, ws[0], [sum(nn_[r] for nn_, _, _ in rows[:1])
                                                                         for r in range(P)],
                               lens0, ts, tw, sum(sum(tc) for _, _, tc in rows), T,
                               float(torch.stack(losses).mean()) if losses else float("nan"))
        rec = {"scenario": args.scenario, "mode": "virtual", "adapt_every": k, "epoch": e, "w": ws[0],
               "w_end": w.alloc.view()["w"], "frozen": w.alloc.view()["frozen"], "t_s": ts,
               "T_emulated": T, "bound": bound, "T_over_bound": T / bound,
               "t_c": sum(sum(tc) for _, _, tc in rows) / S, "loss": float(torch.stack(losses).mean()) if losses else None}
        if k > 0:
            rec["w_segments"] = ws
        print(json.dumps(rec), flush=True)
        w.epoch += 1
    # the measured-cost bound: t1(n) captured and timed at EVERY row count a rank can get (n = g·w, floor <= w
    # <= C − (P−1)·floor); the best integer allocation under the same emulation (what any controller could
    # reach) is the min-max of the measured per-rank step costs — vs the linear Σspeed bound above, which
    # assumes t_s ∝ samples and is unattainable with a fixed per-step cost.  The affine fit
    # t1(n) ≈ a + b·n of the same table is reported beside it.
    v = w.alloc.view()
    wmax = C - (P - 1) * cfg.floor
    # --opt-stride k: time every k-th unit count (plus the ends and the final allocation's) and interpolate
    # linearly between them (VGG-16 captures cost seconds each); 1 = every unit count
    # (0 = automatic: every unit count, but every 8th for VGG-16, whose 61 graph captures at every row count
    # outgrew the shared CUDA-graph pool on one GPU)
    stride = args.opt_stride if args.opt_stride > 0 else (8 if model == "vgg16" else 1)
    meas = sorted(set(range(cfg.floor, wmax + 1, stride)) | {wmax} | set(v["w"]) - {0})
    t1m = {u: w.t1(g * u) for u in meas}
    t1tab = {}
    for u in range(cfg.floor, wmax + 1):
        if u in t1m:
            t1tab[u] = t1m[u]
        else:
            a_ = max(x for x in meas if x < u)
            b_ = min(x for x in meas if x > u)
            t1tab[u] = t1m[a_] + (t1m[b_] - t1m[a_]) * (u - a_) / (b_ - a_)
    pts = sorted((g * u, t) for u, t in t1m.items())
    a0, b0 = fit_affine([p_[0] for p_ in pts], [p_[1] for p_ in pts])
    c0s = w.c0_ns / 1e9
    t_step, w_opt = minmax_alloc(lambda r, u: step_cost(t1tab[u], g * u, sigma[r], args.spin, c0s) if u <= wmax
                                 else float("inf"), P, C, cfg.floor)
    tc_mean = last_tc if last_tc is not None else 0.0
    S = v["S"]
    bound_aff = S * (t_step + tc_mean)
    # the controller's own fixed point under the measured costs (the allocation it froze at), for context
    w_fin = v["w"]
    t_fin = max(step_cost(t1tab[u], g * u, sigma[r], args.spin, c0s) for r, u in enumerate(w_fin) if u > 0)
    print(json.dumps({"scenario": args.scenario, "mode": "virtual", "spin": args.spin, "adapt_every": k,
                      "static": args.static, "epochs": args.epochs, "T_total": totals["T"],
                      "bound_total": totals["bound"], "T_over_bound": totals["T"] / totals["bound"],
                      "t1_points": pts, "affine_fit": {"a_s": a0, "b_s_per_row": b0}, "c0_s_per_row": c0s,
                      "opt_w": w_opt, "opt_step_s": t_step, "opt_bound_epoch_s": bound_aff,
                      "final_w_model_step_s": t_fin, "last_epoch_T": last_T,
                      "last_epoch_T_over_opt_bound": (last_T / bound_aff) if last_T else None,
                      "last_epoch_T_over_linear_bound": (last_T / last_bound) if last_T else None,
                      "final_w": w_fin}), flush=True)
    for c in comms:
        c.destroy()


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--scenario", default="c2", choices=sorted(SCENARIOS))
    ap.add_argument("--epochs", type=int, default=8)
    ap.add_argument("--N", type=int, default=0, help="override the data set size (shorter epochs)")
    ap.add_argument("--static", action="store_true", help="disable the self-adaptive controller")
    ap.add_argument("--micro", type=int, default=0,
                    help="max rows per microbatch (default 1024 ResNet / 256 VGG); a rank whose n_r crosses a "
                         "multiple of it pays one more fixed per-microbatch cost")
    ap.add_argument("--virtual", action="store_true", help="all ranks on one GPU, serially (see run_virtual)")
    ap.add_argument("--adapt-every", type=int, default=0,
                    help="N3: controller every k aggregation steps over the step-interleaved shard (0 = per epoch)")
    ap.add_argument("--never-freeze", action="store_true", help="keep adapting after the ratio is stable")
    ap.add_argument("--ema", type=float, default=1.0, help="EMA weight on t_s (1 = raw, S:166)")
    ap.add_argument("--model", default="proportional", choices=["proportional", "affine"],
                    help="controller step-cost model: the paper's Eq. 10, or the affine extension (DESIGN §3 #49)")
    ap.add_argument("--metrics-csv", default="", help="append the per-(epoch, rank) metrics CSV (SURVEY §5) here")
    ap.add_argument("--opt-stride", type=int, default=0,
                    help="measured-cost bound: time t1 at every k-th unit count and interpolate (1 = all; "
                         "0 = all, every 8th for VGG-16)")
    ap.add_argument("--spin", default="t1", choices=["t1", "sample"],
                    help="K4 emulation: t1 = (σ−1)·t1(n_r) per step; sample = (σ−1)·c0·n_r (SURVEY §8(a) a4)")
    args = ap.parse_args()
    if args.virtual:
        return run_virtual(args)

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
    comm = pr.comm_init(rank, world, local, config=pr.comm_config(algo=pr.ALGO_AUTO))
    policy = make_policy(args)
    cfg = RunConfig(N=N, shape=shape, model=model, ratios=ratios, C=C, g=g, slowdown=sigma,
                    adaptive=adaptive and not args.static, micro=args.micro or (256 if model == "vgg16" else 1024),
                    adapt_every=args.adapt_every, policy=policy, slowdown_schedule=SCHEDULES.get(args.scenario),
                    spin=args.spin)
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
            if args.metrics_csv:
                lens = wk.alloc.view()["len"]                 # the shards of this epoch (updated at the next boundary)
                write_metrics_rows(args.metrics_csv, args.scenario, e, rec["w"], [int(x) for x in n],
                                   lens, ts, [x - min(ars) for x in ars], min(ars), Tmax, rec["loss"])
    comm.destroy()
    dist.destroy_process_group()


if __name__ == "__main__":
    main()
