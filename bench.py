#!/usr/bin/env python
"""Benchmark of the proportional-allocation + weighted-ring-allreduce training path (arXiv 2111.08272).

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference]
    python -m torch.distributed.run --nproc-per-node N --master-addr 127.0.0.1 ... bench.py --gpus N ...

A "step" is ONE EPOCH of Algorithm 1 — the unit at which the paper re-allocates and the
unit of the metric "epoch time at 1/2/4/8 B200" (BASELINE.json) — and it runs every row of
SURVEY §8(a): controller update + allgather of t_s (a10, a5), per-epoch shard (a2, K1), then S
aggregation steps of gather (a3, K2) -> ResNet-18 forward/backward with gradient accumulation (a4)
-> weighted ring allreduce of the 11,689,512-element fp32 gradient (a6-a8, K3; identity at N=1) ->
SGD (a9).  Workload: CIFAR-10-shaped synthetic data 50,000×3×32×32 u8 resident in HBM (153.6 MB >
L2 126 MB, so every epoch streams it from HBM), global batch B = 1024 (g = 16, C = 64) split by the
allocation at N = 1; across N weak scaling by default (1,024 samples per GPU per aggregation, C = 64·N,
the epoch shrinks to 50,000 // (1,024·N) aggregations), --strong keeps B = 1,024 for every N.

value   = whole-job samples/s over the K timed epochs (device time, CUDA events, max over ranks)
e2e     = the same with the data set in pinned HOST memory: the gather reads every sampled row over
          PCIe inside the timed region, and every step's loss is read back to the host
roofline= the library's dominant kernel in the timed region (by total live time: the fused SGD update
          at N=1 — 48 launches per epoch — K3 at N>1; K2 and the others are reported beside it), achieved
          algorithmic bytes / live CUDA-event duration vs the measured peak
cpu_baseline / --impl reference: the CPU oracle (oracle/) + a torch-CPU forward/backward on a bounded
          sample of one aggregation step, on the host cores.
"""

from __future__ import annotations

import argparse
import json
import os
import statistics
import subprocess
import sys
import threading
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

METRIC = "epoch throughput (samples/s; epoch time = S·B/value) of the proportional-allocation + weighted-ring-allreduce training step"
N_DATA, G_UNIT, C_UNITS = 50_000, 16, 64
STRONG = "--strong" in sys.argv          # the oracle legs follow the same batch rule as the timed arm
ROW_BYTES = 3 * 32 * 32
L_RESNET18 = 11_689_512
NVLINK_PEER_GBS = 770.0      # B200_PROFILING.md: measured peer copy per direction (900 nominal)


def parse():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=5)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--e2e-epochs", type=int, default=2)
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--overlap", action="store_true",
                    help="N1: bucketed weighted allreduce overlapped with backward (N > 1)")
    ap.add_argument("--bucket-mb", type=float, default=8.0)
    ap.add_argument("--no-colocated", action="store_true")
    ap.add_argument("--data-n", type=int, default=N_DATA,
                    help="data-set rows (default 50,000; smaller only for profiling runs: S = N // 1024)")
    ap.add_argument("--strong", action="store_true",
                    help="strong scaling: keep the global batch at 1,024 for every N (default: weak — 1,024 "
                         "samples per GPU per aggregation, global batch 1,024·N)")
    ap.add_argument("--kernel-shares", action="store_true",
                    help="also report each library kernel's share of the timed step (live CUDA events)")
    return ap.parse_args()


def peaks():
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as f:
            d = json.load(f)
        return float(d["hbm_gbs"]), "measured"
    except Exception:
        return 6650.0, "fallback"


# ---------------------------------------------------------------------------------------------------
class ClockSampler:
    """nvidia-smi clocks / throttle reasons sampled every 200 ms during the timed region."""

    Q = ("clocks.sm,clocks.max.sm,clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
         "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, device):
        self.device, self.proc, self.lines = device, None, []

    def start(self):
        if os.environ.get("PR_BENCH_NO_CLOCKS") == "1":    # diagnostics only: the contract wants the samples
            return
        try:
            self.proc = subprocess.Popen(["nvidia-smi", f"--query-gpu={self.Q}", "--format=csv,noheader,nounits",
                                          "-lms", "200", "-i", str(self.device)], stdout=subprocess.PIPE,
                                         stderr=subprocess.DEVNULL, text=True)
            self.t = threading.Thread(target=self._read, daemon=True)
            self.t.start()
        except Exception:
            self.proc = None

    def _read(self):
        for line in self.proc.stdout:
            self.lines.append(line.strip())

    def stop(self):
        if not self.proc:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvidia-smi unavailable"]}
        self.proc.terminate()
        try:
            self.proc.wait(5)
        except Exception:
            self.proc.kill()
        sm, mx, reasons = [], [], set()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        for ln in self.lines:
            p = [x.strip() for x in ln.split(",")]
            if len(p) < 6:
                continue
            try:
                sm.append(float(p[0]))
                mx.append(float(p[1]))
            except ValueError:
                continue
            for nm, v in zip(names, p[2:6]):
                if v.lower().startswith("active"):
                    reasons.add(nm)
        return {"sm_mhz": statistics.median(sm) if sm else None, "sm_max_mhz": max(mx) if mx else None,
                "reasons": sorted(reasons), "samples": len(sm)}


# ---------------------------------------------------------------------------------------------------
def run_ours(args):
    import torch
    import torch.distributed as dist

    import paper_2111_08272_b200 as pr
    from paper_2111_08272_b200.trainer import RunConfig, Worker

    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    assert world == args.gpus, f"--gpus {args.gpus} but WORLD_SIZE={world}"
    # PR_BENCH_SHARED_GPU=1: every rank on cuda:0 with a gloo group — a functional check of the N>1 path
    # on a one-GPU box (timings are then meaningless: the ranks time-share one GPU)
    shared = os.environ.get("PR_BENCH_SHARED_GPU") == "1"
    if shared:
        local = 0
    torch.cuda.set_device(local)
    tdev = "cpu" if shared else "cuda"
    if world > 1:
        if shared:
            dist.init_process_group("gloo")
        else:
            dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    # AUTO: the 46.76 MB step buffer takes the ring (with K7 fused); N1's buckets take the two-shot at P >= 8
    comm = pr.comm_init(rank, world, local, config=pr.comm_config(algo=pr.ALGO_AUTO)) if world > 1 else None
    units = units_for(world, args.strong)
    cfg = RunConfig(N=args.data_n, ratios=[1] * world, C=units, g=G_UNIT, adaptive=True, micro=1024,
                    overlap=args.overlap, bucket_mb=args.bucket_mb)
    wk = Worker(cfg, rank, world, local, comm)

    def barrier():
        if world > 1:
            dist.barrier()

    def epoch(record=False, loss_to_host=False, w=wk):
        w.boundary()                             # a10 + t_s exchange (Algorithm 1 steps 1-3)
        return w.run_epoch(record=record, loss_to_host=loss_to_host)

    for _ in range(args.warmup):
        epoch()
    torch.cuda.synchronize()
    barrier()
    wk.launches = 0
    wk.gather_events.clear()
    wk.ar_events.clear()
    wk.sgd_events.clear()
    clocks = ClockSampler(local)
    clocks.start()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    torch.cuda.synchronize()
    e0.record()
    samples = 0
    recs = []
    marks, host_ms = [], []
    for _ in range(args.steps):
        rec = epoch(record=True)
        marks.append(torch.cuda.Event(enable_timing=True))
        marks[-1].record()
        host_ms.append(round(wk.host_enqueue_s * 1e3, 2))
        recs.append(rec)
        samples += rec["S"] * wk.alloc.view()["B"]
    e1.record()
    torch.cuda.synchronize()
    barrier()
    clk = clocks.stop()
    ms = e0.elapsed_time(e1)
    if world > 1:
        t = torch.tensor([ms], device=tdev)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        ms = float(t)
    launches = wk.launches
    ms_epoch = ms / args.steps
    value = samples / (ms / 1e3)

    # ---- roofline of the library's dominant kernel (live CUDA events in the timed region) ----------
    hbm, peak_kind = peaks()
    g_ms = [a.elapsed_time(b) for a, b, _ in wk.gather_events]
    g_rows = [n for _, _, n in wk.gather_events]
    g_bytes = statistics.mean(g_rows) * (ROW_BYTES + 2 * ROW_BYTES + 8 + 8 + 8)
    g_avg = statistics.mean(g_ms) if g_ms else float("nan")
    gather_roof = {"kernel": "gather_kernel<U8_TO_BF16_AFFINE> channels-last (K2, LSU, one launch per epoch)",
                   "bound": "hbm",
                   "achieved": g_bytes / (g_avg * 1e-3) / 1e9, "peak": hbm, "unit": "GB/s",
                   "peak_kind": peak_kind, "launches": len(g_ms), "avg_us": g_avg * 1e3,
                   "bytes_per_launch": g_bytes, "total_ms": sum(g_ms)}
    gather_roof["frac"] = gather_roof["achieved"] / hbm
    mix = mix_ceiling()
    if mix:
        gather_roof["mix_ceiling"] = {"gbs": mix, "frac": gather_roof["achieved"] / mix,
                                      "source": "tools/probes/widen_probe.cu: sequential stream with K2's 1:2 "
                                                "read:write byte mix (profiles/round1_k2_mix_ceiling.txt)"}
    gather_roof["traffic"] = traffic_from_profiles("gather")
    roof = gather_roof
    sgd_roof = None
    if wk.sgd_events:
        u_ms = [a.elapsed_time(b) for a, b in wk.sgd_events]
        u_avg = statistics.mean(u_ms)
        u_bytes = 16.0 * wk.L                      # read θ, ḡ; write θ, ḡ = 0 (fp32)
        sgd_roof = {"kernel": "sgd_kernel (a9: SGD + gradient reset, one launch per aggregation step)",
                    "bound": "hbm", "achieved": u_bytes / (u_avg * 1e-3) / 1e9, "peak": hbm, "unit": "GB/s",
                    "peak_kind": peak_kind, "launches": len(u_ms), "avg_us": u_avg * 1e3,
                    "bytes_per_launch": u_bytes, "total_ms": sum(u_ms), "traffic": traffic_from_profiles("sgd")}
        sgd_roof["frac"] = sgd_roof["achieved"] / hbm
        if sgd_roof["total_ms"] > roof["total_ms"]:
            roof = sgd_roof
    allreduce = None
    if world > 1 and wk.ar_events:
        a_ms = [a.elapsed_time(b) for a, b in wk.ar_events]
        a_avg = statistics.mean(a_ms)
        Z = wk.L * 4
        bus = Z * 2 * (world - 1) / world / (a_avg * 1e-3) / 1e9
        kname = ("ring_kernel<float> (K3 with K7 fused: weighted allreduce + SGD + gradient reset)"
                 if getattr(wk, "pflat", None) is not None and not wk._overlap else "ring_kernel<float> (K3)")
        allreduce = {"kernel": kname, "bound": "nvlink", "achieved": bus, "peak": NVLINK_PEER_GBS,
                     "unit": "GB/s", "peak_kind": "B200_PROFILING.md measured peer copy per direction",
                     "frac": bus / NVLINK_PEER_GBS, "avg_us": a_avg * 1e3, "bytes": Z, "launches": len(a_ms),
                     "frac_of_900_nominal": bus / 900.0, "total_ms": sum(a_ms), "traffic": None}
        if allreduce["total_ms"] > roof["total_ms"]:
            roof = allreduce
        if not shared:
            allreduce["nccl_baseline"] = nccl_baseline(wk, world, rank)

    # ---- e2e: host-resident data set, per-step loss read back --------------------------------------
    e2e = None
    if args.e2e_epochs > 0:
        cfg_h = RunConfig(N=args.data_n, ratios=[1] * world, C=units, g=G_UNIT, adaptive=True, micro=1024,
                          host_data=True, overlap=args.overlap, bucket_mb=args.bucket_mb)
        wk_h = Worker(cfg_h, rank, world, local, comm, data=wk.X.cpu(), labels=wk.Y.cpu())
        wk_h.model.load_state_dict(wk.model.state_dict())
        for _ in range(3):                                 # warm-up: the allocation freezes, after
            epoch(w=wk_h)                                  # which every epoch prefetches the next one's rows
        torch.cuda.synchronize()
        barrier()
        h0, h1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        h0.record()
        hs = 0
        for _ in range(args.e2e_epochs):
            r = epoch(w=wk_h, loss_to_host=True)
            hs += r["S"] * wk_h.alloc.view()["B"]
        h1.record()
        torch.cuda.synchronize()
        barrier()
        hms = h0.elapsed_time(h1)
        if world > 1:
            t = torch.tensor([hms], device=tdev)
            dist.all_reduce(t, op=dist.ReduceOp.MAX)
            hms = float(t)
        v = wk_h.alloc.view()
        e2e = {"value": hs / (hms / 1e3), "unit": "samples/s",
               "h2d_bytes_per_step": v["S"] * v["n"][rank] * (ROW_BYTES + 8),
               "d2h_bytes_per_step": v["S"] * 4,
               "note": "data set in pinned host memory; rows gathered over PCIe by K2 inside the timed region; "
                       "every step's loss copied to pinned host memory and read by the host one step late (no per-step GPU idle)"}

    # ---- co-located ring (1 GPU): all P ranks of K3 on this GPU, HBM-bound proxy of the NVLink path --
    colocated = None
    if world == 1 and not args.no_colocated:
        colocated = colocated_allreduce(hbm, peak_kind)

    if rank == 0:
        cpu = None if args.no_cpu_baseline else cpu_baseline(world)
        out = {
            "metric": METRIC, "value": value, "unit": "samples/s", "n_gpus": world, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": ms_epoch, "higher_is_better": True,
            "scaling": "strong" if args.strong else "weak",
            "vs_baseline": None, "dtype": "f32", "data": "synthetic",
            "config": bench_config(world, bool(args.overlap and world > 1), args.strong),
            "epoch_time_s": ms_epoch / 1e3,
            "epoch_ms_each": [round(a.elapsed_time(b), 2) for a, b in zip([e0] + marks[:-1], marks)],
            "host_enqueue_ms_each": host_ms,
            "roofline": {k: roof[k] for k in ("bound", "achieved", "peak", "unit", "frac", "traffic")},
            "roofline_detail": roof,
            "gather": gather_roof,
            "sgd": sgd_roof,
            "allreduce": allreduce,
            "allreduce_colocated": colocated,
            "e2e": e2e,
            "gpu_launches": launches,
            "clocks": clk,
            "cpu_baseline": cpu,
            "alloc_w": wk.alloc.view()["w"],
            "loss_last_epoch": recs[-1]["loss"],
            # share of the timed region spent in each library kernel (live events; compare with the ncu
            # launch list of the same command in profiles/)
            "kernel_shares": {"gather_kernel": gather_roof["total_ms"] / ms,
                              "sgd_kernel": (sgd_roof["total_ms"] / ms) if sgd_roof else 0.0,
                              "ring_kernel": (allreduce["total_ms"] / ms) if allreduce else 0.0},
        }
        if args.data_n != N_DATA:
            out["config"]["workload"] += f" [PROFILING VARIANT: N={args.data_n}]"
        print(json.dumps(out))
    if comm is not None:
        comm.destroy()
    if world > 1:
        dist.destroy_process_group()


def mix_ceiling():
    """Best GB/s of the sequential 1:2 read:write streaming probe (context for K2's roofline)."""
    try:
        import re
        with open(os.path.join(ROOT, "profiles", "round1_k2_mix_ceiling.txt")) as f:
            v = [float(m.group(1)) for m in re.finditer(r"widen .*?([0-9.]+) GB/s", f.read())]
        return max(v) if v else None
    except OSError:
        return None


def units_for(world, strong=False):
    """Allocation units C per aggregation: 64 units of g = 16 samples per GPU (weak scaling: 1,024 samples
    per GPU per step at equal speeds), or 64 in total (strong: the global batch stays 1,024)."""
    return C_UNITS if strong else C_UNITS * world


def bench_config(world, overlap=False, strong=False):
    """The workload both arms name (our arm and --impl reference print the same config)."""
    C = units_for(world, strong)
    B = G_UNIT * C
    return {"workload": f"resnet18-cifar10-shaped-50k, global batch {B} (g={G_UNIT}, C={C}), equal start, "
                        "self-adaptive allocation, fp32 gradients (11,689,512), bf16 autocast compute",
            "model": "resnet18 (1000-class head, random init)", "global_batch": B,
            "seq_len": None, "parallelism": f"dp{world}", "step": f"one epoch (S={N_DATA // B} aggregations)",
            "overlap": overlap, "l2": "inputs larger than L2 (153.6 MB data set streamed every epoch)"}


def nccl_baseline(wk, world, rank, reps=20):
    """K5: the same weighted average through NCCL on the same buffer — premul-sum
    (ncclRedOpCreatePreMulSum via torch) and scale + SUM — against K3, all timed back to back."""
    import torch
    import torch.distributed as dist

    import paper_2111_08272_b200 as pr

    n_r = wk.alloc.view()["n"][rank]
    sumn = wk.alloc.view()["B"]
    s = n_r / sumn
    buf = wk.flat
    Z = buf.numel() * 4

    def timed(fn):
        for _ in range(5):
            fn()
        torch.cuda.synchronize()
        dist.barrier()
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record()
        for _ in range(reps):
            fn()
        b.record()
        torch.cuda.synchronize()
        t = torch.tensor([a.elapsed_time(b) / reps], device="cuda")
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        us = float(t) * 1e3
        return {"us": us, "busbw_GBs": Z * 2 * (world - 1) / world / (us * 1e-6) / 1e9}

    out = {"propring_K3": timed(lambda: pr.weighted_allreduce(wk.comm, buf, n_r))}
    if getattr(wk, "pflat", None) is not None:
        # rows a6-a9 fused (K7 in K3); lr = 0 leaves the parameters bit-identical (θ + (−0)·d = θ)
        out["propring_K3_K7_fused"] = timed(lambda: pr.weighted_allreduce_sgd(wk.comm, buf, wk.pflat, n_r, 0.0, 0.0,
                                                                              zero_grad=False))
    try:
        op = dist._make_nccl_premul_sum(s)
        out["nccl_premul_sum"] = timed(lambda: dist.all_reduce(buf, op=op))
    except Exception as e:   # noqa: BLE001
        out["nccl_premul_sum"] = {"error": repr(e)[:200]}

    def scale_sum():
        buf.mul_(s)
        dist.all_reduce(buf)

    out["nccl_scale_then_sum"] = timed(scale_sum)
    buf.zero_()
    return out


def traffic_from_profiles(kind):
    """dram bytes per launch from the committed ncu --set full capture (profiles/ncu_traffic.json)."""
    try:
        with open(os.path.join(ROOT, "profiles", "ncu_traffic.json")) as f:
            return json.load(f).get(kind, {}).get("dram_bytes_per_launch")
    except Exception:
        return None


def colocated_allreduce(hbm, peak_kind, P=8, reps=20):
    import torch

    import paper_2111_08272_b200 as pr

    comms = pr.comm_init_local(P, torch.cuda.current_device(), pr.comm_config())
    L = L_RESNET18
    bufs = [torch.randn(L, device="cuda") for _ in range(P)]
    n = [64, 64, 64, 64, 128, 128, 256, 256][:P]
    for _ in range(5):
        pr.weighted_allreduce_local(comms, bufs, n)
    torch.cuda.synchronize()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record()
    for _ in range(reps):
        pr.weighted_allreduce_local(comms, bufs, n)
    b.record()
    torch.cuda.synchronize()
    t = a.elapsed_time(b) / reps
    Z = L * 4
    # algorithmic HBM bytes of one call, all P ranks (direct all-gather): per rank
    # hop0 2·Z/P, P−2 middle hops 3·Z/P, last hop 4·Z/P, P−2 forwards 2·Z/P  => (6 + 5(P−2))·Z/P
    byts = P * (6 + 5 * (P - 2)) * Z / P
    # rows a6-a9 fused (K7 inside K3) vs composed (ring + K7 per rank), same setting
    store = [torch.randn(2 * L, device="cuda") for _ in range(P)]
    grads, thetas = [x[:L] for x in store], [x[L:] for x in store]

    def timed(fn):
        for _ in range(3):
            fn()
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        for _ in range(reps):
            fn()
        e1.record()
        torch.cuda.synchronize()
        return e0.elapsed_time(e1) / reps * 1e3

    def composed():
        pr.weighted_allreduce_local(comms, grads, n)
        for r in range(P):
            pr.sgd_update(thetas[r], grads[r], 1e-6, 0.0, zero_grad=True)

    fused_us = timed(lambda: pr.weighted_allreduce_sgd_local(comms, grads, thetas, n, 1e-6, 0.0, zero_grad=True))
    composed_us = timed(composed)
    for c in comms:
        c.destroy()
    # C1 (BASELINE configs[0]): the logistic-regression gradient (1,024 fp32 = 4 KiB), 2 ranks, n = [25, 75];
    # AUTO takes the one-shot LL path; 20 calls captured in one CUDA graph = device time per call
    c1 = pr.comm_init_local(2, torch.cuda.current_device(), pr.comm_config(algo=pr.ALGO_AUTO))
    g1 = [torch.randn(1024, device="cuda") for _ in range(2)]
    st = torch.cuda.Stream()
    with torch.cuda.stream(st):
        pr.weighted_allreduce_local(c1, g1, [25, 75], stream=st)
        torch.cuda.synchronize()
        gr = torch.cuda.CUDAGraph()
        with torch.cuda.graph(gr, stream=st):
            for _ in range(20):
                pr.weighted_allreduce_local(c1, g1, [25, 75], stream=st)
    gr.replay()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    gr.replay()
    e1.record()
    torch.cuda.synchronize()
    c1_us = e0.elapsed_time(e1) / 20 * 1e3
    del gr
    for c in c1:
        c.destroy()
    # per-rank CTA throughput with the cross-GPU configuration (32 channels, 1 MiB slots): 2 ranks on this
    # GPU leave HBM far from saturated, so this is what one rank's channels can push — the bound a real
    # NVLink run would face before the link's 770 GB/s (tools/sweep_cta.py)
    cx = pr.comm_init_local(2, torch.cuda.current_device(), pr.comm_config(channels=32, slot_bytes=1 << 20))
    Lx = (256 << 20) // 4
    gx = [torch.randn(Lx, device="cuda") for _ in range(2)]
    for _ in range(2):
        pr.weighted_allreduce_local(cx, gx, [1, 2])
    torch.cuda.synchronize()
    e0.record()
    for _ in range(5):
        pr.weighted_allreduce_local(cx, gx, [1, 2])
    e1.record()
    torch.cuda.synchronize()
    x_us = e0.elapsed_time(e1) / 5 * 1e3
    per_rank_bus = Lx * 4 * 2 * (2 - 1) / 2 / (x_us * 1e-6) / 1e9
    del gx
    for c in cx:
        c.destroy()
    return {"kernel": "ring_kernel<float> (K3), all ranks on one GPU", "P": P, "bytes_per_rank": Z,
            "fused_a6_a9_us": fused_us, "composed_a6_a9_us": composed_us,
            "c1_allreduce_4KiB_P2_us": c1_us,
            "cross_gpu_config_per_rank_busbw_equiv": {"GBs": per_rank_bus, "us": x_us, "bytes": Lx * 4, "P": 2,
                                                      "channels": 32, "vs_nvlink_770": per_rank_bus / NVLINK_PEER_GBS},
            "n_local": n, "avg_us": t * 1e3, "bound": "hbm", "achieved": byts / (t * 1e-3) / 1e9, "peak": hbm,
            "unit": "GB/s", "frac": byts / (t * 1e-3) / 1e9 / hbm, "peak_kind": peak_kind,
            "algorithmic_bytes_per_call": byts,
            "note": "P virtual ranks co-resident on one GPU exercise the same kernel and protocol; peer stores "
                    "land in local HBM, so this is an HBM roofline, not an NVLink number (the algorithmic bytes "
                    "count every staging round trip at HBM, part of which the 126 MB L2 serves: frac can exceed 1)"}


# ---------------------------------------------------------------------------------------------------
def oracle_step(P, sample_rows, X, Y, grads, model, rank=0, a=None, epoch=0):
    """One aggregation step of the CPU reference: oracle shard slice + gather + torch-CPU fwd/bwd on a
    bounded sample + oracle fp64 weighted average of P gradient buffers + controller update."""
    import numpy as np
    import torch
    import torch.nn.functional as F

    from oracle import allocation as OA
    from oracle import gather as OG
    from oracle import permutation as OP
    from oracle import wavg as OW

    if a is None:
        a = OA.alloc_init(N_DATA, [1] * P, C=units_for(P, STRONG), g=G_UNIT)
    n_r = a.n[rank]
    idx = OP.shard_indices(N_DATA, a.off[rank] + 0, min(a.len[rank], n_r), 1234, epoch)
    xb, yb = OG.gather_rows(X, idx[:sample_rows], OG.U8_TO_F32_AFFINE, scale=np.float32([1 / 51.5865, 1 / 50.847, 1 / 51.255]),
                            shift=np.float32([125.307, 122.961, 113.8575]), plane=1024, Y=Y)
    x = torch.from_numpy(xb).view(-1, 3, 32, 32)
    loss = F.cross_entropy(model(x), torch.from_numpy(yb))
    model.zero_grad()
    loss.backward()
    ref, _ = OW.weighted_average(grads, a.n)
    OA.alloc_update(a, [1.0] * P) if not a.frozen else None
    return float(loss.detach()), ref.shape[0]


def cpu_reference_setup(P):
    import numpy as np
    import torch

    import synth
    from paper_2111_08272_b200.trainer import build_model

    X = synth.images_u8(N_DATA, seed=0).reshape(N_DATA, -1)
    Y = synth.labels(N_DATA, 10, seed=1)
    grads = synth.gradients(max(P, 1), L_RESNET18, seed_base=1000).astype(np.float64)
    model = build_model("resnet18", 1000)
    return X, Y, grads, model, torch.get_num_threads()


def cpu_baseline(P, sample_rows=16, steps=2):
    X, Y, grads, model, cores = cpu_reference_setup(P)
    oracle_step(P, sample_rows, X, Y, grads, model)          # warm-up
    t0 = time.perf_counter()
    for s in range(steps):
        oracle_step(P, sample_rows, X, Y, grads, model, epoch=s)
    dt = (time.perf_counter() - t0) / steps
    return {"value": sample_rows / dt, "unit": "samples/s", "cores": cores, "kind": "oracle",
            "sample": f"{steps} aggregation steps, each: oracle shard slice + oracle gather of {sample_rows} rows + "
                      f"torch-CPU fp32 ResNet-18 fwd/bwd on those rows + oracle fp64 weighted average of "
                      f"{max(P, 1)}×{L_RESNET18} gradients + controller; samples/s = rows/step time"}


def run_reference(args):
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    if rank != 0:
        return
    X, Y, grads, model, cores = cpu_reference_setup(args.gpus)
    sample_rows = 16
    for w in range(args.warmup):
        oracle_step(args.gpus, sample_rows, X, Y, grads, model, epoch=w)
    t0 = time.perf_counter()
    for s in range(args.steps):
        oracle_step(args.gpus, sample_rows, X, Y, grads, model, epoch=s)
    dt = time.perf_counter() - t0
    value = args.steps * sample_rows / dt
    out = {"impl": "reference", "metric": METRIC, "value": value, "unit": "samples/s", "n_gpus": args.gpus,
           "steps": args.steps, "warmup": args.warmup, "ms_per_step": dt / args.steps * 1e3,
           "higher_is_better": True, "scaling": "strong" if args.strong else "weak", "vs_baseline": None,
           "dtype": "f64", "data": "synthetic",
           "config": bench_config(args.gpus, False, args.strong),
           "cpu_baseline": {"value": value, "unit": "samples/s", "cores": cores, "kind": "oracle",
                            "sample": f"bounded sample of the workload: each step = one aggregation step on "
                                      f"{sample_rows} rows (oracle shard + gather, torch-CPU fp32 ResNet-18 "
                                      f"fwd/bwd, oracle fp64 weighted average of P x 11,689,512 gradients, "
                                      f"controller); samples/s = rows / step time"},
           "e2e": {"value": value, "unit": "samples/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    print(json.dumps(out))


if __name__ == "__main__":
    a = parse()
    if a.impl == "reference":
        run_reference(a)
    else:
        run_ours(a)
