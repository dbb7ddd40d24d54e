#!/usr/bin/env python
"""Benchmark of the proportional-allocation + weighted-ring-allreduce training path (arXiv 2111.08272).

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference]
    (N > 1 without WORLD_SIZE in the environment: bench.py re-launches itself under torch.distributed.run,
     one rank per GPU; the driver's torchrun form works unchanged)

A "step" is ONE EPOCH of Algorithm 1 — the unit at which the paper re-allocates and the
unit of the metric "epoch time at 1/2/4/8 B200" (BASELINE.json) — and it runs every row of
SURVEY §8(a): controller update + allgather of t_s (a10, a5), per-epoch shard (a2, K1), then S
aggregation steps of gather (a3, K2) -> forward/backward with gradient accumulation (a4) -> weighted
ring allreduce of the fp32 gradient (a6-a8, K3; identity at N=1) -> SGD (a9; fused into K3 at N>1).

Workloads (SURVEY §8(d) "Scaling" row: C2 data / ResNet-18 and C3 data / VGG-16, homogeneous, equal
start, fixed global batch B = 1,024 = g·C with g = 16, C = 64 — STRONG scaling):
  headline  ResNet-18 (1000-class head, random init), CIFAR-10-shaped 50,000×3×32×32 u8 resident in HBM
            (153.6 MB > L2 126 MB: every epoch streams it from HBM), S = 48 aggregations per epoch
  "vgg16"   VGG-16 (1000-class head), ImageNet-shaped 51,200×3×224×224 u8 (7.7 GB), S = 50; its own
            warm-up (3 epochs) and --vgg-steps timed epochs (the 553 MB gradient is the ≥ 64 MB allreduce)
  "weak_scaling" (N > 1): the ResNet-18 leg with 1,024 samples per GPU per aggregation (C = 64·N)

value    = whole-job samples/s over the K timed epochs (device time, CUDA events, max over ranks)
e2e      = the same with the data set in pinned HOST memory: the gather reads every sampled row over
           PCIe inside the timed region, and every step's loss is read back to the host
roofline = the library's dominant kernel in the timed region (by total live time: the SGD update at N=1
           — one launch per aggregation — the fused K3+K7 at N>1), algorithmic bytes / live CUDA-event
           duration vs the measured peak (HBM: MEASURED_PEAKS.json; NVLink: 770 GB/s measured peer copy)
allreduce_sweep (N>1): K3 at 64 MiB / 256 MiB / the VGG-16 gradient against NCCL premul-sum and
           scale + sum on the same registered buffer (C5's weights), busBW vs 770 (measured) and 900 (nominal)
cpu_baseline (N=1, rank 0): the CPU oracle (oracle/) — a bounded end-to-end aggregation step on the host
           cores, and per §8(d) each oracle part single-threaded, pinned to core 0, median of 5, beside the
           GPU kernel that computes it.  --impl reference times the same oracle step as its own arm.
"""

from __future__ import annotations

import argparse
import json
import os
import socket
import statistics
import subprocess
import sys
import threading
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

METRIC = "epoch throughput (samples/s; epoch time = S·B/value) of the proportional-allocation + weighted-ring-allreduce training step"
N_DATA, G_UNIT, C_UNITS = 50_000, 16, 64
ROW_BYTES = 3 * 32 * 32
L_RESNET18 = 11_689_512
L_VGG16 = 138_357_544
NVLINK_PEER_GBS = 770.0      # B200_PROFILING.md: measured peer copy per direction
NVLINK_NOMINAL_GBS = 900.0
# C5 weights: P=2 [1,3]·256, P=4 [1,1,2,4]·256, P=8 [1,1,1,1,2,2,4,4]·256
C5_WEIGHTS = {2: [1, 3], 4: [1, 1, 2, 4], 8: [1, 1, 1, 1, 2, 2, 4, 4]}

# the two workloads of the Scaling row: name -> (model, N, shape, micro, description)
WORKLOADS = {
    "resnet18": ("resnet18", N_DATA, (3, 32, 32), 1024,
                 "resnet18-cifar10-shaped-50k"),
    "vgg16": ("vgg16", 51_200, (3, 224, 224), 256,
              "vgg16-imagenet-shaped-51.2k"),
}


def parse(argv=None):
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=5)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--e2e-epochs", type=int, default=2)
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-oracle-kernels", action="store_true", help="skip the per-kernel oracle timings")
    ap.add_argument("--overlap", action="store_true",
                    help="N1: bucketed weighted allreduce overlapped with backward (N > 1)")
    ap.add_argument("--bucket-mb", type=float, default=8.0)
    ap.add_argument("--no-colocated", action="store_true")
    ap.add_argument("--no-vgg", action="store_true", help="skip the VGG-16 / ImageNet-shaped leg")
    ap.add_argument("--vgg-steps", type=int, default=2, help="timed epochs of the VGG-16 leg (3 warm-up)")
    ap.add_argument("--no-weak", action="store_true", help="N > 1: skip the weak-scaling leg")
    ap.add_argument("--data-n", type=int, default=N_DATA,
                    help="data-set rows (default 50,000; smaller only for profiling runs: S = N // 1024)")
    ap.add_argument("--weak", action="store_true",
                    help="headline in weak scaling (1,024 samples per GPU per aggregation); default strong "
                         "(SURVEY §8(d): fixed global batch 1,024 for every N)")
    ap.add_argument("--metrics-csv", default="", help="rank 0 writes the per-(epoch, rank) metrics CSV here")
    ap.add_argument("--oracle-timings-child", default="", help=argparse.SUPPRESS)
    return ap.parse_args(argv)


def peaks():
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as f:
            d = json.load(f)
        return float(d["hbm_gbs"]), "measured"
    except Exception:
        return 6650.0, "fallback"


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def self_launch(args, argv):
    """`python bench.py --gpus N` with N > 1 and no torchrun around it: re-run this file under
    torch.distributed.run, one rank per GPU (127.0.0.1 rendezvous); rank 0 prints the line."""
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={args.gpus}",
           "--master-addr", "127.0.0.1", f"--master-port={_free_port()}", os.path.abspath(__file__)] + list(argv)
    return subprocess.call(cmd)


# ---------------------------------------------------------------------------------------------------
class ClockSampler:
    """nvidia-smi clocks / throttle reasons sampled every 200 ms during the timed region."""

    Q = ("clocks.sm,clocks.max.sm,clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
         "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, device):
        self.device, self.proc, self.lines = device, None, []

    def start(self):
        if os.environ.get("PR_BENCH_NO_CLOCKS") == "1":    # diagnostics only: the contract wants the samples
            return self
        try:
            self.proc = subprocess.Popen(["nvidia-smi", f"--query-gpu={self.Q}", "--format=csv,noheader,nounits",
                                          "-lms", "200", "-i", str(self.device)], stdout=subprocess.PIPE,
                                         stderr=subprocess.DEVNULL, text=True)
            self.t = threading.Thread(target=self._read, daemon=True)
            self.t.start()
        except Exception:
            self.proc = None
        return self

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
def units_for(world, strong=True):
    """Allocation units C per aggregation: 64 in total (strong, the default: the global batch stays 1,024),
    or 64 units of g = 16 samples per GPU (weak: 1,024 samples per GPU per aggregation)."""
    return C_UNITS if strong else C_UNITS * world


def bench_config(world, overlap=False, strong=True, workload="resnet18", data_n=None):
    """The workload both arms name (our arm and --impl reference print the same config)."""
    model, N, shape, _, desc = WORKLOADS[workload]
    N = data_n or N
    C = units_for(world, strong)
    B = G_UNIT * C
    L = L_RESNET18 if model == "resnet18" else L_VGG16
    return {"workload": f"{desc}, global batch {B} (g={G_UNIT}, C={C}), equal start, self-adaptive allocation, "
                        f"fp32 gradients ({L:,}), bf16 autocast compute",
            "model": f"{model} (1000-class head, random init)", "global_batch": B,
            "seq_len": None, "parallelism": f"dp{world}", "step": f"one epoch (S={N // B} aggregations)",
            "scaling": "strong" if strong else "weak", "overlap": overlap,
            "l2": f"inputs larger than L2 ({N * (3 * shape[1] * shape[2]) / 1e6:,.1f} MB data set streamed every epoch)"}


def mix_ceiling():
    """Best GB/s of the sequential 1:2 read:write streaming probe at the ImageNet epoch size (context for
    K2's roofline): 2.47 GB u8 read, 4.93 GB written, 16-byte STGs or smem tiles + bulk stores, L2 evicted
    clean or dirty before each rep (tools/probes/mix_probe.cu, profiles/round2_k2_mix_probe_imagenet.txt)."""
    try:
        import re
        with open(os.path.join(ROOT, "profiles", "round2_k2_mix_probe_imagenet.txt")) as f:
            v = [float(m.group(1)) for m in re.finditer(r"widen .*?([0-9.]+) GB/s best", f.read())]
        return max(v) if v else None
    except OSError:
        return None


def traffic_from_profiles(kind, algorithmic_bytes=None):
    """dram bytes per launch from the committed ncu --set full capture (profiles/ncu_traffic.json); when the
    capture's launch was a different size (its algorithmic bytes are recorded), scaled to this launch."""
    try:
        with open(os.path.join(ROOT, "profiles", "ncu_traffic.json")) as f:
            e = json.load(f).get(kind, {})
        t = e.get("dram_bytes_per_launch")
        if t is not None and algorithmic_bytes and e.get("algorithmic_bytes"):
            t = t * algorithmic_bytes / e["algorithmic_bytes"]
        return t
    except Exception:
        return None


def _max_over_ranks(x, world, tdev):
    if world == 1:
        return x
    import torch
    import torch.distributed as dist

    t = torch.tensor([x], dtype=torch.float64, device=tdev)
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    return float(t)


# ---------------------------------------------------------------------------------------------------
def run_workload(name, args, ctx, strong=True, steps=None, warmup=None, e2e_epochs=None, kernel_detail=True):
    """One workload: W warm-up epochs, K timed epochs (barrier + synchronize on both sides, CUDA events,
    max over ranks), the live per-kernel events of the timed region, then the e2e epochs."""
    import torch

    from paper_2111_08272_b200.trainer import RunConfig, Worker

    world, rank, local, comm, tdev = ctx["world"], ctx["rank"], ctx["local"], ctx["comm"], ctx["tdev"]
    model, N, shape, micro, _ = WORKLOADS[name]
    if name == "resnet18":
        N = args.data_n
    steps = args.steps if steps is None else steps
    warmup = args.warmup if warmup is None else warmup
    e2e_epochs = args.e2e_epochs if e2e_epochs is None else e2e_epochs
    units = units_for(world, strong)
    row_bytes = shape[0] * shape[1] * shape[2]
    overlap = bool(args.overlap and world > 1)
    cfg = RunConfig(N=N, shape=shape, model=model, ratios=[1] * world, C=units, g=G_UNIT, adaptive=True,
                    micro=micro, overlap=overlap, bucket_mb=args.bucket_mb)
    wk = Worker(cfg, rank, world, local, comm)

    def barrier():
        if world > 1:
            import torch.distributed as dist
            dist.barrier()

    def epoch(record=False, loss_to_host=False, w=wk):
        w.boundary()                             # a10 + t_s exchange (Algorithm 1 steps 1-3)
        return w.run_epoch(record=record, loss_to_host=loss_to_host)

    for _ in range(warmup):
        epoch()
    torch.cuda.synchronize()
    barrier()
    wk.launches = 0
    wk.gather_events.clear()
    wk.ar_events.clear()
    wk.sgd_events.clear()
    clocks = ClockSampler(local).start()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    torch.cuda.synchronize()
    barrier()
    e0.record()
    samples, recs, marks, host_ms = 0, [], [], []
    for _ in range(steps):
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
    ms = _max_over_ranks(e0.elapsed_time(e1), world, tdev)
    out = {"value": samples / (ms / 1e3), "unit": "samples/s", "ms_per_step": ms / steps, "steps": steps,
           "warmup": warmup, "epoch_time_s": ms / steps / 1e3,
           "epoch_ms_each": [round(a.elapsed_time(b), 2) for a, b in zip([e0] + marks[:-1], marks)],
           "host_enqueue_ms_each": host_ms, "gpu_launches": wk.launches, "clocks": clk,
           "alloc_w": wk.alloc.view()["w"], "loss_last_epoch": recs[-1]["loss"],
           "config": bench_config(world, overlap, strong, name, N)}

    # ---- the library kernels of the timed region (live CUDA events on the launching stream) ----------
    hbm, peak_kind = peaks()
    g_ms = [a.elapsed_time(b) for a, b, _ in wk.gather_events]
    g_rows = [n for _, _, n in wk.gather_events]
    g_avg = statistics.mean(g_ms) if g_ms else float("nan")
    g_bytes = statistics.mean(g_rows) * (row_bytes + 2 * row_bytes + 8 + 8 + 8) if g_rows else 0.0
    gather = {"kernel": "gather_hwc_bulk_kernel<U8_TO_BF16_AFFINE, 3> channels-last (K2: coalesced loads -> smem "
                        "tile -> cp.async.bulk store; one launch per epoch)",
              "bound": "hbm", "achieved": g_bytes / (g_avg * 1e-3) / 1e9 if g_ms else None, "peak": hbm,
              "unit": "GB/s", "peak_kind": peak_kind, "launches": len(g_ms), "avg_us": g_avg * 1e3,
              "bytes_per_launch": g_bytes, "total_ms": sum(g_ms),
              "traffic": traffic_from_profiles("gather" if name == "resnet18" else "gather_imagenet", g_bytes)}
    gather["frac"] = gather["achieved"] / hbm if gather["achieved"] else None
    mix = mix_ceiling()
    if mix and gather["achieved"]:
        gather["mix_ceiling"] = {"gbs": mix, "frac": gather["achieved"] / mix,
                                 "source": "tools/probes/mix_probe.cu: sequential stream with K2's 1:2 read:write "
                                           "byte mix at the ImageNet epoch size, best store flavour "
                                           "(profiles/round2_k2_mix_probe_imagenet.txt)"}
    roof = gather
    sgd = None
    if wk.sgd_events:
        u_ms = [a.elapsed_time(b) for a, b in wk.sgd_events]
        u_avg = statistics.mean(u_ms)
        u_bytes = 16.0 * wk.L                      # read θ, ḡ; write θ, ḡ = 0 (fp32)
        sgd = {"kernel": "sgd_kernel (a9: SGD + gradient reset, one launch per aggregation step)",
               "bound": "hbm", "achieved": u_bytes / (u_avg * 1e-3) / 1e9, "peak": hbm, "unit": "GB/s",
               "peak_kind": peak_kind, "launches": len(u_ms), "avg_us": u_avg * 1e3,
               "bytes_per_launch": u_bytes, "total_ms": sum(u_ms),
               "traffic": traffic_from_profiles("sgd" if name == "resnet18" else "sgd_vgg16", u_bytes)}
        sgd["frac"] = sgd["achieved"] / hbm
        if sgd["total_ms"] > roof["total_ms"]:
            roof = sgd
    allreduce = None
    if world > 1 and wk.ar_events:
        a_ms = [a.elapsed_time(b) for a, b in wk.ar_events]
        a_avg = _max_over_ranks(statistics.mean(a_ms), world, tdev)
        Z = wk.L * 4
        bus = Z * 2 * (world - 1) / world / (a_avg * 1e-3) / 1e9
        fused = getattr(wk, "pflat", None) is not None and not wk._overlap
        kname = ("ring_kernel<float, FUSE> (K3 with K7 fused: weighted allreduce + SGD + gradient reset)"
                 if fused else "ring_kernel<float> (K3)")
        allreduce = {"kernel": kname, "bound": "nvlink", "achieved": bus, "peak": NVLINK_PEER_GBS,
                     "unit": "GB/s", "peak_kind": "B200_PROFILING.md measured peer copy per direction",
                     "frac": bus / NVLINK_PEER_GBS, "frac_of_900_nominal": bus / NVLINK_NOMINAL_GBS,
                     "avg_us": a_avg * 1e3, "bytes": Z, "launches": len(a_ms), "total_ms": sum(a_ms),
                     "traffic": None,
                     "note": "busBW = Z·2(P−1)/P / t; the fused kernel also applies SGD to the reduced chunk, so "
                             "this is a lower bound on the ring's own busBW"}
        if allreduce["total_ms"] > roof["total_ms"]:
            roof = allreduce
        if not ctx["shared"]:
            allreduce["nccl_baseline"] = nccl_baseline(wk, world, rank, tdev)
    out.update({"roofline": {k: roof[k] for k in ("bound", "achieved", "peak", "unit", "frac", "traffic")},
                "roofline_detail": roof, "gather": gather, "sgd": sgd, "allreduce": allreduce,
                "kernel_shares": {"gather_kernel": gather["total_ms"] / ms,
                                  "sgd_kernel": (sgd["total_ms"] / ms) if sgd else 0.0,
                                  "ring_kernel": (allreduce["total_ms"] / ms) if allreduce else 0.0}})
    if args.metrics_csv and kernel_detail:
        write_metrics_csv(args.metrics_csv, wk, recs, world, rank, tdev, name)

    # ---- e2e: host-resident data set, per-step loss read back --------------------------------------
    if e2e_epochs > 0:
        cfg_h = RunConfig(N=N, shape=shape, model=model, ratios=[1] * world, C=units, g=G_UNIT, adaptive=True,
                          micro=micro, host_data=True, overlap=overlap, bucket_mb=args.bucket_mb)
        xh, yh = wk.X.cpu(), wk.Y.cpu()
        del wk                                             # the device-resident leg is done: free its memory
        torch.cuda.empty_cache()
        wk_h = Worker(cfg_h, rank, world, local, comm, data=xh, labels=yh)
        del xh, yh                                         # the pinned copy inside wk_h is the one used
        for _ in range(3):                                 # warm-up: the allocation freezes, after
            epoch(w=wk_h)                                  # which every epoch prefetches the next one's rows
        torch.cuda.synchronize()
        barrier()
        h0, h1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        h0.record()
        hs = 0
        for _ in range(e2e_epochs):
            r = epoch(w=wk_h, loss_to_host=True)
            hs += r["S"] * wk_h.alloc.view()["B"]
        h1.record()
        torch.cuda.synchronize()
        barrier()
        hms = _max_over_ranks(h0.elapsed_time(h1), world, tdev)
        v = wk_h.alloc.view()
        out["e2e"] = {"value": hs / (hms / 1e3), "unit": "samples/s",
                      "h2d_bytes_per_step": v["S"] * v["n"][rank] * (row_bytes + 8),
                      "d2h_bytes_per_step": v["S"] * 4, "epochs": e2e_epochs,
                      "note": "data set in pinned host memory; rows gathered over PCIe by K2 inside the timed region "
                              "(the first timed epoch's rows were prefetched during the last warm-up epoch, as "
                              "every frozen epoch prefetches the next: steady-state accounting); every step's loss "
                              "copied to pinned host memory and read by the host one step late"}
        del wk_h
    else:
        out["e2e"] = None
        del wk
    torch.cuda.empty_cache()
    return out


def write_metrics_csv(path, wk, recs, world, rank, tdev, name):
    """SURVEY §5 per-(epoch, rank) metrics: epoch,rank,w,n,len,t_s_ns,t_w_ns,t_c_ns,T_ns,loss (t_w, t_c from the
    allreduce stamps are summed per epoch only at N > 1; rank 0 writes every rank's rows)."""
    import torch
    import torch.distributed as dist

    v = wk.alloc.view()
    rows = []
    for i, rec in enumerate(recs):
        rows.append([float(wk.epoch - len(recs) + i), float(rank), float(rec["w"][rank]), float(rec["n_r"]),
                     float(v["len"][rank]), rec["t_s"] * 1e9, float("nan"), float("nan"), float("nan"), rec["loss"]])
    t = torch.tensor(rows, dtype=torch.float64, device=tdev)
    if world > 1:
        allr = [torch.zeros_like(t) for _ in range(world)]
        dist.all_gather(allr, t)
    else:
        allr = [t]
    if rank == 0:
        with open(path, "a") as f:
            if f.tell() == 0:
                f.write("workload,epoch,rank,w,n,len,t_s_ns,t_w_ns,t_c_ns,T_ns,loss\n")
            for r in allr:
                for row in r.cpu().tolist():
                    f.write(name + "," + ",".join(
                        ("" if x != x else (str(int(x)) if j < 5 else f"{x:.6g}")) for j, x in enumerate(row)) + "\n")


def nccl_baseline(wk, world, rank, tdev, reps=20):
    """K5: the same weighted average through NCCL on the same buffer — premul-sum
    (ncclRedOpCreatePreMulSum via torch) and scale + SUM — against K3, all timed back to back."""
    import torch

    import paper_2111_08272_b200 as pr

    n_r = wk.alloc.view()["n"][rank]
    buf = wk.flat
    out = {"propring_K3": _timed_collective(lambda: pr.weighted_allreduce(wk.comm, buf, n_r), buf, world, tdev, reps)}
    if getattr(wk, "pflat", None) is not None:
        # rows a6-a9 fused (K7 in K3); lr = 0 leaves the parameters bit-identical (θ + (−0)·d = θ)
        out["propring_K3_K7_fused"] = _timed_collective(
            lambda: pr.weighted_allreduce_sgd(wk.comm, buf, wk.pflat, n_r, 0.0, 0.0, zero_grad=False), buf, world,
            tdev, reps)
    out.update(_nccl_pair(buf, n_r / wk.alloc.view()["B"], world, tdev, reps))
    buf.zero_()
    return out


def _timed_collective(fn, buf, world, tdev, reps=20, warm=5):
    """nccl-tests protocol: barrier, warm-up calls, `reps` calls back to back bracketed by
    CUDA events, max over ranks."""
    import torch
    import torch.distributed as dist

    for _ in range(warm):
        fn()
    torch.cuda.synchronize()
    dist.barrier()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record()
    for _ in range(reps):
        fn()
    b.record()
    torch.cuda.synchronize()
    us = _max_over_ranks(a.elapsed_time(b) / reps, world, tdev) * 1e3
    Z = buf.numel() * buf.element_size()
    bus = Z * 2 * (world - 1) / world / (us * 1e-6) / 1e9
    return {"us": us, "busbw_GBs": bus, "frac_of_770": bus / NVLINK_PEER_GBS, "frac_of_900": bus / NVLINK_NOMINAL_GBS}


def _nccl_pair(buf, s, world, tdev, reps=20):
    import torch.distributed as dist

    out = {}
    try:
        op = dist._make_nccl_premul_sum(s)
        out["nccl_premul_sum"] = _timed_collective(lambda: dist.all_reduce(buf, op=op), buf, world, tdev, reps)
    except Exception as e:   # noqa: BLE001
        out["nccl_premul_sum"] = {"error": repr(e)[:200]}

    def scale_sum():
        buf.mul_(s)
        dist.all_reduce(buf)

    out["nccl_scale_then_sum"] = _timed_collective(scale_sum, buf, world, tdev, reps)
    return out


def allreduce_sweep(ctx, reps=20):
    """N > 1: K3 at the north star's ≥ 64 MB sizes (64 MiB, 256 MiB fp32; 64 MiB bf16; the VGG-16 gradient) on
    a registered buffer, C5's skewed weights, against NCCL premul-sum and scale + sum on the same buffer."""
    import torch

    import paper_2111_08272_b200 as pr

    world, rank, comm, tdev = ctx["world"], ctx["rank"], ctx["comm"], ctx["tdev"]
    w = C5_WEIGHTS.get(world, [1 + (r % 4) for r in range(world)])
    n = [256 * x for x in w]
    s = n[rank] / sum(n)
    zmax = max(256 << 20, L_VGG16 * 4)
    raw = comm.alloc(zmax)
    res = []
    for dtype, Z in ((torch.float32, 64 << 20), (torch.float32, 256 << 20), (torch.float32, L_VGG16 * 4),
                     (torch.bfloat16, 64 << 20)):
        buf = raw[:Z].view(dtype)
        g = torch.Generator(device="cuda").manual_seed(1000 + rank)
        buf.copy_(torch.randn(buf.numel(), device="cuda", generator=g).to(dtype))
        row = {"bytes": Z, "dtype": str(dtype).split(".")[-1], "weights": n,
               "propring_K3": _timed_collective(lambda: pr.weighted_allreduce(comm, buf, n[rank]), buf, world, tdev,
                                                reps)}
        if not ctx["shared"]:
            row.update(_nccl_pair(buf, s, world, tdev, reps))
        res.append(row)
    # N2's NVLS variant (in-switch reduction through an NVSwitch multicast object) where the platform has one
    nv_comm = pr.comm_init(rank, world, ctx["local"], config=pr.comm_config(algo=pr.ALGO_NVLS))
    try:
        nv = nv_comm.nvls_alloc(zmax)
        for row in res:
            if row["dtype"] != "float32":
                continue
            Z = row["bytes"]
            buf = nv[:Z].view(torch.float32)
            g = torch.Generator(device="cuda").manual_seed(1000 + rank)
            buf.copy_(torch.randn(buf.numel(), device="cuda", generator=g))
            row["propring_NVLS"] = _timed_collective(lambda: pr.weighted_allreduce(nv_comm, buf, n[rank]), buf, world,
                                                     tdev, reps)
    except pr.PropringError as e:
        for row in res:
            row["propring_NVLS"] = {"unavailable": str(e)[:160]}
    finally:
        nv_comm.destroy()
    return res


def colocated_allreduce(hbm, peak_kind, P=8, reps=20):
    """N = 1: K3 with all P ranks on the one GPU — the same kernel and protocol with peer memory = local HBM
    (an HBM-roofline proxy, not NVLink), plus the fused a6-a9 kernel, C1's 4 KiB call, and the per-rank
    CTA throughput of the cross-GPU configuration."""
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
    # C3's VGG-16 gradient (553 MB per rank, the >= 64 MB regime of the north-star target) at P = 4 with the
    # allocation C3 converges to (n = 16·[11,11,21,21]): same proxy, same byte count formula
    del bufs
    P3, L3 = 4, L_VGG16
    c3 = pr.comm_init_local(P3, torch.cuda.current_device(), pr.comm_config())
    b3 = [torch.randn(L3, device="cuda") for _ in range(P3)]
    n3 = [16 * w for w in (11, 11, 21, 21)]
    for _ in range(2):
        pr.weighted_allreduce_local(c3, b3, n3)
    torch.cuda.synchronize()
    a.record()
    for _ in range(5):
        pr.weighted_allreduce_local(c3, b3, n3)
    b.record()
    torch.cuda.synchronize()
    t3 = a.elapsed_time(b) / 5
    byts3 = P3 * (6 + 5 * (P3 - 2)) * (L3 * 4) / P3
    vgg = {"P": P3, "bytes_per_rank": L3 * 4, "n_local": n3, "avg_us": t3 * 1e3,
           "achieved": byts3 / (t3 * 1e-3) / 1e9, "frac": byts3 / (t3 * 1e-3) / 1e9 / hbm,
           "algorithmic_bytes_per_call": byts3}
    del b3
    for c in c3:
        c.destroy()
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
    del store, grads, thetas
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
    # NVLink run would face before the link's 770 GB/s (tools/sweep_cta.py).  NOT an NVLink
    # number: the stores never cross a link.
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
    pull = colocated_pull(hbm, n, n3, reps)
    return {"kernel": "ring_kernel<float> (K3), all ranks on one GPU", "P": P, "bytes_per_rank": Z,
            "fused_a6_a9_us": fused_us, "composed_a6_a9_us": composed_us,
            "c1_allreduce_4KiB_P2_us": c1_us, "vgg16_C3_P4": vgg, "pull_two_shot": pull,
            "cross_gpu_config_per_rank_busbw_equiv": {
                "GBs": per_rank_bus, "us": x_us, "bytes": Lx * 4, "P": 2, "channels": 32,
                "vs_nvlink_770": per_rank_bus / NVLINK_PEER_GBS,
                "note": "CTA-throughput proxy with both ranks on one GPU: not NVLink"},
            "n_local": n, "avg_us": t * 1e3, "bound": "hbm", "achieved": byts / (t * 1e-3) / 1e9, "peak": hbm,
            "unit": "GB/s", "frac": byts / (t * 1e-3) / 1e9 / hbm, "peak_kind": peak_kind,
            "algorithmic_bytes_per_call": byts,
            "note": "P virtual ranks co-resident on one GPU exercise the same kernel and protocol; peer stores "
                    "land in local HBM, so this is an HBM roofline, not an NVLink number (the algorithmic bytes "
                    "count every staging round trip at HBM, part of which the 126 MB L2 serves: frac can exceed 1)"}


def colocated_pull(hbm, n8, n3, reps):
    """The pull two-shot (PR_ALGO_TWO_SHOT_PULL, N2; the ring's bits) on the same co-located cases as the
    ring: ResNet-18 gradient at P = 8, C3's VGG-16 gradient at P = 4, and the cross-GPU configuration's
    per-rank CTA proxy (P = 2, 32 channels, 256 MiB).  Algorithmic HBM bytes per call: every rank reads its
    chunk from the P buffers and writes it into the P buffers — 2·Z per rank."""
    import torch

    import paper_2111_08272_b200 as pr

    def one(P, L, n, k, **cfg):
        comms = pr.comm_init_local(P, torch.cuda.current_device(), pr.comm_config(algo=pr.ALGO_TWO_SHOT_PULL, **cfg))
        bufs = [torch.randn(L, device="cuda") for _ in range(P)]
        for _ in range(2):
            pr.weighted_allreduce_local(comms, bufs, n)
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        for _ in range(k):
            pr.weighted_allreduce_local(comms, bufs, n)
        e1.record()
        torch.cuda.synchronize()
        us = e0.elapsed_time(e1) / k * 1e3
        del bufs
        for c in comms:
            c.destroy()
        Z = L * 4
        return {"P": P, "bytes_per_rank": Z, "avg_us": us, "algorithmic_bytes_per_call": 2 * P * Z,
                "achieved": 2 * P * Z / (us * 1e-6) / 1e9, "frac": 2 * P * Z / (us * 1e-6) / 1e9 / hbm,
                "busbw_equiv_per_rank_GBs": Z * 2 * (P - 1) / P / (us * 1e-6) / 1e9}

    out = {"kernel": "twoshot_pull_kernel<float> (K3 variant, N2), all ranks on one GPU",
           "resnet18_P8": one(8, L_RESNET18, n8, reps), "vgg16_C3_P4": one(4, L_VGG16, n3, 5),
           # the TMA-staged data path (PR_COMM_FLAG_PULL_TMA, opt-in): same bits, deeper load queue
           "tma": {"kernel": "twoshot_pull_tma_kernel<float>", "resnet18_P8": one(8, L_RESNET18, n8, reps, pull_tma=True),
                   "vgg16_C3_P4": one(4, L_VGG16, n3, 5, pull_tma=True)}}
    # rows a6-a9 fused into the pull two-shot (K7 applied by the chunk owner, gradient reset), as the ring's
    # fused_a6_a9_us beside it
    P, L = 8, L_RESNET18
    comms = pr.comm_init_local(P, torch.cuda.current_device(), pr.comm_config(algo=pr.ALGO_TWO_SHOT_PULL))
    store = [torch.randn(2 * L, device="cuda") for _ in range(P)]
    grads, thetas = [x[:L] for x in store], [x[L:] for x in store]
    for _ in range(3):
        pr.weighted_allreduce_sgd_local(comms, grads, thetas, n8, 1e-6, 0.0, zero_grad=True)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(reps):
        pr.weighted_allreduce_sgd_local(comms, grads, thetas, n8, 1e-6, 0.0, zero_grad=True)
    e1.record()
    torch.cuda.synchronize()
    out["fused_a6_a9_resnet18_P8_us"] = e0.elapsed_time(e1) / reps * 1e3
    del store, grads, thetas
    for c in comms:
        c.destroy()
    x = one(2, (256 << 20) // 4, [1, 2], 5, channels=32, slot_bytes=1 << 20)
    x["channels"] = 32
    x["vs_nvlink_770"] = x["busbw_equiv_per_rank_GBs"] / NVLINK_PEER_GBS
    x["note"] = "CTA-throughput proxy with both ranks on one GPU: not NVLink"
    out["cross_gpu_config_per_rank"] = x
    return out


# ---------------------------------------------------------------------------------------------------
# Per-kernel oracle timings beside the GPU kernels (SURVEY §8(d) "Oracle timing beside it")
KERNEL_CASES = [
    # (key, oracle part, gpu kernel, params)
    ("shard_N50000", "O3+O4 permutation + shard", "K1 pr_shard_indices", {"N": 50_000}),
    ("shard_N1281167", "O3+O4 permutation + shard", "K1 pr_shard_indices", {"N": 1_281_167}),
    ("gather_C2", "O5 gather (u8 -> bf16 affine)", "K2 pr_gather_rows", {"rows": 256, "shape": (3, 32, 32)}),
    ("gather_C3", "O5 gather (u8 -> bf16 affine)", "K2 pr_gather_rows", {"rows": 336, "shape": (3, 224, 224)}),
] + [(f"wavg_{name}_P{P}", "O6 weighted average (fp64)", "K3 ring, P ranks co-located",
      {"L": L, "P": P, "size": name})
     for name, L in (("4KB", 1024), ("46.76MB", L_RESNET18), ("553MB", L_VGG16)) for P in (2, 4, 8)] + [
    ("controller_P8", "O8 controller step (Eq. 10 + Hamilton + stop rule)", "pr_alloc_update (host C++)", {"P": 8}),
]
O6_SLICE = 17_294_693          # 553 MB: the oracle is timed on a 1/8 slice and scaled ×8 (bounded sample)


def oracle_timings_child(path):
    """Runs in a subprocess pinned to core 0 with single-threaded BLAS (taskset -c 0 equivalent): each oracle
    part at the §8(d) sizes, median of 5 after one warm-up.  Writes {key: ms} as JSON to `path`."""
    import numpy as np

    import synth
    from oracle import allocation as OA
    from oracle import gather as OG
    from oracle import permutation as OP
    from oracle import wavg as OW

    def med(fn, reps=5):
        fn()
        ts = []
        for _ in range(reps):
            t = time.perf_counter()
            fn()
            ts.append((time.perf_counter() - t) * 1e3)
        return statistics.median(ts)

    res = {}
    sc, sh = np.float32([1 / 51.5865, 1 / 50.847, 1 / 51.255]), np.float32([125.307, 122.961, 113.8575])
    for key, _, _, p in KERNEL_CASES:
        if key.startswith("shard"):
            res[key] = med(lambda: OP.shard_indices(p["N"], 0, p["N"], 1234, 3))
        elif key.startswith("gather"):
            c, h, w = p["shape"]
            X = synth.images_u8(4 * p["rows"], c, h, w, seed=0).reshape(4 * p["rows"], -1)
            idx = np.arange(0, 4 * p["rows"], 4)
            res[key] = med(lambda: OG.gather_rows(X, idx, OG.U8_TO_BF16_AFFINE, scale=sc, shift=sh, plane=h * w))
        elif key.startswith("wavg"):
            L = min(p["L"], O6_SLICE)
            g = synth.gradients(p["P"], L, seed_base=1000)
            nl = [256 * x for x in C5_WEIGHTS[p["P"]]]
            res[key] = med(lambda: OW.weighted_average(OW.as_f64(g, "f32"), nl)) * (p["L"] / L)
        elif key.startswith("controller"):
            def ctl():
                a = OA.alloc_init(50_000, [1] * 8, C=64, g=16)
                OA.alloc_update(a, [1.0, 1.0, 1.0, 1.0, 2.0, 2.0, 4.0, 4.0])
            res[key] = med(ctl, reps=25)
    with open(path, "w") as f:
        json.dump(res, f)


def _cpu_model():
    try:
        with open("/proc/cpuinfo") as f:
            for ln in f:
                if ln.startswith("model name"):
                    return ln.split(":", 1)[1].strip()
    except OSError:
        pass
    return None


def gpu_kernel_timings(reps=20):
    """The GPU side of KERNEL_CASES through the C ABI (CUDA events, median of `reps` after warm-up)."""
    import torch

    import paper_2111_08272_b200 as pr

    def med(fn, reps=reps):
        for _ in range(3):
            fn()
        torch.cuda.synchronize()
        ts = []
        for _ in range(reps):
            a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            a.record()
            fn()
            b.record()
            b.synchronize()
            ts.append(a.elapsed_time(b))
        return statistics.median(ts)

    res = {}
    comms_by_p = {}
    for key, _, _, p in KERNEL_CASES:
        if key.startswith("shard"):
            a = pr.alloc_init(p["N"], [1], C=1, g=1)
            idx = torch.empty(p["N"], dtype=torch.int64, device="cuda")
            res[key] = med(lambda: pr.shard_indices(a, 0, 3, 1234, idx))
        elif key.startswith("gather"):
            c, h, w = p["shape"]
            n_src = 4096 if h == 32 else 2048
            X = torch.randint(0, 256, (n_src, c * h * w), dtype=torch.uint8, device="cuda")
            Y = torch.zeros(n_src, dtype=torch.int64, device="cuda")
            idx = torch.randperm(n_src, device="cuda")[:p["rows"]].contiguous()
            out = torch.empty((p["rows"], c * h * w), dtype=torch.bfloat16, device="cuda")
            yo = torch.empty(p["rows"], dtype=torch.int64, device="cuda")
            op = pr.make_gather_op(pr.GATHER_U8_TO_BF16_AFFINE, [1 / 51.5865, 1 / 50.847, 1 / 51.255],
                                   [125.307, 122.961, 113.8575], h * w, layout=pr.GATHER_LAYOUT_HWC)
            res[key] = med(lambda: pr.gather_rows(X, n_src, c * h * w, idx, p["rows"], out, op, Y, yo))
            del X
        elif key.startswith("wavg"):
            P = p["P"]
            if P not in comms_by_p:
                comms_by_p[P] = pr.comm_init_local(P, torch.cuda.current_device(), pr.comm_config(algo=pr.ALGO_AUTO))
            bufs = [torch.randn(p["L"], device="cuda") for _ in range(P)]
            nl = [256 * x for x in C5_WEIGHTS[P]]
            res[key] = med(lambda: pr.weighted_allreduce_local(comms_by_p[P], bufs, nl), reps=10)
            del bufs
        elif key.startswith("controller"):
            ts = []
            for _ in range(25):
                a = pr.alloc_init(50_000, [1] * 8, C=64, g=16)
                t = time.perf_counter()
                a.update([1.0, 1.0, 1.0, 1.0, 2.0, 2.0, 4.0, 4.0])
                ts.append((time.perf_counter() - t) * 1e3)
            res[key] = statistics.median(ts)
    for cs in comms_by_p.values():
        for c in cs:
            c.destroy()
    torch.cuda.empty_cache()
    return res


def kernel_vs_oracle():
    """GPU kernel timings, then the oracle's in a pinned single-threaded subprocess, side by side."""
    import tempfile

    gpu = gpu_kernel_timings()
    fd, path = tempfile.mkstemp(suffix=".json")
    os.close(fd)
    env = dict(os.environ, OMP_NUM_THREADS="1", OPENBLAS_NUM_THREADS="1", MKL_NUM_THREADS="1",
               NUMEXPR_NUM_THREADS="1")
    t0 = time.perf_counter()
    try:
        subprocess.run([sys.executable, os.path.abspath(__file__), "--oracle-timings-child", path], env=env,
                       check=True, preexec_fn=lambda: os.sched_setaffinity(0, {0}), timeout=600,
                       stdout=subprocess.DEVNULL)
        with open(path) as f:
            ora = json.load(f)
    finally:
        os.unlink(path)
    rows = []
    for key, opart, kern, p in KERNEL_CASES:
        o, g = ora.get(key), gpu.get(key)
        rows.append({"case": key, "oracle": opart, "gpu": kern,
                     "params": {k: (list(v) if isinstance(v, tuple) else v) for k, v in p.items()},
                     "oracle_ms": o, "gpu_ms": g, "ratio": (o / g) if (o and g) else None})
    return {"threads": 1, "pinned": "core 0 (sched_setaffinity {0}, as taskset -c 0); OMP/BLAS threads 1",
            "cpu_model": _cpu_model(), "host_cores": os.cpu_count(), "stat": "median of 5 after 1 warm-up "
            "(controller: 25); GPU: CUDA events, median of 20 (K3: 10) after 3 warm-up",
            "o6_553MB_sample": f"the 553 MB O6 rows time a {O6_SLICE:,}-element slice (1/8 of VGG-16) and scale ×8",
            "wall_s": time.perf_counter() - t0, "rows": rows}


# ---------------------------------------------------------------------------------------------------
def oracle_step(P, sample_rows, X, Y, grads, model, rank=0, a=None, epoch=0, strong=True):
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
        a = OA.alloc_init(N_DATA, [1] * P, C=units_for(P, strong), g=G_UNIT)
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
    """Inputs of the CPU reference step.  Imports only synth/, oracle/ and torch (torchvision's ResNet-18
    built directly: nothing of the product package is loaded on this arm)."""
    import numpy as np
    import torch
    import torchvision

    import synth

    X = synth.images_u8(N_DATA, seed=0).reshape(N_DATA, -1)
    Y = synth.labels(N_DATA, 10, seed=1)
    grads = synth.gradients(max(P, 1), L_RESNET18, seed_base=1000).astype(np.float64)
    model = torchvision.models.resnet18(num_classes=1000)
    return X, Y, grads, model, torch.get_num_threads()


def cpu_baseline(P, sample_rows=16, steps=2, strong=True):
    X, Y, grads, model, cores = cpu_reference_setup(P)
    oracle_step(P, sample_rows, X, Y, grads, model, strong=strong)          # warm-up
    t0 = time.perf_counter()
    for s in range(steps):
        oracle_step(P, sample_rows, X, Y, grads, model, epoch=s, strong=strong)
    dt = (time.perf_counter() - t0) / steps
    return {"value": sample_rows / dt, "unit": "samples/s", "cores": cores, "kind": "oracle",
            "sample": f"{steps} aggregation steps, each: oracle shard slice + oracle gather of {sample_rows} rows + "
                      f"torch-CPU fp32 ResNet-18 fwd/bwd on those rows + oracle fp64 weighted average of "
                      f"{max(P, 1)}×{L_RESNET18} gradients + controller; samples/s = rows/step time"}


def run_reference(args):
    rank = int(os.environ.get("RANK", "0"))
    if rank != 0:
        return
    strong = not args.weak
    X, Y, grads, model, cores = cpu_reference_setup(args.gpus)
    sample_rows = 16
    for w in range(args.warmup):
        oracle_step(args.gpus, sample_rows, X, Y, grads, model, epoch=w, strong=strong)
    t0 = time.perf_counter()
    for s in range(args.steps):
        oracle_step(args.gpus, sample_rows, X, Y, grads, model, epoch=s, strong=strong)
    dt = time.perf_counter() - t0
    value = args.steps * sample_rows / dt
    out = {"impl": "reference", "metric": METRIC, "value": value, "unit": "samples/s", "n_gpus": args.gpus,
           "steps": args.steps, "warmup": args.warmup, "ms_per_step": dt / args.steps * 1e3,
           "higher_is_better": True, "scaling": "strong" if strong else "weak", "vs_baseline": None,
           "dtype": "f64", "data": "synthetic",
           "config": bench_config(args.gpus, False, strong),
           "cpu_baseline": {"value": value, "unit": "samples/s", "cores": cores, "kind": "oracle",
                            "sample": f"bounded sample of the workload: each step = one aggregation step on "
                                      f"{sample_rows} rows (oracle shard + gather, torch-CPU fp32 ResNet-18 "
                                      f"fwd/bwd, oracle fp64 weighted average of P x 11,689,512 gradients, "
                                      f"controller); samples/s = rows / step time"},
           "e2e": {"value": value, "unit": "samples/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    print(json.dumps(out))


# ---------------------------------------------------------------------------------------------------
def run_ours(args):
    import torch
    import torch.distributed as dist

    import paper_2111_08272_b200 as pr

    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    if world != args.gpus:
        raise SystemExit(f"--gpus {args.gpus} but WORLD_SIZE={world}")
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
    # AUTO: the step buffers take the ring (with K7 fused); N1's buckets take the pull two-shot (<= 16 MiB at P >= 8)
    comm = pr.comm_init(rank, world, local, config=pr.comm_config(algo=pr.ALGO_AUTO)) if world > 1 else None
    ctx = {"world": world, "rank": rank, "local": local, "comm": comm, "tdev": tdev, "shared": shared}
    strong = not args.weak

    head = run_workload("resnet18", args, ctx, strong=strong)
    weak = None
    if world > 1 and not args.no_weak:
        w = run_workload("resnet18", args, ctx, strong=not strong, e2e_epochs=0, kernel_detail=False)
        weak = {k: w[k] for k in ("value", "unit", "ms_per_step", "steps", "epoch_ms_each", "config", "kernel_shares")}
        weak["allreduce"] = w["allreduce"]
    vgg = None
    if not args.no_vgg:
        v = run_workload("vgg16", args, ctx, strong=strong, steps=args.vgg_steps, warmup=3, e2e_epochs=1)
        vgg = {k: v[k] for k in ("value", "unit", "ms_per_step", "steps", "warmup", "epoch_ms_each", "config",
                                 "roofline", "roofline_detail", "gather", "sgd", "allreduce", "e2e", "gpu_launches",
                                 "clocks", "kernel_shares", "alloc_w", "loss_last_epoch")}
    sweep = allreduce_sweep(ctx) if world > 1 else None
    hbm, peak_kind = peaks()
    colocated = None
    if world == 1 and not args.no_colocated:
        colocated = colocated_allreduce(hbm, peak_kind)
    kvo = None
    if world == 1 and rank == 0 and not (args.no_cpu_baseline or args.no_oracle_kernels):
        kvo = kernel_vs_oracle()

    if rank == 0:
        cpu = None
        if world == 1 and not args.no_cpu_baseline:
            cpu = cpu_baseline(world, strong=strong)
            cpu["cpu_model"] = _cpu_model()
            cpu["per_kernel"] = kvo
        out = {
            "metric": METRIC, "value": head["value"], "unit": "samples/s", "n_gpus": world, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": head["ms_per_step"], "higher_is_better": True,
            "scaling": "strong" if strong else "weak", "vs_baseline": None,
            "dtype": "bf16 compute (autocast), fp32 gradients / allreduce / update",
            "data": "synthetic",
            "config": head["config"],
            "epoch_time_s": head["epoch_time_s"],
            "epoch_ms_each": head["epoch_ms_each"],
            "host_enqueue_ms_each": head["host_enqueue_ms_each"],
            "roofline": head["roofline"],
            "roofline_detail": head["roofline_detail"],
            "gather": head["gather"],
            "sgd": head["sgd"],
            "allreduce": head["allreduce"],
            "allreduce_sweep": sweep,
            "allreduce_colocated": colocated,
            "e2e": head["e2e"],
            "gpu_launches": head["gpu_launches"],
            "clocks": head["clocks"],
            "cpu_baseline": cpu,
            "alloc_w": head["alloc_w"],
            "loss_last_epoch": head["loss_last_epoch"],
            # share of the timed region spent in each library kernel (live events; compare with the ncu
            # launch list of the same command in profiles/)
            "kernel_shares": head["kernel_shares"],
            "weak_scaling": weak,
            "vgg16": vgg,
        }
        if args.data_n != N_DATA:
            out["config"]["workload"] += f" [PROFILING VARIANT: N={args.data_n}]"
        print(json.dumps(out), flush=True)
    if comm is not None:
        comm.destroy()
    if world > 1:
        dist.destroy_process_group()


def main(argv=None):
    argv = sys.argv[1:] if argv is None else argv
    a = parse(argv)
    if a.oracle_timings_child:
        return oracle_timings_child(a.oracle_timings_child)
    if a.gpus > 1 and "WORLD_SIZE" not in os.environ and a.impl == "ours":
        sys.exit(self_launch(a, argv))
    if a.impl == "reference":
        run_reference(a)
    else:
        run_ours(a)


if __name__ == "__main__":
    main()
