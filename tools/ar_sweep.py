#!/usr/bin/env python
"""C5 (BASELINE configs[4]): weighted allreduce sweep, 1 MiB … 1 GiB, fp32/bf16, skewed weights, vs NCCL.

Multi-GPU (one rank per GPU):
    torchrun --nproc-per-node P --master-addr 127.0.0.1 tools/ar_sweep.py [--max-mib 1024]
Co-located (all P ranks on one GPU, HBM-bound proxy; no NCCL):
    python tools/ar_sweep.py --colocated 8

Per size/dtype: K3 time (max over ranks), bus bandwidth Z·2(P−1)/P/t, fraction of the 770 GB/s
measured peer bandwidth (900 nominal); NCCL premul-sum and scale+sum on the same buffer; parity of
K3 against the CPU oracle's fp64 weighted mean on 10^6 sampled elements.
Weights: P=2 [1,3]·256, P=4 [1,1,2,4]·256, P=8 [1,1,1,1,2,2,4,4]·256.
"""

import argparse
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import numpy as np  # noqa: E402
import torch  # noqa: E402

import paper_2111_08272_b200 as pr  # noqa: E402

WEIGHTS = {1: [1], 2: [1, 3], 3: [1, 2, 3], 4: [1, 1, 2, 4], 8: [1, 1, 1, 1, 2, 2, 4, 4]}


def weights(P):
    return [256 * w for w in WEIGHTS.get(P, [1 + (r % 4) for r in range(P)])]


def fill(buf, rank, dtype):
    g = torch.Generator(device="cuda").manual_seed(1000 + rank)
    x = torch.randn(buf.numel(), device="cuda", generator=g)
    buf.copy_(x.to(dtype))


def check_parity(out, P, n, dtype, L, rank_fill, sample=1_000_000):
    """fp64 oracle on sampled elements (oracle/wavg.py arithmetic on the same inputs)."""
    from oracle import wavg as W

    idx = torch.randint(0, L, (min(sample, L),), device="cuda")
    g = []
    for r in range(P):
        b = torch.empty(L, dtype=dtype, device="cuda")
        rank_fill(b, r)
        g.append(b[idx].double().cpu().numpy())
    ref, den = W.weighted_average(np.stack(g), n)
    err, zb = W.error_metric(out[idx].double().cpu().numpy(), ref, den)
    return err, zb


def sizes(max_mib):
    s, z = [], 1 << 20
    while z <= max_mib << 20:
        s.append(z)
        z <<= 1
    return s


def run_colocated(P, max_mib, reps, algo=0):
    comms = pr.comm_init_local(P, 0, pr.comm_config(algo=algo))
    n = weights(P)
    for dtype, es in ((torch.float32, 4), (torch.bfloat16, 2)):
        for Z in sizes(max_mib):
            L = Z // es
            bufs = [torch.empty(L, dtype=dtype, device="cuda") for _ in range(P)]
            for r in range(P):
                fill(bufs[r], r, dtype)
            pr.weighted_allreduce_local(comms, bufs, n)
            torch.cuda.synchronize()
            err, zb = check_parity(bufs[0], P, n, dtype, L, lambda b, r: fill(b, r, dtype))
            for _ in range(3):
                pr.weighted_allreduce_local(comms, bufs, n)
            a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            a.record()
            for _ in range(reps):
                pr.weighted_allreduce_local(comms, bufs, n)
            b.record()
            torch.cuda.synchronize()
            us = a.elapsed_time(b) / reps * 1e3
            hbm = (6 + 5 * (P - 2)) * Z / (us * 1e-6) / 1e9
            print(json.dumps({"mode": "colocated", "algo": algo, "P": P, "dtype": str(dtype).split(".")[-1], "bytes": Z, "us": us,
                              "hbm_algorithmic_GBs": hbm, "max_err": err, "zero_violations": zb}), flush=True)
            del bufs
    for c in comms:
        c.destroy()


def run_multi(max_mib, reps, algo=0, channels=0, min_slice=0, bulk=False, l2pf=False):
    import torch.distributed as dist

    local = int(os.environ.get("LOCAL_RANK", "0"))
    shared = os.environ.get("PR_BENCH_SHARED_GPU") == "1"   # functional check: every rank on cuda:0, gloo
    if shared:
        local = 0
    torch.cuda.set_device(local)
    if shared:
        dist.init_process_group("gloo")
    else:
        dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    rank, P = dist.get_rank(), dist.get_world_size()
    comm = pr.comm_init(rank, P, local, config=pr.comm_config(algo=algo, channels=channels, min_slice_bytes=min_slice,
                                                              pull_tma=os.environ.get("PR_AR_SWEEP_PULL_TMA") == "1",
                                                              bulk_store=bulk, l2_prefetch=l2pf))
    n = weights(P)
    s = n[rank] / sum(n)
    Zmax = max_mib << 20
    # NVLS (algo 5): the buffers must live in the communicator's NVLS region (multicast-bound memory)
    raw = comm.nvls_alloc(Zmax) if algo == pr.ALGO_NVLS else comm.alloc(Zmax)
    for dtype, es in ((torch.float32, 4), (torch.bfloat16, 2)):
        for Z in sizes(max_mib):
            L = Z // es
            buf = raw[:Z].view(dtype)

            def timed(fn):
                for _ in range(3):
                    fn()
                torch.cuda.synchronize()
                dist.barrier()
                a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                a.record()
                for _ in range(reps):
                    fn()
                b.record()
                torch.cuda.synchronize()
                t = torch.tensor([a.elapsed_time(b) / reps], device="cpu" if shared else "cuda")
                dist.all_reduce(t, op=dist.ReduceOp.MAX)
                return float(t) * 1e3

            fill(buf, rank, dtype)
            pr.weighted_allreduce(comm, buf, n[rank])
            torch.cuda.synchronize()
            err, zb = check_parity(buf, P, n, dtype, L, lambda b, r: fill(b, r, dtype)) if rank == 0 else (0, 0)
            us = timed(lambda: pr.weighted_allreduce(comm, buf, n[rank]))
            res = {"mode": "nvlink", "P": P, "dtype": str(dtype).split(".")[-1], "bytes": Z, "us": us,
                   "busbw_GBs": Z * 2 * (P - 1) / P / (us * 1e-6) / 1e9, "max_err": err, "zero_violations": zb}
            res["frac_of_770"] = res["busbw_GBs"] / 770.0
            if shared:
                if rank == 0:
                    print(json.dumps(res), flush=True)
                continue
            try:
                op = dist._make_nccl_premul_sum(s)
                t = timed(lambda: dist.all_reduce(buf, op=op))
                res["nccl_premul_us"] = t
            except Exception as e:  # noqa: BLE001
                res["nccl_premul_error"] = repr(e)[:120]

            def scale_sum():
                buf.mul_(s)
                dist.all_reduce(buf)

            res["nccl_scale_sum_us"] = timed(scale_sum)
            if rank == 0:
                print(json.dumps(res), flush=True)
    comm.destroy()
    dist.destroy_process_group()


if __name__ == "__main__":
    ap = argparse.ArgumentParser()
    ap.add_argument("--colocated", type=int, default=0)
    ap.add_argument("--max-mib", type=int, default=1024)
    ap.add_argument("--reps", type=int, default=20)
    ap.add_argument("--algo", type=int, default=0, help="0 ring, 1 two-shot, 2 auto, 3 LL ring, 4 one-shot LL, 5 NVLS, 6 pull two-shot")
    ap.add_argument("--channels", type=int, default=0, help="CTAs per rank (multi-GPU mode; 0 = topology default)")
    ap.add_argument("--min-slice", type=int, default=0, help="ring min_slice_bytes (0 = slot-sized slices)")
    ap.add_argument("--bulk", action="store_true", help="ring data path with TMA bulk stores")
    ap.add_argument("--l2pf", action="store_true", help="ring: L2 prefetch of each slice's own gradient")
    a = ap.parse_args()
    if a.colocated:
        run_colocated(a.colocated, a.max_mib, a.reps, a.algo)
    else:
        run_multi(a.max_mib, a.reps, a.algo, a.channels, a.min_slice, a.bulk, a.l2pf)
