"""Run each library kernel in isolation at bench sizes (target for `ncu --set full`, one GPU).

    python tools/profile_kernels.py [gather|gather_imagenet|shard|ring|pull|pull_cta|ring_cta|all] [reps]

gather          K2 at the bench step size: 1024 CIFAR rows (3,072 B u8 -> 6,144 B bf16)
gather_imagenet K2 at the C3 fast-rank size: 336 ImageNet-shaped rows (150,528 B -> 301,056 B)
shard           K1 over N = 1,281,167 (whole permutation)
ring            K3, 8 ranks co-located on this GPU, 11,689,512 fp32 each (ResNet-18 gradients)
Also prints CUDA-event timings (outside ncu these are the kernel's live durations).
"""

import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import torch  # noqa: E402

import paper_2111_08272_b200 as pr  # noqa: E402


def timed(fn, reps):
    fn()
    torch.cuda.synchronize()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record()
    for _ in range(reps):
        fn()
    b.record()
    torch.cuda.synchronize()
    return a.elapsed_time(b) / reps * 1e3   # us


def gather(rows, row_bytes, nsrc, reps, plane, impls=(1, 2), layout=0, seq=False):
    X = torch.randint(0, 256, (nsrc, row_bytes), dtype=torch.uint8, device="cuda")
    Y = torch.randint(0, 10, (nsrc,), dtype=torch.int64, device="cuda")
    # distinct rows, like a shard of the per-epoch permutation (sampling with replacement would let
    # repeated rows hit in L2 and flatter the kernel)
    idx = torch.arange(rows, device="cuda") if seq else torch.randperm(nsrc, device="cuda")[:rows] if rows <= nsrc else torch.randint(0, nsrc, (rows,), device="cuda")
    out = torch.empty((rows, row_bytes), dtype=torch.bfloat16, device="cuda")
    lab = torch.empty(rows, dtype=torch.int64, device="cuda")
    for impl in impls:
        op = pr.make_gather_op(pr.GATHER_U8_TO_BF16_AFFINE, [0.02, 0.02, 0.02], [120.0, 120.0, 110.0], plane,
                               impl=impl, layout=layout)
        us = timed(lambda: pr.gather_rows(X, nsrc, row_bytes, idx, rows, out, op, Y, lab), reps)
        byts = rows * (3 * row_bytes + 24)
        print(f"gather[{ {1: 'LSU', 2: 'TMA', 3: 'BULK'}[impl]}{',HWC' if layout else ''}] rows={rows} row_bytes={row_bytes}: {us:.2f} us, "
              f"{byts / us / 1e3:.1f} GB/s algorithmic")


def shard(reps):
    N = 1281167
    out = torch.empty(N, dtype=torch.int64, device="cuda")
    us = timed(lambda: pr.permute(N, 1234, 3, 0, N, out), reps)
    print(f"permute N={N}: {us:.2f} us, {N / us:.1f} M indices/s")


def sgd(reps, L=11_689_512):
    th = torch.randn(L, device="cuda")
    g = torch.randn(L, device="cuda")
    us = timed(lambda: pr.sgd_update(th, g, 1e-2, 1e-4, zero_grad=True), reps)
    print(f"sgd L={L}: {us:.2f} us, {16 * L / us / 1e3:.1f} GB/s algorithmic")


def ring_fused(reps, P=8, L=11_689_512, only_fused=False):
    """Rows a6-a9: composed (K3 ring + K7 per rank) vs fused (K7 inside K3), 8 ranks co-located."""
    comms = pr.comm_init_local(P, 0)
    store = [torch.randn(2 * L, device="cuda") for _ in range(P)]
    grads, thetas = [s_[:L] for s_ in store], [s_[L:] for s_ in store]
    n = [64, 64, 64, 64, 128, 128, 256, 256][:P]

    def composed():
        pr.weighted_allreduce_local(comms, grads, n)
        for r in range(P):
            pr.sgd_update(thetas[r], grads[r], 1e-6, 0.0, zero_grad=False)

    def fused():
        pr.weighted_allreduce_sgd_local(comms, grads, thetas, n, 1e-6, 0.0, zero_grad=False)

    if only_fused:
        print(f"a6-a9 fused P={P} L={L}: {timed(fused, reps):.1f} us")
        for c in comms:
            c.destroy()
        return
    uc, uf = timed(composed, reps), timed(fused, reps)
    print(f"a6-a9 P={P} L={L}: composed (ring + {P}x K7) {uc:.1f} us, fused {uf:.1f} us")
    for c in comms:
        c.destroy()


def ring(reps, P=8, L=11_689_512, **cfg):
    comms = pr.comm_init_local(P, 0, pr.comm_config(**cfg))
    bufs = [torch.randn(L, device="cuda") for _ in range(P)]
    n = [64, 64, 64, 64, 128, 128, 256, 256][:P]
    us = timed(lambda: pr.weighted_allreduce_local(comms, bufs, n), reps)
    byts = (6 + 5 * (P - 2)) * L * 4
    print(f"ring P={P} L={L}: {us:.1f} us, {byts / us / 1e3:.1f} GB/s algorithmic HBM (all ranks)")
    for c in comms:
        c.destroy()


def pull(reps, P=8, L=11_689_512, **cfg):
    """K3 pull two-shot (PR_ALGO_TWO_SHOT_PULL); algorithmic HBM bytes co-located: every rank reads its
    chunk from P buffers (Z) and writes it into P buffers (Z) -> 2·Z per rank."""
    comms = pr.comm_init_local(P, 0, pr.comm_config(algo=pr.ALGO_TWO_SHOT_PULL, **cfg))
    bufs = [torch.randn(L, device="cuda") for _ in range(P)]
    n = [64, 64, 64, 64, 128, 128, 256, 256][:P]
    us = timed(lambda: pr.weighted_allreduce_local(comms, bufs, n), reps)
    byts = 2 * P * L * 4
    print(f"pull two-shot P={P} L={L}: {us:.1f} us, {byts / us / 1e3:.1f} GB/s algorithmic HBM (all ranks), "
          f"bus-equivalent per rank {L * 4 * 2 * (P - 1) / P / us / 1e3:.1f} GB/s")
    for c in comms:
        c.destroy()


if __name__ == "__main__":
    what = sys.argv[1] if len(sys.argv) > 1 else "all"
    reps = int(sys.argv[2]) if len(sys.argv) > 2 else 20
    if what in ("gather", "all"):
        gather(1024, 3072, 50000, reps, 1024)
    if what in ("gather_epoch", "all"):
        gather(49152, 3072, 50000, reps, 1024)          # one launch per epoch (48 steps x 1024 rows)
    if what in ("gather_epoch_hwc", "all"):
        gather(49152, 3072, 50000, reps, 1024, impls=(2, 1) if what == "all" else (2,), layout=1)
    if what == "gather_epoch_hwc_lsu":                 # exactly the bench's launch (channels-last, LSU)
        gather(49152, 3072, 50000, reps, 1024, impls=(1,), layout=1)
    if what == "gather_epoch_hwc_lsu_seq":             # same bytes, rows in order: cost of the scatter
        gather(49152, 3072, 50000, reps, 1024, impls=(1,), layout=1, seq=True)
    if what in ("gather_imagenet", "all"):
        gather(336, 150528, 2000, reps, 50176)
    if what == "gather_imagenet_hwc":                  # the C3 step launch, channels-last, LSU vs TMA
        gather(336, 150528, 2000, reps, 50176, impls=(1, 2), layout=1)
    if what == "gather_imagenet_epoch_hwc":            # a VGG-16 epoch-size launch (16,384 distinct rows, 7.4 GB)
        gather(16384, 150528, 16384, reps, 50176, impls=(1, 2), layout=1)
    if what == "gather_bulk_ab":                       # channels-last: LSU vs bulk-store kernel at the bench's sizes
        for rows, rb, nsrc, plane in ((1024, 3072, 50000, 1024), (49152, 3072, 50000, 1024),
                                      (336, 150528, 2000, 50176), (16384, 150528, 16384, 50176)):
            gather(rows, rb, nsrc, reps, plane, impls=(1, 3), layout=1)
    if what == "gather_imagenet_epoch_hwc_bulk":       # the VGG-16 leg's launch with the bulk-store kernel
        gather(16384, 150528, 16384, reps, 50176, impls=(3,), layout=1)
    if what == "gather_epoch_hwc_bulk":
        gather(49152, 3072, 50000, reps, 1024, impls=(3,), layout=1)
    if what in ("shard", "all"):
        shard(reps)
    if what in ("sgd", "all"):
        sgd(reps)
    if what == "sgd_vgg16":                            # the VGG-16 leg's update (138,357,544 fp32)
        sgd(reps, L=138_357_544)
    if what == "gather_imagenet_epoch_hwc_lsu":        # the VGG-16 leg's launch kind (LSU, channels-last)
        gather(16384, 150528, 16384, reps, 50176, impls=(1,), layout=1)
    if what == "pull":                                  # co-located ResNet-18 gradient, 8 ranks, default channels
        pull(reps)
    if what == "pull_fused":                            # a6-a9 fused into the pull two-shot, P = 8 co-located
        P, L = 8, 11_689_512
        comms = pr.comm_init_local(P, 0, pr.comm_config(algo=pr.ALGO_TWO_SHOT_PULL))
        store = [torch.randn(2 * L, device="cuda") for _ in range(P)]
        grads, thetas = [x[:L] for x in store], [x[L:] for x in store]
        n = [64, 64, 64, 64, 128, 128, 256, 256]
        us = timed(lambda: pr.weighted_allreduce_sgd_local(comms, grads, thetas, n, 1e-6, 0.0, zero_grad=True), reps)
        print(f"fused pull two-shot a6-a9 P={P} L={L}: {us:.1f} us")
        for c in comms:
            c.destroy()
    if what == "pull_vgg":                              # C3's VGG-16 gradient, P = 4, register-queued pull
        pull(max(2, reps // 4), P=4, L=138_357_544)
    if what == "pull_tma_vgg":                          # the same, TMA-staged (PR_COMM_FLAG_PULL_TMA)
        pull(max(2, reps // 4), P=4, L=138_357_544, pull_tma=True)
    if what == "pull_cta":                              # per-channel regime: P = 2, 4 channels, 256 MiB
        pull(max(2, reps // 4), P=2, L=(256 << 20) // 4, channels=4)
    if what == "ring_cta":                              # the ring in the same per-channel regime
        ring(max(2, reps // 4), P=2, L=(256 << 20) // 4, channels=4)
    if what == "ring_sizes":                            # default channels: P = 2 / 4 / 8 at the ResNet-18 and VGG-16 sizes
        for P in (2, 4, 8):
            for L in (11_689_512, 138_357_544):
                ring(max(2, reps // (4 if L > 2e7 else 1)), P=P, L=L)
    if what == "ring_cta":                              # the cross-GPU configuration, 2 ranks: per-channel CTA path
        ring(reps, P=2, L=(256 << 20) // 4, channels=32, slot_bytes=1 << 20)
    if what in ("ring_fused", "all"):
        ring_fused(reps)
    if what == "ring_fused_only":
        ring_fused(reps, only_fused=True)
    if what in ("ring", "all"):
        ring(reps)
