"""GPU parity of K3, the sample-count-weighted ring allreduce, through the C ABI.

All P ranks run on the one test GPU (pr_comm_init_local: same kernel, same flag/credit protocol, peer
memory = local memory).  Checks:
  * bit-identical to the oracle's ring-order replay (oracle/ring_emu.c) — catches any chunk, offset,
    order or rounding bug;
  * within the north-star tolerance of the fp64 weighted mean (1e-5 fp32, 2e-2 bf16), with the
    cancellation-aware metric of DESIGN.md §3 #16;
  * equal weights vs torch's mean (library routine); n_r = 0 contributes nothing, even NaN;
  * back-to-back calls (monotone counters), direct and staged all-gather, error latching.
"""

import numpy as np
import pytest
import torch

import synth
from oracle import gather as OG
from oracle import wavg as W

pytestmark = pytest.mark.gpu
pr = pytest.importorskip("paper_2111_08272_b200")

TOL = {"f32": 1e-5, "bf16": 2e-2}


@pytest.fixture(scope="module", autouse=True)
def _cuda():
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")


_GROUPS = {}


def group(P, **cfg):
    key = (P, tuple(sorted(cfg.items())))
    if key not in _GROUPS:
        _GROUPS[key] = pr.comm_init_local(P, 0, pr.comm_config(watchdog_ns=5_000_000_000, **cfg))
    return _GROUPS[key]


def _inputs(P, L, dtype, kind="gaussian", seed=0):
    g32 = synth.gradients(P, L, seed_base=1000 + seed, kind=kind)
    if dtype == "bf16":
        host = OG.f32_to_bf16_bits(g32)
        dev = [torch.from_numpy(host[r].view(np.int16).copy()).cuda().view(torch.bfloat16) for r in range(P)]
    else:
        host = g32
        dev = [torch.from_numpy(g32[r].copy()).cuda() for r in range(P)]
    return host, dev


def _result_host(t, dtype):
    return t.view(torch.int16).cpu().numpy().view(np.uint16) if dtype == "bf16" else t.cpu().numpy()


def _check(P, L, dtype, n, comms, kind="gaussian", seed=0, stream=None):
    host, dev = _inputs(P, L, dtype, kind, seed)
    pr.weighted_allreduce_local(comms, dev, n, stream=stream)
    torch.cuda.synchronize()
    for c in comms:
        assert c.status() == 0
    emu = W.ring_emulate(host, n, dtype)
    ref, den = W.weighted_average(W.as_f64(host, dtype), n)
    outs = [_result_host(d, dtype) for d in dev]
    for r in range(P):
        assert np.array_equal(outs[r].view(np.uint8), emu.view(np.uint8)), f"rank {r} differs from ring replay"
    err, zb = W.error_metric(W.as_f64(outs[0], dtype), ref, den)
    assert zb == 0 and err <= TOL[dtype], err
    return outs


@pytest.mark.parametrize("dtype", ["f32", "bf16"])
@pytest.mark.parametrize("P", [2, 3, 4, 5, 7, 8])
def test_counts_and_weights(P, dtype):
    comms = group(P)
    rng = np.random.Generator(np.random.PCG64(P))
    for L in (1, 7, P, P + 1, 1000, 4099, 2 ** 20 + 3):
        for wkind in ("equal", "skewed", "zero"):
            if wkind == "equal":
                n = [256] * P
            elif wkind == "skewed":
                n = [int(x) * 64 for x in rng.integers(1, 9, P)]
            else:
                n = [int(x) * 16 for x in rng.integers(1, 5, P)]
                n[int(rng.integers(0, P))] = 0
            _check(P, L, dtype, n, comms, kind="mixed" if L % 2 else "gaussian", seed=L)


@pytest.mark.parametrize("P", [2, 4, 8])
def test_large_buffer_64MiB(P):
    comms = group(P)
    L = 64 * 2 ** 20 // 4
    n = [int(x) for x in [64, 64, 64, 64, 128, 128, 256, 256][:P]]
    _check(P, L, "f32", n, comms)


def test_resnet18_size_sampled_parity_against_oracle():
    """Full-size C2/C4 gradient (11,689,512 fp32) at P=8: ring replay on every element."""
    P = 8
    comms = group(P)
    _check(P, 11_689_512, "f32", [64, 64, 64, 64, 128, 128, 256, 256], comms)


def test_vgg16_size_C3_full_parity():
    """Full-size C3 gradient (VGG-16, 138,357,544 fp32 = 553 MB per rank) at P=4 with the allocation C3
    converges to (w = [11,11,21,21], g = 16): ring replay on every element + fp64 tolerance."""
    P = 4
    comms = group(P)
    _check(P, 138_357_544, "f32", [16 * w for w in (11, 11, 21, 21)], comms)


def test_c5_maximum_size_1GiB():
    """C5's largest buffer (2^30 B per rank, fp32) at P = 2 with C5's skewed weights [1,3]·256, and bf16
    256 MiB per rank (2^27 elements) at P = 4 [1,1,2,4]·256 — ring replay on every element + the fp64
    tolerance, mixed-scale inputs."""
    _check(2, 2 ** 28, "f32", [256, 768], group(2), kind="mixed", seed=30)
    _check(4, 2 ** 27, "bf16", [256, 256, 512, 1024], group(4), kind="mixed", seed=31)


def test_pull_tma_channels_graph_replay_and_full_sizes():
    """The TMA-staged pull: few and many channels, `.sys` scope, back-to-back calls, graph replay, the
    ResNet-18 gradient at P = 8 and C3's VGG-16 gradient at P = 4 (ring replay on every element)."""
    for cfg in (dict(channels=1), dict(channels=3, sys_scope=True, threads=128)):
        for P in (2, 4, 7):
            comms = group(P, algo=pr.ALGO_TWO_SHOT_PULL, pull_tma=True, **cfg)
            for it, L in enumerate((999, 300_001, 5)):
                _check(P, L, "f32" if it % 2 == 0 else "bf16", [5] * (P - 1) + [it], comms, seed=L + 1)
    P, L = 3, 40_000
    comms = group(P, algo=pr.ALGO_TWO_SHOT_PULL, pull_tma=True)
    host, dev = _inputs(P, L, "f32", seed=23)
    src = [d.clone() for d in dev]
    n = [3, 1, 2]
    s = torch.cuda.Stream()
    g = torch.cuda.CUDAGraph()
    with torch.cuda.stream(s):
        pr.weighted_allreduce_local(comms, dev, n, stream=s)
        torch.cuda.synchronize()
        with torch.cuda.graph(g, stream=s):
            pr.weighted_allreduce_local(comms, dev, n, stream=s)
    emu = W.ring_emulate(host, n, "f32")
    for _ in range(3):
        for d, s0 in zip(dev, src):
            d.copy_(s0)
        g.replay()
        torch.cuda.synchronize()
        assert all(np.array_equal(d.cpu().numpy(), emu) for d in dev)
    _check_sampled(8, SIZES["resnet18"], SKEW, group(8, algo=pr.ALGO_TWO_SHOT_PULL, pull_tma=True), seed=61)
    _check_sampled(4, SIZES["vgg16"], SKEW[-4:], group(4, algo=pr.ALGO_TWO_SHOT_PULL, pull_tma=True), seed=62)


def test_c5_maximum_size_1GiB_pull_two_shot():
    """The same C5 maximum-size cases through the pull two-shot (and P = 8 at 64 MiB fp32)."""
    _check(2, 2 ** 28, "f32", [256, 768], group(2, algo=pr.ALGO_TWO_SHOT_PULL), kind="mixed", seed=32)
    _check(4, 2 ** 27, "bf16", [256, 256, 512, 1024], group(4, algo=pr.ALGO_TWO_SHOT_PULL), kind="mixed", seed=33)
    _check(8, 2 ** 24, "f32", [64, 64, 64, 64, 128, 128, 256, 256], group(8, algo=pr.ALGO_TWO_SHOT_PULL), seed=34)


def test_resnet18_size_bf16_P8():
    """C5's bf16 leg at the ResNet-18 size, skewed weights 1:1:1:1:2:2:4:4."""
    P = 8
    comms = group(P)
    _check(P, 11_689_512, "bf16", [64, 64, 64, 64, 128, 128, 256, 256], comms, kind="mixed")


def test_equal_weights_match_torch_mean():
    P, L = 4, 100_003
    comms = group(P)
    host, dev = _inputs(P, L, "f32")
    mean = torch.stack(dev).double().mean(0)                      # library routine
    den = torch.stack(dev).double().abs().sum(0) / P + 1e-300     # Σ|s·g| (before the in-place reduce)
    pr.weighted_allreduce_local(comms, dev, [32] * P)
    torch.cuda.synchronize()
    assert float(((dev[0].double() - mean).abs() / den).max()) <= 1e-5


def test_power_of_two_equal_weights_is_scaled_sum_bit_exact():
    P, L = 8, 333_333
    comms = group(P)
    host, dev = _inputs(P, L, "f32", seed=5)
    pr.weighted_allreduce_local(comms, dev, [10] * P)
    torch.cuda.synchronize()
    cs = W.chunk_elems(L, P, 4)
    plain = np.zeros(L, dtype=np.float32)
    for c in range(P):
        lo, hi = c * cs, min((c + 1) * cs, L)
        acc = host[c, lo:hi].copy()
        for h in range(1, P):
            acc = (acc + host[(c + h) % P, lo:hi]).astype(np.float32)
        plain[lo:hi] = acc
    assert np.array_equal(dev[3].cpu().numpy(), plain * np.float32(1 / 8))


def test_zero_sample_rank_with_nan_does_not_propagate():
    P, L = 4, 10_000
    comms = group(P)
    host, dev = _inputs(P, L, "f32")
    dev[2].fill_(float("nan"))
    host[2, :] = np.nan
    n = [10, 20, 0, 30]
    pr.weighted_allreduce_local(comms, dev, n)
    torch.cuda.synchronize()
    out = dev[2].cpu().numpy()
    assert np.all(np.isfinite(out))
    assert np.array_equal(out, W.ring_emulate(host, n, "f32"))


def test_identity_P1_and_zero_samples_error():
    comms = group(1)
    x = torch.randn(1000, device="cuda")
    y = x.clone()
    pr.weighted_allreduce_local(comms, [x], [5])
    assert torch.equal(x, y)
    with pytest.raises(pr.PropringError) as e:
        pr.weighted_allreduce_local(comms, [x], [0])
    assert e.value.code == pr.PR_ERR_ZERO_SAMPLES


def test_all_zero_samples_latches_error_and_leaves_buffers():
    comms = pr.comm_init_local(3, 0, pr.comm_config(watchdog_ns=2_000_000_000))
    host, dev = _inputs(3, 5000, "f32")
    before = [d.clone() for d in dev]
    with pytest.raises(pr.PropringError):
        pr.weighted_allreduce_local(comms, dev, [0, 0, 0])   # host-side check
    for c in comms:
        c.destroy()


def test_back_to_back_calls_and_streams():
    """Many calls in a row (monotone counters, parity-double-buffered handshake), different sizes."""
    P = 5
    comms = group(P)
    s = torch.cuda.Stream()
    with torch.cuda.stream(s):
        for it, L in enumerate([10, 100_000, 3, 77_777, 1_000_000, 5, 12_345]):
            _check(P, L, "f32" if it % 2 else "bf16", [it + 1, 2, 3, 4 * it, 5], comms, seed=it, stream=s)


def test_staged_allgather_path():
    for P in (2, 3, 8):
        comms = group(P, force_staged=True)
        for L in (5, 4099, 2 ** 20 + 3):
            _check(P, L, "f32", [1 + r for r in range(P)], comms, seed=L)
            _check(P, L, "bf16", [3] * P, comms, seed=L)


@pytest.mark.parametrize("P", [2, 5, 8])
def test_system_scope_protocol(P):
    """The multi-GPU flavour of the protocol (.sys release/acquire) on the one test GPU."""
    comms = group(P, sys_scope=True)
    for L in (7, 4099, 2 ** 20 + 3, 11_689_512):
        _check(P, L, "f32", [64, 64, 64, 64, 128, 128, 256, 256][:P], comms, seed=L)
    _check(P, 2 ** 20 + 3, "bf16", [3] * P, comms)
    comms2 = group(P, sys_scope=True, force_staged=True)
    _check(P, 300_001, "f32", [1 + r for r in range(P)], comms2)


@pytest.mark.parametrize("cfg", [dict(channels=1, slots=2, slot_bytes=256, stages=2, tile_bytes=256), dict(channels=3, slots=3, slot_bytes=4096),
                                 dict(channels=32, slots=8, slot_bytes=65536, threads=256, stages=4, tile_bytes=8192),
                                 dict(channels=3, slots=4, slot_bytes=1024, force_staged=True),
                                 dict(channels=2, slots=5, slot_bytes=512, threads=64)])
def test_config_variants(cfg):
    for P in (2, 5):
        comms = group(P, **cfg)
        for L in (1, 999, 300_001):
            _check(P, L, "f32", [7] * (P - 1) + [1], comms, seed=L)
            _check(P, L, "bf16", [2] * P, comms, seed=L)


def test_cuda_graph_replay():
    """Device-resident counters make the call capturable: replaying the graph gives the same result."""
    P, L = 4, 50_000
    comms = group(P)
    host, dev = _inputs(P, L, "f32", seed=9)
    src = [d.clone() for d in dev]
    n = [1, 2, 3, 4]
    s = torch.cuda.Stream()
    g = torch.cuda.CUDAGraph()
    with torch.cuda.stream(s):
        pr.weighted_allreduce_local(comms, dev, n, stream=s)   # warm-up outside capture
        torch.cuda.synchronize()
        with torch.cuda.graph(g, stream=s):
            pr.weighted_allreduce_local(comms, dev, n, stream=s)
    emu = W.ring_emulate(host, n, "f32")
    for _ in range(3):
        for d, s0 in zip(dev, src):
            d.copy_(s0)
        g.replay()
        torch.cuda.synchronize()
        for d in dev:
            assert np.array_equal(d.cpu().numpy(), emu)


def test_length_mismatch_and_timeout_latch():
    """Per-rank launches of a local group on separate streams: count mismatch -> LENGTH_MISMATCH on
    every rank with buffers untouched; a missing peer -> PEER_TIMEOUT."""
    P = 2
    comms = pr.comm_init_local(P, 0, pr.comm_config(channels=2, watchdog_ns=1_000_000_000))
    a = torch.randn(1000, device="cuda")
    b = torch.randn(1000, device="cuda")
    a0, b0 = a.clone(), b.clone()
    s0, s1 = torch.cuda.Stream(), torch.cuda.Stream()
    torch.cuda.synchronize()
    pr.weighted_allreduce(comms[0], a, 1, stream=s0, count=1000)
    pr.weighted_allreduce(comms[1], b, 1, stream=s1, count=999)
    torch.cuda.synchronize()
    assert comms[0].status() == pr.PR_ERR_LENGTH_MISMATCH and comms[1].status() == pr.PR_ERR_LENGTH_MISMATCH
    assert torch.equal(a, a0) and torch.equal(b, b0)
    for c in comms:
        c.destroy()
    comms = pr.comm_init_local(P, 0, pr.comm_config(channels=2, watchdog_ns=300_000_000))
    pr.weighted_allreduce(comms[0], a, 1, stream=s0)
    torch.cuda.synchronize()
    assert comms[0].status() == pr.PR_ERR_PEER_TIMEOUT
    with pytest.raises(pr.PropringError) as e:
        pr.weighted_allreduce(comms[0], a, 1, stream=s0)
    assert e.value.code == pr.PR_ERR_PEER_TIMEOUT
    for c in comms:
        c.destroy()


def test_pull_two_shot_mismatch_unregistered_and_timeout_latch():
    """Pull two-shot error paths, per-rank launches on separate streams: count mismatch -> LENGTH_MISMATCH on
    every rank, buffers untouched; buffers that cannot be addressed directly (force_staged) -> INVALID on
    every rank; a missing peer -> PEER_TIMEOUT.  (Ranks picking different kernels: tests/test_multiproc.py.)"""
    P, L = 2, 1 << 18
    s0, s1 = torch.cuda.Stream(), torch.cuda.Stream()
    comms = pr.comm_init_local(P, 0, pr.comm_config(channels=2, watchdog_ns=1_000_000_000, algo=pr.ALGO_TWO_SHOT_PULL))
    a, b = torch.randn(L, device="cuda"), torch.randn(L, device="cuda")
    a0, b0 = a.clone(), b.clone()
    torch.cuda.synchronize()
    pr.weighted_allreduce(comms[0], a, 1, stream=s0, count=L)
    pr.weighted_allreduce(comms[1], b, 1, stream=s1, count=L - 1)
    torch.cuda.synchronize()
    assert comms[0].status() == pr.PR_ERR_LENGTH_MISMATCH and comms[1].status() == pr.PR_ERR_LENGTH_MISMATCH
    assert torch.equal(a, a0) and torch.equal(b, b0)
    for c in comms:
        c.destroy()
    comms = pr.comm_init_local(P, 0, pr.comm_config(channels=2, watchdog_ns=1_000_000_000, force_staged=True,
                                                    algo=pr.ALGO_TWO_SHOT_PULL))
    pr.weighted_allreduce(comms[0], a, 1, stream=s0)
    pr.weighted_allreduce(comms[1], b, 1, stream=s1)
    torch.cuda.synchronize()
    assert comms[0].status() == pr.PR_ERR_INVALID and comms[1].status() == pr.PR_ERR_INVALID
    assert torch.equal(a, a0) and torch.equal(b, b0)
    for c in comms:
        c.destroy()
    comms = pr.comm_init_local(P, 0, pr.comm_config(channels=2, watchdog_ns=300_000_000, algo=pr.ALGO_TWO_SHOT_PULL))
    pr.weighted_allreduce(comms[0], a, 1, stream=s0)
    torch.cuda.synchronize()
    assert comms[0].status() == pr.PR_ERR_PEER_TIMEOUT
    for c in comms:
        c.destroy()


def test_timestamps_and_status():
    P = 3
    comms = group(P)
    host, dev = _inputs(P, 1 << 20, "f32")
    pr.weighted_allreduce_local(comms, dev, [1, 2, 3])
    torch.cuda.synchronize()
    for c in comms:
        t = c.timestamps()
        assert 0 < t[0] <= t[1] <= t[2]


# ---- two-shot variant: same bits as the ring -------------------------------------------

@pytest.mark.parametrize("dtype", ["f32", "bf16"])
@pytest.mark.parametrize("P", [2, 3, 5, 8])
def test_two_shot_bit_identical_to_ring_replay(P, dtype):
    comms = group(P, algo=pr.ALGO_TWO_SHOT)
    rng = np.random.Generator(np.random.PCG64(100 + P))
    for L in (1, 7, P + 1, 4099, 2 ** 20 + 3):
        n = [int(x) * 16 for x in rng.integers(1, 9, P)]
        if L % 2:
            n[int(rng.integers(0, P))] = 0
        _check(P, L, dtype, n, comms, kind="mixed" if L % 3 == 0 else "gaussian", seed=L)


def test_two_shot_small_slots_many_slices_and_sys_scope():
    for cfg in (dict(ts_slots=2, ts_slot_bytes=256, channels=3), dict(ts_slots=3, ts_slot_bytes=4096, sys_scope=True)):
        for P in (2, 4):
            comms = group(P, algo=pr.ALGO_TWO_SHOT, **cfg)
            for L in (999, 300_001):
                _check(P, L, "f32", [5] * (P - 1) + [1], comms, seed=L)
                _check(P, L, "bf16", [2] * P, comms, seed=L)


@pytest.mark.parametrize("tma", [False, True])
@pytest.mark.parametrize("dtype", ["f32", "bf16"])
@pytest.mark.parametrize("P", [2, 3, 4, 5, 8])
def test_pull_two_shot_bit_identical_to_ring_replay(P, dtype, tma):
    """PR_ALGO_TWO_SHOT_PULL: chunk r read straight out of every rank's buffer, reduced in the ring's order
    with the ring's rounding — the ring replay's bits, including n_r = 0 ranks and ragged tails; with
    PR_COMM_FLAG_PULL_TMA the source tiles are staged in shared memory by TMA (same bits)."""
    comms = group(P, algo=pr.ALGO_TWO_SHOT_PULL, pull_tma=tma)
    rng = np.random.Generator(np.random.PCG64(300 + P))
    for L in (1, 7, P + 1, 4099, 2 ** 20 + 3):
        n = [int(x) * 16 for x in rng.integers(1, 9, P)]
        if L % 2:
            n[int(rng.integers(0, P))] = 0
        _check(P, L, dtype, n, comms, kind="mixed" if L % 3 == 0 else "gaussian", seed=L)


def test_pull_two_shot_channels_sys_scope_and_graph_replay():
    for cfg in (dict(channels=1), dict(channels=3, sys_scope=True), dict(channels=64, threads=128)):
        for P in (2, 4, 7):
            comms = group(P, algo=pr.ALGO_TWO_SHOT_PULL, **cfg)
            for it, L in enumerate((999, 300_001, 5)):                # back to back: monotone counters
                _check(P, L, "f32" if it % 2 == 0 else "bf16", [5] * (P - 1) + [it], comms, seed=L)
    P, L = 3, 40_000
    comms = group(P, algo=pr.ALGO_TWO_SHOT_PULL)
    host, dev = _inputs(P, L, "f32", seed=22)
    src = [d.clone() for d in dev]
    n = [3, 1, 2]
    s = torch.cuda.Stream()
    g = torch.cuda.CUDAGraph()
    with torch.cuda.stream(s):
        pr.weighted_allreduce_local(comms, dev, n, stream=s)
        torch.cuda.synchronize()
        with torch.cuda.graph(g, stream=s):
            pr.weighted_allreduce_local(comms, dev, n, stream=s)
    emu = W.ring_emulate(host, n, "f32")
    for _ in range(3):
        for d, s0 in zip(dev, src):
            d.copy_(s0)
        g.replay()
        torch.cuda.synchronize()
        assert all(np.array_equal(d.cpu().numpy(), emu) for d in dev)


@pytest.mark.parametrize("P,L", [(8, 11_689_512), (4, 138_357_544)])
def test_pull_two_shot_full_sizes_against_oracle(P, L):
    """ResNet-18 gradient at P = 8 and VGG-16 at P = 4 (C3): sampled elements against the fp64 weighted mean
    (the oracle's definition, one element at a time) and every rank identical to rank 0."""
    comms = group(P, algo=pr.ALGO_TWO_SHOT_PULL)
    g = torch.Generator(device="cuda").manual_seed(L % 1000 + P)
    dev = [torch.randn(L, device="cuda", generator=g) for _ in range(P)]
    idx = torch.from_numpy(np.random.Generator(np.random.PCG64(L)).integers(0, L, 20000)).cuda()
    samp = np.stack([d[idx].cpu().numpy() for d in dev])
    n = [int(x) for x in np.random.Generator(np.random.PCG64(P)).integers(1, 400, P)]
    pr.weighted_allreduce_local(comms, dev, n)
    torch.cuda.synchronize()
    assert all(c.status() == 0 for c in comms)
    ref, den = W.weighted_average(samp.astype(np.float64), n)
    err, zb = W.error_metric(dev[0][idx].cpu().numpy().astype(np.float64), ref, den)
    assert zb == 0 and err <= TOL["f32"], err
    assert all(torch.equal(d, dev[0]) for d in dev[1:])


def test_auto_mixes_algorithms_back_to_back():
    """ALGO_AUTO: LL ring up to ll_max_bytes (256 KiB), pull two-shot up to ts_max_bytes, ring above; interleaved
    calls share the handshake sequence (the LL line flag) and the counters."""
    P = 4
    comms = group(P, algo=pr.ALGO_AUTO, ts_max_bytes=1 << 20)
    for it, L in enumerate([100, 2 ** 20, 3, 300_000, 5_000_000, 17]):   # 400 B .. 20 MB
        _check(P, L, "f32" if it % 2 else "bf16", [it + 1, 2, 0 if it == 3 else 3, 4], comms, seed=it)


def test_two_shot_graph_replay():
    P, L = 3, 40_000
    comms = group(P, algo=pr.ALGO_TWO_SHOT)
    host, dev = _inputs(P, L, "f32", seed=21)
    src = [d.clone() for d in dev]
    n = [3, 1, 2]
    s = torch.cuda.Stream()
    g = torch.cuda.CUDAGraph()
    with torch.cuda.stream(s):
        pr.weighted_allreduce_local(comms, dev, n, stream=s)
        torch.cuda.synchronize()
        with torch.cuda.graph(g, stream=s):
            pr.weighted_allreduce_local(comms, dev, n, stream=s)
    emu = W.ring_emulate(host, n, "f32")
    for _ in range(3):
        for d, s0 in zip(dev, src):
            d.copy_(s0)
        g.replay()
        torch.cuda.synchronize()
        assert all(np.array_equal(d.cpu().numpy(), emu) for d in dev)


# ---- LL ring: the ring's schedule and rounding with a low-latency line protocol (same bits) ------------

LL_ALGOS = {"ll": dict(algo=pr.ALGO_LL, ll_max_bytes=1 << 20), "oneshot": dict(algo=pr.ALGO_ONESHOT, os_max_bytes=1 << 20)}


@pytest.mark.parametrize("algo", ["ll", "oneshot"])
@pytest.mark.parametrize("dtype", ["f32", "bf16"])
@pytest.mark.parametrize("P", [2, 3, 4, 5, 8])
def test_ll_ring_bit_identical_to_ring_replay(P, dtype, algo):
    comms = group(P, **LL_ALGOS[algo])
    rng = np.random.Generator(np.random.PCG64(200 + P))
    for L in (1, 2, 3, 5, 7, P + 1, 1000, 4099, 65_537, 2 ** 18 - 1):   # ragged last lines (fp32 1/2, bf16 1..4)
        n = [int(x) * 16 for x in rng.integers(1, 9, P)]
        if L % 2:
            n[int(rng.integers(0, P))] = 0
        _check(P, L, dtype, n, comms, kind="mixed" if L % 3 == 0 else "gaussian", seed=L)


@pytest.mark.parametrize("algo", ["ll", "oneshot"])
def test_ll_ring_many_calls_reuse_regions_and_sys_scope(algo):
    """The line flag is the call's handshake sequence: back-to-back calls rewrite the same regions, and a
    stale line from the previous call must never pass (the results would then differ from the replay)."""
    for cfg in (dict(channels=3), dict(channels=16, sys_scope=True), dict(channels=1, threads=64)):
        P = 4
        comms = group(P, **LL_ALGOS[algo], **cfg)
        for it in range(12):
            L = [999, 65_536, 3, 40_001][it % 4]
            _check(P, L, "f32" if it % 3 else "bf16", [it % 5, 2, 3, 1 + it], comms, seed=100 + it)


@pytest.mark.parametrize("cfg", [dict(algo=pr.ALGO_LL, ll_max_bytes=4096), dict(algo=pr.ALGO_ONESHOT, os_max_bytes=4096)])
def test_ll_ring_above_ll_max_takes_the_ring(cfg):
    P = 3
    comms = group(P, **cfg)
    for L in (1000, 1025, 300_000):        # 4,000 B (LL), 4,100 B and 1.2 MB (ring)
        _check(P, L, "f32", [1, 2, 3], comms, seed=L)


@pytest.mark.parametrize("algo", ["ll", "oneshot"])
def test_ll_ring_graph_replay(algo):
    P, L = 3, 40_000
    comms = group(P, **LL_ALGOS[algo])
    host, dev = _inputs(P, L, "f32", seed=31)
    src = [d.clone() for d in dev]
    n = [3, 0, 2]
    s = torch.cuda.Stream()
    g = torch.cuda.CUDAGraph()
    with torch.cuda.stream(s):
        pr.weighted_allreduce_local(comms, dev, n, stream=s)
        torch.cuda.synchronize()
        with torch.cuda.graph(g, stream=s):
            pr.weighted_allreduce_local(comms, dev, n, stream=s)
    emu = W.ring_emulate(host, n, "f32")
    for _ in range(3):
        for d, s0 in zip(dev, src):
            d.copy_(s0)
        g.replay()
        torch.cuda.synchronize()
        assert all(np.array_equal(d.cpu().numpy(), emu) for d in dev)


@pytest.mark.parametrize("algo", [pr.ALGO_LL, pr.ALGO_ONESHOT])
def test_ll_ring_length_mismatch_and_timeout_latch(algo):
    P = 2
    comms = pr.comm_init_local(P, 0, pr.comm_config(channels=2, algo=algo, watchdog_ns=1_000_000_000))
    a = torch.randn(1000, device="cuda")
    b = torch.randn(1000, device="cuda")
    a0, b0 = a.clone(), b.clone()
    s0, s1 = torch.cuda.Stream(), torch.cuda.Stream()
    torch.cuda.synchronize()
    pr.weighted_allreduce(comms[0], a, 1, stream=s0, count=1000)
    pr.weighted_allreduce(comms[1], b, 1, stream=s1, count=999)
    torch.cuda.synchronize()
    assert comms[0].status() == pr.PR_ERR_LENGTH_MISMATCH and comms[1].status() == pr.PR_ERR_LENGTH_MISMATCH
    assert torch.equal(a, a0) and torch.equal(b, b0)
    for c in comms:
        c.destroy()
    comms = pr.comm_init_local(P, 0, pr.comm_config(channels=2, algo=algo, watchdog_ns=300_000_000))
    pr.weighted_allreduce(comms[0], a, 1, stream=s0)
    torch.cuda.synchronize()
    assert comms[0].status() == pr.PR_ERR_PEER_TIMEOUT
    for c in comms:
        c.destroy()


# ---- rows a6-a9 fused: K7 (SGD + reset) inside K3's ring -------------------------------------------------

def _fused_case(P, L, n, comms, seed, cfg_delta=True, lr=1e-2, wd=1e-4):
    """One [grad | theta] allocation per rank (theta at the same offset everywhere), replicated theta."""
    Lp = (L + 3) // 4 * 4
    g = synth.gradients(P, L, seed_base=seed)
    theta0 = synth.gradients(1, L, seed_base=seed + 500)[0]
    store = [torch.zeros(2 * Lp + (0 if cfg_delta else 4 * (r + 1)), device="cuda") for r in range(P)]
    off = [Lp if cfg_delta else Lp + 4 * (r + 1) for r in range(P)]
    grads = [store[r][:L] for r in range(P)]
    thetas = [store[r][off[r]:off[r] + L] for r in range(P)]
    for r in range(P):
        grads[r].copy_(torch.from_numpy(g[r]))
        thetas[r].copy_(torch.from_numpy(theta0))
    # composed reference on copies: ring allreduce, then K7 on every rank
    rg = [torch.from_numpy(g[r].copy()).cuda() for r in range(P)]
    rt = [torch.from_numpy(theta0.copy()).cuda() for r in range(P)]
    pr.weighted_allreduce_local(comms, rg, n)
    for r in range(P):
        pr.sgd_update(rt[r], rg[r], lr, wd, zero_grad=True)
    pr.weighted_allreduce_sgd_local(comms, grads, thetas, n, lr, wd, zero_grad=True)
    torch.cuda.synchronize()
    assert all(c.status() == 0 for c in comms)
    for r in range(P):
        assert torch.equal(thetas[r], rt[r]), f"rank {r}: fused θ' differs from ring + K7"
        assert torch.count_nonzero(grads[r]) == 0
    return g, theta0, thetas[0].cpu().numpy()


@pytest.mark.parametrize("P", [2, 3, 4, 8])
def test_fused_allreduce_sgd_bit_identical_to_composed(P):
    comms = group(P)
    rng = np.random.Generator(np.random.PCG64(300 + P))
    for L in (1, 7, 1000, 4099, 2 ** 20 + 3):
        n = [int(x) * 16 for x in rng.integers(1, 9, P)]
        if L % 2:
            n[int(rng.integers(0, P))] = 0
        _fused_case(P, L, n, comms, seed=L)


def test_fused_allreduce_sgd_resnet18_size_against_oracle():
    """Full ResNet-18 gradient at P = 8: fused θ' = composed θ' bit for bit, and within K7's two roundings of
    the oracle (ring replay for ḡ, fp64 SGD)."""
    from oracle import linmodel as LM

    P, L = 8, 11_689_512
    n = [64, 64, 64, 64, 128, 128, 256, 256]
    g, theta0, out = _fused_case(P, L, n, group(P), seed=77)
    gbar = W.ring_emulate(g, n, "f32").astype(np.float64)
    ref = LM.sgd_step(theta0.astype(np.float64), gbar, float(np.float32(1e-2)), float(np.float32(1e-4)))
    bound = 2.0 ** -24 * (np.abs(ref) + np.float32(1e-2) * np.abs(gbar + np.float32(1e-4) * theta0)) * 1.01
    assert np.all(np.abs(out.astype(np.float64) - ref) <= bound + 1e-45)


@pytest.mark.parametrize("tma", [False, True])
@pytest.mark.parametrize("P", [2, 3, 4, 5, 8])
def test_fused_pull_two_shot_bit_identical_to_composed(P, tma):
    """Rows a6-a9 in the pull two-shot: the owner of chunk r applies K7 and stores θ' into every rank's θ;
    same bits as ring + K7, gradients reset (zero_grad) or left untouched (zero_grad=False)."""
    comms = group(P, algo=pr.ALGO_TWO_SHOT_PULL, pull_tma=tma)
    rng = np.random.Generator(np.random.PCG64(310 + P))
    for L in (1, 7, 1000, 4099, 2 ** 20 + 3):
        n = [int(x) * 16 for x in rng.integers(1, 9, P)]
        if L % 2:
            n[int(rng.integers(0, P))] = 0
        _fused_case(P, L, n, comms, seed=L + 3)
    L = 5003
    g = synth.gradients(P, L, seed_base=8)
    theta0 = torch.from_numpy(synth.gradients(1, L, seed_base=9)[0]).cuda()
    store = [torch.zeros(2 * 5004, device="cuda") for _ in range(P)]
    grads, thetas = [x[:L] for x in store], [x[5004:5004 + L] for x in store]
    for r in range(P):
        grads[r].copy_(torch.from_numpy(g[r]))
        thetas[r].copy_(theta0)
    n = [1 + r for r in range(P)]
    pr.weighted_allreduce_sgd_local(comms, grads, thetas, n, 0.05, 1e-3, zero_grad=False)
    ref_g = [torch.from_numpy(g[r].copy()).cuda() for r in range(P)]
    pr.weighted_allreduce_local(group(P), ref_g, n)                    # the ring's ḡ
    ref = theta0.clone()
    pr.sgd_update(ref, ref_g[0], 0.05, 1e-3, zero_grad=False)
    torch.cuda.synchronize()
    for r in range(P):
        assert torch.equal(thetas[r], ref)
        assert np.array_equal(grads[r].cpu().numpy(), g[r])              # zero_grad=False: untouched


def test_fused_pull_two_shot_resnet18_size_and_graph_replay():
    from oracle import linmodel as LM

    P, L = 8, 11_689_512
    n = [64, 64, 64, 64, 128, 128, 256, 256]
    g, theta0, out = _fused_case(P, L, n, group(P, algo=pr.ALGO_TWO_SHOT_PULL), seed=78)
    gbar = W.ring_emulate(g, n, "f32").astype(np.float64)
    ref = LM.sgd_step(theta0.astype(np.float64), gbar, float(np.float32(1e-2)), float(np.float32(1e-4)))
    bound = 2.0 ** -24 * (np.abs(ref) + np.float32(1e-2) * np.abs(gbar + np.float32(1e-4) * theta0)) * 1.01
    assert np.all(np.abs(out.astype(np.float64) - ref) <= bound + 1e-45)
    P, L = 3, 40_000
    comms = group(P, algo=pr.ALGO_TWO_SHOT_PULL)
    store = [torch.zeros(2 * L, device="cuda") for _ in range(P)]
    grads, thetas = [s_[:L] for s_ in store], [s_[L:] for s_ in store]
    g = synth.gradients(P, L, seed_base=43)
    theta0 = torch.from_numpy(synth.gradients(1, L, seed_base=44)[0]).cuda()
    n = [3, 1, 2]
    s = torch.cuda.Stream()
    gr = torch.cuda.CUDAGraph()
    with torch.cuda.stream(s):
        pr.weighted_allreduce_sgd_local(comms, grads, thetas, n, 0.1, 0.0, stream=s)
        torch.cuda.synchronize()
        with torch.cuda.graph(gr, stream=s):
            pr.weighted_allreduce_sgd_local(comms, grads, thetas, n, 0.1, 0.0, stream=s)
    rg = [torch.from_numpy(g[r].copy()).cuda() for r in range(P)]
    pr.weighted_allreduce_local(comms, rg, n)
    ref = theta0.clone()
    pr.sgd_update(ref, rg[0].clone(), 0.1, 0.0)
    for _ in range(3):
        for r in range(P):
            grads[r].copy_(torch.from_numpy(g[r]))
            thetas[r].copy_(theta0)
        gr.replay()
        torch.cuda.synchronize()
        assert all(torch.equal(t, ref) for t in thetas)
        assert all(torch.count_nonzero(x) == 0 for x in grads)


def test_fused_allreduce_sgd_small_slices_staged_and_layout_fallbacks():
    for cfg in (dict(channels=3, slots=4, slot_bytes=4096, tile_bytes=1024, stages=3), dict(force_staged=True),
                dict(algo=pr.ALGO_AUTO)):
        comms = group(4, **cfg)
        for L in (999, 300_001):
            _fused_case(4, L, [3, 0, 5, 1], comms, seed=L + 9)
    # θ at different offsets on different ranks: the host composes the two operations instead
    _fused_case(3, 5000, [1, 2, 3], group(3), seed=5, cfg_delta=False)


def test_fused_allreduce_sgd_graph_replay():
    P, L = 3, 40_000
    comms = group(P)
    Lp = L
    store = [torch.zeros(2 * Lp, device="cuda") for _ in range(P)]
    grads, thetas = [s_[:L] for s_ in store], [s_[Lp:] for s_ in store]
    g = synth.gradients(P, L, seed_base=41)
    theta0 = torch.from_numpy(synth.gradients(1, L, seed_base=42)[0]).cuda()
    n = [3, 1, 2]
    s = torch.cuda.Stream()
    gr = torch.cuda.CUDAGraph()
    with torch.cuda.stream(s):
        pr.weighted_allreduce_sgd_local(comms, grads, thetas, n, 0.1, 0.0, stream=s)
        torch.cuda.synchronize()
        with torch.cuda.graph(gr, stream=s):
            pr.weighted_allreduce_sgd_local(comms, grads, thetas, n, 0.1, 0.0, stream=s)
    rg = [torch.from_numpy(g[r].copy()).cuda() for r in range(P)]
    pr.weighted_allreduce_local(comms, rg, n)
    ref = theta0.clone()
    pr.sgd_update(ref, rg[0].clone(), 0.1, 0.0)
    for _ in range(3):
        for r in range(P):
            grads[r].copy_(torch.from_numpy(g[r]))
            thetas[r].copy_(theta0)
        gr.replay()
        torch.cuda.synchronize()
        assert all(torch.equal(t, ref) for t in thetas)


def test_randomized_configs_all_algorithms():
    """Seeded sweep over communicator configurations × algorithms × P × counts × dtypes × weights: every
    result bit-identical to the oracle's ring replay (and, for fused calls, to ring + K7)."""
    rng = np.random.Generator(np.random.PCG64(2024))
    algos = [pr.ALGO_RING, pr.ALGO_TWO_SHOT, pr.ALGO_LL, pr.ALGO_ONESHOT, pr.ALGO_AUTO, pr.ALGO_TWO_SHOT_PULL]
    for case in range(80):
        P = int(rng.choice([2, 3, 4, 5, 6, 7, 8]))
        stages = int(rng.integers(2, 7))
        tile = int(rng.choice([256, 1024, 4096, 16384]))
        cfg = dict(channels=int(rng.integers(1, 9)), slots=int(rng.choice([2, 4, 6, 8])),
                   slot_bytes=int(rng.choice([256, 4096, 65536, 262144])), stages=stages, tile_bytes=tile,
                   threads=int(rng.choice([64, 128, 256, 512])), algo=int(rng.choice(algos)),
                   sys_scope=bool(rng.integers(0, 2)), ts_slot_bytes=int(rng.choice([256, 4096, 65536])),
                   ll_max_bytes=int(rng.choice([4096, 262144])), os_max_bytes=int(rng.choice([1024, 65536])))
        if cfg["algo"] == pr.ALGO_TWO_SHOT_PULL:                 # both pull data paths (a separate stream of
            cfg["pull_tma"] = bool(np.random.Generator(np.random.PCG64(case)).integers(0, 2))   # draws)
        comms = pr.comm_init_local(P, 0, pr.comm_config(watchdog_ns=5_000_000_000, **cfg))
        try:
            for _ in range(2):
                L = int(rng.choice([1, 3, 17, 1000, 4097, 65_537, 300_001]))
                dtype = "f32" if rng.integers(0, 2) else "bf16"
                n = [int(x) for x in rng.integers(0, 5, P)]
                if sum(n) == 0:
                    n[0] = 1
                _check(P, L, dtype, n, comms, kind="mixed" if L % 2 else "gaussian", seed=case * 7 + L)
            if cfg["algo"] in (pr.ALGO_RING, pr.ALGO_AUTO, pr.ALGO_TWO_SHOT_PULL):
                _fused_case(P, int(rng.choice([7, 5000, 200_003])), [1 + (r % 3) for r in range(P)], comms,
                            seed=case + 900)
        finally:
            for c in comms:
                c.destroy()


@pytest.mark.parametrize("min_slice", [4096, 65536])
def test_ring_min_slice_bit_identical(min_slice):
    """min_slice_bytes > 0 slices each chunk share into up to slots/2 slices: same bits (plain and fused)."""
    for P in (2, 4, 8):
        comms = group(P, min_slice_bytes=min_slice, slots=8)
        for L in (7, 4099, 300_001, 2 ** 21 + 5):
            _check(P, L, "f32" if L % 2 else "bf16", [1 + (r % 3) for r in range(P)], comms, seed=L + P)
        _fused_case(P, 200_003, [2] * P, comms, seed=P + 77)


# ---- the cross-GPU default configuration (VERDICT r1 "What's weak" #3c) --------------------------------
# Ranks on different GPUs resolve to 32 channels × 1 MiB staging slots with .sys-scope flags (resolve_config
# in ring.cu): the configuration an 8-GPU run executes.  Forced here on one GPU (sys_scope=True), at the
# gradient sizes of the bench's two models, P = 2 / 4 / 8, ring and fused a6-a9.
CROSS = dict(channels=32, slot_bytes=1 << 20, sys_scope=True)
# P = 8 co-located needs 8 × 32 channel CTAs resident at once (a cooperative launch): with 512 consumer
# threads and 6 × 2 × 16 KiB of stages one CTA fills an SM (148 < 256), so P = 8 runs the same channels,
# slots, slot size and scope — the same chunk / slice / flag geometry — with 256 consumer threads and 8 KiB
# tiles (two CTAs per SM).  Tile size and thread count only change how a slice is cut into TMA tiles.
CROSS8 = dict(CROSS, threads=256, tile_bytes=8192)
SIZES = {"resnet18": 11_689_512, "vgg16": 138_357_544}
SKEW = [64, 64, 64, 64, 128, 128, 256, 256]


def _check_sampled(P, L, n, comms, seed, samples=1_000_000):
    """Ring replay on every element; the fp64 weighted mean (O6) on `samples` seeded positions (C5's rule
    for buffers above 64 MiB: the fp64 arrays of P × L would not fit the host comfortably)."""
    host, dev = _inputs(P, L, "f32", seed=seed)
    pr.weighted_allreduce_local(comms, dev, n)
    torch.cuda.synchronize()
    assert all(c.status() == 0 for c in comms)
    emu = W.ring_emulate(host, n, "f32")
    for r in range(P):
        assert np.array_equal(dev[r].cpu().numpy(), emu), f"rank {r} differs from ring replay"
    pos = np.sort(np.random.Generator(np.random.PCG64(seed)).choice(L, size=min(samples, L), replace=False))
    ref, den = W.weighted_average(W.as_f64(host[:, pos], "f32"), n)
    err, zb = W.error_metric(emu[pos].astype(np.float64), ref, den)
    assert zb == 0 and err <= TOL["f32"], err


@pytest.mark.parametrize("model", ["resnet18", "vgg16"])
@pytest.mark.parametrize("P", [2, 4, 8])
def test_cross_gpu_default_config_ring(P, model):
    _check_sampled(P, SIZES[model], SKEW[-P:], group(P, **(CROSS8 if P == 8 else CROSS)), seed=P + len(model))


@pytest.mark.parametrize("model", ["resnet18", "vgg16"])
@pytest.mark.parametrize("P", [2, 4, 8])
def test_cross_gpu_default_config_fused(P, model):
    """a6-a9 in one kernel under the cross-GPU configuration: θ' bit-identical to ring + K7, and within K7's
    two roundings of the oracle (ring replay for ḡ, fp64 SGD) on sampled positions."""
    from oracle import linmodel as LM

    L = SIZES[model]
    n = SKEW[-P:]
    g, theta0, out = _fused_case(P, L, n, group(P, **(CROSS8 if P == 8 else CROSS)), seed=100 + P)
    gbar = W.ring_emulate(g, n, "f32")
    pos = np.random.Generator(np.random.PCG64(P)).choice(L, size=min(1_000_000, L), replace=False)
    gb, t0 = gbar[pos].astype(np.float64), theta0[pos].astype(np.float64)
    ref = LM.sgd_step(t0, gb, float(np.float32(1e-2)), float(np.float32(1e-4)))
    bound = 2.0 ** -24 * (np.abs(ref) + np.float32(1e-2) * np.abs(gb + np.float32(1e-4) * t0)) * 1.01
    assert np.all(np.abs(out[pos].astype(np.float64) - ref) <= bound + 1e-45)


CROSS_PULL = dict(CROSS, algo=pr.ALGO_TWO_SHOT_PULL)
CROSS_PULL8 = dict(CROSS_PULL, threads=256)      # 8 × 32 CTAs co-resident: two 256-thread CTAs per SM


@pytest.mark.parametrize("model", ["resnet18", "vgg16"])
@pytest.mark.parametrize("P", [2, 4, 8])
def test_cross_gpu_default_config_pull(P, model):
    """The pull two-shot under the cross-GPU configuration (32 channels, `.sys` scope): the ring replay on
    every element, the fp64 mean on sampled positions; and its fused a6-a9 form = ring + K7 bit for bit."""
    cfg = CROSS_PULL8 if P == 8 else CROSS_PULL
    _check_sampled(P, SIZES[model], SKEW[-P:], group(P, **cfg), seed=P + len(model) + 50)
    if model == "resnet18":
        _fused_case(P, SIZES[model], SKEW[-P:], group(P, **cfg), seed=150 + P)


def test_auto_with_unregistered_or_staged_buffers_skips_two_shot():
    """AUTO at a two-shot size (1-4 MiB) on a group whose buffers cannot take the direct
    all-gather (force_staged) must take the staged ring, not latch PR_ERR_INVALID in the two-shot."""
    P = 4
    comms = group(P, algo=pr.ALGO_AUTO, force_staged=True)
    for L in (300_001, 1 << 20):
        _check(P, L, "f32", [1, 2, 3, 4], comms, seed=L)
    assert all(c.status() == 0 for c in comms)


# ---- the TMA bulk-store data path (PR_COMM_FLAG_BULK_STORE) ------------------------------------------------
@pytest.mark.parametrize("dtype", ["f32", "bf16"])
@pytest.mark.parametrize("P", [2, 3, 4, 8])
def test_bulk_store_ring_bit_identical_to_ring_replay(P, dtype):
    """Results written back to shared memory and pushed by one thread with cp.async.bulk stores: the same
    bits as the ring replay (direct and staged all-gather, .gpu and .sys scope, ragged tails)."""
    for cfg in (dict(bulk_store=True), dict(bulk_store=True, force_staged=True),
                dict(bulk_store=True, sys_scope=True, channels=4, slot_bytes=4096, tile_bytes=1024, stages=3)):
        comms = group(P, **cfg)
        rng = np.random.Generator(np.random.PCG64(77 + P))
        for L in (1, 7, P + 1, 1000, 4099, 65_537, 2 ** 20 + 3):
            n = [int(x) * 16 for x in rng.integers(0, 5, P)]
            if sum(n) == 0:
                n[0] = 16
            _check(P, L, dtype, n, comms, kind="mixed" if L % 2 else "gaussian", seed=L + P)


@pytest.mark.parametrize("P", [2, 4, 8])
def test_bulk_store_fused_and_full_sizes(P):
    comms = group(P, bulk_store=True)
    for L in (7, 4099, 300_001):
        _fused_case(P, L, [1 + (r % 3) for r in range(P)], comms, seed=L + 31)
    _check(P, 11_689_512, "f32", SKEW[-P:], comms, seed=5)
    comms = group(P, **(dict(CROSS8) if P == 8 else dict(CROSS)), bulk_store=True)
    _check_sampled(P, 11_689_512, SKEW[-P:], comms, seed=P + 11)
    _fused_case(P, 11_689_512, SKEW[-P:], comms, seed=P + 13)


def test_bulk_store_randomized_configs_and_graph_replay():
    rng = np.random.Generator(np.random.PCG64(4242))
    for case in range(30):
        P = int(rng.choice([2, 3, 4, 5, 8]))
        cfg = dict(channels=int(rng.integers(1, 9)), slots=int(rng.choice([2, 4, 8])),
                   slot_bytes=int(rng.choice([256, 4096, 65536, 262144])), stages=int(rng.integers(2, 7)),
                   tile_bytes=int(rng.choice([256, 1024, 4096, 16384])), threads=int(rng.choice([64, 256, 512])),
                   sys_scope=bool(rng.integers(0, 2)), force_staged=bool(rng.integers(0, 2)), bulk_store=True)
        comms = pr.comm_init_local(P, 0, pr.comm_config(watchdog_ns=5_000_000_000, **cfg))
        try:
            for _ in range(2):
                L = int(rng.choice([1, 3, 17, 1000, 4097, 65_537, 300_001]))
                n = [int(x) for x in rng.integers(0, 5, P)]
                if sum(n) == 0:
                    n[0] = 1
                _check(P, L, "f32" if rng.integers(0, 2) else "bf16", n, comms, seed=case * 11 + L)
            if not cfg["force_staged"]:
                _fused_case(P, int(rng.choice([7, 5000, 200_003])), [1 + (r % 3) for r in range(P)], comms,
                            seed=case + 700)
        finally:
            for c in comms:
                c.destroy()
    # graph replay: counters carried on the device across replays
    P, L = 4, 100_003
    comms = group(P, bulk_store=True)
    host, dev = _inputs(P, L, "f32", seed=3)
    n = [3, 1, 2, 5]
    emu = W.ring_emulate(host, n, "f32")
    s = torch.cuda.Stream()
    gr = torch.cuda.CUDAGraph()
    with torch.cuda.stream(s):
        pr.weighted_allreduce_local(comms, dev, n, stream=s)
        torch.cuda.synchronize()
        with torch.cuda.graph(gr, stream=s):
            pr.weighted_allreduce_local(comms, dev, n, stream=s)
    for _ in range(3):
        for r in range(P):
            dev[r].copy_(torch.from_numpy(host[r]))
        gr.replay()
        torch.cuda.synchronize()
        assert all(np.array_equal(d.cpu().numpy(), emu) for d in dev)


# ---- NVLS (N2): the multicast kernel's logic through its software emulation on one GPU ---------------------
@pytest.mark.parametrize("P", [2, 3, 4, 8])
def test_nvls_kernel_emulated_within_tolerance(P):
    """PR_ALGO_NVLS in a local group runs nvls_kernel<EMU>: the same phases (weights applied in place, a
    per-channel cross-rank barrier, chunk-owner reduce + store to every rank, a second barrier), with the
    switch's ld_reduce / multicast store replaced by their definition over the ranks' buffers — one GPU has
    no multicast object.  Switch order is unspecified (DESIGN.md §3 #48): tolerance vs the fp64 mean, all
    ranks identical, a zero-sample rank holding NaN contributes nothing, back-to-back calls and bf16 (which
    takes the ring) included."""
    comms = group(P, algo=pr.ALGO_NVLS, channels=4)
    rng = np.random.Generator(np.random.PCG64(500 + P))
    for L in (1, 7, P + 1, 1000, 4099, 2 ** 20 + 3):
        n = [int(x) * 16 for x in rng.integers(1, 6, P)]
        if L % 2:
            n[int(rng.integers(0, P))] = 0
        host, dev = _inputs(P, L, "f32", kind="mixed" if L % 2 else "gaussian", seed=L + P)
        for r in range(P):
            if n[r] == 0:
                dev[r].fill_(float("nan"))
        pr.weighted_allreduce_local(comms, dev, n)
        pr.weighted_allreduce_local(comms, [d.clone() for d in dev], n)      # back to back (seq advances)
        torch.cuda.synchronize()
        assert all(c.status() == 0 for c in comms)
        outs = [d.cpu().numpy() for d in dev]
        assert all(np.array_equal(outs[0], o) for o in outs[1:])
        h64 = W.as_f64(host, "f32")
        ref, den = W.weighted_average(h64, n)
        err, zb = W.error_metric(outs[0].astype(np.float64), ref, den)
        assert zb == 0 and err <= TOL["f32"], (L, err)
    _check(P, 4099, "bf16", [1 + r for r in range(P)], comms, seed=9)         # bf16: the ring's bits


@pytest.mark.parametrize("P", [2, 3, 8])
def test_l2_prefetch_ring_bit_identical_to_ring_replay(P):
    """PR_COMM_FLAG_L2_PREFETCH only adds cp.async.bulk.prefetch.L2 hints: same bits as the ring replay, fp32
    and bf16, direct and staged."""
    for staged in (False, True):
        comms = group(P, l2_prefetch=True, force_staged=staged, channels=4, slot_bytes=1 << 16)
        for L in (1, 7, 4099, 2 ** 20 + 3):
            for dtype in ("f32", "bf16"):
                _check(P, L, dtype, [16 * (r + 1) for r in range(P)], comms, kind="mixed", seed=L + P)
