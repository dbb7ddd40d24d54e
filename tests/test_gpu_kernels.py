"""GPU parity: K1 sharder, K2 gather, K4 spin, called through the C ABI, against the CPU oracle.

Bar: bit-exact for indices and gathered bytes (integer / byte work, and the affine
conversion whose definition fixes every rounding).
"""

import numpy as np
import pytest
import torch

import synth
from oracle import allocation as A
from oracle import gather as OG
from oracle import permutation as PM

pytestmark = pytest.mark.gpu

pr = pytest.importorskip("paper_2111_08272_b200")


@pytest.fixture(scope="module", autouse=True)
def _cuda():
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    torch.cuda.init()


def _dev(x):
    return torch.from_numpy(np.ascontiguousarray(x)).cuda()


# ---------------------------------------------------------------- K1 ----------------------------

def test_philox_device_matches_kat_oracle_and_curand():
    rng = np.random.Generator(np.random.PCG64(1))
    ctr = rng.integers(0, 2 ** 32, (4096, 4), dtype=np.uint64).astype(np.uint32)
    ctr[0] = 0
    ctr[1] = 0xFFFFFFFF
    ctr[2] = [0x243F6A88, 0x85A308D3, 0x13198A2E, 0x03707344]
    for key in (0, 0xFFFFFFFFFFFFFFFF, 0x299F31D0A4093822, 1234567):
        d = _dev(ctr.view(np.int32))
        mine = torch.empty(ctr.size, dtype=torch.int32, device="cuda")
        cur = torch.empty_like(mine)
        pr.test_philox(d, key, False, mine)
        pr.test_philox(d, key, True, cur)
        torch.cuda.synchronize()
        m = mine.cpu().numpy().view(np.uint32).reshape(-1, 4)
        c = cur.cpu().numpy().view(np.uint32).reshape(-1, 4)
        assert np.array_equal(m, c)                           # library routine (cuRAND)
        o = np.stack(PM.philox4x32_10(tuple(ctr[:, j] for j in range(4)), (key & 0xFFFFFFFF, key >> 32)), 1)
        assert np.array_equal(m, o)                           # oracle
    # published KAT through the device function
    d = _dev(np.array([[0, 0, 0, 0]], dtype=np.uint32).view(np.int32))
    out = torch.empty(4, dtype=torch.int32, device="cuda")
    pr.test_philox(d, 0, False, out)
    assert out.cpu().numpy().view(np.uint32).tolist() == [0x6627E8D5, 0xE169C58D, 0xBC57AC4C, 0x9B00DBD8]


@pytest.mark.parametrize("N", [1, 2, 3, 10, 1000, 50000, 1281167, 2 ** 24])
def test_permute_bit_exact(N):
    rng = np.random.Generator(np.random.PCG64(N))
    for _ in range(3 if N < 2 ** 20 else 1):
        seed = int(rng.integers(0, 2 ** 63)) * 2 + int(rng.integers(0, 2))
        ep = int(rng.integers(0, 2 ** 40))
        out = torch.empty(N, dtype=torch.int64, device="cuda")
        pr.permute(N, seed, ep, 0, N, out)
        got = out.cpu().numpy()
        if N <= 2 ** 21:
            assert np.array_equal(got, PM.permute(np.arange(N), N, seed, ep))
        else:   # full size: sampled positions one by one + the bijection property
            pos = rng.integers(0, N, 20000)
            assert np.array_equal(got[pos], PM.permute(pos, N, seed, ep))
        assert np.array_equal(np.sort(got), np.arange(N))


def test_permute_subrange_and_edges():
    N = 12345
    full = torch.empty(N, dtype=torch.int64, device="cuda")
    pr.permute(N, 9, 4, 0, N, full)
    part = torch.empty(1000, dtype=torch.int64, device="cuda")
    pr.permute(N, 9, 4, 11345, 1000, part)
    assert torch.equal(full[11345:], part)
    pr.permute(N, 9, 4, 5, 0, part)          # empty range: no-op
    with pytest.raises(pr.PropringError):
        pr.permute(N, 9, 4, 12000, 1000, part)


def test_permute_warp_range_boundaries():
    """K1's lane-refill walk hands each warp a contiguous range of ceil(count / warps) outputs; counts
    around 32 · k (partial last warp, one lane, ranges shorter than a warp) and offset ranges must give
    the oracle's π element for element, including the largest grid (148 · 32 warps) with a ragged tail."""
    rng = np.random.Generator(np.random.PCG64(77))
    for N in (5, 33, 257, 4099, 65537):
        full = PM.permute(np.arange(N), N, 31, 2)
        for count in sorted({1, 2, 31, 32, 33, 63, 64, 65, N // 2, N - 1, N} - {0}):
            if count > N:
                continue
            begin = int(rng.integers(0, N - count + 1))
            out = torch.full((count + 5,), -7, dtype=torch.int64, device="cuda")
            pr.permute(N, 31, 2, begin, count, out)
            got = out.cpu().numpy()
            assert np.array_equal(got[:count], full[begin:begin + count]), (N, begin, count)
            assert (got[count:] == -7).all()                  # nothing written past count
    for N in (148 * 32 * 7 + 13,                               # every refill warp 7 outputs + a ragged tail
              148 * 4 * 256 * 3 + 77):                         # ranges of 24 per lane (the full grid) + a ragged tail
        out = torch.empty(N, dtype=torch.int64, device="cuda")
        pr.permute(N, 5, 9, 0, N, out)
        assert np.array_equal(out.cpu().numpy(), PM.permute(np.arange(N), N, 5, 9))


@pytest.mark.parametrize("N,ratios,C,g", [(1000, [1, 3], 4, 25), (50000, [1, 2], 3, 128),
                                          (51200, [1, 1, 1, 1], 64, 16), (50000, [1, 1, 1, 1, 2, 2, 4, 4], 64, 16),
                                          (1281167, [3, 1, 4, 1, 5], 14, 2)])
def test_shard_indices_bit_exact(N, ratios, C, g):
    a = pr.alloc_init(N, ratios, C=C, g=g)
    o = A.alloc_init(N, ratios, C=C, g=g)
    for epoch in (0, 1, 7):
        seen = []
        for r in range(len(ratios)):
            out = torch.empty(o.len[r], dtype=torch.int64, device="cuda")
            pr.shard_indices(a, r, epoch, 1234, out)
            got = out.cpu().numpy()
            assert np.array_equal(got, PM.shard_indices(N, o.off[r], o.len[r], 1234, epoch))
            seen.append(got)
        allv = np.concatenate(seen)
        assert np.array_equal(np.sort(allv), np.arange(N))
    small = torch.empty(o.len[0] - 1, dtype=torch.int64, device="cuda")
    with pytest.raises(pr.PropringError) as e:
        pr.shard_indices(a, 0, 0, 1, small)
    assert e.value.code == pr.PR_ERR_CAPACITY


@pytest.mark.parametrize("N,ratios,C,g", [(1000, [1, 3], 4, 25), (50000, [1, 1, 1, 1, 2, 2, 4, 4], 64, 16),
                                          (1281167, [3, 1, 4, 1, 5], 14, 2)])
def test_shard_steps_bit_exact(N, ratios, C, g):
    a = pr.alloc_init(N, ratios, C=C, g=g)
    v = a.view()
    B, S = g * sum(v["w"]), v["S"]
    for step0, nsteps in ((0, 1), (1, 3), (S - 2, 2), (0, S)):
        if nsteps * B > 4_000_000:
            continue
        seen = []
        for r in range(len(ratios)):
            n_r, o_r = v["n"][r], g * sum(v["w"][:r])
            out = torch.empty(nsteps * n_r + 3, dtype=torch.int64, device="cuda")
            pr.shard_steps(a, r, 5, 77, step0, nsteps, out)
            got = out[:nsteps * n_r].cpu().numpy()
            assert np.array_equal(got, PM.shard_steps(N, B, o_r, n_r, 77, 5, step0, nsteps))
            seen.append(got)
        assert np.unique(np.concatenate(seen)).size == nsteps * B
    out = torch.empty(v["n"][0], dtype=torch.int64, device="cuda")
    for bad in ((S, 1), (-1, 1), (S - 1, 2)):
        with pytest.raises(pr.PropringError) as e:
            pr.shard_steps(a, 0, 0, 1, bad[0], bad[1], out)
        assert e.value.code == pr.PR_ERR_INVALID
    with pytest.raises(pr.PropringError) as e:
        pr.shard_steps(a, 0, 0, 1, 0, 2, out)
    assert e.value.code == pr.PR_ERR_CAPACITY


# ---------------------------------------------------------------- K2 ----------------------------

MEAN = [123.675, 116.28, 103.53]
STD = [58.395, 57.12, 57.375]


@pytest.mark.parametrize("row_bytes,plane", [(16, 16), (48, 16), (48, 8), (3072, 1024), (150528, 50176)])
@pytest.mark.parametrize("n", [0, 1, 31, 32, 33, 4096])
def test_gather_bit_exact(row_bytes, plane, n):
    if row_bytes == 150528 and n == 4096:
        n = 300
    nsrc = max(64, n // 2)
    channels = row_bytes // plane
    rng = np.random.Generator(np.random.PCG64(row_bytes + n))
    X = rng.integers(0, 256, (nsrc, row_bytes), dtype=np.uint8)
    Y = rng.integers(0, 1000, nsrc, dtype=np.int64)
    idx = rng.integers(0, nsrc, n, dtype=np.int64)
    scale = np.array([1.0 / STD[c % 3] for c in range(channels)], dtype=np.float32)
    shift = np.array([MEAN[c % 3] for c in range(channels)], dtype=np.float32)
    dX, dY, didx = _dev(X), _dev(Y), _dev(idx)
    for op, impl in [(o, i) for o in (pr.GATHER_COPY, pr.GATHER_U8_TO_F32_AFFINE, pr.GATHER_U8_TO_BF16_AFFINE)
                     for i in (pr.GATHER_IMPL_LSU, pr.GATHER_IMPL_TMA)]:
        width = {0: 1, 1: 4, 2: 2}[op]
        out = torch.full((max(n, 1) * row_bytes * width,), 0x5A, dtype=torch.uint8, device="cuda")
        lab = torch.full((max(n, 1),), -7, dtype=torch.int64, device="cuda")
        gop = pr.make_gather_op(op, scale, shift, plane, impl=impl)
        pr.gather_rows(dX, nsrc, row_bytes, didx, n, out, gop, dY, lab)
        torch.cuda.synchronize()
        if n == 0:
            assert int((out != 0x5A).sum()) == 0
            continue
        ref, rlab = OG.gather_rows(X, idx, op, scale, shift, plane, Y=Y)
        assert np.array_equal(out.cpu().numpy(), np.ascontiguousarray(ref).view(np.uint8).reshape(-1))
        assert np.array_equal(lab.cpu().numpy(), rlab)


@pytest.mark.parametrize("channels,plane", [(1, 32), (2, 48), (3, 16), (3, 1024), (4, 64), (3, 50176)])
@pytest.mark.parametrize("n", [1, 9, 33, 700])
def test_gather_hwc_bit_exact(channels, plane, n):
    """Channels-last output (PR_GATHER_LAYOUT_HWC): whole-row units and per-plane pixel-block units."""
    if plane == 50176 and n == 700:
        n = 40
    row_bytes = channels * plane
    nsrc = max(64, n)
    rng = np.random.Generator(np.random.PCG64(channels * 100000 + plane + n))
    X = rng.integers(0, 256, (nsrc, row_bytes), dtype=np.uint8)
    idx = rng.integers(0, nsrc, n, dtype=np.int64)
    scale = np.array([1.0 / STD[c % 3] for c in range(channels)], dtype=np.float32)
    shift = np.array([MEAN[c % 3] for c in range(channels)], dtype=np.float32)
    dX, didx = _dev(X), _dev(idx)
    Y = rng.integers(0, 1000, nsrc, dtype=np.int64)
    dY = _dev(Y)
    for op, width, impl in [(o, w, i) for o, w in ((pr.GATHER_U8_TO_BF16_AFFINE, 2), (pr.GATHER_U8_TO_F32_AFFINE, 4))
                            for i in (pr.GATHER_IMPL_LSU, pr.GATHER_IMPL_TMA, pr.GATHER_IMPL_BULK)]:
        out = torch.full((n * row_bytes * width + 64,), 0x5A, dtype=torch.uint8, device="cuda")
        lab = torch.full((n,), -7, dtype=torch.int64, device="cuda")
        gop = pr.make_gather_op(op, scale, shift, plane, impl=impl, layout=pr.GATHER_LAYOUT_HWC)
        pr.gather_rows(dX, nsrc, row_bytes, didx, n, out, gop, dY, lab)
        ref, rlab = OG.gather_rows(X, idx, op, scale, shift, plane, layout="hwc", Y=Y)
        got = out.cpu().numpy()
        assert np.array_equal(got[:n * row_bytes * width], np.ascontiguousarray(ref).view(np.uint8).reshape(-1))
        assert (got[n * row_bytes * width:] == 0x5A).all()          # nothing written past the output
        assert np.array_equal(lab.cpu().numpy(), rlab)


@pytest.mark.parametrize("channels,plane,n", [(3, 1024, 4097), (3, 1360, 333), (1, 4096, 3), (4, 16, 1),
                                              (3, 50176, 7), (2, 8192, 5)])
def test_gather_hwc_bulk_unit_boundaries(channels, plane, n):
    """The bulk-store kernel's units are 4096 consecutive OUTPUT pixels: units that span several rows, start
    mid-row, end mid-row, a ragged last unit, and rows longer than a unit — bit-exact against the oracle, with
    the bytes past the output untouched."""
    row_bytes = channels * plane
    nsrc = max(16, n)
    rng = np.random.Generator(np.random.PCG64(7 * plane + n))
    X = rng.integers(0, 256, (nsrc, row_bytes), dtype=np.uint8)
    idx = rng.integers(0, nsrc, n, dtype=np.int64)
    scale = np.array([1.0 / STD[c % 3] for c in range(channels)], dtype=np.float32)
    shift = np.array([MEAN[c % 3] for c in range(channels)], dtype=np.float32)
    dX, didx = _dev(X), _dev(idx)
    for op, width in ((pr.GATHER_U8_TO_BF16_AFFINE, 2), (pr.GATHER_U8_TO_F32_AFFINE, 4)):
        out = torch.full((n * row_bytes * width + 4096,), 0x5A, dtype=torch.uint8, device="cuda")
        gop = pr.make_gather_op(op, scale, shift, plane, impl=pr.GATHER_IMPL_BULK, layout=pr.GATHER_LAYOUT_HWC)
        pr.gather_rows(dX, nsrc, row_bytes, didx, n, out, gop)
        ref, _ = OG.gather_rows(X, idx, op, scale, shift, plane, layout="hwc")
        got = out.cpu().numpy()
        assert np.array_equal(got[:n * row_bytes * width], np.ascontiguousarray(ref).view(np.uint8).reshape(-1))
        assert (got[n * row_bytes * width:] == 0x5A).all()


def test_gather_bulk_rejects_chw():
    X = torch.zeros((4, 3 * 16), dtype=torch.uint8, device="cuda")
    idx = torch.zeros(2, dtype=torch.int64, device="cuda")
    out = torch.empty((2, 48), dtype=torch.bfloat16, device="cuda")
    with pytest.raises(pr.PropringError):
        pr.gather_rows(X, 4, 48, idx, 2, out, pr.make_gather_op(pr.GATHER_U8_TO_BF16_AFFINE, [1.0] * 3, [0.0] * 3,
                                                                16, impl=pr.GATHER_IMPL_BULK))


def test_gather_hwc_rejects_unsupported():
    X = torch.zeros((4, 5 * 16), dtype=torch.uint8, device="cuda")
    idx = torch.zeros(2, dtype=torch.int64, device="cuda")
    out = torch.empty((2, 80), dtype=torch.bfloat16, device="cuda")
    with pytest.raises(pr.PropringError):      # 5 channels > 4
        pr.gather_rows(X, 4, 80, idx, 2, out, pr.make_gather_op(pr.GATHER_U8_TO_BF16_AFFINE, [1.0] * 5, [0.0] * 5,
                                                                16, layout=pr.GATHER_LAYOUT_HWC))


def test_gather_step_slices_of_a_shard_and_alignment_errors():
    X = synth.images_u8(2000, seed=0).reshape(2000, -1)
    a = pr.alloc_init(2000, [1, 2], C=3, g=16)
    v = a.view()
    idx = torch.empty(v["len"][1], dtype=torch.int64, device="cuda")
    pr.shard_indices(a, 1, 3, 99, idx)
    dX = _dev(X)
    n = v["n"][1]
    out = torch.empty((n, 3072), dtype=torch.bfloat16, device="cuda")
    scale = [1 / s for s in STD]
    gop = pr.make_gather_op(pr.GATHER_U8_TO_BF16_AFFINE, scale, MEAN, 1024)
    for s in range(v["S"]):
        pr.gather_rows(dX, 2000, 3072, idx[s * n:], n, out, gop)
        ref, _ = OG.step_gather(X, idx.cpu().numpy(), s, n, op=OG.U8_TO_BF16_AFFINE,
                                scale=np.float32(scale), shift=np.float32(MEAN), plane=1024)
        assert np.array_equal(out.view(torch.int16).cpu().numpy().view(np.uint16), ref)
    with pytest.raises(pr.PropringError) as e:
        pr.gather_rows(dX, 2000, 3000, idx, 1, out)
    assert e.value.code == pr.PR_ERR_ALIGN


def test_gather_epoch_size_tma_vs_oracle():
    """The bench's per-epoch launch (48 steps x 1024 CIFAR rows, AUTO -> TMA): bit-exact on sampled rows."""
    X = synth.images_u8(50000, seed=0).reshape(50000, -1)
    a = pr.alloc_init(50000, [1], C=64, g=16)
    idx = torch.empty(50000, dtype=torch.int64, device="cuda")
    pr.shard_indices(a, 0, 5, 1234, idx)
    rows = 48 * 1024
    out = torch.empty((rows, 3072), dtype=torch.bfloat16, device="cuda")
    scale = [1 / s for s in STD]
    pr.gather_rows(_dev(X), 50000, 3072, idx, rows, out, pr.make_gather_op(pr.GATHER_U8_TO_BF16_AFFINE, scale, MEAN, 1024))
    pick = np.random.Generator(np.random.PCG64(3)).integers(0, rows, 500)
    ref, _ = OG.gather_rows(X, idx.cpu().numpy()[pick], OG.U8_TO_BF16_AFFINE, np.float32(scale), np.float32(MEAN), 1024)
    got = out.view(torch.int16).cpu().numpy().view(np.uint16)[pick]
    assert np.array_equal(got, ref)


def test_gather_from_mapped_host_memory():
    """The e2e path: rows read straight from pinned host memory over PCIe."""
    X = synth.images_u8(512, seed=5).reshape(512, -1)
    hX = torch.from_numpy(X).pin_memory()
    idx = torch.randint(0, 512, (100,), dtype=torch.int64).cuda()
    out = torch.empty((100, 3072), dtype=torch.uint8, device="cuda")
    ptr = hX.data_ptr()   # UVA: pinned host memory is addressable from the device
    pr.gather_rows(ptr, 512, 3072, idx, 100, out)
    assert torch.equal(out.cpu(), hX[idx.cpu()])
    # the trainer's e2e form: channels-last bf16 from host memory (AUTO -> LSU kernel), 4096 rows
    big = torch.from_numpy(synth.images_u8(4096, seed=6).reshape(4096, -1)).pin_memory()
    idx2 = torch.randint(0, 4096, (4096,), dtype=torch.int64)
    ob = torch.empty((4096, 3072), dtype=torch.bfloat16, device="cuda")
    scale = [1 / s for s in STD]
    pr.gather_rows(big.data_ptr(), 4096, 3072, idx2.cuda(), 4096, ob,
                   pr.make_gather_op(pr.GATHER_U8_TO_BF16_AFFINE, scale, MEAN, 1024, layout=pr.GATHER_LAYOUT_HWC))
    ref, _ = OG.gather_rows(big.numpy(), idx2.numpy(), OG.U8_TO_BF16_AFFINE, np.float32(scale), np.float32(MEAN), 1024,
                            layout="hwc")
    assert np.array_equal(ob.view(torch.int16).cpu().numpy().view(np.uint16), ref)


# ---------------------------------------------------------------- K4 ----------------------------

def test_spin_duration():
    pr.spin(1000)                     # first launch pays the lazy module load
    torch.cuda.synchronize()
    for ns in (50_000, 1_000_000):
        s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        s.record()
        pr.spin(ns)
        e.record()
        e.synchronize()
        ms = s.elapsed_time(e)
        # %globaltimer advances in coarse ticks (tens of us on B200): bound the absolute overshoot;
        # emulated slowdowns are ms-scale ((σ−1)·c0·n_r), where this is < 5% (the 1 ms case)
        assert ns / 1e6 * 0.99 <= ms <= ns / 1e6 * 1.02 + 0.05


def test_stamp_ring_orders_and_wraps():
    ring = torch.zeros(1 + 4, dtype=torch.int64, device="cuda")
    for _ in range(6):
        pr.stamp(ring)
        pr.spin(20_000)
    torch.cuda.synchronize()
    r = ring.cpu().tolist()
    assert r[0] == 6
    s2, s3, s4, s5 = r[3], r[4], r[1], r[2]          # stamps 4 and 5 wrapped onto slots 0 and 1
    assert s3 - s2 >= 20_000 and s4 - s3 >= 20_000 and s5 - s4 >= 20_000
    with pytest.raises(pr.PropringError):
        pr.stamp(torch.zeros(1, dtype=torch.int64, device="cuda"))


# ---- a9: fused SGD update (Eq. 1, wd P:235) ----------------------------------------------------------

def _sgd_ref(theta, g, lr, wd):
    """Oracle O7's sgd_step in fp64 on the fp32 inputs with lr, wd rounded to fp32 (the kernel's definition)."""
    from oracle import linmodel as LM

    return LM.sgd_step(theta.astype(np.float64), g.astype(np.float64), float(np.float32(lr)), float(np.float32(wd)))


@pytest.mark.parametrize("n", [1, 3, 4, 5, 1000, 4099, 11_689_512])
def test_sgd_update_within_one_rounding_of_oracle(n):
    rng = np.random.Generator(np.random.PCG64(n))
    theta = (rng.standard_normal(n) * np.exp(rng.standard_normal(n))).astype(np.float32)
    g = (rng.standard_normal(n) * np.exp(2 * rng.standard_normal(n))).astype(np.float32)
    lr, wd = 1e-2, 1e-4
    dt, dg = torch.from_numpy(theta).cuda(), torch.from_numpy(g).cuda()
    pr.sgd_update(dt, dg, lr, wd, zero_grad=True)
    torch.cuda.synchronize()
    out = dt.cpu().numpy().astype(np.float64)
    ref = _sgd_ref(theta, g, lr, wd)
    # two roundings: |err| <= u·|θ'| + lr·u·|g + wd·θ| (u = 2^-24), plus slack for the fp32 lr/wd
    bound = 2.0 ** -24 * (np.abs(ref) + np.float32(lr) * np.abs(g.astype(np.float64) + np.float32(wd) * theta)) * 1.01
    assert np.all(np.abs(out - ref) <= bound + 1e-45)
    assert torch.count_nonzero(dg) == 0
    # library routine: torch.optim.SGD on the same values, within the same bound
    p = torch.nn.Parameter(torch.from_numpy(theta).cuda())
    p.grad = torch.from_numpy(g).cuda()
    torch.optim.SGD([p], lr=lr, weight_decay=wd).step()
    assert np.all(np.abs(p.detach().cpu().numpy().astype(np.float64) - out) <= 2 * bound + 1e-45)


def test_sgd_update_keep_grad_and_errors():
    theta = torch.randn(1001, device="cuda")
    g = torch.randn(1001, device="cuda")
    g0 = g.clone()
    pr.sgd_update(theta, g, 0.1, 0.0, zero_grad=False)
    assert torch.equal(g, g0)
    pr.sgd_update(theta[:0], g[:0], 0.1)                  # n = 0: no launch
    with pytest.raises(pr.PropringError) as e:
        pr.sgd_update(theta[1:], g[1:], 0.1)             # 4-byte offset: not 16-byte aligned
    assert e.value.code == pr.PR_ERR_ALIGN
    with pytest.raises(ValueError):
        pr.sgd_update(theta.double(), g.double(), 0.1)
