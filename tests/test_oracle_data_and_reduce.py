"""Pins for oracle O5 (gather), O6 (weighted average + ring emulation), O7 (linear model), O9 (model)."""

import numpy as np
import pytest
import torch

import synth
from oracle import allocation as A
from oracle import epoch_model as EM
from oracle import gather as G
from oracle import linmodel as LM
from oracle import wavg as W


# ---------------------------------------------------------------- O5 ----------------------------

def test_gather_copy_is_bit_copy():
    X = synth.images_u8(50, seed=3).reshape(50, -1)
    idx = np.array([4, 4, 0, 49, 17])
    out, lab = G.gather_rows(X, idx, G.COPY, Y=np.arange(50) * 10)
    assert out.tobytes() == b"".join(X[i].tobytes() for i in idx)
    assert lab.tolist() == [40, 40, 0, 490, 170]


def test_gather_affine_matches_exact_rounding():
    X = synth.images_u8(20, seed=4)
    idx = np.arange(20)[::-1]
    scale = np.array([1 / 58.395, 1 / 57.12, 1 / 57.375], dtype=np.float32)
    shift = np.array([123.675, 116.28, 103.53], dtype=np.float32)
    out, _ = G.gather_rows(X, idx, G.U8_TO_F32_AFFINE, scale, shift, plane=32 * 32)
    rows = X.reshape(20, -1)[idx].astype(np.float64)
    ch = np.arange(rows.shape[1]) // 1024
    d = (rows - shift.astype(np.float64)[ch]).astype(np.float32).astype(np.float64)   # first rounding
    exact = d * scale.astype(np.float64)[ch]
    # second rounding: within half an ulp of fp32
    assert np.all(np.abs(out.astype(np.float64) - exact) <= 0.5 * np.spacing(np.abs(out)).astype(np.float64))
    bf, _ = G.gather_rows(X, idx, G.U8_TO_BF16_AFFINE, scale, shift, plane=1024)
    ref = torch.from_numpy(out).to(torch.bfloat16).view(torch.int16).numpy().view(np.uint16)  # library RNE
    assert np.array_equal(bf, ref)


def test_gather_hwc_layout_is_channels_last_permute():
    """layout="hwc" = the CHW result permuted to channels-last (torch permute/contiguous: library routine)."""
    X = synth.images_u8(7, seed=6)
    idx = np.array([3, 0, 6, 6])
    scale = np.array([0.5, 0.25, 0.125], dtype=np.float32)
    shift = np.array([1.0, 2.0, 3.0], dtype=np.float32)
    chw, _ = G.gather_rows(X, idx, G.U8_TO_F32_AFFINE, scale, shift, plane=1024)
    hwc, _ = G.gather_rows(X, idx, G.U8_TO_F32_AFFINE, scale, shift, plane=1024, layout="hwc")
    ref = torch.from_numpy(chw).view(4, 3, 32, 32).permute(0, 2, 3, 1).contiguous().view(4, -1).numpy()
    assert np.array_equal(hwc, ref)
    assert hwc[1, 5 * 3 + 2] == chw[1, 2 * 1024 + 5]       # element (c=2, p=5) of row 1


def test_bf16_rne_against_torch_random_bits():
    rng = np.random.Generator(np.random.PCG64(8))
    bits = rng.integers(0, 2 ** 32, 200000, dtype=np.uint64).astype(np.uint32)
    x = bits.view(np.float32)
    x = x[np.isfinite(x)]
    mine = G.f32_to_bf16_bits(x)
    ref = torch.from_numpy(x.copy()).to(torch.bfloat16).view(torch.int16).numpy().view(np.uint16)
    assert np.array_equal(mine, ref)


# ---------------------------------------------------------------- O6 ----------------------------

def test_wavg_equal_weights_is_mean_and_identity():
    g = synth.gradients(4, 1000).astype(np.float64)
    ref, den = W.weighted_average(g, [7, 7, 7, 7])
    assert np.allclose(ref, g.mean(axis=0), rtol=1e-14, atol=1e-15)
    ref1, _ = W.weighted_average(g[:1], [5])
    assert np.array_equal(ref1, g[0])


def test_wavg_disjoint_supports():
    g = np.array([[1.0, 0, 0], [0, 2.0, 0], [0, 0, 3.0]])
    ref, _ = W.weighted_average(g, [1, 1, 1])
    assert np.allclose(ref, [1 / 3, 2 / 3, 1.0], rtol=1e-15)       # S:199 analogue
    ref, _ = W.weighted_average(g, [1, 0, 3])                      # n=0 rank skipped
    assert np.allclose(ref, [0.25, 0.0, 2.25])   # 1·1/4, 0, 3·3/4


def test_wavg_matches_full_batch_sum():
    """Σ_r (n_r/Σn)·mean_r = global mean of all samples (Eq. 1)."""
    rng = np.random.Generator(np.random.PCG64(9))
    n = [3, 9, 1, 27]
    samples = [rng.standard_normal((k, 50)) for k in n]
    ref, _ = W.weighted_average(np.stack([s.mean(axis=0) for s in samples]), n)
    assert np.allclose(ref, np.concatenate(samples).mean(axis=0), rtol=1e-12, atol=1e-14)


@pytest.mark.parametrize("P", [2, 3, 4, 5, 7, 8])
@pytest.mark.parametrize("L", [1, 7, 8, 33, 1000, 4099])
def test_ring_emulation_within_bound(P, L):
    rng = np.random.Generator(np.random.PCG64(P * 1000 + L))
    n = [int(x) for x in rng.integers(1, 9, P)]
    for kind in ("gaussian", "mixed"):
        g32 = synth.gradients(P, L, seed_base=L, kind=kind)
        y = W.ring_emulate(g32, n, "f32")
        ref, den = W.weighted_average(W.as_f64(g32, "f32"), n)
        err, zb = W.error_metric(y, ref, den)
        # first-order bound: P roundings to fp32 (u = 2^-24) + fp32 quantisation of n_r/Σn (2^-24)
        assert zb == 0 and err <= (P + 1) * 2.0 ** -24 * 1.01
        gb = G.f32_to_bf16_bits(g32)
        yb = W.ring_emulate(gb, n, "bf16")
        ref, den = W.weighted_average(W.as_f64(gb, "bf16"), n)
        err, zb = W.error_metric(W.as_f64(yb, "bf16"), ref, den)
        # bf16 has an 8-bit significand: u = 2^-8 per rounding (each preceded by an fp32 rounding)
        assert zb == 0 and err <= P * (2.0 ** -8 + 2.0 ** -23) * 1.01


@pytest.mark.parametrize("P", [2, 4, 8])
def test_ring_emulation_power_of_two_equals_scaled_ring_sum(P):
    """s = 2^-k is exact, so the weighted ring equals s × (unweighted ring-order fp32 sum), bit for bit."""
    L = 1001
    g = synth.gradients(P, L, seed_base=3)
    y = W.ring_emulate(g, [5] * P, "f32")
    cs = W.chunk_elems(L, P, 4)
    plain = np.zeros(L, dtype=np.float32)
    for c in range(P):
        lo, hi = c * cs, min((c + 1) * cs, L)
        acc = g[c, lo:hi].copy()
        for h in range(1, P):
            acc = (acc + g[(c + h) % P, lo:hi]).astype(np.float32)
        plain[lo:hi] = acc
    assert np.array_equal(y, (plain * np.float32(1.0 / P)).astype(np.float32))


def test_ring_emulation_zero_rank_nan_does_not_propagate():
    g = synth.gradients(3, 64)
    g[1, :] = np.nan
    y = W.ring_emulate(g, [4, 0, 4], "f32")
    assert np.all(np.isfinite(y))
    ref, den = W.weighted_average(W.as_f64(g, "f32"), [4, 0, 4])
    err, _ = W.error_metric(y, ref, den)
    assert err < 1e-6


def test_chunking_rule():
    assert W.chunk_elems(1000, 8, 4) == 128
    assert W.chunk_elems(7, 8, 4) == 4
    assert W.chunk_elems(1, 2, 2) == 8


# ---------------------------------------------------------------- O7 ----------------------------

def test_linmodel_gradient_finite_differences():
    X, y, _ = synth.logistic_problem(200, 16)
    rng = np.random.Generator(np.random.PCG64(1))
    theta = rng.standard_normal(16) * 0.3
    g = LM.grad_mean(theta, X, y)
    eps = 1e-6
    fd = np.array([(LM.loss(theta + eps * e, X, y) - LM.loss(theta - eps * e, X, y)) / (2 * eps)
                   for e in np.eye(16)])
    assert np.max(np.abs(fd - g)) / np.max(np.abs(g)) < 1e-6


def test_linmodel_weighted_shards_equal_full_batch():
    X, y, _ = synth.logistic_problem()
    theta = np.linspace(-0.1, 0.1, X.shape[1])
    rows = [np.arange(0, 25), np.arange(25, 100)]
    ws = LM.weighted_step_gradient(theta, X, y, rows)
    full = X[:100].T @ (1.0 / (1.0 + np.exp(-(X[:100] @ theta))) - y[:100]) / 100
    assert np.max(np.abs(ws - full)) <= 1e-12 * np.max(np.abs(full))


def test_linmodel_trajectory_hand_derived_two_steps():
    """Pin of O7's trajectory() (VERDICT r1 "What's weak" #2) with a case worked by hand, so a shifted step
    (wrong rows, θ appended before the update, a dropped weight decay or weight) fails here on the CPU.

    D = 1, N = 6, two ranks with n = [1, 2] (weights 1/3, 2/3), shards rank 0 = rows [0, 1], rank 1 =
    rows [2, 3, 4, 5]; x = [1, 2, 1, -1, 3, 0.5], y = [1, 0, 0, 1, 1, 0]; η = 0.5, λ = 0.1, θ_0 = 0.
      step 0 rows: rank 0 {0}, rank 1 {2, 3}.  σ(0) = 1/2 so residuals σ − y = [-1/2 | 1/2, -1/2]:
        g_0 = 1/3·(1·(−1/2)) + 2/3·½·(1·½ + (−1)·(−½)) = −1/6 + 1/3 = 1/6
        θ_1 = 0 − ½·(1/6 + 0.1·0) = −1/12
      step 1 rows: rank 0 {1}, rank 1 {4, 5}, at θ_1 = −1/12:
        g_1 = 1/3·2·σ(−1/6) + 2/3·½·(3·(σ(−1/4) − 1) + ½·σ(−1/24))
        θ_2 = θ_1 − ½·(g_1 + 0.1·θ_1)
    """
    import math

    def sig(z):
        return 1.0 / (1.0 + math.exp(-z))

    X = np.array([[1.0], [2.0], [1.0], [-1.0], [3.0], [0.5]])
    y = np.array([1.0, 0.0, 0.0, 1.0, 1.0, 0.0])
    shards = [np.array([0, 1]), np.array([2, 3, 4, 5])]
    traj = LM.trajectory(X, y, shards, [1, 2], 2, 0.5, 0.1)
    th1 = -1.0 / 12.0
    g1 = (1 / 3) * 2 * sig(-1 / 6) + (2 / 3) * 0.5 * (3 * (sig(-1 / 4) - 1) + 0.5 * sig(-1 / 24))
    th2 = th1 - 0.5 * (g1 + 0.1 * th1)
    assert len(traj) == 3
    assert traj[0][0] == 0.0
    assert abs(traj[1][0] - th1) <= 1e-15
    assert abs(traj[2][0] - th2) <= 1e-15
    # the step gradient at θ_0 is the hand value 1/6
    assert abs(LM.weighted_step_gradient(np.zeros(1), X, y, LM.step_rows(shards, [1, 2], 0))[0] - 1 / 6) <= 1e-15


def test_linmodel_allocation_invariance():
    """[1,3] vs [2,2] over the same global rows per step give the same θ."""
    X, y, _ = synth.logistic_problem()
    order = np.arange(1000)

    def traj(split):
        theta = np.zeros(X.shape[1])
        for s in range(10):
            glob = order[s * 100:(s + 1) * 100]
            rows = [glob[:split], glob[split:]]
            theta = LM.sgd_step(theta, LM.weighted_step_gradient(theta, X, y, rows), 0.1)
        return theta

    a, b = traj(25), traj(50)
    assert np.max(np.abs(a - b)) <= 1e-12


# ---------------------------------------------------------------- O9 ----------------------------

def test_model_cost_2_to_1_thirty_percent():
    """S:418 / S:411: costs 1:2 ms, C=20: adaptive freezes at [13,7], 30% below equal allocation."""
    speeds = [1000.0, 500.0]
    recs = EM.run(N=20 * 50, P=2, C=20, g=1, speeds=speeds, epochs=6)
    assert recs[0]["w"] == [10, 10] and recs[-1]["w"] == [13, 7] and recs[-1]["frozen"]
    red = 1.0 - recs[-1]["T"] / recs[0]["T"]
    assert 0.29 < red < 0.31


def test_model_cost_5_to_1():
    recs = EM.run(N=20 * 50, P=2, C=20, g=1, speeds=[1000.0, 200.0], epochs=6)
    assert recs[-1]["w"] == [17, 3]
    assert 0.65 < 1.0 - recs[-1]["T"] / recs[0]["T"] < 0.67


def test_model_capacity_monotone():
    """adding a worker or replacing the slow one strictly reduces the frozen epoch time."""
    base = EM.run(N=2000, P=2, C=20, g=1, speeds=[1000.0, 500.0], epochs=8)[-1]["T"]
    add = EM.run(N=2000, P=3, C=20, g=1, speeds=[1000.0, 500.0, 500.0], epochs=8)[-1]["T"]
    rep = EM.run(N=2000, P=2, C=20, g=1, speeds=[1000.0, 1000.0], epochs=8)[-1]["T"]
    assert add < base and rep < base


def test_model_affine_overhead_four_epochs():
    """Speeds 1:1:2:2 with a per-step overhead: converges to [11,11,21,21] within <= 5 updates."""
    recs = EM.run(N=51200, P=4, C=64, g=16, speeds=[1000.0, 1000.0, 2000.0, 2000.0], epochs=8,
                  overhead=[0.05] * 4)
    ws = [r["w"] for r in recs]
    assert ws[0] == [16, 16, 16, 16]
    k = next(i for i, r in enumerate(recs) if r["frozen"])
    assert k <= 6 and ws[-1] == [11, 11, 21, 21]


def test_model_bound_and_equal_prediction():
    S, B = 10, 1024
    assert EM.bound(S, B, [1.0, 3.0]) == pytest.approx(10 * 1024 / 4.0)
    assert EM.equal_prediction(S, B, [1.0, 3.0]) == pytest.approx(10 * 512 / 1.0)
