"""Pins for oracle O1 (apportionment), O2 (static allocation) and O8 (controller).

Each test checks the oracle against something other than itself: hand-derived worked examples
(tests/golden, cited), brute force over tiny inputs, the Appendix linear system solved by a
library routine, and invariants the paper states (Eq. 4/5 conservation, Eq. 8 equilibrium).
"""

import itertools
import math
import random
from fractions import Fraction

import numpy as np
import pytest

from conftest import read_golden, ints, floats
from oracle import allocation as A
from oracle.apportion import hamilton, hamilton_exact


# ---------------------------------------------------------------- O1 ----------------------------

def _parse_kv(s):
    out = {}
    for tok in s.split():
        k, v = tok.split("=")
        out[k] = v
    return out


def test_golden_spec_examples():
    rows = read_golden("spec_allocator_examples.txt")
    assert len(rows) >= 9
    for kind, inp, exp in rows:
        kv = _parse_kv(inp)
        if kind == "apportion":
            got = hamilton(floats(kv["q"]), int(kv["total"]), int(kv["floor"]))
            assert got == ints(exp), (inp, got)
        elif kind == "update":
            w = ints(kv["w"])
            a = A.alloc_init(10 ** 6, w, C=int(kv["C"]), g=1, floor=1)
            A.alloc_update(a, floats(kv["t"]))
            assert a.w == ints(exp), (inp, a.w)
        elif kind == "rates":
            v = [wi / ti for wi, ti in zip(ints(kv["w"]), floats(kv["t"]))]
            assert v == floats(exp)
        elif kind == "closed_form":
            u = A.increments_closed_form(ints(kv["w"]), floats(kv["v"]))
            assert np.allclose(u, floats(exp), rtol=1e-12, atol=1e-12)
        else:
            raise AssertionError(kind)


def _brute_force_lr(num, den, total):
    """All integer vectors >= 0 with sum = total; L1-closest to num/den; ties -> lexicographically largest."""
    P = len(num)
    best, best_cost = None, None
    for a in itertools.product(range(total + 1), repeat=P):
        if sum(a) != total:
            continue
        cost = sum(abs(Fraction(x) - Fraction(n, den)) for x, n in zip(a, num))
        if best is None or cost < best_cost or (cost == best_cost and a > best):
            best, best_cost = a, cost
    return list(best)


def test_hamilton_brute_force_tiny():
    rng = random.Random(7)
    cases = 0
    for P in (1, 2, 3, 4):
        for total in range(0, 13):
            for _ in range(6):
                den = rng.choice([1, 2, 3, 4, 5, 7, 8, 16])
                # random composition of total·den into P non-negative parts
                cuts = sorted(rng.randint(0, total * den) for _ in range(P - 1))
                parts = [b - a for a, b in zip([0] + cuts, cuts + [total * den])]
                exp = _brute_force_lr(parts, den, total)
                assert hamilton_exact(parts, den, total) == exp, (parts, den, total)
                if den in (1, 2, 4, 8, 16):  # quotas exactly representable in fp64
                    q = [p / den for p in parts]
                    assert hamilton(q, total, 0) == exp
                cases += 1
    assert cases > 200


def test_hamilton_quota_and_sum_properties():
    rng = np.random.Generator(np.random.PCG64(3))
    for _ in range(2000):
        P = int(rng.integers(1, 17))
        C = int(rng.integers(P, 400))
        v = rng.uniform(0.01, 10.0, P)
        q = A.controller_quotas([1] * P, 1.0 / v, C)
        a = hamilton(q, C, 0)
        assert sum(a) == C
        assert all(abs(ai - qi) < 1.0 for ai, qi in zip(a, q))   # quota property
        b = hamilton(q, C, 1)
        assert sum(b) == C and min(b) >= 1
        if min(a) >= 1:
            assert a == b


def test_hamilton_floor_clamp():
    assert hamilton([0.2, 0.3, 19.5], 20, 1) == [1, 1, 18]
    assert hamilton([0.0, 0.0, 20.0], 20, 2) == [2, 2, 16]
    with pytest.raises(ValueError):
        hamilton([1.0, 1.0], 2, 2)


# ---------------------------------------------------------------- O2 ----------------------------

def test_golden_shard_sizes():
    for N, ratios, C, g, w, n, S, ln in read_golden("shard_sizes.txt"):
        N, C, g, S = int(N), int(C), int(g), int(S)
        if S == 0:
            length, off = A.shard_sizes(N, ints(w), C)
            assert length == ints(ln)
            continue
        a = A.alloc_init(N, floats(ratios), C=C, g=g, floor=1)
        assert a.w == ints(w) and a.n == ints(n) and a.S == S and a.len == ints(ln)
        assert sum(a.len) == N and a.off[0] == 0
        assert all(a.off[i + 1] == a.off[i] + a.len[i] for i in range(a.P - 1))
        assert all(abs(li - Fraction(N * wi, C)) < 1 for li, wi in zip(a.len, a.w))  # ±1 sample
        assert all(li >= S * ni for li, ni in zip(a.len, a.n))  # S·n_r fits in every shard


def test_init_errors():
    with pytest.raises(A.InfeasibleFloor):
        A.alloc_init(100, [1, 1, 1], C=2, g=1, floor=1)
    with pytest.raises(A.DatasetTooSmall):
        A.alloc_init(10, [1, 1], C=20, g=1)
    with pytest.raises(ValueError):
        A.alloc_init(10, [1, -1], C=2)
    with pytest.raises(ValueError):
        A.alloc_init(10, [1, float("nan")], C=2)


def test_init_real_ratios_rounds_to_C():
    a = A.alloc_init(10000, [1.0, 2.5, 0.7], C=20, g=4)
    assert sum(a.w) == 20 and a.w == hamilton([20 * 1.0 / 4.2, 20 * 2.5 / 4.2, 20 * 0.7 / 4.2], 20, 1)


# ---------------------------------------------------------------- O8 ----------------------------

def test_zero_timing_leaves_state_unchanged():
    a = A.alloc_init(1000, [1, 1], C=20, g=1)
    before = (list(a.w), a.epoch, list(a.history))
    for bad in ([0.0, 1.0], [1.0, -1.0], [float("nan"), 1.0], [float("inf"), 1.0]):
        with pytest.raises(A.ZeroTiming):
            A.alloc_update(a, bad)
        assert (a.w, a.epoch, a.history) == before


def test_appendix_linear_system_equals_closed_form():
    """Eq. 22 == solve of A·u=b (Eqs. 19-21), n in [2,16] x 1000."""
    rng = np.random.Generator(np.random.PCG64(11))
    for _ in range(1000):
        n = int(rng.integers(2, 17))
        w = rng.integers(1, 50, n).astype(float)
        v = rng.uniform(0.1, 20.0, n)
        u_cf = np.array(A.increments_closed_form(w, v))
        u_ge = np.array(A.increments_linear_system(w, v))
        Am, b = A.appendix_system(w, v)
        u_np = np.linalg.solve(np.array(Am), np.array(b))      # library routine
        scale = max(1.0, float(np.abs(u_cf).max()))
        assert np.max(np.abs(u_cf - u_ge)) <= 1e-9 * scale
        assert np.max(np.abs(u_cf - u_np)) <= 1e-9 * scale
        assert abs(u_cf.sum()) <= 1e-9 * w.sum()                # Eq. 5


def test_update_equals_rounded_eq22():
    """w^(k+1) = w^(k) + u (Eq. 10 = Eq. 9 + w) before rounding; Hamilton after."""
    rng = np.random.Generator(np.random.PCG64(12))
    for _ in range(300):
        P = int(rng.integers(2, 9))
        C = int(rng.integers(4 * P, 200))
        a = A.alloc_init(10 ** 6, [1] * P, C=C, g=1)
        t = rng.uniform(0.5, 4.0, P)
        w0 = list(a.w)
        q = A.controller_quotas(w0, t, C)
        v = [wi / ti for wi, ti in zip(w0, t)]
        u = A.increments_linear_system(w0, v)
        assert np.allclose(q, np.array(w0) + np.array(u), rtol=1e-9, atol=1e-9)
        A.alloc_update(a, t)
        assert sum(a.w) == C                                   # Eq. 4
        assert all(abs(x - y) < 1.0 for x, y in zip(a.w, q)) or min(a.w) == 1


def test_equilibrium_eq8_and_fixed_point():
    """Linear costs t_i = w_i·c_i: one update lands on w ∝ v (Eq. 8); equal t is a fixed point."""
    rng = np.random.Generator(np.random.PCG64(13))
    for _ in range(200):
        P = int(rng.integers(2, 9))
        C = 240
        cost = rng.uniform(0.5, 3.0, P)
        w = A.hamilton([C / P] * P, C, 1)
        t = [wi * ci for wi, ci in zip(w, cost)]
        q = A.controller_quotas(w, t, C)
        v = [wi / ti for wi, ti in zip(w, t)]
        ratio = [qi / vi for qi, vi in zip(q, v)]
        assert max(ratio) - min(ratio) <= 1e-9 * max(ratio)      # D·w_j/(C·v_j) equal for all pairs
    a = A.alloc_init(10 ** 6, [8, 8, 8], C=24)
    assert A.alloc_update(a, [3.0, 3.0, 3.0]) is False and a.w == [8, 8, 8]


def test_scale_invariance():
    rng = np.random.Generator(np.random.PCG64(14))
    for _ in range(200):
        P = int(rng.integers(2, 9))
        t = rng.uniform(0.5, 4.0, P)
        a = A.alloc_init(10 ** 6, [1] * P, C=64)
        b = A.alloc_init(10 ** 6, [1] * P, C=64)
        A.alloc_update(a, t)
        A.alloc_update(b, t * 4.0)        # power of two: exact scaling of every quotient
        assert a.w == b.w


def test_stop_rule_freezes_within_five_epochs():
    """costs [1ms, 2ms], C=20, start [10,10] -> [13,7], frozen within <= 5 epochs."""
    a = A.alloc_init(10 ** 6, [10, 10], C=20, g=1)
    cost = [1e-3, 2e-3]
    epochs = 0
    while not a.frozen:
        A.alloc_update(a, [wi * ci for wi, ci in zip(a.w, cost)])
        epochs += 1
        assert epochs <= 5
    assert a.w == [13, 7]
    hist = list(a.history)
    assert A.alloc_update(a, [1.0, 100.0]) is False and a.history == hist   # frozen: no-op
    assert A.is_stable([[8, 12], [7, 13]], 2, 0) is False
    assert A.is_stable([[8, 12], [7, 13]], 2, 1) is True
    assert A.is_stable([[7, 13]], 2, 1) is False


def test_three_worker_equilibrium():
    """costs [1,1,2] ms, C=20 -> [8,8,4]."""
    a = A.alloc_init(10 ** 6, [7, 7, 6], C=20, g=1)
    cost = [1.0, 1.0, 2.0]
    for _ in range(5):
        A.alloc_update(a, [wi * ci for wi, ci in zip(a.w, cost)])
    assert a.w == [8, 8, 4]


def test_ema_smoothing_definition():
    a = A.alloc_init(10 ** 6, [10, 10], C=20)
    a.ema_alpha = 0.5
    a.never_freeze = True
    A.alloc_update(a, [1.0, 1.0])
    A.alloc_update(a, [3.0, 1.0])
    assert a.t_prev == [0.5 * 3.0 + 0.5 * 1.0, 1.0]


# ---- affine step-cost model (DESIGN.md §3 #49; opt-in extension, not the paper's Eq. 10) -------------

def _brute_minmax(models, C, floor):
    """Every composition of C into len(models) parts >= floor: the smallest achievable max cost."""
    import itertools

    P = len(models)
    best = None
    for w in itertools.product(range(floor, C - floor * (P - 1) + 1), repeat=P):
        if sum(w) != C:
            continue
        m = max(a + b * float(x) for (a, b), x in zip(models, w))
        best = m if best is None or m < best else best
    return best


def test_minmax_greedy_is_the_brute_force_optimum():
    """Pin of the greedy: for increasing affine costs its max equals the exhaustive min-max (P <= 4,
    C <= 12, floor 1 or 2), and the result is a valid allocation."""
    rng = np.random.Generator(np.random.PCG64(49))
    for case in range(400):
        P = int(rng.integers(1, 5))
        floor = int(rng.integers(1, 3))
        C = int(rng.integers(P * floor, 13))
        models = [(float(rng.choice([0.0, rng.uniform(0, 3)])), float(rng.uniform(0.1, 4))) for _ in range(P)]
        w = A.minmax_greedy(models, C, floor)
        assert sum(w) == C and min(w) >= floor
        got = max(a + b * float(x) for (a, b), x in zip(models, w))
        assert got == _brute_minmax(models, C, floor), (models, C, floor, w)


def test_affine_fit_recovers_exact_lines_and_matches_polyfit():
    """Pin of the least-squares fit: noise-free t = a + b·w is recovered to rounding; noisy data agree with
    numpy.polyfit (library routine) to 1e-9; one distinct w -> None; a falling line -> the proportional
    fallback through the latest point."""
    rng = np.random.Generator(np.random.PCG64(7))
    for _ in range(200):
        a, b = float(rng.uniform(0, 5)), float(rng.uniform(0.01, 3))
        ws = [int(x) for x in rng.integers(1, 40, int(rng.integers(2, 9)))]
        if len(set(ws)) < 2:
            ws.append(ws[0] + 1)
        fa, fb = A.affine_fit(ws, [a + b * w for w in ws])
        assert abs(fa - a) <= 1e-9 * (1 + a) and abs(fb - b) <= 1e-9 * b
        ts = [a + b * w + float(rng.normal(0, 0.01)) for w in ws]
        f = A.affine_fit(ws, ts)
        pb, pa = np.polyfit(np.array(ws, float), np.array(ts), 1)
        if pb > 0 and pa >= 0:
            assert abs(f[0] - pa) <= 1e-9 * (1 + abs(pa)) and abs(f[1] - pb) <= 1e-9 * (1 + abs(pb))
        else:
            assert f == (0.0, ts[-1] / ws[-1])
    assert A.affine_fit([4, 4, 4], [1.0, 1.1, 0.9]) is None
    assert A.affine_fit([2, 4], [3.0, 1.0]) == (0.0, 1.0 / 4)


def test_affine_model_first_update_is_eq10_and_second_reaches_the_optimum():
    """From a uniform start no rank has two distinct w, so the first update IS Eq. 10 + Hamilton; with
    noise-free affine costs the second update (two observations per rank) lands on the exact min-max
    allocation of the true costs (brute force over P = 3, C = 12), and the stop rule then freezes it."""
    cost = [(2.0, 0.5), (2.0, 1.0), (2.0, 2.0)]                  # fixed cost 2, speeds 4:2:1

    def times(w):
        return [a + b * float(x) for (a, b), x in zip(cost, w)]

    a = A.alloc_init(10_000, [1, 1, 1], C=12, g=1)
    e = A.alloc_init(10_000, [1, 1, 1], C=12, g=1)
    a.model = "affine"
    A.alloc_update(a, times(a.w))
    A.alloc_update(e, times(e.w))
    assert a.w == e.w
    A.alloc_update(a, times(a.w))
    assert max(times(a.w)) == _brute_minmax(cost, 12, 1)
    A.alloc_update(a, times(a.w))
    A.alloc_update(a, times(a.w))
    assert a.frozen


def test_affine_model_on_linear_costs_is_eq8_up_to_rounding():
    """Linear costs (a = 0, the paper's model, Eq. 6-8): the affine model's allocation is the min-max of
    b_i·w_i, i.e. w ∝ v_i = 1/b_i (Eq. 8) to within one unit per rank."""
    b = [1.0, 1.0, 2.0, 4.0]                                      # speeds 4:4:2:1 -> 16:16:8:4 of C = 44
    a = A.alloc_init(10_000, [1, 1, 1, 1], C=44, g=1)
    a.model = "affine"
    a.never_freeze = True
    for _ in range(4):
        A.alloc_update(a, [bi * float(w) for bi, w in zip(b, a.w)])
    assert all(abs(x - y) <= 1 for x, y in zip(a.w, [16, 16, 8, 4]))
