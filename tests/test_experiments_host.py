"""CPU checks of experiments.py's host logic: the affine-cost min-max bound (the best integer allocation
for step costs a + b·n under either K4 emulation) against brute force, and the affine fit."""

import itertools
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import experiments as E  # noqa: E402


def _cost(a, b, g, x, s, spin, c0):
    return E.step_cost(a + b * g * x, g * x, s, spin, c0)


def _brute(a, b, sigma, g, C, floor, spin, c0):
    best = None
    for w in itertools.product(range(floor, C + 1), repeat=len(sigma)):
        if sum(w) != C:
            continue
        t = max(_cost(a, b, g, x, s, spin, c0) for x, s in zip(w, sigma))
        best = t if best is None else min(best, t)
    return best


def test_affine_minmax_is_the_integer_optimum():
    rng = np.random.Generator(np.random.PCG64(5))
    for _ in range(60):
        P = int(rng.integers(2, 5))
        C = int(rng.integers(P, 13))
        sigma = [float(x) for x in rng.choice([1.0, 1.5, 2.0, 4.0], P)]
        a, b = float(rng.uniform(0, 2e-3)), float(rng.uniform(1e-7, 5e-6))
        spin = "t1" if rng.random() < 0.5 else "sample"
        c0 = float(rng.uniform(1e-6, 2e-5))
        T, w = E.affine_minmax(a, b, sigma, 16, C, 1, spin, c0)
        assert sum(w) == C and min(w) >= 1
        assert max(_cost(a, b, 16, x, s, spin, c0) for x, s in zip(w, sigma)) <= T + 1e-15
        assert abs(T - _brute(a, b, sigma, 16, C, 1, spin, c0)) <= 1e-15


def test_affine_minmax_linear_costs_give_the_proportional_allocation():
    # no fixed cost: the optimum is w ∝ v (Eq. 8), e.g. C4's speeds 1:1:1:1:2:2:4:4 -> [4,4,4,4,8,8,16,16]
    T, w = E.affine_minmax(0.0, 1e-6, [4, 4, 4, 4, 2, 2, 1, 1], 16, 64)
    assert w == [4, 4, 4, 4, 8, 8, 16, 16] and abs(T - 256e-6) < 1e-15


def test_minmax_alloc_on_a_measured_table():
    """A non-affine cost table (a step at a microbatch boundary): the greedy min-max is still the optimum."""
    tab = {u: 1e-3 + 2e-6 * 16 * u + (0.8e-3 if u > 8 else 0.0) for u in range(1, 17)}
    sigma = [3.0, 1.0, 1.0]
    T, w = E.minmax_alloc(lambda r, u: sigma[r] * tab[u], 3, 16)
    best = min(max(sigma[r] * tab[x] for r, x in enumerate(ws))
               for ws in itertools.product(range(1, 15), repeat=3) if sum(ws) == 16)
    assert sum(w) == 16 and abs(T - best) < 1e-15


def test_minmax_alloc_non_monotone_costs():
    """A measured table is not monotone (cuDNN picks a different algorithm per batch size): a feasible
    allocation may skip over a costly unit count; the DP still finds the exact optimum."""
    rng = np.random.Generator(np.random.PCG64(9))
    for _ in range(40):
        P, C = 3, int(rng.integers(3, 13))
        tab = [[float(x) for x in rng.uniform(1.0, 2.0, C + 1)] for _ in range(P)]
        T, w = E.minmax_alloc(lambda r, u: tab[r][u], P, C)
        best = min(max(tab[r][x] for r, x in enumerate(ws))
                   for ws in itertools.product(range(1, C + 1), repeat=P) if sum(ws) == C)
        assert sum(w) == C and min(w) >= 1 and abs(T - best) < 1e-15
        assert max(tab[r][x] for r, x in enumerate(w)) <= T


def test_fit_affine():
    a, b = E.fit_affine([64, 128, 256], [1.3e-3 + 1.5e-6 * n for n in (64, 128, 256)])
    assert abs(a - 1.3e-3) < 1e-12 and abs(b - 1.5e-6) < 1e-15
    assert E.fit_affine([100], [2.0]) == (2.0, 0.0)


def test_make_policy_from_command_line():
    """--model affine / --ema / --never-freeze each reach Alloc.set_policy, alone or together (the EMA is no
    longer dropped when the stop rule stays on)."""
    import argparse

    import paper_2111_08272_b200 as pr

    def ns(**kw):
        d = dict(never_freeze=False, scenario="c4", ema=1.0, model="proportional")
        d.update(kw)
        return argparse.Namespace(**d)

    assert E.make_policy(ns()) is None
    assert E.make_policy(ns(ema=0.5)) == {"ema_alpha": 0.5}
    assert E.make_policy(ns(model="affine")) == {"model": pr.ALLOC_MODEL_AFFINE}
    assert E.make_policy(ns(never_freeze=True, model="affine")) == {"never_freeze": True, "model": pr.ALLOC_MODEL_AFFINE}
    assert E.make_policy(ns(scenario="n3-swap")) == {"never_freeze": True}
    a = pr.alloc_init(50_000, [1] * 8, C=64, g=16)
    a.set_policy(**E.make_policy(ns(model="affine", ema=0.7)))
