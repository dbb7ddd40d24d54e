"""O9 epoch-time model and the Σspeed-balanced bound.  TEST INFRASTRUCTURE ONLY (see oracle/__init__.py).

Timing decomposition (§3.2.1): T_i = t_c^i + t_s^i + t_w^i per aggregation; t_c equal
for all workers (Eq. 2); every worker leaves the barrier together (Eq. 3), so
t_w^i = max_j t_s^j − t_s^i.  Speeds v_i (samples/s).

Model: per aggregation, rank r computes for a_r + n_r/v_r seconds (a_r = fixed
per-step overhead, optional multiplicative lognormal noise σ, seeded); the step lasts
max_r(compute_r) + t_c; an epoch is S aggregations.  The controller (O8) is iterated over epochs.

  bound   T_ideal = S·(B/Σv + t_c)                        (perfect balance, continuous w)
  equal   S·(max_r (B/P)/v_r + t_c)                        (equal allocation)

Pins: S:411-418 acceptance examples (costs 1:2 -> [13,7], 30% below equal; [1,1,2] -> [8,8,4];
capacity monotonicity) and the paper's "4-5 epochs" for the affine-overhead model.
End-to-end measured epoch times on the GPU are judged against this bound (parity unpinned by the
paper: no epoch time survives in its text).
"""

from __future__ import annotations

import numpy as np

from .allocation import alloc_init, alloc_update, ZeroTiming


def step_compute(n_local, speeds, overhead=None, noise=0.0, rng=None):
    """Per-rank compute seconds for one aggregation."""
    P = len(n_local)
    a = [0.0] * P if overhead is None else list(overhead)
    t = np.array([a[r] + n_local[r] / speeds[r] for r in range(P)], dtype=np.float64)
    if noise > 0.0:
        t = t * np.exp(noise * rng.standard_normal(P))
    return t


def epoch(alloc, speeds, t_c=0.0, overhead=None, noise=0.0, rng=None):
    """One epoch: returns dict(t_s per rank, t_w per rank, T epoch seconds)."""
    ts = np.zeros(alloc.P)
    tw = np.zeros(alloc.P)
    T = 0.0
    for _ in range(alloc.S):
        c = step_compute(alloc.n, speeds, overhead, noise, rng)
        m = float(c.max())
        ts += c
        tw += m - c
        T += m + t_c
    return {"t_s": ts, "t_w": tw, "T": T}


def bound(S, B, speeds, t_c=0.0):
    return S * (B / float(np.sum(speeds)) + t_c)


def equal_prediction(S, B, speeds, t_c=0.0):
    P = len(speeds)
    return S * (max((B / P) / v for v in speeds) + t_c)


def run(N, P, C, g, speeds, epochs, ratios=None, t_c=0.0, overhead=None, noise=0.0, seed=0,
        adaptive=True, floor=1):
    """Algorithm 1 over the model: epoch 0 uses the initial ratios; from the next epoch
    boundary on, t_s of the last epoch drives Eq. 10.  Returns per-epoch records."""
    rng = np.random.Generator(np.random.PCG64(seed))
    a = alloc_init(N, ratios if ratios is not None else [1] * P, C=C, g=g, floor=floor)
    out = []
    for e in range(epochs):
        rec = epoch(a, speeds, t_c, overhead, noise, rng)
        rec["w"] = list(a.w)
        rec["frozen"] = a.frozen
        out.append(rec)
        if adaptive:
            try:
                alloc_update(a, rec["t_s"])
            except ZeroTiming:
                pass
    return out
