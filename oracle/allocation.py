"""O2 static allocation and O8 self-adaptive controller.  TEST INFRASTRUCTURE ONLY (see oracle/__init__.py).

Follows the paper's algorithm step by step:

* Static allocation (§3.1): "we set the weight w_1..w_n ... we assigned a corresponding
  proportion of training samples to each worker from the total dataset"; D_i = D·w_i/Σw;
  the total batch per aggregation is minibatch·Σw (P:69 end).  Reading (DESIGN.md §3 #1):
  w_i counts units of g samples, n_i = g·w_i, B = g·C.  Shard sizes by exact-integer Hamilton
  (§3 #9, departs from SPEC's remainder-to-last S:64).  S = floor(N/B) aggregations per epoch, each
  rank uses the first S·n_r positions of its shard (§3 #10).
* Self-adaptive allocation (Algorithm 1; Eq. 10):
      w_i^(k+1) = (w_i^(k)/t_s^i) / Σ_j (w_j^(k)/t_s^j) · Σ_j w_j^(k)
  then integer rounding (Hamilton, §3 #3), stop rule "could be cancelled when the ratio is
  not fluctuating" (window=2, tol=1, §3 #7).  First epoch t_s = 0 -> ZeroTiming, no
  update (§3 #6).
* Eq. 9 = Appendix Eq. 22 closed-form increment u, and the Appendix linear
  system A·u = b (Eqs. 15-21) solved by Gaussian elimination as an oracle cross-check.

* Affine step-cost model (opt-in extension, DESIGN.md §3 #49 — NOT in the paper): the paper's model is
  t_s ∝ samples (Eq. 6-8); with a fixed per-step cost each rank's epoch time is fitted as
  t_i(w) = a_i + b_i·w by least squares over its last `fit_window` (w, t) observations, and the next
  allocation is the integer min-max allocation min_{Σw=C, w>=floor} max_i a_i + b_i·w_i, built by handing
  out units one at a time to the rank with the smallest cost after taking it (ties to the lowest rank).
  Fewer than two distinct w for a rank: a_i = 0, b_i = t_i/w_i; a fit with b <= 0 or a < 0: the same
  proportional model through the latest observation.  No rank with two distinct w: Eq. 10 exactly.

The fp64 operation order of `controller_quotas` is part of the definition (bit-exact with the host
library; DESIGN.md §3 #35):  v_i = w_i / t_i;  S_v = ((v_0 + v_1) + ...) left to right;
q_i = (C·v_i) / S_v.
"""

from __future__ import annotations

import math
from dataclasses import dataclass, field

from .apportion import hamilton, hamilton_exact


class ZeroTiming(ValueError):
    """S:98 ZeroTiming — some t_s <= 0 or non-finite; the allocation is left unchanged."""


class InfeasibleFloor(ValueError):
    """S:128 InfeasibleFloor — C < P·floor."""


class DatasetTooSmall(ValueError):
    """S:326 DatasetTooSmall — N < B = g·C."""


@dataclass
class Allocation:
    N: int
    P: int
    C: int
    g: int
    floor: int
    w: list
    n: list = field(default_factory=list)
    len: list = field(default_factory=list)
    off: list = field(default_factory=list)
    B: int = 0
    S: int = 0
    epoch: int = 0
    frozen: bool = False
    history: list = field(default_factory=list)
    window: int = 2
    tol: int = 1
    never_freeze: bool = False
    ema_alpha: float = 1.0
    t_prev: list | None = None
    model: str = "proportional"       # or "affine" (§3 #49)
    fit_window: int = 8
    t_hist: list = field(default_factory=list)   # t used by update k (history[k] was in effect)


def shard_sizes(N: int, w, C: int):
    """D_i = D·w_i/Σw rounded by exact-integer Hamilton; off = exclusive prefix sum."""
    length = hamilton_exact([N * wi for wi in w], C, N)
    off = []
    acc = 0
    for x in length:
        off.append(acc)
        acc += x
    return length, off


def _derive(a: Allocation) -> Allocation:
    a.n = [a.g * wi for wi in a.w]
    a.B = a.g * a.C
    a.len, a.off = shard_sizes(a.N, a.w, a.C)
    a.S = a.N // a.B
    return a


def alloc_init(N: int, ratios, C: int = 0, g: int = 1, floor: int = 1) -> Allocation:
    """O2: w = Hamilton(C·r_i/Σr, C, floor).  C = 0 means C = Σr (ratios must then be integers)."""
    P = len(ratios)
    r = [float(x) for x in ratios]
    if P < 1 or N < 1 or g < 1 or floor < 0 or any((not math.isfinite(x)) or x <= 0 for x in r):
        raise ValueError("invalid")
    if C == 0:
        if any(x != math.floor(x) for x in r):
            raise ValueError("C=0 requires integer ratios")
        C = int(sum(int(x) for x in r))
    if C < P * floor:
        raise InfeasibleFloor()
    if N < g * C:
        raise DatasetTooSmall()
    s = 0.0
    for x in r:
        s = s + x
    q = [(float(C) * x) / s for x in r]
    w = hamilton(q, C, floor)
    a = Allocation(N=N, P=P, C=C, g=g, floor=floor, w=w)
    _derive(a)
    a.history = [list(w)]
    return a


def controller_quotas(w, t, C: int):
    """Eq. 10 before rounding: q_i = C·(w_i/t_i)/Σ_j(w_j/t_j), fixed fp64 order."""
    v = [float(wi) / float(ti) for wi, ti in zip(w, t)]
    s = 0.0
    for x in v:
        s = s + x
    return [(float(C) * x) / s for x in v]


def is_stable(history, window: int, tol: int) -> bool:
    """the last `window` vectors pairwise differ by <= tol in every component."""
    if len(history) < window:
        return False
    tail = history[-window:]
    for i in range(len(tail)):
        for j in range(i + 1, len(tail)):
            if max(abs(x - y) for x, y in zip(tail[i], tail[j])) > tol:
                return False
    return True


def affine_fit(ws, ts):
    """Least-squares t = a + b·w over one rank's observations (chronological), fixed fp64 order:
    means by left-to-right sums, then Σ(w−mw)², Σ(w−mw)(t−mt) left to right; b = sxy/sxx, a = mt − b·mw.
    None when fewer than two distinct w; (0, t/w of the latest) when b <= 0 or a < 0."""
    if all(x == ws[0] for x in ws):
        return None
    n = len(ws)
    sw = 0.0
    st = 0.0
    for x, y in zip(ws, ts):
        sw = sw + float(x)
        st = st + y
    mw = sw / float(n)
    mt = st / float(n)
    sxx = 0.0
    sxy = 0.0
    for x, y in zip(ws, ts):
        d = float(x) - mw
        sxx = sxx + d * d
        sxy = sxy + d * (y - mt)
    b = sxy / sxx
    a = mt - b * mw
    if b > 0.0 and a >= 0.0 and math.isfinite(a) and math.isfinite(b):
        return a, b
    return 0.0, ts[-1] / float(ws[-1])


def minmax_greedy(models, C: int, floor: int):
    """Integer min-max allocation for increasing affine costs: every rank at the floor, then each remaining
    unit to the rank whose cost a + b·(w+1) is smallest (ties to the lowest rank)."""
    w = [floor] * len(models)
    for _ in range(C - len(models) * floor):
        best, bc = 0, None
        for i, (a, b) in enumerate(models):
            c = a + b * float(w[i] + 1)
            if bc is None or c < bc:
                best, bc = i, c
        w[best] += 1
    return w


def alloc_update(a: Allocation, t_s) -> bool:
    """O8, Algorithm 1 steps 1-3.  Returns `changed`.  Mutates `a` only on success."""
    if a.frozen:
        return False
    t = [float(x) for x in t_s]
    if len(t) != a.P:
        raise ValueError("invalid")
    if any((not math.isfinite(x)) or x <= 0.0 for x in t):
        raise ZeroTiming()
    if a.ema_alpha != 1.0 and a.t_prev is not None:
        t = [a.ema_alpha * x + (1.0 - a.ema_alpha) * y for x, y in zip(t, a.t_prev)]
    w_new = None
    if a.model == "affine":
        obs = list(zip(a.history[:len(a.t_hist)], a.t_hist))[-(a.fit_window - 1):] + [(list(a.w), t)]
        models = []
        for i in range(a.P):
            f = affine_fit([o[0][i] for o in obs], [o[1][i] for o in obs])
            models.append(f)
        if any(f is not None for f in models):
            models = [f if f is not None else (0.0, t[i] / float(a.w[i])) for i, f in enumerate(models)]
            w_new = minmax_greedy(models, a.C, a.floor)
    if w_new is None:
        q = controller_quotas(a.w, t, a.C)
        w_new = hamilton(q, a.C, a.floor)
    changed = w_new != a.w
    a.t_prev = t
    a.t_hist.append(list(t))
    a.w = w_new
    a.history.append(list(w_new))
    a.epoch += 1
    _derive(a)
    if not a.never_freeze and is_stable(a.history, a.window, a.tol):
        a.frozen = True
    return changed


# ---- Eq. 9 / Eq. 22 and the Appendix linear system (oracle-only cross-check) -------------------

def increments_closed_form(w, v):
    """Eq. 9 = Eq. 22: u_i = v_i/Σv · Σw − w_i."""
    sv = math.fsum(v)
    sw = math.fsum(w)
    return [vi / sv * sw - wi for vi, wi in zip(v, w)]


def appendix_system(w, v):
    """Eqs. 15-21: rows i<n: 1/v_i at i, −1/v_{i+1} at i+1; last row all ones (Eq. 17).
    b_i = w_{i+1}/v_{i+1} − w_i/v_i for i<n, b_n = 0 (Eq. 20)."""
    n = len(w)
    A = [[0.0] * n for _ in range(n)]
    b = [0.0] * n
    for i in range(n - 1):
        A[i][i] = 1.0 / v[i]
        A[i][i + 1] = -1.0 / v[i + 1]
        b[i] = w[i + 1] / v[i + 1] - w[i] / v[i]
    A[n - 1] = [1.0] * n
    return A, b


def solve_gauss(A, b):
    """Plain Gaussian elimination with partial pivoting."""
    n = len(b)
    M = [list(map(float, row)) + [float(bi)] for row, bi in zip(A, b)]
    for col in range(n):
        piv = max(range(col, n), key=lambda r: abs(M[r][col]))
        if M[piv][col] == 0.0:
            raise ZeroDivisionError("singular")
        M[col], M[piv] = M[piv], M[col]
        for r in range(col + 1, n):
            f = M[r][col] / M[col][col]
            for c in range(col, n + 1):
                M[r][c] -= f * M[col][c]
    x = [0.0] * n
    for r in range(n - 1, -1, -1):
        s = M[r][n]
        for c in range(r + 1, n):
            s -= M[r][c] * x[c]
        x[r] = s / M[r][r]
    return x


def increments_linear_system(w, v):
    """Solve the Appendix system A·u = b (Eq. 21)."""
    A, b = appendix_system(w, v)
    return solve_gauss(A, b)
