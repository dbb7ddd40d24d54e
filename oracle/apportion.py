"""O1 — integer apportionment (largest remainder / Hamilton).  TEST INFRASTRUCTURE ONLY (see oracle/__init__.py).

Paper: "The reason why rounding decimals of u_i is that w^(k+1) is integer" (§3.2.3) — the
paper fixes only that the new allocation is integer.  Reading (DESIGN.md §3 #3):
largest remainder with ties to the lowest rank, so Σ stays exactly the target (Eq. 4).
Floor: clamp violators at `floor` and re-apportion the rest
proportionally to their original quotas, repeated until no rank violates.

Two entry points:
  hamilton_exact(num, den, total)      quotas num_i/den (exact integers; shard sizes D_i)
  hamilton(q, total, floor)            real fp64 quotas (controller, Eq. 10)
The fp64 operation order in `hamilton` is part of the definition (the C++ host library must
reproduce the same doubles bit for bit; DESIGN.md §3 #35).
"""

from __future__ import annotations

import math


def _largest_remainder_pick(fracs, remaining):
    """Indices of the `remaining` largest fractional parts; ties -> lowest index (stable sort)."""
    order = sorted(range(len(fracs)), key=lambda i: (-fracs[i], i))
    return set(order[:remaining])


def hamilton_exact(num, den: int, total: int):
    """Largest remainder over exact rational quotas num_i/den whose sum is `total`.

    base_i = floor(num_i/den); the total - Σbase leftover units go to the largest remainders
    num_i mod den, ties to the lowest index.  Pure integer arithmetic.
    """
    num = [int(x) for x in num]
    den = int(den)
    if den <= 0:
        raise ValueError("den must be positive")
    if sum(num) != total * den:
        raise ValueError("quotas must sum to total")
    base = [x // den for x in num]
    rem = [x % den for x in num]
    left = total - sum(base)
    pick = _largest_remainder_pick(rem, left)
    return [b + (1 if i in pick else 0) for i, b in enumerate(base)]


def _hamilton_plain(q, total: int):
    """Floor-free largest remainder over fp64 quotas (one pass)."""
    base = [int(math.floor(x)) for x in q]
    fracs = [x - math.floor(x) for x in q]          # exact in fp64 for x >= 0
    left = total - sum(base)
    if left < 0 or left > len(q):
        raise ArithmeticError(f"quotas inconsistent with total: leftover {left}")
    pick = _largest_remainder_pick(fracs, left)
    return [b + (1 if i in pick else 0) for i, b in enumerate(base)]


def hamilton(q, total: int, floor: int = 0):
    """Largest remainder over fp64 quotas q (Σq ≈ total) with a per-rank minimum `floor`.

    Step 1: a = plain largest remainder of q.  If every a_i >= floor, return a.
    Step 2: ranks with a_i < floor are fixed at floor; the remaining total T' = total - floor·|fixed|
            is re-apportioned among the other ranks with quotas q_i·T'/S (S = Σ of their original q,
            summed left to right in rank order; the product is formed first, then the division).
    Repeat step 2 until no rank violates.  Requires total >= len(q)·floor (else InfeasibleFloor).
    """
    n = len(q)
    if total < n * floor:
        raise ValueError("InfeasibleFloor")
    q = [float(x) for x in q]
    fixed = [False] * n
    while True:
        active = [i for i in range(n) if not fixed[i]]
        t_rem = total - floor * (n - len(active))
        if len(active) == n:
            qa = [q[i] for i in active]
        else:
            s = 0.0
            for i in active:
                s = s + q[i]
            qa = [(q[i] * float(t_rem)) / s for i in active]
        a = _hamilton_plain(qa, t_rem)
        viol = [active[j] for j in range(len(active)) if a[j] < floor]
        if not viol:
            out = [floor] * n
            for j, i in enumerate(active):
                out[i] = a[j]
            return out
        for i in viol:
            fixed[i] = True
