"""Pins for oracle O3 (per-epoch permutation) and O4 (shard indices).

Philox4x32-10 is pinned by the published Random123 known-answer vectors; π by bijectivity,
near-uniformity on tiny domains, and the regression vectors an independent implementation of the
same written definition produced during the survey ("Feistel cycle-walk π").
"""

import math

import numpy as np

from conftest import read_golden
from oracle import allocation as A
from oracle import permutation as PM


def test_philox_known_answers():
    rows = read_golden("philox4x32_10_kat.txt")
    assert len(rows) == 3
    for (line,) in rows:
        lhs, rhs = line.split("->")
        v = [int(x, 16) for x in lhs.split()]
        exp = [int(x, 16) for x in rhs.split()]
        out = PM.philox4x32_10(([v[0]], [v[1]], [v[2]], [v[3]]), (v[4], v[5]))
        assert [int(o[0]) for o in out] == exp


def test_survey_regression_vectors():
    """N=10, seed 1234: epoch 0 and 1."""
    assert PM.permute(np.arange(10), 10, 1234, 0).tolist() == [6, 0, 8, 4, 1, 5, 9, 3, 7, 2]
    assert PM.permute(np.arange(10), 10, 1234, 1).tolist() == [3, 4, 1, 0, 5, 6, 9, 2, 7, 8]


def test_feistel_is_bijection_on_domain():
    for N in (1, 2, 5, 16, 17, 1000, 4096):
        b, _, _ = PM.feistel_params(N)
        dom = np.arange(1 << b, dtype=np.uint64)
        y = PM.feistel(dom, N, 99, 3)
        assert np.array_equal(np.sort(y), dom)


def test_permutation_bijective_small_all():
    rng = np.random.Generator(np.random.PCG64(5))
    Ns = list(range(1, 257)) + sorted(set(int(x) for x in rng.integers(257, 4097, 60))) + [4096]
    for N in Ns:
        seed = int(rng.integers(0, 2 ** 63))
        ep = int(rng.integers(0, 2 ** 40))
        y = PM.permute(np.arange(N), N, seed, ep)
        assert np.array_equal(np.sort(y), np.arange(N)), N


def test_permutation_bijective_large():
    for N in (50000, 1281167):
        y = PM.permute(np.arange(N), N, 1234, 7)
        assert np.array_equal(np.sort(y), np.arange(N))


def test_permutation_uniform_tiny():
    """N=3: all 6 permutations appear over 6000 epochs, chi-square near uniform."""
    counts = {}
    for e in range(6000):
        key = tuple(PM.permute(np.arange(3), 3, 42, e).tolist())
        counts[key] = counts.get(key, 0) + 1
    assert len(counts) == 6
    chi2 = sum((c - 1000) ** 2 / 1000 for c in counts.values())
    assert chi2 < 25.0   # 5 dof; p ~ 1e-4


def test_epochs_and_seeds_differ():
    a = PM.permute(np.arange(1000), 1000, 1, 0)
    b = PM.permute(np.arange(1000), 1000, 1, 1)
    c = PM.permute(np.arange(1000), 1000, 2, 0)
    assert not np.array_equal(a, b) and not np.array_equal(a, c)


def test_shards_disjoint_and_cover():
    for N, ratios, C in ((1000, [1, 3], 4), (50000, [1, 1, 1, 1, 2, 2, 4, 4], 64), (12345, [3, 5, 7], 15)):
        a = A.alloc_init(N, ratios, C=C, g=1)
        shards = [PM.shard_indices(N, a.off[r], a.len[r], 77, 2) for r in range(a.P)]
        allv = np.concatenate(shards)
        assert allv.size == N and np.array_equal(np.sort(allv), np.arange(N))
        assert all(s.size == a.len[r] for r, s in enumerate(shards))


def test_shard_steps_reduces_to_contiguous_shard_at_one_rank():
    # P = 1 (w = [C]): step s takes positions [s·B, (s+1)·B), so S steps are the first S·B of the shard
    N, C, g = 5000, 4, 25
    a = A.alloc_init(N, [1], C=C, g=g)
    B, S = g * C, N // (g * C)
    got = PM.shard_steps(N, B, 0, B, 3, 1, 0, S)
    assert np.array_equal(got, PM.shard_indices(N, 0, a.len[0], 3, 1)[:S * B])


def test_shard_steps_disjoint_under_reallocation():
    # the allocation changes every 3 steps; each step's rows over ranks are exactly π([s·B, (s+1)·B))
    N, C, g = 6000, 8, 10
    B, S = g * C, N // (g * C)
    plans = [[1, 1, 2, 4], [4, 2, 1, 1], [2, 2, 2, 2], [1, 1, 1, 5]]
    seen = []
    for s in range(S):
        w = plans[(s // 3) % len(plans)]
        o = np.concatenate([[0], np.cumsum(w)[:-1]]) * g
        step = [PM.shard_steps(N, B, int(o[r]), g * w[r], 5, 2, s, 1) for r in range(4)]
        assert sorted(np.concatenate(step).tolist()) == sorted(PM.shard_indices(N, s * B, B, 5, 2).tolist())
        seen.extend(np.concatenate(step).tolist())
    assert len(set(seen)) == S * B


def test_shard_steps_segments_compose():
    N, B, o, n = 10007, 96, 32, 40
    whole = PM.shard_steps(N, B, o, n, 11, 4, 7, 20)
    parts = np.concatenate([PM.shard_steps(N, B, o, n, 11, 4, 7, 5), PM.shard_steps(N, B, o, n, 11, 4, 12, 15)])
    assert np.array_equal(whole, parts)
    assert np.array_equal(whole[:n], PM.shard_indices(N, 7 * B + o, n, 11, 4))
