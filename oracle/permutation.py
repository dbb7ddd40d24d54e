"""O3 per-epoch permutation π_{seed,e} and O4 shard indices.  TEST INFRASTRUCTURE ONLY (see oracle/__init__.py).

The paper assigns "a corresponding proportion of training samples to each worker from the total
dataset" and redistributes the sub-datasets every epoch (Algorithm 1 step 3), but is
SILENT on shuffling.  Build-defined reading (DESIGN.md §3 #8):

  b = max(2, bitlen(N−1)) rounded up to even;  h = b/2;  mask = 2^h − 1
  F_k(R) = Philox4x32-10(ctr = (R, k, lo32(e), hi32(e)), key = (lo32(seed), hi32(seed)))[0] & mask
  feistel(x): (L, R) = (x >> h, x & mask); for k = 0..3: (L, R) <- (R, L xor F_k(R)); return (L << h) | R
  π(j): y = feistel(j); while y >= N: y = feistel(y)          (cycle walking)
  shard r:  idx_r[t] = π(off_r + t),  t < len_r                   (O4)

Philox4x32-10 is the Salmon et al. (SC'11, Random123) counter-based generator: multipliers
0xD2511F53 / 0xCD9E8D57, Weyl key increments 0x9E3779B9 / 0xBB67AE85, 10 rounds.  Pinned by the
published known-answer vectors (tests/golden/philox4x32_10_kat.txt).  The π values themselves are
pinned only by bijectivity / uniformity invariants and by this written definition (parity of the
values is "definition-pinned": no paper value exists).
Vectorised with numpy uint32/uint64 integer arithmetic; no floating point anywhere.
"""

from __future__ import annotations

import numpy as np

PHILOX_M0 = 0xD2511F53
PHILOX_M1 = 0xCD9E8D57
PHILOX_W0 = 0x9E3779B9
PHILOX_W1 = 0xBB67AE85
_U32 = 0xFFFFFFFF


def philox4x32_10(ctr, key):
    """Philox4x32-10 on arrays.  ctr: 4 uint32 arrays (broadcastable); key: 2 python ints / arrays.

    Round:  (hi0, lo0) = M0·c0;  (hi1, lo1) = M1·c2;
            c = (hi1 ^ c1 ^ k0,  lo1,  hi0 ^ c3 ^ k1,  lo0)
    Key schedule between rounds: k0 += W0, k1 += W1 (mod 2^32).  Returns 4 uint32 arrays.
    """
    c0, c1, c2, c3 = (np.asarray(c, dtype=np.uint64) & _U32 for c in ctr)
    k0 = np.uint64(int(key[0]) & _U32)
    k1 = np.uint64(int(key[1]) & _U32)
    m0 = np.uint64(PHILOX_M0)
    m1 = np.uint64(PHILOX_M1)
    mask = np.uint64(_U32)
    s32 = np.uint64(32)
    for rnd in range(10):
        if rnd > 0:
            k0 = np.uint64((int(k0) + PHILOX_W0) & _U32)
            k1 = np.uint64((int(k1) + PHILOX_W1) & _U32)
        p0 = m0 * c0
        p1 = m1 * c2
        hi0, lo0 = p0 >> s32, p0 & mask
        hi1, lo1 = p1 >> s32, p1 & mask
        c0, c1, c2, c3 = (hi1 ^ c1 ^ k0) & mask, lo1, (hi0 ^ c3 ^ k1) & mask, lo0
    return tuple(x.astype(np.uint32) for x in (c0, c1, c2, c3))


def feistel_params(N: int):
    """(b, h, mask): domain 2^b >= N with b even, b >= 2."""
    if N < 1:
        raise ValueError("N >= 1")
    b = max(2, int(N - 1).bit_length())
    if b % 2:
        b += 1
    h = b // 2
    if h > 32:
        raise ValueError("N too large for a 32-bit-half Feistel network")
    return b, h, (1 << h) - 1


def feistel(x, N: int, seed: int, epoch: int):
    """One pass of the 4-round balanced Feistel network on the 2^b domain (uint64 arrays)."""
    _, h, mask = feistel_params(N)
    x = np.asarray(x, dtype=np.uint64)
    sh = np.uint64(h)
    m = np.uint64(mask)
    L = x >> sh
    R = x & m
    key = (seed & _U32, (seed >> 32) & _U32)
    e_lo = np.uint64(epoch & _U32)
    e_hi = np.uint64((epoch >> 32) & _U32)
    for k in range(4):
        f = philox4x32_10((R, np.uint64(k), e_lo, e_hi), key)[0].astype(np.uint64) & m
        L, R = R, L ^ f
    return (L << sh) | R


def permute(j, N: int, seed: int, epoch: int):
    """π_{seed,epoch}(j) for an array of positions j in [0, N), by cycle walking."""
    j = np.asarray(j, dtype=np.uint64)
    y = feistel(j, N, seed, epoch)
    todo = np.nonzero(y >= np.uint64(N))[0]
    while todo.size:
        y[todo] = feistel(y[todo], N, seed, epoch)
        todo = todo[y[todo] >= np.uint64(N)]
    return y.astype(np.int64)


def shard_indices(N: int, off: int, length: int, seed: int, epoch: int):
    """O4: idx[t] = π(off + t) for t < length."""
    return permute(np.arange(off, off + length, dtype=np.uint64), N, seed, epoch)


def shard_steps(N: int, B: int, o: int, n: int, seed: int, epoch: int, step0: int, nsteps: int):
    """Step-interleaved shard (DESIGN.md §3 #43): aggregation step s owns the permuted
    positions [s·B, (s+1)·B) and the rank takes the n of them starting at o = g·Σ_{j<r} w_j:
    idx[(s − step0)·n + t] = π(s·B + o + t) for step0 <= s < step0 + nsteps, t < n."""
    pos = [s * B + o + t for s in range(step0, step0 + nsteps) for t in range(n)]
    return permute(np.array(pos, dtype=np.uint64), N, seed, epoch)
