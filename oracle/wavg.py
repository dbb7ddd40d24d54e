"""O6 sample-count-weighted average of the per-rank gradients.  TEST INFRASTRUCTURE ONLY (see oracle/__init__.py).

Eq. 1: w_k = w_{k−1} − η·(1/N)·Σ_{i=1..N} ∇f_i(w_{k−1}), with N = Σ_i minibatch·w_i.
If rank r holds the local MEAN gradient g_r over its n_r samples (DESIGN.md §3 #11), the global mean is

    ref[j] = Σ_r (n_r / Σn) · g_r[j]                                   (plain definition, fp64)

computed here over the dtype-rounded inputs.  A rank with n_r = 0 contributes nothing (§3 #33).

Error metric (DESIGN.md §3 #16, cancellation-aware):  err[j] = |y[j] − ref[j]| / Σ_r |s_r·g_r[j]|;
where the denominator is 0, y[j] must be exactly 0.

ring_emulate(): the bit-exact ring-order replay (oracle/ring_emu.c) for the chunking rule
cs = round_up(ceil(count/P), 16 bytes / element size) (DESIGN.md §3 #14).
"""

from __future__ import annotations

import ctypes
import os
import subprocess

import numpy as np

from .gather import bf16_bits_to_f32

_HERE = os.path.dirname(os.path.abspath(__file__))
_SO = os.path.join(_HERE, "libringemu.so")
_lib = None


def build_c(force: bool = False) -> str:
    """Compile oracle/ring_emu.c (plain C, -O2 -ffp-contract=off) into oracle/libringemu.so."""
    src = os.path.join(_HERE, "ring_emu.c")
    if force or not os.path.exists(_SO) or os.path.getmtime(_SO) < os.path.getmtime(src):
        subprocess.check_call(["gcc", "-O2", "-ffp-contract=off", "-fno-tree-vectorize", "-shared",
                               "-fPIC", "-o", _SO, src, "-lm"])
    return _SO


def _load():
    global _lib
    if _lib is None:
        _lib = ctypes.CDLL(build_c())
        i64, ip = ctypes.c_int64, ctypes.c_void_p
        _lib.ring_emulate_f32.argtypes = [ctypes.c_int, i64, i64, ip, ip, ip, ip]
        _lib.ring_emulate_bf16.argtypes = [ctypes.c_int, i64, i64, ip, ip, ip, ip]
    return _lib


def weights(n_local):
    """s_r = n_r / Σn in fp64 (Eq. 1 with N = Σn)."""
    total = sum(int(x) for x in n_local)
    if total == 0:
        raise ZeroDivisionError("ZeroSampleCount (S:317)")
    return [int(x) / total for x in n_local]


def weights_f32(n_local):
    """The fp32 weights a kernel multiplies by: fp32(n_r / Σn) with the division in fp64."""
    return np.array(weights(n_local), dtype=np.float64).astype(np.float32)


def as_f64(g, dtype: str):
    """Dtype-rounded inputs widened to fp64. g: float32 array, or uint16 bf16 bits when dtype='bf16'."""
    if dtype == "bf16":
        return bf16_bits_to_f32(g).astype(np.float64)
    return np.asarray(g, dtype=np.float32).astype(np.float64)


def weighted_average(g64, n_local):
    """ref = Σ_r (n_r/Σn)·g_r in fp64 (g64: [P, L] float64).  Skips ranks with n_r = 0."""
    s = weights(n_local)
    ref = np.zeros(g64.shape[1], dtype=np.float64)
    den = np.zeros(g64.shape[1], dtype=np.float64)
    for r in range(g64.shape[0]):
        if int(n_local[r]) == 0:
            continue
        term = s[r] * g64[r]
        ref += term
        den += np.abs(term)
    return ref, den


def error_metric(y64, ref, den):
    """Cancellation-aware elementwise error (DESIGN.md §3 #16).  Returns (max_err, zero_violations)."""
    y64 = np.asarray(y64, dtype=np.float64)
    nz = den > 0
    err = np.zeros_like(ref)
    err[nz] = np.abs(y64[nz] - ref[nz]) / den[nz]
    zero_bad = int(np.count_nonzero(y64[~nz] != 0.0))
    return (float(err.max()) if err.size else 0.0), zero_bad


def chunk_elems(count: int, P: int, elem_bytes: int) -> int:
    """cs = round_up(ceil(count/P), 16/elem_bytes)  (DESIGN.md §3 #14)."""
    vec = 16 // elem_bytes
    per = -(-count // P)
    return -(-per // vec) * vec


def ring_emulate(g, n_local, dtype: str = "f32"):
    """Bit-exact ring-order replay.  g: [P, L] float32 (dtype f32) or uint16 bf16 bits (dtype bf16)."""
    lib = _load()
    P, L = g.shape
    s = weights_f32(n_local)
    act = np.array([1 if int(x) > 0 else 0 for x in n_local], dtype=np.int32)
    if dtype == "f32":
        g = np.ascontiguousarray(g, dtype=np.float32)
        out = np.zeros(L, dtype=np.float32)
        cs = chunk_elems(L, P, 4)
        lib.ring_emulate_f32(P, L, cs, g.ctypes.data, s.ctypes.data, act.ctypes.data, out.ctypes.data)
    elif dtype == "bf16":
        g = np.ascontiguousarray(g, dtype=np.uint16)
        out = np.zeros(L, dtype=np.uint16)
        cs = chunk_elems(L, P, 2)
        lib.ring_emulate_bf16(P, L, cs, g.ctypes.data, s.ctypes.data, act.ctypes.data, out.ctypes.data)
    else:
        raise ValueError(dtype)
    return out
