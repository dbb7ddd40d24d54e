"""O5 step-batch gather.  TEST INFRASTRUCTURE ONLY (see oracle/__init__.py).

Algorithm 1 step 4: "Proportionally draw samples from the sub-data set for training"; static
allocation: "Worker i draws w_i samples from subdataset".  The paper is silent on the
data-plane details, so the operation is build-defined (DESIGN.md §3 #38):

  for step s, rows t' in [0, n):  out[t', :] = op(X[idx[s·n + t'], :]),   lab[t'] = Y[idx[s·n + t']]

  COPY               bit copy of the row bytes
  U8_TO_F32_AFFINE   (float32(x) − shift_c) · scale_c, two separately rounded fp32 operations (no FMA)
  U8_TO_BF16_AFFINE  the same fp32 value, then round-to-nearest-even to bfloat16
  channel c = k // plane for element k of a CHW row (plane = H·W)
  layout "hwc" (channels-last output): element (c, p) of the row is stored at p·C + c

Pins: COPY is the identity on bytes; the affine value is within 0.5 ulp(fp32) of each rounding of the
exact fp64 value; RNE-to-bf16 agrees with torch's CPU float32->bfloat16 conversion (a library routine).
"""

from __future__ import annotations

import numpy as np

COPY = 0
U8_TO_F32_AFFINE = 1
U8_TO_BF16_AFFINE = 2


def f32_to_bf16_bits(x):
    """Round-to-nearest-even float32 -> bfloat16, returned as uint16 bit patterns.

    Definition: keep the top 16 bits of the IEEE binary32 encoding after adding 0x7FFF + lsb, where
    lsb is bit 16 of the input (ties go to the even result).  NaN maps to a quiet NaN.
    """
    b = np.ascontiguousarray(x, dtype=np.float32).view(np.uint32).astype(np.uint64)
    lsb = (b >> np.uint64(16)) & np.uint64(1)
    r = ((b + np.uint64(0x7FFF) + lsb) >> np.uint64(16)).astype(np.uint16)
    nan = np.isnan(np.asarray(x, dtype=np.float32))
    if nan.any():
        r = np.where(nan, ((b >> np.uint64(16)).astype(np.uint16) | np.uint16(0x0040)), r)
    return r


def bf16_bits_to_f32(bits):
    """Exact widening bfloat16 (uint16 bits) -> float32."""
    return (np.asarray(bits, dtype=np.uint16).astype(np.uint32) << np.uint32(16)).view(np.float32)


def gather_rows(X, idx, op: int = COPY, scale=None, shift=None, plane: int = 1, Y=None, layout: str = "chw"):
    """Gather rows X[idx] and apply `op`.  X: [N, R] (uint8 for the affine ops).  Returns (out, lab).
    layout="hwc": the affine output row is stored channels-last (element (c, p) at p·C + c)."""
    X = np.asarray(X)
    idx = np.asarray(idx, dtype=np.int64)
    rows = X.reshape(X.shape[0], -1)[idx]
    lab = None if Y is None else np.asarray(Y)[idx]
    if op == COPY:
        return rows.copy(), lab
    if rows.dtype != np.uint8:
        raise TypeError("affine ops take uint8 rows")
    k = np.arange(rows.shape[1])
    ch = k // plane
    sc = np.asarray(scale, dtype=np.float32)[ch]
    sh = np.asarray(shift, dtype=np.float32)[ch]
    v = rows.astype(np.float32)
    v = np.subtract(v, sh, dtype=np.float32)      # first fp32 rounding
    v = np.multiply(v, sc, dtype=np.float32)      # second fp32 rounding
    if layout == "hwc":                           # channels-last: element (c, p) -> position p·C + c
        C = rows.shape[1] // plane
        v = np.ascontiguousarray(v.reshape(v.shape[0], C, plane).transpose(0, 2, 1)).reshape(v.shape[0], -1)
    elif layout != "chw":
        raise ValueError(layout)
    if op == U8_TO_F32_AFFINE:
        return v, lab
    if op == U8_TO_BF16_AFFINE:
        return f32_to_bf16_bits(v), lab
    raise ValueError(op)


def step_gather(X, idx_shard, step: int, n: int, **kw):
    """Rows of aggregation step `step`: positions [step·n, (step+1)·n) of the rank's shard."""
    return gather_rows(X, np.asarray(idx_shard)[step * n:(step + 1) * n], **kw)
