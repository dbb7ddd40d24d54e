"""Seeded synthetic input generators shared by the oracle tests, the GPU parity tests and bench.py.

This module holds NONE of the method's arithmetic (no allocation, permutation, gather, weighting or
reduction).  It only draws seeded random inputs with the shapes and distributions of the paper's
workloads (SURVEY.md §8(d) "Concrete synthetic inputs per config"):

* CIFAR-10-shaped images  uint8 [N, 3, 32, 32]   (paper §4: ResNet18/50, VGG on CIFAR10)
* ImageNet-shaped images  uint8 [N, 3, 224, 224] (VGG-16 with a 1000-class head, BASELINE configs[2])
* labels                  int64 uniform over the class count
* per-rank gradient buffers (Gaussian, or "mixed-scale" g·exp(3·N(0,1)) for precision tests)
* the 1,024-feature logistic-regression problem of BASELINE configs[0]

Both sides of every parity test receive the same arrays from here.
"""

from __future__ import annotations

import numpy as np

__all__ = [
    "images_u8",
    "labels",
    "gradients",
    "logistic_problem",
    "step_times",
]


def _rng(seed: int) -> np.random.Generator:
    return np.random.Generator(np.random.PCG64(int(seed)))


def images_u8(n: int, c: int = 3, h: int = 32, w: int = 32, seed: int = 0) -> np.ndarray:
    """Uniform 0..255 uint8 images in CHW layout, [n, c, h, w] ("uniform (seed 0)")."""
    return _rng(seed).integers(0, 256, size=(n, c, h, w), dtype=np.uint8)


def labels(n: int, classes: int = 10, seed: int = 1) -> np.ndarray:
    """Uniform class labels int64 [n] ("labels uniform 0..9 (seed 1)")."""
    return _rng(seed).integers(0, classes, size=(n,), dtype=np.int64)


def gradients(p: int, length: int, seed_base: int = 1000, kind: str = "gaussian") -> np.ndarray:
    """Per-rank gradient buffers float32 [p, length]; rank r uses seed seed_base + r.

    kind="gaussian": N(0, 1).  kind="mixed": N(0,1)·exp(3·N(0,1)) (mixed magnitudes, for precision).
    """
    out = np.empty((p, length), dtype=np.float32)
    for r in range(p):
        g = _rng(seed_base + r)
        x = g.standard_normal(length)
        if kind == "mixed":
            x = x * np.exp(3.0 * g.standard_normal(length))
        elif kind != "gaussian":
            raise ValueError(kind)
        out[r] = x.astype(np.float32)
    return out


def logistic_problem(n: int = 1000, d: int = 1024, seeds=(0, 1, 2)):
    """BASELINE configs[0]: X ~ N(0,1) [n,d] fp64; θ* ~ N(0, 1/d); labels y_j = [u_j < sigmoid(x_j·θ*)].

    The label draw uses a sigmoid only to synthesise a plausible data set; it is data generation, not
    the method (the method is the gradient / weighting, which lives in oracle/ and in the CUDA path).
    """
    X = _rng(seeds[0]).standard_normal((n, d))
    theta_star = _rng(seeds[1]).standard_normal(d) / np.sqrt(d)
    u = _rng(seeds[2]).random(n)
    y = (u < 1.0 / (1.0 + np.exp(-(X @ theta_star)))).astype(np.float64)
    return X, y, theta_star


def step_times(p: int, seed: int, lo: float = 0.5, hi: float = 5.0) -> np.ndarray:
    """Random positive per-rank epoch times (seconds), float64 [p], for controller property tests."""
    return _rng(seed).uniform(lo, hi, size=p)
