"""O7 linear-model closed form.  TEST INFRASTRUCTURE ONLY (see oracle/__init__.py).

Convergence analysis (§3.1.2, Eq. 1): with N = Σ_i minibatch·w_i, the aggregated update is
the mean gradient over all N samples, so the allocation does not change the trajectory.  For
logistic regression without bias (BASELINE configs[0]; DESIGN.md §3 #30):

    loss(θ; X, y) = mean_j −[y_j log σ(x_j·θ) + (1−y_j) log(1−σ(x_j·θ))]
    ∇ = Xᵀ(σ(Xθ) − y) / n                       (local mean gradient over n rows)
    Σ_r (n_r/B)·g_r = ∇ over the union of the step's rows             (Eq. 1)
    θ ← θ − η(∇ + λθ)                                                   (SGD, wd λ)

fp64 throughout.  Pins: central finite differences of `loss` (gradient formula), and the exact
identity above checked against the full-batch gradient of the union (tests/test_oracle_linmodel.py).
"""

from __future__ import annotations

import numpy as np


def sigmoid(z):
    return 1.0 / (1.0 + np.exp(-z))


def loss(theta, X, y):
    z = X @ theta
    # log σ(z) = −log(1+e^{−z}); log(1−σ(z)) = −log(1+e^{z})
    return float(np.mean(y * np.logaddexp(0.0, -z) + (1.0 - y) * np.logaddexp(0.0, z)))


def grad_mean(theta, X, y):
    """Local mean gradient over the rows of X."""
    return X.T @ (sigmoid(X @ theta) - y) / X.shape[0]


def sgd_step(theta, g, lr, wd=0.0):
    return theta - lr * (g + wd * theta)


def step_rows(idx_shards, n_local, step):
    """Row ids rank r uses at aggregation `step`: its shard positions [step·n_r, (step+1)·n_r)."""
    return [np.asarray(idx)[step * n:(step + 1) * n] for idx, n in zip(idx_shards, n_local)]


def weighted_step_gradient(theta, X, y, rows_per_rank):
    """Σ_r (n_r/Σn)·g_r with g_r the local mean gradient of rank r's rows (plain definition)."""
    n = [len(r) for r in rows_per_rank]
    tot = sum(n)
    out = np.zeros_like(theta)
    for rows, nr in zip(rows_per_rank, n):
        if nr:
            out += (nr / tot) * grad_mean(theta, X[rows], y[rows])
    return out


def trajectory(X, y, idx_shards, n_local, steps, lr, wd=0.0, theta0=None):
    """θ_0 = 0 (or theta0) and `steps` SGD updates with the weighted step gradient (O7)."""
    theta = np.zeros(X.shape[1]) if theta0 is None else np.array(theta0, dtype=np.float64)
    out = [theta.copy()]
    for s in range(steps):
        g = weighted_step_gradient(theta, X, y, step_rows(idx_shards, n_local, s))
        theta = sgd_step(theta, g, lr, wd)
        out.append(theta.copy())
    return out
