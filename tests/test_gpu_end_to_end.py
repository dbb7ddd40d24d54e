"""End-to-end parity for BASELINE configs[0] (C1): 2 workers, 1,000-sample synthetic data set, 1,024-param
logistic regression, static ratio 1:3, 10 aggregation steps.

GPU path: pr_alloc_init -> pr_shard_indices (K1) -> per step pr_gather_rows (K2, fp32 rows) -> each rank's
local mean gradient X_rᵀ(σ(X_r θ) − y_r)/n_r (torch fp32 on the GPU, the harness's a4) ->
pr_weighted_allreduce_local (K3) -> SGD.  Oracle: allocation + permutation + O7 closed form in fp64
(Eq. 1: the weighted average of the shard means equals the full-batch gradient).
"""

import numpy as np
import pytest
import torch

import synth
from oracle import allocation as OA
from oracle import linmodel as OL
from oracle import permutation as OP

pytestmark = pytest.mark.gpu
pr = pytest.importorskip("paper_2111_08272_b200")


@pytest.fixture(scope="module", autouse=True)
def _cuda():
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")


@pytest.mark.parametrize("ratios", [[1, 3], [2, 2], [3, 1]])
def test_c1_logistic_regression_trajectory(ratios):
    N, D, C, g, steps, lr, seed, epoch = 1000, 1024, 4, 25, 10, 0.1, 1234, 0
    X, y, _ = synth.logistic_problem(N, D)
    # ---- GPU path through the ABI -----------------------------------------------------------------
    a = pr.alloc_init(N, ratios, C=C, g=g)
    v = a.view()
    assert v["n"] == [g * r for r in ratios] and v["S"] == 10
    P = len(ratios)
    dX = torch.from_numpy(X.astype(np.float32)).cuda()
    dy = torch.from_numpy(y.astype(np.float32)).cuda()
    comms = pr.comm_init_local(P, 0, pr.comm_config(channels=2, watchdog_ns=5_000_000_000))
    idx = []
    for r in range(P):
        t = torch.empty(v["len"][r], dtype=torch.int64, device="cuda")
        pr.shard_indices(a, r, epoch, seed, t)
        idx.append(t)
    theta = torch.zeros(D, dtype=torch.float32, device="cuda")
    grads_gpu, thetas_gpu = [], [theta.clone()]
    rows_buf = [torch.empty((v["n"][r], D), dtype=torch.float32, device="cuda") for r in range(P)]
    for s in range(steps):
        bufs = []
        for r in range(P):
            n = v["n"][r]
            pr.gather_rows(dX, N, D * 4, idx[r][s * n:], n, rows_buf[r])               # K2 (COPY)
            yr = dy[idx[r][s * n:(s + 1) * n]]
            xr = rows_buf[r]
            bufs.append(xr.t() @ (torch.sigmoid(xr @ theta) - yr) / n)                 # local mean (a4)
        pr.weighted_allreduce_local(comms, bufs, v["n"])                               # K3
        torch.cuda.synchronize()
        assert torch.equal(bufs[0], bufs[1])
        grads_gpu.append(bufs[0].double().cpu().numpy())
        theta = theta - lr * bufs[0]                                                   # Eq. 1
        thetas_gpu.append(theta.clone())
    for c in comms:
        c.destroy()
    # ---- oracle -------------------------------------------------------------------------------------
    o = OA.alloc_init(N, ratios, C=C, g=g)
    shards = [OP.shard_indices(N, o.off[r], o.len[r], seed, epoch) for r in range(P)]
    assert all(np.array_equal(shards[r], idx[r].cpu().numpy()) for r in range(P))
    traj = OL.trajectory(X, y, shards, o.n, steps, lr)
    for s in range(steps):
        th = thetas_gpu[s].double().cpu().numpy()
        rows = OL.step_rows(shards, o.n, s)
        ref = OL.weighted_step_gradient(th, X, y, rows)                 # Eq. 1 at the GPU path's own θ_s
        # the same step from the full-batch closed form over the union of the step's rows (Eq. 1)
        full = OL.grad_mean(th, X[np.concatenate(rows)], y[np.concatenate(rows)])
        assert np.max(np.abs(ref - full)) <= 1e-12 * np.max(np.abs(full))
        # element by element, cancellation-aware over the per-sample terms of the sum (DESIGN.md §3 #45)
        allr = np.concatenate(rows)
        den = np.abs(X[allr]).T @ np.abs(OL.sigmoid(X[allr] @ th) - y[allr]) / len(allr)
        err = np.abs(grads_gpu[s] - ref)
        assert np.all(err <= 1e-5 * den), (s, float(np.max(err / den)))
        # θ_{s+1} = θ_s − η·ḡ_s: one fp32 multiply and one subtraction (torch) of the GPU's own ḡ_s
        nxt = thetas_gpu[s + 1].double().cpu().numpy()
        want = th - float(np.float32(lr)) * grads_gpu[s]
        assert np.all(np.abs(nxt - want) <= 2.0 ** -23 * (np.abs(want) + lr * np.abs(grads_gpu[s])) + 1e-45), s
    for s in range(steps + 1):
        tg = thetas_gpu[s].double().cpu().numpy()
        assert np.linalg.norm(tg - traj[s]) <= 1e-5 * max(1e-30, np.linalg.norm(traj[s])) + 1e-9
