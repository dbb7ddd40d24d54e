"""Oracle parity of the harness rows the bench runs through `Worker` (VERDICT r1 "What's weak" #3a, #3d).

Two processes on the one test GPU, one rank each (CUDA-IPC communicator, gloo bootstrap), run the REAL
Worker code path and hand their observations to the parent, which checks them against the oracle:

* C1 (BASELINE configs[0]: 2 workers, 1,000 samples, 1,024-weight logistic regression, ratio 1:3, 10
  steps) through `Worker.run_epoch`: K1 shard -> K2 epoch gather (fp32 COPY) -> a4 in microbatches of 10
  rows (3 and 8 microbatches per step, ragged last one: P:69 steps (1)-(3), each microbatch loss scaled by
  mb/n_r) inside the captured step graph -> K3 weighted ring allreduce -> a9.  Checked per step, element
  by element: the reduced gradient ḡ_s against the oracle's Eq. 1 weighted gradient (O7) at the rank's
  own θ_s, with the cancellation-aware metric of a sum over samples (DESIGN.md §3 #45); θ_{s+1} against
  the oracle's SGD step applied to (θ_s, ḡ_s) within its roundings; the shard against O4 bit for bit;
  θ identical on both ranks; and the fused a6-a9 kernel's θ trajectory against the composed one.
* N1: the bucketed allreduce launched from backward hooks inside the captured step
  (`overlap=True`), on a 3-layer fp32 MLP cut into several buckets.  Each step's reduced buffer is checked
  element by element against O6 (`oracle.wavg.weighted_average` of the ranks' local gradients, 1e-5
  cancellation-aware) and bucket by bucket against the ring-order replay (`ring_emulate`) bit for bit.
"""

import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

pytestmark = pytest.mark.gpu


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _spawn(target, world=2, timeout=600, **kw):
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    ps = [ctx.Process(target=target, args=(r, world, port, q), kwargs=kw) for r in range(world)]
    for p in ps:
        p.start()
    res = dict(q.get(timeout=timeout) for _ in ps)
    for p in ps:
        p.join(60)
    for r in range(world):
        if isinstance(res[r], str):
            raise AssertionError(f"rank {r}: {res[r]}")
    return res


def _c1_worker(rank, world, port, q, micro=10):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        import paper_2111_08272_b200 as pr
        from paper_2111_08272_b200.trainer import RunConfig, Worker

        torch.cuda.set_device(0)
        out = {}
        for fused in (False, True):
            comm = pr.comm_init(rank, world, 0, config=pr.comm_config(channels=2, watchdog_ns=60_000_000_000))
            cfg = RunConfig(N=1000, shape=(1024,), classes=2, model="logreg", ratios=[1, 3], C=4, g=25, lr=0.1,
                            wd=1e-4, micro=micro, bf16_compute=False, channels_last=False, fused_sgd=fused)
            w = Worker(cfg, rank, world, 0, comm)
            gbar, theta = [], []

            def params(wk):
                return torch.cat([p.detach().flatten() for p in wk.model.parameters()]).clone()

            def on_reduced(wk):
                gbar.append(wk.flat.detach().clone())
                theta.append(params(wk))

            def on_step(wk):
                if fused:
                    theta.append(params(wk))

            w.on_reduced, w.on_step = on_reduced, on_step
            theta0 = params(w)
            rec = w.run_epoch()
            torch.cuda.synchronize()
            final = params(w)
            idx = w.idx[:w.alloc.view()["len"][rank]].cpu().numpy()
            out[fused] = {"gbar": [g.cpu().numpy() for g in gbar], "theta": [t.cpu().numpy() for t in theta],
                          "theta0": theta0.cpu().numpy(), "final": final.cpu().numpy(), "idx": idx,
                          "S": rec["S"], "status": comm.status(), "n": w.alloc.view()["n"]}
            del w
            comm.destroy()
        q.put((rank, out))
    except Exception as e:  # noqa: BLE001
        import traceback

        q.put((rank, repr(e) + traceback.format_exc()))
    finally:
        dist.destroy_process_group()


def _per_sample_abs(theta, X, y, rows_per_rank):
    """Σ_r (n_r/B)·(1/n_r)·Σ_{i∈r} |x_ij|·|σ(x_i·θ) − y_i| = (1/B)·Σ_i |x_ij|·|res_i|: the absolute sum of the
    per-sample terms whose signed sum is ḡ_j — the cancellation-aware denominator for a gradient that is
    itself computed as a sum over samples in fp32 (DESIGN.md §3 #45)."""
    from oracle import linmodel as OL

    rows = np.concatenate(rows_per_rank)
    res = OL.sigmoid(X[rows] @ theta) - y[rows]
    return np.abs(X[rows]).T @ np.abs(res) / len(rows)


@pytest.mark.parametrize("micro", [10, 1024])
def test_c1_through_worker_matches_oracle_elementwise(micro):
    import synth
    from oracle import allocation as OA
    from oracle import linmodel as OL
    from oracle import permutation as OP

    res = _spawn(_c1_worker, micro=micro)
    N, D, lr, wd = 1000, 1024, float(np.float32(0.1)), float(np.float32(1e-4))
    X, y, _ = synth.logistic_problem(N, D)
    o = OA.alloc_init(N, [1, 3], C=4, g=25)
    shards = [OP.shard_indices(N, o.off[r], o.len[r], 1234, 0) for r in range(2)]
    for r in range(2):
        assert res[r][False]["status"] == 0 and res[r][True]["status"] == 0
        assert np.array_equal(res[r][False]["idx"], shards[r]) and res[r][False]["n"] == o.n
    plain0, plain1 = res[0][False], res[1][False]
    S = plain0["S"]
    assert S == 10 and len(plain0["gbar"]) == S and not np.any(plain0["theta0"])           # θ_0 = 0 (C1)
    for s in range(S):
        # the ranks hold the same reduced gradient and the same parameters (direct all-gather)
        assert np.array_equal(plain0["gbar"][s], plain1["gbar"][s])
        assert np.array_equal(plain0["theta"][s], plain1["theta"][s])
        th = plain0["theta"][s].astype(np.float64)
        rows = OL.step_rows(shards, o.n, s)
        ref = OL.weighted_step_gradient(th, X, y, rows)                                        # Eq. 1 (O7)
        den = _per_sample_abs(th, X, y, rows)
        err = np.abs(plain0["gbar"][s].astype(np.float64) - ref)
        assert np.all(err <= 1e-5 * den), (s, float(np.max(err / den)))
        # a9: θ_{s+1} = θ_s − η(ḡ_s + λθ_s) within the roundings of the fp32 update (torch SGD: 2 ops)
        nxt = plain0["theta"][s + 1] if s + 1 < S else plain0["final"]
        g = plain0["gbar"][s].astype(np.float64)
        want = OL.sgd_step(th, g, lr, wd)
        bound = 2.0 ** -23 * (np.abs(want) + lr * (np.abs(g) + wd * np.abs(th))) + 1e-45
        assert np.all(np.abs(nxt.astype(np.float64) - want) <= bound), s
    # the whole trajectory stays on the oracle's fp64 trajectory (normwise; drift is amplified by the Jacobian)
    traj = OL.trajectory(X, y, shards, o.n, S, lr, wd)
    tfinal = plain0["final"].astype(np.float64)
    assert np.linalg.norm(tfinal - traj[S]) <= 1e-5 * np.linalg.norm(traj[S])
    # the fused a6-a9 kernel (K7 inside K3) follows the same trajectory as ring + separate update
    fz0, fz1 = res[0][True], res[1][True]
    assert np.array_equal(fz0["final"], fz1["final"])
    for s in range(S):
        a, b = fz0["theta"][s].astype(np.float64), (plain0["theta"][s + 1] if s + 1 < S else plain0["final"])
        assert np.linalg.norm(a - b) <= 1e-5 * np.linalg.norm(b), s


def _n1_worker(rank, world, port, q, algo=0):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        import paper_2111_08272_b200 as pr
        from paper_2111_08272_b200.trainer import RunConfig, Worker

        torch.cuda.set_device(0)
        comm = pr.comm_init(rank, world, 0, config=pr.comm_config(channels=4, watchdog_ns=60_000_000_000, algo=algo))
        cfg = RunConfig(N=4096, shape=(1024,), classes=10, model="mlp", num_classes=10, ratios=[1, 3], C=4, g=64,
                        lr=0.05, wd=1e-4, micro=96, bf16_compute=False, channels_last=False, fused_sgd=False,
                        overlap=True, bucket_mb=0.004)
        w = Worker(cfg, rank, world, 0, comm)
        v = w.alloc.view()
        n_r, S = v["n"][rank], 4
        w.prepare(n_r)
        xe, ye, _, _ = w._data(0, n_r, v["S"], False)
        local, red, determ = [], [], True
        for s in range(S):
            x, y = xe[s * n_r:(s + 1) * n_r], ye[s * n_r:(s + 1) * n_r]
            w.compute(x, y, n_r)                          # eager, no bucket armed: this rank's local gradient
            g1 = w.flat.clone()
            w.flat.zero_()
            w.compute(x, y, n_r)
            determ = determ and bool(torch.equal(g1, w.flat))
            w.flat.zero_()
            w.compute_graphed(x, y, n_r)                  # the N1 step: backward + bucket allreduces, joined
            red.append(w.flat.clone())
            w.allreduce_and_update(n_r)                   # overlap without the fused update: SGD + reset
            local.append(g1)
        torch.cuda.synchronize()
        out = {"local": [t.cpu().numpy() for t in local], "red": [t.cpu().numpy() for t in red], "n": v["n"],
               "buckets": [(lo, hi) for lo, hi, _ in w._buckets], "determ": determ, "status": comm.status()}
        del w
        comm.destroy()
        q.put((rank, out))
    except Exception as e:  # noqa: BLE001
        import traceback

        q.put((rank, repr(e) + traceback.format_exc()))
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("algo", ["ring", "pull"])
def test_n1_overlapped_buckets_match_oracle_elementwise(algo):
    """N1's buckets through the ring and through the pull two-shot (AUTO's two-shot slot): every bucket the
    oracle's ring replay of its range."""
    from oracle import wavg as OW

    import paper_2111_08272_b200 as pr
    res = _spawn(_n1_worker, algo={"ring": pr.ALGO_RING, "pull": pr.ALGO_TWO_SHOT_PULL}[algo])
    r0, r1 = res[0], res[1]
    assert r0["status"] == 0 and r1["status"] == 0
    assert len(r0["buckets"]) >= 3, r0["buckets"]                     # the model is cut into several buckets
    n = r0["n"]
    for s in range(len(r0["red"])):
        assert np.array_equal(r0["red"][s], r1["red"][s])            # every bucket all-gathered to both ranks
        g = np.stack([r0["local"][s], r1["local"][s]])
        ref, den = OW.weighted_average(OW.as_f64(g, "f32"), n)        # O6 over the whole buffer
        err, zbad = OW.error_metric(r0["red"][s].astype(np.float64), ref, den)
        assert zbad == 0 and err <= 1e-5, (s, err)
        if r0["determ"] and r1["determ"]:
            # each bucket is one K3 call over [lo, hi): its bits are the ring-order replay of that range
            for lo, hi in r0["buckets"]:
                emu = OW.ring_emulate(np.ascontiguousarray(g[:, lo:hi]), n, "f32")
                assert np.array_equal(r0["red"][s][lo:hi], emu), (s, lo, hi)


def _n1_fused_worker(rank, world, port, q, algo=0):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        import paper_2111_08272_b200 as pr
        from paper_2111_08272_b200.trainer import RunConfig, Worker

        torch.cuda.set_device(0)
        torch.manual_seed(5)
        comm = pr.comm_init(rank, world, 0, config=pr.comm_config(channels=4, watchdog_ns=60_000_000_000, algo=algo))
        cfg = RunConfig(N=4096, shape=(1024,), classes=10, model="mlp", num_classes=10, ratios=[1, 3], C=4, g=64,
                        lr=0.05, wd=1e-4, micro=96, bf16_compute=False, channels_last=False, fused_sgd=True,
                        overlap=True, bucket_mb=0.004)
        w = Worker(cfg, rank, world, 0, comm)
        v = w.alloc.view()
        n_r = v["n"][rank]
        w.prepare(n_r)
        xe, ye, _, _ = w._data(0, n_r, v["S"], False)
        theta0 = w.pflat.clone()
        for s in range(4):
            w.compute_graphed(xe[s * n_r:(s + 1) * n_r], ye[s * n_r:(s + 1) * n_r], n_r)
            w.allreduce_and_update(n_r)                   # every bucket's update ran fused with its allreduce
        torch.cuda.synchronize()
        out = {"theta0": theta0.cpu().numpy(), "theta": w.pflat.cpu().numpy(), "status": comm.status(),
               "grad_zero": bool(torch.count_nonzero(w.flat) == 0)}
        del w
        comm.destroy()
        q.put((rank, out))
    except Exception as e:  # noqa: BLE001
        import traceback

        q.put((rank, repr(e) + traceback.format_exc()))
    finally:
        dist.destroy_process_group()


def test_n1_fused_buckets_pull_equals_ring():
    """N1 with the update fused per bucket (two processes over IPC): the pull two-shot's fused kernel and the
    ring's fused kernel give the same θ bit for bit, identical on both ranks, gradients reset."""
    import paper_2111_08272_b200 as pr

    ring = _spawn(_n1_fused_worker, algo=pr.ALGO_RING)
    pull = _spawn(_n1_fused_worker, algo=pr.ALGO_TWO_SHOT_PULL)
    for res in (ring, pull):
        assert res[0]["status"] == 0 and res[1]["status"] == 0
        assert np.array_equal(res[0]["theta"], res[1]["theta"])
        assert res[0]["grad_zero"] and res[1]["grad_zero"]
    assert np.array_equal(ring[0]["theta0"], pull[0]["theta0"])        # same initial parameters
    assert not np.array_equal(ring[0]["theta"], ring[0]["theta0"])     # the steps moved θ
    assert np.array_equal(ring[0]["theta"], pull[0]["theta"])


def _n3_async_worker(rank, world, port, q):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        import paper_2111_08272_b200 as pr
        from paper_2111_08272_b200.trainer import RunConfig, Worker

        torch.cuda.set_device(0)
        comm = pr.comm_init(rank, world, 0, config=pr.comm_config(channels=2, watchdog_ns=60_000_000_000))
        # K6 asynchronous: device value in, pinned host out, no synchronisation inside the call
        d = torch.tensor(1.5 + rank, dtype=torch.float64, device="cuda")
        h = torch.zeros(world, dtype=torch.float64, pin_memory=True)
        comm.allgather_f64_async(d, h)
        ev = torch.cuda.Event()
        ev.record()
        ev.synchronize()
        ag_ok = h.tolist() == [1.5 + r for r in range(world)]
        sync_ok = comm.allgather_f64(7.0 + rank) == [7.0 + r for r in range(world)]
        # N3 with the asynchronous exchange: rank 0 emulated 3x slower; the replicated controller must move
        # units to rank 1 and every rank must take the same decisions
        cfg = RunConfig(N=4096, shape=(1024,), classes=10, model="mlp", num_classes=10, ratios=[1, 1], C=16, g=16,
                        micro=256, bf16_compute=False, channels_last=False, adaptive=True, adapt_every=4,
                        adapt_lag=1, slowdown=[3.0, 1.0], policy={"never_freeze": True})
        w = Worker(cfg, rank, world, 0, comm)
        recs = [w.run_epoch() for _ in range(2)]
        torch.cuda.synchronize()
        hist = [list(map(int, w.alloc.history(i))) for i in range(w.alloc.view()["hist_len"])]
        segs = [(sg["w"], sg.get("t_s")) for r_ in recs for sg in r_["segments"]]
        out = {"ag_ok": ag_ok, "sync_ok": sync_ok, "hist": hist, "segs": segs, "status": comm.status(),
               "t_s": [r_["t_s"] for r_ in recs]}
        del w
        comm.destroy()
        q.put((rank, out))
    except Exception as e:  # noqa: BLE001
        import traceback

        q.put((rank, repr(e) + traceback.format_exc()))
    finally:
        dist.destroy_process_group()


def test_n3_asynchronous_exchange_two_processes():
    """K6 without a host synchronisation (pr_stamp_seconds + pr_comm_allgather_f64_async) and N3's one-segment-
    lag controller on it: both ranks see the same times, take the same decisions, and the slow rank sheds
    units (VERDICT r1 "What's weak" #11)."""
    res = _spawn(_n3_async_worker)
    r0, r1 = res[0], res[1]
    assert r0["ag_ok"] and r1["ag_ok"] and r0["sync_ok"] and r1["sync_ok"]
    assert r0["status"] == 0 and r1["status"] == 0
    assert r0["hist"] == r1["hist"] and r0["segs"] == r1["segs"]
    assert len(r0["hist"]) > 3 and r0["hist"][0] == [8, 8]
    last = r0["hist"][-1]
    assert sum(last) == 16 and last[1] > last[0], r0["hist"]
    for wv, ts in r0["segs"]:
        assert ts is not None and len(ts) == 2 and min(ts) > 0
    assert min(r0["t_s"]) > 0 and min(r1["t_s"]) > 0
