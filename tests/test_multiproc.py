"""World-size-2 tests of the N>1 path.

CPU (gloo, runs here): the replicated control plane — every rank computes the same allocation from the
same t_s allgather, shards are disjoint and cover the data set, and the byte-exchange callback that
bootstraps pr_comm_init (CUDA-IPC handle allgather) is a correct rank-ordered allgather.
GPU (marked): two processes on the one test GPU bootstrap a real pr_comm_init over CUDA IPC and run
the weighted allreduce (needs the two contexts to be co-resident; skipped if the box cannot).
"""

import ctypes
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _cpu_worker(rank, world, port, q):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        import paper_2111_08272_b200 as pr
        from oracle import allocation as A
        from oracle import permutation as PM

        # exchange callback = rank-ordered byte allgather
        fn = pr.torch_exchange()
        send = (b"rank%d-" % rank) * 3
        recv = ctypes.create_string_buffer(len(send) * world)
        rc = fn(None, ctypes.cast(ctypes.c_char_p(send), ctypes.c_void_p), len(send), ctypes.addressof(recv))
        assert rc == 0
        assert recv.raw == b"".join((b"rank%d-" % r) * 3 for r in range(world))

        # replicated controller: per-rank measured times -> allgather -> identical update everywhere
        a = pr.alloc_init(51200, [1] * world, C=64, g=16)
        speeds = [1000.0, 2000.0]
        for epoch in range(6):
            v = a.view()
            t_local = torch.tensor([v["S"] * v["n"][rank] / speeds[rank] + 0.01], dtype=torch.float64)
            allt = [torch.zeros(1, dtype=torch.float64) for _ in range(world)]
            dist.all_gather(allt, t_local)
            a.update([float(x) for x in allt])
        w = torch.tensor(a.view()["w"])
        ws = [torch.zeros_like(w) for _ in range(world)]
        dist.all_gather(ws, w)
        assert all(torch.equal(ws[0], x) for x in ws)
        v = a.view()
        assert sum(v["w"]) == 64 and v["w"][1] > v["w"][0]
        # each rank derives only its own shard; together they partition the data set
        mine = PM.shard_indices(v["N"], v["off"][rank], v["len"][rank], 7, 3)
        parts = [None] * world
        dist.all_gather_object(parts, mine.tolist())
        allv = np.concatenate([np.asarray(p, dtype=np.int64) for p in parts])
        assert np.array_equal(np.sort(allv), np.arange(v["N"]))
        q.put((rank, "ok"))
    except Exception as e:  # report to the parent
        q.put((rank, repr(e)))
    finally:
        dist.destroy_process_group()


def test_gloo_world2_control_plane():
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    ps = [ctx.Process(target=_cpu_worker, args=(r, 2, port, q)) for r in range(2)]
    for p in ps:
        p.start()
    res = dict(q.get(timeout=240) for _ in ps)
    for p in ps:
        p.join(60)
    assert res == {0: "ok", 1: "ok"}, res


def _gpu_worker(rank, world, port, q):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        import paper_2111_08272_b200 as pr
        import synth
        from oracle import wavg as W

        torch.cuda.set_device(0)
        bad = []
        # every algorithm over real CUDA-IPC peer windows; the LL ring also at forced system scope
        for algo, sys_scope in ((pr.ALGO_RING, False), (pr.ALGO_TWO_SHOT, False), (pr.ALGO_LL, False),
                                (pr.ALGO_LL, True), (pr.ALGO_ONESHOT, True), (pr.ALGO_TWO_SHOT_PULL, False),
                                (pr.ALGO_TWO_SHOT_PULL, True)):
            comm = pr.comm_init(rank, world, 0, config=pr.comm_config(channels=2, watchdog_ns=30_000_000_000,
                                                                      algo=algo, sys_scope=sys_scope))
            L = 4099
            g = synth.gradients(world, L, seed_base=11)
            buf = comm.alloc(L * 4, dtype=torch.float32)
            n = [3, 5]
            for _ in range(3):                      # repeated calls: counters / line flags advance
                buf.copy_(torch.from_numpy(g[rank]))
                pr.weighted_allreduce(comm, buf, n[rank])
            torch.cuda.synchronize()
            st = comm.status()
            ok = st == 0 and np.array_equal(buf.cpu().numpy(), W.ring_emulate(g, n, "f32"))
            t = comm.allgather_f64(1.5 + rank)
            ok = ok and t == [1.5, 2.5]
            if not ok:
                bad.append(f"algo={algo} sys={sys_scope} status={st}")
            if algo in (pr.ALGO_RING, pr.ALGO_TWO_SHOT_PULL) and not sys_scope:
                # rows a6-a9 fused (K7 in K3) over IPC: one [grad | theta] region per rank
                raw = comm.alloc(2 * 4100 * 4, dtype=torch.float32)
                gr, th = raw[:L], raw[4100:4100 + L]
                theta0 = torch.from_numpy(synth.gradients(1, L, seed_base=12)[0]).cuda()
                gr.copy_(torch.from_numpy(g[rank]))
                th.copy_(theta0)
                pr.weighted_allreduce_sgd(comm, gr, th, n[rank], 0.05, 1e-4)
                torch.cuda.synchronize()
                ref_g = torch.from_numpy(W.ring_emulate(g, n, "f32")).cuda()
                ref = theta0.clone()
                pr.sgd_update(ref, ref_g, 0.05, 1e-4)
                torch.cuda.synchronize()
                if not (comm.status() == 0 and torch.equal(th, ref) and torch.count_nonzero(gr) == 0):
                    bad.append(f"fused status={comm.status()}")
            dist.barrier()
            comm.destroy()
        # AUTO at a two-shot size, rank 0 on its registered buffer (-> pull two-shot), rank 1 on an unregistered
        # tensor (-> ring): the algorithm travels in the handshake, so both latch LENGTH_MISMATCH, no hang
        comm = pr.comm_init(rank, world, 0, config=pr.comm_config(channels=2, watchdog_ns=30_000_000_000,
                                                                  algo=pr.ALGO_AUTO))
        L = 1 << 18
        reg = comm.alloc(L * 4, dtype=torch.float32)
        buf = reg if rank == 0 else torch.zeros(L, device="cuda")
        buf.fill_(1.0 + rank)
        try:
            pr.weighted_allreduce(comm, buf, 1)
        except pr.PropringError:
            pass
        torch.cuda.synchronize()
        if comm.status() != pr.PR_ERR_LENGTH_MISMATCH or not bool((buf == 1.0 + rank).all()):
            bad.append(f"mixed kernels status={comm.status()}")
        dist.barrier()
        comm.destroy()
        # a registration that fails on any rank leaves nothing behind (the next one gets region 0
        # and the direct all-gather works); NVLS (N2) is set up or refused on every rank together
        comm = pr.comm_init(rank, world, 0, config=pr.comm_config(channels=2, watchdog_ns=30_000_000_000,
                                                                  algo=pr.ALGO_NVLS))
        try:
            comm.register(torch.zeros(1024, pin_memory=True))       # host memory: no CUDA-IPC handle
            bad.append("registering host memory succeeded")
        except pr.PropringError as e:
            if e.code != pr.PR_ERR_CUDA:
                bad.append(f"register error {e.code}")
        L = 4099
        g = synth.gradients(world, L, seed_base=21)
        n = [3, 5]
        buf = comm.alloc(L * 4, dtype=torch.float32)
        buf.copy_(torch.from_numpy(g[rank]))
        pr.weighted_allreduce(comm, buf, n[rank])                  # outside any NVLS region: the ring
        torch.cuda.synchronize()
        if not (comm.status() == 0 and np.array_equal(buf.cpu().numpy(), W.ring_emulate(g, n, "f32"))):
            bad.append(f"ring after failed register: status={comm.status()}")
        try:
            nv = comm.nvls_alloc(L * 4, dtype=torch.float32)
            nv_code = 0
        except pr.PropringError as e:
            nv, nv_code = None, e.code
        codes = [None] * world
        dist.all_gather_object(codes, nv_code)
        if len(set(codes)) != 1 or nv_code not in (0, pr.PR_ERR_UNSUPPORTED):
            bad.append(f"nvls codes {codes}")
        if nv is not None:                                         # a box with NVSwitch multicast
            nv.copy_(torch.from_numpy(g[rank]))
            pr.weighted_allreduce(comm, nv, n[rank])
            torch.cuda.synchronize()
            ref, den = W.weighted_average(W.as_f64(g, "f32"), n)
            err, zb = W.error_metric(nv.double().cpu().numpy(), ref, den)
            if not (comm.status() == 0 and zb == 0 and err <= 1e-5):
                bad.append(f"nvls err={err} status={comm.status()}")
        dist.barrier()
        comm.destroy()
        q.put((rank, "ok" if not bad else "; ".join(bad)))
    except Exception as e:
        q.put((rank, repr(e)))
    finally:
        dist.destroy_process_group()


@pytest.mark.gpu
def test_ipc_two_processes_one_gpu():
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    ps = [ctx.Process(target=_gpu_worker, args=(r, 2, port, q)) for r in range(2)]
    for p in ps:
        p.start()
    res = dict(q.get(timeout=300) for _ in ps)
    for p in ps:
        p.join(60)
    assert res == {0: "ok", 1: "ok"}, res


def _overlap_worker(rank, world, port, q):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        import gc

        import paper_2111_08272_b200 as pr
        from paper_2111_08272_b200.trainer import RunConfig, Worker

        torch.cuda.set_device(0)
        res, p0 = {}, None
        for ov in (False, True):
            comm = pr.comm_init(rank, world, 0, config=pr.comm_config(watchdog_ns=60_000_000_000))
            cfg = RunConfig(N=2048, ratios=[1, 3], C=4, g=64, micro=1024, overlap=ov, bucket_mb=4.0)
            w = Worker(cfg, rank, world, 0, comm)
            if p0 is None:
                p0 = torch.cat([p.detach().flatten() for p in w.model.parameters()]).cpu()
            rec = w.run_epoch()
            torch.cuda.synchronize()
            params = torch.cat([p.detach().flatten() for p in w.model.parameters()]).cpu()
            nb = len(w._buckets) if ov else 0
            st = comm.status()
            del w
            gc.collect()
            comm.destroy()
            res[ov] = (params, rec["t_s"], nb, st)
        d_base, d_ov = res[False][0] - p0, res[True][0] - p0
        rel = float((d_ov - d_base).norm() / d_base.norm())
        # every bucket reduced: the ranks hold bit-identical parameters after the overlapped epoch
        mine = res[True][0].double()
        other = [torch.zeros_like(mine) for _ in range(world)]
        dist.all_gather(other, mine)
        same = all(torch.equal(o, other[0]) for o in other)
        ok = (rel < 1e-2 and same and res[True][2] > 1 and res[True][1] > 0 and res[False][1] > 0
              and res[True][3] == 0 and res[False][3] == 0)
        q.put((rank, "ok" if ok else f"rel={rel} same={same} buckets={res[True][2]} t_s={res[True][1]}"))
    except Exception as e:
        import traceback

        q.put((rank, repr(e) + traceback.format_exc()))
    finally:
        dist.destroy_process_group()


@pytest.mark.gpu
def test_overlapped_bucket_allreduce_two_processes():
    """N1: bucketed allreduce launched from backward hooks inside the captured step gives the same training
    step as the allreduce after backward, and leaves the ranks with identical parameters."""
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    ps = [ctx.Process(target=_overlap_worker, args=(r, 2, port, q)) for r in range(2)]
    for p in ps:
        p.start()
    res = dict(q.get(timeout=600) for _ in ps)
    for p in ps:
        p.join(60)
    assert res == {0: "ok", 1: "ok"}, res


def _torchrun(args, env_extra, timeout=900):
    import subprocess
    import sys

    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    env = dict(os.environ, **env_extra)
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", "--nproc-per-node=2", "--master-addr",
           "127.0.0.1", f"--master-port={_free_port()}"] + args
    return subprocess.run(cmd, cwd=root, env=env, capture_output=True, text=True, timeout=timeout)


@pytest.mark.gpu
@pytest.mark.parametrize("model", ["proportional", "affine"])
def test_experiments_multiprocess_path_two_ranks(tmp_path, model):
    """experiments.py's one-rank-per-process path — real barrier inside K3, measured t_w, the K6 t_s allgather,
    the replicated controller (the paper's Eq. 10 and the affine step-cost model) — with 2 processes sharing
    the test GPU (PR_BENCH_SHARED_GPU=1: functional only, the ranks time-share one GPU), plus the per-(epoch,
    rank) metrics CSV of SURVEY §5."""
    import json

    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    csv = tmp_path / "m.csv"
    r = _torchrun(["experiments.py", "--scenario", "c2-5x", "--epochs", "3", "--N", "8192", "--model", model,
                   "--metrics-csv", str(csv)], {"PR_BENCH_SHARED_GPU": "1"})
    assert r.returncode == 0, r.stderr[-3000:]
    recs = [json.loads(ln) for ln in r.stdout.splitlines() if ln.startswith("{")]
    assert [x["epoch"] for x in recs] == [0, 1, 2]
    for x in recs:
        assert len(x["t_s"]) == 2 and len(x["t_w"]) == 2 and min(x["t_w"]) == 0.0
        assert x["T"] > 0 and x["bound"] > 0 and sum(x["w"]) == 12
    rows = csv.read_text().splitlines()
    assert rows[0] == "scenario,epoch,rank,w,n,len,t_s_ns,t_w_ns,t_c_ns,T_ns,loss" and len(rows) == 1 + 3 * 2
    for ln in rows[1:]:
        f = ln.split(",")
        assert f[0] == "c2-5x" and int(f[3]) * 32 == int(f[4]) and int(f[6]) > 0


@pytest.mark.gpu
def test_bench_two_ranks_self_launch_shared_gpu():
    """`PR_BENCH_SHARED_GPU=1 python bench.py --gpus 2` (no torchrun around it: bench.py re-launches itself)
    prints one valid JSON line from rank 0 — the driver's N > 1 form, functional on a one-GPU box."""
    import json
    import subprocess
    import sys

    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    env = dict(os.environ, PR_BENCH_SHARED_GPU="1")
    env.pop("WORLD_SIZE", None)
    r = subprocess.run([sys.executable, "bench.py", "--gpus", "2", "--steps", "2", "--warmup", "3", "--no-vgg",
                        "--e2e-epochs", "1", "--data-n", "8192"], cwd=root, env=env, capture_output=True, text=True,
                       timeout=900)
    assert r.returncode == 0, r.stderr[-3000:]
    lines = [ln for ln in r.stdout.splitlines() if ln.startswith("{")]
    assert len(lines) == 1
    d = json.loads(lines[0])
    assert d["n_gpus"] == 2 and d["scaling"] == "strong" and d["config"]["global_batch"] == 1024
    assert d["value"] > 0 and d["e2e"]["value"] > 0 and d["gpu_launches"] > 0
    assert d["allreduce"]["bound"] == "nvlink" and d["weak_scaling"]["config"]["global_batch"] == 2048
    assert [row["bytes"] for row in d["allreduce_sweep"]][:2] == [64 << 20, 256 << 20]
