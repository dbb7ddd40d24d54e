"""GPU checks of the harness (rows a3-a5, a9) built on the library.

* the epoch-level gather (one K2 launch per epoch) yields exactly the per-step batches of P:150, bitwise;
* the channels-last + CUDA-graph step computes the same training step as the eager NCHW step (losses
  and parameters agree to bf16-autocast noise);
* t_s is positive and the controller runs at the epoch boundary.
"""

import numpy as np
import pytest
import torch

pytestmark = pytest.mark.gpu
pr = pytest.importorskip("paper_2111_08272_b200")


@pytest.fixture(scope="module", autouse=True)
def _cuda():
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")


def _worker(**kw):
    from paper_2111_08272_b200.trainer import RunConfig, Worker

    cfg = RunConfig(N=4096, ratios=[1], C=64, g=16, micro=1024, adaptive=True, **kw)
    return Worker(cfg, 0, 1, 0, None)


def test_epoch_gather_equals_step_gathers():
    for cl in (False, True):
        w = _worker(channels_last=cl)
        v = w.alloc.view()
        n, S = v["n"][0], v["S"]
        pr.shard_indices(w.alloc, 0, 3, w.cfg.seed, w.idx)
        xe, ye = w.gather(0, S * n)
        for s in range(S):
            x, y = w.gather(s * n, n)
            assert torch.equal(x.view(torch.int16), xe[s * n:(s + 1) * n].view(torch.int16))
            assert torch.equal(y, ye[s * n:(s + 1) * n])


def test_graphed_channels_last_step_matches_eager():
    a = _worker(channels_last=True, graphs=True)
    b = _worker(channels_last=False, graphs=False)
    for _ in range(3):
        ra, rb = a.run_epoch(), b.run_epoch()
        assert abs(ra["loss"] - rb["loss"]) <= 2e-2 * abs(rb["loss"])
        assert ra["t_s"] > 0 and rb["t_s"] > 0
    pa = torch.cat([p.detach().float().flatten() for p in a.model.parameters()])
    pb = torch.cat([p.detach().float().flatten() for p in b.model.parameters()])
    assert float((pa - pb).norm() / pb.norm()) < 1e-2


def test_boundary_runs_controller():
    w = _worker()
    assert w.boundary() is False              # first boundary: no t_s yet
    w.run_epoch()
    w.boundary()                              # P = 1: Eq. 10 keeps w = [C]
    v = w.alloc.view()
    assert v["w"] == [64] and v["epoch"] == 1


def test_segmented_epoch_matches_contiguous_at_one_rank():
    # N3 at P = 1: the step-interleaved shard of step s is positions [s·B, (s+1)·B) = the contiguous
    # shard's step s, so the segmented epoch trains on the same batches (same losses up to bf16 noise)
    a = _worker(adapt_every=3, policy={"never_freeze": True})
    b = _worker()
    ra, rb = a.run_epoch(), b.run_epoch()
    S = rb["S"]
    assert [sg["steps"] for sg in ra["segments"]] == [3] * (S // 3) + ([S % 3] if S % 3 else [])
    assert abs(ra["loss"] - rb["loss"]) <= 2e-2 * abs(rb["loss"])
    assert a.alloc.view()["hist_len"] == 1 + len(ra["segments"])   # one controller call per segment
    assert a.gstep == S and a.boundary() is False


def test_slowdown_schedule_lookup():
    w = _worker(slowdown=[2.0], slowdown_schedule=[(5, [3.0]), (9, [1.5])])
    seen = []
    for s in (0, 4, 5, 8, 9, 100):
        w.gstep = s
        seen.append(w.sigma())
    assert seen == [2.0, 2.0, 3.0, 3.0, 1.5, 1.5]


def test_checkpoint_resume_continues_the_same_run():
    """resume from Worker.state_dict() between epochs = the uninterrupted run: same allocation
    state and history length, same shards (π depends only on (seed, epoch)), same training up to cuDNN /
    bf16 reassociation noise."""
    import io

    a = _worker()
    for _ in range(2):
        a.boundary()
        a.run_epoch()
    buf = io.BytesIO()
    torch.save(a.state_dict(), buf)
    alloc_epoch = a.alloc.view()["epoch"]
    for _ in range(2):
        a.boundary()
        a.run_epoch()
    b = _worker()
    buf.seek(0)
    b.load_state_dict(torch.load(buf, weights_only=False))
    assert b.epoch == 2 and b.alloc.view()["epoch"] == alloc_epoch
    for _ in range(2):
        b.boundary()
        b.run_epoch()
    va, vb = a.alloc.view(), b.alloc.view()
    assert (va["w"], va["epoch"], va["hist_len"], va["frozen"]) == (vb["w"], vb["epoch"], vb["hist_len"], vb["frozen"])
    assert a.epoch == b.epoch == 4 and a.gstep == b.gstep
    ia, ib = torch.empty_like(a.idx), torch.empty_like(b.idx)
    pr.shard_indices(a.alloc, 0, a.epoch, a.cfg.seed, ia)
    pr.shard_indices(b.alloc, 0, b.epoch, b.cfg.seed, ib)
    assert torch.equal(ia, ib)
    pa = torch.cat([p.detach().float().flatten() for p in a.model.parameters()])
    pb = torch.cat([p.detach().float().flatten() for p in b.model.parameters()])
    assert float((pa - pb).norm() / pa.norm()) < 1e-3
    with pytest.raises(ValueError):
        sd = a.state_dict()
        sd["P"] = 2
        b.load_state_dict(sd)


def test_fused_sgd_matches_torch_sgd_training():
    """a9 through pr_sgd_update (flat parameter views) trains like torch.optim.SGD + memset."""
    a = _worker(fused_sgd=True)
    b = _worker(fused_sgd=False)
    for _ in range(2):
        ra, rb = a.run_epoch(), b.run_epoch()
        assert abs(ra["loss"] - rb["loss"]) <= 2e-2 * abs(rb["loss"])
    pa = torch.cat([p.detach().float().flatten() for p in a.model.parameters()])
    pb = torch.cat([p.detach().float().flatten() for p in b.model.parameters()])
    assert float((pa - pb).norm() / pb.norm()) < 1e-3
    # the parameters really are views of the flat buffer the kernel updates
    p0 = next(a.model.parameters())
    assert p0.untyped_storage().data_ptr() == a.pflat.untyped_storage().data_ptr()
    assert torch.count_nonzero(a.flat) == 0               # gradient reset fused into the update
