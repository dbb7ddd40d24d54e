"""Small invocation of every library kernel, for compute-sanitizer (memcheck / racecheck / synccheck).

    compute-sanitizer --tool memcheck python tools/sanitize_workload.py
Checks results against the oracle as it goes (a sanitizer run must also be a correct run).
"""

import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import numpy as np  # noqa: E402
import torch  # noqa: E402

import paper_2111_08272_b200 as pr  # noqa: E402
import synth  # noqa: E402
from oracle import gather as OG  # noqa: E402
from oracle import permutation as OP  # noqa: E402
from oracle import wavg as OW  # noqa: E402


def main():
    torch.cuda.init()
    # K1
    out = torch.empty(1000, dtype=torch.int64, device="cuda")
    pr.permute(1000, 7, 3, 0, 1000, out)
    assert np.array_equal(out.cpu().numpy(), OP.permute(np.arange(1000), 1000, 7, 3))
    # K2: both kernels, CHW and HWC, a long-row case
    for row_bytes, plane, n in ((3072, 1024, 40), (3 * 12544, 12544, 5)):
        X = synth.images_u8(64, seed=1).reshape(64, -1)[:, :row_bytes] if row_bytes == 3072 else \
            np.random.Generator(np.random.PCG64(2)).integers(0, 256, (8, row_bytes), dtype=np.uint8)
        nsrc = X.shape[0]
        idx = np.arange(n) % nsrc
        dX, didx = torch.from_numpy(np.ascontiguousarray(X)).cuda(), torch.from_numpy(idx).cuda()
        for impl in (pr.GATHER_IMPL_LSU, pr.GATHER_IMPL_TMA, pr.GATHER_IMPL_BULK):
            for layout, lname in ((pr.GATHER_LAYOUT_CHW, "chw"), (pr.GATHER_LAYOUT_HWC, "hwc")):
                if impl == pr.GATHER_IMPL_BULK and layout == pr.GATHER_LAYOUT_CHW:
                    continue                                  # channels-last only
                o = torch.empty((n, row_bytes), dtype=torch.bfloat16, device="cuda")
                op = pr.make_gather_op(pr.GATHER_U8_TO_BF16_AFFINE, [0.02] * 3, [100.0] * 3, plane, impl=impl,
                                       layout=layout)
                pr.gather_rows(dX, nsrc, row_bytes, didx, n, o, op)
                ref, _ = OG.gather_rows(X, idx, OG.U8_TO_BF16_AFFINE, np.float32([0.02] * 3), np.float32([100.0] * 3),
                                        plane, layout=lname)
                assert np.array_equal(o.view(torch.int16).cpu().numpy().view(np.uint16), ref), (impl, lname)
    # K2 TMA with stage reuse (more units than CTAs): 8192 rows -> 1024 units over 296 CTAs
    X = synth.images_u8(256, seed=3).reshape(256, -1)
    idx = np.random.Generator(np.random.PCG64(4)).integers(0, 256, 8192)
    o = torch.empty((8192, 3072), dtype=torch.bfloat16, device="cuda")
    op = pr.make_gather_op(pr.GATHER_U8_TO_BF16_AFFINE, [0.02] * 3, [100.0] * 3, 1024, impl=pr.GATHER_IMPL_TMA)
    pr.gather_rows(torch.from_numpy(X).cuda(), 256, 3072, torch.from_numpy(idx).cuda(), 8192, o, op)
    ref, _ = OG.gather_rows(X, idx, OG.U8_TO_BF16_AFFINE, np.float32([0.02] * 3), np.float32([100.0] * 3), 1024)
    assert np.array_equal(o.view(torch.int16).cpu().numpy().view(np.uint16), ref)
    # K2 bulk-store kernel with smem-tile reuse (2,048 units over at most 592 CTAs: every CTA rewrites both
    # tiles behind cp.async.bulk.wait_group.read) and labels
    Y = np.arange(256, dtype=np.int64) * 3
    lab = torch.empty(8192, dtype=torch.int64, device="cuda")
    op = pr.make_gather_op(pr.GATHER_U8_TO_BF16_AFFINE, [0.02] * 3, [100.0] * 3, 1024, impl=pr.GATHER_IMPL_BULK,
                           layout=pr.GATHER_LAYOUT_HWC)
    pr.gather_rows(torch.from_numpy(X).cuda(), 256, 3072, torch.from_numpy(idx).cuda(), 8192, o, op,
                   torch.from_numpy(Y).cuda(), lab)
    ref, rlab = OG.gather_rows(X, idx, OG.U8_TO_BF16_AFFINE, np.float32([0.02] * 3), np.float32([100.0] * 3), 1024,
                               Y=Y, layout="hwc")
    assert np.array_equal(o.view(torch.int16).cpu().numpy().view(np.uint16), ref)
    assert np.array_equal(lab.cpu().numpy(), rlab)
    # K4
    pr.spin(10_000)
    # K3: local groups, both scopes, direct and staged, ragged counts
    for flags in (dict(), dict(sys_scope=True), dict(force_staged=True), dict(algo=pr.ALGO_TWO_SHOT),
                  dict(algo=pr.ALGO_LL), dict(algo=pr.ALGO_LL, sys_scope=True), dict(algo=pr.ALGO_ONESHOT),
                  dict(min_slice_bytes=512), dict(bulk_store=True), dict(bulk_store=True, force_staged=True),
                  dict(bulk_store=True, sys_scope=True), dict(algo=pr.ALGO_AUTO, force_staged=True)):
        comms = pr.comm_init_local(3, 0, pr.comm_config(channels=2, slots=4, slot_bytes=4096, stages=2,
                                                        tile_bytes=2048, threads=64, **flags))
        for L in (5, 3001):
            g = synth.gradients(3, L, seed_base=L)
            bufs = [torch.from_numpy(g[r].copy()).cuda() for r in range(3)]
            pr.weighted_allreduce_local(comms, bufs, [1, 0, 3])
            torch.cuda.synchronize()
            assert all(c.status() == 0 for c in comms)
            assert np.array_equal(bufs[1].cpu().numpy(), OW.ring_emulate(g, [1, 0, 3], "f32"))
            hb = OG.f32_to_bf16_bits(g)                     # bf16 leg (odd L: ragged last line / tail)
            bb = [torch.from_numpy(hb[r].view(np.int16).copy()).cuda().view(torch.bfloat16) for r in range(3)]
            pr.weighted_allreduce_local(comms, bb, [2, 5, 0])
            torch.cuda.synchronize()
            assert all(c.status() == 0 for c in comms)
            assert np.array_equal(bb[0].view(torch.int16).cpu().numpy().view(np.uint16),
                                  OW.ring_emulate(hb, [2, 5, 0], "bf16"))
        for c in comms:
            c.destroy()
    # K3 with K7 fused (rows a6-a9): [grad | theta] per rank, against ring + K7 composed (STG and bulk paths)
    for bulk in (False, True):
        comms = pr.comm_init_local(3, 0, pr.comm_config(channels=2, slots=4, slot_bytes=4096, stages=2, tile_bytes=2048,
                                                        threads=64, bulk_store=bulk))
        for L in (5, 3001):
            Lp = (L + 3) // 4 * 4
            g = synth.gradients(3, L, seed_base=L + 1)
            th0 = torch.from_numpy(synth.gradients(1, L, seed_base=L + 2)[0]).cuda()
            store = [torch.zeros(2 * Lp, device="cuda") for _ in range(3)]
            gr, th = [s_[:L] for s_ in store], [s_[Lp:Lp + L] for s_ in store]
            for r in range(3):
                gr[r].copy_(torch.from_numpy(g[r]))
                th[r].copy_(th0)
            pr.weighted_allreduce_sgd_local(comms, gr, th, [2, 0, 1], 0.1, 1e-4)
            ref = th0.clone()
            pr.sgd_update(ref, torch.from_numpy(OW.ring_emulate(g, [2, 0, 1], "f32")).cuda(), 0.1, 1e-4)
            torch.cuda.synchronize()
            assert all(c.status() == 0 for c in comms)
            assert all(torch.equal(t, ref) for t in th) and all(torch.count_nonzero(x) == 0 for x in gr)
        for c in comms:
            c.destroy()
    # a6 timestamps on the device + K6's device-side value path (pr_stamp / pr_stamp_seconds)
    ring = torch.zeros(9, dtype=torch.int64, device="cuda")
    for _ in range(4):
        pr.stamp(ring)
    d = torch.zeros((), dtype=torch.float64, device="cuda")
    pr.stamp_seconds(ring, d)
    torch.cuda.synchronize()
    assert float(d) >= 0.0
    print("sanitize workload: ok")


if __name__ == "__main__":
    main()
