"""A/B of a ring data-path option against the default, same call, same box, alternating:

    python tools/ab_bulk.py [bulk_store|l2_prefetch]

bulk_store (PR_COMM_FLAG_BULK_STORE): TMA bulk stores instead of 16-byte STGs; l2_prefetch
(PR_COMM_FLAG_L2_PREFETCH): each slice's own gradient prefetched into L2 before the flag waits.  Measures:
  (a) per-rank CTA throughput, P = 2 co-located (HBM far from saturated: each channel CTA's own data path is
      the limit, the regime of a multi-GPU rank), 256 MiB fp32, 16 / 32 channels, 1 MiB slots, .gpu / .sys;
  (b) P = 8 co-located at the ResNet-18 gradient size (HBM-bound proxy), plain ring and fused a6-a9.
Prints one JSON line per measurement."""

import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import paper_2111_08272_b200 as pr  # noqa: E402


def timed(fn, reps=5, warm=2):
    for _ in range(warm):
        fn()
    torch.cuda.synchronize()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record()
    for _ in range(reps):
        fn()
    b.record()
    torch.cuda.synchronize()
    return a.elapsed_time(b) / reps * 1e3


def main():
    opt = sys.argv[1] if len(sys.argv) > 1 else "bulk_store"
    L2 = (256 << 20) // 4
    x2 = [torch.randn(L2, device="cuda") for _ in range(2)]
    L8 = 11_689_512
    x8 = [torch.randn(2 * L8, device="cuda") for _ in range(8)]
    g8, t8 = [x[:L8] for x in x8], [x[L8:] for x in x8]
    n8 = [64, 64, 64, 64, 128, 128, 256, 256]
    for rep in range(2):
        for bulk in (False, True):
            for ch, sysv in ((16, False), (32, False), (32, True)):
                cs = pr.comm_init_local(2, 0, pr.comm_config(channels=ch, slot_bytes=1 << 20, sys_scope=sysv,
                                                             **{opt: bulk}))
                us = timed(lambda: pr.weighted_allreduce_local(cs, x2, [1, 2]))
                bus = L2 * 4 / (us * 1e-6) / 1e9
                print(json.dumps({"rep": rep, "test": "P2_cta", opt: bulk, "channels": ch, "sys": sysv,
                                  "us": round(us, 1), "busbw_equiv_GBs": round(bus, 1),
                                  "per_channel_GBs": round(bus / ch, 2)}), flush=True)
                for c in cs:
                    c.destroy()
            cs = pr.comm_init_local(8, 0, pr.comm_config(**{opt: bulk}))
            us = timed(lambda: pr.weighted_allreduce_local(cs, g8, n8), reps=20)
            uf = timed(lambda: pr.weighted_allreduce_sgd_local(cs, g8, t8, n8, 1e-6, 0.0, zero_grad=False), reps=20)
            print(json.dumps({"rep": rep, "test": "P8_resnet18", opt: bulk, "ring_us": round(us, 1),
                              "fused_us": round(uf, 1)}), flush=True)
            for c in cs:
                c.destroy()


if __name__ == "__main__":
    main()
