"""Two-shot (N2) configuration sweep, co-located: ts_slot_bytes x ts_slots x channels at P = 2 and 8."""
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import paper_2111_08272_b200 as pr  # noqa: E402

for P in (2, 8):
    for ch in (16,):
        for tsb in (65536, 262144, 1048576):
            for tss in (2, 4):
                comms = pr.comm_init_local(P, 0, pr.comm_config(algo=pr.ALGO_TWO_SHOT, channels=ch, ts_slot_bytes=tsb,
                                                                ts_slots=tss))
                raws = [c.alloc(16 << 20) for c in comms]
                for Z in (1 << 20, 4 << 20, 16 << 20):
                    bufs = [r[:Z].view(torch.float32) for r in raws]
                    n = [1 + q for q in range(P)]
                    for _ in range(3):
                        pr.weighted_allreduce_local(comms, bufs, n)
                    torch.cuda.synchronize()
                    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                    a.record()
                    for _ in range(10):
                        pr.weighted_allreduce_local(comms, bufs, n)
                    b.record()
                    torch.cuda.synchronize()
                    us = a.elapsed_time(b) / 10 * 1e3
                    print(json.dumps({"P": P, "channels": ch, "ts_slot_bytes": tsb, "ts_slots": tss, "bytes": Z,
                                      "us": round(us, 1)}), flush=True)
                del raws
                for c in comms:
                    c.destroy()
