"""K1 A/B: one-thread-per-index cycle walk (PR_K1_KERNEL=direct) vs the lane-refill walk (default).

    python tools/ab_k1.py            # both kernels (refill at 8-64 warps per SM), each in its own process
                                     # (the switches are read once per process)
    python tools/ab_k1.py --child    # one kernel (the environment decides), JSON lines on stdout

Sizes: the whole permutation at N = 50,000 (C2/C4) and 1,281,167 (the scale point of SURVEY §8(a) a2),
one rank's shard at C3 (12,800 of 51,200), and the N3 step-interleaved shard (pr_shard_steps) at C4.
Device time per call from CUDA events (median of 5 runs of 20 back-to-back calls, after warm-up);
the refill run also checks its outputs bit-for-bit against the direct kernel's (saved to /tmp).
"""

import json
import os
import subprocess
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))


def child():
    import numpy as np
    import torch

    import paper_2111_08272_b200 as pr

    kind = os.environ.get("PR_K1_KERNEL", "refill")
    if kind != "direct":
        kind += "/W=" + os.environ.get("PR_K1_WARPS_PER_SM", "default")
    cases = []

    def permute_case(N, begin, count):
        out = torch.empty(count, dtype=torch.int64, device="cuda")
        return f"permute N={N} [{begin},{begin + count})", (lambda: pr.permute(N, 1234, 3, begin, count, out)), out, N

    cases.append(permute_case(50000, 0, 50000))
    cases.append(permute_case(1281167, 0, 1281167))
    cases.append(permute_case(51200, 12800, 12800))
    a = pr.alloc_init(50000, [1, 1, 1, 1, 2, 2, 4, 4], C=64, g=16)
    v = a.view()
    S, n7 = v["S"], v["n"][7]
    o7 = torch.empty(S * n7, dtype=torch.int64, device="cuda")
    cases.append(("shard_steps C4 rank 7 all steps", lambda: pr.shard_steps(a, 7, 5, 77, 0, S, o7), o7, 50000))
    st = torch.cuda.current_stream()
    for name, fn, out, N in cases:
        for _ in range(3):
            fn()
        torch.cuda.synchronize()
        runs = []
        for _ in range(5):
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record(st)
            for _ in range(20):
                fn()
            e1.record(st)
            torch.cuda.synchronize()
            runs.append(e0.elapsed_time(e1) / 20 * 1e3)
        us = sorted(runs)[2]
        got = out.cpu().numpy()
        key = name.replace(" ", "_").replace("=", "").replace("[", "").replace(")", "").replace(",", "_")
        path = f"/tmp/k1_{key}.npy"
        same = None
        if kind == "direct":
            np.save(path, got)
        elif os.path.exists(path):
            same = bool(np.array_equal(np.load(path), got))
        print(json.dumps({"kernel": kind, "case": name, "count": int(got.size), "us": round(us, 2),
                          "G_indices_per_s": round(got.size / us / 1e3, 3), "bit_exact_vs_direct": same}),
              flush=True)


def main():
    here = os.path.abspath(__file__)
    env = dict(os.environ, PR_K1_KERNEL="direct")
    subprocess.run([sys.executable, here, "--child"], env=env, check=True)
    for w in ("8", "16", "24", "32", "64", ""):
        env = dict(os.environ, PR_K1_KERNEL="refill")
        if w:
            env["PR_K1_WARPS_PER_SM"] = w
        else:
            env.pop("PR_K1_WARPS_PER_SM", None)
        subprocess.run([sys.executable, here, "--child"], env=env, check=True)


if __name__ == "__main__":
    child() if "--child" in sys.argv else main()
