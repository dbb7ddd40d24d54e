"""Summarise experiments.py --virtual JSON lines (run with tools/run_hetero_r2*.sh) into one row per run,
recomputing the measured-cost optimum from the recorded t1 table with experiments.minmax_alloc.

    python tools/hetero_table.py profiles/round2_heterogeneity_runs.jsonl [...]
"""

import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import experiments as E  # noqa: E402


def interp(m, wmax):
    """t1 at every unit count 1..wmax from the measured ones (linear between neighbours, as --opt-stride)."""
    out = {}
    for u in range(1, wmax + 1):
        if u in m:
            out[u] = m[u]
        else:
            a = max(x for x in m if x < u)
            b = min(x for x in m if x > u)
            out[u] = m[a] + (m[b] - m[a]) * (u - a) / (b - a)
    return out


def main(paths):
    print("| run | emulation | final w | last-epoch T (s) | T / linear bound | measured-cost optimum w | T / optimum |")
    print("|---|---|---|---|---|---|---|")
    for path in paths:
        for ln in open(path):
            d = json.loads(ln)
            if "T_total" not in d:
                continue
            model, N, shape, P, ratios, C, g, sigma, adaptive = E.SCENARIOS[d["scenario"]]
            t1 = interp({n // g: t for n, t in d["t1_points"] if n % g == 0}, C - (P - 1))
            c0 = d["c0_s_per_row"]
            S = N // (g * C)
            tc = d["opt_bound_epoch_s"] / S - d["opt_step_s"]
            wmax = C - (P - 1)
            T, w = E.minmax_alloc(lambda r, u: E.step_cost(t1[u], g * u, sigma[r], d["spin"], c0) if u <= wmax and u in t1
                                  else float("inf"), P, C)
            bound = S * (T + tc)
            print(f"| {d['run']} | {d['spin']} | {d['final_w']} | {d['last_epoch_T']:.4f} | "
                  f"{d['last_epoch_T_over_linear_bound']:.3f} | {w} | {d['last_epoch_T'] / bound:.3f} |")


if __name__ == "__main__":
    main(sys.argv[1:])
