"""Summarise ncu captures into profiles/ (run here, on the CPU host).

    python tools/summarize_ncu.py <round-tag> gpurun_out/prof_*.ncu-rep [--launches gpurun_out/launches.csv]

Writes profiles/<tag>_ncu_summary.md (key metrics + top stall reasons per captured kernel, and the
launch-list shares of the bench command) and updates profiles/ncu_traffic.json (dram bytes per launch
of each library kernel, read by bench.py's roofline `traffic`).
"""

import csv
import io
import json
import os
import subprocess
import sys
from collections import defaultdict

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
KEYS = [
    ("gpu__time_duration.sum", "duration"),
    ("dram__bytes_read.sum", "dram read"),
    ("dram__bytes_write.sum", "dram write"),
    ("gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed", "DRAM % peak"),
    ("sm__throughput.avg.pct_of_peak_sustained_elapsed", "SM % peak"),
    ("sm__warps_active.avg.pct_of_peak_sustained_active", "warps active %"),
    ("launch__registers_per_thread", "regs/thread"),
    ("launch__grid_size", "grid"),
    ("launch__block_size", "block"),
    ("lts__t_bytes.sum", "L2 bytes"),
]
SCALE = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "nsecond": 1e-3, "usecond": 1, "msecond": 1e3,
         "ns": 1e-3, "us": 1, "ms": 1e3}


def raw(rep):
    out = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    return rows[0], rows[1], rows[2:]


def val(hdr, units, row, key):
    if key not in hdr:
        return None, ""
    i = hdr.index(key)
    try:
        return float(row[i].replace(",", "")), units[i]
    except ValueError:
        return row[i], units[i]


def stalls(hdr, row):
    out = []
    for i, h in enumerate(hdr):
        if h.startswith("smsp__average_warp_latency_issue_stalled_") and h.endswith(".ratio"):
            try:
                out.append((float(row[i]), h.replace("smsp__average_warp_latency_issue_stalled_", "").replace(".ratio", "")))
            except ValueError:
                pass
    return sorted(out, reverse=True)[:5]


def main():
    tag = sys.argv[1]
    reps = [a for a in sys.argv[2:] if a.endswith(".ncu-rep")]
    launches = sys.argv[sys.argv.index("--launches") + 1] if "--launches" in sys.argv else None
    lines = [f"# ncu summary — {tag}", "", "Captured with `ncu --set full --clock-control none --import-source on` "
             "(kernel replay, cold caches, serialised) by `tools/ncu_round.sh` / `tools/ncu_round2.sh` on one B200; "
             "raw reports stay in gpurun_out/ (scratch).", ""]
    traffic_path = os.path.join(ROOT, "profiles", "ncu_traffic.json")
    traffic = json.load(open(traffic_path)) if os.path.exists(traffic_path) else {}
    for rep in reps:
        hdr, units, rows = raw(rep)
        name = os.path.basename(rep).replace(".ncu-rep", "")
        for row in rows:
            kname = row[hdr.index("Kernel Name")]
            lines += [f"## {name}: `{kname[:110]}`", "", "| metric | value |", "|---|---|"]
            d = {}
            for key, label in KEYS:
                v, u = val(hdr, units, row, key)
                if v is None:
                    continue
                if isinstance(v, float) and u in SCALE and key.startswith(("dram__bytes", "lts__t_bytes")):
                    v = v * SCALE[u]
                    u = "byte"
                if isinstance(v, float) and u in ("nsecond", "usecond", "msecond", "ns", "us", "ms") and key == "gpu__time_duration.sum":
                    v = v * SCALE[u]
                    u = "usecond"
                d[key] = v
                lines.append(f"| {label} (`{key}`) | {v:,.3f} {u} |" if isinstance(v, float) else f"| {label} | {v} |")
            st = stalls(hdr, row)
            if st:
                lines.append("| top stall reasons (cycles/instr) | " + ", ".join(f"{n} {x:.1f}" for x, n in st) + " |")
            lines.append("")
            kind = ("gather_imagenet" if "gather" in kname and "imagenet" in name else
                    "sgd_vgg16" if "sgd_kernel" in kname and "vgg" in name else
                    "gather" if "gather" in kname else "sgd" if "sgd_kernel" in kname else
                    "ring_ll" if "ring_ll" in kname else
                    "ring_fused" if ("ring_kernel<float, 1" in kname or "ring_kernel<float, true" in kname) else
                    "twoshot" if "twoshot" in kname else "ring_cta" if ("ring" in kname and "cta" in name) else
                    "ring_colocated" if "ring" in kname else
                    "permute" if "permute" in kname else name)
            if "dram__bytes_read.sum" in d and "dram__bytes_write.sum" in d:
                traffic[kind] = {"dram_bytes_per_launch": d["dram__bytes_read.sum"] + d["dram__bytes_write.sum"],
                                 "capture": f"{tag}/{name}", "duration_us": d.get("gpu__time_duration.sum")}
    if launches and os.path.exists(launches):
        per = defaultdict(lambda: [0, 0.0])
        total = 0.0
        with open(launches) as f:
            text = f.read()
        start = text.find('"ID"')
        rdr = csv.DictReader(io.StringIO(text[start:]))
        for r in rdr:
            if r.get("Metric Name") != "gpu__time_duration.sum":
                continue
            try:
                t = float(r["Metric Value"].replace(",", ""))
            except (KeyError, ValueError):
                continue
            unit = r.get("Metric Unit", "nsecond")
            t = t * SCALE.get(unit, 1e-3)   # -> us
            k = r["Kernel Name"]
            per[k][0] += 1
            per[k][1] += t
            total += t
        mine = ("gather_tma_kernel", "gather_kernel", "gather_hwc_bulk_kernel", "permute_kernel", "walk_refill_kernel", "walk_direct_kernel", "ring_kernel", "ring_ll_kernel", "twoshot_kernel",
                "sgd_kernel", "spin_kernel", "stamp_kernel", "allgather_f64", "oneshot_ll_kernel", "nvls_kernel",
                "stamp_seconds_kernel")
        lines += ["## Launch list of the bench command (`ncu --metrics gpu__time_duration.sum`)", "",
                  f"Total kernel time {total / 1e3:.2f} ms over {sum(v[0] for v in per.values())} launches "
                  "(cold-cache, serialised: compare shares, not absolutes).", "",
                  "| kernel | launches | total us | share |", "|---|---|---|---|"]
        for k, (n, t) in sorted(per.items(), key=lambda kv: -kv[1][1])[:25]:
            flag = " **(library)**" if any(m in k for m in mine) else ""
            lines.append(f"| `{k[:90]}`{flag} | {n} | {t:,.1f} | {t / total:.4f} |")
        lib = {k: v for k, v in per.items() if any(m in k for m in mine)}
        lines += ["", "Library kernels:", ""]
        for k, (n, t) in sorted(lib.items(), key=lambda kv: -kv[1][1]):
            lines.append(f"* `{k[:100]}`: {n} launches, {t:,.1f} us, share {t / total:.4f}")
        lines.append("")
    os.makedirs(os.path.join(ROOT, "profiles"), exist_ok=True)
    with open(os.path.join(ROOT, "profiles", f"{tag}_ncu_summary.md"), "w") as f:
        f.write("\n".join(lines) + "\n")
    with open(traffic_path, "w") as f:
        json.dump(traffic, f, indent=1)
    print("\n".join(lines))


if __name__ == "__main__":
    main()
