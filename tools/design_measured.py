"""Regenerate DESIGN.md §8's "Measured (N = 1)" and "Per-kernel oracle timing" blocks from a bench line.

    python tools/design_measured.py profiles/round2_bench_n1.json
"""

import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def blocks(d):
    v, ac = d["vgg16"], d["allreduce_colocated"]
    m = f"""Driver-format line of this round's final code (`python bench.py`, defaults: 5 timed + 3 warm-up epochs; clocks
{d['clocks']['sm_mhz']:.0f}/{d['clocks']['sm_max_mhz']:.0f} MHz, throttle reasons {d['clocks']['reasons'] or 'none'}):

| leg | value | kernel evidence |
|---|---|---|
| ResNet-18 / CIFAR-shaped 50k, B = 1,024 | {d['value'] / 1e3:.1f}k samples/s ({d['ms_per_step']:.1f} ms per epoch); e2e {d['e2e']['value'] / 1e3:.1f}k | K7 {d['roofline_detail']['avg_us']:.1f} µs per launch = {d['roofline']['frac']:.3f} of {d['roofline']['peak']:.0f} GB/s; K2 {d['gather']['avg_us']:.1f} µs = {d['gather']['frac']:.3f} ({d['gather']['mix_ceiling']['frac']:.3f} of the mix ceiling) |
| VGG-16 / ImageNet-shaped 51.2k, B = 1,024 | {v['value'] / 1e3:.2f}k samples/s ({v['ms_per_step'] / 1e3:.2f} s per epoch); e2e {v['e2e']['value'] / 1e3:.2f}k | K7 {v['roofline_detail']['avg_us']:.0f} µs = {v['roofline']['frac']:.3f}; K2 {v['gather']['avg_us'] / 1e3:.2f} ms = {v['gather']['frac']:.3f} ({v['gather']['mix_ceiling']['frac']:.3f} of the mix ceiling); clocks {v['clocks']['sm_mhz']:.0f} MHz, {', '.join(v['clocks']['reasons']) or 'no throttle reason'} |
| K3 co-located (8 ranks, ResNet-18 gradient) | {ac['avg_us']:.0f} µs; fused a6-a9 {ac['fused_a6_a9_us']:.0f} µs vs composed {ac['composed_a6_a9_us']:.0f} µs | HBM proxy {ac['frac']:.2f} of the copy peak (algorithmic) |
| K3 cross-GPU config, per-rank CTA proxy (2 ranks, 32 ch) | {ac['cross_gpu_config_per_rank_busbw_equiv']['GBs']:.0f} GB/s bus-equivalent | not NVLink |
| K3 pull two-shot (N2), same co-located cases | ResNet-18 P = 8 {ac['pull_two_shot']['resnet18_P8']['avg_us']:.0f} µs (fused a6-a9 {ac['pull_two_shot'].get('fused_a6_a9_resnet18_P8_us', float('nan')):.0f} µs); VGG-16 P = 4 {ac['pull_two_shot']['vgg16_C3_P4']['avg_us']:.0f} µs (ring {ac['vgg16_C3_P4']['avg_us']:.0f}); cross-GPU proxy {ac['pull_two_shot']['cross_gpu_config_per_rank']['busbw_equiv_per_rank_GBs']:.0f} GB/s | HBM {ac['pull_two_shot']['resnet18_P8']['frac']:.2f} / {ac['pull_two_shot']['vgg16_C3_P4']['frac']:.2f} of the copy peak (2·Z per rank algorithmic) |
| K3 pull two-shot, TMA-staged (opt-in) | ResNet-18 P = 8 {ac['pull_two_shot']['tma']['resnet18_P8']['avg_us']:.0f} µs; VGG-16 P = 4 {ac['pull_two_shot']['tma']['vgg16_C3_P4']['avg_us']:.0f} µs | HBM {ac['pull_two_shot']['tma']['resnet18_P8']['frac']:.2f} / {ac['pull_two_shot']['tma']['vgg16_C3_P4']['frac']:.2f} |

Library kernels are {100 * sum(d['kernel_shares'].values()):.1f} % of the ResNet-18 epoch at N = 1 (the rest is cuDNN forward/backward; at
P = 1 the allreduce is an identity), {100 * sum(v['kernel_shares'].values()):.2f} % of the VGG-16 epoch.  `gpu_launches` {d['gpu_launches']}."""
    rows = d["cpu_baseline"]["per_kernel"]["rows"]
    o = "| case | oracle (1 core) | GPU kernel | ratio |\n|---|---|---|---|\n"
    for r in rows:
        o += f"| {r['case']} ({r['oracle']} vs {r['gpu']}) | {r['oracle_ms']:.3f} ms | {r['gpu_ms'] * 1e3:.1f} µs | {r['ratio']:.1f}× |\n"
    pk = d["cpu_baseline"]["per_kernel"]
    o += (f"\nCPU: {pk['cpu_model']}, {pk['host_cores']} host cores, oracle pinned to core 0.  The 4 KB rows are launch "
          f"latency on the GPU side (P co-located ranks launched eagerly; the oracle wins there); the end-to-end "
          f"oracle step ({d['cpu_baseline']['cores']} threads) is {d['cpu_baseline']['value']:.0f} samples/s.\n")
    return m, o


def main(path):
    d = json.load(open(path))
    m, o = blocks(d)
    p = os.path.join(ROOT, "DESIGN.md")
    s = open(p).read()
    h1 = s.index("### Measured (N = 1")
    h2 = s.index("### Per-kernel oracle timing")
    h3 = s.index("## 9. What differs")
    s = (s[:h1] + f"### Measured (N = 1, `{os.path.relpath(path, ROOT)}`)\n\n" + m + "\n\n" +
         "### Per-kernel oracle timing beside the GPU kernels (same run)\n\n" + o + "\n" + s[h3:])
    open(p, "w").write(s)


if __name__ == "__main__":
    main(sys.argv[1])
