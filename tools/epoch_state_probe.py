"""Why does the ResNet-18 bench epoch sit at either ~126 or ~134 ms (whole runs, or switching mid-run)?

    python tools/epoch_state_probe.py [epochs] [processes]

The bench's N = 1 ResNet-18 workload (RunConfig as bench.py), 3 warm-up epochs, then per epoch: the epoch
time (CUDA events), t_s (the sum of the per-step compute events, a5), the host enqueue time, and NVML's SM /
memory clocks, power, temperature and throttle reasons sampled right after the epoch.  Run in `processes`
fresh processes one after another (the state may be per process: cuDNN's autotuned algorithms are chosen at
capture).  One JSON line per epoch.
"""

import json
import os
import subprocess
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def child(epochs):
    import pynvml
    import torch

    from paper_2111_08272_b200.trainer import RunConfig, Worker

    pynvml.nvmlInit()
    h = pynvml.nvmlDeviceGetHandleByIndex(0)
    cfg = RunConfig(N=50_000, shape=(3, 32, 32), model="resnet18", ratios=[1], C=64, g=16, adaptive=True, micro=1024)
    wk = Worker(cfg, 0, 1, 0, None)
    for e in range(3 + epochs):
        wk.boundary()
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        torch.cuda.synchronize()
        a.record()
        t0 = time.perf_counter()
        rec = wk.run_epoch()
        b.record()
        torch.cuda.synchronize()
        if e < 3:
            continue
        print(json.dumps({
            "pid": os.getpid(), "epoch": e, "epoch_ms": round(a.elapsed_time(b), 2), "t_s_ms": round(rec["t_s"] * 1e3, 2),
            "host_ms": round((time.perf_counter() - t0) * 1e3, 2), "host_enqueue_ms": round(wk.host_enqueue_s * 1e3, 2),
            "sm_mhz": pynvml.nvmlDeviceGetClockInfo(h, pynvml.NVML_CLOCK_SM),
            "mem_mhz": pynvml.nvmlDeviceGetClockInfo(h, pynvml.NVML_CLOCK_MEM),
            "power_w": pynvml.nvmlDeviceGetPowerUsage(h) / 1000, "temp_c": pynvml.nvmlDeviceGetTemperature(h, 0),
            "throttle": pynvml.nvmlDeviceGetCurrentClocksThrottleReasons(h)}), flush=True)


if __name__ == "__main__":
    if len(sys.argv) > 3 and sys.argv[3] == "--child":
        child(int(sys.argv[1]))
    else:
        epochs = int(sys.argv[1]) if len(sys.argv) > 1 else 12
        procs = int(sys.argv[2]) if len(sys.argv) > 2 else 3
        for _ in range(procs):
            subprocess.call([sys.executable, os.path.abspath(__file__), str(epochs), "1", "--child"])
