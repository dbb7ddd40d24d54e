#!/bin/bash
# Fused pull two-shot (a6-a9): parity (allreduce file + IPC + worker parity), and co-located timing vs the fused ring.
mkdir -p gpurun_out
timeout 1800 python -m pytest tests/test_gpu_allreduce.py tests/test_multiproc.py tests/test_gpu_worker_parity.py -q -x -p no:cacheprovider -m gpu > gpurun_out/pf_pytest.log 2>&1
echo "pytest exit $?" >> gpurun_out/pf_pytest.log
tail -n 3 gpurun_out/pf_pytest.log
timeout 300 python - <<'PY' > gpurun_out/pf_times.jsonl 2>&1
import json, sys, torch
sys.path.insert(0, ".")
import paper_2111_08272_b200 as pr
P, L = 8, 11_689_512
n = [64, 64, 64, 64, 128, 128, 256, 256]
for name, algo in (("ring", pr.ALGO_RING), ("pull", pr.ALGO_TWO_SHOT_PULL)):
    comms = pr.comm_init_local(P, 0, pr.comm_config(algo=algo))
    store = [torch.randn(2 * L, device="cuda") for _ in range(P)]
    grads, thetas = [x[:L] for x in store], [x[L:] for x in store]
    def timed(fn, k=20):
        for _ in range(3): fn()
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        for _ in range(k): fn()
        e1.record(); torch.cuda.synchronize()
        return e0.elapsed_time(e1) / k * 1e3
    fz = timed(lambda: pr.weighted_allreduce_sgd_local(comms, grads, thetas, n, 1e-6, 0.0, zero_grad=True))
    fn = timed(lambda: pr.weighted_allreduce_sgd_local(comms, grads, thetas, n, 1e-6, 0.0, zero_grad=False))
    def composed():
        pr.weighted_allreduce_local(comms, grads, n)
        for r in range(P): pr.sgd_update(thetas[r], grads[r], 1e-6, 0.0, zero_grad=True)
    cz = timed(composed)
    print(json.dumps({"algo": name, "P": P, "L": L, "fused_zero_grad_us": round(fz, 1), "fused_keep_grad_us": round(fn, 1),
                      "composed_us": round(cz, 1)}), flush=True)
    for c in comms: c.destroy()
    del store, grads, thetas
PY
cat gpurun_out/pf_times.jsonl
