"""Run-to-run spread of the harness step (row a4): ResNet-18, 1,024 CIFAR-shaped rows, channels-last, bf16
autocast, CUDA graph — with cuDNN autotuning (benchmark=True, the trainer's setting) and without.
    python tools/model_variance.py [benchmark 0|1] [benchmark_limit]"""

import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

bench = sys.argv[1] == "1" if len(sys.argv) > 1 else True
torch.backends.cudnn.benchmark = bench
if len(sys.argv) > 2:
    torch.backends.cudnn.benchmark_limit = int(sys.argv[2])
from tools.model_speed import run  # noqa: E402

print(f"cudnn.benchmark={bench} limit={torch.backends.cudnn.benchmark_limit}: {run(True, True):.3f} ms per 1,024-row step")
