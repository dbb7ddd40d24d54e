"""Algorithm 1 end to end on one GPU (experiments.py --virtual): emulated 2× straggler, ResNet-18 in its
linear-cost regime.  The controller must reach Eq. 10's fixed point w ∝ v ([8,16] of C = 24 for
σ = [2,1]) after one update, freeze, and the emulated epoch time must be within 10% of the
Σspeed-balanced bound (north star) and well below the equal-allocation epoch."""

import json
import os
import subprocess
import sys

import pytest
import torch

pytestmark = pytest.mark.gpu
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def test_c2_lin_converges_and_meets_bound():
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    out = subprocess.run([sys.executable, os.path.join(ROOT, "experiments.py"), "--virtual", "--scenario", "c2-lin",
                          "--epochs", "3", "--N", "24576"], capture_output=True, text=True, timeout=600, cwd=ROOT)
    recs = [r for r in (json.loads(l) for l in out.stdout.splitlines() if l.startswith("{")) if "epoch" in r]
    assert len(recs) == 3, out.stderr[-2000:]
    assert recs[0]["w"] == [12, 12]
    assert recs[1]["w"] == [8, 16] and recs[2]["w"] == [8, 16] and recs[2]["frozen"]
    assert recs[2]["T_over_bound"] <= 1.10
    assert recs[2]["T_emulated"] < 0.75 * recs[0]["T_emulated"]
