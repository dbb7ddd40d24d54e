"""t1(n): graphed channels-last forward/backward time vs rows per step (ResNet-18 CIFAR / VGG-16 ImageNet)."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402
from paper_2111_08272_b200.trainer import RunConfig, Worker  # noqa: E402

which = sys.argv[1] if len(sys.argv) > 1 else "resnet18"
if which == "resnet18":
    cfg = RunConfig(N=8192, ratios=[1], C=1, g=16, micro=4096)
    ns = [64, 128, 256, 512, 1024, 2048, 4096]
else:
    cfg = RunConfig(N=1024, shape=(3, 224, 224), model="vgg16", ratios=[1], C=1, g=16, micro=256)
    ns = [16, 32, 64, 128, 256]
w = Worker(cfg, 0, 1, 0, None)
for n in ns:
    w.prepare(n)
    print(which, n, f"{w._graphs[n][4] / 1e6:.3f} ms", f"{w._graphs[n][4] / n:.1f} ns/sample", flush=True)
