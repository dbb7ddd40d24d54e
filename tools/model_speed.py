"""Harness (row a4) speed probe: ResNet-18 forward/backward on 1,024 CIFAR-shaped rows, bf16 autocast,
NCHW vs channels_last, eager vs CUDA graph.  Prints ms per aggregation step."""

import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402
import torch.nn.functional as F  # noqa: E402
import torchvision  # noqa: E402


def run(channels_last, graph, n=1024, reps=20):
    torch.manual_seed(0)
    m = torchvision.models.resnet18(num_classes=1000).cuda()
    if channels_last:
        m = m.to(memory_format=torch.channels_last)
    opt = torch.optim.SGD(m.parameters(), lr=0.01, weight_decay=1e-4)
    x = torch.randn(n, 3, 32, 32, device="cuda").to(torch.bfloat16)
    if channels_last:
        x = x.contiguous(memory_format=torch.channels_last)
    y = torch.randint(0, 10, (n,), device="cuda")

    def step():
        with torch.autocast("cuda", dtype=torch.bfloat16):
            loss = F.cross_entropy(m(x).float(), y)
        loss.backward()
        opt.step()
        opt.zero_grad(set_to_none=False)

    s = torch.cuda.Stream()
    s.wait_stream(torch.cuda.current_stream())
    with torch.cuda.stream(s):
        for _ in range(3):
            step()
    torch.cuda.current_stream().wait_stream(s)
    fn = step
    if graph:
        g = torch.cuda.CUDAGraph()
        opt.zero_grad(set_to_none=False)
        with torch.cuda.graph(g):
            step()
        fn = g.replay
    torch.cuda.synchronize()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record()
    for _ in range(reps):
        fn()
    b.record()
    torch.cuda.synchronize()
    return a.elapsed_time(b) / reps


if __name__ == "__main__":
    torch.backends.cudnn.benchmark = True
    for cl in (False, True):
        for gr in (False, True):
            try:
                print(f"channels_last={cl} graph={gr}: {run(cl, gr):.2f} ms/step", flush=True)
            except Exception as e:
                print(f"channels_last={cl} graph={gr}: ERROR {e}", flush=True)
