#!/usr/bin/env python
"""Practical HBM ceilings for K2's read:write mix (1 byte read : 2 bytes written for u8 -> bf16), measured
with plain PyTorch elementwise kernels on the same sizes as the epoch gather (49,152 rows x 3,072 B):
  cast   x_u8.to(bf16)            151 MB read, 302 MB written (K2's mix, contiguous)
  copy   y.copy_(x) bf16          302 MB read, 302 MB written (1:1, the MEASURED_PEAKS kind)
  fill   y.fill_(1)               302 MB written only
  read   x.sum() on int64 view    151 MB read only
"""
import torch

rows, rb = 49152, 3072
x = torch.randint(0, 256, (rows, rb), dtype=torch.uint8, device="cuda")
y = torch.empty((rows, rb), dtype=torch.bfloat16, device="cuda")
z = torch.empty_like(y)
flush = torch.empty(256 << 20, dtype=torch.uint8, device="cuda")


def t(fn, reps=20):
    fn()
    tot = 0.0
    for _ in range(reps):
        flush.zero_()
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record()
        fn()
        b.record()
        b.synchronize()
        tot += a.elapsed_time(b)
    return tot / reps * 1e3


xv = x.view(torch.int64)
for name, fn, by in [("cast u8->bf16", lambda: y.copy_(x), rows * rb * 3),
                     ("copy bf16", lambda: z.copy_(y), rows * rb * 4),
                     ("fill bf16", lambda: y.fill_(1), rows * rb * 2),
                     ("read u8 (sum)", lambda: xv.sum(), rows * rb)]:
    us = t(fn)
    print(f"{name:16s} {us:8.2f} us  {by / us / 1e3:8.1f} GB/s")

# the driver's memset (cudaMemsetAsync) as a second write-only reference
import ctypes
import glob
import os

cands = glob.glob(os.path.join(os.path.dirname(torch.__file__), "lib", "libcudart*.so*")) + \
    glob.glob("/usr/local/cuda/lib64/libcudart.so*")
if cands:
    rt = ctypes.CDLL(cands[0])
    rt.cudaMemsetAsync.argtypes = [ctypes.c_void_p, ctypes.c_int, ctypes.c_size_t, ctypes.c_void_p]
    nb = rows * rb * 2
    us = t(lambda: rt.cudaMemsetAsync(y.data_ptr(), 0, nb, torch.cuda.current_stream().cuda_stream))
    print(f"{'memset':16s} {us:8.2f} us  {nb / us / 1e3:8.1f} GB/s")
    big = torch.empty(4 << 30, dtype=torch.uint8, device="cuda")
    us = t(lambda: rt.cudaMemsetAsync(big.data_ptr(), 0, big.numel(), torch.cuda.current_stream().cuda_stream), 5)
    print(f"{'memset 4 GiB':16s} {us:8.2f} us  {big.numel() / us / 1e3:8.1f} GB/s")
    us = t(lambda: big.fill_(3), 5)
    print(f"{'fill 4 GiB':16s} {us:8.2f} us  {big.numel() / us / 1e3:8.1f} GB/s")
