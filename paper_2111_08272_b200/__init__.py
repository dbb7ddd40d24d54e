"""propring — B200-native proportional task allocation + sample-count-weighted ring allreduce.

The data-parallel hot path of arXiv 2111.08272 ("Task allocation for decentralized training in
heterogeneous environment"), as a C-ABI library (include/propring.h, libpropring.so built for sm_100a)
with this thin binding on top.  Every function here marshals arguments and calls the library; all
device work runs in the library's kernels.  PyTorch supplies device memory, streams and process groups.

    alloc_init(N, ratios, C, g, floor)      -> Alloc           static allocation
    Alloc.update(step_times)                -> changed          self-adaptive Eq. 10
    shard_indices(alloc, rank, epoch, seed, out)               per-epoch shard
    shard_steps(alloc, rank, epoch, seed, step0, nsteps, out)  step-interleaved shard (N3)
    gather_rows(src, idx, out, op, ...)                        step-batch gather
    comm_init(rank, P, device, group) / comm_init_local(P)     NVLink peer-memory communicator
    weighted_allreduce(comm, buf, n_local)                     Σ_r (n_r/Σn)·buf_r     (Eq. 1)
"""

from __future__ import annotations

import ctypes

from ._lib import (LIB, AllocPolicy, AllocView, CommConfig, EXCHANGE_FN, GatherOp, PR_MAX_RANKS,
                   PR_GATHER_MAX_CHANNELS)

PR_OK = 0
PR_ERR_INVALID = -1
PR_ERR_INFEASIBLE_FLOOR = -2
PR_ERR_DATASET_TOO_SMALL = -3
PR_ERR_ZERO_TIMING = -4
PR_ERR_CUDA = -5
PR_ERR_ALIGN = -6
PR_ERR_NO_P2P = -7
PR_ERR_LENGTH_MISMATCH = -8
PR_ERR_ZERO_SAMPLES = -9
PR_ERR_PEER_TIMEOUT = -10
PR_ERR_CAPACITY = -11
PR_ERR_INTERNAL = -12
PR_ERR_UNSUPPORTED = -13

GATHER_COPY = 0
GATHER_U8_TO_F32_AFFINE = 1
GATHER_U8_TO_BF16_AFFINE = 2
DTYPE_F32 = 0
DTYPE_BF16 = 1


# pr_alloc_policy.model (include/propring.h): the paper's Eq. 10, or the affine step-cost extension
ALLOC_MODEL_PROPORTIONAL = 0
ALLOC_MODEL_AFFINE = 1

class PropringError(RuntimeError):
    def __init__(self, code: int, where: str):
        self.code = code
        msg = LIB.pr_strerror(code).decode()
        if code == PR_ERR_CUDA:
            msg += f" ({LIB.pr_last_cuda_error().decode()})"
        super().__init__(f"{where}: {msg} [{code}]")


def _check(rc: int, where: str):
    if rc != PR_OK:
        raise PropringError(rc, where)


def version() -> int:
    return LIB.pr_version()


def _ptr(t):
    """Device (or host) address of a tensor / numpy array / int."""
    if t is None:
        return None
    if isinstance(t, int):
        return t
    if hasattr(t, "data_ptr"):
        return t.data_ptr()
    return t.ctypes.data


def _stream(stream):
    if stream is None:
        import torch
        return torch.cuda.current_stream().cuda_stream
    if isinstance(stream, int):
        return stream
    return stream.cuda_stream


# ---------------------------------------------------------------------------------------------------
# Allocation
# ---------------------------------------------------------------------------------------------------

class Alloc:
    """Owner of a pr_alloc handle (host state, replicated on every rank)."""

    def __init__(self, handle):
        self._h = handle

    def __del__(self):
        h, self._h = getattr(self, "_h", None), None
        if h:
            LIB.pr_alloc_destroy(h)

    @property
    def handle(self):
        return self._h

    def update(self, step_times) -> bool:
        P = self.view()["P"]
        arr = (ctypes.c_double * P)(*[float(x) for x in step_times])
        ch = ctypes.c_int32(0)
        _check(LIB.pr_alloc_update(self._h, arr, ctypes.byref(ch)), "pr_alloc_update")
        return bool(ch.value)

    def set_policy(self, window=2, tol=1, never_freeze=False, ema_alpha=1.0, model=ALLOC_MODEL_PROPORTIONAL,
                   fit_window=8):
        pol = AllocPolicy(window=window, never_freeze=1 if never_freeze else 0, tol=tol, ema_alpha=ema_alpha,
                          model=model, fit_window=fit_window)
        _check(LIB.pr_alloc_set_policy(self._h, ctypes.byref(pol)), "pr_alloc_set_policy")

    def view(self) -> dict:
        v = AllocView()
        _check(LIB.pr_alloc_query(self._h, ctypes.byref(v)), "pr_alloc_query")
        P = v.P
        return {"N": v.N, "P": P, "frozen": bool(v.frozen), "C": v.C, "g": v.g, "floor": v.floor, "B": v.B,
                "S": v.S, "epoch": v.epoch, "hist_len": v.hist_len, "w": list(v.w[:P]), "n": list(v.n[:P]),
                "len": list(v.len[:P]), "off": list(v.off[:P])}

    def history(self, k: int):
        P = self.view()["P"]
        out = (ctypes.c_int64 * P)()
        _check(LIB.pr_alloc_history(self._h, k, out), "pr_alloc_history")
        return list(out)

    def save(self) -> bytes:
        size = ctypes.c_size_t(0)
        _check(LIB.pr_alloc_save(self._h, None, 0, ctypes.byref(size)), "pr_alloc_save")
        buf = ctypes.create_string_buffer(size.value)
        _check(LIB.pr_alloc_save(self._h, buf, size.value, ctypes.byref(size)), "pr_alloc_save")
        return buf.raw[:size.value]

    @staticmethod
    def load(data: bytes) -> "Alloc":
        h = ctypes.c_void_p()
        buf = ctypes.create_string_buffer(data, len(data))
        _check(LIB.pr_alloc_load(ctypes.byref(h), buf, len(data)), "pr_alloc_load")
        return Alloc(h.value)


def alloc_init(N: int, ratios, C: int = 0, g: int = 1, floor: int = 1) -> Alloc:
    """Static allocation: w = Hamilton(C·r/Σr), n = g·w, shards D_i = D·w_i/Σw."""
    P = len(ratios)
    arr = (ctypes.c_double * P)(*[float(x) for x in ratios])
    h = ctypes.c_void_p()
    _check(LIB.pr_alloc_init(ctypes.byref(h), int(N), P, arr, int(C), int(g), int(floor)), "pr_alloc_init")
    return Alloc(h.value)


def alloc_update(alloc: Alloc, step_times) -> bool:
    return alloc.update(step_times)


# ---------------------------------------------------------------------------------------------------
# Sharder, gather, spin
# ---------------------------------------------------------------------------------------------------

def shard_indices(alloc: Alloc, rank: int, epoch: int, seed: int, out, stream=None):
    """out[t] = π_{seed,epoch}(off_rank + t), t < len_rank (K1).  out: int64 CUDA tensor."""
    _check(LIB.pr_shard_indices(alloc.handle, rank, epoch, seed & (2 ** 64 - 1), _ptr(out), out.numel(),
                                _stream(stream)), "pr_shard_indices")
    return out


def shard_steps(alloc: Alloc, rank: int, epoch: int, seed: int, step0: int, nsteps: int, out, stream=None):
    """Step-interleaved shard (N3): out[(s-step0)·n_r + t] = π(s·B + o_rank + t) for steps
    [step0, step0+nsteps) — the allocation may change between any two steps.  out: int64 CUDA tensor."""
    _check(LIB.pr_shard_steps(alloc.handle, rank, epoch, seed & (2 ** 64 - 1), step0, nsteps, _ptr(out),
                              out.numel(), _stream(stream)), "pr_shard_steps")
    return out


def permute(N: int, seed: int, epoch: int, begin: int, count: int, out, stream=None):
    _check(LIB.pr_permute(N, seed & (2 ** 64 - 1), epoch, begin, count, _ptr(out), _stream(stream)), "pr_permute")
    return out


GATHER_IMPL_AUTO = 0
GATHER_IMPL_LSU = 1
GATHER_IMPL_TMA = 2
GATHER_IMPL_BULK = 3
GATHER_LAYOUT_CHW = 0
GATHER_LAYOUT_HWC = 1


def make_gather_op(op=GATHER_COPY, scale=None, shift=None, plane=1, impl=GATHER_IMPL_AUTO,
                   layout=GATHER_LAYOUT_CHW):
    """pr_gather_op: per-channel affine (channels = len(scale), plane = H·W), kernel choice, output layout."""
    g = GatherOp()
    g.op = op
    g.impl = impl
    g.layout = layout
    if op != GATHER_COPY:
        n = len(scale)
        g.channels = n
        g.plane = plane
        for i in range(n):
            g.scale[i] = float(scale[i])
            g.shift[i] = float(shift[i])
    return g


def gather_rows(src, n_src: int, row_bytes: int, idx, n: int, out, op=None, lab_src=None, lab_dst=None,
                stream=None):
    """out[t] = op(src[idx[t]]), lab_dst[t] = lab_src[idx[t]] for t < n (K2).  src may be a device
    pointer or a mapped pinned host pointer (int)."""
    opp = ctypes.byref(op) if op is not None else None
    _check(LIB.pr_gather_rows(_ptr(src), n_src, row_bytes, _ptr(idx), n, _ptr(out), opp, _ptr(lab_src),
                              _ptr(lab_dst), _stream(stream)), "pr_gather_rows")
    return out


def spin(ns: int, stream=None):
    """Emulated slowdown (K4): busy-wait `ns` nanoseconds on the stream."""
    _check(LIB.pr_spin(int(ns), _stream(stream)), "pr_spin")


def stamp(ring, stream=None):
    """Append the device %globaltimer (ns) to ring[1 + (ring[0]++ mod cap)] (a5 t_s stamps inside graphs).
    ring: int64 CUDA tensor of 1 + cap entries; zero ring[0] to restart."""
    _check(LIB.pr_stamp(_ptr(ring), ring.numel() - 1, _stream(stream)), "pr_stamp")


def stamp_seconds(ring, out, stream=None):
    """out (device float64 scalar tensor) = Σ over ring's (start, end) stamp pairs, in seconds (a5 on device)."""
    _check(LIB.pr_stamp_seconds(_ptr(ring), ring.numel() - 1, _ptr(out), _stream(stream)), "pr_stamp_seconds")


def sgd_update(theta, grad, lr: float, wd: float = 0.0, zero_grad: bool = True, stream=None):
    """a9: θ ← θ − lr·(g + wd·θ) (two fp32 FMAs) and, if zero_grad, g ← 0 — one pass over flat fp32
    buffers (Eq. 1; wd P:235)."""
    if str(theta.dtype) != "torch.float32" or theta.dtype != grad.dtype or theta.numel() != grad.numel():
        raise ValueError("theta and grad must be fp32 buffers of equal length")
    _check(LIB.pr_sgd_update(_ptr(theta), _ptr(grad), theta.numel(), float(lr), float(wd), int(bool(zero_grad)),
                             _stream(stream)), "pr_sgd_update")


def test_philox(ctr, key: int, use_curand: bool, out, stream=None):
    n = ctr.numel() // 4
    _check(LIB.pr_test_philox(_ptr(ctr), n, key, 1 if use_curand else 0, _ptr(out), _stream(stream)),
           "pr_test_philox")
    return out


# ---------------------------------------------------------------------------------------------------
# Communicator + weighted ring allreduce
# ---------------------------------------------------------------------------------------------------

COMM_FLAG_FORCE_STAGED = 1
COMM_FLAG_SYS_SCOPE = 2
COMM_FLAG_BULK_STORE = 4
COMM_FLAG_L2_PREFETCH = 8
COMM_FLAG_PULL_TMA = 16
ALGO_RING = 0
ALGO_TWO_SHOT = 1
ALGO_AUTO = 2
ALGO_LL = 3
ALGO_ONESHOT = 4
ALGO_NVLS = 5
ALGO_TWO_SHOT_PULL = 6


def comm_config(channels=0, slots=8, threads=512, slot_bytes=0, watchdog_ns=10_000_000_000,
                force_staged=False, stages=0, tile_bytes=0, sys_scope=False, algo=ALGO_RING, ts_slots=2,
                ts_slot_bytes=256 * 1024, ts_max_bytes=4 << 20, ll_max_bytes=256 * 1024,
                os_max_bytes=64 * 1024, min_slice_bytes=0, bulk_store=False, l2_prefetch=False, pull_tma=False):
    """K3 launch/pipeline configuration.  channels / slot_bytes / stages / tile_bytes = 0: chosen at init from
    the topology (one GPU: 128/P channels (16 at P = 8, at most 64) / 256 KiB / 7 / 16 KiB, the co-located
    optimum of tools/sweep_ring.py; ranks on different GPUs: 32 / 1 MiB / 7 / 16 KiB, from the per-channel
    throughput of tools/sweep_cta.py).
    sys_scope=True forces system-scope synchronisation even when all ranks share one GPU (tests).
    algo: ALGO_RING (the paper's ring), ALGO_LL (the ring with the low-latency line protocol, buffers up to
    ll_max_bytes), ALGO_ONESHOT (one hop, buffers up to os_max_bytes), ALGO_TWO_SHOT, ALGO_TWO_SHOT_PULL (the
    two-shot with its first phase as loads from the peers' registered buffers), or ALGO_AUTO (one-shot up to
    os_max_bytes, LL up to ll_max_bytes, the pull two-shot for registered buffers up to ts_max_bytes, ring
    above)."""
    flags = ((COMM_FLAG_FORCE_STAGED if force_staged else 0) | (COMM_FLAG_SYS_SCOPE if sys_scope else 0)
             | (COMM_FLAG_BULK_STORE if bulk_store else 0) | (COMM_FLAG_L2_PREFETCH if l2_prefetch else 0)
             | (COMM_FLAG_PULL_TMA if pull_tma else 0))
    return CommConfig(channels=channels, slots=slots, threads=threads, flags=flags, slot_bytes=slot_bytes,
                      watchdog_ns=watchdog_ns, stages=stages, tile_bytes=tile_bytes, algo=algo, ts_slots=ts_slots,
                      ts_slot_bytes=ts_slot_bytes, ts_max_bytes=ts_max_bytes, ll_max_bytes=ll_max_bytes,
                      os_max_bytes=os_max_bytes, min_slice_bytes=min_slice_bytes)


class _DeviceBuffer:
    """__cuda_array_interface__ view of library-owned device memory (pr_comm_alloc)."""

    def __init__(self, ptr, nbytes, device):
        self.__cuda_array_interface__ = {"shape": (nbytes,), "typestr": "|u1", "data": (ptr, False), "version": 3}
        self.device = device


class Comm:
    def __init__(self, handle, keepalive=None):
        self._h = handle
        self._keep = keepalive
        self._owned = []

    @property
    def handle(self):
        return self._h

    def rank_size(self):
        r, s = ctypes.c_int32(), ctypes.c_int32()
        _check(LIB.pr_comm_rank(self._h, ctypes.byref(r), ctypes.byref(s)), "pr_comm_rank")
        return r.value, s.value

    def register(self, tensor):
        _check(LIB.pr_comm_register(self._h, _ptr(tensor), tensor.numel() * tensor.element_size()),
               "pr_comm_register")

    def alloc(self, nbytes: int, dtype=None, device=None):
        """Library-owned, IPC-registered device memory wrapped as a torch tensor (uint8 or `dtype`)."""
        import torch
        p = ctypes.c_void_p()
        _check(LIB.pr_comm_alloc(self._h, nbytes, ctypes.byref(p)), "pr_comm_alloc")
        dev = device if device is not None else torch.device("cuda", torch.cuda.current_device())
        t = torch.as_tensor(_DeviceBuffer(p.value, nbytes, dev), device=dev)
        self._owned.append(t)
        return t.view(dtype) if dtype is not None else t

    def nvls_alloc(self, nbytes: int, dtype=None, device=None):
        """NVLS region (collective): this rank's unicast view of memory bound to one NVSwitch multicast object
        across all ranks, as a torch tensor.  Raises PropringError(PR_ERR_UNSUPPORTED) where the platform has
        no multicast (every rank together)."""
        import torch
        p = ctypes.c_void_p()
        _check(LIB.pr_comm_nvls_alloc(self._h, nbytes, ctypes.byref(p)), "pr_comm_nvls_alloc")
        dev = device if device is not None else torch.device("cuda", torch.cuda.current_device())
        t = torch.as_tensor(_DeviceBuffer(p.value, nbytes, dev), device=dev)
        self._owned.append(t)
        return t.view(dtype) if dtype is not None else t

    def allgather_f64(self, x: float, stream=None):
        P = self.rank_size()[1]
        out = (ctypes.c_double * P)()
        _check(LIB.pr_comm_allgather_f64(self._h, float(x), out, _stream(stream)), "pr_comm_allgather_f64")
        return list(out)

    def allgather_f64_async(self, d_local, h_out, stream=None):
        """K6 without a host synchronisation: d_local (device float64 scalar) -> h_out (pinned float64 [P]),
        stream-ordered; read h_out after an event recorded behind this call."""
        _check(LIB.pr_comm_allgather_f64_async(self._h, _ptr(d_local), _ptr(h_out), _stream(stream)),
               "pr_comm_allgather_f64_async")

    def status(self) -> int:
        return LIB.pr_comm_status(self._h)

    def timestamps(self):
        out = (ctypes.c_int64 * 3)()
        _check(LIB.pr_comm_timestamps(self._h, out), "pr_comm_timestamps")
        return list(out)

    def destroy(self):
        h, self._h = self._h, None
        self._owned = []
        if h:
            LIB.pr_comm_destroy(h)


def torch_exchange(group=None):
    """A pr_exchange_fn over a torch.distributed process group (byte allgather, rank-ordered)."""
    import torch
    import torch.distributed as dist

    def _fn(ctx, send, length, recv):
        try:
            backend = dist.get_backend(group)
            dev = torch.device("cuda", torch.cuda.current_device()) if backend == "nccl" else torch.device("cpu")
            src = torch.frombuffer(bytearray(ctypes.string_at(send, length)), dtype=torch.uint8).to(dev)
            world = dist.get_world_size(group)
            outs = [torch.empty(length, dtype=torch.uint8, device=dev) for _ in range(world)]
            dist.all_gather(outs, src, group=group)
            data = b"".join(o.cpu().numpy().tobytes() for o in outs)
            ctypes.memmove(recv, data, len(data))
            return 0
        except Exception:   # never raise through C
            return 1

    return EXCHANGE_FN(_fn)


def comm_init(rank: int, P: int, device: int, exchange=None, config=None) -> Comm:
    """One process per GPU: CUDA-IPC bootstrap over `exchange` (default: the torch default group)."""
    fn = exchange if exchange is not None else torch_exchange()
    h = ctypes.c_void_p()
    cfg = ctypes.byref(config) if config is not None else None
    _check(LIB.pr_comm_init(ctypes.byref(h), rank, P, device, fn, None, cfg), "pr_comm_init")
    return Comm(h.value, keepalive=fn)


def comm_init_local(P: int, device: int = 0, config=None):
    """P ranks in this process on one device (test / emulation mode)."""
    arr = (ctypes.c_void_p * P)()
    cfg = ctypes.byref(config) if config is not None else None
    _check(LIB.pr_comm_init_local(arr, P, device, cfg), "pr_comm_init_local")
    return [Comm(arr[r]) for r in range(P)]


def _dtype_code(t):
    import torch
    if t.dtype == torch.float32:
        return DTYPE_F32
    if t.dtype == torch.bfloat16:
        return DTYPE_BF16
    raise TypeError(f"unsupported dtype {t.dtype}")


def weighted_allreduce(comm: Comm, buf, n_local: int, stream=None, count=None):
    """buf <- Σ_r (n_r/Σn)·buf_r in place (K3; Eq. 1).  buf: contiguous fp32/bf16 CUDA tensor."""
    cnt = buf.numel() if count is None else count
    _check(LIB.pr_weighted_allreduce(comm.handle, _ptr(buf), cnt, _dtype_code(buf), int(n_local), _stream(stream)),
           "pr_weighted_allreduce")
    return buf


def weighted_allreduce_sgd(comm: Comm, grad, theta, n_local: int, lr: float, wd: float = 0.0, zero_grad: bool = True,
                           stream=None):
    """Rows a6-a9 in one call: θ ← θ − lr·(ḡ + wd·θ) with ḡ = Σ_r (n_r/Σn)·grad_r, and grad ← 0 — one fused
    kernel (K7 in K3) when the ring takes the call and grad/theta share a registered region at the same
    offset on every rank, else the composed pair (same bits).  fp32 only."""
    if str(grad.dtype) != "torch.float32" or grad.dtype != theta.dtype or grad.numel() != theta.numel():
        raise ValueError("grad and theta must be fp32 buffers of equal length")
    _check(LIB.pr_weighted_allreduce_sgd(comm.handle, _ptr(grad), _ptr(theta), grad.numel(), int(n_local), float(lr),
                                         float(wd), int(bool(zero_grad)), _stream(stream)), "pr_weighted_allreduce_sgd")


def weighted_allreduce_sgd_local(comms, grads, thetas, n_local, lr: float, wd: float = 0.0, zero_grad: bool = True,
                                 stream=None):
    """Local-group form of weighted_allreduce_sgd (all ranks in one launch)."""
    P = len(comms)
    hs = (ctypes.c_void_p * P)(*[c.handle for c in comms])
    gs = (ctypes.c_void_p * P)(*[_ptr(b) for b in grads])
    ts = (ctypes.c_void_p * P)(*[_ptr(b) for b in thetas])
    ns = (ctypes.c_int64 * P)(*[int(x) for x in n_local])
    _check(LIB.pr_weighted_allreduce_sgd_local(hs, gs, ts, grads[0].numel(), ns, float(lr), float(wd),
                                               int(bool(zero_grad)), _stream(stream)), "pr_weighted_allreduce_sgd_local")


def weighted_allreduce_local(comms, bufs, n_local, stream=None, count=None):
    """All ranks of a comm_init_local group in one launch."""
    P = len(comms)
    hs = (ctypes.c_void_p * P)(*[c.handle for c in comms])
    bs = (ctypes.c_void_p * P)(*[_ptr(b) for b in bufs])
    ns = (ctypes.c_int64 * P)(*[int(x) for x in n_local])
    cnt = bufs[0].numel() if count is None else count
    _check(LIB.pr_weighted_allreduce_local(hs, bs, cnt, _dtype_code(bufs[0]), ns, _stream(stream)),
           "pr_weighted_allreduce_local")
    return bufs
