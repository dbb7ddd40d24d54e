"""Training harness around the library: Algorithm 1 on one rank of a P-rank job.

Rows of SURVEY §8(a) handled here (the rest are library calls):
  a4  local compute + gradient accumulation: "accumulate gradients without back propagation [= without
      a parameter update] ... until w_i samples are transferred" (P:69 steps (1)-(3)).  The rank's n_r
      samples are processed in microbatches of at most `micro` rows; each microbatch loss is scaled by
      mb/n_r so the flat gradient buffer ends up holding the LOCAL MEAN gradient (DESIGN.md §3 #11).
      Emulated heterogeneity: a K4 spin of (σ_r − 1)·t1(n_r) after each step's graph replay, t1(n_r) the
      rank's own measured step time for its n_r rows at σ = 1 (prepare()), slows rank r by the factor σ_r
      (the eager path without graphs falls back to a per-sample calibration, c0·n_r).
  a5  t_s capture: CUDA events around data movement + compute + spin, summed over the epoch (P:102,
      P:152; DESIGN.md §3 #4-#5); one event synchronisation per epoch, not per step.
  a9  SGD update, Eq. 1 with weight decay: the library's fused pr_sgd_update over the
      flat parameter / reduced-gradient buffers (also resets the gradient for the next aggregation);
      fused_sgd=False uses torch.optim.SGD + a memset instead.
Library rows: a1/a10 alloc_init / Alloc.update (+ pr_comm_allgather_f64 for the t_s exchange),
a2 shard_indices, a3 gather_rows, a6-a8 weighted_allreduce.

Data movement (a3): by default ONE K2 launch per epoch gathers the rows of all S aggregation steps
(S·n_r rows, in step order) into a resident buffer — the same rows in the same order as S per-step
gathers, but HBM-bound instead of launch-latency-bound; its time is part of t_s.  gather="step"
issues one launch per aggregation step instead.

Parameters' .grad are views into one flat fp32 buffer allocated by the communicator (CUDA-IPC
registered), so backward() accumulates straight into the buffer the ring reduces in place.
"""

from __future__ import annotations

import time
from dataclasses import dataclass, field

import torch
import torch.nn.functional as F

import paper_2111_08272_b200 as pr

CIFAR_MEAN = [125.307, 122.961, 113.8575]
CIFAR_STD = [51.5865, 50.847, 51.255]


@dataclass
class RunConfig:
    N: int = 50_000
    shape: tuple = (3, 32, 32)
    classes: int = 10
    model: str = "resnet18"                 # resnet18 | vgg16 (u8 images) | logreg | mlp (fp32 feature rows)
    num_classes: int = 1000                 # head size of the gradient buffer (DESIGN.md §3 #31)
    ratios: list = field(default_factory=lambda: [1])
    C: int = 0
    g: int = 128
    floor: int = 1
    seed: int = 1234
    lr: float = 1e-2
    wd: float = 1e-4
    micro: int = 512                        # max rows per microbatch
    slowdown: list | None = None            # σ_r per rank (emulated heterogeneity)
    adaptive: bool = False                  # Algorithm 1 self-adaptive allocation
    host_data: bool = False                 # e2e: data set in pinned host memory, gathered over PCIe
    bf16_compute: bool = True               # autocast for the model's forward/backward
    gather: str = "epoch"                   # "epoch": one K2 launch per epoch; "step": one per step
    channels_last: bool = True              # K2 writes HWC rows; the model runs channels-last (no transposes)
    graphs: bool = True                     # capture each step's forward/backward (+ spin) in a CUDA graph
    # N3: intra-epoch controller.  adapt_every = k > 0 runs the epoch as segments of k
    # aggregation steps over the step-interleaved shard (pr_shard_steps) and calls the controller at every
    # segment boundary with that segment's t_s; 0 = once per epoch (Algorithm 1 as written).
    adapt_every: int = 0
    # N3 exchange cadence: 0 = the segment's t_s is read on the host (CUDA events) and exchanged with the
    # synchronous K6 before the next segment; 1 = t_s is summed on the device from %globaltimer stamps and
    # exchanged with the asynchronous K6 (pinned host result, no stream synchronisation), and the
    # controller applies segment j's times before segment j + 2 (one segment of lag, DESIGN.md §3 #47)
    adapt_lag: int = 0
    policy: dict | None = None              # Alloc.set_policy kwargs (e.g. never_freeze, ema_alpha)
    # time-varying stragglers: [(global_step, [σ_r ...]), ...]; σ at step s = the last entry with step <= s
    slowdown_schedule: list | None = None
    # N1: overlap the weighted allreduce with backward.  The flat gradient buffer is cut into
    # ~bucket_mb buckets in reverse parameter order; each bucket's K3 is launched on a comm stream from a
    # post-accumulate-grad hook as soon as its last gradient is final (in bucket order on every rank).
    # Needs graphs=True (the overlapped step is one captured graph per n_r).
    overlap: bool = False
    bucket_mb: float = 8.0
    # a9 through the library's fused kernel (pr_sgd_update: SGD + gradient reset in one pass over flat
    # fp32 parameter / gradient buffers) instead of torch.optim.SGD + a separate memset
    fused_sgd: bool = True
    # K4 emulation of a rank σ_r× slower (DESIGN.md §3 #46): "t1" spins (σ_r − 1)·t1(n_r) after each step —
    # the rank's whole step (fixed + per-sample cost) takes σ_r× its own σ = 1 time; "sample" spins
    # (σ_r − 1)·c0·n_r — SURVEY §8(a) a4's per-sample spin, c0 = t1(n)/n at the first n_r this rank runs
    # (only the per-sample part is slowed; every rank pays the same fixed cost).
    spin: str = "t1"


FEATURE_MODELS = ("logreg", "mlp")           # fp32 feature rows (gathered by K2's COPY op), no images


def build_model(name: str, num_classes: int, in_features: int = 1024):
    """The harness's model (row a4).  logreg: BASELINE configs[0]'s 1,024-weight logistic regression without
    bias (DESIGN.md §3 #30), θ_0 = 0; mlp: a small fp32 multi-layer model whose several
    parameter tensors give N1 several buckets in the parity tests."""
    import torch.nn as nn

    if name == "logreg":
        m = nn.Linear(in_features, 1, bias=False)
        nn.init.zeros_(m.weight)
        return m
    if name == "mlp":
        return nn.Sequential(nn.Linear(in_features, 256), nn.ReLU(), nn.Linear(256, 128), nn.ReLU(),
                             nn.Linear(128, num_classes))
    import torchvision

    if name == "resnet18":
        return torchvision.models.resnet18(num_classes=num_classes)
    if name == "vgg16":
        return torchvision.models.vgg16(num_classes=num_classes)
    raise ValueError(name)


class Worker:
    """One rank: owns the data set copy, the model, the flat gradient buffer and the communicator."""

    def __init__(self, cfg: RunConfig, rank: int = 0, world: int = 1, device: int = 0, comm=None,
                 data=None, labels=None):
        self.cfg, self.rank, self.P = cfg, rank, world
        self.dev = torch.device("cuda", device)
        torch.cuda.set_device(self.dev)
        self.comm = comm
        self.stream = torch.cuda.current_stream(self.dev)
        self.alloc = pr.alloc_init(cfg.N, cfg.ratios, C=cfg.C, g=cfg.g, floor=cfg.floor)
        if cfg.policy:
            self.alloc.set_policy(**cfg.policy)
        self.gstep = 0                                # global aggregation-step counter (slowdown schedule)
        self.features = cfg.model in FEATURE_MODELS
        if self.features and (cfg.channels_last or cfg.bf16_compute):
            raise ValueError("feature models run fp32 rows: set channels_last=False, bf16_compute=False")
        self.row_elems = int(torch.tensor(cfg.shape).prod())          # output elements per gathered row
        self.row_bytes = self.row_elems * (4 if self.features else 1)  # source bytes per row (fp32 / u8)
        if data is None:                              # synthetic data set, replicated per rank
            import synth

            if self.features:
                xf, yf, _ = synth.logistic_problem(cfg.N, self.row_elems)
                data = torch.from_numpy(xf.astype("float32"))
                labels = torch.from_numpy(yf.astype("int64")) if cfg.model == "logreg" else \
                    torch.from_numpy(synth.labels(cfg.N, cfg.classes, seed=1))
            else:
                data = torch.from_numpy(synth.images_u8(cfg.N, *cfg.shape, seed=0).reshape(cfg.N, -1))
                labels = torch.from_numpy(synth.labels(cfg.N, cfg.classes, seed=1))
        self.X = data.pin_memory() if cfg.host_data else data.to(self.dev)
        self.Y = labels.to(self.dev)
        # K2 kernel chosen here, as the library's AUTO rule would (host data -> LSU, channels-last -> the
        # bulk-store kernel, CHW -> TMA), so the launch does no host-side pointer query
        lsu = cfg.host_data
        if self.features:                             # fp32 rows: a byte-exact copy (O5 COPY)
            self.gop = pr.make_gather_op(pr.GATHER_COPY, impl=pr.GATHER_IMPL_LSU)
        else:
            C, H, W = cfg.shape
            self.gop = pr.make_gather_op(pr.GATHER_U8_TO_BF16_AFFINE if cfg.bf16_compute else pr.GATHER_U8_TO_F32_AFFINE,
                                         [1.0 / s for s in CIFAR_STD[:C]], CIFAR_MEAN[:C], H * W,
                                         impl=pr.GATHER_IMPL_LSU if lsu else
                                         pr.GATHER_IMPL_BULK if cfg.channels_last else pr.GATHER_IMPL_TMA,
                                         layout=pr.GATHER_LAYOUT_HWC if cfg.channels_last else pr.GATHER_LAYOUT_CHW)
        torch.backends.cudnn.benchmark = True
        # try every cuDNN algorithm when autotuning (default: the first 10 heuristics' picks): the
        # ResNet-18 step settles at 2.90-2.91 ms instead of 3.08-3.09 (tools/model_variance.py, 6 runs each)
        torch.backends.cudnn.benchmark_limit = 0
        torch.manual_seed(cfg.seed)                   # identical initial weights on every rank
        self.model = build_model(cfg.model, cfg.num_classes, self.row_elems).to(self.dev)
        if cfg.channels_last:
            self.model = self.model.to(memory_format=torch.channels_last)
        self._graphs = {}                             # n_r -> captured step
        self._pool = None
        params = list(self.model.parameters())
        self.L = sum(p.numel() for p in params)
        self._raw = None
        Lp = (self.L + 3) // 4 * 4
        if comm is not None and cfg.fused_sgd:
            # one IPC-registered region [grad | θ], θ at the same offset on every rank: the fused a6-a9 call
            # (K7 inside K3's ring) all-gathers θ' straight into every rank's parameters
            self._raw = comm.alloc(2 * Lp * 4, dtype=torch.float32)
            self.flat = self._raw[:self.L]
        elif comm is not None:
            self.flat = comm.alloc(self.L * 4, dtype=torch.float32)   # IPC-registered: direct all-gather
        else:
            self.flat = torch.zeros(self.L, dtype=torch.float32, device=self.dev)
        off = 0
        for p in params:   # .grad = a view of the flat buffer with the parameter's own (channels-last) strides
            p.grad = self.flat[off:off + p.numel()].as_strided(p.shape, p.stride())
            off += p.numel()
        self.pflat = None
        if cfg.fused_sgd:  # parameters become views of one flat fp32 buffer laid out like the gradient
            self.pflat = (self._raw[Lp:Lp + self.L] if self._raw is not None
                          else torch.empty(self.L, dtype=torch.float32, device=self.dev))
            off = 0
            with torch.no_grad():
                for p in params:
                    v = self.pflat[off:off + p.numel()].as_strided(p.shape, p.stride())
                    v.copy_(p.data)
                    p.data = v
                    off += p.numel()
            self.opt = None
        else:
            self.opt = torch.optim.SGD(params, lr=cfg.lr, weight_decay=cfg.wd)
        self._overlap = bool(cfg.overlap and comm is not None and world > 1)
        if cfg.overlap and not cfg.graphs:
            raise ValueError("overlap=True needs graphs=True")
        if self._overlap:
            self._setup_buckets(params)
        self.idx = torch.empty(cfg.N, dtype=torch.int64, device=self.dev)   # any shard size after re-allocation
        self.xdt = torch.bfloat16 if cfg.bf16_compute else torch.float32
        self.c0_ns = 0.0                               # calibrated per-sample compute time (ns) at σ = 1
        self.launches = 0                              # library kernels launched (for the bench)
        self.ar_events, self.gather_events, self.sgd_events = [], [], []
        self.epoch = 0
        self.last_ts = 0.0
        self.history = []
        # observation hooks (tests, diagnostics): on_reduced(worker) runs after the step's weighted
        # allreduce and before the update when the reduced gradient exists as a buffer (not with the
        # fused a6-a9 kernel); on_step(worker) runs after the update.  Host-side, in enqueue order.
        self.on_reduced = None
        self.on_step = None

    # ---- N1: bucketed allreduce overlapped with backward ----------------------------------------------
    def _setup_buckets(self, params):
        """Buckets = contiguous ranges [lo, hi) of the flat buffer, filled in reverse parameter order (the
        order backward finalises gradients), closed at >= bucket_mb and at 16-byte boundaries (K3 alignment)."""
        import functools

        spans, off = [], 0
        for p in params:
            spans.append((off, off + p.numel()))
            off += p.numel()
        limit = max(4, int(self.cfg.bucket_mb * 2 ** 20 / 4))
        self._buckets, bucket_of, cur, hi = [], {}, [], None
        for i in reversed(range(len(params))):
            lo = spans[i][0]
            hi = spans[i][1] if hi is None else hi
            cur.append(i)
            if (hi - lo >= limit and lo % 4 == 0) or i == 0:
                for j in cur:
                    bucket_of[j] = len(self._buckets)
                self._buckets.append((lo, hi, len(cur)))
                cur, hi = [], None
        self._ready = [0] * len(self._buckets)
        self._next, self._armed, self._n_armed = 0, False, 0
        self._bucket_ev = [torch.cuda.Event() for _ in self._buckets]
        self.comm_stream = torch.cuda.Stream(self.dev)
        self.stamps = torch.zeros(1 + 2 * (self.cfg.N + 1), dtype=torch.int64, device=self.dev)
        for i, p in enumerate(params):
            p.register_post_accumulate_grad_hook(functools.partial(self._grad_ready, bucket_of[i]))

    def _grad_ready(self, b, _param):
        """Post-accumulate-grad hook (runs while backward is captured): launch every bucket that is complete,
        in bucket order, on the comm stream after the work that produced it."""
        if not self._armed:
            return
        self._ready[b] += 1
        while self._next < len(self._buckets) and self._ready[self._next] == self._buckets[self._next][2]:
            lo, hi, _ = self._buckets[self._next]
            ev = self._bucket_ev[self._next]
            ev.record(torch.cuda.current_stream(self.dev))
            self.comm_stream.wait_event(ev)
            self._bucket_call(lo, hi, self._n_armed, self.comm_stream)
            self._next += 1

    def _bucket_call(self, lo, hi, n, stream):
        """One bucket's a6-a8 — or, with the flat [grad | θ] region, a6-a9 fused (K7 inside K3): the bucket's
        layers have finished their backward on every rank (the handshake waits for all), so their θ can be
        updated while backward continues on earlier layers (which never read these weights again; the
        forward's bf16 weight copies are what backward saved)."""
        if self.pflat is not None:
            pr.weighted_allreduce_sgd(self.comm, self.flat[lo:hi], self.pflat[lo:hi], n, self.cfg.lr, self.cfg.wd,
                                      zero_grad=True, stream=stream)
        else:
            pr.weighted_allreduce(self.comm, self.flat[lo:hi], n, stream=stream)

    # ---- a3: data movement --------------------------------------------------------------------------
    def gather(self, first: int, rows: int, record=False, stream=None, persistent=False):
        """K2: rows [first, first+rows) of this rank's shard -> (x [rows, C·H·W], y [rows]).
        persistent: write into one of two epoch buffers kept for the run (ping-pong: the next epoch's
        prefetch never touches the buffer the current epoch reads), so no allocation happens per epoch."""
        st = self.stream if stream is None else stream
        if persistent:
            if not hasattr(self, "_ebuf"):
                self._ebuf, self._eflip = [None, None], 0
            self._eflip ^= 1
            b = self._ebuf[self._eflip]
            if b is None or b[0].shape[0] < max(rows, 1):
                b = (torch.empty((max(rows, 1), self.row_elems), dtype=self.xdt, device=self.dev),
                     torch.empty(max(rows, 1), dtype=torch.int64, device=self.dev))
                self._ebuf[self._eflip] = b
            x, y = b[0][:max(rows, 1)], b[1][:max(rows, 1)]
        else:
            with torch.cuda.stream(st):               # outputs allocated on (and owned by) the launching stream
                x = torch.empty((max(rows, 1), self.row_elems), dtype=self.xdt, device=self.dev)
                y = torch.empty(max(rows, 1), dtype=torch.int64, device=self.dev)
        if rows > 0:
            if record:
                g0, g1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                g0.record(st)
            pr.gather_rows(self.X.data_ptr(), self.cfg.N, self.row_bytes, self.idx[first:], rows, x, self.gop, self.Y,
                           y, stream=st)
            self.launches += 1
            if record:
                g1.record(st)
                self.gather_events.append((g0, g1, rows))
        return x, y

    # ---- a4: forward/backward with gradient accumulation (P:69 steps (1)-(3)) --------------------------
    def _input(self, x, n_r: int):
        if self.features:
            return x[:n_r]
        C, H, W = self.cfg.shape
        if self.cfg.channels_last:                    # HWC rows -> logical NCHW with channels-last strides
            return x[:n_r].view(n_r, H, W, C).permute(0, 3, 1, 2)
        return x[:n_r].view(n_r, C, H, W)

    def compute(self, x, y, n_r: int, overlap: bool = False):
        cfg = self.cfg
        x = self._input(x, n_r)
        losses = []
        for m0 in range(0, n_r, cfg.micro):
            xm, ym = x[m0:m0 + cfg.micro], y[m0:m0 + cfg.micro]
            with torch.autocast("cuda", dtype=torch.bfloat16, enabled=cfg.bf16_compute):
                out = self.model(xm)
                if cfg.model == "logreg":   # mean binary cross-entropy: ∇ = Xᵀ(σ(Xθ) − y)/n (O7)
                    loss = F.binary_cross_entropy_with_logits(out.float().squeeze(1), ym.float())
                else:
                    loss = F.cross_entropy(out.float(), ym)
            if overlap and m0 + cfg.micro >= n_r:             # N1: the last microbatch finalises every grad
                self._ready, self._next, self._armed, self._n_armed = [0] * len(self._buckets), 0, True, n_r
            (loss * (xm.shape[0] / n_r)).backward()           # local mean over n_r (DESIGN §3 #11)
            losses.append(loss.detach() * xm.shape[0])
        if overlap:
            self._armed = False
            if self._next != len(self._buckets):
                raise RuntimeError(f"N1: {self._next} of {len(self._buckets)} buckets launched")
            cur = torch.cuda.current_stream(self.dev)
            pr.stamp(self.stamps, stream=cur)                  # end of this rank's compute (t_s, a5)
            cur.wait_stream(self.comm_stream)                  # join: the update needs the reduced buffer
        ns = self._spin_ns(n_r)
        if ns > 0:
            pr.spin(ns)                                      # K4 on the current (possibly capturing) stream
            self.launches += 1
        return torch.stack(losses).sum() / n_r

    def sigma(self, rank: int | None = None) -> float:
        """Emulated slowdown σ of `rank` at the current global step (K4 target)."""
        rank = self.rank if rank is None else rank
        sched = self.cfg.slowdown_schedule
        if sched:
            cur = None
            for step, sig in sched:
                if step <= self.gstep:
                    cur = sig
            if cur is not None:
                return float(cur[rank])
        return float(self.cfg.slowdown[rank]) if self.cfg.slowdown else 1.0

    def _spin_ns(self, n_r: int, t1_ns: float = 0.0) -> int:
        """K4 spin of this rank at the current step: (σ−1)·t1(n_r) ("t1"), or (σ−1)·c0·n_r ("sample", and the
        eager path without a captured t1)."""
        sigma = self.sigma() if self.cfg.slowdown or self.cfg.slowdown_schedule else 1.0
        if sigma <= 1.0:
            return 0
        if self.cfg.spin == "t1" and t1_ns > 0:
            return int((sigma - 1.0) * t1_ns)
        return int((sigma - 1.0) * self.c0_ns * n_r) if self.c0_ns > 0 else 0

    def prepare(self, n_r: int, calib_reps: int = 3):
        """Capture the forward/backward of n_r rows in a CUDA graph and time its replay, t1(n_r) — the
        rank's compute time at σ = 1.  Done OUTSIDE any timed region (warm-up and capture would otherwise
        pollute t_s).  Capture is rank-local (no collective inside), so a rank whose n_r changes
        re-captures alone."""
        if n_r <= 0 or n_r in self._graphs:
            return
        xs = torch.randn((n_r, self.row_elems), device=self.dev).to(self.xdt)
        ys = torch.randint(0, self.cfg.classes, (n_r,), device=self.dev)
        side = torch.cuda.Stream(self.dev)
        side.wait_stream(self.stream)
        launches, save, save_sched = self.launches, self.cfg.slowdown, self.cfg.slowdown_schedule
        self.cfg.slowdown = self.cfg.slowdown_schedule = None  # the spin is launched after the replay
        with torch.cuda.stream(side):
            self.compute(xs, ys, n_r)                         # warm-up (cuDNN autotune, allocator)
        self.stream.wait_stream(side)
        g = torch.cuda.CUDAGraph()
        if self._pool is None:
            self._pool = torch.cuda.graph_pool_handle()
        # one memory pool for every n_r's graph: the graphs replay one at a time on one stream and keep no
        # temporaries live between replays, so a re-allocation that visits many n_r costs no extra memory
        with torch.cuda.graph(g, pool=self._pool, stream=side):
            loss = self.compute(xs, ys, n_r)
        self.stream.wait_stream(side)
        self.cfg.slowdown, self.cfg.slowdown_schedule, self.launches = save, save_sched, launches
        g.replay()                                            # warm replay, then t1(n_r)
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record(self.stream)
        for _ in range(calib_reps):
            g.replay()
        b.record(self.stream)
        b.synchronize()
        self.flat.zero_()                                     # discard the warm-up/calibration gradients
        g2 = loss2 = None
        if self._overlap:
            # N1: a second graph of the same step whose backward launches the bucket allreduces (capture
            # executes nothing, so no collective runs here; the plain graph above gave t1 without them)
            g2 = torch.cuda.CUDAGraph()
            side.wait_stream(self.stream)
            self.cfg.slowdown = self.cfg.slowdown_schedule = None
            with torch.cuda.graph(g2, pool=self._pool, stream=side):
                loss2 = self.compute(xs, ys, n_r, overlap=True)
            self.stream.wait_stream(side)
            self.cfg.slowdown, self.cfg.slowdown_schedule = save, save_sched
        t1_ns = a.elapsed_time(b) * 1e6 / calib_reps
        if self.c0_ns == 0.0:
            self.c0_ns = t1_ns / n_r                           # per-sample cost at the first n_r ("sample" spin)
        self._graphs[n_r] = (g, xs, ys, loss, t1_ns, g2, loss2)

    def compute_graphed(self, x, y, n_r: int):
        """a4 through the captured graph; emulated slowdown σ_r (K4): a rank σ× slower takes σ× its own
        measured compute time, so the spin is (σ_r − 1)·t1(n_r) for the n_r it actually processes."""
        self.prepare(n_r)
        g, xs, ys, loss, t1_ns, g2, loss2 = self._graphs[n_r]
        xs.copy_(x[:n_r])
        ys.copy_(y[:n_r])
        ns = self._spin_ns(n_r, t1_ns)
        if g2 is not None:
            # N1: stamp, slowdown first (a slower GPU finishes every bucket later), then the step whose
            # backward overlaps the bucket allreduces; the graph stamps the end of compute before its join
            pr.stamp(self.stamps, stream=self.stream)
            if ns > 0:
                pr.spin(ns, stream=self.stream)
            g2.replay()
            self.launches += 2 + len(self._buckets) + (ns > 0)
            return loss2.clone()
        g.replay()
        if ns > 0:
            pr.spin(ns, stream=self.stream)
            self.launches += 1
        return loss.clone()

    def t1(self, n_r: int) -> float:
        """Measured σ = 1 step time t1(n_r) in seconds (captures the step first if needed)."""
        self.prepare(n_r)
        return self._graphs[n_r][4] / 1e9

    # ---- a6-a9: weighted ring allreduce + SGD (Algorithm 1 steps 5-6) ---------------------------------
    def allreduce_and_update(self, n_r: int, record=False):
        self._allreduce_and_update(n_r, record)
        if self.on_step is not None:
            self.on_step(self)

    def _allreduce_and_update(self, n_r: int, record=False):
        if self._overlap and n_r == 0:                        # N1: an idle rank still joins every bucket
            for lo, hi, _ in self._buckets:
                self._bucket_call(lo, hi, 0, self.stream)
                self.launches += 1
        elif self.P > 1 and not self._overlap:
            if record:
                a0, a1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                a0.record(self.stream)
            if self.pflat is not None:
                # a6-a9 in one call: weighted ring allreduce with K7 fused (θ' all-gathered, gradient reset)
                pr.weighted_allreduce_sgd(self.comm, self.flat, self.pflat, n_r, self.cfg.lr, self.cfg.wd,
                                          zero_grad=True, stream=self.stream)
            else:
                pr.weighted_allreduce(self.comm, self.flat, n_r, stream=self.stream)
            self.launches += 1
            if record:
                a1.record(self.stream)
                self.ar_events.append((a0, a1))
            if self.pflat is not None:
                return
        if self._overlap and self.pflat is not None:
            return                                            # every bucket's update ran fused with its allreduce
        if self.on_reduced is not None:
            self.on_reduced(self)                             # the reduced gradient ḡ is in self.flat
        if self.pflat is not None:
            if record:
                u0, u1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                u0.record(self.stream)
            pr.sgd_update(self.pflat, self.flat, self.cfg.lr, self.cfg.wd, zero_grad=True, stream=self.stream)
            self.launches += 1
            if record:
                u1.record(self.stream)
                self.sgd_events.append((u0, u1))
        else:
            self.opt.step()
            self.flat.zero_()

    def _compute_time(self, ev) -> float:
        """Σ over the recorded steps of this rank's compute time in seconds (a5).  With N1 the step's CUDA
        events would include the overlapped allreduce (and the wait for peers), so the device stamps taken
        before the spin and at the end of backward are used instead (DESIGN §3 #4: t_s excludes waiting)."""
        if self._overlap:
            k = int(self.stamps[0])
            st = self.stamps[1:1 + k].cpu()
            return float((st[1::2] - st[0::2]).sum()) / 1e9
        return sum(a.elapsed_time(b) for a, b in ev) / 1e3

    # ---- one epoch (Algorithm 1 outer loop) -----------------------------------------------------------
    def _data(self, epoch: int, n_r: int, S: int, record: bool, stream=None):
        """a2 + a3 of `epoch`: the shard (K1) and — epoch-level gather — all S step batches (K2)."""
        st = self.stream if stream is None else stream
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(st)
        pr.shard_indices(self.alloc, self.rank, epoch, self.cfg.seed, self.idx, stream=st)
        self.launches += 1
        xe = ye = None
        if self.cfg.gather == "epoch":
            xe, ye = self.gather(0, S * n_r, record, stream=st, persistent=True)
        e1.record(st)
        self._idx_free = torch.cuda.Event()           # self.idx is free for the next shard once this has run
        self._idx_free.record(st)
        return xe, ye, e0, e1

    def run_epoch(self, record=False, loss_to_host=False):
        cfg = self.cfg
        if cfg.adapt_every > 0:
            return self.run_epoch_segments(record, loss_to_host)
        v = self.alloc.view()
        n_r, S = v["n"][self.rank], v["S"]
        if cfg.graphs:
            self.prepare(n_r)                                 # capture + t1(n_r) outside the timed region
        t_host0 = time.perf_counter()
        pre, self._prefetched = getattr(self, "_prefetched", None), None
        if pre is not None and pre[0] == (self.epoch, n_r):
            xe, ye, e0, e1 = pre[1]                           # enqueued at the end of the previous epoch
            if pre[2] is not None:                            # ... on the side stream: join it here
                self.stream.wait_event(pre[2])
        else:
            xe, ye, e0, e1 = self._data(self.epoch, n_r, S, record)
        ev = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(S)]
        if self._overlap:
            self.stamps[0].zero_()
        losses, host_losses = [], []
        for s in range(S):
            ev[s][0].record(self.stream)
            if n_r > 0:
                if cfg.gather == "epoch":
                    x, y = xe[s * n_r:(s + 1) * n_r], ye[s * n_r:(s + 1) * n_r]
                else:
                    x, y = self.gather(s * n_r, n_r, record)
                loss = self.compute_graphed(x, y, n_r) if cfg.graphs else self.compute(x, y, n_r)
            else:
                loss = torch.zeros((), device=self.dev)
            ev[s][1].record(self.stream)
            self.allreduce_and_update(n_r, record)
            self.gstep += 1
            losses.append(loss)
            if loss_to_host:
                # D2H of the step's result (e2e contract), read one step late: the copy is enqueued behind
                # this step and the host blocks on the PREVIOUS step's copy, so the GPU never idles for it
                self._loss_readback(loss, host_losses)
        if cfg.gather == "epoch" and v["frozen"]:
            # frozen allocation: the next epoch's shard cannot change at the boundary, so its K1 + K2
            # are enqueued now and run while the host synchronises for t_s and runs the controller
            if cfg.host_data:
                # rows come over PCIe (e2e): gather the next epoch on a side stream, beside this epoch's steps
                # (the host is ahead of the GPU here; the side stream only waits for the last use of idx)
                if not hasattr(self, "_side"):
                    self._side = torch.cuda.Stream(self.dev)
                self._side.wait_event(self._idx_free)
                data = self._data(self.epoch + 1, n_r, S, record, stream=self._side)
                done = torch.cuda.Event()
                done.record(self._side)
                self._prefetched = ((self.epoch + 1, n_r), data, done)
            else:
                self._prefetched = ((self.epoch + 1, n_r), self._data(self.epoch + 1, n_r, S, record), None)
        self.host_enqueue_s = time.perf_counter() - t_host0   # diagnostics: host time to enqueue the epoch
        ev[-1][1].synchronize()
        while loss_to_host and getattr(self, "_pending", None):
            self._read_loss(host_losses)
        t_s = e0.elapsed_time(e1) / 1e3 + self._compute_time(ev)                      # seconds (a5)
        self.epoch += 1
        rec = {"t_s": t_s, "loss": float(torch.stack(losses).mean()), "S": S, "n_r": n_r, "w": v["w"]}
        self.history.append(rec)
        self.last_ts = t_s
        return rec

    def _loss_readback(self, loss, host_losses):
        """Enqueue the step's loss D2H copy into a pinned 2-slot ring; block on and read the PREVIOUS step's."""
        if not hasattr(self, "_loss_pinned"):
            self._loss_pinned = torch.empty(2, dtype=torch.float32, pin_memory=True)
            self._loss_ev = [torch.cuda.Event(), torch.cuda.Event()]
            self._pending, self._ls = [], 0
        slot = self._ls % 2
        self._ls += 1
        self._loss_pinned[slot:slot + 1].copy_(loss.detach().float().reshape(1), non_blocking=True)
        self._loss_ev[slot].record(self.stream)
        self._pending.append(slot)
        while len(self._pending) > 1:
            self._read_loss(host_losses)

    def _read_loss(self, host_losses):
        slot = self._pending.pop(0)
        self._loss_ev[slot].synchronize()
        host_losses.append(float(self._loss_pinned[slot]))

    def run_epoch_segments(self, record=False, loss_to_host=False):
        """N3: the epoch as segments of k = adapt_every aggregation steps over the step-interleaved shard.
        Per segment: K1 (pr_shard_steps) + K2 for k·n_r rows, k steps of a4 + a6-a9, then the segment's
        t_s (a5) is exchanged (K6) and the controller (a10) may change w before the next segment.  Step s
        always trains on the same B permuted positions whatever w is (DESIGN §3 #43)."""
        cfg = self.cfg
        if cfg.adapt_lag:
            return self._run_epoch_segments_async(record, loss_to_host)
        S = self.alloc.view()["S"]
        k = cfg.adapt_every
        losses, host_losses, segs = [], [], []
        t_epoch, s0 = 0.0, 0
        while s0 < S:
            v = self.alloc.view()
            n_r, ns = v["n"][self.rank], min(k, S - s0)
            if cfg.graphs:
                self.prepare(n_r)
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record(self.stream)
            pr.shard_steps(self.alloc, self.rank, self.epoch, cfg.seed, s0, ns, self.idx, stream=self.stream)
            self.launches += 1
            xe, ye = self.gather(0, ns * n_r, record)
            e1.record(self.stream)
            ev = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(ns)]
            if self._overlap:
                self.stamps[0].zero_()
            for j in range(ns):
                ev[j][0].record(self.stream)
                if n_r > 0:
                    x, y = xe[j * n_r:(j + 1) * n_r], ye[j * n_r:(j + 1) * n_r]
                    loss = self.compute_graphed(x, y, n_r) if cfg.graphs else self.compute(x, y, n_r)
                else:
                    loss = torch.zeros((), device=self.dev)
                ev[j][1].record(self.stream)
                self.allreduce_and_update(n_r, record)
                self.gstep += 1
                losses.append(loss)
                if loss_to_host:
                    self._loss_readback(loss, host_losses)
            ev[-1][1].synchronize()
            while loss_to_host and getattr(self, "_pending", None):
                self._read_loss(host_losses)
            t_seg = e0.elapsed_time(e1) / 1e3 + self._compute_time(ev)
            t_epoch += t_seg
            changed = False
            if self.comm is not None:
                ts = self.comm.allgather_f64(t_seg, stream=self.stream)
                self.launches += 1
            else:
                ts = [t_seg]
            if cfg.adaptive:
                changed = self.alloc.update(ts)
            segs.append({"s0": s0, "steps": ns, "w": v["w"], "t_s": ts, "changed": changed})
            s0 += ns
        self.epoch += 1
        self.last_ts = t_epoch
        rec = {"t_s": t_epoch, "loss": float(torch.stack(losses).mean()), "S": S,
               "n_r": self.alloc.view()["n"][self.rank], "w": segs[0]["w"], "segments": segs}
        self.history.append(rec)
        return rec

    def _run_epoch_segments_async(self, record=False, loss_to_host=False):
        """N3 with the asynchronous exchange (adapt_lag = 1): per segment, t_s (a5) is summed on the device
        from stamp pairs (data movement, then every step's compute) and all-gathered by the asynchronous K6
        into pinned host memory; the host never waits for the segment it just enqueued — before enqueuing
        segment j + 1 it reads segment j − 1's times (long finished) and runs the controller on them."""
        cfg = self.cfg
        if self._overlap:
            raise ValueError("adapt_lag=1 with overlap is not supported (N1 owns the step stamps)")
        S = self.alloc.view()["S"]
        k = cfg.adapt_every
        if not hasattr(self, "_segring"):
            self._segring = torch.zeros(1 + 2 * (k + 1), dtype=torch.int64, device=self.dev)
            self._d_ts = [torch.zeros((), dtype=torch.float64, device=self.dev) for _ in range(2)]
            self._h_ts = [torch.zeros(self.P, dtype=torch.float64, pin_memory=True) for _ in range(2)]
            self._seg_pending, self._seg_count = [], 0
        losses, host_losses, segs = [], [], []
        t_epoch, s0 = 0.0, 0

        def consume(block_until):
            nonlocal t_epoch
            while self._seg_pending and self._seg_pending[0]["seq"] <= block_until:
                p = self._seg_pending.pop(0)
                p["ev"].synchronize()                       # recorded a segment ago: already complete
                ts = [float(x) for x in self._h_ts[p["slot"]]]
                t_epoch += ts[self.rank]
                changed = self.alloc.update(ts) if cfg.adaptive else False
                p["seg"].update({"t_s": ts, "changed": changed})

        while s0 < S:
            consume(self._seg_count - 2)                    # segment j − 1's times decide segment j + 1
            v = self.alloc.view()
            n_r, ns = v["n"][self.rank], min(k, S - s0)
            if cfg.graphs:
                self.prepare(n_r)
            ring = self._segring
            ring[0].zero_()
            pr.stamp(ring, stream=self.stream)              # a5: data movement of the segment ...
            pr.shard_steps(self.alloc, self.rank, self.epoch, cfg.seed, s0, ns, self.idx, stream=self.stream)
            xe, ye = self.gather(0, ns * n_r, record)
            pr.stamp(ring, stream=self.stream)
            self.launches += 3
            for j in range(ns):
                pr.stamp(ring, stream=self.stream)          # ... then each step's compute (+ K4 spin)
                if n_r > 0:
                    x, y = xe[j * n_r:(j + 1) * n_r], ye[j * n_r:(j + 1) * n_r]
                    loss = self.compute_graphed(x, y, n_r) if cfg.graphs else self.compute(x, y, n_r)
                else:
                    loss = torch.zeros((), device=self.dev)
                pr.stamp(ring, stream=self.stream)
                self.launches += 2
                self.allreduce_and_update(n_r, record)
                self.gstep += 1
                losses.append(loss)
                if loss_to_host:
                    self._loss_readback(loss, host_losses)
            slot = self._seg_count % 2
            pr.stamp_seconds(ring, self._d_ts[slot], stream=self.stream)
            if self.comm is not None:
                self.comm.allgather_f64_async(self._d_ts[slot], self._h_ts[slot], stream=self.stream)
            else:
                self._h_ts[slot][:1].copy_(self._d_ts[slot].reshape(1), non_blocking=True)
            self.launches += 2
            ev = torch.cuda.Event()
            ev.record(self.stream)
            seg = {"s0": s0, "steps": ns, "w": v["w"]}
            segs.append(seg)
            self._seg_pending.append({"seq": self._seg_count, "slot": slot, "ev": ev, "seg": seg})
            self._seg_count += 1
            s0 += ns
        consume(self._seg_count)                            # epoch end: apply what is left (one wait)
        while loss_to_host and getattr(self, "_pending", None):
            self._read_loss(host_losses)
        self.epoch += 1
        self.last_ts = t_epoch
        rec = {"t_s": t_epoch, "loss": float(torch.stack(losses).mean()), "S": S,
               "n_r": self.alloc.view()["n"][self.rank], "w": segs[0]["w"], "segments": segs}
        self.history.append(rec)
        return rec

    def boundary(self):
        """Algorithm 1 steps 1-3: exchange t_s (K6), Eq. 10 + rounding, redistribute."""
        if self.epoch == 0 or self.cfg.adapt_every > 0:
            return False                              # "t_s ... is set to 0" / N3 adapts per segment
        if self.comm is not None:
            ts = self.comm.allgather_f64(self.last_ts, stream=self.stream)
            self.launches += 1
        else:
            ts = [self.last_ts]
        if not self.cfg.adaptive:
            return False
        return self.alloc.update(ts)

    def calibrate(self, steps: int = 3):
        """c0 = seconds per sample of this rank's compute at σ = 1 (for the K4 spin)."""
        v = self.alloc.view()
        n_r = v["n"][self.rank]
        pr.shard_indices(self.alloc, self.rank, 0, self.cfg.seed, self.idx, stream=self.stream)
        x, y = self.gather(0, n_r)
        save, save_sched = self.cfg.slowdown, self.cfg.slowdown_schedule
        self.cfg.slowdown = self.cfg.slowdown_schedule = None
        for _ in range(2):
            self.compute(x, y, n_r)
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record(self.stream)
        for _ in range(steps):
            self.compute(x, y, n_r)
        b.record(self.stream)
        b.synchronize()
        self.flat.zero_()
        self.cfg.slowdown, self.cfg.slowdown_schedule = save, save_sched
        self.c0_ns = a.elapsed_time(b) * 1e6 / (steps * n_r)
        return self.c0_ns

    # ---- checkpoint / resume -------------------------------------------------------------
    # The method's state is the allocation (w, history, frozen, epoch: pr_alloc_save, POD bytes) plus the
    # harness's epoch / step counters and last t_s; the permutation is a pure function of (seed, epoch),
    # so a resumed run draws exactly the shards the uninterrupted run would have.  Model and optimizer
    # state are torch state dicts.  Call between epochs (no prefetched epoch in flight).
    def state_dict(self) -> dict:
        torch.cuda.synchronize(self.dev)
        return {"version": 1, "rank": self.rank, "P": self.P, "alloc": self.alloc.save(),
                "epoch": self.epoch, "gstep": self.gstep, "last_ts": self.last_ts, "c0_ns": self.c0_ns,
                "model": {k: v.detach().clone() for k, v in self.model.state_dict().items()},
                "opt": self.opt.state_dict() if self.opt is not None else None, "history": list(self.history)}

    def load_state_dict(self, sd: dict) -> None:
        if sd.get("version") != 1 or sd["P"] != self.P or sd["rank"] != self.rank:
            raise ValueError("checkpoint is for another job layout")
        self.alloc = pr.Alloc.load(sd["alloc"])
        self.epoch, self.gstep, self.last_ts, self.c0_ns = sd["epoch"], sd["gstep"], sd["last_ts"], sd["c0_ns"]
        with torch.no_grad():
            self.model.load_state_dict(sd["model"])
        if self.opt is not None and sd["opt"] is not None:
            self.opt.load_state_dict(sd["opt"])
        self.history = list(sd["history"])
        self._prefetched = None
