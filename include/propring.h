/*
 * propring — proportional task allocation + sample-count-weighted ring allreduce for B200 (sm_100a).
 *
 * C ABI of libpropring.so: the data-parallel hot path of arXiv 2111.08272, "Task allocation for
 * decentralized training in heterogeneous environment" (Chao, Liao, Gao).
 * Citation keys: P:n = PAPER.md line n (paper source), S:n = SPEC.md line n, DESIGN §3 #k = the k-th
 * reading of a silent/ambiguous passage listed in DESIGN.md §3.
 *
 * Conventions (every call):
 *   - returns int: PR_OK (0) on success, a negative PR_ERR_* code otherwise; nothing aborts on user
 *     error and no C++ exception crosses the ABI;
 *   - output parameters are written only on success;
 *   - "d_" pointers are CUDA device pointers (or host pointers mapped into the device address space),
 *     "h_"/plain pointers are host memory; all memory passed in stays caller-owned unless stated;
 *   - `stream` is a cudaStream_t (passed as void* so this header needs no CUDA include); device work
 *     is enqueued asynchronously and stream-ordered;
 *   - pr_alloc handles are pure host state, not thread-safe per handle; pr_comm calls are serialised
 *     per communicator and are collective (same order on every rank), like NCCL.
 */
#ifndef PROPRING_H
#define PROPRING_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define PR_VERSION 10100       /* 1.1.0 */
#define PR_MAX_RANKS 64

/* ---- error codes (SPEC error names in parentheses) ------------------------------------------- */
#define PR_OK                      0
#define PR_ERR_INVALID            -1   /* bad argument, null handle, bad version/size               */
#define PR_ERR_INFEASIBLE_FLOOR   -2   /* C < P·floor (InfeasibleFloor)                       */
#define PR_ERR_DATASET_TOO_SMALL  -3   /* N < B = g·C (DatasetTooSmall)                       */
#define PR_ERR_ZERO_TIMING        -4   /* a step time <= 0, NaN or Inf (ZeroTiming)            */
#define PR_ERR_CUDA               -5   /* a CUDA runtime call failed                                  */
#define PR_ERR_ALIGN              -6   /* pointer or row size not 16-byte aligned                    */
#define PR_ERR_NO_P2P             -7   /* peer access between two ranks' GPUs is not possible        */
#define PR_ERR_LENGTH_MISMATCH    -8   /* ranks called the allreduce with different count/dtype (LengthMismatch) */
#define PR_ERR_ZERO_SAMPLES       -9   /* Σ n_local = 0 (ZeroSampleCount)                     */
#define PR_ERR_PEER_TIMEOUT      -10   /* watchdog expired waiting for a peer (TransportClosed) */
#define PR_ERR_CAPACITY          -11   /* output capacity too small                                  */
#define PR_ERR_INTERNAL          -12   /* invariant violated inside the library (a bug)              */
#define PR_ERR_UNSUPPORTED       -13   /* the platform lacks a capability (NVSwitch multicast for NVLS) */

const char *pr_strerror(int code);
int pr_version(void);

/* =================================================================================================
 * 1. Allocation (host control plane) — §8(a) rows a1 and a10
 * ================================================================================================= */

typedef struct pr_alloc pr_alloc;

/* Read-only snapshot of an allocation.  Arrays are indexed by rank (first P entries valid). */
typedef struct {
    int64_t N;        /* dataset rows D                                                      */
    int32_t P;        /* workers                                                                      */
    int32_t frozen;   /* 1 once the stop rule fired                                           */
    int64_t C;        /* Σ w_i, units per aggregation, constant (Eq. 4)                    */
    int64_t g;        /* samples per unit: the paper's "minibatch" (DESIGN §3 #1)        */
    int64_t floor;    /* minimum units per worker                                             */
    int64_t B;        /* global samples per aggregation = g·C ("minibatch*(Σw_i)")        */
    int64_t S;        /* aggregations per epoch = floor(N / B) (DESIGN §3 #10)                        */
    int64_t epoch;    /* number of successful pr_alloc_update calls                                   */
    int64_t hist_len; /* number of allocation vectors in the history (initial one included)           */
    int64_t w[PR_MAX_RANKS];   /* units per aggregation w_i^(k)                        */
    int64_t n[PR_MAX_RANKS];   /* samples per aggregation n_i = g·w_i                                 */
    int64_t len[PR_MAX_RANKS]; /* shard sizes D_i = D·w_i/Σw, exact-integer Hamilton (DESIGN §3 #9) */
    int64_t off[PR_MAX_RANKS]; /* shard offsets: exclusive prefix sum of len in rank order             */
} pr_alloc_view;

/* Step-time model of the controller.  PROPORTIONAL is the paper's: t_i ∝ w_i (Eq. 6-8), the
 * update is Eq. 10 + Hamilton.  AFFINE is an opt-in extension (DESIGN.md §3 #49) for steps with a fixed
 * per-step cost, where Eq. 10's fixed point (all t_i equal) is not the balanced optimum: each rank's
 * t_i(w) = a_i + b_i·w is fitted by least squares over its last fit_window (w, t) observations (fewer than
 * two distinct w: a_i = 0, b_i = t_i/w_i; a fit with b <= 0 or a < 0: the same proportional fallback), and
 * w' = the integer min-max allocation: min over Σw = C, w >= floor of max_i a_i + b_i·w_i (greedy, ties to
 * the lowest rank).  While no rank has two distinct w (the first update from a uniform start), the update
 * is Eq. 10 exactly.  Requires floor >= 1. */
#define PR_ALLOC_MODEL_PROPORTIONAL 0
#define PR_ALLOC_MODEL_AFFINE       1

/* Stop-rule / smoothing policy of the self-adaptive controller. */
typedef struct {
    int32_t window;        /* stable when the last `window` vectors differ by <= tol (default 2)     */
    int32_t never_freeze;  /* 1: keep re-allocating every epoch (default 0)                          */
    int64_t tol;           /* per-component tolerance in units (default 1)                           */
    double  ema_alpha;     /* t_eff = a·t + (1−a)·t_eff_prev; 1.0 = raw last-epoch times (default)   */
    int32_t model;         /* PR_ALLOC_MODEL_* (default PROPORTIONAL)                               */
    int32_t fit_window;    /* AFFINE: observations per rank in the fit, 2..64 (default 8)             */
} pr_alloc_policy;

/* Static allocation (§3.1; a1).  w = Hamilton(C·r_i/Σr, floor) with ties to the lowest rank
 * (identity when the ratios are integers summing to C); n_i = g·w_i; len = Hamilton(N·w_i/C) in exact
 * integer arithmetic; off = prefix sum; S = floor(N/(g·C)).
 *   ratios: host double[P], each finite and > 0.  C = 0 means C = Σratios (ratios must be integers).
 *   Errors: PR_ERR_INVALID (P<1 or P>PR_MAX_RANKS, N<1, g<1, floor<0, bad ratio, C<0),
 *           PR_ERR_INFEASIBLE_FLOOR, PR_ERR_DATASET_TOO_SMALL.
 *   Deterministic and replicated: every rank calls it with identical arguments and gets identical state.
 *   Ownership: *out is library-owned; free with pr_alloc_destroy. */
int pr_alloc_init(pr_alloc **out, int64_t N, int32_t P, const double *ratios, int64_t C, int64_t g,
                  int64_t floor);
int pr_alloc_set_policy(pr_alloc *a, const pr_alloc_policy *policy);

/* Self-adaptive update (Algorithm 1 steps 1-3; Eq. 10; rounding P:181; a10).
 *   step_times: host double[P], rank i's gradient-computing time t_s^i of the last epoch in seconds
 *   (per-epoch sum of CUDA-event step times; DESIGN §3 #4-#5).  Any t <= 0 / NaN / Inf ->
 *   PR_ERR_ZERO_TIMING with the state unchanged (the first epoch's "t_s is set to 0").
 *   v_i = w_i / t_i;  S_v = Σ v left to right;  q_i = (C·v_i)/S_v;  w' = Hamilton(q, C, floor);
 *   history += w'; epoch += 1; then the stop rule may freeze the allocation.
 *   If already frozen: no-op, *changed = 0, PR_OK.  changed (may be NULL): 1 if w' != w. */
int pr_alloc_update(pr_alloc *a, const double *step_times, int32_t *changed);
int pr_alloc_query(const pr_alloc *a, pr_alloc_view *out);
/* k-th allocation vector of the history (0 = initial); w_out: host int64[P]. */
int pr_alloc_history(const pr_alloc *a, int64_t k, int64_t *w_out);
/* Checkpoint (POD bytes: w, history, frozen flag, policy, EMA state, the t of every update).  *size receives the byte count;
 * with buf == NULL only the size is returned.  PR_ERR_CAPACITY if cap is too small. */
int pr_alloc_save(const pr_alloc *a, void *buf, size_t cap, size_t *size);
int pr_alloc_load(pr_alloc **out, const void *buf, size_t size);
void pr_alloc_destroy(pr_alloc *a);

/* =================================================================================================
 * 2. Sharder (K1) and gather (K2) — §8(a) rows a2 and a3
 * ================================================================================================= */

/* Per-epoch permutation + proportional split ("assigned a corresponding proportion", Algorithm 1
 * step 3 "Redistribute the subdataset"; shuffle is build-defined, DESIGN §3 #8):
 *   d_out[t] = π_{seed,epoch}(off_rank + t), t < len_rank, where π is a 4-round Feistel network with
 *   Philox4x32-10 round functions on a 2^b domain, cycle-walked into [0, N).
 *   d_out: caller-owned device int64[cap], cap >= len_rank.  Async on stream.
 *   Errors: PR_ERR_INVALID (rank out of range), PR_ERR_CAPACITY, PR_ERR_CUDA. */
int pr_shard_indices(const pr_alloc *a, int32_t rank, int64_t epoch, uint64_t seed, int64_t *d_out,
                     int64_t cap, void *stream);
/* Step-interleaved shard for intra-epoch re-allocation ("Load ... will change
 * slightly" P:98; DESIGN §3 #43).  Aggregation step s of the epoch owns permuted positions
 * [s·B, (s+1)·B), B = g·C; rank r takes the n_r = g·w_r positions starting at o_r = g·Σ_{j<r} w_j:
 *   d_out[(s − step0)·n_r + t] = π_{seed,epoch}(s·B + o_r + t),  step0 <= s < step0 + nsteps, t < n_r.
 * Because B is fixed (Σw = C, Eq. 4), the step's sample set does not depend on w, so the allocation may
 * change between any two steps and the ranks' rows stay disjoint.  Requires step0 + nsteps <= S.
 * d_out: caller-owned device int64[cap], cap >= nsteps·n_r.  Async on stream.
 * Errors: PR_ERR_INVALID (rank or step range), PR_ERR_CAPACITY, PR_ERR_CUDA. */
int pr_shard_steps(const pr_alloc *a, int32_t rank, int64_t epoch, uint64_t seed, int64_t step0,
                   int64_t nsteps, int64_t *d_out, int64_t cap, void *stream);
/* The permutation itself on positions [begin, begin+count): d_out[t] = π_{seed,epoch}(begin + t).
 * Requires 1 <= N <= 2^62 and begin + count <= N. */
int pr_permute(int64_t N, uint64_t seed, int64_t epoch, int64_t begin, int64_t count, int64_t *d_out,
               void *stream);

#define PR_GATHER_COPY              0  /* bit copy of each row                                       */
#define PR_GATHER_U8_TO_F32_AFFINE  1  /* (float(x) − shift_c)·scale_c, two fp32 roundings, no FMA   */
#define PR_GATHER_U8_TO_BF16_AFFINE 2  /* the same value rounded to bfloat16 (RNE)                   */
#define PR_GATHER_MAX_CHANNELS 16
#define PR_GATHER_IMPL_AUTO 0   /* device source, >= 1 MiB: channels-last -> BULK; CHW >= 8 MiB -> TMA; else LSU */
#define PR_GATHER_IMPL_LSU  1   /* warp per 2 KiB segment, ld.global.nc 16-byte vectors                 */
#define PR_GATHER_IMPL_TMA  2   /* cp.async.bulk rows / segments into a 4-stage smem ring (mbarrier)    */
#define PR_GATHER_IMPL_BULK 3   /* channels-last output only: coalesced loads -> smem tile in output
                                   order -> one cp.async.bulk store per 4096 output pixels (device
                                   sources; a host source runs the LSU kernel); PR_ERR_INVALID for CHW */
#define PR_GATHER_LAYOUT_CHW 0  /* output row in the input's channel-major order                        */
#define PR_GATHER_LAYOUT_HWC 1  /* channels-last output: element (c, p) at p·channels + c; needs
                                   channels <= 4 and plane % 16 == 0 (both kernels)                     */

typedef struct {
    int32_t op;                              /* PR_GATHER_*                                           */
    int32_t channels;                        /* affine ops: number of channels (<= 16)               */
    int64_t plane;                           /* affine ops: elements per channel (H·W of a CHW row)   */
    float scale[PR_GATHER_MAX_CHANNELS];     /* per-channel multiplier                                */
    float shift[PR_GATHER_MAX_CHANNELS];     /* per-channel subtrahend                                */
    int32_t impl;                            /* PR_GATHER_IMPL_* (results are identical)              */
    int32_t layout;                          /* PR_GATHER_LAYOUT_* of the output row (affine ops)     */
} pr_gather_op;

/* Step-batch gather (Algorithm 1 step 4, "Proportionally draw samples from the sub-data set"):
 *   for t < n:  dst[t, :] = op(src[idx[t], :]);  if d_lab_src: d_lab_dst[t] = d_lab_src[idx[t]].
 *   d_src: [n_src, row_bytes] bytes (device memory, or mapped pinned host memory for the e2e path);
 *   d_idx: int64[n] in [0, n_src) (out-of-range is a contract violation);
 *   d_dst: COPY -> [n, row_bytes] bytes; U8_TO_F32 -> [n, row_bytes] float; U8_TO_BF16 -> bf16.
 *   op == NULL means COPY.  row_bytes, d_src and d_dst must be 16-byte aligned (PR_ERR_ALIGN);
 *   for affine ops channels·plane must equal row_bytes (PR_ERR_INVALID).  n = 0 is a no-op. */
int pr_gather_rows(const void *d_src, int64_t n_src, int64_t row_bytes, const int64_t *d_idx, int64_t n,
                   void *d_dst, const pr_gather_op *op, const int64_t *d_lab_src, int64_t *d_lab_dst,
                   void *stream);

/* Emulated heterogeneity (K4): a 32-thread kernel that busy-waits on %globaltimer for `ns`
 * nanoseconds on `stream` (the per-rank calibrated slowdown of the north star). ns <= 0: no launch. */
int pr_spin(int64_t ns, void *stream);

/* t_s capture (row a5) where CUDA events cannot bracket the compute — inside a captured
 * graph whose tail also joins an overlapped allreduce (N1): a 1-thread kernel appends the %globaltimer
 * value (ns) to a caller-owned device ring, stream-ordered:
 *   i = d_ring[0]++ (atomic);  d_ring[1 + i mod cap] = now.
 * The caller zeroes d_ring[0] and reads the ring after the stream completes.  cap >= 1.
 * Errors: PR_ERR_INVALID, PR_ERR_CUDA. */
int pr_stamp(int64_t *d_ring, int64_t cap, void *stream);

/* t_s of a segment from pr_stamp pairs, on the device (row a5 without a host synchronisation, for the
 * asynchronous controller exchange below): *d_out = Σ_{i < k/2} (ring[2 + 2i] − ring[1 + 2i]) · 1e-9 s,
 * k = min(ring[0], cap) stamps recorded as (start, end) pairs.  d_ring: device int64[1 + cap];
 * d_out: device double.  Stream-ordered.  Errors: PR_ERR_INVALID, PR_ERR_CUDA. */
int pr_stamp_seconds(const int64_t *d_ring, int64_t cap, double *d_out, void *stream);

/* SGD update, §8(a) row a9: Eq. 1 with weight decay, applied to the reduced
 * gradient, fused with the gradient reset for the next aggregation:
 *   θ[i] ← fma(−lr, fma(wd, θ[i], g[i]), θ[i]);   if zero_grad: g[i] ← 0
 * in fp32 (lr, wd rounded to fp32), each fma rounded once (RN).  d_theta, d_grad: device fp32 [n],
 * 16-byte aligned, caller-owned; async on `stream`.  Errors: PR_ERR_INVALID (n < 0, null pointer),
 * PR_ERR_ALIGN, PR_ERR_CUDA. */
int pr_sgd_update(float *d_theta, float *d_grad, int64_t n, double lr, double wd, int32_t zero_grad, void *stream);

/* =================================================================================================
 * 3. Weighted ring allreduce (K3) — §8(a) rows a6, a7, a8
 * ================================================================================================= */

typedef struct pr_comm pr_comm;

#define PR_DTYPE_F32  0
#define PR_DTYPE_BF16 1

#define PR_COMM_FLAG_FORCE_STAGED 1   /* all-gather through staging even when buffers are registered */
#define PR_COMM_FLAG_BULK_STORE   4   /* ring data path: results pushed with TMA bulk stores (one thread,
                                         * whole tiles) instead of 16-byte stores from every consumer lane */
#define PR_COMM_FLAG_L2_PREFETCH  8   /* ring data path: each slice's own-gradient range is prefetched into
                                         * L2 (cp.async.bulk.prefetch.L2) before the slice's flag waits */
#define PR_COMM_FLAG_PULL_TMA    16   /* pull two-shot: the P source tiles staged in shared memory by TMA bulk
                                        loads (4 stages, up to 192 KiB in flight per channel) instead of
                                        register-queued loads — for peer reads over NVLink; same bits */
#define PR_COMM_FLAG_SYS_SCOPE    2   /* system-scope release/acquire even when every rank shares one GPU
                                         (by default .gpu scope is used exactly when that is the case) */

/* Fields marked (topology) may be 0 = chosen at init from where the ranks are: all on one GPU (local
 * groups, co-located processes) -> the HBM-bound optimum; on different GPUs -> more channels with larger
 * tiles and slots, since each rank then has only its own channels' SMs. */
typedef struct {
    int32_t channels;     /* ring channels = CTAs per rank (topology: 128/P, <= 64, one GPU / 32 across) */
    int32_t slots;        /* staging slots per channel, >= 2 (default 8)                    */
    int32_t threads;      /* consumer threads per CTA, <= 512 (default 512)                                         */
    int32_t flags;        /* PR_COMM_FLAG_* (default 0)                                                */
    int64_t slot_bytes;   /* bytes per staging slot, multiple of 256 (topology: 256 KiB / 1 MiB)      */
    int64_t watchdog_ns;  /* spin-wait deadline per call (default 10 s); <= 0 disables               */
    int32_t stages;       /* TMA smem pipeline depth per CTA, 2..16, stages·2·tile <= 224 KiB (0: 7)    */
    int32_t tile_bytes;   /* bytes per input per pipeline stage, multiple of 16, <= 32768 (0: 16 KiB) */
    int32_t algo;         /* PR_ALGO_* (default PR_ALGO_RING)                                         */
    int32_t ts_slots;     /* two-shot staging slots per (channel, source), >= 2 (default 2)          */
    int64_t ts_slot_bytes;/* two-shot slice bytes, multiple of 256 (default 262144)                  */
    int64_t ts_max_bytes; /* PR_ALGO_AUTO: two-shot for buffers up to this many bytes (default 4 MiB)  */
    int64_t ll_max_bytes; /* largest buffer the LL ring handles (PR_ALGO_LL; PR_ALGO_AUTO picks it up to
                             here); sizes the LL regions of the window, <= 64 MiB (default 256 KiB)  */
    int64_t os_max_bytes; /* largest buffer the one-shot LL path handles (PR_ALGO_ONESHOT; PR_ALGO_AUTO
                             picks it up to here), <= 16 MiB (default 64 KiB)                         */
    int64_t min_slice_bytes; /* ring: 0 = slot-sized slices (default); > 0 (multiple of 16) = cut each
                             channel's share of a chunk into up to slots/2 slices of >= this many bytes,
                             so every phase keeps several slices in flight (an A/B knob for NVLink)  */
} pr_comm_config;

/* Allreduce algorithm.  Both compute the same bits (the two-shot reducer adds the contributions in the
 * ring's order with the ring's per-hop rounding).  Two-shot: each rank pushes its raw
 * slice of chunk d to rank d (one hop), rank d reduces and stores the result into every peer's
 * registered buffer (second hop) — 2 synchronisation phases instead of 2(P−1); it needs every rank's
 * buffer registered (else PR_ERR_INVALID is latched on all ranks). */
#define PR_ALGO_RING     0
#define PR_ALGO_TWO_SHOT 1
#define PR_ALGO_AUTO     2   /* one-shot up to os_max_bytes, LL ring up to ll_max_bytes, the PULL two-shot
                                 (registered buffers) up to ts_max_bytes (× 2 for P >= 4, × 4 for P >= 8),
                                 ring above */
/* LL ring: the ring's schedule, order and rounding (same bits) with a low-latency line protocol — every
 * 16-byte line pushed to the next rank carries 8 payload bytes and the call's sequence number in both
 * 64-bit halves, so the receiver polls the data itself (no fence / flag / credit round trip per hop).
 * Half the bandwidth of the ring, a fraction of its per-hop latency: for buffers <= ll_max_bytes
 * (larger buffers given PR_ALGO_LL take the ring).  Works with unregistered buffers. */
#define PR_ALGO_LL       3
/* One-shot LL: one hop — every rank pushes its raw buffer as LL lines to every peer and reduces all P
 * contributions itself, per element in the ring's order for that element's chunk with the ring's
 * per-hop rounding (same bits).  (P−1)·2·Z bytes sent per rank: for buffers <= os_max_bytes (larger
 * buffers given PR_ALGO_ONESHOT take the ring).  Works with unregistered buffers. */
#define PR_ALGO_ONESHOT  4
#define PR_ALGO_NVLS     5   /* NVSwitch in-switch reduction: fp32 buffers inside the NVLS
                              * region (pr_comm_nvls_alloc); each rank weights its buffer in place, then
                              * reduces its chunk with multimem.ld_reduce and multicasts it with multimem.st.
                              * The switch's summation order is unspecified: within tolerance of the fp64
                              * mean, NOT the ring's bits.  Buffers outside the region take the ring. */
/* Pull two-shot (round 2): after the handshake rank r LOADS its chunk r from every rank's registered
 * buffer (instead of each rank pushing it into r's staging), reduces it in the ring's order with the
 * ring's rounding (same bits) and stores the result into every rank's buffer.  Stores per rank fall from
 * (2P−1)/P·Z to Z — the SM store path is what bounds a channel.  Needs every rank's buffer registered
 * (else PR_ERR_INVALID is latched on all ranks).  PR_ALGO_AUTO takes it instead of the push two-shot
 * (registered buffers up to ts_max_bytes); above that AUTO keeps the ring (the paper's algorithm), since the
 * pull's peer loads are unmeasured over NVLink.  pr_weighted_allreduce_sgd fuses the update into it too. */
#define PR_ALGO_TWO_SHOT_PULL 6

/* Byte allgather supplied by the caller (e.g. over a torch process group): every rank passes `len`
 * bytes in `send` and receives the P·len bytes of all ranks, rank-ordered, in `recv`.  Returns 0 on
 * success. */
typedef int (*pr_exchange_fn)(void *ctx, const void *send, size_t len, void *recv);

/* One process per GPU (collective over P processes).  Allocates this rank's flag page + staging
 * (cudaMalloc), exports it with CUDA IPC, exchanges the handles through `fn`, and maps every peer's
 * memory (NVLink 5 / NVSwitch P2P).  cfg may be NULL (defaults).  device = CUDA ordinal of this rank.
 * Errors: PR_ERR_INVALID, PR_ERR_NO_P2P, PR_ERR_CUDA. */
int pr_comm_init(pr_comm **out, int32_t rank, int32_t P, int32_t device, pr_exchange_fn fn, void *ctx,
                 const pr_comm_config *cfg);
/* Single-process group of P ranks on ONE device (test and emulation mode: the P ranks' memories are
 * all local, the ring protocol and kernel are the same).  out: host pr_comm*[P]. */
int pr_comm_init_local(pr_comm **out, int32_t P, int32_t device, const pr_comm_config *cfg);

/* Collective: register [d_buf, d_buf+bytes) so that the all-gather phase stores the reduced chunks
 * straight into every peer's buffer (no staging copy).  d_buf must be the base of a cudaMalloc
 * allocation (CUDA IPC requirement) — pr_comm_alloc returns such memory.  Buffers passed to
 * pr_weighted_allreduce inside a registered region take the direct path when every rank's buffer is
 * registered, else the staged path.  Registered memory stays caller-owned. */
int pr_comm_register(pr_comm *c, void *d_buf, size_t bytes);
/* Collective: allocate `bytes` of device memory (zeroed) on this rank's device and register it.
 * Library-owned; released by pr_comm_destroy. */
int pr_comm_alloc(pr_comm *c, size_t bytes, void **d_ptr);

/* Sample-count-weighted ring allreduce, in place (Eq. 1; ring of P:63 / S:195):
 *     buf <- Σ_r (n_r / Σn) · buf_r
 * where buf_r is rank r's LOCAL MEAN gradient over its n_r = n_local samples (DESIGN §3 #11).
 * One kernel: handshake (seq, count, dtype, n_r) with every peer = the barrier of P:54/P:63 (its
 * duration is t_w), Σn and s_r = fp32(n_r/Σn) (fp64 division); P−1 reduce-scatter hops where each
 * rank's contribution is scaled as it enters the ring (hop 0: y = s_r·g_r; later hops y = fma(s_r, g_r,
 * recv), fp32 math, round-to-nearest-even to the dtype); P−1 all-gather hops (bit copies).
 *   count: elements; dt: PR_DTYPE_F32 / PR_DTYPE_BF16; d_buf 16-byte aligned (PR_ERR_ALIGN);
 *   n_local >= 0: a rank with n_local = 0 contributes exactly nothing (never multiplied).
 *   P = 1: identity (no launch) unless n_local = 0 (PR_ERR_ZERO_SAMPLES).
 * Every rank must call with the same count and dtype in the same order; a mismatch is detected in the
 * handshake and latched as PR_ERR_LENGTH_MISMATCH on every rank with buf untouched; Σn = 0 latches
 * PR_ERR_ZERO_SAMPLES; a peer that never arrives latches PR_ERR_PEER_TIMEOUT after watchdog_ns.
 * Latched device errors are returned by pr_comm_status() once the stream has completed, and by the
 * next call.  Async; stream-ordered; the caller keeps buf alive until the stream completes. */
int pr_weighted_allreduce(pr_comm *c, void *d_buf, int64_t count, int32_t dt, int64_t n_local,
                          void *stream);
/* Local-group form: one cooperative launch runs all P ranks of a pr_comm_init_local group (rank r uses
 * d_bufs[r], n_local[r]); comms: host pr_comm*[P] in rank order.  (pr_weighted_allreduce on a single
 * rank of a local group launches that rank alone: the caller must issue all P ranks' calls on distinct
 * streams so that they are co-resident — used to exercise the mismatch / timeout paths.) */
int pr_weighted_allreduce_local(pr_comm *const *comms, void *const *d_bufs, int64_t count, int32_t dt,
                                const int64_t *n_local, void *stream);

/* Rows a6-a9 in one call (K7 fused into K3): the weighted allreduce of the fp32 local-mean gradient
 * d_grad (as pr_weighted_allreduce) followed by pr_sgd_update(d_theta, ḡ, lr, wd, zero_grad) — with the TMA
 * ring and registered buffers, ONE kernel: the owner of each reduced chunk applies the update to its θ
 * chunk and the all-gather carries θ' (into every rank's d_theta) instead of ḡ; the gradient is reset as
 * the reduce-scatter consumes it.  With the pull two-shot (PR_ALGO_TWO_SHOT_PULL, or AUTO at its sizes)
 * likewise one kernel: the owner of chunk r stores θ' into every rank's θ, and each rank resets its own
 * gradient after the final wait (when every peer has read it).  d_theta must hold identical values on every rank (replicated
 * parameters) and lie at the same byte offset from d_grad inside the same registered region on every rank
 * (e.g. one pr_comm_alloc of 2·count floats: [grad | theta]); else — or when the configured algorithm for
 * this size is neither the ring nor the pull two-shot — the call is composed of the two operations (same
 * bits).  After the call
 * d_theta holds θ' on every rank; d_grad holds 0 if zero_grad, else unspecified (the reduced ḡ is not
 * materialised in the fused path).  Errors: as pr_weighted_allreduce (+ PR_ERR_INVALID latched when the
 * ranks' θ layouts differ). */
int pr_weighted_allreduce_sgd(pr_comm *c, float *d_grad, float *d_theta, int64_t count, int64_t n_local, double lr,
                              double wd, int32_t zero_grad, void *stream);
/* Local-group form of pr_weighted_allreduce_sgd (all P ranks in one launch). */
int pr_weighted_allreduce_sgd_local(pr_comm *const *comms, float *const *d_grads, float *const *d_thetas,
                                    int64_t count, const int64_t *n_local, double lr, double wd, int32_t zero_grad,
                                    void *stream);

/* Algorithm 1 step 1: every rank contributes `local` and receives all P values in rank
 * order into host out[P].  Synchronous (waits for `stream`). */
int pr_comm_allgather_f64(pr_comm *c, double local, double *out, void *stream);

/* The same exchange without a host synchronisation (K6 asynchronous): the local value is read from
 * device memory when the kernel runs (d_local: device double, e.g. written by pr_stamp_seconds) and the
 * P values land in h_out[P] — PINNED host memory (cudaHostAlloc / torch pin_memory), written by the
 * device — stream-ordered.  The caller records an event behind the call and reads h_out after it; the
 * controller can then act one segment later without stalling the stream.  Errors: PR_ERR_INVALID
 * (local group, null pointer, h_out not device-accessible), PR_ERR_CUDA; peer timeouts latch in
 * pr_comm_status. */
int pr_comm_allgather_f64_async(pr_comm *c, const double *d_local, double *h_out, void *stream);

/* NVLS region (collective, every rank with the same bytes): allocates `bytes` (rounded up
 * to the multicast granularity) on every rank's device, binds all of them to ONE NVSwitch multicast
 * object and maps both aliases; *d_ptr = this rank's unicast address (zeroed).  A weighted allreduce with
 * config.algo = PR_ALGO_NVLS on an fp32 buffer inside it reduces in the switch.  At most one region per
 * communicator; freed by pr_comm_destroy.  The multicast handle travels as a fabric handle when the
 * platform has one, else as a file descriptor duplicated with pidfd_getfd.
 * Errors (on every rank together): PR_ERR_UNSUPPORTED (no multicast: a single-GPU or non-NVSwitch
 * system, a container without the fabric), PR_ERR_INVALID (local group, P < 2, a region exists). */
int pr_comm_nvls_alloc(pr_comm *c, size_t bytes, void **d_ptr);

/* Latched device error of the last completed call (PR_OK if none). Non-blocking host read. */
int pr_comm_status(pr_comm *c);
/* %globaltimer stamps (ns) of the last completed call on this rank: [0] kernel entry, [1] handshake
 * complete (barrier left: t_w = [1]−[0]), [2] kernel exit (t_c = [2]−[1]).  out: host int64[3]. */
int pr_comm_timestamps(pr_comm *c, int64_t *out);
/* Rank and size of a communicator. */
int pr_comm_rank(const pr_comm *c, int32_t *rank, int32_t *size);
/* Collective teardown (frees staging, flags, pr_comm_alloc memory, closes IPC mappings). */
void pr_comm_destroy(pr_comm *c);

/* =================================================================================================
 * 4. Test hooks (parity pins against library routines; no hot-path role)
 * ================================================================================================= */

/* d_out[4·i + j] = word j of Philox4x32-10(ctr_i, key) computed by the library's device function,
 * ctr_i = (d_ctr[4i..4i+3]) ; with use_curand != 0 the same through cuRAND's curand_Philox4x32_10
 * (the library routine pin of SURVEY §8(c) O3 (ii)).  n counters. */
int pr_test_philox(const uint32_t *d_ctr, int64_t n, uint64_t key, int32_t use_curand, uint32_t *d_out,
                   void *stream);

#ifdef __cplusplus
}
#endif

#endif /* PROPRING_H */
