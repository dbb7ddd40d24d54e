// K3 — sample-count-weighted ring allreduce over NVLink 5 / NVSwitch peer memory (+ its communicator).
//
// Paper: Ring AllReduce (§2.2): n workers on a ring, the gradient cut into n parts; a reduce-scatter
// phase ("the kth worker ... send the kth data to the next worker, and at the same time receive the k−1th
// data from the previous worker") then an all-gather phase ("each worker sends the integrated part to the
// next worker"), preceded by the barrier that synchronises all workers — the wait the
// method shrinks (t_w).  Eq. 1: the update is the mean over N = Σ_i minibatch·w_i
// samples, so with buf_r = rank r's local mean over n_r samples the reduction is buf = Σ_r (n_r/Σn)·buf_r.
// Readings: #11 local-mean convention, #13 ring schedule, #14 chunk boundaries, #15 order
// and rounding, #32 Σn exchanged in the handshake, #33 n_r = 0 contributes nothing, #36 the n_r/Σn scale
// is applied where a contribution enters the ring (hop 0: y = s·g; later: y = fma(s, g, recv)).
//
// Design (B200): ONE kernel per call, one CTA per ring "channel".  Each channel owns a contiguous slice
// of every chunk and runs an independent ring with its own flags and K staging slots:
//   * all synchronisation is local polling (ld.acquire.sys) + remote signalling (st.release.sys), i.e.
//     every NVLink transaction is a store: data is PUSHED into the next rank's staging slot (reduce-scatter)
//     or straight into the next rank's registered gradient buffer (all-gather, no staging copy);
//   * monotone 64-bit counters (ready / credit / ag_ready) — never reset, so back-to-back calls and
//     CUDA-graph replays need no host involvement; handshake entries are double-buffered by seq parity;
//   * every spin has a %globaltimer deadline (watchdog) that latches PR_ERR_PEER_TIMEOUT.
// Data path per slice (ring_kernel): a producer warp polls the flags and TMA-loads the rank's own tile and
// the received tile into a shared-memory ring; 16 consumer warps do the fp32 math (one instantiation per
// hop arithmetic) and push 16-byte vectors to the peer; a signal warp publishes each slice's flag off the
// data path.  The handshake is written in fence-free LL lines (seq | payload per 64-bit element).
// Variants with the same bits: ring_ll_kernel (LL lines per hop, small buffers),
// oneshot_ll_kernel (one hop, tiny buffers), twoshot_kernel (2 phases), and ring_kernel<float, true>
// (K7's SGD fused into the last reduce-scatter hop; the all-gather carries θ').  Channel count, tile and
// slot sizes default from the topology (resolve_config): CTAs per rank are the bound across GPUs.
#include <cuda.h>            // driver-API types only: entry points are fetched with cudaGetDriverEntryPoint
#include <cuda_bf16.h>
#include <sys/syscall.h>
#include <unistd.h>

#include <algorithm>
#include <cstring>
#include <mutex>
#include <new>
#include <string>
#include <vector>

#include "common.h"

#define PR_MAX_REGS 8

namespace {


// ---- window layout (one cudaMalloc per rank, CUDA-IPC exported) ------------------------------------
struct ChanFlags {          // written by peers, polled locally
    unsigned long long rs_ready;   uint64_t p0[15];   // by prev: slices it has stored into my staging slots
    unsigned long long rs_credit;  uint64_t p1[15];   // by next: my slot-slices it has consumed (slot reuse)
    unsigned long long ag_ready;   uint64_t p2[15];   // by prev: direct all-gather slices written into my buf
};
struct HsEntry {            // handshake entry, written by rank q into every peer's page (slot [parity][q]):
    uint64_t line[16];      // five LL lines: (seq32 | count, n, dtype/reg_id, offset, θ-delta halves), see
};                          // handshake(); lines 5-7 unused (padding to 128 B)
struct ChanState {          // local only: cumulative counters carried across calls
    unsigned long long seq;         // handshake sequence number
    unsigned long long slot_base;   // staging-slot slices produced (= consumed: uniform slicing)
    unsigned long long ag_base;     // direct all-gather slices sent (= received)
    unsigned long long ts_base;     // two-shot slices processed (every rank processes the same number)
    uint64_t pad[12];
};
struct TsFlags {            // two-shot flags, one counter per peer (index = the peer that writes it)
    unsigned long long ready[PR_MAX_RANKS];    // by q: slices of its raw contribution stored in my staging
    unsigned long long credit[PR_MAX_RANKS];   // by q: slices of MY contribution it has consumed
    unsigned long long ag[PR_MAX_RANKS];       // by q: slices of its reduced chunk stored into my buffer
};
struct AgEntry {
    unsigned long long seq;
    double v;
};
struct NvFlags {            // NVLS: by q, the call sequence whose phase A (scale) / B (reduce + multicast) it finished
    unsigned long long a[PR_MAX_RANKS];
    unsigned long long b[PR_MAX_RANKS];
};
static_assert(sizeof(ChanFlags) == 384, "flags");
static_assert(sizeof(HsEntry) == 128, "hs");
static_assert(sizeof(ChanState) == 128, "state");

struct DevTable {
    int32_t rank, P, channels, slots;
    int32_t stages, tile_bytes;     // TMA pipeline: depth, bytes per input per stage
    int32_t sysscope, l2pf;         // 1: some peer is another GPU (use .sys release/acquire); 1: L2 prefetch of g
    int64_t slot_bytes;
    int64_t watchdog_ns;
    uint64_t off_flags, off_hs, off_state, off_ag, off_staging, window_bytes;
    uint64_t off_ts_flags, off_ts_staging;
    int32_t ts_slots, pad1;
    int64_t ts_slot_bytes;
    uint64_t off_ll;                // LL ring: [channels][2P−2 phases][ll_region_bytes]
    int64_t ll_region_bytes;        // 16-byte lines, 8 payload bytes each, for one channel's share of a chunk
    int64_t min_slice_bytes;        // > 0: cut each chunk share into up to slots/2 slices of >= this (ring)
    uint64_t off_os;                // one-shot LL: [channels][P sources][os_region_bytes]
    int64_t os_region_bytes;        // LL lines for one channel's share of the whole buffer
    uint64_t off_nv;                // NVLS barrier counters: [channels] NvFlags
    uint8_t* nv_uc;                 // NVLS region: this rank's unicast mapping (null: none) ...
    uint8_t* nv_mc;                 // ... and the multicast mapping of the same offsets (all ranks' memory)
    int64_t nv_bytes;
    volatile int* status;           // host-mapped
    volatile long long* stamps;     // host-mapped [3]
    uint8_t* win[PR_MAX_RANKS];
    uint8_t* reg[PR_MAX_REGS][PR_MAX_RANKS];
};

struct RankCall {
    const DevTable* tab;
    void* buf;
    int64_t n_local;
    int32_t reg_id;
    int32_t pad;
    int64_t reg_off;
    int64_t th_delta;   // fused update (K7 in K3): θ = buf + th_delta bytes, identical on every rank
};

struct LaunchArgs {
    int64_t count;
    int32_t dtype;
    int32_t nranks;     // entries in calls[] (gridDim.y)
    int32_t fuse;       // 1: the all-gather carries θ' = SGD(θ, ḡ) computed by the chunk owner (K7 in K3)
    int32_t zero;       // fused: reset the gradient buffer as it is consumed
    float nlr, wd;      // fused: −lr, weight decay (fp32, as pr_sgd_update)
    int32_t algo;       // PR_ALGO_* this rank launched: part of the handshake, so ranks that picked
    int32_t pad;        // different kernels latch PR_ERR_LENGTH_MISMATCH instead of waiting forever
    RankCall calls[PR_MAX_RANKS];
};

uint64_t align_up(uint64_t x, uint64_t a) { return (x + a - 1) / a * a; }

void layout(DevTable& t) {
    t.off_flags = 0;
    uint64_t o = (uint64_t)t.channels * sizeof(ChanFlags);
    t.off_hs = o = align_up(o, 256);
    o += (uint64_t)t.channels * 2 * t.P * sizeof(HsEntry);
    t.off_state = o = align_up(o, 256);
    o += (uint64_t)t.channels * sizeof(ChanState);
    t.off_ag = o = align_up(o, 256);
    o += 2ull * t.P * sizeof(AgEntry);
    t.off_staging = o = align_up(o, 4096);
    o += (uint64_t)t.channels * t.slots * (uint64_t)t.slot_bytes;
    t.off_ts_flags = o = align_up(o, 4096);
    o += (uint64_t)t.channels * sizeof(TsFlags);
    t.off_ts_staging = o = align_up(o, 4096);
    o += (uint64_t)t.channels * t.P * t.ts_slots * (uint64_t)t.ts_slot_bytes;
    t.off_ll = o = align_up(o, 4096);
    o += (uint64_t)t.channels * (uint64_t)(t.P > 1 ? 2 * t.P - 2 : 0) * (uint64_t)t.ll_region_bytes;
    t.off_os = o = align_up(o, 4096);
    o += (uint64_t)t.channels * (uint64_t)t.P * (uint64_t)t.os_region_bytes;
    t.off_nv = o = align_up(o, 4096);
    o += (uint64_t)t.channels * sizeof(NvFlags);
    t.window_bytes = align_up(o, 4096);
}

// ---- device helpers --------------------------------------------------------------------------------
__device__ __forceinline__ unsigned long long gtimer() {
    unsigned long long t;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
    return t;
}
// Memory scope of the protocol: .sys when a peer window lives on another GPU (NVLink peer memory), .gpu
// when every rank of the group shares this device (local groups, co-located processes) — the cheapest
// scope that is still correct.
__device__ __forceinline__ unsigned long long ld_acquire(const unsigned long long* p, bool sys) {
    unsigned long long v;
    if (sys) asm volatile("ld.acquire.sys.global.u64 %0, [%1];" : "=l"(v) : "l"(p) : "memory");
    else asm volatile("ld.acquire.gpu.global.u64 %0, [%1];" : "=l"(v) : "l"(p) : "memory");
    return v;
}
__device__ __forceinline__ void st_release(unsigned long long* p, unsigned long long v, bool sys) {
    if (sys) asm volatile("st.release.sys.global.u64 [%0], %1;" ::"l"(p), "l"(v) : "memory");
    else asm volatile("st.release.gpu.global.u64 [%0], %1;" ::"l"(p), "l"(v) : "memory");
}
__device__ __forceinline__ void st_relaxed_u64(unsigned long long* p, unsigned long long v, bool sys) {
    if (sys) asm volatile("st.relaxed.sys.global.u64 [%0], %1;" ::"l"(p), "l"(v) : "memory");
    else asm volatile("st.relaxed.gpu.global.u64 [%0], %1;" ::"l"(p), "l"(v) : "memory");
}
__device__ __forceinline__ long long ld_relaxed_s64(const void* p, bool sys) {
    long long v;
    if (sys) asm volatile("ld.relaxed.sys.global.s64 %0, [%1];" : "=l"(v) : "l"(p) : "memory");
    else asm volatile("ld.relaxed.gpu.global.s64 %0, [%1];" : "=l"(v) : "l"(p) : "memory");
    return v;
}
__device__ __forceinline__ void st_relaxed_s64(void* p, long long v, bool sys) {
    if (sys) asm volatile("st.relaxed.sys.global.s64 [%0], %1;" ::"l"(p), "l"(v) : "memory");
    else asm volatile("st.relaxed.gpu.global.s64 [%0], %1;" ::"l"(p), "l"(v) : "memory");
}
__device__ __forceinline__ void st_v4(void* p, uint4 v) {
    asm volatile("st.global.v4.u32 [%0], {%1,%2,%3,%4};" ::"l"(p), "r"(v.x), "r"(v.y), "r"(v.z), "r"(v.w)
                 : "memory");
}

__device__ __forceinline__ ChanFlags* flags_of(uint8_t* w, const DevTable* t, int ch) {
    return reinterpret_cast<ChanFlags*>(w + t->off_flags) + ch;
}
__device__ __forceinline__ HsEntry* hs_of(uint8_t* w, const DevTable* t, int ch, int par, int q) {
    return reinterpret_cast<HsEntry*>(w + t->off_hs) + ((size_t)ch * 2 + par) * t->P + q;
}
__device__ __forceinline__ ChanState* state_of(uint8_t* w, const DevTable* t, int ch) {
    return reinterpret_cast<ChanState*>(w + t->off_state) + ch;
}
__device__ __forceinline__ uint8_t* slot_of(uint8_t* w, const DevTable* t, int ch, unsigned long long J) {
    return w + t->off_staging + ((size_t)ch * t->slots + (size_t)(J % (unsigned long long)t->slots)) * t->slot_bytes;
}

enum Mode { M_SCALE = 0, M_FMA = 1, M_COPY = 2, M_ZERO = 3 };

// Element traits: fp32 math on 16-byte vectors of the storage dtype.
template <typename T> struct Vec;
template <> struct Vec<float> {
    static constexpr int V = 4;
    __device__ static float ld(const float* p) { float v; asm volatile("ld.global.cg.f32 %0, [%1];" : "=f"(v) : "l"(p)); return v; }
    __device__ static void st(float* p, float v) { *p = v; }
    __device__ static float to_f(float v) { return v; }
    __device__ static float from_f(float v) { return v; }
    __device__ static uint4 op(int mode, float s, uint4 g, uint4 in) {
        uint4 y;
        const uint32_t gi[4] = {g.x, g.y, g.z, g.w}, ii[4] = {in.x, in.y, in.z, in.w};
        uint32_t o[4];
#pragma unroll
        for (int j = 0; j < 4; ++j) {
            const float gv = __uint_as_float(gi[j]), iv = __uint_as_float(ii[j]);
            float r;
            if (mode == M_SCALE) r = __fmul_rn(s, gv);
            else if (mode == M_FMA) r = __fmaf_rn(s, gv, iv);
            else if (mode == M_COPY) r = iv;
            else r = 0.0f;
            o[j] = __float_as_uint(r);
        }
        y.x = o[0]; y.y = o[1]; y.z = o[2]; y.w = o[3];
        return y;
    }
};
template <> struct Vec<__nv_bfloat16> {
    static constexpr int V = 8;
    __device__ static __nv_bfloat16 ld(const __nv_bfloat16* p) {
        unsigned short v;
        asm volatile("ld.global.cg.u16 %0, [%1];" : "=h"(v) : "l"(p));
        return __ushort_as_bfloat16(v);
    }
    __device__ static void st(__nv_bfloat16* p, __nv_bfloat16 v) { *p = v; }
    __device__ static float to_f(__nv_bfloat16 v) { return __bfloat162float(v); }
    __device__ static __nv_bfloat16 from_f(float v) { return __float2bfloat16_rn(v); }
    __device__ static float lo(uint32_t w) { return __uint_as_float(w << 16); }
    __device__ static float hi(uint32_t w) { return __uint_as_float(w & 0xffff0000u); }
    __device__ static uint32_t pack(float a, float b) {
        return (uint32_t)__bfloat16_as_ushort(__float2bfloat16_rn(a)) |
               ((uint32_t)__bfloat16_as_ushort(__float2bfloat16_rn(b)) << 16);
    }
    __device__ static float one(int mode, float s, float gv, float iv) {
        if (mode == M_SCALE) return __fmul_rn(s, gv);
        if (mode == M_FMA) return __fmaf_rn(s, gv, iv);
        if (mode == M_COPY) return iv;
        return 0.0f;
    }
    __device__ static uint4 op(int mode, float s, uint4 g, uint4 in) {
        if (mode == M_COPY) return in;
        const uint32_t gi[4] = {g.x, g.y, g.z, g.w}, ii[4] = {in.x, in.y, in.z, in.w};
        uint32_t o[4];
#pragma unroll
        for (int j = 0; j < 4; ++j)
            o[j] = pack(one(mode, s, lo(gi[j]), lo(ii[j])), one(mode, s, hi(gi[j]), hi(ii[j])));
        return make_uint4(o[0], o[1], o[2], o[3]);
    }
};

// ---- TMA (bulk copy) + mbarrier helpers ------------------------------------------------------------
constexpr int kMaxStages = 16;      // smem pipeline depth limit (tiles in flight per CTA)

__device__ __forceinline__ uint32_t smem_u32(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }
__device__ __forceinline__ void mbar_init(uint64_t* b, uint32_t count) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(b)), "r"(count) : "memory");
}
__device__ __forceinline__ void mbar_arrive_expect_tx(uint64_t* b, uint32_t tx) {
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(b)), "r"(tx) : "memory");
}
__device__ __forceinline__ void mbar_arrive(uint64_t* b) {
    asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_u32(b)) : "memory");
}
__device__ __forceinline__ void mbar_wait(uint64_t* b, uint32_t parity) {
    asm volatile(
        "{\n\t.reg .pred P1;\n"
        "LAB_WAIT:\n\t"
        "mbarrier.try_wait.parity.shared::cta.b64 P1, [%0], %1;\n\t"
        "@P1 bra DONE;\n\t"
        "bra LAB_WAIT;\n"
        "DONE:\n\t}" ::"r"(smem_u32(b)),
        "r"(parity)
        : "memory");
}
// TMA bulk copy global -> shared, completion counted in bytes on `bar` (SASS: UBLKCP)
__device__ __forceinline__ void tma_load(void* dst, const void* src, uint32_t bytes, uint64_t* bar) {
    asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
                     smem_u32(dst)),
                 "l"(src), "r"(bytes), "r"(smem_u32(bar))
                 : "memory");
}
// generic-proxy writes (peer stores observed through an acquire) -> visible to the async proxy (TMA)
// cp.async.bulk.prefetch.L2: bring [p, p+bytes) into L2 ahead of the TMA loads (16-byte aligned and sized)
__device__ __forceinline__ void prefetch_l2(const void* p, uint32_t bytes) {
    asm volatile("cp.async.bulk.prefetch.L2.global [%0], %1;" ::"l"(p), "r"(bytes) : "memory");
}
__device__ __forceinline__ void fence_proxy_async_global() { asm volatile("fence.proxy.async.global;" ::: "memory"); }
// this thread's st.shared writes -> visible to a later bulk store's (async proxy) reads of shared memory
__device__ __forceinline__ void fence_proxy_async_smem() { asm volatile("fence.proxy.async.shared::cta;" ::: "memory"); }
// TMA bulk store shared -> global (local or NVLink peer memory), bulk-group completion (SASS: UBLKCP)
__device__ __forceinline__ void tma_store(void* dst, const void* src, uint32_t bytes) {
    asm volatile("cp.async.bulk.global.shared::cta.bulk_group [%0], [%1], %2;" ::"l"(dst), "r"(smem_u32(src)), "r"(bytes)
                 : "memory");
}
__device__ __forceinline__ void bulk_commit() { asm volatile("cp.async.bulk.commit_group;" ::: "memory"); }
// all but the newest N bulk groups have finished READING shared memory (the source tiles may be reused)
template <int N> __device__ __forceinline__ void bulk_wait_read() {
    asm volatile("cp.async.bulk.wait_group.read %0;" ::"n"(N) : "memory");
}
// all but the newest N bulk groups are COMPLETE (their global writes performed)
template <int N> __device__ __forceinline__ void bulk_wait() { asm volatile("cp.async.bulk.wait_group %0;" ::"n"(N) : "memory"); }

struct Shared {
    int err;
    int direct;
    long long sumn;
    void* next_buf;
    unsigned long long fin_slot, fin_ag;   // producer's final counters, for the epilogue
    uint64_t full[kMaxStages];             // producer -> consumers: tile landed in smem (TMA tx bytes)
    uint64_t stored[kMaxStages];           // consumers -> signal warp: tile's stores issued
    uint64_t empty[kMaxStages];            // consumers + signal warp -> producer: stage reusable
    int tile_ok[kMaxStages];
};

__device__ __forceinline__ void latch(const DevTable* t, int code) {
    if (*t->status == 0) *t->status = code;
}

// Spin until *p >= target; false on watchdog expiry.
__device__ __forceinline__ bool wait_ge(const unsigned long long* p, unsigned long long target,
                                        unsigned long long deadline, bool sys) {
    while (ld_acquire(p, sys) < target) {
        if (gtimer() > deadline) return false;
    }
    return true;
}

enum Kind { K_FIRST = 0, K_MID = 1, K_LAST = 2, K_AGMID = 3, K_AGLAST = 4 };

// The schedule: rounds of G slices; each round walks the 2P−1 phases (see the comment in ring_kernel).
template <typename F>
__device__ __forceinline__ void for_each_step(int P, int r, int64_t nsl, int64_t G, F&& f) {
    for (int64_t i0 = 0; i0 < nsl; i0 += G) {
        const int64_t gend = min(i0 + G, nsl);
        for (int h = 0; h < 2 * P - 1; ++h) {
            int kind, c;
            if (h == 0) { kind = K_FIRST; c = r; }
            else if (h <= P - 2) { kind = K_MID; c = (r - h + P) % P; }
            else if (h == P - 1) { kind = K_LAST; c = (r + 1) % P; }
            else if (h <= 2 * P - 3) { kind = K_AGMID; c = (r + 1 - (h - (P - 1)) + P) % P; }
            else { kind = K_AGLAST; c = (r + 2) % P; }
            for (int64_t i = i0; i < gend; ++i) f(kind, c, i);
        }
    }
}

// Handshake = the barrier; its duration is t_w.  Publishes (seq, count, dtype, n_r,
// registration) into every rank's page and waits for all P entries of this call (entries are
// double-buffered by seq parity).  Returns Σn and whether every rank's buffer is registered; fills ns[q]
// (n of rank q) and bufs[q] (rank q's buffer mapped in this process, if registered) when given.
//
// Entries use the LL line format (see ring_ll_kernel): the 64-byte entry is four 16-byte lines of two
// 64-bit elements, each (seq32 << 32 | 32 payload bits).  A 64-bit aligned element is single-copy
// atomic, so a reader that sees the call's sequence number in all eight elements has the whole entry —
// no release fence before a flag store (a MEMBAR.SYS at system scope, the dominant cost of a flag
// round trip).  Ordering against the previous call's data is given by stream order: a rank publishes
// its entry for call k only after its kernel for call k−1 has completed.
struct HsOut {
    int err;
    int direct;
    long long sumn;
};
__device__ __forceinline__ void st_line64(void* p, unsigned long long a, unsigned long long b, bool sys) {
    if (sys) asm volatile("st.relaxed.sys.global.v2.b64 [%0], {%1,%2};" ::"l"(p), "l"(a), "l"(b) : "memory");
    else asm volatile("st.relaxed.gpu.global.v2.b64 [%0], {%1,%2};" ::"l"(p), "l"(a), "l"(b) : "memory");
}
__device__ __forceinline__ void ld_line64(const void* p, unsigned long long& a, unsigned long long& b, bool sys) {
    if (sys) asm volatile("ld.relaxed.sys.global.v2.b64 {%0,%1}, [%2];" : "=l"(a), "=l"(b) : "l"(p) : "memory");
    else asm volatile("ld.relaxed.gpu.global.v2.b64 {%0,%1}, [%2];" : "=l"(a), "=l"(b) : "l"(p) : "memory");
}
__device__ __forceinline__ unsigned long long tag(uint32_t flag, uint32_t w) { return ((unsigned long long)flag << 32) | w; }
__device__ __forceinline__ void hs_publish(HsEntry* e, uint32_t flag, long long count, long long n, uint32_t dtype,
                                           int32_t reg_id, long long offset, long long th_delta, bool sys) {
    unsigned long long* L = reinterpret_cast<unsigned long long*>(e);
    st_line64(L + 8, tag(flag, (uint32_t)th_delta), tag(flag, (uint32_t)((unsigned long long)th_delta >> 32)), sys);
    st_line64(L + 0, tag(flag, (uint32_t)count), tag(flag, (uint32_t)((unsigned long long)count >> 32)), sys);
    st_line64(L + 2, tag(flag, (uint32_t)n), tag(flag, (uint32_t)((unsigned long long)n >> 32)), sys);
    st_line64(L + 4, tag(flag, dtype), tag(flag, (uint32_t)reg_id), sys);
    st_line64(L + 6, tag(flag, (uint32_t)offset), tag(flag, (uint32_t)((unsigned long long)offset >> 32)), sys);
}
// Poll one entry until all eight elements carry `flag`; false on watchdog expiry.
__device__ __forceinline__ bool hs_read(const HsEntry* e, uint32_t flag, unsigned long long deadline, bool sys,
                                        long long& count, long long& n, uint32_t& dtype, int32_t& reg_id,
                                        long long& offset, long long& th_delta) {
    const unsigned long long* L = reinterpret_cast<const unsigned long long*>(e);
    unsigned long long w[10];
    for (;;) {
        ld_line64(L + 0, w[0], w[1], sys);
        ld_line64(L + 2, w[2], w[3], sys);
        ld_line64(L + 4, w[4], w[5], sys);
        ld_line64(L + 6, w[6], w[7], sys);
        ld_line64(L + 8, w[8], w[9], sys);
        bool ok = true;
#pragma unroll
        for (int k = 0; k < 10; ++k) ok = ok && (uint32_t)(w[k] >> 32) == flag;
        if (ok) break;
        if (gtimer() > deadline) return false;
    }
    count = (long long)(((w[1] & 0xffffffffull) << 32) | (w[0] & 0xffffffffull));
    n = (long long)(((w[3] & 0xffffffffull) << 32) | (w[2] & 0xffffffffull));
    dtype = (uint32_t)w[4];
    reg_id = (int32_t)(uint32_t)w[5];
    offset = (long long)(((w[7] & 0xffffffffull) << 32) | (w[6] & 0xffffffffull));
    th_delta = (long long)(((w[9] & 0xffffffffull) << 32) | (w[8] & 0xffffffffull));
    return true;
}
// The call's kind as published in the handshake: dtype | fused update << 8 | algorithm << 16.
__device__ __forceinline__ uint32_t call_kind(const LaunchArgs& A) {
    return (uint32_t)A.dtype | ((uint32_t)A.fuse << 8) | ((uint32_t)A.algo << 16);
}

// Executed by ALL 32 lanes of warp 0: lane q publishes into rank q's page and polls entry q of this
// page (ranks q, q+32, …), so the P peers are contacted in parallel; Σn, "all registered" and the error
// code are combined with warp shuffles (DESIGN.md §3 #37).  The result is valid in every lane.
__device__ HsOut handshake(const LaunchArgs& A, const RankCall& rc, const DevTable* tab, ChanState* st, int ch, bool sys,
                           unsigned long long deadline, long long* ns, uint8_t** bufs) {
    const int r = tab->rank, P = tab->P;
    const int lane = threadIdx.x & 31;
    uint8_t* my = tab->win[r];
    const unsigned long long seq = st->seq + 1;
    const int par = (int)(seq & 1ull);
    const uint32_t flag = (uint32_t)(seq & 0xffffffffull);
    for (int q = lane; q < P; q += 32)
        hs_publish(hs_of(tab->win[q], tab, ch, par, r), flag, A.count, rc.n_local, call_kind(A), rc.reg_id,
                   rc.reg_off, rc.th_delta, sys);
    int err = 0, direct = 1;
    long long sumn = 0;
    for (int q = lane; q < P; q += 32) {
        long long cnt, n, off, thd;
        uint32_t dt;
        int32_t rid;
        if (!hs_read(hs_of(my, tab, ch, par, q), flag, deadline, sys, cnt, n, dt, rid, off, thd)) {
            err = PR_ERR_PEER_TIMEOUT;
            break;
        }
        // the dtype word carries the fused-update flag and the algorithm: every rank makes the same kind of call
        if (cnt != A.count || dt != call_kind(A)) err = PR_ERR_LENGTH_MISMATCH;
        if (A.fuse && thd != rc.th_delta) err = err ? err : PR_ERR_INVALID;   // θ-layout differs across ranks
        sumn += n;
        if (rid < 0) direct = 0;
        if (ns) ns[q] = n;
        if (bufs) bufs[q] = rid >= 0 ? (uint8_t*)((uintptr_t)tab->reg[rid][q] + (uintptr_t)off) : nullptr;
    }
#pragma unroll
    for (int o = 16; o; o >>= 1) {                    // warp-shuffle reductions
        sumn += __shfl_xor_sync(0xffffffffu, sumn, o);
        err = min(err, __shfl_xor_sync(0xffffffffu, err, o));   // error codes are negative
    }
    direct = __all_sync(0xffffffffu, direct);
    HsOut out{err, direct, sumn};
    if (!out.err && out.sumn <= 0) out.err = PR_ERR_ZERO_SAMPLES;
    __syncwarp();
    if (lane == 0) st->seq = seq;
    return out;
}

// K7's arithmetic on a 16-byte vector (fp32 only: the fused update requires fp32 buffers):
// θ' = fma(−η, fma(λ, θ, ḡ), θ), exactly as pr_sgd_update.
template <typename T> __device__ __forceinline__ uint4 sgd_v4(uint4 t, uint4 g, float nlr, float wd);
template <> __device__ __forceinline__ uint4 sgd_v4<float>(uint4 t, uint4 g, float nlr, float wd) {
    const uint32_t ti[4] = {t.x, t.y, t.z, t.w}, gi[4] = {g.x, g.y, g.z, g.w};
    uint32_t o[4];
#pragma unroll
    for (int j = 0; j < 4; ++j) {
        const float tv = __uint_as_float(ti[j]);
        o[j] = __float_as_uint(__fmaf_rn(nlr, __fmaf_rn(wd, tv, __uint_as_float(gi[j])), tv));
    }
    return make_uint4(o[0], o[1], o[2], o[3]);
}
template <> __device__ __forceinline__ uint4 sgd_v4<__nv_bfloat16>(uint4, uint4 g, float, float) { return g; }

// The consumers' per-tile inner loop with the hop's arithmetic fixed at compile time: a runtime `mode`
// inside the loop compiled to a branch + reconvergence per element (≈ 50 instructions per 16-byte vector
// in the ncu source view of a CTA-bound run); with MODE constant it is ≈ 15 (2 LDS, 4 FFMA, 1-3 STG).
// out1/out2/zg/thp are already offset to the tile's first element; out2, zg, thp may be null (uniform).
// BULK: y goes back into the received tile in shared memory (`is`, same thread, same slot: read then
// write) and the signal thread pushes the whole tile with one TMA bulk store per destination; a COPY
// hop then has no per-vector work at all (the loaded tile IS the output).
template <typename T, int MODE, bool FUSE, bool BULK>
__device__ __forceinline__ void tile_vectors(const uint4* __restrict__ gs, uint4* is, int nv, int cid,
                                             int nc, float s, T* out1, T* out2, T* zg, const T* thp, float nlr,
                                             float wd) {
    constexpr int V = Vec<T>::V;
    if constexpr (BULK && MODE == M_COPY && !FUSE) {
        return;
    } else {
    if (BULK && MODE == M_COPY && !thp && !zg) return;
    for (int v = cid; v < nv; v += nc) {
        const uint4 a = (MODE == M_SCALE || MODE == M_FMA) ? gs[v] : make_uint4(0, 0, 0, 0);
        const uint4 b = (MODE == M_FMA || MODE == M_COPY) ? is[v] : make_uint4(0, 0, 0, 0);
        uint4 y = Vec<T>::op(MODE, s, a, b);
        if (FUSE && thp) y = sgd_v4<T>(*reinterpret_cast<const uint4*>(thp + (int64_t)v * V), y, nlr, wd);
        if (FUSE && zg) st_v4(zg + (int64_t)v * V, make_uint4(0, 0, 0, 0));
        if (BULK) {
            is[v] = y;
        } else {
            st_v4(out1 + (int64_t)v * V, y);
            if (out2) st_v4(out2 + (int64_t)v * V, y);
        }
    }
    if (BULK) fence_proxy_async_smem();                   // the bulk store reads these smem writes
    }
}

template <typename T>
struct SliceArgs {
    T* out1;                     // destination of the slice (next rank's slot, or a buffer)
    T* out2;                     // second destination or null
    T* zg;                       // fused: own gradient to reset, or null
    const T* thp;                // fused: own θ of the reduced chunk, or null
    const T* gsrc;               // own gradient of the slice (ragged tail only)
    const T* isrc;               // received data of the slice (ragged tail only)
    int64_t len, te, nt;         // slice elements, tile elements, tiles
    float s, nlr, wd;
};

// Consumers' loop over one slice's tiles with the hop's arithmetic fixed (MODE).  Per tile: wait for the
// TMA bytes, compute + store the full 16-byte vectors (tile_vectors), the ragged tail (only at the end of
// the buffer), then one arrive per warp on `stored`.  Pointers advance by a tile; no per-tile branching on
// the mode, no 64-bit multiplies (these dominated a CTA-bound run once the element loop was tight).
template <typename T, int MODE, bool FUSE, bool BULK>
__device__ __forceinline__ void consume_slice(Shared& sh, uint8_t* smem, int kTileBytes, int kStages, int& stg, uint32_t& ph,
                                              int cid, int nc, int lane, const SliceArgs<T>& a) {
    constexpr int V = Vec<T>::V;
    T* o1 = a.out1;
    T* o2 = a.out2;
    T* zp = a.zg;
    const T* tp = a.thp;
    int64_t left = a.len;
    for (int64_t t = 0; t < a.nt; ++t) {
        const int ne = (int)(left < a.te ? left : a.te);
        mbar_wait(&sh.full[stg], ph);
        const bool ok = sh.tile_ok[stg] != 0;
        const int nv = (ne * (int)sizeof(T)) / 16;
        const uint4* gs = reinterpret_cast<const uint4*>(smem + (size_t)stg * 2 * kTileBytes);
        uint4* is = reinterpret_cast<uint4*>(smem + (size_t)stg * 2 * kTileBytes + kTileBytes);
        if (ok) {
            tile_vectors<T, MODE, FUSE, BULK>(gs, is, nv, cid, nc, a.s, o1, o2, zp, tp, a.nlr, a.wd);
            if (nv * V < ne) {                                      // ragged tail: end of the buffer only
                const int64_t e0 = a.len - left;
                for (int e = nv * V + cid; e < ne; e += nc) {
                    const float gv = (MODE == M_SCALE || MODE == M_FMA) ? Vec<T>::to_f(Vec<T>::ld(a.gsrc + e0 + e)) : 0.0f;
                    const float iv = (MODE == M_FMA || MODE == M_COPY) ? Vec<T>::to_f(Vec<T>::ld(a.isrc + e0 + e)) : 0.0f;
                    float rr;
                    if (MODE == M_SCALE) rr = __fmul_rn(a.s, gv);
                    else if (MODE == M_FMA) rr = __fmaf_rn(a.s, gv, iv);
                    else rr = (MODE == M_COPY) ? iv : 0.0f;
                    T y = (MODE == M_COPY) ? Vec<T>::ld(a.isrc + e0 + e) : Vec<T>::from_f(rr);
                    if (FUSE && tp) {
                        const float tv = Vec<T>::to_f(tp[e]);
                        y = Vec<T>::from_f(__fmaf_rn(a.nlr, __fmaf_rn(a.wd, tv, Vec<T>::to_f(y)), tv));
                    }
                    if (FUSE && zp) Vec<T>::st(zp + e, Vec<T>::from_f(0.0f));
                    Vec<T>::st(o1 + e, y);
                    if (o2) Vec<T>::st(o2 + e, y);
                }
            }
        }
        __syncwarp();
        if (lane == 0) mbar_arrive(&sh.stored[stg]);   // release.cta: this warp's smem reads and stores precede
        if (++stg == kStages) {
            stg = 0;
            ph ^= 1u;
        }
        left -= ne;
        o1 += ne;
        if (o2) o2 += ne;
        if (FUSE && zp) zp += ne;
        if (FUSE && tp) tp += ne;
    }
}

// FUSE (compile time): the K7-fused variant; the plain ring is compiled without any of its code.
// BULK (compile time, PR_COMM_FLAG_BULK_STORE): consumers write each tile's result back into shared memory
// and the signal thread pushes it with TMA bulk stores (cp.async.bulk.global.shared::cta) instead of 16-byte
// STGs from every consumer lane; a slice's ready flag is released once its bulk groups have completed.
template <typename T, bool FUSE, bool BULK>
__global__ void __launch_bounds__(576, 1) ring_kernel(const __grid_constant__ LaunchArgs A) {
    extern __shared__ __align__(128) uint8_t smem[];   // [stages][2][tile_bytes]: g tile, recv tile
    __shared__ Shared sh;
    const RankCall& rc = A.calls[blockIdx.y];
    const DevTable* tab = rc.tab;
    const int ch = blockIdx.x;
    const int r = tab->rank, P = tab->P;
    const int next = (r + 1) % P, prev = (r + P - 1) % P;
    uint8_t* my = tab->win[r];
    ChanState* st = state_of(my, tab, ch);
    ChanFlags* myf = flags_of(my, tab, ch);
    ChanFlags* nxf = flags_of(tab->win[next], tab, ch);
    ChanFlags* pvf = flags_of(tab->win[prev], tab, ch);
    const bool t0 = threadIdx.x == 0;
    const bool sys = tab->sysscope != 0;
    const int nc = blockDim.x - 64;                 // consumer threads (warps 2..): warp 0 producer, warp 1 signal
    const int kStages = tab->stages;
    const int kTileBytes = tab->tile_bytes;
    unsigned long long deadline = ~0ull;

    // ---- handshake = the barrier; its duration is t_w ---------------------------------
    if (threadIdx.x < 32) {                           // warp 0 (the producer warp) runs the handshake
        const unsigned long long start = gtimer();
        if (tab->watchdog_ns > 0) deadline = start + (unsigned long long)tab->watchdog_ns;
        if (t0) {
            if (ch == 0) tab->stamps[0] = (long long)start;
            for (int k = 0; k < kStages; ++k) {
                mbar_init(&sh.full[k], 1);
                mbar_init(&sh.stored[k], (uint32_t)(nc / 32));
                mbar_init(&sh.empty[k], 1);                 // the signal warp, after `stored`
            }
            asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
        }
        __shared__ uint8_t* s_bufs[PR_MAX_RANKS];
        const HsOut hs = handshake(A, rc, tab, st, ch, sys, deadline, nullptr, s_bufs);
        if (t0) {
            sh.err = hs.err ? hs.err : ((A.fuse && !hs.direct) ? PR_ERR_INVALID : 0);   // fused: direct AG only
            sh.direct = hs.direct;
            sh.sumn = hs.sumn;
            sh.next_buf = hs.direct ? (void*)s_bufs[next] : nullptr;
            if (ch == 0) tab->stamps[1] = (long long)gtimer();
        }
    }
    __syncthreads();
    if (sh.err) {
        if (t0) latch(tab, sh.err);
        return;
    }

    // ---- geometry (DESIGN.md §3 #14) ----------------------------------------------------------------
    constexpr int V = Vec<T>::V;
    const int64_t TE = kTileBytes / (int64_t)sizeof(T);          // tile elements
    const int64_t count = A.count;
    const int64_t per = (count + P - 1) / P;
    const int64_t cs = (per + V - 1) / V * V;                      // chunk elements
    const int64_t subp = (cs + tab->channels - 1) / tab->channels;
    const int64_t sub = (subp + V - 1) / V * V;                   // this channel's share of a chunk
    // slice elements: one staging slot; with min_slice_bytes > 0 the chunk share is cut into up to
    // G = slots/2 slices (each >= min_slice_bytes) so that a phase keeps G slices in flight — per phase
    // max(G·τ, τ + L) instead of τ + L when the share fits one slot (a latency-bound regime on NVLink;
    // co-located it did not pay).  A pure function of (count, P, config): same on every rank.
    int64_t sl = tab->slot_bytes / (int64_t)sizeof(T);
    if (tab->min_slice_bytes > 0) {
        const int64_t G0 = (int64_t)(tab->slots / 2);
        const int64_t want = ((sub + G0 - 1) / G0 + V - 1) / V * V;
        sl = min(sl, max(want, (int64_t)(tab->min_slice_bytes / (int64_t)sizeof(T))));
    }
    const int64_t te = min(TE, sl);
    const int64_t nsl = sub > 0 ? (sub + sl - 1) / sl : 0;
    const float s = (float)((double)rc.n_local / (double)sh.sumn);  // n_r/Σn: fp64 division, fp32 weight
    const bool act = rc.n_local > 0;
    const bool direct = sh.direct != 0;
    T* buf = reinterpret_cast<T*>(rc.buf);
    T* nbuf = reinterpret_cast<T*>(sh.next_buf);
    // fused update (K7 in K3): the owner of a reduced chunk applies SGD to its θ and the all-gather carries
    // θ' (own θ and the next rank's θ = buf + th_delta bytes, the same layout on every rank)
    constexpr bool fuse = FUSE;
    T* th = fuse ? reinterpret_cast<T*>(reinterpret_cast<uint8_t*>(rc.buf) + rc.th_delta) : buf;
    T* nth = (fuse && nbuf) ? reinterpret_cast<T*>(reinterpret_cast<uint8_t*>(sh.next_buf) + rc.th_delta) : nbuf;
    const unsigned long long K = (unsigned long long)tab->slots;
    // Rounds of G = K/2 slices per chunk walk all 2P−1 phases:
    //   phase 0             RS hop 0     chunk r            y = s·g                 -> next's slot
    //   phase h, 1..P−2     RS hop h     chunk (r−h) mod P  y = fma(s, g, recv)     -> next's slot
    //   phase P−1           last RS hop  chunk (r+1) mod P  y = fma(s, g, recv)     -> own buf + next (AG hop 0)
    //   phase P−1+k, k≥1    AG hop k     chunk (r+1−k)      forward                 -> next
    //   phase 2P−2          AG receive   chunk (r+2) mod P  (staged: slot -> own buf)
    // G <= K/2 keeps the schedule deadlock-free (a producer never needs a credit its consumer can only
    // return after its own blocked production) and leaves G−1 slices of slack per hop to hide the flag
    // latency.  Every rank executes the same (round, phase, slice) sequence, so slot numbers match.
    const int64_t G = (int64_t)(K / 2);

    auto range = [&](int c, int64_t i, int64_t& lo, int64_t& len) {
        const int64_t clo = (int64_t)c * cs;
        const int64_t chi = min(clo + cs, count);
        const int64_t a = clo + (int64_t)ch * sub + i * sl;
        const int64_t b = min(min(a + sl, clo + min((int64_t)(ch + 1) * sub, cs)), chi);
        lo = a;
        len = b > a ? b - a : 0;
    };
    auto reads_slot = [&](int k) { return k == K_MID || k == K_LAST || (!direct && (k == K_AGMID || k == K_AGLAST)); };
    auto writes_slot = [&](int k) { return k == K_FIRST || k == K_MID || (!direct && (k == K_LAST || k == K_AGMID)); };
    auto waits_ag = [&](int k) { return direct && (k == K_AGMID || k == K_AGLAST); };
    auto sends_ag = [&](int k) { return direct && (k == K_LAST || k == K_AGMID); };
    auto needs_g = [&](int k) { return act && (k == K_FIRST || k == K_MID || k == K_LAST); };
    auto needs_in = [&](int k) { return k != K_FIRST && !(direct && k == K_AGLAST); };
    auto ntiles = [&](int k, int64_t len) -> int64_t {
        if (direct && k == K_AGLAST) return 0;
        return (len + te - 1) / te;
    };
    auto mode_of = [&](int k) -> int {
        if (k == K_FIRST) return act ? M_SCALE : M_ZERO;
        if (k == K_MID || k == K_LAST) return act ? M_FMA : M_COPY;
        return M_COPY;
    };
    // where a hop's result goes: the next rank's staging slot, own buffer, and/or the next rank's buffer
    auto dests = [&](int kind, int64_t lo, unsigned long long prodJ, T*& out1, T*& out2) {
        T* nslot = reinterpret_cast<T*>(slot_of(tab->win[next], tab, ch, prodJ));
        out2 = nullptr;
        if (kind == K_FIRST || kind == K_MID) out1 = nslot;
        else if (kind == K_LAST) { out1 = th + lo; out2 = direct ? nth + lo : nslot; }
        else if (kind == K_AGMID) { if (direct) out1 = nth + lo; else { out1 = buf + lo; out2 = nslot; } }
        else out1 = buf + lo;                                   // K_AGLAST (staged)
    };

    if (threadIdx.x < 32) {
        // ================= producer: flags -> TMA bulk loads into the smem ring =======================
        if (t0) {
            unsigned long long prodJ = st->slot_base, consJ = st->slot_base, agC = st->ag_base;
            uint32_t tc = 0;
            int stg = 0;
            uint32_t eph = 1;   // parity of the `empty` phase a reuse of stage stg waits for (first use: none)
            bool bad = false;
            for_each_step(P, r, nsl, G, [&](int kind, int c, int64_t i) {
                int64_t lo, len;
                range(c, i, lo, len);
                if (tab->l2pf && !bad && needs_g(kind)) {
                    // PR_COMM_FLAG_L2_PREFETCH: the own gradient of this slice does not depend on any peer;
                    // start pulling it into L2 before the flag waits so the tiles' TMA loads hit L2
                    const uint8_t* p0 = reinterpret_cast<const uint8_t*>(buf + lo);
                    const int64_t bytes = (len * (int64_t)sizeof(T)) & ~15ll;
                    for (int64_t o = 0; o < bytes; o += 65536) prefetch_l2(p0 + o, (uint32_t)min((int64_t)65536, bytes - o));
                }
                if (!bad) {
                    bool ok = true;
                    if (reads_slot(kind)) ok = wait_ge(&myf->rs_ready, consJ + 1, deadline, sys);
                    if (ok && waits_ag(kind)) ok = wait_ge(&myf->ag_ready, agC + 1, deadline, sys);
                    if (ok && writes_slot(kind) && prodJ + 1 > K) ok = wait_ge(&myf->rs_credit, prodJ + 1 - K, deadline, sys);
                    if (!ok) {
                        bad = true;
                        *(volatile int*)&sh.err = PR_ERR_PEER_TIMEOUT;
                        latch(tab, PR_ERR_PEER_TIMEOUT);
                    }
                    if (reads_slot(kind) || waits_ag(kind)) fence_proxy_async_global();
                }
                const int64_t nt = ntiles(kind, len);
                const T* gsrc = buf + lo;
                const T* isrc = (kind == K_AGMID && direct) ? th + lo
                                                            : reinterpret_cast<const T*>(slot_of(my, tab, ch, consJ));
                for (int64_t t = 0; t < nt; ++t, ++tc) {
                    // stage / phase maintained incrementally: a runtime `%` and `/` per tile on this one
                    // thread were a measurable share of its serial per-tile issue time
                    if (tc >= (uint32_t)kStages) mbar_wait(&sh.empty[stg], eph);
                    const int64_t e0 = t * te;
                    const int64_t ne = min(te, len - e0);
                    const uint32_t vb = (uint32_t)((ne * (int64_t)sizeof(T)) & ~15ll);   // whole 16 B vectors
                    uint8_t* gs = smem + (size_t)stg * 2 * kTileBytes;
                    uint8_t* is = gs + kTileBytes;
                    uint32_t tx = 0;
                    if (!bad && vb) {
                        if (needs_g(kind)) tx += vb;
                        if (needs_in(kind)) tx += vb;
                    }
                    sh.tile_ok[stg] = bad ? 0 : 1;
                    if (!bad && vb) {      // copies first, then the arrive that carries their byte count
                        if (needs_g(kind)) tma_load(gs, gsrc + e0, vb, &sh.full[stg]);
                        if (needs_in(kind)) tma_load(is, isrc + e0, vb, &sh.full[stg]);
                    }
                    mbar_arrive_expect_tx(&sh.full[stg], tx);
                    if (++stg == kStages) {
                        stg = 0;
                        eph ^= 1u;
                    }
                }
                if (reads_slot(kind)) ++consJ;
                if (writes_slot(kind)) ++prodJ;
                if (waits_ag(kind)) ++agC;
            });
            sh.fin_slot = consJ;                   // hand the final counters to the epilogue
            sh.fin_ag = agC;
        }
    } else if (threadIdx.x < 64) {
        // ================= signal warp: per-slice release of ready flags, off the data path ===========
        // Waits until the consumers' stores of a slice's tiles are issued (stored barrier, release.cta by
        // every consumer warp), then one sys-scope release makes the whole slice visible to the peer.
        if (threadIdx.x == 32 && BULK) {
            // BULK: the signal thread also moves the data.  Per tile: wait `stored` (the consumers' results
            // are in the tile's smem, fenced for the async proxy), issue one bulk store per destination,
            // commit; the stage is handed back to the producer once its bulk group has finished reading
            // smem (one group of slack).  A slice's flag is released after all its groups COMPLETED.
            unsigned long long prodJ = st->slot_base, agP = st->ag_base, consJ = st->slot_base;
            int stg = 0, prev_stg = -1;
            uint32_t ph = 0;
            for_each_step(P, r, nsl, G, [&](int kind, int c, int64_t i) {
                int64_t lo, len;
                range(c, i, lo, len);
                const int64_t nt = ntiles(kind, len);
                const bool sends = sends_ag(kind) || writes_slot(kind);
                T* out1;
                T* out2;
                dests(kind, lo, prodJ, out1, out2);
                bool ok = true;
                for (int64_t t = 0; t < nt; ++t) {
                    mbar_wait(&sh.stored[stg], ph);
                    ok = ok && sh.tile_ok[stg] != 0;
                    const int64_t e0 = t * te;
                    const int64_t ne = min(te, len - e0);
                    const uint32_t vb = (uint32_t)((ne * (int64_t)sizeof(T)) & ~15ll);
                    const uint8_t* src = smem + (size_t)stg * 2 * kTileBytes + kTileBytes;
                    if (ok && vb) {
                        tma_store(out1 + e0, src, vb);
                        if (out2) tma_store(out2 + e0, src, vb);
                    }
                    bulk_commit();
                    bulk_wait_read<1>();                    // the previous tile's stores have read their smem
                    if (prev_stg >= 0) mbar_arrive(&sh.empty[prev_stg]);
                    prev_stg = stg;
                    if (++stg == kStages) {
                        stg = 0;
                        ph ^= 1u;
                    }
                    if (t == nt - 1) {
                        bulk_wait<0>();                     // the slice's writes are performed ...
                        fence_proxy_async_global();         // ... and ordered before the generic release
                        if (sends && ok) {
                            if (sends_ag(kind)) st_release(&nxf->ag_ready, agP + 1, sys);
                            else st_release(&nxf->rs_ready, prodJ + 1, sys);
                        }
                        if (reads_slot(kind) && ok) st_relaxed_u64(&pvf->rs_credit, consJ + 1, sys);
                    }
                }
                if (nt == 0 && !*(volatile int*)&sh.err) {   // empty slice: nothing to wait for
                    if (sends) {
                        if (sends_ag(kind)) st_release(&nxf->ag_ready, agP + 1, sys);
                        else st_release(&nxf->rs_ready, prodJ + 1, sys);
                    }
                    if (reads_slot(kind)) st_relaxed_u64(&pvf->rs_credit, consJ + 1, sys);
                }
                if (sends_ag(kind)) ++agP;
                else if (writes_slot(kind)) ++prodJ;
                if (reads_slot(kind)) ++consJ;
            });
            bulk_wait<0>();
            if (prev_stg >= 0) mbar_arrive(&sh.empty[prev_stg]);
        } else if (threadIdx.x == 32) {
            unsigned long long prodJ = st->slot_base, agP = st->ag_base, consJ = st->slot_base;            int stg = 0;
            uint32_t ph = 0;
            for_each_step(P, r, nsl, G, [&](int kind, int c, int64_t i) {
                int64_t lo, len;
                range(c, i, lo, len);
                const int64_t nt = ntiles(kind, len);
                const bool sends = sends_ag(kind) || writes_slot(kind);
                bool ok = true;
                for (int64_t t = 0; t < nt; ++t) {
                    // wait for EVERY tile's phase: try_wait.parity cannot tell phase k+1 from k−1, so a
                    // skipped phase would let a later wait on this stage return early (found by synccheck)
                    mbar_wait(&sh.stored[stg], ph);
                    ok = ok && sh.tile_ok[stg] != 0;
                    // stage free: consumers read it before arriving on `stored`; the chain consumer ->
                    // stored -> signal -> empty -> producer is transitive (release/acquire at each step)
                    mbar_arrive(&sh.empty[stg]);
                    if (++stg == kStages) {
                        stg = 0;
                        ph ^= 1u;
                    }
                    if (t == nt - 1 && sends && ok) {
                        if (sends_ag(kind)) st_release(&nxf->ag_ready, agP + 1, sys);
                        else st_release(&nxf->rs_ready, prodJ + 1, sys);
                    }
                    // the slice's received slot is consumed (every tile's TMA landed before its consumers
                    // arrived on `stored`): hand it back to the previous rank
                    if (t == nt - 1 && reads_slot(kind) && ok) st_relaxed_u64(&pvf->rs_credit, consJ + 1, sys);
                }
                if (nt == 0 && !*(volatile int*)&sh.err) {   // empty slice: nothing to wait for
                    if (sends) {
                        if (sends_ag(kind)) st_release(&nxf->ag_ready, agP + 1, sys);
                        else st_release(&nxf->rs_ready, prodJ + 1, sys);
                    }
                    if (reads_slot(kind)) st_relaxed_u64(&pvf->rs_credit, consJ + 1, sys);
                }
                if (sends_ag(kind)) ++agP;
                else if (writes_slot(kind)) ++prodJ;
                if (reads_slot(kind)) ++consJ;
            });
        }
    } else {
        // ================= consumers: smem -> fp32 math -> 16 B stores to local + peer memory ==========
        const int cid = threadIdx.x - 64;
        const int lane = threadIdx.x & 31;
        unsigned long long prodJ = st->slot_base, consJ = st->slot_base;
        int stg = 0;
        uint32_t ph = 0;
        for_each_step(P, r, nsl, G, [&](int kind, int c, int64_t i) {
            int64_t lo, len;
            range(c, i, lo, len);
            const int64_t nt = ntiles(kind, len);
            const int mode = mode_of(kind);
            T* out1;
            T* out2;
            dests(kind, lo, prodJ, out1, out2);
            const T* gsrc = buf + lo;
            const T* isrc = (kind == K_AGMID && direct) ? th + lo
                                                        : reinterpret_cast<const T*>(slot_of(my, tab, ch, consJ));
            const bool upd = FUSE && kind == K_LAST;                // reduced chunk final here: apply SGD
            const bool zg = FUSE && A.zero && kind <= K_LAST;        // own gradient consumed: reset it
            SliceArgs<T> sa{out1, out2, zg ? buf + lo : nullptr, upd ? th + lo : nullptr, gsrc, isrc, len, te, nt, s,
                            A.nlr, A.wd};   // (slot credits are returned by the signal warp)
            // the hop's arithmetic is fixed per instantiation: one switch per slice, none per tile / element
            switch (mode) {
                case M_SCALE: consume_slice<T, M_SCALE, FUSE, BULK>(sh, smem, kTileBytes, kStages, stg, ph, cid, nc, lane, sa); break;
                case M_FMA: consume_slice<T, M_FMA, FUSE, BULK>(sh, smem, kTileBytes, kStages, stg, ph, cid, nc, lane, sa); break;
                case M_COPY: consume_slice<T, M_COPY, FUSE, BULK>(sh, smem, kTileBytes, kStages, stg, ph, cid, nc, lane, sa); break;
                default: consume_slice<T, M_ZERO, FUSE, BULK>(sh, smem, kTileBytes, kStages, stg, ph, cid, nc, lane, sa); break;
            }
            if (reads_slot(kind)) ++consJ;
            if (writes_slot(kind)) ++prodJ;
        });
    }
    __syncthreads();
    if (t0) {
        if (!*(volatile int*)&sh.err) {
            st->slot_base = sh.fin_slot;   // == prodJ: all ranks produce/consume equally
            st->ag_base = sh.fin_ag;
        }
        if (ch == 0) tab->stamps[2] = (long long)gtimer();
    }
}

// =====================================================================================================
// Two-shot variant: 2 synchronisation phases instead of 2(P−1) — NVSwitch gives every
// peer full bandwidth, so the ring's hop chain is only needed for its order, not its topology.
//   phase A  rank r pushes its RAW slice i of every other chunk d into rank d's staging [src r]
//   phase B  rank d reduces chunk d's slice i in the ring's order (d, d+1, …, d+P−1) with the ring's
//            per-hop rounding — so the result is bit-identical to ring_kernel — and stores it into its
//            own buffer and every peer's registered buffer (direct all-gather)
// Per-peer counters in TsFlags: ready (data landed), credit (slot consumed), ag (reduced slice landed).
// K2 >= 2 staging slots per (channel, source): to push slice i+1 a rank needs the credit for slice
// i+1−K2, returned by the destination's phase B of that slice, which precedes its phase A of slice
// i+2−K2 ≤ i — so the schedule cannot deadlock.
// =====================================================================================================
__device__ __forceinline__ uint4 ld_cg_v4(const void* p) {     // L2-coherent load of peer-written data
    uint4 v;
    asm volatile("ld.global.cg.v4.u32 {%0,%1,%2,%3}, [%4];" : "=r"(v.x), "=r"(v.y), "=r"(v.z), "=r"(v.w) : "l"(p));
    return v;
}
__device__ __forceinline__ TsFlags* ts_flags_of(uint8_t* w, const DevTable* t, int ch) {
    return reinterpret_cast<TsFlags*>(w + t->off_ts_flags) + ch;
}
__device__ __forceinline__ uint8_t* ts_slot_of(uint8_t* w, const DevTable* t, int ch, int src, unsigned long long J) {
    return w + t->off_ts_staging +
           (((size_t)ch * t->P + src) * t->ts_slots + (size_t)(J % (unsigned long long)t->ts_slots)) * t->ts_slot_bytes;
}
template <typename T> __device__ __forceinline__ float rnd_dtype(float x);
template <> __device__ __forceinline__ float rnd_dtype<float>(float x) { return x; }
template <> __device__ __forceinline__ float rnd_dtype<__nv_bfloat16>(float x) {
    return __bfloat162float(__float2bfloat16_rn(x));
}
template <typename T> __device__ __forceinline__ float lane_f(const uint4& v, int j);
template <> __device__ __forceinline__ float lane_f<float>(const uint4& v, int j) {
    const uint32_t w[4] = {v.x, v.y, v.z, v.w};
    return __uint_as_float(w[j]);
}
template <> __device__ __forceinline__ float lane_f<__nv_bfloat16>(const uint4& v, int j) {
    const uint32_t w[4] = {v.x, v.y, v.z, v.w};
    return (j & 1) ? __uint_as_float(w[j >> 1] & 0xffff0000u) : __uint_as_float(w[j >> 1] << 16);
}
template <typename T> __device__ __forceinline__ uint4 pack_f(const float* f);
template <> __device__ __forceinline__ uint4 pack_f<float>(const float* f) {
    return make_uint4(__float_as_uint(f[0]), __float_as_uint(f[1]), __float_as_uint(f[2]), __float_as_uint(f[3]));
}
template <> __device__ __forceinline__ uint4 pack_f<__nv_bfloat16>(const float* f) {
    return make_uint4(Vec<__nv_bfloat16>::pack(f[0], f[1]), Vec<__nv_bfloat16>::pack(f[2], f[3]),
                      Vec<__nv_bfloat16>::pack(f[4], f[5]), Vec<__nv_bfloat16>::pack(f[6], f[7]));
}

// Executed by all 32 lanes of one warp: lane l waits on the counter of peer (r+1+l) mod P (and l+32, …),
// so the P−1 acquire polls are in flight together instead of one after another (one flag latency per
// wait point, not P−1).  True in every lane iff every peer reached `target` before the deadline.
__device__ __forceinline__ bool warp_wait_peers(const unsigned long long* arr, unsigned long long target, int r, int P,
                                                unsigned long long deadline, bool sys) {
    bool ok = true;
    for (int l = (int)(threadIdx.x & 31); l < P - 1; l += 32)
        ok = ok && wait_ge(&arr[(r + 1 + l) % P], target, deadline, sys);
    return __all_sync(0xffffffffu, ok);
}

// Two-shot phase B on one slice: every element reduced over the P sources in the ring's order for chunk r
// with the ring's per-hop rounding.  Source pointers, weights and activity are resolved once per slice into
// shared memory (src[h] is source h = rank (r+h) mod P: the own gradient or its staging slot), so the
// vector loop does P cache-global loads, P FMAs per element and P stores — no slot-address arithmetic or
// modulo per element (that was most of the instructions).  PP > 0: P known at compile time (unrolled).
template <typename T, int PP>
__device__ __forceinline__ void ts_reduce(int P, int64_t nv, const uint8_t* const* src, const float* wt, const int* act,
                                          uint8_t* const* dst) {
    constexpr int V = Vec<T>::V;
    const int np = PP > 0 ? PP : P;
    for (int64_t v = threadIdx.x; v < nv; v += blockDim.x) {
        float acc[V];
#pragma unroll
        for (int j = 0; j < V; ++j) acc[j] = 0.0f;
#pragma unroll
        for (int h = 0; h < (PP > 0 ? PP : 1); ++h) {
            if (PP == 0) break;
            if (!act[h]) continue;                            // n_q = 0 contributes nothing (never multiplied)
            const uint4 x = ld_cg_v4(src[h] + (size_t)v * 16);
            const float sq = wt[h];
#pragma unroll
            for (int j = 0; j < V; ++j)
                acc[j] = rnd_dtype<T>(h == 0 ? __fmul_rn(sq, lane_f<T>(x, j)) : __fmaf_rn(sq, lane_f<T>(x, j), acc[j]));
        }
        if (PP == 0) {
            for (int h = 0; h < np; ++h) {
                if (!act[h]) continue;
                const uint4 x = ld_cg_v4(src[h] + (size_t)v * 16);
                const float sq = wt[h];
#pragma unroll
                for (int j = 0; j < V; ++j)
                    acc[j] = rnd_dtype<T>(h == 0 ? __fmul_rn(sq, lane_f<T>(x, j)) : __fmaf_rn(sq, lane_f<T>(x, j), acc[j]));
            }
        }
        const uint4 y = pack_f<T>(acc);
#pragma unroll 8
        for (int q = 0; q < np; ++q) st_v4(dst[q] + (size_t)v * 16, y);
    }
}

template <typename T>
__global__ void __launch_bounds__(512, 1) twoshot_kernel(const __grid_constant__ LaunchArgs A) {
    __shared__ int s_err;
    __shared__ long long s_sumn;
    __shared__ long long s_n[PR_MAX_RANKS];
    __shared__ uint8_t* s_bufs[PR_MAX_RANKS];
    __shared__ float s_w[PR_MAX_RANKS];
    __shared__ const uint8_t* s_src[PR_MAX_RANKS];
    __shared__ uint8_t* s_dst[PR_MAX_RANKS];
    __shared__ float s_wt[PR_MAX_RANKS];
    __shared__ int s_act[PR_MAX_RANKS];
    const RankCall& rc = A.calls[blockIdx.y];
    const DevTable* tab = rc.tab;
    const int ch = blockIdx.x;
    const int r = tab->rank, P = tab->P;
    uint8_t* my = tab->win[r];
    ChanState* st = state_of(my, tab, ch);
    TsFlags* mf = ts_flags_of(my, tab, ch);
    const bool t0 = threadIdx.x == 0;
    const bool sys = tab->sysscope != 0;
    unsigned long long deadline = ~0ull;
    if (threadIdx.x < 32) {                           // warp 0 runs the handshake
        const unsigned long long start = gtimer();
        if (tab->watchdog_ns > 0) deadline = start + (unsigned long long)tab->watchdog_ns;
        if (t0 && ch == 0) tab->stamps[0] = (long long)start;
        const HsOut hs = handshake(A, rc, tab, st, ch, sys, deadline, s_n, s_bufs);
        __syncwarp();
        for (int q = (int)threadIdx.x; q < P; q += 32)
            s_w[q] = hs.sumn > 0 ? (float)((double)s_n[q] / (double)hs.sumn) : 0.0f;
        if (t0) {
            s_err = hs.err ? hs.err : (hs.direct ? 0 : PR_ERR_INVALID);   // two-shot needs registered buffers
            s_sumn = hs.sumn;
            if (ch == 0) tab->stamps[1] = (long long)gtimer();
        }
    }
    __syncthreads();
    if (s_err) {
        if (t0) latch(tab, s_err);
        return;
    }
    constexpr int V = Vec<T>::V;
    const int64_t count = A.count;
    const int64_t per = (count + P - 1) / P;
    const int64_t cs = (per + V - 1) / V * V;
    const int64_t subp = (cs + tab->channels - 1) / tab->channels;
    const int64_t sub = (subp + V - 1) / V * V;
    const int64_t sl = tab->ts_slot_bytes / (int64_t)sizeof(T);
    const int64_t nsl = sub > 0 ? (sub + sl - 1) / sl : 0;
    const unsigned long long K2 = (unsigned long long)tab->ts_slots;
    const unsigned long long base = st->ts_base;
    T* buf = reinterpret_cast<T*>(rc.buf);
    auto range = [&](int c, int64_t i, int64_t& lo, int64_t& len) {
        const int64_t clo = (int64_t)c * cs;
        const int64_t chi = min(clo + cs, count);
        const int64_t a = clo + (int64_t)ch * sub + i * sl;
        const int64_t b = min(min(a + sl, clo + min((int64_t)(ch + 1) * sub, cs)), chi);
        lo = a;
        len = b > a ? b - a : 0;
    };
    __shared__ int s_abort;
    if (t0) s_abort = 0;
    auto sync_ok = [&]() -> bool {
        __syncthreads();
        return s_abort == 0;
    };
    auto fail = [&]() {
        s_abort = 1;
        latch(tab, PR_ERR_PEER_TIMEOUT);
    };
    for (int64_t i = 0; i < nsl; ++i) {
        const unsigned long long J = base + (unsigned long long)i;
        // ---- phase A: raw slice i of every chunk d != r -> rank d's staging [src r], all peers at once --------
        if (threadIdx.x < 32 && J + 1 > K2)
            if (!warp_wait_peers(mf->credit, J + 1 - K2, r, P, deadline, sys) && t0) fail();
        if (!sync_ok()) return;
        for (int k = 1; k < P; ++k) {                               // no barrier between destinations
            const int d = (r + k) % P;
            int64_t lo, len;
            range(d, i, lo, len);
            T* dst = reinterpret_cast<T*>(ts_slot_of(tab->win[d], tab, ch, r, J));
            const int64_t nv = len / V;
            for (int64_t v = threadIdx.x; v < nv; v += blockDim.x)
                st_v4(dst + v * V, *reinterpret_cast<const uint4*>(buf + lo + v * V));
            for (int64_t e = nv * V + threadIdx.x; e < len; e += blockDim.x) dst[e] = buf[lo + e];
        }
        __syncthreads();
        if ((int)threadIdx.x < P - 1) {                              // one releasing thread per peer
            const int d = (r + 1 + (int)threadIdx.x) % P;
            st_release(&ts_flags_of(tab->win[d], tab, ch)->ready[r], J + 1, sys);
        }
        // ---- phase B: reduce chunk r's slice i in ring order, store into every rank's buffer -------------
        int64_t lo, len;
        range(r, i, lo, len);
        if (threadIdx.x < 32)
            if (!warp_wait_peers(mf->ready, J + 1, r, P, deadline, sys) && t0) fail();
        if (!sync_ok()) return;
        const int64_t nv = len / V;
        for (int h = (int)threadIdx.x; h < P; h += (int)blockDim.x) {     // resolve the P sources once
            const int q = (r + h) % P;
            s_src[h] = q == r ? reinterpret_cast<const uint8_t*>(buf + lo) : ts_slot_of(my, tab, ch, q, J);
            s_wt[h] = s_w[q];
            s_act[h] = s_n[q] > 0 ? 1 : 0;
            s_dst[h] = reinterpret_cast<uint8_t*>(reinterpret_cast<T*>(s_bufs[h]) + lo);
        }
        __syncthreads();
        if (P == 8) ts_reduce<T, 8>(P, nv, s_src, s_wt, s_act, s_dst);
        else if (P == 4) ts_reduce<T, 4>(P, nv, s_src, s_wt, s_act, s_dst);
        else if (P == 2) ts_reduce<T, 2>(P, nv, s_src, s_wt, s_act, s_dst);
        else ts_reduce<T, 0>(P, nv, s_src, s_wt, s_act, s_dst);
        for (int64_t e = nv * V + threadIdx.x; e < len; e += blockDim.x) {   // ragged tail: end of buffer
            float acc = 0.0f;
            for (int h = 0; h < P; ++h) {
                const int q = (r + h) % P;
                const T xv = (q == r) ? buf[lo + e] : reinterpret_cast<const T*>(ts_slot_of(my, tab, ch, q, J))[e];
                if (s_n[q] <= 0) continue;
                acc = rnd_dtype<T>(h == 0 ? __fmul_rn(s_w[q], Vec<T>::to_f(xv)) : __fmaf_rn(s_w[q], Vec<T>::to_f(xv), acc));
            }
            for (int q = 0; q < P; ++q) reinterpret_cast<T*>(s_bufs[q])[lo + e] = Vec<T>::from_f(acc);
        }
        __syncthreads();
        if ((int)threadIdx.x < P - 1) {                              // one releasing thread per peer
            const int q = (r + 1 + (int)threadIdx.x) % P;
            TsFlags* qf = ts_flags_of(tab->win[q], tab, ch);
            st_relaxed_u64(&qf->credit[r], J + 1, sys);       // its slot in my staging is free again
            st_release(&qf->ag[r], J + 1, sys);               // my reduced slice i is in its buffer
        }
    }
    // every other rank's reduced chunk has landed in my buffer
    if (threadIdx.x < 32)
        if (!warp_wait_peers(mf->ag, base + (unsigned long long)nsl, r, P, deadline, sys) && t0) fail();
    __syncthreads();
    if (t0) {
        if (!s_abort) st->ts_base = base + (unsigned long long)nsl;
        if (ch == 0) tab->stamps[2] = (long long)gtimer();
    }
}

// =====================================================================================================
// Pull two-shot (PR_ALGO_TWO_SHOT_PULL, round 2): the two-shot's reduction with phase A replaced by loads.
// After the handshake (the barrier: every rank's gradient is final) rank r reads its chunk r straight out
// of the P ranks' registered buffers, in the ring's order for chunk r (r, r+1, …, r+P−1) with the ring's
// per-hop rounding — the ring's bits — and stores the result into all P buffers.  No staging, no per-slice
// flags: one release per peer at the end ("my reduced chunk is in your buffer, and I have finished reading
// yours") and one wait for all P−1 of them.  No hazard between ranks: chunk r of every buffer is read and
// then written only by rank r (same thread, same address, program order).
// Why: a channel's bound is the SM's store path (≈ 62 GB/s per SM).  The ring and the push
// two-shot store (2P−1)/P·Z per rank for a bus volume of 2(P−1)/P·Z — 1.5 (P = 2) to 1.07 (P = 8) stored
// bytes per bus byte; pulling phase A leaves only phase B's Z of stores: P/(2(P−1)) = 1.0 (P = 2) to 0.57
// (P = 8).  The loads are the same Z per rank (own chunk + P−1 peer slices), issued as P independent
// 16-byte L2-coherent loads per vector and thread.
// =====================================================================================================
// The pull two-shot's reduction: like ts_reduce, but U vectors per thread per iteration with all U·P loads
// issued before any store.  The own buffer is both a source and a destination, so the compiler cannot
// hoist the next iteration's loads above this iteration's stores by itself; with P = 2 one vector per
// iteration left 2 loads in flight per thread and the channel latency-bound.
// FUSE (fp32): ḡ is not stored; θ' = K7(θ, ḡ) from the owner's θ replica (`thp`) goes to the P θ buffers (dst).
template <typename T, int PP, int U, bool FUSE>
__device__ __forceinline__ void ts_pull_reduce(int64_t nv, const uint8_t* const* src, const float* wt, const int* act,
                                               uint8_t* const* dst, const uint8_t* thp, float nlr, float wd) {
    constexpr int V = Vec<T>::V;
    const int64_t B = blockDim.x;
    for (int64_t v0 = threadIdx.x; v0 < nv; v0 += B * U) {
        uint4 x[U][PP];
#pragma unroll
        for (int u = 0; u < U; ++u) {
            const int64_t v = v0 + u * B;
#pragma unroll
            for (int h = 0; h < PP; ++h)
                x[u][h] = (v < nv && act[h]) ? ld_cg_v4(src[h] + (size_t)v * 16) : make_uint4(0, 0, 0, 0);
        }
#pragma unroll
        for (int u = 0; u < U; ++u) {
            const int64_t v = v0 + u * B;
            if (v >= nv) break;
            float acc[V];
#pragma unroll
            for (int j = 0; j < V; ++j) acc[j] = 0.0f;
#pragma unroll
            for (int h = 0; h < PP; ++h) {
                if (!act[h]) continue;                        // n_q = 0 contributes nothing (never multiplied)
                const float sq = wt[h];
#pragma unroll
                for (int j = 0; j < V; ++j)
                    acc[j] = rnd_dtype<T>(h == 0 ? __fmul_rn(sq, lane_f<T>(x[u][h], j))
                                                 : __fmaf_rn(sq, lane_f<T>(x[u][h], j), acc[j]));
            }
            uint4 y = pack_f<T>(acc);
            if (FUSE) y = sgd_v4<T>(*reinterpret_cast<const uint4*>(thp + (size_t)v * 16), y, nlr, wd);
#pragma unroll
            for (int q = 0; q < PP; ++q) st_v4(dst[q] + (size_t)v * 16, y);
        }
    }
}

// Any P (not unrolled), one vector per iteration; FUSE as above.
template <typename T, bool FUSE>
__device__ __forceinline__ void ts_pull_reduce_any(int P, int64_t nv, const uint8_t* const* src, const float* wt,
                                                   const int* act, uint8_t* const* dst, const uint8_t* thp, float nlr,
                                                   float wd) {
    constexpr int V = Vec<T>::V;
    for (int64_t v = threadIdx.x; v < nv; v += blockDim.x) {
        float acc[V];
#pragma unroll
        for (int j = 0; j < V; ++j) acc[j] = 0.0f;
        for (int h = 0; h < P; ++h) {
            if (!act[h]) continue;
            const uint4 x = ld_cg_v4(src[h] + (size_t)v * 16);
            const float sq = wt[h];
#pragma unroll
            for (int j = 0; j < V; ++j)
                acc[j] = rnd_dtype<T>(h == 0 ? __fmul_rn(sq, lane_f<T>(x, j)) : __fmaf_rn(sq, lane_f<T>(x, j), acc[j]));
        }
        uint4 y = pack_f<T>(acc);
        if (FUSE) y = sgd_v4<T>(*reinterpret_cast<const uint4*>(thp + (size_t)v * 16), y, nlr, wd);
        for (int q = 0; q < P; ++q) st_v4(dst[q] + (size_t)v * 16, y);
    }
}

// FUSE (fp32, rows a6-a9 in one kernel as ring_kernel<float, true>): the owner of chunk r applies K7 to its θ
// replica and stores θ' into the P θ buffers (buf + th_delta on every rank) instead of ḡ; ḡ is never
// materialised.  With A.zero each rank resets its own gradient after the final wait (every peer has then
// finished reading it).  Same bits as ring + K7.
template <typename T, bool FUSE>
__global__ void __launch_bounds__(512, 1) twoshot_pull_kernel(const __grid_constant__ LaunchArgs A) {
    __shared__ int s_err;
    __shared__ long long s_n[PR_MAX_RANKS];
    __shared__ uint8_t* s_bufs[PR_MAX_RANKS];
    __shared__ float s_w[PR_MAX_RANKS];
    __shared__ const uint8_t* s_src[PR_MAX_RANKS];
    __shared__ uint8_t* s_dst[PR_MAX_RANKS];
    __shared__ float s_wt[PR_MAX_RANKS];
    __shared__ int s_act[PR_MAX_RANKS];
    __shared__ int s_abort;
    const RankCall& rc = A.calls[blockIdx.y];
    const DevTable* tab = rc.tab;
    const int ch = blockIdx.x;
    const int r = tab->rank, P = tab->P;
    uint8_t* my = tab->win[r];
    ChanState* st = state_of(my, tab, ch);
    TsFlags* mf = ts_flags_of(my, tab, ch);
    const bool t0 = threadIdx.x == 0;
    const bool sys = tab->sysscope != 0;
    unsigned long long deadline = ~0ull;
    if (threadIdx.x < 32) {                           // warp 0 runs the handshake
        const unsigned long long start = gtimer();
        if (tab->watchdog_ns > 0) deadline = start + (unsigned long long)tab->watchdog_ns;
        if (t0 && ch == 0) tab->stamps[0] = (long long)start;
        const HsOut hs = handshake(A, rc, tab, st, ch, sys, deadline, s_n, s_bufs);
        __syncwarp();
        for (int q = (int)threadIdx.x; q < P; q += 32)
            s_w[q] = hs.sumn > 0 ? (float)((double)s_n[q] / (double)hs.sumn) : 0.0f;
        if (t0) {
            s_err = hs.err ? hs.err : (hs.direct ? 0 : PR_ERR_INVALID);   // reads and writes registered buffers
            if (FUSE && A.fuse == 0) s_err = PR_ERR_INVALID;
            s_abort = 0;
            if (ch == 0) tab->stamps[1] = (long long)gtimer();
        }
    }
    __syncthreads();
    if (s_err) {
        if (t0) latch(tab, s_err);
        return;
    }
    constexpr int V = Vec<T>::V;
    const int64_t count = A.count;
    const int64_t per = (count + P - 1) / P;
    const int64_t cs = (per + V - 1) / V * V;
    const int64_t subp = (cs + tab->channels - 1) / tab->channels;
    const int64_t sub = (subp + V - 1) / V * V;
    const unsigned long long base = st->ts_base;
    // this channel's share of chunk r (the ring's chunk / channel geometry, DESIGN.md §3 #14)
    const int64_t clo = (int64_t)r * cs;
    const int64_t lo = clo + (int64_t)ch * sub;
    const int64_t hi = min(clo + min((int64_t)(ch + 1) * sub, cs), count);
    const int64_t len = hi > lo ? hi - lo : 0;
    const int64_t nv = len / V;
    for (int h = (int)threadIdx.x; h < P; h += (int)blockDim.x) {     // the P sources in ring order, once
        const int q = (r + h) % P;
        s_src[h] = reinterpret_cast<const uint8_t*>(reinterpret_cast<const T*>(s_bufs[q]) + lo);
        s_wt[h] = s_w[q];
        s_act[h] = s_n[q] > 0 ? 1 : 0;
        // destinations: the P gradient buffers, or (FUSE) the P θ buffers = gradient + th_delta bytes
        s_dst[h] = reinterpret_cast<uint8_t*>(reinterpret_cast<T*>(s_bufs[h] + (FUSE ? rc.th_delta : 0)) + lo);
    }
    __syncthreads();
    const uint8_t* thp = FUSE ? reinterpret_cast<const uint8_t*>(reinterpret_cast<const T*>(
                                    reinterpret_cast<const uint8_t*>(rc.buf) + rc.th_delta) + lo)
                              : nullptr;
    if (len > 0) {
        // U = 16/P: 16 loads (256 B) in flight per thread at every P — 128 KiB per channel, for the latency of
        // peer reads (U = 8/P measured 0-11 % slower per channel co-located, profiles/round2_k3_pull_deep_ab.jsonl)
        if (P == 8) ts_pull_reduce<T, 8, 2, FUSE>(nv, s_src, s_wt, s_act, s_dst, thp, A.nlr, A.wd);
        else if (P == 4) ts_pull_reduce<T, 4, 4, FUSE>(nv, s_src, s_wt, s_act, s_dst, thp, A.nlr, A.wd);
        else if (P == 2) ts_pull_reduce<T, 2, 8, FUSE>(nv, s_src, s_wt, s_act, s_dst, thp, A.nlr, A.wd);
        else ts_pull_reduce_any<T, FUSE>(P, nv, s_src, s_wt, s_act, s_dst, thp, A.nlr, A.wd);
        for (int64_t e = nv * V + threadIdx.x; e < len; e += blockDim.x) {   // ragged tail: end of buffer
            float acc = 0.0f;
            for (int h = 0; h < P; ++h) {
                const int q = (r + h) % P;
                if (s_n[q] <= 0) continue;
                const T xv = reinterpret_cast<const T*>(s_bufs[q])[lo + e];
                acc = rnd_dtype<T>(h == 0 ? __fmul_rn(s_w[q], Vec<T>::to_f(xv)) : __fmaf_rn(s_w[q], Vec<T>::to_f(xv), acc));
            }
            if (FUSE) {
                const float tv = Vec<T>::to_f(reinterpret_cast<const T*>(thp)[e]);
                acc = __fmaf_rn(A.nlr, __fmaf_rn(A.wd, tv, acc), tv);
            }
            for (int q = 0; q < P; ++q) reinterpret_cast<T*>(s_dst[q])[e] = Vec<T>::from_f(acc);
        }
    }
    __syncthreads();
    if ((int)threadIdx.x < P - 1) {                                  // one releasing thread per peer
        const int q = (r + 1 + (int)threadIdx.x) % P;
        st_release(&ts_flags_of(tab->win[q], tab, ch)->ag[r], base + 1, sys);
    }
    if (threadIdx.x < 32)
        if (!warp_wait_peers(mf->ag, base + 1, r, P, deadline, sys) && t0) {
            s_abort = 1;
            latch(tab, PR_ERR_PEER_TIMEOUT);
        }
    __syncthreads();
    if (FUSE && A.zero && !s_abort) {
        // every peer has read its slices of this rank's gradient: reset this channel's share of every chunk
        T* g = reinterpret_cast<T*>(rc.buf);
        for (int c = 0; c < P; ++c) {
            const int64_t a0 = (int64_t)c * cs + (int64_t)ch * sub;
            const int64_t a1 = min((int64_t)c * cs + min((int64_t)(ch + 1) * sub, cs), count);
            const int64_t zl = a1 > a0 ? a1 - a0 : 0;
            const int64_t zv = zl / V;
            for (int64_t v = threadIdx.x; v < zv; v += blockDim.x) st_v4(g + a0 + v * V, make_uint4(0, 0, 0, 0));
            for (int64_t e = zv * V + threadIdx.x; e < zl; e += blockDim.x) g[a0 + e] = Vec<T>::from_f(0.0f);
        }
    }
    if (t0) {
        if (!s_abort) st->ts_base = base + 1;   // the push two-shot's counters stay consistent (targets are >=)
        if (ch == 0) tab->stamps[2] = (long long)gtimer();
    }
}

// TMA-staged pull (PR_COMM_FLAG_PULL_TMA, opt-in): the same reduction, order, rounding and flags as
// twoshot_pull_kernel, but the P source tiles are brought into shared memory by one producer thread with
// cp.async.bulk (kPullStages deep, up to 192 KiB in flight per channel instead of 128 KiB in registers)
// and the consumer warps reduce from shared memory.  For peer reads over NVLink, whose round trip the
// register-queued loads expose; co-located the two are compared in profiles/round2_k3_pull_tma_ab.jsonl.
constexpr int kPullStages = 4;
__host__ __device__ constexpr int pull_tile_bytes(int P) {
    return ((196608 / (kPullStages * P)) & ~15) < 32768 ? ((196608 / (kPullStages * P)) & ~15) : 32768;
}

template <typename T, bool FUSE>
__global__ void __launch_bounds__(544, 1) twoshot_pull_tma_kernel(const __grid_constant__ LaunchArgs A) {
    extern __shared__ __align__(128) uint8_t smem[];   // [kPullStages][P][tile]
    __shared__ uint64_t full[kPullStages], empty[kPullStages];
    __shared__ int s_err;
    __shared__ long long s_n[PR_MAX_RANKS];
    __shared__ uint8_t* s_bufs[PR_MAX_RANKS];
    __shared__ float s_w[PR_MAX_RANKS];
    __shared__ const uint8_t* s_src[PR_MAX_RANKS];
    __shared__ uint8_t* s_dst[PR_MAX_RANKS];
    __shared__ float s_wt[PR_MAX_RANKS];
    __shared__ int s_act[PR_MAX_RANKS];
    __shared__ int s_abort;
    const RankCall& rc = A.calls[blockIdx.y];
    const DevTable* tab = rc.tab;
    const int ch = blockIdx.x;
    const int r = tab->rank, P = tab->P;
    uint8_t* my = tab->win[r];
    ChanState* st = state_of(my, tab, ch);
    TsFlags* mf = ts_flags_of(my, tab, ch);
    const bool t0 = threadIdx.x == 0;
    const bool sys = tab->sysscope != 0;
    const int nc = blockDim.x - 32;                   // consumer threads (warps 1..); warp 0: producer
    unsigned long long deadline = ~0ull;
    if (threadIdx.x < 32) {
        const unsigned long long start = gtimer();
        if (tab->watchdog_ns > 0) deadline = start + (unsigned long long)tab->watchdog_ns;
        if (t0) {
            if (ch == 0) tab->stamps[0] = (long long)start;
            for (int k = 0; k < kPullStages; ++k) {
                mbar_init(&full[k], 1);
                mbar_init(&empty[k], (uint32_t)(nc / 32));
            }
            asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
        }
        const HsOut hs = handshake(A, rc, tab, st, ch, sys, deadline, s_n, s_bufs);
        __syncwarp();
        for (int q = (int)threadIdx.x; q < P; q += 32)
            s_w[q] = hs.sumn > 0 ? (float)((double)s_n[q] / (double)hs.sumn) : 0.0f;
        if (t0) {
            s_err = hs.err ? hs.err : (hs.direct ? 0 : PR_ERR_INVALID);
            if (FUSE && A.fuse == 0) s_err = PR_ERR_INVALID;
            s_abort = 0;
            if (ch == 0) tab->stamps[1] = (long long)gtimer();
        }
    }
    __syncthreads();
    if (s_err) {
        if (t0) latch(tab, s_err);
        return;
    }
    constexpr int V = Vec<T>::V;
    const int64_t count = A.count;
    const int64_t per = (count + P - 1) / P;
    const int64_t cs = (per + V - 1) / V * V;
    const int64_t subp = (cs + tab->channels - 1) / tab->channels;
    const int64_t sub = (subp + V - 1) / V * V;
    const unsigned long long base = st->ts_base;
    const int64_t clo = (int64_t)r * cs;
    const int64_t lo = clo + (int64_t)ch * sub;
    const int64_t hi = min(clo + min((int64_t)(ch + 1) * sub, cs), count);
    const int64_t len = hi > lo ? hi - lo : 0;
    const int64_t nv = len / V;
    for (int h = (int)threadIdx.x; h < P; h += (int)blockDim.x) {
        const int q = (r + h) % P;
        s_src[h] = reinterpret_cast<const uint8_t*>(reinterpret_cast<const T*>(s_bufs[q]) + lo);
        s_wt[h] = s_w[q];
        s_act[h] = s_n[q] > 0 ? 1 : 0;
        s_dst[h] = reinterpret_cast<uint8_t*>(reinterpret_cast<T*>(s_bufs[h] + (FUSE ? rc.th_delta : 0)) + lo);
    }
    __syncthreads();
    const uint8_t* thp = FUSE ? reinterpret_cast<const uint8_t*>(reinterpret_cast<const T*>(
                                    reinterpret_cast<const uint8_t*>(rc.buf) + rc.th_delta) + lo)
                              : nullptr;
    const int tb = pull_tile_bytes(P);
    const int64_t vbytes = nv * 16;
    const int64_t ntiles = (vbytes + tb - 1) / tb;
    if (threadIdx.x < 32) {
        if (t0) {                                     // producer: P bulk loads per tile into one stage
            fence_proxy_async_global();               // peers' gradients (acquired in the handshake) -> TMA
            uint32_t nact = 0;
            for (int h = 0; h < P; ++h) nact += (uint32_t)s_act[h];
            for (int64_t t = 0; t < ntiles; ++t) {
                const int stg = (int)(t % kPullStages);
                if (t >= kPullStages) mbar_wait(&empty[stg], (uint32_t)(((t / kPullStages) - 1) & 1));
                const uint32_t bytes = (uint32_t)min((int64_t)tb, vbytes - t * tb);
                mbar_arrive_expect_tx(&full[stg], bytes * nact);
                for (int h = 0; h < P; ++h)
                    if (s_act[h])
                        tma_load(smem + ((size_t)stg * P + h) * tb, s_src[h] + t * tb, bytes, &full[stg]);
            }
        }
    } else {
        const int cid = threadIdx.x - 32;
        const int lane = threadIdx.x & 31;
        for (int64_t t = 0; t < ntiles; ++t) {
            const int stg = (int)(t % kPullStages);
            mbar_wait(&full[stg], (uint32_t)((t / kPullStages) & 1));
            const int64_t bytes = min((int64_t)tb, vbytes - t * tb);
            const int nvt = (int)(bytes / 16);
            const uint8_t* tile = smem + (size_t)stg * P * tb;
            for (int v = cid; v < nvt; v += nc) {
                float acc[V];
#pragma unroll
                for (int j = 0; j < V; ++j) acc[j] = 0.0f;
                for (int h = 0; h < P; ++h) {
                    if (!s_act[h]) continue;
                    const uint4 x = *reinterpret_cast<const uint4*>(tile + (size_t)h * tb + (size_t)v * 16);
                    const float sq = s_wt[h];
#pragma unroll
                    for (int j = 0; j < V; ++j)
                        acc[j] = rnd_dtype<T>(h == 0 ? __fmul_rn(sq, lane_f<T>(x, j)) : __fmaf_rn(sq, lane_f<T>(x, j), acc[j]));
                }
                uint4 y = pack_f<T>(acc);
                const size_t off = (size_t)t * tb + (size_t)v * 16;
                if (FUSE) y = sgd_v4<T>(*reinterpret_cast<const uint4*>(thp + off), y, A.nlr, A.wd);
                for (int q = 0; q < P; ++q) st_v4(s_dst[q] + off, y);
            }
            __syncwarp();
            if (lane == 0) mbar_arrive(&empty[stg]);   // this warp's smem reads of the stage are done
        }
        for (int64_t e = nv * V + cid; e < len; e += nc) {   // ragged tail: end of buffer
            float acc = 0.0f;
            for (int h = 0; h < P; ++h) {
                const int q = (r + h) % P;
                if (s_n[q] <= 0) continue;
                const T xv = reinterpret_cast<const T*>(s_bufs[q])[lo + e];
                acc = rnd_dtype<T>(h == 0 ? __fmul_rn(s_w[q], Vec<T>::to_f(xv)) : __fmaf_rn(s_w[q], Vec<T>::to_f(xv), acc));
            }
            if (FUSE) {
                const float tv = Vec<T>::to_f(reinterpret_cast<const T*>(thp)[e]);
                acc = __fmaf_rn(A.nlr, __fmaf_rn(A.wd, tv, acc), tv);
            }
            for (int q = 0; q < P; ++q) reinterpret_cast<T*>(s_dst[q])[e] = Vec<T>::from_f(acc);
        }
    }
    __syncthreads();
    if ((int)threadIdx.x < P - 1) {
        const int q = (r + 1 + (int)threadIdx.x) % P;
        st_release(&ts_flags_of(tab->win[q], tab, ch)->ag[r], base + 1, sys);
    }
    if (threadIdx.x < 32)
        if (!warp_wait_peers(mf->ag, base + 1, r, P, deadline, sys) && t0) {
            s_abort = 1;
            latch(tab, PR_ERR_PEER_TIMEOUT);
        }
    __syncthreads();
    if (FUSE && A.zero && !s_abort) {
        T* g = reinterpret_cast<T*>(rc.buf);
        for (int c = 0; c < P; ++c) {
            const int64_t a0 = (int64_t)c * cs + (int64_t)ch * sub;
            const int64_t a1 = min((int64_t)c * cs + min((int64_t)(ch + 1) * sub, cs), count);
            const int64_t zl = a1 > a0 ? a1 - a0 : 0;
            const int64_t zv = zl / V;
            for (int64_t v = threadIdx.x; v < zv; v += blockDim.x) st_v4(g + a0 + v * V, make_uint4(0, 0, 0, 0));
            for (int64_t e = zv * V + threadIdx.x; e < zl; e += blockDim.x) g[a0 + e] = Vec<T>::from_f(0.0f);
        }
    }
    if (t0) {
        if (!s_abort) st->ts_base = base + 1;
        if (ch == 0) tab->stamps[2] = (long long)gtimer();
    }
}

// =====================================================================================================
// LL ring (low-latency protocol for small buffers): the SAME ring schedule, order and per-hop rounding as
// ring_kernel — so the result is bit-identical — but every 16-byte line a rank pushes carries its own
// validity: two 64-bit elements, each (flag << 32 | 32 payload bits), flag = the call's handshake sequence.
// A 64-bit aligned element is single-copy atomic, so a receiver that sees the flag in an element also
// sees that element's payload: no release fence, no separate ready flag, no credit — the receiver polls
// the data itself.  Each phase h has its own region in the next rank's window (2P−2 regions), so a line is
// written once per call; the handshake (a barrier: every rank has finished the previous call) makes
// reusing the regions in the next call safe.  Half of every line is flag, so this trades bandwidth for
// latency: one store + one poll per hop instead of store → fence → flag → poll → TMA load.
// Each thread owns the same line positions in every phase, so a thread runs its own mini-ring and the
// CTA never synchronises between phases.
// =====================================================================================================
__device__ __forceinline__ void st_ll(void* p, uint32_t d0, uint32_t d1, uint32_t flag, bool sys) {
    st_line64(p, tag(flag, d0), tag(flag, d1), sys);
}
// one 32-bit payload word: 1 fp32 or 2 bf16 (the ring's Vec<T>::op on a quarter vector)
template <typename T> __device__ __forceinline__ uint32_t ll_op(int mode, float s, uint32_t g, uint32_t in);
template <> __device__ __forceinline__ uint32_t ll_op<float>(int mode, float s, uint32_t g, uint32_t in) {
    const float gv = __uint_as_float(g), iv = __uint_as_float(in);
    float r;
    if (mode == M_SCALE) r = __fmul_rn(s, gv);
    else if (mode == M_FMA) r = __fmaf_rn(s, gv, iv);
    else if (mode == M_COPY) r = iv;
    else r = 0.0f;
    return __float_as_uint(r);
}
template <> __device__ __forceinline__ uint32_t ll_op<__nv_bfloat16>(int mode, float s, uint32_t g, uint32_t in) {
    using B = Vec<__nv_bfloat16>;
    if (mode == M_COPY) return in;
    return B::pack(B::one(mode, s, B::lo(g), B::lo(in)), B::one(mode, s, B::hi(g), B::hi(in)));
}
// load / store the elements of one line (8 bytes = E elements); `nv` < E only on the buffer's last line
template <typename T> __device__ __forceinline__ void ld_line(const T* p, int nv, uint32_t& w0, uint32_t& w1) {
    constexpr int E = 8 / (int)sizeof(T);
    if (nv == E) {
        asm volatile("ld.global.v2.u32 {%0,%1}, [%2];" : "=r"(w0), "=r"(w1) : "l"(p));
        return;
    }
    uint16_t h[4] = {0, 0, 0, 0};
    const uint16_t* q = reinterpret_cast<const uint16_t*>(p);
    for (int k = 0; k < nv * (int)sizeof(T) / 2; ++k) h[k] = q[k];
    w0 = (uint32_t)h[0] | ((uint32_t)h[1] << 16);
    w1 = (uint32_t)h[2] | ((uint32_t)h[3] << 16);
}
template <typename T> __device__ __forceinline__ void st_line(T* p, int nv, uint32_t w0, uint32_t w1) {
    constexpr int E = 8 / (int)sizeof(T);
    if (nv == E) {
        asm volatile("st.global.v2.u32 [%0], {%1,%2};" ::"l"(p), "r"(w0), "r"(w1) : "memory");
        return;
    }
    const uint16_t h[4] = {(uint16_t)(w0 & 0xffffu), (uint16_t)(w0 >> 16), (uint16_t)(w1 & 0xffffu), (uint16_t)(w1 >> 16)};
    uint16_t* q = reinterpret_cast<uint16_t*>(p);
    for (int k = 0; k < nv * (int)sizeof(T) / 2; ++k) q[k] = h[k];
}

template <typename T>
__global__ void __launch_bounds__(512, 1) ring_ll_kernel(const __grid_constant__ LaunchArgs A) {
    __shared__ int s_err;
    __shared__ long long s_sumn;
    __shared__ unsigned s_flag;
    const RankCall& rc = A.calls[blockIdx.y];
    const DevTable* tab = rc.tab;
    const int ch = blockIdx.x;
    const int r = tab->rank, P = tab->P;
    const int next = (r + 1) % P;
    uint8_t* my = tab->win[r];
    ChanState* st = state_of(my, tab, ch);
    const bool t0 = threadIdx.x == 0;
    const bool sys = tab->sysscope != 0;
    unsigned long long deadline = ~0ull;
    if (threadIdx.x < 32) {                           // warp 0: the handshake = the barrier
        const unsigned long long start = gtimer();
        if (t0 && ch == 0) tab->stamps[0] = (long long)start;
        if (tab->watchdog_ns > 0) deadline = start + (unsigned long long)tab->watchdog_ns;
        const HsOut hs = handshake(A, rc, tab, st, ch, sys, deadline, nullptr, nullptr);
        if (t0) {
            s_err = hs.err;
            s_sumn = hs.sumn;
            s_flag = (unsigned)(st->seq & 0xffffffffull);   // this call's sequence: the line flag
            if (ch == 0) tab->stamps[1] = (long long)gtimer();
        }
    }
    __syncthreads();
    if (s_err) {
        if (t0) latch(tab, s_err);
        return;
    }
    if (tab->watchdog_ns > 0) deadline = gtimer() + (unsigned long long)tab->watchdog_ns;
    constexpr int V = Vec<T>::V;
    constexpr int E = 8 / (int)sizeof(T);                          // elements per line
    const int64_t count = A.count;
    const int64_t per = (count + P - 1) / P;
    const int64_t cs = (per + V - 1) / V * V;                      // chunk elements (as ring_kernel)
    const int64_t subp = (cs + tab->channels - 1) / tab->channels;
    const int64_t sub = (subp + V - 1) / V * V;                   // this channel's share of a chunk
    const float s = (float)((double)rc.n_local / (double)s_sumn);  // n_r/Σn: fp64 division, fp32 weight
    const bool act = rc.n_local > 0;
    const uint32_t flag = s_flag;
    T* buf = reinterpret_cast<T*>(rc.buf);
    uint8_t* my_ll = my + tab->off_ll + (size_t)ch * (size_t)(2 * P - 2) * (size_t)tab->ll_region_bytes;
    uint8_t* nx_ll = tab->win[next] + tab->off_ll + (size_t)ch * (size_t)(2 * P - 2) * (size_t)tab->ll_region_bytes;
    bool bad = false;
    for (int h = 0; h < 2 * P - 1 && !bad; ++h) {
        int kind, c;
        if (h == 0) { kind = K_FIRST; c = r; }
        else if (h <= P - 2) { kind = K_MID; c = (r - h + P) % P; }
        else if (h == P - 1) { kind = K_LAST; c = (r + 1) % P; }
        else if (h <= 2 * P - 3) { kind = K_AGMID; c = (r + 1 - (h - (P - 1)) + P) % P; }
        else { kind = K_AGLAST; c = (r + 2) % P; }
        const int64_t clo = (int64_t)c * cs;
        const int64_t chi = min(clo + cs, count);
        const int64_t lo = clo + (int64_t)ch * sub;
        const int64_t hi = min(clo + min((int64_t)(ch + 1) * sub, cs), chi);
        const int64_t len = hi > lo ? hi - lo : 0;
        const int64_t nl = (len + E - 1) / E;
        int mode;
        if (kind == K_FIRST) mode = act ? M_SCALE : M_ZERO;
        else if (kind == K_MID || kind == K_LAST) mode = act ? M_FMA : M_COPY;
        else mode = M_COPY;
        const bool needs_g = act && kind <= K_LAST;
        const uint8_t* in_reg = h > 0 ? my_ll + (size_t)(h - 1) * tab->ll_region_bytes : nullptr;
        uint8_t* out_reg = h < 2 * P - 2 ? nx_ll + (size_t)h * tab->ll_region_bytes : nullptr;
        for (int64_t j = threadIdx.x; j < nl; j += blockDim.x) {
            const int nv = (int)min((int64_t)E, len - j * E);
            T* p = buf + lo + j * E;
            uint32_t g0 = 0, g1 = 0, i0 = 0, i1 = 0;
            if (needs_g) ld_line<T>(p, nv, g0, g1);
            if (in_reg) {                                          // poll the line until both halves carry this call's flag
                unsigned long long a, b;
                for (;;) {
                    ld_line64(in_reg + (size_t)j * 16, a, b, sys);
                    if ((uint32_t)(a >> 32) == flag && (uint32_t)(b >> 32) == flag) break;
                    if (gtimer() > deadline) { bad = true; break; }
                }
                if (bad) break;
                i0 = (uint32_t)a;
                i1 = (uint32_t)b;
            }
            const uint32_t y0 = ll_op<T>(mode, s, g0, i0), y1 = ll_op<T>(mode, s, g1, i1);
            if (out_reg) st_ll(out_reg + (size_t)j * 16, y0, y1, flag, sys);
            if (kind >= K_LAST) st_line<T>(p, nv, y0, y1);          // reduced / gathered chunk -> own buffer
        }
    }
    if (bad) latch(tab, PR_ERR_PEER_TIMEOUT);
    __syncthreads();
    if (t0 && ch == 0) tab->stamps[2] = (long long)gtimer();
}

// =====================================================================================================
// One-shot LL (tiny buffers): ONE hop.  Every rank pushes its raw buffer, as LL lines, into a per-source
// region of every peer's window; every rank then reduces all P contributions itself — per element in the
// ring's order for that element's chunk c (c, c+1, …, c+P−1) with the ring's per-hop rounding, exactly as
// the two-shot reducer — so all ranks compute the ring's bits without a second hop.  Traffic per rank is
// (P−1)·2·Z bytes, so this is for buffers of a few tens of KiB, where the ring's 2P−2 hops are all latency.
// =====================================================================================================
template <typename T>
__global__ void __launch_bounds__(512, 1) oneshot_ll_kernel(const __grid_constant__ LaunchArgs A) {
    __shared__ int s_err;
    __shared__ long long s_n[PR_MAX_RANKS];
    __shared__ float s_w[PR_MAX_RANKS];
    __shared__ unsigned s_flag;
    const RankCall& rc = A.calls[blockIdx.y];
    const DevTable* tab = rc.tab;
    const int ch = blockIdx.x;
    const int r = tab->rank, P = tab->P;
    uint8_t* my = tab->win[r];
    ChanState* st = state_of(my, tab, ch);
    const bool t0 = threadIdx.x == 0;
    const bool sys = tab->sysscope != 0;
    unsigned long long deadline = ~0ull;
    if (threadIdx.x < 32) {
        const unsigned long long start = gtimer();
        if (t0 && ch == 0) tab->stamps[0] = (long long)start;
        if (tab->watchdog_ns > 0) deadline = start + (unsigned long long)tab->watchdog_ns;
        const HsOut hs = handshake(A, rc, tab, st, ch, sys, deadline, s_n, nullptr);
        __syncwarp();
        for (int q = (int)threadIdx.x; q < P; q += 32)
            s_w[q] = hs.sumn > 0 ? (float)((double)s_n[q] / (double)hs.sumn) : 0.0f;
        if (t0) {
            s_err = hs.err;
            s_flag = (unsigned)(st->seq & 0xffffffffull);
            if (ch == 0) tab->stamps[1] = (long long)gtimer();
        }
    }
    __syncthreads();
    if (s_err) {
        if (t0) latch(tab, s_err);
        return;
    }
    if (tab->watchdog_ns > 0) deadline = gtimer() + (unsigned long long)tab->watchdog_ns;
    constexpr int V = Vec<T>::V;
    constexpr int E = 8 / (int)sizeof(T);
    const int64_t count = A.count;
    const int64_t per = (count + P - 1) / P;
    const int64_t cs = (per + V - 1) / V * V;                      // the ring's chunk (sets the order)
    const int64_t subp = (count + tab->channels - 1) / tab->channels;
    const int64_t sub = (subp + V - 1) / V * V;                   // this channel's share of the buffer
    const int64_t lo = min((int64_t)ch * sub, count);
    const int64_t len = min(lo + sub, count) - lo;
    const int64_t nl = (len + E - 1) / E;
    const uint32_t flag = s_flag;
    T* buf = reinterpret_cast<T*>(rc.buf);
    const size_t reg = (size_t)tab->os_region_bytes;
    // push: my raw lines -> region [ch][src = r] of every peer
    for (int64_t j = threadIdx.x; j < nl; j += blockDim.x) {
        const int nv = (int)min((int64_t)E, len - j * E);
        uint32_t w0 = 0, w1 = 0;
        ld_line<T>(buf + lo + j * E, nv, w0, w1);
        for (int k = 1; k < P; ++k) {
            const int q = (r + k) % P;
            uint8_t* dst = tab->win[q] + tab->off_os + ((size_t)ch * P + r) * reg + (size_t)j * 16;
            st_ll(dst, w0, w1, flag, sys);
        }
    }
    // reduce: every element in its chunk's ring order, the ring's rounding (as twoshot_kernel)
    bool bad = false;
    for (int64_t j = threadIdx.x; j < nl && !bad; j += blockDim.x) {
        const int nv = (int)min((int64_t)E, len - j * E);
        const int64_t e0 = lo + j * E;
        const int c = (int)(e0 / cs);                              // a line never straddles a chunk
        float acc[E];
#pragma unroll
        for (int k = 0; k < E; ++k) acc[k] = 0.0f;
        for (int h = 0; h < P; ++h) {
            const int q = (c + h) % P;
            if (s_n[q] <= 0) continue;                             // n_q = 0 contributes nothing
            uint32_t w0, w1;
            if (q == r) {
                ld_line<T>(buf + e0, nv, w0, w1);
            } else {
                const uint8_t* src = my + tab->off_os + ((size_t)ch * P + q) * reg + (size_t)j * 16;
                unsigned long long a, b;
                for (;;) {
                    ld_line64(src, a, b, sys);
                    if ((uint32_t)(a >> 32) == flag && (uint32_t)(b >> 32) == flag) break;
                    if (gtimer() > deadline) { bad = true; break; }
                }
                if (bad) break;
                w0 = (uint32_t)a;
                w1 = (uint32_t)b;
            }
            const uint4 xv = make_uint4(w0, w1, 0u, 0u);
            const float sq = s_w[q];
#pragma unroll
            for (int k = 0; k < E; ++k)
                acc[k] = rnd_dtype<T>(h == 0 ? __fmul_rn(sq, lane_f<T>(xv, k)) : __fmaf_rn(sq, lane_f<T>(xv, k), acc[k]));
        }
        if (bad) break;
        uint32_t y0, y1;
        if (sizeof(T) == 4) {
            y0 = __float_as_uint(acc[0]);
            y1 = __float_as_uint(acc[1 % E]);
        } else {
            y0 = Vec<__nv_bfloat16>::pack(acc[0], acc[1 % E]);
            y1 = Vec<__nv_bfloat16>::pack(acc[2 % E], acc[3 % E]);
        }
        // own gradient line j was read above by this same thread (push and reduce): safe to overwrite
        st_line<T>(buf + e0, nv, y0, y1);
    }
    if (bad) latch(tab, PR_ERR_PEER_TIMEOUT);
    __syncthreads();
    if (t0 && ch == 0) tab->stamps[2] = (long long)gtimer();
}

// =====================================================================================================
// NVLS: the reduction done inside the NVSwitch.  The gradient buffer lives in an NVLS
// region (pr_comm_nvls_alloc: every rank's memory bound to one multicast object), so one
// multimem.ld_reduce through the multicast address returns Σ_q x_q[j] summed by the switch, and one
// multimem.st writes the result into every rank's memory.  The switch adds raw values, so the weights are
// applied first (phase A: x_r ← s_r·g_r in place, or 0 when n_r = 0 — a zero rank contributes exactly
// zero, never 0·g, DESIGN.md §3 #33); then (phase B) rank r reduces chunk r's channel share and
// multicasts it.  Per-channel barriers between the phases go through the windows' NvFlags (release /
// acquire at .sys scope), with fence.proxy.alias around them: phase A writes through the unicast alias,
// phase B reads and writes the same bytes through the multicast alias.  Reduction order inside the switch
// is unspecified: the result is checked against the fp64 weighted mean within tolerance, not bit for bit
// (DESIGN.md §3 #48).  fp32 only.
// =====================================================================================================
__device__ __forceinline__ void fence_proxy_alias() { asm volatile("fence.proxy.alias;" ::: "memory"); }
__device__ __forceinline__ float4 mm_ld_reduce_v4(const float* mc) {
    float4 r;
    asm volatile("multimem.ld_reduce.relaxed.sys.global.add.v4.f32 {%0,%1,%2,%3}, [%4];"
                 : "=f"(r.x), "=f"(r.y), "=f"(r.z), "=f"(r.w)
                 : "l"(mc)
                 : "memory");
    return r;
}
__device__ __forceinline__ void mm_st_v4(float* mc, float4 v) {
    asm volatile("multimem.st.relaxed.sys.global.v4.f32 [%0], {%1,%2,%3,%4};" ::"l"(mc), "f"(v.x), "f"(v.y), "f"(v.z),
                 "f"(v.w)
                 : "memory");
}
__device__ __forceinline__ float mm_ld_reduce_f32(const float* mc) {
    float r;
    asm volatile("multimem.ld_reduce.relaxed.sys.global.add.f32 %0, [%1];" : "=f"(r) : "l"(mc) : "memory");
    return r;
}
__device__ __forceinline__ void mm_st_f32(float* mc, float v) {
    asm volatile("multimem.st.relaxed.sys.global.f32 [%0], %1;" ::"l"(mc), "f"(v) : "memory");
}
__device__ __forceinline__ float ld_cg_f32(const float* p) {
    float v;
    asm volatile("ld.global.cg.f32 %0, [%1];" : "=f"(v) : "l"(p));
    return v;
}
__device__ __forceinline__ NvFlags* nv_of(uint8_t* w, const DevTable* t, int ch) {
    return reinterpret_cast<NvFlags*>(w + t->off_nv) + ch;
}

// EMU (local groups only, for tests): the switch operations are replaced by their definition over the
// ranks' unicast buffers — ld_reduce = Σ_q x_q[j] in rank order, st = a store into every rank's buffer —
// so the kernel's phases, geometry, barriers, tails and zero ranks are exercised on one GPU, where no
// multicast object can be created.
template <bool EMU>
__global__ void __launch_bounds__(512, 1) nvls_kernel(const __grid_constant__ LaunchArgs A) {
    __shared__ int s_err;
    __shared__ long long s_sumn;
    __shared__ unsigned long long s_seq;
    __shared__ uint8_t* s_bufs[PR_MAX_RANKS];
    const RankCall& rc = A.calls[blockIdx.y];
    const DevTable* tab = rc.tab;
    const int ch = blockIdx.x;
    const int r = tab->rank, P = tab->P;
    uint8_t* my = tab->win[r];
    ChanState* st = state_of(my, tab, ch);
    const bool t0 = threadIdx.x == 0;
    unsigned long long deadline = ~0ull;
    if (threadIdx.x < 32) {                           // warp 0: the handshake = the barrier
        const unsigned long long start = gtimer();
        if (t0 && ch == 0) tab->stamps[0] = (long long)start;
        if (tab->watchdog_ns > 0) deadline = start + (unsigned long long)tab->watchdog_ns;
        const HsOut hs = handshake(A, rc, tab, st, ch, tab->sysscope != 0, deadline, nullptr, EMU ? s_bufs : nullptr);
        if (t0) {
            s_err = hs.err ? hs.err : ((EMU && !hs.direct) ? PR_ERR_INVALID : 0);
            s_sumn = hs.sumn;
            s_seq = st->seq;
            if (ch == 0) tab->stamps[1] = (long long)gtimer();
        }
    }
    __syncthreads();
    if (s_err) {
        if (t0) latch(tab, s_err);
        return;
    }
    if (tab->watchdog_ns > 0) deadline = gtimer() + (unsigned long long)tab->watchdog_ns;
    const unsigned long long seq = s_seq;
    const int64_t count = A.count;
    const int64_t per = (count + P - 1) / P;
    const int64_t cs = (per + 3) / 4 * 4;                             // chunk (as the ring, 16 bytes)
    const int64_t subp = (cs + tab->channels - 1) / tab->channels;
    const int64_t sub = (subp + 3) / 4 * 4;
    const float s = (float)((double)rc.n_local / (double)s_sumn);    // n_r/Σn: fp64 division, fp32 weight
    const bool act = rc.n_local > 0;
    float* buf = reinterpret_cast<float*>(rc.buf);
    float* mcb = EMU ? nullptr : reinterpret_cast<float*>(tab->nv_mc + (reinterpret_cast<uint8_t*>(rc.buf) - tab->nv_uc));
    auto range = [&](int c, int64_t& lo, int64_t& len) {
        const int64_t clo = (int64_t)c * cs;
        const int64_t chi = min(clo + cs, count);
        lo = clo + (int64_t)ch * sub;
        const int64_t hi = min(clo + min((int64_t)(ch + 1) * sub, cs), chi);
        len = hi > lo ? hi - lo : 0;
    };
    auto barrier = [&](bool phase_b) -> bool {       // channel ch of every rank reached this point of call seq
        fence_proxy_alias();
        __threadfence_system();
        __syncthreads();
        bool ok = true;
        if (threadIdx.x < 32) {
            for (int q = (int)threadIdx.x; q < P; q += 32) {
                NvFlags* f = nv_of(tab->win[q], tab, ch);
                st_release(phase_b ? &f->b[r] : &f->a[r], seq, true);
            }
            NvFlags* mf = nv_of(my, tab, ch);
            for (int q = (int)threadIdx.x; q < P; q += 32)
                ok = ok && wait_ge(phase_b ? &mf->b[q] : &mf->a[q], seq, deadline, true);
            ok = __all_sync(0xffffffffu, ok);
            if (!ok && t0) latch(tab, PR_ERR_PEER_TIMEOUT);
            if (t0) s_err = ok ? 0 : PR_ERR_PEER_TIMEOUT;
        }
        __syncthreads();
        fence_proxy_alias();
        return s_err == 0;
    };
    // phase A: this channel's share of every chunk of the own buffer, weighted in place (unicast alias)
    for (int c = 0; c < P; ++c) {
        int64_t lo, len;
        range(c, lo, len);
        const int64_t nv = len / 4;
        float4* v4 = reinterpret_cast<float4*>(buf + lo);
        for (int64_t v = threadIdx.x; v < nv; v += blockDim.x) {
            float4 x = v4[v];
            x = act ? make_float4(__fmul_rn(s, x.x), __fmul_rn(s, x.y), __fmul_rn(s, x.z), __fmul_rn(s, x.w))
                    : make_float4(0.f, 0.f, 0.f, 0.f);
            v4[v] = x;
        }
        for (int64_t e = nv * 4 + threadIdx.x; e < len; e += blockDim.x) buf[lo + e] = act ? __fmul_rn(s, buf[lo + e]) : 0.f;
    }
    if (!barrier(false)) return;
    // phase B: chunk r's share: switch-reduced sum -> multicast into every rank's buffer
    {
        int64_t lo, len;
        range(r, lo, len);
        const int64_t nv = len / 4;
        if constexpr (EMU) {
            for (int64_t e = threadIdx.x; e < len; e += blockDim.x) {
                float acc = 0.0f;
                for (int q = 0; q < P; ++q) acc = __fadd_rn(acc, ld_cg_f32(reinterpret_cast<const float*>(s_bufs[q]) + lo + e));
                for (int q = 0; q < P; ++q) reinterpret_cast<float*>(s_bufs[q])[lo + e] = acc;
            }
        } else {
            for (int64_t v = threadIdx.x; v < nv; v += blockDim.x) {
                float* p = mcb + lo + 4 * v;
                mm_st_v4(p, mm_ld_reduce_v4(p));
            }
            for (int64_t e = nv * 4 + threadIdx.x; e < len; e += blockDim.x) {
                float* p = mcb + lo + e;
                mm_st_f32(p, mm_ld_reduce_f32(p));
            }
        }
    }
    barrier(true);                                    // every rank's multicast stores into my memory landed
    __syncthreads();
    if (t0 && ch == 0) tab->stamps[2] = (long long)gtimer();
}

__global__ void allgather_f64_kernel(const DevTable* tab, unsigned long long seq, double v, const double* vp,
                                     double* out) {
    if (threadIdx.x != 0) return;
    if (vp) v = *vp;                                   // asynchronous form: the value is on the device
    const bool sys = tab->sysscope != 0;
    const int r = tab->rank, P = tab->P;
    const int par = (int)(seq & 1ull);
    unsigned long long deadline = ~0ull;
    if (tab->watchdog_ns > 0) deadline = gtimer() + (unsigned long long)tab->watchdog_ns;
    for (int q = 0; q < P; ++q) {
        AgEntry* e = reinterpret_cast<AgEntry*>(tab->win[q] + tab->off_ag) + par * P + r;
        st_relaxed_s64(&e->v, __double_as_longlong(v), sys);
        st_release(&e->seq, seq, sys);
    }
    for (int q = 0; q < P; ++q) {
        AgEntry* e = reinterpret_cast<AgEntry*>(tab->win[r] + tab->off_ag) + par * P + q;
        if (!wait_ge(&e->seq, seq, deadline, sys)) { latch(tab, PR_ERR_PEER_TIMEOUT); return; }
        out[q] = __longlong_as_double(ld_relaxed_s64(&e->v, sys));
    }
}

}  // namespace

// =====================================================================================================
// Host side: communicator
// =====================================================================================================

namespace {
thread_local std::string g_cuda_err;

struct Reg {
    uint8_t* base = nullptr;
    size_t bytes = 0;
    bool owned = false;
    std::vector<uint8_t*> peer;   // mapped base of rank q's region (own = base); IPC-opened for q != rank
};

struct Hello {
    cudaIpcMemHandle_t handle;
    int32_t P, rank, device, channels, slots, threads, stages, tile_bytes, algo, ts_slots;
    int64_t ts_slot_bytes, ts_max_bytes, ll_max_bytes, os_max_bytes, min_slice_bytes;
    int64_t slot_bytes, window_bytes;
    uint64_t bytes;   // registration size
    unsigned char uuid[16];   // device identity: peers on another GPU need .sys-scope synchronisation
};
}  // namespace

void pr_internal_set_cuda_error(cudaError_t e, const char* what) {
    g_cuda_err = std::string(what) + ": " + cudaGetErrorString(e);
}
extern "C" const char* pr_last_cuda_error(void) { return g_cuda_err.c_str(); }

struct pr_comm {
    int32_t rank = 0, P = 1, device = 0;
    bool local = false;
    pr_comm_config cfg{};
    DevTable tab{};
    DevTable* d_tab = nullptr;
    uint8_t* win = nullptr;                 // own window
    std::vector<uint8_t*> opened;           // IPC-opened peer pointers (to close)
    int* h_status = nullptr;                // host-mapped status [0], stamps at +64 B
    long long* h_stamps = nullptr;
    double* h_ag = nullptr;                 // host-mapped allgather output
    std::vector<Reg> regs;
    pr_exchange_fn fn = nullptr;
    void* ctx = nullptr;
    unsigned long long ag_seq = 0;
    // NVLS region (pr_comm_nvls_alloc): multicast object, this rank's physical memory, the two mappings
    unsigned long long nv_mc_handle = 0, nv_mem_handle = 0;
    uintptr_t nv_uc = 0, nv_mc = 0;
    size_t nv_size = 0;
};

namespace {

pr_comm_config default_config() {
    pr_comm_config c;
    c.channels = 0;          // topology (resolve_config)
    c.slots = 8;
    c.threads = 512;
    c.flags = 0;
    c.slot_bytes = 0;        // topology
    c.watchdog_ns = 10ll * 1000 * 1000 * 1000;
    c.stages = 0;            // topology
    c.tile_bytes = 0;        // topology
    c.algo = PR_ALGO_RING;
    c.ts_slots = 2;
    c.ts_slot_bytes = 256 * 1024;   // tools/sweep_twoshot.py: P = 2, 16 MiB 92 -> 67 us vs 64 KiB; P = 8 neutral
    c.ts_max_bytes = 4ll << 20;     // measured crossover (co-located P = 4, 8): two-shot wins up to ~4 MiB
    c.ll_max_bytes = 256 * 1024;
    c.os_max_bytes = 64 * 1024;
    c.min_slice_bytes = 0;
    return c;
}

// Topology defaults for the fields a caller leaves 0 (channels, stages, tile_bytes, slot_bytes).  Same GPU
// (co-located ranks share the HBM and the SMs): 16 channels of 7 × 16 KiB stages, 256 KiB slots — the
// HBM-bound optimum of tools/sweep_ring.py.  Ranks on different GPUs: each rank has only its own
// channels' SMs, and a channel CTA moves ≈ 22-27 GB/s of bus bandwidth (its SM↔L2 traffic is ≈ 3.5
// bytes per bus byte; tools/sweep_cta.py, P = 2 co-located with HBM far from saturated), so 770 GB/s per
// direction needs > 30 of them: 32 channels of 7 × 16 KiB stages and 1 MiB slots (≈ 860 GB/s
// bus-equivalent per rank in that proxy).  Same GPU with fewer than 8 ranks: the 16-channel
// optimum was found at P = 8, where 128 CTAs saturate HBM; at P = 4 the same 16 channels per rank (64 CTAs)
// left the VGG-16 gradient CTA-bound (0.76 of HBM), so a co-located group keeps ≈ 128 CTAs in total:
// 128 / P channels per rank (at most 64) — which also keeps P > 8 groups co-resident (one CTA per SM).
void resolve_config(pr_comm_config& c, bool cross_gpu, int P) {
    // (P = 1 runs no ring: keep the window small)
    if (c.channels == 0) c.channels = cross_gpu ? 32 : (P <= 1 ? 16 : std::max(1, std::min(64, 128 / P)));
    // 7 × 2 × 16 KiB = 224 KiB of the 227 KB a CTA may use: the co-located P = 8 ResNet-18 ring 243 -> 234 µs
    // against 6 stages (profiles/round2_k3_stages7.jsonl)
    if (c.stages == 0) c.stages = 7;
    if (c.tile_bytes == 0) c.tile_bytes = 16384;
    if (c.slot_bytes == 0) c.slot_bytes = cross_gpu ? (1ll << 20) : (256 * 1024);
}

int check_config(const pr_comm_config& c) {
    if ((c.flags & ~(PR_COMM_FLAG_FORCE_STAGED | PR_COMM_FLAG_SYS_SCOPE | PR_COMM_FLAG_BULK_STORE |
                     PR_COMM_FLAG_L2_PREFETCH | PR_COMM_FLAG_PULL_TMA)) || c.channels < 1 || c.channels > 128 || c.slots < 2 || c.slots > 64 || c.threads < 32 || c.threads > 512 ||
        c.threads % 32 || c.slot_bytes < 256 || c.slot_bytes % 256 || c.slot_bytes > (64ll << 20) ||
        c.stages < 2 || c.stages > kMaxStages || c.tile_bytes < 256 || c.tile_bytes % 16 || c.tile_bytes > 32768 ||
        (int64_t)c.stages * 2 * c.tile_bytes > 224 * 1024 || c.algo < PR_ALGO_RING || c.algo > PR_ALGO_TWO_SHOT_PULL ||
        c.ll_max_bytes < 0 || c.ll_max_bytes > (64ll << 20) || c.os_max_bytes < 0 || c.os_max_bytes > (16ll << 20) ||
        c.min_slice_bytes < 0 || c.min_slice_bytes % 16 ||
        c.ts_slots < 2 || c.ts_slots > 16 || c.ts_slot_bytes < 256 || c.ts_slot_bytes % 256 ||
        c.ts_slot_bytes > (16ll << 20) || c.ts_max_bytes < 0)
        return PR_ERR_INVALID;
    return PR_OK;
}

// Bytes of one LL region: 2 × (one channel's share of a chunk of the largest LL buffer), for either dtype
// (chunk and share are rounded up to 16 bytes exactly as the kernels round them in elements).
// Bytes of one one-shot region: 2 × (one channel's share of the largest one-shot buffer).
uint64_t os_region_bytes(const pr_comm_config& c, int P) {
    if (P < 2 || c.os_max_bytes <= 0) return 0;
    return 2 * align_up(((uint64_t)c.os_max_bytes + c.channels - 1) / c.channels, 16);
}

uint64_t ll_region_bytes(const pr_comm_config& c, int P) {
    if (P < 2 || c.ll_max_bytes <= 0) return 0;
    const uint64_t per = ((uint64_t)c.ll_max_bytes + P - 1) / P;
    const uint64_t cs = align_up(per, 16);
    const uint64_t sub = align_up((cs + c.channels - 1) / c.channels, 16);
    return 2 * sub;
}

int alloc_common(pr_comm* c) {
    PR_CUDA_TRY(cudaSetDevice(c->device));
    DevTable& t = c->tab;
    t.rank = c->rank;
    t.P = c->P;
    t.channels = c->cfg.channels;
    t.slots = c->cfg.slots;
    t.slot_bytes = c->cfg.slot_bytes;
    t.watchdog_ns = c->cfg.watchdog_ns;
    t.stages = c->cfg.stages;
    t.tile_bytes = c->cfg.tile_bytes;
    t.ts_slots = c->cfg.ts_slots;
    t.ts_slot_bytes = c->cfg.ts_slot_bytes;
    t.ll_region_bytes = (int64_t)ll_region_bytes(c->cfg, c->P);
    t.min_slice_bytes = c->cfg.min_slice_bytes;
    t.os_region_bytes = (int64_t)os_region_bytes(c->cfg, c->P);
    layout(t);
    PR_CUDA_TRY(cudaMalloc((void**)&c->win, t.window_bytes));
    PR_CUDA_TRY(cudaMemset(c->win, 0, t.window_bytes));
    void* h = nullptr;
    PR_CUDA_TRY(cudaHostAlloc(&h, 4096, cudaHostAllocMapped | cudaHostAllocPortable));
    std::memset(h, 0, 4096);
    c->h_status = reinterpret_cast<int*>(h);
    c->h_stamps = reinterpret_cast<long long*>((char*)h + 64);
    c->h_ag = reinterpret_cast<double*>((char*)h + 256);
    void* d = nullptr;
    PR_CUDA_TRY(cudaHostGetDevicePointer(&d, h, 0));
    t.status = reinterpret_cast<volatile int*>(d);
    t.stamps = reinterpret_cast<volatile long long*>((char*)d + 64);
    PR_CUDA_TRY(cudaMalloc((void**)&c->d_tab, sizeof(DevTable)));
    return PR_OK;
}

int push_table(pr_comm* c) {
    PR_CUDA_TRY(cudaMemcpy(c->d_tab, &c->tab, sizeof(DevTable), cudaMemcpyHostToDevice));
    return PR_OK;
}

int exchange(pr_comm* c, const void* send, size_t len, void* recv) {
    if (!c->fn) return PR_ERR_INVALID;
    return c->fn(c->ctx, send, len, recv) == 0 ? PR_OK : PR_ERR_INVALID;
}

void nvls_release(pr_comm* c);

void free_comm(pr_comm* c) {
    if (!c) return;
    cudaSetDevice(c->device);
    nvls_release(c);
    for (auto& rg : c->regs) {
        for (int q = 0; q < (int)rg.peer.size(); ++q)
            if (!c->local && q != c->rank && rg.peer[q]) cudaIpcCloseMemHandle(rg.peer[q]);
        if (rg.owned && rg.base) cudaFree(rg.base);
    }
    for (auto* p : c->opened) cudaIpcCloseMemHandle(p);
    if (c->win) cudaFree(c->win);
    if (c->d_tab) cudaFree(c->d_tab);
    if (c->h_status) cudaFreeHost(c->h_status);
    delete c;
}

int find_reg(const pr_comm* c, const void* buf, size_t bytes, int32_t* id, int64_t* off) {
    if (c->cfg.flags & PR_COMM_FLAG_FORCE_STAGED) {
        *id = -1;
        *off = 0;
        return PR_OK;
    }
    if (c->local) {   // local group: every pointer is directly addressable; region 0 has base 0
        *id = 0;
        *off = (int64_t)(uintptr_t)buf;
        return PR_OK;
    }
    const uint8_t* b = reinterpret_cast<const uint8_t*>(buf);
    for (size_t i = 0; i < c->regs.size(); ++i) {
        const Reg& rg = c->regs[i];
        if (b >= rg.base && b + bytes <= rg.base + rg.bytes) {
            *id = (int32_t)i;
            *off = (int64_t)(b - rg.base);
            return PR_OK;
        }
    }
    *id = -1;
    *off = 0;
    return PR_OK;
}

size_t dtype_size(int32_t dt) { return dt == PR_DTYPE_F32 ? 4 : (dt == PR_DTYPE_BF16 ? 2 : 0); }

// The algorithm a call takes: a pure function of (config, count, dtype, P, registered).
// AUTO's two-shot limit grows with P: the ring pays 2P−2 flag round trips per call, the two-shot 2; at
// `.sys` scope and P = 8 the two-shot won up to 16 MiB (tools/ar_latency.py --sys), at P = 2 the ring wins
// from 4 MiB — so ts_max_bytes × 4 for P >= 8, × 2 for P >= 4 (kept for the pull two-shot, which beat
// the ring at every size co-located — unmeasured over NVLink).  Both two-shots read / write every peer's
// registered buffer, so AUTO takes one only for a registered buffer (and never under FORCE_STAGED); an
// explicit PR_ALGO_TWO_SHOT[_PULL] on an unregistered buffer latches PR_ERR_INVALID.
// `registered` is per rank: a job whose ranks differ there picks different kernels, and the handshake
// (which carries the algorithm) turns that into PR_ERR_LENGTH_MISMATCH on every rank.
int pick_algo(const pr_comm_config& cfg, int64_t count, int32_t dtype, int P, bool registered, bool in_nvls = false) {
    const int64_t bytes = count * (dtype == PR_DTYPE_F32 ? 4 : 2);
    // NVLS only when asked for, on an fp32 buffer inside the communicator's NVLS region; otherwise the ring
    if (cfg.algo == PR_ALGO_NVLS) return (in_nvls && dtype == PR_DTYPE_F32 && P > 1) ? PR_ALGO_NVLS : PR_ALGO_RING;
    if (cfg.algo == PR_ALGO_TWO_SHOT_PULL) return PR_ALGO_TWO_SHOT_PULL;   // explicit only (see the header)
    const int64_t ts_max = cfg.ts_max_bytes * (P >= 8 ? 4 : (P >= 4 ? 2 : 1));
    const bool direct_ok = registered && !(cfg.flags & PR_COMM_FLAG_FORCE_STAGED);
    if ((cfg.algo == PR_ALGO_ONESHOT || cfg.algo == PR_ALGO_AUTO) && bytes <= cfg.os_max_bytes) return PR_ALGO_ONESHOT;
    if ((cfg.algo == PR_ALGO_LL || cfg.algo == PR_ALGO_AUTO) && bytes <= cfg.ll_max_bytes) return PR_ALGO_LL;
    if (cfg.algo == PR_ALGO_TWO_SHOT) return PR_ALGO_TWO_SHOT;
    // AUTO's two-shot slot takes the pull variant (round 2): same bits, same registration requirement, and
    // faster than the push two-shot at every size / P / scope measured (profiles/round2_k3_pull_latency.txt)
    if (cfg.algo == PR_ALGO_AUTO && direct_ok && bytes <= ts_max) return PR_ALGO_TWO_SHOT_PULL;
    return PR_ALGO_RING;
}

// One launch of a K3 variant: grid (channels, ranks in this launch); cooperative for local groups (all P
// ranks' CTAs must be co-resident).
int launch_k3(void* fn, const LaunchArgs& a, int nranks, int channels, int block, size_t smem, cudaStream_t s,
              bool coop) {
    void* args[] = {(void*)&a};
    const dim3 grid((unsigned)channels, (unsigned)nranks), blk((unsigned)block);
    if (coop) {
        PR_CUDA_TRY(cudaLaunchCooperativeKernel(fn, grid, blk, args, smem, s));
    } else {
        PR_CUDA_TRY(cudaLaunchKernel(fn, grid, blk, args, smem, s));
    }
    return PR_OK;
}

int launch_ring(LaunchArgs& a, int nranks, int P, int device, const pr_comm_config& cfg, cudaStream_t s, bool coop,
                bool in_nvls = false) {
    const int32_t threads = cfg.threads, channels = cfg.channels;
    const bool f32 = a.dtype == PR_DTYPE_F32;
    bool registered = true;
    for (int r = 0; r < nranks; ++r) registered = registered && a.calls[r].reg_id >= 0;
    // the fused update (K7 inside K3) exists in the TMA ring and the pull two-shot (callers check fusable_algo)
    int algo = pick_algo(cfg, a.count, a.dtype, P, registered, in_nvls);
    if (a.fuse && algo != PR_ALGO_TWO_SHOT_PULL) algo = PR_ALGO_RING;
    a.algo = algo;
    switch (algo) {
        case PR_ALGO_NVLS:   // a local group (coop) runs the emulation: no multicast object on one device
            return launch_k3(coop ? (void*)nvls_kernel<true> : (void*)nvls_kernel<false>, a, nranks, channels, threads,
                             0, s, coop);
        case PR_ALGO_ONESHOT:
            return launch_k3(f32 ? (void*)oneshot_ll_kernel<float> : (void*)oneshot_ll_kernel<__nv_bfloat16>, a, nranks,
                             channels, threads, 0, s, coop);
        case PR_ALGO_LL:
            return launch_k3(f32 ? (void*)ring_ll_kernel<float> : (void*)ring_ll_kernel<__nv_bfloat16>, a, nranks,
                             channels, threads, 0, s, coop);
        case PR_ALGO_TWO_SHOT:
            return launch_k3(f32 ? (void*)twoshot_kernel<float> : (void*)twoshot_kernel<__nv_bfloat16>, a, nranks,
                             channels, threads, 0, s, coop);
        case PR_ALGO_TWO_SHOT_PULL:
            if (cfg.flags & PR_COMM_FLAG_PULL_TMA) {
                void* fn = a.fuse ? (void*)twoshot_pull_tma_kernel<float, true>
                                  : f32 ? (void*)twoshot_pull_tma_kernel<float, false>
                                        : (void*)twoshot_pull_tma_kernel<__nv_bfloat16, false>;
                const size_t smem = (size_t)kPullStages * P * pull_tile_bytes(P);
                static std::mutex mu;
                static bool attr_set[PR_MAX_DEVICES][3];
                const int di = a.fuse ? 2 : (f32 ? 0 : 1);
                if (device < 0 || device >= PR_MAX_DEVICES) return PR_ERR_INVALID;
                {
                    std::lock_guard<std::mutex> lk(mu);
                    if (!attr_set[device][di]) {
                        PR_CUDA_TRY(cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, 196608));
                        attr_set[device][di] = true;
                    }
                }
                return launch_k3(fn, a, nranks, channels, threads + 32, smem, s, coop);
            }
            return launch_k3(a.fuse ? (void*)twoshot_pull_kernel<float, true>
                                    : f32 ? (void*)twoshot_pull_kernel<float, false>
                                          : (void*)twoshot_pull_kernel<__nv_bfloat16, false>,
                             a, nranks, channels, threads, 0, s, coop);
        default: break;
    }
    const bool bulk = (cfg.flags & PR_COMM_FLAG_BULK_STORE) != 0;
    void* fn = bulk ? (a.fuse ? (void*)ring_kernel<float, true, true>
                              : f32 ? (void*)ring_kernel<float, false, true> : (void*)ring_kernel<__nv_bfloat16, false, true>)
                    : (a.fuse ? (void*)ring_kernel<float, true, false>
                              : f32 ? (void*)ring_kernel<float, false, false> : (void*)ring_kernel<__nv_bfloat16, false, false>);
    const size_t smem = (size_t)cfg.stages * 2 * cfg.tile_bytes;
    // the dynamic-smem opt-in is a per-device function attribute: cached per (device, instantiation)
    static std::mutex mu;
    static size_t attr_set[PR_MAX_DEVICES][6];
    const int di = (a.fuse ? 2 : (f32 ? 0 : 1)) + (bulk ? 3 : 0);
    if (device < 0 || device >= PR_MAX_DEVICES) return PR_ERR_INVALID;
    {
        std::lock_guard<std::mutex> lk(mu);
        if (attr_set[device][di] < smem) {
            PR_CUDA_TRY(cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
            attr_set[device][di] = smem;
        }
    }
    // producer warp + signal warp + `threads` consumer threads per channel CTA
    return launch_k3(fn, a, nranks, channels, threads + 64, smem, s, coop);
}

// ---- NVLS region: driver entry points fetched at run time (no link-time libcuda dependency: the library
// must load on a GPU-less host) ---------------------------------------------------------------------------
struct DrvApi {
    bool ok = false;
    CUresult (*devGet)(CUdevice*, int);
    CUresult (*devAttr)(int*, CUdevice_attribute, CUdevice);
    CUresult (*mcGran)(size_t*, const CUmulticastObjectProp*, CUmulticastGranularity_flags);
    CUresult (*mcCreate)(CUmemGenericAllocationHandle*, const CUmulticastObjectProp*);
    CUresult (*mcAdd)(CUmemGenericAllocationHandle, CUdevice);
    CUresult (*mcBind)(CUmemGenericAllocationHandle, size_t, CUmemGenericAllocationHandle, size_t, size_t,
                       unsigned long long);
    CUresult (*mcUnbind)(CUmemGenericAllocationHandle, CUdevice, size_t, size_t);
    CUresult (*memCreate)(CUmemGenericAllocationHandle*, size_t, const CUmemAllocationProp*, unsigned long long);
    CUresult (*memRelease)(CUmemGenericAllocationHandle);
    CUresult (*addrReserve)(CUdeviceptr*, size_t, size_t, CUdeviceptr, unsigned long long);
    CUresult (*addrFree)(CUdeviceptr, size_t);
    CUresult (*memMap)(CUdeviceptr, size_t, size_t, CUmemGenericAllocationHandle, unsigned long long);
    CUresult (*memUnmap)(CUdeviceptr, size_t);
    CUresult (*setAccess)(CUdeviceptr, size_t, const CUmemAccessDesc*, size_t);
    CUresult (*exportH)(void*, CUmemGenericAllocationHandle, CUmemAllocationHandleType, unsigned long long);
    CUresult (*importH)(CUmemGenericAllocationHandle*, void*, CUmemAllocationHandleType);
};

const DrvApi& drv() {
    static DrvApi d;
    static std::once_flag once;
    std::call_once(once, [] {
        auto get = [](const char* name, void** fp) {
            cudaDriverEntryPointQueryResult q;
            return cudaGetDriverEntryPoint(name, fp, cudaEnableDefault, &q) == cudaSuccess &&
                   q == cudaDriverEntryPointSuccess && *fp;
        };
        bool ok = true;
        ok = ok && get("cuDeviceGet", (void**)&d.devGet);
        ok = ok && get("cuDeviceGetAttribute", (void**)&d.devAttr);
        ok = ok && get("cuMulticastGetGranularity", (void**)&d.mcGran);
        ok = ok && get("cuMulticastCreate", (void**)&d.mcCreate);
        ok = ok && get("cuMulticastAddDevice", (void**)&d.mcAdd);
        ok = ok && get("cuMulticastBindMem", (void**)&d.mcBind);
        ok = ok && get("cuMulticastUnbind", (void**)&d.mcUnbind);
        ok = ok && get("cuMemCreate", (void**)&d.memCreate);
        ok = ok && get("cuMemRelease", (void**)&d.memRelease);
        ok = ok && get("cuMemAddressReserve", (void**)&d.addrReserve);
        ok = ok && get("cuMemAddressFree", (void**)&d.addrFree);
        ok = ok && get("cuMemMap", (void**)&d.memMap);
        ok = ok && get("cuMemUnmap", (void**)&d.memUnmap);
        ok = ok && get("cuMemSetAccess", (void**)&d.setAccess);
        ok = ok && get("cuMemExportToShareableHandle", (void**)&d.exportH);
        ok = ok && get("cuMemImportFromShareableHandle", (void**)&d.importH);
        d.ok = ok;
        cudaGetLastError();
    });
    return d;
}

void nvls_release(pr_comm* c) {
    if (!c->nv_size) return;
    const DrvApi& d = drv();
    CUdevice dev = 0;
    d.devGet(&dev, c->device);
    if (c->nv_mc) { d.memUnmap((CUdeviceptr)c->nv_mc, c->nv_size); d.addrFree((CUdeviceptr)c->nv_mc, c->nv_size); }
    if (c->nv_uc) { d.memUnmap((CUdeviceptr)c->nv_uc, c->nv_size); d.addrFree((CUdeviceptr)c->nv_uc, c->nv_size); }
    if (c->nv_mc_handle && c->nv_mem_handle) d.mcUnbind((CUmemGenericAllocationHandle)c->nv_mc_handle, dev, 0, c->nv_size);
    if (c->nv_mem_handle) d.memRelease((CUmemGenericAllocationHandle)c->nv_mem_handle);
    if (c->nv_mc_handle) d.memRelease((CUmemGenericAllocationHandle)c->nv_mc_handle);
    c->nv_uc = c->nv_mc = 0;
    c->nv_mc_handle = c->nv_mem_handle = 0;
    c->nv_size = 0;
    c->tab.nv_uc = c->tab.nv_mc = nullptr;
    c->tab.nv_bytes = 0;
}

struct NvHello {
    int32_t err;        // this rank failed a step so far (every rank fails together)
    int32_t kind;       // rank 0's export: 1 fabric handle, 2 POSIX file descriptor (pid + fd)
    int32_t pid, fd;
    unsigned char fabric[64];
};

// One collective step of the setup: every rank contributes its error flag (and rank 0 its handle);
// returns the first error of any rank.
int nv_sync(pr_comm* c, NvHello& me, std::vector<NvHello>& all) {
    all.assign(c->P, NvHello{});
    if (exchange(c, &me, sizeof(NvHello), all.data())) return PR_ERR_INVALID;
    for (const NvHello& h : all)
        if (h.err) return h.err;
    return PR_OK;
}

}  // namespace

// NVLS region: see include/propring.h.  Collective.
extern "C" int pr_comm_nvls_alloc(pr_comm* c, size_t bytes, void** d_ptr) {
    if (!c || !d_ptr || bytes == 0 || c->local || c->P < 2 || c->nv_size) return PR_ERR_INVALID;
    PR_CUDA_TRY(cudaSetDevice(c->device));
    const DrvApi& d = drv();
    NvHello me{};
    std::vector<NvHello> all;
    CUdevice dev = 0;
    int mc_ok = 0;
    if (!d.ok || d.devGet(&dev, c->device) != CUDA_SUCCESS ||
        d.devAttr(&mc_ok, CU_DEVICE_ATTRIBUTE_MULTICAST_SUPPORTED, dev) != CUDA_SUCCESS || !mc_ok)
        me.err = PR_ERR_UNSUPPORTED;
    CUmulticastObjectProp mp;
    std::memset(&mp, 0, sizeof(mp));
    mp.numDevices = (unsigned)c->P;
    mp.size = bytes;
    size_t gran = 0;
    if (!me.err) {
        mp.handleTypes = CU_MEM_HANDLE_TYPE_POSIX_FILE_DESCRIPTOR;
        if (d.mcGran(&gran, &mp, CU_MULTICAST_GRANULARITY_RECOMMENDED) != CUDA_SUCCESS || !gran) me.err = PR_ERR_UNSUPPORTED;
    }
    const size_t size = gran ? (bytes + gran - 1) / gran * gran : 0;
    mp.size = size;
    CUmemGenericAllocationHandle mc = 0, mem = 0;
    CUmemAllocationHandleType htype = CU_MEM_HANDLE_TYPE_POSIX_FILE_DESCRIPTOR;
    // step 1: rank 0 creates the multicast object and exports it (fabric handle as bytes if the platform
    // has one, else a file descriptor the peers duplicate with pidfd_getfd)
    if (c->rank == 0 && !me.err) {
        mp.handleTypes = (CUmemAllocationHandleType)(CU_MEM_HANDLE_TYPE_FABRIC | CU_MEM_HANDLE_TYPE_POSIX_FILE_DESCRIPTOR);
        if (d.mcCreate(&mc, &mp) == CUDA_SUCCESS &&
            d.exportH(me.fabric, mc, CU_MEM_HANDLE_TYPE_FABRIC, 0) == CUDA_SUCCESS) {
            me.kind = 1;
        } else {
            if (mc) d.memRelease(mc);
            mc = 0;
            mp.handleTypes = CU_MEM_HANDLE_TYPE_POSIX_FILE_DESCRIPTOR;
            int fd = -1;
            if (d.mcCreate(&mc, &mp) == CUDA_SUCCESS &&
                d.exportH(&fd, mc, CU_MEM_HANDLE_TYPE_POSIX_FILE_DESCRIPTOR, 0) == CUDA_SUCCESS) {
                me.kind = 2;
                me.pid = (int32_t)getpid();
                me.fd = fd;
            } else {
                me.err = PR_ERR_UNSUPPORTED;
            }
        }
    }
    int rc = nv_sync(c, me, all);
    // step 2: the peers import it
    if (!rc && c->rank != 0) {
        const NvHello& h0 = all[0];
        if (h0.kind == 1) {
            htype = CU_MEM_HANDLE_TYPE_FABRIC;
            if (d.importH(&mc, (void*)h0.fabric, CU_MEM_HANDLE_TYPE_FABRIC) != CUDA_SUCCESS) me.err = PR_ERR_UNSUPPORTED;
        } else {
            const int pfd = (int)syscall(SYS_pidfd_open, h0.pid, 0);
            const int fd = pfd >= 0 ? (int)syscall(SYS_pidfd_getfd, pfd, h0.fd, 0) : -1;
            if (fd < 0 || d.importH(&mc, (void*)(uintptr_t)fd, CU_MEM_HANDLE_TYPE_POSIX_FILE_DESCRIPTOR) != CUDA_SUCCESS)
                me.err = PR_ERR_UNSUPPORTED;
            if (fd >= 0) close(fd);
            if (pfd >= 0) close(pfd);
        }
    } else if (!rc && c->rank == 0) {
        htype = all[0].kind == 1 ? CU_MEM_HANDLE_TYPE_FABRIC : CU_MEM_HANDLE_TYPE_POSIX_FILE_DESCRIPTOR;
    }
    if (!rc) rc = nv_sync(c, me, all);
    if (c->rank == 0 && me.kind == 2 && me.fd >= 0) close(me.fd);   // every peer has duplicated it
    // step 3: every rank adds its device to the team — all of them before anyone binds memory (a multicast
    // object accepts bindings only once its team is complete) — then allocates and binds its memory and
    // maps both aliases
    if (!rc) {
        if (d.mcAdd(mc, dev) != CUDA_SUCCESS) me.err = PR_ERR_UNSUPPORTED;
        rc = nv_sync(c, me, all);
    }
    CUdeviceptr uc = 0, mcp = 0;
    if (!rc) {
        CUmemAllocationProp ap;
        std::memset(&ap, 0, sizeof(ap));
        ap.type = CU_MEM_ALLOCATION_TYPE_PINNED;
        ap.location.type = CU_MEM_LOCATION_TYPE_DEVICE;
        ap.location.id = c->device;
        ap.requestedHandleTypes = htype;
        CUmemAccessDesc acc;
        acc.location.type = CU_MEM_LOCATION_TYPE_DEVICE;
        acc.location.id = c->device;
        acc.flags = CU_MEM_ACCESS_FLAGS_PROT_READWRITE;
        if (d.memCreate(&mem, size, &ap, 0) != CUDA_SUCCESS ||
            d.mcBind(mc, 0, mem, 0, size, 0) != CUDA_SUCCESS || d.addrReserve(&uc, size, gran, 0, 0) != CUDA_SUCCESS ||
            d.memMap(uc, size, 0, mem, 0) != CUDA_SUCCESS || d.setAccess(uc, size, &acc, 1) != CUDA_SUCCESS ||
            d.addrReserve(&mcp, size, gran, 0, 0) != CUDA_SUCCESS || d.memMap(mcp, size, 0, mc, 0) != CUDA_SUCCESS ||
            d.setAccess(mcp, size, &acc, 1) != CUDA_SUCCESS || cudaMemset((void*)uc, 0, size) != cudaSuccess ||
            cudaDeviceSynchronize() != cudaSuccess)
            me.err = PR_ERR_UNSUPPORTED;
        cudaGetLastError();
        rc = nv_sync(c, me, all);
    }
    c->nv_mc_handle = mc;
    c->nv_mem_handle = mem;
    c->nv_uc = (uintptr_t)uc;
    c->nv_mc = (uintptr_t)mcp;
    c->nv_size = size;
    if (!rc) {
        c->tab.nv_uc = (uint8_t*)uc;
        c->tab.nv_mc = (uint8_t*)mcp;
        c->tab.nv_bytes = (int64_t)size;
        rc = push_table(c);
    }
    if (rc) {
        nvls_release(c);
        return rc;
    }
    *d_ptr = (void*)uc;
    return PR_OK;
}

extern "C" int pr_comm_init(pr_comm** out, int32_t rank, int32_t P, int32_t device, pr_exchange_fn fn, void* ctx,
                            const pr_comm_config* cfg) {
    if (!out || !fn || P < 1 || P > PR_MAX_RANKS || rank < 0 || rank >= P || device < 0) return PR_ERR_INVALID;
    pr_comm* c = new (std::nothrow) pr_comm();
    if (!c) return PR_ERR_INTERNAL;
    c->rank = rank; c->P = P; c->device = device; c->fn = fn; c->ctx = ctx;
    c->cfg = cfg ? *cfg : default_config();
    // probe exchange: are the ranks on different GPUs?  (decides the topology defaults of fields left 0)
    struct Probe {
        unsigned char uuid[16];
    } mine{}, *probes = nullptr;
    {
        cudaDeviceProp prop;
        if (cudaGetDeviceProperties(&prop, device) == cudaSuccess) std::memcpy(mine.uuid, &prop.uuid, 16);
    }
    std::vector<Probe> all_probe(P);
    probes = all_probe.data();
    if (int xrc = exchange(c, &mine, sizeof(Probe), probes)) { free_comm(c); return xrc; }
    bool cross = false;
    for (int q = 0; q < P; ++q) cross = cross || std::memcmp(probes[q].uuid, mine.uuid, 16) != 0;
    resolve_config(c->cfg, cross, P);
    int rc = check_config(c->cfg);
    if (!rc) rc = alloc_common(c);
    Hello me;
    std::memset(&me, 0, sizeof(me));
    if (!rc) {
        cudaError_t e = cudaIpcGetMemHandle(&me.handle, c->win);
        if (e != cudaSuccess) { pr_internal_set_cuda_error(e, "cudaIpcGetMemHandle(window)"); rc = PR_ERR_CUDA; }
    }
    me.P = P; me.rank = rank; me.device = device; me.channels = c->cfg.channels; me.slots = c->cfg.slots;
    me.threads = c->cfg.threads; me.slot_bytes = c->cfg.slot_bytes; me.window_bytes = (int64_t)c->tab.window_bytes;
    me.stages = c->cfg.stages; me.tile_bytes = c->cfg.tile_bytes;
    me.algo = c->cfg.algo; me.ts_slots = c->cfg.ts_slots; me.ts_slot_bytes = c->cfg.ts_slot_bytes;
    me.ts_max_bytes = c->cfg.ts_max_bytes;
    me.ll_max_bytes = c->cfg.ll_max_bytes;
    me.os_max_bytes = c->cfg.os_max_bytes;
    me.min_slice_bytes = c->cfg.min_slice_bytes;
    {
        cudaDeviceProp prop;
        if (cudaGetDeviceProperties(&prop, device) == cudaSuccess) std::memcpy(me.uuid, &prop.uuid, 16);
    }
    me.bytes = rc ? 1 : 0;   // error flag travels with the hello so every rank fails together
    std::vector<Hello> all(P);
    int xrc = exchange(c, &me, sizeof(Hello), all.data());
    if (xrc) { free_comm(c); return xrc; }
    for (int q = 0; q < P; ++q) {
        const Hello& h = all[q];
        if (h.bytes) rc = rc ? rc : PR_ERR_CUDA;
        if (h.P != P || h.rank != q || h.channels != me.channels || h.slots != me.slots || h.slot_bytes != me.slot_bytes ||
            h.threads != me.threads || h.stages != me.stages || h.tile_bytes != me.tile_bytes || h.algo != me.algo ||
            h.ts_slots != me.ts_slots || h.ts_slot_bytes != me.ts_slot_bytes || h.ts_max_bytes != me.ts_max_bytes ||
            h.ll_max_bytes != me.ll_max_bytes || h.os_max_bytes != me.os_max_bytes ||
            h.min_slice_bytes != me.min_slice_bytes)
            rc = rc ? rc : PR_ERR_INVALID;
    }
    if (rc) { free_comm(c); return rc; }
    for (int q = 0; q < P; ++q) {
        if (q == rank) { c->tab.win[q] = c->win; continue; }
        void* p = nullptr;
        cudaError_t e = cudaIpcOpenMemHandle(&p, all[q].handle, cudaIpcMemLazyEnablePeerAccess);
        if (e != cudaSuccess) {
            pr_internal_set_cuda_error(e, "cudaIpcOpenMemHandle(window)");
            rc = (e == cudaErrorPeerAccessUnsupported || e == cudaErrorInvalidDevice) ? PR_ERR_NO_P2P : PR_ERR_CUDA;
            break;
        }
        c->opened.push_back((uint8_t*)p);
        c->tab.win[q] = (uint8_t*)p;
    }
    c->tab.sysscope = (c->cfg.flags & PR_COMM_FLAG_SYS_SCOPE) ? 1 : 0;
    c->tab.l2pf = (c->cfg.flags & PR_COMM_FLAG_L2_PREFETCH) ? 1 : 0;
    for (int q = 0; q < P; ++q)
        if (std::memcmp(all[q].uuid, me.uuid, 16) != 0) c->tab.sysscope = 1;   // a peer on another GPU
    if (!rc) rc = push_table(c);
    // barrier: nobody signals into a window before every rank has mapped every window
    int flag = rc ? 1 : 0;
    std::vector<int> flags(P);
    if (exchange(c, &flag, sizeof(int), flags.data())) rc = rc ? rc : PR_ERR_INVALID;
    for (int q = 0; q < P; ++q) if (flags[q]) rc = rc ? rc : PR_ERR_CUDA;
    if (rc) { free_comm(c); return rc; }
    *out = c;
    return PR_OK;
}

extern "C" int pr_comm_init_local(pr_comm** out, int32_t P, int32_t device, const pr_comm_config* cfg) {
    if (!out || P < 1 || P > PR_MAX_RANKS || device < 0) return PR_ERR_INVALID;
    pr_comm_config cf = cfg ? *cfg : default_config();
    resolve_config(cf, false, P);                                 // one device
    if (int rc = check_config(cf)) return rc;
    std::vector<pr_comm*> cs(P, nullptr);
    int rc = PR_OK;
    for (int r = 0; r < P && !rc; ++r) {
        cs[r] = new (std::nothrow) pr_comm();
        if (!cs[r]) { rc = PR_ERR_INTERNAL; break; }
        cs[r]->rank = r; cs[r]->P = P; cs[r]->device = device; cs[r]->local = true; cs[r]->cfg = cf;
        rc = alloc_common(cs[r]);
    }
    if (!rc) {
        for (int r = 0; r < P; ++r) {
            for (int q = 0; q < P; ++q) {
                cs[r]->tab.win[q] = cs[q]->win;
                cs[r]->tab.reg[0][q] = nullptr;   // local region 0: the whole address space, base 0
            }
            cs[r]->tab.sysscope = (cf.flags & PR_COMM_FLAG_SYS_SCOPE) ? 1 : 0;   // one device: .gpu suffices
            cs[r]->tab.l2pf = (cf.flags & PR_COMM_FLAG_L2_PREFETCH) ? 1 : 0;
            if ((rc = push_table(cs[r]))) break;
        }
    }
    if (rc) {
        for (auto* c : cs) free_comm(c);
        return rc;
    }
    for (int r = 0; r < P; ++r) out[r] = cs[r];
    return PR_OK;
}

extern "C" int pr_comm_register(pr_comm* c, void* d_buf, size_t bytes) {
    if (!c || !d_buf || bytes == 0) return PR_ERR_INVALID;
    if (c->local) return PR_OK;
    if ((int)c->regs.size() >= PR_MAX_REGS) return PR_ERR_CAPACITY;
    PR_CUDA_TRY(cudaSetDevice(c->device));
    Hello me;
    std::memset(&me, 0, sizeof(me));
    int rc = PR_OK;
    cudaError_t e = cudaIpcGetMemHandle(&me.handle, d_buf);
    if (e != cudaSuccess) { pr_internal_set_cuda_error(e, "cudaIpcGetMemHandle(register)"); rc = PR_ERR_CUDA; }
    me.rank = c->rank;
    me.bytes = bytes;
    me.P = rc;   // error travels with the message
    std::vector<Hello> all(c->P);
    if (exchange(c, &me, sizeof(Hello), all.data())) return PR_ERR_INVALID;
    for (auto& h : all) if (h.P) rc = rc ? rc : h.P;
    if (rc) return rc;
    Reg rg;
    rg.base = (uint8_t*)d_buf;
    rg.bytes = bytes;
    rg.peer.assign(c->P, nullptr);
    for (int q = 0; q < c->P && !rc; ++q) {
        if (q == c->rank) { rg.peer[q] = rg.base; continue; }
        void* p = nullptr;
        cudaError_t e2 = cudaIpcOpenMemHandle(&p, all[q].handle, cudaIpcMemLazyEnablePeerAccess);
        if (e2 != cudaSuccess) { pr_internal_set_cuda_error(e2, "cudaIpcOpenMemHandle(register)"); rc = PR_ERR_CUDA; break; }
        rg.peer[q] = (uint8_t*)p;
    }
    // collective outcome: the registration exists on every rank or on none (region ids must agree across
    // ranks — a peer's handshake names its region by id), so nothing is recorded before all ranks succeeded
    int flag = rc ? 1 : 0;
    std::vector<int> flags(c->P);
    if (exchange(c, &flag, sizeof(int), flags.data())) rc = rc ? rc : PR_ERR_INVALID;
    for (int f : flags) if (f) rc = rc ? rc : PR_ERR_CUDA;
    const int id = (int)c->regs.size();
    if (!rc) {
        for (int q = 0; q < c->P; ++q) c->tab.reg[id][q] = rg.peer[q];
        rc = push_table(c);
        if (rc) for (int q = 0; q < c->P; ++q) c->tab.reg[id][q] = nullptr;
    }
    if (rc) {   // undo: close what this rank opened; the region is not recorded
        for (int q = 0; q < c->P; ++q)
            if (q != c->rank && rg.peer[q]) cudaIpcCloseMemHandle(rg.peer[q]);
        return rc;
    }
    c->regs.push_back(rg);
    return PR_OK;
}

extern "C" int pr_comm_alloc(pr_comm* c, size_t bytes, void** d_ptr) {
    if (!c || !d_ptr || bytes == 0) return PR_ERR_INVALID;
    PR_CUDA_TRY(cudaSetDevice(c->device));
    void* p = nullptr;
    PR_CUDA_TRY(cudaMalloc(&p, bytes));
    if (cudaError_t e = cudaMemset(p, 0, bytes)) {
        pr_internal_set_cuda_error(e, "cudaMemset(pr_comm_alloc)");
        cudaFree(p);
        return PR_ERR_CUDA;
    }
    if (c->local) {
        Reg rg;
        rg.base = (uint8_t*)p; rg.bytes = bytes; rg.owned = true;
        c->regs.push_back(rg);
        *d_ptr = p;
        return PR_OK;
    }
    int rc = pr_comm_register(c, p, bytes);
    if (rc) { cudaFree(p); return rc; }
    c->regs.back().owned = true;
    *d_ptr = p;
    return PR_OK;
}

extern "C" int pr_weighted_allreduce(pr_comm* c, void* d_buf, int64_t count, int32_t dt, int64_t n_local,
                                     void* stream) {
    if (!c || count < 0 || n_local < 0 || !dtype_size(dt) || (count > 0 && !d_buf)) return PR_ERR_INVALID;
    if (((uintptr_t)d_buf & 15)) return PR_ERR_ALIGN;
    if (int st = *(volatile int*)c->h_status) return st;
    if (c->P == 1) return n_local > 0 ? PR_OK : PR_ERR_ZERO_SAMPLES;
    LaunchArgs a;
    std::memset(&a, 0, sizeof(a));
    a.count = count;
    a.dtype = dt;
    a.nranks = 1;
    a.calls[0].tab = c->d_tab;
    a.calls[0].buf = d_buf;
    a.calls[0].n_local = n_local;
    find_reg(c, d_buf, (size_t)count * dtype_size(dt), &a.calls[0].reg_id, &a.calls[0].reg_off);
    const uintptr_t b = (uintptr_t)d_buf;
    const bool in_nvls = c->nv_uc && b >= c->nv_uc && b + (size_t)count * dtype_size(dt) <= c->nv_uc + c->nv_size;
    PR_CUDA_TRY(cudaSetDevice(c->device));
    return launch_ring(a, 1, c->P, c->device, c->cfg, (cudaStream_t)stream, false, in_nvls);
}

extern "C" int pr_weighted_allreduce_local(pr_comm* const* comms, void* const* d_bufs, int64_t count, int32_t dt,
                                           const int64_t* n_local, void* stream) {
    if (!comms || !d_bufs || !n_local || count < 0 || !dtype_size(dt)) return PR_ERR_INVALID;
    const pr_comm* c0 = comms[0];
    if (!c0 || !c0->local) return PR_ERR_INVALID;
    const int P = c0->P;
    int64_t sumn = 0;
    for (int r = 0; r < P; ++r) {
        const pr_comm* c = comms[r];
        if (!c || !c->local || c->rank != r || c->P != P || c->device != c0->device) return PR_ERR_INVALID;
        if (n_local[r] < 0 || (count > 0 && !d_bufs[r])) return PR_ERR_INVALID;
        if ((uintptr_t)d_bufs[r] & 15) return PR_ERR_ALIGN;
        if (int st = *(volatile int*)c->h_status) return st;
        sumn += n_local[r];
    }
    if (sumn <= 0) return PR_ERR_ZERO_SAMPLES;   // every n is visible here: fail before launching
    if (P == 1) return PR_OK;
    LaunchArgs a;
    std::memset(&a, 0, sizeof(a));
    a.count = count;
    a.dtype = dt;
    a.nranks = P;
    for (int r = 0; r < P; ++r) {
        a.calls[r].tab = comms[r]->d_tab;
        a.calls[r].buf = d_bufs[r];
        a.calls[r].n_local = n_local[r];
        find_reg(comms[r], d_bufs[r], 0, &a.calls[r].reg_id, &a.calls[r].reg_off);
    }
    PR_CUDA_TRY(cudaSetDevice(c0->device));
    // PR_ALGO_NVLS in a local group: the software emulation of the multicast kernel (nvls_kernel<true>)
    return launch_ring(a, P, P, c0->device, c0->cfg, (cudaStream_t)stream, true, /*in_nvls=*/true);
}

// ---- K7 fused into K3: weighted allreduce + SGD update (+ gradient reset) ---------------------------
extern "C" int pr_weighted_allreduce_sgd(pr_comm* c, float* d_grad, float* d_theta, int64_t count, int64_t n_local,
                                         double lr, double wd, int32_t zero_grad, void* stream) {
    if (!c || count < 0 || n_local < 0 || (count > 0 && (!d_grad || !d_theta))) return PR_ERR_INVALID;
    if (((uintptr_t)d_grad & 15) || ((uintptr_t)d_theta & 15)) return PR_ERR_ALIGN;
    if (int st = *(volatile int*)c->h_status) return st;
    if (c->P == 1) {
        if (n_local <= 0) return PR_ERR_ZERO_SAMPLES;
        return pr_sgd_update(d_theta, d_grad, count, lr, wd, zero_grad, stream);
    }
    LaunchArgs a;
    std::memset(&a, 0, sizeof(a));
    a.count = count;
    a.dtype = PR_DTYPE_F32;
    a.nranks = 1;
    a.calls[0].tab = c->d_tab;
    a.calls[0].buf = d_grad;
    a.calls[0].n_local = n_local;
    find_reg(c, d_grad, (size_t)count * 4, &a.calls[0].reg_id, &a.calls[0].reg_off);
    int32_t trid = -1;
    int64_t toff = 0;
    find_reg(c, d_theta, (size_t)count * 4, &trid, &toff);
    const int falgo = pick_algo(c->cfg, count, PR_DTYPE_F32, c->P, a.calls[0].reg_id >= 0);
    const bool fusable = (falgo == PR_ALGO_RING || falgo == PR_ALGO_TWO_SHOT_PULL) &&
                         a.calls[0].reg_id >= 0 && trid == a.calls[0].reg_id && !(c->cfg.flags & PR_COMM_FLAG_FORCE_STAGED);
    if (!fusable) {   // composed: the same bits (the ring's ḡ, then K7's two FMAs)
        if (int rc = pr_weighted_allreduce(c, d_grad, count, PR_DTYPE_F32, n_local, stream)) return rc;
        return pr_sgd_update(d_theta, d_grad, count, lr, wd, zero_grad, stream);
    }
    a.fuse = 1;
    a.zero = zero_grad ? 1 : 0;
    a.nlr = (float)(-lr);
    a.wd = (float)wd;
    a.calls[0].th_delta = (int64_t)((const uint8_t*)d_theta - (const uint8_t*)d_grad);
    PR_CUDA_TRY(cudaSetDevice(c->device));
    return launch_ring(a, 1, c->P, c->device, c->cfg, (cudaStream_t)stream, false);
}

extern "C" int pr_weighted_allreduce_sgd_local(pr_comm* const* comms, float* const* d_grads, float* const* d_thetas,
                                               int64_t count, const int64_t* n_local, double lr, double wd,
                                               int32_t zero_grad, void* stream) {
    if (!comms || !d_grads || !d_thetas || !n_local || count < 0) return PR_ERR_INVALID;
    const pr_comm* c0 = comms[0];
    if (!c0 || !c0->local) return PR_ERR_INVALID;
    const int P = c0->P;
    int64_t sumn = 0;
    bool same_delta = true;
    const int64_t d0 = (int64_t)((const uint8_t*)d_thetas[0] - (const uint8_t*)d_grads[0]);
    for (int r = 0; r < P; ++r) {
        const pr_comm* c = comms[r];
        if (!c || !c->local || c->rank != r || c->P != P || c->device != c0->device) return PR_ERR_INVALID;
        if (n_local[r] < 0 || (count > 0 && (!d_grads[r] || !d_thetas[r]))) return PR_ERR_INVALID;
        if (((uintptr_t)d_grads[r] & 15) || ((uintptr_t)d_thetas[r] & 15)) return PR_ERR_ALIGN;
        if (int st = *(volatile int*)c->h_status) return st;
        sumn += n_local[r];
        same_delta = same_delta && (int64_t)((const uint8_t*)d_thetas[r] - (const uint8_t*)d_grads[r]) == d0;
    }
    if (sumn <= 0) return PR_ERR_ZERO_SAMPLES;
    PR_CUDA_TRY(cudaSetDevice(c0->device));
    const int falgo = P > 1 ? pick_algo(c0->cfg, count, PR_DTYPE_F32, P, true) : PR_ALGO_RING;
    const bool fusable = P > 1 && (falgo == PR_ALGO_RING || falgo == PR_ALGO_TWO_SHOT_PULL) && same_delta &&
                         !(c0->cfg.flags & PR_COMM_FLAG_FORCE_STAGED);
    if (!fusable) {
        if (P > 1) {
            if (int rc = pr_weighted_allreduce_local(comms, (void* const*)d_grads, count, PR_DTYPE_F32, n_local, stream))
                return rc;
        }
        for (int r = 0; r < P; ++r)
            if (int rc = pr_sgd_update(d_thetas[r], d_grads[r], count, lr, wd, zero_grad, stream)) return rc;
        return PR_OK;
    }
    LaunchArgs a;
    std::memset(&a, 0, sizeof(a));
    a.count = count;
    a.dtype = PR_DTYPE_F32;
    a.nranks = P;
    a.fuse = 1;
    a.zero = zero_grad ? 1 : 0;
    a.nlr = (float)(-lr);
    a.wd = (float)wd;
    for (int r = 0; r < P; ++r) {
        a.calls[r].tab = comms[r]->d_tab;
        a.calls[r].buf = d_grads[r];
        a.calls[r].n_local = n_local[r];
        a.calls[r].th_delta = d0;
        find_reg(comms[r], d_grads[r], 0, &a.calls[r].reg_id, &a.calls[r].reg_off);
    }
    return launch_ring(a, P, P, c0->device, c0->cfg, (cudaStream_t)stream, true);
}

extern "C" int pr_comm_allgather_f64(pr_comm* c, double local, double* out, void* stream) {
    if (!c || !out || c->local) return PR_ERR_INVALID;
    if (int st = *(volatile int*)c->h_status) return st;
    if (c->P == 1) { out[0] = local; return PR_OK; }
    PR_CUDA_TRY(cudaSetDevice(c->device));
    double* d_out = nullptr;
    PR_CUDA_TRY(cudaHostGetDevicePointer((void**)&d_out, c->h_ag, 0));
    c->ag_seq += 1;
    allgather_f64_kernel<<<1, 32, 0, (cudaStream_t)stream>>>(c->d_tab, c->ag_seq, local, nullptr, d_out);
    PR_CUDA_TRY(cudaGetLastError());
    PR_CUDA_TRY(cudaStreamSynchronize((cudaStream_t)stream));
    if (int st = *(volatile int*)c->h_status) return st;
    for (int q = 0; q < c->P; ++q) out[q] = ((volatile double*)c->h_ag)[q];
    return PR_OK;
}

extern "C" int pr_comm_allgather_f64_async(pr_comm* c, const double* d_local, double* h_out, void* stream) {
    if (!c || !d_local || !h_out || c->local) return PR_ERR_INVALID;
    if (int st = *(volatile int*)c->h_status) return st;
    PR_CUDA_TRY(cudaSetDevice(c->device));
    cudaPointerAttributes at;
    if (cudaPointerGetAttributes(&at, h_out) != cudaSuccess || at.type != cudaMemoryTypeHost || !at.devicePointer) {
        cudaGetLastError();
        return PR_ERR_INVALID;                         // must be pinned host memory the device can write
    }
    if (c->P == 1) {                                   // identity: one stream-ordered copy
        PR_CUDA_TRY(cudaMemcpyAsync(at.devicePointer, d_local, sizeof(double), cudaMemcpyDeviceToDevice,
                                    (cudaStream_t)stream));
        return PR_OK;
    }
    c->ag_seq += 1;
    allgather_f64_kernel<<<1, 32, 0, (cudaStream_t)stream>>>(c->d_tab, c->ag_seq, 0.0, d_local,
                                                            reinterpret_cast<double*>(at.devicePointer));
    PR_CUDA_TRY(cudaGetLastError());
    return PR_OK;
}

extern "C" int pr_comm_status(pr_comm* c) {
    if (!c) return PR_ERR_INVALID;
    return *(volatile int*)c->h_status;
}

extern "C" int pr_comm_timestamps(pr_comm* c, int64_t* out) {
    if (!c || !out) return PR_ERR_INVALID;
    for (int i = 0; i < 3; ++i) out[i] = ((volatile long long*)c->h_stamps)[i];
    return PR_OK;
}

extern "C" int pr_comm_rank(const pr_comm* c, int32_t* rank, int32_t* size) {
    if (!c) return PR_ERR_INVALID;
    if (rank) *rank = c->rank;
    if (size) *size = c->P;
    return PR_OK;
}

extern "C" void pr_comm_destroy(pr_comm* c) {
    if (!c) return;
    if (!c->local && c->fn && c->P > 1) {   // collective: nobody unmaps while a peer may still signal
        cudaSetDevice(c->device);
        cudaDeviceSynchronize();
        int flag = 0;
        std::vector<int> flags(c->P);
        exchange(c, &flag, sizeof(int), flags.data());
    }
    free_comm(c);
}

// ---- misc ABI ----------------------------------------------------------------------------------------
extern "C" const char* pr_strerror(int code) {
    switch (code) {
        case PR_OK: return "ok";
        case PR_ERR_INVALID: return "invalid argument";
        case PR_ERR_INFEASIBLE_FLOOR: return "infeasible floor (C < P*floor)";
        case PR_ERR_DATASET_TOO_SMALL: return "dataset too small (N < g*C)";
        case PR_ERR_ZERO_TIMING: return "zero/invalid step timing";
        case PR_ERR_CUDA: return "CUDA error";
        case PR_ERR_ALIGN: return "misaligned pointer or row size";
        case PR_ERR_NO_P2P: return "no peer access between GPUs";
        case PR_ERR_LENGTH_MISMATCH: return "ranks disagree on count/dtype";
        case PR_ERR_ZERO_SAMPLES: return "sum of n_local is zero";
        case PR_ERR_PEER_TIMEOUT: return "peer timeout (watchdog)";
        case PR_ERR_CAPACITY: return "capacity too small";
        case PR_ERR_INTERNAL: return "internal error";
        case PR_ERR_UNSUPPORTED: return "not supported on this platform (NVLS multicast)";
        default: return "unknown error";
    }
}

extern "C" int pr_version(void) { return PR_VERSION; }
