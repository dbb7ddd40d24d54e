// K2 — step-batch gather of sampled rows into the local batch, with the u8 -> f32/bf16 affine fused
// (and optionally the CHW -> HWC "channels-last" layout change the model's tensor-core convs want).
//
// Paper: Algorithm 1 step 4, "Proportionally draw samples from the sub-data set for training";
// static allocation, "Worker i draws w_i samples from subdataset".  Data-plane definition is
// build-defined (DESIGN.md §3 #38, #41): dst[t,:] = op(src[idx[t],:]), lab_dst[t] = lab_src[idx[t]];
// with PR_GATHER_LAYOUT_HWC the output element (c, p) of a CHW row is stored at p·C + c.
//
// HBM-bound: per row, row_bytes read + out_bytes written (+8 B index, +16 B label).  Three kernels with
// identical results:
//   gather_hwc_bulk_kernel  channels-last output: coalesced loads, conversion into a smem tile in output
//                      order, one cp.async.bulk store per 4096 output pixels (below; the AUTO choice for
//                      channels-last launches of >= 1 MiB from device memory);
//   gather_tma_kernel  persistent CTAs; a producer warp prefetches row indices and issues cp.async.bulk
//                      copies (whole rows, 24 KiB segments, or per-channel pixel blocks) into a 4-stage
//                      mbarrier ring; 8 consumer warps convert from smem and store 16-byte vectors.
//   gather_kernel      (LSU) a warp per 2 KiB segment, 4 ld.global.nc 16-byte loads in flight per lane;
//                      chosen for small launches and host-memory sources (the e2e path).
// Conversion: u8 -> exact float via PRMT into 0x4B000000 then −2^23, (x − shift)·scale with packed
// FADD2/FMUL2 (per-lane IEEE RN, identical to the scalar two-op definition), cvt.rn.bf16x2.f32.
#include <cuda_bf16.h>

#include <cstdlib>

#include "common.h"

namespace {

constexpr int kWarpsPerCta = 8;
constexpr int kVecPerLane = 4;                            // 16-byte input vectors per lane per work item
constexpr int kSegVec = 32 * kVecPerLane;                 // input vectors per work item (2 KiB)
constexpr int kMaxHwcChannels = 4;

struct GatherParams {
    const uint8_t* src;
    int64_t row_bytes;
    const int64_t* idx;
    int64_t n;
    uint8_t* dst;
    int32_t op;
    int32_t channels;
    int64_t plane;
    float scale[PR_GATHER_MAX_CHANNELS];
    float shift[PR_GATHER_MAX_CHANNELS];
    const int64_t* lab_src;
    int64_t* lab_dst;
    int32_t hwc;          // 1: channels-last output
};

__device__ __forceinline__ uint4 ld_nc_v4(const void* p) {
    uint4 r;
    asm volatile("ld.global.nc.L1::no_allocate.v4.u32 {%0,%1,%2,%3}, [%4];"
                 : "=r"(r.x), "=r"(r.y), "=r"(r.z), "=r"(r.w)
                 : "l"(p));
    return r;
}

__device__ __forceinline__ void st_v4(void* p, uint4 v) {
    asm volatile("st.global.v4.u32 [%0], {%1,%2,%3,%4};" ::"l"(p), "r"(v.x), "r"(v.y), "r"(v.z), "r"(v.w)
                 : "memory");
}

// (float(x) − shift) · scale: two separately rounded fp32 operations (no contraction).
__device__ __forceinline__ float affine(uint32_t x, float sc, float sh) {
    return __fmul_rn(__fsub_rn((float)x, sh), sc);
}

__device__ __forceinline__ uint32_t pack_bf16x2(float lo, float hi) {
    const __nv_bfloat162 h = __floats2bfloat162_rn(lo, hi);     // one cvt.rn.bf16x2.f32
    return *reinterpret_cast<const uint32_t*>(&h);
}

// Packed fp32 pairs (Blackwell FADD2/FMUL2): per-lane IEEE round-to-nearest, identical to two scalar ops.
__device__ __forceinline__ uint64_t pk2(float lo, float hi) {
    uint64_t r;
    asm("mov.b64 %0, {%1,%2};" : "=l"(r) : "f"(lo), "f"(hi));
    return r;
}
__device__ __forceinline__ uint64_t add2(uint64_t a, uint64_t b) {
    uint64_t r;
    asm("add.rn.f32x2 %0, %1, %2;" : "=l"(r) : "l"(a), "l"(b));
    return r;
}
__device__ __forceinline__ uint64_t mul2(uint64_t a, uint64_t b) {
    uint64_t r;
    asm("mul.rn.f32x2 %0, %1, %2;" : "=l"(r) : "l"(a), "l"(b));
    return r;
}
// bytes j and j+1 of w as exact floats 2^23 + x (PRMT into the mantissa of 0x4B000000)
__device__ __forceinline__ uint64_t u8pair_magic(uint32_t w, int j) {
    const uint32_t a = __byte_perm(w, 0x4B000000u, 0x7540u + j);
    const uint32_t b = __byte_perm(w, 0x4B000000u, 0x7540u + j + 1);
    return (uint64_t)a | ((uint64_t)b << 32);
}
// f[0..2k) = (x − shift)·scale for the 4·k bytes of w[0..k), one channel
template <int K>
__device__ __forceinline__ void affine_words(const uint32_t* w, float sc, float sh, float* f) {
    const uint64_t m23 = pk2(-8388608.0f, -8388608.0f);
    const uint64_t nsh = pk2(-sh, -sh);
    const uint64_t sc2 = pk2(sc, sc);
#pragma unroll
    for (int j = 0; j < 4 * K; j += 2) {
        const uint64_t xf = add2(u8pair_magic(w[j >> 2], j & 3), m23);   // exact: x
        const uint64_t y = mul2(add2(xf, nsh), sc2);                     // RN(RN(x − shift)·scale)
        f[j] = __uint_as_float((uint32_t)y);
        f[j + 1] = __uint_as_float((uint32_t)(y >> 32));
    }
}

template <int OP>
__device__ __forceinline__ void convert_store(const GatherParams& p, uint8_t* drow, int64_t v, uint4 x) {
    if (OP == PR_GATHER_COPY) {
        st_v4(drow + v * 16, x);
        return;
    }
    const uint32_t w[4] = {x.x, x.y, x.z, x.w};
    float f[16];
    const uint32_t k0 = (uint32_t)v * 16u;  // element index of the first byte (row_bytes < 2^31)
    const uint32_t plane = (uint32_t)p.plane;
    if (plane % 16u == 0) {                 // one channel per 16-byte vector
        const int c = (int)(k0 / plane);
        affine_words<4>(w, p.scale[c], p.shift[c], f);
    } else {
#pragma unroll
        for (int j = 0; j < 16; ++j) {
            const int c = (int)((k0 + (uint32_t)j) / plane);
            f[j] = affine((w[j >> 2] >> (8 * (j & 3))) & 0xffu, p.scale[c], p.shift[c]);
        }
    }
    if (OP == PR_GATHER_U8_TO_BF16_AFFINE) {
        uint8_t* d = drow + v * 32;
        st_v4(d, make_uint4(pack_bf16x2(f[0], f[1]), pack_bf16x2(f[2], f[3]), pack_bf16x2(f[4], f[5]),
                            pack_bf16x2(f[6], f[7])));
        st_v4(d + 16, make_uint4(pack_bf16x2(f[8], f[9]), pack_bf16x2(f[10], f[11]), pack_bf16x2(f[12], f[13]),
                                 pack_bf16x2(f[14], f[15])));
    } else {
        uint8_t* d = drow + v * 64;
#pragma unroll
        for (int q = 0; q < 4; ++q)
            st_v4(d + 16 * q, make_uint4(__float_as_uint(f[4 * q]), __float_as_uint(f[4 * q + 1]),
                                         __float_as_uint(f[4 * q + 2]), __float_as_uint(f[4 * q + 3])));
    }
}

// Channels-last: PX (8 or 16) consecutive pixels of all C channels (ww = PX/4 words per channel) -> the
// PX·C interleaved outputs (value k = pixel k / C, channel k mod C) as NV = PX·C·es/16 16-byte vectors o[]
// (es = 2 for bf16, 4 for f32).
template <int OP, int C, int PX>
__device__ __forceinline__ void hwc_convert_words(const GatherParams& p, const uint32_t* ww, uint4* o) {
    float f[C][PX];
#pragma unroll
    for (int c = 0; c < C; ++c) affine_words<PX / 4>(ww + c * (PX / 4), p.scale[c], p.shift[c], f[c]);
    if (OP == PR_GATHER_U8_TO_BF16_AFFINE) {
#pragma unroll
        for (int q = 0; q < C * PX / 8; ++q) {
            uint32_t h[4];
#pragma unroll
            for (int j = 0; j < 4; ++j) {
                const int k = 8 * q + 2 * j;
                h[j] = pack_bf16x2(f[k % C][k / C], f[(k + 1) % C][(k + 1) / C]);
            }
            o[q] = make_uint4(h[0], h[1], h[2], h[3]);
        }
    } else {
#pragma unroll
        for (int q = 0; q < C * PX / 4; ++q) {
            uint32_t h[4];
#pragma unroll
            for (int j = 0; j < 4; ++j) {
                const int k = 4 * q + j;
                h[j] = __float_as_uint(f[k % C][k / C]);
            }
            o[q] = make_uint4(h[0], h[1], h[2], h[3]);
        }
    }
}

template <int OP, int C, int PX>
__device__ __forceinline__ void hwc_convert(const GatherParams& p, const uint8_t* s, int64_t ps, uint4* o) {
    uint32_t ww[C * PX / 4];
#pragma unroll
    for (int c = 0; c < C; ++c) {
        if (PX == 16) {
            const uint4 w = *reinterpret_cast<const uint4*>(s + c * ps);
            ww[4 * c] = w.x; ww[4 * c + 1] = w.y; ww[(4 * c + 2) % (C * PX / 4)] = w.z; ww[(4 * c + 3) % (C * PX / 4)] = w.w;
        } else {
            const uint2 w = *reinterpret_cast<const uint2*>(s + c * ps);
            ww[2 * c] = w.x; ww[2 * c + 1] = w.y;
        }
    }
    hwc_convert_words<OP, C, PX>(p, ww, o);
}

// TMA consumer path: 8 pixels from the smem stage straight to the HWC output row (8·C·es bytes per lane).
template <int OP, int C>
__device__ __forceinline__ void hwc_store(const GatherParams& p, uint8_t* drow, int64_t pix0, const uint8_t* s,
                                          int64_t ps) {
    constexpr int NV = C * 8 * (OP == PR_GATHER_U8_TO_BF16_AFFINE ? 2 : 4) / 16;
    uint4 o[NV];
    hwc_convert<OP, C, 8>(p, s, ps, o);
    uint8_t* d = drow + pix0 * C * (OP == PR_GATHER_U8_TO_BF16_AFFINE ? 2 : 4);
#pragma unroll
    for (int q = 0; q < NV; ++q) st_v4(d + 16 * q, o[q]);
}

template <int OP>
__device__ __forceinline__ void hwc_dispatch(const GatherParams& p, uint8_t* drow, int64_t pix0, const uint8_t* s,
                                             int64_t ps) {
    switch (p.channels) {
        case 1: hwc_store<OP, 1>(p, drow, pix0, s, ps); break;
        case 2: hwc_store<OP, 2>(p, drow, pix0, s, ps); break;
        case 3: hwc_store<OP, 3>(p, drow, pix0, s, ps); break;
        default: hwc_store<OP, 4>(p, drow, pix0, s, ps); break;
    }
}

// Channels-last LSU loop: a warp item is 32 lanes × 8 pixels of one row.  ITEMS items per iteration: all
// their loads (C 8-byte loads per item per lane, coalesced across the warp) are issued before any
// conversion/store, so ITEMS·C loads are in flight per lane.  Measured (epoch gather, 49,152 DISTINCT rows,
// tools/ab_gather.sh): ITEMS 1 / 2 / 3 at 64 regs (4 CTAs per SM) 85.6 / 89.7 / 95.3 µs; ITEMS 2 at 96 regs
// (2 CTAs per SM) 104.8 µs — more loads in flight do not help; occupancy does, up to 4 CTAs per SM (48
// regs, 5 CTAs: 96 µs).
#ifndef PR_HWC_ITEMS
#define PR_HWC_ITEMS 1
#endif
template <int OP, int C>
__device__ __forceinline__ void hwc_lsu_loop(const GatherParams& p, int64_t warp, int64_t nwarps, int lane) {
    constexpr int ITEMS = PR_HWC_ITEMS;
    constexpr int es = OP == PR_GATHER_U8_TO_BF16_AFFINE ? 2 : 4;
    constexpr int NV = C * 8 * es / 16;
    const int64_t groups = p.plane / 8, gsegs = (groups + 31) / 32;
    const int64_t total = p.n * gsegs;
    const int64_t out_row = p.row_bytes * es;
    for (int64_t it0 = warp; it0 < total; it0 += (int64_t)ITEMS * nwarps) {
        uint32_t ww[ITEMS][C * 2];
        int64_t drow_off[ITEMS];
        bool ok[ITEMS];
#pragma unroll
        for (int u = 0; u < ITEMS; ++u) {
            const int64_t it = it0 + (int64_t)u * nwarps;
            const int64_t row = it / gsegs, gi = (it - row * gsegs) * 32 + lane;
            ok[u] = it < total && gi < groups;
            drow_off[u] = row * out_row + gi * 8 * C * es;
            if (ok[u]) {
                const uint8_t* s = p.src + __ldg(p.idx + row) * p.row_bytes + gi * 8;
#pragma unroll
                for (int c = 0; c < C; ++c) {
                    const uint2 w = *reinterpret_cast<const uint2*>(s + c * p.plane);
                    ww[u][2 * c] = w.x;
                    ww[u][2 * c + 1] = w.y;
                }
            }
        }
#pragma unroll
        for (int u = 0; u < ITEMS; ++u) {
            if (!ok[u]) continue;
            uint4 o[NV];
            hwc_convert_words<OP, C, 8>(p, ww[u], o);
            uint8_t* d = p.dst + drow_off[u];
#pragma unroll
            for (int q = 0; q < NV; ++q) st_v4(d + 16 * q, o[q]);
        }
    }
}

#ifndef PR_GATHER_MINB
#define PR_GATHER_MINB 4
#endif
template <int OP>
__global__ void __launch_bounds__(32 * kWarpsPerCta, PR_GATHER_MINB) gather_kernel(const __grid_constant__ GatherParams p) {
    const int lane = threadIdx.x & 31;
    const int64_t warp = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
    const int64_t nwarps = ((int64_t)gridDim.x * blockDim.x) >> 5;
    const int64_t vpr = p.row_bytes / 16;                      // input vectors per row
    const int64_t segs = (vpr + kSegVec - 1) / kSegVec;         // work items per row
    const int64_t out_mul = (OP == PR_GATHER_COPY) ? 1 : (OP == PR_GATHER_U8_TO_BF16_AFFINE ? 2 : 4);
    const int64_t items = p.n * segs;

    if (p.lab_dst) {                                            // labels: one thread per row
        const int64_t nthreads = (int64_t)gridDim.x * blockDim.x;
        for (int64_t t = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; t < p.n; t += nthreads)
            p.lab_dst[t] = p.lab_src[p.idx[t]];
    }
    if (OP != PR_GATHER_COPY && p.hwc) {
        // channels-last: a warp item is 32 lanes × 8 pixels of one row; per lane C 8-byte loads (one per
        // plane, coalesced across the warp) and 8·C·es bytes of interleaved output stored directly.
        // Measured alternatives (epoch gather, 49,152 rows, same box): this 83.5 us; 16-pixel items 99 us;
        // per-warp smem staging for fully coalesced stores 85-86 us; ld.global.nc 3% slower; a software-
        // pipelined loop (next item's loads before this item's stores) 87.8 us; grids of 2-80 waves slower
        // than one resident wave.  A write-only probe reaches 6.6 TB/s (tools/probes/write_probe.cu).
        switch (p.channels) {
            case 1: hwc_lsu_loop<OP, 1>(p, warp, nwarps, lane); break;
            case 2: hwc_lsu_loop<OP, 2>(p, warp, nwarps, lane); break;
            case 3: hwc_lsu_loop<OP, 3>(p, warp, nwarps, lane); break;
            default: hwc_lsu_loop<OP, 4>(p, warp, nwarps, lane); break;
        }
        return;
    }
    for (int64_t it = warp; it < items; it += nwarps) {
        const int64_t row = it / segs;
        const int64_t seg = it - row * segs;
        const int64_t src_row = __ldg(p.idx + row);
        const uint8_t* srow = p.src + src_row * p.row_bytes;
        uint8_t* drow = p.dst + row * p.row_bytes * out_mul;
        const int64_t v0 = seg * kSegVec + lane;
        uint4 x[kVecPerLane];
#pragma unroll
        for (int u = 0; u < kVecPerLane; ++u) {
            const int64_t v = v0 + 32 * u;
            if (v < vpr) x[u] = ld_nc_v4(srow + v * 16);
        }
#pragma unroll
        for (int u = 0; u < kVecPerLane; ++u) {
            const int64_t v = v0 + 32 * u;
            if (v < vpr) convert_store<OP>(p, drow, v, x[u]);
        }
    }
}

// ---- TMA-staged variant --------------------------------------------------------------------------------
// A unit is up to kTmaSeg input bytes: several whole rows (one bulk copy each), one 24 KiB segment of a
// long row (CHW output), or one pixel block of a long row across all C planes (HWC output, C copies).
// The producer warp prefetches the next unit's row indices (lane-parallel) while lane 0 issues copies.
constexpr int kTmaStages = 4;
constexpr int kTmaSeg = 24576;                // input bytes per unit
constexpr int kTmaConsumerWarps = 8;

__device__ __forceinline__ uint32_t smem_u32(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }
__device__ __forceinline__ void mbar_init(uint64_t* b, uint32_t c) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(b)), "r"(c) : "memory");
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
__device__ __forceinline__ void tma_load(void* dst, const void* src, uint32_t bytes, uint64_t* bar) {
    asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
                     smem_u32(dst)),
                 "l"(src), "r"(bytes), "r"(smem_u32(bar))
                 : "memory");
}

struct TmaGeom {
    int64_t rpu;     // rows per unit (> 1: whole rows)
    int64_t upr;     // units per row (rpu == 1)
    int64_t pb;      // HWC pixel block (rpu == 1 && hwc), pixels
    int64_t units;
};

__host__ __device__ inline TmaGeom tma_geom(int64_t n, int64_t row_bytes, int hwc, int64_t channels, int64_t plane) {
    TmaGeom g;
    g.rpu = 1;
    g.pb = 0;
    if (row_bytes <= kTmaSeg / 2) {
        g.rpu = kTmaSeg / row_bytes < 32 ? kTmaSeg / row_bytes : 32;
        g.upr = 1;
        g.units = (n + g.rpu - 1) / g.rpu;
    } else if (hwc) {
        g.pb = (kTmaSeg / channels) / 16 * 16;
        g.upr = (plane + g.pb - 1) / g.pb;
        g.units = n * g.upr;
    } else {
        g.upr = (row_bytes + kTmaSeg - 1) / kTmaSeg;
        g.units = n * g.upr;
    }
    return g;
}

template <int OP>
__global__ void __launch_bounds__(32 * (kTmaConsumerWarps + 1)) gather_tma_kernel(const __grid_constant__ GatherParams p) {
    extern __shared__ __align__(128) uint8_t smem[];   // [kTmaStages][kTmaSeg]
    __shared__ uint64_t full[kTmaStages], empty[kTmaStages];
    const TmaGeom geo = tma_geom(p.n, p.row_bytes, p.hwc, p.channels, p.plane);
    const int64_t G = gridDim.x;
    const int64_t out_mul = (OP == PR_GATHER_COPY) ? 1 : (OP == PR_GATHER_U8_TO_BF16_AFFINE ? 2 : 4);
    if (threadIdx.x == 0) {
        for (int k = 0; k < kTmaStages; ++k) {
            mbar_init(&full[k], 1);
            mbar_init(&empty[k], kTmaConsumerWarps);
        }
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    if (p.lab_dst) {                                                 // labels: one thread per row
        const int64_t nthreads = (int64_t)gridDim.x * blockDim.x;
        for (int64_t t = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; t < p.n; t += nthreads)
            p.lab_dst[t] = p.lab_src[p.idx[t]];
    }
    __syncthreads();
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    auto fetch = [&](int64_t u) -> int64_t {          // source row(s) of unit u (lane j: j-th row)
        if (u >= geo.units) return 0;
        if (geo.rpu > 1) {
            const int64_t row = u * geo.rpu + lane;
            return (lane < geo.rpu && row < p.n) ? __ldg(p.idx + row) : 0;
        }
        return __ldg(p.idx + u / geo.upr);
    };
    if (warp == 0) {
        uint32_t k = 0;
        int64_t cur = fetch(blockIdx.x);
        for (int64_t u = blockIdx.x; u < geo.units; u += G, ++k) {
            const int64_t nxt = fetch(u + G);                         // prefetch: hides the idx latency
            const int stg = (int)(k % kTmaStages);
            if (lane == 0 && k >= (uint32_t)kTmaStages) mbar_wait(&empty[stg], ((k / kTmaStages) - 1) & 1);
            uint8_t* dst = smem + (size_t)stg * kTmaSeg;
            if (geo.rpu > 1) {
                const int64_t nrows = min(geo.rpu, p.n - u * geo.rpu);
                if (lane == 0) mbar_arrive_expect_tx(&full[stg], (uint32_t)(nrows * p.row_bytes));
                for (int j = 0; j < nrows; ++j) {
                    const int64_t srow = __shfl_sync(0xffffffffu, cur, j);
                    if (lane == 0) tma_load(dst + j * p.row_bytes, p.src + srow * p.row_bytes, (uint32_t)p.row_bytes,
                                            &full[stg]);
                }
            } else if (lane == 0) {
                const int64_t b = u % geo.upr;
                if (geo.pb) {                                         // HWC: pixel block of every plane
                    const int64_t p0 = b * geo.pb;
                    const uint32_t np = (uint32_t)min(geo.pb, p.plane - p0);
                    mbar_arrive_expect_tx(&full[stg], np * (uint32_t)p.channels);
                    for (int c = 0; c < p.channels; ++c)
                        tma_load(dst + c * geo.pb, p.src + cur * p.row_bytes + c * p.plane + p0, np, &full[stg]);
                } else {
                    const int64_t off = b * kTmaSeg;
                    const uint32_t bytes = (uint32_t)min((int64_t)kTmaSeg, p.row_bytes - off);
                    mbar_arrive_expect_tx(&full[stg], bytes);
                    tma_load(dst, p.src + cur * p.row_bytes + off, bytes, &full[stg]);
                }
            }
            cur = nxt;
        }
    } else {
        // consumer warps: smem -> convert -> 16-byte stores, lanes on consecutive vectors / pixel groups
        const int cw = warp - 1;
        const int64_t vpr = p.row_bytes / 16;
        uint32_t k = 0;
        for (int64_t u = blockIdx.x; u < geo.units; u += G, ++k) {
            const int stg = (int)(k % kTmaStages);
            mbar_wait(&full[stg], (k / kTmaStages) & 1);
            const uint8_t* sb = smem + (size_t)stg * kTmaSeg;
            const uint4* sv = reinterpret_cast<const uint4*>(sb);
            if (geo.rpu > 1) {
                const int64_t nrows = min(geo.rpu, p.n - u * geo.rpu);
                for (int64_t rl = cw; rl < nrows; rl += kTmaConsumerWarps) {
                    uint8_t* drow = p.dst + (u * geo.rpu + rl) * p.row_bytes * out_mul;
                    if (OP != PR_GATHER_COPY && p.hwc) {
                        for (int64_t gi = lane; gi < p.plane / 8; gi += 32)
                            hwc_dispatch<OP>(p, drow, gi * 8, sb + rl * p.row_bytes + gi * 8, p.plane);
                    } else {
                        for (int64_t v = lane; v < vpr; v += 32) convert_store<OP>(p, drow, v, sv[rl * vpr + v]);
                    }
                }
            } else {
                const int64_t row = u / geo.upr, b = u - row * geo.upr;
                uint8_t* drow = p.dst + row * p.row_bytes * out_mul;
                if (OP != PR_GATHER_COPY && geo.pb) {
                    const int64_t p0 = b * geo.pb, np = min(geo.pb, p.plane - p0);
                    for (int64_t gi = threadIdx.x - 32; gi < np / 8; gi += 32 * kTmaConsumerWarps)
                        hwc_dispatch<OP>(p, drow, p0 + gi * 8, sb + gi * 8, geo.pb);
                } else {
                    const int64_t off = b * kTmaSeg;
                    const int64_t nv = min((int64_t)kTmaSeg, p.row_bytes - off) / 16;
                    for (int64_t v = threadIdx.x - 32; v < nv; v += 32 * kTmaConsumerWarps)
                        convert_store<OP>(p, drow, off / 16 + v, sv[v]);
                }
            }
            __syncwarp();
            if (lane == 0) mbar_arrive(&empty[stg]);
        }
    }
}

// ---- Bulk-store variant (channels-last output) ----------------------------------------------------------
// The output of a channels-last gather is one contiguous stream: dst pixel q (row t = q / plane, pixel
// p = q mod plane) sits at q·C·es.  A unit is kBulkPx consecutive output pixels (several short rows or a
// block of a long row): every thread loads kBulkGroups 8-pixel groups (C 8-byte loads each, coalesced per
// plane across the warp, all issued before any conversion), converts them into the unit's smem tile in
// output order (16-byte smem stores, conflict-free at the 48-byte lane stride), and one thread pushes the
// whole tile with a single cp.async.bulk store.  Two tiles per CTA: a tile is rewritten only after its
// previous bulk store has read it.  Why: a 1:2 read:write stream with 16-byte STGs tops out at 5.97 TB/s
// on B200, with smem tiles + bulk stores at 6.28 TB/s (tools/probes/mix_probe.cu, ImageNet-sized) —
// full-line writes in large bursts.  t = q / plane by a 64-bit multiply-high with m = ceil(2^64 / plane),
// exact while q·plane < 2^64 (checked on the host).
constexpr int kBulkThreads = 256;
constexpr int kBulkGroupsDefault = 2;                            // 8-pixel groups per thread per unit
constexpr int64_t kBulkAutoBytes = 1 << 20;                      // AUTO: input bytes from which the bulk kernel runs

__device__ __forceinline__ void bulk_store(void* dst, const void* src, uint32_t bytes) {
    asm volatile("cp.async.bulk.global.shared::cta.bulk_group [%0], [%1], %2;" ::"l"(dst), "r"(smem_u32(src)),
                 "r"(bytes)
                 : "memory");
    asm volatile("cp.async.bulk.commit_group;" ::: "memory");
}

template <int OP, int C, int kBulkGroups>
__global__ void __launch_bounds__(kBulkThreads) gather_hwc_bulk_kernel(const __grid_constant__ GatherParams p,
                                                                       uint64_t magic) {
    extern __shared__ __align__(128) uint8_t tiles[];             // [2][kBulkPx · C · es]
    constexpr int64_t kBulkPx = 8 * kBulkThreads * kBulkGroups;      // output pixels per unit
    constexpr int es = OP == PR_GATHER_U8_TO_BF16_AFFINE ? 2 : 4;
    constexpr int NV = C * 8 * es / 16;                              // 16-byte vectors per 8-pixel group
    constexpr int64_t kTile = kBulkPx * C * es;
    if (p.lab_dst) {                                                 // labels: one thread per row
        const int64_t nthreads = (int64_t)gridDim.x * blockDim.x;
        for (int64_t t = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; t < p.n; t += nthreads)
            p.lab_dst[t] = p.lab_src[p.idx[t]];
    }
    const uint64_t plane = (uint64_t)p.plane;
    const uint64_t total = (uint64_t)p.n * plane;
    const uint64_t units = (total + kBulkPx - 1) / kBulkPx;
    int buf = 0;
    for (uint64_t u = blockIdx.x; u < units; u += gridDim.x) {
        uint8_t* tile = tiles + buf * kTile;
        if (threadIdx.x == 0) asm volatile("cp.async.bulk.wait_group.read 1;" ::: "memory");
        __syncthreads();                                             // the tile's previous store has read it
        const uint64_t q0 = u * kBulkPx;
        const uint64_t npx = min((uint64_t)kBulkPx, total - q0);
        uint32_t ww[kBulkGroups][C * 2];
#pragma unroll
        for (int g = 0; g < kBulkGroups; ++g) {
            const uint64_t px = 8ull * (threadIdx.x + (uint64_t)g * kBulkThreads);
            if (px < npx) {
                const uint64_t q = q0 + px;
                const uint64_t t = __umul64hi(q, magic);
                const uint8_t* s = p.src + __ldg(p.idx + t) * p.row_bytes + (q - t * plane);
#pragma unroll
                for (int c = 0; c < C; ++c) {
                    const uint2 w = *reinterpret_cast<const uint2*>(s + c * p.plane);
                    ww[g][2 * c] = w.x;
                    ww[g][2 * c + 1] = w.y;
                }
            }
        }
#pragma unroll
        for (int g = 0; g < kBulkGroups; ++g) {
            const uint64_t px = 8ull * (threadIdx.x + (uint64_t)g * kBulkThreads);
            if (px < npx) {
                uint4 o[NV];
                hwc_convert_words<OP, C, 8>(p, ww[g], o);
                uint4* d = reinterpret_cast<uint4*>(tile + px * C * es);
#pragma unroll
                for (int v = 0; v < NV; ++v) d[v] = o[v];
            }
        }
        asm volatile("fence.proxy.async.shared::cta;" ::: "memory");  // generic smem writes -> bulk copy
        __syncthreads();
        if (threadIdx.x == 0) bulk_store(p.dst + q0 * C * es, tile, (uint32_t)(npx * C * es));
        buf ^= 1;
    }
    if (threadIdx.x == 0) asm volatile("cp.async.bulk.wait_group 0;" ::: "memory");
}

template <int OP, int G>
const void* bulk_fn_g(int C) {
    switch (C) {
        case 1: return (const void*)gather_hwc_bulk_kernel<OP, 1, G>;
        case 2: return (const void*)gather_hwc_bulk_kernel<OP, 2, G>;
        case 3: return (const void*)gather_hwc_bulk_kernel<OP, 3, G>;
        default: return (const void*)gather_hwc_bulk_kernel<OP, 4, G>;
    }
}
template <int OP>
const void* bulk_fn(int C, int G) {
    return G == 1 ? bulk_fn_g<OP, 1>(C) : bulk_fn_g<OP, 2>(C);
}

// Launch of the bulk-store kernel; false when the geometry is outside its exactness range (caller falls back).
int launch_hwc_bulk(const GatherParams& p, cudaStream_t s, bool* launched) {
    *launched = false;
    const unsigned __int128 pl = (unsigned __int128)(uint64_t)p.plane;
    if ((unsigned __int128)(uint64_t)p.n * pl * pl >= ((unsigned __int128)1 << 64)) return PR_OK;
    const uint64_t magic = (uint64_t)((((unsigned __int128)1 << 64) + pl - 1) / pl);
    // A/B knob: groups per thread, 1 or 2 (measured, 4 bench launch sizes: 2 = 1 within noise; 4 is 5-20 %
    // slower and its f32 4-channel tiles would not fit in shared memory)
    static const int G = [] {
        const char* e = getenv("PR_GATHER_BULK_GROUPS");
        const int v = e ? atoi(e) : kBulkGroupsDefault;
        return v == 1 ? 1 : 2;
    }();
    const int64_t upx = 8 * kBulkThreads * G;
    const int es = p.op == PR_GATHER_U8_TO_BF16_AFFINE ? 2 : 4;
    const int C = p.channels;
    const size_t smem = 2 * (size_t)upx * C * es;
    const void* fn = p.op == PR_GATHER_U8_TO_BF16_AFFINE ? bulk_fn<PR_GATHER_U8_TO_BF16_AFFINE>(C, G)
                                                         : bulk_fn<PR_GATHER_U8_TO_F32_AFFINE>(C, G);
    // per device, per (op, C): dynamic-smem opt-in and the resident grid
    static std::mutex mu;
    static int grid_of[PR_MAX_DEVICES][2][kMaxHwcChannels + 1];
    int dev = 0;
    PR_CUDA_TRY(cudaGetDevice(&dev));
    if (dev < 0 || dev >= PR_MAX_DEVICES) return PR_ERR_INVALID;
    const int oi = p.op == PR_GATHER_U8_TO_BF16_AFFINE ? 1 : 0;
    int grid = 0;
    {
        std::lock_guard<std::mutex> lk(mu);
        if (!grid_of[dev][oi][C]) {
            PR_CUDA_TRY(cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
            int sms = 0, per = 0;
            PR_CUDA_TRY(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev));
            PR_CUDA_TRY(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per, fn, kBulkThreads, smem));
            static const int cap = [] {
                const char* e = getenv("PR_GATHER_BULK_CTAS");      // A/B knob: CTAs per SM (default 8)
                const int v = e ? atoi(e) : 8;
                return v < 1 ? 8 : v;
            }();
            grid_of[dev][oi][C] = sms * (per < 1 ? 1 : (per < cap ? per : cap));
        }
        grid = grid_of[dev][oi][C];
    }
    const int64_t units = ((int64_t)p.n * p.plane + upx - 1) / upx;
    const int blocks = (int)(units < grid ? (units > 0 ? units : 1) : grid);
    void* args[] = {(void*)&p, (void*)&magic};
    PR_CUDA_TRY(cudaLaunchKernel(fn, dim3(blocks), dim3(kBulkThreads), args, smem, s));
    *launched = true;
    return PR_OK;
}

}  // namespace

extern "C" int pr_gather_rows(const void* d_src, int64_t n_src, int64_t row_bytes, const int64_t* d_idx, int64_t n,
                              void* d_dst, const pr_gather_op* op, const int64_t* d_lab_src, int64_t* d_lab_dst,
                              void* stream) {
    if (n < 0 || n_src < 0 || row_bytes <= 0) return PR_ERR_INVALID;
    if (n == 0) return PR_OK;
    if (!d_src || !d_idx || !d_dst || (d_lab_dst && !d_lab_src)) return PR_ERR_INVALID;
    if (row_bytes >= ((int64_t)1 << 31)) return PR_ERR_INVALID;
    if (row_bytes % 16 || ((uintptr_t)d_src & 15) || ((uintptr_t)d_dst & 15)) return PR_ERR_ALIGN;
    GatherParams p;
    p.src = (const uint8_t*)d_src;
    p.row_bytes = row_bytes;
    p.idx = d_idx;
    p.n = n;
    p.dst = (uint8_t*)d_dst;
    p.op = op ? op->op : PR_GATHER_COPY;
    p.channels = 1;
    p.plane = row_bytes;
    p.hwc = 0;
    for (int i = 0; i < PR_GATHER_MAX_CHANNELS; ++i) { p.scale[i] = 1.0f; p.shift[i] = 0.0f; }
    if (p.op != PR_GATHER_COPY) {
        if (p.op != PR_GATHER_U8_TO_F32_AFFINE && p.op != PR_GATHER_U8_TO_BF16_AFFINE) return PR_ERR_INVALID;
        if (op->channels < 1 || op->channels > PR_GATHER_MAX_CHANNELS || op->plane < 1 ||
            op->plane * op->channels != row_bytes)
            return PR_ERR_INVALID;
        p.channels = op->channels;
        p.plane = op->plane;
        for (int i = 0; i < op->channels; ++i) { p.scale[i] = op->scale[i]; p.shift[i] = op->shift[i]; }
        if (op->layout == PR_GATHER_LAYOUT_HWC) {
            if (op->channels > kMaxHwcChannels || op->plane % 16) return PR_ERR_INVALID;
            p.hwc = 1;
        } else if (op->layout != PR_GATHER_LAYOUT_CHW) {
            return PR_ERR_INVALID;
        }
    }
    p.lab_src = d_lab_src;
    p.lab_dst = d_lab_dst;
    cudaStream_t s = (cudaStream_t)stream;
    const int impl = op ? op->impl : PR_GATHER_IMPL_AUTO;
    // TMA staging pays off once a launch moves enough bytes to be bandwidth-bound; rows
    // read from pinned host memory (the e2e path) stream over PCIe through the LSU kernel.
    bool host_src = false;
    if (impl != PR_GATHER_IMPL_TMA) {
        cudaPointerAttributes at;
        if (cudaPointerGetAttributes(&at, d_src) == cudaSuccess) host_src = at.type == cudaMemoryTypeHost;
        else cudaGetLastError();
    }
    // Measured on B200: CHW output, >= 8 MiB: TMA 5.26 vs LSU 4.89 TB/s; HWC output: LSU
    // 5.61 vs TMA 4.90 TB/s (each lane's per-plane 8-byte loads coalesce; no extra smem pass).
    if (impl == PR_GATHER_IMPL_BULK && !p.hwc) return PR_ERR_INVALID;   // channels-last output only
    if (p.hwc && !host_src &&
        (impl == PR_GATHER_IMPL_BULK || (impl == PR_GATHER_IMPL_AUTO && n * row_bytes >= kBulkAutoBytes))) {
        bool launched = false;
        const int rc = launch_hwc_bulk(p, s, &launched);
        if (rc != PR_OK || launched) return rc;
        if (impl == PR_GATHER_IMPL_BULK) return PR_ERR_INVALID;      // outside the kernel's index range
    }
    const bool tma = impl == PR_GATHER_IMPL_TMA ||
                     (impl == PR_GATHER_IMPL_AUTO && !host_src && !p.hwc && n * row_bytes >= (8ll << 20));
    if (tma) {
        const size_t smem = (size_t)kTmaStages * kTmaSeg;
        const TmaGeom geo = tma_geom(n, row_bytes, p.hwc, p.channels, p.plane);
        const int64_t blocks = geo.units < 148 * 2 ? geo.units : 148 * 2;
        const dim3 block(32 * (kTmaConsumerWarps + 1));
        // the dynamic-smem opt-in is a per-device function attribute: set once per device
        static std::mutex mu;
        static bool attr[PR_MAX_DEVICES];
        int dev = 0;
        PR_CUDA_TRY(cudaGetDevice(&dev));
        if (dev < 0 || dev >= PR_MAX_DEVICES) return PR_ERR_INVALID;
        {
            std::lock_guard<std::mutex> lk(mu);
            if (!attr[dev]) {
                PR_CUDA_TRY(cudaFuncSetAttribute(gather_tma_kernel<PR_GATHER_COPY>,
                                                 cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
                PR_CUDA_TRY(cudaFuncSetAttribute(gather_tma_kernel<PR_GATHER_U8_TO_F32_AFFINE>,
                                                 cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
                PR_CUDA_TRY(cudaFuncSetAttribute(gather_tma_kernel<PR_GATHER_U8_TO_BF16_AFFINE>,
                                                 cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
                attr[dev] = true;
            }
        }
        switch (p.op) {
            case PR_GATHER_COPY: gather_tma_kernel<PR_GATHER_COPY><<<(unsigned)blocks, block, smem, s>>>(p); break;
            case PR_GATHER_U8_TO_F32_AFFINE:
                gather_tma_kernel<PR_GATHER_U8_TO_F32_AFFINE><<<(unsigned)blocks, block, smem, s>>>(p);
                break;
            default: gather_tma_kernel<PR_GATHER_U8_TO_BF16_AFFINE><<<(unsigned)blocks, block, smem, s>>>(p);
        }
        PR_CUDA_TRY(cudaGetLastError());
        return PR_OK;
    }
    const int64_t vpr = row_bytes / 16;
    const int64_t items = n * ((vpr + kSegVec - 1) / kSegVec);
    // grid = one resident wave (SMs × CTAs per SM from the occupancy calculator): a grid-stride loop over
    // a grid larger than what fits leaves the second wave of CTAs as a tail
    // (per device: SM counts may differ between the devices one process drives)
    static std::mutex mu_res;
    static int resident_dev[PR_MAX_DEVICES][3];
    const int opi = p.op < 0 || p.op > 2 ? 2 : p.op;
    int rdev = 0;
    PR_CUDA_TRY(cudaGetDevice(&rdev));
    if (rdev < 0 || rdev >= PR_MAX_DEVICES) return PR_ERR_INVALID;
    int resident_n = 0;
    {
        std::lock_guard<std::mutex> lk(mu_res);
        if (!resident_dev[rdev][opi]) {
            int sms = 0, per_sm = 0;
            PR_CUDA_TRY(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, rdev));
            const void* fn = opi == 0 ? (const void*)gather_kernel<PR_GATHER_COPY>
                             : opi == 1 ? (const void*)gather_kernel<PR_GATHER_U8_TO_F32_AFFINE>
                                        : (const void*)gather_kernel<PR_GATHER_U8_TO_BF16_AFFINE>;
            PR_CUDA_TRY(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, fn, 32 * kWarpsPerCta, 0));
            resident_dev[rdev][opi] = sms * (per_sm > 0 ? per_sm : 1);
        }
        resident_n = resident_dev[rdev][opi];
    }
    int64_t blocks = (items + kWarpsPerCta - 1) / kWarpsPerCta;
#ifndef PR_GATHER_GRID
    if (blocks > resident_n) blocks = resident_n;
    if (host_src) {
        // rows read over PCIe: a few CTAs keep enough loads in flight for the link, and the rest of the GPU
        // stays free for the compute this gather runs beside (the trainer prefetches on a side stream).
        // Bench e2e, ResNet-18 leg (profiles/round2_e2e_host_grid_ab.jsonl): 16 / 32 CTAs 368-370k samples/s,
        // 64 364-366k, 128 364-365k.
        static const int host_grid = [] {
            const char* e = getenv("PR_GATHER_HOST_GRID");
            const int v = e ? atoi(e) : 32;
            return v < 1 ? 32 : v;
        }();
        if (blocks > host_grid) blocks = host_grid;
    }
#else
    if (blocks > PR_GATHER_GRID) blocks = PR_GATHER_GRID;
#endif
    if (blocks < 1) blocks = 1;
    switch (p.op) {
        case PR_GATHER_COPY: gather_kernel<PR_GATHER_COPY><<<(unsigned)blocks, 32 * kWarpsPerCta, 0, s>>>(p); break;
        case PR_GATHER_U8_TO_F32_AFFINE:
            gather_kernel<PR_GATHER_U8_TO_F32_AFFINE><<<(unsigned)blocks, 32 * kWarpsPerCta, 0, s>>>(p);
            break;
        default: gather_kernel<PR_GATHER_U8_TO_BF16_AFFINE><<<(unsigned)blocks, 32 * kWarpsPerCta, 0, s>>>(p);
    }
    PR_CUDA_TRY(cudaGetLastError());
    return PR_OK;
}

// ---- K4: emulated heterogeneity --------------------------------------------------------------------
namespace {
__global__ void spin_kernel(int64_t ns) {
    if (threadIdx.x != 0) return;
    uint64_t t0, t;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t0));
    do {
        asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
    } while ((int64_t)(t - t0) < ns);
}
}  // namespace

extern "C" int pr_spin(int64_t ns, void* stream) {
    if (ns <= 0) return PR_OK;
    spin_kernel<<<1, 32, 0, (cudaStream_t)stream>>>(ns);
    PR_CUDA_TRY(cudaGetLastError());
    return PR_OK;
}

// ---- a5: device-side step stamps ---------------------------------------------------------------------
namespace {
__global__ void stamp_kernel(int64_t* ring, int64_t cap) {
    uint64_t t;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
    const unsigned long long i = atomicAdd(reinterpret_cast<unsigned long long*>(ring), 1ull);
    ring[1 + (int64_t)(i % (unsigned long long)cap)] = (int64_t)t;
}
// Σ over the recorded (start, end) pairs, in seconds; one warp (lane-strided partial sums + shuffle).
__global__ void stamp_seconds_kernel(const int64_t* ring, int64_t cap, double* out) {
    const int64_t k = min(ring[0], cap);
    long long acc = 0;
    for (int64_t i = threadIdx.x; 2 * i + 1 < k; i += 32) acc += ring[2 + 2 * i] - ring[1 + 2 * i];
#pragma unroll
    for (int o = 16; o; o >>= 1) acc += __shfl_xor_sync(0xffffffffu, acc, o);
    if (threadIdx.x == 0) *out = (double)acc * 1e-9;
}
}  // namespace

extern "C" int pr_stamp_seconds(const int64_t* d_ring, int64_t cap, double* d_out, void* stream) {
    if (!d_ring || !d_out || cap < 1) return PR_ERR_INVALID;
    stamp_seconds_kernel<<<1, 32, 0, (cudaStream_t)stream>>>(d_ring, cap, d_out);
    PR_CUDA_TRY(cudaGetLastError());
    return PR_OK;
}

extern "C" int pr_stamp(int64_t* d_ring, int64_t cap, void* stream) {
    if (!d_ring || cap < 1) return PR_ERR_INVALID;
    stamp_kernel<<<1, 1, 0, (cudaStream_t)stream>>>(d_ring, cap);
    PR_CUDA_TRY(cudaGetLastError());
    return PR_OK;
}
