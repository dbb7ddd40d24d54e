// K1 — per-epoch permutation + proportional split (the sharder), sm_100a.
//
// Paper: each worker "holds unequal subdataset" in proportion w_i/Σw (§3.1) and the sub-datasets
// are redistributed every epoch (Algorithm 1 step 3).  The shuffle is build-defined (DESIGN.md
// §3 #8): π_{seed,e} = 4-round Feistel network on a 2^b domain (b even, 2^b >= N) whose round function is
// word 0 of Philox4x32-10(ctr = (R, k, lo32 e, hi32 e), key = (lo32 seed, hi32 seed)), cycle-walked into
// [0, N).  Shard r = π(off_r .. off_r + len_r − 1).
//
// Bound: integer ALU (≈4 Philox-10 evaluations per Feistel pass, ≈M/N passes per index); the only
// memory traffic is the 8-byte index written per output.  Default kernel: lane-refill
// cycle walk, one contiguous range of outputs per warp (walk_refill_kernel below).
#include <curand_philox4x32_x.h>
#include <stdlib.h>
#include <string.h>

#include "common.h"

namespace {

constexpr uint32_t kM0 = 0xD2511F53u, kM1 = 0xCD9E8D57u;
constexpr uint32_t kW0 = 0x9E3779B9u, kW1 = 0xBB67AE85u;

__device__ __forceinline__ uint4 philox_round(uint4 c, uint32_t k0, uint32_t k1) {
    const uint32_t hi0 = __umulhi(kM0, c.x), lo0 = kM0 * c.x;
    const uint32_t hi1 = __umulhi(kM1, c.z), lo1 = kM1 * c.z;
    return make_uint4(hi1 ^ c.y ^ k0, lo1, hi0 ^ c.w ^ k1, lo0);
}

__device__ __forceinline__ uint4 philox4x32_10(uint4 c, uint32_t k0, uint32_t k1) {
#pragma unroll
    for (int r = 0; r < 10; ++r) {
        if (r) { k0 += kW0; k1 += kW1; }
        c = philox_round(c, k0, k1);
    }
    return c;
}

struct FeistelKey {
    uint32_t k0, k1, e_lo, e_hi;
    uint32_t h;         // half width in bits (1..32)
    uint64_t mask;      // 2^h − 1
};

__device__ __forceinline__ uint64_t feistel(uint64_t x, const FeistelKey& fk) {
    uint64_t L = x >> fk.h, R = x & fk.mask;
#pragma unroll
    for (uint32_t k = 0; k < 4; ++k) {
        const uint4 o = philox4x32_10(make_uint4((uint32_t)R, k, fk.e_lo, fk.e_hi), fk.k0, fk.k1);
        const uint64_t f = (uint64_t)o.x & fk.mask;
        const uint64_t t = L ^ f;
        L = R;
        R = t;
    }
    return (L << fk.h) | R;
}

constexpr int kRefillWarpsPerSM = 16;   // A/B at N = 1,281,167 (profiles/round2_k1_refill_ab.jsonl): 8 → 68.2 µs, 16 → 62.1, 24 → 63.0, 32 → 68.2, 64 → 78.8

// Index maps: output position i -> the Feistel input whose cycle-walked image is out[i].
struct RangeMap {  // pr_permute / pr_shard_indices: π(begin + i)
    uint64_t begin;
    __device__ __forceinline__ uint64_t operator()(uint64_t i) const { return begin + i; }
};
struct StepMap {   // pr_shard_steps (N3): π(s·B + o + t), s = step0 + i / n, t = i mod n
    uint64_t B, o, n, step0;
    __device__ __forceinline__ uint64_t operator()(uint64_t i) const {
        const uint64_t q = i / n;
        return (step0 + q) * B + o + (i - q * n);
    }
};

// One thread per output index (round 1).  A warp runs as long as its longest cycle walk: with
// p = N/M accepted draws the walk length is geometric(p), so at N = 1,281,167 (p = 0.305, mean 3.27
// Feistel passes) the warp's maximum over 32 lanes is ≈ 3× the mean and two thirds of the issued
// Feistel passes belong to lanes that have already finished.  Kept for the A/B (PR_K1_KERNEL=direct).
template <class Map>
__global__ void __launch_bounds__(256) walk_direct_kernel(uint64_t N, FeistelKey fk, Map map, uint64_t count,
                                                          int64_t* __restrict__ out) {
    const uint64_t stride = (uint64_t)gridDim.x * blockDim.x;
    for (uint64_t i = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; i < count; i += stride) {
        uint64_t y = feistel(map(i), fk);
        while (y >= N) y = feistel(y, fk);  // cycle walking: terminates, π restricted to [0, N) is a bijection
        out[i] = (int64_t)y;
    }
}

// Lane-refill walk (round 2, default): each warp owns a contiguous range of output positions and every
// lane carries one walk in flight.  Per iteration all lanes take one Feistel pass; a lane whose image
// fell inside [0, N) stores it and takes the warp's next position (ballot + popc hands positions out in
// lane order), the others keep walking.  Every issued pass is useful work until the warp's range runs
// dry, so the issue cost per index is the mean walk (M/N passes), not the warp's maximum.  Same π, same
// bits; only the order in which the outputs are written changes.
template <class Map>
__global__ void __launch_bounds__(256) walk_refill_kernel(uint64_t N, FeistelKey fk, Map map, uint64_t count,
                                                          uint64_t per_warp, int64_t* __restrict__ out) {
    const unsigned lane = threadIdx.x & 31u;
    const unsigned below = (1u << lane) - 1u;
    const uint64_t warp = ((uint64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
    const uint64_t jb = warp * per_warp;
    if (jb >= count) return;  // warp-uniform
    const uint64_t je = (jb + per_warp < count) ? jb + per_warp : count;
    uint64_t j = jb + lane;
    bool active = j < je;
    uint64_t x = active ? map(j) : 0;
    uint64_t next = jb + 32;
    while (__any_sync(0xffffffffu, active)) {
        const uint64_t y = feistel(x, fk);
        const bool done = active && y < N;
        const unsigned dm = __ballot_sync(0xffffffffu, done);
        if (done) {
            out[j] = (int64_t)y;
            j = next + __popc(dm & below);
            active = j < je;
            if (active) x = map(j);
        } else {
            x = y;  // keep walking (inactive lanes compute on a dead value)
        }
        next += __popc(dm);
    }
}

int refill_warps_per_sm() {   // A/B knob PR_K1_WARPS_PER_SM (8..64, multiple of 8); see launch_walk
    static const int w = [] {
        const char* e = getenv("PR_K1_WARPS_PER_SM");
        const int v = e ? atoi(e) : 0;
        return (v >= 8 && v <= 64 && v % 8 == 0) ? v : kRefillWarpsPerSM;
    }();
    return w;
}

bool use_direct_kernel() {
    static const bool direct = [] {
        const char* e = getenv("PR_K1_KERNEL");
        return e && !strcmp(e, "direct");
    }();
    return direct;
}

// Launch K1 over `count` outputs.  Refill: warps = min(148·W, ceil(count/32)) (each lane ≥ 1 position),
// contiguous ranges of ceil(count/warps) positions.  W = warps per SM trades the range's tail (the last
// lanes' walks finish while the rest of the warp idles: fewer, longer ranges amortise it) against latency
// hiding (IMAD.WIDE chains; the fmaheavy pipe saturates with a few warps per scheduler).
template <class Map>
int launch_walk(uint64_t N, const FeistelKey& fk, Map map, uint64_t count, int64_t* d_out, cudaStream_t st) {
    if (use_direct_kernel()) {
        uint64_t blocks = (count + 255) / 256;
        if (blocks > 148 * 8) blocks = 148 * 8;
        walk_direct_kernel<Map><<<(unsigned)blocks, 256, 0, st>>>(N, fk, map, count, d_out);
    } else {
        uint64_t warps = (count + 31) / 32;
        const uint64_t wmax = 148ull * (uint64_t)refill_warps_per_sm();
        if (warps > wmax) warps = wmax;
        const uint64_t per_warp = (count + warps - 1) / warps;
        warps = (count + per_warp - 1) / per_warp;
        const uint64_t blocks = (warps + 7) / 8;
        walk_refill_kernel<Map><<<(unsigned)blocks, 256, 0, st>>>(N, fk, map, count, per_warp, d_out);
    }
    PR_CUDA_TRY(cudaGetLastError());
    return PR_OK;
}

__global__ void philox_test_kernel(const uint32_t* __restrict__ ctr, int64_t n, uint32_t k0, uint32_t k1,
                                   int use_curand, uint32_t* __restrict__ out) {
    const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= n) return;
    const uint4 c = make_uint4(ctr[4 * i], ctr[4 * i + 1], ctr[4 * i + 2], ctr[4 * i + 3]);
    uint4 o;
    if (use_curand) {
        o = curand_Philox4x32_10(c, make_uint2(k0, k1));
    } else {
        o = philox4x32_10(c, k0, k1);
    }
    out[4 * i] = o.x; out[4 * i + 1] = o.y; out[4 * i + 2] = o.z; out[4 * i + 3] = o.w;
}

FeistelKey make_key(int64_t N, uint64_t seed, int64_t epoch) {
    uint32_t b = 0;
    for (uint64_t v = (uint64_t)(N - 1); v; v >>= 1) ++b;  // bitlen(N − 1)
    if (b < 2) b = 2;
    if (b & 1) ++b;
    FeistelKey fk;
    fk.h = b / 2;
    fk.mask = (fk.h >= 64) ? ~0ull : ((1ull << fk.h) - 1ull);
    fk.k0 = (uint32_t)(seed & 0xffffffffu);
    fk.k1 = (uint32_t)(seed >> 32);
    fk.e_lo = (uint32_t)((uint64_t)epoch & 0xffffffffu);
    fk.e_hi = (uint32_t)((uint64_t)epoch >> 32);
    return fk;
}

}  // namespace

extern "C" int pr_permute(int64_t N, uint64_t seed, int64_t epoch, int64_t begin, int64_t count, int64_t* d_out,
                          void* stream) {
    if (N < 1 || N > ((int64_t)1 << 62) || begin < 0 || count < 0 || begin + count > N) return PR_ERR_INVALID;
    if (count == 0) return PR_OK;
    if (!d_out) return PR_ERR_INVALID;
    const FeistelKey fk = make_key(N, seed, epoch);
    return launch_walk((uint64_t)N, fk, RangeMap{(uint64_t)begin}, (uint64_t)count, d_out, (cudaStream_t)stream);
}

extern "C" int pr_shard_indices(const pr_alloc* a, int32_t rank, int64_t epoch, uint64_t seed, int64_t* d_out,
                                int64_t cap, void* stream) {
    int64_t N, off, len;
    int rc = pr_internal_shard_range(a, rank, &N, &off, &len);
    if (rc) return rc;
    if (cap < len) return PR_ERR_CAPACITY;
    return pr_permute(N, seed, epoch, off, len, d_out, stream);
}

extern "C" int pr_shard_steps(const pr_alloc* a, int32_t rank, int64_t epoch, uint64_t seed, int64_t step0,
                              int64_t nsteps, int64_t* d_out, int64_t cap, void* stream) {
    int64_t N, B, S, o, n;
    int rc = pr_internal_step_layout(a, rank, &N, &B, &S, &o, &n);
    if (rc) return rc;
    if (step0 < 0 || nsteps < 0 || step0 + nsteps > S) return PR_ERR_INVALID;
    const int64_t count = nsteps * n;
    if (cap < count) return PR_ERR_CAPACITY;
    if (count == 0) return PR_OK;
    if (!d_out) return PR_ERR_INVALID;
    const FeistelKey fk = make_key(N, seed, epoch);
    return launch_walk((uint64_t)N, fk, StepMap{(uint64_t)B, (uint64_t)o, (uint64_t)n, (uint64_t)step0},
                       (uint64_t)count, d_out, (cudaStream_t)stream);
}

extern "C" int pr_test_philox(const uint32_t* d_ctr, int64_t n, uint64_t key, int32_t use_curand, uint32_t* d_out,
                              void* stream) {
    if (n < 0 || (n > 0 && (!d_ctr || !d_out))) return PR_ERR_INVALID;
    if (n == 0) return PR_OK;
    philox_test_kernel<<<(unsigned)((n + 255) / 256), 256, 0, (cudaStream_t)stream>>>(
        d_ctr, n, (uint32_t)(key & 0xffffffffu), (uint32_t)(key >> 32), use_curand, d_out);
    PR_CUDA_TRY(cudaGetLastError());
    return PR_OK;
}
