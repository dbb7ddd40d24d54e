// racecheck probe: does compute-sanitizer's racecheck model a TWO-hop mbarrier release chain?
// Same TMA ring as K3 (ring.cu) reduced to its synchronisation skeleton, 2 stages, 64 rounds:
//   producer warp:  wait empty[s] (parity) -> arrive.expect_tx full[s] -> cp.async.bulk global->smem stage s
//   consumer warps: wait full[s] -> read stage s (ld.shared) -> __syncwarp -> lane 0 arrives on
//                   HOPS == 1: empty[s]               (one hop: consumer -> producer, as K2's TMA gather)
//                   HOPS == 2: stored[s]; the signal warp waits stored[s] and arrives on empty[s] (as K3)
// Both are correct under the PTX memory model (mbarrier arrive = release, try_wait = acquire, causality
// order is transitive).  Build: nvcc -gencode arch=compute_100a,code=sm_100a -O2 -lineinfo -DHOPS=1|2
// Run:   compute-sanitizer --tool racecheck ./racecheck_chain
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>

#ifndef HOPS
#define HOPS 2
#endif
constexpr int kStages = 2, kRounds = 64, kStageBytes = 4096, kConsumers = 4;

__device__ __forceinline__ uint32_t su32(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }
__device__ __forceinline__ void mb_init(uint64_t* b, int c) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(su32(b)), "r"(c) : "memory");
}
__device__ __forceinline__ void mb_arrive(uint64_t* b) {
    asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(su32(b)) : "memory");
}
__device__ __forceinline__ void mb_expect(uint64_t* b, uint32_t tx) {
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(su32(b)), "r"(tx) : "memory");
}
__device__ __forceinline__ void mb_wait(uint64_t* b, uint32_t parity) {
    asm volatile(
        "{\n\t.reg .pred P1;\n\tWAIT:\n\t"
        "mbarrier.try_wait.parity.shared::cta.b64 P1, [%0], %1;\n\t"
        "@!P1 bra WAIT;\n\t}" ::"r"(su32(b)), "r"(parity) : "memory");
}
__device__ __forceinline__ void tma_load(void* dst, const void* src, uint32_t bytes, uint64_t* bar) {
    asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];"
                 ::"r"(su32(dst)), "l"(src), "r"(bytes), "r"(su32(bar)) : "memory");
}

__global__ void chain(const uint4* __restrict__ src, unsigned long long* out) {
    __shared__ alignas(128) uint4 stage[kStages][kStageBytes / 16];
    __shared__ uint64_t full[kStages], empty[kStages], stored[kStages];
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    if (threadIdx.x == 0) {
        for (int s = 0; s < kStages; ++s) {
            mb_init(&full[s], 1);
            mb_init(&empty[s], HOPS == 1 ? kConsumers : 1);
            mb_init(&stored[s], kConsumers);
        }
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    __syncthreads();
    if (warp == 0) {                                   // producer
        if (lane == 0)
            for (int r = 0; r < kRounds; ++r) {
                const int s = r % kStages;
                if (r >= kStages) mb_wait(&empty[s], ((r / kStages) - 1) & 1);
                mb_expect(&full[s], kStageBytes);
                tma_load(stage[s], src + (size_t)r * (kStageBytes / 16), kStageBytes, &full[s]);
            }
    } else if (warp <= kConsumers) {                   // consumers
        unsigned long long acc = 0;
        for (int r = 0; r < kRounds; ++r) {
            const int s = r % kStages;
            mb_wait(&full[s], (r / kStages) & 1);
            for (int i = lane + 32 * (warp - 1); i < kStageBytes / 16; i += 32 * kConsumers) acc += stage[s][i].x;
            __syncwarp();
            if (lane == 0) mb_arrive(HOPS == 1 ? &empty[s] : &stored[s]);
        }
        atomicAdd(out, acc);
    } else if (HOPS == 2 && warp == kConsumers + 1) {  // signal warp (K3's middle hop)
        if (lane == 0)
            for (int r = 0; r < kRounds; ++r) {
                const int s = r % kStages;
                mb_wait(&stored[s], (r / kStages) & 1);
                mb_arrive(&empty[s]);
            }
    }
}

int main() {
    const size_t n = (size_t)kRounds * kStageBytes / 16;
    uint4* src;
    unsigned long long* out;
    cudaMalloc(&src, n * 16);
    cudaMalloc(&out, 8);
    uint4* h = new uint4[n];
    unsigned long long expect = 0;
    for (size_t i = 0; i < n; ++i) { h[i] = make_uint4((unsigned)i, 0, 0, 0); expect += (unsigned)i; }
    cudaMemcpy(src, h, n * 16, cudaMemcpyHostToDevice);
    cudaMemset(out, 0, 8);
    chain<<<1, 32 * (kConsumers + 2)>>>(src, out);
    unsigned long long got = 0;
    cudaMemcpy(&got, out, 8, cudaMemcpyDeviceToHost);
    printf("HOPS=%d sum %s (%llu vs %llu) %s\n", HOPS, got == expect ? "ok" : "BAD", got, expect,
           cudaGetErrorString(cudaGetLastError()));
    return got == expect ? 0 : 1;
}
