// Write-bandwidth probe: which store flavour reaches HBM write peak on B200 (K2 is write-heavy: 1 B read
// for 2 B written).  Build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o write_probe write_probe.cu
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>

template <int MODE>
__global__ void wr(uint4* __restrict__ d, size_t n, uint32_t v) {
    const size_t stride = (size_t)gridDim.x * blockDim.x;
    const uint4 x = make_uint4(v, v + 1, v + 2, v + 3);
    for (size_t i = (size_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += stride) {
        uint4* p = d + i;
        if (MODE == 0) asm volatile("st.global.v4.u32 [%0], {%1,%2,%3,%4};" ::"l"(p), "r"(x.x), "r"(x.y), "r"(x.z), "r"(x.w) : "memory");
        if (MODE == 1) asm volatile("st.global.cs.v4.u32 [%0], {%1,%2,%3,%4};" ::"l"(p), "r"(x.x), "r"(x.y), "r"(x.z), "r"(x.w) : "memory");
        if (MODE == 2) asm volatile("st.global.L1::no_allocate.v4.u32 [%0], {%1,%2,%3,%4};" ::"l"(p), "r"(x.x), "r"(x.y), "r"(x.z), "r"(x.w) : "memory");
        if (MODE == 3) {   // 256-bit store (sm_100), evict-first; i indexes 32-byte units here
            if (2 * i + 1 < n) asm volatile("st.global.L2::evict_first.v8.b32 [%0], {%1,%2,%3,%4,%1,%2,%3,%4};" ::"l"(d + 2 * i), "r"(x.x), "r"(x.y), "r"(x.z), "r"(x.w) : "memory");
        }
        if (MODE == 5) {   // 256-bit store (sm_100)
            if (2 * i + 1 < n) asm volatile("st.global.v8.b32 [%0], {%1,%2,%3,%4,%1,%2,%3,%4};" ::"l"(d + 2 * i), "r"(x.x), "r"(x.y), "r"(x.z), "r"(x.w) : "memory");
        }
        if (MODE == 4) asm volatile("st.global.wt.v4.u32 [%0], {%1,%2,%3,%4};" ::"l"(p), "r"(x.x), "r"(x.y), "r"(x.z), "r"(x.w) : "memory");
    }
}

// unrolled: each thread writes 4 consecutive-stride vectors per iteration
template <int MODE>
__global__ void wr4(uint4* __restrict__ d, size_t n, uint32_t v) {
    const size_t stride = (size_t)gridDim.x * blockDim.x;
    const uint4 x = make_uint4(v, v + 1, v + 2, v + 3);
    for (size_t i = (size_t)blockIdx.x * blockDim.x + threadIdx.x; i + 3 * stride < n; i += 4 * stride) {
#pragma unroll
        for (int u = 0; u < 4; ++u) {
            uint4* p = d + i + u * stride;
            if (MODE == 0) asm volatile("st.global.v4.u32 [%0], {%1,%2,%3,%4};" ::"l"(p), "r"(x.x), "r"(x.y), "r"(x.z), "r"(x.w) : "memory");
            if (MODE == 1) asm volatile("st.global.cs.v4.u32 [%0], {%1,%2,%3,%4};" ::"l"(p), "r"(x.x), "r"(x.y), "r"(x.z), "r"(x.w) : "memory");
        }
    }
}

int main() {
    const size_t bytes = 302ull << 20;   // the epoch gather's output
    const size_t n = bytes / 16;
    uint4* d;
    cudaMalloc(&d, bytes);
    uint8_t* fl;
    cudaMalloc(&fl, 256 << 20);
    int sms;
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
    cudaEvent_t a, b;
    cudaEventCreate(&a);
    cudaEventCreate(&b);
    const char* names[] = {"st.global", "st.global.cs", "st.L1::no_allocate", "st.v8 L2::evict_first", "st.global.wt", "st.v8.b32"};
    for (int grid_mul : {4, 8, 16, 64}) {
        for (int m = 0; m < 8; ++m) {
            float best = 1e9;
            for (int r = 0; r < 10; ++r) {
                cudaMemsetAsync(fl, r, 256 << 20);
                cudaEventRecord(a);
                const int g = sms * grid_mul, t = 256;
                switch (m) {
                    case 0: wr<0><<<g, t>>>(d, n, r); break;
                    case 1: wr<1><<<g, t>>>(d, n, r); break;
                    case 2: wr<2><<<g, t>>>(d, n, r); break;
                    case 3: wr<3><<<g, t>>>(d, n, r); break;
                    case 4: wr<4><<<g, t>>>(d, n, r); break;
                    case 5: wr<5><<<g, t>>>(d, n, r); break;
                    case 6: wr4<0><<<g, t>>>(d, n, r); break;
                    case 7: wr4<1><<<g, t>>>(d, n, r); break;
                }
                cudaEventRecord(b);
                cudaEventSynchronize(b);
                float ms;
                cudaEventElapsedTime(&ms, a, b);
                if (ms < best) best = ms;
            }
            printf("grid %3dxSM %-22s %s %8.2f us %8.1f GB/s\n", grid_mul, m < 6 ? names[m] : (m == 6 ? "unroll4 st.global" : "unroll4 st.global.cs"),
                   "", best * 1e3, bytes / (best * 1e-3) / 1e9);
        }
    }
    float best = 1e9;
    for (int r = 0; r < 10; ++r) {
        cudaMemsetAsync(fl, r, 256 << 20);
        cudaEventRecord(a);
        cudaMemsetAsync(d, r + 1, bytes);
        cudaEventRecord(b);
        cudaEventSynchronize(b);
        float ms;
        cudaEventElapsedTime(&ms, a, b);
        if (ms < best) best = ms;
    }
    printf("cudaMemsetAsync                         %8.2f us %8.1f GB/s\n", best * 1e3, bytes / (best * 1e-3) / 1e9);
    printf("%s\n", cudaGetErrorString(cudaGetLastError()));
    return 0;
}
