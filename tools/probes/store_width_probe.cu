// Per-SM store throughput with 128-bit vs 256-bit global stores (STG.E.128 vs STG.E.ENL2.256), few CTAs
// (HBM idle): is K3's per-channel bound (the SM -> crossbar store path, profiles/round2_ring_cta_ncu_summary.md)
// a request-count limit that wider stores relieve?  Also a copy (load + store) per width.
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o store_width_probe store_width_probe.cu
#include <cstdint>
#include <cstdio>
#include <cuda_runtime.h>

template <int W>   // bytes per thread per store: 16 or 32
__global__ void __launch_bounds__(512) fill(float* __restrict__ d, size_t n_floats, float v) {
    const size_t per = W / 4;
    const size_t stride = (size_t)gridDim.x * blockDim.x * per;
    for (size_t i = ((size_t)blockIdx.x * blockDim.x + threadIdx.x) * per; i < n_floats; i += stride) {
        if (W == 16) {
            asm volatile("st.global.v4.f32 [%0], {%1,%1,%1,%1};" ::"l"(d + i), "f"(v) : "memory");
        } else {
            asm volatile("st.global.v8.f32 [%0], {%1,%1,%1,%1,%1,%1,%1,%1};" ::"l"(d + i), "f"(v) : "memory");
        }
    }
}

template <int W>
__global__ void __launch_bounds__(512) copy(float* __restrict__ d, const float* __restrict__ s, size_t n_floats) {
    const size_t per = W / 4;
    const size_t stride = (size_t)gridDim.x * blockDim.x * per;
    for (size_t i = ((size_t)blockIdx.x * blockDim.x + threadIdx.x) * per; i < n_floats; i += stride) {
        if (W == 16) {
            float a, b, c, e;
            asm volatile("ld.global.v4.f32 {%0,%1,%2,%3}, [%4];" : "=f"(a), "=f"(b), "=f"(c), "=f"(e) : "l"(s + i));
            asm volatile("st.global.v4.f32 [%0], {%1,%2,%3,%4};" ::"l"(d + i), "f"(a), "f"(b), "f"(c), "f"(e) : "memory");
        } else {
            float a0, a1, a2, a3, a4, a5, a6, a7;
            asm volatile("ld.global.v8.f32 {%0,%1,%2,%3,%4,%5,%6,%7}, [%8];"
                         : "=f"(a0), "=f"(a1), "=f"(a2), "=f"(a3), "=f"(a4), "=f"(a5), "=f"(a6), "=f"(a7)
                         : "l"(s + i));
            asm volatile("st.global.v8.f32 [%0], {%1,%2,%3,%4,%5,%6,%7,%8};" ::"l"(d + i), "f"(a0), "f"(a1), "f"(a2),
                         "f"(a3), "f"(a4), "f"(a5), "f"(a6), "f"(a7)
                         : "memory");
        }
    }
}

int main() {
    const size_t bytes = 512ull << 20, n = bytes / 4;
    float *d, *s;
    cudaMalloc(&d, bytes);
    cudaMalloc(&s, bytes);
    cudaMemset(s, 0, bytes);
    cudaEvent_t a, b;
    cudaEventCreate(&a);
    cudaEventCreate(&b);
    auto run = [&](const char* name, int ctas, auto launch, double moved) {
        launch();
        cudaDeviceSynchronize();
        cudaEventRecord(a);
        for (int r = 0; r < 5; ++r) launch();
        cudaEventRecord(b);
        cudaEventSynchronize(b);
        float ms;
        cudaEventElapsedTime(&ms, a, b);
        const double t = ms / 5 * 1e-3;
        printf("%-10s ctas %3d  %8.1f us  %7.1f GB/s total  %6.1f GB/s per CTA (stored bytes)\n", name, ctas, t * 1e6,
               moved / t / 1e9, moved / t / 1e9 / ctas);
    };
    for (int ctas : {16, 32, 64, 148}) {
        run("fill v4", ctas, [&] { fill<16><<<ctas, 512>>>(d, n, 1.0f); }, (double)bytes);
        run("fill v8", ctas, [&] { fill<32><<<ctas, 512>>>(d, n, 1.0f); }, (double)bytes);
        run("copy v4", ctas, [&] { copy<16><<<ctas, 512>>>(d, s, n); }, (double)bytes);
        run("copy v8", ctas, [&] { copy<32><<<ctas, 512>>>(d, s, n); }, (double)bytes);
    }
    printf("%s\n", cudaGetErrorString(cudaDeviceSynchronize()));
    return 0;
}
