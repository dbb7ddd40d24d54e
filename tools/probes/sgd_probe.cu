// K7 (SGD + gradient reset) variants at the ResNet-18 / VGG-16 sizes: loads in flight per thread (unroll U),
// grid size, and the L2 state the kernel starts from.  "after-bwd" rewrites the gradient buffer right before
// the update (what backward leaves: the gradient lines dirty in L2, θ clean); "clean" evicts L2 with a read.
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o sgd_probe sgd_probe.cu
#include <cstdint>
#include <cstdio>
#include <cuda_runtime.h>

template <int U, bool REV>
__global__ void __launch_bounds__(256) sgd_u(float* __restrict__ th, float* __restrict__ g, int64_t n4, float nlr, float wd) {
    const int64_t stride = (int64_t)gridDim.x * blockDim.x;
    float4* t4 = reinterpret_cast<float4*>(th);
    float4* g4 = reinterpret_cast<float4*>(g);
    const int64_t tid = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    for (int64_t i0 = tid; i0 < n4; i0 += U * stride) {
        float4 t[U], d[U];
#pragma unroll
        for (int u = 0; u < U; ++u) {
            int64_t i = i0 + u * stride;
            if (REV) i = n4 - 1 - i;
            if (i0 + u * stride < n4) { t[u] = t4[i]; d[u] = g4[i]; }
        }
#pragma unroll
        for (int u = 0; u < U; ++u) {
            int64_t i = i0 + u * stride;
            if (REV) i = n4 - 1 - i;
            if (i0 + u * stride < n4) {
                float4 x = t[u];
                x.x = __fmaf_rn(nlr, __fmaf_rn(wd, x.x, d[u].x), x.x);
                x.y = __fmaf_rn(nlr, __fmaf_rn(wd, x.y, d[u].y), x.y);
                x.z = __fmaf_rn(nlr, __fmaf_rn(wd, x.z, d[u].z), x.z);
                x.w = __fmaf_rn(nlr, __fmaf_rn(wd, x.w, d[u].w), x.w);
                t4[i] = x;
                g4[i] = make_float4(0.f, 0.f, 0.f, 0.f);
            }
        }
    }
}

__global__ void fill(float* p, int64_t n, float v) {
    for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) p[i] = v;
}
__global__ void readflush(const uint4* __restrict__ f, size_t n, unsigned* sink) {
    uint32_t acc = 0;
    for (size_t i = (size_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (size_t)gridDim.x * blockDim.x) acc ^= f[i].x;
    if (acc == 0x12345678u) *sink = acc;
}

int main() {
    int sms;
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
    uint4* fl;
    unsigned* sink;
    cudaMalloc(&fl, 256 << 20);
    cudaMalloc(&sink, 4);
    cudaMemset(fl, 1, 256 << 20);
    cudaEvent_t a, b;
    cudaEventCreate(&a);
    cudaEventCreate(&b);
    for (int64_t L : {11689512LL, 138357544LL}) {
        float *th, *g;
        cudaMalloc(&th, L * 4);
        cudaMalloc(&g, L * 4);
        fill<<<sms * 4, 256>>>(th, L, 1.0f);
        const int64_t n4 = L / 4;
        for (int state = 0; state < 2; ++state) {
            auto run = [&](const char* name, auto launch) {
                float best = 1e9, sum = 0;
                const int reps = 20;
                for (int r = 0; r < reps; ++r) {
                    readflush<<<sms * 4, 256>>>(fl, (256 << 20) / 16, sink);
                    if (state == 1) fill<<<sms * 4, 256>>>(g, L, 1e-3f);   // backward just wrote ḡ
                    cudaEventRecord(a);
                    launch();
                    cudaEventRecord(b);
                    cudaEventSynchronize(b);
                    float ms;
                    cudaEventElapsedTime(&ms, a, b);
                    if (r >= 3) sum += ms;
                    if (ms < best) best = ms;
                }
                const double mean = sum / (reps - 3);
                printf("L=%-10lld %-9s %-26s best %8.2f us mean %8.2f us  %7.1f GB/s mean (algorithmic 16 B/elem)\n",
                       (long long)L, state ? "after-bwd" : "clean", name, best * 1e3, mean * 1e3, 16.0 * L / (mean * 1e-3) / 1e9);
            };
            for (int per : {4, 6, 8}) {
                const int g0 = sms * per;
                char nm[64];
                snprintf(nm, sizeof nm, "U1 grid %dxSM", per);
                run(nm, [&] { sgd_u<1, false><<<g0, 256>>>(th, g, n4, -1e-6f, 0.f); });
                snprintf(nm, sizeof nm, "U2 grid %dxSM", per);
                run(nm, [&] { sgd_u<2, false><<<g0, 256>>>(th, g, n4, -1e-6f, 0.f); });
                snprintf(nm, sizeof nm, "U4 grid %dxSM", per);
                run(nm, [&] { sgd_u<4, false><<<g0, 256>>>(th, g, n4, -1e-6f, 0.f); });
                snprintf(nm, sizeof nm, "U2 rev grid %dxSM", per);
                run(nm, [&] { sgd_u<2, true><<<g0, 256>>>(th, g, n4, -1e-6f, 0.f); });
            }
        }
        cudaFree(th);
        cudaFree(g);
    }
    printf("%s\n", cudaGetErrorString(cudaDeviceSynchronize()));
    return 0;
}
