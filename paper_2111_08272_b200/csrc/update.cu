// a9 — the SGD update of Eq. 1 with weight decay, fused with the gradient reset that
// starts the next aggregation (Algorithm 1 step 4 accumulates into a zeroed buffer):
//
//     d      = fma(λ, θ, ḡ)          (ḡ + λθ, one rounding)
//     θ'     = fma(−η, d, θ)         (θ − η·d, one rounding)
//     ḡ      = 0                     (if zero_grad)
//
// on the flat fp32 parameter and gradient buffers (the parameters' .data/.grad are views into them), in
// ONE pass: 16 bytes per element (read θ, ḡ; write θ, ḡ) instead of the per-tensor optimizer kernels plus a
// separate memset.  HBM-bound; float4 vectors, grid = one resident wave, grid-stride.
#include "common.h"

namespace {

__global__ void __launch_bounds__(256) sgd_kernel(float* __restrict__ th, float* __restrict__ g, int64_t n,
                                                   float nlr, float wd, int zero) {
    const int64_t n4 = n / 4;
    const int64_t stride = (int64_t)gridDim.x * blockDim.x;
    float4* t4 = reinterpret_cast<float4*>(th);
    float4* g4 = reinterpret_cast<float4*>(g);
    for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n4; i += stride) {
        float4 t = t4[i];
        const float4 d = g4[i];
        t.x = __fmaf_rn(nlr, __fmaf_rn(wd, t.x, d.x), t.x);
        t.y = __fmaf_rn(nlr, __fmaf_rn(wd, t.y, d.y), t.y);
        t.z = __fmaf_rn(nlr, __fmaf_rn(wd, t.z, d.z), t.z);
        t.w = __fmaf_rn(nlr, __fmaf_rn(wd, t.w, d.w), t.w);
        t4[i] = t;
        if (zero) g4[i] = make_float4(0.f, 0.f, 0.f, 0.f);
    }
    for (int64_t i = 4 * n4 + (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += stride) {
        th[i] = __fmaf_rn(nlr, __fmaf_rn(wd, th[i], g[i]), th[i]);
        if (zero) g[i] = 0.0f;
    }
}

}  // namespace

extern "C" int pr_sgd_update(float* d_theta, float* d_grad, int64_t n, double lr, double wd, int32_t zero_grad,
                             void* stream) {
    if (n < 0 || (n > 0 && (!d_theta || !d_grad))) return PR_ERR_INVALID;
    if (((uintptr_t)d_theta & 15) || ((uintptr_t)d_grad & 15)) return PR_ERR_ALIGN;
    if (n == 0) return PR_OK;
    // one resident wave, per device (thread-safe: a process may drive several devices)
    static std::mutex mu;
    static int grid_dev[PR_MAX_DEVICES];
    int dev = 0, grid = 0;
    PR_CUDA_TRY(cudaGetDevice(&dev));
    if (dev < 0 || dev >= PR_MAX_DEVICES) return PR_ERR_INVALID;
    {
        std::lock_guard<std::mutex> lk(mu);
        if (!grid_dev[dev]) {
            int sms = 0, per = 0;
            PR_CUDA_TRY(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev));
            PR_CUDA_TRY(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per, sgd_kernel, 256, 0));
            grid_dev[dev] = sms * (per > 0 ? per : 1);
        }
        grid = grid_dev[dev];
    }
    const int64_t need = (n / 4 + 255) / 256 + 1;
    const int blocks = (int)(need < grid ? need : grid);
    sgd_kernel<<<blocks, 256, 0, (cudaStream_t)stream>>>(d_theta, d_grad, n, (float)(-lr), (float)wd, zero_grad ? 1 : 0);
    PR_CUDA_TRY(cudaGetLastError());
    return PR_OK;
}
