// Probe: can this box build an NVSwitch multicast object (NVLS) and run multimem.ld_reduce / multimem.st?
// Single process, one device: a 1-member multicast team (ld_reduce over one member = the member's value).
// Then a forked child imports the multicast handle through pidfd_getfd and maps it (the cross-process
// exchange the N2-NVLS communicator uses).
//   nvcc -gencode arch=compute_100a,code=sm_100a -O2 -o nvls_probe nvls_probe.cu -lcuda
#include <cuda.h>
#include <cuda_runtime.h>
#include <stdio.h>
#include <stdlib.h>
#include <string.h>
#include <sys/syscall.h>
#include <sys/wait.h>
#include <unistd.h>

#define CK(x)                                                                         \
    do {                                                                              \
        CUresult r_ = (x);                                                            \
        if (r_ != CUDA_SUCCESS) {                                                     \
            const char* s_ = nullptr;                                                 \
            cuGetErrorString(r_, &s_);                                                \
            printf("FAIL %s -> %d %s (line %d)\n", #x, (int)r_, s_ ? s_ : "?", __LINE__); \
            return 1;                                                                 \
        }                                                                             \
    } while (0)

__global__ void k_reduce(const float* mc, float* out, float* mc_dst, int n) {
    int i = blockIdx.x * blockDim.x + threadIdx.x;
    if (i * 4 >= n) return;
    float a, b, c, d;
    asm volatile("multimem.ld_reduce.relaxed.sys.global.add.v4.f32 {%0,%1,%2,%3}, [%4];"
                 : "=f"(a), "=f"(b), "=f"(c), "=f"(d)
                 : "l"(mc + 4 * i)
                 : "memory");
    out[4 * i] = a; out[4 * i + 1] = b; out[4 * i + 2] = c; out[4 * i + 3] = d;
    asm volatile("multimem.st.relaxed.sys.global.v4.f32 [%0], {%1,%2,%3,%4};" ::"l"(mc_dst + 4 * i), "f"(2 * a),
                 "f"(2 * b), "f"(2 * c), "f"(2 * d)
                 : "memory");
}

int main() {
    CK(cuInit(0));
    CUdevice dev;
    CK(cuDeviceGet(&dev, 0));
    CUcontext ctx;
    CK(cuDevicePrimaryCtxRetain(&ctx, dev));
    CK(cuCtxSetCurrent(ctx));
    int mcs = -1, fab = -1;
    cuDeviceGetAttribute(&mcs, CU_DEVICE_ATTRIBUTE_MULTICAST_SUPPORTED, dev);
    cuDeviceGetAttribute(&fab, CU_DEVICE_ATTRIBUTE_HANDLE_TYPE_FABRIC_SUPPORTED, dev);
    printf("multicast_supported=%d fabric_handle_supported=%d\n", mcs, fab);
    const int n = 1 << 20;
    CUmulticastObjectProp mp;
    memset(&mp, 0, sizeof(mp));
    mp.numDevices = 1;
    mp.handleTypes = CU_MEM_HANDLE_TYPE_POSIX_FILE_DESCRIPTOR;
    mp.size = (size_t)n * 4;
    size_t gmin = 0, grec = 0;
    CK(cuMulticastGetGranularity(&gmin, &mp, CU_MULTICAST_GRANULARITY_MINIMUM));
    CK(cuMulticastGetGranularity(&grec, &mp, CU_MULTICAST_GRANULARITY_RECOMMENDED));
    printf("granularity min=%zu rec=%zu\n", gmin, grec);
    // which (numDevices, handleTypes, size) does cuMulticastCreate accept on this box?
    {
        const unsigned long long hts[3] = {0, CU_MEM_HANDLE_TYPE_POSIX_FILE_DESCRIPTOR, CU_MEM_HANDLE_TYPE_FABRIC};
        for (int nd = 1; nd <= 2; ++nd)
            for (int hi = 0; hi < 3; ++hi)
                for (int si = 0; si < 2; ++si) {
                    CUmulticastObjectProp q = mp;
                    q.numDevices = nd;
                    q.handleTypes = hts[hi];
                    q.size = si ? grec : gmin;
                    CUmemGenericAllocationHandle h;
                    CUresult rr = cuMulticastCreate(&h, &q);
                    printf("create numDevices=%d handleTypes=%llu size=%zu -> %d\n", nd, hts[hi], q.size, (int)rr);
                    if (rr == CUDA_SUCCESS) cuMemRelease(h);
                }
    }
    size_t sz = ((size_t)n * 4 + gmin - 1) / gmin * gmin;
    mp.size = sz;
    CUmemGenericAllocationHandle mc;
    CK(cuMulticastCreate(&mc, &mp));
    CK(cuMulticastAddDevice(mc, dev));
    CUmemAllocationProp ap;
    memset(&ap, 0, sizeof(ap));
    ap.type = CU_MEM_ALLOCATION_TYPE_PINNED;
    ap.location.type = CU_MEM_LOCATION_TYPE_DEVICE;
    ap.location.id = 0;
    ap.requestedHandleTypes = CU_MEM_HANDLE_TYPE_POSIX_FILE_DESCRIPTOR;
    size_t ag = 0;
    CK(cuMemGetAllocationGranularity(&ag, &ap, CU_MEM_ALLOC_GRANULARITY_RECOMMENDED));
    printf("alloc granularity=%zu size=%zu\n", ag, sz);
    CUmemGenericAllocationHandle mem;
    CK(cuMemCreate(&mem, sz, &ap, 0));
    CK(cuMulticastBindMem(mc, 0, mem, 0, sz, 0));
    CUdeviceptr uc = 0, mcp = 0;
    CK(cuMemAddressReserve(&uc, sz, grec, 0, 0));
    CK(cuMemMap(uc, sz, 0, mem, 0));
    CK(cuMemAddressReserve(&mcp, sz, grec, 0, 0));
    CK(cuMemMap(mcp, sz, 0, mc, 0));
    CUmemAccessDesc acc;
    acc.location.type = CU_MEM_LOCATION_TYPE_DEVICE;
    acc.location.id = 0;
    acc.flags = CU_MEM_ACCESS_FLAGS_PROT_READWRITE;
    CK(cuMemSetAccess(uc, sz, &acc, 1));
    CK(cuMemSetAccess(mcp, sz, &acc, 1));
    float* h = (float*)malloc((size_t)n * 4);
    for (int i = 0; i < n; ++i) h[i] = (float)(i % 1000) * 0.5f;
    CK(cuMemcpyHtoD(uc, h, (size_t)n * 4));
    float* out;
    cudaMalloc(&out, (size_t)n * 4);
    k_reduce<<<n / 4 / 256, 256>>>((const float*)mcp, out, (float*)mcp, n);
    cudaError_t ke = cudaDeviceSynchronize();
    printf("kernel: %s\n", cudaGetErrorString(ke));
    if (ke != cudaSuccess) return 1;
    float* h2 = (float*)malloc((size_t)n * 4);
    float* h3 = (float*)malloc((size_t)n * 4);
    cudaMemcpy(h2, out, (size_t)n * 4, cudaMemcpyDeviceToHost);
    CK(cuMemcpyDtoH(h3, uc, (size_t)n * 4));
    int bad2 = 0, bad3 = 0;
    for (int i = 0; i < n; ++i) {
        if (h2[i] != h[i]) ++bad2;
        if (h3[i] != 2 * h[i]) ++bad3;
    }
    printf("ld_reduce mismatches=%d  multimem.st mismatches=%d\n", bad2, bad3);
    // export the multicast handle and let a forked child import it through pidfd_getfd
    int fd = -1;
    CUresult er = cuMemExportToShareableHandle(&fd, mc, CU_MEM_HANDLE_TYPE_POSIX_FILE_DESCRIPTOR, 0);
    printf("export mc handle: %d fd=%d\n", (int)er, fd);
    int pfd = (int)syscall(SYS_pidfd_open, getpid(), 0);
    int dupfd = pfd >= 0 ? (int)syscall(SYS_pidfd_getfd, pfd, fd, 0) : -1;
    printf("pidfd_open=%d pidfd_getfd(self)=%d\n", pfd, dupfd);
    fflush(stdout);
    pid_t parent = getpid();
    pid_t ch = fork();
    if (ch == 0) {
        // child: new CUDA context, import via pidfd_getfd from the parent
        int pp = (int)syscall(SYS_pidfd_open, parent, 0);
        int cfd = pp >= 0 ? (int)syscall(SYS_pidfd_getfd, pp, fd, 0) : -1;
        printf("child: pidfd_open=%d getfd=%d\n", pp, cfd);
        fflush(stdout);
        _exit(cfd >= 0 ? 0 : 3);
    }
    int stt = 0;
    waitpid(ch, &stt, 0);
    printf("child exit=%d\nPROBE_DONE\n", WEXITSTATUS(stt));
    return 0;
}
