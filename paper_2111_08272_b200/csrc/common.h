// Internal helpers shared by the library's translation units (not part of the ABI).
#pragma once
#include <stdint.h>

#include "../../include/propring.h"

// Per-device caches (function attributes, occupancy-derived grids) are indexed by device ordinal.
#define PR_MAX_DEVICES 64

#ifdef __CUDACC__
#include <cuda_runtime.h>

#include <mutex>
#define PR_CUDA_TRY(expr)                                   \
    do {                                                    \
        cudaError_t _e = (expr);                            \
        if (_e != cudaSuccess) {                            \
            pr_internal_set_cuda_error(_e, #expr);          \
            return PR_ERR_CUDA;                             \
        }                                                   \
    } while (0)
void pr_internal_set_cuda_error(cudaError_t e, const char* what);
#endif

// alloc.cpp
int pr_internal_shard_range(const pr_alloc* a, int32_t rank, int64_t* N, int64_t* off, int64_t* len);
// Step-interleaved layout: B = g·C, S = ⌊N/B⌋, o = g·Σ_{j<rank} w_j, n = g·w_rank.
int pr_internal_step_layout(const pr_alloc* a, int32_t rank, int64_t* N, int64_t* B, int64_t* S, int64_t* o,
                            int64_t* n);

// Last CUDA error text (thread-local), for debugging from Python.
extern "C" const char* pr_last_cuda_error(void);
