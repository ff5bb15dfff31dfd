// common.cuh -- shared device/host helpers of the ravgmg CUDA library (sm_100a).
#pragma once
#include <cuda_runtime.h>
#include <stdint.h>
#include <stdio.h>
#include <string>

#include "../../include/ravgmg.h"

namespace rav {

// ---- error handling ---------------------------------------------------------
void set_error(const char* fmt, ...);
const char* get_error();

#define RAV_CUDA(expr)                                                                 \
    do {                                                                               \
        cudaError_t _e = (expr);                                                       \
        if (_e != cudaSuccess) {                                                       \
            ::rav::set_error("%s:%d: %s: %s", __FILE__, __LINE__, #expr,               \
                             cudaGetErrorString(_e));                                  \
            return _e == cudaErrorMemoryAllocation ? RAV_ERR_OOM : RAV_ERR_CUDA;       \
        }                                                                              \
    } while (0)

#define RAV_CHECK_LAUNCH() RAV_CUDA(cudaGetLastError())

#define RAV_TRY(expr)                                                                  \
    do {                                                                               \
        rav_status _s = (expr);                                                        \
        if (_s != RAV_OK) return _s;                                                   \
    } while (0)

inline cudaStream_t as_stream(void* s) { return reinterpret_cast<cudaStream_t>(s); }

int num_sms();

// number of blocks for a grid-stride loop over `items` with `per_block` items per block,
// capped at `waves` x (#SMs x resident blocks per SM)
inline int64_t cdiv(int64_t a, int64_t b) { return (a + b - 1) / b; }

// launch counter (kernels issued by the current API call; graph replays count their nodes)
extern thread_local int64_t g_launches;
inline void count_launch(int64_t k = 1) { g_launches += k; }

// ---- device helpers -----------------------------------------------------------
__device__ __forceinline__ double warp_sum(double v) {
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
    return v;
}

template <int G>
__device__ __forceinline__ double group_sum(double v) {
#pragma unroll
    for (int o = G / 2; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
    return v;
}

// streaming (evict-first) loads for data read exactly once per sweep
__device__ __forceinline__ double ld_stream(const double* p) { return __ldcs(p); }
__device__ __forceinline__ double2 ld_stream2(const double2* p) { return __ldcs(p); }
__device__ __forceinline__ int ld_stream_i(const int* p) { return __ldcs(p); }

}  // namespace rav
