// common.cuh -- shared device/host helpers of the ravgmg CUDA library (sm_100a).
#pragma once
#include <cuda_runtime.h>
#include <stdint.h>
#include <stdio.h>
#include <string>
#include <utility>

#include <nvtx3/nvToolsExt.h>

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

// NVTX range around a C-ABI call (setup / smooth / cycle phases in nsys / ncu timelines)
struct NvtxRange {
    explicit NvtxRange(const char* name) { nvtxRangePushA(name); }
    ~NvtxRange() { nvtxRangePop(); }
};

int num_sms();

// number of blocks for a grid-stride loop over `items` with `per_block` items per block,
// capped at `waves` x (#SMs x resident blocks per SM)
inline int64_t cdiv(int64_t a, int64_t b) { return (a + b - 1) / b; }

// launch counter (kernels issued by the current API call; graph replays count their nodes)
extern thread_local int64_t g_launches;
inline void count_launch(int64_t k = 1) { g_launches += k; }

// ---- programmatic dependent launch (PDL) ------------------------------------------
// The hot-loop kernels (residual, RAV sweep) let their successor launch while their last
// CTAs drain (griddepcontrol.launch_dependents at entry); the successor prefetches the
// stream data that does not depend on its predecessor into L2, then waits
// (griddepcontrol.wait: the predecessor has completed and its writes are visible).
__device__ __forceinline__ void pdl_trigger() { asm volatile("griddepcontrol.launch_dependents;" ::: "memory"); }
__device__ __forceinline__ void pdl_wait() { asm volatile("griddepcontrol.wait;" ::: "memory"); }
__device__ __forceinline__ void prefetch_l2(const void* p) { asm volatile("prefetch.global.L2 [%0];" ::"l"(p)); }
// bulk L2 prefetch by the TMA unit (one instruction, 16-byte aligned address, size a multiple of 16)
__device__ __forceinline__ void bulk_prefetch_l2(const void* p, uint32_t bytes) {
    asm volatile("cp.async.bulk.prefetch.L2.global [%0], %1;" ::"l"(p), "r"(bytes) : "memory");
}

bool pdl_enabled();

template <typename... KArgs, typename... Args>
cudaError_t launch_maybe_pdl(void (*kernel)(KArgs...), dim3 grid, dim3 block, size_t smem, cudaStream_t s,
                             Args&&... args) {
    cudaLaunchConfig_t cfg{};
    cfg.gridDim = grid;
    cfg.blockDim = block;
    cfg.dynamicSmemBytes = smem;
    cfg.stream = s;
    cudaLaunchAttribute attr[1];
    attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    attr[0].val.programmaticStreamSerializationAllowed = 1;
    cfg.attrs = attr;
    cfg.numAttrs = pdl_enabled() ? 1 : 0;
    return cudaLaunchKernelEx(&cfg, kernel, std::forward<Args>(args)...);
}

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

// the D components of a node (dof = D * node + c): one 16-byte load when D = 2 and aligned
template <int D>
__device__ __forceinline__ void ld_node(const double* __restrict__ p, double* out) {
    if (D == 2 && (reinterpret_cast<uintptr_t>(p) & 15) == 0) {
        const double2 v = __ldg(reinterpret_cast<const double2*>(p));
        out[0] = v.x;
        out[D - 1] = v.y;
    } else {
#pragma unroll
        for (int c = 0; c < D; ++c) out[c] = __ldg(p + c);
    }
}

// streaming (evict-first) loads for data read exactly once per sweep
__device__ __forceinline__ double ld_stream(const double* p) { return __ldcs(p); }
__device__ __forceinline__ double2 ld_stream2(const double2* p) { return __ldcs(p); }
__device__ __forceinline__ int ld_stream_i(const int* p) { return __ldcs(p); }

}  // namespace rav
