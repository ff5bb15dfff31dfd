// p2p.cu -- peer-memory transport for the slab exchanges (SURVEY section 8 row e: "K4 writes
// interface partials directly into the neighbor's symmetric-memory buffer (peer stores over
// NVLink), followed by a flag wait").
//
// Every rank exports its receive buffers and flag words with CUDA IPC; a neighbour imports
// them once at setup.  Per exchange, on the sender's stream: wait until the receiver has
// consumed the slot's previous use (stream wait on a flag), store the payload into the
// receiver's buffer (a copy kernel with peer stores -- over NVLink between GPUs), and
// publish the sequence number in the receiver's flag (stream write with release
// semantics).  On the receiver's stream: wait for the flag (stream wait, followed by a
// flush of remote writes where the device supports it), consume, and hand the slot back.
// No host round trip and no kernel ever spins: the waits are stream memory operations
// (cuStreamWaitValue32 / cuStreamWriteValue32, resolved through cudaGetDriverEntryPoint).
#include <cuda.h>

#include "internal.cuh"

namespace rav {
namespace {

typedef CUresult (*PFN_wait32)(CUstream, CUdeviceptr, cuuint32_t, unsigned int);
typedef CUresult (*PFN_write32)(CUstream, CUdeviceptr, cuuint32_t, unsigned int);
typedef CUresult (*PFN_devattr)(int*, CUdevice_attribute, CUdevice);

struct DriverOps {
    PFN_wait32 wait = nullptr;
    PFN_write32 write = nullptr;
    unsigned int wait_flags = CU_STREAM_WAIT_VALUE_GEQ;
    bool ok = false;
};

static const DriverOps& driver_ops() {
    static DriverOps ops = [] {
        DriverOps o;
        cudaDriverEntryPointQueryResult q;
        void* fn = nullptr;
        if (cudaGetDriverEntryPoint("cuStreamWaitValue32", &fn, cudaEnableDefault, &q) == cudaSuccess &&
            q == cudaDriverEntryPointSuccess)
            o.wait = reinterpret_cast<PFN_wait32>(fn);
        fn = nullptr;
        if (cudaGetDriverEntryPoint("cuStreamWriteValue32", &fn, cudaEnableDefault, &q) == cudaSuccess &&
            q == cudaDriverEntryPointSuccess)
            o.write = reinterpret_cast<PFN_write32>(fn);
        fn = nullptr;
        int dev = 0, flush = 0;
        cudaGetDevice(&dev);
        if (cudaGetDriverEntryPoint("cuDeviceGetAttribute", &fn, cudaEnableDefault, &q) == cudaSuccess &&
            q == cudaDriverEntryPointSuccess &&
            reinterpret_cast<PFN_devattr>(fn)(&flush, CU_DEVICE_ATTRIBUTE_CAN_FLUSH_REMOTE_WRITES, dev) ==
                CUDA_SUCCESS &&
            flush)
            o.wait_flags |= CU_STREAM_WAIT_VALUE_FLUSH;
        cudaGetLastError();
        o.ok = o.wait && o.write;
        return o;
    }();
    return ops;
}

__global__ void copy_kernel(int64_t n, const double* __restrict__ src, double* __restrict__ dst) {
    for (int64_t k = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; k < n; k += (int64_t)gridDim.x * blockDim.x)
        dst[k] = src[k];
}

}  // namespace
}  // namespace rav

using namespace rav;

extern "C" {

rav_status rav_device_alloc(int64_t bytes, void** dev_ptr) {
    if (bytes <= 0 || !dev_ptr) { set_error("rav_device_alloc: bad argument"); return RAV_ERR_ARG; }
    RAV_CUDA(cudaMalloc(dev_ptr, (size_t)bytes));
    RAV_CUDA(cudaMemset(*dev_ptr, 0, (size_t)bytes));
    return RAV_OK;
}

rav_status rav_device_free(void* dev_ptr) {
    if (dev_ptr) RAV_CUDA(cudaFree(dev_ptr));
    return RAV_OK;
}

rav_status rav_ipc_export(void* dev_ptr, unsigned char* handle) {
    if (!dev_ptr || !handle) { set_error("rav_ipc_export: NULL argument"); return RAV_ERR_ARG; }
    cudaIpcMemHandle_t h;
    RAV_CUDA(cudaIpcGetMemHandle(&h, dev_ptr));
    memcpy(handle, &h, sizeof(h));
    return RAV_OK;
}

rav_status rav_ipc_import(const unsigned char* handle, void** dev_ptr) {
    if (!handle || !dev_ptr) { set_error("rav_ipc_import: NULL argument"); return RAV_ERR_ARG; }
    cudaIpcMemHandle_t h;
    memcpy(&h, handle, sizeof(h));
    RAV_CUDA(cudaIpcOpenMemHandle(dev_ptr, h, cudaIpcMemLazyEnablePeerAccess));
    return RAV_OK;
}

rav_status rav_ipc_close(void* dev_ptr) {
    if (!dev_ptr) return RAV_OK;
    RAV_CUDA(cudaIpcCloseMemHandle(dev_ptr));
    return RAV_OK;
}

rav_status rav_stream_wait(void* stream, uint32_t* flag, uint32_t value) {
    const DriverOps& o = driver_ops();
    if (!o.ok) { set_error("rav_stream_wait: stream memory operations unavailable"); return RAV_ERR_CUDA; }
    if (!flag) { set_error("rav_stream_wait: NULL flag"); return RAV_ERR_ARG; }
    if (o.wait(reinterpret_cast<CUstream>(stream), reinterpret_cast<CUdeviceptr>(flag), value, o.wait_flags) !=
        CUDA_SUCCESS) {
        set_error("rav_stream_wait: cuStreamWaitValue32 failed");
        return RAV_ERR_CUDA;
    }
    return RAV_OK;
}

rav_status rav_stream_signal(void* stream, uint32_t* flag, uint32_t value) {
    const DriverOps& o = driver_ops();
    if (!o.ok) { set_error("rav_stream_signal: stream memory operations unavailable"); return RAV_ERR_CUDA; }
    if (!flag) { set_error("rav_stream_signal: NULL flag"); return RAV_ERR_ARG; }
    if (o.write(reinterpret_cast<CUstream>(stream), reinterpret_cast<CUdeviceptr>(flag), value,
                CU_STREAM_WRITE_VALUE_DEFAULT) != CUDA_SUCCESS) {
        set_error("rav_stream_signal: cuStreamWriteValue32 failed");
        return RAV_ERR_CUDA;
    }
    return RAV_OK;
}

rav_status rav_peer_put(const double* src, double* remote_dst, int64_t n, void* stream) {
    if (n < 0 || (n > 0 && (!src || !remote_dst))) { set_error("rav_peer_put: bad argument"); return RAV_ERR_ARG; }
    g_launches = 0;
    if (n == 0) return RAV_OK;
    const int blocks = (int)std::min<int64_t>(cdiv(n, 256), (int64_t)num_sms() * 4);
    copy_kernel<<<blocks, 256, 0, as_stream(stream)>>>(n, src, remote_dst);
    count_launch();
    RAV_CHECK_LAUNCH();
    return RAV_OK;
}

}  // extern "C"
