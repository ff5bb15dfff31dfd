// linalg.cu -- CSR kernels of the hot path (SURVEY section 8 rows a2 "residual
// SpMV" and a7 "transfers"): r = b - L x (Eq. 10), y = alpha A x + beta y,
// deterministic residual norms, CSR upload / transpose.
//
// Layout: CSR with int64 row pointers and int32 sorted columns.  A group of G
// lanes (G = 8 for the ~25-nnz rows of 2D Q2-Q1, 32 for the ~90-375-nnz rows
// of 3D) owns one row; consecutive groups own consecutive rows, so a warp
// streams one contiguous range of val/col with no padding.  val/col are read
// with evict-first streaming loads (they are touched once per sweep); x is
// read through L1/L2 (it is L2-resident between the sweep and the residual).
#include <cub/cub.cuh>

#include "internal.cuh"

namespace rav {

template <int G>
__global__ void __launch_bounds__(256) residual_kernel(int64_t n, const int64_t* __restrict__ rp,
                                                       const int32_t* __restrict__ ci,
                                                       const double* __restrict__ val,
                                                       const double* __restrict__ x,
                                                       const double* __restrict__ b, double* __restrict__ r) {
    // warp-uniform trip count: every lane reaches the shuffles (rows past n are masked)
    const int lane = threadIdx.x % G;
    const int64_t groups = (int64_t)gridDim.x * (blockDim.x / G);
    const int64_t first = (int64_t)blockIdx.x * (blockDim.x / G) + threadIdx.x / G;
    const int64_t warp_first = first - (threadIdx.x % 32) / G;
    for (int64_t base = warp_first; base < n; base += groups) {
        const int64_t row = base + (threadIdx.x % 32) / G;
        double acc = 0.0;
        if (row < n) {
            const int64_t s = rp[row], e = rp[row + 1];
            for (int64_t k = s + lane; k < e; k += G) acc += ld_stream(val + k) * __ldg(x + ld_stream_i(ci + k));
        }
        acc = group_sum<G>(acc);
        if (lane == 0 && row < n) r[row] = b[row] - acc;
    }
}

template <int G>
__global__ void __launch_bounds__(256) spmv_kernel(int64_t n, const int64_t* __restrict__ rp,
                                                   const int32_t* __restrict__ ci,
                                                   const double* __restrict__ val,
                                                   const double* __restrict__ x, double* __restrict__ y,
                                                   double alpha, double beta) {
    const int lane = threadIdx.x % G;
    const int64_t groups = (int64_t)gridDim.x * (blockDim.x / G);
    const int64_t first = (int64_t)blockIdx.x * (blockDim.x / G) + threadIdx.x / G;
    const int64_t warp_first = first - (threadIdx.x % 32) / G;
    for (int64_t base = warp_first; base < n; base += groups) {
        const int64_t row = base + (threadIdx.x % 32) / G;
        double acc = 0.0;
        if (row < n) {
            const int64_t s = rp[row], e = rp[row + 1];
            for (int64_t k = s + lane; k < e; k += G) acc += ld_stream(val + k) * __ldg(x + ld_stream_i(ci + k));
        }
        acc = group_sum<G>(acc);
        if (lane == 0 && row < n) y[row] = (beta == 0.0 ? 0.0 : beta * y[row]) + alpha * acc;
    }
}


// sum of squares of (b - A x) per block (fixed order => deterministic)
template <int G>
__global__ void __launch_bounds__(256) resnorm_kernel(int64_t n, const int64_t* __restrict__ rp,
                                                      const int32_t* __restrict__ ci,
                                                      const double* __restrict__ val,
                                                      const double* __restrict__ x,
                                                      const double* __restrict__ b, double* __restrict__ part) {
    __shared__ double red[256 / G];
    const int lane = threadIdx.x % G, grp = threadIdx.x / G;
    const int64_t groups = (int64_t)gridDim.x * (blockDim.x / G);
    double mine = 0.0;
    const int64_t first = (int64_t)blockIdx.x * (blockDim.x / G) + grp;
    const int64_t warp_first = first - (threadIdx.x % 32) / G;
    for (int64_t base = warp_first; base < n; base += groups) {
        const int64_t row = base + (threadIdx.x % 32) / G;
        double acc = 0.0;
        if (row < n) {
            const int64_t s = rp[row], e = rp[row + 1];
            for (int64_t k = s + lane; k < e; k += G) acc += ld_stream(val + k) * __ldg(x + ld_stream_i(ci + k));
        }
        acc = group_sum<G>(acc);
        if (row < n) {
            double rr = b[row] - acc;
            mine += rr * rr;
        }
    }
    if (lane == 0) red[grp] = mine;
    __syncthreads();
    if (threadIdx.x == 0) {
        double t = 0.0;
        for (int i = 0; i < 256 / G; ++i) t += red[i];
        part[blockIdx.x] = t;
    }
}

// one CTA of 1024 threads, four independent accumulators per thread (fixed order: deterministic);
// a full c3 grid has 82k partials, which one 256-thread serial chain took 147 us to sum
__global__ void __launch_bounds__(1024) sum_parts_kernel(const double* __restrict__ part, int nblk, double* out) {
    __shared__ double red[1024];
    double t0 = 0.0, t1 = 0.0, t2 = 0.0, t3 = 0.0;
    int i = threadIdx.x;
    for (; i + 3 * 1024 < nblk; i += 4 * 1024) {
        t0 += part[i];
        t1 += part[i + 1024];
        t2 += part[i + 2 * 1024];
        t3 += part[i + 3 * 1024];
    }
    for (; i < nblk; i += 1024) t0 += part[i];
    red[threadIdx.x] = (t0 + t1) + (t2 + t3);
    __syncthreads();
    for (int o = 512; o > 0; o >>= 1) {
        if (threadIdx.x < o) red[threadIdx.x] += red[threadIdx.x + o];
        __syncthreads();
    }
    if (threadIdx.x == 0) *out = red[0];
}

static int spmv_blocks(int64_t n, int G) {
    int64_t rows_per_block = 256 / G;
    int64_t b = cdiv(n, rows_per_block);
    int64_t cap = (int64_t)num_sms() * 8;
    return (int)(b < 1 ? 1 : (b > cap ? cap : b));
}

rav_status launch_residual(const Csr& A, const double* x, const double* b, double* r, cudaStream_t s,
                           const void* xpf, int64_t xpf_bytes) {
    if (A.n_rows == 0) return RAV_OK;
    if (A.nb.nslices > 0) return launch_nb_residual(A, x, b, r, nullptr, 0, s, nullptr, xpf, xpf_bytes);
    if (A.sell.nslices > 0) return launch_sell_residual(A, x, b, r, nullptr, 0, s);
    int nb = spmv_blocks(A.n_rows, A.lanes);
    if (A.lanes == 32)
        residual_kernel<32><<<nb, 256, 0, s>>>(A.n_rows, A.rp, A.ci, A.val, x, b, r);
    else if (A.lanes == 16)
        residual_kernel<16><<<nb, 256, 0, s>>>(A.n_rows, A.rp, A.ci, A.val, x, b, r);
    else
        residual_kernel<8><<<nb, 256, 0, s>>>(A.n_rows, A.rp, A.ci, A.val, x, b, r);
    count_launch();
    RAV_CHECK_LAUNCH();
    return RAV_OK;
}

rav_status launch_spmv(const Csr& A, const double* x, double* y, double alpha, double beta, cudaStream_t s) {
    if (A.n_rows == 0) return RAV_OK;
    // transfers (P: 1-9 entries per row, R = P^T: up to ~25) are short-row matrices: lanes per row
    // from the mean row length, one pass of the whole grid (no grid-stride cap)
    const double mean = (double)A.nnz / (double)A.n_rows;
    const int G = mean > 48.0 ? 32 : (mean > 12.0 ? 8 : (mean > 5.0 ? 4 : 2));
    const int nb = (int)std::max<int64_t>(1, std::min<int64_t>(cdiv(A.n_rows * G, 256), (int64_t)1 << 30));
    if (G == 32)
        spmv_kernel<32><<<nb, 256, 0, s>>>(A.n_rows, A.rp, A.ci, A.val, x, y, alpha, beta);
    else if (G == 8)
        spmv_kernel<8><<<nb, 256, 0, s>>>(A.n_rows, A.rp, A.ci, A.val, x, y, alpha, beta);
    else if (G == 4)
        spmv_kernel<4><<<nb, 256, 0, s>>>(A.n_rows, A.rp, A.ci, A.val, x, y, alpha, beta);
    else
        spmv_kernel<2><<<nb, 256, 0, s>>>(A.n_rows, A.rp, A.ci, A.val, x, y, alpha, beta);
    count_launch();
    RAV_CHECK_LAUNCH();
    return RAV_OK;
}

int residual_norm_blocks() { return num_sms() * 4; }

// r = b - A x and *out = ||r||^2 in one pass over A when a fused kernel exists (node-blocked / SELL)
int64_t residual_part_capacity(const Csr& A) {
    int64_t c = residual_norm_blocks();
    if (A.nb.nslices > 0) c = std::max(c, nb_full_blocks(A.nb));
    if (A.sell.nslices > 0) c = std::max(c, sell_full_blocks(A.sell));
    return c;
}

rav_status launch_residual_and_norm2(const Csr& A, const double* x, const double* b, double* r, double* part,
                                     int nblk, double* out, cudaStream_t s) {
    if (A.nb.nslices > 0 || A.sell.nslices > 0) {
        int used = nblk;
        if (A.nb.nslices > 0) RAV_TRY(launch_nb_residual(A, x, b, r, part, nblk, s, &used));
        else RAV_TRY(launch_sell_residual(A, x, b, r, part, nblk, s, &used));
        sum_parts_kernel<<<1, 1024, 0, s>>>(part, used, out);
        count_launch();
        RAV_CHECK_LAUNCH();
        return RAV_OK;
    }
    RAV_TRY(launch_residual(A, x, b, r, s));
    return launch_dot(r, r, A.n_rows, part, nblk, out, 0, s);
}

rav_status launch_residual_norm2(const Csr& A, const double* x, const double* b, double* part, int nblk,
                                 double* out, cudaStream_t s) {
    if (A.nb.nslices > 0 || A.sell.nslices > 0) {
        int used = nblk;
        if (A.nb.nslices > 0) RAV_TRY(launch_nb_residual(A, x, b, nullptr, part, nblk, s, &used));
        else RAV_TRY(launch_sell_residual(A, x, b, nullptr, part, nblk, s, &used));
        sum_parts_kernel<<<1, 1024, 0, s>>>(part, used, out);
        count_launch();
        RAV_CHECK_LAUNCH();
        return RAV_OK;
    }
    if (A.lanes == 32)
        resnorm_kernel<32><<<nblk, 256, 0, s>>>(A.n_rows, A.rp, A.ci, A.val, x, b, part);
    else if (A.lanes == 16)
        resnorm_kernel<16><<<nblk, 256, 0, s>>>(A.n_rows, A.rp, A.ci, A.val, x, b, part);
    else
        resnorm_kernel<8><<<nblk, 256, 0, s>>>(A.n_rows, A.rp, A.ci, A.val, x, b, part);
    count_launch();
    RAV_CHECK_LAUNCH();
    sum_parts_kernel<<<1, 1024, 0, s>>>(part, nblk, out);
    count_launch();
    RAV_CHECK_LAUNCH();
    return RAV_OK;
}

// partial dot products per block (fixed order => deterministic)
__global__ void __launch_bounds__(256) dot_kernel(int64_t n, const double* __restrict__ a,
                                                  const double* __restrict__ b, double* __restrict__ part) {
    __shared__ double red[8];
    double t = 0.0;
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x)
        t = fma(a[i], b[i], t);
    t = warp_sum(t);
    if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = t;
    __syncthreads();
    if (threadIdx.x == 0) {
        double u = 0.0;
        for (int w = 0; w < 8; ++w) u += red[w];
        part[blockIdx.x] = u;
    }
}

__global__ void sum_parts_acc_kernel(const double* __restrict__ part, int nblk, double* out, int accumulate) {
    __shared__ double red[256];
    double t = 0.0;
    for (int i = threadIdx.x; i < nblk; i += blockDim.x) t += part[i];
    red[threadIdx.x] = t;
    __syncthreads();
    for (int o = 128; o > 0; o >>= 1) {
        if (threadIdx.x < o) red[threadIdx.x] += red[threadIdx.x + o];
        __syncthreads();
    }
    if (threadIdx.x == 0) *out = accumulate ? *out + red[0] : red[0];
}

rav_status launch_dot(const double* a, const double* b, int64_t n, double* part, int nblk, double* out,
                      int accumulate, cudaStream_t s) {
    const int blocks = (int)std::max<int64_t>(1, std::min<int64_t>(cdiv(std::max<int64_t>(n, 1), 256), nblk));
    dot_kernel<<<blocks, 256, 0, s>>>(n, a, b, part);
    count_launch();
    RAV_CHECK_LAUNCH();
    sum_parts_acc_kernel<<<1, 256, 0, s>>>(part, blocks, out, accumulate);
    count_launch();
    RAV_CHECK_LAUNCH();
    return RAV_OK;
}

// w[k] += alpha * sum_{i < nv} coef[i] * V[i * ld + k]   (coef on the device; Krylov updates)
__global__ void __launch_bounds__(256) multi_axpy_kernel(int64_t n, int nv, const double* __restrict__ V, int64_t ld,
                                                         const double* __restrict__ coef, double alpha,
                                                         double* __restrict__ w) {
    for (int64_t k = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; k < n; k += (int64_t)gridDim.x * blockDim.x) {
        double s = 0.0;
        for (int i = 0; i < nv; ++i) s = fma(coef[i], V[i * ld + k], s);
        w[k] = fma(alpha, s, w[k]);
    }
}

// out[i] = sum_k V[i ld + k] w[k] for i < nv <= MD_NV in one pass over w and the nv vectors
// (Gram-Schmidt of FGMRES); per-block partials part[b MD_NV + i], summed in fixed block order
constexpr int MD_NV = 32;
__global__ void __launch_bounds__(256, 2) multi_dot_kernel(int64_t n, int nv, const double* __restrict__ V, int64_t ld,
                                                        const double* __restrict__ w, double* __restrict__ part) {
    double acc[MD_NV];
#pragma unroll
    for (int i = 0; i < MD_NV; ++i) acc[i] = 0.0;
    for (int64_t k = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; k < n; k += (int64_t)gridDim.x * blockDim.x) {
        const double wk = w[k];
#pragma unroll
        for (int i = 0; i < MD_NV; ++i)
            if (i < nv) acc[i] = fma(V[i * ld + k], wk, acc[i]);
    }
    __shared__ double red[8][MD_NV];
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
#pragma unroll
    for (int i = 0; i < MD_NV; ++i) {
        if (i < nv) {
            const double v = warp_sum(acc[i]);
            if (lane == 0) red[warp][i] = v;
        }
    }
    __syncthreads();
    if (threadIdx.x < nv) {
        double t = 0.0;
        for (int q = 0; q < 8; ++q) t += red[q][threadIdx.x];
        part[(int64_t)blockIdx.x * MD_NV + threadIdx.x] = t;
    }
}

__global__ void multi_dot_sum_kernel(int nblk, int nv, const double* __restrict__ part, double* __restrict__ out) {
    if (threadIdx.x < nv) {
        double t = 0.0;
        for (int b = 0; b < nblk; ++b) t += part[(int64_t)b * MD_NV + threadIdx.x];
        out[threadIdx.x] = t;
    }
}

int multi_dot_max() { return MD_NV; }
int multi_dot_blocks() { return num_sms() * 4; }

rav_status launch_multi_dot(int64_t n, int nv, const double* V, int64_t ld, const double* w, double* part, double* out,
                            cudaStream_t s) {
    if (nv <= 0) return RAV_OK;
    if (nv > MD_NV) { set_error("multi_dot: at most %d vectors", MD_NV); return RAV_ERR_ARG; }
    const int blocks = (int)std::max<int64_t>(1, std::min<int64_t>(cdiv(std::max<int64_t>(n, 1), 256), multi_dot_blocks()));
    multi_dot_kernel<<<blocks, 256, 0, s>>>(n, nv, V, ld, w, part);
    count_launch();
    multi_dot_sum_kernel<<<1, 32, 0, s>>>(blocks, nv, part, out);
    count_launch();
    RAV_CHECK_LAUNCH();
    return RAV_OK;
}

__global__ void scale_kernel(int64_t n, const double* __restrict__ src, double s, double* __restrict__ dst) {
    for (int64_t k = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; k < n; k += (int64_t)gridDim.x * blockDim.x)
        dst[k] = s * src[k];
}

rav_status launch_multi_axpy(int64_t n, int nv, const double* V, int64_t ld, const double* coef, double alpha,
                             double* w, cudaStream_t s) {
    if (n == 0 || nv == 0) return RAV_OK;
    const int blocks = (int)std::min<int64_t>(cdiv(n, 256), (int64_t)num_sms() * 8);
    multi_axpy_kernel<<<blocks, 256, 0, s>>>(n, nv, V, ld, coef, alpha, w);
    count_launch();
    RAV_CHECK_LAUNCH();
    return RAV_OK;
}

rav_status launch_scale(int64_t n, const double* src, double sc, double* dst, cudaStream_t s) {
    if (n == 0) return RAV_OK;
    const int blocks = (int)std::min<int64_t>(cdiv(n, 256), (int64_t)num_sms() * 8);
    scale_kernel<<<blocks, 256, 0, s>>>(n, src, sc, dst);
    count_launch();
    RAV_CHECK_LAUNCH();
    return RAV_OK;
}

// pack / unpack for the slab exchanges
__global__ void index_op_kernel(int op, const double* __restrict__ src, const int32_t* __restrict__ idx, int64_t n,
                                double* __restrict__ dst, double value) {
    for (int64_t k = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; k < n; k += (int64_t)gridDim.x * blockDim.x) {
        const int32_t i = idx[k];
        if (op == 0) dst[k] = src[i];
        else if (op == 1) dst[i] = src[k];
        else if (op == 2) dst[i] += src[k];
        else if (op == 4) dst[k] = src[i] - dst[k];
        else dst[i] = value;
    }
}

static bool is_device_ptr(const void* p) {
    cudaPointerAttributes a;
    if (cudaPointerGetAttributes(&a, p) != cudaSuccess) { cudaGetLastError(); return false; }
    return a.type == cudaMemoryTypeDevice || a.type == cudaMemoryTypeManaged;
}

__global__ void row_len_max_kernel(int64_t n, const int64_t* rp, unsigned long long* mx, unsigned long long* sum) {
    unsigned long long m = 0, t = 0;
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
        unsigned long long l = (unsigned long long)(rp[i + 1] - rp[i]);
        m = l > m ? l : m;
        t += l;
    }
    atomicMax(mx, m);
    (void)sum;
    (void)t;
}

// input validation of a CSR (include/ravgmg.h: "columns sorted ascending within each row"):
// bit 0: row_ptr not monotone / not starting at 0, bit 1: column out of range, bit 2: columns
// not strictly increasing within a row
__global__ void csr_check_kernel(int64_t n, int64_t ncols, const int64_t* rp, const int32_t* ci, unsigned int* err) {
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
        const int64_t a = rp[i], b = rp[i + 1];
        if ((i == 0 && a != 0) || b < a) { atomicOr(err, 1u); continue; }
        for (int64_t k = a; k < b; ++k) {
            const int32_t c = ci[k];
            if (c < 0 || c >= ncols) atomicOr(err, 2u);
            if (k > a && c <= ci[k - 1]) atomicOr(err, 4u);
        }
    }
}

rav_status csr_upload(const rav_csr* A, Csr& out, cudaStream_t s) {
    if (!A || A->n_rows < 0 || !A->row_ptr) { set_error("rav_csr: NULL or negative size"); return RAV_ERR_ARG; }
    out.n_rows = A->n_rows;
    out.n_cols = A->n_cols;
    int64_t nnz = 0;
    cudaMemcpyKind kind = A->on_device ? cudaMemcpyDeviceToDevice : cudaMemcpyHostToDevice;
    if (A->on_device != is_device_ptr(A->row_ptr)) {
        set_error("rav_csr: on_device flag does not match the row_ptr pointer kind");
        return RAV_ERR_ARG;
    }
    RAV_CUDA(cudaMemcpyAsync(&nnz, A->row_ptr + A->n_rows, sizeof(int64_t),
                             A->on_device ? cudaMemcpyDeviceToHost : cudaMemcpyHostToHost, s));
    RAV_CUDA(cudaStreamSynchronize(s));
    if (nnz < 0) { set_error("rav_csr: negative nnz"); return RAV_ERR_ARG; }
    out.nnz = nnz;
    RAV_CUDA(cudaMalloc(&out.rp, sizeof(int64_t) * (out.n_rows + 1)));
    RAV_CUDA(cudaMalloc(&out.ci, sizeof(int32_t) * (nnz > 0 ? nnz : 1)));
    RAV_CUDA(cudaMalloc(&out.val, sizeof(double) * (nnz > 0 ? nnz : 1)));
    RAV_CUDA(cudaMemcpyAsync(out.rp, A->row_ptr, sizeof(int64_t) * (out.n_rows + 1), kind, s));
    if (nnz > 0) {
        RAV_CUDA(cudaMemcpyAsync(out.ci, A->col, sizeof(int32_t) * nnz, kind, s));
        RAV_CUDA(cudaMemcpyAsync(out.val, A->val, sizeof(double) * nnz, kind, s));
    }
    if (out.n_rows > 0) {
        unsigned int* err = nullptr;
        RAV_CUDA(cudaMallocAsync(&err, sizeof(unsigned int), s));
        RAV_CUDA(cudaMemsetAsync(err, 0, sizeof(unsigned int), s));
        const int nb = (int)std::min<int64_t>(cdiv(out.n_rows, 256), (int64_t)num_sms() * 16);
        csr_check_kernel<<<nb, 256, 0, s>>>(out.n_rows, out.n_cols, out.rp, out.ci, err);
        count_launch();
        RAV_CHECK_LAUNCH();
        unsigned int h_err = 0;
        RAV_CUDA(cudaMemcpyAsync(&h_err, err, sizeof(h_err), cudaMemcpyDeviceToHost, s));
        cudaFreeAsync(err, s);
        RAV_CUDA(cudaStreamSynchronize(s));
        if (h_err) {
            set_error("rav_csr: %s", (h_err & 1) ? "row_ptr must start at 0 and be non-decreasing"
                                     : (h_err & 2) ? "column index out of range"
                                                   : "columns must be strictly increasing within a row");
            csr_free(out);
            return RAV_ERR_ARG;
        }
    }
    // lanes per row from the mean row length
    double mean = out.n_rows > 0 ? (double)nnz / (double)out.n_rows : 0.0;
    out.lanes = mean > 64.0 ? 32 : (mean > 24.0 ? 8 : 8);
    if (mean > 64.0) out.lanes = 32;
    RAV_CUDA(cudaStreamSynchronize(s));
    return RAV_OK;
}

void csr_free(Csr& A) {
    sell_free(A.sell);
    nb_free(A.nb);
    if (A.rp) cudaFree(A.rp);
    if (A.ci) cudaFree(A.ci);
    if (A.val) cudaFree(A.val);
    A.rp = nullptr;
    A.ci = nullptr;
    A.val = nullptr;
}

__global__ void col_count_kernel(int64_t nnz, const int32_t* ci, int64_t* cnt) {
    for (int64_t k = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; k < nnz; k += (int64_t)gridDim.x * blockDim.x)
        atomicAdd((unsigned long long*)(cnt + ci[k]), 1ULL);
}

__global__ void transpose_fill_kernel(int64_t n, const int64_t* rp, const int32_t* ci, const double* val,
                                      const int64_t* trp, int64_t* cursor, int32_t* tci, double* tval) {
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x)
        for (int64_t k = rp[i]; k < rp[i + 1]; ++k) {
            int64_t c = ci[k];
            int64_t p = trp[c] + (int64_t)atomicAdd((unsigned long long*)(cursor + c), 1ULL);
            tci[p] = (int32_t)i;
            tval[p] = val[k];
        }
}

// insertion sort of each transposed row by column => deterministic order
__global__ void row_sort_kernel(int64_t n, const int64_t* rp, int32_t* ci, double* val) {
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
        int64_t s = rp[i], e = rp[i + 1];
        for (int64_t a = s + 1; a < e; ++a) {
            int32_t kc = ci[a];
            double kv = val[a];
            int64_t b = a - 1;
            while (b >= s && ci[b] > kc) { ci[b + 1] = ci[b]; val[b + 1] = val[b]; --b; }
            ci[b + 1] = kc;
            val[b + 1] = kv;
        }
    }
}

rav_status csr_transpose(const Csr& A, Csr& At, cudaStream_t s) {
    At.n_rows = A.n_cols;
    At.n_cols = A.n_rows;
    At.nnz = A.nnz;
    int64_t *cnt = nullptr, *cursor = nullptr;
    RAV_CUDA(cudaMalloc(&At.rp, sizeof(int64_t) * (At.n_rows + 1)));
    RAV_CUDA(cudaMalloc(&At.ci, sizeof(int32_t) * (A.nnz > 0 ? A.nnz : 1)));
    RAV_CUDA(cudaMalloc(&At.val, sizeof(double) * (A.nnz > 0 ? A.nnz : 1)));
    RAV_CUDA(cudaMallocAsync(&cnt, sizeof(int64_t) * (At.n_rows > 0 ? At.n_rows : 1), s));
    RAV_CUDA(cudaMallocAsync(&cursor, sizeof(int64_t) * (At.n_rows > 0 ? At.n_rows : 1), s));
    RAV_CUDA(cudaMemsetAsync(cnt, 0, sizeof(int64_t) * At.n_rows, s));
    RAV_CUDA(cudaMemsetAsync(cursor, 0, sizeof(int64_t) * At.n_rows, s));
    int nb = (int)std::min<int64_t>(cdiv(A.nnz > 0 ? A.nnz : 1, 256), (int64_t)num_sms() * 16);
    col_count_kernel<<<nb, 256, 0, s>>>(A.nnz, A.ci, cnt);
    count_launch();
    RAV_CHECK_LAUNCH();
    RAV_TRY(gen::counts_to_rowptr(cnt, At.rp, At.n_rows, s));
    int nbr = (int)std::min<int64_t>(cdiv(A.n_rows > 0 ? A.n_rows : 1, 256), (int64_t)num_sms() * 16);
    transpose_fill_kernel<<<nbr, 256, 0, s>>>(A.n_rows, A.rp, A.ci, A.val, At.rp, cursor, At.ci, At.val);
    count_launch();
    RAV_CHECK_LAUNCH();
    int nbt = (int)std::min<int64_t>(cdiv(At.n_rows > 0 ? At.n_rows : 1, 256), (int64_t)num_sms() * 16);
    row_sort_kernel<<<nbt, 256, 0, s>>>(At.n_rows, At.rp, At.ci, At.val);
    count_launch();
    RAV_CHECK_LAUNCH();
    cudaFreeAsync(cnt, s);
    cudaFreeAsync(cursor, s);
    double mean = At.n_rows > 0 ? (double)At.nnz / At.n_rows : 0.0;
    At.lanes = mean > 64.0 ? 32 : 8;
    RAV_CUDA(cudaStreamSynchronize(s));
    return RAV_OK;
}

}  // namespace rav

extern "C" rav_status rav_index_op(int op, const double* src, const int32_t* idx, int64_t n, double* dst,
                                   double value, void* stream) {
    using namespace rav;
    if (op < 0 || op > 4 || n < 0 || (n > 0 && (!idx || !dst || (op != 3 && !src)))) {
        set_error("rav_index_op: bad argument");
        return RAV_ERR_ARG;
    }
    g_launches = 0;
    if (n == 0) return RAV_OK;
    const int blocks = (int)std::min<int64_t>(cdiv(n, 256), (int64_t)num_sms() * 8);
    index_op_kernel<<<blocks, 256, 0, as_stream(stream)>>>(op, src, idx, n, dst, value);
    count_launch();
    RAV_CHECK_LAUNCH();
    return RAV_OK;
}

// ------------------------------------------------------------------------------------
// pressure normalisation (reading R4)
// ------------------------------------------------------------------------------------
namespace rav {

// s[0] = the shift: mode 0 x[pin], mode 1 the mean of x[n_vel .. n) (partials summed in fixed
// block order, so the result is bitwise reproducible)
__global__ void pressure_shift_kernel(int64_t np, double* __restrict__ xp, const double* __restrict__ s,
                                      double scale) {
    const double sh = s[0] * scale;
    for (int64_t k = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; k < np; k += (int64_t)gridDim.x * blockDim.x)
        xp[k] -= sh;
}

__global__ void __launch_bounds__(256) sum_kernel(int64_t n, const double* __restrict__ a, double* __restrict__ part) {
    __shared__ double red[8];
    double t = 0.0;
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x)
        t += a[i];
    t = warp_sum(t);
    if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = t;
    __syncthreads();
    if (threadIdx.x == 0) {
        double u = 0.0;
        for (int w = 0; w < 8; ++w) u += red[w];
        part[blockIdx.x] = u;
    }
}

// shift: one device double; part: >= residual_norm_blocks() doubles of device scratch
rav_status launch_pressure_normalize(double* x, int64_t n_vel, int64_t n, int mode, int64_t pin, double* shift,
                                     double* part, cudaStream_t s) {
    const int64_t np = n - n_vel;
    if (np <= 0) return RAV_OK;
    double scale = 1.0;
    if (mode == 0) {
        RAV_CUDA(cudaMemcpyAsync(shift, x + pin, sizeof(double), cudaMemcpyDeviceToDevice, s));
    } else {
        const int nblk = residual_norm_blocks();
        const int blocks = (int)std::max<int64_t>(1, std::min<int64_t>(cdiv(np, 256), nblk));
        sum_kernel<<<blocks, 256, 0, s>>>(np, x + n_vel, part);
        count_launch();
        RAV_CHECK_LAUNCH();
        sum_parts_acc_kernel<<<1, 256, 0, s>>>(part, blocks, shift, 0);
        count_launch();
        RAV_CHECK_LAUNCH();
        scale = 1.0 / (double)np;
    }
    const int blocks = (int)std::min<int64_t>(cdiv(np, 256), (int64_t)num_sms() * 8);
    pressure_shift_kernel<<<blocks, 256, 0, s>>>(np, x + n_vel, shift, scale);
    count_launch();
    RAV_CHECK_LAUNCH();
    return RAV_OK;
}

}  // namespace rav

extern "C" rav_status rav_pressure_normalize(double* x, int64_t n_vel, int64_t n, int mode, int64_t pin,
                                             void* stream) {
    using namespace rav;
    if (!x || n_vel < 0 || n < n_vel || (mode != 0 && mode != 1) || (mode == 0 && (pin < n_vel || pin >= n))) {
        set_error("rav_pressure_normalize: bad argument (need 0 <= n_vel <= n, mode 0/1, n_vel <= pin < n for mode 0)");
        return RAV_ERR_ARG;
    }
    if (!is_device_ptr(x)) { set_error("rav_pressure_normalize: x must be a device pointer"); return RAV_ERR_ARG; }
    g_launches = 0;
    static thread_local double* work = nullptr;
    if (!work) RAV_CUDA(cudaMalloc(&work, sizeof(double) * (residual_norm_blocks() + 1)));
    return launch_pressure_normalize(x, n_vel, n, mode, pin, work, work + 1, as_stream(stream));
}
