// sell.cu -- SELL-32-sigma copy of the level operator for the residual SpMV
// (r = b - L x, Eq. 10).
//
// The CSR rows of a Q2-Q1 operator have a handful of distinct lengths (2D: 13,
// 21, 34 for velocity rows of cell-centre / edge / vertex nodes, 50 for
// pressure rows), interleaved along the DoF numbering.  Sorting rows by length
// inside windows of SIGMA = 4096 rows and storing slices of 32 rows
// column-major turns the residual into one thread per row with fully coalesced
// 256-byte (val) / 128-byte (col) warp loads, no row-pointer chase and no
// shuffles; padding is < 1%.  Each row is summed in its CSR column order by one
// thread, so the residual is deterministic (run to run and across launch shapes).
#include <algorithm>
#include <cub/cub.cuh>

#include "internal.cuh"

namespace rav {

constexpr int SELL_C = 32;
constexpr int SELL_SIGMA = 4096;   // multiple of SELL_C: slices never straddle windows
constexpr int SELL_THREADS = 256;

__global__ void row_len_kernel(int64_t n, const int64_t* rp, int32_t* len, int32_t* idx) {
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
        len[i] = (int32_t)(rp[i + 1] - rp[i]);
        idx[i] = (int32_t)i;
    }
}

__global__ void window_offsets_kernel(int64_t n, int64_t nw, int64_t* off) {
    for (int64_t w = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; w <= nw; w += (int64_t)gridDim.x * blockDim.x)
        off[w] = w * SELL_SIGMA < n ? w * SELL_SIGMA : n;
}

// slice size = 32 * (length of its first, i.e. longest, row)
__global__ void slice_size_kernel(int64_t n, int64_t nslices, const int32_t* slen, int64_t* sz) {
    for (int64_t s = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; s < nslices; s += (int64_t)gridDim.x * blockDim.x)
        sz[s] = (int64_t)SELL_C * slen[s * SELL_C];
}

__global__ void sell_fill_kernel(int64_t n, int64_t nslices, const int64_t* rp, const int32_t* ci, const double* val,
                                 const int32_t* perm, const int64_t* sptr, int32_t* scol, double* sval) {
    const int64_t total = nslices * SELL_C;
    for (int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; t < total; t += (int64_t)gridDim.x * blockDim.x) {
        const int64_t s = t / SELL_C;
        const int l = (int)(t % SELL_C);
        const int64_t w = (sptr[s + 1] - sptr[s]) / SELL_C;
        const int64_t base = sptr[s] + l;
        if (t < n) {
            const int32_t row = perm[t];
            const int64_t a = rp[row], len = rp[row + 1] - a;
            for (int64_t k = 0; k < w; ++k) {
                scol[base + k * SELL_C] = k < len ? ci[a + k] : row;
                sval[base + k * SELL_C] = k < len ? val[a + k] : 0.0;
            }
        } else {
            for (int64_t k = 0; k < w; ++k) {
                scol[base + k * SELL_C] = 0;
                sval[base + k * SELL_C] = 0.0;
            }
        }
    }
}

__global__ void __launch_bounds__(SELL_THREADS) sell_residual_kernel(int64_t n, int64_t nslices,
                                                                     const int64_t* __restrict__ sptr,
                                                                     const int32_t* __restrict__ scol,
                                                                     const double* __restrict__ sval,
                                                                     const int32_t* __restrict__ perm,
                                                                     const double* __restrict__ x,
                                                                     const double* __restrict__ b,
                                                                     double* __restrict__ r, double* __restrict__ part) {
    __shared__ double red[SELL_THREADS / 32];
    double mine = 0.0;
    const int64_t total = nslices * SELL_C;
    for (int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; t - threadIdx.x < total;
         t += (int64_t)gridDim.x * blockDim.x) {
        if (t < total) {
            const int64_t s = t / SELL_C;
            const int l = (int)(t % SELL_C);
            const int64_t s0 = sptr[s];
            const int w = (int)((sptr[s + 1] - s0) / SELL_C);
            const double* v = sval + s0 + l;
            const int32_t* c = scol + s0 + l;
            double acc = 0.0;
            int k = 0;
            for (; k + 4 <= w; k += 4) {
                const int c0 = __ldcs(c + (k + 0) * SELL_C), c1 = __ldcs(c + (k + 1) * SELL_C);
                const int c2 = __ldcs(c + (k + 2) * SELL_C), c3 = __ldcs(c + (k + 3) * SELL_C);
                const double v0 = __ldcs(v + (k + 0) * SELL_C), v1 = __ldcs(v + (k + 1) * SELL_C);
                const double v2 = __ldcs(v + (k + 2) * SELL_C), v3 = __ldcs(v + (k + 3) * SELL_C);
                const double x0 = __ldg(x + c0), x1 = __ldg(x + c1), x2 = __ldg(x + c2), x3 = __ldg(x + c3);
                acc += v0 * x0;
                acc += v1 * x1;
                acc += v2 * x2;
                acc += v3 * x3;
            }
            for (; k < w; ++k) acc += __ldcs(v + k * SELL_C) * __ldg(x + __ldcs(c + k * SELL_C));
            if (t < n) {
                const int32_t row = perm[t];
                const double rr = b[row] - acc;
                if (r) r[row] = rr;
                mine += rr * rr;
            }
        }
    }
    if (part) {
        mine = warp_sum(mine);
        if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = mine;
        __syncthreads();
        if (threadIdx.x == 0) {
            double sum = 0.0;
            for (int i = 0; i < SELL_THREADS / 32; ++i) sum += red[i];
            part[blockIdx.x] = sum;
        }
    }
}

rav_status sell_build(Csr& A, cudaStream_t s) {
    Sell& S = A.sell;
    const int64_t n = A.n_rows;
    if (n == 0 || A.n_rows != A.n_cols) return RAV_OK;
    S.nslices = cdiv(n, SELL_C);
    const int64_t nslots = S.nslices * SELL_C;
    const int64_t nw = cdiv(n, SELL_SIGMA);
    int32_t *len = nullptr, *idx = nullptr, *slen = nullptr;
    int64_t *woff = nullptr, *sz = nullptr;
    RAV_CUDA(cudaMallocAsync(&len, sizeof(int32_t) * n, s));
    RAV_CUDA(cudaMallocAsync(&idx, sizeof(int32_t) * n, s));
    RAV_CUDA(cudaMallocAsync(&slen, sizeof(int32_t) * nslots, s));
    RAV_CUDA(cudaMallocAsync(&woff, sizeof(int64_t) * (nw + 1), s));
    RAV_CUDA(cudaMallocAsync(&sz, sizeof(int64_t) * S.nslices, s));
    RAV_CUDA(cudaMalloc(&S.perm, sizeof(int32_t) * nslots));
    RAV_CUDA(cudaMalloc(&S.sptr, sizeof(int64_t) * (S.nslices + 1)));
    RAV_CUDA(cudaMemsetAsync(slen, 0, sizeof(int32_t) * nslots, s));
    RAV_CUDA(cudaMemsetAsync(S.perm, 0, sizeof(int32_t) * nslots, s));
    const int nb = (int)std::max<int64_t>(1, std::min<int64_t>(cdiv(n, 256), (int64_t)num_sms() * 16));
    row_len_kernel<<<nb, 256, 0, s>>>(n, A.rp, len, idx);
    count_launch();
    RAV_CHECK_LAUNCH();
    window_offsets_kernel<<<(int)std::max<int64_t>(1, cdiv(nw + 1, 256)), 256, 0, s>>>(n, nw, woff);
    count_launch();
    RAV_CHECK_LAUNCH();
    size_t tmp = 0;
    RAV_CUDA(cub::DeviceSegmentedRadixSort::SortPairsDescending(nullptr, tmp, len, slen, idx, S.perm, (int)n, (int)nw,
                                                                woff, woff + 1, 0, 8 * sizeof(int32_t), s));
    void* d_tmp = nullptr;
    RAV_CUDA(cudaMallocAsync(&d_tmp, tmp + 16, s));
    RAV_CUDA(cub::DeviceSegmentedRadixSort::SortPairsDescending(d_tmp, tmp, len, slen, idx, S.perm, (int)n, (int)nw,
                                                                woff, woff + 1, 0, 8 * sizeof(int32_t), s));
    slice_size_kernel<<<(int)std::max<int64_t>(1, std::min<int64_t>(cdiv(S.nslices, 256), (int64_t)num_sms() * 16)),
                        256, 0, s>>>(n, S.nslices, slen, sz);
    count_launch();
    RAV_CHECK_LAUNCH();
    RAV_TRY(gen::counts_to_rowptr(sz, S.sptr, S.nslices, s));
    RAV_CUDA(cudaMemcpyAsync(&S.stored, S.sptr + S.nslices, sizeof(int64_t), cudaMemcpyDeviceToHost, s));
    RAV_CUDA(cudaStreamSynchronize(s));
    RAV_CUDA(cudaMalloc(&S.col, sizeof(int32_t) * std::max<int64_t>(1, S.stored)));
    RAV_CUDA(cudaMalloc(&S.val, sizeof(double) * std::max<int64_t>(1, S.stored)));
    const int nbf = (int)std::max<int64_t>(1, std::min<int64_t>(cdiv(nslots, 256), (int64_t)num_sms() * 16));
    sell_fill_kernel<<<nbf, 256, 0, s>>>(n, S.nslices, A.rp, A.ci, A.val, S.perm, S.sptr, S.col, S.val);
    count_launch();
    RAV_CHECK_LAUNCH();
    cudaFreeAsync(d_tmp, s);
    cudaFreeAsync(len, s);
    cudaFreeAsync(idx, s);
    cudaFreeAsync(slen, s);
    cudaFreeAsync(woff, s);
    cudaFreeAsync(sz, s);
    RAV_CUDA(cudaStreamSynchronize(s));
    return RAV_OK;
}

void sell_free(Sell& S) {
    if (S.sptr) cudaFree(S.sptr);
    if (S.col) cudaFree(S.col);
    if (S.val) cudaFree(S.val);
    if (S.perm) cudaFree(S.perm);
    S = Sell{};
}

int64_t sell_full_blocks(const Sell& S) { return cdiv(S.nslices * SELL_C, SELL_THREADS); }

rav_status launch_sell_residual(const Csr& A, const double* x, const double* b, double* r, double* part, int nblk,
                                cudaStream_t s, int* used) {
    const Sell& S = A.sell;
    const int64_t full = sell_full_blocks(S);
    const int blocks = (int)(part ? std::min<int64_t>(full, nblk) : full);   // one partial norm per block
    if (used) *used = blocks;
    sell_residual_kernel<<<blocks, SELL_THREADS, 0, s>>>(A.n_rows, S.nslices, S.sptr, S.col, S.val, S.perm, x, b, r,
                                                         part);
    count_launch();
    RAV_CHECK_LAUNCH();
    return RAV_OK;
}

}  // namespace rav
