// coarse.cu -- coarsest-grid direct solve ("We
// use LU factorization to solve the coarse system to machine accuracy").
// The coarsest operator (<= a few hundred DoFs) is densified with DoF `pin`
// removed (R4: the pressure null space is fixed only here), factored once by
// Gaussian elimination with partial pivoting in one CTA; the inverse is formed
// from the factors at setup (one warp per column) and every V-cycle applies it
// as one dense mat-vec in one CTA (fallback above 2048 unknowns: the row swaps
// and two triangular solves in one warp).
#include <algorithm>

#include "internal.cuh"

namespace rav {

__global__ void densify_kernel(int64_t n, const int64_t* rp, const int32_t* ci, const double* val, int64_t pin,
                               int m, double* D) {
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
        if (i == pin) continue;
        int64_t ii = (pin >= 0 && i > pin) ? i - 1 : i;
        for (int64_t k = rp[i]; k < rp[i + 1]; ++k) {
            int64_t j = ci[k];
            if (j == pin) continue;
            int64_t jj = (pin >= 0 && j > pin) ? j - 1 : j;
            D[ii * m + jj] = val[k];
        }
    }
}

// in-place LU with partial pivoting (P A = L U), one CTA; fail = first failing column + 1
__global__ void __launch_bounds__(512) coarse_lu_kernel(int m, double* A, int32_t* piv, int* fail) {
    __shared__ int s_p;
    __shared__ double s_rn_tol;
    extern __shared__ double rn[];
    const int tid = threadIdx.x, nt = blockDim.x;
    for (int r = tid; r < m; r += nt) {
        double mx = 0.0;
        for (int c = 0; c < m; ++c) mx = fmax(mx, fabs(A[(size_t)r * m + c]));
        rn[r] = mx;
    }
    if (tid == 0) *fail = 0;
    __syncthreads();
    for (int c = 0; c < m; ++c) {
        if (tid < 32) {
            double best = -1.0;
            int bi = c;
            for (int r = c + tid; r < m; r += 32) {
                double v = fabs(A[(size_t)r * m + c]);
                if (v > best) { best = v; bi = r; }
            }
            for (int o = 16; o > 0; o >>= 1) {
                double ob = __shfl_xor_sync(0xffffffffu, best, o);
                int oi = __shfl_xor_sync(0xffffffffu, bi, o);
                if (ob > best || (ob == best && oi < bi)) { best = ob; bi = oi; }
            }
            if (tid == 0) {
                s_p = bi;
                piv[c] = bi;
                s_rn_tol = 1e-14 * rn[bi];
                if (!(best > s_rn_tol)) *fail = c + 1;
            }
        }
        __syncthreads();
        if (*fail) return;
        const int p = s_p;
        if (p != c) {
            for (int t = tid; t < m; t += nt) {
                double u = A[(size_t)c * m + t];
                A[(size_t)c * m + t] = A[(size_t)p * m + t];
                A[(size_t)p * m + t] = u;
            }
            if (tid == 0) { double u = rn[c]; rn[c] = rn[p]; rn[p] = u; }
        }
        __syncthreads();
        const double inv = 1.0 / A[(size_t)c * m + c];
        for (int r = c + 1 + tid; r < m; r += nt) A[(size_t)r * m + c] *= inv;
        __syncthreads();
        const int nr = m - c - 1;
        for (int t = tid; t < nr * nr; t += nt) {
            int r = c + 1 + t / nr, col = c + 1 + t % nr;
            A[(size_t)r * m + col] -= A[(size_t)r * m + c] * A[(size_t)c * m + col];
        }
        __syncthreads();
    }
}

// x = A^{-1} b on the pinned system; one warp
__global__ void coarse_solve_kernel(int64_t n, int64_t pin, int m, const double* __restrict__ LU,
                                    const int32_t* __restrict__ piv, const double* __restrict__ b, double* x) {
    extern __shared__ double y[];
    const int lane = threadIdx.x;
    for (int64_t i = lane; i < n; i += 32) {
        if (i == pin) continue;
        int64_t ii = (pin >= 0 && i > pin) ? i - 1 : i;
        y[ii] = b[i];
    }
    __syncwarp();
    if (lane == 0)
        for (int k = 0; k < m; ++k) {
            int p = piv[k];
            if (p != k) { double u = y[k]; y[k] = y[p]; y[p] = u; }
        }
    __syncwarp();
    for (int i = 0; i < m; ++i) {               // L (unit) forward
        double s = 0.0;
        for (int j = lane; j < i; j += 32) s += LU[(size_t)i * m + j] * y[j];
        s = warp_sum(s);
        if (lane == 0) y[i] -= s;
        __syncwarp();
    }
    for (int i = m - 1; i >= 0; --i) {          // U backward
        double s = 0.0;
        for (int j = i + 1 + lane; j < m; j += 32) s += LU[(size_t)i * m + j] * y[j];
        s = warp_sum(s);
        if (lane == 0) y[i] = (y[i] - s) / LU[(size_t)i * m + i];
        __syncwarp();
    }
    for (int64_t i = lane; i < n; i += 32) {
        if (i == pin) { x[i] = 0.0; continue; }
        int64_t ii = (pin >= 0 && i > pin) ? i - 1 : i;
        x[i] = y[ii];
    }
}

// column w of A^{-1} from the LU factors (one warp per column; setup only)
__global__ void coarse_inverse_kernel(int m, const double* __restrict__ LU, const int32_t* __restrict__ piv,
                                      double* __restrict__ inv) {
    extern __shared__ double ysh[];
    const int w = blockIdx.x, lane = threadIdx.x;
    double* y = ysh;
    for (int i = lane; i < m; i += 32) y[i] = (i == w) ? 1.0 : 0.0;
    __syncwarp();
    if (lane == 0)
        for (int k = 0; k < m; ++k) {
            int p = piv[k];
            if (p != k) { double u = y[k]; y[k] = y[p]; y[p] = u; }
        }
    __syncwarp();
    for (int i = 0; i < m; ++i) {
        double t = 0.0;
        for (int j = lane; j < i; j += 32) t += LU[(size_t)i * m + j] * y[j];
        t = warp_sum(t);
        if (lane == 0) y[i] -= t;
        __syncwarp();
    }
    for (int i = m - 1; i >= 0; --i) {
        double t = 0.0;
        for (int j = i + 1 + lane; j < m; j += 32) t += LU[(size_t)i * m + j] * y[j];
        t = warp_sum(t);
        if (lane == 0) y[i] = (y[i] - t) / LU[(size_t)i * m + i];
        __syncwarp();
    }
    for (int i = lane; i < m; i += 32) inv[(size_t)i * m + w] = y[i];
}

// x = A^{-1} b with the precomputed inverse: one CTA, a warp per row, pinned DoF set to 0
__global__ void __launch_bounds__(512) coarse_apply_kernel(int64_t n, int64_t pin, int m, const double* __restrict__ inv,
                                                           const double* __restrict__ b, double* __restrict__ x) {
    extern __shared__ double yb[];
    for (int64_t i = threadIdx.x; i < n; i += blockDim.x) {
        if (i == pin) continue;
        yb[(pin >= 0 && i > pin) ? i - 1 : i] = b[i];
    }
    __syncthreads();
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5, nw = blockDim.x >> 5;
    for (int r = warp; r < m; r += nw) {
        double t = 0.0;
        for (int j = lane; j < m; j += 32) t = fma(inv[(size_t)r * m + j], yb[j], t);
        t = warp_sum(t);
        if (lane == 0) x[(pin >= 0 && r >= pin) ? r + 1 : r] = t;
    }
    if (pin >= 0 && threadIdx.x == 0) x[pin] = 0.0;
}

rav_status coarse_factor(const Csr& A, int64_t pin, CoarseLU& C, cudaStream_t s) {
    C.n = A.n_rows;
    C.pin = pin;
    C.m = (int)(pin >= 0 ? A.n_rows - 1 : A.n_rows);
    if (C.m < 1 || C.m > 6000) { set_error("coarsest system size %d out of range [1, 6000]", C.m); return RAV_ERR_ARG; }
    RAV_CUDA(cudaMalloc(&C.lu, sizeof(double) * (size_t)C.m * C.m));
    RAV_CUDA(cudaMalloc(&C.piv, sizeof(int32_t) * C.m));
    RAV_CUDA(cudaMemsetAsync(C.lu, 0, sizeof(double) * (size_t)C.m * C.m, s));
    densify_kernel<<<(int)std::max<int64_t>(1, cdiv(C.n, 128)), 128, 0, s>>>(C.n, A.rp, A.ci, A.val, pin, C.m, C.lu);
    count_launch();
    RAV_CHECK_LAUNCH();
    int* fail = nullptr;
    RAV_CUDA(cudaMallocAsync(&fail, sizeof(int), s));
    coarse_lu_kernel<<<1, 512, sizeof(double) * C.m, s>>>(C.m, C.lu, C.piv, fail);
    count_launch();
    RAV_CHECK_LAUNCH();
    int h_fail = 0;
    RAV_CUDA(cudaMemcpyAsync(&h_fail, fail, sizeof(int), cudaMemcpyDeviceToHost, s));
    cudaFreeAsync(fail, s);
    RAV_CUDA(cudaStreamSynchronize(s));
    if (h_fail) {
        set_error("singular coarsest system (column %d)", h_fail - 1);
        return RAV_ERR_SINGULAR_COARSE;
    }
    // explicit inverse from the LU factors: every V-cycle's coarse solve becomes one dense
    // mat-vec in one CTA (the per-cycle triangular solves were 2m dependent warp steps)
    if (C.m <= 2048) {
        RAV_CUDA(cudaMalloc(&C.inv, sizeof(double) * (size_t)C.m * C.m));
        coarse_inverse_kernel<<<C.m, 32, sizeof(double) * C.m, s>>>(C.m, C.lu, C.piv, C.inv);
        count_launch();
        RAV_CHECK_LAUNCH();
        RAV_CUDA(cudaStreamSynchronize(s));
    }
    return RAV_OK;
}

rav_status launch_coarse_solve(const CoarseLU& C, const double* b, double* x, cudaStream_t s) {
    if (C.inv) coarse_apply_kernel<<<1, 512, sizeof(double) * C.m, s>>>(C.n, C.pin, C.m, C.inv, b, x);
    else coarse_solve_kernel<<<1, 32, sizeof(double) * C.m, s>>>(C.n, C.pin, C.m, C.lu, C.piv, b, x);
    count_launch();
    RAV_CHECK_LAUNCH();
    return RAV_OK;
}

void coarse_free(CoarseLU& C) {
    if (C.lu) cudaFree(C.lu);
    if (C.piv) cudaFree(C.piv);
    if (C.inv) cudaFree(C.inv);
    C = CoarseLU{};
}

}  // namespace rav
