// sweep.cu -- the restricted additive Vanka sweep (
// P:124 Eq. 13): given r = b - L x (one residual for all patches),
//     x_j += omega * sum_{i : j restricted in patch i} (W_i R_i r)_j
// with W_i = diag(w_i) L_i^{-1}[restricted, :] precomputed by setup.cu.
// The corrections of the (up to 2^d) patches that share a DoF through the
// partition-of-unity weights (R3) are combined with red.global.add.f64
// (order-independent up to rounding, R16).
//
// The sweep is HBM-bound (~0.23 flop/byte): the only large stream is the
// factor rows (7.75 KB per 2D patch).  Two kernels:
//  * sweep_thread_kernel<NT>: one patch per thread, factor rows in the SoA
//    chunk layout of setup.cu, so every warp-wide LDG.128 reads 512
//    contiguous bytes with an evict-first hint; NT accumulators in registers,
//    the residual gathered once per column (r stays L2-resident: 19 MB at c2).
//  * sweep_warp_kernel: one warp per patch (any n_i, nres_i; 3D 376 x 82),
//    r_i staged in shared memory, lanes stream the row-major rows coalesced,
//    warp-shuffle reductions.
#include <algorithm>

#include "internal.cuh"

namespace rav {

template <int NT>
__global__ void __launch_bounds__(128) sweep_thread_kernel(int64_t nchunks, int NMAX, const double2* __restrict__ W,
                                                           const int32_t* __restrict__ DT,
                                                           const int32_t* __restrict__ NR,
                                                           const double* __restrict__ r, double* __restrict__ x,
                                                           double omega) {
    const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    const int64_t chunk = i >> 5;
    const int lane = threadIdx.x & 31;
    if (chunk >= nchunks) return;
    const int64_t pairs = (int64_t)NMAX * NT / 2;
    const double2* wp = W + chunk * pairs * 32 + lane;
    const int32_t* dp = DT + chunk * (int64_t)NMAX * 32 + lane;
    double acc[NT];
#pragma unroll
    for (int k = 0; k < NT; ++k) acc[k] = 0.0;
    for (int j0 = 0; j0 < NMAX; j0 += 2) {
        const double r0 = __ldg(r + __ldcs(dp + j0 * 32));
        const double r1 = __ldg(r + __ldcs(dp + (j0 + 1) * 32));
        const double2* wq = wp + (int64_t)(j0 * NT / 2) * 32;
#pragma unroll
        for (int q = 0; q < NT; ++q) {
            const double2 v = __ldcs(wq + q * 32);
            const int e0 = 2 * q, e1 = 2 * q + 1;
            if (e0 < NT) acc[e0] = fma(v.x, r0, acc[e0]); else acc[e0 - NT] = fma(v.x, r1, acc[e0 - NT]);
            if (e1 < NT) acc[e1] = fma(v.y, r0, acc[e1]); else acc[e1 - NT] = fma(v.y, r1, acc[e1 - NT]);
        }
    }
    const int m = NR[i];
#pragma unroll
    for (int k = 0; k < NT; ++k)
        if (k < m) atomicAdd(x + dp[k * 32], omega * acc[k]);
}

// Symmetric-block variant (layout 3 of setup.cu): the restricted x restricted block
// of L_i^{-1} is symmetric, so the NT x NT leading block is streamed as its upper
// triangle (each entry feeds two accumulators), the remaining columns as NT-row
// slabs, and the partition-of-unity weights are applied once per row at the end:
//   c_k = w_k ( sum_{j<NT} Linv[min(k,j)][max(k,j)] r_j + sum_{j>=NT} Linv[k][j] r_j ).
// 2D PoU: 798 stored entries per patch instead of 988 (-19%).
template <int NT>
__global__ void __launch_bounds__(128) sweep_sym_kernel(int64_t nchunks, int NMAX, const double2* __restrict__ W,
                                                        const int32_t* __restrict__ DT,
                                                        const double* __restrict__ WT,
                                                        const int32_t* __restrict__ NR,
                                                        const double* __restrict__ r, double* __restrict__ x,
                                                        double omega) {
    constexpr int TRI = NT * (NT + 1) / 2;
    constexpr int NTRI = TRI + (TRI & 1);
    const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    const int64_t chunk = i >> 5;
    const int lane = threadIdx.x & 31;
    if (chunk >= nchunks) return;
    const int64_t pairs = ((int64_t)NTRI + (int64_t)(NMAX - NT) * NT) / 2;
    const double2* wp = W + chunk * pairs * 32 + lane;
    const int32_t* dp = DT + chunk * (int64_t)NMAX * 32 + lane;
    double acc[NT], rr[NT];
#pragma unroll
    for (int k = 0; k < NT; ++k) {
        acc[k] = 0.0;
        rr[k] = __ldg(r + __ldcs(dp + k * 32));
    }
    double2 pv = make_double2(0.0, 0.0);
#pragma unroll
    for (int j = 0; j < NT; ++j) {
#pragma unroll
        for (int k = 0; k <= j; ++k) {
            const int e = j * (j + 1) / 2 + k;
            if ((e & 1) == 0) pv = __ldcs(wp + (e >> 1) * 32);
            const double v = (e & 1) ? pv.y : pv.x;
            acc[k] = fma(v, rr[j], acc[k]);
            if (k != j) acc[j] = fma(v, rr[k], acc[j]);
        }
    }
    const double2* wq0 = wp + (NTRI / 2) * 32;
    for (int j0 = NT; j0 < NMAX; j0 += 2) {
        const double r0 = __ldg(r + __ldcs(dp + j0 * 32));
        const double r1 = __ldg(r + __ldcs(dp + (j0 + 1) * 32));
        const double2* wq = wq0 + (int64_t)((j0 - NT) * NT / 2) * 32;
#pragma unroll
        for (int q = 0; q < NT; ++q) {
            const double2 v = __ldcs(wq + q * 32);
            const int e0 = 2 * q, e1 = 2 * q + 1;
            if (e0 < NT) acc[e0] = fma(v.x, r0, acc[e0]); else acc[e0 - NT] = fma(v.x, r1, acc[e0 - NT]);
            if (e1 < NT) acc[e1] = fma(v.y, r0, acc[e1]); else acc[e1 - NT] = fma(v.y, r1, acc[e1 - NT]);
        }
    }
    const int m = NR[i];
    const double* wt = WT + chunk * NT * 32 + lane;
#pragma unroll
    for (int k = 0; k < NT; ++k)
        if (k < m) atomicAdd(x + dp[k * 32], omega * (wt[k * 32] * acc[k]));
}

constexpr int WK_THREADS = 256;

__global__ void __launch_bounds__(WK_THREADS) sweep_warp_kernel(int64_t np, int nmax, const int64_t* __restrict__ poffs,
                                                                const int32_t* __restrict__ pdofs,
                                                                const int32_t* __restrict__ nres,
                                                                const int64_t* __restrict__ foffs,
                                                                const double* __restrict__ fac,
                                                                const double* __restrict__ r, double* __restrict__ x,
                                                                double omega) {
    extern __shared__ double sm[];
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    double* rl = sm + (size_t)warp * nmax;
    const int wpb = WK_THREADS / 32;
    for (int64_t i = (int64_t)blockIdx.x * wpb + warp; i < np; i += (int64_t)gridDim.x * wpb) {
        const int64_t off = poffs[i];
        const int n = (int)(poffs[i + 1] - off);
        const int m = nres[i];
        for (int j = lane; j < n; j += 32) rl[j] = __ldg(r + pdofs[off + j]);
        __syncwarp();
        const double* Wi = fac + foffs[i];
        for (int k0 = 0; k0 < m; k0 += 4) {
            double acc[4] = {0.0, 0.0, 0.0, 0.0};
            const int kr = min(4, m - k0);
            for (int j = lane; j < n; j += 32) {
                const double rj = rl[j];
#pragma unroll
                for (int t = 0; t < 4; ++t)
                    if (t < kr) acc[t] = fma(ld_stream(Wi + (int64_t)(k0 + t) * n + j), rj, acc[t]);
            }
#pragma unroll
            for (int t = 0; t < 4; ++t) {
                double s = warp_sum(acc[t]);
                if (lane == 0 && t < kr) atomicAdd(x + pdofs[off + k0 + t], omega * s);
            }
        }
        __syncwarp();
    }
}

template <int NT>
static void launch_thread(const Factors& F, const double* r, double* x, double omega, cudaStream_t s) {
    int64_t threads = F.nchunks * 32;
    int blocks = (int)cdiv(threads, 128);
    sweep_thread_kernel<NT><<<blocks, 128, 0, s>>>(F.nchunks, F.NMAX, reinterpret_cast<const double2*>(F.facT),
                                                  F.DT, F.NR, r, x, omega);
}

template <int NT>
static void launch_sym(const Factors& F, const double* r, double* x, double omega, cudaStream_t s) {
    int64_t threads = F.nchunks * 32;
    int blocks = (int)cdiv(threads, 128);
    sweep_sym_kernel<NT><<<blocks, 128, 0, s>>>(F.nchunks, F.NMAX, reinterpret_cast<const double2*>(F.facT), F.DT,
                                               F.WT, F.NR, r, x, omega);
}

rav_status launch_sweep(const PatchSet& P, const Factors& F, const double* r, double* x, double omega,
                        cudaStream_t s) {
    if (F.layout == 6) return launch_diag_sweep(P, F, r, x, omega, s);
    if (F.layout >= 4) return launch_schur_sweep(P, F, r, x, omega, s);
    if (F.layout == 3) {
        switch (F.NT) {
            case 3: launch_sym<3>(F, r, x, omega, s); break;
            case 4: launch_sym<4>(F, r, x, omega, s); break;
            case 8: launch_sym<8>(F, r, x, omega, s); break;
            case 9: launch_sym<9>(F, r, x, omega, s); break;
            case 12: launch_sym<12>(F, r, x, omega, s); break;
            case 16: launch_sym<16>(F, r, x, omega, s); break;
            case 19: launch_sym<19>(F, r, x, omega, s); break;
            case 24: launch_sym<24>(F, r, x, omega, s); break;
            case 32: launch_sym<32>(F, r, x, omega, s); break;
            default: set_error("unsupported NT %d", F.NT); return RAV_ERR_ARG;
        }
    } else if (F.layout == 2) {
        switch (F.NT) {
            case 3: launch_thread<3>(F, r, x, omega, s); break;
            case 4: launch_thread<4>(F, r, x, omega, s); break;
            case 8: launch_thread<8>(F, r, x, omega, s); break;
            case 9: launch_thread<9>(F, r, x, omega, s); break;
            case 12: launch_thread<12>(F, r, x, omega, s); break;
            case 16: launch_thread<16>(F, r, x, omega, s); break;
            case 19: launch_thread<19>(F, r, x, omega, s); break;
            case 24: launch_thread<24>(F, r, x, omega, s); break;
            case 32: launch_thread<32>(F, r, x, omega, s); break;
            default: set_error("unsupported NT %d", F.NT); return RAV_ERR_ARG;
        }
    } else {
        size_t shmem = sizeof(double) * (size_t)P.nmax * (WK_THREADS / 32);
        if (shmem > 48 * 1024)
            RAV_CUDA(cudaFuncSetAttribute(sweep_warp_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)shmem));
        int blocks = (int)std::min<int64_t>(cdiv(P.n_patches, WK_THREADS / 32), (int64_t)num_sms() * 16);
        sweep_warp_kernel<<<blocks, WK_THREADS, shmem, s>>>(P.n_patches, P.nmax, P.offs, P.dofs, P.nres, F.foffs,
                                                            F.fac, r, x, omega);
    }
    count_launch();
    RAV_CHECK_LAUNCH();
    return RAV_OK;
}

}  // namespace rav
