// xfer.cu -- stencil form of the nested-grid transfers of structured levels (SURVEY section 8
// row a7).  The prolongation of a uniformly refined tensor-product grid is the tensor
// product of 1D interpolation stencils:
//   Q2 velocity (lattice index f of the fine (4 n_c + 1)-node line, coarse (2 n_c + 1)):
//     f even: coarse node f / 2, weight 1; f = 4e + 1 / 4e + 3: coarse nodes 2e, 2e+1, 2e+2 with
//     the Q2 basis at t = 1/4 / 3/4: (3/8, 3/4, -1/8) / (-1/8, 3/4, 3/8);
//   Q1 (pressure vertices; Q1-Q1 velocity): f even: f / 2, weight 1; f odd: (f -+ 1) / 2, 1/2 each;
// Dirichlet nodes (velocity on the boundary) are dropped on both sides; R = P^T.  So instead of
// streaming the CSR of P and of P^T (c3 fine level: about 2 GB per V-cycle at 2.8 TB/s), the
// kernels read the input vector and write the output vector only.
//   prolongation: one thread per fine node (all d components) / fine vertex;
//   restriction:  one thread per coarse node / vertex, gathering the transpose stencil
//     Q2: coarse c even: fine 2c-3, 2c-1, 2c, 2c+1, 2c+3 with (-1/8, 3/8, 1, 3/8, -1/8);
//         c odd: fine 2c-1, 2c, 2c+1 with (3/4, 1, 3/4);
//     Q1: fine 2c-1, 2c, 2c+1 with (1/2, 1, 1/2).
// Sums run over the stencil in ascending DoF order.  xs_verify checks the stencil form against
// the level's own CSR P / P^T on seeded vectors before it is used.
// Slab windows (multi-GPU levels, rav_grid win = 1): the vectors are windows of layers along the
// last axis; the prolongation fills only the fine rows of the owned layers (the others keep their
// value: rav_gen_prolongation leaves those rows empty) and the restriction gathers only from them
// (P_own^T r), writing every coarse window entry.
#include "internal.cuh"

namespace rav {
namespace {

struct XArgs {
    int dim, P;                 // P: velocity lattice refinement (2: Q2, 1: Q1)
    int nc[3];                  // coarse cells per axis (fine: 2 nc)
    int64_t nfree_f, nfree_c;   // free velocity nodes (of the windows)
    int64_t nvert_f, nvert_c;   // vertices (pressure DoFs, of the windows)
    int64_t nvel_f, nvel_c;     // dim * nfree
    // last-axis windows (global lattice layers, inclusive): see XStruct
    int fn_lo, fn_hi, fv_lo, fv_hi, rn_lo, rn_hi, rv_lo, rv_hi, cn_lo, cn_hi, cv_lo, cv_hi;
};

// Per-axis stencils as fixed-length candidate lists (weight 0 = absent), so that every loop
// below unrolls completely and the lists stay in registers.
// prolongation, fine lattice index f (3 candidates)
__device__ __forceinline__ void q2_interp(int f, int ncx, int* idx, double* w) {
    if (!(f & 1)) {
        idx[0] = f >> 1; w[0] = 1.0;
        idx[1] = idx[2] = 0; w[1] = w[2] = 0.0;
        return;
    }
    int e = f >> 2;
    if (e > ncx - 1) e = ncx - 1;
    idx[0] = 2 * e; idx[1] = 2 * e + 1; idx[2] = 2 * e + 2;
    const bool first = (f & 3) == 1;
    w[0] = first ? 0.375 : -0.125;
    w[1] = 0.75;
    w[2] = first ? -0.125 : 0.375;
}
__device__ __forceinline__ void q1_interp(int f, int* idx, double* w) {
    if (!(f & 1)) {
        idx[0] = f >> 1; w[0] = 1.0;
        idx[1] = idx[2] = 0; w[1] = w[2] = 0.0;
        return;
    }
    idx[0] = (f - 1) >> 1; w[0] = 0.5;
    idx[1] = (f + 1) >> 1; w[1] = 0.5;
    idx[2] = 0; w[2] = 0.0;
}
// restriction (transpose stencils, 5 candidates), fine indices restricted to [lo, hi]
__device__ __forceinline__ void q2_gather(int c, int lo, int hi, int* idx, double* w) {
    const bool odd = c & 1;
#pragma unroll
    for (int k = 0; k < 5; ++k) {
        const int off = odd ? k - 1 : (k == 0 ? -3 : (k == 4 ? 3 : k - 2));
        const double v = odd ? (k == 1 ? 1.0 : (k < 3 ? 0.75 : 0.0))
                             : (k == 2 ? 1.0 : ((k == 1 || k == 3) ? 0.375 : -0.125));
        idx[k] = 2 * c + off;
        w[k] = (idx[k] >= lo && idx[k] <= hi) ? v : 0.0;
    }
}
__device__ __forceinline__ void q1_gather(int c, int lo, int hi, int* idx, double* w) {
#pragma unroll
    for (int k = 0; k < 5; ++k) {
        idx[k] = 2 * c + k - 1;
        const double v = k == 1 ? 1.0 : (k < 3 ? 0.5 : 0.0);
        w[k] = (idx[k] >= lo && idx[k] <= hi) ? v : 0.0;
    }
}

// y_f = beta y_f + alpha P x_c
template <int DIM>
__global__ void __launch_bounds__(256) xs_prolong_kernel(XArgs X, const double* __restrict__ xc,
                                                         double* __restrict__ yf, double alpha, double beta) {
    constexpr int N2 = DIM > 2 ? 3 : 1;
    const int64_t total = X.nfree_f + X.nvert_f;
    const int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (t >= total) return;
    int idx[3][3];
    double wt[3][3];
    if (t < X.nfree_f) {   // fine velocity node: lattice coordinates 1 .. P nf - 1
        int64_t r = t;
#pragma unroll
        for (int k = 0; k < DIM; ++k) {
            const int m = 2 * X.P * X.nc[k] - 1;
            const int a = k < DIM - 1 ? (int)(r % m) + 1 : (int)r + X.fn_lo;   // last axis: the window's layers
            if (k < DIM - 1) r /= m;
            else if (a < X.rn_lo || a > X.rn_hi) return;                      // not an owned row
            if (X.P == 2) q2_interp(a, X.nc[k], idx[k], wt[k]);
            else q1_interp(a, idx[k], wt[k]);
        }
        double acc[DIM];
#pragma unroll
        for (int c = 0; c < DIM; ++c) acc[c] = 0.0;
#pragma unroll
        for (int s2 = 0; s2 < N2; ++s2)
#pragma unroll
            for (int s1 = 0; s1 < 3; ++s1)
#pragma unroll
                for (int s0 = 0; s0 < 3; ++s0) {
                    double w = wt[0][s0] * wt[1][s1];
                    if (DIM > 2) w *= wt[2][s2];
                    int64_t id = 0, st = 1;
                    bool free_ = w != 0.0;
#pragma unroll
                    for (int k = 0; k < DIM; ++k) {
                        const int ak = k == 0 ? idx[0][s0] : (k == 1 ? idx[1][s1] : idx[2][s2]);
                        const int m = X.P * X.nc[k];
                        free_ = free_ && ak > 0 && ak < m && (k < DIM - 1 || (ak >= X.cn_lo && ak <= X.cn_hi));
                        id += (int64_t)(k < DIM - 1 ? ak - 1 : ak - X.cn_lo) * st;
                        st *= m - 1;
                    }
                    if (!free_) continue;
                    double xv[DIM];
                    ld_node<DIM>(xc + id * DIM, xv);
#pragma unroll
                    for (int c = 0; c < DIM; ++c) acc[c] = fma(w, xv[c], acc[c]);
                }
        double* yp = yf + t * DIM;
        if (DIM == 2 && (reinterpret_cast<uintptr_t>(yp) & 15) == 0) {
            double2 y = beta == 0.0 ? make_double2(0.0, 0.0) : *reinterpret_cast<const double2*>(yp);
            y.x = (beta == 0.0 ? 0.0 : beta * y.x) + alpha * acc[0];
            y.y = (beta == 0.0 ? 0.0 : beta * y.y) + alpha * acc[DIM - 1];
            *reinterpret_cast<double2*>(yp) = y;
        } else {
#pragma unroll
            for (int c = 0; c < DIM; ++c) yp[c] = (beta == 0.0 ? 0.0 : beta * yp[c]) + alpha * acc[c];
        }
    } else {               // fine vertex (pressure)
        int64_t r = t - X.nfree_f;
#pragma unroll
        for (int k = 0; k < DIM; ++k) {
            const int m = 2 * X.nc[k] + 1;
            const int v = k < DIM - 1 ? (int)(r % m) : (int)r + X.fv_lo;
            if (k < DIM - 1) r /= m;
            else if (v < X.rv_lo || v > X.rv_hi) return;
            q1_interp(v, idx[k], wt[k]);
        }
        double acc = 0.0;
#pragma unroll
        for (int s2 = 0; s2 < N2; ++s2)
#pragma unroll
            for (int s1 = 0; s1 < 3; ++s1)
#pragma unroll
                for (int s0 = 0; s0 < 3; ++s0) {
                    double w = wt[0][s0] * wt[1][s1];
                    if (DIM > 2) w *= wt[2][s2];
                    if (w == 0.0) continue;
                    int64_t id = 0, st = 1;
                    bool in = true;
#pragma unroll
                    for (int k = 0; k < DIM; ++k) {
                        const int ak = k == 0 ? idx[0][s0] : (k == 1 ? idx[1][s1] : idx[2][s2]);
                        in = in && (k < DIM - 1 || (ak >= X.cv_lo && ak <= X.cv_hi));
                        id += (int64_t)(k < DIM - 1 ? ak : ak - X.cv_lo) * st;
                        st *= X.nc[k] + 1;
                    }
                    if (!in) continue;
                    acc = fma(w, __ldg(xc + X.nvel_c + id), acc);
                }
        double* yp = yf + X.nvel_f + (t - X.nfree_f);
        *yp = (beta == 0.0 ? 0.0 : beta * *yp) + alpha * acc;
    }
}

// b_c = P^T r_f
template <int DIM>
__global__ void __launch_bounds__(256) xs_restrict_kernel(XArgs X, const double* __restrict__ rf,
                                                          double* __restrict__ bc) {
    constexpr int N2 = DIM > 2 ? 5 : 1;
    const int64_t total = X.nfree_c + X.nvert_c;
    const int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (t >= total) return;
    int idx[3][5];
    double wt[3][5];
    if (t < X.nfree_c) {   // coarse velocity node
        int64_t r = t;
#pragma unroll
        for (int k = 0; k < DIM; ++k) {
            const int m = X.P * X.nc[k] - 1;
            const int c = k < DIM - 1 ? (int)(r % m) + 1 : (int)r + X.cn_lo;
            if (k < DIM - 1) r /= m;
            const int lo = k < DIM - 1 ? 1 : X.rn_lo, hi = k < DIM - 1 ? 2 * X.P * X.nc[k] - 1 : X.rn_hi;
            if (X.P == 2) q2_gather(c, lo, hi, idx[k], wt[k]);
            else q1_gather(c, lo, hi, idx[k], wt[k]);
        }
        double acc[DIM];
#pragma unroll
        for (int c = 0; c < DIM; ++c) acc[c] = 0.0;
#pragma unroll
        for (int s2 = 0; s2 < N2; ++s2)
#pragma unroll
            for (int s1 = 0; s1 < 5; ++s1)
#pragma unroll
                for (int s0 = 0; s0 < 5; ++s0) {
                    double w = wt[0][s0] * wt[1][s1];
                    if (DIM > 2) w *= wt[2][s2];
                    if (w == 0.0) continue;
                    int64_t id = 0, st = 1;
#pragma unroll
                    for (int k = 0; k < DIM; ++k) {
                        const int ak = k == 0 ? idx[0][s0] : (k == 1 ? idx[1][s1] : idx[2][s2]);
                        id += (int64_t)(k < DIM - 1 ? ak - 1 : ak - X.fn_lo) * st;
                        st *= 2 * X.P * X.nc[k] - 1;
                    }
                    double rv[DIM];
                    ld_node<DIM>(rf + id * DIM, rv);
#pragma unroll
                    for (int c = 0; c < DIM; ++c) acc[c] = fma(w, rv[c], acc[c]);
                }
        double* bp = bc + t * DIM;
        if (DIM == 2 && (reinterpret_cast<uintptr_t>(bp) & 15) == 0)
            *reinterpret_cast<double2*>(bp) = make_double2(acc[0], acc[DIM - 1]);
        else {
#pragma unroll
            for (int c = 0; c < DIM; ++c) bp[c] = acc[c];
        }
    } else {               // coarse vertex
        int64_t r = t - X.nfree_c;
#pragma unroll
        for (int k = 0; k < DIM; ++k) {
            const int m = X.nc[k] + 1;
            const int c = k < DIM - 1 ? (int)(r % m) : (int)r + X.cv_lo;
            if (k < DIM - 1) r /= m;
            q1_gather(c, k < DIM - 1 ? 0 : X.rv_lo, k < DIM - 1 ? 2 * X.nc[k] : X.rv_hi, idx[k], wt[k]);
        }
        double acc = 0.0;
#pragma unroll
        for (int s2 = 0; s2 < N2; ++s2)
#pragma unroll
            for (int s1 = 0; s1 < 5; ++s1)
#pragma unroll
                for (int s0 = 0; s0 < 5; ++s0) {
                    double w = wt[0][s0] * wt[1][s1];
                    if (DIM > 2) w *= wt[2][s2];
                    if (w == 0.0) continue;
                    int64_t id = 0, st = 1;
#pragma unroll
                    for (int k = 0; k < DIM; ++k) {
                        const int ak = k == 0 ? idx[0][s0] : (k == 1 ? idx[1][s1] : idx[2][s2]);
                        id += (int64_t)(k < DIM - 1 ? ak : ak - X.fv_lo) * st;
                        st *= 2 * X.nc[k] + 1;
                    }
                    acc = fma(w, __ldg(rf + X.nvel_f + id), acc);
                }
        bc[X.nvel_c + (t - X.nfree_c)] = acc;
    }
}

// seeded test vector in [-1, 1) (splitmix64 of the index)
__global__ void xs_seed_kernel(int64_t n, uint64_t seed, double* v) {
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
        uint64_t z = seed + 0x9E3779B97F4A7C15ull * (uint64_t)(i + 1);
        z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ull;
        z = (z ^ (z >> 27)) * 0x94D049BB133111EBull;
        z ^= z >> 31;
        v[i] = (double)(z >> 11) * (1.0 / 4503599627370496.0) - 1.0;
    }
}

// out[0] = max |a - b|, out[1] = max |a| as order-preserving bit patterns of non-negative doubles
__global__ void xs_diff_kernel(int64_t n, const double* a, const double* b, unsigned long long* out) {
    unsigned long long d = 0, m = 0;
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
        const double e = fabs(a[i] - b[i]);
        const unsigned long long be = e != e ? ~0ull : (unsigned long long)__double_as_longlong(e);
        d = be > d ? be : d;
        const unsigned long long ba = (unsigned long long)__double_as_longlong(fabs(a[i]));
        m = ba > m ? ba : m;
    }
    atomicMax(out, d);
    atomicMax(out + 1, m);
}

XArgs make_args(const XStruct& S) {
    XArgs X{};
    X.dim = S.dim;
    X.P = S.P;
    for (int k = 0; k < 3; ++k) X.nc[k] = k < S.dim ? S.nc[k] : 1;
    X.fn_lo = S.fn_lo; X.fn_hi = S.fn_hi; X.fv_lo = S.fv_lo; X.fv_hi = S.fv_hi;
    X.rn_lo = S.rn_lo; X.rn_hi = S.rn_hi; X.rv_lo = S.rv_lo; X.rv_hi = S.rv_hi;
    X.cn_lo = S.cn_lo; X.cn_hi = S.cn_hi; X.cv_lo = S.cv_lo; X.cv_hi = S.cv_hi;
    X.nfree_f = X.nfree_c = X.nvert_f = X.nvert_c = 1;
    for (int k = 0; k < S.dim; ++k) {   // last axis: the window's layers
        const bool last = k == S.dim - 1;
        X.nfree_f *= last ? (int64_t)(S.fn_hi - S.fn_lo + 1) : (int64_t)(2 * S.P * X.nc[k] - 1);
        X.nfree_c *= last ? (int64_t)(S.cn_hi - S.cn_lo + 1) : (int64_t)(S.P * X.nc[k] - 1);
        X.nvert_f *= last ? (int64_t)(S.fv_hi - S.fv_lo + 1) : (int64_t)(2 * X.nc[k] + 1);
        X.nvert_c *= last ? (int64_t)(S.cv_hi - S.cv_lo + 1) : (int64_t)(X.nc[k] + 1);
    }
    X.nvel_f = S.dim * X.nfree_f;
    X.nvel_c = S.dim * X.nfree_c;
    return X;
}

}  // namespace

rav_status xs_build(const rav_grid* f, const rav_grid* c, int64_t n_fine, int64_t n_coarse, XStruct& S) {
    S = XStruct{};
    if (!f || !c) { set_error("structured transfer: NULL grid"); return RAV_ERR_ARG; }
    if (f->dim != c->dim || (f->dim != 2 && f->dim != 3)) { set_error("structured transfer: dim mismatch"); return RAV_ERR_ARG; }
    const int Pf = f->vel_order == 1 ? 1 : 2, Pc = c->vel_order == 1 ? 1 : 2;
    if (Pf != Pc) { set_error("structured transfer: element pairs differ"); return RAV_ERR_ARG; }
    for (int k = 0; k < f->dim; ++k)
        if (c->ncell[k] < 1 || f->ncell[k] != 2 * c->ncell[k]) {
            set_error("structured transfer: the fine grid must be the uniform refinement of the coarse one");
            return RAV_ERR_ARG;
        }
    S.dim = f->dim;
    S.P = Pf;
    for (int k = 0; k < 3; ++k) S.nc[k] = k < f->dim ? c->ncell[k] : 1;
    // last-axis windows: whole grids take every free node layer / vertex layer
    const int L = f->dim - 1;
    const int fnm = Pf * f->ncell[L] - 1, cnm = Pf * c->ncell[L] - 1;   // free node layers 1 .. m
    if (f->win) {
        S.fn_lo = f->node_lo; S.fn_hi = f->node_hi; S.fv_lo = f->vert_lo; S.fv_hi = f->vert_hi;
        S.rn_lo = f->rnode_lo; S.rn_hi = f->rnode_hi; S.rv_lo = f->rvert_lo; S.rv_hi = f->rvert_hi;
    } else {
        S.fn_lo = S.rn_lo = 1; S.fn_hi = S.rn_hi = fnm;
        S.fv_lo = S.rv_lo = 0; S.fv_hi = S.rv_hi = f->ncell[L];
    }
    if (c->win) {
        S.cn_lo = c->node_lo; S.cn_hi = c->node_hi; S.cv_lo = c->vert_lo; S.cv_hi = c->vert_hi;
    } else {
        S.cn_lo = 1; S.cn_hi = cnm; S.cv_lo = 0; S.cv_hi = c->ncell[L];
    }
    if (S.fn_lo < 1 || S.fn_hi > fnm || S.fn_lo > S.fn_hi || S.cn_lo < 1 || S.cn_hi > cnm || S.cn_lo > S.cn_hi ||
        S.fv_lo < 0 || S.fv_hi > f->ncell[L] || S.cv_lo < 0 || S.cv_hi > c->ncell[L] ||
        S.rn_lo < S.fn_lo || S.rn_hi > S.fn_hi || S.rv_lo < S.fv_lo || S.rv_hi > S.fv_hi) {
        set_error("structured transfer: inconsistent slab windows");
        return RAV_ERR_ARG;
    }
    const XArgs X = make_args(S);
    if (X.nvel_f + X.nvert_f != n_fine || X.nvel_c + X.nvert_c != n_coarse) {
        set_error("structured transfer: grid sizes (%lld x %lld) do not match P (%lld x %lld)",
                  (long long)(X.nvel_f + X.nvert_f), (long long)(X.nvel_c + X.nvert_c), (long long)n_fine,
                  (long long)n_coarse);
        return RAV_ERR_ARG;
    }
    S.n_fine = n_fine;
    S.n_coarse = n_coarse;
    S.on = 1;
    return RAV_OK;
}

rav_status launch_xs_prolong(const XStruct& S, const double* xc, double* yf, double alpha, double beta,
                             cudaStream_t s) {
    const XArgs X = make_args(S);
    const int64_t total = X.nfree_f + X.nvert_f;
    const unsigned blocks = (unsigned)std::max<int64_t>(1, cdiv(total, 256));
    if (S.dim == 2) xs_prolong_kernel<2><<<blocks, 256, 0, s>>>(X, xc, yf, alpha, beta);
    else xs_prolong_kernel<3><<<blocks, 256, 0, s>>>(X, xc, yf, alpha, beta);
    count_launch();
    RAV_CHECK_LAUNCH();
    return RAV_OK;
}

rav_status launch_xs_restrict(const XStruct& S, const double* rf, double* bc, cudaStream_t s) {
    const XArgs X = make_args(S);
    const int64_t total = X.nfree_c + X.nvert_c;
    const unsigned blocks = (unsigned)std::max<int64_t>(1, cdiv(total, 256));
    if (S.dim == 2) xs_restrict_kernel<2><<<blocks, 256, 0, s>>>(X, rf, bc);
    else xs_restrict_kernel<3><<<blocks, 256, 0, s>>>(X, rf, bc);
    count_launch();
    RAV_CHECK_LAUNCH();
    return RAV_OK;
}

// apply both forms to seeded vectors; |stencil - CSR| <= 1e-13 max|CSR result| or RAV_ERR_ARG
rav_status xs_verify(const XStruct& S, const Csr& P, const Csr& PT, cudaStream_t s) {
    const int64_t nf = S.n_fine, nc = S.n_coarse;
    double *vc = nullptr, *vf = nullptr, *y1 = nullptr, *y2 = nullptr;
    unsigned long long* dd = nullptr;
    const int64_t big = std::max(nf, nc);
    RAV_CUDA(cudaMallocAsync(&vc, sizeof(double) * std::max<int64_t>(1, nc), s));
    RAV_CUDA(cudaMallocAsync(&vf, sizeof(double) * std::max<int64_t>(1, nf), s));
    RAV_CUDA(cudaMallocAsync(&y1, sizeof(double) * std::max<int64_t>(1, big), s));
    RAV_CUDA(cudaMallocAsync(&y2, sizeof(double) * std::max<int64_t>(1, big), s));
    RAV_CUDA(cudaMallocAsync(&dd, sizeof(unsigned long long) * 4, s));
    RAV_CUDA(cudaMemsetAsync(dd, 0, sizeof(unsigned long long) * 4, s));
    const int gb = (int)std::min<int64_t>(cdiv(big, 256), (int64_t)num_sms() * 8);
    xs_seed_kernel<<<gb, 256, 0, s>>>(nc, 0x5eed1ull, vc);
    xs_seed_kernel<<<gb, 256, 0, s>>>(nf, 0x5eed2ull, vf);
    RAV_CHECK_LAUNCH();
    RAV_TRY(launch_spmv(P, vc, y1, 1.0, 0.0, s));
    RAV_TRY(launch_xs_prolong(S, vc, y2, 1.0, 0.0, s));
    xs_diff_kernel<<<gb, 256, 0, s>>>(nf, y1, y2, dd);
    RAV_TRY(launch_spmv(PT, vf, y1, 1.0, 0.0, s));
    RAV_TRY(launch_xs_restrict(S, vf, y2, s));
    xs_diff_kernel<<<gb, 256, 0, s>>>(nc, y1, y2, dd + 2);
    RAV_CHECK_LAUNCH();
    unsigned long long h[4] = {0, 0, 0, 0};
    RAV_CUDA(cudaMemcpyAsync(h, dd, sizeof(h), cudaMemcpyDeviceToHost, s));
    RAV_CUDA(cudaStreamSynchronize(s));
    for (void* p : {(void*)vc, (void*)vf, (void*)y1, (void*)y2, (void*)dd}) cudaFreeAsync(p, s);
    double v[4];
    memcpy(v, h, sizeof(v));
    const bool ok = h[0] != ~0ull && h[2] != ~0ull && v[0] <= 1e-13 * v[1] && v[2] <= 1e-13 * v[3];
    if (!ok) {
        set_error("structured transfer does not match the level's P (max diff %.3e / %.3e, P^T %.3e / %.3e)", v[0],
                  v[1], v[2], v[3]);
        return RAV_ERR_ARG;
    }
    return RAV_OK;
}

}  // namespace rav
