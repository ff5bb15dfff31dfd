// schur.cu -- factored ("Schur") format of the restricted rows of L_i^{-1} for
// Vanka patches of Taylor-Hood-type saddle-point operators (SURVEY section 8
// rows a4/a5; P:114 L_i = R_i L R_i^T, Eq. 13).
//
// A Vanka patch holds one pressure DoF p and the velocity DoFs of nn nodes.
// For the Laplacian-form viscous term (Eq. 7) the velocity block of L is
// I_d (x) A_s (the same scalar matrix for every component, no coupling between
// components), so with b the velocity-pressure column of L_i and c = L_pp:
//
//   L_i = [ I_d(x)A_s  b ]      L_i^{-1} = [ I(x)A_s^{-1} + g S^{-1} g^T   -g S^{-1} ]
//         [ b^T        c ]                 [ -S^{-1} g^T                    S^{-1}  ]
//
// g = (I(x)A_s^{-1}) b, S = c - b^T g (the Schur complement of the pressure DoF).
// Applied to r_i = (r_u, r_p):  t = S^{-1} (g^T r_u - r_p),
//   du_(k,c) = (A_s^{-1} r_c)_k + g_(k,c) t,   dp = -t,
// which is exactly row (k,c) / row p of L_i^{-1} times r_i.  Only the restricted
// rows of A_s^{-1} (restricted nodes k, P:122 / R3), g, 1/S and the weights are
// stored: 2D PoU 240 doubles per patch instead of 969 rows entries (3D: 3779
// instead of 30832).  setup verifies the structure on every patch and the
// caller falls back to the generic row formats when it does not hold.
//
// The setup solves A_s [G | Y] = [b_0 .. b_{d-1} | e_k (k restricted)] by
// Gaussian elimination with partial pivoting in shared memory (one CTA per
// patch; 2D nn = 25, 3D nn = 125).
#include <algorithm>
#include <climits>
#include <vector>

#include <cub/cub.cuh>

#include "internal.cuh"

namespace rav {

constexpr int ST = 128;

struct SchurArgs {
    const int64_t* rp;
    const int32_t* ci;
    const double* val;
    int64_t np;
    const int64_t* poffs;
    const int32_t* pdofs;
    const double* pw;
    int64_t nvel;
    int D;           // velocity components (interleaved: dof = D * node + c)
    int nnmax;       // max nodes per patch
    int mnmax;       // max restricted nodes per patch
    int ld;          // leading dimension of the augmented matrix (>= nnmax + D + mnmax)
    int layout;      // 4: thread SoA chunks, 5: per-patch (warp kernel), 6: diagonal Vanka (per patch)
    // thread layout (4)
    int MT, NN;
    int64_t pairs;   // double2 pairs per chunk
    double* facT;
    int32_t* ND;     // [chunk][NN][32] node dof (component 0)
    int32_t* PD;     // [chunk][32] pressure dof
    int32_t* NR;     // [chunk][32] restricted node count
    double* AUX;     // [chunk][MT + 2][32]: w_k (k < MT), w_p, 1/S
    // per-patch layout (5)
    const int64_t* foffs;  // per patch: Y (MT x nn col-major, stride MT), g (nn*D), aux (MT + 2)
    double* fac;
    int32_t* nodes;  // per patch node dofs: nodeoffs[i] ... (nn_i)
    const int64_t* nodeoffs;
    int32_t* pdof;   // per patch pressure dof
    int32_t* nres_nodes;
    unsigned int* fail;          // bit 0: structure does not hold; bit 1: singular
    unsigned long long* bad;     // smallest singular patch
    unsigned long long* alg;     // sum of algorithmic bytes of the stored data
    int comp_verified;           // the node-blocked build verified equal component blocks and no
                                 // cross-component entries for the whole operator (nb.cu)
    int gj;                      // 3D: blocked Gauss-Jordan on the FP64 tensor cores (gj_dmma)
    int hbits;                   // node hash table of 2^hbits slots (>= 2 nnmax) in shared memory
};

__device__ __forceinline__ int64_t tri_col_start(int j, int D) { return (int64_t)j * (j + 1) / 2 + (int64_t)j * D; }

// ---- 3D local solves on the FP64 tensor cores --------------------------------------------------
// D = C + A B for 8x8 (C, D) / 8x4 (A) / 4x8 (B) f64 tiles: one DMMA (mma.sync m8n8k4 f64; sm_100a
// has no tcgen05 kind for f64).  Fragments: a = A[lane/4][lane%4], b = B[lane%4][lane/4],
// c = C[lane/4][2 (lane%4) + {0,1}].
__device__ __forceinline__ void dmma884(double (&c)[2], double a, double b) {
    asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};"
                 : "+d"(c[0]), "+d"(c[1])
                 : "d"(a), "d"(b));
}

constexpr int GJ_NB = 16;    // 8-wide block rows / columns of A_s (nn <= 128)
constexpr int GJ_NJ = 20;    // + 4 block columns of right-hand sides (D + mn <= 32)
constexpr int GJ_LDP = 168;  // stride of a published block row (B-fragment reads: 2 wavefronts)
constexpr int GJ_BUF = 8 * GJ_LDP + 3 * 64;   // published block row, Dinv, and the next diagonal helper tiles

// In-place inverse of an 8 x 8 tile held in accumulator layout (thread (g, t) = lane (4g + t) holds
// D[g][2t], D[g][2t + 1]): Gauss-Jordan, 8 pivots, rows and columns by shuffles.  Pivot row
// 8K + p below 1e-14 ||row||_inf (S:268's tolerance) sets *s_fail = 2.
__device__ __forceinline__ void gj_inv8(double& d0, double& d1, int g, int t, int K, int nn, const double* rn,
                                        int* s_fail) {
#pragma unroll
    for (int p = 0; p < 8; ++p) {
        const double f0 = __shfl_sync(0xffffffffu, d0, 4 * g + (p >> 1));
        const double f1 = __shfl_sync(0xffffffffu, d1, 4 * g + (p >> 1));
        const double r0 = __shfl_sync(0xffffffffu, d0, 4 * p + t);
        const double r1 = __shfl_sync(0xffffffffu, d1, 4 * p + t);
        const double f = (p & 1) ? f1 : f0;                       // D[g][p]
        const double piv = __shfl_sync(0xffffffffu, f, 4 * p);   // D[p][p]
        const int pr = 8 * K + p;
        if (g == 0 && t == 0 && pr < nn && !(fabs(piv) > 1e-14 * rn[pr])) *s_fail = 2;
        const double inv = 1.0 / piv;
#pragma unroll
        for (int h = 0; h < 2; ++h) {
            const int col = 2 * t + h;
            const double rp = (h ? r1 : r0) * inv;
            double& d = h ? d1 : d0;
            d = g == p ? (col == p ? inv : rp) : (col == p ? -f * inv : fma(-f, rp, d));
        }
    }
}

// A-operand fragments (row g, columns 4 kk + t, kk = 0, 1) of an 8 x 8 tile held in accumulator
// layout: held by lane 4g + 2kk + t/2, slot t & 1
__device__ __forceinline__ void gj_afrag(double d0, double d1, int g, int t, double& A0, double& A1) {
    const double x00 = __shfl_sync(0xffffffffu, d0, 4 * g + (t >> 1));
    const double x01 = __shfl_sync(0xffffffffu, d1, 4 * g + (t >> 1));
    const double x10 = __shfl_sync(0xffffffffu, d0, 4 * g + 2 + (t >> 1));
    const double x11 = __shfl_sync(0xffffffffu, d1, 4 * g + 2 + (t >> 1));
    A0 = (t & 1) ? x01 : x00;
    A1 = (t & 1) ? x11 : x10;
}

// X = A_s^{-1} [b_0 .. b_{D-1} | e_k (k < mn)] (g and the restricted columns of A_s^{-1}, which are
// its restricted rows: A_s is symmetric) for a symmetric positive definite A_s, nn <= 128,
// D + mn <= 32: block Gauss-Jordan elimination without pivoting in 8 x 8 blocks, 16 warps, the
// block updates on the FP64 tensor cores.  Warp I owns block row I of the augmented matrix
// [A_s | R] (rows 8I .. 8I+7, 160 columns) as 20 m8n8k4 accumulator tiles in registers.  The pivot
// rows are never scaled: at step K the buffer K & 1 holds block row K (published by warp K) and
// Dinv_K, the inverse of its diagonal block; every other warp I forms its multiplier
// L = M_IK Dinv_K (two DMMA) and subtracts L M_KJ from its tiles J > K (two DMMA per tile).  At
// the end block row I holds [.. M_II .. | R_I] and X_I = Dinv_I R_I.  The serial part -- the next
// diagonal block's update and 8 x 8 inversion -- is done at step K by warp K, whose own row has
// nothing to update at that step, from the tiles (K+1, K) and (K+1, K+1) that warp K+1 published
// after step K-1: Dinv_{K+1} = (M_{K+1,K+1} - M_{K+1,K} Dinv_K M_{K,K+1})^{-1}.  So it overlaps
// the other warps' tensor-core updates instead of following them.  One barrier per step (double
// buffered).  Rows and columns nn .. 127 are an identity block.  On return (after a barrier) rows
// j < nn of X are in M[j ld + nn + q], q < D + mn, where the elimination path leaves them.
__device__ void gj_dmma(double* M, int ld, int nn, int D, int mn, const double* bcol, const double* rn,
                        int* s_fail) {
    const int tid = threadIdx.x, I = tid >> 5, lane = tid & 31, g = lane >> 2, t = lane & 3;
    const int row = 8 * I + g;
    double c[GJ_NJ][2];
#pragma unroll
    for (int J = 0; J < GJ_NJ; ++J)
#pragma unroll
        for (int h = 0; h < 2; ++h) {
            const int col = 8 * J + 2 * t + h;
            double v;
            if (J < GJ_NB) {
                v = (row < nn && col < nn) ? M[(size_t)row * ld + col] : (row == col ? 1.0 : 0.0);
            } else {
                const int q = col - 8 * GJ_NB;
                v = row >= nn ? 0.0 : q < D ? bcol[row * D + q] : (q - D < mn && row == q - D) ? 1.0 : 0.0;
            }
            c[J][h] = v;
        }
    __syncthreads();   // M is free: from here on it holds the two publication buffers
    // buffer layout: block row [8][GJ_LDP] | Dinv [8][8] | tile (K+1, K) [8][8] | tile (K+1, K+1) [8][8]
    auto put = [&](double* T, double v0, double v1) {
        *reinterpret_cast<double2*>(T + g * 8 + 2 * t) = make_double2(v0, v1);
    };
    double di0 = 0.0, di1 = 0.0;   // Dinv_I (accumulator layout)
    if (I == 0) {
        di0 = c[0][0];
        di1 = c[0][1];
        gj_inv8(di0, di1, g, t, 0, nn, rn, s_fail);
#pragma unroll
        for (int J = 1; J < GJ_NJ; ++J)
            *reinterpret_cast<double2*>(M + g * GJ_LDP + 8 * J + 2 * t) = make_double2(c[J][0], c[J][1]);
        put(M + 8 * GJ_LDP, di0, di1);
    } else if (I == 1) {
        put(M + 8 * GJ_LDP + 64, c[0][0], c[0][1]);
        put(M + 8 * GJ_LDP + 128, c[1][0], c[1][1]);
    }
#pragma unroll   // compile-time K: every tile index below is static (a runtime K made the selects dynamic indexing)
    for (int K = 0; K < GJ_NB; ++K) {
        __syncthreads();
        const double* P = M + (K & 1) * GJ_BUF;    // block row K
        const double* Dv = P + 8 * GJ_LDP;         // Dinv_K
        double* Q = M + ((K + 1) & 1) * GJ_BUF;    // publications for step K + 1
        if (I == K) {   // helper: Dinv_{K+1}
            if (K > 0) {
                di0 = Dv[g * 8 + 2 * t];
                di1 = Dv[g * 8 + 2 * t + 1];
            }
            if (K + 1 < GJ_NB) {
                const double* T1 = Dv + 64;
                const double* T2 = Dv + 128;
                double L[2] = {0.0, 0.0}, A0, A1;
                dmma884(L, T1[g * 8 + t], Dv[t * 8 + g]);             // L = M_{K+1,K} Dinv_K
                dmma884(L, T1[g * 8 + 4 + t], Dv[(4 + t) * 8 + g]);
                gj_afrag(L[0], L[1], g, t, A0, A1);
                double X[2] = {T2[g * 8 + 2 * t], T2[g * 8 + 2 * t + 1]};
                dmma884(X, -A0, P[t * GJ_LDP + 8 * (K + 1) + g]);     // - L M_{K,K+1}
                dmma884(X, -A1, P[(4 + t) * GJ_LDP + 8 * (K + 1) + g]);
                gj_inv8(X[0], X[1], g, t, K + 1, nn, rn, s_fail);
                put(Q + 8 * GJ_LDP, X[0], X[1]);
            }
        } else {
            double A0, A1, L[2] = {0.0, 0.0};
            gj_afrag(c[K][0], c[K][1], g, t, A0, A1);
            dmma884(L, A0, Dv[t * 8 + g]);           // L = M_IK Dinv_K
            dmma884(L, A1, Dv[(4 + t) * 8 + g]);
            gj_afrag(L[0], L[1], g, t, A0, A1);
            A0 = -A0;
            A1 = -A1;
#pragma unroll
            for (int J = K + 1; J < GJ_NJ; ++J) {
                if (J == K + 1 && I == K + 1) continue;   // its diagonal tile: only Dinv is used
                dmma884(c[J], A0, P[t * GJ_LDP + 8 * J + g]);
                dmma884(c[J], A1, P[(4 + t) * GJ_LDP + 8 * J + g]);
            }
            if (K + 1 < GJ_NB && I == K + 1) {
#pragma unroll
                for (int J = K + 2; J < GJ_NJ; ++J)
                    *reinterpret_cast<double2*>(Q + g * GJ_LDP + 8 * J + 2 * t) = make_double2(c[J][0], c[J][1]);
            }
            if (K + 2 < GJ_NB && I == K + 2) {
                put(Q + 8 * GJ_LDP + 64, c[K + 1][0], c[K + 1][1]);
                put(Q + 8 * GJ_LDP + 128, c[K + 2][0], c[K + 2][1]);
            }
        }
    }
    __syncthreads();
    // X_I = Dinv_I R_I: R_I through a per-warp shared-memory tile into B-fragment layout
    double* R = M + 2 * GJ_BUF + I * (8 * 34);
#pragma unroll
    for (int J = GJ_NB; J < GJ_NJ; ++J)
        *reinterpret_cast<double2*>(R + g * 34 + 8 * (J - GJ_NB) + 2 * t) = make_double2(c[J][0], c[J][1]);
    __syncwarp();
    double A0, A1;
    gj_afrag(di0, di1, g, t, A0, A1);
#pragma unroll
    for (int J = GJ_NB; J < GJ_NJ; ++J) {
        double x[2] = {0.0, 0.0};
        dmma884(x, A0, R[t * 34 + 8 * (J - GJ_NB) + g]);
        dmma884(x, A1, R[(4 + t) * 34 + 8 * (J - GJ_NB) + g]);
        c[J][0] = x[0];
        c[J][1] = x[1];
    }
    __syncthreads();
#pragma unroll
    for (int J = GJ_NB; J < GJ_NJ; ++J)
#pragma unroll
        for (int h = 0; h < 2; ++h) {
            const int q = 8 * (J - GJ_NB) + 2 * t + h;
            if (row < nn && q < D + mn) M[(size_t)row * ld + nn + q] = c[J][h];
        }
    __syncthreads();
}

// NT threads per CTA: 128 for the small 2D patches (several CTAs per SM), 512 for the
// 3D patches whose ~150 KB of shared memory allow one CTA per SM
template <int NT>
__global__ void __launch_bounds__(NT) schur_factor_kernel(SchurArgs a) {
    extern __shared__ double smem[];
    const int tid = threadIdx.x;
    const int D = a.D;
    double* M = smem;                                         // nnmax x ld
    double* rn = M + (size_t)a.nnmax * a.ld;                  // nnmax
    double* bcol = rn + a.nnmax;                              // nnmax * D (B column of L_i)
    double* wnode = bcol + (size_t)a.nnmax * D;               // nnmax weights (per node)
    int32_t* ndof = (int32_t*)(wnode + a.nnmax);              // nnmax: dof of component 0
    int32_t* hkey = ndof + a.nnmax;                           // node id (dof / D) -> local index:
    int32_t* hval = hkey + (1 << a.hbits);                    // open addressing, linear probing
    const unsigned hmask = (1u << a.hbits) - 1;
    auto hslot = [&](int nd) { return ((unsigned)nd * 2654435761u) >> (32 - a.hbits); };
    auto hfind = [&](int nd) {   // local index of node nd in the patch, or -1
        for (unsigned h = hslot(nd);; h = (h + 1) & hmask) {
            const int k = hkey[h];
            if (k == nd) return (int)hval[h];
            if (k < 0) return -1;
        }
    };
    __shared__ int s_nn, s_mn, s_pd, s_fail, s_piv, s_sym, s_np, s_pidx;
    __shared__ double s_wp, s_cpp;

    for (int64_t i = blockIdx.x; i < a.np; i += gridDim.x) {
        const int64_t off = a.poffs[i];
        const int n = (int)(a.poffs[i + 1] - off);
        __syncthreads();
        // the patch's DoF list and weights into shared memory by all threads (M is free here and
        // holds nnmax * ld >= n doubles + ints), then the sequential scan reads shared memory only
        double* stw = M;
        int32_t* std_ = reinterpret_cast<int32_t*>(M + n);
        const bool staged = (size_t)n * 12 + 8 <= (size_t)a.nnmax * a.ld * 8;
        if (staged)
            for (int t = tid; t < n; t += NT) {
                std_[t] = a.pdofs[off + t];
                stw[t] = a.pw[off + t];
            }
        __syncthreads();
        // node table + structure checks, in parallel over the staged DoF list (a single thread
        // scanning it held the other warps at the barrier).  The list must be: node groups of D
        // consecutive entries (dof = node D + c, c = 0 .. D-1, one weight per group, no node twice
        // in a row), restricted (w > 0) groups first, and exactly one pressure DoF anywhere.
        if (staged) {
            if (tid == 0) { s_np = 0; s_pidx = -1; s_fail = 0; s_cpp = 0.0; s_mn = 0; }
            __syncthreads();
            for (int t = tid; t < n; t += NT)
                if (std_[t] >= a.nvel) {
                    atomicAdd(&s_np, 1);
                    s_pidx = t;
                }
            __syncthreads();
            const int nvent = n - s_np;     // velocity entries
            const int pidx = s_pidx;
            if (tid == 0 && (s_np != 1 || nvent % D != 0 || nvent / D < 1 || nvent / D > a.nnmax)) s_fail = 1;
            __syncthreads();
            if (!s_fail) {
                for (int t = tid; t < n; t += NT) {
                    if (t == pidx) continue;
                    const int v = t - (t > pidx ? 1 : 0);          // index among the velocity entries
                    const int dof = std_[t];
                    const double w = stw[t];
                    const int c = dof % D;
                    if (v % D == 0) {
                        if (c != 0) atomicOr((unsigned int*)&s_fail, 1u);
                        const int j = v / D;
                        ndof[j] = dof;
                        wnode[j] = w;
                    } else {
                        const int tp = (t - 1 == pidx) ? t - 2 : t - 1;   // previous velocity entry
                        if (dof != std_[tp] + 1 || c == 0 || w != stw[tp]) atomicOr((unsigned int*)&s_fail, 1u);
                    }
                }
            }
            __syncthreads();
            if (!s_fail) {
                const int nn = nvent / D;
                for (int j = tid; j < nn; j += NT) {
                    if (wnode[j] > 0.0) {
                        atomicAdd(&s_mn, 1);
                        if (j > 0 && !(wnode[j - 1] > 0.0)) atomicOr((unsigned int*)&s_fail, 1u);   // restricted first
                    }
                    if (j > 0 && ndof[j] == ndof[j - 1]) atomicOr((unsigned int*)&s_fail, 1u);
                }
            }
            __syncthreads();
            if (tid == 0) {
                s_nn = nvent / D;
                s_pd = pidx >= 0 ? std_[pidx] : -1;
                s_wp = pidx >= 0 ? stw[pidx] : 0.0;
                if (s_mn > a.mnmax) s_fail = 1;
            }
        } else {   // DoF list larger than the staging space: the sequential scan from global memory
            if (tid == 0) {
                // node table + structure checks (sequential: n <= a few hundred)
                int nn = 0, mn = 0, pd = -1, fail = 0, cnt = 0, cur = -1;
                double wcur = 0.0, wp = 0.0;
                bool in_rest = true;
                for (int t = 0; t < n && !fail; ++t) {
                    const int dof = staged ? std_[t] : a.pdofs[off + t];
                    const double w = staged ? stw[t] : a.pw[off + t];
                    if (dof >= a.nvel) {
                        if (pd >= 0) fail = 1;
                        pd = dof;
                        wp = w;
                        continue;
                    }
                    const int node = dof / D, c = dof % D;
                    if (node != cur) {
                        if (cur >= 0 && cnt != D) fail = 1;
                        if (c != 0 || nn >= a.nnmax) { fail = 1; break; }
                        cur = node;
                        cnt = 1;
                        wcur = w;
                        ndof[nn] = dof;
                        wnode[nn] = w;
                        if (w > 0.0) {
                            if (!in_rest) fail = 1;   // restricted nodes must come first
                            ++mn;
                        } else {
                            in_rest = false;
                        }
                        ++nn;
                    } else {
                        if (c != cnt || w != wcur) fail = 1;
                        ++cnt;
                    }
                }
                if (cur >= 0 && cnt != D) fail = 1;
                if (pd < 0 || nn < 1 || mn > a.mnmax) fail = 1;
                s_nn = nn;
                s_mn = mn;
                s_pd = pd;
                s_wp = wp;
                s_cpp = 0.0;
                s_fail = fail;
            }
        }
        __syncthreads();
        if (s_fail) {
            if (tid == 0) atomicOr(a.fail, 1u);
            continue;
        }
        const int nn = s_nn, mn = s_mn, pd = s_pd;
        const int W = nn + D + mn, ld = a.ld;
        for (int t = tid; t < nn * ld; t += NT) M[t] = 0.0;
        for (int t = tid; t < nn * D; t += NT) bcol[t] = 0.0;
        for (int t = tid; t <= (int)hmask; t += NT) hkey[t] = -1;
        __syncthreads();
        for (int t = tid; t < nn; t += NT) {   // the patch's nodes into the hash table
            const int nd = ndof[t] / D;
            for (unsigned h = hslot(nd);; h = (h + 1) & hmask) {
                const int old = atomicCAS(&hkey[h], -1, nd);
                if (old == -1) { hval[h] = t; break; }
                if (old == nd) { atomicOr((unsigned int*)&s_fail, 1u); break; }   // a node twice
            }
        }
        __syncthreads();
        // gather A_s (component 0 rows), the B column, and verify components 1..D-1.  With the
        // component structure verified for the whole operator (nb.cu), the component-0 rows of A_s
        // are gathered by a merge of the sorted row with the sorted node list and nothing else is
        // re-checked
        if (a.comp_verified) {
            // one warp per component-0 row, its lanes over the row's entries; the lane that meets the
            // patch's pressure column also takes the other components' B entries, at the same offset of
            // their rows (verified identical structure).  The loads are issued ahead of their use:
            // lane m first loads the row starts of the warp's m-th row and of the next D - 1 component
            // rows, then two rows at a time every lane loads all its (column, value) pairs
            // (GATHER_U per row) before the searches and stores -- the dependent global round trips
            // of a serial walk held the CTA (one per SM in 3D) most of the kernel's time.
            constexpr int NW = NT / 32, GATHER_U = 5;
            const int warp = tid >> 5, lane = tid & 31;
            const int nrw = nn > warp ? (nn - warp + NW - 1) / NW : 0;   // rows j = warp + NW m
            int64_t rs[4] = {0, 0, 0, 0};                               // rp[row + c], c <= D (D <= 3)
            for (int m0 = 0; m0 < nrw; m0 += 32) {
                if (m0 + lane < nrw) {
                    const int row = ndof[warp + NW * (m0 + lane)];
#pragma unroll
                    for (int c = 0; c < 4; ++c)
                        if (c <= D) rs[c] = __ldg(a.rp + row + c);
                }
                const int mend = min(nrw, m0 + 32);
                for (int m = m0; m < mend; m += 2) {
                    int64_t k0[2], k1[2];
                    int col[2][GATHER_U];
                    double vv[2][GATHER_U];
#pragma unroll
                    for (int r = 0; r < 2; ++r) {
                        const int src = min(m + r, mend - 1) - m0;
                        k0[r] = __shfl_sync(0xffffffffu, rs[0], src);
                        k1[r] = m + r < mend ? __shfl_sync(0xffffffffu, rs[1], src) : k0[r];
#pragma unroll
                        for (int u = 0; u < GATHER_U; ++u) {
                            const int64_t k = k0[r] + lane + 32 * u;
                            const bool ok = k < k1[r];
                            col[r][u] = ok ? __ldg(a.ci + k) : -1;
                            vv[r][u] = ok ? __ldg(a.val + k) : 0.0;
                        }
                    }
#pragma unroll
                    for (int r = 0; r < 2; ++r) {
                        if (m + r >= mend) break;
                        const int j = warp + NW * (m + r);
                        const int src = m + r - m0;
                        int64_t kc[3];
#pragma unroll
                        for (int c = 1; c < 3; ++c) kc[c] = __shfl_sync(0xffffffffu, rs[c], src);
                        auto put = [&](int cl, double v, int64_t k) {
                            if (cl < 0) return;
                            if (cl == pd) {
                                bcol[j * D] = v;
#pragma unroll
                                for (int c = 1; c < 3; ++c)
                                    if (c < D) bcol[j * D + c] = __ldg(a.val + kc[c] + (k - k0[r]));
                                return;
                            }
                            if (cl >= a.nvel) return;
                            const int l = hfind(cl / D);
                            if (l >= 0) M[(size_t)j * ld + l] = v;
                        };
#pragma unroll
                        for (int u = 0; u < GATHER_U; ++u) put(col[r][u], vv[r][u], k0[r] + lane + 32 * u);
                        for (int64_t k = k0[r] + 32 * GATHER_U + lane; k < k1[r]; k += 32)   // long rows
                            put(__ldg(a.ci + k), __ldg(a.val + k), k);
                    }
                }
            }
        }
        for (int t = tid; t < nn * D && !a.comp_verified; t += NT) {
            const int j = t / D, c = t % D;
            const int row = ndof[j] + c;
            for (int64_t k = a.rp[row]; k < a.rp[row + 1]; ++k) {
                const int col = a.ci[k];
                const double v = a.val[k];
                if (col == pd) { bcol[j * D + c] = v; continue; }
                if (col >= a.nvel) continue;    // other pressure DoFs are outside the patch
                const int cc = col % D;
                const int l = hfind(col / D);
                if (l < 0) continue;
                if (cc != c) {
                    if (v != 0.0) atomicOr((unsigned int*)&s_fail, 1u);
                    continue;
                }
                if (c == 0) M[(size_t)j * ld + l] = v;
            }
        }
        __syncthreads();
        for (int t = tid; t < nn * (D - 1) && !a.comp_verified; t += NT) {
            const int j = t / (D - 1), c = 1 + t % (D - 1);
            const int row = ndof[j] + c;
            for (int64_t k = a.rp[row]; k < a.rp[row + 1]; ++k) {
                const int col = a.ci[k];
                if (col >= a.nvel || col % D != c) continue;
                const int l = hfind(col / D);
                if (l < 0) continue;
                if (M[(size_t)j * ld + l] != a.val[k]) atomicOr((unsigned int*)&s_fail, 1u);
            }
        }
        // pressure row: symmetric B and C_pp (entries in parallel: one thread walking a 3D pressure
        // row of 375 entries with dependent global loads kept the other warps at the barrier)
        for (int64_t k = a.rp[pd] + tid; k < a.rp[pd + 1]; k += NT) {
            const int col = a.ci[k];
            if (col == pd) { s_cpp = a.val[k]; continue; }
            if (col >= a.nvel) continue;
            const int l = hfind(col / D);
            if (l < 0) continue;
            if (bcol[l * D + col % D] != a.val[k]) atomicOr((unsigned int*)&s_fail, 1u);
        }
        __syncthreads();
        if (s_fail) {
            if (tid == 0) atomicOr(a.fail, 1u);
            continue;
        }
        if (a.layout == 6) {
            // diagonal Vanka (R17): A_s -> diag(A_s); closed form g_j = b_j / a_jj,
            // S = c - sum b_j g_j; per patch [1/a_jj (nn) | g (nn*D) | w (nn) | w_p | 1/S]
            double* base = a.fac + a.foffs[i];
            double* g = base + nn;
            double* aux = g + (size_t)nn * D;
            for (int t = tid; t < nn; t += NT) {
                const double dj = M[(size_t)t * ld + t];
                base[t] = 1.0 / dj;
                if (!(fabs(dj) > 0.0)) atomicOr((unsigned int*)&s_fail, 2u);
                aux[t] = wnode[t];
            }
            for (int t = tid; t < nn * D; t += NT) g[t] = bcol[t] / M[(size_t)(t / D) * ld + (t / D)];
            for (int j = tid; j < nn; j += NT) a.nodes[a.nodeoffs[i] + j] = ndof[j];
            __syncthreads();
            if (tid < 32) {
                double sacc = 0.0, sa = 0.0;
                for (int t = tid; t < nn * D; t += 32) {
                    const double pr = bcol[t] * g[t];
                    sacc += pr;
                    sa += fabs(pr);
                }
                sacc = warp_sum(sacc);
                sa = warp_sum(sa);
                if (tid == 0) {
                    const double S = s_cpp - sacc;
                    if (!(fabs(S) > 1e-14 * (sa + fabs(s_cpp)))) s_fail = 2;
                    aux[nn] = s_wp;
                    aux[nn + 1] = 1.0 / S;
                    a.pdof[i] = pd;
                    a.nres_nodes[i] = mn;
                    atomicAdd(a.alg, 8ull * ((unsigned long long)nn * (D + 2) + 2) + 4ull * (nn + 1));
                }
            }
            __syncthreads();
            if (s_fail) {
                if (tid == 0) { atomicOr(a.fail, 2u); atomicMin(a.bad, (unsigned long long)i); }
            }
            continue;
        }
        // right-hand sides: B columns, then e_k for the restricted nodes
        for (int t = tid; t < nn * D; t += NT) M[(size_t)(t / D) * ld + nn + (t % D)] = bcol[t];
        for (int k = tid; k < mn; k += NT) M[(size_t)k * ld + nn + D + k] = 1.0;
        // row norms ||row||_inf (pivot tolerance) and the symmetry test of A_s: one warp per row, its
        // lanes over the columns.  A symmetric A_s (every generated operator: the principal block of
        // the SPD viscous operator) is eliminated without pivoting; an unsymmetric block keeps
        // partial pivoting
        if (tid == 0) s_sym = 1;
        __syncthreads();
        for (int r = tid >> 5; r < nn; r += NT / 32) {
            double mx = 0.0;
            bool sym = true;
            for (int c = tid & 31; c < nn; c += 32) {
                const double v = M[(size_t)r * ld + c];
                mx = fmax(mx, fabs(v));
                if (c > r && v != M[(size_t)c * ld + r]) sym = false;
            }
#pragma unroll
            for (int o = 16; o > 0; o >>= 1) mx = fmax(mx, __shfl_xor_sync(0xffffffffu, mx, o));
            if ((tid & 31) == 0) rn[r] = mx;
            if (!sym) s_sym = 0;
        }
        __syncthreads();
        const bool nopiv = s_sym != 0;
        bool gj = false;   // solved on the tensor cores (gj_dmma): no elimination / back substitution
        if constexpr (NT == 512) {
            if (a.gj && nopiv && D == 3 && nn <= 8 * GJ_NB && D + mn <= 8 * (GJ_NJ - GJ_NB)) {
                gj_dmma(M, ld, nn, D, mn, bcol, rn, &s_fail);
                gj = true;
            }
        }
        // Gaussian elimination with partial pivoting (A_s symmetric: A_s^T = A_s)
        for (int c = 0; c < nn && !gj; ++c) {
            if (nopiv) {
                const double piv = M[(size_t)c * ld + c];
                if (tid == 0 && !(fabs(piv) > 1e-14 * rn[c])) s_fail = 2;
                const double inv = 1.0 / piv;
                const int nr = nn - c - 1, ncol = W - c - 1;
                if (nr > 0 && ncol > 0) {
                    const int dq = NT / ncol, dr = NT % ncol;
                    int rr = tid / ncol, cc = tid % ncol;
                    for (int t = tid; t < nr * ncol; t += NT) {
                        const int r = c + 1 + rr, col = c + 1 + cc;
                        M[(size_t)r * ld + col] -= (M[(size_t)r * ld + c] * inv) * M[(size_t)c * ld + col];
                        rr += dq;
                        cc += dr;
                        if (cc >= ncol) { cc -= ncol; ++rr; }
                    }
                }
                __syncthreads();
                continue;
            }
            if (tid < 32) {
                double best = -1.0;
                int bi = c;
                for (int r = c + tid; r < nn; r += 32) {
                    double v = fabs(M[(size_t)r * ld + c]);
                    if (v > best) { best = v; bi = r; }
                }
#pragma unroll
                for (int o = 16; o > 0; o >>= 1) {
                    double ob = __shfl_xor_sync(0xffffffffu, best, o);
                    int oi = __shfl_xor_sync(0xffffffffu, bi, o);
                    if (ob > best || (ob == best && oi < bi)) { best = ob; bi = oi; }
                }
                if (tid == 0) {
                    s_piv = bi;
                    if (!(best > 1e-14 * rn[bi])) s_fail = 2;
                }
            }
            __syncthreads();
            if (s_fail) break;
            const int p = s_piv;
            if (p != c) {
                for (int t = c + tid; t < W; t += NT) {
                    double u = M[(size_t)c * ld + t];
                    M[(size_t)c * ld + t] = M[(size_t)p * ld + t];
                    M[(size_t)p * ld + t] = u;
                }
                if (tid == 0) { double u = rn[c]; rn[c] = rn[p]; rn[p] = u; }
            }
            __syncthreads();
            const double inv = 1.0 / M[(size_t)c * ld + c];
            const int nr = nn - c - 1, ncol = W - c - 1;
            if (nr > 0 && ncol > 0) {
                // flattened (row, column) walk with incremental indices: one division per thread and
                // pivot instead of a division and a remainder per updated entry
                const int dq = NT / ncol, dr = NT % ncol;
                int rr = tid / ncol, cc = tid % ncol;
                for (int t = tid; t < nr * ncol; t += NT) {
                    const int r = c + 1 + rr, col = c + 1 + cc;
                    M[(size_t)r * ld + col] -= (M[(size_t)r * ld + c] * inv) * M[(size_t)c * ld + col];
                    rr += dq;
                    cc += dr;
                    if (cc >= ncol) { cc -= ncol; ++rr; }
                }
            }
            __syncthreads();
        }
        if (s_fail) {
            if (tid == 0) { atomicOr(a.fail, 2u); atomicMin(a.bad, (unsigned long long)i); }
            continue;
        }
        const int nrhs = D + mn;
        for (int c = nn - 1; c >= 0 && !gj; --c) {
            for (int t = tid; t < nrhs; t += NT) M[(size_t)c * ld + nn + t] /= M[(size_t)c * ld + c];
            __syncthreads();
            {
                const int dq = NT / nrhs, dr = NT % nrhs;
                int r = tid / nrhs, k = tid % nrhs;
                for (int t = tid; t < c * nrhs; t += NT) {
                    M[(size_t)r * ld + nn + k] -= M[(size_t)r * ld + c] * M[(size_t)c * ld + nn + k];
                    r += dq;
                    k += dr;
                    if (k >= nrhs) { k -= nrhs; ++r; }
                }
            }
            __syncthreads();
        }
        // Schur complement S = c - b^T g (one warp)
        if (tid < 32) {
            double s = 0.0, sa = 0.0;
            for (int t = tid; t < nn * D; t += 32) {
                const double pr = bcol[t] * M[(size_t)(t / D) * ld + nn + (t % D)];
                s += pr;
                sa += fabs(pr);
            }
            s = warp_sum(s);
            sa = warp_sum(sa);
            if (tid == 0) {
                const double S = s_cpp - s;
                if (!(fabs(S) > 1e-14 * (sa + fabs(s_cpp)))) s_fail = 2;
                rn[0] = 1.0 / S;   // reuse rn[0] for 1/S
            }
        }
        __syncthreads();
        if (s_fail) {
            if (tid == 0) { atomicOr(a.fail, 2u); atomicMin(a.bad, (unsigned long long)i); }
            continue;
        }
        const double Sinv = rn[0];
        if (tid == 0) {   // algorithmic bytes: A_s^{-1} restricted rows (triangle in layout 4), g, weights, 1/S, indices
            const unsigned long long yb = a.layout == 4 ? (unsigned long long)mn * (mn + 1) / 2 + (unsigned long long)mn * (nn - mn)
                                                        : (unsigned long long)mn * nn;
            atomicAdd(a.alg, 8ull * (yb + (unsigned long long)nn * D + mn + 2) + 4ull * (nn + 1));
        }
        // Y[k][j] = (A_s^{-1})_{kj} = M[j][nn + D + k];  g[j][c] = M[j][nn + c]
        if (a.layout == 4) {
            const int64_t chunk = i >> 5;
            const int lane = (int)(i & 31);
            double* base = a.facT + chunk * a.pairs * 64;
            const int MT = a.MT;
            const int64_t tri = tri_col_start(MT, D);
            const int64_t tri_pad = tri + (tri & 1);
            // entries: column j < MT: Y[0..j][j], g[j][0..D-1]; column j >= MT: Y[0..MT-1][j], g[j][.]
            for (int t = tid; t < nn * (MT + D); t += NT) {
                const int j = t / (MT + D), q = t % (MT + D);
                int64_t e;
                double v;
                if (q < MT) {
                    const int k = q;
                    if (j < MT && k > j) continue;
                    v = k < mn ? M[(size_t)j * ld + nn + D + k] : 0.0;
                    e = j < MT ? tri_col_start(j, D) + k : tri_pad + (int64_t)(j - MT) * (MT + D) + k;
                } else {
                    const int c = q - MT;
                    v = M[(size_t)j * ld + nn + c];
                    e = j < MT ? tri_col_start(j, D) + (j + 1) + c : tri_pad + (int64_t)(j - MT) * (MT + D) + MT + c;
                }
                base[((e >> 1) * 32 + lane) * 2 + (e & 1)] = v;
            }
            for (int j = tid; j < a.NN; j += NT)
                a.ND[(chunk * a.NN + j) * 32 + lane] = j < nn ? ndof[j] : ndof[0];
            for (int k = tid; k < MT; k += NT)
                a.AUX[(chunk * (MT + 2) + k) * 32 + lane] = k < mn ? wnode[k] : 0.0;
            if (tid == 0) {
                a.AUX[(chunk * (MT + 2) + MT) * 32 + lane] = s_wp;
                a.AUX[(chunk * (MT + 2) + MT + 1) * 32 + lane] = Sinv;
                a.PD[chunk * 32 + lane] = pd;
                a.NR[chunk * 32 + lane] = mn;
            }
        } else {
            const int MT = a.MT;
            double* Y = a.fac + a.foffs[i];            // MT x nn, column-major (stride MT)
            double* g = Y + (size_t)MT * nn;           // nn * D
            double* aux = g + (size_t)nn * D;          // MT weights, w_p, 1/S
            for (int t = tid; t < nn * MT; t += NT) {
                const int j = t / MT, k = t % MT;
                Y[t] = k < mn ? M[(size_t)j * ld + nn + D + k] : 0.0;
            }
            for (int t = tid; t < nn * D; t += NT) g[t] = M[(size_t)(t / D) * ld + nn + (t % D)];
            for (int k = tid; k < MT; k += NT) aux[k] = k < mn ? wnode[k] : 0.0;
            for (int j = tid; j < nn; j += NT) a.nodes[a.nodeoffs[i] + j] = ndof[j];
            if (tid == 0) {
                aux[MT] = s_wp;
                aux[MT + 1] = Sinv;
                a.pdof[i] = pd;
                a.nres_nodes[i] = mn;
            }
        }
    }
}

// ------------------------------------------------------------------------------------
// sweeps
// ------------------------------------------------------------------------------------

// one patch per thread (2D): MT restricted nodes, D components, NN nodes per patch (runtime)
// DET: the corrections go to per-patch slots cbuf[i (MT D + 1) + k D + c] (pressure: slot MT D)
// instead of atomics; det_gather_kernel adds them to x in ascending patch order (rav_opts.deterministic)
// NDP: node indices from (nbase[i], pattern table ntbl[npid[i] * NN + j]) instead of the ND array
// RA: r is 16-byte aligned (checked at launch): node gathers without the per-load alignment test
// OB: the interface exchange fused into the sweep (Outbox, internal.cuh): ghost-written DoFs of
// flagged patches go to the consumers' receive buffers
// PA: warp-level pre-aggregation of the scatter (x-neighbouring patches share the nodes of one
// column of their restricted 3 x 3 blocks): a lane adds its right neighbour's contribution to a
// shared node to its own before the atomic, the neighbour skips that atomic.  The match is by node
// index on both lanes (the same predicate), so any patch shape is handled correctly; only the
// slot pairs tried ((2,0), (5,3), (8,6): R9's lexicographic order) assume the interior pattern.
template <int MT, int D, int NRB, bool DET, bool NDP, bool RA, bool OB, bool WTB = false, bool PA = false>
__device__ __forceinline__ void schur_thread_body(int64_t np, int64_t nchunks, int NN, int64_t pairs,
                                                                 const double2* __restrict__ W,
                                                                 const int32_t* __restrict__ ND,
                                                                 const int32_t* __restrict__ npid,
                                                                 const int32_t* __restrict__ nbase,
                                                                 const int32_t* __restrict__ ntbl,
                                                                 const int32_t* __restrict__ PD,
                                                                 const int32_t* __restrict__ NR,
                                                                 const double* __restrict__ AUX,
                                                                 const double* __restrict__ r,
                                                                 double* __restrict__ x, double omega,
                                                                 double* __restrict__ cbuf, int pf, ObView ob,
                                                                 const double* __restrict__ wtab = nullptr,
                                                                 const int32_t* __restrict__ ntab = nullptr,
                                                                 const double* __restrict__ SINV = nullptr) {
    static_assert(!WTB || NDP, "the weight table is indexed by the node pattern");
    constexpr int TRI = MT * (MT + 1) / 2 + MT * D;
    constexpr int TRI_PAD = TRI + (TRI & 1);
    constexpr int RC = MT + D;   // entries per rectangular column
    const int64_t gw = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;   // warp -> chunk
    const int64_t chunk = OB && ob.rot ? (gw < ob.rot ? gw + nchunks - ob.rot : gw - ob.rot) : gw;
    const int lane = threadIdx.x & 31;
    const int64_t i = chunk * 32 + lane;
    pdl_trigger();
    if (gw >= nchunks) return;
    const double2* wp = W + chunk * pairs * 32 + lane;
    const int32_t* np_ = NDP ? nullptr : ND + chunk * (int64_t)NN * 32 + lane;
    const int32_t pid_i = NDP ? npid[i] : 0;
    const int32_t* ntp = NDP ? ntbl + (int64_t)pid_i * NN : nullptr;   // L1-resident pattern row
    const int32_t nb0 = NDP ? nbase[i] : 0;
    const bool flagged = OB && i < np && ob.pflag[i];   // loaded early: needed only at the scatter
    // warp-uniform: the chunks without a ghost-writing patch (nearly all) keep the plain scatter
    const bool fw = OB && __any_sync(0xffffffffu, flagged);
#define ND_AT(j) (NDP ? nb0 + __ldg(ntp + (j)) : __ldcs(np_ + (j) * 32))
    {   // before r exists: the chunk's node indices and first factor lines into L2
        const char* wc = reinterpret_cast<const char*>(W + chunk * pairs * 32);
        if (!NDP) {
            const char* nc = reinterpret_cast<const char*>(ND + chunk * (int64_t)NN * 32);
            for (int ln = lane; ln < NN; ln += 32) prefetch_l2(nc + (size_t)ln * 128);
        }
        const int lines = (int)(pairs * 4 < 128 ? pairs * 4 : 128);
        for (int ln = lane; ln < lines; ln += 32) prefetch_l2(wc + (size_t)ln * 128);
        // NRB > 0: the first pf rectangular blocks by one bulk prefetch (the rest rolls inside the loop)
        if (NRB > 0 && pf > 0 && lane == 0)
            bulk_prefetch_l2(wc + (size_t)(TRI_PAD / 2) * 512, (uint32_t)(min(pf, NRB) * RC * 512));
    }
    pdl_wait();
    auto ldr = [&](const double* p, double* out) {
        if constexpr (RA && D == 2) {
            const double2 v = __ldg(reinterpret_cast<const double2*>(p));
            out[0] = v.x;
            out[D - 1] = v.y;
        } else {
            ld_node<D>(p, out);
        }
    };
    double acc[MT][D], rr[MT][D], gR[MT][D];
    double gacc = 0.0;
    const int pd = PD[i];
    const double rpd = __ldg(r + pd);   // the pressure residual with the patch's other gathers, not at the end
#pragma unroll
    for (int k = 0; k < MT; ++k) {
        const int nd = ND_AT(k);
        ldr(r + nd, rr[k]);
#pragma unroll
        for (int c = 0; c < D; ++c) acc[k][c] = 0.0;
    }
    double2 pv = make_double2(0.0, 0.0);
#pragma unroll
    for (int j = 0; j < MT; ++j) {
        constexpr int dummy = 0;
        (void)dummy;
#pragma unroll
        for (int q = 0; q <= j + D; ++q) {
            const int e = j * (j + 1) / 2 + j * D + q;
            if ((e & 1) == 0) pv = __ldcs(wp + (e >> 1) * 32);
            const double v = (e & 1) ? pv.y : pv.x;
            if (q <= j) {
                const int k = q;
#pragma unroll
                for (int c = 0; c < D; ++c) {
                    acc[k][c] = fma(v, rr[j][c], acc[k][c]);
                    if (k != j) acc[j][c] = fma(v, rr[k][c], acc[j][c]);
                }
            } else {
                const int c = q - j - 1;
                gR[j][c] = v;
                gacc = fma(v, rr[j][c], gacc);
            }
        }
    }
    // rectangular columns, two at a time (2 * RC entries = RC pairs)
    const double2* wq0 = wp + (TRI_PAD / 2) * 32;
    const int nrb = NRB > 0 ? NRB : (NN - MT) / 2;
#pragma unroll
    for (int b = 0; b < (NRB > 0 ? NRB : 1 << 20); ++b) {
        if (NRB == 0 && b >= nrb) break;
        const int j0 = MT + 2 * b;
        if (NRB > 0 && pf > 0 && lane == 0 && b + pf < NRB)   // rolling: block b + pf into L2
            bulk_prefetch_l2(W + chunk * pairs * 32 + (int64_t)(TRI_PAD / 2 + (b + pf) * RC) * 32, (uint32_t)(RC * 512));
        double ra[D], rb[D];
        const int n0 = ND_AT(j0), n1 = ND_AT(j0 + 1);
        ldr(r + n0, ra);
        ldr(r + n1, rb);
        const double2* wq = wq0 + (int64_t)((j0 - MT) / 2) * RC * 32;
#pragma unroll
        for (int p = 0; p < RC; ++p) {
            const double2 v2 = __ldcs(wq + p * 32);
#pragma unroll
            for (int h = 0; h < 2; ++h) {
                const int e = 2 * p + h;
                const double v = h ? v2.y : v2.x;
                const bool second = e >= RC;
                const int q = second ? e - RC : e;
                if (q < MT) {
#pragma unroll
                    for (int c = 0; c < D; ++c) acc[q][c] = fma(v, second ? rb[c] : ra[c], acc[q][c]);
                } else {
                    gacc = fma(v, second ? rb[q - MT] : ra[q - MT], gacc);
                }
            }
        }
    }
    // WTB: weights, w_p and the restricted count from the node pattern's row (L1), 1/S from SINV
    const double* aux = WTB ? nullptr : AUX + chunk * (MT + 2) * 32 + lane;
    const double* wt = WTB ? wtab + (int64_t)pid_i * (MT + 1) : nullptr;
    const double t = (WTB ? __ldcs(SINV + i) : aux[(MT + 1) * 32]) * (gacc - rpd);
    if constexpr (PA) {
        static_assert(MT == 9 && WTB && !DET && !OB, "pre-aggregated scatter: the 2D PoU table kernel");
        const bool live = i < np;   // the padding slots of the last chunk take part in the shuffles
        const int m = live ? __ldg(ntab + pid_i) : 0;
        int ndk[MT];
        double val[MT][D];
#pragma unroll
        for (int k = 0; k < MT; ++k) {
            ndk[k] = k < m ? ND_AT(k) : -1;
            const double wk = k < m ? omega * __ldg(wt + k) : 0.0;
#pragma unroll
            for (int c = 0; c < D; ++c) val[k][c] = wk * fma(gR[k][c], t, acc[k][c]);
        }
#pragma unroll
        for (int p = 0; p < 3; ++p) {
            const int kr = 3 * p + 2, kl = 3 * p;
            const int pn = __shfl_down_sync(0xffffffffu, ndk[kl], 1);
            const int on = __shfl_up_sync(0xffffffffu, ndk[kr], 1);
            const bool take = lane < 31 && ndk[kr] >= 0 && pn == ndk[kr];
#pragma unroll
            for (int c = 0; c < D; ++c) {
                const double pvc = __shfl_down_sync(0xffffffffu, val[kl][c], 1);
                if (take) val[kr][c] += pvc;
            }
            if (lane > 0 && ndk[kl] >= 0 && on == ndk[kl]) ndk[kl] = -1;   // the left neighbour adds it
        }
        if (!live) return;
#pragma unroll
        for (int k = 0; k < MT; ++k) {
            if (ndk[k] >= 0) {
#pragma unroll
                for (int c = 0; c < D; ++c) atomicAdd(x + ndk[k] + c, val[k][c]);
            }
        }
        const double wpr = __ldg(wt + MT);
        if (wpr != 0.0) atomicAdd(x + pd, omega * wpr * (-t));
        return;
    }
    if (i >= np) return;   // padding slots of the last chunk
    const int m = WTB ? __ldg(ntab + pid_i) : NR[i];
    double* cb = DET ? cbuf + i * (MT * D + 1) : nullptr;
    // the scatter (restricted prolongation, Eq. 13): one straight-line loop per target kind,
    // the warp-uniform branch outside it (a branch per store turned the reductions into returning
    // atomics under divergence management)
    auto scatter = [&](auto&& add) {
#pragma unroll
        for (int k = 0; k < MT; ++k) {
            if (k < m) {
                const double wk = omega * (WTB ? __ldg(wt + k) : aux[k * 32]);
                const int nd = ND_AT(k);
#pragma unroll
                for (int c = 0; c < D; ++c) add(nd + c, wk * fma(gR[k][c], t, acc[k][c]), k * D + c);
            }
        }
    };
    if constexpr (DET) {
        scatter([&](int, double v, int slot) { cb[slot] = v; });
    } else if constexpr (OB) {
        if (fw) {
            if (flagged) ob_wait_acks(ob);
            scatter([&](int dof, double v, int) { ob_add(ob, flagged, x, dof, v); });
        } else {
            scatter([&](int dof, double v, int) { red_add(x + dof, v); });
        }
    } else {
        scatter([&](int dof, double v, int) { atomicAdd(x + dof, v); });
    }
    const double wpr = WTB ? __ldg(wt + MT) : aux[MT * 32];
    if (wpr != 0.0) {
        if (DET) cb[MT * D] = omega * wpr * (-t);
        else if (OB) red_add(x + pd, omega * wpr * (-t));
        else atomicAdd(x + pd, omega * wpr * (-t));
    }
}

#undef ND_AT

template <int MT, int D, int NRB = 0, bool DET = false, bool NDP = false, bool RA = false, bool OB = false,
          bool WTB = false, bool PA = false>
__global__ void __launch_bounds__(128, 4) schur_sweep_thread_kernel(int64_t np, int64_t nchunks, int NN, int64_t pairs,
                                                                 const double2* __restrict__ W,
                                                                 const int32_t* __restrict__ ND,
                                                                 const int32_t* __restrict__ npid,
                                                                 const int32_t* __restrict__ nbase,
                                                                 const int32_t* __restrict__ ntbl,
                                                                 const int32_t* __restrict__ PD,
                                                                 const int32_t* __restrict__ NR,
                                                                 const double* __restrict__ AUX,
                                                                 const double* __restrict__ r,
                                                                 double* __restrict__ x, double omega,
                                                                 double* __restrict__ cbuf, int pf, Outbox ob,
                                                                 const double* __restrict__ wtab,
                                                                 const int32_t* __restrict__ ntab,
                                                                 const double* __restrict__ SINV) {
    schur_thread_body<MT, D, NRB, DET, NDP, RA, OB, WTB, PA>(np, nchunks, NN, pairs, W, ND, npid, nbase, ntbl, PD, NR, AUX,
                                                         r, x, omega, cbuf, pf, ob_view(ob), wtab, ntab, SINV);
    if constexpr (OB) {   // a writer: this warp's chunk holds a ghost-writing patch
        const int64_t gw = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
        const int64_t chunk = ob.rot ? (gw < ob.rot ? gw + nchunks - ob.rot : gw - ob.rot) : gw;
        const int64_t i = chunk * 32 + (threadIdx.x & 31);
        if (__any_sync(0xffffffffu, gw < nchunks && i < np && ob.pflag[i])) ob_writer_done(ob);
    }
}

// one patch per warp (3D and large patches): lane k owns restricted node k
// MTC > 0: compile-time number of restricted nodes (27 for the 3D PoU interior shape): the column
// loads then use immediate offsets from a running pointer instead of 64-bit index arithmetic
template <int D, bool DET = false, int WB = 8, int MTC = 0, bool OB = false>
__global__ void __launch_bounds__(256) schur_sweep_warp_kernel(int64_t np, int MT, int nnmax,
                                                               const int64_t* __restrict__ foffs,
                                                               const int64_t* __restrict__ nodeoffs,
                                                               const int32_t* __restrict__ nodes,
                                                               const int32_t* __restrict__ pdof,
                                                               const int32_t* __restrict__ nresn,
                                                               const double* __restrict__ fac,
                                                               const double* __restrict__ r, double* __restrict__ x,
                                                               double omega, double* __restrict__ cbuf, int wpf,
                                                               Outbox ob) {
    extern __shared__ double sm[];
    const ObView obv = ob_view(ob);
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    double* rl = sm + (size_t)warp * nnmax * D;
    for (int64_t i = (int64_t)blockIdx.x * 8 + warp; i < np; i += (int64_t)gridDim.x * 8) {
        if (lane == 0 && wpf > 0) {   // this patch's (and with wpf = 2 the next one's) factor block into L2
            const int64_t last = wpf > 1 ? min(i + (int64_t)gridDim.x * 8, np - 1) : i;
            for (int64_t k = i; k <= last; k += (int64_t)gridDim.x * 8) {
                const uintptr_t a0 = reinterpret_cast<uintptr_t>(fac + foffs[k]) & ~(uintptr_t)15;
                const uintptr_t a1 = (reinterpret_cast<uintptr_t>(fac + foffs[k + 1]) + 15) & ~(uintptr_t)15;
                bulk_prefetch_l2(reinterpret_cast<const void*>(a0), (uint32_t)(a1 - a0));
            }
        }
        const int64_t no = nodeoffs[i];
        const int nn = (int)(nodeoffs[i + 1] - no);
        if (lane == 0) {   // the operands of the chain's end (weights, 1/S, counts, pressure DoF) into L2 now
            prefetch_l2(fac + foffs[i] + (size_t)(MTC > 0 ? MTC : MT) * nn + (size_t)nn * D);
            prefetch_l2(pdof + i);
            prefetch_l2(nresn + i);
        }
        {   // gather r of the patch's nodes: lane takes nodes lane + 32u (independent index loads first)
            int nd[4];
#pragma unroll
            for (int u = 0; u < 4; ++u) nd[u] = lane + 32 * u < nn ? __ldg(nodes + no + lane + 32 * u) : -1;
#pragma unroll
            for (int u = 0; u < 4; ++u)
                if (nd[u] >= 0) {
#pragma unroll
                    for (int c = 0; c < D; ++c) rl[(lane + 32 * u) * D + c] = __ldg(r + nd[u] + c);
                }
            for (int j = lane + 128; j < nn; j += 32) {
                const int n1 = __ldg(nodes + no + j);
#pragma unroll
                for (int c = 0; c < D; ++c) rl[j * D + c] = __ldg(r + n1 + c);
            }
        }
        __syncwarp();
        const double* Y = fac + foffs[i];
        const double* g = Y + (size_t)MT * nn;
        const double* aux = g + (size_t)nn * D;
        double acc[D];
#pragma unroll
        for (int c = 0; c < D; ++c) acc[c] = 0.0;
        if constexpr (MTC > 0) {
            if (lane < MTC) {
                const double* yp = Y + lane;
                const double* rp = rl;
                int j = 0;
                for (; j + WB <= nn; j += WB, yp += WB * MTC, rp += WB * D) {
                    double y[WB];
#pragma unroll
                    for (int u = 0; u < WB; ++u) y[u] = __ldcs(yp + u * MTC);
#pragma unroll
                    for (int u = 0; u < WB; ++u)
#pragma unroll
                        for (int c = 0; c < D; ++c) acc[c] = fma(y[u], rp[u * D + c], acc[c]);
                }
                for (; j < nn; ++j, yp += MTC, rp += D) {
                    const double y = __ldcs(yp);
#pragma unroll
                    for (int c = 0; c < D; ++c) acc[c] = fma(y, rp[c], acc[c]);
                }
            }
        } else if (lane < MT) {
            // batches of WB independent column loads in flight per lane (the loop is latency-bound otherwise)
            int j = 0;
            for (; j + WB <= nn; j += WB) {
                double y[WB];
#pragma unroll
                for (int u = 0; u < WB; ++u) y[u] = __ldcs(Y + (size_t)(j + u) * MT + lane);
#pragma unroll
                for (int u = 0; u < WB; ++u)
#pragma unroll
                    for (int c = 0; c < D; ++c) acc[c] = fma(y[u], rl[(j + u) * D + c], acc[c]);
            }
            for (; j < nn; ++j) {
                const double y = __ldcs(Y + (size_t)j * MT + lane);
#pragma unroll
                for (int c = 0; c < D; ++c) acc[c] = fma(y, rl[j * D + c], acc[c]);
            }
        }
        double gs = 0.0;
        for (int t = lane; t < nn * D; t += 32) gs = fma(__ldcs(g + t), rl[t], gs);
        gs = warp_sum(gs);
        const double t = aux[MT + 1] * (gs - __ldg(r + pdof[i]));
        double* cb = DET ? cbuf + i * ((int64_t)MT * D + 1) : nullptr;
        if (lane < nresn[i]) {
            const double wk = omega * aux[lane];
            const int nd = nodes[no + lane];
            const bool flagged = OB && obv.pflag[i];
            if (OB && flagged) ob_wait_acks(obv);
#pragma unroll
            for (int c = 0; c < D; ++c) {
                const double v = wk * fma(g[lane * D + c], t, acc[c]);
                if (DET) cb[lane * D + c] = v;
                else if (OB) ob_add(obv, flagged, x, nd + c, v);
                else atomicAdd(x + nd + c, v);
            }
        }
        if (lane == 0) {
            if (DET) cb[MT * D] = omega * aux[MT] * (-t);
            else if (OB) red_add(x + pdof[i], omega * aux[MT] * (-t));
            else atomicAdd(x + pdof[i], omega * aux[MT] * (-t));
        }
        if constexpr (OB)   // a writer: this patch is ghost-writing (warp-uniform: one patch per warp)
            if (obv.pflag[i]) ob_writer_done(ob);
        __syncwarp();
    }
}

// coarse levels (few patches): one CTA of 8 warps per patch, warp w takes the columns j = w
// (mod 8) of A_s^{-1} and of g, the partial sums meet in shared memory -- 8x less serial latency
// per patch than schur_sweep_warp_kernel when the grid cannot fill the GPU anyway
template <int D, bool DET = false>
__global__ void __launch_bounds__(256) schur_sweep_cta_kernel(int64_t np, int MT, int nnmax,
                                                              const int64_t* __restrict__ foffs,
                                                              const int64_t* __restrict__ nodeoffs,
                                                              const int32_t* __restrict__ nodes,
                                                              const int32_t* __restrict__ pdof,
                                                              const int32_t* __restrict__ nresn,
                                                              const double* __restrict__ fac,
                                                              const double* __restrict__ r, double* __restrict__ x,
                                                              double omega, double* __restrict__ cbuf) {
    extern __shared__ double sm[];
    double* rl = sm;                                  // nnmax * D
    double* part = rl + (size_t)nnmax * D;            // 8 warps x 32 lanes x D
    __shared__ double gpart[8];
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    for (int64_t i = blockIdx.x; i < np; i += gridDim.x) {
        const int64_t no = nodeoffs[i];
        const int nn = (int)(nodeoffs[i + 1] - no);
        const double* Y = fac + foffs[i];
        const double* g = Y + (size_t)MT * nn;
        const double* aux = g + (size_t)nn * D;
        // warp 0's end-of-patch operands (1/S, the pressure residual, its weight, the restricted count,
        // node and g entries) issued with the gather instead of after the column loop and the barrier
        double e_sinv = 0.0, e_rp = 0.0, e_wl = 0.0, e_wp = 0.0, e_g[D];
        int e_nres = 0, e_nd = 0, e_pd = 0;
        if (warp == 0) {
            e_pd = pdof[i];
            e_nres = nresn[i];
            e_sinv = aux[MT + 1];
            e_wp = aux[MT];
            e_rp = __ldg(r + e_pd);
            if (lane < MT && lane < nn) {
                e_wl = aux[lane];
                e_nd = nodes[no + lane];
#pragma unroll
                for (int c = 0; c < D; ++c) e_g[c] = g[lane * D + c];
            }
        }
        for (int t = threadIdx.x; t < nn * D; t += blockDim.x) rl[t] = __ldg(r + nodes[no + t / D] + (t % D));
        __syncthreads();
        double acc[D];
#pragma unroll
        for (int c = 0; c < D; ++c) acc[c] = 0.0;
        if (lane < MT)
            for (int j = warp; j < nn; j += 8) {
                const double y = __ldcs(Y + (size_t)j * MT + lane);
#pragma unroll
                for (int c = 0; c < D; ++c) acc[c] = fma(y, rl[j * D + c], acc[c]);
            }
#pragma unroll
        for (int c = 0; c < D; ++c) part[(warp * 32 + lane) * D + c] = acc[c];
        double gs = 0.0;
        for (int t = threadIdx.x; t < nn * D; t += blockDim.x) gs = fma(__ldcs(g + t), rl[t], gs);
        gs = warp_sum(gs);
        if (lane == 0) gpart[warp] = gs;
        __syncthreads();
        if (warp == 0) {
            double gt = 0.0;
            for (int w = 0; w < 8; ++w) gt += gpart[w];
            const double t = e_sinv * (gt - e_rp);
            double* cb = DET ? cbuf + i * ((int64_t)MT * D + 1) : nullptr;
            if (lane < e_nres) {
                const double wk = omega * e_wl;
#pragma unroll
                for (int c = 0; c < D; ++c) {
                    double a = 0.0;
                    for (int w = 0; w < 8; ++w) a += part[(w * 32 + lane) * D + c];
                    const double v = wk * fma(e_g[c], t, a);
                    if (DET) cb[lane * D + c] = v;
                    else atomicAdd(x + e_nd + c, v);
                }
            }
            if (lane == 0) {
                if (DET) cb[MT * D] = omega * e_wp * (-t);
                else atomicAdd(x + e_pd, omega * e_wp * (-t));
            }
        }
        __syncthreads();
    }
}

// ------------------------------------------------------------------------------------
// host side
// ------------------------------------------------------------------------------------

static int pick_MT(int mnmax) {
    static const int cand[] = {1, 2, 4, 9, 16, 27, 32};
    for (int c : cand)
        if (c >= mnmax) return c;
    return -1;
}

// ---- node-index patterns of the thread layout (structured patches) ----------------------------
// slot i's node list ND[(chunk NN + j) 32 + lane] = base + pattern offsets; few distinct patterns
__device__ __forceinline__ uint64_t nd_fnv(uint64_t h, uint32_t v) {
    for (int k = 0; k < 4; ++k) { h ^= (v >> (8 * k)) & 0xffu; h *= 1099511628211ull; }
    return h;
}

__global__ void nd_hash_kernel(int64_t nslots, int NN, const int32_t* ND, uint64_t* key, int32_t* idx, int32_t* base) {
    for (int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; t < nslots; t += (int64_t)gridDim.x * blockDim.x) {
        const int64_t chunk = t >> 5;
        const int lane = (int)(t & 31);
        const int32_t* p = ND + chunk * (int64_t)NN * 32 + lane;
        const int32_t b0 = p[0];
        uint64_t h = 1469598103934665603ull;
        for (int j = 0; j < NN; ++j) h = nd_fnv(h, (uint32_t)(p[j * 32] - b0));
        key[t] = h;
        idx[t] = (int32_t)t;
        base[t] = b0;
    }
}

__global__ void nd_flag_kernel(int64_t n, const uint64_t* skey, int32_t* flag) {
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x)
        flag[i] = (i == 0 || skey[i] != skey[i - 1]) ? 1 : 0;
}

__global__ void nd_pid_kernel(int64_t n, const int32_t* sidx, const int32_t* flag, const int32_t* seg, int32_t* pid,
                              int32_t* rep) {
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
        pid[sidx[i]] = seg[i] - 1;
        if (flag[i]) rep[seg[i] - 1] = sidx[i];
    }
}

__global__ void nd_table_kernel(int npat, int NN, const int32_t* rep, const int32_t* ND, int32_t* tbl) {
    for (int p = blockIdx.x * blockDim.x + threadIdx.x; p < npat; p += gridDim.x * blockDim.x) {
        const int64_t t = rep[p];
        const int32_t* q = ND + (t >> 5) * (int64_t)NN * 32 + (t & 31);
        for (int j = 0; j < NN; ++j) tbl[(int64_t)p * NN + j] = q[j * 32] - q[0];
    }
}

__global__ void nd_verify_kernel(int64_t nslots, int NN, const int32_t* ND, const int32_t* pid, const int32_t* base,
                                 const int32_t* tbl, unsigned int* err) {
    for (int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; t < nslots; t += (int64_t)gridDim.x * blockDim.x) {
        const int32_t* q = ND + (t >> 5) * (int64_t)NN * 32 + (t & 31);
        for (int j = 0; j < NN; ++j)
            if (q[j * 32] != base[t] + tbl[(int64_t)pid[t] * NN + j]) atomicOr(err, 1u);
    }
}

// ---- per-pattern weight table of the thread layout (see Factors::wtab) -------------------------
__global__ void wt_rep_kernel(int64_t np, const int32_t* npid, int32_t* rep) {
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < np; i += (int64_t)gridDim.x * blockDim.x)
        atomicMin(rep + npid[i], (int32_t)i);
}
__global__ void wt_fill_kernel(int npat, int64_t np, int MT, const int32_t* rep, const double* AUX,
                               const int32_t* NR, double* wtab, int32_t* ntab) {
    for (int p = blockIdx.x * blockDim.x + threadIdx.x; p < npat; p += gridDim.x * blockDim.x) {
        const int i = rep[p];
        if (i >= np) {   // a pattern of padding slots only (rep kept its 0x7f7f7f7f fill)
            for (int k = 0; k <= MT; ++k) wtab[(int64_t)p * (MT + 1) + k] = 0.0;
            ntab[p] = 0;
            continue;
        }
        const int64_t chunk = i >> 5;
        const int lane = i & 31;
        for (int k = 0; k <= MT; ++k) wtab[(int64_t)p * (MT + 1) + k] = AUX[(chunk * (MT + 2) + k) * 32 + lane];
        ntab[p] = NR[i];
    }
}
// every slot against its pattern's row (padding slots i >= np: weights 0, count 0 -- the sweep
// returns before using them); SINV for all slots; Sum (NR + 1) of the real patches for the byte model
__global__ void wt_verify_kernel(int64_t ns, int64_t np, int MT, const int32_t* npid, const double* AUX,
                                 const int32_t* NR, const double* wtab, const int32_t* ntab, double* SINV,
                                 unsigned int* err, unsigned long long* cnt) {
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < ns; i += (int64_t)gridDim.x * blockDim.x) {
        const int64_t chunk = i >> 5;
        const int lane = (int)(i & 31);
        SINV[i] = AUX[(chunk * (MT + 2) + MT + 1) * 32 + lane];
        if (i >= np) continue;
        const int p = npid[i];
        if (ntab[p] != NR[i]) atomicOr(err, 1u);
        for (int k = 0; k <= MT; ++k)
            if (__double_as_longlong(wtab[(int64_t)p * (MT + 1) + k]) !=
                __double_as_longlong(AUX[(chunk * (MT + 2) + k) * 32 + lane]))
                atomicOr(err, 1u);
        atomicAdd(cnt, (unsigned long long)(NR[i] + 1));
    }
}

static rav_status schur_wt_compress(Factors& F, int64_t np, cudaStream_t s) {
    const int64_t ns = F.nchunks * 32;
    const int npat = F.nnpat, MT = F.MT;
    if (npat <= 0 || (int64_t)npat * (MT + 1) * 8 > (4 << 20)) return RAV_OK;
    int32_t* rep = nullptr;
    unsigned int* err = nullptr;
    unsigned long long* cnt = nullptr;
    double *wtab = nullptr, *sinv = nullptr;
    int32_t* ntab = nullptr;
    RAV_CUDA(cudaMallocAsync(&rep, sizeof(int32_t) * npat, s));
    RAV_CUDA(cudaMemsetAsync(rep, 0x7f, sizeof(int32_t) * npat, s));   // 0x7f7f7f7f: above any slot
    RAV_CUDA(cudaMallocAsync(&err, sizeof(unsigned int), s));
    RAV_CUDA(cudaMemsetAsync(err, 0, sizeof(unsigned int), s));
    RAV_CUDA(cudaMallocAsync(&cnt, sizeof(unsigned long long), s));
    RAV_CUDA(cudaMemsetAsync(cnt, 0, sizeof(unsigned long long), s));
    RAV_CUDA(cudaMalloc(&wtab, sizeof(double) * (size_t)npat * (MT + 1)));
    RAV_CUDA(cudaMalloc(&ntab, sizeof(int32_t) * npat));
    RAV_CUDA(cudaMalloc(&sinv, sizeof(double) * ns));
    const int nb = (int)std::max<int64_t>(1, std::min<int64_t>(cdiv(ns, 256), (int64_t)num_sms() * 16));
    wt_rep_kernel<<<nb, 256, 0, s>>>(np, F.npid, rep);
    count_launch();
    wt_fill_kernel<<<(int)cdiv(npat, 128), 128, 0, s>>>(npat, np, MT, rep, F.WT, F.NR, wtab, ntab);
    count_launch();
    wt_verify_kernel<<<nb, 256, 0, s>>>(ns, np, MT, F.npid, F.WT, F.NR, wtab, ntab, sinv, err, cnt);
    count_launch();
    RAV_CHECK_LAUNCH();
    unsigned int h_err = 0;
    unsigned long long h_cnt = 0;
    RAV_CUDA(cudaMemcpyAsync(&h_err, err, sizeof(h_err), cudaMemcpyDeviceToHost, s));
    RAV_CUDA(cudaMemcpyAsync(&h_cnt, cnt, sizeof(h_cnt), cudaMemcpyDeviceToHost, s));
    for (void* p : {(void*)rep, (void*)err, (void*)cnt}) cudaFreeAsync(p, s);
    RAV_CUDA(cudaStreamSynchronize(s));
    if (h_err) {
        for (void* p : {(void*)wtab, (void*)ntab, (void*)sinv}) cudaFree(p);
        return RAV_OK;
    }
    F.wtab = wtab;
    F.ntab = ntab;
    F.SINV = sinv;
    F.alg_bytes -= 8 * (int64_t)h_cnt;   // the streamed weights and w_p (1/S stays, now in SINV)
    return RAV_OK;
}

static rav_status schur_nd_compress(Factors& F, int64_t np, cudaStream_t s) {
    (void)np;
    const int64_t ns = F.nchunks * 32;
    const int NN = F.NN;
    uint64_t *key = nullptr, *skey = nullptr;
    int32_t *idx = nullptr, *sidx = nullptr, *flag = nullptr, *seg = nullptr, *rep = nullptr;
    int32_t *pid = nullptr, *base = nullptr, *tbl = nullptr;
    unsigned int* err = nullptr;
    RAV_CUDA(cudaMallocAsync(&key, sizeof(uint64_t) * ns, s));
    RAV_CUDA(cudaMallocAsync(&skey, sizeof(uint64_t) * ns, s));
    RAV_CUDA(cudaMallocAsync(&idx, sizeof(int32_t) * ns, s));
    RAV_CUDA(cudaMallocAsync(&sidx, sizeof(int32_t) * ns, s));
    RAV_CUDA(cudaMallocAsync(&flag, sizeof(int32_t) * ns, s));
    RAV_CUDA(cudaMallocAsync(&seg, sizeof(int32_t) * ns, s));
    RAV_CUDA(cudaMalloc(&pid, sizeof(int32_t) * ns));
    RAV_CUDA(cudaMalloc(&base, sizeof(int32_t) * ns));
    const int nb = (int)std::max<int64_t>(1, std::min<int64_t>(cdiv(ns, 256), (int64_t)num_sms() * 16));
    nd_hash_kernel<<<nb, 256, 0, s>>>(ns, NN, F.DT, key, idx, base);
    count_launch();
    RAV_CHECK_LAUNCH();
    size_t tmp = 0, tmp2 = 0;
    RAV_CUDA(cub::DeviceRadixSort::SortPairs(nullptr, tmp, key, skey, idx, sidx, (int)ns, 0, 64, s));
    RAV_CUDA(cub::DeviceScan::InclusiveSum(nullptr, tmp2, flag, seg, (int)ns, s));
    void* d_tmp = nullptr;
    RAV_CUDA(cudaMallocAsync(&d_tmp, std::max(tmp, tmp2) + 16, s));
    RAV_CUDA(cub::DeviceRadixSort::SortPairs(d_tmp, tmp, key, skey, idx, sidx, (int)ns, 0, 64, s));
    nd_flag_kernel<<<nb, 256, 0, s>>>(ns, skey, flag);
    count_launch();
    RAV_CUDA(cub::DeviceScan::InclusiveSum(d_tmp, tmp2, flag, seg, (int)ns, s));
    int32_t npat = 0;
    RAV_CUDA(cudaMemcpyAsync(&npat, seg + ns - 1, sizeof(int32_t), cudaMemcpyDeviceToHost, s));
    RAV_CUDA(cudaStreamSynchronize(s));
    bool ok = npat > 0 && (int64_t)npat * NN * 4 <= (4 << 20);
    if (ok) {
        RAV_CUDA(cudaMallocAsync(&rep, sizeof(int32_t) * npat, s));
        RAV_CUDA(cudaMalloc(&tbl, sizeof(int32_t) * (int64_t)npat * NN));
        RAV_CUDA(cudaMallocAsync(&err, sizeof(unsigned int), s));
        RAV_CUDA(cudaMemsetAsync(err, 0, sizeof(unsigned int), s));
        nd_pid_kernel<<<nb, 256, 0, s>>>(ns, sidx, flag, seg, pid, rep);
        count_launch();
        nd_table_kernel<<<(int)cdiv(npat, 128), 128, 0, s>>>(npat, NN, rep, F.DT, tbl);
        count_launch();
        nd_verify_kernel<<<nb, 256, 0, s>>>(ns, NN, F.DT, pid, base, tbl, err);
        count_launch();
        RAV_CHECK_LAUNCH();
        unsigned int h_err = 0;
        RAV_CUDA(cudaMemcpyAsync(&h_err, err, sizeof(h_err), cudaMemcpyDeviceToHost, s));
        RAV_CUDA(cudaStreamSynchronize(s));
        ok = h_err == 0;
    }
    for (void* p : {(void*)key, (void*)skey, (void*)idx, (void*)sidx, (void*)flag, (void*)seg, (void*)rep, (void*)err,
                    d_tmp})
        if (p) cudaFreeAsync(p, s);
    RAV_CUDA(cudaStreamSynchronize(s));
    if (!ok) {
        for (void* p : {(void*)pid, (void*)base, (void*)tbl})
            if (p) cudaFree(p);
        return RAV_OK;
    }
    F.npid = pid;
    F.nbase = base;
    F.ntbl = tbl;
    F.nnpat = npat;
    return RAV_OK;
}

rav_status schur_factorize(const Csr& A, const PatchSet& P, int64_t nvel, int D, int kernel_choice, int mode,
                           Factors& F, int64_t* bad_patch, bool* applicable, cudaStream_t s) {
    *applicable = false;
    if (D < 1 || D > 3 || nvel <= 0) return RAV_OK;
    // node bounds from the patch sizes (one pressure DoF per patch)
    const int nnmax = (P.nmax - 1) / D;
    const int mnmax = std::max(1, (P.nresmax - 1) / D);
    if (nnmax < 1 || nnmax > 200) return RAV_OK;
    const int MT = mode == 1 ? 1 : pick_MT(mnmax);
    if (MT < 0) return RAV_OK;
    if (mode == 2) kernel_choice = RAV_KERNEL_WARP;   // MV: per-patch layout (full rows)
    SchurArgs a{};
    a.rp = A.rp;
    a.ci = A.ci;
    a.val = A.val;
    a.np = P.n_patches;
    a.poffs = P.offs;
    a.pdofs = P.dofs;
    a.pw = P.w;
    a.nvel = nvel;
    a.D = D;
    a.nnmax = nnmax;
    a.mnmax = MT;
    a.ld = nnmax + D + MT;
    if ((a.ld & 15) == 0) a.ld += 1;
    a.MT = MT;
    if (mode == 1) a.mnmax = nnmax;   // diagonal Vanka: any number of weighted nodes
    // small levels (few patches: latency-bound) take the per-patch layout, whose CTA / warp kernels
    // spread one patch over many lanes; the thread-per-patch SoA layout needs many patches to fill the GPU
    static const int64_t small = [] {
        const char* e = getenv("RAV_SCHUR_SMALL");
        return e ? atoll(e) : 4096;
    }();
    const bool thread = mode == 0 && kernel_choice != RAV_KERNEL_WARP && D == 2 && MT <= 9 && nnmax <= 32 &&
                        (P.n_patches >= small || kernel_choice == RAV_KERNEL_SCHUR);
    F.nchunks = cdiv(P.n_patches, 32);
    F.mode = mode;
    if (mode == 1) {
        F.layout = 6;
        F.D = D;
        F.NN = nnmax;
        std::vector<int64_t> ho(P.n_patches + 1), fo(P.n_patches + 1), no(P.n_patches + 1);
        RAV_CUDA(cudaMemcpy(ho.data(), P.offs, sizeof(int64_t) * (P.n_patches + 1), cudaMemcpyDeviceToHost));
        fo[0] = 0;
        no[0] = 0;
        for (int64_t i = 0; i < P.n_patches; ++i) {
            const int64_t nn = (ho[i + 1] - ho[i] - 1) / D;
            fo[i + 1] = fo[i] + nn * (D + 2) + 2;
            no[i + 1] = no[i] + nn;
        }
        RAV_CUDA(cudaMalloc(&F.foffs, sizeof(int64_t) * (P.n_patches + 1)));
        RAV_CUDA(cudaMalloc(&F.nodeoffs, sizeof(int64_t) * (P.n_patches + 1)));
        RAV_CUDA(cudaMalloc(&F.fac, sizeof(double) * std::max<int64_t>(1, fo.back())));
        RAV_CUDA(cudaMalloc(&F.nodes, sizeof(int32_t) * std::max<int64_t>(1, no.back())));
        RAV_CUDA(cudaMalloc(&F.PD, sizeof(int32_t) * P.n_patches));
        RAV_CUDA(cudaMalloc(&F.NR, sizeof(int32_t) * P.n_patches));
        RAV_CUDA(cudaMemcpy(F.foffs, fo.data(), sizeof(int64_t) * (P.n_patches + 1), cudaMemcpyHostToDevice));
        RAV_CUDA(cudaMemcpy(F.nodeoffs, no.data(), sizeof(int64_t) * (P.n_patches + 1), cudaMemcpyHostToDevice));
        F.bytes = (int64_t)sizeof(double) * fo.back() + sizeof(int32_t) * no.back();
        F.lead = F.fac;
        F.lead_bytes = (int64_t)sizeof(double) * fo.back();
        a.layout = 6;
        a.foffs = F.foffs;
        a.fac = F.fac;
        a.nodes = F.nodes;
        a.nodeoffs = F.nodeoffs;
        a.pdof = F.PD;
        a.nres_nodes = F.NR;
    } else if (thread) {
        F.layout = 4;
        F.MT = MT;
        F.D = D;
        F.NN = std::max(MT, nnmax);
        if ((F.NN - MT) & 1) F.NN += 1;
        int64_t tri = (int64_t)MT * (MT + 1) / 2 + (int64_t)MT * D;
        tri += tri & 1;
        F.pairs = (tri + (int64_t)(F.NN - MT) * (MT + D)) / 2;
        size_t fb = sizeof(double) * 2 * F.pairs * 32 * F.nchunks;
        RAV_CUDA(cudaMalloc(&F.facT, fb));
        RAV_CUDA(cudaMalloc(&F.DT, sizeof(int32_t) * F.NN * 32 * F.nchunks));
        RAV_CUDA(cudaMalloc(&F.PD, sizeof(int32_t) * 32 * F.nchunks));
        RAV_CUDA(cudaMalloc(&F.NR, sizeof(int32_t) * 32 * F.nchunks));
        RAV_CUDA(cudaMalloc(&F.WT, sizeof(double) * (MT + 2) * 32 * F.nchunks));
        RAV_CUDA(cudaMemsetAsync(F.facT, 0, fb, s));
        RAV_CUDA(cudaMemsetAsync(F.DT, 0, sizeof(int32_t) * F.NN * 32 * F.nchunks, s));
        RAV_CUDA(cudaMemsetAsync(F.PD, 0, sizeof(int32_t) * 32 * F.nchunks, s));
        RAV_CUDA(cudaMemsetAsync(F.NR, 0, sizeof(int32_t) * 32 * F.nchunks, s));
        RAV_CUDA(cudaMemsetAsync(F.WT, 0, sizeof(double) * (MT + 2) * 32 * F.nchunks, s));
        F.bytes = (int64_t)fb;
        F.lead = F.facT;
        F.lead_bytes = (int64_t)fb;
        a.layout = 4;
        a.NN = F.NN;
        a.pairs = F.pairs;
        a.facT = F.facT;
        a.ND = F.DT;
        a.PD = F.PD;
        a.NR = F.NR;
        a.AUX = F.WT;
    } else {
        F.layout = 5;
        F.MT = MT;
        F.D = D;
        F.NN = nnmax;
        // per-patch sizes: nn_i = (n_i - 1) / D nodes -> MT*nn + nn*D + MT + 2 doubles
        std::vector<int64_t> ho(P.n_patches + 1), fo(P.n_patches + 1), no(P.n_patches + 1);
        RAV_CUDA(cudaMemcpy(ho.data(), P.offs, sizeof(int64_t) * (P.n_patches + 1), cudaMemcpyDeviceToHost));
        fo[0] = 0;
        no[0] = 0;
        for (int64_t i = 0; i < P.n_patches; ++i) {
            const int64_t nn = (ho[i + 1] - ho[i] - 1) / D;
            int64_t sz = (int64_t)MT * nn + nn * D + MT + 2;
            sz += sz & 1;
            fo[i + 1] = fo[i] + sz;
            no[i + 1] = no[i] + nn;
        }
        RAV_CUDA(cudaMalloc(&F.foffs, sizeof(int64_t) * (P.n_patches + 1)));
        RAV_CUDA(cudaMalloc(&F.nodeoffs, sizeof(int64_t) * (P.n_patches + 1)));
        RAV_CUDA(cudaMalloc(&F.fac, sizeof(double) * std::max<int64_t>(1, fo.back())));
        RAV_CUDA(cudaMalloc(&F.nodes, sizeof(int32_t) * std::max<int64_t>(1, no.back())));
        RAV_CUDA(cudaMalloc(&F.PD, sizeof(int32_t) * P.n_patches));
        RAV_CUDA(cudaMalloc(&F.NR, sizeof(int32_t) * P.n_patches));
        RAV_CUDA(cudaMemcpy(F.foffs, fo.data(), sizeof(int64_t) * (P.n_patches + 1), cudaMemcpyHostToDevice));
        RAV_CUDA(cudaMemcpy(F.nodeoffs, no.data(), sizeof(int64_t) * (P.n_patches + 1), cudaMemcpyHostToDevice));
        RAV_CUDA(cudaMemsetAsync(F.fac, 0, sizeof(double) * std::max<int64_t>(1, fo.back()), s));
        F.bytes = (int64_t)sizeof(double) * fo.back() + sizeof(int32_t) * no.back();
        F.lead = F.fac;
        F.lead_bytes = (int64_t)sizeof(double) * fo.back();
        a.layout = 5;
        a.foffs = F.foffs;
        a.fac = F.fac;
        a.nodes = F.nodes;
        a.nodeoffs = F.nodeoffs;
        a.pdof = F.PD;
        a.nres_nodes = F.NR;
    }
    unsigned int* fail = nullptr;
    unsigned long long* bad = nullptr;
    unsigned long long* alg = nullptr;
    RAV_CUDA(cudaMallocAsync(&fail, sizeof(unsigned int), s));
    RAV_CUDA(cudaMallocAsync(&bad, sizeof(unsigned long long), s));
    RAV_CUDA(cudaMallocAsync(&alg, sizeof(unsigned long long), s));
    RAV_CUDA(cudaMemsetAsync(fail, 0, sizeof(unsigned int), s));
    RAV_CUDA(cudaMemsetAsync(bad, 0xff, sizeof(unsigned long long), s));
    RAV_CUDA(cudaMemsetAsync(alg, 0, sizeof(unsigned long long), s));
    a.fail = fail;
    a.comp_verified = (A.nb.nslices > 0 && A.nb.D == D) ? 1 : 0;
    static const int gj = [] {   // 3D local solves by the tensor-core Gauss-Jordan (gj_dmma)
        const char* e = getenv("RAV_SCHUR_GJ");
        return e ? atoi(e) : 1;
    }();
    a.gj = gj;
    a.bad = bad;
    a.alg = alg;
    a.hbits = 4;
    while ((1 << a.hbits) < 2 * a.nnmax) ++a.hbits;
    const size_t shmem = sizeof(double) * ((size_t)a.nnmax * a.ld + a.nnmax + (size_t)a.nnmax * D + a.nnmax) +
                         sizeof(int32_t) * (a.nnmax + 2 * ((size_t)1 << a.hbits)) + 64;
    if (shmem > 220 * 1024) {
        factors_free(F);
        cudaFreeAsync(fail, s);
        cudaFreeAsync(bad, s);
        return RAV_OK;
    }
    if (shmem > 48 * 1024) {
        RAV_CUDA(cudaFuncSetAttribute(schur_factor_kernel<128>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)shmem));
        RAV_CUDA(cudaFuncSetAttribute(schur_factor_kernel<512>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)shmem));
    }
    const int per_sm = (int)std::max<size_t>(1, std::min<size_t>(16, (220 * 1024) / shmem));
    const int grid = (int)std::min<int64_t>(P.n_patches, (int64_t)num_sms() * per_sm);
    // one or two CTAs per SM (3D): 512 threads, measured c4 factor 260 -> see DESIGN; else 128
    if (per_sm <= 2) schur_factor_kernel<512><<<grid, 512, shmem, s>>>(a);
    else schur_factor_kernel<128><<<grid, 128, shmem, s>>>(a);
    count_launch();
    RAV_CHECK_LAUNCH();
    unsigned int h_fail = 0;
    unsigned long long h_bad = 0, h_alg = 0;
    RAV_CUDA(cudaMemcpyAsync(&h_fail, fail, sizeof(h_fail), cudaMemcpyDeviceToHost, s));
    RAV_CUDA(cudaMemcpyAsync(&h_bad, bad, sizeof(h_bad), cudaMemcpyDeviceToHost, s));
    RAV_CUDA(cudaMemcpyAsync(&h_alg, alg, sizeof(h_alg), cudaMemcpyDeviceToHost, s));
    cudaFreeAsync(fail, s);
    cudaFreeAsync(bad, s);
    cudaFreeAsync(alg, s);
    RAV_CUDA(cudaStreamSynchronize(s));
    F.alg_bytes = (int64_t)h_alg;
    if (h_fail & 1u) {   // structure does not hold: caller uses the generic formats
        factors_free(F);
        return RAV_OK;
    }
    *applicable = true;
    if (h_fail & 2u) {
        if (bad_patch) *bad_patch = (int64_t)h_bad;
        set_error("singular local system in patch %lld", (long long)h_bad);
        return RAV_ERR_SINGULAR_LOCAL;
    }
    if (bad_patch) *bad_patch = -1;
    // node-index patterns: measured with the bulk prefetch, c2 109.4 -> 106.3 us, c3 1477 -> 1445 us (on);
    // before the prefetch 113.3 -> 111.2 us at c2 and no change at c3
    static const bool ndc = [] {
        const char* e = getenv("RAV_SCHUR_NDC");
        return !(e && atoi(e) == 0);
    }();
    if (F.layout == 4 && mode == 0 && ndc) {
        RAV_TRY(schur_nd_compress(F, P.n_patches, s));
        if (F.npid) {   // streamed index bytes: pattern id + base + pressure DoF instead of nn + 1 indices
            const int64_t sum_nn = (P.entries - P.n_patches) / D;
            F.alg_bytes += -4 * (sum_nn + P.n_patches) + 12 * P.n_patches;
            static const bool wt = [] {
                const char* e = getenv("RAV_SCHUR_WTAB");
                return !(e && atoi(e) == 0);
            }();
            if (wt) RAV_TRY(schur_wt_compress(F, P.n_patches, s));
        }
    }
    return RAV_OK;
}

// ---- canonical rows export (parity tests): W[a][b] = w_a * (L_i^{-1})[a][b] ------------
struct SchurView {
    int layout, MT, D, NN;
    int64_t pairs;
    const double* facT;
    const int32_t* ND;
    const double* AUX;
    const int64_t* foffs;
    const double* fac;
    const int32_t* nodes;
    const int64_t* nodeoffs;
};

__device__ double sv_entry(const SchurView& v, int64_t i, int64_t e) {
    const int64_t chunk = i >> 5;
    const int lane = (int)(i & 31);
    return v.facT[((chunk * v.pairs + (e >> 1)) * 32 + lane) * 2 + (e & 1)];
}
__device__ double sv_Y(const SchurView& v, int64_t i, int nn, int k, int j) {   // (A_s^{-1})_{kj}, k restricted
    if (v.layout == 5) return v.fac[v.foffs[i] + (int64_t)j * v.MT + k];
    const int64_t tri = tri_col_start(v.MT, v.D), tri_pad = tri + (tri & 1);
    if (j < v.MT) {
        if (k <= j) return sv_entry(v, i, tri_col_start(j, v.D) + k);
        return sv_entry(v, i, tri_col_start(k, v.D) + j);
    }
    return sv_entry(v, i, tri_pad + (int64_t)(j - v.MT) * (v.MT + v.D) + k);
}
__device__ double sv_g(const SchurView& v, int64_t i, int nn, int j, int c) {
    if (v.layout == 5) return v.fac[v.foffs[i] + (int64_t)v.MT * nn + (int64_t)j * v.D + c];
    const int64_t tri = tri_col_start(v.MT, v.D), tri_pad = tri + (tri & 1);
    if (j < v.MT) return sv_entry(v, i, tri_col_start(j, v.D) + j + 1 + c);
    return sv_entry(v, i, tri_pad + (int64_t)(j - v.MT) * (v.MT + v.D) + v.MT + c);
}
__device__ double sv_aux(const SchurView& v, int64_t i, int nn, int q) {   // q < MT: w_k; MT: w_p; MT+1: 1/S
    if (v.layout == 5) return v.fac[v.foffs[i] + (int64_t)v.MT * nn + (int64_t)nn * v.D + q];
    const int64_t chunk = i >> 5;
    return v.AUX[(chunk * (v.MT + 2) + q) * 32 + (i & 31)];
}

__global__ void export_schur_kernel(int64_t np, const int64_t* offs, const int32_t* dofs, const double* w,
                                    const int64_t* roffs, int64_t nvel, SchurView v, double* rows) {
    for (int64_t i = blockIdx.x; i < np; i += gridDim.x) {
        const int64_t off = offs[i];
        const int n = (int)(offs[i + 1] - off);
        const int D = v.D;
        const int nn = (n - 1) / D;
        int m = 0;
        for (int t = 0; t < n; ++t) m += w[off + t] > 0.0;
        const double Sinv = sv_aux(v, i, nn, v.MT + 1);
        // local DoF -> node index: restricted nodes first in patch order; node j of DoF = rank among nodes
        for (int t = threadIdx.x; t < m * n; t += blockDim.x) {
            const int ra = t / n, cb = t % n;
            const int da = dofs[off + ra], db = dofs[off + cb];
            // node index of a velocity DoF: count distinct nodes before it in patch order
            auto node_of = [&](int idx) {
                int cnt = 0, prev = -1;
                for (int u = 0; u <= idx; ++u) {
                    const int du = dofs[off + u];
                    if (du >= nvel) continue;
                    const int nd = du / D;
                    if (nd != prev) { ++cnt; prev = nd; }
                }
                return cnt - 1;
            };
            double val;
            if (da < nvel) {
                const int k = node_of(ra), ca = da % D;
                const double wk = w[off + ra];
                if (db < nvel) {
                    const int j = node_of(cb), cc = db % D;
                    val = (ca == cc ? sv_Y(v, i, nn, k, j) : 0.0) + sv_g(v, i, nn, k, ca) * Sinv * sv_g(v, i, nn, j, cc);
                } else {
                    val = -sv_g(v, i, nn, k, ca) * Sinv;
                }
                val *= wk;
            } else {
                const double wp = w[off + ra];
                if (db < nvel) val = -Sinv * sv_g(v, i, nn, node_of(cb), db % D);
                else val = Sinv;
                val *= wp;
            }
            rows[roffs[i] + t] = val;
        }
    }
}

__global__ void rows_size_kernel(int64_t np, const int64_t* offs, const int32_t* nres, int64_t* sz);

rav_status export_schur_rows(const PatchSet& P, const Factors& F, int64_t nvel, double* rows, cudaStream_t s) {
    int64_t *sz = nullptr, *roffs = nullptr;
    RAV_CUDA(cudaMallocAsync(&sz, sizeof(int64_t) * P.n_patches, s));
    RAV_CUDA(cudaMallocAsync(&roffs, sizeof(int64_t) * (P.n_patches + 1), s));
    const int nb = (int)std::min<int64_t>(cdiv(P.n_patches, 256), (int64_t)num_sms() * 16);
    rows_size_kernel<<<nb, 256, 0, s>>>(P.n_patches, P.offs, P.nres, sz);
    count_launch();
    RAV_TRY(gen::counts_to_rowptr(sz, roffs, P.n_patches, s));
    SchurView v{F.layout, F.MT, F.D, F.NN, F.pairs, F.facT, F.DT, F.WT, F.foffs, F.fac, F.nodes, F.nodeoffs};
    const int g = (int)std::min<int64_t>(P.n_patches, (int64_t)num_sms() * 8);
    export_schur_kernel<<<g, 128, 0, s>>>(P.n_patches, P.offs, P.dofs, P.w, roffs, nvel, v, rows);
    count_launch();
    RAV_CHECK_LAUNCH();
    cudaFreeAsync(sz, s);
    cudaFreeAsync(roffs, s);
    RAV_CUDA(cudaStreamSynchronize(s));
    return RAV_OK;
}

// ---- diagonal Vanka sweep (R17, layout 6): one warp per patch, lanes over nodes ------------
//   t = S^{-1} (g^T r_u - r_p),  du_j = r_j / a_jj + g_j t  (weights w_j),  dp = -t
template <int D>
__global__ void __launch_bounds__(256) diag_sweep_kernel(int64_t np, const int64_t* __restrict__ foffs,
                                                         const int64_t* __restrict__ nodeoffs,
                                                         const int32_t* __restrict__ nodes,
                                                         const int32_t* __restrict__ pdof,
                                                         const double* __restrict__ fac,
                                                         const double* __restrict__ r, double* __restrict__ x,
                                                         double omega) {
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    for (int64_t i = (int64_t)blockIdx.x * 8 + warp; i < np; i += (int64_t)gridDim.x * 8) {
        const int64_t no = nodeoffs[i];
        const int nn = (int)(nodeoffs[i + 1] - no);
        const double* dinv = fac + foffs[i];
        const double* g = dinv + nn;
        const double* aux = g + (size_t)nn * D;
        double gs = 0.0;
        for (int t = lane; t < nn * D; t += 32) gs = fma(__ldcs(g + t), __ldg(r + nodes[no + t / D] + t % D), gs);
        gs = warp_sum(gs);
        const int pd = pdof[i];
        const double t = aux[nn + 1] * (gs - __ldg(r + pd));
        for (int j = lane; j < nn; j += 32) {
            const double wj = aux[j];
            if (wj == 0.0) continue;
            const int nd = nodes[no + j];
            const double dj = __ldcs(dinv + j);
#pragma unroll
            for (int c = 0; c < D; ++c)
                atomicAdd(x + nd + c, omega * wj * fma(g[j * D + c], t, dj * __ldg(r + nd + c)));
        }
        if (lane == 0 && aux[nn] != 0.0) atomicAdd(x + pd, omega * aux[nn] * (-t));
    }
}

// the same with GL lanes per patch (32 / GL patches per warp): short patches keep all lanes busy
template <int D, int GL>
__global__ void __launch_bounds__(256) diag_sweep_group_kernel(int64_t np, const int64_t* __restrict__ foffs,
                                                               const int64_t* __restrict__ nodeoffs,
                                                               const int32_t* __restrict__ nodes,
                                                               const int32_t* __restrict__ pdof,
                                                               const double* __restrict__ fac,
                                                               const double* __restrict__ r, double* __restrict__ x,
                                                               double omega) {
    const int64_t gid = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) / GL;
    const int q = threadIdx.x % GL;
    const int64_t ngroups = (int64_t)gridDim.x * blockDim.x / GL;
    // warp-uniform trip count: every lane reaches the group shuffles
    for (int64_t base = gid - (threadIdx.x % 32) / GL; base < np; base += ngroups) {
        const int64_t i = base + (threadIdx.x % 32) / GL;
        const bool live = i < np;
        int64_t no = 0;
        int nn = 0;
        const double *dinv = fac, *g = fac, *aux = fac;
        if (live) {
            no = nodeoffs[i];
            nn = (int)(nodeoffs[i + 1] - no);
            dinv = fac + foffs[i];
            g = dinv + nn;
            aux = g + (size_t)nn * D;
        }
        double gs = 0.0;
        for (int t = q; t < nn * D; t += GL) gs = fma(__ldcs(g + t), __ldg(r + nodes[no + t / D] + t % D), gs);
        gs = group_sum<GL>(gs);
        if (!live) continue;
        const int pd = pdof[i];
        const double t = aux[nn + 1] * (gs - __ldg(r + pd));
        for (int j = q; j < nn; j += GL) {
            const double wj = aux[j];
            if (wj == 0.0) continue;
            const int nd = nodes[no + j];
            const double dj = __ldcs(dinv + j);
            double rv[D];
            ld_node<D>(r + nd, rv);
#pragma unroll
            for (int c = 0; c < D; ++c) atomicAdd(x + nd + c, omega * wj * fma(g[j * D + c], t, dj * rv[c]));
        }
        if (q == 0 && aux[nn] != 0.0) atomicAdd(x + pd, omega * aux[nn] * (-t));
    }
}

// ---- multicoloured multiplicative Vanka (Eq. 11, R10): one colour per launch --------
// Patches of one colour share no DoF and are not coupled through L, so they are
// relaxed concurrently; each computes a fresh local residual on its own rows
// (Eq. 15) and applies the full L_i^{-1} (Schur form, all nodes) with
// prolongation R_i^T.  Result = sequential MV in colour order.
// RR: the colour's fresh residual r = b - L x was computed by the residual kernel just before (the
// patches of one colour share no DoF and are not coupled through L, so it is each patch's fresh
// local residual of Eq. 15); the kernel gathers it instead of re-reading the patch rows of L
template <int D, bool RR = false>
__global__ void __launch_bounds__(256) mv_color_kernel(int64_t ncol, const int32_t* __restrict__ plist, int MT,
                                                       int nnmax, const int64_t* __restrict__ foffs,
                                                       const int64_t* __restrict__ nodeoffs,
                                                       const int32_t* __restrict__ nodes,
                                                       const int32_t* __restrict__ pdof,
                                                       const double* __restrict__ fac,
                                                       const int64_t* __restrict__ rp, const int32_t* __restrict__ ci,
                                                       const double* __restrict__ val,
                                                       const double* __restrict__ b, double* __restrict__ x,
                                                       double omega) {
    extern __shared__ double sm[];
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    double* rl = sm + (size_t)warp * (nnmax * D + 1);
    for (int64_t q = (int64_t)blockIdx.x * 8 + warp; q < ncol; q += (int64_t)gridDim.x * 8) {
        const int64_t i = plist[q];
        const int64_t no = nodeoffs[i];
        const int nn = (int)(nodeoffs[i + 1] - no);
        const int pd = pdof[i];
        if constexpr (RR) {
            for (int t = lane; t <= nn * D; t += 32) rl[t] = __ldg(b + (t < nn * D ? nodes[no + t / D] + t % D : pd));
        } else
        // fresh local residual on the patch rows (Eq. 15): 4 lanes per row, 8 rows per pass
        for (int t0 = 0; t0 <= nn * D; t0 += 8) {
            const int t = t0 + (lane >> 2), q = lane & 3;
            double s = 0.0;
            int row = 0;
            if (t <= nn * D) {
                row = t < nn * D ? nodes[no + t / D] + t % D : pd;
                for (int64_t k = rp[row] + q; k < rp[row + 1]; k += 4) s = fma(val[k], x[ci[k]], s);
            }
            s = group_sum<4>(s);
            if (q == 0 && t <= nn * D) rl[t] = b[row] - s;
        }
        __syncwarp();
        const double* Y = fac + foffs[i];
        const double* g = Y + (size_t)MT * nn;
        const double* aux = g + (size_t)nn * D;
        double gs = 0.0;
        for (int t = lane; t < nn * D; t += 32) gs = fma(g[t], rl[t], gs);
        gs = warp_sum(gs);
        const double tt = aux[MT + 1] * (gs - rl[nn * D]);
        for (int k0 = 0; k0 < nn; k0 += 32) {
            const int k = k0 + lane;
            double acc[D];
#pragma unroll
            for (int c = 0; c < D; ++c) acc[c] = 0.0;
            if (k < nn)
                for (int j = 0; j < nn; ++j) {
                    const double y = Y[(size_t)j * MT + k];
#pragma unroll
                    for (int c = 0; c < D; ++c) acc[c] = fma(y, rl[j * D + c], acc[c]);
                }
            __syncwarp();
            if (k < nn) {
                const int nd = nodes[no + k];
#pragma unroll
                for (int c = 0; c < D; ++c) x[nd + c] += omega * fma(g[k * D + c], tt, acc[c]);
            }
        }
        if (lane == 0) x[pd] += omega * (-tt);
        __syncwarp();
    }
}

rav_status launch_diag_sweep(const PatchSet& P, const Factors& F, const double* r, double* x, double omega,
                             cudaStream_t s) {
    const int blocks = (int)std::min<int64_t>(cdiv(P.n_patches, 8), (int64_t)num_sms() * 16);
    if (F.D == 3)
        diag_sweep_kernel<3><<<blocks, 256, 0, s>>>(P.n_patches, F.foffs, F.nodeoffs, F.nodes, F.PD, F.fac, r, x, omega);
    else if (F.D == 2 && F.NN <= 32) {   // 2D: 8 lanes per patch (measured in bench c5)
        const int gb = (int)std::max<int64_t>(1, cdiv(P.n_patches * 8, 256));
        diag_sweep_group_kernel<2, 8><<<gb, 256, 0, s>>>(P.n_patches, F.foffs, F.nodeoffs, F.nodes, F.PD, F.fac, r, x,
                                                         omega);
    } else if (F.D == 2)
        diag_sweep_kernel<2><<<blocks, 256, 0, s>>>(P.n_patches, F.foffs, F.nodeoffs, F.nodes, F.PD, F.fac, r, x, omega);
    else
        diag_sweep_kernel<1><<<blocks, 256, 0, s>>>(P.n_patches, F.foffs, F.nodeoffs, F.nodes, F.PD, F.fac, r, x, omega);
    count_launch();
    RAV_CHECK_LAUNCH();
    return RAV_OK;
}

rav_status launch_mv_color_r(const Factors& F, int64_t ncol, const int32_t* plist, const double* r, double* x,
                             double omega, cudaStream_t s) {
    if (ncol <= 0) return RAV_OK;
    const size_t shmem = sizeof(double) * (size_t)(F.NN * F.D + 1) * 8;
    const int blocks = (int)std::min<int64_t>(cdiv(ncol, 8), (int64_t)num_sms() * 16);
    if (F.D == 3)
        mv_color_kernel<3, true><<<blocks, 256, shmem, s>>>(ncol, plist, F.MT, F.NN, F.foffs, F.nodeoffs, F.nodes, F.PD,
                                                            F.fac, nullptr, nullptr, nullptr, r, x, omega);
    else if (F.D == 2)
        mv_color_kernel<2, true><<<blocks, 256, shmem, s>>>(ncol, plist, F.MT, F.NN, F.foffs, F.nodeoffs, F.nodes, F.PD,
                                                            F.fac, nullptr, nullptr, nullptr, r, x, omega);
    else
        mv_color_kernel<1, true><<<blocks, 256, shmem, s>>>(ncol, plist, F.MT, F.NN, F.foffs, F.nodeoffs, F.nodes, F.PD,
                                                            F.fac, nullptr, nullptr, nullptr, r, x, omega);
    count_launch();
    RAV_CHECK_LAUNCH();
    return RAV_OK;
}

rav_status launch_mv_color(const Csr& A, const Factors& F, int64_t ncol, const int32_t* plist, const double* b,
                           double* x, double omega, cudaStream_t s) {
    if (ncol <= 0) return RAV_OK;
    const size_t shmem = sizeof(double) * (size_t)(F.NN * F.D + 1) * 8;
    const int blocks = (int)std::min<int64_t>(cdiv(ncol, 8), (int64_t)num_sms() * 16);
    if (F.D == 3)
        mv_color_kernel<3><<<blocks, 256, shmem, s>>>(ncol, plist, F.MT, F.NN, F.foffs, F.nodeoffs, F.nodes, F.PD, F.fac,
                                                      A.rp, A.ci, A.val, b, x, omega);
    else if (F.D == 2)
        mv_color_kernel<2><<<blocks, 256, shmem, s>>>(ncol, plist, F.MT, F.NN, F.foffs, F.nodeoffs, F.nodes, F.PD, F.fac,
                                                      A.rp, A.ci, A.val, b, x, omega);
    else
        mv_color_kernel<1><<<blocks, 256, shmem, s>>>(ncol, plist, F.MT, F.NN, F.foffs, F.nodeoffs, F.nodes, F.PD, F.fac,
                                                      A.rp, A.ci, A.val, b, x, omega);
    count_launch();
    RAV_CHECK_LAUNCH();
    return RAV_OK;
}

template <int MT, bool DET, bool OB = false>
static void launch_schur_thread(int64_t np, const Factors& F, const double* r, double* x, double omega,
                                cudaStream_t s, const Outbox& ob = Outbox{}) {
    const double2* W = reinterpret_cast<const double2*>(F.facT);
    // 2D PoU interior shape (25 nodes, 9 restricted): compile-time rectangular loop (122 -> 113 us at c2)
    const bool shape = MT == 9 && F.NN == 25;
    const bool ra = (reinterpret_cast<uintptr_t>(r) & 15) == 0;
    auto kern = F.npid ? (shape ? (ra ? (F.wtab ? schur_sweep_thread_kernel<MT, 2, 8, DET, true, true, OB, true>
                                               : schur_sweep_thread_kernel<MT, 2, 8, DET, true, true, OB>)
                                      : schur_sweep_thread_kernel<MT, 2, 8, DET, true, false, OB>)
                                : schur_sweep_thread_kernel<MT, 2, 0, DET, true, false, OB>)
                       : shape ? schur_sweep_thread_kernel<MT, 2, 8, DET, false, false, OB>
                               : schur_sweep_thread_kernel<MT, 2, 0, DET, false, false, OB>;
    // the pre-aggregated scatter (PA) for the 2D PoU table kernel; RAV_SCHUR_PA=0: off.  Measured (B200,
    // profiles/r02pa_*): sweep alone c2 96.5 -> 95.2 us, c3 1358 -> 1337 us; c2 step 16.01 -> 15.70 ms
    static const int pa = [] {
        const char* e = getenv("RAV_SCHUR_PA");
        return e ? atoi(e) : 1;
    }();
    if constexpr (MT == 9 && !DET && !OB) {
        if (pa && F.npid && shape && ra && F.wtab) kern = schur_sweep_thread_kernel<9, 2, 8, false, true, true, false, true, true>;
    }
    // rectangular blocks prefetched ahead by the bulk-copy unit (0: off).  Measured (rav_apply alone):
    // c2 115.0 / 109.7 / 108.9 / 110.3 / 117.0 us for 0 / 1 / 2 / 3 / 5; c3 1606 -> 1474 us at 2.  Re-tuned with
    // the weight table and the pre-aggregated scatter (profiles/r02k_*): c2 101.9 / 92.5 / 95.2 / 96.0 us for
    // 0 / 1 / 2 / 3, c3 1470 / 1336 / 1338 us for 0 / 1 / 2: one block ahead is the default
    static const int pf = [] {
        const char* e = getenv("RAV_SCHUR_PF");
        return e ? atoi(e) : 1;
    }();
    // threads per block (a chunk per warp; the register budget gives 16 warps per SM at any of these).
    // One-warp blocks let an SM take the next chunk as soon as one warp retires instead of when four
    // have: c2 sweep 92.9 / 91.3 / 91.15 us at 128 / 64 / 32 (profiles/r02n_bs_sweep.txt), c3 equal
    static const int bs = [] {
        const char* e = getenv("RAV_SCHUR_BS");
        const int v = e ? atoi(e) : 32;
        return v == 128 || v == 64 ? v : 32;
    }();
    launch_maybe_pdl(kern, dim3((unsigned)cdiv(F.nchunks * 32, bs)), dim3(bs), 0, s, np, F.nchunks, F.NN, F.pairs, W,
                     (const int32_t*)F.DT, (const int32_t*)F.npid, (const int32_t*)F.nbase, (const int32_t*)F.ntbl,
                     (const int32_t*)F.PD, (const int32_t*)F.NR, (const double*)F.WT, r, x, omega, F.cbuf, pf, ob,
                     (const double*)F.wtab, (const int32_t*)F.ntab, (const double*)F.SINV);
}

static int64_t schur_cta_max() {   // patch count below which a CTA (8 warps) takes one patch
    static const int64_t cta_max = [] {
        const char* e = getenv("RAV_SCHUR_CTA_MAX");
        return e ? atoll(e) : 2048;
    }();
    return cta_max;
}

template <int D, bool DET, bool OB = false>
static void launch_schur_perpatch(const PatchSet& P, const Factors& F, const double* r, double* x, double omega,
                                  cudaStream_t s, const Outbox& ob = Outbox{}) {
    const int64_t cta_max = schur_cta_max();
    if (!OB && P.n_patches < cta_max && F.MT <= 32) {   // coarse levels: a CTA per patch (latency)
        const size_t shmem = sizeof(double) * ((size_t)F.NN * D + 8 * 32 * (size_t)D);
        schur_sweep_cta_kernel<D, DET><<<(int)std::max<int64_t>(1, P.n_patches), 256, shmem, s>>>(
            P.n_patches, F.MT, F.NN, F.foffs, F.nodeoffs, F.nodes, F.PD, F.NR, F.fac, r, x, omega, F.cbuf);
    } else {
        const size_t shmem = sizeof(double) * (size_t)F.NN * D * 8;
        // grid cap in blocks per SM.  c4 (WB 8): 218 us at 8 (one persistent wave), 189 at 16, 185 at 32
        // (one patch per warp); WB 16 / 24 within 2%
        static const int bps = [] {
            const char* e = getenv("RAV_SCHUR_WBPS");
            return e ? atoi(e) : 32;
        }();
        const int blocks = (int)std::min<int64_t>(cdiv(P.n_patches, 8), (int64_t)num_sms() * bps);
        static const int wpf = [] {   // per-patch bulk prefetch (c4, batched loads: 188.4 us off, 194.9 on)
            const char* e = getenv("RAV_SCHUR_WPF");
            return e ? atoi(e) : 0;
        }();
        static const int wb = [] {    // column loads in flight per lane
            const char* e = getenv("RAV_SCHUR_WB");
            return e ? atoi(e) : 8;
        }();
        static const int mtc = [] {   // compile-time restricted-node count for the 3D PoU shape
            const char* e = getenv("RAV_SCHUR_MTC");
            return e ? atoi(e) : 1;
        }();
        auto kern = (mtc && D == 3 && F.MT == 27) ? (wb >= 16 ? schur_sweep_warp_kernel<D, DET, 16, 27, OB>
                                                              : schur_sweep_warp_kernel<D, DET, 8, 27, OB>)
                  : wb >= 24 ? schur_sweep_warp_kernel<D, DET, 24, 0, OB>
                  : wb >= 16 ? schur_sweep_warp_kernel<D, DET, 16, 0, OB> : schur_sweep_warp_kernel<D, DET, 8, 0, OB>;
        kern<<<blocks, 256, shmem, s>>>(P.n_patches, F.MT, F.NN, F.foffs, F.nodeoffs, F.nodes, F.PD, F.NR, F.fac, r, x,
                                        omega, F.cbuf, wpf, ob);
    }
}

// deterministic mode, phase 2: x[dof_u] += (sum of its slots in ascending patch order)
__global__ void det_gather_kernel(int64_t nu, const int32_t* __restrict__ dof, const int64_t* __restrict__ off,
                                  const int32_t* __restrict__ slot, const double* __restrict__ cbuf,
                                  double* __restrict__ x) {
    for (int64_t u = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; u < nu; u += (int64_t)gridDim.x * blockDim.x) {
        double t = 0.0;
        for (int64_t e = off[u]; e < off[u + 1]; ++e) t += cbuf[slot[e]];
        x[dof[u]] += t;
    }
}

rav_status launch_schur_sweep(const PatchSet& P, const Factors& F, const double* r, double* x, double omega,
                              cudaStream_t s) {
    const bool det = F.cbuf != nullptr;
    if (F.layout == 4) {
        switch (F.MT * 2 + (det ? 1 : 0)) {
            case 2: launch_schur_thread<1, false>(P.n_patches, F, r, x, omega, s); break;
            case 3: launch_schur_thread<1, true>(P.n_patches, F, r, x, omega, s); break;
            case 4: launch_schur_thread<2, false>(P.n_patches, F, r, x, omega, s); break;
            case 5: launch_schur_thread<2, true>(P.n_patches, F, r, x, omega, s); break;
            case 8: launch_schur_thread<4, false>(P.n_patches, F, r, x, omega, s); break;
            case 9: launch_schur_thread<4, true>(P.n_patches, F, r, x, omega, s); break;
            case 18: launch_schur_thread<9, false>(P.n_patches, F, r, x, omega, s); break;
            case 19: launch_schur_thread<9, true>(P.n_patches, F, r, x, omega, s); break;
            default: set_error("schur thread kernel: unsupported MT %d", F.MT); return RAV_ERR_ARG;
        }
    } else if (F.D == 3) {
        if (det) launch_schur_perpatch<3, true>(P, F, r, x, omega, s);
        else launch_schur_perpatch<3, false>(P, F, r, x, omega, s);
    } else if (F.D == 2) {
        if (det) launch_schur_perpatch<2, true>(P, F, r, x, omega, s);
        else launch_schur_perpatch<2, false>(P, F, r, x, omega, s);
    } else {
        if (det) launch_schur_perpatch<1, true>(P, F, r, x, omega, s);
        else launch_schur_perpatch<1, false>(P, F, r, x, omega, s);
    }
    count_launch();
    RAV_CHECK_LAUNCH();
    if (det) {
        const int blocks = (int)std::max<int64_t>(1, std::min<int64_t>(cdiv(F.det_n, 256), (int64_t)num_sms() * 16));
        det_gather_kernel<<<blocks, 256, 0, s>>>(F.det_n, F.det_dof, F.det_off, F.det_slot, F.cbuf, x);
        count_launch();
        RAV_CHECK_LAUNCH();
    }
    return RAV_OK;
}

bool schur_fusable(const PatchSet& P, const Factors& F) {
    if (F.cbuf) return false;   // deterministic mode keeps its two-phase scatter
    if (F.layout == 4) return F.D == 2 && (F.MT == 1 || F.MT == 2 || F.MT == 4 || F.MT == 9);
    return F.layout == 5 && F.D >= 1 && F.D <= 3;
}

rav_status launch_schur_sweep_ob(const PatchSet& P, const Factors& F, const double* r, double* x, double omega,
                                 const Outbox& ob, cudaStream_t s) {
    if (!schur_fusable(P, F)) { set_error("fused sweep: unsupported factor layout"); return RAV_ERR_ARG; }
    if (F.layout == 4) {
        switch (F.MT) {
            case 1: launch_schur_thread<1, false, true>(P.n_patches, F, r, x, omega, s, ob); break;
            case 2: launch_schur_thread<2, false, true>(P.n_patches, F, r, x, omega, s, ob); break;
            case 4: launch_schur_thread<4, false, true>(P.n_patches, F, r, x, omega, s, ob); break;
            default: launch_schur_thread<9, false, true>(P.n_patches, F, r, x, omega, s, ob); break;
        }
    } else if (F.D == 3) {
        launch_schur_perpatch<3, false, true>(P, F, r, x, omega, s, ob);
    } else if (F.D == 2) {
        launch_schur_perpatch<2, false, true>(P, F, r, x, omega, s, ob);
    } else {
        launch_schur_perpatch<1, false, true>(P, F, r, x, omega, s, ob);
    }
    count_launch();
    RAV_CHECK_LAUNCH();
    return RAV_OK;
}


// ---- deterministic scatter tables ------------------------------------------------------------
// (dof, slot) pairs of every written correction: restricted node k < m_i, component c -> slot
// i (MT D + 1) + k D + c; the pressure DoF (weight != 0) -> slot i (MT D + 1) + MT D.  Unused
// slots get key INT_MAX and sort to the end.
__global__ void det_pairs_kernel(int64_t np, int layout, int MT, int D, int NN, const int32_t* __restrict__ ND,
                                 const int32_t* __restrict__ NR, const int32_t* __restrict__ PD,
                                 const double* __restrict__ AUX, const int64_t* __restrict__ foffs,
                                 const int64_t* __restrict__ nodeoffs, const int32_t* __restrict__ nodes,
                                 const double* __restrict__ fac, int32_t* __restrict__ key, int32_t* __restrict__ val) {
    const int spp = MT * D + 1;
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < np; i += (int64_t)gridDim.x * blockDim.x) {
        const int m = NR[i];
        double wp;
        if (layout == 4) {
            const int64_t chunk = i >> 5;
            const int lane = (int)(i & 31);
            wp = AUX[(chunk * (MT + 2) + MT) * 32 + lane];
            for (int k = 0; k < MT; ++k)
                for (int cc = 0; cc < D; ++cc) {
                    const int64_t sl = i * spp + k * D + cc;
                    key[sl] = k < m ? ND[(chunk * NN + k) * 32 + lane] + cc : INT_MAX;
                    val[sl] = (int32_t)sl;
                }
        } else {
            const int64_t no = nodeoffs[i];
            const int nn = (int)(nodeoffs[i + 1] - no);
            wp = fac[foffs[i] + (int64_t)MT * nn + (int64_t)nn * D + MT];
            for (int k = 0; k < MT; ++k)
                for (int cc = 0; cc < D; ++cc) {
                    const int64_t sl = i * spp + k * D + cc;
                    key[sl] = k < m ? nodes[no + k] + cc : INT_MAX;
                    val[sl] = (int32_t)sl;
                }
        }
        const int64_t sp = i * spp + MT * D;
        key[sp] = wp != 0.0 ? PD[i] : INT_MAX;
        val[sp] = (int32_t)sp;
    }
}

rav_status schur_det_setup(const PatchSet& P, Factors& F, cudaStream_t s) {
    if (F.layout != 4 && F.layout != 5) {
        set_error("rav_setup: deterministic scatter is implemented for the Schur formats only");
        return RAV_ERR_ARG;
    }
    const int64_t spp = (int64_t)F.MT * F.D + 1;
    const int64_t ns = P.n_patches * spp;
    if (ns >= INT32_MAX) { set_error("rav_setup: too many correction slots for deterministic mode"); return RAV_ERR_ARG; }
    RAV_CUDA(cudaMalloc(&F.cbuf, sizeof(double) * std::max<int64_t>(1, ns)));
    int32_t *key = nullptr, *val = nullptr, *skey = nullptr, *uniq = nullptr, *cnt32 = nullptr;
    int64_t *cnt = nullptr, *nrun = nullptr;
    RAV_CUDA(cudaMallocAsync(&key, sizeof(int32_t) * ns, s));
    RAV_CUDA(cudaMallocAsync(&val, sizeof(int32_t) * ns, s));
    RAV_CUDA(cudaMallocAsync(&skey, sizeof(int32_t) * ns, s));
    RAV_CUDA(cudaMalloc(&F.det_slot, sizeof(int32_t) * ns));
    const int blocks = (int)std::max<int64_t>(1, std::min<int64_t>(cdiv(P.n_patches, 128), (int64_t)num_sms() * 16));
    det_pairs_kernel<<<blocks, 128, 0, s>>>(P.n_patches, F.layout, F.MT, F.D, F.NN, F.DT, F.NR, F.PD, F.WT, F.foffs,
                                            F.nodeoffs, F.nodes, F.fac, key, val);
    count_launch();
    RAV_CHECK_LAUNCH();
    size_t tmp = 0;
    RAV_CUDA(cub::DeviceRadixSort::SortPairs(nullptr, tmp, key, skey, val, F.det_slot, (int)ns, 0, 32, s));
    void* d_tmp = nullptr;
    RAV_CUDA(cudaMallocAsync(&d_tmp, tmp + 16, s));
    // LSD radix sort is stable: equal DoFs keep ascending slots = ascending patches
    RAV_CUDA(cub::DeviceRadixSort::SortPairs(d_tmp, tmp, key, skey, val, F.det_slot, (int)ns, 0, 32, s));
    RAV_CUDA(cudaMallocAsync(&uniq, sizeof(int32_t) * ns, s));
    RAV_CUDA(cudaMallocAsync(&cnt32, sizeof(int32_t) * ns, s));
    RAV_CUDA(cudaMallocAsync(&nrun, sizeof(int64_t), s));
    size_t tmp2 = 0;
    RAV_CUDA(cub::DeviceRunLengthEncode::Encode(nullptr, tmp2, skey, uniq, cnt32, nrun, (int)ns, s));
    void* d_tmp2 = nullptr;
    RAV_CUDA(cudaMallocAsync(&d_tmp2, tmp2 + 16, s));
    RAV_CUDA(cub::DeviceRunLengthEncode::Encode(d_tmp2, tmp2, skey, uniq, cnt32, nrun, (int)ns, s));
    int64_t h_nrun = 0;
    RAV_CUDA(cudaMemcpyAsync(&h_nrun, nrun, sizeof(int64_t), cudaMemcpyDeviceToHost, s));
    RAV_CUDA(cudaStreamSynchronize(s));
    int32_t last = 0;
    if (h_nrun > 0) RAV_CUDA(cudaMemcpy(&last, uniq + h_nrun - 1, sizeof(int32_t), cudaMemcpyDeviceToHost));
    const int64_t nu = (h_nrun > 0 && last == INT_MAX) ? h_nrun - 1 : h_nrun;   // drop the unused-slot run
    F.det_n = nu;
    RAV_CUDA(cudaMalloc(&F.det_dof, sizeof(int32_t) * std::max<int64_t>(1, nu)));
    RAV_CUDA(cudaMalloc(&F.det_off, sizeof(int64_t) * (nu + 1)));
    RAV_CUDA(cudaMallocAsync(&cnt, sizeof(int64_t) * std::max<int64_t>(1, nu), s));
    if (nu > 0) {
        RAV_CUDA(cudaMemcpyAsync(F.det_dof, uniq, sizeof(int32_t) * nu, cudaMemcpyDeviceToDevice, s));
        // widen the counts and scan them into offsets
        std::vector<int32_t> hc(nu);
        RAV_CUDA(cudaMemcpyAsync(hc.data(), cnt32, sizeof(int32_t) * nu, cudaMemcpyDeviceToHost, s));
        RAV_CUDA(cudaStreamSynchronize(s));
        std::vector<int64_t> ho(nu + 1, 0);
        for (int64_t u = 0; u < nu; ++u) ho[u + 1] = ho[u] + hc[u];
        RAV_CUDA(cudaMemcpy(F.det_off, ho.data(), sizeof(int64_t) * (nu + 1), cudaMemcpyHostToDevice));
    } else {
        RAV_CUDA(cudaMemsetAsync(F.det_off, 0, sizeof(int64_t), s));
    }
    for (void* p : {(void*)key, (void*)val, (void*)skey, (void*)uniq, (void*)cnt32, (void*)cnt, (void*)nrun, d_tmp,
                    d_tmp2})
        cudaFreeAsync(p, s);
    RAV_CUDA(cudaStreamSynchronize(s));
    return RAV_OK;
}

}  // namespace rav
