// gen.cu -- device-side generator of the structured Taylor-Hood Q2-Q1 Stokes
// levels (SURVEY section 8 rows a1 "level operators", a3 "patch builder", a7
// "transfers").  Row-parallel, deterministic assembly: every CSR entry is
// computed by the thread owning its row as a sum over the elements shared by
// its row and column DoFs (Eq. 7) -- no atomics, no COO sort, and
// entries (i,j) and (j,i) are produced by the same arithmetic in the same
// order, so L = L^T bitwise.
#include <cub/cub.cuh>
#include <math_constants.h>

#include <vector>

#include "common.cuh"
#include "internal.cuh"

namespace rav {
namespace gen {


struct Grid {
    int dim;
    int n[3];        // cells per axis
    double h[3];
    double vol;      // prod h
    int kind;
    int eta_mode;
    double eta0;
    int nm;
    double amp[8];
    int mode[8][3];
    double phase[8][3];
    double gmin, gmax;
    int64_t nfree, nvel, nvert, ndof, nel;
    // window along the last axis (rav_grid.win); whole grid when win == 0
    int last;
    int64_t nlow_free, nlow_vert;   // free nodes / vertices per layer of the last axis
    int64_t vel_off, vert_off;      // global velocity-DoF / vertex offsets of the window
    int64_t nvel_loc, nvert_loc, ndof_loc;
    int rnode_lo, rnode_hi, rvert_lo, rvert_hi;
    int64_t patch_off, npatch;      // first global vertex with a patch, number of patches
    // element pair: P = 2 Taylor-Hood Q2-Q1 (velocity nodes on the (2n+1)^d lattice, R1),
    // P = 1 stabilized Q1-Q1 (velocity on the vertices, C of P:78 Eq. 8, R18)
    int P, ngp;                     // velocity lattice refinement, Gauss points per axis (P + 1)
    double gt[3], gw[3];            // Gauss rule on [0,1] (3-point for Q2-Q1 R7, 2-point for Q1-Q1 R18)
    double beta, he2;               // stabilization beta_0 and squared element diameter
};

static Grid make_grid(const rav_grid* g) {
    Grid G{};
    G.dim = g->dim;
    G.P = g->vel_order == 1 ? 1 : 2;
    G.ngp = G.P + 1;
    if (G.P == 2) {
        const double a = 0.5 * 0.77459666924148337704;  // sqrt(3/5)/2
        G.gt[0] = 0.5 - a; G.gt[1] = 0.5; G.gt[2] = 0.5 + a;
        G.gw[0] = 5.0 / 18.0; G.gw[1] = 8.0 / 18.0; G.gw[2] = 5.0 / 18.0;
    } else {
        const double a = 0.5 * 0.57735026918962576451;  // sqrt(1/3)/2
        G.gt[0] = 0.5 - a; G.gt[1] = 0.5 + a;
        G.gw[0] = 0.5; G.gw[1] = 0.5;
    }
    G.beta = g->beta;
    G.vol = 1.0;
    G.nfree = 1;
    G.nvert = 1;
    G.nel = 1;
    for (int k = 0; k < 3; ++k) {
        G.n[k] = k < g->dim ? g->ncell[k] : 1;
        G.h[k] = k < g->dim ? g->len[k] / g->ncell[k] : 1.0;
    }
    for (int k = 0; k < g->dim; ++k) {
        G.vol *= G.h[k];
        G.nfree *= (int64_t)(G.P * G.n[k] - 1);
        G.he2 += G.h[k] * G.h[k];
        G.nvert *= (int64_t)(G.n[k] + 1);
        G.nel *= G.n[k];
    }
    G.kind = g->kind;
    G.eta_mode = g->eta_mode;
    G.eta0 = g->eta0;
    G.nm = g->n_modes;
    for (int m = 0; m < 8; ++m) {
        G.amp[m] = g->amp[m];
        for (int k = 0; k < 3; ++k) {
            G.mode[m][k] = g->mode[m][k];
            G.phase[m][k] = g->phase[m][k];
        }
    }
    G.gmin = g->gmin;
    G.gmax = g->gmax;
    G.nvel = (int64_t)g->dim * G.nfree;
    G.ndof = G.nvel + G.nvert;
    G.last = g->dim - 1;
    G.nlow_free = G.nfree / (G.P * G.n[G.last] - 1);
    G.nlow_vert = G.nvert / (G.n[G.last] + 1);
    int node_lo = 1, node_hi = G.P * G.n[G.last] - 1, vert_lo = 0, vert_hi = G.n[G.last];
    G.rnode_lo = node_lo; G.rnode_hi = node_hi; G.rvert_lo = vert_lo; G.rvert_hi = vert_hi;
    int pv_lo = 0, pv_hi = G.n[G.last];
    if (g->win) {
        node_lo = std::max(1, g->node_lo);
        node_hi = std::min(G.P * G.n[G.last] - 1, g->node_hi);
        vert_lo = std::max(0, g->vert_lo);
        vert_hi = std::min(G.n[G.last], g->vert_hi);
        G.rnode_lo = g->rnode_lo; G.rnode_hi = g->rnode_hi;
        G.rvert_lo = g->rvert_lo; G.rvert_hi = g->rvert_hi;
        pv_lo = std::max(0, g->pvert_lo);
        pv_hi = std::min(G.n[G.last], g->pvert_hi);
    }
    G.vel_off = (int64_t)g->dim * G.nlow_free * (node_lo - 1);
    G.nvel_loc = (int64_t)g->dim * G.nlow_free * std::max(0, node_hi - node_lo + 1);
    G.vert_off = G.nlow_vert * vert_lo;
    G.nvert_loc = G.nlow_vert * std::max(0, vert_hi - vert_lo + 1);
    G.ndof_loc = G.nvel_loc + G.nvert_loc;
    G.patch_off = G.nlow_vert * pv_lo;
    G.npatch = G.nlow_vert * std::max(0, pv_hi - pv_lo + 1);
    return G;
}

// local index of a global velocity DoF / vertex in the window, -1 outside
__device__ __forceinline__ int64_t loc_vel(const Grid& G, int64_t gdof) {
    const int64_t l = gdof - G.vel_off;
    return (l >= 0 && l < G.nvel_loc) ? l : -1;
}
__device__ __forceinline__ int64_t loc_vert(const Grid& G, int64_t vid) {
    const int64_t l = vid - G.vert_off;
    return (l >= 0 && l < G.nvert_loc) ? G.nvel_loc + l : -1;
}

static rav_status check_grid(const rav_grid* g) {
    if (!g || (g->dim != 2 && g->dim != 3)) { set_error("rav_grid: dim must be 2 or 3"); return RAV_ERR_ARG; }
    for (int k = 0; k < g->dim; ++k)
        if (g->ncell[k] < 1 || !(g->len[k] > 0)) { set_error("rav_grid: bad ncell/len"); return RAV_ERR_ARG; }
    if (g->kind == 1 && g->dim != 2) { set_error("rav_grid: manufactured solution is 2D only"); return RAV_ERR_ARG; }
    if (g->kind < 0 || g->kind > 2) { set_error("rav_grid: bad kind"); return RAV_ERR_ARG; }
    if (g->n_modes < 0 || g->n_modes > 8) { set_error("rav_grid: n_modes > 8"); return RAV_ERR_ARG; }
    if (g->eta_mode == 1 && !(g->gmax > g->gmin)) { set_error("rav_grid: gmax <= gmin"); return RAV_ERR_ARG; }
    if (g->vel_order != 0 && g->vel_order != 1 && g->vel_order != 2) { set_error("rav_grid: vel_order must be 1 or 2"); return RAV_ERR_ARG; }
    if (g->vel_order == 1 && g->win) { set_error("rav_grid: slab windows are implemented for Q2-Q1 only"); return RAV_ERR_ARG; }
    if (g->vel_order == 1 && !(g->beta > 0.0)) { set_error("rav_grid: Q1-Q1 needs beta > 0 (P:80)"); return RAV_ERR_ARG; }
    if (g->win && (g->node_lo > g->node_hi || g->vert_lo > g->vert_hi || g->pvert_lo > g->pvert_hi)) {
        set_error("rav_grid: empty window");
        return RAV_ERR_ARG;
    }
    return RAV_OK;
}


// ---- 1D bases -------------------------------------------------------------------
__device__ __forceinline__ double q2v(int l, double t) {
    return l == 0 ? (2.0 * t - 1.0) * (t - 1.0) : (l == 1 ? 4.0 * t * (1.0 - t) : t * (2.0 * t - 1.0));
}
__device__ __forceinline__ double q2d(int l, double t) {
    return l == 0 ? 4.0 * t - 3.0 : (l == 1 ? 4.0 - 8.0 * t : 4.0 * t - 1.0);
}
__device__ __forceinline__ double q1v(int m, double t) { return m == 0 ? 1.0 - t : t; }
__device__ __forceinline__ double q1d(int m, double t) { (void)t; return m == 0 ? -1.0 : 1.0; }
// velocity basis of the element pair (P = 2: Q2, P = 1: Q1)
__device__ __forceinline__ double vbv(int P, int l, double t) { return P == 2 ? q2v(l, t) : q1v(l, t); }
__device__ __forceinline__ double vbd(int P, int l, double t) { return P == 2 ? q2d(l, t) : q1d(l, t); }

// ---- lattice helpers --------------------------------------------------------------
__device__ __forceinline__ int64_t free_id(const Grid& G, const int* a) {
    int64_t id = 0, s = 1;
    for (int k = 0; k < G.dim; ++k) {
        int m = G.P * G.n[k];
        if (a[k] <= 0 || a[k] >= m) return -1;
        id += (int64_t)(a[k] - 1) * s;
        s *= (m - 1);
    }
    return id;
}
__device__ __forceinline__ int64_t vert_id(const Grid& G, const int* v) {
    int64_t id = 0, s = 1;
    for (int k = 0; k < G.dim; ++k) { id += (int64_t)v[k] * s; s *= (G.n[k] + 1); }
    return id;
}
__device__ __forceinline__ int64_t elem_id(const Grid& G, const int* e) {
    int64_t id = 0, s = 1;
    for (int k = 0; k < G.dim; ++k) { id += (int64_t)e[k] * s; s *= G.n[k]; }
    return id;
}
// range of elements along one axis containing velocity lattice node index a
__device__ __forceinline__ void node_elems(int P, int a, int n, int& lo, int& hi) {
    if (P == 1) { lo = a - 1; hi = a; }
    else if (a & 1) { lo = hi = (a - 1) >> 1; }
    else { lo = (a >> 1) - 1; hi = a >> 1; }
    if (lo < 0) lo = 0;
    if (hi > n - 1) hi = n - 1;
}
__device__ __forceinline__ void vert_elems(int v, int n, int& lo, int& hi) {
    lo = v - 1 < 0 ? 0 : v - 1;
    hi = v > n - 1 ? n - 1 : v;
}

// Dirichlet data (R8): cavity lid u = e_x on the interior of the top face
__device__ __forceinline__ double dirichlet(const Grid& G, const int* a, int c) {
    if (G.kind != 0 || c != 0) return 0.0;
    int top = G.dim - 1;
    if (a[top] != G.P * G.n[top]) return 0.0;
    for (int k = 0; k < top; ++k)
        if (a[k] <= 0 || a[k] >= G.P * G.n[k]) return 0.0;
    return 1.0;
}

// ---- coefficient tables at quadrature points (R12, R13) -------------------------------
__device__ void eta_grad(const Grid& G, const double* x, double& eta, double* ge) {
    ge[0] = ge[1] = ge[2] = 0.0;
    if (G.eta_mode == 0) { eta = G.eta0; return; }
    double g = 0.0, dg[3] = {0.0, 0.0, 0.0};
    for (int m = 0; m < G.nm; ++m) {
        double cs[3] = {1.0, 1.0, 1.0}, sn[3] = {0.0, 0.0, 0.0};
        for (int k = 0; k < G.dim; ++k) sincos(CUDART_PI * G.mode[m][k] * x[k] + G.phase[m][k], &sn[k], &cs[k]);
        double p = G.amp[m];
        for (int k = 0; k < G.dim; ++k) p *= cs[k];
        g += p;
        for (int k = 0; k < G.dim; ++k) {
            double t = -G.amp[m] * CUDART_PI * G.mode[m][k] * sn[k];
            for (int j = 0; j < G.dim; ++j) if (j != k) t *= cs[j];
            dg[k] += t;
        }
    }
    double sc = log(100.0) / (G.gmax - G.gmin);
    eta = exp(log(0.1) + (g - G.gmin) * sc);
    for (int k = 0; k < G.dim; ++k) ge[k] = eta * sc * dg[k];
}

// f = -div(eta grad u) + grad p for u = curl(sin^2 pi x sin^2 pi y), p = cos pi x cos pi y
__device__ void mms_force(const Grid& G, const double* x, double* f) {
    const double pi = CUDART_PI;
    double eta, ge[3];
    eta_grad(G, x, eta, ge);
    double sx, cx, sy, cy, s2x, c2x, s2y, c2y;
    sincos(pi * x[0], &sx, &cx);
    sincos(pi * x[1], &sy, &cy);
    sincos(2.0 * pi * x[0], &s2x, &c2x);
    sincos(2.0 * pi * x[1], &s2y, &c2y);
    const double pi2 = pi * pi, pi3 = pi2 * pi;
    // u0 = pi sx^2 s2y ; u1 = -pi s2x sy^2
    double u0x = pi2 * s2x * s2y, u0y = 2.0 * pi2 * sx * sx * c2y;
    double lap0 = 2.0 * pi3 * c2x * s2y - 4.0 * pi3 * sx * sx * s2y;
    double u1x = -2.0 * pi2 * c2x * sy * sy, u1y = -pi2 * s2x * s2y;
    double lap1 = 4.0 * pi3 * s2x * sy * sy - 2.0 * pi3 * s2x * c2y;
    f[0] = -eta * lap0 - (ge[0] * u0x + ge[1] * u0y) - pi * sx * cy;
    f[1] = -eta * lap1 - (ge[0] * u1x + ge[1] * u1y) - pi * cx * sy;
}

// one thread per (element, quadrature point): eta and (MMS) f
__global__ void coef_kernel(Grid G, double* eta_tab, double* f_tab) {
    const int NG = G.dim == 2 ? G.ngp * G.ngp : G.ngp * G.ngp * G.ngp;
    int64_t total = G.nel * NG;
    for (int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; t < total;
         t += (int64_t)gridDim.x * blockDim.x) {
        int64_t el = t / NG;
        int q = (int)(t % NG);
        int e[3] = {0, 0, 0};
        int64_t r = el;
        for (int k = 0; k < G.dim; ++k) { e[k] = (int)(r % G.n[k]); r /= G.n[k]; }
        double x[3] = {0, 0, 0};
        int qq = q;
        for (int k = 0; k < G.dim; ++k) { x[k] = (e[k] + G.gt[qq % G.ngp]) * G.h[k]; qq /= G.ngp; }
        double eta, ge[3];
        eta_grad(G, x, eta, ge);
        eta_tab[t] = eta;
        if (f_tab) {
            double f[3] = {0.0, 0.0, 0.0};
            if (G.kind == 1) mms_force(G, x, f);
            f_tab[2 * t] = f[0];
            f_tab[2 * t + 1] = f[1];
        }
    }
}

// ---- entry formulas -------------------------------------------------------------------
// Basis values at the quadrature points of the reference element, formed once per CTA (the same
// expressions the entry formulas evaluated inline before, so the entries do not change): velocity
// basis v[l][q] and derivative / h_k d[k][l][q]; Q1 (pressure) basis pv[m][q], pd[k][m][q].
// Removes the per-entry basis polynomials and FP64 divisions from the row-gather assembly.
struct BasisTab {
    double v[3][3];
    double d[3][3][3];
    double pv[2][3];
    double pd[3][2][3];
};
__device__ void basis_tab_init(const Grid& G, BasisTab& T) {
    for (int idx = threadIdx.x; idx < 9 + 27 + 6 + 18; idx += blockDim.x) {
        if (idx < 9) {
            const int l = idx / 3, q = idx % 3;
            T.v[l][q] = (q < G.ngp && l <= G.P) ? vbv(G.P, l, G.gt[q]) : 0.0;
        } else if (idx < 36) {
            const int t = idx - 9, k = t / 9, l = (t / 3) % 3, q = t % 3;
            T.d[k][l][q] = (q < G.ngp && l <= G.P) ? vbd(G.P, l, G.gt[q]) / G.h[k] : 0.0;
        } else if (idx < 42) {
            const int t = idx - 36, m = t / 3, q = t % 3;
            T.pv[m][q] = q < G.ngp ? q1v(m, G.gt[q]) : 0.0;
        } else {
            const int t = idx - 42, k = t / 6, m = (t / 3) % 2, q = t % 3;
            T.pd[k][m][q] = q < G.ngp ? q1d(m, G.gt[q]) / G.h[k] : 0.0;
        }
    }
}

// Element matrices (row a1).  A_e[i][j] = int_e eta grad phi_i . grad phi_j (i <= j, local node
// index i = l_x + (P+1) l_y [+ (P+1)^2 l_z]) is formed once per element by elem_a_kernel with the
// quadrature of the former per-entry loop; an entry then sums A_e over the elements its two nodes
// share, in the same element order.  The B block is the same for every element of a uniform
// level: B_e[i][m][c] = -int_e psi_m d_c phi_i, formed once per CTA in shared memory.
__device__ __forceinline__ int pair_index(int NL, int i, int j) {   // i <= j
    return i * NL - i * (i - 1) / 2 + (j - i);
}

__global__ void elem_a_kernel(Grid G, const double* __restrict__ eta_tab, double* __restrict__ Ae) {
    __shared__ BasisTab T;
    basis_tab_init(G, T);
    __syncthreads();
    const int P1 = G.P + 1;
    const int NL = G.dim == 2 ? P1 * P1 : P1 * P1 * P1;
    const int NPAIR = NL * (NL + 1) / 2;
    const int g = G.ngp, NG = G.dim == 2 ? g * g : g * g * g;
    for (int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; t < G.nel * NPAIR;
         t += (int64_t)gridDim.x * blockDim.x) {
        const int64_t el = t / NPAIR;
        int pr = (int)(t % NPAIR), i = 0;
        while (pr >= NL - i) { pr -= NL - i; ++i; }
        const int j = i + pr;
        int la[3] = {0, 0, 0}, lb[3] = {0, 0, 0};
        for (int k = 0, ii = i, jj = j; k < G.dim; ++k) { la[k] = ii % P1; ii /= P1; lb[k] = jj % P1; jj /= P1; }
        const double* et = eta_tab + el * NG;
        double s = 0.0;
        for (int q = 0; q < NG; ++q) {
            int qk[3] = {q % g, (q / g) % g, q / (g * g)};
            double va[3], vb[3], da[3], db[3], w = G.vol;
            for (int k = 0; k < G.dim; ++k) {
                w *= G.gw[qk[k]];
                va[k] = T.v[la[k]][qk[k]]; vb[k] = T.v[lb[k]][qk[k]];
                da[k] = T.d[k][la[k]][qk[k]]; db[k] = T.d[k][lb[k]][qk[k]];
            }
            double dot = 0.0;
            for (int k = 0; k < G.dim; ++k) {
                double ga = da[k], gb = db[k];
                for (int m = 0; m < G.dim; ++m) if (m != k) { ga *= va[m]; gb *= vb[m]; }
                dot += ga * gb;
            }
            s += (w * et[q]) * dot;
        }
        Ae[t] = s;
    }
}

struct ElemB {
    double b[27][8][3];
};
__device__ void elem_b_init(const Grid& G, const BasisTab& T, ElemB& E) {
    const int P1 = G.P + 1;
    const int NL = G.dim == 2 ? P1 * P1 : P1 * P1 * P1;
    const int NV = G.dim == 2 ? 4 : 8;
    const int g = G.ngp, NG = G.dim == 2 ? g * g : g * g * g;
    for (int idx = threadIdx.x; idx < NL * NV * G.dim; idx += blockDim.x) {
        const int c = idx % G.dim, m = (idx / G.dim) % NV, i = idx / (G.dim * NV);
        int lb[3] = {0, 0, 0}, lm[3] = {0, 0, 0};
        for (int k = 0, ii = i, mm = m; k < G.dim; ++k) { lb[k] = ii % P1; ii /= P1; lm[k] = mm % 2; mm /= 2; }
        double s = 0.0;
        for (int q = 0; q < NG; ++q) {
            int qk[3] = {q % g, (q / g) % g, q / (g * g)};
            double w = G.vol, psi = 1.0, dphi = 1.0;
            for (int k = 0; k < G.dim; ++k) {
                w *= G.gw[qk[k]];
                psi *= T.pv[lm[k]][qk[k]];
                dphi *= (k == c) ? T.d[k][lb[k]][qk[k]] : T.v[lb[k]][qk[k]];
            }
            s -= (w * psi) * dphi;
        }
        E.b[i][m][c] = s;
    }
}

// int_e eta grad phi_a . grad phi_b over the elements shared by nodes a and b
__device__ double a_entry(const Grid& G, const double* __restrict__ Ae, const int* a, const int* b) {
    int lo[3] = {0, 0, 0}, hi[3] = {0, 0, 0};
    for (int k = 0; k < G.dim; ++k) {
        int la, ha, lb, hb;
        node_elems(G.P, a[k], G.n[k], la, ha);
        node_elems(G.P, b[k], G.n[k], lb, hb);
        lo[k] = max(la, lb);
        hi[k] = min(ha, hb);
        if (lo[k] > hi[k]) return 0.0;
    }
    const int P1 = G.P + 1;
    const int NL = G.dim == 2 ? P1 * P1 : P1 * P1 * P1;
    const int NPAIR = NL * (NL + 1) / 2;
    double s = 0.0;
    int e[3] = {0, 0, 0};
    for (e[2] = lo[2]; e[2] <= hi[2]; ++e[2])
        for (e[1] = lo[1]; e[1] <= hi[1]; ++e[1])
            for (e[0] = lo[0]; e[0] <= hi[0]; ++e[0]) {
                int ia = 0, ib = 0;
                for (int k = G.dim - 1; k >= 0; --k) {
                    ia = ia * P1 + (a[k] - G.P * e[k]);
                    ib = ib * P1 + (b[k] - G.P * e[k]);
                }
                s += __ldg(Ae + elem_id(G, e) * NPAIR + pair_index(NL, min(ia, ib), max(ia, ib)));
            }
    return s;
}

// -int_e psi_v d_c phi_b over the elements shared by node b and vertex v
__device__ double b_entry(const Grid& G, const ElemB& E, const int* b, int c, const int* v) {
    int lo[3] = {0, 0, 0}, hi[3] = {0, 0, 0};
    for (int k = 0; k < G.dim; ++k) {
        int lb, hb, lv, hv;
        node_elems(G.P, b[k], G.n[k], lb, hb);
        vert_elems(v[k], G.n[k], lv, hv);
        lo[k] = max(lb, lv);
        hi[k] = min(hb, hv);
        if (lo[k] > hi[k]) return 0.0;
    }
    const int P1 = G.P + 1;
    double s = 0.0;
    int e[3] = {0, 0, 0};
    for (e[2] = lo[2]; e[2] <= hi[2]; ++e[2])
        for (e[1] = lo[1]; e[1] <= hi[1]; ++e[1])
            for (e[0] = lo[0]; e[0] <= hi[0]; ++e[0]) {
                int ib = 0, im = 0;
                for (int k = G.dim - 1; k >= 0; --k) {
                    ib = ib * P1 + (b[k] - G.P * e[k]);
                    im = im * 2 + (v[k] - e[k]);
                }
                s += E.b[ib][im][c];
            }
    return s;
}

// int f_c phi_a over the elements containing node a (2D manufactured forcing)
__device__ double f_entry(const Grid& G, const BasisTab& T, const double* f_tab, const int* a, int c) {
    if (G.kind != 1) return 0.0;
    int lo[3] = {0, 0, 0}, hi[3] = {0, 0, 0};
    for (int k = 0; k < G.dim; ++k) node_elems(G.P, a[k], G.n[k], lo[k], hi[k]);
    const int g = G.ngp, NG = g * g;
    double s = 0.0;
    int e[3] = {0, 0, 0};
    for (e[1] = lo[1]; e[1] <= hi[1]; ++e[1])
        for (e[0] = lo[0]; e[0] <= hi[0]; ++e[0]) {
            int la[2] = {a[0] - G.P * e[0], a[1] - G.P * e[1]};
            int64_t el = elem_id(G, e);
            for (int q = 0; q < NG; ++q) {
                double w = G.vol * G.gw[q % g] * G.gw[q / g];
                s += (w * f_tab[2 * (el * NG + q) + c]) * (T.v[la[0]][q % g] * T.v[la[1]][q / g]);
            }
        }
    return s;
}

// Q1-Q1 stabilization (Eq. 8, R18): -beta_0 h_e^2 int (1/eta) grad psi_v . grad psi_u over the
// elements shared by vertices v and u
__device__ double c_entry(const Grid& G, const BasisTab& T, const double* eta_tab, const int* v, const int* u) {
    int lo[3] = {0, 0, 0}, hi[3] = {0, 0, 0};
    for (int k = 0; k < G.dim; ++k) {
        int lv, hv, lu, hu;
        vert_elems(v[k], G.n[k], lv, hv);
        vert_elems(u[k], G.n[k], lu, hu);
        lo[k] = max(lv, lu);
        hi[k] = min(hv, hu);
        if (lo[k] > hi[k]) return 0.0;
    }
    const int g = G.ngp, NG = G.dim == 2 ? g * g : g * g * g;
    double s = 0.0;
    int e[3] = {0, 0, 0};
    for (e[2] = lo[2]; e[2] <= hi[2]; ++e[2])
        for (e[1] = lo[1]; e[1] <= hi[1]; ++e[1])
            for (e[0] = lo[0]; e[0] <= hi[0]; ++e[0]) {
                int lv[3], lu[3];
                for (int k = 0; k < 3; ++k) { lv[k] = v[k] - e[k]; lu[k] = u[k] - e[k]; }
                const double* et = eta_tab + elem_id(G, e) * NG;
                for (int q = 0; q < NG; ++q) {
                    int qk[3] = {q % g, (q / g) % g, q / (g * g)};
                    double vv[3], vu[3], dv[3], du[3], w = G.vol;
                    for (int k = 0; k < G.dim; ++k) {
                        w *= G.gw[qk[k]];
                        vv[k] = T.pv[lv[k]][qk[k]]; vu[k] = T.pv[lu[k]][qk[k]];
                        dv[k] = T.pd[k][lv[k]][qk[k]]; du[k] = T.pd[k][lu[k]][qk[k]];
                    }
                    double dot = 0.0;
                    for (int k = 0; k < G.dim; ++k) {
                        double gv = dv[k], gu = du[k];
                        for (int j = 0; j < G.dim; ++j) if (j != k) { gv *= vv[j]; gu *= vu[j]; }
                        dot += gv * gu;
                    }
                    s -= G.beta * G.he2 * (w / et[q]) * dot;
                }
            }
    return s;
}

// ---- row decoding -----------------------------------------------------------------------
__device__ __forceinline__ void decode_vel_row(const Grid& G, int64_t row, int* a, int& c) {
    int64_t fi = row / G.dim;
    c = (int)(row % G.dim);
    a[0] = a[1] = a[2] = 0;
    for (int k = 0; k < G.dim; ++k) {
        int m = G.P * G.n[k] - 1;
        a[k] = (int)(fi % m) + 1;
        fi /= m;
    }
}
__device__ __forceinline__ void decode_vertex(const Grid& G, int64_t vi, int* v) {
    v[0] = v[1] = v[2] = 0;
    for (int k = 0; k < G.dim; ++k) { v[k] = (int)(vi % (G.n[k] + 1)); vi /= (G.n[k] + 1); }
}

// ---- operator: count / fill ---------------------------------------------------------------
// Row pattern (structural, R2): velocity row (a, c): same-component velocity DoFs of
// the nodes of all elements containing a, then the pressure DoFs of their vertices;
// pressure row v: all velocity DoFs of the nodes of the elements containing v.
// decode a LOCAL row of the window: velocity (node a, component c) or vertex a;
// false when the row lies outside the row window (empty row)
__device__ __forceinline__ bool decode_local_row(const Grid& G, int64_t row, int* a, int& c, bool& vel) {
    vel = row < G.nvel_loc;
    if (vel) {
        decode_vel_row(G, row + G.vel_off, a, c);
        return a[G.last] >= G.rnode_lo && a[G.last] <= G.rnode_hi;
    }
    decode_vertex(G, row - G.nvel_loc + G.vert_off, a);
    c = 0;
    return a[G.last] >= G.rvert_lo && a[G.last] <= G.rvert_hi;
}

__global__ void op_count_kernel(Grid G, int64_t* cnt) {
    for (int64_t row = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; row < G.ndof_loc;
         row += (int64_t)gridDim.x * blockDim.x) {
        int lo[3] = {0, 0, 0}, hi[3] = {0, 0, 0}, a[3] = {0, 0, 0}, c = 0;
        bool vel;
        if (!decode_local_row(G, row, a, c, vel)) { cnt[row] = 0; continue; }
        for (int k = 0; k < G.dim; ++k) {
            if (vel) node_elems(G.P, a[k], G.n[k], lo[k], hi[k]);
            else vert_elems(a[k], G.n[k], lo[k], hi[k]);
        }
        int64_t nodes = 1, verts = 1;
        for (int k = 0; k < G.dim; ++k) {
            // free lattice nodes in [P lo, P hi + P] intersected with [1, P n - 1]
            int l = max(G.P * lo[k], 1), h = min(G.P * hi[k] + G.P, G.P * G.n[k] - 1);
            nodes *= (h - l + 1);
            verts *= (hi[k] - lo[k] + 2);
        }
        // velocity row: velocity + pressure (B); pressure row: velocity (B^T) [+ pressure (C), Q1-Q1]
        cnt[row] = vel ? nodes + verts : nodes * G.dim + (G.P == 1 ? verts : 0);
    }
}

__global__ void op_fill_kernel(Grid G, const double* eta_tab, const double* __restrict__ Ae, const double* f_tab,
                               const int64_t* rp, int32_t* col, double* val, double* rhs, unsigned int* err) {
    __shared__ BasisTab T;
    __shared__ ElemB E;
    basis_tab_init(G, T);
    __syncthreads();
    elem_b_init(G, T, E);
    __syncthreads();
    for (int64_t row = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; row < G.ndof_loc;
         row += (int64_t)gridDim.x * blockDim.x) {
        int64_t p = rp[row];
        int lo[3] = {0, 0, 0}, hi[3] = {0, 0, 0}, a[3] = {0, 0, 0}, c = 0;
        bool vel;
        if (!decode_local_row(G, row, a, c, vel)) { rhs[row] = 0.0; continue; }
        for (int k = 0; k < G.dim; ++k) {
            if (vel) node_elems(G.P, a[k], G.n[k], lo[k], hi[k]);
            else vert_elems(a[k], G.n[k], lo[k], hi[k]);
        }
        double lift = 0.0;
        int bl[3] = {0, 0, 0}, bh[3] = {0, 0, 0};
        for (int k = 0; k < G.dim; ++k) { bl[k] = G.P * lo[k]; bh[k] = G.P * hi[k] + G.P; }
        int b[3] = {0, 0, 0};
        for (b[2] = bl[2]; b[2] <= bh[2]; ++b[2])
            for (b[1] = bl[1]; b[1] <= bh[1]; ++b[1])
                for (b[0] = bl[0]; b[0] <= bh[0]; ++b[0]) {
                    int64_t fb = free_id(G, b);
                    if (vel) {
                        if (fb >= 0) {
                            const int64_t lc = loc_vel(G, fb * G.dim + c);
                            if (lc < 0) atomicOr(err, 1u);
                            col[p] = (int32_t)lc;
                            val[p] = a_entry(G, Ae, a, b);
                            ++p;
                        } else {
                            double ud = dirichlet(G, b, c);
                            if (ud != 0.0) lift -= a_entry(G, Ae, a, b) * ud;
                        }
                    } else {
                        for (int cc = 0; cc < G.dim; ++cc) {
                            if (fb >= 0) {
                                const int64_t lc = loc_vel(G, fb * G.dim + cc);
                                if (lc < 0) atomicOr(err, 1u);
                                col[p] = (int32_t)lc;
                                val[p] = b_entry(G, E, b, cc, a);
                                ++p;
                            } else {
                                double ud = dirichlet(G, b, cc);
                                if (ud != 0.0) lift -= b_entry(G, E, b, cc, a) * ud;
                            }
                        }
                    }
                }
        if (vel || G.P == 1) {   // B entries of a velocity row / C entries of a Q1-Q1 pressure row
            int v[3] = {0, 0, 0};
            for (v[2] = lo[2]; v[2] <= (G.dim > 2 ? hi[2] + 1 : 0); ++v[2])
                for (v[1] = lo[1]; v[1] <= hi[1] + 1; ++v[1])
                    for (v[0] = lo[0]; v[0] <= hi[0] + 1; ++v[0]) {
                        const int64_t lc = loc_vert(G, vert_id(G, v));
                        if (lc < 0) atomicOr(err, 1u);
                        col[p] = (int32_t)lc;
                        val[p] = vel ? b_entry(G, E, a, c, v) : c_entry(G, T, eta_tab, a, v);
                        ++p;
                    }
        }
        rhs[row] = vel ? f_entry(G, T, f_tab, a, c) + lift : lift;
    }
}

// ---- patches -------------------------------------------------------------------
__device__ __forceinline__ double patch_weight(int mode, int dim, int P, const int* a, const int* v) {
    if (mode == 2) return 1.0;
    double w = 1.0;
    for (int k = 0; k < dim; ++k) {
        int off = a[k] - P * v[k];
        if (P == 1) {          // Q1-Q1: the velocity DoFs on the pressure node
            if (off != 0) return 0.0;
            continue;
        }
        if (mode == 0) {
            if (off < -1 || off > 1) return 0.0;
            if (off != 0) w *= 0.5;
        } else if (off != 0 && off != 1) {
            return 0.0;
        }
    }
    return w;
}

__global__ void patch_count_kernel(Grid G, int64_t* cnt) {
    for (int64_t pi = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; pi < G.npatch;
         pi += (int64_t)gridDim.x * blockDim.x) {
        int v[3];
        decode_vertex(G, pi + G.patch_off, v);
        int64_t nodes = 1;
        for (int k = 0; k < G.dim; ++k) {
            int l = max(G.P * v[k] - G.P, 1), h = min(G.P * v[k] + G.P, G.P * G.n[k] - 1);
            nodes *= (h - l + 1);
        }
        cnt[pi] = nodes * G.dim + 1;
    }
}

__global__ void patch_fill_kernel(Grid G, int mode, const int64_t* offs, int32_t* dofs, double* w,
                                  unsigned int* err) {
    for (int64_t pi = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; pi < G.npatch;
         pi += (int64_t)gridDim.x * blockDim.x) {
        const int64_t vi = pi + G.patch_off;
        int v[3];
        decode_vertex(G, vi, v);
        int l[3] = {0, 0, 0}, h[3] = {0, 0, 0};
        for (int k = 0; k < G.dim; ++k) { l[k] = max(G.P * v[k] - G.P, 1); h[k] = min(G.P * v[k] + G.P, G.P * G.n[k] - 1); }
        int64_t p = offs[pi];
        for (int pass = 0; pass < 2; ++pass) {
            if (pass == 1) {
                const int64_t lp = loc_vert(G, vi);
                if (lp < 0) atomicOr(err, 1u);
                dofs[p] = (int32_t)lp;
                w[p] = 1.0;
                ++p;
            }
            int a[3] = {0, 0, 0};
            for (a[2] = l[2]; a[2] <= h[2]; ++a[2])
                for (a[1] = l[1]; a[1] <= h[1]; ++a[1])
                    for (a[0] = l[0]; a[0] <= h[0]; ++a[0]) {
                        double wt = patch_weight(mode, G.dim, G.P, a, v);
                        if ((pass == 0) != (wt > 0.0)) continue;
                        int64_t fa = free_id(G, a);
                        for (int c = 0; c < G.dim; ++c) {
                            const int64_t lc = loc_vel(G, fa * G.dim + c);
                            if (lc < 0) atomicOr(err, 1u);
                            dofs[p] = (int32_t)lc;
                            w[p] = wt;
                            ++p;
                        }
                    }
        }
    }
}

// ---- prolongation ------------------------------------------------------------------------
__device__ __forceinline__ int interp_q2(int af, int nc, int* idx, double* wt) {
    if (!(af & 1)) { idx[0] = af >> 1; wt[0] = 1.0; return 1; }
    int e = af >> 2;
    if (e > nc - 1) e = nc - 1;
    double t = (af - 4.0 * e) * 0.25;
    for (int i = 0; i < 3; ++i) { idx[i] = 2 * e + i; wt[i] = q2v(i, t); }
    return 3;
}
__device__ __forceinline__ int interp_q1(int bf, int* idx, double* wt) {
    if (!(bf & 1)) { idx[0] = bf >> 1; wt[0] = 1.0; return 1; }
    idx[0] = (bf - 1) >> 1; wt[0] = 0.5;
    idx[1] = (bf + 1) >> 1; wt[1] = 0.5;
    return 2;
}

template <bool FILL>
__global__ void prol_kernel(Grid F, Grid Cg, int64_t* cnt_or_rp, int32_t* ci, double* val, unsigned int* err) {
    // rows: LOCAL DoFs of the fine window (rows outside its row window are empty);
    // columns: LOCAL DoFs of the coarse window (= global ids when it is the whole grid)
    for (int64_t row = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; row < F.ndof_loc;
         row += (int64_t)gridDim.x * blockDim.x) {
        int idx[3][3] = {{0, 0, 0}, {0, 0, 0}, {0, 0, 0}};
        double wt[3][3] = {{1, 0, 0}, {1, 0, 0}, {1, 0, 0}};
        int cnt[3] = {1, 1, 1};
        int a[3] = {0, 0, 0}, comp = 0;
        bool vel;
        if (!decode_local_row(F, row, a, comp, vel)) {
            if (!FILL) cnt_or_rp[row] = 0;
            continue;
        }
        for (int k = 0; k < F.dim; ++k)
            cnt[k] = (vel && F.P == 2) ? interp_q2(a[k], Cg.n[k], idx[k], wt[k]) : interp_q1(a[k], idx[k], wt[k]);
        int64_t p = FILL ? cnt_or_rp[row] : 0;
        int64_t c = 0;
        for (int s2 = 0; s2 < cnt[2]; ++s2)
            for (int s1 = 0; s1 < cnt[1]; ++s1)
                for (int s0 = 0; s0 < cnt[0]; ++s0) {
                    int ac[3] = {idx[0][s0], idx[1][s1], F.dim > 2 ? idx[2][s2] : 0};
                    double w = wt[0][s0] * wt[1][s1];
                    if (F.dim > 2) w *= wt[2][s2];
                    int64_t colid;
                    if (vel) {
                        int64_t fc = free_id(Cg, ac);
                        if (fc < 0) continue;
                        colid = loc_vel(Cg, fc * F.dim + comp);
                    } else {
                        colid = loc_vert(Cg, vert_id(Cg, ac));
                    }
                    if (colid < 0) { atomicOr(err, 1u); continue; }
                    if (FILL) { ci[p + c] = (int32_t)colid; val[p + c] = w; }
                    ++c;
                }
        if (!FILL) cnt_or_rp[row] = c;
    }
}

// ---- scan helper: rp[0] = 0, rp[i+1] = sum cnt[0..i] -------------------------------------------
rav_status counts_to_rowptr(const int64_t* cnt, int64_t* rp, int64_t n, cudaStream_t s) {
    RAV_CUDA(cudaMemsetAsync(rp, 0, sizeof(int64_t), s));
    size_t tmp = 0;
    RAV_CUDA(cub::DeviceScan::InclusiveSum(nullptr, tmp, cnt, rp + 1, n, s));
    void* d_tmp = nullptr;
    RAV_CUDA(cudaMallocAsync(&d_tmp, tmp > 0 ? tmp : 1, s));
    cudaError_t e = cub::DeviceScan::InclusiveSum(d_tmp, tmp, cnt, rp + 1, n, s);
    cudaFreeAsync(d_tmp, s);
    RAV_CUDA(e);
    return RAV_OK;
}

static int grid_for(int64_t n, int bs) {
    int64_t b = cdiv(n, bs);
    int64_t cap = (int64_t)num_sms() * 32;
    return (int)(b < 1 ? 1 : (b > cap ? cap : b));
}

// ---- Q1-Q1 element matrices of arbitrary square cells (adaptive meshes, R20) ----------------------
// cell c: origin (cx[c], cy[c]), side hc[c].  out[c * Q1_CELL_DOUBLES + ...]:
//   A[a][b] (16): int eta grad phi_a . grad phi_b          a, b: corners (x fastest)
//   B[a][k][m] (32): -int psi_m d_k phi_a
//   C[m][m'] (16): -beta h_e^2 int (1/eta) grad psi_m . grad psi_m'     (Eq. 8, R18)
//   F[a][k] (8): int f_k phi_a
__global__ void q1_cell_kernel(Grid G, int64_t ncell, const double* __restrict__ cx, const double* __restrict__ cy,
                               const double* __restrict__ hc, double* __restrict__ out) {
    for (int64_t c = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; c < ncell; c += (int64_t)gridDim.x * blockDim.x) {
        const double h = hc[c], he2 = 2.0 * h * h;
        double A[16] = {0}, B[32] = {0}, Cm[16] = {0}, F[8] = {0};
        for (int q = 0; q < 4; ++q) {
            const double t0 = G.gt[q & 1], t1 = G.gt[q >> 1];
            const double w = G.gw[q & 1] * G.gw[q >> 1] * h * h;
            double x[3] = {cx[c] + t0 * h, cy[c] + t1 * h, 0.0};
            double eta, ge[3], f[3] = {0.0, 0.0, 0.0};
            eta_grad(G, x, eta, ge);
            if (G.kind == 1) mms_force(G, x, f);
            double phi[4], gx[4], gy[4];
            for (int a = 0; a < 4; ++a) {
                const int ax = a & 1, ay = a >> 1;
                phi[a] = q1v(ax, t0) * q1v(ay, t1);
                gx[a] = q1d(ax, t0) / h * q1v(ay, t1);
                gy[a] = q1v(ax, t0) * q1d(ay, t1) / h;
            }
            for (int a = 0; a < 4; ++a) {
                for (int b = 0; b < 4; ++b) {
                    const double dot = gx[a] * gx[b] + gy[a] * gy[b];
                    A[a * 4 + b] += (w * eta) * dot;
                    Cm[a * 4 + b] -= G.beta * he2 * (w / eta) * dot;
                }
                for (int m = 0; m < 4; ++m) {
                    B[(a * 2 + 0) * 4 + m] -= (w * phi[m]) * gx[a];
                    B[(a * 2 + 1) * 4 + m] -= (w * phi[m]) * gy[a];
                }
                F[a * 2 + 0] += (w * f[0]) * phi[a];
                F[a * 2 + 1] += (w * f[1]) * phi[a];
            }
        }
        double* o = out + c * 72;
        for (int i = 0; i < 16; ++i) o[i] = A[i];
        for (int i = 0; i < 32; ++i) o[16 + i] = B[i];
        for (int i = 0; i < 16; ++i) o[48 + i] = Cm[i];
        for (int i = 0; i < 8; ++i) o[64 + i] = F[i];
    }
}

rav_status q1_cell_matrices(const rav_grid* g, int64_t ncell, const double* cx, const double* cy, const double* hc,
                            double* out) {
    RAV_TRY(check_grid(g));
    Grid G = make_grid(g);
    if (G.P != 1 || G.dim != 2) { set_error("q1_cell_matrices: 2D Q1-Q1 only"); return RAV_ERR_ARG; }
    double *d_in = nullptr, *d_out = nullptr;
    RAV_CUDA(cudaMalloc(&d_in, sizeof(double) * 3 * std::max<int64_t>(1, ncell)));
    RAV_CUDA(cudaMalloc(&d_out, sizeof(double) * 72 * std::max<int64_t>(1, ncell)));
    RAV_CUDA(cudaMemcpy(d_in, cx, sizeof(double) * ncell, cudaMemcpyHostToDevice));
    RAV_CUDA(cudaMemcpy(d_in + ncell, cy, sizeof(double) * ncell, cudaMemcpyHostToDevice));
    RAV_CUDA(cudaMemcpy(d_in + 2 * ncell, hc, sizeof(double) * ncell, cudaMemcpyHostToDevice));
    q1_cell_kernel<<<grid_for(std::max<int64_t>(1, ncell), 128), 128>>>(G, ncell, d_in, d_in + ncell, d_in + 2 * ncell,
                                                                        d_out);
    count_launch();
    RAV_CHECK_LAUNCH();
    RAV_CUDA(cudaMemcpy(out, d_out, sizeof(double) * 72 * ncell, cudaMemcpyDeviceToHost));
    cudaFree(d_in);
    cudaFree(d_out);
    return RAV_OK;
}

}  // namespace gen
}  // namespace rav

using namespace rav;
using namespace rav::gen;

extern "C" rav_status rav_gen_sizes(const rav_grid* g, int weights, void* stream, int64_t* n_dofs,
                                    int64_t* n_vel, int64_t* nnz, int64_t* n_patches,
                                    int64_t* patch_entries) {
    RAV_TRY(check_grid(g));
    if (weights < 0 || weights > 2) { set_error("rav_gen_sizes: weights must be 0, 1 or 2"); return RAV_ERR_ARG; }
    Grid G = make_grid(g);
    cudaStream_t s = as_stream(stream);
    if (n_dofs) *n_dofs = G.ndof_loc;
    if (n_vel) *n_vel = G.nvel_loc;
    if (n_patches) *n_patches = G.npatch;
    int64_t *cnt = nullptr, *rp = nullptr;
    int64_t nmax = std::max<int64_t>(1, std::max(G.ndof_loc, G.npatch));
    RAV_CUDA(cudaMallocAsync(&cnt, sizeof(int64_t) * nmax, s));
    RAV_CUDA(cudaMallocAsync(&rp, sizeof(int64_t) * (nmax + 1), s));
    int64_t h_nnz = 0, h_pe = 0;
    if (nnz && G.ndof_loc > 0) {
        op_count_kernel<<<grid_for(G.ndof_loc, 256), 256, 0, s>>>(G, cnt);
        count_launch();
        RAV_CHECK_LAUNCH();
        RAV_TRY(counts_to_rowptr(cnt, rp, G.ndof_loc, s));
        RAV_CUDA(cudaMemcpyAsync(&h_nnz, rp + G.ndof_loc, sizeof(int64_t), cudaMemcpyDeviceToHost, s));
    }
    if (patch_entries && G.npatch > 0) {
        patch_count_kernel<<<grid_for(G.npatch, 256), 256, 0, s>>>(G, cnt);
        count_launch();
        RAV_CHECK_LAUNCH();
        RAV_TRY(counts_to_rowptr(cnt, rp, G.npatch, s));
        RAV_CUDA(cudaMemcpyAsync(&h_pe, rp + G.npatch, sizeof(int64_t), cudaMemcpyDeviceToHost, s));
    }
    cudaFreeAsync(cnt, s);
    cudaFreeAsync(rp, s);
    RAV_CUDA(cudaStreamSynchronize(s));
    if (nnz) *nnz = h_nnz;
    if (patch_entries) *patch_entries = h_pe;
    if (h_nnz > INT32_MAX * 4LL) { set_error("nnz too large"); return RAV_ERR_ARG; }
    if (G.ndof_loc > INT32_MAX) { set_error("n_dofs exceeds int32 column index range"); return RAV_ERR_ARG; }
    return RAV_OK;
}

extern "C" rav_status rav_gen_operator(const rav_grid* g, int64_t* row_ptr, int32_t* col, double* val,
                                       double* rhs, void* stream) {
    RAV_TRY(check_grid(g));
    if (!row_ptr || !col || !val || !rhs) { set_error("rav_gen_operator: NULL buffer"); return RAV_ERR_ARG; }
    Grid G = make_grid(g);
    cudaStream_t s = as_stream(stream);
    const int NG = G.dim == 2 ? G.ngp * G.ngp : G.ngp * G.ngp * G.ngp;
    double *eta_tab = nullptr, *f_tab = nullptr;
    int64_t* cnt = nullptr;
    unsigned int* err = nullptr;
    RAV_CUDA(cudaMallocAsync(&eta_tab, sizeof(double) * G.nel * NG, s));
    if (G.kind == 1) RAV_CUDA(cudaMallocAsync(&f_tab, sizeof(double) * G.nel * NG * 2, s));
    RAV_CUDA(cudaMallocAsync(&cnt, sizeof(int64_t) * std::max<int64_t>(1, G.ndof_loc), s));
    RAV_CUDA(cudaMallocAsync(&err, sizeof(unsigned int), s));
    RAV_CUDA(cudaMemsetAsync(err, 0, sizeof(unsigned int), s));
    coef_kernel<<<grid_for(G.nel * NG, 256), 256, 0, s>>>(G, eta_tab, f_tab);
    count_launch();
    RAV_CHECK_LAUNCH();
    const int P1 = G.P + 1, NL = G.dim == 2 ? P1 * P1 : P1 * P1 * P1;
    const int64_t npair = (int64_t)NL * (NL + 1) / 2;
    double* Ae = nullptr;
    RAV_CUDA(cudaMallocAsync(&Ae, sizeof(double) * std::max<int64_t>(1, G.nel * npair), s));
    elem_a_kernel<<<grid_for(G.nel * npair, 256), 256, 0, s>>>(G, eta_tab, Ae);
    count_launch();
    RAV_CHECK_LAUNCH();
    op_count_kernel<<<grid_for(G.ndof_loc, 256), 256, 0, s>>>(G, cnt);
    count_launch();
    RAV_CHECK_LAUNCH();
    RAV_TRY(counts_to_rowptr(cnt, row_ptr, G.ndof_loc, s));
    op_fill_kernel<<<grid_for(G.ndof_loc, 128), 128, 0, s>>>(G, eta_tab, Ae, f_tab, row_ptr, col, val, rhs, err);
    count_launch();
    RAV_CHECK_LAUNCH();
    unsigned int h_err = 0;
    RAV_CUDA(cudaMemcpyAsync(&h_err, err, sizeof(h_err), cudaMemcpyDeviceToHost, s));
    cudaFreeAsync(Ae, s);
    cudaFreeAsync(eta_tab, s);
    if (f_tab) cudaFreeAsync(f_tab, s);
    cudaFreeAsync(cnt, s);
    cudaFreeAsync(err, s);
    RAV_CUDA(cudaStreamSynchronize(s));
    if (h_err) { set_error("rav_gen_operator: a row of the row window couples outside the DoF window"); return RAV_ERR_ARG; }
    return RAV_OK;
}

extern "C" rav_status rav_gen_patches(const rav_grid* g, int weights, int64_t* offs, int32_t* dofs,
                                      double* w, void* stream) {
    RAV_TRY(check_grid(g));
    if (weights < 0 || weights > 2) { set_error("rav_gen_patches: weights must be 0, 1 or 2"); return RAV_ERR_ARG; }
    if (!offs || !dofs || !w) { set_error("rav_gen_patches: NULL buffer"); return RAV_ERR_ARG; }
    Grid G = make_grid(g);
    cudaStream_t s = as_stream(stream);
    int64_t* cnt = nullptr;
    unsigned int* err = nullptr;
    RAV_CUDA(cudaMallocAsync(&cnt, sizeof(int64_t) * std::max<int64_t>(1, G.npatch), s));
    RAV_CUDA(cudaMallocAsync(&err, sizeof(unsigned int), s));
    RAV_CUDA(cudaMemsetAsync(err, 0, sizeof(unsigned int), s));
    patch_count_kernel<<<grid_for(G.npatch, 256), 256, 0, s>>>(G, cnt);
    count_launch();
    RAV_CHECK_LAUNCH();
    RAV_TRY(counts_to_rowptr(cnt, offs, G.npatch, s));
    patch_fill_kernel<<<grid_for(G.npatch, 128), 128, 0, s>>>(G, weights, offs, dofs, w, err);
    count_launch();
    RAV_CHECK_LAUNCH();
    unsigned int h_err = 0;
    RAV_CUDA(cudaMemcpyAsync(&h_err, err, sizeof(h_err), cudaMemcpyDeviceToHost, s));
    cudaFreeAsync(cnt, s);
    cudaFreeAsync(err, s);
    RAV_CUDA(cudaStreamSynchronize(s));
    if (h_err) { set_error("rav_gen_patches: a patch reaches outside the DoF window"); return RAV_ERR_ARG; }
    return RAV_OK;
}

static rav_status check_nested(const rav_grid* f, const rav_grid* c) {
    RAV_TRY(check_grid(f));
    RAV_TRY(check_grid(c));
    if (f->dim != c->dim) { set_error("prolongation: dim mismatch"); return RAV_ERR_ARG; }
    if ((f->vel_order == 1) != (c->vel_order == 1)) { set_error("prolongation: element pair mismatch"); return RAV_ERR_ARG; }
    for (int k = 0; k < f->dim; ++k)
        if (f->ncell[k] != 2 * c->ncell[k]) { set_error("prolongation: fine ncell must be 2 x coarse"); return RAV_ERR_ARG; }
    return RAV_OK;
}

// count (FILL = false into cnt) or fill the prolongation; err set when a column leaves the coarse window
static rav_status prol_pass(const Grid& F, const Grid& Cg, int64_t* rp_or_cnt, int32_t* ci, double* val, bool fill,
                            cudaStream_t s) {
    unsigned int* err = nullptr;
    RAV_CUDA(cudaMallocAsync(&err, sizeof(unsigned int), s));
    RAV_CUDA(cudaMemsetAsync(err, 0, sizeof(unsigned int), s));
    if (fill) prol_kernel<true><<<grid_for(F.ndof_loc, 256), 256, 0, s>>>(F, Cg, rp_or_cnt, ci, val, err);
    else prol_kernel<false><<<grid_for(F.ndof_loc, 256), 256, 0, s>>>(F, Cg, rp_or_cnt, nullptr, nullptr, err);
    count_launch();
    RAV_CHECK_LAUNCH();
    unsigned int h_err = 0;
    RAV_CUDA(cudaMemcpyAsync(&h_err, err, sizeof(h_err), cudaMemcpyDeviceToHost, s));
    cudaFreeAsync(err, s);
    RAV_CUDA(cudaStreamSynchronize(s));
    if (h_err) { set_error("prolongation: a row of the fine row window interpolates from outside the coarse window"); return RAV_ERR_ARG; }
    return RAV_OK;
}

extern "C" rav_status rav_gen_prolongation_nnz(const rav_grid* fine, const rav_grid* coarse, void* stream,
                                               int64_t* nnz) {
    RAV_TRY(check_nested(fine, coarse));
    if (!nnz) { set_error("rav_gen_prolongation_nnz: NULL nnz"); return RAV_ERR_ARG; }
    Grid F = make_grid(fine), Cg = make_grid(coarse);
    cudaStream_t s = as_stream(stream);
    int64_t *cnt = nullptr, *rp = nullptr;
    const int64_t nr = std::max<int64_t>(1, F.ndof_loc);
    RAV_CUDA(cudaMallocAsync(&cnt, sizeof(int64_t) * nr, s));
    RAV_CUDA(cudaMallocAsync(&rp, sizeof(int64_t) * (nr + 1), s));
    rav_status st = prol_pass(F, Cg, cnt, nullptr, nullptr, false, s);
    int64_t h = 0;
    if (st == RAV_OK && F.ndof_loc > 0) {
        st = counts_to_rowptr(cnt, rp, F.ndof_loc, s);
        if (st == RAV_OK) RAV_CUDA(cudaMemcpyAsync(&h, rp + F.ndof_loc, sizeof(int64_t), cudaMemcpyDeviceToHost, s));
    }
    cudaFreeAsync(cnt, s);
    cudaFreeAsync(rp, s);
    RAV_CUDA(cudaStreamSynchronize(s));
    *nnz = h;
    return st;
}

extern "C" rav_status rav_gen_prolongation(const rav_grid* fine, const rav_grid* coarse, int64_t* rp,
                                           int32_t* ci, double* val, void* stream) {
    RAV_TRY(check_nested(fine, coarse));
    if (!rp) { set_error("rav_gen_prolongation: NULL buffer"); return RAV_ERR_ARG; }
    Grid F = make_grid(fine), Cg = make_grid(coarse);
    cudaStream_t s = as_stream(stream);
    if (F.ndof_loc == 0) { RAV_CUDA(cudaMemsetAsync(rp, 0, sizeof(int64_t), s)); return RAV_OK; }
    int64_t* cnt = nullptr;
    RAV_CUDA(cudaMallocAsync(&cnt, sizeof(int64_t) * F.ndof_loc, s));
    rav_status st = prol_pass(F, Cg, cnt, nullptr, nullptr, false, s);
    if (st == RAV_OK) st = counts_to_rowptr(cnt, rp, F.ndof_loc, s);
    if (st == RAV_OK) st = prol_pass(F, Cg, rp, ci, val, true, s);
    cudaFreeAsync(cnt, s);
    RAV_CUDA(cudaStreamSynchronize(s));
    return st;
}

// 4^d multicolouring of the generated patches (R10): patch of vertex (i, j[, k]) gets colour
// (i mod 4) + 4 (j mod 4) [+ 16 (k mod 4)] by GLOBAL vertex coordinates (a slab window colours its
// patches like the whole grid, so every rank relaxes the same colour at the same time); patches
// ascending inside each colour.  Host outputs in the rav_set_colors layout.
extern "C" rav_status rav_gen_colors(const rav_grid* g, int64_t* color_offs, int32_t* patch_ids) {
    RAV_TRY(check_grid(g));
    if (!color_offs || !patch_ids) { set_error("rav_gen_colors: NULL buffer"); return RAV_ERR_ARG; }
    const Grid G = make_grid(g);
    const int nc = g->dim == 2 ? 16 : 64;
    int64_t nv[3] = {1, 1, 1};
    for (int k = 0; k < g->dim; ++k) nv[k] = (int64_t)G.n[k] + 1;
    std::vector<int> col(G.npatch);
    std::vector<int64_t> cnt(nc + 1, 0);
    for (int64_t q = 0; q < G.npatch; ++q) {
        int64_t v = G.patch_off + q, c = 0, mult = 1;
        for (int k = 0; k < g->dim; ++k) {
            c += (v % nv[k]) % 4 * mult;
            v /= nv[k];
            mult *= 4;
        }
        col[q] = (int)c;
        cnt[c + 1]++;
    }
    for (int c = 0; c < nc; ++c) cnt[c + 1] += cnt[c];
    for (int c = 0; c <= nc; ++c) color_offs[c] = cnt[c];
    for (int64_t q = 0; q < G.npatch; ++q) patch_ids[cnt[col[q]]++] = (int32_t)q;
    return RAV_OK;
}
