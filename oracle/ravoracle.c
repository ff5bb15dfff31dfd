/*
 * ravoracle.c -- the parity ORACLE for the restricted additive Vanka (RAV)
 * multigrid hot path of Saberi, Meschke, Vogel, "A restricted additive Vanka
 * smoother for geometric multigrid" (arXiv 2103.10127; /root/reference/PAPER.md).
 *
 * TEST INFRASTRUCTURE ONLY.  Only tests/, __graft_entry__.smoke() and bench.py's
 * cpu_baseline / --impl reference legs may load this library.  The product path
 * (paper_2103_10127_b200/, include/ravgmg.h) never links, includes or calls it,
 * and this file includes nothing from the product tree.
 *
 * Plain, slow, obviously-correct CPU code.  Every function cites the passage it
 * follows.  Citation convention: "P:n" = PAPER.md line n, "S:n" = SPEC.md line n,
 * "R<k>" = the reading k listed in DESIGN.md / SURVEY.md section 8.
 *
 *   assembly        P:66-74 Eqs. 5-7 (Taylor-Hood Q2-Q1, C = 0: R1; or the paper's
 *                   stabilized Q1-Q1 with C of P:78 Eq. 8: R18), Dirichlet
 *                   condensation S:207 (R8), 3-point Gauss per axis (R7)
 *   patches         P:108 (structural Bt-row support, R2), P:122 (restricted
 *                   prolongation; partition-of-unity weights R3)
 *   local solves    P:114 L_i = R_i L R_i^T; S:254-268 LU with partial pivoting,
 *                   rows of L_i^{-1} by transposed solves
 *   smoothers       P:104 Eq. 10; MV P:112 Eq. 11 + Eq. 15; AV P:118
 *                   Eq. 12; RAV P:124 Eq. 13; diagonal Vanka R17
 *   multigrid       P:84-90 (V-cycle, nested transfers, coarse LU)
 *                   (stopping rule, damping), R4 (pin only in the coarsest LU)
 *
 * Pin status of each function: see oracle/__init__.py and DESIGN.md section 3.
 */
#include <math.h>
#include <stdint.h>
#include <stdlib.h>
#include <string.h>
#ifdef _OPENMP
#include <omp.h>
#endif

#define OR_MAXMODES 8

/* Problem description (mirrors the dict of seeded_inputs.problem). */
typedef struct {
    int32_t dim;           /* 2 or 3 */
    int32_t ncell[3];      /* cells per axis (axis 2 unused when dim == 2) */
    double  len[3];        /* box lengths */
    int32_t kind;          /* 0 cavity lid, 1 manufactured solution (2D), 2 homogeneous */
    int32_t eta_mode;      /* 0 constant eta0, 1 Fourier field (R12) */
    double  eta0;
    int32_t n_modes;
    double  amp[OR_MAXMODES];
    int32_t mode[OR_MAXMODES][3];
    double  phase[OR_MAXMODES][3];
    double  gmin, gmax;
    int32_t vel_order;     /* 2 (or 0): Taylor-Hood Q2-Q1 (R1); 1: stabilized Q1-Q1 (R18) */
    double  beta;          /* Q1-Q1 stabilization constant beta_0 of R18 */
} or_desc;

/* ------------------------------------------------------------------------- */
/* Grid bookkeeping (R9): Q2 nodes on the (2n+1)^d lattice, vertices on the    */
/* (n+1)^d lattice.  Free velocity DoFs = interior nodes, numbered            */
/* lexicographically (x fastest), components interleaved; then all vertices   */
/* (pressure) lexicographically.                                              */
/* ------------------------------------------------------------------------- */

static int axes(const or_desc* D) { return D->dim; }
/* velocity lattice refinement P: velocity nodes on the (P n + 1)^d lattice, vertices = nodes P a */
static int vorder(const or_desc* D) { return D->vel_order == 1 ? 1 : 2; }

int64_t or_n_free_nodes(const or_desc* D) {
    int64_t m = 1;
    for (int k = 0; k < axes(D); ++k) m *= (int64_t)(vorder(D) * D->ncell[k] - 1);
    return m;
}

int64_t or_n_vertices(const or_desc* D) {
    int64_t m = 1;
    for (int k = 0; k < axes(D); ++k) m *= (int64_t)(D->ncell[k] + 1);
    return m;
}

int64_t or_n_velocity(const or_desc* D) { return (int64_t)D->dim * or_n_free_nodes(D); }
int64_t or_n_dofs(const or_desc* D) { return or_n_velocity(D) + or_n_vertices(D); }

/* free-node index of lattice node a, or -1 when a lies on the boundary */
static int64_t free_node(const or_desc* D, const int* a) {
    int64_t idx = 0, stride = 1;
    for (int k = 0; k < axes(D); ++k) {
        int m = vorder(D) * D->ncell[k];
        if (a[k] <= 0 || a[k] >= m) return -1;
        idx += (int64_t)(a[k] - 1) * stride;
        stride *= (int64_t)(m - 1);
    }
    return idx;
}

static int64_t vertex_id(const or_desc* D, const int* v) {
    int64_t idx = 0, stride = 1;
    for (int k = 0; k < axes(D); ++k) {
        idx += (int64_t)v[k] * stride;
        stride *= (int64_t)(D->ncell[k] + 1);
    }
    return idx;
}

static int64_t pdof(const or_desc* D, const int* v) { return or_n_velocity(D) + vertex_id(D, v); }

/* Dirichlet value of velocity component c at boundary node a (R8):
 * cavity lid u = e_x on the top face (y = 1 in 2D, z = 1 in 3D) excluding the
 * face's boundary edges/corners, zero elsewhere; all other kinds: zero. */
static double dirichlet_value(const or_desc* D, const int* a, int c) {
    if (D->kind != 0 || c != 0) return 0.0;
    int top = D->dim - 1;
    if (a[top] != vorder(D) * D->ncell[top]) return 0.0;
    for (int k = 0; k < top; ++k)
        if (a[k] <= 0 || a[k] >= vorder(D) * D->ncell[k]) return 0.0;
    return 1.0;
}

/* ------------------------------------------------------------------------- */
/* Coefficients: viscosity eta(x) (constant or R12 Fourier field) and the     */
/* manufactured forcing f = -div(eta grad u) + grad p of R13 (Eq. 1).   */
/* ------------------------------------------------------------------------- */

static void eta_and_grad(const or_desc* D, const double* x, double* eta, double* geta) {
    for (int k = 0; k < 3; ++k) geta[k] = 0.0;
    if (D->eta_mode == 0) { *eta = D->eta0; return; }
    double g = 0.0, dg[3] = {0, 0, 0};
    for (int m = 0; m < D->n_modes; ++m) {
        double cs[3], sn[3];
        for (int k = 0; k < D->dim; ++k) {
            double arg = M_PI * D->mode[m][k] * x[k] + D->phase[m][k];
            cs[k] = cos(arg);
            sn[k] = sin(arg);
        }
        double prod = D->amp[m];
        for (int k = 0; k < D->dim; ++k) prod *= cs[k];
        g += prod;
        for (int k = 0; k < D->dim; ++k) {
            double t = D->amp[m] * (-M_PI * D->mode[m][k] * sn[k]);
            for (int j = 0; j < D->dim; ++j) if (j != k) t *= cs[j];
            dg[k] += t;
        }
    }
    double scale = log(100.0) / (D->gmax - D->gmin);
    double ge = log(0.1) + (g - D->gmin) * scale;
    *eta = exp(ge);
    for (int k = 0; k < D->dim; ++k) geta[k] = (*eta) * scale * dg[k];
}

/* exact MMS velocity/pressure (R13), 2D */
static void mms_exact(const double* x, double* u, double* p) {
    double sx = sin(M_PI * x[0]), sy = sin(M_PI * x[1]);
    u[0] = M_PI * sx * sx * sin(2 * M_PI * x[1]);
    u[1] = -M_PI * sin(2 * M_PI * x[0]) * sy * sy;
    *p = cos(M_PI * x[0]) * cos(M_PI * x[1]);
}

static void forcing(const or_desc* D, const double* x, double* f) {
    f[0] = f[1] = f[2] = 0.0;
    if (D->kind != 1) return;
    const double pi = M_PI, X = x[0], Y = x[1];
    double eta, ge[3];
    eta_and_grad(D, x, &eta, ge);
    double sx = sin(pi * X), sy = sin(pi * Y);
    double s2x = sin(2 * pi * X), s2y = sin(2 * pi * Y), c2x = cos(2 * pi * X), c2y = cos(2 * pi * Y);
    /* u0 = pi sin^2(pi x) sin(2 pi y) */
    double u0x = pi * pi * s2x * s2y;
    double u0y = 2 * pi * pi * sx * sx * c2y;
    double lap0 = 2 * pi * pi * pi * c2x * s2y - 4 * pi * pi * pi * sx * sx * s2y;
    /* u1 = -pi sin(2 pi x) sin^2(pi y) */
    double u1x = -2 * pi * pi * c2x * sy * sy;
    double u1y = -pi * pi * s2x * s2y;
    double lap1 = 4 * pi * pi * pi * s2x * sy * sy - 2 * pi * pi * pi * s2x * c2y;
    /* p = cos(pi x) cos(pi y) */
    double px = -pi * sin(pi * X) * cos(pi * Y);
    double py = -pi * cos(pi * X) * sin(pi * Y);
    f[0] = -eta * lap0 - (ge[0] * u0x + ge[1] * u0y) + px;
    f[1] = -eta * lap1 - (ge[0] * u1x + ge[1] * u1y) + py;
}

/* ------------------------------------------------------------------------- */
/* Reference element: 1D Q2 Lagrange basis on [0,1] with nodes 0, 1/2, 1;     */
/* Q1 basis 1-t, t; 3-point Gauss rule (R7).                                   */
/* ------------------------------------------------------------------------- */

static double q2(int i, double t) {
    if (i == 0) return 2.0 * (t - 0.5) * (t - 1.0);
    if (i == 1) return 4.0 * t * (1.0 - t);
    return t * (2.0 * t - 1.0);
}
static double dq2(int i, double t) {
    if (i == 0) return 4.0 * t - 3.0;
    if (i == 1) return 4.0 - 8.0 * t;
    return 4.0 * t - 1.0;
}
static double q1(int i, double t) { return i == 0 ? 1.0 - t : t; }
static double dq1(int i, double t) { (void)t; return i == 0 ? -1.0 : 1.0; }
/* velocity basis of order P (2: Q2, 1: Q1) */
static double vb(int P, int i, double t) { return P == 2 ? q2(i, t) : q1(i, t); }
static double dvb(int P, int i, double t) { return P == 2 ? dq2(i, t) : dq1(i, t); }

static const double GAUSS3_T[3] = {0.5 - 0.5 * 0.77459666924148337704, 0.5,
                                   0.5 + 0.5 * 0.77459666924148337704};
static const double GAUSS3_W[3] = {5.0 / 18.0, 8.0 / 18.0, 5.0 / 18.0};
/* 2-point Gauss rule on [0,1] for Q1-Q1 ("2x2 Gauss", R18) */
static const double GAUSS2_T[2] = {0.5 - 0.5 * 0.57735026918962576451, 0.5 + 0.5 * 0.57735026918962576451};
static const double GAUSS2_W[2] = {0.5, 0.5};

static int ipow(int b, int e) { int r = 1; while (e-- > 0) r *= b; return r; }

/* Element matrices of element e (Eq. 7, Eq. 8):
 *   Ae[a][b]     = int eta grad(phi_a) . grad(phi_b)          (per velocity component)
 *   Be[a][c][m]  = - int psi_m d_c phi_a                       (B := -(div v, p))
 *   Ce[m][m']    = - beta_0 h_e^2 int (1/eta) grad psi_m . grad psi_m'   (Q1-Q1 only, R18;
 *                  h_e = element diameter; Eq. 8 read on the pressure basis)
 *   Fe[a][c]     = int f_c phi_a
 * a, b: local velocity nodes ((P+1)^d), m: local vertices (2^d).  Gauss rule with
 * P+1 points per axis (R7 / R18). */
static void element_matrices_at(const or_desc* D, const double* org, const double* hin, double* Ae, double* Be,
                                double* Ce, double* Fe);

static void element_matrices(const or_desc* D, const int* e, double* Ae, double* Be, double* Ce, double* Fe) {
    double h[3] = {1.0, 1.0, 1.0}, org[3] = {0.0, 0.0, 0.0};
    for (int k = 0; k < D->dim; ++k) { h[k] = D->len[k] / D->ncell[k]; org[k] = e[k] * h[k]; }
    element_matrices_at(D, org, h, Ae, Be, Ce, Fe);
}

/* the same element matrices for the cell [org, org + h] (adaptive meshes, R20) */
int or_element_matrices(const or_desc* D, const double* org, const double* h, double* Ae, double* Be, double* Ce,
                        double* Fe) {
    element_matrices_at(D, org, h, Ae, Be, Ce, Fe);
    return 0;
}

static void element_matrices_at(const or_desc* D, const double* org, const double* hin, double* Ae, double* Be,
                                double* Ce, double* Fe) {
    const int d = D->dim, P = vorder(D), NQ = ipow(P + 1, d), NV = ipow(2, d), NP1 = P + 1, NG = ipow(NP1, d);
    const double* GT = P == 2 ? GAUSS3_T : GAUSS2_T;
    const double* GW = P == 2 ? GAUSS3_W : GAUSS2_W;
    double h[3], h2 = 0.0;
    for (int k = 0; k < d; ++k) { h[k] = hin[k]; h2 += h[k] * h[k]; }
    memset(Ae, 0, sizeof(double) * NQ * NQ);
    memset(Be, 0, sizeof(double) * NQ * 3 * NV);
    memset(Ce, 0, sizeof(double) * NV * NV);
    memset(Fe, 0, sizeof(double) * NQ * 3);
    double phi[27], grad[27][3], psi[8], gpsi[8][3];
    for (int q = 0; q < NG; ++q) {
        double t[3], x[3], w = 1.0;
        for (int k = 0; k < d; ++k) {
            int qk = (q / ipow(NP1, k)) % NP1;
            t[k] = GT[qk];
            w *= GW[qk] * h[k];
            x[k] = org[k] + t[k] * h[k];
        }
        double eta, ge[3], f[3];
        eta_and_grad(D, x, &eta, ge);
        forcing(D, x, f);
        for (int a = 0; a < NQ; ++a) {
            int ak[3];
            for (int k = 0; k < d; ++k) ak[k] = (a / ipow(NP1, k)) % NP1;
            double v = 1.0;
            for (int k = 0; k < d; ++k) v *= vb(P, ak[k], t[k]);
            phi[a] = v;
            for (int k = 0; k < d; ++k) {
                double g = dvb(P, ak[k], t[k]) / h[k];
                for (int j = 0; j < d; ++j) if (j != k) g *= vb(P, ak[j], t[j]);
                grad[a][k] = g;
            }
        }
        for (int m = 0; m < NV; ++m) {
            double v = 1.0;
            for (int k = 0; k < d; ++k) v *= q1((m >> k) & 1, t[k]);
            psi[m] = v;
            for (int k = 0; k < d; ++k) {
                double g = dq1((m >> k) & 1, t[k]) / h[k];
                for (int j = 0; j < d; ++j) if (j != k) g *= q1((m >> j) & 1, t[j]);
                gpsi[m][k] = g;
            }
        }
        for (int a = 0; a < NQ; ++a) {
            for (int b = a; b < NQ; ++b) {
                double dot = 0.0;
                for (int k = 0; k < d; ++k) dot += grad[a][k] * grad[b][k];
                Ae[a * NQ + b] += w * eta * dot;
            }
            for (int c = 0; c < d; ++c) {
                for (int m = 0; m < NV; ++m) Be[(a * 3 + c) * NV + m] -= w * psi[m] * grad[a][c];
                Fe[a * 3 + c] += w * f[c] * phi[a];
            }
        }
        if (P == 1)
            for (int m = 0; m < NV; ++m)
                for (int m2 = m; m2 < NV; ++m2) {
                    double dot = 0.0;
                    for (int k = 0; k < d; ++k) dot += gpsi[m][k] * gpsi[m2][k];
                    Ce[m * NV + m2] -= D->beta * h2 * (w / eta) * dot;
                }
    }
    for (int a = 0; a < NQ; ++a)
        for (int b = 0; b < a; ++b) Ae[a * NQ + b] = Ae[b * NQ + a]; /* symmetric by definition */
    for (int m = 0; m < NV; ++m)
        for (int m2 = 0; m2 < m; ++m2) Ce[m * NV + m2] = Ce[m2 * NV + m];
}

/* ------------------------------------------------------------------------- */
/* CSR helpers                                                                */
/* ------------------------------------------------------------------------- */

static int cmp_i64(const void* x, const void* y) {
    int64_t a = *(const int64_t*)x, b = *(const int64_t*)y;
    return (a > b) - (a < b);
}

static int64_t csr_find(const int64_t* rp, const int32_t* ci, int64_t row, int64_t col) {
    int64_t lo = rp[row], hi = rp[row + 1] - 1;
    while (lo <= hi) {
        int64_t mid = (lo + hi) / 2;
        if (ci[mid] == col) return mid;
        if (ci[mid] < col) lo = mid + 1; else hi = mid - 1;
    }
    return -1;
}

/* Row pattern: the DoFs that share an element with the row's node/vertex.
 * Structural (R2): entries are kept even when they evaluate to zero.
 * For a velocity row (node a, component c): same-component velocity DoFs and
 * pressure DoFs of all elements containing a.  For a pressure row (vertex v):
 * all velocity DoFs of all elements containing v, plus (Q1-Q1, C != 0) the
 * pressure DoFs of those elements.  Taylor-Hood: C = 0 => no p-p entries. */
static int64_t row_pattern(const or_desc* D, int64_t row, int64_t* out) {
    const int d = D->dim, P = vorder(D);
    const int64_t nu = or_n_velocity(D);
    int node[3] = {0, 0, 0}, is_vel = row < nu, comp = 0;
    int elo[3] = {0, 0, 0}, ehi[3] = {0, 0, 0};
    if (is_vel) {
        int64_t fi = row / d;
        comp = (int)(row % d);
        for (int k = 0; k < d; ++k) {
            int m = P * D->ncell[k] - 1;
            node[k] = (int)(fi % m) + 1;
            fi /= m;
        }
        for (int k = 0; k < d; ++k) {
            /* elements along axis k containing lattice index node[k] */
            if (P == 1) { elo[k] = node[k] - 1; ehi[k] = node[k]; }
            else if (node[k] % 2 == 0) { elo[k] = node[k] / 2 - 1; ehi[k] = node[k] / 2; }
            else { elo[k] = ehi[k] = (node[k] - 1) / 2; }
            if (elo[k] < 0) elo[k] = 0;
            if (ehi[k] > D->ncell[k] - 1) ehi[k] = D->ncell[k] - 1;
        }
    } else {
        int64_t vi = row - nu;
        int v[3];
        for (int k = 0; k < d; ++k) { v[k] = (int)(vi % (D->ncell[k] + 1)); vi /= (D->ncell[k] + 1); }
        for (int k = 0; k < d; ++k) {
            elo[k] = v[k] - 1 < 0 ? 0 : v[k] - 1;
            ehi[k] = v[k] > D->ncell[k] - 1 ? D->ncell[k] - 1 : v[k];
        }
    }
    int64_t cnt = 0;
    /* nodes of the union of those elements: lattice box [P elo, P ehi + P] */
    int lo[3] = {0, 0, 0}, hi[3] = {0, 0, 0};
    for (int k = 0; k < d; ++k) { lo[k] = P * elo[k]; hi[k] = P * ehi[k] + P; }
    int b[3] = {0, 0, 0};
    int tot = 1;
    for (int k = 0; k < d; ++k) tot *= (hi[k] - lo[k] + 1);
    for (int t = 0; t < tot; ++t) {
        int r = t;
        for (int k = 0; k < d; ++k) { b[k] = lo[k] + r % (hi[k] - lo[k] + 1); r /= (hi[k] - lo[k] + 1); }
        int64_t fb = free_node(D, b);
        if (fb < 0) continue;
        if (is_vel) out[cnt++] = fb * d + comp;
        else for (int c = 0; c < d; ++c) out[cnt++] = fb * d + c;
    }
    if (is_vel || P == 1) {   /* B entries of a velocity row; C entries of a Q1-Q1 pressure row */
        int vt = 1;
        for (int k = 0; k < d; ++k) vt *= (ehi[k] - elo[k] + 2);
        for (int t = 0; t < vt; ++t) {
            int r = t, v[3] = {0, 0, 0};
            for (int k = 0; k < d; ++k) { v[k] = elo[k] + r % (ehi[k] - elo[k] + 2); r /= (ehi[k] - elo[k] + 2); }
            out[cnt++] = pdof(D, v);
        }
    }
    qsort(out, (size_t)cnt, sizeof(int64_t), cmp_i64);
    return cnt;
}

/* Number of stored entries of L (pass 1 of assembly). */
int64_t or_assemble_nnz(const or_desc* D) {
    int64_t n = or_n_dofs(D), nnz = 0;
    int64_t buf[512];
    for (int64_t i = 0; i < n; ++i) nnz += row_pattern(D, i, buf);
    return nnz;
}

/* Assemble L = [A B; B^T 0] and b (Eq. 6, Eq. 7) over the free DoFs,
 * element by element, with Dirichlet condensation (R8):
 *   b_free = F_free - L_{free,D} u_D.
 * Caller allocates rp[n+1], ci[nnz], val[nnz], rhs[n]. */
int or_assemble(const or_desc* D, int64_t* rp, int32_t* ci, double* val, double* rhs) {
    const int d = D->dim, P = vorder(D), NQ = ipow(P + 1, d), NV = ipow(2, d);
    const int64_t n = or_n_dofs(D);
    int64_t buf[512];
    rp[0] = 0;
    for (int64_t i = 0; i < n; ++i) {
        int64_t c = row_pattern(D, i, buf);
        for (int64_t j = 0; j < c; ++j) ci[rp[i] + j] = (int32_t)buf[j];
        rp[i + 1] = rp[i] + c;
    }
    memset(val, 0, sizeof(double) * rp[n]);
    memset(rhs, 0, sizeof(double) * n);
    double* Ae = malloc(sizeof(double) * NQ * NQ);
    double* Be = malloc(sizeof(double) * NQ * 3 * NV);
    double* Ce = malloc(sizeof(double) * NV * NV);
    double* Fe = malloc(sizeof(double) * NQ * 3);
    int64_t nel = 1;
    for (int k = 0; k < d; ++k) nel *= D->ncell[k];
    for (int64_t el = 0; el < nel; ++el) {
        int e[3] = {0, 0, 0};
        int64_t r = el;
        for (int k = 0; k < d; ++k) { e[k] = (int)(r % D->ncell[k]); r /= D->ncell[k]; }
        element_matrices(D, e, Ae, Be, Ce, Fe);
        int64_t gn[27];           /* free-node index of each local node or -1 */
        int an[27][3];
        for (int a = 0; a < NQ; ++a) {
            for (int k = 0; k < 3; ++k) an[a][k] = 0;
            for (int k = 0; k < d; ++k) an[a][k] = P * e[k] + (a / ipow(P + 1, k)) % (P + 1);
            gn[a] = free_node(D, an[a]);
        }
        int64_t gp[8];
        for (int m = 0; m < NV; ++m) {
            int v[3] = {0, 0, 0};
            for (int k = 0; k < d; ++k) v[k] = e[k] + ((m >> k) & 1);
            gp[m] = pdof(D, v);
        }
        for (int a = 0; a < NQ; ++a) {
            for (int c = 0; c < d; ++c) {
                if (gn[a] >= 0) {
                    int64_t row = gn[a] * d + c;
                    rhs[row] += Fe[a * 3 + c];
                    for (int b = 0; b < NQ; ++b) {
                        if (gn[b] >= 0) {
                            int64_t pos = csr_find(rp, ci, row, gn[b] * d + c);
                            val[pos] += Ae[a * NQ + b];
                        } else {
                            rhs[row] -= Ae[a * NQ + b] * dirichlet_value(D, an[b], c);
                        }
                    }
                    for (int m = 0; m < NV; ++m) {
                        int64_t pos = csr_find(rp, ci, row, gp[m]);
                        val[pos] += Be[(a * 3 + c) * NV + m];
                        int64_t pos2 = csr_find(rp, ci, gp[m], row);
                        val[pos2] += Be[(a * 3 + c) * NV + m];
                    }
                } else {
                    double ud = dirichlet_value(D, an[a], c);
                    if (ud != 0.0)
                        for (int m = 0; m < NV; ++m) rhs[gp[m]] -= Be[(a * 3 + c) * NV + m] * ud;
                }
            }
        }
        if (P == 1)   /* stabilization C (Eq. 8) */
            for (int m = 0; m < NV; ++m)
                for (int m2 = 0; m2 < NV; ++m2) val[csr_find(rp, ci, gp[m], gp[m2])] += Ce[m * NV + m2];
    }
    free(Ae); free(Be); free(Ce); free(Fe);
    return 0;
}

/* y = b - L x  (Eq. 10, the residual).  Rows are independent; each row is
 * summed in column order by one thread, so the result does not depend on the
 * thread count. */
void or_residual(int64_t n, const int64_t* rp, const int32_t* ci, const double* val,
                 const double* x, const double* b, double* r) {
#pragma omp parallel for schedule(static, 4096)
    for (int64_t i = 0; i < n; ++i) {
        double s = 0.0;
        for (int64_t k = rp[i]; k < rp[i + 1]; ++k) s += val[k] * x[ci[k]];
        r[i] = b[i] - s;
    }
}

/* y = M x for a general CSR (transfers) */
void or_spmv(int64_t nrows, const int64_t* rp, const int32_t* ci, const double* val,
             const double* x, double* y) {
#pragma omp parallel for schedule(static, 4096)
    for (int64_t i = 0; i < nrows; ++i) {
        double s = 0.0;
        for (int64_t k = rp[i]; k < rp[i + 1]; ++k) s += val[k] * x[ci[k]];
        y[i] = s;
    }
}

/* y = M^T x  (restriction R = P^T), plain scatter in row order */
void or_spmv_t(int64_t nrows, int64_t ncols, const int64_t* rp, const int32_t* ci,
               const double* val, const double* x, double* y) {
    memset(y, 0, sizeof(double) * ncols);
    for (int64_t i = 0; i < nrows; ++i)
        for (int64_t k = rp[i]; k < rp[i + 1]; ++k) y[ci[k]] += val[k] * x[i];
}

/* ------------------------------------------------------------------------- */
/* Vanka patches (R2, R3)                                              */
/* ------------------------------------------------------------------------- */

/* weights_mode: 0 = partition-of-unity psi_v(x_j) (R3), 1 = 0/1 ownership
 * node a -> vertex floor(a/2) (the paper's 0/1 G_i extended), 2 = all ones
 * (full prolongation R^T: additive Vanka, Eq. 12). */
static double patch_weight(int mode, int d, int P, const int* a, const int* v) {
    if (mode == 2) return 1.0;
    double w = 1.0;
    for (int k = 0; k < d; ++k) {
        int off = a[k] - P * v[k];
        if (P == 1) {          /* Q1-Q1: the velocity DoFs on the pressure node */
            if (off != 0) return 0.0;
            continue;
        }
        if (mode == 0) {
            if (off < -1 || off > 1) return 0.0;
            w *= (off == 0) ? 1.0 : 0.5;
        } else {
            if (off != 0 && off != 1) return 0.0;
        }
    }
    return w;
}

/* Patch of vertex v: the free velocity DoFs on the Q2 nodes of all elements
 * touching v (the structural support of row p_v of B^T) plus p_v.
 * Order: restricted DoFs (weight > 0) ascending, then the others ascending. */
static int64_t build_patch(const or_desc* D, int mode, const int* v, int64_t* dofs, double* w) {
    const int d = D->dim, P = vorder(D);
    int lo[3] = {0, 0, 0}, hi[3] = {0, 0, 0};
    for (int k = 0; k < d; ++k) {
        lo[k] = P * v[k] - P < 0 ? 0 : P * v[k] - P;
        hi[k] = P * v[k] + P > P * D->ncell[k] ? P * D->ncell[k] : P * v[k] + P;
    }
    int64_t cnt_r = 0, cnt_o = 0;
    int64_t rd[1200], od[1200];
    double rw[1200];
    int tot = 1;
    for (int k = 0; k < d; ++k) tot *= (hi[k] - lo[k] + 1);
    for (int t = 0; t < tot; ++t) {
        int a[3] = {0, 0, 0}, r = t;
        for (int k = 0; k < d; ++k) { a[k] = lo[k] + r % (hi[k] - lo[k] + 1); r /= (hi[k] - lo[k] + 1); }
        int64_t fa = free_node(D, a);
        if (fa < 0) continue;
        double wt = patch_weight(mode, d, P, a, v);
        for (int c = 0; c < d; ++c) {
            if (wt > 0.0) { rd[cnt_r] = fa * d + c; rw[cnt_r] = wt; cnt_r++; }
            else od[cnt_o++] = fa * d + c;
        }
    }
    /* lexicographic node loop with x fastest already yields ascending DoFs */
    int64_t c = 0;
    for (int64_t i = 0; i < cnt_r; ++i) { dofs[c] = rd[i]; w[c] = rw[i]; c++; }
    dofs[c] = pdof(D, v); w[c] = 1.0; c++;           /* pressure DoF, weight 1 */
    for (int64_t i = 0; i < cnt_o; ++i) { dofs[c] = od[i]; w[c] = 0.0; c++; }
    return c;
}

/* total number of patch entries (pass 1) */
int64_t or_patch_entries(const or_desc* D, int mode) {
    int64_t nv = or_n_vertices(D), tot = 0;
    int64_t dofs[1200];
    double w[1200];
    for (int64_t vi = 0; vi < nv; ++vi) {
        int v[3] = {0, 0, 0};
        int64_t r = vi;
        for (int k = 0; k < D->dim; ++k) { v[k] = (int)(r % (D->ncell[k] + 1)); r /= (D->ncell[k] + 1); }
        tot += build_patch(D, mode, v, dofs, w);
    }
    return tot;
}

/* one patch per vertex, in vertex (= pressure DoF) order */
int or_patches(const or_desc* D, int mode, int64_t* offs, int32_t* dofs, double* w) {
    int64_t nv = or_n_vertices(D);
    int64_t tmpd[1200];
    double tmpw[1200];
    offs[0] = 0;
    for (int64_t vi = 0; vi < nv; ++vi) {
        int v[3] = {0, 0, 0};
        int64_t r = vi;
        for (int k = 0; k < D->dim; ++k) { v[k] = (int)(r % (D->ncell[k] + 1)); r /= (D->ncell[k] + 1); }
        int64_t c = build_patch(D, mode, v, tmpd, tmpw);
        for (int64_t j = 0; j < c; ++j) { dofs[offs[vi] + j] = (int32_t)tmpd[j]; w[offs[vi] + j] = tmpw[j]; }
        offs[vi + 1] = offs[vi] + c;
    }
    return 0;
}

/* ------------------------------------------------------------------------- */
/* Dense LU with partial pivoting: P M = L U, in place, row-major. */
/* Pivot tolerance 1e-14 * ||original row||_inf.                      */
/* ------------------------------------------------------------------------- */

int or_lu_factor(int n, double* M, int32_t* piv) {
    double* rn = malloc(sizeof(double) * (n > 0 ? n : 1));
    for (int i = 0; i < n; ++i) {
        double m = 0.0;
        for (int j = 0; j < n; ++j) if (fabs(M[i * n + j]) > m) m = fabs(M[i * n + j]);
        rn[i] = m;
    }
    for (int k = 0; k < n; ++k) {
        int p = k;
        double best = fabs(M[k * n + k]);
        for (int i = k + 1; i < n; ++i)
            if (fabs(M[i * n + k]) > best) { best = fabs(M[i * n + k]); p = i; }
        piv[k] = p;
        if (p != k) {
            for (int j = 0; j < n; ++j) { double t = M[k * n + j]; M[k * n + j] = M[p * n + j]; M[p * n + j] = t; }
            double t = rn[k]; rn[k] = rn[p]; rn[p] = t;
        }
        if (!(best > 1e-14 * rn[k])) { free(rn); return k + 1; }   /* singular */
        for (int i = k + 1; i < n; ++i) {
            double f = M[i * n + k] / M[k * n + k];
            M[i * n + k] = f;
            for (int j = k + 1; j < n; ++j) M[i * n + j] -= f * M[k * n + j];
        }
    }
    free(rn);
    return 0;
}

/* solve M x = b with the factors (x holds b on entry) */
void or_lu_solve(int n, const double* LU, const int32_t* piv, double* x) {
    for (int k = 0; k < n; ++k) if (piv[k] != k) { double t = x[k]; x[k] = x[piv[k]]; x[piv[k]] = t; }
    for (int i = 0; i < n; ++i) for (int j = 0; j < i; ++j) x[i] -= LU[i * n + j] * x[j];
    for (int i = n - 1; i >= 0; --i) {
        for (int j = i + 1; j < n; ++j) x[i] -= LU[i * n + j] * x[j];
        x[i] /= LU[i * n + i];
    }
}

/* solve M^T x = b (S:254 lu_solve_transposed): M^T = U^T L^T P */
void or_lu_solve_t(int n, const double* LU, const int32_t* piv, double* x) {
    for (int i = 0; i < n; ++i) {              /* U^T z = b */
        for (int j = 0; j < i; ++j) x[i] -= LU[j * n + i] * x[j];
        x[i] /= LU[i * n + i];
    }
    for (int i = n - 1; i >= 0; --i)           /* L^T w = z (unit diagonal) */
        for (int j = i + 1; j < n; ++j) x[i] -= LU[j * n + i] * x[j];
    for (int k = n - 1; k >= 0; --k) if (piv[k] != k) { double t = x[k]; x[k] = x[piv[k]]; x[piv[k]] = t; }
}

/* dense extract L_i = R_i L R_i^T */
static void extract_local(const int64_t* rp, const int32_t* ci, const double* val,
                          int ni, const int32_t* dofs, double* Li) {
    for (int a = 0; a < ni; ++a)
        for (int b = 0; b < ni; ++b) {
            int64_t pos = csr_find(rp, ci, dofs[a], dofs[b]);
            Li[a * ni + b] = pos >= 0 ? val[pos] : 0.0;
        }
}

/* ------------------------------------------------------------------------- */
/* Local factorizations                               */
/*   fmt 0 ROWS : for each restricted local k (weight > 0):                   */
/*                W_i[k][:] = w_k * (row k of L_i^{-1})  via L_i^T y = e_k    */
/*   fmt 1 LU   : LU of L_i (MV: full local solve)                            */
/*   fmt 2 DIAG : LU of L_i with its velocity-velocity block replaced by its  */
/*                diagonal (diagonal Vanka, R17)                              */
/* Storage offsets are computed by the caller: ROWS uses sum nres_i * n_i,    */
/* LU/DIAG use sum n_i^2 (+ n_i pivots).                                      */
/* Returns -1 on success or the id of the first singular patch.               */
/* ------------------------------------------------------------------------- */

int64_t or_factor(int64_t n, int64_t nvel, const int64_t* rp, const int32_t* ci, const double* val,
                  int64_t npatch, const int64_t* poffs, const int32_t* pdofs, const double* pw,
                  int fmt, const int64_t* foffs, double* fac, int32_t* piv_all, const int64_t* pivoffs) {
    int64_t bad = -1;
    (void)n;
#pragma omp parallel for schedule(dynamic, 64)
    for (int64_t i = 0; i < npatch; ++i) {
        int ni = (int)(poffs[i + 1] - poffs[i]);
        const int32_t* dofs = pdofs + poffs[i];
        const double* w = pw + poffs[i];
        double* Li = malloc(sizeof(double) * ni * ni);
        int32_t* piv = malloc(sizeof(int32_t) * ni);
        extract_local(rp, ci, val, ni, dofs, Li);
        if (fmt == 2)
            for (int a = 0; a < ni; ++a)
                for (int b = 0; b < ni; ++b)
                    if (a != b && dofs[a] < nvel && dofs[b] < nvel) Li[a * ni + b] = 0.0;
        int st = or_lu_factor(ni, Li, piv);
        if (st != 0) {
#pragma omp critical
            { if (bad < 0 || i < bad) bad = i; }
        } else if (fmt == 0) {
            double* y = malloc(sizeof(double) * ni);
            int64_t o = foffs[i];
            for (int k = 0; k < ni; ++k) {
                if (!(w[k] > 0.0)) continue;
                for (int j = 0; j < ni; ++j) y[j] = (j == k) ? 1.0 : 0.0;
                or_lu_solve_t(ni, Li, piv, y);       /* y = row k of L_i^{-1} */
                for (int j = 0; j < ni; ++j) fac[o + j] = w[k] * y[j];
                o += ni;
            }
            free(y);
        } else {
            memcpy(fac + foffs[i], Li, sizeof(double) * ni * ni);
            memcpy(piv_all + pivoffs[i], piv, sizeof(int32_t) * ni);
        }
        free(Li); free(piv);
    }
    return bad;
}

/* ------------------------------------------------------------------------- */
/* Smoothers (one application = one sweep; nu sweeps)                        */
/* ------------------------------------------------------------------------- */

/* Additive sweep with precomputed weighted rows (RAV P:124 Eq. 13 with PoU or
 * ownership weights; AV P:118 Eq. 12 with unit weights):
 *   r = b - L x ;  Delta = sum_i R_i^T (W_i R_i r)  (ascending i) ;  x += omega Delta
 * The patch products c_ik = (W_i R_i r)_k are independent (computed in parallel
 * over patches into their own slots, foffs-aligned per restricted row); the sum
 * into Delta runs serially in ascending patch order, so every thread count gives
 * the same bits. */
void or_additive_sweeps(int64_t n, const int64_t* rp, const int32_t* ci, const double* val,
                        int64_t npatch, const int64_t* poffs, const int32_t* pdofs, const double* pw,
                        const int64_t* foffs, const double* fac,
                        double* x, const double* b, double omega, int nu) {
    double* r = malloc(sizeof(double) * n);
    double* delta = malloc(sizeof(double) * n);
    /* slot of restricted row k of patch i: coffs[i] + (its rank among the restricted entries) */
    int64_t* coffs = malloc(sizeof(int64_t) * (npatch + 1));
    coffs[0] = 0;
    for (int64_t i = 0; i < npatch; ++i) {
        int64_t m = 0;
        for (int64_t k = poffs[i]; k < poffs[i + 1]; ++k) m += pw[k] > 0.0;
        coffs[i + 1] = coffs[i] + m;
    }
    double* c = malloc(sizeof(double) * (coffs[npatch] > 0 ? coffs[npatch] : 1));
    for (int s = 0; s < nu; ++s) {
        or_residual(n, rp, ci, val, x, b, r);
#pragma omp parallel for schedule(dynamic, 256)
        for (int64_t i = 0; i < npatch; ++i) {
            int ni = (int)(poffs[i + 1] - poffs[i]);
            const int32_t* dofs = pdofs + poffs[i];
            const double* w = pw + poffs[i];
            const double* row = fac + foffs[i];
            int64_t q = coffs[i];
            for (int k = 0; k < ni; ++k) {
                if (!(w[k] > 0.0)) continue;
                double t = 0.0;
                for (int j = 0; j < ni; ++j) t += row[j] * r[dofs[j]];
                c[q++] = t;
                row += ni;
            }
        }
        memset(delta, 0, sizeof(double) * n);
        for (int64_t i = 0; i < npatch; ++i) {
            int64_t q = coffs[i];
            for (int64_t k = poffs[i]; k < poffs[i + 1]; ++k)
                if (pw[k] > 0.0) delta[pdofs[k]] += c[q++];
        }
        for (int64_t j = 0; j < n; ++j) x[j] += omega * delta[j];
    }
    free(r); free(delta); free(coffs); free(c);
}

/* Additive sweep with full local LU solves (diagonal Vanka, R17; also usable
 * for AV with fmt LU): r = b - L x; Delta = sum_i R_i^T (w_i o L_i^{-1} R_i r).
 * Local solves in parallel into per-patch slots (poffs-aligned), the sum into
 * Delta serially in ascending patch order (thread-count independent bits). */
void or_additive_lu_sweeps(int64_t n, const int64_t* rp, const int32_t* ci, const double* val,
                           int64_t npatch, const int64_t* poffs, const int32_t* pdofs, const double* pw,
                           const int64_t* foffs, const double* fac, const int32_t* piv_all,
                           const int64_t* pivoffs, double* x, const double* b, double omega, int nu) {
    double* r = malloc(sizeof(double) * n);
    double* delta = malloc(sizeof(double) * n);
    double* loc = malloc(sizeof(double) * (poffs[npatch] > 0 ? poffs[npatch] : 1));
    for (int s = 0; s < nu; ++s) {
        or_residual(n, rp, ci, val, x, b, r);
#pragma omp parallel for schedule(dynamic, 256)
        for (int64_t i = 0; i < npatch; ++i) {
            int ni = (int)(poffs[i + 1] - poffs[i]);
            const int32_t* dofs = pdofs + poffs[i];
            double* li = loc + poffs[i];
            for (int j = 0; j < ni; ++j) li[j] = r[dofs[j]];
            or_lu_solve(ni, fac + foffs[i], piv_all + pivoffs[i], li);
        }
        memset(delta, 0, sizeof(double) * n);
        for (int64_t i = 0; i < npatch; ++i)
            for (int64_t k = poffs[i]; k < poffs[i + 1]; ++k) delta[pdofs[k]] += pw[k] * loc[k];
        for (int64_t j = 0; j < n; ++j) x[j] += omega * delta[j];
    }
    free(r); free(delta); free(loc);
}

/* Multiplicative Vanka (Eq. 11) in the given patch order: for each patch,
 * a fresh local residual x_m = b_m - L_{m,k} x_k on the patch rows (P:221
 * Eq. 15), a full local solve, and x += omega R_i^T d. */
void or_mv_sweeps(int64_t n, const int64_t* rp, const int32_t* ci, const double* val,
                  int64_t npatch, const int64_t* poffs, const int32_t* pdofs,
                  const int64_t* foffs, const double* fac, const int32_t* piv_all,
                  const int64_t* pivoffs, const int32_t* order,
                  double* x, const double* b, double omega, int nu) {
    (void)n;
    double* loc = malloc(sizeof(double) * 1200);
    for (int s = 0; s < nu; ++s) {
        for (int64_t t = 0; t < npatch; ++t) {
            int64_t i = order ? order[t] : t;
            int ni = (int)(poffs[i + 1] - poffs[i]);
            const int32_t* dofs = pdofs + poffs[i];
            for (int a = 0; a < ni; ++a) {
                int64_t row = dofs[a];
                double sum = 0.0;
                for (int64_t k = rp[row]; k < rp[row + 1]; ++k) sum += val[k] * x[ci[k]];
                loc[a] = b[row] - sum;
            }
            or_lu_solve(ni, fac + foffs[i], piv_all + pivoffs[i], loc);
            for (int a = 0; a < ni; ++a) x[dofs[a]] += omega * loc[a];
        }
    }
    free(loc);
}

/* ------------------------------------------------------------------------- */
/* Grid transfers: nested interpolation Q2 (velocity) and Q1           */
/* (pressure) from the coarse grid (ncell/2) to the fine grid; Dirichlet rows */
/* and columns dropped.  P: fine free DoFs x coarse free DoFs.  R = P^T.      */
/* ------------------------------------------------------------------------- */

/* 1D Q2 interpolation of coarse lattice nodes onto fine lattice index af:
 * the fine node sits at coarse-lattice position af/2.  Returns the count. */
static int interp_q2_1d(int af, int ncoarse, int* idx, double* wt) {
    if (af % 2 == 0) { idx[0] = af / 2; wt[0] = 1.0; return 1; }
    int e = af / 4;                       /* coarse element containing the node */
    if (e > ncoarse - 1) e = ncoarse - 1;
    double t = (af - 4.0 * e) / 4.0;      /* 1/4 or 3/4 */
    for (int i = 0; i < 3; ++i) { idx[i] = 2 * e + i; wt[i] = q2(i, t); }
    return 3;
}

static int interp_q1_1d(int bf, int* idx, double* wt) {
    if (bf % 2 == 0) { idx[0] = bf / 2; wt[0] = 1.0; return 1; }
    idx[0] = (bf - 1) / 2; wt[0] = 0.5;
    idx[1] = (bf + 1) / 2; wt[1] = 0.5;
    return 2;
}

static int64_t prolong_row(const or_desc* F, const or_desc* C, int64_t row, int64_t* cols, double* vals) {
    const int d = F->dim;
    const int64_t nuf = or_n_velocity(F);
    int idx[3][3];
    double wt[3][3];
    int cnt[3] = {1, 1, 1};
    int comp = -1;
    if (row < nuf) {
        int64_t fi = row / d;
        comp = (int)(row % d);
        for (int k = 0; k < d; ++k) {
            int m = vorder(F) * F->ncell[k] - 1;
            int a = (int)(fi % m) + 1;
            fi /= m;
            cnt[k] = vorder(F) == 2 ? interp_q2_1d(a, C->ncell[k], idx[k], wt[k]) : interp_q1_1d(a, idx[k], wt[k]);
        }
    } else {
        int64_t vi = row - nuf;
        for (int k = 0; k < d; ++k) {
            int b = (int)(vi % (F->ncell[k] + 1));
            vi /= (F->ncell[k] + 1);
            cnt[k] = interp_q1_1d(b, idx[k], wt[k]);
        }
    }
    int64_t c = 0;
    int tot = 1;
    for (int k = 0; k < d; ++k) tot *= cnt[k];
    for (int t = 0; t < tot; ++t) {
        int r = t, a[3] = {0, 0, 0};
        double w = 1.0;
        for (int k = 0; k < d; ++k) { int s = r % cnt[k]; r /= cnt[k]; a[k] = idx[k][s]; w *= wt[k][s]; }
        if (w == 0.0) continue;
        if (comp >= 0) {
            int64_t fc = free_node(C, a);
            if (fc < 0) continue;                  /* coarse Dirichlet column dropped */
            cols[c] = fc * d + comp;
        } else {
            cols[c] = pdof(C, a);
        }
        vals[c] = w;
        c++;
    }
    /* sort by column (insertion sort, tiny rows) */
    for (int64_t i = 1; i < c; ++i) {
        int64_t kc = cols[i]; double kv = vals[i]; int64_t j = i - 1;
        while (j >= 0 && cols[j] > kc) { cols[j + 1] = cols[j]; vals[j + 1] = vals[j]; --j; }
        cols[j + 1] = kc; vals[j + 1] = kv;
    }
    return c;
}

int64_t or_prolongation_nnz(const or_desc* F, const or_desc* C) {
    int64_t n = or_n_dofs(F), nnz = 0;
    int64_t cols[64];
    double vals[64];
    for (int64_t i = 0; i < n; ++i) nnz += prolong_row(F, C, i, cols, vals);
    return nnz;
}

int or_prolongation(const or_desc* F, const or_desc* C, int64_t* rp, int32_t* ci, double* val) {
    int64_t n = or_n_dofs(F);
    int64_t cols[64];
    double vals[64];
    rp[0] = 0;
    for (int64_t i = 0; i < n; ++i) {
        int64_t c = prolong_row(F, C, i, cols, vals);
        for (int64_t j = 0; j < c; ++j) { ci[rp[i] + j] = (int32_t)cols[j]; val[rp[i] + j] = vals[j]; }
        rp[i + 1] = rp[i] + c;
    }
    return 0;
}

/* ------------------------------------------------------------------------- */
/* Multigrid (R4, R11)                            */
/* ------------------------------------------------------------------------- */

typedef struct {
    int64_t n, nvel;
    const int64_t* rp; const int32_t* ci; const double* val;          /* L_l */
    int64_t npatch;
    const int64_t* poffs; const int32_t* pdofs; const double* pw;     /* patches */
    const int64_t* foffs; const double* fac;                          /* rows or LU */
    const int32_t* piv; const int64_t* pivoffs;
    const int32_t* order;                                             /* MV order */
    const int64_t* prp; const int32_t* pci; const double* pval;       /* P: level l-1 -> l */
    int64_t nc;                                                       /* columns of P */
} or_level;

typedef struct {
    int64_t n;          /* coarsest system size */
    int64_t pin;        /* pinned DoF (removed from the LU), -1 for none */
    const double* lu;   /* (n-1)^2 or n^2 */
    const int32_t* piv;
} or_coarse;

/* Factor the dense coarsest matrix with the pressure pin (R4: the pin lives
 * only here).  A is n x n dense row-major; out lu (m x m, m = n - (pin>=0)). */
int or_coarse_factor(int64_t n, const double* A, int64_t pin, double* lu, int32_t* piv) {
    int m = (int)(pin >= 0 ? n - 1 : n);
    int ii = 0;
    for (int64_t i = 0; i < n; ++i) {
        if (i == pin) continue;
        int jj = 0;
        for (int64_t j = 0; j < n; ++j) {
            if (j == pin) continue;
            lu[ii * m + jj] = A[i * n + j];
            jj++;
        }
        ii++;
    }
    return or_lu_factor(m, lu, piv);
}

void or_coarse_solve(const or_coarse* C, const double* rhs, double* x) {
    int m = (int)(C->pin >= 0 ? C->n - 1 : C->n);
    double* t = malloc(sizeof(double) * (m > 0 ? m : 1));
    int ii = 0;
    for (int64_t i = 0; i < C->n; ++i) if (i != C->pin) t[ii++] = rhs[i];
    or_lu_solve(m, C->lu, C->piv, t);
    ii = 0;
    for (int64_t i = 0; i < C->n; ++i) x[i] = (i == C->pin) ? 0.0 : t[ii++];
    free(t);
}

/* smoother: 0 additive rows (RAV / AV), 1 multiplicative (MV), 2 additive LU (diag Vanka) */
static void smooth(const or_level* L, int smoother, double* x, const double* b, double omega, int nu) {
    if (nu <= 0) return;
    if (smoother == 0)
        or_additive_sweeps(L->n, L->rp, L->ci, L->val, L->npatch, L->poffs, L->pdofs, L->pw,
                           L->foffs, L->fac, x, b, omega, nu);
    else if (smoother == 1)
        or_mv_sweeps(L->n, L->rp, L->ci, L->val, L->npatch, L->poffs, L->pdofs, L->foffs, L->fac,
                     L->piv, L->pivoffs, L->order, x, b, omega, nu);
    else
        or_additive_lu_sweeps(L->n, L->rp, L->ci, L->val, L->npatch, L->poffs, L->pdofs, L->pw,
                              L->foffs, L->fac, L->piv, L->pivoffs, x, b, omega, nu);
}

/* One V-cycle on level l (0 = coarsest) (Fig. 1):
 * pre-smooth, restrict the residual, recurse from a zero guess (or the coarse
 * LU at level 0), prolongate and add, post-smooth. */
void or_vcycle(const or_level* levels, const or_coarse* C, int l, int smoother,
               double* x, const double* b, int pre, int post, double omega) {
    if (l == 0) { or_coarse_solve(C, b, x); return; }
    const or_level* L = &levels[l];
    const or_level* Lc = &levels[l - 1];
    smooth(L, smoother, x, b, omega, pre);
    double* r = malloc(sizeof(double) * L->n);
    double* rc = malloc(sizeof(double) * Lc->n);
    double* ec = calloc((size_t)Lc->n, sizeof(double));
    double* ef = malloc(sizeof(double) * L->n);
    or_residual(L->n, L->rp, L->ci, L->val, x, b, r);
    or_spmv_t(L->n, Lc->n, L->prp, L->pci, L->pval, r, rc);
    or_vcycle(levels, C, l - 1, smoother, ec, rc, pre, post, omega);
    or_spmv(L->n, L->prp, L->pci, L->pval, ec, ef);
    for (int64_t i = 0; i < L->n; ++i) x[i] += ef[i];
    smooth(L, smoother, x, b, omega, post);
    free(r); free(rc); free(ec); free(ef);
}

static double norm2(int64_t n, const double* v) {
    double s = 0.0;
    for (int64_t i = 0; i < n; ++i) s += v[i] * v[i];
    return sqrt(s);
}

/* GMG as a stand-alone fixed-point iteration: V-cycles
 * until ||b - L x_k||_2 <= rtol ||b - L x_0||_2 or maxit.  hist[0..k] holds
 * the residual norms.  Returns k. */
int or_mg_solve(const or_level* levels, const or_coarse* C, int nlev, int smoother,
                double* x, const double* b, int pre, int post, double omega,
                double rtol, int maxit, double* hist) {
    const or_level* L = &levels[nlev - 1];
    double* r = malloc(sizeof(double) * L->n);
    or_residual(L->n, L->rp, L->ci, L->val, x, b, r);
    double r0 = norm2(L->n, r);
    hist[0] = r0;
    int k = 0;
    if (r0 == 0.0) { free(r); return 0; }
    while (k < maxit) {
        or_vcycle(levels, C, nlev - 1, smoother, x, b, pre, post, omega);
        or_residual(L->n, L->rp, L->ci, L->val, x, b, r);
        double rk = norm2(L->n, r);
        k++;
        hist[k] = rk;
        if (!(rk == rk)) break;          /* NaN: diverged */
        if (rk <= rtol * r0) break;
    }
    free(r);
    return k;
}

/* ------------------------------------------------------------------------- */
/* Sampled RAV sweep for full-size parity (one sweep): x_new at sampled DoFs  */
/* computed one by one.  mask[j] != 0 marks sampled DoFs; only patches whose  */
/* restricted set meets the sample are factorized (Eq. 13).             */
/* ------------------------------------------------------------------------- */

int64_t or_rav_sweep_sampled(int64_t n, const int64_t* rp, const int32_t* ci, const double* val,
                             int64_t npatch, const int64_t* poffs, const int32_t* pdofs, const double* pw,
                             const double* x, const double* b, double omega, const uint8_t* mask,
                             double* xnew /* length n; only sampled entries written */,
                             double* mag /* NULL or length n: rounding scale at sampled entries */) {
    /* mag[j] = |x_j| + omega sum over patches |w_k (L_i^{-T} e_k)_a| (|b_a| + sum |L_a.| |x| + |r_a|):
     * the magnitude of the terms that make up x_new[j] (a scale for element-wise parity bounds,
     * not part of the method) */
    double* delta = calloc((size_t)n, sizeof(double));
    double* dmag = mag ? calloc((size_t)n, sizeof(double)) : NULL;
    int64_t bad = -1;
    for (int64_t i = 0; i < npatch; ++i) {
        int ni = (int)(poffs[i + 1] - poffs[i]);
        const int32_t* dofs = pdofs + poffs[i];
        const double* w = pw + poffs[i];
        int hit = 0;
        for (int k = 0; k < ni; ++k) if (w[k] > 0.0 && mask[dofs[k]]) hit = 1;
        if (!hit) continue;
        double* Li = malloc(sizeof(double) * ni * ni);
        int32_t* piv = malloc(sizeof(int32_t) * ni);
        double* ri = malloc(sizeof(double) * ni);
        double* ra = malloc(sizeof(double) * ni);
        double* y = malloc(sizeof(double) * ni);
        extract_local(rp, ci, val, ni, dofs, Li);
        if (or_lu_factor(ni, Li, piv) != 0) { if (bad < 0) bad = i; }
        else {
            for (int a = 0; a < ni; ++a) {
                int64_t row = dofs[a];
                double s = 0.0, sa = 0.0;
                for (int64_t k = rp[row]; k < rp[row + 1]; ++k) {
                    s += val[k] * x[ci[k]];
                    sa += fabs(val[k] * x[ci[k]]);
                }
                ri[a] = b[row] - s;
                ra[a] = fabs(b[row]) + sa + fabs(ri[a]);
            }
            for (int k = 0; k < ni; ++k) {
                if (!(w[k] > 0.0) || !mask[dofs[k]]) continue;
                for (int j = 0; j < ni; ++j) y[j] = (j == k) ? 1.0 : 0.0;
                or_lu_solve_t(ni, Li, piv, y);
                double c = 0.0, ca = 0.0;
                for (int j = 0; j < ni; ++j) {
                    c += w[k] * y[j] * ri[j];
                    ca += fabs(w[k] * y[j]) * ra[j];
                }
                delta[dofs[k]] += c;
                if (dmag) dmag[dofs[k]] += ca;
            }
        }
        free(Li); free(piv); free(ri); free(ra); free(y);
    }
    for (int64_t j = 0; j < n; ++j)
        if (mask[j]) {
            xnew[j] = x[j] + omega * delta[j];
            if (mag) mag[j] = fabs(x[j]) + omega * dmag[j];
        }
    free(delta);
    free(dmag);
    return bad;
}

/* ------------------------------------------------------------------------- */
/* Discretization error against the manufactured solution (R13): L2 norms of  */
/* u - u_h and (p_h - mean p_h) - p (mean of p over the box is 0), 4-point    */
/* Gauss per axis.  2D only.                                                 */
/* ------------------------------------------------------------------------- */

void or_mms_errors(const or_desc* D, const double* xsol, double* err_u, double* err_p) {
    static const double G4T[4] = {-0.86113631159405257522, -0.33998104358485626480,
                                  0.33998104358485626480, 0.86113631159405257522};
    static const double G4W[4] = {0.34785484513745385737, 0.65214515486254614263,
                                  0.65214515486254614263, 0.34785484513745385737};
    double h0 = D->len[0] / D->ncell[0], h1 = D->len[1] / D->ncell[1];
    double area = D->len[0] * D->len[1];
    double pint = 0.0;
    /* pass 1: mean of p_h */
    for (int e1 = 0; e1 < D->ncell[1]; ++e1)
        for (int e0 = 0; e0 < D->ncell[0]; ++e0)
            for (int q1i = 0; q1i < 4; ++q1i)
                for (int q0i = 0; q0i < 4; ++q0i) {
                    double t0 = 0.5 * (1 + G4T[q0i]), t1 = 0.5 * (1 + G4T[q1i]);
                    double w = 0.25 * G4W[q0i] * G4W[q1i] * h0 * h1;
                    double ph = 0.0;
                    for (int m = 0; m < 4; ++m) {
                        int v[3] = {e0 + (m & 1), e1 + ((m >> 1) & 1), 0};
                        ph += q1(m & 1, t0) * q1((m >> 1) & 1, t1) * xsol[pdof(D, v)];
                    }
                    pint += w * ph;
                }
    double pmean = pint / area;
    double eu = 0.0, ep = 0.0;
    for (int e1 = 0; e1 < D->ncell[1]; ++e1)
        for (int e0 = 0; e0 < D->ncell[0]; ++e0)
            for (int q1i = 0; q1i < 4; ++q1i)
                for (int q0i = 0; q0i < 4; ++q0i) {
                    double t0 = 0.5 * (1 + G4T[q0i]), t1 = 0.5 * (1 + G4T[q1i]);
                    double w = 0.25 * G4W[q0i] * G4W[q1i] * h0 * h1;
                    double x[3] = {(e0 + t0) * h0, (e1 + t1) * h1, 0.0};
                    double uh[2] = {0, 0}, ph = 0.0;
                    const int P = vorder(D), NP1 = P + 1;
                    for (int a = 0; a < NP1 * NP1; ++a) {
                        int an[3] = {P * e0 + a % NP1, P * e1 + a / NP1, 0};
                        double phi = vb(P, a % NP1, t0) * vb(P, a / NP1, t1);
                        int64_t fn = free_node(D, an);
                        for (int c = 0; c < 2; ++c)
                            uh[c] += phi * (fn >= 0 ? xsol[fn * 2 + c] : dirichlet_value(D, an, c));
                    }
                    for (int m = 0; m < 4; ++m) {
                        int v[3] = {e0 + (m & 1), e1 + ((m >> 1) & 1), 0};
                        ph += q1(m & 1, t0) * q1((m >> 1) & 1, t1) * xsol[pdof(D, v)];
                    }
                    double ue[2], pe;
                    mms_exact(x, ue, &pe);
                    eu += w * ((uh[0] - ue[0]) * (uh[0] - ue[0]) + (uh[1] - ue[1]) * (uh[1] - ue[1]));
                    ep += w * (ph - pmean - pe) * (ph - pmean - pe);
                }
    *err_u = sqrt(eu);
    *err_p = sqrt(ep);
}

/* viscosity at a point (test hook) */
double or_eta(const or_desc* D, double x, double y, double z) {
    double p[3] = {x, y, z}, e, g[3];
    eta_and_grad(D, p, &e, g);
    return e;
}

void or_set_num_threads(int t) {
#ifdef _OPENMP
    if (t > 0) omp_set_num_threads(t);
#else
    (void)t;
#endif
}

int or_num_threads(void) {
#ifdef _OPENMP
    return omp_get_max_threads();
#else
    return 1;
#endif
}
