/*
 * ravgmg.h -- C-ABI of the B200-native restricted additive Vanka (RAV)
 * geometric-multigrid hot path (Saberi, Meschke, Vogel, arXiv 2103.10127).
 *
 * Citations: "P:n" = /root/reference/PAPER.md line n (section / equation named),
 * "S:n" = SPEC.md line n, "R<k>" = reading k of DESIGN.md section 2.
 *
 * Conventions (all entry points):
 *  - Plain C types only; every function is extern "C" and never throws.
 *  - Every call returns rav_status; on failure rav_last_error() returns a
 *    thread-local, human-readable message (valid until the next failing call
 *    on the same thread).
 *  - Floating point is IEEE binary64 throughout.  Indices: int32 column/DoF
 *    indices, int64 row pointers / offsets.
 *  - "device" pointers are CUDA global-memory pointers on the current device
 *    (e.g. torch tensor data_ptr()); "host" pointers are ordinary CPU memory.
 *    Functions that accept either detect the kind with cudaPointerGetAttributes.
 *  - stream: a cudaStream_t passed as void* (NULL = legacy default stream).
 *    Work is stream-ordered; functions that return sizes or status from the
 *    device synchronize the stream before returning.
 *  - Ownership: buffers passed in are caller-owned.  rav_setup / mg_setup COPY
 *    what they need into library-owned device memory, so callers may free
 *    their inputs afterwards.  Contexts are released with rav_destroy /
 *    mg_destroy.
 */
#ifndef RAVGMG_H
#define RAVGMG_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef enum {
    RAV_OK = 0,
    RAV_ERR_ARG = 1,              /* invalid argument (sizes, NULL, empty patch S:302) */
    RAV_ERR_SINGULAR_LOCAL = 2,   /* a local system L_i is singular */
    RAV_ERR_SINGULAR_COARSE = 3,  /* the pinned coarsest system is singular */
    RAV_ERR_OOM = 4,              /* device allocation failed */
    RAV_ERR_CUDA = 5,             /* a CUDA runtime error */
    RAV_ERR_COMM = 6,             /* multi-rank exchange error */
    RAV_ERR_DIVERGED = 7          /* NaN/Inf residual during mg_solve */
} rav_status;

/* ------------------------------------------------------------------------- */
/* Structured Q2-Q1 problem generator      */
/* ------------------------------------------------------------------------- */

/* Uniform grid of ncell[0] x ncell[1] (x ncell[2]) cells on the box
 * [0,len0] x [0,len1] (x [0,len2]), Taylor-Hood Q2-Q1 (R1).
 * kind: 0 lid-driven cavity (u = e_x on the top face interior, no-slip
 *         elsewhere, f = 0, R8),
 *       1 manufactured solution u = curl(sin^2 pi x sin^2 pi y),
 *         p = cos pi x cos pi y (2D only, R13), homogeneous Dirichlet,
 *       2 homogeneous (f = 0, u = 0 on the boundary).
 * eta_mode: 0 constant eta0; 1 eta = exp(ln 0.1 + (g - gmin)/(gmax - gmin) ln 100),
 *         g(x) = sum_k amp[k] prod_d cos(pi mode[k][d] x_d + phase[k][d]) (R12).
 * DoF numbering (R9): free Q2 nodes lexicographic (x fastest), velocity
 * components interleaved (dof = dim * node + c); then all vertices
 * lexicographic (pressure).  Dirichlet DoFs are eliminated. */
typedef struct {
    int32_t dim;
    int32_t ncell[3];
    double  len[3];
    int32_t kind;
    int32_t eta_mode;
    double  eta0;
    int32_t n_modes;            /* <= 8 */
    double  amp[8];
    int32_t mode[8][3];
    double  phase[8][3];
    double  gmin, gmax;
    /* Slab window along the LAST axis (multi-GPU, SURVEY section 8 row e).  win = 0:
     * the whole grid.  win = 1: the level is generated for one rank.  Ranges are
     * inclusive, in global lattice indices of the last axis (Q2 node layers run
     * 0..2n, vertex layers 0..n).  Local DoFs = free nodes with last index in
     * [node_lo, node_hi] (a contiguous range of the global velocity numbering,
     * same order) followed by vertices in [vert_lo, vert_hi]; rows are assembled
     * only for nodes in [rnode_lo, rnode_hi] and vertices in [rvert_lo,
     * rvert_hi] (other rows are empty, b = 0); patches exist for the vertices in
     * [pvert_lo, pvert_hi].  Columns must fall inside the window (else
     * RAV_ERR_ARG).  Transfers: see rav_gen_prolongation. */
    int32_t win;
    int32_t node_lo, node_hi, vert_lo, vert_hi;
    int32_t rnode_lo, rnode_hi, rvert_lo, rvert_hi;
    int32_t pvert_lo, pvert_hi;
    /* Element pair: vel_order 2 (or 0) = Taylor-Hood Q2-Q1, C = 0 (R1; the BASELINE
     * configs); 1 = the paper's stabilized equal-order Q1-Q1: velocity on
     * the vertices, C = -beta sum_e h_e^2 ((1/eta) grad q, grad p)_e (Eq. 8 read
     * on the pressure basis with beta(x) = beta / eta(x), h_e = element diameter:
     * reading R18), 2-point Gauss rule per axis.  beta > 0 is required for Q1-Q1.
     * Q1-Q1 levels support the whole-grid generator and transfers (win = 0). */
    int32_t vel_order;
    double  beta;
} rav_grid;

/* Sizes of the generated level: n_dofs = n_vel + n_pres; nnz of L; number of
 * patches (= vertices) and total patch entries for the given weights mode
 * (0 partition of unity R3, 1 0/1 ownership, 2 all ones = additive Vanka).
 * Runs counting kernels on `stream` and synchronizes it. */
rav_status rav_gen_sizes(const rav_grid* g, int weights, void* stream,
                         int64_t* n_dofs, int64_t* n_vel, int64_t* nnz,
                         int64_t* n_patches, int64_t* patch_entries);

/* Assemble L = [A B; B^T 0] (Eq. 6, Eq. 7; C = 0 for Taylor-Hood)
 * in CSR with sorted columns and the right-hand side b (Eq. 5 with the
 * Dirichlet lift b_free = F_free - L_{free,D} u_D).  3-point Gauss
 * rule per axis (R7).  The pattern is STRUCTURAL (R2): entries that evaluate
 * to 0 are stored.  Device buffers, caller-allocated: row_ptr[n_dofs+1],
 * col[nnz], val[nnz], rhs[n_dofs]. */
rav_status rav_gen_operator(const rav_grid* g, int64_t* row_ptr, int32_t* col, double* val,
                            double* rhs, void* stream);

/* Vanka patches: one per vertex v (in vertex order), holding every
 * free velocity DoF on the Q2 nodes of the elements touching v plus p_v.
 * Per patch the restricted DoFs (weight > 0, P:122 / R3) come first in
 * ascending order, then the others ascending.  Device buffers:
 * offs[n_patches+1], dofs[patch_entries], w[patch_entries]. */
rav_status rav_gen_patches(const rav_grid* g, int weights, int64_t* offs, int32_t* dofs,
                           double* w, void* stream);

/* Nested prolongation P from `coarse` (ncell/2) to `fine`: Q2
 * interpolation for velocity, Q1 for pressure, Dirichlet rows/columns
 * dropped.  Rows = fine DoFs, columns = coarse DoFs, sorted.  nnz first
 * (synchronizes), then fill device buffers rp[n_fine+1], ci[nnz], val[nnz].
 * Windows (multi-rank cycles): rows are the LOCAL DoFs of the fine grid's
 * window, and only rows inside its row window [rnode_lo, rnode_hi] /
 * [rvert_lo, rvert_hi] are filled (the others are empty) -- a rank passes its
 * OWNED layers there.  Columns are LOCAL DoFs of the coarse grid's window
 * (global ids when coarse->win = 0); a row interpolating from outside the
 * coarse window is RAV_ERR_ARG.  n_fine = the fine window's n_dofs. */
rav_status rav_gen_prolongation_nnz(const rav_grid* fine, const rav_grid* coarse, void* stream,
                                    int64_t* nnz);
rav_status rav_gen_prolongation(const rav_grid* fine, const rav_grid* coarse, int64_t* rp,
                                int32_t* ci, double* val, void* stream);

/* Multicolouring of the generated patches for RAV_VARIANT_MV (Eq. 11; reading
 * R10): the patch of vertex (i, j[, k]) gets colour (i mod 4) + 4 (j mod 4)
 * [+ 16 (k mod 4)] from its GLOBAL vertex coordinates (a slab window colours its
 * patches as the whole grid does); patches ascending inside each colour.  Same-colour
 * patches are >= 4 vertices apart, so they share no DoF and are not coupled through L.
 * Host outputs in the rav_set_colors layout: color_offs[4^dim + 1] and
 * patch_ids[n_patches] (local patch ids of the window).  Integer host work, no stream. */
rav_status rav_gen_colors(const rav_grid* g, int64_t* color_offs, int32_t* patch_ids);

/* ------------------------------------------------------------------------- */
/* Adaptive quadtree hierarchies with hanging nodes */
/* ------------------------------------------------------------------------- */

/* The paper's grid hierarchies (Table 1; reading R20): base is the
 * problem on an n0 x n0 coarse grid of the unit square (ncell[0] = ncell[1] = n0,
 * len = 1, 2D, stabilized Q1-Q1: vel_order 1, beta > 0, win = 0).  Level 0 (the
 * coarsest) is that grid; level k+1 splits every leaf of level k closer to the
 * boundary than bands[k] cells of the current finest size (bands[k] <= 0: the R20
 * default (2, 3, 5, 8, 13, 19), which reproduces Table 1), then restores 2:1 edge
 * balance.  uniform = 1 splits every leaf instead (the structured grids).  Hanging
 * vertices (edge midpoints of coarser neighbours) are constrained to the mean of the
 * edge's end points and eliminated.  Numbering: non-hanging vertices by
 * (y, x); velocity DoFs 2 * free_vertex + c, then one pressure DoF per non-hanging
 * vertex.  Per level: the operator (CSR, sorted columns, structural pattern), the
 * right-hand side, the Vanka patches (restricted = velocity on the pressure node,
 * P:122; order: restricted, p, others) and for levels >= 1 the prolongation from
 * level - 1.  The mesh logic runs on the host at creation (setup); the
 * element matrices on the device.  Outputs go to caller buffers, host or device. */
typedef struct {
    rav_grid base;
    int32_t n_levels;           /* >= 1 */
    int32_t bands[16];          /* per refinement step, in finest cells (<= 0: default) */
    int32_t uniform;
} rav_adaptive_desc;

typedef struct rav_adaptive rav_adaptive;
rav_status rav_adaptive_create(const rav_adaptive_desc* desc, rav_adaptive** out);
rav_status rav_adaptive_sizes(const rav_adaptive* a, int level, int64_t* n_dofs, int64_t* n_vel, int64_t* nnz,
                              int64_t* n_patches, int64_t* patch_entries, int64_t* prol_nnz, int64_t* n_cells);
/* rp[n+1], ci[nnz], val[nnz], rhs[n], poffs[n_patches+1], pdofs/pw[patch_entries],
 * prp[n+1], pci/pval[prol_nnz] (prolongation ignored on level 0); NULL skips a buffer. */
rav_status rav_adaptive_fill(const rav_adaptive* a, int level, int64_t* rp, int32_t* ci, double* val, double* rhs,
                             int64_t* poffs, int32_t* pdofs, double* pw, int64_t* prp, int32_t* pci, double* pval);
void rav_adaptive_destroy(rav_adaptive* a);

/* ------------------------------------------------------------------------- */
/* Smoother: RAV (Eq. 13) and its additive relatives                    */
/* ------------------------------------------------------------------------- */

/* A sparse matrix in CSR.  Columns sorted ascending within each row.  Setup calls
 * validate it (row_ptr[0] = 0 and non-decreasing, 0 <= col < n_cols, strictly
 * increasing columns per row) and return RAV_ERR_ARG otherwise. */
typedef struct {
    int64_t n_rows, n_cols;
    const int64_t* row_ptr;     /* n_rows + 1 */
    const int32_t* col;         /* row_ptr[n_rows] */
    const double*  val;
    int32_t on_device;          /* 1: device pointers, 0: host pointers */
} rav_csr;

/* Subdomains S_{x,Omega_sd,i}: patch i holds dofs[offs[i]..offs[i+1]).
 * weight[j] > 0 marks a DoF of the restricted prolongation R~_i with
 * its partition-of-unity weight (R3); restricted DoFs need not be listed
 * first (setup reorders internally).  weight == 1 on every entry gives the
 * additive Vanka operator of Eq. 12. */
typedef struct {
    int64_t n_patches;
    const int64_t* offs;        /* n_patches + 1 */
    const int32_t* dofs;
    const double*  weight;
    int32_t on_device;
} rav_patches;

enum {
    RAV_VARIANT_ROWS = 0,       /* additive: RAV (Eq. 13) / AV (Eq. 12) from the weights */
    RAV_VARIANT_DIAG = 1,       /* diagonal Vanka: A_i replaced by diag(A_i) (R17); closed form
                                   when block_dim > 0 and the patch structure allows it */
    RAV_VARIANT_MV = 2          /* multiplicative Vanka (Eq. 11) in colours (R10): per colour
                                   all patches relax concurrently with a fresh local residual
                                   (Eq. 15) and full prolongation R_i^T; needs block_dim > 0,
                                   the Schur structure and rav_set_colors.  Same-colour patches
                                   must share no DoF and not be coupled through L (the caller's
                                   colouring guarantees it; then the result equals sequential MV
                                   in colour-major order). */
};

enum {
    RAV_KERNEL_AUTO = 0,        /* RAV_KERNEL_SCHUR when block_dim > 0 and every patch has the Schur
                                   structure; otherwise RAV_KERNEL_SYM when the patch shape allows,
                                   else WARP */
    RAV_KERNEL_WARP = 1,        /* general warp-per-patch kernel (any n_i, nres_i), rows row-major */
    RAV_KERNEL_THREAD = 2,      /* thread-per-patch kernel, full weighted rows (nres <= 32, n <= 64) */
    RAV_KERNEL_SYM = 3,         /* thread-per-patch kernel storing the symmetric restricted block of
                                   L_i^{-1} once (upper triangle) + weights: 17% fewer bytes in 2D */
    RAV_KERNEL_SCHUR = 4        /* factored rows (needs block_dim > 0): every patch must hold one
                                   pressure DoF p and complete velocity nodes, with velocity block
                                   I_d (x) A_s (no cross-component coupling) and symmetric B; then
                                   L_i^{-1} = [I(x)A_s^{-1} + g S^{-1} g^T, -g S^{-1}; -S^{-1} g^T,
                                   S^{-1}] (g = A_s^{-1} b, S = L_pp - b^T g) and only the restricted
                                   rows of A_s^{-1}, g and 1/S are stored (2D: 4x fewer bytes than
                                   rows; 3D: 8x).  AUTO tries it first when block_dim > 0 and falls
                                   back to SYM / WARP when any patch lacks the structure. */
};

typedef struct {
    int32_t variant;            /* RAV_VARIANT_* */
    int32_t kernel;             /* RAV_KERNEL_* */
    int32_t deterministic;      /* 1: run-to-run bitwise reproducible scatter (R16): the sweep writes
                                   every correction to its own slot and a second kernel adds them
                                   to x per DoF in ascending patch order (no atomics).  Schur formats
                                   only (RAV_ERR_ARG otherwise); MV is deterministic by construction.
                                   0: corrections are added with floating-point reductions in
                                   arrival order; the 2D thread sweep first sums, inside a warp, the
                                   corrections of x-neighbouring patches to a shared node (DESIGN 5.1,
                                   RAV_SCHUR_PA): Eq. 13's sum in another order, equal to the
                                   oracle's to rounding, not run-to-run bitwise */
    int64_t n_vel;              /* DoFs < n_vel are velocity (needed by DIAG and SCHUR) */
    void*   stream;             /* cudaStream_t */
    int32_t block_dim;          /* velocity components interleaved as dof = block_dim * node + c
                                   (enables RAV_KERNEL_SCHUR); 0 = unknown */
} rav_opts;

typedef struct rav_ctx rav_ctx;

/* Build the smoother for L x = b: for every patch gather
 * L_i = R_i L R_i^T from the CSR and store what the sweep needs of L_i^{-1}
 * (P:225-227).  Default for Vanka-shaped patches (block_dim > 0, see
 * RAV_KERNEL_SCHUR): the exact block form -- A_s is eliminated per patch and the
 * restricted rows of A_s^{-1}, g = A_s^{-1} b and 1/S are stored.  Other
 * patches: Gaussian elimination with partial pivoting on L_i^T (pivot tolerance
 * 1e-14 * ||row||_inf) and the restricted rows
 * W_i = diag(w_i) L_i^{-1}[restricted, :].
 * On RAV_ERR_SINGULAR_LOCAL, *bad_patch (if non-NULL) holds the smallest
 * failing patch id.  Empty patches are RAV_ERR_ARG. */
rav_status rav_setup(const rav_csr* A, const rav_patches* P, const rav_opts* opts,
                     rav_ctx** out, int64_t* bad_patch);

/* nu sweeps of x <- x + omega * sum_i R~_i^T L_i^{-1} R_i (b - L x)
 * (Eq. 10 with S_RAV of P:124 Eq. 13, scalar damping omega, R5).
 * x (in/out) and b are length n_rows, both device or both host pointers;
 * host buffers are staged through library-owned device buffers (the copies
 * are part of the call).  Stream-ordered on the context stream. */
rav_status rav_smooth(rav_ctx* ctx, double* x, const double* b, int nu, double omega);

/* rav_smooth on nprob independent problems held in HOST buffers: problem k
 * runs nu sweeps on x[k] (in/out, n_rows doubles) with right-hand side b[k]
 * (b[k] may repeat a pointer).  The library stages them through two device
 * buffer pairs and a copy stream of its own, so the host->device copy of
 * problem k+1 and the device->host copy of problem k-1 overlap the sweeps of
 * problem k (pinned host memory makes the copies asynchronous; pageable
 * memory still works, without the overlap).  Each problem's result equals
 * rav_smooth on it (to the atomic scatter's rounding order; bitwise in
 * deterministic mode).  Needs a context stream (rav_opts.stream).  Returns
 * when every x[k] holds its result.  Errors: RAV_ERR_ARG for NULL / device
 * pointers or no stream; RAV_ERR_CUDA. */
rav_status rav_smooth_batch(rav_ctx* ctx, int64_t nprob, double* const* x, const double* const* b, int nu,
                            double omega);

/* x += omega * sum_i R~_i^T W_i R_i r for a given residual r (device
 * pointers): one application of the smoother operator S_RAV of P:124 Eq. 13
 * to r, i.e. the sweep kernel alone (used to time it in isolation). */
rav_status rav_apply(rav_ctx* ctx, const double* r, double* x, double omega);

/* r = b - L x (device pointers).  The residual SpMV of P:104 Eq. 10.  With
 * block_dim > 0 and a Taylor-Hood structure, rav_setup keeps a node-blocked
 * copy of L (A once per node, stencil-compressed columns, the B / B^T values
 * -- which carry no viscosity -- from a verified table when they repeat).  With
 * one lane per row (2D fine levels) each row is summed in the CSR row's order,
 * so r equals the CSR residual up to FMA contraction; several lanes per row (3D,
 * coarse levels) sum interleaved partial sums (rounding-level differences).
 * Falls back to a SELL copy of the CSR otherwise. */
rav_status rav_residual(rav_ctx* ctx, const double* x, const double* b, double* r);

/* Export the stored factor rows in the canonical layout (for parity tests):
 * for patch i, rows k of its restricted DoFs (in the patch's own order of
 * the restricted entries), each of length n_i, concatenated; plus per-entry
 * DoF lists.  Sizes via rav_rows_size.  Device output buffers. */
rav_status rav_rows_size(const rav_ctx* ctx, int64_t* total);
rav_status rav_export_rows(const rav_ctx* ctx, double* rows);

/* Algorithmic roofline bytes of one application (SURVEY section 8 row d):
 * bytes_sweep = the bytes the stored format must move: Schur formats (default)
 * the factored rows (restricted rows of A_s^{-1}, g, weights, 1/S) + node
 * indices as counted at setup; RAV_KERNEL_SYM the symmetric restricted block
 * once + one weight per restricted row; other kernels 8 sum nres_i n_i + 4
 * sum n_i (patch DoF lists); plus r read, x read + write.  bytes_residual =
 * the node-blocked copy's bytes (values, pattern ids / bases or columns) +
 * its row permutation and slice headers + x, b, r (24 n) when it exists,
 * else the CSR's 12 nnz + 8 (n+1) + 24 n.  flops = 2 sum nres_i n_i + 2 nnz. */
rav_status rav_sweep_bytes(const rav_ctx* ctx, double* bytes_sweep, double* bytes_residual,
                           double* flops);

/* Colouring for RAV_VARIANT_MV (host arrays): colour c holds patches
 * patch_ids[color_offs[c] .. color_offs[c+1]) and colours run in order c = 0,
 * 1, ...; patch_ids must be a permutation of 0..n_patches-1.  Copied. */
rav_status rav_set_colors(rav_ctx* ctx, int n_colors, const int64_t* color_offs, const int32_t* patch_ids);

/* One colour of multiplicative Vanka (RAV_VARIANT_MV after rav_set_colors): every
 * patch of colour `color` relaxes concurrently with a fresh local residual
 * (Eq. 15) and x += omega L_i^{-1} r_i on all its DoFs (Eq. 11).  Device
 * pointers.  rav_smooth runs all colours in order; this entry point lets a
 * multi-rank driver exchange interface values between colours. */
rav_status rav_apply_color(rav_ctx* ctx, int color, double* x, const double* b, double omega);

/* Greedy multicolouring of arbitrary patches for RAV_VARIANT_MV (R10 / R20):
 * patches i and j conflict when j holds a DoF of patch i or a DoF coupled to it
 * through L; patches are coloured in ascending order with the smallest free colour,
 * so same-colour patches may relax concurrently and the colour-major sweep is a
 * sequential MV sweep.  A, P: host or device.  Outputs (host): *n_colors,
 * color_offs[n_patches + 1] (capacity; n_colors + 1 used), patch_ids[n_patches]
 * (colour-major, ascending inside a colour) -- the rav_set_colors layout. */
rav_status rav_color_patches(const rav_csr* A, const rav_patches* P, int64_t* n_colors, int64_t* color_offs,
                             int32_t* patch_ids);

/* Name of the sweep kernel / factor format chosen by rav_setup (static string). */
const char* rav_kernel_name(const rav_ctx* ctx);

rav_status rav_set_stream(rav_ctx* ctx, void* stream);
void rav_destroy(rav_ctx* ctx);

/* ------------------------------------------------------------------------- */
/* Geometric multigrid                                   */
/* ------------------------------------------------------------------------- */

typedef struct mg_ctx mg_ctx;

/* Levels are ordered coarsest first: A[0] is the coarsest operator, A[L-1]
 * the finest.  P[l] (l >= 1) is the nested prolongation from level l-1 to
 * level l (rows = DoFs of level l); P[0] and patches[0] are ignored.  The
 * coarsest system is solved by a dense LU with partial pivoting in
 * which DoF `coarse_pin` is removed and set to 0 (R4: the pressure null
 * space is fixed only here; coarse_pin < 0 disables the pin).  Smoothers on
 * levels 1..L-1 are built with rav_setup(opts). */
rav_status mg_setup(int n_levels, const rav_csr* A, const rav_patches* patches, const rav_csr* P,
                    const int64_t* n_vel /* per level (DoFs < n_vel[l] are velocity), NULL =
                                            opts->n_vel on every level */,
                    int64_t coarse_pin, const rav_opts* opts, mg_ctx** out,
                    int* bad_level, int64_t* bad_patch);

/* One V-cycle (Fig. 1): pre smoothing steps, restriction of the
 * residual (R = P^T), recursive coarse correction from a zero guess, coarse
 * LU at level 0, prolongation and addition, post smoothing steps.  x, b:
 * device pointers on the finest level. */
rav_status mg_vcycle(mg_ctx* ctx, double* x, const double* b, int pre, int post, double omega);

/* Stand-alone multigrid iteration: V-cycles until
 * ||b - L x_k||_2 <= rtol ||b - L x_0||_2 or maxit (R11).  *iters = k;
 * hist (host, maxit + 1 doubles, may be NULL) receives ||r_0||..||r_k||.
 * x, b: device or host pointers (host buffers are staged).  Returns
 * RAV_ERR_DIVERGED on a NaN/Inf residual; non-convergence is RAV_OK with
 * *iters == maxit. */
rav_status mg_solve(mg_ctx* ctx, double* x, const double* b, int pre, int post, double omega,
                    double rtol, int maxit, int* iters, double* hist);

/* Flexible GMRES(restart) on the finest level, right-preconditioned by one
 * V-cycle from a zero guess ("the geometric multigrid method can
 * also be used as a preconditioner in a Krylov subspace solver"; reading R19).
 * Arnoldi with classical Gram-Schmidt and one reorthogonalisation pass, Givens
 * rotations on the host.  A restart cycle ends when the least-squares residual
 * estimate <= rtol ||b - L x_0||_2, after `restart` steps, or after maxit
 * Arnoldi steps (= preconditioner applications); x is then updated and the TRUE
 * residual ||b - L x||_2 is computed: the solve stops only when it meets rtol
 * (else it restarts).  *iters = steps taken; hist (host, maxit + 1, may be NULL)
 * = ||r_0||, the estimate after every step, with the entry of each cycle's last
 * step replaced by the true residual (so hist[*iters] is always ||b - L x||).  x (in/out), b: DEVICE pointers.
 * Work space (restart + 1 + restart vectors of n_fine doubles) is allocated on
 * the first call and kept in the context.  RAV_ERR_DIVERGED on NaN/Inf. */
rav_status mg_fgmres(mg_ctx* ctx, double* x, const double* b, int pre, int post, double omega, int restart,
                     double rtol, int maxit, int* iters, double* hist);

/* ------------------------------------------------------------------------- */
/* Exchange helpers for the slab-partitioned sweep (SURVEY section 8 row e)    */
/* ------------------------------------------------------------------------- */
/* Device pointers, stream-ordered.  op: 0 gather  dst[k] = src[idx[k]]
 *                                       1 scatter dst[idx[k]] = src[k]
 *                                       2 scatter-add dst[idx[k]] += src[k]
 *                                         (indices unique within one call)
 *                                       3 fill dst[idx[k]] = value (src unused)
 *                                       4 gather-difference dst[k] = src[idx[k]] - dst[k] */
rav_status rav_index_op(int op, const double* src, const int32_t* idx, int64_t n, double* dst, double value,
                        void* stream);

/* Transfer operator of a host-driven (multi-rank) cycle (SURVEY section
 * 8 rows a7 / e): rav_xfer_setup copies P (rav_csr, host or device, n_rows =
 * fine DoFs, n_cols = coarse DoFs) and builds R = P^T on the device.
 * rav_prolong: xf += alpha P xc.  rav_restrict: bc = P^T rf (bc overwritten).
 * Device pointers, stream-ordered on the transfer's stream. */
typedef struct rav_xfer rav_xfer;
rav_status rav_xfer_setup(const rav_csr* P, void* stream, rav_xfer** out);
rav_status rav_prolong(rav_xfer* t, const double* xc, double* xf, double alpha);
rav_status rav_restrict(rav_xfer* t, const double* rf, double* bc);
rav_status rav_xfer_set_stream(rav_xfer* t, void* stream);
/* Switch the transfer to its stencil form (P:88 -- the nested interpolation of
 * a uniformly refined tensor-product grid: Q2 1D weights 1 / (3/8, 3/4, -1/8),
 * Q1 weights 1 / (1/2, 1/2), Dirichlet nodes dropped; R = P^T): the kernels
 * read the input and write the output vector, no matrix.  fine / coarse: the
 * rav_grid descriptors of the two levels (fine ncell = 2 coarse ncell, same
 * element pair; slab windows as in rav_gen_prolongation).  Before switching, both forms are applied to
 * seeded vectors and must agree to 1e-13 relative; otherwise RAV_ERR_ARG and
 * the CSR form stays.  In 3D only the prolongation switches (the 125-point
 * restriction gather measured slower than the CSR P^T).  Synchronizes the
 * transfer's stream. */
rav_status rav_xfer_set_structured(rav_xfer* t, const rav_grid* fine, const rav_grid* coarse);
void rav_xfer_destroy(rav_xfer* t);

/* *out = sum_{i<n} a[i] b[i] (accumulate = 1: *out += ...), device pointers,
 * fixed reduction order (bitwise reproducible).  Used for the residual norm
 * of the stopping test (R11) over a rank's owned DoFs. */
rav_status rav_dot(const double* a, const double* b, int64_t n, double* out, int accumulate, void* stream);


/* ------------------------------------------------------------------------- */
/* Slab-partitioned (multi-GPU) smoother and V-cycle in the library           */
/* (SURVEY section 8 rows a11 / b / e; within a sweep every       */
/* patch is independent, so RAV shards by patches with one interface exchange  */
/* per sweep)                                                                  */
/* ------------------------------------------------------------------------- */
/* The finest levels are cut into subdomains (slabs of patches); global
 * subdomain ids are 0 .. n_sub_total-1 and subdomain g lives on process
 * sub_proc[g].  A process drives one or more subdomains (n_local >= 1) on its
 * current device: one per GPU in production; several on one GPU to emulate a
 * multi-GPU run with one process (the exchanges between subdomains of the same
 * process are then plain device reads of the neighbour's buffers -- no kernel
 * ever waits on another).  Per sweep on a partitioned level, for every local
 * subdomain: r = b - L x on its rows; x := 0 on its ghost-written DoFs; the RAV
 * sweep of its patches (Eq. 13); then (1) the partial corrections on
 * ghost-written DoFs go to their owners, which add them (interface-correction
 * sum), (2) the owners' values refresh every ghost copy (halo refresh).  The
 * V-cycle restricts / prolongs with each subdomain's windowed
 * transfer, sums coarse partials at the owners, and below the partitioned
 * levels runs an agglomerated multigrid context (mg_setup, identical on every
 * process) on the sum of all subdomains' restricted residuals.  Collectives
 * between processes are NCCL point-to-point sends / receives and all-gathers
 * on the context stream (loaded at run time from the process's libnccl.so.2);
 * sums over subdomains run in ascending subdomain order, so every process sees
 * bitwise-identical coarse right-hand sides and norms, and a run emulated on one
 * GPU reproduces the multi-GPU bits.  Everything a cycle launches (NCCL
 * included) is captured once as a CUDA graph per argument set. */

typedef struct rav_comm rav_comm;

/* A new NCCL unique id (process 0 calls it; the caller broadcasts the 128
 * bytes to the other processes, e.g. with torch.distributed). */
rav_status rav_comm_unique_id(unsigned char id[128]);

/* Communicator of process `proc` of `nprocs` on the current device.  nccl_id =
 * NULL: no NCCL (only valid for nprocs = 1; every subdomain is local).  With an
 * id, ncclCommInitRank(nprocs, id, proc) -- collective over the processes; with
 * nprocs = 1 this gives a one-rank communicator whose self sends / receives can
 * carry the local exchanges (mgd_setup flag via_comm) to verify the NCCL path on
 * one GPU.  RAV_ERR_COMM when libnccl.so.2 cannot be loaded or NCCL fails. */
rav_status rav_comm_create(int nprocs, int proc, const unsigned char* nccl_id, rav_comm** out);
void rav_comm_destroy(rav_comm* c);

/* One neighbour of a subdomain on one level (host arrays of LOCAL DoF ids of
 * the subdomain's window, order agreed with the neighbour's lists):
 * corr_send  ghost-written DoFs owned by `peer` whose partial corrections go to it;
 * corr_recv  owned DoFs receiving `peer`'s partial corrections (same order as its corr_send);
 * halo_send  owned DoFs `peer` holds as ghosts (its halo_recv, same order);
 * halo_recv  ghost DoFs owned by `peer`, refreshed from its halo_send. */
typedef struct {
    int32_t peer;                       /* global subdomain id */
    int64_t n_corr_send, n_corr_recv, n_halo_send, n_halo_recv;
    const int32_t* corr_send;
    const int32_t* corr_recv;
    const int32_t* halo_send;
    const int32_t* halo_recv;
} rav_neighbor;

/* One subdomain's share of one partitioned level (copied at setup). */
typedef struct {
    rav_csr A;                          /* the subdomain's window of the level operator (rows assembled
                                           for the DoFs its patches read) */
    rav_patches P;                      /* its patches (only they write corrections) */
    int64_t n_vel;                      /* window DoFs < n_vel are velocity */
    int32_t n_neighbors;
    const rav_neighbor* neighbors;
    int64_t n_ghost_written;            /* ghost DoFs its patches write (zeroed before each sweep) */
    const int32_t* ghost_written;
    int64_t owned[4];                   /* owned DoFs: [owned[0], owned[1]) and [owned[2], owned[3]) */
    rav_csr P_coarse;                   /* prolongation from the next level: rows = this window's DoFs
                                           (owned rows filled), columns = the next partitioned level's
                                           window of the same subdomain, or -- on the last partitioned
                                           level -- the agglomerated level's global DoFs */
    int32_t n_colors;                   /* RAV_VARIANT_MV: colouring of the patches (rav_set_colors */
    const int64_t* color_offs;          /*   layout; the same colour index on every subdomain) */
    const int32_t* color_ids;
    /* Optional (NULL = the CSR P_coarse is applied): the rav_grid descriptors P_coarse was generated
     * from -- this level's window with its row window on the OWNED layers (as passed to
     * rav_gen_prolongation) and the next partitioned level's window, or the agglomerated level's
     * whole grid.  With both, mgd_setup switches the transfer to its stencil form (rav_xfer_set_
     * structured's contract, slab windows included: the prolongation fills the owned rows only,
     * the restriction gathers from them) after checking it against P_coarse on seeded vectors
     * (1e-13); a mismatch keeps the CSR form. */
    const rav_grid* grid_fine;
    const rav_grid* grid_coarse;
} rav_subdomain;

typedef struct mgd_ctx mgd_ctx;

/* Build the partitioned hierarchy: subs[k * n_local + i] = local subdomain i
 * (global id local_ids[i], ascending) on partitioned level k = 0 (finest) ..
 * n_levels-1.  coarse: the agglomerated hierarchy below (mg_setup on the whole
 * grids; caller-owned, must outlive the context; its stream is set to
 * opts->stream), or NULL for smoothing only (mgd_smooth).  Transport (via_comm):
 * 0 = messages to other processes through NCCL, between local subdomains the
 * receiver reads the sender's packed buffer; 1 = every message through NCCL
 * (the local ones by self sends: verification on one GPU); 2 = the peer-memory
 * transport: the pack kernel stores each message straight into the consumer's
 * receive buffer (CUDA IPC mapping of the other process's block over NVLink, a
 * plain pointer for a local subdomain) and releases the consumer's flag; the
 * consumer's unpack kernel acquires it and releases the producer's ack; no
 * NCCL call on the data path (NCCL only carries the setup's handle exchange
 * and the per-cycle coarse-rhs / norm all-gathers between processes).  Waits
 * are bounded (~4 s): a timeout is reported as RAV_ERR_COMM by the next
 * mgd_solve / mgd_residual_norm.  RAV / AV / diagonal Vanka only (MV: RAV_ERR_ARG).
 * Every message size is checked against the peer's list (RAV_ERR_ARG on a
 * mismatch).  opts as for rav_setup. */
rav_status mgd_setup(rav_comm* comm, int n_sub_total, const int32_t* sub_proc, int n_local,
                     const int32_t* local_ids, int n_levels, const rav_subdomain* subs, mg_ctx* coarse,
                     const rav_opts* opts, int via_comm, mgd_ctx** out);

/* nu slab-partitioned sweeps on the finest partitioned level: x[i], b[i] are
 * device vectors of local subdomain i's window (x in/out; ghost copies are
 * current on return).  RAV / AV / diagonal Vanka: one interface-correction sum
 * and one halo refresh per sweep; RAV_VARIANT_MV: per colour (Eq. 11). */
rav_status mgd_smooth(mgd_ctx* ctx, double* const* x, const double* const* b, int nu, double omega);

/* One distributed V-cycle (x in/out, ghosts current on return). */
rav_status mgd_vcycle(mgd_ctx* ctx, double* const* x, const double* const* b, int pre, int post, double omega);

/* V-cycles until ||b - L x_k|| <= rtol ||b - L x_0|| over the OWNED DoFs of all
 * subdomains (R11) or maxit; *iters, hist (host, maxit + 1) as in mg_solve.
 * Host work per cycle: one graph launch and one 8-byte read of the norm. */
rav_status mgd_solve(mgd_ctx* ctx, double* const* x, const double* const* b, int pre, int post, double omega,
                     double rtol, int maxit, int* iters, double* hist);

/* ||b - L x||_2 over the owned DoFs of all subdomains (host result, synchronizes). */
rav_status mgd_residual_norm(mgd_ctx* ctx, double* const* x, const double* const* b, double* norm);

/* Kernel launches (graph nodes) of the last mgd_* call. */
int64_t mgd_last_launches(const mgd_ctx* ctx);
/* Host time of the last mgd_solve: seconds spent enqueueing the cycles (graph launches,
 * the first call's capture included) and waiting for each cycle's norm, and the cycle count. */
rav_status mgd_host_time(const mgd_ctx* ctx, double* enqueue_s, double* wait_s, int* cycles);
rav_status mgd_set_stream(mgd_ctx* ctx, void* stream);
void mgd_destroy(mgd_ctx* ctx);

/* Colouring of the smoother on level `level` (1 .. n_levels-1) for
 * RAV_VARIANT_MV (same contract as rav_set_colors). */
rav_status mg_set_colors(mg_ctx* ctx, int level, int n_colors, const int64_t* color_offs,
                         const int32_t* patch_ids);

/* Stencil-form transfers for every level (see rav_xfer_set_structured):
 * grids[0 .. n_levels-1] are the levels' rav_grid descriptors, coarsest first,
 * each the uniform refinement of the one before.  Every level is verified
 * against its CSR P before any is switched; on RAV_ERR_ARG nothing changes.
 * Synchronizes the context's stream. */
rav_status mg_set_structured_transfers(mg_ctx* ctx, const rav_grid* grids);

/* Number of GPU kernel launches issued by the most recent rav_smooth,
 * mg_vcycle or mg_solve call on this context (graph nodes included). */
int64_t rav_last_launches(const rav_ctx* ctx);

/* Pressure normalisation (reading R4).  The
 * pressure of the enclosed-flow Stokes system is defined only up to a constant: the
 * operators keep every pressure DoF and the constant is fixed only inside the
 * coarsest solve (mg_setup coarse_pin), so the fine-level pressure of an iterate
 * carries whatever constant the cycles leave.  This call fixes it after a solve:
 * mode 0: p <- p - p[pin] (config c1's "pressure pinned at one corner vertex": with the
 *         generator's numbering (R9) pin = n_vel is vertex 0, the corner (0, 0[, 0]));
 * mode 1: p <- p - mean(p) (arithmetic mean of the n - n_vel pressure DoFs, summed in
 *         a fixed order: bitwise reproducible).
 * x: device pointer of length n, DoFs [n_vel, n) are pressure.  Stream-ordered.
 * RAV_ERR_ARG for n_vel > n, mode not 0/1, pin outside [n_vel, n) in mode 0. */
rav_status rav_pressure_normalize(double* x, int64_t n_vel, int64_t n, int mode, int64_t pin, void* stream);
int64_t mg_last_launches(const mg_ctx* ctx);
/* Algorithmic HBM bytes of one V(pre, post) cycle of mg_solve (the roofline of the V-cycle
 * metric): per smoothed level, (pre + post) sweeps of the sweep kernel and one residual launch per
 * sweep (below the finest level the first sweep's residual is b itself) + the restriction's
 * residual on the finest level, each at rav_sweep_bytes' figures; the transfers' vector traffic
 * (stencil form) or CSR bytes; the coarse solve's explicit inverse. */
rav_status mg_cycle_bytes(const mg_ctx* ctx, int pre, int post, double* bytes);
/* rav_pressure_normalize on the finest level of the hierarchy (its n_vel from
 * mg_setup; mode 0 pins the first pressure DoF, i.e. vertex 0 in the generator's
 * numbering).  x: device pointer, stream-ordered on the context stream. */
rav_status mg_normalize_pressure(mg_ctx* ctx, double* x, int mode);
rav_status mg_set_stream(mg_ctx* ctx, void* stream);
void mg_destroy(mg_ctx* ctx);

/* Thread-local message of the last failure on this thread ("" if none). */
const char* rav_last_error(void);

/* Library version string. */
const char* rav_version(void);

#ifdef __cplusplus
}
#endif
#endif /* RAVGMG_H */
