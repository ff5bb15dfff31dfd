// internal.cuh -- launchers shared between the translation units of libravgmg.
#pragma once
#include "common.cuh"

namespace rav {

namespace gen {
rav_status counts_to_rowptr(const int64_t* cnt, int64_t* rp, int64_t n, cudaStream_t s);
// Q1-Q1 element matrices (A 16, B 32, C 16, F 8 doubles per cell, see gen.cu) of square cells
// (host arrays in and out; runs on the device) -- the adaptive generator's assembly input
rav_status q1_cell_matrices(const rav_grid* g, int64_t ncell, const double* cx, const double* cy, const double* hc,
                            double* out);
}

// ---- linalg.cu ------------------------------------------------------------------------
// SELL-32-sigma copy of a square operator for the residual kernel (sell.cu):
// rows sorted by length (descending) inside windows of SIGMA rows, slices of
// 32 rows stored column-major (entry k of slot l at sptr[s] + 32 k + l), padded
// with (col = row, val = 0) to the slice's longest row.
struct Sell {
    int64_t nslices = 0;
    int64_t* sptr = nullptr;   // nslices + 1
    int32_t* col = nullptr;
    double* val = nullptr;
    int32_t* perm = nullptr;   // slot -> row
    int64_t stored = 0;        // sptr[nslices] (padded entries)
};

// node-blocked copy (nb.cu) for operators whose velocity block is I_d (x) A_s
struct NodeBlocked {
    int D = 0;
    int64_t nnodes = 0, nblock = 0, nslices = 0, nvel = 0;
    int32_t* perm = nullptr;   // slot -> block row (node rows first, then pressure rows)
    int32_t *wa = nullptr, *wb = nullptr;
    int64_t *cptr = nullptr, *vptr = nullptr;
    int32_t* col = nullptr;
    double* val = nullptr;
    int pair = 0;              // D = 2: values stored as 16-byte pairs (nb.cu, slot layout)
    int64_t bytes = 0;
    // stencil-compressed columns (structured operators): slot t's columns are base + the offsets
    // of its pattern pid[t] (tbl[pid * W + k]; A entries first, then B); col is then freed
    int32_t *pid = nullptr, *baseA = nullptr, *baseB = nullptr, *tbl = nullptr;
    int W = 0, npat = 0;
    // B-value compression (after the column compression): the B / B^T values of a slot (its d
    // values per B entry, in entry order) are a vector of the small table vtbl at offset vofs[t];
    // the slice value arrays then hold only the A entries (32 A values per slice)
    int32_t* vofs = nullptr;
    double* vtbl = nullptr;
    int64_t nvtbl = 0, nbvec = 0;
};

struct Csr {
    int64_t n_rows = 0, n_cols = 0, nnz = 0;
    int64_t* rp = nullptr;
    int32_t* ci = nullptr;
    double* val = nullptr;
    int lanes = 8;  // lanes per row used by the row-group SpMV kernels
    Sell sell;      // built for smoother operators (rav_setup); empty otherwise
    NodeBlocked nb; // preferred over sell when the structure allows it
};
rav_status sell_build(Csr& A, cudaStream_t s);
void sell_free(Sell& S);
rav_status nb_build(Csr& A, int64_t nvel, int D, cudaStream_t s);
void nb_free(NodeBlocked& N);
// r = b - A x via the node-blocked / SELL copy (r may be null); if part != nullptr also one partial sum
// of r^2 per block, with min(full grid, nblk) blocks (*used = blocks launched)
// xpf / xpf_bytes (optional): the NEXT kernel's leading stream (the sweep's first factor chunks),
// bulk-prefetched into L2 by the residual's last warps while the residual, bound by gather
// latency, leaves HBM bandwidth unused
rav_status launch_nb_residual(const Csr& A, const double* x, const double* b, double* r, double* part, int nblk,
                              cudaStream_t s, int* used = nullptr, const void* xpf = nullptr, int64_t xpf_bytes = 0);
rav_status launch_sell_residual(const Csr& A, const double* x, const double* b, double* r, double* part, int nblk,
                                cudaStream_t s, int* used = nullptr);
int64_t nb_full_blocks(const NodeBlocked& N);
int64_t sell_full_blocks(const Sell& S);
// partial-sum capacity for which the fused residual-norm kernels run on their full grid
int64_t residual_part_capacity(const Csr& A);

rav_status csr_upload(const rav_csr* A, Csr& out, cudaStream_t s);
void csr_free(Csr& A);
rav_status csr_transpose(const Csr& A, Csr& At, cudaStream_t s);

// r = b - A x
rav_status launch_residual(const Csr& A, const double* x, const double* b, double* r, cudaStream_t s,
                           const void* xpf = nullptr, int64_t xpf_bytes = 0);
// y = alpha * A x + beta * y
rav_status launch_spmv(const Csr& A, const double* x, double* y, double alpha, double beta, cudaStream_t s);
// partial sums of squares of (b - A x) into part[nblk]; then total into *out (device)
rav_status launch_residual_norm2(const Csr& A, const double* x, const double* b, double* part, int nblk,
                                 double* out, cudaStream_t s);
int residual_norm_blocks();
// r = b - A x and *out = ||r||^2 (one pass over A when the node-blocked / SELL copy exists)
rav_status launch_residual_and_norm2(const Csr& A, const double* x, const double* b, double* r, double* part,
                                     int nblk, double* out, cudaStream_t s);
// *out (device) = sum_i a[i] b[i] (+ *out if accumulate), deterministic (part: >= nblk doubles)
rav_status launch_dot(const double* a, const double* b, int64_t n, double* part, int nblk, double* out,
                      int accumulate, cudaStream_t s);
// w += alpha * sum_i coef[i] V[i * ld + .] (coef: device, nv entries); dst = s * src
// out[i] = V_i . w for i < nv <= multi_dot_max() (part: multi_dot_blocks() * multi_dot_max() doubles)
int multi_dot_max();
int multi_dot_blocks();
rav_status launch_multi_dot(int64_t n, int nv, const double* V, int64_t ld, const double* w, double* part, double* out,
                            cudaStream_t s);
rav_status launch_multi_axpy(int64_t n, int nv, const double* V, int64_t ld, const double* coef, double alpha,
                             double* w, cudaStream_t s);
rav_status launch_scale(int64_t n, const double* src, double sc, double* dst, cudaStream_t s);
// a10 / R4: mode 0 p -= p[pin], mode 1 p -= mean(p) over x[n_vel .. n); shift: 1 device double,
// part: >= residual_norm_blocks() device doubles
rav_status launch_pressure_normalize(double* x, int64_t n_vel, int64_t n, int mode, int64_t pin, double* shift,
                                     double* part, cudaStream_t s);

// ---- setup.cu -------------------------------------------------------------------------
struct PatchSet {
    int64_t n_patches = 0, entries = 0;
    int64_t* offs = nullptr;   // device, reordered: restricted first
    int32_t* dofs = nullptr;
    double* w = nullptr;
    int32_t* nres = nullptr;   // restricted count per patch
    int nmax = 0, nresmax = 0;
    int64_t rows_total = 0;    // sum nres_i * n_i
    int64_t nres_total = 0;    // sum nres_i
    int64_t sym_total = 0;     // sum nres_i (nres_i + 1) / 2 + nres_i (n_i - nres_i)
};

struct Factors {
    int layout = 0;            // 1 general (row-major per patch), 2 thread-per-patch SoA chunks
    // general
    int64_t* foffs = nullptr;  // n_patches + 1
    double* fac = nullptr;
    // SoA
    int NT = 0, NMAX = 0, NTRI = 0;
    double* WT = nullptr;      // layout 3: nchunks * NT * 32 row weights; layout 4: aux (weights, w_p, 1/S)
    // Schur formats (schur.cu): layout 4 thread SoA chunks, layout 5 per patch (warp kernel)
    int MT = 0, D = 0, NN = 0;
    int64_t pairs = 0;
    int32_t* PD = nullptr;     // pressure DoF per patch slot
    int32_t* nodes = nullptr;  // layout 5: node dofs per patch
    int64_t* nodeoffs = nullptr;
    int64_t alg_bytes = 0;     // algorithmic bytes of the stored factor data (per application)
    int mode = 0;              // schur_factorize mode
    int64_t nchunks = 0;
    double* facT = nullptr;    // nchunks * (NMAX*NT/2) * 32 double2
    int32_t* DT = nullptr;     // nchunks * NMAX * 32
    int32_t* NR = nullptr;     // nchunks * 32 restricted counts (0 for padding)
    int64_t bytes = 0;
    // the sweep's leading factor stream in the order its first wave reads it (layout 4: facT,
    // chunk-major; layouts 5 / 6: fac, patch-major): what a preceding residual prefetches into L2
    const void* lead = nullptr;
    int64_t lead_bytes = 0;
    // layout 4 node-index compression: node j of slot i = nbase[i] + ntbl[npid[i] * NN + j] (DT freed)
    int32_t *npid = nullptr, *nbase = nullptr, *ntbl = nullptr;
    int nnpat = 0;
    // layout 4 weight table (with the node patterns): the restricted weights, w_p and the restricted
    // count of a slot are those of its node pattern (PoU weights are geometric), verified bitwise;
    // the sweep then streams only 1/S per patch (SINV) instead of the MT + 2 aux values and NR
    double* wtab = nullptr;     // nnpat * (MT + 1): weights k < MT, then w_p
    int32_t* ntab = nullptr;    // nnpat: restricted node count
    double* SINV = nullptr;     // nchunks * 32: 1/S per slot
    // deterministic scatter (rav_opts.deterministic, Schur formats): per-patch correction slots and,
    // per written DoF, its slots in ascending patch order
    double* cbuf = nullptr;
    int64_t det_n = 0;          // number of written DoFs
    int32_t* det_dof = nullptr;
    int64_t* det_off = nullptr; // det_n + 1
    int32_t* det_slot = nullptr;
};

// build the deterministic-scatter tables of a Schur format (layouts 4 / 5)
rav_status schur_det_setup(const PatchSet& P, Factors& F, cudaStream_t s);

rav_status patches_upload(const rav_patches* P, int64_t n_dofs, PatchSet& out, cudaStream_t s);
void patches_free(PatchSet& P);
// factorize all patches; bad_patch = smallest singular patch or -1
rav_status factorize(const Csr& A, const PatchSet& P, int variant, int64_t nvel, int kernel_choice,
                     Factors& F, int64_t* bad_patch, cudaStream_t s);
void factors_free(Factors& F);
rav_status export_rows(const PatchSet& P, const Factors& F, double* rows, cudaStream_t s);
bool thread_kernel_supported(int nresmax, int nmax);

// ---- schur.cu -------------------------------------------------------------------------
// Try the factored Schur format (velocity block I_D (x) A_s, one pressure DoF per patch).
// *applicable = false (and F untouched) when the structure does not hold.
// mode: 0 restricted rows (RAV / AV), 1 diagonal Vanka (layout 6), 2 full rows for multicoloured MV
rav_status schur_factorize(const Csr& A, const PatchSet& P, int64_t nvel, int D, int kernel_choice, int mode,
                           Factors& F, int64_t* bad_patch, bool* applicable, cudaStream_t s);
rav_status launch_diag_sweep(const PatchSet& P, const Factors& F, const double* r, double* x, double omega,
                             cudaStream_t s);
rav_status launch_mv_color(const Csr& A, const Factors& F, int64_t ncol, const int32_t* plist, const double* b,
                           double* x, double omega, cudaStream_t s);
// one MV colour from a residual r = b - L x computed just before (instead of the patch rows of L)
rav_status launch_mv_color_r(const Factors& F, int64_t ncol, const int32_t* plist, const double* r, double* x,
                             double omega, cudaStream_t s);
rav_status launch_schur_sweep(const PatchSet& P, const Factors& F, const double* r, double* x, double omega,
                              cudaStream_t s);

// ---- the interface exchange fused into the sweep (mgd peer transport, dist.cu) ----------------
// The corrections a subdomain's patches make to DoFs a neighbour owns (ghost-written DoFs) are
// added by the sweep's own scatter straight into that neighbour's receive buffer (over NVLink when
// it is another GPU), instead of into x followed by a pack kernel and a message.  The sweep waits
// (thread 0 of each CTA) for the consumers' acks of the previous message before any scatter, and
// its last CTA releases the consumers' flags.
struct Outbox {
    const int32_t* rmap = nullptr;          // per local DoF: (q << 24) | slot for ghost-written DoFs, else -1
    const uint8_t* pflag = nullptr;         // per patch: 1 when it writes a ghost-written DoF
    int nq = 0;                             // consumers (<= 2: the slab's neighbours)
    double* buf[2] = {nullptr, nullptr};    // consumer q's receive buffer for these corrections
    unsigned long long* sig[2] = {nullptr, nullptr};   // consumer q's flag
    unsigned long long* ack[2] = {nullptr, nullptr};   // own ack words (released by consumer q)
    int sys[2] = {0, 0};                    // consumer q is another GPU: system-scope release
    unsigned long long* seq = nullptr;      // this producer's message counter
    unsigned int* done = nullptr;           // writers of the launch that finished
    unsigned int nflag = 0;                 // writers per launch: chunks (thread kernel) / patches (warp
                                            // kernel) holding a ghost-writing patch
    int64_t rot = 0;                        // thread kernel: warp w takes chunk (w - rot) mod nchunks, so
                                            // the trailing writer chunks run in the first wave, not the last
    unsigned int* timeout = nullptr;        // set when a bounded wait expires
};

__device__ __forceinline__ unsigned long long ob_ld_acquire(const unsigned long long* p, int sys) {
    unsigned long long v;
    if (sys) asm volatile("ld.acquire.sys.global.u64 %0, [%1];" : "=l"(v) : "l"(p) : "memory");
    else asm volatile("ld.acquire.gpu.global.u64 %0, [%1];" : "=l"(v) : "l"(p) : "memory");
    return v;
}
__device__ __forceinline__ void ob_st_release(unsigned long long* p, unsigned long long v, int sys) {
    if (sys) asm volatile("st.release.sys.global.u64 [%0], %1;" ::"l"(p), "l"(v) : "memory");
    else asm volatile("st.release.gpu.global.u64 [%0], %1;" ::"l"(p), "l"(v) : "memory");
}
// spin until *p >= v (bounded: ~4 s, then *err |= 1 and go on -- never a hung GPU)
__device__ __forceinline__ void ob_wait_geq(const unsigned long long* p, unsigned long long v, int sys,
                                            unsigned int* err) {
    for (long long spin = 0; ob_ld_acquire(p, sys) < v; ++spin) {
        if (spin > (1ll << 24)) {
            if (err) atomicOr(err, 1u);
            return;
        }
        __nanosleep(256);
    }
}
// the hot-loop view of an Outbox, passed by value (a reference to the kernel parameter would put
// the whole struct in local memory)
struct ObView {
    const int32_t* rmap;
    const uint8_t* pflag;
    double* buf0;
    double* buf1;
    const unsigned long long* ack0;
    const unsigned long long* ack1;
    const unsigned long long* seq;
    unsigned int* timeout;
    int nq, sys0, sys1;
    int64_t rot;
};
__device__ __forceinline__ ObView ob_view(const Outbox& o) {
    return ObView{o.rmap, o.pflag, o.buf[0], o.buf[1], o.ack[0], o.ack[1], o.seq, o.timeout, o.nq, o.sys[0], o.sys[1],
                  o.rot};
}
// before a thread's first store into a receive buffer: the consumers have consumed the previous
// message (ack >= this launch's message number - 1; *seq changes only at the launch's end)
__device__ __forceinline__ void ob_wait_acks(const ObView& o) {
    const unsigned long long s = *reinterpret_cast<const volatile unsigned long long*>(o.seq);
    if (o.nq > 0) ob_wait_geq(o.ack0, s, o.sys0, o.timeout);
    if (o.nq > 1) ob_wait_geq(o.ack1, s, o.sys1, o.timeout);
}
// *p += v as a fire-and-forget reduction (kernels that also hold fences compiled atomicAdd to
// returning ATOMG: +15% on the sweep)
__device__ __forceinline__ void red_add(double* p, double v) {
    asm volatile("red.relaxed.gpu.global.add.f64 [%0], %1;" ::"l"(p), "d"(v) : "memory");
}
// x[dof] += v, or the consumer's receive buffer when dof is ghost-written (patches with pflag)
__device__ __forceinline__ void ob_add(const ObView& o, bool flagged, double* x, int dof, double v) {
    if (flagged) {
        const int m = o.rmap[dof];
        if (m >= 0) {
            red_add((m >> 24 ? o.buf1 : o.buf0) + (m & 0xffffff), v);
            return;
        }
    }
    red_add(x + dof, v);
}
// after a writer (a chunk / patch with ghost-writing patches; every lane of the warp calls it) has
// made its scatters: fence, count it; the launch's last writer releases the consumers' flags with
// the next message number.  Only writers count -- a single counter hit by every warp of the grid
// cost ~15% of the sweep -- and only writers' stores go to the receive buffers (the stores to x
// reach the consumer's add kernel through the kernel boundary).  Static indices: the parameter
// stays in constant space.
__device__ __forceinline__ void ob_writer_done(const Outbox& o) {
    __syncwarp();
    if ((threadIdx.x & 31) == 0) {
        __threadfence();
        if (atomicAdd(o.done, 1u) == o.nflag - 1) {
            __threadfence();
            *o.done = 0;
            const unsigned long long t = *reinterpret_cast<volatile unsigned long long*>(o.seq) + 1;
            *o.seq = t;
#pragma unroll
            for (int q = 0; q < 2; ++q)
                if (q < o.nq) ob_st_release(o.sig[q], t, o.sys[q]);
        }
    }
}
// can the sweep of this smoother run fused (the Schur thread kernel, or the per-patch warp kernel)?
bool schur_fusable(const PatchSet& P, const Factors& F);
rav_status launch_schur_sweep_ob(const PatchSet& P, const Factors& F, const double* r, double* x, double omega,
                                 const Outbox& ob, cudaStream_t s);
rav_status export_schur_rows(const PatchSet& P, const Factors& F, int64_t nvel, double* rows, cudaStream_t s);

// ---- sweep.cu -------------------------------------------------------------------------
rav_status launch_sweep(const PatchSet& P, const Factors& F, const double* r, double* x, double omega,
                        cudaStream_t s);

// ---- coarse.cu ------------------------------------------------------------------------
// ---- xfer.cu: stencil form of the nested transfers of uniformly refined structured grids -----
// (3D restriction stays on the CSR P^T: its 125-point gather per coarse node is latency-bound,
// measured 34 vs 19 us at the c4 fine level; the 3D prolongation uses the stencil, 15 vs 22 us)
struct XStruct {
    int on = 0;
    int dim = 0, P = 2;    // P: velocity lattice refinement (2: Q2-Q1, 1: Q1-Q1)
    int nc[3] = {1, 1, 1}; // coarse cells per axis
    int64_t n_fine = 0, n_coarse = 0;
    // slab windows along the last axis (global lattice layers, inclusive; whole grids: everything):
    // fine window node / vertex layers, the fine rows P fills (owned layers), coarse window layers
    int fn_lo = 0, fn_hi = -1, fv_lo = 0, fv_hi = -1;
    int rn_lo = 0, rn_hi = -1, rv_lo = 0, rv_hi = -1;
    int cn_lo = 0, cn_hi = -1, cv_lo = 0, cv_hi = -1;
};
rav_status xs_build(const rav_grid* fine, const rav_grid* coarse, int64_t n_fine, int64_t n_coarse, XStruct& S);
rav_status xs_verify(const XStruct& S, const Csr& P, const Csr& PT, cudaStream_t s);
rav_status launch_xs_prolong(const XStruct& S, const double* xc, double* yf, double alpha, double beta,
                             cudaStream_t s);
rav_status launch_xs_restrict(const XStruct& S, const double* rf, double* bc, cudaStream_t s);

struct CoarseLU {
    int64_t n = 0, pin = -1;
    int m = 0;
    double* lu = nullptr;      // m x m
    int32_t* piv = nullptr;
    double* inv = nullptr;     // m x m explicit inverse (m <= 2048), row-major
};
rav_status coarse_factor(const Csr& A, int64_t pin, CoarseLU& C, cudaStream_t s);
rav_status launch_coarse_solve(const CoarseLU& C, const double* b, double* x, cudaStream_t s);
void coarse_free(CoarseLU& C);

}  // namespace rav
