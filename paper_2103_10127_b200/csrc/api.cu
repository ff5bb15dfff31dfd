// api.cu -- the C-ABI of include/ravgmg.h: smoother and multigrid contexts,
// stream-ordered execution, CUDA-graph capture of sweep sequences and of whole
// V-cycles (the coarse levels are launch-bound), host-buffer staging.
#include <stdarg.h>

#include <algorithm>
#include <vector>

#include "ctx.cuh"

namespace rav {

static thread_local char g_err[1024] = "";
thread_local int64_t g_launches = 0;

void set_error(const char* fmt, ...) {
    va_list ap;
    va_start(ap, fmt);
    vsnprintf(g_err, sizeof(g_err), fmt, ap);
    va_end(ap);
}
const char* get_error() { return g_err; }

bool pdl_enabled() {
    static const bool on = [] {
        const char* e = getenv("RAV_PDL");
        return !(e && atoi(e) == 0);
    }();
    return on;
}

int num_sms() {
    static int n = 0;
    if (n == 0) {
        int dev = 0;
        cudaGetDevice(&dev);
        if (cudaDeviceGetAttribute(&n, cudaDevAttrMultiProcessorCount, dev) != cudaSuccess || n <= 0) n = 148;
    }
    return n;
}

static bool is_device_ptr(const void* p) {
    cudaPointerAttributes a;
    if (cudaPointerGetAttributes(&a, p) != cudaSuccess) { cudaGetLastError(); return false; }
    return a.type == cudaMemoryTypeDevice || a.type == cudaMemoryTypeManaged;
}

}  // namespace rav

using namespace rav;

namespace rav {

// r_ready: c->r already holds b - L x for the incoming x (the stopping test of mg_solve
// computed it), so the first sweep skips its residual pass
// x_zero: x is zero on entry (coarse-level corrections, FGMRES preconditioner applications), so the
// first sweep's residual is b itself and is read from b instead of being computed
// bytes of the sweep's leading factor stream the residual before it prefetches into L2 (RAV_XPF_MB)
static int64_t xpf_bytes() {
    static const int64_t v = [] {
        const char* e = getenv("RAV_XPF_MB");
        return (int64_t)((e ? atof(e) : 48.0) * 1048576.0);   // measured c2 step: 0 168.7, 32 166.5, 48 165.9, 64 166.4, 96 169.8 us
    }();
    return v;
}

rav_status smooth_launches(rav_ctx* c, double* x, const double* b, int nu, double omega, bool r_ready,
                           bool x_zero) {
    for (int k = 0; k < nu; ++k) {
        if (c->variant == RAV_VARIANT_MV) {   // colour by colour, fresh local residuals (Eq. 11, 15)
            for (size_t q = 0; q + 1 < c->coffs.size(); ++q) {
                if (c->A.nb.nslices > 0) {   // the colour's residual by the node-blocked kernel, then the patches
                    RAV_TRY(launch_residual(c->A, x, b, c->r, c->stream));
                    RAV_TRY(launch_mv_color_r(c->F, c->coffs[q + 1] - c->coffs[q], c->plist + c->coffs[q], c->r, x,
                                              omega, c->stream));
                } else {
                    RAV_TRY(launch_mv_color(c->A, c->F, c->coffs[q + 1] - c->coffs[q], c->plist + c->coffs[q], b,
                                            x, omega, c->stream));
                }
            }
            continue;
        }
        if (k == 0 && x_zero && !r_ready) {   // r = b - L 0 = b
            RAV_TRY(launch_sweep(c->P, c->F, b, x, omega, c->stream));
            continue;
        }
        if (!(r_ready && k == 0))
            RAV_TRY(launch_residual(c->A, x, b, c->r, c->stream, c->F.lead, std::min(c->F.lead_bytes, xpf_bytes())));
        RAV_TRY(launch_sweep(c->P, c->F, c->r, x, omega, c->stream));
    }
    return RAV_OK;
}

}  // namespace rav

extern "C" {

const char* rav_last_error(void) { return rav::get_error(); }
const char* rav_version(void) { return "ravgmg 0.1 (sm_100a)"; }

rav_status rav_setup(const rav_csr* A, const rav_patches* P, const rav_opts* opts, rav_ctx** out,
                     int64_t* bad_patch) {
    NvtxRange nvtx_range("rav_setup");
    if (!out || !A || !P) { set_error("rav_setup: NULL argument"); return RAV_ERR_ARG; }
    *out = nullptr;
    if (bad_patch) *bad_patch = -1;
    rav_opts o{};
    if (opts) o = *opts;
    if (o.variant != RAV_VARIANT_ROWS && o.variant != RAV_VARIANT_DIAG && o.variant != RAV_VARIANT_MV) {
        set_error("rav_setup: bad variant");
        return RAV_ERR_ARG;
    }
    if (A->n_rows != A->n_cols) { set_error("rav_setup: L must be square"); return RAV_ERR_ARG; }
    rav_ctx* c = new rav_ctx();
    c->stream = as_stream(o.stream);
    c->variant = o.variant;
    c->nvel = o.n_vel;
    rav_status st = csr_upload(A, c->A, c->stream);
    static const int mv_nb = [] {   // MV: colour residuals by the node-blocked kernel (0: patch rows of L)
        const char* e = getenv("RAV_MV_NB");
        return e ? atoi(e) : 1;
    }();
    if (st == RAV_OK && (o.variant != RAV_VARIANT_MV || mv_nb) && o.block_dim > 0 && o.kernel != RAV_KERNEL_WARP)
        st = nb_build(c->A, o.n_vel, o.block_dim, c->stream);
    if (st == RAV_OK && o.variant != RAV_VARIANT_MV && c->A.nb.nslices == 0) st = sell_build(c->A, c->stream);
    if (st == RAV_OK) st = patches_upload(P, A->n_rows, c->P, c->stream);
    bool done = false;
    const bool want_schur = o.block_dim > 0 && (o.kernel == RAV_KERNEL_AUTO || o.kernel == RAV_KERNEL_SCHUR);
    if (st == RAV_OK && (want_schur || o.variant == RAV_VARIANT_MV)) {
        const int mode = o.variant == RAV_VARIANT_DIAG ? 1 : (o.variant == RAV_VARIANT_MV ? 2 : 0);
        st = schur_factorize(c->A, c->P, o.n_vel, o.block_dim, o.kernel, mode, c->F, bad_patch, &done, c->stream);
        if (st == RAV_OK && !done && (o.kernel == RAV_KERNEL_SCHUR || o.variant == RAV_VARIANT_MV)) {
            set_error("rav_setup: %s needs block_dim > 0 and patches with one pressure DoF and an I_d (x) A_s "
                      "velocity block", o.variant == RAV_VARIANT_MV ? "RAV_VARIANT_MV" : "RAV_KERNEL_SCHUR");
            st = RAV_ERR_ARG;
        }
    }
    if (st == RAV_OK && !done) {
        if (o.kernel == RAV_KERNEL_SCHUR) {
            set_error("rav_setup: RAV_KERNEL_SCHUR needs variant ROWS and block_dim > 0");
            st = RAV_ERR_ARG;
        } else {
            st = factorize(c->A, c->P, o.variant, o.n_vel, o.kernel, c->F, bad_patch, c->stream);
        }
    }
    if (st == RAV_OK && o.deterministic && o.variant != RAV_VARIANT_MV) {
        if (c->F.layout == 4 || c->F.layout == 5) {
            st = schur_det_setup(c->P, c->F, c->stream);
        } else {
            set_error("rav_setup: deterministic scatter needs the Schur format (block_dim > 0, Vanka-shaped patches)");
            st = RAV_ERR_ARG;
        }
    }
    if (st == RAV_OK) {
        cudaError_t e = cudaMalloc(&c->r, sizeof(double) * std::max<int64_t>(1, c->A.n_rows));
        if (e != cudaSuccess) { set_error("rav_setup: %s", cudaGetErrorString(e)); st = RAV_ERR_OOM; }
    }
    if (st != RAV_OK) { rav_destroy(c); return st; }
    *out = c;
    return RAV_OK;
}

rav_status rav_set_colors(rav_ctx* c, int n_colors, const int64_t* color_offs, const int32_t* patch_ids) {
    if (!c || n_colors < 1 || !color_offs || !patch_ids) { set_error("rav_set_colors: bad argument"); return RAV_ERR_ARG; }
    if (color_offs[0] != 0 || color_offs[n_colors] != c->P.n_patches) {
        set_error("rav_set_colors: colours must partition the %lld patches", (long long)c->P.n_patches);
        return RAV_ERR_ARG;
    }
    std::vector<char> seen(c->P.n_patches, 0);
    for (int64_t q = 0; q < c->P.n_patches; ++q) {
        const int32_t i = patch_ids[q];
        if (i < 0 || i >= c->P.n_patches || seen[i]) { set_error("rav_set_colors: not a permutation"); return RAV_ERR_ARG; }
        seen[i] = 1;
    }
    c->coffs.assign(color_offs, color_offs + n_colors + 1);
    if (c->plist) cudaFree(c->plist);
    RAV_CUDA(cudaMalloc(&c->plist, sizeof(int32_t) * c->P.n_patches));
    RAV_CUDA(cudaMemcpy(c->plist, patch_ids, sizeof(int32_t) * c->P.n_patches, cudaMemcpyHostToDevice));
    c->graphs_reset();
    return RAV_OK;
}

rav_status rav_apply_color(rav_ctx* c, int color, double* x, const double* b, double omega) {
    if (!c || !x || !b) { set_error("rav_apply_color: NULL argument"); return RAV_ERR_ARG; }
    if (c->variant != RAV_VARIANT_MV || c->coffs.empty()) {
        set_error("rav_apply_color: needs RAV_VARIANT_MV and rav_set_colors");
        return RAV_ERR_ARG;
    }
    if (color < 0 || color + 1 >= (int)c->coffs.size()) { set_error("rav_apply_color: bad colour"); return RAV_ERR_ARG; }
    g_launches = 0;
    RAV_TRY(launch_mv_color(c->A, c->F, c->coffs[color + 1] - c->coffs[color], c->plist + c->coffs[color], b, x, omega,
                            c->stream));
    c->last_launches = g_launches;
    return RAV_OK;
}

rav_status rav_set_stream(rav_ctx* c, void* stream) {
    if (!c) { set_error("NULL ctx"); return RAV_ERR_ARG; }
    if (c->stream != as_stream(stream)) c->graphs_reset();
    c->stream = as_stream(stream);
    return RAV_OK;
}

rav_status rav_smooth(rav_ctx* c, double* x, const double* b, int nu, double omega) {
    NvtxRange nvtx_range("rav_smooth");
    if (!c || !x || !b || nu < 0) { set_error("rav_smooth: bad argument"); return RAV_ERR_ARG; }
    g_launches = 0;
    if (nu == 0) { c->last_launches = 0; return RAV_OK; }
    const int64_t n = c->A.n_rows;
    bool dx = is_device_ptr(x), db = is_device_ptr(b);
    if (dx != db) { set_error("rav_smooth: x and b must both be device or both host pointers"); return RAV_ERR_ARG; }
    double* X = x;
    const double* B = b;
    if (!dx) {
        if (!c->hx) {
            RAV_CUDA(cudaMalloc(&c->hx, sizeof(double) * n));
            RAV_CUDA(cudaMalloc(&c->hb, sizeof(double) * n));
        }
        RAV_CUDA(cudaMemcpyAsync(c->hx, x, sizeof(double) * n, cudaMemcpyHostToDevice, c->stream));
        RAV_CUDA(cudaMemcpyAsync(c->hb, b, sizeof(double) * n, cudaMemcpyHostToDevice, c->stream));
        X = c->hx;
        B = c->hb;
    }
    if (c->variant == RAV_VARIANT_MV && c->coffs.empty()) {
        set_error("rav_smooth: RAV_VARIANT_MV needs rav_set_colors first");
        return RAV_ERR_ARG;
    }
    bool use_graph = c->stream != nullptr && (nu >= 2 || c->variant == RAV_VARIANT_MV);
    int gi = c->graph[0].match(X, B, nu, 0, 0, omega) ? 0 : (c->graph[1].match(X, B, nu, 0, 0, omega) ? 1 : -1);
    if (gi < 0) {
        gi = c->graph_next;
        c->graph_next ^= 1;
    }
    RAV_TRY(run_graph(c->graph[gi], c->stream, use_graph, X, B, nu, 0, 0, omega, c->last_launches,
                      [&]() { return smooth_launches(c, X, B, nu, omega); }));
    if (!dx) {
        RAV_CUDA(cudaMemcpyAsync(x, c->hx, sizeof(double) * n, cudaMemcpyDeviceToHost, c->stream));
        RAV_CUDA(cudaStreamSynchronize(c->stream));
    }
    return RAV_OK;
}

rav_status rav_smooth_batch(rav_ctx* c, int64_t nprob, double* const* x, const double* const* b, int nu,
                            double omega) {
    NvtxRange nvtx_range("rav_smooth_batch");
    if (!c || nprob < 0 || nu < 0 || (nprob > 0 && (!x || !b))) { set_error("rav_smooth_batch: bad argument"); return RAV_ERR_ARG; }
    for (int64_t k = 0; k < nprob; ++k)
        if (!x[k] || !b[k] || is_device_ptr(x[k]) || is_device_ptr(b[k])) {
            set_error("rav_smooth_batch: problem %lld: x and b must be host pointers", (long long)k);
            return RAV_ERR_ARG;
        }
    if (c->variant == RAV_VARIANT_MV && c->coffs.empty()) {
        set_error("rav_smooth_batch: RAV_VARIANT_MV needs rav_set_colors first");
        return RAV_ERR_ARG;
    }
    g_launches = 0;
    if (nprob == 0 || nu == 0) { c->last_launches = 0; return RAV_OK; }
    if (!c->stream) { set_error("rav_smooth_batch: needs a context stream (rav_opts.stream)"); return RAV_ERR_ARG; }
    const int64_t n = c->A.n_rows;
    const size_t bytes = sizeof(double) * (size_t)n;
    if (!c->hx) {
        RAV_CUDA(cudaMalloc(&c->hx, bytes));
        RAV_CUDA(cudaMalloc(&c->hb, bytes));
    }
    if (!c->hx2) {
        RAV_CUDA(cudaMalloc(&c->hx2, bytes));
        RAV_CUDA(cudaMalloc(&c->hb2, bytes));
    }
    if (!c->cstream) RAV_CUDA(cudaStreamCreateWithFlags(&c->cstream, cudaStreamNonBlocking));
    for (int k = 0; k < 2; ++k) {
        if (!c->ev_in[k]) RAV_CUDA(cudaEventCreateWithFlags(&c->ev_in[k], cudaEventDisableTiming));
        if (!c->ev_done[k]) RAV_CUDA(cudaEventCreateWithFlags(&c->ev_done[k], cudaEventDisableTiming));
    }
    double* X[2] = {c->hx, c->hx2};
    double* B[2] = {c->hb, c->hb2};
    // copy stream: in(0), in(1), out(0), in(2), out(1), ... -- in(k + 2) reuses slot k after out(k);
    // the sweeps of problem k wait for in(k), out(k) waits for them
    auto put = [&](int64_t k) -> rav_status {
        const int s = (int)(k & 1);
        RAV_CUDA(cudaMemcpyAsync(X[s], x[k], bytes, cudaMemcpyHostToDevice, c->cstream));
        RAV_CUDA(cudaMemcpyAsync(B[s], b[k], bytes, cudaMemcpyHostToDevice, c->cstream));
        RAV_CUDA(cudaEventRecord(c->ev_in[s], c->cstream));
        return RAV_OK;
    };
    int64_t launches = 0;
    RAV_TRY(put(0));
    if (nprob > 1) RAV_TRY(put(1));
    for (int64_t k = 0; k < nprob; ++k) {
        const int s = (int)(k & 1);
        RAV_CUDA(cudaStreamWaitEvent(c->stream, c->ev_in[s], 0));
        int gi = c->graph[0].match(X[s], B[s], nu, 0, 0, omega) ? 0
                 : (c->graph[1].match(X[s], B[s], nu, 0, 0, omega) ? 1 : -1);
        if (gi < 0) {
            gi = c->graph_next;
            c->graph_next ^= 1;
        }
        int64_t l = 0;
        RAV_TRY(run_graph(c->graph[gi], c->stream, true, X[s], B[s], nu, 0, 0, omega, l,
                          [&]() { return smooth_launches(c, X[s], B[s], nu, omega); }));
        launches += l;
        RAV_CUDA(cudaEventRecord(c->ev_done[s], c->stream));
        RAV_CUDA(cudaStreamWaitEvent(c->cstream, c->ev_done[s], 0));
        RAV_CUDA(cudaMemcpyAsync(x[k], X[s], bytes, cudaMemcpyDeviceToHost, c->cstream));
        if (k + 2 < nprob) RAV_TRY(put(k + 2));
    }
    RAV_CUDA(cudaStreamSynchronize(c->cstream));
    RAV_CUDA(cudaStreamSynchronize(c->stream));
    c->last_launches = launches;
    return RAV_OK;
}

rav_status rav_residual(rav_ctx* c, const double* x, const double* b, double* r) {
    NvtxRange nvtx_range("rav_residual");
    if (!c || !x || !b || !r) { set_error("rav_residual: NULL argument"); return RAV_ERR_ARG; }
    g_launches = 0;
    RAV_TRY(launch_residual(c->A, x, b, r, c->stream));
    c->last_launches = g_launches;
    return RAV_OK;
}

rav_status rav_apply(rav_ctx* c, const double* r, double* x, double omega) {
    NvtxRange nvtx_range("rav_apply");
    if (!c || !x || !r) { set_error("rav_apply: NULL argument"); return RAV_ERR_ARG; }
    g_launches = 0;
    RAV_TRY(launch_sweep(c->P, c->F, r, x, omega, c->stream));
    c->last_launches = g_launches;
    return RAV_OK;
}

rav_status rav_rows_size(const rav_ctx* c, int64_t* total) {
    if (!c || !total) { set_error("NULL argument"); return RAV_ERR_ARG; }
    *total = c->P.rows_total;
    return RAV_OK;
}

rav_status rav_export_rows(const rav_ctx* c, double* rows) {
    if (!c || !rows) { set_error("NULL argument"); return RAV_ERR_ARG; }
    if (c->F.layout == 6) {
        set_error("rav_export_rows: not available for the diagonal-Vanka format");
        return RAV_ERR_ARG;
    }
    if (c->F.layout >= 4) RAV_TRY(export_schur_rows(c->P, c->F, c->nvel, rows, c->stream));
    else RAV_TRY(export_rows(c->P, c->F, rows, c->stream));
    RAV_CUDA(cudaStreamSynchronize(c->stream));
    return RAV_OK;
}

rav_status rav_sweep_bytes(const rav_ctx* c, double* bytes_sweep, double* bytes_residual, double* flops) {
    if (!c) { set_error("NULL ctx"); return RAV_ERR_ARG; }
    const double n = (double)c->A.n_rows, nnz = (double)c->A.nnz;
    // algorithmic bytes (SURVEY section 8 row d): factor rows 8 sum nres_i n_i, patch DoF
    // indices 4 sum n_i, x read+write, r gathered once (compulsory vectors)
    // layout 3 streams the symmetric restricted block once (+ one weight per restricted row)
    double rows = c->F.layout == 3 ? 8.0 * (double)(c->P.sym_total + c->P.nres_total)
                                   : 8.0 * (double)c->P.rows_total;
    double idx = 4.0 * (double)c->P.entries;
    if (c->F.layout >= 4) {   // Schur formats: factored rows + node indices (counted at setup)
        rows = (double)c->F.alg_bytes;
        idx = 0.0;
    }
    double sweep = rows + idx + 8.0 * n /* r */ + 16.0 * n /* x rmw */;
    double resid = 12.0 * nnz + 8.0 * (n + 1) + 8.0 * n /* x */ + 8.0 * n /* b */ + 8.0 * n /* r write */;
    if (c->A.nb.nslices > 0)   // node-blocked copy: its own entries + per-row permutation + vectors
        resid = (double)c->A.nb.bytes + 4.0 * (double)c->A.nb.nblock + 24.0 * (double)c->A.nb.nslices + 24.0 * n;
    if (bytes_sweep) *bytes_sweep = sweep;
    if (bytes_residual) *bytes_residual = resid;
    if (flops) *flops = 2.0 * (double)c->P.rows_total + 2.0 * nnz;
    return RAV_OK;
}

int64_t rav_last_launches(const rav_ctx* c) { return c ? c->last_launches : 0; }

const char* rav_kernel_name(const rav_ctx* c) {
    if (!c) return "";
    switch (c->F.layout) {
        case 1: return "sweep_warp_kernel (rows, row-major per patch)";
        case 2: return "sweep_thread_kernel (rows, SoA chunks)";
        case 3: return "sweep_sym_kernel (symmetric restricted block, SoA chunks)";
        case 4: return "schur_sweep_thread_kernel (factored Schur rows, SoA chunks)";
        case 5: return c->variant == RAV_VARIANT_MV ? "mv_color_kernel (multicoloured MV, full Schur rows)"
                                                    : "schur_sweep_warp_kernel (factored Schur rows, per patch)";
        case 6: return "diag_sweep_kernel (diagonal Vanka, closed form)";
        default: return "unknown";
    }
}

void rav_destroy(rav_ctx* c) {
    if (!c) return;
    if (c->stream) cudaStreamSynchronize(c->stream);
    else cudaDeviceSynchronize();
    c->graphs_reset();
    csr_free(c->A);
    patches_free(c->P);
    factors_free(c->F);
    if (c->r) cudaFree(c->r);
    if (c->hx) cudaFree(c->hx);
    if (c->hb) cudaFree(c->hb);
    if (c->hx2) cudaFree(c->hx2);
    if (c->hb2) cudaFree(c->hb2);
    if (c->cstream) {
        cudaStreamSynchronize(c->cstream);
        cudaStreamDestroy(c->cstream);
    }
    for (int k = 0; k < 2; ++k) {
        if (c->ev_in[k]) cudaEventDestroy(c->ev_in[k]);
        if (c->ev_done[k]) cudaEventDestroy(c->ev_done[k]);
    }
    if (c->plist) cudaFree(c->plist);
    delete c;
}

// ------------------------------------------------------------------------------------
// multigrid
// ------------------------------------------------------------------------------------

void mg_destroy(mg_ctx* m) {
    if (!m) return;
    if (m->stream) cudaStreamSynchronize(m->stream);
    else cudaDeviceSynchronize();
    m->cyc.reset();
    for (int l = 0; l < (int)m->lv.size(); ++l) {
        mg_level& L = m->lv[l];
        if (L.sm) rav_destroy(L.sm);
        else csr_free(L.A);
        csr_free(L.P);
        csr_free(L.PT);
        if (L.x) cudaFree(L.x);
        if (L.b) cudaFree(L.b);
        if (L.r) cudaFree(L.r);
    }
    coarse_free(m->C);
    if (m->part) cudaFree(m->part);
    if (m->norm2) cudaFree(m->norm2);
    if (m->h_norm2) cudaFreeHost(m->h_norm2);
    if (m->hx) cudaFree(m->hx);
    if (m->hb) cudaFree(m->hb);
    for (double* p : {m->kV, m->kZ, m->kw, m->kr, m->kh, m->kpart, m->kzero, m->kmd})
        if (p) cudaFree(p);
    delete m;
}

rav_status mg_setup(int n_levels, const rav_csr* A, const rav_patches* patches, const rav_csr* P,
                    const int64_t* n_vel, int64_t coarse_pin, const rav_opts* opts, mg_ctx** out, int* bad_level,
                    int64_t* bad_patch) {
    NvtxRange nvtx_range("mg_setup");
    if (!out || !A || n_levels < 1 || (n_levels > 1 && (!patches || !P))) {
        set_error("mg_setup: bad argument");
        return RAV_ERR_ARG;
    }
    *out = nullptr;
    if (bad_level) *bad_level = -1;
    if (bad_patch) *bad_patch = -1;
    rav_opts o{};
    if (opts) o = *opts;
    mg_ctx* m = new mg_ctx();
    m->L = n_levels;
    m->lv.resize(n_levels);
    m->stream = as_stream(o.stream);
    rav_status st = RAV_OK;
    for (int l = 0; l < n_levels && st == RAV_OK; ++l) {
        mg_level& L = m->lv[l];
        if (l == 0) {
            L.nvel = n_vel ? n_vel[0] : o.n_vel;
            st = csr_upload(&A[0], L.A, m->stream);
            if (st == RAV_OK) st = coarse_factor(L.A, coarse_pin, m->C, m->stream);
        } else {
            if (P[l].n_rows != A[l].n_rows || P[l].n_cols != A[l - 1].n_rows) {
                set_error("mg_setup: P[%d] must be n_%d x n_%d", l, l, l - 1);
                st = RAV_ERR_ARG;
                break;
            }
            int64_t bp = -1;
            rav_opts ol = o;
            if (n_vel) ol.n_vel = n_vel[l];
            L.nvel = ol.n_vel;
            st = rav_setup(&A[l], &patches[l], &ol, &L.sm, &bp);
            if (st == RAV_ERR_SINGULAR_LOCAL) {
                if (bad_level) *bad_level = l;
                if (bad_patch) *bad_patch = bp;
            }
            if (st != RAV_OK) break;
            L.A = L.sm->A;  // shallow view (owned by the smoother)
            st = csr_upload(&P[l], L.P, m->stream);
            if (st == RAV_OK) st = csr_transpose(L.P, L.PT, m->stream);
        }
        if (st != RAV_OK) break;
        int64_t n = L.A.n_rows;
        cudaError_t e = cudaMalloc(&L.r, sizeof(double) * std::max<int64_t>(1, n));
        if (e == cudaSuccess && l < n_levels - 1) {
            e = cudaMalloc(&L.x, sizeof(double) * std::max<int64_t>(1, n));
            if (e == cudaSuccess) e = cudaMalloc(&L.b, sizeof(double) * std::max<int64_t>(1, n));
        }
        if (e != cudaSuccess) { set_error("mg_setup: %s", cudaGetErrorString(e)); st = RAV_ERR_OOM; }
    }
    if (st == RAV_OK) {
        int64_t cap = residual_norm_blocks();
        for (auto& L : m->lv) cap = std::max(cap, residual_part_capacity(L.A));
        m->part_cap = (int)cap;
        cudaError_t e = cudaMalloc(&m->part, sizeof(double) * cap);
        if (e == cudaSuccess) e = cudaMalloc(&m->norm2, sizeof(double));
        if (e == cudaSuccess) e = cudaMallocHost(&m->h_norm2, sizeof(double));
        if (e != cudaSuccess) { set_error("mg_setup: %s", cudaGetErrorString(e)); st = RAV_ERR_OOM; }
    }
    if (st != RAV_OK) {
        // the smoother contexts own their operators; avoid double frees of the views
        for (auto& L : m->lv)
            if (L.sm) L.A = Csr{};
        mg_destroy(m);
        return st;
    }
    for (auto& L : m->lv)
        if (L.sm) L.sm->stream = m->stream;
    *out = m;
    return RAV_OK;
}

rav_status mg_set_structured_transfers(mg_ctx* m, const rav_grid* grids) {
    if (!m || !grids) { set_error("mg_set_structured_transfers: NULL argument"); return RAV_ERR_ARG; }
    std::vector<XStruct> xs(m->L);
    for (int l = 1; l < m->L; ++l) {
        mg_level& L = m->lv[l];
        RAV_TRY(xs_build(&grids[l], &grids[l - 1], L.P.n_rows, L.P.n_cols, xs[l]));
        RAV_TRY(xs_verify(xs[l], L.P, L.PT, m->stream));
    }
    for (int l = 1; l < m->L; ++l) m->lv[l].xs = xs[l];
    m->cyc.reset();   // the captured cycle used the CSR transfers
    return RAV_OK;
}

rav_status mg_set_stream(mg_ctx* m, void* stream) {
    if (!m) { set_error("NULL ctx"); return RAV_ERR_ARG; }
    if (m->stream != as_stream(stream)) m->cyc.reset();
    m->stream = as_stream(stream);
    for (auto& L : m->lv)
        if (L.sm) rav_set_stream(L.sm, stream);
    return RAV_OK;
}

}  // extern "C"

namespace rav {

// V-cycle on level l (Fig. 1): x and b are the level's iterate / rhs
// x_zero: x is zero on entry (every level below the finest; FGMRES's z_j), see smooth_launches
rav_status vcycle_launches(mg_ctx* m, int l, double* x, const double* b, int pre, int post, double omega,
                           bool r_ready, bool x_zero) {
    cudaStream_t s = m->stream;
    if (l == 0) return launch_coarse_solve(m->C, b, x, s);
    mg_level& L = m->lv[l];
    mg_level& Lc = m->lv[l - 1];
    RAV_TRY(smooth_launches(L.sm, x, b, pre, omega, r_ready, x_zero));
    if (pre == 0 && r_ready) RAV_CUDA(cudaMemcpyAsync(L.r, L.sm->r, sizeof(double) * L.A.n_rows, cudaMemcpyDeviceToDevice, s));
    else RAV_TRY(launch_residual(L.A, x, b, L.r, s));
    if (L.xs.on && L.xs.dim == 2) RAV_TRY(launch_xs_restrict(L.xs, L.r, Lc.b, s));   // b_{l-1} = P^T r_l
    else RAV_TRY(launch_spmv(L.PT, L.r, Lc.b, 1.0, 0.0, s));
    if (l - 1 > 0) RAV_CUDA(cudaMemsetAsync(Lc.x, 0, sizeof(double) * Lc.A.n_rows, s));
    RAV_TRY(vcycle_launches(m, l - 1, Lc.x, Lc.b, pre, post, omega, false, l - 1 > 0));
    if (L.xs.on) RAV_TRY(launch_xs_prolong(L.xs, Lc.x, x, 1.0, 1.0, s));   // x_l += P x_{l-1}
    else RAV_TRY(launch_spmv(L.P, Lc.x, x, 1.0, 1.0, s));
    RAV_TRY(smooth_launches(L.sm, x, b, post, omega));
    return RAV_OK;
}

// one cycle whose first smoothing sweep reuses the residual of the previous stopping test,
// then the stopping test's residual (kept in the smoother's r for the next cycle) + its norm
static rav_status cycle_and_norm(mg_ctx* m, double* x, const double* b, int pre, int post, double omega) {
    mg_level& F = m->lv[m->L - 1];
    const bool reuse = F.sm && F.sm->variant != RAV_VARIANT_MV;
    RAV_TRY(vcycle_launches(m, m->L - 1, x, b, pre, post, omega, reuse));
    if (reuse)
        RAV_TRY(launch_residual_and_norm2(F.A, x, b, F.sm->r, m->part, m->part_cap, m->norm2, m->stream));
    else
        RAV_TRY(launch_residual_norm2(F.A, x, b, m->part, m->part_cap, m->norm2, m->stream));
    RAV_CUDA(cudaMemcpyAsync(m->h_norm2, m->norm2, sizeof(double), cudaMemcpyDeviceToHost, m->stream));
    return RAV_OK;
}

}  // namespace rav

extern "C" {

rav_status mg_vcycle(mg_ctx* m, double* x, const double* b, int pre, int post, double omega) {
    NvtxRange nvtx_range("mg_vcycle");
    if (!m || !x || !b || pre < 0 || post < 0) { set_error("mg_vcycle: bad argument"); return RAV_ERR_ARG; }
    g_launches = 0;
    if (m->L == 1) {
        RAV_TRY(launch_coarse_solve(m->C, b, x, m->stream));
        m->last_launches = g_launches;
        return RAV_OK;
    }
    RAV_TRY(vcycle_launches(m, m->L - 1, x, b, pre, post, omega));
    m->last_launches = g_launches;
    return RAV_OK;
}

rav_status mg_solve(mg_ctx* m, double* x, const double* b, int pre, int post, double omega, double rtol, int maxit,
                    int* iters, double* hist) {
    NvtxRange nvtx_range("mg_solve");
    if (!m || !x || !b || maxit < 0 || pre < 0 || post < 0) { set_error("mg_solve: bad argument"); return RAV_ERR_ARG; }
    g_launches = 0;
    int64_t total = 0;
    mg_level& F = m->lv[m->L - 1];
    const int64_t n = F.A.n_rows;
    bool dx = is_device_ptr(x), db = is_device_ptr(b);
    if (dx != db) { set_error("mg_solve: x and b must both be device or both host pointers"); return RAV_ERR_ARG; }
    double* X = x;
    const double* B = b;
    cudaStream_t s = m->stream;
    if (!dx) {
        if (!m->hx) {
            RAV_CUDA(cudaMalloc(&m->hx, sizeof(double) * n));
            RAV_CUDA(cudaMalloc(&m->hb, sizeof(double) * n));
        }
        RAV_CUDA(cudaMemcpyAsync(m->hx, x, sizeof(double) * n, cudaMemcpyHostToDevice, s));
        RAV_CUDA(cudaMemcpyAsync(m->hb, b, sizeof(double) * n, cudaMemcpyHostToDevice, s));
        X = m->hx;
        B = m->hb;
    }
    if (m->L > 1 && F.sm->variant != RAV_VARIANT_MV)   // r0 stays in the smoother's r for the first sweep
        RAV_TRY(launch_residual_and_norm2(F.A, X, B, F.sm->r, m->part, m->part_cap, m->norm2, s));
    else
        RAV_TRY(launch_residual_norm2(F.A, X, B, m->part, m->part_cap, m->norm2, s));
    RAV_CUDA(cudaMemcpyAsync(m->h_norm2, m->norm2, sizeof(double), cudaMemcpyDeviceToHost, s));
    RAV_CUDA(cudaStreamSynchronize(s));
    total += g_launches;
    double r0 = sqrt(*m->h_norm2);
    if (hist) hist[0] = r0;
    int k = 0;
    rav_status st = RAV_OK;
    if (!(r0 == r0) || isinf(r0)) st = RAV_ERR_DIVERGED;
    bool use_graph = s != nullptr && m->L > 1;
    while (st == RAV_OK && r0 > 0.0 && k < maxit) {
        int64_t launches = 0;
        st = run_graph(m->cyc, s, use_graph, X, B, pre, post, 0, omega, launches,
                       [&]() { return cycle_and_norm(m, X, B, pre, post, omega); });
        if (st != RAV_OK) break;
        total += launches;
        cudaError_t e = cudaStreamSynchronize(s);
        if (e != cudaSuccess) { set_error("mg_solve: %s", cudaGetErrorString(e)); st = RAV_ERR_CUDA; break; }
        double rk = sqrt(*m->h_norm2);
        ++k;
        if (hist) hist[k] = rk;
        if (!(rk == rk) || isinf(rk)) { set_error("mg_solve: residual is not finite at cycle %d", k); st = RAV_ERR_DIVERGED; break; }
        if (rk <= rtol * r0) break;
    }
    if (iters) *iters = k;
    if (!dx && st == RAV_OK) {
        RAV_CUDA(cudaMemcpyAsync(x, m->hx, sizeof(double) * n, cudaMemcpyDeviceToHost, s));
        RAV_CUDA(cudaStreamSynchronize(s));
    }
    m->last_launches = total;
    return st;
}

int64_t mg_last_launches(const mg_ctx* m) { return m ? m->last_launches : 0; }

rav_status mg_cycle_bytes(const mg_ctx* m, int pre, int post, double* bytes) {
    if (!m || !bytes || pre < 0 || post < 0) { set_error("mg_cycle_bytes: bad arguments"); return RAV_ERR_ARG; }
    double tot = 0.0;
    for (int l = 1; l < m->L; ++l) {
        const mg_level& L = m->lv[l];
        const double nf = (double)L.A.n_rows, nc = (double)m->lv[l - 1].A.n_rows;
        double bs = 0.0, br = 0.0;
        RAV_TRY(rav_sweep_bytes(L.sm, &bs, &br, nullptr));
        // residual launches: one per sweep but the first below the finest level (x = 0: it reads b),
        // + the restriction's; the finest level's first sweep reuses the stopping test's residual,
        // which mg_solve adds (same count)
        const int nres = pre + post + (l == m->L - 1 ? 1 : 0);
        tot += (pre + post) * bs + nres * br;
        if (L.xs.on) tot += 8.0 * (nc + 2.0 * nf) + (L.xs.dim == 2 ? 8.0 * (nf + nc) : 12.0 * L.PT.nnz + 8.0 * (nf + 2.0 * nc));
        else tot += 2.0 * (12.0 * (double)L.P.nnz) + 8.0 * (3.0 * nf + 2.0 * nc);
        if (l - 1 > 0) tot += 8.0 * nc;   // zeroing the coarse correction
    }
    tot += 8.0 * (double)m->C.m * (double)m->C.m;   // the coarse solve's explicit inverse
    *bytes = tot;
    return RAV_OK;
}

rav_status mg_normalize_pressure(mg_ctx* m, double* x, int mode) {
    if (!m || !x || (mode != 0 && mode != 1)) { set_error("mg_normalize_pressure: bad argument"); return RAV_ERR_ARG; }
    if (!is_device_ptr(x)) { set_error("mg_normalize_pressure: x must be a device pointer"); return RAV_ERR_ARG; }
    mg_level& F = m->lv[m->L - 1];
    if (F.nvel <= 0 || F.nvel >= F.A.n_rows) {
        set_error("mg_normalize_pressure: the finest level has no pressure block (n_vel not given at mg_setup)");
        return RAV_ERR_ARG;
    }
    g_launches = 0;
    RAV_TRY(launch_pressure_normalize(x, F.nvel, F.A.n_rows, mode, F.nvel, m->norm2, m->part, m->stream));
    m->last_launches = g_launches;
    return RAV_OK;
}

rav_status mg_set_colors(mg_ctx* m, int level, int n_colors, const int64_t* color_offs, const int32_t* patch_ids) {
    if (!m || level < 1 || level >= m->L) { set_error("mg_set_colors: bad level"); return RAV_ERR_ARG; }
    RAV_TRY(rav_set_colors(m->lv[level].sm, n_colors, color_offs, patch_ids));
    m->cyc.reset();
    return RAV_OK;
}

}  // extern "C"

// ------------------------------------------------------------------------------------
// transfers and reductions for host-driven (multi-rank) cycles
// ------------------------------------------------------------------------------------

struct rav_xfer {
    Csr P, PT;
    XStruct xs;
    cudaStream_t stream = nullptr;
    int64_t last_launches = 0;
};

extern "C" {

rav_status rav_xfer_setup(const rav_csr* P, void* stream, rav_xfer** out) {
    if (!P || !out) { set_error("rav_xfer_setup: NULL argument"); return RAV_ERR_ARG; }
    *out = nullptr;
    rav_xfer* t = new rav_xfer();
    t->stream = as_stream(stream);
    rav_status st = csr_upload(P, t->P, t->stream);
    if (st == RAV_OK) st = csr_transpose(t->P, t->PT, t->stream);
    if (st != RAV_OK) { rav_xfer_destroy(t); return st; }
    *out = t;
    return RAV_OK;
}

rav_status rav_prolong(rav_xfer* t, const double* xc, double* xf, double alpha) {
    if (!t || !xc || !xf) { set_error("rav_prolong: NULL argument"); return RAV_ERR_ARG; }
    g_launches = 0;
    if (t->xs.on) RAV_TRY(launch_xs_prolong(t->xs, xc, xf, alpha, 1.0, t->stream));
    else RAV_TRY(launch_spmv(t->P, xc, xf, alpha, 1.0, t->stream));
    t->last_launches = g_launches;
    return RAV_OK;
}

rav_status rav_restrict(rav_xfer* t, const double* rf, double* bc) {
    if (!t || !rf || !bc) { set_error("rav_restrict: NULL argument"); return RAV_ERR_ARG; }
    g_launches = 0;
    if (t->xs.on && t->xs.dim == 2) RAV_TRY(launch_xs_restrict(t->xs, rf, bc, t->stream));
    else RAV_TRY(launch_spmv(t->PT, rf, bc, 1.0, 0.0, t->stream));
    t->last_launches = g_launches;
    return RAV_OK;
}

rav_status rav_xfer_set_structured(rav_xfer* t, const rav_grid* fine, const rav_grid* coarse) {
    if (!t || !fine || !coarse) { set_error("rav_xfer_set_structured: NULL argument"); return RAV_ERR_ARG; }
    XStruct S;
    RAV_TRY(xs_build(fine, coarse, t->P.n_rows, t->P.n_cols, S));
    RAV_TRY(xs_verify(S, t->P, t->PT, t->stream));
    t->xs = S;
    return RAV_OK;
}

rav_status rav_xfer_set_stream(rav_xfer* t, void* stream) {
    if (!t) { set_error("NULL xfer"); return RAV_ERR_ARG; }
    t->stream = as_stream(stream);
    return RAV_OK;
}

void rav_xfer_destroy(rav_xfer* t) {
    if (!t) return;
    if (t->stream) cudaStreamSynchronize(t->stream);
    else cudaDeviceSynchronize();
    csr_free(t->P);
    csr_free(t->PT);
    delete t;
}

rav_status rav_dot(const double* a, const double* b, int64_t n, double* out, int accumulate, void* stream) {
    if (n < 0 || !out || (n > 0 && (!a || !b))) { set_error("rav_dot: bad argument"); return RAV_ERR_ARG; }
    g_launches = 0;
    static thread_local double* part = nullptr;
    const int nblk = residual_norm_blocks();
    if (!part) RAV_CUDA(cudaMalloc(&part, sizeof(double) * nblk));
    return launch_dot(a, b, n, part, nblk, out, accumulate, as_stream(stream));
}

}  // extern "C"

// ------------------------------------------------------------------------------------
// flexible GMRES with the V-cycle as preconditioner (reading R19)
// ------------------------------------------------------------------------------------

namespace rav {

static rav_status kry_alloc(mg_ctx* m, int restart, int64_t n) {
    if (m->kry_m == restart && m->kV) return RAV_OK;
    for (double** p : {&m->kV, &m->kZ, &m->kw, &m->kr, &m->kh, &m->kpart, &m->kzero, &m->kmd})
        if (*p) { cudaFree(*p); *p = nullptr; }
    RAV_CUDA(cudaMalloc(&m->kV, sizeof(double) * (size_t)(restart + 1) * n));
    RAV_CUDA(cudaMalloc(&m->kZ, sizeof(double) * (size_t)restart * n));
    RAV_CUDA(cudaMalloc(&m->kw, sizeof(double) * n));
    RAV_CUDA(cudaMalloc(&m->kr, sizeof(double) * n));
    RAV_CUDA(cudaMalloc(&m->kh, sizeof(double) * (2 * (restart + 1) + 2)));
    RAV_CUDA(cudaMalloc(&m->kpart, sizeof(double) * residual_norm_blocks()));
    RAV_CUDA(cudaMalloc(&m->kzero, sizeof(double) * n));
    RAV_CUDA(cudaMemset(m->kzero, 0, sizeof(double) * n));
    RAV_CUDA(cudaMalloc(&m->kmd, sizeof(double) * (size_t)multi_dot_blocks() * multi_dot_max()));
    m->kry_m = restart;
    return RAV_OK;
}

// *out (host) = ||v||_2
static rav_status kry_norm(mg_ctx* m, const double* v, int64_t n, double* dev_slot, double* out) {
    RAV_TRY(launch_dot(v, v, n, m->kpart, residual_norm_blocks(), dev_slot, 0, m->stream));
    RAV_CUDA(cudaMemcpyAsync(out, dev_slot, sizeof(double), cudaMemcpyDeviceToHost, m->stream));
    RAV_CUDA(cudaStreamSynchronize(m->stream));
    *out = sqrt(*out);
    return RAV_OK;
}

}  // namespace rav

extern "C" rav_status mg_fgmres(mg_ctx* m, double* x, const double* b, int pre, int post, double omega, int restart,
                                double rtol, int maxit, int* iters, double* hist) {
    rav::NvtxRange nvtx_range("mg_fgmres");
    using namespace rav;
    if (!m || !x || !b || restart < 1 || restart > 200 || maxit < 0 || pre < 0 || post < 0) {
        set_error("mg_fgmres: bad argument");
        return RAV_ERR_ARG;
    }
    if (!is_device_ptr(x) || !is_device_ptr(b)) { set_error("mg_fgmres: x and b must be device pointers"); return RAV_ERR_ARG; }
    g_launches = 0;
    cudaStream_t s = m->stream;
    mg_level& F = m->lv[m->L - 1];
    const int64_t n = F.A.n_rows;
    RAV_TRY(kry_alloc(m, restart, n));
    const int M = restart;
    double* V = m->kV;
    double* Z = m->kZ;
    double* hd = m->kh;                       // [0, M+1): pass-1 dots, [M+1, 2M+2): pass-2 dots, [2M+2]: norm
    std::vector<double> H((size_t)(M + 1) * M), cs(M), sn(M), g(M + 1), hh(2 * (M + 1) + 1), y(M);
    RAV_TRY(launch_residual(F.A, x, b, m->kr, s));
    double beta = 0.0;
    RAV_TRY(kry_norm(m, m->kr, n, hd + 2 * M + 2, &beta));
    const double r0 = beta;
    if (hist) hist[0] = r0;
    int k = 0;
    rav_status st = RAV_OK;
    if (!(r0 == r0) || isinf(r0)) st = RAV_ERR_DIVERGED;
    bool done = r0 == 0.0;
    while (st == RAV_OK && !done && k < maxit) {
        RAV_TRY(launch_scale(n, m->kr, 1.0 / beta, V, s));
        std::fill(H.begin(), H.end(), 0.0);
        std::fill(g.begin(), g.end(), 0.0);
        g[0] = beta;
        int j = 0, jn = 0;
        for (j = 0; j < M; ++j) {
            double* vj = V + (size_t)j * n;
            double* zj = Z + (size_t)j * n;
            RAV_CUDA(cudaMemsetAsync(zj, 0, sizeof(double) * n, s));
            if (m->L == 1) RAV_TRY(launch_coarse_solve(m->C, vj, zj, s));
            else RAV_TRY(vcycle_launches(m, m->L - 1, zj, vj, pre, post, omega, false, true));   // z_j = M^{-1} v_j
            // w' = -L z_j through the level's residual kernel (node-blocked, ~half the CSR bytes) with a zero
            // right-hand side.  The sign is not flipped back: CGS on w' gives h'_i = -h_i and leaves -w, so
            // the Hessenberg column takes -(h'_1 + h'_2) and v_{j+1} = w' / (-||w'||).
            RAV_TRY(launch_residual(F.A, zj, m->kzero, m->kw, s));
            for (int pass = 0; pass < 2; ++pass) {                                    // CGS2
                double* hp = hd + pass * (M + 1);
                if (j + 1 <= multi_dot_max()) {   // all projections in one pass over w
                    RAV_TRY(launch_multi_dot(n, j + 1, V, n, m->kw, m->kmd, hp, s));
                } else {
                    for (int i = 0; i <= j; ++i)
                        RAV_TRY(launch_dot(V + (size_t)i * n, m->kw, n, m->kpart, residual_norm_blocks(), hp + i, 0, s));
                }
                RAV_TRY(launch_multi_axpy(n, j + 1, V, n, hp, -1.0, m->kw, s));
            }
            RAV_TRY(launch_dot(m->kw, m->kw, n, m->kpart, residual_norm_blocks(), hd + 2 * M + 2, 0, s));
            RAV_CUDA(cudaMemcpyAsync(hh.data(), hd, sizeof(double) * (2 * (M + 1) + 1), cudaMemcpyDeviceToHost, s));
            RAV_CUDA(cudaStreamSynchronize(s));
            for (int i = 0; i <= j; ++i) H[(size_t)i * M + j] = -(hh[i] + hh[M + 1 + i]);
            const double hn = sqrt(hh[2 * M + 2]);
            H[(size_t)(j + 1) * M + j] = hn;
            for (int i = 0; i < j; ++i) {   // previous Givens rotations
                const double a = H[(size_t)i * M + j], c = H[(size_t)(i + 1) * M + j];
                H[(size_t)i * M + j] = cs[i] * a + sn[i] * c;
                H[(size_t)(i + 1) * M + j] = -sn[i] * a + cs[i] * c;
            }
            const double a = H[(size_t)j * M + j], c = H[(size_t)(j + 1) * M + j];
            const double rr = hypot(a, c);
            cs[j] = rr > 0.0 ? a / rr : 1.0;
            sn[j] = rr > 0.0 ? c / rr : 0.0;
            H[(size_t)j * M + j] = rr;
            H[(size_t)(j + 1) * M + j] = 0.0;
            g[j + 1] = -sn[j] * g[j];
            g[j] = cs[j] * g[j];
            const double res = fabs(g[j + 1]);
            ++k;
            if (hist) hist[k] = res;
            jn = j + 1;
            if (!(res == res) || isinf(res)) { set_error("mg_fgmres: residual is not finite at step %d", k); st = RAV_ERR_DIVERGED; break; }
            if (res <= rtol * r0 || k >= maxit || hn == 0.0) { done = true; break; }
            RAV_TRY(launch_scale(n, m->kw, -1.0 / hn, V + (size_t)(j + 1) * n, s));
        }
        if (st != RAV_OK) break;
        // y = H^{-1} g (upper triangular, jn x jn); x += Z y
        for (int i = jn - 1; i >= 0; --i) {
            double t = g[i];
            for (int q = i + 1; q < jn; ++q) t -= H[(size_t)i * M + q] * y[q];
            y[i] = t / H[(size_t)i * M + i];
        }
        RAV_CUDA(cudaMemcpyAsync(hd, y.data(), sizeof(double) * jn, cudaMemcpyHostToDevice, s));
        RAV_TRY(launch_multi_axpy(n, jn, Z, n, hd, 1.0, x, s));
        RAV_TRY(launch_residual(F.A, x, b, m->kr, s));
        RAV_TRY(kry_norm(m, m->kr, n, hd + 2 * M + 2, &beta));
        // the stopping test and the reported history use the TRUE residual ||b - L x|| after the update,
        // not only the least-squares estimate: an estimate that met rtol while the true residual did
        // not triggers a restart
        if (hist) hist[k] = beta;
        if (!(beta == beta) || isinf(beta)) { set_error("mg_fgmres: residual is not finite at step %d", k); st = RAV_ERR_DIVERGED; break; }
        if (done && beta > rtol * r0 && k < maxit) done = false;
    }
    if (iters) *iters = k;
    m->last_launches = g_launches;
    return st;
}
