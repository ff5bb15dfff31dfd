// ctx.cuh -- the smoother / multigrid context structures of the C-ABI (include/ravgmg.h),
// shared by api.cu (single-domain entry points) and dist.cu (the slab-partitioned
// multi-subdomain cycle, which drives the same contexts per subdomain).
#pragma once
#include <vector>

#include "internal.cuh"

namespace rav {

// A captured sequence of launches, keyed by its arguments.
struct GraphCache {
    cudaGraphExec_t exec = nullptr;
    cudaGraph_t graph = nullptr;
    const void* k0 = nullptr;
    const void* k1 = nullptr;
    int i0 = -1, i1 = -1, i2 = -1;
    double d0 = 0.0;
    int64_t nodes = 0;
    bool match(const void* a, const void* b, int x, int y, int z, double w) const {
        return exec && a == k0 && b == k1 && x == i0 && y == i1 && z == i2 && w == d0;
    }
    void reset() {
        if (exec) cudaGraphExecDestroy(exec);
        if (graph) cudaGraphDestroy(graph);
        exec = nullptr;
        graph = nullptr;
    }
};

}  // namespace rav

using namespace rav;

struct rav_ctx {
    Csr A;
    PatchSet P;
    Factors F;
    int variant = 0;
    int64_t nvel = 0;
    cudaStream_t stream = nullptr;
    double* r = nullptr;        // residual work vector
    double* hx = nullptr;       // staging for host x / b
    double* hb = nullptr;
    // rav_smooth_batch: a second staging pair, a copy stream and per-slot events (the copies of
    // one problem overlap the sweeps of the next)
    double* hx2 = nullptr;
    double* hb2 = nullptr;
    cudaStream_t cstream = nullptr;
    cudaEvent_t ev_in[2] = {nullptr, nullptr}, ev_done[2] = {nullptr, nullptr};
    // captured sweep chains for the two most recent (x, b, nu, omega) keys: a caller that alternates
    // between two buffer pairs (double-buffered host transfers) replays without re-capturing
    GraphCache graph[2];
    int graph_next = 0;         // entry to replace on a miss
    void graphs_reset() { graph[0].reset(); graph[1].reset(); }
    int64_t last_launches = 0;
    // multicoloured MV (RAV_VARIANT_MV): colour c = patches plist[coffs[c] .. coffs[c+1])
    std::vector<int64_t> coffs;
    int32_t* plist = nullptr;
};

struct mg_level {
    rav_ctx* sm = nullptr;  // smoother (levels >= 1)
    Csr A;                  // level operator (owned by sm for l >= 1; own copy at l = 0)
    Csr P, PT;              // prolongation from l-1 and its transpose (restriction)
    XStruct xs;             // stencil form of P (mg_set_structured_transfers), used when xs.on
    double* x = nullptr;    // level iterate (l < L-1)
    double* b = nullptr;    // level right-hand side (l < L-1)
    double* r = nullptr;    // level residual
    int64_t nvel = 0;       // DoFs < nvel are velocity
};

struct mg_ctx {
    int L = 0;
    std::vector<mg_level> lv;
    CoarseLU C;
    cudaStream_t stream = nullptr;
    double* part = nullptr;     // residual-norm partials
    int part_cap = 0;           // their number (full grid of the finest fused residual kernel)
    double* norm2 = nullptr;    // device scalar
    double* h_norm2 = nullptr;  // pinned host scalar
    double* hx = nullptr;
    double* hb = nullptr;
    GraphCache cyc;             // one V-cycle + residual norm
    int64_t last_launches = 0;
    // FGMRES work space (mg_fgmres): V (m+1) x n, Z m x n, w, r, device coefficients
    int kry_m = 0;
    double *kV = nullptr, *kZ = nullptr, *kw = nullptr, *kr = nullptr, *kh = nullptr, *kpart = nullptr;
    double *kzero = nullptr, *kmd = nullptr;   // zero right-hand side (w = L z via the residual), multi-dot partials
};


namespace rav {

// the sweep chain of one smoother context (residual + sweep per sweep; see api.cu)
rav_status smooth_launches(rav_ctx* c, double* x, const double* b, int nu, double omega, bool r_ready = false,
                           bool x_zero = false);
// the launches of one V-cycle on level l of a multigrid context (see api.cu)
rav_status vcycle_launches(mg_ctx* m, int l, double* x, const double* b, int pre, int post, double omega,
                           bool r_ready = false, bool x_zero = false);

// run `body` either directly or through a cached CUDA graph on stream s
template <class Body>
inline rav_status run_graph(GraphCache& G, cudaStream_t s, bool use_graph, const void* k0, const void* k1, int i0,
                            int i1, int i2, double d0, int64_t& launches, Body body) {
    if (!use_graph) {
        int64_t before = g_launches;
        RAV_TRY(body());
        launches = g_launches - before;
        return RAV_OK;
    }
    if (!G.match(k0, k1, i0, i1, i2, d0)) {
        G.reset();
        int64_t before = g_launches;
        RAV_CUDA(cudaStreamBeginCapture(s, cudaStreamCaptureModeThreadLocal));
        rav_status st = body();
        cudaGraph_t g = nullptr;
        cudaError_t e = cudaStreamEndCapture(s, &g);
        if (st != RAV_OK) { if (g) cudaGraphDestroy(g); return st; }
        RAV_CUDA(e);
        G.graph = g;
        RAV_CUDA(cudaGraphInstantiate(&G.exec, g, 0));
        G.k0 = k0; G.k1 = k1; G.i0 = i0; G.i1 = i1; G.i2 = i2; G.d0 = d0;
        G.nodes = g_launches - before;
        g_launches = before;
    }
    RAV_CUDA(cudaGraphLaunch(G.exec, s));
    g_launches += G.nodes;
    launches = G.nodes;
    return RAV_OK;
}

}  // namespace rav
