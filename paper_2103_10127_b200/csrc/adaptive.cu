// adaptive.cu -- adaptive quadtree hierarchies with hanging nodes for the paper's
// stabilized Q1-Q1 pair ("hanging nodes ... are
// handled as constraints and removed from the global system of equations", P:146,
// Table 1; reading R20 in DESIGN.md).
//
// Host-side setup (mesh generation, constraints, sparse patterns); the element
// matrices are computed on the device (gen::q1_cell_matrices); every sweep, residual,
// transfer and cycle on these levels runs through the generic rav_setup / mg_setup
// path on the GPU (Schur-factored patches: the constrained velocity block is still
// I_2 (x) A_s and every patch holds one pressure DoF).
//
// Mesh: an integer lattice of N = n0 2^(L-1) units per side; level 1 = the n0 x n0
// grid; level k+1 splits every leaf of level k within bands[k-1] finest cells of the
// boundary, then restores 2:1 edge balance on a per-unit size map (split the coarser
// of any two edge-adjacent units whose sizes differ by more than 2x, until none).
// Hanging vertex: the midpoint of a leaf edge that is a corner of another leaf; its
// value is the mean of the edge's end points (recursively).  Non-hanging vertices are
// numbered by (y, x); free velocity = non-hanging, off the boundary.
#include <algorithm>
#include <cstring>
#include <map>
#include <unordered_map>
#include <unordered_set>
#include <vector>

#include "internal.cuh"

namespace rav {
namespace {

struct Cell {
    int x, y, s;
};

static inline uint64_t vkey(int x, int y) { return ((uint64_t)(uint32_t)y << 32) | (uint32_t)x; }

// per-unit size map of a leaf set (side N x N); builds the leaves back from it
struct SizeMap {
    int N;
    std::vector<int> sz;   // size of the leaf covering unit (i, j), row-major j * N + i
    explicit SizeMap(int n) : N(n), sz((size_t)n * n, 0) {}
    void paint(const Cell& c) {
        for (int j = c.y; j < c.y + c.s; ++j)
            for (int i = c.x; i < c.x + c.s; ++i) sz[(size_t)j * N + i] = c.s;
    }
    std::vector<Cell> leaves() const {
        std::vector<Cell> out;
        for (int j = 0; j < N; ++j)
            for (int i = 0; i < N; ++i) {
                const int s = sz[(size_t)j * N + i];
                if (i % s == 0 && j % s == 0) out.push_back({i, j, s});
            }
        return out;
    }
};

static void split_leaf(SizeMap& M, int i, int j) {   // the leaf covering unit (i, j)
    const int s = M.sz[(size_t)j * M.N + i];
    if (s <= 1) return;
    const int x0 = i / s * s, y0 = j / s * s;
    M.paint({x0, y0, s / 2});
    M.paint({x0 + s / 2, y0, s / 2});
    M.paint({x0, y0 + s / 2, s / 2});
    M.paint({x0 + s / 2, y0 + s / 2, s / 2});
}

static void balance_2to1(SizeMap& M) {
    const int N = M.N;
    bool changed = true;
    while (changed) {
        changed = false;
        for (int j = 0; j < N; ++j)
            for (int i = 0; i < N; ++i) {
                const int s = M.sz[(size_t)j * N + i];
                const int nb[2][2] = {{i + 1, j}, {i, j + 1}};
                for (auto& q : nb) {
                    if (q[0] >= N || q[1] >= N) continue;
                    const int t = M.sz[(size_t)q[1] * N + q[0]];
                    if (s > 2 * t) { split_leaf(M, i, j); changed = true; }
                    else if (t > 2 * s) { split_leaf(M, q[0], q[1]); changed = true; }
                }
            }
    }
}

struct Level {
    int N = 0;
    std::vector<Cell> cells;
    std::vector<int> sizes;                                  // distinct leaf sizes, descending
    std::unordered_map<uint64_t, std::pair<uint64_t, uint64_t>> hang;   // vertex -> coarse edge end points
    std::vector<uint64_t> regular;                           // non-hanging vertices by (y, x)
    std::unordered_map<uint64_t, int> vel_id, p_id;
    int64_t nvel = 0, n = 0;
    // assembled system and smoother / transfer data
    std::vector<int64_t> rp;
    std::vector<int32_t> ci;
    std::vector<double> val, rhs;
    std::vector<int64_t> poffs;
    std::vector<int32_t> pdofs;
    std::vector<double> pw;
    std::vector<int64_t> prp;
    std::vector<int32_t> pci;
    std::vector<double> pval;
};

static inline uint64_t ckey(int x, int y, int s) { return vkey(x, y) * 64 + (uint64_t)__builtin_ctz((unsigned)s); }

static const Cell* find_leaf(const Level& L, int px, int py, const std::vector<Cell>& cells,
                             const std::unordered_map<uint64_t, int>& index) {
    for (int s : L.sizes) {
        auto it = index.find(ckey(px / s * s, py / s * s, s));
        if (it != index.end()) return &cells[it->second];
    }
    return nullptr;
}

static void expand(const Level& L, uint64_t v, double w, std::map<uint64_t, double>& acc) {
    auto it = L.hang.find(v);
    if (it == L.hang.end()) { acc[v] += w; return; }
    expand(L, it->second.first, 0.5 * w, acc);
    expand(L, it->second.second, 0.5 * w, acc);
}

static void finish_mesh(Level& L) {
    const int N = L.N;
    std::unordered_set<uint64_t> verts;
    std::vector<int> sz;
    for (const Cell& c : L.cells) {
        verts.insert(vkey(c.x, c.y));
        verts.insert(vkey(c.x + c.s, c.y));
        verts.insert(vkey(c.x, c.y + c.s));
        verts.insert(vkey(c.x + c.s, c.y + c.s));
        sz.push_back(c.s);
    }
    std::sort(sz.begin(), sz.end(), std::greater<int>());
    sz.erase(std::unique(sz.begin(), sz.end()), sz.end());
    L.sizes = sz;
    for (const Cell& c : L.cells) {
        if (c.s % 2) continue;
        const int h = c.s / 2;
        const int e[4][6] = {{c.x + h, c.y, c.x, c.y, c.x + c.s, c.y},
                             {c.x + h, c.y + c.s, c.x, c.y + c.s, c.x + c.s, c.y + c.s},
                             {c.x, c.y + h, c.x, c.y, c.x, c.y + c.s},
                             {c.x + c.s, c.y + h, c.x + c.s, c.y, c.x + c.s, c.y + c.s}};
        for (auto& q : e)
            if (verts.count(vkey(q[0], q[1]))) L.hang[vkey(q[0], q[1])] = {vkey(q[2], q[3]), vkey(q[4], q[5])};
    }
    for (uint64_t v : verts)
        if (!L.hang.count(v)) L.regular.push_back(v);
    std::sort(L.regular.begin(), L.regular.end());   // key = (y << 32) | x: (y, x) order
    int nf = 0;
    for (size_t k = 0; k < L.regular.size(); ++k) {
        const uint64_t v = L.regular[k];
        const int x = (int)(uint32_t)v, y = (int)(v >> 32);
        L.p_id[v] = (int)k;
        if (x > 0 && y > 0 && x < N && y < N) L.vel_id[v] = nf++;
    }
    L.nvel = 2 * (int64_t)nf;
    L.n = L.nvel + (int64_t)L.regular.size();
}

static double lid(const Level& L, uint64_t v, int kind, int c) {
    const int x = (int)(uint32_t)v, y = (int)(v >> 32);
    return (kind == 0 && c == 0 && y == L.N && x > 0 && x < L.N) ? 1.0 : 0.0;
}

static rav_status assemble(const rav_grid* g, Level& L) {
    const int64_t nc = (int64_t)L.cells.size();
    std::vector<double> cx(nc), cy(nc), hc(nc), em((size_t)72 * nc);
    std::vector<int64_t> order(nc);
    for (int64_t c = 0; c < nc; ++c) order[c] = c;
    std::sort(order.begin(), order.end(), [&](int64_t a, int64_t b) {
        const Cell &p = L.cells[a], &q = L.cells[b];
        return p.y != q.y ? p.y < q.y : (p.x != q.x ? p.x < q.x : p.s < q.s);
    });
    for (int64_t k = 0; k < nc; ++k) {
        const Cell& c = L.cells[order[k]];
        cx[k] = (double)c.x / L.N;
        cy[k] = (double)c.y / L.N;
        hc[k] = (double)c.s / L.N;
    }
    RAV_TRY(gen::q1_cell_matrices(g, nc, cx.data(), cy.data(), hc.data(), em.data()));
    struct T {
        int64_t r, c;
        double v;
    };
    std::vector<T> trip;
    trip.reserve((size_t)nc * 200);
    L.rhs.assign(L.n, 0.0);
    for (int64_t k = 0; k < nc; ++k) {
        const Cell& c = L.cells[order[k]];
        const double* A = &em[(size_t)72 * k];
        const double* B = A + 16;
        const double* Cm = A + 48;
        const double* F = A + 64;
        std::vector<std::pair<uint64_t, double>> ex[4];
        for (int a = 0; a < 4; ++a) {
            std::map<uint64_t, double> acc;
            expand(L, vkey(c.x + (a & 1) * c.s, c.y + (a >> 1) * c.s), 1.0, acc);
            ex[a].assign(acc.begin(), acc.end());
        }
        for (int a = 0; a < 4; ++a)
            for (int comp = 0; comp < 2; ++comp)
                for (auto& ua : ex[a]) {
                    auto fv = L.vel_id.find(ua.first);
                    if (fv == L.vel_id.end()) {   // Dirichlet velocity: lift into the pressure rows
                        const double gval = lid(L, ua.first, g->kind, comp);
                        for (int m = 0; m < 4; ++m)
                            for (auto& um : ex[m])
                                L.rhs[L.nvel + L.p_id[um.first]] -= ua.second * um.second * B[(a * 2 + comp) * 4 + m] * gval;
                        continue;
                    }
                    const int64_t r = 2 * (int64_t)fv->second + comp;
                    L.rhs[r] += ua.second * F[a * 2 + comp];
                    for (int b = 0; b < 4; ++b)
                        for (auto& ub : ex[b]) {
                            const double v = ua.second * ub.second * A[a * 4 + b];
                            auto fb = L.vel_id.find(ub.first);
                            if (fb != L.vel_id.end()) trip.push_back({r, 2 * (int64_t)fb->second + comp, v});
                            else L.rhs[r] -= v * lid(L, ub.first, g->kind, comp);
                        }
                    for (int m = 0; m < 4; ++m)
                        for (auto& um : ex[m]) {
                            const double v = ua.second * um.second * B[(a * 2 + comp) * 4 + m];
                            const int64_t p = L.nvel + L.p_id[um.first];
                            trip.push_back({r, p, v});
                            trip.push_back({p, r, v});
                        }
                }
        for (int m = 0; m < 4; ++m)
            for (auto& um : ex[m])
                for (int m2 = 0; m2 < 4; ++m2)
                    for (auto& um2 : ex[m2])
                        trip.push_back({L.nvel + L.p_id[um.first], L.nvel + L.p_id[um2.first],
                                        um.second * um2.second * Cm[m * 4 + m2]});
    }
    std::stable_sort(trip.begin(), trip.end(), [](const T& a, const T& b) { return a.r != b.r ? a.r < b.r : a.c < b.c; });
    L.rp.assign(L.n + 1, 0);
    L.ci.clear();
    L.val.clear();
    for (size_t k = 0; k < trip.size();) {
        size_t e = k;
        double v = 0.0;
        while (e < trip.size() && trip[e].r == trip[k].r && trip[e].c == trip[k].c) v += trip[e++].v;
        L.ci.push_back((int32_t)trip[k].c);
        L.val.push_back(v);
        L.rp[trip[k].r + 1]++;
        k = e;
    }
    for (int64_t i = 0; i < L.n; ++i) L.rp[i + 1] += L.rp[i];
    return RAV_OK;
}

static void build_patches(Level& L) {
    L.poffs.assign(1, 0);
    L.pdofs.clear();
    L.pw.clear();
    for (uint64_t v : L.regular) {
        const int64_t p = L.nvel + L.p_id[v];
        std::vector<int32_t> rest, others;
        auto fv = L.vel_id.find(v);
        if (fv != L.vel_id.end()) rest = {2 * fv->second, 2 * fv->second + 1};
        for (int64_t k = L.rp[p]; k < L.rp[p + 1]; ++k) {
            const int32_t c = L.ci[k];
            if (c < L.nvel && std::find(rest.begin(), rest.end(), c) == rest.end()) others.push_back(c);
        }
        for (int32_t d : rest) { L.pdofs.push_back(d); L.pw.push_back(1.0); }
        L.pdofs.push_back((int32_t)p);
        L.pw.push_back(1.0);
        for (int32_t d : others) { L.pdofs.push_back(d); L.pw.push_back(0.0); }
        L.poffs.push_back((int64_t)L.pdofs.size());
    }
}

static void build_prolongation(Level& F, const Level& Cc) {
    std::unordered_map<uint64_t, int> index;
    for (size_t k = 0; k < Cc.cells.size(); ++k) index[ckey(Cc.cells[k].x, Cc.cells[k].y, Cc.cells[k].s)] = (int)k;
    auto interp = [&](uint64_t v, bool velocity) {
        const int x = (int)(uint32_t)v, y = (int)(v >> 32);
        const Cell* c = find_leaf(Cc, std::min(x, Cc.N - 1), std::min(y, Cc.N - 1), Cc.cells, index);
        const double tx = (double)(x - c->x) / c->s, ty = (double)(y - c->y) / c->s;
        std::map<uint64_t, double> acc;
        for (int a = 0; a < 4; ++a) {
            const double wa = ((a & 1) ? tx : 1.0 - tx) * ((a >> 1) ? ty : 1.0 - ty);
            if (wa == 0.0) continue;
            std::map<uint64_t, double> e;
            expand(Cc, vkey(c->x + (a & 1) * c->s, c->y + (a >> 1) * c->s), 1.0, e);
            for (auto& t : e) {
                if (velocity && !Cc.vel_id.count(t.first)) continue;   // Dirichlet columns dropped
                acc[t.first] += wa * t.second;
            }
        }
        return acc;
    };
    F.prp.assign(1, 0);
    F.pci.clear();
    F.pval.clear();
    std::vector<uint64_t> freev(F.vel_id.size());
    for (auto& kv : F.vel_id) freev[kv.second] = kv.first;
    for (uint64_t v : freev) {
        auto acc = interp(v, true);
        for (int comp = 0; comp < 2; ++comp) {
            std::vector<std::pair<int32_t, double>> row;
            for (auto& t : acc) row.push_back({2 * Cc.vel_id.at(t.first) + comp, t.second});
            std::sort(row.begin(), row.end());
            for (auto& t : row) { F.pci.push_back(t.first); F.pval.push_back(t.second); }
            F.prp.push_back((int64_t)F.pci.size());
        }
    }
    for (uint64_t v : F.regular) {
        auto acc = interp(v, false);
        std::vector<std::pair<int32_t, double>> row;
        for (auto& t : acc) row.push_back({(int32_t)(Cc.nvel + Cc.p_id.at(t.first)), t.second});
        std::sort(row.begin(), row.end());
        for (auto& t : row) { F.pci.push_back(t.first); F.pval.push_back(t.second); }
        F.prp.push_back((int64_t)F.pci.size());
    }
}

static const int kDefaultBands[] = {2, 3, 5, 8, 13, 19};   // R20 (reproduces Table 1)

}  // namespace
}  // namespace rav

struct rav_adaptive {
    std::vector<rav::Level> lv;
};

using namespace rav;

template <class Tv>
static rav_status copy_out(Tv* dst, const std::vector<Tv>& src) {
    if (!dst || src.empty()) return RAV_OK;
    RAV_CUDA(cudaMemcpy(dst, src.data(), sizeof(Tv) * src.size(), cudaMemcpyDefault));
    return RAV_OK;
}

extern "C" {

rav_status rav_adaptive_create(const rav_adaptive_desc* d, rav_adaptive** out) {
    NvtxRange nvtx_range("rav_adaptive_create");
    if (!d || !out) { set_error("rav_adaptive_create: NULL argument"); return RAV_ERR_ARG; }
    *out = nullptr;
    const rav_grid& g = d->base;
    if (g.dim != 2 || g.vel_order != 1 || !(g.beta > 0.0) || g.win) {
        set_error("rav_adaptive_create: 2D stabilized Q1-Q1 (vel_order 1, beta > 0), whole domain only");
        return RAV_ERR_ARG;
    }
    const int n0 = g.ncell[0];
    if (n0 < 1 || g.ncell[1] != n0 || g.len[0] != 1.0 || g.len[1] != 1.0) {
        set_error("rav_adaptive_create: the coarse grid must be n0 x n0 on the unit square");
        return RAV_ERR_ARG;
    }
    if (d->n_levels < 1 || d->n_levels > 12) { set_error("rav_adaptive_create: 1 <= n_levels <= 12"); return RAV_ERR_ARG; }
    const int L = d->n_levels;
    const int S1 = 1 << (L - 1);
    const int N = n0 * S1;
    if ((int64_t)N * N > (int64_t)1 << 28) { set_error("rav_adaptive_create: hierarchy too deep"); return RAV_ERR_ARG; }
    rav_adaptive* A = new rav_adaptive();
    A->lv.resize(L);
    SizeMap M(N);
    for (int j = 0; j < n0; ++j)
        for (int i = 0; i < n0; ++i) M.paint({i * S1, j * S1, S1});
    for (int k = 0; k < L; ++k) {
        if (k > 0) {   // level k -> k+1 (1-based): split the leaves within the band, then balance
            const int bk = d->bands[k - 1] > 0 ? d->bands[k - 1] : kDefaultBands[std::min(k, 6) - 1];
            const int band = d->uniform ? N + 1 : bk * (N / (n0 << (k - 1)));
            for (const Cell& c : M.leaves()) {
                const int dist = std::min(std::min(c.x, c.y), std::min(N - (c.x + c.s), N - (c.y + c.s)));
                if (dist < band && c.s > 1) split_leaf(M, c.x, c.y);
            }
            balance_2to1(M);
        }
        Level& Lk = A->lv[k];
        Lk.N = N;
        Lk.cells = M.leaves();
        finish_mesh(Lk);
        rav_status st = assemble(&g, Lk);
        if (st != RAV_OK) { delete A; return st; }
        build_patches(Lk);
        if (k > 0) build_prolongation(Lk, A->lv[k - 1]);
    }
    *out = A;
    return RAV_OK;
}

rav_status rav_adaptive_sizes(const rav_adaptive* A, int level, int64_t* n_dofs, int64_t* n_vel, int64_t* nnz,
                              int64_t* n_patches, int64_t* patch_entries, int64_t* prol_nnz, int64_t* n_cells) {
    if (!A || level < 0 || level >= (int)A->lv.size()) { set_error("rav_adaptive_sizes: bad level"); return RAV_ERR_ARG; }
    const Level& L = A->lv[level];
    if (n_dofs) *n_dofs = L.n;
    if (n_vel) *n_vel = L.nvel;
    if (nnz) *nnz = (int64_t)L.ci.size();
    if (n_patches) *n_patches = (int64_t)L.regular.size();
    if (patch_entries) *patch_entries = (int64_t)L.pdofs.size();
    if (prol_nnz) *prol_nnz = (int64_t)L.pci.size();
    if (n_cells) *n_cells = (int64_t)L.cells.size();
    return RAV_OK;
}

rav_status rav_adaptive_fill(const rav_adaptive* A, int level, int64_t* rp, int32_t* ci, double* val, double* rhs,
                             int64_t* poffs, int32_t* pdofs, double* pw, int64_t* prp, int32_t* pci, double* pval) {
    if (!A || level < 0 || level >= (int)A->lv.size()) { set_error("rav_adaptive_fill: bad level"); return RAV_ERR_ARG; }
    const Level& L = A->lv[level];
    RAV_TRY(copy_out(rp, L.rp));
    RAV_TRY(copy_out(ci, L.ci));
    RAV_TRY(copy_out(val, L.val));
    RAV_TRY(copy_out(rhs, L.rhs));
    RAV_TRY(copy_out(poffs, L.poffs));
    RAV_TRY(copy_out(pdofs, L.pdofs));
    RAV_TRY(copy_out(pw, L.pw));
    if (level > 0) {
        RAV_TRY(copy_out(prp, L.prp));
        RAV_TRY(copy_out(pci, L.pci));
        RAV_TRY(copy_out(pval, L.pval));
    }
    return RAV_OK;
}

void rav_adaptive_destroy(rav_adaptive* A) { delete A; }

}  // extern "C"

// ---- greedy multicolouring of arbitrary Vanka patches (multiplicative Vanka, R10 / R20) -------
// Patches i and j conflict when j holds a DoF of patch i or a DoF coupled to patch i through L
// (then relaxing them concurrently is not the sequential sweep).  Greedy in ascending patch
// order, smallest free colour.  Host algorithm (setup); inputs host or device.
namespace {

template <class Tv>
static rav_status to_host(std::vector<Tv>& dst, const Tv* src, int64_t n) {
    dst.resize(std::max<int64_t>(n, 0));
    if (n > 0) RAV_CUDA(cudaMemcpy(dst.data(), src, sizeof(Tv) * n, cudaMemcpyDefault));
    return RAV_OK;
}

}  // namespace

extern "C" rav_status rav_color_patches(const rav_csr* A, const rav_patches* P, int64_t* n_colors,
                                        int64_t* color_offs, int32_t* patch_ids) {
    if (!A || !P || !n_colors || !color_offs || !patch_ids || A->n_rows < 0 || P->n_patches < 0) {
        set_error("rav_color_patches: bad argument");
        return RAV_ERR_ARG;
    }
    const int64_t n = A->n_rows, np = P->n_patches;
    std::vector<int64_t> rp, po;
    std::vector<int32_t> ci, pd;
    RAV_TRY(to_host(rp, A->row_ptr, n + 1));
    RAV_TRY(to_host(ci, A->col, rp.empty() ? 0 : rp[n]));
    RAV_TRY(to_host(po, P->offs, np + 1));
    RAV_TRY(to_host(pd, P->dofs, po.empty() ? 0 : po[np]));
    // DoF -> patches holding it
    std::vector<int64_t> dp(n + 1, 0);
    for (int32_t d : pd) dp[d + 1]++;
    for (int64_t i = 0; i < n; ++i) dp[i + 1] += dp[i];
    std::vector<int32_t> dl(pd.size());
    {
        std::vector<int64_t> cur(dp.begin(), dp.end() - 1);
        for (int64_t i = 0; i < np; ++i)
            for (int64_t k = po[i]; k < po[i + 1]; ++k) dl[cur[pd[k]]++] = (int32_t)i;
    }
    std::vector<int32_t> color(np, -1);
    std::vector<int64_t> seen(np, -1);   // last patch that marked j as a neighbour
    std::vector<int64_t> used;           // colour -> last patch that found it taken
    int32_t ncol = 0;
    for (int64_t i = 0; i < np; ++i) {
        auto visit = [&](int32_t d) {
            for (int64_t q = dp[d]; q < dp[d + 1]; ++q) {
                const int32_t j = dl[q];
                if (j >= i || seen[j] == i) continue;
                seen[j] = i;
                used[color[j]] = i;
            }
        };
        for (int64_t k = po[i]; k < po[i + 1]; ++k) {
            const int32_t d = pd[k];
            visit(d);
            for (int64_t e = rp[d]; e < rp[d + 1]; ++e) visit(ci[e]);
        }
        int32_t c = 0;
        while (c < ncol && used[c] == i) ++c;
        if (c == ncol) { ++ncol; used.push_back(-1); }
        color[i] = c;
    }
    std::vector<int64_t> cnt(ncol + 1, 0);
    for (int32_t c : color) cnt[c + 1]++;
    for (int c = 0; c < ncol; ++c) cnt[c + 1] += cnt[c];
    for (int c = 0; c <= ncol; ++c) color_offs[c] = cnt[c];
    std::vector<int64_t> cur(cnt.begin(), cnt.end() - 1);
    for (int64_t i = 0; i < np; ++i) patch_ids[cur[color[i]]++] = (int32_t)i;
    *n_colors = ncol;
    return RAV_OK;
}
