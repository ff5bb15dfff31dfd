// nb.cu -- node-blocked copy of a Taylor-Hood level operator for the residual
// r = b - L x (Eq. 10).
//
// For the Laplacian-form viscous term (Eq. 7) the velocity block of L is
// I_d (x) A_s: the rows of the d components of a node carry the same columns
// (shifted by the component) and bitwise-equal values, and they share their
// pressure columns.  The node-blocked copy stores, per velocity NODE row j:
//   A entries  (node k, a_jk)            one value for all components
//   B entries  (pressure p, b_jp^c c<d)  d values per column
// and per pressure row v:
//   BT entries (node k, b_vk^c c<d)      d values per node
// i.e. 12*nnz(A)/d + (4 + 8d)*nnz(B)/d*2 bytes instead of 12*nnz: -35% at c2.
// Block rows are sorted by length in windows of 4096 and stored as SELL slices
// of 32 rows (column-major), one thread per block row producing all d residual
// components (x gathered as d contiguous values).  For d = 2 the values are
// stored as 16-byte pairs per slot (two consecutive A entries; the two
// components of a B / BT entry), so a warp-wide load moves 512 contiguous bytes.  Each component sums its A
// entries then its B entries in ascending column order -- the CSR order -- so
// the result equals the CSR residual up to FMA contraction.
//
// nb_build verifies the structure (d divides n_vel, component rows with equal
// patterns/values, no cross-component entries, pressure rows with complete
// node groups); on failure the SELL copy is used instead.
#include <algorithm>
#include <vector>
#include <cub/cub.cuh>

#include "internal.cuh"

namespace rav {

constexpr int NB_C = 32;
constexpr int NB_SIGMA = 4096;

// per block row: (#A entries, #B entries) for node rows, (#BT entries, 0) for pressure rows
__global__ void nb_count_kernel(int64_t nnodes, int64_t npres, int D, int64_t nvel, const int64_t* rp,
                                const int32_t* ci, const double* val, int32_t* na, int32_t* nb,
                                unsigned int* fail) {
    const int64_t total = nnodes + npres;
    for (int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; t < total; t += (int64_t)gridDim.x * blockDim.x) {
        if (t < nnodes) {
            const int64_t r0 = t * D;
            const int64_t s0 = rp[r0], e0 = rp[r0 + 1];
            int a = 0, b = 0;
            for (int64_t k = s0; k < e0; ++k) {
                const int c = ci[k];
                if (c < nvel) {
                    if (c % D != 0) atomicOr(fail, 1u);
                    ++a;
                } else {
                    ++b;
                }
            }
            for (int cc = 1; cc < D; ++cc) {       // rows of the other components: same pattern, same values
                const int64_t s = rp[r0 + cc], e = rp[r0 + cc + 1];
                if (e - s != e0 - s0) { atomicOr(fail, 1u); continue; }
                for (int64_t k = 0; k < e - s; ++k) {
                    const int c0 = ci[s0 + k], c1 = ci[s + k];
                    if (c0 < nvel) {
                        if (c1 != c0 + cc || val[s + k] != val[s0 + k]) atomicOr(fail, 1u);
                    } else if (c1 != c0) {
                        atomicOr(fail, 1u);
                    }
                }
            }
            na[t] = a;
            nb[t] = b;
        } else {
            const int64_t row = nvel + (t - nnodes);
            const int64_t s = rp[row], e = rp[row + 1];
            if ((e - s) % D != 0) atomicOr(fail, 1u);
            for (int64_t k = s; k < e; ++k)
                if (ci[k] >= nvel || ci[k] % D != (k - s) % D || ((k - s) % D != 0 && ci[k] != ci[k - 1] + 1))
                    atomicOr(fail, 1u);
            na[t] = 0;                         // pressure rows: only "B-type" entries (node, d values)
            nb[t] = (int32_t)((e - s) / D);
        }
    }
}

__global__ void nb_key_kernel(int64_t n, const int32_t* na, const int32_t* nb, int D,
                              int32_t* key, int32_t* idx) {
    for (int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; t < n; t += (int64_t)gridDim.x * blockDim.x) {
        const int32_t br = (int32_t)t;
        key[t] = na[br] * 12 + nb[br] * (4 + 8 * D);   // bytes of the block row
        idx[t] = br;
    }
}


__global__ void nb_windows_kernel(int64_t n, int64_t nw, int64_t* off) {
    for (int64_t w = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; w <= nw; w += (int64_t)gridDim.x * blockDim.x)
        off[w] = w * NB_SIGMA < n ? w * NB_SIGMA : n;
}

// per slice: widths (max over its 32 rows) and sizes in bytes-units
__global__ void nb_slice_kernel(int64_t n, int64_t nslices, int D, const int32_t* perm, const int32_t* na,
                                const int32_t* nb, int32_t* wa, int32_t* wb, int64_t* scol, int64_t* sval) {
    for (int64_t s = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; s < nslices; s += (int64_t)gridDim.x * blockDim.x) {
        int a = 0, b = 0;
        for (int l = 0; l < NB_C; ++l) {
            const int64_t t = s * NB_C + l;
            if (t < n) {
                a = max(a, na[perm[t]]);
                b = max(b, nb[perm[t]]);
            }
        }
        wa[s] = a;
        wb[s] = b;
        scol[s] = (int64_t)NB_C * (a + b);
        sval[s] = (int64_t)NB_C * (a + (int64_t)b * D);
    }
}

// value layout of a slice of width (A, B), lane l, relative to the slice's first value:
//   plain: A entry k at k*32 + l; B entry (k, c) at A*32 + (k*D + c)*32 + l
//   pair (D = 2): A entries (2p, 2p+1) at (p*32 + l)*2 + {0,1}, an odd last A entry at
//                 (A & ~1)*32 + l; B entry (k, c) at A*32 + (k*32 + l)*2 + c
// Both occupy 32*(A + D*B) values; the pair layout keeps every 16-byte slot pair contiguous.
__device__ __forceinline__ int64_t nb_ia(bool pair, int A, int k, int l) {
    if (!pair) return (int64_t)k * NB_C + l;
    const int A2 = A & ~1;
    return k < A2 ? ((int64_t)(k >> 1) * NB_C + l) * 2 + (k & 1) : (int64_t)A2 * NB_C + l;
}
__device__ __forceinline__ int64_t nb_ib(bool pair, int D, int A, int k, int c, int l) {
    return (int64_t)A * NB_C + (pair ? ((int64_t)k * NB_C + l) * 2 + c : ((int64_t)k * D + c) * NB_C + l);
}

// slot t = 32 s + l; node rows: A cols/vals then B cols / D vals; pressure rows: BT cols (node dof of comp 0) / D vals
__global__ void nb_fill_kernel(int64_t n, int64_t nnodes, int64_t nslices, int D, int64_t nvel, const int64_t* rp,
                               const int32_t* ci, const double* val, const int32_t* perm, const int32_t* wa,
                               const int32_t* wb, const int64_t* cptr, const int64_t* vptr, int32_t* col,
                               double* v, int pair_i) {
    const bool pair = pair_i != 0;
    const int64_t total = nslices * NB_C;
    for (int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; t < total; t += (int64_t)gridDim.x * blockDim.x) {
        const int64_t s = t / NB_C;
        const int l = (int)(t % NB_C);
        const int A = wa[s], B = wb[s];
        int32_t* cA = col + cptr[s] + l;
        int32_t* cB = cA + (int64_t)A * NB_C;
        double* vs = v + vptr[s];
#define NB_VA(k) vs[nb_ia(pair, A, (k), l)]
#define NB_VB(k, c) vs[nb_ib(pair, D, A, (k), (c), l)]
        if (t >= n) {
            for (int k = 0; k < A; ++k) { cA[k * NB_C] = 0; NB_VA(k) = 0.0; }
            for (int k = 0; k < B; ++k) {
                cB[k * NB_C] = 0;
                for (int c = 0; c < D; ++c) NB_VB(k, c) = 0.0;
            }
            continue;
        }
        const int64_t br = perm[t];
        if (br < nnodes) {
            const int64_t r0 = br * D;
            const int64_t s0 = rp[r0], e0 = rp[r0 + 1];
            int a = 0, b = 0;
            for (int64_t k = s0; k < e0; ++k) {
                const int c = ci[k];
                if (c < nvel) {
                    cA[a * NB_C] = c;
                    NB_VA(a) = val[k];
                    ++a;
                } else {
                    cB[b * NB_C] = c;
                    for (int cc = 0; cc < D; ++cc) NB_VB(b, cc) = val[rp[r0 + cc] + (k - s0)];
                    ++b;
                }
            }
            // padding entries (value 0) repeat the row's first column: offset 0 from the pattern base,
            // so padded rows add few stencil patterns (a per-row column here made the pattern count
            // grow with the number of windows and disabled the compression at c3)
            const int32_t padA = a > 0 ? cA[0] : (int32_t)r0, padB = b > 0 ? cB[0] : (int32_t)nvel;
            for (; a < A; ++a) { cA[a * NB_C] = padA; NB_VA(a) = 0.0; }
            for (; b < B; ++b) {
                cB[b * NB_C] = padB;
                for (int cc = 0; cc < D; ++cc) NB_VB(b, cc) = 0.0;
            }
        } else {
            const int64_t row = nvel + (br - nnodes);
            const int64_t s0 = rp[row], e0 = rp[row + 1];
            for (int a = 0; a < A; ++a) { cA[a * NB_C] = 0; NB_VA(a) = 0.0; }
            int q = 0;
            for (int64_t k = s0; k < e0; k += D, ++q) {
                cB[q * NB_C] = ci[k];   // component-0 dof of the node
                for (int cc = 0; cc < D; ++cc) NB_VB(q, cc) = val[k + cc];
            }
            const int32_t padB = q > 0 ? cB[0] : 0;
            for (; q < B; ++q) {
                cB[q * NB_C] = padB;
                for (int cc = 0; cc < D; ++cc) NB_VB(q, cc) = 0.0;
            }
        }
#undef NB_VA
#undef NB_VB
    }
}

// G lanes per block row (G = 1: one thread per row; G > 1 for the long rows of 3D): a warp
// covers 32/G consecutive slots of one slice, lane q of a group takes entries q, q+G, ...
// of its row (for a fixed k the 32/G rows of the warp are contiguous, so every 32-byte
// sector is fully used), then the group sums by shuffles.
// column access: explicit (SELL column array) or stencil-compressed (base + pattern offset)
struct NbCols {
    const int32_t* __restrict__ col;      // explicit
    const int32_t* __restrict__ pid;      // compressed
    const int32_t* __restrict__ baseA;
    const int32_t* __restrict__ baseB;
    const int32_t* __restrict__ tbl;
    int W;
    int bulk;   // prologue: the warp's whole slice into L2 by one bulk prefetch
    const int32_t* __restrict__ vofs;   // VB: per slot, offset of its B-value vector in vtbl
    const double* __restrict__ vtbl;
    const char* xpf;    // the next kernel's leading bytes: prefetched into L2 by the last xpf_warps warps,
    int64_t xpf_bytes;  // NB_XPF_SEG bytes each
    int64_t xpf_warps;
};
constexpr int64_t NB_XPF_SEG = 8192;

// XA: x is 16-byte aligned (checked once at launch), so the node gathers of the pair layout are
// single 16-byte loads without the per-load alignment test of ld_node
// VB: B / B^T values from the table cols.vtbl (L1-resident) instead of the slice's value stream
template <int D, int G, int UA, int MINB = 1, bool PAT = false, bool PR = false, bool XA = false, bool VB = false>
__global__ void __launch_bounds__(256, MINB) nb_residual_kernel(int64_t n, int64_t nnodes, int64_t nslices, int64_t nvel,
                                                          const int32_t* __restrict__ perm,
                                                          const int32_t* __restrict__ wa,
                                                          const int32_t* __restrict__ wb,
                                                          const int64_t* __restrict__ cptr,
                                                          const int64_t* __restrict__ vptr,
                                                          NbCols cols,
                                                          const double* __restrict__ v, const double* __restrict__ x,
                                                          const double* __restrict__ b, double* __restrict__ r,
                                                          double* __restrict__ part) {
    static_assert(!PR || D == 2, "pair layout is 2D only");
    static_assert(!VB || PAT, "B-value table: compressed columns only");
    auto ldx2 = [&](const double* p, double* out) {
        if constexpr (XA) {
            const double2 v = __ldg(reinterpret_cast<const double2*>(p));
            out[0] = v.x;
            out[1] = v.y;
        } else {
            ld_node<2>(p, out);
        }
    };
    const int32_t* __restrict__ col = cols.col;
    __shared__ double red[8];
    double mine = 0.0;
    const int64_t total = nslices * NB_C * G;
    const int q = threadIdx.x % G;
    // 16-byte vector access to b / r for the d = 2 node rows (uniform: depends on the pointers only)
    const bool v2 = PR && ((reinterpret_cast<uintptr_t>(b) | reinterpret_cast<uintptr_t>(r)) & 15) == 0;
    pdl_trigger();
    if (G > 1 && cols.bulk) {   // the first warp of each slice prefetches the whole slice
        const int64_t t0 = (blockIdx.x * (int64_t)blockDim.x + (threadIdx.x & ~31)) / G;
        const int64_t s0 = t0 / NB_C;
        if (s0 < nslices && t0 % NB_C == 0 && (threadIdx.x & 31) == 0 && vptr[s0 + 1] > vptr[s0])
            bulk_prefetch_l2(v + vptr[s0], (uint32_t)((vptr[s0 + 1] - vptr[s0]) * 8));
    }
    if (G == 1) {   // before x exists: this warp's first slice lines (values, columns) into L2
        const int64_t s0 = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) / NB_C;
        const int lane = threadIdx.x & 31;
        if (s0 < nslices) {
            const char* vb = reinterpret_cast<const char*>(v + vptr[s0]);
            if (cols.bulk) {
                if (lane == 0 && vptr[s0 + 1] > vptr[s0]) bulk_prefetch_l2(vb, (uint32_t)((vptr[s0 + 1] - vptr[s0]) * 8));
                if (PAT && lane == 1) prefetch_l2(cols.pid + s0 * NB_C);
                if (PAT && lane == 2) prefetch_l2(cols.baseA + s0 * NB_C);
                if (PAT && lane == 3) prefetch_l2(cols.baseB + s0 * NB_C);
                if (!PAT && lane >= 16) prefetch_l2(reinterpret_cast<const char*>(col + cptr[s0]) + (size_t)(lane - 16) * 128);
            } else if (PAT) prefetch_l2(vb + (size_t)lane * 128);
            else if (lane < 16) prefetch_l2(vb + (size_t)lane * 128);
            else prefetch_l2(reinterpret_cast<const char*>(col + cptr[s0]) + (size_t)(lane - 16) * 128);
        }
    }
    if (cols.xpf_warps > 0 && (threadIdx.x & 31) == 0) {   // static data: before the dependency wait
        const int64_t tw = ((int64_t)gridDim.x * blockDim.x) >> 5;
        const int64_t gw = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
        const int64_t k = gw - (tw - cols.xpf_warps);
        if (k >= 0) {
            const int64_t off = k * NB_XPF_SEG;
            if (off < cols.xpf_bytes)
                bulk_prefetch_l2(cols.xpf + off, (uint32_t)min((int64_t)NB_XPF_SEG, cols.xpf_bytes - off));
        }
    }
    pdl_wait();
    for (int64_t tt = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; tt - threadIdx.x < total;
         tt += (int64_t)gridDim.x * blockDim.x) {
        const bool live = tt < total;
        const int64_t t = live ? tt / G : 0;       // slot
        const int64_t s = t / NB_C;
        const int l = (int)(t % NB_C);
        const int A = live ? wa[s] : 0, B = live ? wb[s] : 0;
        const int32_t* cA = PAT ? nullptr : col + (live ? cptr[s] : 0) + l;
        const int32_t* cB = PAT ? nullptr : cA + (int64_t)A * NB_C;
        // PAT: column of entry k = base + tbl[pid * W + k] (the pattern table is L1-resident)
        const int32_t* tp = PAT ? cols.tbl + (int64_t)(live ? cols.pid[t] : 0) * cols.W : nullptr;
        const int32_t bA = PAT && live ? cols.baseA[t] : 0, bB = PAT && live ? cols.baseB[t] : 0;
        const double* vbt = VB ? cols.vtbl + (live ? cols.vofs[t] : 0) : nullptr;   // B values of the slot
#define NB_VB2(k) (VB ? __ldg(reinterpret_cast<const double2*>(vbt) + (k)) : __ldcs(pB + (int64_t)(k) * NB_C))
#define NB_COLA(k) (PAT ? bA + __ldg(tp + (k)) : __ldcs(cA + (k) * NB_C))
#define NB_COLB(k) (PAT ? bB + __ldg(tp + A + (k)) : __ldcs(cB + (k) * NB_C))
        const double* vs = v + (live ? vptr[s] : 0);   // the slice's values (layout: nb_ia / nb_ib)
        const double* vA = vs + l;                     // plain layout
        const double* vB = vA + (int64_t)A * NB_C;
        const double2* pA = reinterpret_cast<const double2*>(vs) + l;                      // pair layout
        const double2* pB = reinterpret_cast<const double2*>(vs + (int64_t)A * NB_C) + l;
        const int64_t br = (live && t < n) ? perm[t] : -1;
        if constexpr (G == 1) {   // one thread per row: per-branch accumulation (no shuffles)
            if (br < 0) continue;
            if (br < nnodes) {
                double acc[D];
#pragma unroll
                for (int c = 0; c < D; ++c) acc[c] = 0.0;
                if constexpr (PR) {
                    const int A2 = A >> 1;
                    // two entries per iteration; a second iteration in flight only with the 48-register cap
                    if constexpr (PAT) {   // offsets of pair p + 1 loaded while pair p is gathered
                        const int2* tp2 = reinterpret_cast<const int2*>(tp);
                        int2 on = A2 > 0 ? __ldg(tp2) : make_int2(0, 0);
#pragma unroll (MINB <= 5 ? 2 : 1)
                        for (int p = 0; p < A2; ++p) {
                            const int2 o = on;
                            if (p + 1 < A2) on = __ldg(tp2 + p + 1);
                            const double2 a = __ldcs(pA + (int64_t)p * NB_C);
                            double x0[2], x1[2];
                            ldx2(x + bA + o.x, x0);
                            ldx2(x + bA + o.y, x1);
                            acc[0] = fma(a.x, x0[0], acc[0]);
                            acc[1] = fma(a.x, x0[1], acc[1]);
                            acc[0] = fma(a.y, x1[0], acc[0]);
                            acc[1] = fma(a.y, x1[1], acc[1]);
                        }
                    } else
#pragma unroll (MINB <= 5 ? 2 : 1)
                    for (int p = 0; p < A2; ++p) {
                        const double2 a = __ldcs(pA + (int64_t)p * NB_C);
                        double x0[2], x1[2];
                        ldx2(x + NB_COLA(2 * p), x0);
                        ldx2(x + NB_COLA(2 * p + 1), x1);
                        acc[0] = fma(a.x, x0[0], acc[0]);
                        acc[1] = fma(a.x, x0[1], acc[1]);
                        acc[0] = fma(a.y, x1[0], acc[0]);
                        acc[1] = fma(a.y, x1[1], acc[1]);
                    }
                    if (A & 1) {
                        const double a = __ldcs(vs + (int64_t)(2 * A2) * NB_C + l);
                        double x0[2];
                        ldx2(x + NB_COLA(A - 1), x0);
                        acc[0] = fma(a, x0[0], acc[0]);
                        acc[1] = fma(a, x0[1], acc[1]);
                    }
#pragma unroll 2
                    for (int k = 0; k < B; ++k) {
                        const double xp = __ldg(x + NB_COLB(k));
                        const double2 bv = NB_VB2(k);
                        acc[0] = fma(bv.x, xp, acc[0]);
                        acc[1] = fma(bv.y, xp, acc[1]);
                    }
                } else {
#pragma unroll UA
                    for (int k = 0; k < A; ++k) {
                        const int cc = NB_COLA(k);
                        const double a = __ldcs(vA + k * NB_C);
                        double xv[D];
                        ld_node<D>(x + cc, xv);
#pragma unroll
                        for (int c = 0; c < D; ++c) acc[c] = fma(a, xv[c], acc[c]);
                    }
#pragma unroll 2
                    for (int k = 0; k < B; ++k) {
                        const double xp = __ldg(x + NB_COLB(k));
#pragma unroll
                        for (int c = 0; c < D; ++c)
                            acc[c] = fma(VB ? __ldg(vbt + k * D + c) : __ldcs(vB + ((int64_t)k * D + c) * NB_C), xp, acc[c]);
                    }
                }
                const int64_t r0 = br * D;
                if (PR && v2) {
                    const double2 bb = __ldg(reinterpret_cast<const double2*>(b + r0));
                    const double2 rr = make_double2(bb.x - acc[0], bb.y - acc[D - 1]);
                    if (r) *reinterpret_cast<double2*>(r + r0) = rr;
                    mine += rr.x * rr.x;
                    mine += rr.y * rr.y;
                } else {
#pragma unroll
                    for (int c = 0; c < D; ++c) {
                        const double rr = b[r0 + c] - acc[c];
                        if (r) r[r0 + c] = rr;
                        mine += rr * rr;
                    }
                }
            } else {
                double acc = 0.0;
                if constexpr (PR) {
#pragma unroll UA
                    for (int k = 0; k < B; ++k) {
                        double xv[2];
                        ldx2(x + NB_COLB(k), xv);
                        const double2 bv = NB_VB2(k);
                        acc = fma(bv.x, xv[0], acc);
                        acc = fma(bv.y, xv[1], acc);
                    }
                } else {
#pragma unroll UA
                    for (int k = 0; k < B; ++k) {
                        const int cc = NB_COLB(k);
#pragma unroll
                        for (int c = 0; c < D; ++c)
                            acc = fma(VB ? __ldg(vbt + k * D + c) : __ldcs(vB + ((int64_t)k * D + c) * NB_C), __ldg(x + cc + c), acc);
                    }
                }
                const int64_t row = nvel + (br - nnodes);
                const double rr = b[row] - acc;
                if (r) r[row] = rr;
                mine += rr * rr;
            }
            continue;
        }
        // the lanes of a group share the row, but a warp may hold node and pressure rows: the group
        // sums run outside the branches with every lane converged (full-mask shuffles)
        double acc[D];
#pragma unroll
        for (int c = 0; c < D; ++c) acc[c] = 0.0;
        // the row's right-hand side, loaded now (not after the accumulation and the group sum): lane q
        // finalises the components c = q, q + G, ... of a node row (lane 0 a pressure row); the
        // butterfly group sum leaves the same total in every lane of the group
        // (3D only: in 2D the extra registers cost more occupancy than the early loads save)
        constexpr bool EB = D == 3;
        constexpr int CPL = (D + G - 1) / G;   // components per lane
        double be[CPL];
#pragma unroll
        for (int u = 0; u < CPL; ++u) {
            const int c = q + u * G;
            be[u] = 0.0;
            if (EB && br >= 0 && br < nnodes && c < D) be[u] = __ldg(b + br * D + c);
            else if (EB && br >= nnodes && c == 0) be[u] = __ldg(b + nvel + (br - nnodes));
        }
        if (br >= 0 && br < nnodes) {
#pragma unroll UA
            for (int k = q; k < A; k += G) {
                const int cc = NB_COLA(k);
                const double a = __ldcs(vs + nb_ia(PR, A, k, l));
                double xv[D];
                ld_node<D>(x + cc, xv);
#pragma unroll
                for (int c = 0; c < D; ++c) acc[c] = fma(a, xv[c], acc[c]);
            }
#pragma unroll 2
            for (int k = q; k < B; k += G) {
                const double xp = __ldg(x + NB_COLB(k));
#pragma unroll
                for (int c = 0; c < D; ++c)
                    acc[c] = fma(VB ? __ldg(vbt + k * D + c) : __ldcs(vs + nb_ib(PR, D, A, k, c, l)), xp, acc[c]);
            }
        } else if (br >= 0) {
#pragma unroll UA
            for (int k = q; k < B; k += G) {
                const int cc = NB_COLB(k);
#pragma unroll
                for (int c = 0; c < D; ++c)
                    acc[0] = fma(VB ? __ldg(vbt + k * D + c) : __ldcs(vs + nb_ib(PR, D, A, k, c, l)), __ldg(x + cc + c), acc[0]);
            }
        }
        if (G > 1) {
            __syncwarp();
#pragma unroll
            for (int c = 0; c < D; ++c) acc[c] = group_sum<G>(acc[c]);
        }
        if (!EB && q == 0 && br >= 0) {
            if (br < nnodes) {
                const int64_t r0 = br * D;
#pragma unroll
                for (int c = 0; c < D; ++c) {
                    const double rr = b[r0 + c] - acc[c];
                    if (r) r[r0 + c] = rr;
                    mine += rr * rr;
                }
            } else {
                const int64_t row = nvel + (br - nnodes);
                const double rr = b[row] - acc[0];
                if (r) r[row] = rr;
                mine += rr * rr;
            }
        }
        if (EB && br >= 0) {
            if (br < nnodes) {
                const int64_t r0 = br * D;
#pragma unroll
                for (int u = 0; u < CPL; ++u) {
                    const int c = q + u * G;
                    if (c < D) {
                        double a = acc[0];
#pragma unroll
                        for (int cc = 1; cc < D; ++cc) a = c == cc ? acc[cc] : a;
                        const double rr = be[u] - a;
                        if (r) r[r0 + c] = rr;
                        mine += rr * rr;
                    }
                }
            } else if (q == 0) {
                const int64_t row = nvel + (br - nnodes);
                const double rr = be[0] - acc[0];
                if (r) r[row] = rr;
                mine += rr * rr;
            }
        }
    }
#undef NB_COLA
#undef NB_COLB
#undef NB_VB2
    if (part) {
        mine = warp_sum(mine);
        if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = mine;
        __syncthreads();
        if (threadIdx.x == 0) {
            double sum = 0.0;
            for (int i = 0; i < (int)(blockDim.x >> 5); ++i) sum += red[i];
            part[blockIdx.x] = sum;
        }
    }
}

// ---- stencil compression of the column arrays (structured operators) ------------------------
// A slot's column list = (A node columns, B pressure columns); its pattern = (A, B, offsets of
// the A columns from the first A column, offsets of the B columns from the first B column).
// Structured grids have a few hundred distinct patterns, so the 4-byte column indices (a
// quarter of the residual's bytes) become a per-slot pattern id and two bases.
__device__ __forceinline__ uint64_t fnv(uint64_t h, uint32_t v) {
    for (int k = 0; k < 4; ++k) { h ^= (v >> (8 * k)) & 0xffu; h *= 1099511628211ull; }
    return h;
}

__global__ void nb_hash_kernel(int64_t nslots, const int32_t* wa, const int32_t* wb, const int64_t* cptr,
                               const int32_t* col, uint64_t* key, int32_t* idx, int32_t* bA, int32_t* bB) {
    for (int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; t < nslots; t += (int64_t)gridDim.x * blockDim.x) {
        const int64_t s = t / NB_C;
        const int l = (int)(t % NB_C);
        const int A = wa[s], B = wb[s];
        const int32_t* cA = col + cptr[s] + l;
        const int32_t* cB = cA + (int64_t)A * NB_C;
        const int32_t a0 = A > 0 ? cA[0] : 0, b0 = B > 0 ? cB[0] : 0;
        uint64_t h = 1469598103934665603ull;
        h = fnv(h, (uint32_t)A);
        h = fnv(h, (uint32_t)B);
        for (int k = 0; k < A; ++k) h = fnv(h, (uint32_t)(cA[k * NB_C] - a0));
        for (int k = 0; k < B; ++k) h = fnv(h, (uint32_t)(cB[k * NB_C] - b0));
        key[t] = h;
        idx[t] = (int32_t)t;
        bA[t] = a0;
        bB[t] = b0;
    }
}

__global__ void nb_segment_kernel(int64_t nslots, const uint64_t* skey, int32_t* flag) {
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < nslots; i += (int64_t)gridDim.x * blockDim.x)
        flag[i] = (i == 0 || skey[i] != skey[i - 1]) ? 1 : 0;
}

__global__ void nb_pid_kernel(int64_t nslots, const int32_t* sidx, const int32_t* flag, const int32_t* seg,
                              int32_t* pid, int32_t* rep) {
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < nslots; i += (int64_t)gridDim.x * blockDim.x) {
        const int32_t p = seg[i] - 1;
        pid[sidx[i]] = p;
        if (flag[i]) rep[p] = sidx[i];
    }
}

__global__ void nb_table_kernel(int npat, int W, const int32_t* rep, const int32_t* wa, const int32_t* wb,
                                const int64_t* cptr, const int32_t* col, int32_t* tbl, int32_t* tw) {
    for (int p = blockIdx.x * blockDim.x + threadIdx.x; p < npat; p += gridDim.x * blockDim.x) {
        const int64_t t = rep[p], s = t / NB_C;
        const int l = (int)(t % NB_C);
        const int A = wa[s], B = wb[s];
        const int32_t* cA = col + cptr[s] + l;
        const int32_t* cB = cA + (int64_t)A * NB_C;
        const int32_t a0 = A > 0 ? cA[0] : 0, b0 = B > 0 ? cB[0] : 0;
        for (int k = 0; k < A; ++k) tbl[(int64_t)p * W + k] = cA[k * NB_C] - a0;
        for (int k = 0; k < B; ++k) tbl[(int64_t)p * W + A + k] = cB[k * NB_C] - b0;
        tw[2 * p] = A;
        tw[2 * p + 1] = B;
    }
}

__global__ void nb_verify_kernel(int64_t nslots, int W, const int32_t* wa, const int32_t* wb, const int64_t* cptr,
                                 const int32_t* col, const int32_t* pid, const int32_t* bA, const int32_t* bB,
                                 const int32_t* tbl, const int32_t* tw, unsigned int* err) {
    for (int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; t < nslots; t += (int64_t)gridDim.x * blockDim.x) {
        const int64_t s = t / NB_C;
        const int l = (int)(t % NB_C);
        const int A = wa[s], B = wb[s], p = pid[t];
        if (tw[2 * p] != A || tw[2 * p + 1] != B) { atomicOr(err, 1u); continue; }
        const int32_t* cA = col + cptr[s] + l;
        const int32_t* cB = cA + (int64_t)A * NB_C;
        for (int k = 0; k < A; ++k)
            if (cA[k * NB_C] != bA[t] + tbl[(int64_t)p * W + k]) atomicOr(err, 1u);
        for (int k = 0; k < B; ++k)
            if (cB[k * NB_C] != bB[t] + tbl[(int64_t)p * W + A + k]) atomicOr(err, 1u);
    }
}

// replace N.col by (pattern id, bases, table) when the patterns are few and verified
static rav_status nb_compress(NodeBlocked& N, cudaStream_t s) {
    const int64_t ns = N.nslices * NB_C;
    std::vector<int32_t> hwa(N.nslices), hwb(N.nslices);
    RAV_CUDA(cudaMemcpy(hwa.data(), N.wa, sizeof(int32_t) * N.nslices, cudaMemcpyDeviceToHost));
    RAV_CUDA(cudaMemcpy(hwb.data(), N.wb, sizeof(int32_t) * N.nslices, cudaMemcpyDeviceToHost));
    int W = 1;
    for (int64_t k = 0; k < N.nslices; ++k) W = std::max(W, hwa[k] + hwb[k]);
    W += W & 1;   // even row stride: entry pairs (2p, 2p + 1) of a row are one aligned 8-byte load
    uint64_t *key = nullptr, *skey = nullptr;
    int32_t *idx = nullptr, *sidx = nullptr, *flag = nullptr, *seg = nullptr, *rep = nullptr, *tw = nullptr;
    int32_t *pid = nullptr, *bA = nullptr, *bB = nullptr, *tbl = nullptr;
    unsigned int* err = nullptr;
    RAV_CUDA(cudaMallocAsync(&key, sizeof(uint64_t) * ns, s));
    RAV_CUDA(cudaMallocAsync(&skey, sizeof(uint64_t) * ns, s));
    RAV_CUDA(cudaMallocAsync(&idx, sizeof(int32_t) * ns, s));
    RAV_CUDA(cudaMallocAsync(&sidx, sizeof(int32_t) * ns, s));
    RAV_CUDA(cudaMallocAsync(&flag, sizeof(int32_t) * ns, s));
    RAV_CUDA(cudaMallocAsync(&seg, sizeof(int32_t) * ns, s));
    RAV_CUDA(cudaMalloc(&pid, sizeof(int32_t) * ns));
    RAV_CUDA(cudaMalloc(&bA, sizeof(int32_t) * ns));
    RAV_CUDA(cudaMalloc(&bB, sizeof(int32_t) * ns));
    const int nb = (int)std::max<int64_t>(1, std::min<int64_t>(cdiv(ns, 256), (int64_t)num_sms() * 16));
    nb_hash_kernel<<<nb, 256, 0, s>>>(ns, N.wa, N.wb, N.cptr, N.col, key, idx, bA, bB);
    count_launch();
    RAV_CHECK_LAUNCH();
    size_t tmp = 0;
    RAV_CUDA(cub::DeviceRadixSort::SortPairs(nullptr, tmp, key, skey, idx, sidx, (int)ns, 0, 64, s));
    void* d_tmp = nullptr;
    RAV_CUDA(cudaMallocAsync(&d_tmp, tmp + 16, s));
    RAV_CUDA(cub::DeviceRadixSort::SortPairs(d_tmp, tmp, key, skey, idx, sidx, (int)ns, 0, 64, s));
    nb_segment_kernel<<<nb, 256, 0, s>>>(ns, skey, flag);
    count_launch();
    size_t tmp2 = 0;
    RAV_CUDA(cub::DeviceScan::InclusiveSum(nullptr, tmp2, flag, seg, (int)ns, s));
    void* d_tmp2 = nullptr;
    RAV_CUDA(cudaMallocAsync(&d_tmp2, tmp2 + 16, s));
    RAV_CUDA(cub::DeviceScan::InclusiveSum(d_tmp2, tmp2, flag, seg, (int)ns, s));
    int32_t npat = 0;
    RAV_CUDA(cudaMemcpyAsync(&npat, seg + ns - 1, sizeof(int32_t), cudaMemcpyDeviceToHost, s));
    RAV_CUDA(cudaStreamSynchronize(s));
    bool ok = npat > 0 && (int64_t)npat * W * 4 <= (16 << 20);   // table must stay cache-sized
    if (ok) {
        RAV_CUDA(cudaMallocAsync(&rep, sizeof(int32_t) * npat, s));
        RAV_CUDA(cudaMallocAsync(&tw, sizeof(int32_t) * 2 * npat, s));
        RAV_CUDA(cudaMalloc(&tbl, sizeof(int32_t) * (int64_t)npat * W));
        RAV_CUDA(cudaMallocAsync(&err, sizeof(unsigned int), s));
        RAV_CUDA(cudaMemsetAsync(err, 0, sizeof(unsigned int), s));
        nb_pid_kernel<<<nb, 256, 0, s>>>(ns, sidx, flag, seg, pid, rep);
        count_launch();
        nb_table_kernel<<<(int)cdiv(npat, 128), 128, 0, s>>>(npat, W, rep, N.wa, N.wb, N.cptr, N.col, tbl, tw);
        count_launch();
        nb_verify_kernel<<<nb, 256, 0, s>>>(ns, W, N.wa, N.wb, N.cptr, N.col, pid, bA, bB, tbl, tw, err);
        count_launch();
        RAV_CHECK_LAUNCH();
        unsigned int h_err = 0;
        RAV_CUDA(cudaMemcpyAsync(&h_err, err, sizeof(h_err), cudaMemcpyDeviceToHost, s));
        RAV_CUDA(cudaStreamSynchronize(s));
        ok = h_err == 0;   // a hash collision keeps the explicit columns
    }
    for (void* p : {(void*)key, (void*)skey, (void*)idx, (void*)sidx, (void*)flag, (void*)seg, (void*)rep, (void*)tw,
                    (void*)err, d_tmp, d_tmp2})
        if (p) cudaFreeAsync(p, s);
    RAV_CUDA(cudaStreamSynchronize(s));
    if (!ok) {
        for (void* p : {(void*)pid, (void*)bA, (void*)bB, (void*)tbl})
            if (p) cudaFree(p);
        return RAV_OK;
    }
    int64_t hc = 0;
    RAV_CUDA(cudaMemcpy(&hc, N.cptr + N.nslices, sizeof(int64_t), cudaMemcpyDeviceToHost));
    cudaFree(N.col);
    N.col = nullptr;
    N.pid = pid;
    N.baseA = bA;
    N.baseB = bB;
    N.tbl = tbl;
    N.W = W;
    N.npat = npat;
    // streamed bytes: values + per-slot (pid, two bases); the table is cache-resident
    N.bytes = N.bytes - 4 * hc + 12 * ns;
    return RAV_OK;
}

// ---- B-value compression ----------------------------------------------------------------------
// The B block carries no viscosity (Eq. 6: b_jp = -(q_p, div phi_j)), so on a uniform level
// the d values of every B / B^T entry repeat from row to row: a slot's B values (entry order,
// d per entry) form one of a few distinct vectors.  They are hashed, deduplicated, verified
// bitwise against a table and dropped from the streamed values (c2: half of the residual's bytes).
// The residual reads the same values in the same order: bitwise the same result.
__global__ void nb_bhash_kernel(int64_t nslots, int D, int pair, const int32_t* wa, const int32_t* wb,
                                const int64_t* vptr, const double* v, uint64_t* key, int32_t* idx) {
    for (int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; t < nslots; t += (int64_t)gridDim.x * blockDim.x) {
        const int64_t s = t / NB_C;
        const int l = (int)(t % NB_C);
        const int A = wa[s], B = wb[s];
        const double* vs = v + vptr[s];
        uint64_t h = 1469598103934665603ull;
        h = fnv(h, (uint32_t)B);
        for (int k = 0; k < B; ++k)
            for (int c = 0; c < D; ++c) {
                const uint64_t u = (uint64_t)__double_as_longlong(vs[nb_ib(pair != 0, D, A, k, c, l)]);
                h = fnv(fnv(h, (uint32_t)u), (uint32_t)(u >> 32));
            }
        key[t] = h;
        idx[t] = (int32_t)t;
    }
}

__global__ void nb_vlen_kernel(int nvec, int D, const int32_t* rep, const int32_t* wb, int64_t* len) {
    for (int p = blockIdx.x * blockDim.x + threadIdx.x; p < nvec; p += gridDim.x * blockDim.x)
        len[p] = (int64_t)wb[rep[p] / NB_C] * D;
}

__global__ void nb_vtbl_kernel(int nvec, int D, int pair, const int32_t* rep, const int32_t* wa, const int32_t* wb,
                               const int64_t* vptr, const double* v, const int64_t* voff, double* vtbl) {
    for (int p = blockIdx.x * blockDim.x + threadIdx.x; p < nvec; p += gridDim.x * blockDim.x) {
        const int64_t t = rep[p], s = t / NB_C;
        const int l = (int)(t % NB_C);
        const int A = wa[s], B = wb[s];
        for (int k = 0; k < B; ++k)
            for (int c = 0; c < D; ++c) vtbl[voff[p] + k * D + c] = v[vptr[s] + nb_ib(pair != 0, D, A, k, c, l)];
    }
}

// per slot: its vector's offset; verify length and every value bitwise
__global__ void nb_vverify_kernel(int64_t nslots, int D, int pair, const int32_t* wa, const int32_t* wb,
                                  const int64_t* vptr, const double* v, const int32_t* sidx, const int32_t* seg,
                                  const int64_t* voff, const int64_t* vlen, const double* vtbl, int32_t* vofs,
                                  unsigned int* err) {
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < nslots; i += (int64_t)gridDim.x * blockDim.x) {
        const int64_t t = sidx[i], s = t / NB_C;
        const int p = seg[i] - 1;
        const int l = (int)(t % NB_C);
        const int A = wa[s], B = wb[s];
        vofs[t] = (int32_t)voff[p];
        if (vlen[p] != (int64_t)B * D) { atomicOr(err, 1u); continue; }
        for (int k = 0; k < B; ++k)
            for (int c = 0; c < D; ++c)
                if (__double_as_longlong(v[vptr[s] + nb_ib(pair != 0, D, A, k, c, l)]) !=
                    __double_as_longlong(vtbl[voff[p] + k * D + c]))
                    atomicOr(err, 1u);
    }
}

// the A part of each slice: its first 32 A values in both layouts (nb_ia < 32 A)
__global__ void nb_asize_kernel(int64_t nslices, const int32_t* wa, int64_t* sz) {
    for (int64_t s = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; s < nslices; s += (int64_t)gridDim.x * blockDim.x)
        sz[s] = (int64_t)NB_C * wa[s];
}
__global__ void nb_acopy_kernel(int64_t nslices, const int64_t* vptr, const int64_t* vptr2, const double* v,
                                double* v2) {
    for (int64_t s = blockIdx.x; s < nslices; s += gridDim.x) {
        const int64_t n = vptr2[s + 1] - vptr2[s];
        for (int64_t i = threadIdx.x; i < n; i += blockDim.x) v2[vptr2[s] + i] = v[vptr[s] + i];
    }
}

static rav_status nb_compress_bvals(NodeBlocked& N, cudaStream_t s) {
    const int64_t ns = N.nslices * NB_C;
    const int D = N.D;
    uint64_t *key = nullptr, *skey = nullptr;
    int32_t *idx = nullptr, *sidx = nullptr, *flag = nullptr, *seg = nullptr, *rep = nullptr, *vofs = nullptr;
    int64_t *vlen = nullptr, *voff = nullptr, *asz = nullptr, *vptr2 = nullptr;
    double *vtbl = nullptr, *v2 = nullptr;
    unsigned int* err = nullptr;
    void *d_tmp = nullptr, *d_tmp2 = nullptr;
    bool ok = true;
    int32_t nvec = 0;
    int64_t nt = 0;
    const int nb = (int)std::max<int64_t>(1, std::min<int64_t>(cdiv(ns, 256), (int64_t)num_sms() * 16));
    RAV_CUDA(cudaMallocAsync(&key, sizeof(uint64_t) * ns, s));
    RAV_CUDA(cudaMallocAsync(&skey, sizeof(uint64_t) * ns, s));
    RAV_CUDA(cudaMallocAsync(&idx, sizeof(int32_t) * ns, s));
    RAV_CUDA(cudaMallocAsync(&sidx, sizeof(int32_t) * ns, s));
    RAV_CUDA(cudaMallocAsync(&flag, sizeof(int32_t) * ns, s));
    RAV_CUDA(cudaMallocAsync(&seg, sizeof(int32_t) * ns, s));
    nb_bhash_kernel<<<nb, 256, 0, s>>>(ns, D, N.pair, N.wa, N.wb, N.vptr, N.val, key, idx);
    count_launch();
    RAV_CHECK_LAUNCH();
    size_t tmp = 0, tmp2 = 0;
    RAV_CUDA(cub::DeviceRadixSort::SortPairs(nullptr, tmp, key, skey, idx, sidx, (int)ns, 0, 64, s));
    RAV_CUDA(cudaMallocAsync(&d_tmp, tmp + 16, s));
    RAV_CUDA(cub::DeviceRadixSort::SortPairs(d_tmp, tmp, key, skey, idx, sidx, (int)ns, 0, 64, s));
    nb_segment_kernel<<<nb, 256, 0, s>>>(ns, skey, flag);
    count_launch();
    RAV_CUDA(cub::DeviceScan::InclusiveSum(nullptr, tmp2, flag, seg, (int)ns, s));
    RAV_CUDA(cudaMallocAsync(&d_tmp2, tmp2 + 16, s));
    RAV_CUDA(cub::DeviceScan::InclusiveSum(d_tmp2, tmp2, flag, seg, (int)ns, s));
    RAV_CUDA(cudaMemcpyAsync(&nvec, seg + ns - 1, sizeof(int32_t), cudaMemcpyDeviceToHost, s));
    RAV_CUDA(cudaStreamSynchronize(s));
    ok = nvec > 0 && nvec <= 65536;
    if (ok) {
        RAV_CUDA(cudaMallocAsync(&rep, sizeof(int32_t) * nvec, s));
        RAV_CUDA(cudaMallocAsync(&vlen, sizeof(int64_t) * nvec, s));
        RAV_CUDA(cudaMallocAsync(&voff, sizeof(int64_t) * (nvec + 1), s));
        int32_t* dummy_pid = nullptr;
        RAV_CUDA(cudaMallocAsync(&dummy_pid, sizeof(int32_t) * ns, s));
        nb_pid_kernel<<<nb, 256, 0, s>>>(ns, sidx, flag, seg, dummy_pid, rep);
        count_launch();
        cudaFreeAsync(dummy_pid, s);
        nb_vlen_kernel<<<(int)cdiv(nvec, 128), 128, 0, s>>>(nvec, D, rep, N.wb, vlen);
        count_launch();
        RAV_TRY(gen::counts_to_rowptr(vlen, voff, nvec, s));
        RAV_CUDA(cudaMemcpyAsync(&nt, voff + nvec, sizeof(int64_t), cudaMemcpyDeviceToHost, s));
        RAV_CUDA(cudaStreamSynchronize(s));
        ok = nt * 8 <= (8 << 20) && nt < (1ll << 31);   // the table stays cache-sized
    }
    if (ok) {
        RAV_CUDA(cudaMalloc(&vtbl, sizeof(double) * std::max<int64_t>(2, nt)));
        RAV_CUDA(cudaMalloc(&vofs, sizeof(int32_t) * ns));
        RAV_CUDA(cudaMallocAsync(&err, sizeof(unsigned int), s));
        RAV_CUDA(cudaMemsetAsync(err, 0, sizeof(unsigned int), s));
        nb_vtbl_kernel<<<(int)cdiv(nvec, 128), 128, 0, s>>>(nvec, D, N.pair, rep, N.wa, N.wb, N.vptr, N.val, voff, vtbl);
        count_launch();
        nb_vverify_kernel<<<nb, 256, 0, s>>>(ns, D, N.pair, N.wa, N.wb, N.vptr, N.val, sidx, seg, voff, vlen, vtbl,
                                             vofs, err);
        count_launch();
        RAV_CHECK_LAUNCH();
        unsigned int h_err = 0;
        RAV_CUDA(cudaMemcpyAsync(&h_err, err, sizeof(h_err), cudaMemcpyDeviceToHost, s));
        RAV_CUDA(cudaStreamSynchronize(s));
        ok = h_err == 0;   // a hash collision keeps the values in the stream
    }
    int64_t hv2 = 0, hv = 0;
    if (ok) {   // the slices' values shrink to their A parts
        RAV_CUDA(cudaMallocAsync(&asz, sizeof(int64_t) * N.nslices, s));
        RAV_CUDA(cudaMalloc(&vptr2, sizeof(int64_t) * (N.nslices + 1)));
        const int nbs = (int)std::max<int64_t>(1, std::min<int64_t>(cdiv(N.nslices, 256), (int64_t)num_sms() * 16));
        nb_asize_kernel<<<nbs, 256, 0, s>>>(N.nslices, N.wa, asz);
        count_launch();
        RAV_TRY(gen::counts_to_rowptr(asz, vptr2, N.nslices, s));
        RAV_CUDA(cudaMemcpyAsync(&hv2, vptr2 + N.nslices, sizeof(int64_t), cudaMemcpyDeviceToHost, s));
        RAV_CUDA(cudaMemcpyAsync(&hv, N.vptr + N.nslices, sizeof(int64_t), cudaMemcpyDeviceToHost, s));
        RAV_CUDA(cudaStreamSynchronize(s));
        RAV_CUDA(cudaMalloc(&v2, sizeof(double) * std::max<int64_t>(2, hv2)));
        nb_acopy_kernel<<<(int)std::max<int64_t>(1, std::min<int64_t>(N.nslices, (int64_t)num_sms() * 16)), 256, 0, s>>>(
            N.nslices, N.vptr, vptr2, N.val, v2);
        count_launch();
        RAV_CHECK_LAUNCH();
    }
    for (void* p : {(void*)key, (void*)skey, (void*)idx, (void*)sidx, (void*)flag, (void*)seg, (void*)rep, (void*)vlen,
                    (void*)voff, (void*)err, (void*)asz, d_tmp, d_tmp2})
        if (p) cudaFreeAsync(p, s);
    RAV_CUDA(cudaStreamSynchronize(s));
    if (!ok) {
        for (void* p : {(void*)vtbl, (void*)vofs})
            if (p) cudaFree(p);
        return RAV_OK;
    }
    cudaFree(N.val);
    cudaFree(N.vptr);
    N.val = v2;
    N.vptr = vptr2;
    N.vofs = vofs;
    N.vtbl = vtbl;
    N.nvtbl = nt;
    N.nbvec = nvec;
    // streamed bytes: the dropped B values out, a 4-byte vector offset per slot in
    N.bytes = N.bytes - 8 * (hv - hv2) + 4 * ns;
    return RAV_OK;
}

rav_status nb_build(Csr& A, int64_t nvel, int D, cudaStream_t s) {
    NodeBlocked& N = A.nb;
    if (D < 2 || D > 3 || nvel <= 0 || nvel % D != 0 || A.n_rows != A.n_cols || nvel >= A.n_rows) return RAV_OK;
    const int64_t nnodes = nvel / D, npres = A.n_rows - nvel, n = nnodes + npres;
    int32_t *na = nullptr, *nbv = nullptr, *key = nullptr, *idx = nullptr, *skey = nullptr;
    int64_t* woff = nullptr;
    unsigned int* fail = nullptr;
    RAV_CUDA(cudaMallocAsync(&na, sizeof(int32_t) * n, s));
    RAV_CUDA(cudaMallocAsync(&nbv, sizeof(int32_t) * n, s));
    RAV_CUDA(cudaMallocAsync(&fail, sizeof(unsigned int), s));
    RAV_CUDA(cudaMemsetAsync(fail, 0, sizeof(unsigned int), s));
    const int nb1 = (int)std::max<int64_t>(1, std::min<int64_t>(cdiv(n, 256), (int64_t)num_sms() * 16));
    nb_count_kernel<<<nb1, 256, 0, s>>>(nnodes, npres, D, nvel, A.rp, A.ci, A.val, na, nbv, fail);
    count_launch();
    RAV_CHECK_LAUNCH();
    unsigned int h_fail = 0;
    RAV_CUDA(cudaMemcpyAsync(&h_fail, fail, sizeof(h_fail), cudaMemcpyDeviceToHost, s));
    RAV_CUDA(cudaStreamSynchronize(s));
    cudaFreeAsync(fail, s);
    if (h_fail) {
        cudaFreeAsync(na, s);
        cudaFreeAsync(nbv, s);
        return RAV_OK;   // structure does not hold: keep the SELL residual
    }
    N.D = D;
    N.nnodes = nnodes;
    N.nblock = n;
    N.nslices = cdiv(n, NB_C);
    const int64_t nw = cdiv(n, NB_SIGMA);
    RAV_CUDA(cudaMallocAsync(&key, sizeof(int32_t) * n, s));
    RAV_CUDA(cudaMallocAsync(&skey, sizeof(int32_t) * n, s));
    RAV_CUDA(cudaMallocAsync(&idx, sizeof(int32_t) * n, s));
    RAV_CUDA(cudaMallocAsync(&woff, sizeof(int64_t) * (nw + 1), s));
    RAV_CUDA(cudaMalloc(&N.perm, sizeof(int32_t) * N.nslices * NB_C));
    RAV_CUDA(cudaMemsetAsync(N.perm, 0, sizeof(int32_t) * N.nslices * NB_C, s));
    nb_key_kernel<<<nb1, 256, 0, s>>>(n, na, nbv, D, key, idx);
    count_launch();
    nb_windows_kernel<<<(int)std::max<int64_t>(1, cdiv(nw + 1, 256)), 256, 0, s>>>(n, nw, woff);
    count_launch();
    RAV_CHECK_LAUNCH();
    size_t tmp = 0;
    RAV_CUDA(cub::DeviceSegmentedRadixSort::SortPairsDescending(nullptr, tmp, key, skey, idx, N.perm, (int)n, (int)nw,
                                                                woff, woff + 1, 0, 8 * sizeof(int32_t), s));
    void* d_tmp = nullptr;
    RAV_CUDA(cudaMallocAsync(&d_tmp, tmp + 16, s));
    RAV_CUDA(cub::DeviceSegmentedRadixSort::SortPairsDescending(d_tmp, tmp, key, skey, idx, N.perm, (int)n, (int)nw,
                                                                woff, woff + 1, 0, 8 * sizeof(int32_t), s));
    int64_t *csz = nullptr, *vsz = nullptr;
    RAV_CUDA(cudaMalloc(&N.wa, sizeof(int32_t) * N.nslices));
    RAV_CUDA(cudaMalloc(&N.wb, sizeof(int32_t) * N.nslices));
    RAV_CUDA(cudaMalloc(&N.cptr, sizeof(int64_t) * (N.nslices + 1)));
    RAV_CUDA(cudaMalloc(&N.vptr, sizeof(int64_t) * (N.nslices + 1)));
    RAV_CUDA(cudaMallocAsync(&csz, sizeof(int64_t) * N.nslices, s));
    RAV_CUDA(cudaMallocAsync(&vsz, sizeof(int64_t) * N.nslices, s));
    const int nbs = (int)std::max<int64_t>(1, std::min<int64_t>(cdiv(N.nslices, 256), (int64_t)num_sms() * 16));
    nb_slice_kernel<<<nbs, 256, 0, s>>>(n, N.nslices, D, N.perm, na, nbv, N.wa, N.wb, csz, vsz);
    count_launch();
    RAV_CHECK_LAUNCH();
    RAV_TRY(gen::counts_to_rowptr(csz, N.cptr, N.nslices, s));
    RAV_TRY(gen::counts_to_rowptr(vsz, N.vptr, N.nslices, s));
    int64_t hc = 0, hv = 0;
    RAV_CUDA(cudaMemcpyAsync(&hc, N.cptr + N.nslices, sizeof(int64_t), cudaMemcpyDeviceToHost, s));
    RAV_CUDA(cudaMemcpyAsync(&hv, N.vptr + N.nslices, sizeof(int64_t), cudaMemcpyDeviceToHost, s));
    RAV_CUDA(cudaStreamSynchronize(s));
    RAV_CUDA(cudaMalloc(&N.col, sizeof(int32_t) * std::max<int64_t>(1, hc)));
    RAV_CUDA(cudaMalloc(&N.val, sizeof(double) * std::max<int64_t>(1, hv)));
    N.bytes = 4 * hc + 8 * hv;
    static const bool pair_env = [] {
        const char* e = getenv("RAV_NB_PAIR");   // 16-byte value pairs for d = 2 (default on)
        return !(e && atoi(e) == 0);
    }();
    N.pair = (D == 2 && pair_env) ? 1 : 0;
    const int nbf = (int)std::max<int64_t>(1, std::min<int64_t>(cdiv(N.nslices * NB_C, 256), (int64_t)num_sms() * 16));
    nb_fill_kernel<<<nbf, 256, 0, s>>>(n, nnodes, N.nslices, D, nvel, A.rp, A.ci, A.val, N.perm, N.wa, N.wb, N.cptr,
                                       N.vptr, N.col, N.val, N.pair);
    count_launch();
    RAV_CHECK_LAUNCH();
    for (void* p : {(void*)na, (void*)nbv, (void*)key, (void*)skey, (void*)idx, (void*)woff, d_tmp, (void*)csz,
                    (void*)vsz})
        cudaFreeAsync(p, s);
    RAV_CUDA(cudaStreamSynchronize(s));
    N.nvel = nvel;
    static const bool compress = [] {
        const char* e = getenv("RAV_NB_COMPRESS");
        return !(e && atoi(e) == 0);
    }();
    if (compress) RAV_TRY(nb_compress(N, s));
    static const bool bvals = [] {
        const char* e = getenv("RAV_NB_BVALS");
        return !(e && atoi(e) == 0);
    }();
    if (bvals && N.tbl) RAV_TRY(nb_compress_bvals(N, s));
    return RAV_OK;
}

void nb_free(NodeBlocked& N) {
    for (void* p : {(void*)N.perm, (void*)N.wa, (void*)N.wb, (void*)N.cptr, (void*)N.vptr, (void*)N.col, (void*)N.val,
                    (void*)N.pid, (void*)N.baseA, (void*)N.baseB, (void*)N.tbl, (void*)N.vofs, (void*)N.vtbl})
        if (p) cudaFree(p);
    N = NodeBlocked{};
}

// threads per block of the residual kernel (128 or 256; the kernel is compiled for <= 256).
// Measured with the B-value table: 128 is 2-4% faster (c2 61.6 -> 60.1 us, c3 872 -> 840 us)
static int nb_block_threads() {
    static const int bs = [] {
        const char* e = getenv("RAV_NB_BS");
        const int v = e ? atoi(e) : 128;
        return v == 128 || v == 64 ? v : 256;
    }();
    return bs;
}

template <int D, int G, int UA, bool PR = false, bool XA = false>
static void nb_launch(const NodeBlocked& N, const double* x, const double* b, double* r, double* part, int nblk,
                      cudaStream_t s, int* used, const void* xpf, int64_t xpf_bytes) {
    static const int bulk = [] {   // measured: c2 85.2 -> 81.1 us, c3 1549 -> 1426 us
        const char* e = getenv("RAV_NB_BULK");
        return e ? atoi(e) : 1;
    }();
    NbCols cols{N.col, N.pid, N.baseA, N.baseB, N.tbl, N.W, bulk, N.vofs, N.vtbl, nullptr, 0, 0};
    const int bs = nb_block_threads();
    const int64_t full = cdiv(N.nslices * NB_C * G, bs);
    // with partial norms: one partial per block, the full grid when the caller's buffer holds it
    const int blocks = (int)(part ? std::min<int64_t>(full, nblk) : full);
    if (used) *used = blocks;
    if (xpf && xpf_bytes >= 16) {   // 16-byte aligned segments, at most half the grid's warps
        const uintptr_t a = (reinterpret_cast<uintptr_t>(xpf) + 15) & ~(uintptr_t)15;
        cols.xpf = reinterpret_cast<const char*>(a);
        cols.xpf_bytes = (xpf_bytes - (int64_t)(a - reinterpret_cast<uintptr_t>(xpf))) & ~(int64_t)15;
        cols.xpf_warps = std::min<int64_t>(cdiv(cols.xpf_bytes, NB_XPF_SEG), (int64_t)blocks * (bs / 32) / 2);
    }
    static const int minb = [] {   // register cap of the one-thread-per-row variant (measured: 6 best, 102 vs 105 us)
        const char* e = getenv("RAV_NB_MINB");
        return e ? atoi(e) : 6;
    }();
    static const int minb3 = [] {   // register cap of the 3D two-lane variant with the B-value table
        const char* e = getenv("RAV_NB_MINB3");   // measured c4: 1 61.4 us, 4 58.8 us (64 registers), 5 60.3 us
        return e ? atoi(e) : 4;
    }();
    if constexpr (D == 3 && G == 2) {
        if (N.vtbl && minb3 >= 4) {
            auto k3 = minb3 >= 5 ? nb_residual_kernel<D, G, UA, 5, true, PR, XA, true>
                                 : nb_residual_kernel<D, G, UA, 4, true, PR, XA, true>;
            launch_maybe_pdl(k3, dim3(blocks), dim3(bs), 0, s, N.nblock, N.nnodes, N.nslices, N.nvel,
                             (const int32_t*)N.perm, (const int32_t*)N.wa, (const int32_t*)N.wb,
                             (const int64_t*)N.cptr, (const int64_t*)N.vptr, cols, (const double*)N.val, x, b, r,
                             part);
            return;
        }
    }
    auto kern = N.vtbl ? ((minb >= 8 && G == 1) ? nb_residual_kernel<D, G, UA, 8, true, PR, XA, true>
                         : (minb >= 6 && G == 1) ? nb_residual_kernel<D, G, UA, 6, true, PR, XA, true>
                         : (minb == 5 && G == 1) ? nb_residual_kernel<D, G, UA, 5, true, PR, XA, true>
                                                 : nb_residual_kernel<D, G, UA, 1, true, PR, XA, true>)
              : N.tbl ? ((minb >= 8 && G == 1) ? nb_residual_kernel<D, G, UA, 8, true, PR, XA>
                         : (minb >= 6 && G == 1) ? nb_residual_kernel<D, G, UA, 6, true, PR, XA>
                         : (minb == 5 && G == 1) ? nb_residual_kernel<D, G, UA, 5, true, PR, XA>
                                                 : nb_residual_kernel<D, G, UA, 1, true, PR, XA>)
              : (minb >= 8 && G == 1) ? nb_residual_kernel<D, G, UA, 8, false, PR>
              : (minb >= 6 && G == 1) ? nb_residual_kernel<D, G, UA, 6, false, PR>
                                      : nb_residual_kernel<D, G, UA, 1, false, PR>;
    launch_maybe_pdl(kern, dim3(blocks), dim3(bs), 0, s, N.nblock, N.nnodes, N.nslices,
                     N.nvel, (const int32_t*)N.perm, (const int32_t*)N.wa, (const int32_t*)N.wb,
                     (const int64_t*)N.cptr, (const int64_t*)N.vptr, cols, (const double*)N.val, x, b,
                     r, part);
}

static int nb_lanes(const NodeBlocked& N) {
    static const int genv = [] {
        const char* e = getenv("RAV_NB_LANES");   // lanes per block row (0: by dimension)
        return e ? atoi(e) : 0;
    }();
    // measured: 3D c4 98 us (G=2) vs 110 (G=1), 111 (G=4); 2D c2 G=1 best.  Small (coarse) levels
    // cannot fill the GPU with one short group per row: their long rows get a full warp (latency)
    static const int64_t t32 = [] {   // block rows below which a row gets a full warp (32 lanes, 3D)
        const char* e = getenv("RAV_NB_T32");
        return e ? atoll(e) : 8192;
    }();
    static const int64_t t8 = [] {    // ... 8 lanes (3D) / 2 lanes (2D)
        const char* e = getenv("RAV_NB_T8");
        return e ? atoll(e) : 131072;
    }();
    const int G = genv > 0 ? genv
                           : N.nblock < t32 ? (N.D == 3 ? 32 : 8)
                           : N.nblock < t8 ? (N.D == 3 ? 8 : 2)
                           : (N.D == 3 ? 2 : 1);
    return G >= 32 ? 32 : (G >= 8 ? 8 : (G >= 4 ? 4 : (G >= 2 ? 2 : 1)));
}


int64_t nb_full_blocks(const NodeBlocked& N) { return cdiv(N.nslices * NB_C * nb_lanes(N), nb_block_threads()); }

rav_status launch_nb_residual(const Csr& A, const double* x, const double* b, double* r, double* part, int nblk,
                              cudaStream_t s, int* used, const void* xpf, int64_t xpf_bytes) {
    const NodeBlocked& N = A.nb;
    const int G = nb_lanes(N);
    if (N.D == 3) {
        if (G == 32) nb_launch<3, 32, 2>(N, x, b, r, part, nblk, s, used, xpf, xpf_bytes);
        else if (G == 8) nb_launch<3, 8, 4>(N, x, b, r, part, nblk, s, used, xpf, xpf_bytes);
        else if (G == 4) nb_launch<3, 4, 4>(N, x, b, r, part, nblk, s, used, xpf, xpf_bytes);
        else if (G == 2) nb_launch<3, 2, 4>(N, x, b, r, part, nblk, s, used, xpf, xpf_bytes);
        else nb_launch<3, 1, 8>(N, x, b, r, part, nblk, s, used, xpf, xpf_bytes);
    } else {
        if (N.pair && (reinterpret_cast<uintptr_t>(x) & 15) == 0 && G == 1) {
            nb_launch<2, 1, 4, true, true>(N, x, b, r, part, nblk, s, used, xpf, xpf_bytes);
        } else if (N.pair) {
            if (G == 32) nb_launch<2, 32, 2, true>(N, x, b, r, part, nblk, s, used, xpf, xpf_bytes);
            else if (G == 8) nb_launch<2, 8, 4, true>(N, x, b, r, part, nblk, s, used, xpf, xpf_bytes);
            else if (G >= 4) nb_launch<2, 4, 4, true>(N, x, b, r, part, nblk, s, used, xpf, xpf_bytes);
            else if (G == 2) nb_launch<2, 2, 4, true>(N, x, b, r, part, nblk, s, used, xpf, xpf_bytes);
            else nb_launch<2, 1, 4, true>(N, x, b, r, part, nblk, s, used, xpf, xpf_bytes);
        } else {
            if (G == 32) nb_launch<2, 32, 2>(N, x, b, r, part, nblk, s, used, xpf, xpf_bytes);
            else if (G == 8) nb_launch<2, 8, 4>(N, x, b, r, part, nblk, s, used, xpf, xpf_bytes);
            else if (G >= 4) nb_launch<2, 4, 4>(N, x, b, r, part, nblk, s, used, xpf, xpf_bytes);
            else if (G == 2) nb_launch<2, 2, 4>(N, x, b, r, part, nblk, s, used, xpf, xpf_bytes);
            else nb_launch<2, 1, 4>(N, x, b, r, part, nblk, s, used, xpf, xpf_bytes);
        }
    }
    count_launch();
    RAV_CHECK_LAUNCH();
    return RAV_OK;
}

}  // namespace rav
