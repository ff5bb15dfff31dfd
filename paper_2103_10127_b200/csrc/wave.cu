// wave.cu -- band-pipelined RAV sweeps (opt-in: RAV_WAVE=1; SURVEY section 8 rows a2 + a5).
//
// A sweep is two grid-wide phases, the residual R (r = b - L x) and the RAV update A
// (x += omega sum_i R_i^T W_i r_i).  Issued as separate kernels, each phase waits for the
// whole previous one (griddepcontrol.wait), so every launch pays a ramp and a partial last
// wave (DESIGN 5.1: about 15 us for A and 9 us for R at c2, size-independent).  Here the
// kernels are still launched back to back with programmatic dependent launch, but a CTA
// waits only for the parts of the previous phase it actually reads or overwrites:
//   * the sweep's chunks are grouped in A-bands (WB_CHUNKS consecutive chunks: patches in
//     vertex order, so a band is a strip of the grid); the residual's CTAs in R-bands
//     (WR_CTAS consecutive CTAs);
//   * residual CTA u of sweep s waits until the A-bands of sweep s-1 that write the x
//     entries it reads, or read the r rows it overwrites, are done;
//   * A-band b of sweep s waits until the R-bands of sweep s that write the r entries it
//     reads, or read the x entries it updates, are done.
// The dependency ranges come from the operator and the patch lists at setup (wave_build);
// an A-band waits on up to three R-band ranges (node rows, pressure rows, the one band that
// holds both).  Completion is counted per band: the CTA barrier, then one release add.  A
// wait: one thread per band polls with relaxed loads and issues an acquire fence, then the
// CTA barrier.  x and r are then read with weak L1-cacheable loads (the fence invalidated
// the SM's L1).  Measured: correct, but no faster than the plain chain (DESIGN 7).
//
// Progress: a kernel of the chain is launched only after every CTA of its predecessor has
// started (the trigger is the first instruction), so every CTA a waiter depends on is
// resident or finished, and the waits form a chain back to the first kernel, which waits
// with griddepcontrol.wait.  A wait that exceeds ~2 s traps (a launch error, not a hang).
#include <climits>
#include <vector>

#include "internal.cuh"

namespace rav {
namespace {

constexpr int W_NBC = 32;       // slots per SELL slice (nb.cu NB_C)
constexpr int WB_CHUNKS = 64;   // chunks per A-band (16 CTAs of 4 one-chunk warps)
constexpr int WR_CTAS = 16;     // residual CTAs (256 slots each) per R-band
constexpr int W_RES_BS = 256;

// x / r loads after a wait: weak, L1-cacheable ld.global (not the non-coherent path: the data
// change during the kernel's lifetime).  The waiting thread's acquire fence invalidates the SM's
// L1 (CCTL.IVALL), so a line cached afterwards already holds every write the CTA waited for.
#ifndef RAV_WAVE_LOAD
#define RAV_WAVE_LOAD 3   // 0: ld.relaxed.gpu; 1: ld.global.cg; 3: weak ld.global (measured equal, fewest constraints)
#endif
__device__ __forceinline__ void ld2_strong(const double* p, double* out) {
#if RAV_WAVE_LOAD == 0
    asm volatile("ld.relaxed.gpu.global.v2.f64 {%0, %1}, [%2];" : "=d"(out[0]), "=d"(out[1]) : "l"(p) : "memory");
#elif RAV_WAVE_LOAD == 3
    // plain C++ load through a pointer without __restrict__: weak ld.global (never the non-coherent
    // path), ordered by the compiler after the wait's barrier, free to be scheduled for ILP
    const double2 v = *reinterpret_cast<const double2*>(p);
    out[0] = v.x; out[1] = v.y;
#else
    const double2 v = __ldcg(reinterpret_cast<const double2*>(p));
    out[0] = v.x; out[1] = v.y;
#endif
}
__device__ __forceinline__ double ld_strong(const double* p) {
#if RAV_WAVE_LOAD == 0
    double v;
    asm volatile("ld.relaxed.gpu.global.f64 %0, [%1];" : "=d"(v) : "l"(p) : "memory");
    return v;
#elif RAV_WAVE_LOAD == 3
    return *p;
#else
    return __ldcg(p);
#endif
}
__device__ __forceinline__ void red_release(unsigned* p, unsigned v) {
    asm volatile("red.release.gpu.global.add.u32 [%0], %1;" ::"l"(p), "r"(v) : "memory");
}
__device__ __forceinline__ unsigned ld_relaxed_u32(const unsigned* p) {
    unsigned v;
    asm volatile("ld.relaxed.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
    return v;
}
// The CTA waits until done[b] >= mult * cnt[b] for every band b of up to three ranges.  Thread k
// polls the k-th band of the concatenated ranges (all polls in flight at once: one L2 round trip
// when the producers are done), with relaxed loads, then issues its own acquire fence; the
// barrier orders the CTA's later loads after every polling thread's fence.
__device__ __forceinline__ void wait_ranges(const unsigned* done, const int32_t* cnt, const int32_t* lo,
                                            const int32_t* hi, int nr, unsigned mult) {
    int k = threadIdx.x, b = -1;
    for (int q = 0; q < nr && b < 0; ++q) {
        const int w = hi[q] >= lo[q] ? hi[q] - lo[q] + 1 : 0;
        if (k < w) b = lo[q] + k;
        else k -= w;
    }
    if (b >= 0) {
        const unsigned target = mult * (unsigned)cnt[b];
        long long it = 0;
        while (ld_relaxed_u32(done + b) < target) {
            __nanosleep(64);
            if (++it > (1ll << 24)) __trap();
        }
        asm volatile("fence.acq_rel.gpu;" ::: "memory");
    }
    __syncthreads();
}

// every thread's writes, then the CTA barrier, then one release add (cumulative over the writes
// the barrier ordered before it)
__device__ __forceinline__ void signal_band(unsigned* done, int b) {
    __syncthreads();
    if (threadIdx.x == 0) red_release(done + b, 1u);
}

// ---- setup: dependency ranges --------------------------------------------------------------
__global__ void w_fill_kernel(int64_t n, int32_t* a, int32_t v) {
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x)
        a[i] = v;
}

// per DoF: the A-bands reading r there (rmin/rmax) and writing x there (wmin/wmax)
__global__ void w_patch_kernel(int64_t np, int64_t nchunks, int NN, int D, const int32_t* __restrict__ ND,
                               const int32_t* __restrict__ PD, const int32_t* __restrict__ NR, int32_t* rmin,
                               int32_t* rmax, int32_t* wmin, int32_t* wmax) {
    for (int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; t < nchunks * 32; t += (int64_t)gridDim.x * blockDim.x) {
        const int64_t chunk = t / 32, i = t;
        const int lane = (int)(t % 32);
        if (i >= np) continue;
        const int b = (int)(chunk / WB_CHUNKS);
        const int m = NR[i];
        for (int j = 0; j < NN; ++j) {
            const int nd = ND[(chunk * NN + j) * 32 + lane];
            for (int c = 0; c < D; ++c) {
                atomicMin(rmin + nd + c, b);
                atomicMax(rmax + nd + c, b);
                if (j < m) { atomicMin(wmin + nd + c, b); atomicMax(wmax + nd + c, b); }
            }
        }
        const int pd = PD[i];
        atomicMin(rmin + pd, b); atomicMax(rmax + pd, b);
        atomicMin(wmin + pd, b); atomicMax(wmax + pd, b);
    }
}

// per residual slot: its rows' R-band (rowR), the R-bands reading x per column (xmin/xmax), and
// per residual CTA the A-band range it waits for (alo/ahi)
__global__ void w_resid_kernel(int64_t nslots, int64_t n, int64_t nnodes, int64_t nvel, int64_t nall, int D,
                               const int32_t* __restrict__ perm, const int64_t* __restrict__ rp,
                               const int32_t* __restrict__ ci, const int32_t* __restrict__ wmin,
                               const int32_t* __restrict__ wmax, const int32_t* __restrict__ rmin,
                               const int32_t* __restrict__ rmax, int32_t* rowR, int32_t* xmin, int32_t* xmax,
                               int32_t* alo, int32_t* ahi) {
    for (int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; t < nslots; t += (int64_t)gridDim.x * blockDim.x) {
        if (t >= n) continue;
        const int64_t u = t / W_RES_BS;
        const int rb = (int)(u / WR_CTAS);
        const int64_t br = perm[t];
        const int nr = br < nnodes ? D : 1;
        int lo = INT_MAX, hi = -1;
        for (int c = 0; c < nr; ++c) {
            const int64_t row = br < nnodes ? br * D + c : nvel + (br - nnodes);
            rowR[row] = rb;
            if (rmax[row] >= 0) { lo = min(lo, rmin[row]); hi = max(hi, rmax[row]); }
            for (int64_t k = rp[row]; k < rp[row + 1]; ++k) {
                const int col = ci[k];
                // R-bands reading x[col], by kind of the reading row (velocity: xmin/xmax[col],
                // pressure: xmin/xmax[n + col])
                const int64_t slot = br < nnodes ? col : nall + col;
                atomicMin(xmin + slot, rb);
                atomicMax(xmax + slot, rb);
                if (wmax[col] >= 0) { lo = min(lo, wmin[col]); hi = max(hi, wmax[col]); }
            }
        }
        if (hi >= 0) { atomicMin(alo + u, lo); atomicMax(ahi + u, hi); }
    }
}

// kind of each R-band: 0 only node rows, 1 only pressure rows, 2 both (the slot order puts all node
// rows first, so only the band at the boundary holds both)
__global__ void w_rkind_kernel(int nR, int64_t nslots, int64_t n, int64_t nnodes, const int32_t* __restrict__ perm,
                               int32_t* rkind) {
    for (int rb = blockIdx.x * blockDim.x + threadIdx.x; rb < nR; rb += gridDim.x * blockDim.x) {
        const int64_t t0 = (int64_t)rb * WR_CTAS * W_RES_BS;
        const int64_t t1 = min(nslots, t0 + (int64_t)WR_CTAS * W_RES_BS) - 1;
        const bool first_p = t0 < n && perm[t0] >= nnodes;
        const int64_t tl = min(t1, n - 1);
        const bool last_p = tl >= t0 && perm[tl] >= nnodes;
        rkind[rb] = first_p ? 1 : (last_p ? 2 : 0);
    }
}

// per A-band: the R-band ranges it waits for, one over the R-bands holding velocity rows and one
// over those holding pressure rows (rlo/rhi[2 b + kind]; with node rows first in the residual's
// slot order the two sets are far apart, and one range would span everything in between)
__global__ void w_band_kernel(int64_t np, int64_t nchunks, int NN, int D, const int32_t* __restrict__ ND,
                              const int32_t* __restrict__ PD, const int32_t* __restrict__ NR,
                              const int32_t* __restrict__ rowR, const int32_t* __restrict__ xmin,
                              const int32_t* __restrict__ xmax, const int32_t* __restrict__ rkind, int64_t nall,
                              int32_t* rlo, int32_t* rhi) {
    for (int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; t < nchunks * 32; t += (int64_t)gridDim.x * blockDim.x) {
        const int64_t chunk = t / 32, i = t;
        const int lane = (int)(t % 32);
        if (i >= np) continue;
        const int b = (int)(chunk / WB_CHUNKS);
        const int m = NR[i];
        int lo[3] = {INT_MAX, INT_MAX, INT_MAX}, hi[3] = {-1, -1, -1};
        auto add = [&](int rb) {
            if (rb < 0) return;
            const int k = rkind[rb];
            lo[k] = min(lo[k], rb);
            hi[k] = max(hi[k], rb);
        };
        auto take = [&](int64_t d, bool written) {
            add(rowR[d]);
            if (written) {
                if (xmax[d] >= 0) { add(xmin[d]); add(xmax[d]); }                  // velocity rows reading x[d]
                if (xmax[nall + d] >= 0) { add(xmin[nall + d]); add(xmax[nall + d]); }   // pressure rows
            }
        };
        for (int j = 0; j < NN; ++j) {
            const int nd = ND[(chunk * NN + j) * 32 + lane];
            for (int c = 0; c < D; ++c) take(nd + c, j < m);
        }
        take(PD[i], true);
        for (int k = 0; k < 3; ++k)
            if (hi[k] >= 0) { atomicMin(rlo + 3 * b + k, lo[k]); atomicMax(rhi + 3 * b + k, hi[k]); }
    }
}

// ---- residual (node-blocked, one thread per 2D block row, stencil-compressed columns, pairs) --
struct WRes {
    int64_t n, nnodes, nslices, nvel;
    const int32_t *perm, *wa, *wb, *pid, *baseA, *baseB, *tbl;
    const int64_t* vptr;
    int W;
    const double* v;
    const int32_t *alo, *ahi, *cntA;
    const unsigned* doneA;
    unsigned* doneR;
};

__global__ void __launch_bounds__(256, 6) wave_residual_kernel(WRes R, const double* x,
                                                               const double* __restrict__ b, double* __restrict__ r,
                                                               int first, unsigned sweep) {
    pdl_trigger();
    const int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;   // slot
    const int64_t s = t / W_NBC;
    const int l = (int)(t % W_NBC);
    const int lane = threadIdx.x & 31;
    if (s < R.nslices && lane == 0) bulk_prefetch_l2(R.v + R.vptr[s], (uint32_t)((R.vptr[s + 1] - R.vptr[s]) * 8));
    if (first) pdl_wait();
    else if (R.ahi[blockIdx.x] >= 0) wait_ranges(R.doneA, R.cntA, R.alo + blockIdx.x, R.ahi + blockIdx.x, 1, sweep);
    const int64_t br = t < R.n ? R.perm[t] : -1;
    if (br >= 0) {
        const int A = R.wa[s], B = R.wb[s];
        const int32_t* tp = R.tbl + (int64_t)R.pid[t] * R.W;
        const int32_t bA = R.baseA[t], bB = R.baseB[t];
        const double* vs = R.v + R.vptr[s];
        const double2* pA = reinterpret_cast<const double2*>(vs) + l;
        const double2* pB = reinterpret_cast<const double2*>(vs + (int64_t)A * W_NBC) + l;
        if (br < R.nnodes) {
            double acc0 = 0.0, acc1 = 0.0;
            const int A2 = A >> 1;
#pragma unroll 1
            for (int p = 0; p < A2; ++p) {
                const double2 a = __ldcs(pA + (int64_t)p * W_NBC);
                double x0[2], x1[2];
                ld2_strong(x + bA + __ldg(tp + 2 * p), x0);
                ld2_strong(x + bA + __ldg(tp + 2 * p + 1), x1);
                acc0 = fma(a.x, x0[0], acc0);
                acc1 = fma(a.x, x0[1], acc1);
                acc0 = fma(a.y, x1[0], acc0);
                acc1 = fma(a.y, x1[1], acc1);
            }
            if (A & 1) {
                const double a = __ldcs(vs + (int64_t)(2 * A2) * W_NBC + l);
                double x0[2];
                ld2_strong(x + bA + __ldg(tp + A - 1), x0);
                acc0 = fma(a, x0[0], acc0);
                acc1 = fma(a, x0[1], acc1);
            }
#pragma unroll 2
            for (int k = 0; k < B; ++k) {
                const double xp = ld_strong(x + bB + __ldg(tp + A + k));
                const double2 bv = __ldcs(pB + (int64_t)k * W_NBC);
                acc0 = fma(bv.x, xp, acc0);
                acc1 = fma(bv.y, xp, acc1);
            }
            const int64_t r0 = br * 2;
            const double2 bb = __ldg(reinterpret_cast<const double2*>(b + r0));
            *reinterpret_cast<double2*>(r + r0) = make_double2(bb.x - acc0, bb.y - acc1);
        } else {
            double acc = 0.0;
#pragma unroll 4
            for (int k = 0; k < B; ++k) {
                double xv[2];
                ld2_strong(x + bB + __ldg(tp + A + k), xv);
                const double2 bv = __ldcs(pB + (int64_t)k * W_NBC);
                acc = fma(bv.x, xv[0], acc);
                acc = fma(bv.y, xv[1], acc);
            }
            const int64_t row = R.nvel + (br - R.nnodes);
            r[row] = b[row] - acc;
        }
    }
    signal_band(R.doneR, (int)(blockIdx.x / WR_CTAS));
}

// ---- RAV update (2D PoU interior shape: 9 restricted nodes, 25 nodes, one patch per thread) ----
struct WSw {
    int64_t np, nchunks, pairs;
    const double2* W;
    const int32_t *ND, *PD, *NR;
    const double* AUX;
    const int32_t *rlo, *rhi, *cntR;
    const unsigned* doneR;
    unsigned* doneA;
};

__global__ void __launch_bounds__(128, 4) wave_sweep_kernel(WSw S, const double* r,
                                                            double* __restrict__ x, double omega, int first,
                                                            unsigned sweep) {   // sweep: R-band count multiplier
    constexpr int MT = 9, D = 2, NRB = 8, NN = 25, PF = 2;
    constexpr int TRI = MT * (MT + 1) / 2 + MT * D;
    constexpr int TRI_PAD = TRI + (TRI & 1);
    constexpr int RC = MT + D;
    pdl_trigger();
    const int64_t chunk = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
    const int lane = threadIdx.x & 31;
    const int64_t i = chunk * 32 + lane;
    const bool live = chunk < S.nchunks;
    const int band = (int)((blockIdx.x * 4) / WB_CHUNKS);
    const double2* wp = S.W + (live ? chunk : 0) * S.pairs * 32 + lane;
    const int32_t* np_ = S.ND + (live ? chunk : 0) * (int64_t)NN * 32 + lane;
    if (live) {
        const char* wc = reinterpret_cast<const char*>(S.W + chunk * S.pairs * 32);
        const char* nc = reinterpret_cast<const char*>(S.ND + chunk * (int64_t)NN * 32);
        if (lane < NN) prefetch_l2(nc + (size_t)lane * 128);
        if (lane == 0) bulk_prefetch_l2(wc, (uint32_t)((TRI_PAD / 2 + PF * RC) * 512));
    }
    if (first) pdl_wait();
    else wait_ranges(S.doneR, S.cntR, S.rlo + 3 * band, S.rhi + 3 * band, 3, sweep);
    if (live) {
        double acc[MT][D], rr[MT][D], gR[MT][D];
        double gacc = 0.0;
#pragma unroll
        for (int k = 0; k < MT; ++k) {
            ld2_strong(r + __ldcs(np_ + k * 32), rr[k]);
#pragma unroll
            for (int c = 0; c < D; ++c) acc[k][c] = 0.0;
        }
        double2 pv = make_double2(0.0, 0.0);
#pragma unroll
        for (int j = 0; j < MT; ++j) {
#pragma unroll
            for (int q = 0; q <= j + D; ++q) {
                const int e = j * (j + 1) / 2 + j * D + q;
                if ((e & 1) == 0) pv = __ldcs(wp + (e >> 1) * 32);
                const double v = (e & 1) ? pv.y : pv.x;
                if (q <= j) {
#pragma unroll
                    for (int c = 0; c < D; ++c) {
                        acc[q][c] = fma(v, rr[j][c], acc[q][c]);
                        if (q != j) acc[j][c] = fma(v, rr[q][c], acc[j][c]);
                    }
                } else {
                    const int c = q - j - 1;
                    gR[j][c] = v;
                    gacc = fma(v, rr[j][c], gacc);
                }
            }
        }
        const double2* wq0 = wp + (TRI_PAD / 2) * 32;
#pragma unroll
        for (int bb = 0; bb < NRB; ++bb) {
            const int j0 = MT + 2 * bb;
            if (lane == 0 && bb + PF < NRB)
                bulk_prefetch_l2(S.W + chunk * S.pairs * 32 + (int64_t)(TRI_PAD / 2 + (bb + PF) * RC) * 32,
                                 (uint32_t)(RC * 512));
            double ra[D], rb[D];
            ld2_strong(r + __ldcs(np_ + j0 * 32), ra);
            ld2_strong(r + __ldcs(np_ + (j0 + 1) * 32), rb);
            const double2* wq = wq0 + (int64_t)bb * RC * 32;
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
        const double* aux = S.AUX + chunk * (MT + 2) * 32 + lane;
        const int pd = S.PD[i];
        const double t = aux[(MT + 1) * 32] * (gacc - ld_strong(r + pd));
        if (i < S.np) {
            const int m = S.NR[i];
#pragma unroll
            for (int k = 0; k < MT; ++k) {
                if (k < m) {
                    const double wk = omega * aux[k * 32];
                    const int nd = __ldcs(np_ + k * 32);
#pragma unroll
                    for (int c = 0; c < D; ++c) atomicAdd(x + nd + c, wk * fma(gR[k][c], t, acc[k][c]));
                }
            }
            const double wpr = aux[MT * 32];
            if (wpr != 0.0) atomicAdd(x + pd, omega * wpr * (-t));
        }
    }
    signal_band(S.doneA, band);
}

static int grid_for(int64_t n) { return (int)std::max<int64_t>(1, std::min<int64_t>(cdiv(n, 256), (int64_t)num_sms() * 16)); }

}  // namespace

void wave_free(Wave& V) {
    for (void* p : {(void*)V.alo, (void*)V.ahi, (void*)V.rlo, (void*)V.rhi, (void*)V.cntA, (void*)V.cntR,
                    (void*)V.done})
        if (p) cudaFree(p);
    V = Wave{};
}

// dependency ranges of the pipelined sweep; V.on stays 0 when the operator / smoother layout is
// not the one the pipelined kernels implement (2D node-blocked residual with compressed columns
// and value pairs, one lane per row; Schur thread layout of the PoU interior shape)
rav_status wave_build(const Csr& A, const Factors& F, int64_t n_patches, int nb_lanes_used, Wave& V,
                      cudaStream_t s) {
    wave_free(V);
    const NodeBlocked& N = A.nb;
    if (!(N.nslices > 0 && N.D == 2 && N.pair && N.tbl && nb_lanes_used == 1)) return RAV_OK;
    // (the node-index compression keeps F.DT, which the pipelined sweep reads)
    if (!(F.layout == 4 && F.MT == 9 && F.NN == 25 && F.D == 2 && !F.cbuf && F.DT)) return RAV_OK;
    const int64_t n = A.n_rows;
    const int64_t nslots = N.nslices * W_NBC;
    const int64_t nres = cdiv(nslots, W_RES_BS);              // residual CTAs
    const int64_t nsw = cdiv(F.nchunks * 32, 128);            // sweep CTAs (4 chunks each)
    V.nA = (int)cdiv(F.nchunks, WB_CHUNKS);
    V.nR = (int)cdiv(nres, WR_CTAS);
    V.nres = nres;
    V.nsw = nsw;
    int32_t *rmin, *rmax, *wmin, *wmax, *rowR, *xmin, *xmax;
    RAV_CUDA(cudaMallocAsync(&rmin, sizeof(int32_t) * n, s));
    RAV_CUDA(cudaMallocAsync(&rmax, sizeof(int32_t) * n, s));
    RAV_CUDA(cudaMallocAsync(&wmin, sizeof(int32_t) * n, s));
    RAV_CUDA(cudaMallocAsync(&wmax, sizeof(int32_t) * n, s));
    RAV_CUDA(cudaMallocAsync(&rowR, sizeof(int32_t) * n, s));
    RAV_CUDA(cudaMallocAsync(&xmin, sizeof(int32_t) * 2 * n, s));
    RAV_CUDA(cudaMallocAsync(&xmax, sizeof(int32_t) * 2 * n, s));
    int32_t* rkind = nullptr;
    RAV_CUDA(cudaMalloc(&V.alo, sizeof(int32_t) * nres));
    RAV_CUDA(cudaMalloc(&V.ahi, sizeof(int32_t) * nres));
    RAV_CUDA(cudaMalloc(&V.rlo, sizeof(int32_t) * 3 * V.nA));
    RAV_CUDA(cudaMalloc(&V.rhi, sizeof(int32_t) * 3 * V.nA));
    RAV_CUDA(cudaMallocAsync(&rkind, sizeof(int32_t) * V.nR, s));
    RAV_CUDA(cudaMalloc(&V.cntA, sizeof(int32_t) * V.nA));
    RAV_CUDA(cudaMalloc(&V.cntR, sizeof(int32_t) * V.nR));
    RAV_CUDA(cudaMalloc(&V.done, sizeof(unsigned) * (V.nA + V.nR)));
    const int g = grid_for(std::max<int64_t>(n, nslots));
    for (auto pr : {std::make_pair(rmin, INT_MAX), std::make_pair(wmin, INT_MAX), std::make_pair(rmax, -1),
                    std::make_pair(wmax, -1), std::make_pair(rowR, -1)})
        w_fill_kernel<<<g, 256, 0, s>>>(n, pr.first, pr.second);
    w_fill_kernel<<<g, 256, 0, s>>>(2 * n, xmin, INT_MAX);
    w_fill_kernel<<<g, 256, 0, s>>>(2 * n, xmax, -1);
    w_fill_kernel<<<g, 256, 0, s>>>(nres, V.alo, INT_MAX);
    w_fill_kernel<<<g, 256, 0, s>>>(nres, V.ahi, -1);
    w_fill_kernel<<<g, 256, 0, s>>>(3 * V.nA, V.rlo, INT_MAX);
    w_fill_kernel<<<g, 256, 0, s>>>(3 * V.nA, V.rhi, -1);
    w_rkind_kernel<<<g, 256, 0, s>>>(V.nR, nslots, N.nblock, N.nnodes, N.perm, rkind);
    RAV_CHECK_LAUNCH();
    w_patch_kernel<<<g, 256, 0, s>>>(n_patches, F.nchunks, F.NN, F.D, F.DT, F.PD, F.NR, rmin, rmax, wmin, wmax);
    w_resid_kernel<<<g, 256, 0, s>>>(nslots, N.nblock, N.nnodes, N.nvel, n, N.D, N.perm, A.rp, A.ci, wmin, wmax,
                                     rmin, rmax, rowR, xmin, xmax, V.alo, V.ahi);
    w_band_kernel<<<g, 256, 0, s>>>(n_patches, F.nchunks, F.NN, F.D, F.DT, F.PD, F.NR, rowR, xmin, xmax, rkind, n,
                                    V.rlo, V.rhi);
    RAV_CHECK_LAUNCH();
    // per-band CTA counts
    std::vector<int32_t> ca(V.nA), cr(V.nR);
    for (int b = 0; b < V.nA; ++b)
        ca[b] = (int32_t)(std::min<int64_t>(nsw, (int64_t)(b + 1) * WB_CHUNKS / 4) - (int64_t)b * WB_CHUNKS / 4);
    for (int b = 0; b < V.nR; ++b)
        cr[b] = (int32_t)(std::min<int64_t>(nres, (int64_t)(b + 1) * WR_CTAS) - (int64_t)b * WR_CTAS);
    RAV_CUDA(cudaMemcpyAsync(V.cntA, ca.data(), sizeof(int32_t) * V.nA, cudaMemcpyHostToDevice, s));
    RAV_CUDA(cudaMemcpyAsync(V.cntR, cr.data(), sizeof(int32_t) * V.nR, cudaMemcpyHostToDevice, s));
    // report the widest ranges (diagnostics)
    std::vector<int32_t> hlo(nres), hhi(nres), blo(3 * V.nA), bhi(3 * V.nA);
    RAV_CUDA(cudaMemcpyAsync(hlo.data(), V.alo, sizeof(int32_t) * nres, cudaMemcpyDeviceToHost, s));
    RAV_CUDA(cudaMemcpyAsync(hhi.data(), V.ahi, sizeof(int32_t) * nres, cudaMemcpyDeviceToHost, s));
    RAV_CUDA(cudaMemcpyAsync(blo.data(), V.rlo, sizeof(int32_t) * 3 * V.nA, cudaMemcpyDeviceToHost, s));
    RAV_CUDA(cudaMemcpyAsync(bhi.data(), V.rhi, sizeof(int32_t) * 3 * V.nA, cudaMemcpyDeviceToHost, s));
    RAV_CUDA(cudaStreamSynchronize(s));
    for (void* p : {(void*)rmin, (void*)rmax, (void*)wmin, (void*)wmax, (void*)rowR, (void*)xmin, (void*)xmax,
                    (void*)rkind})
        cudaFreeAsync(p, s);
    V.maxA = V.maxR = 0;
    for (int64_t u = 0; u < nres; ++u)
        if (hhi[u] >= 0) V.maxA = std::max(V.maxA, hhi[u] - hlo[u] + 1);
    for (int b = 0; b < V.nA; ++b) {
        int w = 0;
        for (int k = 0; k < 3; ++k)
            if (bhi[3 * b + k] >= 0) w += bhi[3 * b + k] - blo[3 * b + k] + 1;
        V.maxR = std::max(V.maxR, w);
    }
    if (getenv("RAV_WAVE_VERBOSE") && atoi(getenv("RAV_WAVE_VERBOSE")) > 1) {
        for (int64_t u = 0; u < nres; u += std::max<int64_t>(1, nres / 40))
            fprintf(stderr, "  R-CTA %lld waits A-bands [%d, %d]\n", (long long)u, hlo[u], hhi[u]);
        for (int b = 0; b < V.nA; b += std::max(1, V.nA / 20))
            fprintf(stderr, "  A-band %d waits R-bands [%d, %d] [%d, %d] [%d, %d]\n", b, blo[3 * b], bhi[3 * b],
                    blo[3 * b + 1], bhi[3 * b + 1], blo[3 * b + 2], bhi[3 * b + 2]);
        int wide = 0;
        for (int64_t u = 0; u < nres; ++u)
            if (hhi[u] - hlo[u] > 8) ++wide;
        fprintf(stderr, "  %d of %lld residual CTAs wait on more than 9 A-bands\n", wide, (long long)nres);
    }
    if (getenv("RAV_WAVE_VERBOSE"))
        fprintf(stderr, "wave: %d A-bands, %d R-bands, %lld residual CTAs, %lld sweep CTAs; widest waits %d A-bands, %d R-bands\n",
                V.nA, V.nR, (long long)nres, (long long)nsw, V.maxA, V.maxR);
    V.on = 1;
    return RAV_OK;
}

// nu sweeps of the pipelined chain; r_ready: r already holds b - L x (the first residual is skipped)
rav_status wave_smooth(const Csr& A, const Factors& F, int64_t n_patches, const Wave& V, double* x, const double* b,
                       double* r, int nu, double omega, bool r_ready, cudaStream_t s) {
    const NodeBlocked& N = A.nb;
    RAV_CUDA(cudaMemsetAsync(V.done, 0, sizeof(unsigned) * (V.nA + V.nR), s));
    unsigned* doneA = V.done;
    unsigned* doneR = V.done + V.nA;
    const WRes R{N.nblock, N.nnodes, N.nslices, N.nvel, N.perm, N.wa, N.wb, N.pid, N.baseA, N.baseB, N.tbl,
                 N.vptr, N.W, N.val, V.alo, V.ahi, V.cntA, doneA, doneR};
    const WSw S{n_patches, F.nchunks, F.pairs, reinterpret_cast<const double2*>(F.facT), F.DT, F.PD, F.NR, F.WT,
                V.rlo, V.rhi, V.cntR, doneR, doneA};
    int nres_done = 0;   // residual kernels issued so far in this chain
    for (int k = 0; k < nu; ++k) {
        const bool skip_r = r_ready && k == 0;
        if (!skip_r) {
            // sweep k's residual waits for the updates of sweeps 0 .. k-1 (done counts k * cnt); the
            // chain's first kernel waits for the previous stream work instead
            RAV_CUDA(launch_maybe_pdl(wave_residual_kernel, dim3((unsigned)V.nres), dim3(W_RES_BS), 0, s, R, x, b, r,
                                      k == 0 ? 1 : 0, (unsigned)k));
            count_launch();
            ++nres_done;
        }
        // the update of sweep k waits for the residual kernels issued so far (done counts
        // nres_done * cnt); with the first residual skipped it is the chain's first kernel
        RAV_CUDA(launch_maybe_pdl(wave_sweep_kernel, dim3((unsigned)V.nsw), dim3(128), 0, s, S, (const double*)r, x,
                                  omega, skip_r ? 1 : 0, (unsigned)nres_done));
        count_launch();
    }
    RAV_CHECK_LAUNCH();
    return RAV_OK;
}

}  // namespace rav
