// setup.cu -- batched local setup of the Vanka subdomains (SURVEY section 8 row
// a4): for every patch i, gather L_i = R_i L R_i^T from the CSR,
// factor L_i^T by Gaussian elimination with partial pivoting and solve
// L_i^T y = e_k for its restricted DoFs k, giving the rows
//     W_i[k][:] = w_k * (row k of L_i^{-1})
// i.e. only the rows RAV applies are ever stored ("only requires the
// storage of certain rows"); the damping omega is applied at sweep time.
//
// One CTA per patch (grid-stride).  The augmented matrix [L_i^T | E] lives in
// shared memory when it fits (2D: 51 x 70 doubles = 28.6 KB, 7 CTAs/SM), else
// in a per-CTA global scratch slot (3D 376 x 458) that stays L2-resident.
//
// Output layouts:
//   general (layout 1): per patch a row-major nres_i x n_i block at foffs[i].
//   SoA (layout 2):     patches in chunks of 32 (one per lane of the sweep
//     kernel); entry e = j*NT + k of patch (chunk, lane) stored at double
//     index ((chunk*PAIRS + e/2)*32 + lane)*2 + e%2, so each warp-wide 16-byte
//     load of the sweep reads 512 contiguous bytes.  DoF lists likewise
//     DT[(chunk*NMAX + j)*32 + lane].
#include <algorithm>
#include <cub/cub.cuh>
#include <vector>

#include "internal.cuh"

namespace rav {

static bool is_dev(const void* p) {
    cudaPointerAttributes a;
    if (cudaPointerGetAttributes(&a, p) != cudaSuccess) { cudaGetLastError(); return false; }
    return a.type == cudaMemoryTypeDevice || a.type == cudaMemoryTypeManaged;
}

// per patch: size, restricted count, validation
__global__ void patch_stats_kernel(int64_t np, const int64_t* offs, const double* w, int64_t ndofs,
                                   const int32_t* dofs, int32_t* nres, int64_t* rows_sz,
                                   unsigned int* nmax, unsigned int* rmax, unsigned int* err) {
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < np; i += (int64_t)gridDim.x * blockDim.x) {
        int64_t s = offs[i], e = offs[i + 1];
        int n = (int)(e - s);
        int m = 0;
        for (int64_t k = s; k < e; ++k) {
            if (w[k] > 0.0) ++m;
            if (dofs[k] < 0 || dofs[k] >= ndofs) atomicOr(err, 2u);
        }
        if (n <= 0) atomicOr(err, 1u);
        nres[i] = m;
        rows_sz[i] = (int64_t)m * n;
        atomicMax(nmax, (unsigned)n);
        atomicMax(rmax, (unsigned)m);
    }
}

// stable partition of each patch: restricted (w > 0) entries first
__global__ void patch_reorder_kernel(int64_t np, const int64_t* offs, const int32_t* dofs, const double* w,
                                     int32_t* odofs, double* ow) {
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < np; i += (int64_t)gridDim.x * blockDim.x) {
        int64_t s = offs[i], e = offs[i + 1], p = s;
        for (int pass = 0; pass < 2; ++pass)
            for (int64_t k = s; k < e; ++k)
                if ((w[k] > 0.0) == (pass == 0)) { odofs[p] = dofs[k]; ow[p] = w[k]; ++p; }
    }
}

rav_status patches_upload(const rav_patches* P, int64_t n_dofs, PatchSet& out, cudaStream_t s) {
    if (!P || P->n_patches < 1 || !P->offs || !P->dofs || !P->weight) {
        set_error("rav_patches: NULL pointer or no patches");
        return RAV_ERR_ARG;
    }
    if (P->on_device != (int)is_dev(P->offs)) {
        set_error("rav_patches: on_device flag does not match the offs pointer kind");
        return RAV_ERR_ARG;
    }
    cudaMemcpyKind kind = P->on_device ? cudaMemcpyDeviceToDevice : cudaMemcpyHostToDevice;
    out.n_patches = P->n_patches;
    int64_t tot = 0;
    RAV_CUDA(cudaMemcpyAsync(&tot, P->offs + P->n_patches, sizeof(int64_t),
                             P->on_device ? cudaMemcpyDeviceToHost : cudaMemcpyHostToHost, s));
    RAV_CUDA(cudaStreamSynchronize(s));
    if (tot < 1) { set_error("rav_patches: no entries"); return RAV_ERR_ARG; }
    out.entries = tot;
    int32_t* tdofs = nullptr;
    double* tw = nullptr;
    int64_t* rows_sz = nullptr;
    unsigned int* stats = nullptr;
    RAV_CUDA(cudaMalloc(&out.offs, sizeof(int64_t) * (out.n_patches + 1)));
    RAV_CUDA(cudaMalloc(&out.dofs, sizeof(int32_t) * tot));
    RAV_CUDA(cudaMalloc(&out.w, sizeof(double) * tot));
    RAV_CUDA(cudaMalloc(&out.nres, sizeof(int32_t) * out.n_patches));
    RAV_CUDA(cudaMallocAsync(&tdofs, sizeof(int32_t) * tot, s));
    RAV_CUDA(cudaMallocAsync(&tw, sizeof(double) * tot, s));
    RAV_CUDA(cudaMallocAsync(&rows_sz, sizeof(int64_t) * out.n_patches, s));
    RAV_CUDA(cudaMallocAsync(&stats, sizeof(unsigned int) * 3, s));
    RAV_CUDA(cudaMemsetAsync(stats, 0, sizeof(unsigned int) * 3, s));
    RAV_CUDA(cudaMemcpyAsync(out.offs, P->offs, sizeof(int64_t) * (out.n_patches + 1), kind, s));
    RAV_CUDA(cudaMemcpyAsync(tdofs, P->dofs, sizeof(int32_t) * tot, kind, s));
    RAV_CUDA(cudaMemcpyAsync(tw, P->weight, sizeof(double) * tot, kind, s));
    int nb = (int)std::min<int64_t>(cdiv(out.n_patches, 256), (int64_t)num_sms() * 16);
    patch_stats_kernel<<<nb, 256, 0, s>>>(out.n_patches, out.offs, tw, n_dofs, tdofs, out.nres, rows_sz,
                                          stats, stats + 1, stats + 2);
    count_launch();
    RAV_CHECK_LAUNCH();
    patch_reorder_kernel<<<nb, 256, 0, s>>>(out.n_patches, out.offs, tdofs, tw, out.dofs, out.w);
    count_launch();
    RAV_CHECK_LAUNCH();
    // total rows size = sum nres_i n_i
    int64_t* d_sum = nullptr;
    size_t tmp = 0;
    RAV_CUDA(cub::DeviceReduce::Sum(nullptr, tmp, rows_sz, (int64_t*)nullptr, out.n_patches, s));
    void* d_tmp = nullptr;
    RAV_CUDA(cudaMallocAsync(&d_tmp, tmp + 16, s));
    RAV_CUDA(cudaMallocAsync(&d_sum, sizeof(int64_t), s));
    RAV_CUDA(cub::DeviceReduce::Sum(d_tmp, tmp, rows_sz, d_sum, out.n_patches, s));
    unsigned int h_stats[3];
    int64_t h_sum = 0;
    RAV_CUDA(cudaMemcpyAsync(h_stats, stats, sizeof(h_stats), cudaMemcpyDeviceToHost, s));
    RAV_CUDA(cudaMemcpyAsync(&h_sum, d_sum, sizeof(int64_t), cudaMemcpyDeviceToHost, s));
    cudaFreeAsync(d_tmp, s);
    cudaFreeAsync(d_sum, s);
    cudaFreeAsync(tdofs, s);
    cudaFreeAsync(tw, s);
    cudaFreeAsync(rows_sz, s);
    cudaFreeAsync(stats, s);
    RAV_CUDA(cudaStreamSynchronize(s));
    if (h_stats[2] & 1u) { set_error("rav_patches: empty patch (S:302)"); return RAV_ERR_ARG; }
    if (h_stats[2] & 2u) { set_error("rav_patches: DoF index out of range"); return RAV_ERR_ARG; }
    out.nmax = (int)h_stats[0];
    out.nresmax = (int)h_stats[1];
    out.rows_total = h_sum;
    {   // host-side totals for the byte model (sum nres, sum of the symmetric-format entries)
        std::vector<int32_t> hn(out.n_patches);
        std::vector<int64_t> ho(out.n_patches + 1);
        RAV_CUDA(cudaMemcpy(hn.data(), out.nres, sizeof(int32_t) * out.n_patches, cudaMemcpyDeviceToHost));
        RAV_CUDA(cudaMemcpy(ho.data(), out.offs, sizeof(int64_t) * (out.n_patches + 1), cudaMemcpyDeviceToHost));
        int64_t sm = 0, ss = 0;
        for (int64_t i = 0; i < out.n_patches; ++i) {
            int64_t m = hn[i], n = ho[i + 1] - ho[i];
            sm += m;
            ss += m * (m + 1) / 2 + m * (n - m);
        }
        out.nres_total = sm;
        out.sym_total = ss;
    }
    if (out.nresmax < 1) { set_error("rav_patches: no restricted DoF (weight > 0) in any patch"); return RAV_ERR_ARG; }
    return RAV_OK;
}

void patches_free(PatchSet& P) {
    if (P.offs) cudaFree(P.offs);
    if (P.dofs) cudaFree(P.dofs);
    if (P.w) cudaFree(P.w);
    if (P.nres) cudaFree(P.nres);
    P = PatchSet{};
}

// ------------------------------------------------------------------------------------
// The factorization kernel
// ------------------------------------------------------------------------------------
struct FactorArgs {
    const int64_t* rp;
    const int32_t* ci;
    const double* val;
    int64_t np;
    const int64_t* poffs;
    const int32_t* pdofs;
    const double* pw;
    const int32_t* pnres;
    int variant;        // 0 rows, 1 diag Vanka
    int64_t nvel;
    int nmax, mmax;     // workspace dims
    int ld;             // leading dimension of the augmented matrix
    // outputs
    int layout;         // 1 general, 2 SoA
    const int64_t* foffs;
    double* fac;
    int NT, NMAX, NTRI;
    double* facT;
    int32_t* DT;
    int32_t* NR;
    double* WT;
    double* gscratch;   // when not using smem: per-CTA slot of nmax*ld doubles
    unsigned long long* bad;
};

constexpr int FT = 128;  // threads per factorization CTA

__global__ void __launch_bounds__(FT) factor_kernel(FactorArgs a) {
    extern __shared__ double smem[];
    const int tid = threadIdx.x;
    // shared layout: [aug (if smem)] [rn: nmax] [sdofs: nmax int] [sperm: nmax int] [misc]
    double* aug;
    double* rn;
    size_t aug_elems = (size_t)a.nmax * a.ld;
    if (a.gscratch) {
        aug = a.gscratch + (size_t)blockIdx.x * aug_elems;
        rn = smem;
    } else {
        aug = smem;
        rn = smem + aug_elems;
    }
    int32_t* sdofs = (int32_t*)(rn + a.nmax);
    int32_t* sperm = sdofs + a.nmax;
    int32_t* ldofs = sperm + a.nmax;
    __shared__ int s_piv;
    __shared__ int s_fail;

    for (int64_t i = blockIdx.x; i < a.np; i += gridDim.x) {
        const int64_t off = a.poffs[i];
        const int n = (int)(a.poffs[i + 1] - off);
        const int m = a.pnres[i];
        const int W = n + m;
        const int ld = a.ld;
        __syncthreads();
        for (int t = tid; t < n; t += FT) ldofs[t] = a.pdofs[off + t];
        for (int t = tid; t < n * ld; t += FT) aug[t] = 0.0;
        if (tid == 0) s_fail = 0;
        __syncthreads();
        // sorted copy of the patch DoFs with their local positions
        for (int t = tid; t < n; t += FT) {
            int d = ldofs[t], rank = 0;
            for (int u = 0; u < n; ++u) rank += (ldofs[u] < d);
            sdofs[rank] = d;
            sperm[rank] = t;
        }
        __syncthreads();
        // gather M = L_i^T: M[a][b] = L[dof_b][dof_a]; thread per local row b scans CSR row dof_b
        for (int b = tid; b < n; b += FT) {
            const int row = ldofs[b];
            const bool vb = row < a.nvel;
            for (int64_t k = a.rp[row]; k < a.rp[row + 1]; ++k) {
                int c = a.ci[k];
                int lo = 0, hi = n - 1, pos = -1;
                while (lo <= hi) {
                    int mid = (lo + hi) >> 1;
                    int sd = sdofs[mid];
                    if (sd == c) { pos = mid; break; }
                    if (sd < c) lo = mid + 1; else hi = mid - 1;
                }
                if (pos < 0) continue;
                int la = sperm[pos];
                if (a.variant == 1 && vb && c < a.nvel && la != b) continue;  // diag Vanka: A_i -> diag(A_i)
                aug[(size_t)la * ld + b] = a.val[k];
            }
        }
        // right-hand sides e_k for the restricted local DoFs k < m (restricted first)
        for (int k = tid; k < m; k += FT) aug[(size_t)k * ld + n + k] = 1.0;
        __syncthreads();
        // row norms of M (pivot tolerance)
        for (int r = tid; r < n; r += FT) {
            double mx = 0.0;
            for (int c = 0; c < n; ++c) mx = fmax(mx, fabs(aug[(size_t)r * ld + c]));
            rn[r] = mx;
        }
        __syncthreads();
        // Gaussian elimination with partial pivoting on [M | E]
        for (int c = 0; c < n; ++c) {
            if (tid < 32) {
                double best = -1.0;
                int bi = c;
                for (int r = c + tid; r < n; r += 32) {
                    double v = fabs(aug[(size_t)r * ld + c]);
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
                    if (!(best > 1e-14 * rn[bi])) s_fail = 1;
                }
            }
            __syncthreads();
            if (s_fail) break;
            const int p = s_piv;
            if (p != c) {
                for (int t = c + tid; t < W; t += FT) {
                    double u = aug[(size_t)c * ld + t];
                    aug[(size_t)c * ld + t] = aug[(size_t)p * ld + t];
                    aug[(size_t)p * ld + t] = u;
                }
                if (tid == 0) { double u = rn[c]; rn[c] = rn[p]; rn[p] = u; }
            }
            __syncthreads();
            const double inv = 1.0 / aug[(size_t)c * ld + c];
            const int nr = n - c - 1, nc = W - c - 1;
            for (int t = tid; t < nr * nc; t += FT) {
                int r = c + 1 + t / nc, col = c + 1 + t % nc;
                double f = aug[(size_t)r * ld + c] * inv;
                aug[(size_t)r * ld + col] -= f * aug[(size_t)c * ld + col];
            }
            __syncthreads();
        }
        if (s_fail) {
            if (tid == 0) atomicMin(a.bad, (unsigned long long)i);
            continue;
        }
        // back substitution, column oriented: Y overwrites the RHS block
        for (int c = n - 1; c >= 0; --c) {
            for (int t = tid; t < m; t += FT) aug[(size_t)c * ld + n + t] /= aug[(size_t)c * ld + c];
            __syncthreads();
            for (int t = tid; t < c * m; t += FT) {
                int r = t / m, k = t % m;
                aug[(size_t)r * ld + n + k] -= aug[(size_t)r * ld + c] * aug[(size_t)c * ld + n + k];
            }
            __syncthreads();
        }
        // store W[k][j] = w_k * Y[j][k]
        if (a.layout == 1) {
            double* dst = a.fac + a.foffs[i];
            for (int t = tid; t < m * n; t += FT) {
                int k = t / n, j = t % n;
                dst[t] = a.pw[off + k] * aug[(size_t)j * ld + n + k];
            }
        } else if (a.layout == 2) {
            const int64_t chunk = i >> 5;
            const int lane = (int)(i & 31);
            const int64_t pairs = (int64_t)a.NMAX * a.NT / 2;
            double* base = a.facT + chunk * pairs * 64;
            for (int t = tid; t < m * n; t += FT) {
                int k = t / n, j = t % n;
                int64_t e = (int64_t)j * a.NT + k;
                base[((e >> 1) * 32 + lane) * 2 + (e & 1)] = a.pw[off + k] * aug[(size_t)j * ld + n + k];
            }
            for (int j = tid; j < a.NMAX; j += FT)
                a.DT[(chunk * a.NMAX + j) * 32 + lane] = j < n ? ldofs[j] : ldofs[0];
            if (tid == 0) a.NR[i] = m;
        } else {
            // layout 3 (symmetric): the restricted x restricted block of L_i^{-1} is symmetric
            // (L_i = R_i L R_i^T with L symmetric), so columns j < NT keep only rows k <= j
            // (entry e = j(j+1)/2 + k, taken from row k); columns j >= NT keep rows k < NT
            // (entry e = NTRI + (j - NT) NT + k).  Values are UNweighted rows of L_i^{-1};
            // the weights w_k go to WT and are applied once per row in the sweep.
            const int64_t chunk = i >> 5;
            const int lane = (int)(i & 31);
            const int NT = a.NT;
            const int64_t pairs = ((int64_t)a.NTRI + (int64_t)(a.NMAX - NT) * NT) / 2;
            double* base = a.facT + chunk * pairs * 64;
            for (int t = tid; t < m * n; t += FT) {
                int k = t / n, j = t % n;
                int64_t e;
                if (j < NT) {
                    if (k > j) continue;           // stored from row j (j < k < m)
                    e = (int64_t)j * (j + 1) / 2 + k;
                } else {
                    e = a.NTRI + (int64_t)(j - NT) * NT + k;
                }
                base[((e >> 1) * 32 + lane) * 2 + (e & 1)] = aug[(size_t)j * ld + n + k];
            }
            for (int j = tid; j < a.NMAX; j += FT)
                a.DT[(chunk * a.NMAX + j) * 32 + lane] = j < n ? ldofs[j] : ldofs[0];
            for (int k = tid; k < m; k += FT) a.WT[(chunk * NT + k) * 32 + lane] = a.pw[off + k];
            if (tid == 0) a.NR[i] = m;
        }
    }
}

__global__ void rows_size_kernel(int64_t np, const int64_t* offs, const int32_t* nres, int64_t* sz);

bool thread_kernel_supported(int nresmax, int nmax) { return nresmax <= 32 && nmax <= 64; }

int pick_NT(int nresmax) {
    static const int cand[] = {3, 4, 8, 9, 12, 16, 19, 24, 32};
    for (int c : cand)
        if (c >= nresmax) return c;
    return -1;
}

rav_status factorize(const Csr& A, const PatchSet& P, int variant, int64_t nvel, int kernel_choice,
                     Factors& F, int64_t* bad_patch, cudaStream_t s) {
    FactorArgs a{};
    a.rp = A.rp;
    a.ci = A.ci;
    a.val = A.val;
    a.np = P.n_patches;
    a.poffs = P.offs;
    a.pdofs = P.dofs;
    a.pw = P.w;
    a.pnres = P.nres;
    a.variant = variant;
    a.nvel = nvel;
    a.nmax = P.nmax;
    a.mmax = P.nresmax;
    a.ld = P.nmax + P.nresmax;
    if ((a.ld & 15) == 0) a.ld += 1;   // avoid power-of-two strides in shared memory
    bool use_thread = kernel_choice != RAV_KERNEL_WARP && thread_kernel_supported(P.nresmax, P.nmax);
    if ((kernel_choice == RAV_KERNEL_THREAD || kernel_choice == RAV_KERNEL_SYM) && !use_thread) {
        set_error("thread-per-patch kernels need nres <= 32 and n <= 64 (got %d, %d)", P.nresmax, P.nmax);
        return RAV_ERR_ARG;
    }
    if (use_thread && kernel_choice != RAV_KERNEL_THREAD) {
        F.layout = 3;
        F.NT = pick_NT(P.nresmax);
        F.NMAX = std::max(F.NT, P.nmax);
        if ((F.NMAX - F.NT) & 1) F.NMAX += 1;
        F.NTRI = F.NT * (F.NT + 1) / 2;
        F.NTRI += F.NTRI & 1;
        F.nchunks = cdiv(P.n_patches, 32);
        int64_t pairs = ((int64_t)F.NTRI + (int64_t)(F.NMAX - F.NT) * F.NT) / 2;
        size_t fac_bytes = sizeof(double) * 2 * pairs * 32 * F.nchunks;
        RAV_CUDA(cudaMalloc(&F.facT, fac_bytes));
        RAV_CUDA(cudaMalloc(&F.DT, sizeof(int32_t) * F.NMAX * 32 * F.nchunks));
        RAV_CUDA(cudaMalloc(&F.NR, sizeof(int32_t) * 32 * F.nchunks));
        RAV_CUDA(cudaMalloc(&F.WT, sizeof(double) * F.NT * 32 * F.nchunks));
        RAV_CUDA(cudaMemsetAsync(F.facT, 0, fac_bytes, s));
        RAV_CUDA(cudaMemsetAsync(F.DT, 0, sizeof(int32_t) * F.NMAX * 32 * F.nchunks, s));
        RAV_CUDA(cudaMemsetAsync(F.NR, 0, sizeof(int32_t) * 32 * F.nchunks, s));
        RAV_CUDA(cudaMemsetAsync(F.WT, 0, sizeof(double) * F.NT * 32 * F.nchunks, s));
        F.bytes = (int64_t)fac_bytes + sizeof(int32_t) * F.NMAX * 32 * F.nchunks + sizeof(double) * F.NT * 32 * F.nchunks;
        a.layout = 3;
        a.NT = F.NT;
        a.NMAX = F.NMAX;
        a.NTRI = F.NTRI;
        a.facT = F.facT;
        a.DT = F.DT;
        a.NR = F.NR;
        a.WT = F.WT;
    } else if (use_thread) {
        F.layout = 2;
        F.NT = pick_NT(P.nresmax);
        F.NMAX = (P.nmax + 1) & ~1;
        F.nchunks = cdiv(P.n_patches, 32);
        int64_t pairs = (int64_t)F.NMAX * F.NT / 2;
        RAV_CUDA(cudaMalloc(&F.facT, sizeof(double) * 2 * pairs * 32 * F.nchunks));
        RAV_CUDA(cudaMalloc(&F.DT, sizeof(int32_t) * F.NMAX * 32 * F.nchunks));
        RAV_CUDA(cudaMalloc(&F.NR, sizeof(int32_t) * 32 * F.nchunks));
        RAV_CUDA(cudaMemsetAsync(F.facT, 0, sizeof(double) * 2 * pairs * 32 * F.nchunks, s));
        RAV_CUDA(cudaMemsetAsync(F.DT, 0, sizeof(int32_t) * F.NMAX * 32 * F.nchunks, s));
        RAV_CUDA(cudaMemsetAsync(F.NR, 0, sizeof(int32_t) * 32 * F.nchunks, s));
        F.bytes = (int64_t)sizeof(double) * 2 * pairs * 32 * F.nchunks + sizeof(int32_t) * F.NMAX * 32 * F.nchunks;
        a.layout = 2;
        a.NT = F.NT;
        a.NMAX = F.NMAX;
        a.facT = F.facT;
        a.DT = F.DT;
        a.NR = F.NR;
    } else {
        F.layout = 1;
        int64_t* sz = nullptr;
        RAV_CUDA(cudaMalloc(&F.foffs, sizeof(int64_t) * (P.n_patches + 1)));
        RAV_CUDA(cudaMalloc(&F.fac, sizeof(double) * (P.rows_total > 0 ? P.rows_total : 1)));
        // foffs from nres_i * n_i
        RAV_CUDA(cudaMallocAsync(&sz, sizeof(int64_t) * P.n_patches, s));
        int nb = (int)std::min<int64_t>(cdiv(P.n_patches, 256), (int64_t)num_sms() * 16);
        rows_size_kernel<<<nb, 256, 0, s>>>(P.n_patches, P.offs, P.nres, sz);
        count_launch();
        RAV_CHECK_LAUNCH();
        RAV_TRY(gen::counts_to_rowptr(sz, F.foffs, P.n_patches, s));
        cudaFreeAsync(sz, s);
        F.bytes = (int64_t)sizeof(double) * P.rows_total;
        a.layout = 1;
        a.foffs = F.foffs;
        a.fac = F.fac;
    }
    unsigned long long* bad = nullptr;
    RAV_CUDA(cudaMallocAsync(&bad, sizeof(unsigned long long), s));
    RAV_CUDA(cudaMemsetAsync(bad, 0xff, sizeof(unsigned long long), s));
    a.bad = bad;
    size_t aug_bytes = sizeof(double) * (size_t)a.nmax * a.ld;
    size_t aux_bytes = sizeof(double) * a.nmax + sizeof(int32_t) * 3 * a.nmax + 64;
    const size_t smem_cap = 100 * 1024;
    int grid;
    size_t shmem;
    if (aug_bytes + aux_bytes <= smem_cap) {
        shmem = aug_bytes + aux_bytes;
        a.gscratch = nullptr;
        int per_sm = (int)std::max<size_t>(1, std::min<size_t>(16, (200 * 1024) / shmem));
        grid = (int)std::min<int64_t>(P.n_patches, (int64_t)num_sms() * per_sm);
    } else {
        shmem = aux_bytes;
        grid = (int)std::min<int64_t>(P.n_patches, (int64_t)num_sms() * 2);
        RAV_CUDA(cudaMallocAsync(&a.gscratch, aug_bytes * grid, s));
    }
    if (shmem > 48 * 1024) RAV_CUDA(cudaFuncSetAttribute(factor_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)shmem));
    factor_kernel<<<grid, FT, shmem, s>>>(a);
    count_launch();
    RAV_CHECK_LAUNCH();
    unsigned long long h_bad = 0;
    RAV_CUDA(cudaMemcpyAsync(&h_bad, bad, sizeof(h_bad), cudaMemcpyDeviceToHost, s));
    cudaFreeAsync(bad, s);
    if (a.gscratch) cudaFreeAsync(a.gscratch, s);
    RAV_CUDA(cudaStreamSynchronize(s));
    if (h_bad != ~0ULL) {
        if (bad_patch) *bad_patch = (int64_t)h_bad;
        set_error("singular local system in patch %lld", (long long)h_bad);
        return RAV_ERR_SINGULAR_LOCAL;
    }
    if (bad_patch) *bad_patch = -1;
    return RAV_OK;
}

__global__ void rows_size_kernel(int64_t np, const int64_t* offs, const int32_t* nres, int64_t* sz) {
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < np; i += (int64_t)gridDim.x * blockDim.x)
        sz[i] = (int64_t)nres[i] * (offs[i + 1] - offs[i]);
}

void factors_free(Factors& F) {
    if (F.foffs) cudaFree(F.foffs);
    if (F.fac) cudaFree(F.fac);
    if (F.facT) cudaFree(F.facT);
    if (F.DT) cudaFree(F.DT);
    if (F.NR) cudaFree(F.NR);
    if (F.WT) cudaFree(F.WT);
    if (F.PD) cudaFree(F.PD);
    if (F.nodes) cudaFree(F.nodes);
    if (F.nodeoffs) cudaFree(F.nodeoffs);
    for (void* p : {(void*)F.cbuf, (void*)F.det_dof, (void*)F.det_off, (void*)F.det_slot, (void*)F.npid,
                    (void*)F.nbase, (void*)F.ntbl, (void*)F.wtab, (void*)F.ntab, (void*)F.SINV})
        if (p) cudaFree(p);
    F = Factors{};
}

// canonical export (general layout) of the SoA factors
__global__ void export_soa_kernel(int64_t np, const int64_t* offs, const int32_t* nres, const int64_t* roffs,
                                  int NT, int NMAX, const double* facT, double* rows) {
    for (int64_t i = blockIdx.x; i < np; i += gridDim.x) {
        int n = (int)(offs[i + 1] - offs[i]);
        int m = nres[i];
        const int64_t chunk = i >> 5;
        const int lane = (int)(i & 31);
        const int64_t pairs = (int64_t)NMAX * NT / 2;
        const double* base = facT + chunk * pairs * 64;
        for (int t = threadIdx.x; t < m * n; t += blockDim.x) {
            int k = t / n, j = t % n;
            int64_t e = (int64_t)j * NT + k;
            rows[roffs[i] + t] = base[((e >> 1) * 32 + lane) * 2 + (e & 1)];
        }
    }
}

// layout 3 -> W[k][j] = w_k * Linv[k][j] (mirrored triangle for restricted columns)
__global__ void export_sym_kernel(int64_t np, const int64_t* offs, const int32_t* nres, const int64_t* roffs,
                                  int NT, int NMAX, int NTRI, const double* facT, const double* WT, double* rows) {
    for (int64_t i = blockIdx.x; i < np; i += gridDim.x) {
        int n = (int)(offs[i + 1] - offs[i]);
        int m = nres[i];
        const int64_t chunk = i >> 5;
        const int lane = (int)(i & 31);
        const int64_t pairs = ((int64_t)NTRI + (int64_t)(NMAX - NT) * NT) / 2;
        const double* base = facT + chunk * pairs * 64;
        for (int t = threadIdx.x; t < m * n; t += blockDim.x) {
            int k = t / n, j = t % n;
            int64_t e;
            if (j < NT) e = k <= j ? (int64_t)j * (j + 1) / 2 + k : (int64_t)k * (k + 1) / 2 + j;
            else e = NTRI + (int64_t)(j - NT) * NT + k;
            rows[roffs[i] + t] = WT[(chunk * NT + k) * 32 + lane] * base[((e >> 1) * 32 + lane) * 2 + (e & 1)];
        }
    }
}

rav_status export_rows(const PatchSet& P, const Factors& F, double* rows, cudaStream_t s) {
    if (F.layout == 1) {
        RAV_CUDA(cudaMemcpyAsync(rows, F.fac, sizeof(double) * P.rows_total, cudaMemcpyDeviceToDevice, s));
        return RAV_OK;
    }
    int64_t *sz = nullptr, *roffs = nullptr;
    RAV_CUDA(cudaMallocAsync(&sz, sizeof(int64_t) * P.n_patches, s));
    RAV_CUDA(cudaMallocAsync(&roffs, sizeof(int64_t) * (P.n_patches + 1), s));
    int nb = (int)std::min<int64_t>(cdiv(P.n_patches, 256), (int64_t)num_sms() * 16);
    rows_size_kernel<<<nb, 256, 0, s>>>(P.n_patches, P.offs, P.nres, sz);
    count_launch();
    RAV_TRY(gen::counts_to_rowptr(sz, roffs, P.n_patches, s));
    int g = (int)std::min<int64_t>(P.n_patches, (int64_t)num_sms() * 8);
    if (F.layout == 3)
        export_sym_kernel<<<g, 128, 0, s>>>(P.n_patches, P.offs, P.nres, roffs, F.NT, F.NMAX, F.NTRI, F.facT, F.WT,
                                            rows);
    else
        export_soa_kernel<<<g, 128, 0, s>>>(P.n_patches, P.offs, P.nres, roffs, F.NT, F.NMAX, F.facT, rows);
    count_launch();
    RAV_CHECK_LAUNCH();
    cudaFreeAsync(sz, s);
    cudaFreeAsync(roffs, s);
    RAV_CUDA(cudaStreamSynchronize(s));
    return RAV_OK;
}

}  // namespace rav
