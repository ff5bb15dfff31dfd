// dist.cu -- the slab-partitioned smoother and V-cycle inside the library (include/ravgmg.h,
// "Slab-partitioned (multi-GPU) smoother and V-cycle"; SURVEY section 8 rows a11 / b / e).
//
// RAV is additive (Eq. 13): within a sweep every patch reads the same residual and the
// corrections are summed, so the patches shard across subdomains with one exchange step per
// sweep: the partial corrections that a subdomain's patches write on DoFs owned
// by a neighbour are sent to the owner and added there, then the owners refresh every ghost
// copy.  This file drives, per process, one or more subdomains (their own rav_ctx smoothers on
// windowed operators) through
//   residual -> zero ghost-written -> sweep -> pack -> send/recv -> add + pack -> send/recv -> unpack
// and the V-cycle of dist.py's protocol (restriction with windowed transfers, coarse partial sums
// to the owners, agglomerated multigrid below the partitioned levels), all stream-ordered and
// captured as CUDA graphs.  Pack / unpack of every subdomain and neighbour of one phase is ONE
// launch (one CTA row per message).  Messages between subdomains of the same process are not
// copied: the receiver reads the sender's packed buffer directly (the launch boundary orders
// them); messages to other processes (or, with via_comm, all of them) are NCCL sends / receives
// in one group per phase, ordered by (source, destination) subdomain so both ends post them in
// the same order.  Sums over subdomains (coarse right-hand side, norms) are formed in ascending
// subdomain order from an all-gather, so they are bitwise identical on every process.
#include <dlfcn.h>
#include <time.h>
#include <nccl.h>   // types and enums only; the functions are resolved from libnccl.so.2 at run time

#include <algorithm>
#include <map>
#include <tuple>
#include <vector>

#include "ctx.cuh"

namespace rav {
namespace {

// ---- NCCL, loaded at run time ------------------------------------------------------------
struct NcclApi {
    ncclResult_t (*GetUniqueId)(ncclUniqueId*) = nullptr;
    ncclResult_t (*CommInitRank)(ncclComm_t*, int, ncclUniqueId, int) = nullptr;
    ncclResult_t (*CommDestroy)(ncclComm_t) = nullptr;
    ncclResult_t (*Send)(const void*, size_t, ncclDataType_t, int, ncclComm_t, cudaStream_t) = nullptr;
    ncclResult_t (*Recv)(void*, size_t, ncclDataType_t, int, ncclComm_t, cudaStream_t) = nullptr;
    ncclResult_t (*AllGather)(const void*, void*, size_t, ncclDataType_t, ncclComm_t, cudaStream_t) = nullptr;
    ncclResult_t (*GroupStart)() = nullptr;
    ncclResult_t (*GroupEnd)() = nullptr;
    const char* (*GetErrorString)(ncclResult_t) = nullptr;
    bool ok = false;
    char why[256] = "";
};

const NcclApi& nccl() {
    static NcclApi a = [] {
        NcclApi n;
        // the process's NCCL (torch's bundled copy when torch is loaded), else the system one
        void* h = dlopen("libnccl.so.2", RTLD_NOW | RTLD_NOLOAD);
        if (!h) h = dlopen("libnccl.so.2", RTLD_NOW | RTLD_LOCAL);
        if (!h) {
            snprintf(n.why, sizeof(n.why), "dlopen(libnccl.so.2): %s", dlerror());
            return n;
        }
#define RAV_NCCL_SYM(field, name) n.field = reinterpret_cast<decltype(n.field)>(dlsym(h, name))
        RAV_NCCL_SYM(GetUniqueId, "ncclGetUniqueId");
        RAV_NCCL_SYM(CommInitRank, "ncclCommInitRank");
        RAV_NCCL_SYM(CommDestroy, "ncclCommDestroy");
        RAV_NCCL_SYM(Send, "ncclSend");
        RAV_NCCL_SYM(Recv, "ncclRecv");
        RAV_NCCL_SYM(AllGather, "ncclAllGather");
        RAV_NCCL_SYM(GroupStart, "ncclGroupStart");
        RAV_NCCL_SYM(GroupEnd, "ncclGroupEnd");
        RAV_NCCL_SYM(GetErrorString, "ncclGetErrorString");
#undef RAV_NCCL_SYM
        n.ok = n.GetUniqueId && n.CommInitRank && n.CommDestroy && n.Send && n.Recv && n.AllGather &&
               n.GroupStart && n.GroupEnd && n.GetErrorString;
        if (!n.ok) snprintf(n.why, sizeof(n.why), "libnccl.so.2 lacks a required symbol");
        return n;
    }();
    return a;
}

#define RAV_NCCL(expr)                                                                           \
    do {                                                                                         \
        ncclResult_t _r = (expr);                                                                \
        if (_r != ncclSuccess) {                                                                 \
            ::rav::set_error("%s:%d: %s: %s", __FILE__, __LINE__, #expr, nccl().GetErrorString(_r)); \
            return RAV_ERR_COMM;                                                                 \
        }                                                                                        \
    } while (0)

bool is_dev(const void* p) {
    cudaPointerAttributes a;
    if (cudaPointerGetAttributes(&a, p) != cudaSuccess) { cudaGetLastError(); return false; }
    return a.type == cudaMemoryTypeDevice || a.type == cudaMemoryTypeManaged;
}

// ---- pack / unpack: one launch per phase, grid.y = message --------------------------------
enum { OP_GATHER = 0, OP_SCATTER = 1, OP_ADD = 2, OP_ZERO = 3, OP_DIFF = 4, OP_ADD_ATOMIC = 5, OP_ADD_CLEAR = 6,
       OP_ADD_ATOMIC_CLEAR = 7 };   // *_CLEAR: the receive buffer is an accumulator (fused sweep): zero it
constexpr int MAX_VEC = 64;

// Peer-memory transport (mgd_setup via_comm = 2): a message is written by the producer's pack
// step straight into the consumer's receive buffer (a peer-mapped allocation over NVLink when the
// consumer is another process / GPU), then the producer's last CTA sets the consumer's flag to the
// message's sequence number (release, system scope).  The consumer's step waits for the flag
// (acquire), applies the message and sets the producer's ack (so the producer does not overwrite
// a buffer that has not been consumed: it waits for ack >= its previous sequence number).  No
// NCCL call, no host involvement: the exchange is the pack / unpack kernels themselves, captured
// in the cycle's CUDA graph (the sequence counters live in device memory).  Every wait is bounded
// (~4 s): on a timeout the kernel records it in g_peer_timeout and goes on, so a broken peer can
// give wrong numbers but never a hung GPU; mgd_* return RAV_ERR_COMM when it is set.
enum { ROLE_NONE = 0, ROLE_PRODUCER = 1, ROLE_CONSUMER = 2 };

struct Step {
    int op;
    int vec;                 // index into the launch's vector table
    const int32_t* idx;      // device
    int64_t n;
    double* buf;             // device message buffer (own, the local sender's, or the peer's receive buffer)
    int role;                // ROLE_*: peer-transport synchronisation of this step
    unsigned long long* sig; // producer: the consumer's flag (remote); consumer: its own flag
    unsigned long long* ack; // producer: its own ack word; consumer: the producer's ack (remote)
    unsigned long long* seq; // this end's message counter (local)
    unsigned int* done;      // CTAs of this step that finished (local)
    int sys;                 // the other end is another process / GPU: system-scope fences, else GPU scope
};
struct VecTab {
    double* v[MAX_VEC];
};

__device__ unsigned int g_peer_timeout = 0;

__device__ __forceinline__ unsigned long long ld_acquire(const unsigned long long* p, int sys) {
    unsigned long long v;
    if (sys) asm volatile("ld.acquire.sys.global.u64 %0, [%1];" : "=l"(v) : "l"(p) : "memory");
    else asm volatile("ld.acquire.gpu.global.u64 %0, [%1];" : "=l"(v) : "l"(p) : "memory");
    return v;
}
__device__ __forceinline__ void st_release(unsigned long long* p, unsigned long long v, int sys) {
    if (sys) asm volatile("st.release.sys.global.u64 [%0], %1;" ::"l"(p), "l"(v) : "memory");
    else asm volatile("st.release.gpu.global.u64 [%0], %1;" ::"l"(p), "l"(v) : "memory");
}
__device__ void wait_geq(const unsigned long long* p, unsigned long long v, int sys) {
    for (long long spin = 0; ld_acquire(p, sys) < v; ++spin) {
        if (spin > (1ll << 24)) {   // ~4 s at 256 ns per poll
            atomicOr(&g_peer_timeout, 1u);
            return;
        }
        __nanosleep(256);
    }
}

__global__ void __launch_bounds__(256) phase_kernel(const Step* __restrict__ steps, VecTab vt) {
    const Step st = steps[blockIdx.y];
    double* V = vt.v[st.vec];
    __shared__ unsigned long long s_target;
    if (st.role != ROLE_NONE) {
        if (threadIdx.x == 0) {
            const unsigned long long s = *reinterpret_cast<volatile unsigned long long*>(st.seq);
            s_target = s + 1;
            if (st.role == ROLE_PRODUCER) wait_geq(st.ack, s, st.sys);   // the previous message was consumed
            else wait_geq(st.sig, s + 1, st.sys);                        // this message has arrived
        }
        __syncthreads();
    }
    for (int64_t k = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; k < st.n; k += (int64_t)gridDim.x * blockDim.x) {
        const int32_t i = st.idx[k];
        switch (st.op) {
            case OP_GATHER: st.buf[k] = V[i]; break;
            case OP_SCATTER: V[i] = st.buf[k]; break;
            case OP_ADD: V[i] += st.buf[k]; break;
            case OP_ZERO: V[i] = 0.0; break;
            case OP_DIFF: st.buf[k] = V[i] - st.buf[k]; break;
            case OP_ADD_CLEAR: V[i] += st.buf[k]; st.buf[k] = 0.0; break;
            case OP_ADD_ATOMIC_CLEAR: atomicAdd(V + i, st.buf[k]); st.buf[k] = 0.0; break;
            default: atomicAdd(V + i, st.buf[k]); break;
        }
    }
    if (st.role != ROLE_NONE) {
        // the CTA's payload stores (producer) / reads (consumer) are ordered before thread 0's fence by
        // the barrier, the CTAs' fences + counter before the last CTA's, and that one before its release
        // of the flag / ack (release at system scope when the other end is another GPU): causality is
        // transitive in the PTX memory model, so one GPU-scope fence per CTA and one system-scope
        // release per message suffice (a system fence per CTA cost ~4 us per launch)
        __syncthreads();
        if (threadIdx.x == 0) __threadfence();
        if (threadIdx.x == 0 && atomicAdd(st.done, 1u) == gridDim.x - 1) {   // the step's last CTA
            __threadfence();
            *st.done = 0;
            *st.seq = s_target;
            st_release(st.role == ROLE_PRODUCER ? st.sig : st.ack, s_target, st.sys);
        }
    }
}

// per patch: does it write (weight > 0) a ghost-written DoF (rmap >= 0)?  (fused sweep)
__global__ void pflag_kernel(int64_t np, const int64_t* __restrict__ offs, const int32_t* __restrict__ dofs,
                             const double* __restrict__ w, const int32_t* __restrict__ rmap, uint8_t* __restrict__ pflag) {
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < np; i += (int64_t)gridDim.x * blockDim.x) {
        uint8_t f = 0;
        for (int64_t k = offs[i]; k < offs[i + 1]; ++k)
            if (w[k] > 0.0 && rmap[dofs[k]] >= 0) f = 1;
        pflag[i] = f;
    }
}

// out[i] = sum_p parts[p * stride + i], p ascending (bitwise reproducible sums over subdomains)
__global__ void ordered_sum_kernel(const double* __restrict__ parts, int np, int64_t stride, int64_t n,
                                   double* __restrict__ out) {
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
        double s = parts[i];
        for (int p = 1; p < np; ++p) s += parts[p * stride + i];
        out[i] = s;
    }
}

struct Phase {                    // the steps of one pack / unpack launch
    std::vector<Step> h;
    Step* d = nullptr;
    int64_t nmax = 0;
};

struct Msg {                      // one NCCL message of an exchange
    int64_t key0, key1, key2;     // ordering key, identical at both ends
    int peer_proc;
    double* buf;
    int64_t n;
    bool send;
};

// one neighbour of one local subdomain: device index lists and message buffers
struct DNb {
    int32_t peer = -1;            // global subdomain id
    int peer_local = -1;          // local index of the peer subdomain (same process), else -1
    bool remote = false;          // carried by NCCL
    int64_t ncs = 0, ncr = 0, nhs = 0, nhr = 0;
    int32_t *cs = nullptr, *cr = nullptr, *hs = nullptr, *hr = nullptr;
    // send buffers (own) and receive buffers (own when remote, else the peer's send buffers)
    double *cs_buf = nullptr, *hs_buf = nullptr, *rs_buf = nullptr;   // rs: reverse halo (hr -> owner)
    double *cr_in = nullptr, *hr_in = nullptr, *rr_in = nullptr;      // rr: reverse halo received at hs
    std::vector<void*> allocs;
    // peer transport, per message type t (0 corrections, 1 halo, 2 reverse halo):
    // producing end: the consumer's receive buffer and flag, own ack; consuming end: own flag, the
    // producer's ack; each end its own sequence counter and CTA counter
    double* out_buf[3] = {nullptr, nullptr, nullptr};
    unsigned long long *out_sig[3] = {nullptr, nullptr, nullptr}, *my_ack[3] = {nullptr, nullptr, nullptr};
    unsigned long long *my_flag[3] = {nullptr, nullptr, nullptr}, *peer_ack[3] = {nullptr, nullptr, nullptr};
    unsigned long long *seq_p[3] = {nullptr, nullptr, nullptr}, *seq_c[3] = {nullptr, nullptr, nullptr};
    unsigned int *done_p[3] = {nullptr, nullptr, nullptr}, *done_c[3] = {nullptr, nullptr, nullptr};
    int64_t n_out(int t) const { return t == 0 ? ncs : t == 1 ? nhs : nhr; }   // produced entries
    int64_t n_in(int t) const { return t == 0 ? ncr : t == 1 ? nhr : nhs; }    // consumed entries
    double*& in_buf(int t) { return t == 0 ? cr_in : t == 1 ? hr_in : rr_in; }
};

struct DSub {                     // one local subdomain on one partitioned level
    int32_t gid = -1;
    rav_ctx* sm = nullptr;
    int64_t n = 0;
    std::vector<DNb> nb;
    int32_t* gw = nullptr;
    int64_t ngw = 0;
    int64_t own[4] = {0, 0, 0, 0};
    Csr P, PT;                    // prolongation from the next level / the agglomerated level
    XStruct xs;                   // its stencil form (rav_subdomain grids), used when xs.on
    double *x = nullptr, *b = nullptr, *r = nullptr;   // x, b: levels > 0 (level 0: caller's)
    bool add_atomic_c = false, add_atomic_r = false;   // corr_recv / halo_send lists overlap
    // the interface exchange fused into the sweep (peer transport): the sweep's scatter adds the
    // ghost-written DoFs' corrections straight into the consumers' receive buffers (Outbox)
    Outbox ob;
    int32_t* rmap = nullptr;      // per local DoF: (q << 24) | slot, else -1
    uint8_t* pflag = nullptr;     // per patch: writes a ghost-written DoF
};

}  // namespace
}  // namespace rav

using namespace rav;

struct rav_comm {
    int nprocs = 1, proc = 0;
    ncclComm_t nc = nullptr;
};

struct mgd_ctx {
    rav_comm* comm = nullptr;
    int nsub = 0, nl = 0, K = 0;
    std::vector<int32_t> sub_proc;
    std::vector<int32_t> local_ids;
    std::vector<std::vector<DSub>> lv;          // [K][nl]
    mg_ctx* coarse = nullptr;
    int64_t nc = 0;                             // agglomerated fine-level size
    double *bc = nullptr, *xc = nullptr;        // agglomerated rhs / iterate
    double *bc_part = nullptr;                  // [nl][nc] per-subdomain restrictions
    double *bc_loc = nullptr, *bc_all = nullptr;// this process's sum, all processes' sums [nprocs][nc]
    double *nrm_part = nullptr;                 // [nl] owned-residual squares
    double *nrm_loc = nullptr, *nrm_all = nullptr, *nrm = nullptr;
    double* h_nrm = nullptr;                    // pinned
    double* dot_part = nullptr;
    int variant = 0;
    std::vector<int64_t> ncolors;               // per level (MV)
    std::vector<std::vector<int32_t*>> plist;   // [K][nl] device colour-major patch lists (MV)
    std::vector<std::vector<std::vector<int64_t>>> coffs;   // [K][nl] colour offsets (MV)
    cudaStream_t stream = nullptr;
    bool via_comm = false;                      // every exchange through NCCL (verification)
    bool peer = false;                          // peer-memory transport (via_comm = 2)
    void* peer_block = nullptr;                 // receive buffers + flags + acks (exported by CUDA IPC)
    void* sync_block = nullptr;                 // sequence / CTA counters (local)
    bool fused = false;                         // peer transport with the exchange fused into the sweep
    void* ob_block = nullptr;                   // the fused sweeps' sequence / CTA counters
    std::vector<void*> peer_opened;             // other processes' peer blocks (cudaIpcOpenMemHandle)
    // pack / unpack phases per level
    struct LvPhases {
        Phase zero_gw, pack_c, add_c, pack_h, unpack_h, pack_r, add_r, diff_c;
        std::vector<Msg> m_corr, m_halo, m_rev;
    };
    std::vector<LvPhases> ph;
    // graphs
    GraphCache g_smooth, g_cycle;
    std::vector<double*> key_x;
    std::vector<const double*> key_b;
    int key_nu = -1, key_pre = -1, key_post = -1;
    double key_om = 0.0;
    int64_t last_launches = 0;
    double host_enqueue_s = 0.0, host_wait_s = 0.0;   // last mgd_solve: graph launches / waits for the norm
    int host_cycles = 0;
};

namespace rav {
namespace {

double now_s() {
    timespec t;
    clock_gettime(CLOCK_MONOTONIC, &t);
    return (double)t.tv_sec + 1e-9 * (double)t.tv_nsec;
}

rav_status upload_idx(const int32_t* h, int64_t n, int32_t** d, std::vector<void*>& allocs) {
    *d = nullptr;
    if (n <= 0) return RAV_OK;
    if (!h) { set_error("mgd_setup: NULL index list of length %lld", (long long)n); return RAV_ERR_ARG; }
    RAV_CUDA(cudaMalloc(d, sizeof(int32_t) * n));
    allocs.push_back(*d);
    RAV_CUDA(cudaMemcpy(*d, h, sizeof(int32_t) * n, cudaMemcpyHostToDevice));
    return RAV_OK;
}

rav_status alloc_buf(int64_t n, double** d, std::vector<void*>& allocs) {
    *d = nullptr;
    if (n <= 0) return RAV_OK;
    RAV_CUDA(cudaMalloc(d, sizeof(double) * n));
    allocs.push_back(*d);
    return RAV_OK;
}

bool unique_union(const std::vector<std::pair<const int32_t*, int64_t>>& lists) {
    std::vector<int32_t> all;
    for (auto& l : lists) all.insert(all.end(), l.first, l.first + l.second);
    std::sort(all.begin(), all.end());
    return std::adjacent_find(all.begin(), all.end()) == all.end();
}

rav_status phase_upload(Phase& P) {
    if (P.h.empty()) return RAV_OK;
    RAV_CUDA(cudaMalloc(&P.d, sizeof(Step) * P.h.size()));
    RAV_CUDA(cudaMemcpy(P.d, P.h.data(), sizeof(Step) * P.h.size(), cudaMemcpyHostToDevice));
    P.nmax = 0;
    for (auto& s : P.h) P.nmax = std::max(P.nmax, s.n);
    return RAV_OK;
}

rav_status run_phase(const Phase& P, const VecTab& vt, cudaStream_t s) {
    if (P.h.empty() || P.nmax == 0) return RAV_OK;
    dim3 grid((unsigned)std::max<int64_t>(1, std::min<int64_t>(cdiv(P.nmax, 256), 64)), (unsigned)P.h.size());
    phase_kernel<<<grid, 256, 0, s>>>(P.d, vt);
    count_launch();
    RAV_CHECK_LAUNCH();
    return RAV_OK;
}

rav_status run_msgs(const mgd_ctx* m, const std::vector<Msg>& msgs, cudaStream_t s) {
    if (msgs.empty()) return RAV_OK;
    const NcclApi& N = nccl();
    RAV_NCCL(N.GroupStart());
    for (const Msg& g : msgs) {
        if (g.send) RAV_NCCL(N.Send(g.buf, (size_t)g.n, ncclFloat64, g.peer_proc, m->comm->nc, s));
        else RAV_NCCL(N.Recv(g.buf, (size_t)g.n, ncclFloat64, g.peer_proc, m->comm->nc, s));
    }
    RAV_NCCL(N.GroupEnd());
    return RAV_OK;
}

// out[0 .. n) = sum over all subdomains of parts[s][0 .. n) (local parts [nl][stride]), ascending
// subdomain order: local partial sum, then (several processes) all-gather + ordered sum
rav_status ordered_allsum(const mgd_ctx* m, const double* parts, int64_t stride, int64_t n, double* loc,
                          double* all, double* out, cudaStream_t s) {
    const int blocks = (int)std::max<int64_t>(1, std::min<int64_t>(cdiv(n, 256), (int64_t)num_sms() * 4));
    const bool multi = m->comm->nprocs > 1 || m->via_comm;   // via_comm: the all-gather path on one rank too
    ordered_sum_kernel<<<blocks, 256, 0, s>>>(parts, m->nl, stride, n, multi ? loc : out);
    count_launch();
    RAV_CHECK_LAUNCH();
    if (!multi) return RAV_OK;
    RAV_NCCL(nccl().AllGather(loc, all, (size_t)n, ncclFloat64, m->comm->nc, s));
    ordered_sum_kernel<<<blocks, 256, 0, s>>>(all, m->comm->nprocs, n, n, out);
    count_launch();
    RAV_CHECK_LAUNCH();
    return RAV_OK;
}

VecTab vt_of(const std::vector<double*>& v) {
    VecTab t{};
    for (size_t i = 0; i < v.size() && i < (size_t)MAX_VEC; ++i) t.v[i] = v[i];
    return t;
}

// ---- the distributed sweep on partitioned level k (x[i], b[i]: local subdomain vectors) ----
// x_zero: every x[i] is zero on entry (the partitioned coarse levels: the correction starts from
// 0, ghosts included), so the first sweep's residual b - L 0 is b itself and is read from b (the
// window's b is complete: owners accumulated, ghosts refreshed), and there is nothing to zero
rav_status dist_sweeps(mgd_ctx* m, int k, const std::vector<double*>& x, const std::vector<const double*>& b, int nu,
                       double omega, bool x_zero = false) {
    cudaStream_t s = m->stream;
    auto& L = m->lv[k];
    auto& P = m->ph[k];
    const VecTab vx = vt_of(x);
    for (int it = 0; it < nu; ++it) {
        if (m->variant == RAV_VARIANT_MV) {   // per colour: old values, relax, changes -> owners, halo
            for (int64_t c = 0; c < m->ncolors[k]; ++c) {
                RAV_TRY(run_phase(P.pack_c, vx, s));
                for (int i = 0; i < m->nl; ++i) {
                    const auto& co = m->coffs[k][i];
                    RAV_TRY(launch_mv_color(L[i].sm->A, L[i].sm->F, co[c + 1] - co[c], m->plist[k][i] + co[c], b[i],
                                            x[i], omega, s));
                }
                RAV_TRY(run_phase(P.diff_c, vx, s));
                RAV_TRY(run_msgs(m, P.m_corr, s));
                RAV_TRY(run_phase(P.add_c, vx, s));
                RAV_TRY(run_phase(P.pack_h, vx, s));
                RAV_TRY(run_msgs(m, P.m_halo, s));
                RAV_TRY(run_phase(P.unpack_h, vx, s));
            }
            continue;
        }
        const bool from_b = x_zero && it == 0;
        if (!from_b) {
            for (int i = 0; i < m->nl; ++i) RAV_TRY(launch_residual(L[i].sm->A, x[i], b[i], L[i].sm->r, s));
            if (!m->fused) RAV_TRY(run_phase(P.zero_gw, vx, s));
        }
        for (int i = 0; i < m->nl; ++i) {
            const double* ri = from_b ? b[i] : L[i].sm->r;
            if (m->fused) RAV_TRY(launch_schur_sweep_ob(L[i].sm->P, L[i].sm->F, ri, x[i], omega, L[i].ob, s));
            else RAV_TRY(launch_sweep(L[i].sm->P, L[i].sm->F, ri, x[i], omega, s));
        }
        if (!m->fused) RAV_TRY(run_phase(P.pack_c, vx, s));
        RAV_TRY(run_msgs(m, P.m_corr, s));
        RAV_TRY(run_phase(P.add_c, vx, s));
        RAV_TRY(run_phase(P.pack_h, vx, s));
        RAV_TRY(run_msgs(m, P.m_halo, s));
        RAV_TRY(run_phase(P.unpack_h, vx, s));
    }
    return RAV_OK;
}

// owner values -> ghost copies of vector v on level k
rav_status dist_halo(mgd_ctx* m, int k, const std::vector<double*>& v) {
    const VecTab t = vt_of(v);
    RAV_TRY(run_phase(m->ph[k].pack_h, t, m->stream));
    RAV_TRY(run_msgs(m, m->ph[k].m_halo, m->stream));
    return run_phase(m->ph[k].unpack_h, t, m->stream);
}

// partial sums held at ghost copies of v -> added into the owners' entries (halo reversed)
rav_status dist_accumulate(mgd_ctx* m, int k, const std::vector<double*>& v) {
    const VecTab t = vt_of(v);
    RAV_TRY(run_phase(m->ph[k].pack_r, t, m->stream));
    RAV_TRY(run_msgs(m, m->ph[k].m_rev, m->stream));
    return run_phase(m->ph[k].add_r, t, m->stream);
}

rav_status coarse_cycle(mg_ctx* c, double* x, const double* b, int pre, int post, double omega) {
    if (c->L == 1) return launch_coarse_solve(c->C, b, x, c->stream);
    return vcycle_launches(c, c->L - 1, x, b, pre, post, omega, false, true);
}

// V-cycle from partitioned level k (dist.DistVCycle._cycle, in the library)
rav_status dist_cycle(mgd_ctx* m, int k, const std::vector<double*>& x, const std::vector<const double*>& b, int pre,
                      int post, double omega, bool x_zero = false) {
    cudaStream_t s = m->stream;
    auto& L = m->lv[k];
    RAV_TRY(dist_sweeps(m, k, x, b, pre, omega, x_zero));
    for (int i = 0; i < m->nl; ++i) RAV_TRY(launch_residual(L[i].sm->A, x[i], b[i], L[i].r, s));
    if (k + 1 < m->K) {
        auto& C = m->lv[k + 1];
        std::vector<double*> cb(m->nl), cx(m->nl);
        std::vector<const double*> cbc(m->nl);
        for (int i = 0; i < m->nl; ++i) {
            cb[i] = C[i].b;
            cx[i] = C[i].x;
            cbc[i] = C[i].b;
            if (L[i].xs.on && L[i].xs.dim == 2) RAV_TRY(launch_xs_restrict(L[i].xs, L[i].r, C[i].b, s));
            else RAV_TRY(launch_spmv(L[i].PT, L[i].r, C[i].b, 1.0, 0.0, s));   // b_c = P_own^T r (window partials)
        }
        RAV_TRY(dist_accumulate(m, k + 1, cb));
        RAV_TRY(dist_halo(m, k + 1, cb));
        for (int i = 0; i < m->nl; ++i) RAV_CUDA(cudaMemsetAsync(C[i].x, 0, sizeof(double) * C[i].n, s));
        RAV_TRY(dist_cycle(m, k + 1, cx, cbc, pre, post, omega, true));
        for (int i = 0; i < m->nl; ++i) {
            if (L[i].xs.on) RAV_TRY(launch_xs_prolong(L[i].xs, C[i].x, x[i], 1.0, 1.0, s));
            else RAV_TRY(launch_spmv(L[i].P, C[i].x, x[i], 1.0, 1.0, s));
        }
    } else {
        for (int i = 0; i < m->nl; ++i) {
            double* bp = m->bc_part + (size_t)i * m->nc;
            if (L[i].xs.on && L[i].xs.dim == 2) RAV_TRY(launch_xs_restrict(L[i].xs, L[i].r, bp, s));
            else RAV_TRY(launch_spmv(L[i].PT, L[i].r, bp, 1.0, 0.0, s));
        }
        RAV_TRY(ordered_allsum(m, m->bc_part, m->nc, m->nc, m->bc_loc, m->bc_all, m->bc, s));
        RAV_CUDA(cudaMemsetAsync(m->xc, 0, sizeof(double) * m->nc, s));
        RAV_TRY(coarse_cycle(m->coarse, m->xc, m->bc, pre, post, omega));
        for (int i = 0; i < m->nl; ++i) {
            if (L[i].xs.on) RAV_TRY(launch_xs_prolong(L[i].xs, m->xc, x[i], 1.0, 1.0, s));
            else RAV_TRY(launch_spmv(L[i].P, m->xc, x[i], 1.0, 1.0, s));
        }
    }
    RAV_TRY(dist_halo(m, k, x));
    return dist_sweeps(m, k, x, b, post, omega);
}

// ||b - L x||^2 over the owned DoFs of every subdomain -> m->nrm (device) -> m->h_nrm (pinned, async)
rav_status dist_norm(mgd_ctx* m, const std::vector<double*>& x, const std::vector<const double*>& b) {
    cudaStream_t s = m->stream;
    auto& L = m->lv[0];
    for (int i = 0; i < m->nl; ++i) {
        RAV_TRY(launch_residual(L[i].sm->A, x[i], b[i], L[i].r, s));
        for (int q = 0; q < 2; ++q) {
            const int64_t a = L[i].own[2 * q], e = L[i].own[2 * q + 1];
            RAV_TRY(launch_dot(L[i].r + a, L[i].r + a, std::max<int64_t>(0, e - a), m->dot_part, residual_norm_blocks(),
                               m->nrm_part + i, q, s));
        }
    }
    RAV_TRY(ordered_allsum(m, m->nrm_part, 1, 1, m->nrm_loc, m->nrm_all, m->nrm, s));
    RAV_CUDA(cudaMemcpyAsync(m->h_nrm, m->nrm, sizeof(double), cudaMemcpyDeviceToHost, s));
    return RAV_OK;
}

rav_status check_vectors(const mgd_ctx* m, double* const* x, const double* const* b, std::vector<double*>& X,
                         std::vector<const double*>& B) {
    if (!x || !b) { set_error("mgd: NULL vector array"); return RAV_ERR_ARG; }
    X.assign(x, x + m->nl);
    B.assign(b, b + m->nl);
    for (int i = 0; i < m->nl; ++i)
        if (!X[i] || !B[i] || !is_dev(X[i]) || !is_dev(B[i])) {
            set_error("mgd: x[%d] / b[%d] must be device pointers", i, i);
            return RAV_ERR_ARG;
        }
    return RAV_OK;
}

bool same_key(const mgd_ctx* m, const std::vector<double*>& X, const std::vector<const double*>& B) {
    if (m->key_x.size() != X.size()) return false;
    for (size_t i = 0; i < X.size(); ++i)
        if (m->key_x[i] != X[i] || m->key_b[i] != B[i]) return false;
    return true;
}

void set_key(mgd_ctx* m, const std::vector<double*>& X, const std::vector<const double*>& B) {
    m->key_x = X;
    m->key_b.assign(B.begin(), B.end());
}

}  // namespace
}  // namespace rav

extern "C" {

rav_status rav_comm_unique_id(unsigned char id[128]) {
    if (!id) { set_error("rav_comm_unique_id: NULL"); return RAV_ERR_ARG; }
    const NcclApi& N = nccl();
    if (!N.ok) { set_error("rav_comm_unique_id: %s", N.why); return RAV_ERR_COMM; }
    ncclUniqueId u;
    RAV_NCCL(N.GetUniqueId(&u));
    memcpy(id, u.internal, NCCL_UNIQUE_ID_BYTES);
    return RAV_OK;
}

rav_status rav_comm_create(int nprocs, int proc, const unsigned char* nccl_id, rav_comm** out) {
    if (!out || nprocs < 1 || proc < 0 || proc >= nprocs || (nprocs > 1 && !nccl_id)) {
        set_error("rav_comm_create: bad argument (nprocs > 1 needs an NCCL id)");
        return RAV_ERR_ARG;
    }
    *out = nullptr;
    rav_comm* c = new rav_comm();
    c->nprocs = nprocs;
    c->proc = proc;
    if (nccl_id) {
        const NcclApi& N = nccl();
        if (!N.ok) { set_error("rav_comm_create: %s", N.why); delete c; return RAV_ERR_COMM; }
        ncclUniqueId u;
        memcpy(u.internal, nccl_id, NCCL_UNIQUE_ID_BYTES);
        ncclResult_t r = N.CommInitRank(&c->nc, nprocs, u, proc);
        if (r != ncclSuccess) {
            set_error("rav_comm_create: ncclCommInitRank: %s", N.GetErrorString(r));
            delete c;
            return RAV_ERR_COMM;
        }
    }
    *out = c;
    return RAV_OK;
}

void rav_comm_destroy(rav_comm* c) {
    if (!c) return;
    if (c->nc) nccl().CommDestroy(c->nc);
    delete c;
}

void mgd_destroy(mgd_ctx* m) {
    if (!m) return;
    if (m->stream) cudaStreamSynchronize(m->stream);
    else cudaDeviceSynchronize();
    m->g_smooth.reset();
    m->g_cycle.reset();
    for (auto& L : m->lv)
        for (auto& S : L) {
            if (S.sm) rav_destroy(S.sm);
            csr_free(S.P);
            csr_free(S.PT);
            for (auto& nb : S.nb)
                for (void* p : nb.allocs) cudaFree(p);
            if (S.gw) cudaFree(S.gw);
            if (S.x) cudaFree(S.x);
            if (S.b) cudaFree(S.b);
            if (S.r) cudaFree(S.r);
        }
    for (auto& P : m->ph)
        for (Phase* q : {&P.zero_gw, &P.pack_c, &P.add_c, &P.pack_h, &P.unpack_h, &P.pack_r, &P.add_r, &P.diff_c})
            if (q->d) cudaFree(q->d);
    for (auto& L : m->plist)
        for (int32_t* p : L)
            if (p) cudaFree(p);
    for (double* p : {m->bc, m->xc, m->bc_part, m->bc_loc, m->bc_all, m->nrm_part, m->nrm_loc, m->nrm_all, m->nrm,
                      m->dot_part})
        if (p) cudaFree(p);
    if (m->h_nrm) cudaFreeHost(m->h_nrm);
    for (void* p : m->peer_opened) cudaIpcCloseMemHandle(p);
    for (auto& L : m->lv)
        for (auto& S : L) {
            if (S.rmap) cudaFree(S.rmap);
            if (S.pflag) cudaFree(S.pflag);
        }
    if (m->ob_block) cudaFree(m->ob_block);
    if (m->peer_block) cudaFree(m->peer_block);
    if (m->sync_block) cudaFree(m->sync_block);
    delete m;
}


// ---- peer-memory transport setup (via_comm = 2) --------------------------------------------
// One allocation per process holds the receive buffers, flags and ack words of all its message
// ends; it is exported with CUDA IPC and the other processes map it (cudaIpcOpenMemHandle:
// NVLink peer access between GPUs).  Each process publishes the offsets of its ends, keyed by
// (type, level, source, destination, role), together with its IPC handle in one NCCL all-gather at
// setup; subdomains of the same process use plain pointers.
static rav_status peer_setup(mgd_ctx* m) {
    struct Ent { int64_t t, k, src, dst, role, off_buf, off_flag, pad; };   // role 0 consumer end, 1 producer end
    struct Slot { int k, i, j, t, role; size_t ob, of; };
    std::vector<Ent> mine;
    std::vector<Slot> slots;
    size_t bytes = 0;
    auto take = [&](size_t b) {
        const size_t o = bytes;
        bytes += (b + 255) & ~(size_t)255;
        return o;
    };
    bool any_remote = false;
    for (int k = 0; k < m->K; ++k)
        for (int i = 0; i < m->nl; ++i) {
            DSub& S = m->lv[k][i];
            for (int j = 0; j < (int)S.nb.size(); ++j) {
                DNb& B = S.nb[j];
                any_remote = any_remote || B.peer_local < 0;
                for (int t = 0; t < 3; ++t) {
                    if (B.n_in(t)) {
                        const size_t ob = take(sizeof(double) * (size_t)B.n_in(t)), of = take(8);
                        slots.push_back({k, i, j, t, 0, ob, of});
                        mine.push_back({t, k, B.peer, S.gid, 0, (int64_t)ob, (int64_t)of, 0});
                    }
                    if (B.n_out(t)) {
                        const size_t of = take(8);
                        slots.push_back({k, i, j, t, 1, 0, of});
                        mine.push_back({t, k, S.gid, B.peer, 1, 0, (int64_t)of, 0});
                    }
                }
            }
        }
    RAV_CUDA(cudaMalloc(&m->peer_block, std::max<size_t>(bytes, 256)));
    RAV_CUDA(cudaMemset(m->peer_block, 0, std::max<size_t>(bytes, 256)));
    const size_t ns = std::max<size_t>(1, slots.size());
    RAV_CUDA(cudaMalloc(&m->sync_block, 16 * ns));
    RAV_CUDA(cudaMemset(m->sync_block, 0, 16 * ns));
    char* base = static_cast<char*>(m->peer_block);
    auto* seqs = static_cast<unsigned long long*>(m->sync_block);
    auto* dones = reinterpret_cast<unsigned int*>(seqs + ns);
    for (size_t q = 0; q < slots.size(); ++q) {
        const Slot& z = slots[q];
        DNb& B = m->lv[z.k][z.i].nb[z.j];
        if (z.role == 0) {
            B.in_buf(z.t) = reinterpret_cast<double*>(base + z.ob);
            B.my_flag[z.t] = reinterpret_cast<unsigned long long*>(base + z.of);
            B.seq_c[z.t] = seqs + q;
            B.done_c[z.t] = dones + q;
        } else {
            B.my_ack[z.t] = reinterpret_cast<unsigned long long*>(base + z.of);
            B.seq_p[z.t] = seqs + q;
            B.done_p[z.t] = dones + q;
        }
    }
    // the other ends: local subdomains directly
    for (int k = 0; k < m->K; ++k)
        for (int i = 0; i < m->nl; ++i) {
            DSub& S = m->lv[k][i];
            for (DNb& B : S.nb) {
                if (B.peer_local < 0) continue;
                DNb* R = nullptr;
                for (DNb& c : m->lv[k][B.peer_local].nb)
                    if (c.peer == S.gid) R = &c;
                if (!R) { set_error("mgd_setup: peer transport: no reverse neighbour"); return RAV_ERR_ARG; }
                for (int t = 0; t < 3; ++t) {
                    if (B.n_out(t)) { B.out_buf[t] = R->in_buf(t); B.out_sig[t] = R->my_flag[t]; }
                    if (B.n_in(t)) B.peer_ack[t] = R->my_ack[t];
                }
            }
        }
    if (any_remote) {   // other processes: IPC handles and offset tables through one NCCL all-gather
        if (!m->comm->nc) { set_error("mgd_setup: the peer transport between processes needs NCCL for setup"); return RAV_ERR_ARG; }
        const NcclApi& N = nccl();
        const int np = m->comm->nprocs;
        int64_t *dcnt = nullptr, *dtab = nullptr;
        RAV_CUDA(cudaMalloc(&dcnt, sizeof(int64_t) * (np + 1)));
        const int64_t cnt = (int64_t)mine.size();
        RAV_CUDA(cudaMemcpy(dcnt + np, &cnt, sizeof(int64_t), cudaMemcpyHostToDevice));
        RAV_NCCL(N.AllGather(dcnt + np, dcnt, 1, ncclInt64, m->comm->nc, m->stream));
        std::vector<int64_t> counts(np);
        RAV_CUDA(cudaMemcpyAsync(counts.data(), dcnt, sizeof(int64_t) * np, cudaMemcpyDeviceToHost, m->stream));
        RAV_CUDA(cudaStreamSynchronize(m->stream));
        const int64_t mx = *std::max_element(counts.begin(), counts.end());
        const int64_t row = 8 + 8 * mx;   // IPC handle (64 bytes) + entries
        std::vector<int64_t> h(row, 0);
        cudaIpcMemHandle_t hd;
        RAV_CUDA(cudaIpcGetMemHandle(&hd, m->peer_block));
        static_assert(sizeof(cudaIpcMemHandle_t) == 64, "IPC handle size");
        memcpy(h.data(), &hd, 64);
        if (cnt) memcpy(h.data() + 8, mine.data(), sizeof(Ent) * mine.size());
        RAV_CUDA(cudaMalloc(&dtab, sizeof(int64_t) * row * (np + 1)));
        RAV_CUDA(cudaMemcpy(dtab + row * np, h.data(), sizeof(int64_t) * row, cudaMemcpyHostToDevice));
        RAV_NCCL(N.AllGather(dtab + row * np, dtab, (size_t)row, ncclInt64, m->comm->nc, m->stream));
        std::vector<int64_t> all((size_t)row * np);
        RAV_CUDA(cudaMemcpyAsync(all.data(), dtab, sizeof(int64_t) * row * np, cudaMemcpyDeviceToHost, m->stream));
        RAV_CUDA(cudaStreamSynchronize(m->stream));
        cudaFree(dcnt);
        cudaFree(dtab);
        std::vector<char*> bases(np, nullptr);
        auto base_of = [&](int q) -> char* {
            if (!bases[q]) {
                cudaIpcMemHandle_t hq;
                memcpy(&hq, all.data() + (size_t)row * q, 64);
                void* p = nullptr;
                if (cudaIpcOpenMemHandle(&p, hq, cudaIpcMemLazyEnablePeerAccess) != cudaSuccess) {
                    cudaGetLastError();
                    return nullptr;
                }
                m->peer_opened.push_back(p);
                bases[q] = static_cast<char*>(p);
            }
            return bases[q];
        };
        auto find = [&](int q, int64_t t, int64_t k, int64_t src, int64_t dst, int64_t role) -> const Ent* {
            const Ent* e = reinterpret_cast<const Ent*>(all.data() + (size_t)row * q + 8);
            for (int64_t u = 0; u < counts[q]; ++u)
                if (e[u].t == t && e[u].k == k && e[u].src == src && e[u].dst == dst && e[u].role == role) return e + u;
            return nullptr;
        };
        for (int k = 0; k < m->K; ++k)
            for (int i = 0; i < m->nl; ++i) {
                DSub& S = m->lv[k][i];
                for (DNb& B : S.nb) {
                    if (B.peer_local >= 0) continue;
                    const int q = m->sub_proc[B.peer];
                    char* bq = base_of(q);
                    if (!bq) { set_error("mgd_setup: cudaIpcOpenMemHandle of process %d failed", q); return RAV_ERR_COMM; }
                    for (int t = 0; t < 3; ++t) {
                        if (B.n_out(t)) {
                            const Ent* e = find(q, t, k, S.gid, B.peer, 0);
                            if (!e) { set_error("mgd_setup: peer transport: message %d %d->%d has no receiver", t, S.gid, B.peer); return RAV_ERR_ARG; }
                            B.out_buf[t] = reinterpret_cast<double*>(bq + e->off_buf);
                            B.out_sig[t] = reinterpret_cast<unsigned long long*>(bq + e->off_flag);
                        }
                        if (B.n_in(t)) {
                            const Ent* e = find(q, t, k, B.peer, S.gid, 1);
                            if (!e) { set_error("mgd_setup: peer transport: message %d %d->%d has no sender", t, B.peer, S.gid); return RAV_ERR_ARG; }
                            B.peer_ack[t] = reinterpret_cast<unsigned long long*>(bq + e->off_flag);
                        }
                    }
                }
            }
    }
    return RAV_OK;
}

static rav_status peer_check() {   // a bounded wait of the peer transport timed out
    unsigned int h = 0;
    RAV_CUDA(cudaMemcpyFromSymbol(&h, g_peer_timeout, sizeof(h)));
    if (h) {
        set_error("mgd: a peer-transport wait timed out (a peer did not reach the same exchange)");
        return RAV_ERR_COMM;
    }
    return RAV_OK;
}

rav_status mgd_setup(rav_comm* comm, int n_sub_total, const int32_t* sub_proc, int n_local, const int32_t* local_ids,
                     int n_levels, const rav_subdomain* subs, mg_ctx* coarse, const rav_opts* opts, int via_comm,
                     mgd_ctx** out) {
    NvtxRange nvtx_range("mgd_setup");
    if (!comm || !out || n_sub_total < 1 || !sub_proc || n_local < 1 || n_local > MAX_VEC || !local_ids ||
        n_levels < 1 || !subs) {
        set_error("mgd_setup: bad argument");
        return RAV_ERR_ARG;
    }
    *out = nullptr;
    if ((comm->nprocs > 1 || via_comm == 1) && !comm->nc) {
        set_error("mgd_setup: exchanges between processes (or via_comm = 1) need a communicator with NCCL");
        return RAV_ERR_ARG;
    }
    if (via_comm == 2 && opts && opts->variant == RAV_VARIANT_MV) {
        set_error("mgd_setup: the peer-memory transport (via_comm = 2) covers RAV / AV / diagonal Vanka");
        return RAV_ERR_ARG;
    }
    rav_opts o{};
    if (opts) o = *opts;
    mgd_ctx* m = new mgd_ctx();
    m->comm = comm;
    m->nsub = n_sub_total;
    m->nl = n_local;
    m->K = n_levels;
    m->sub_proc.assign(sub_proc, sub_proc + n_sub_total);
    m->local_ids.assign(local_ids, local_ids + n_local);
    m->coarse = coarse;
    m->stream = as_stream(o.stream);
    m->variant = o.variant;
    m->via_comm = via_comm == 1;
    m->peer = via_comm == 2;
    m->fused = m->peer && o.variant != RAV_VARIANT_MV && o.variant != RAV_VARIANT_DIAG && !o.deterministic;
    rav_status st = RAV_OK;
    std::map<int32_t, int> local_of;
    for (int i = 0; i < n_local; ++i) {
        const int32_t g = local_ids[i];
        if (g < 0 || g >= n_sub_total || sub_proc[g] != comm->proc || (i > 0 && g <= local_ids[i - 1])) {
            set_error("mgd_setup: local_ids must be ascending subdomains of this process");
            mgd_destroy(m);
            return RAV_ERR_ARG;
        }
        local_of[g] = i;
    }
    m->lv.assign(n_levels, std::vector<DSub>(n_local));
    m->ph.resize(n_levels);
    m->ncolors.assign(n_levels, 0);
    m->plist.assign(n_levels, std::vector<int32_t*>(n_local, nullptr));
    m->coffs.assign(n_levels, std::vector<std::vector<int64_t>>(n_local));
    for (int k = 0; k < n_levels && st == RAV_OK; ++k) {
        for (int i = 0; i < n_local && st == RAV_OK; ++i) {
            const rav_subdomain& D = subs[(size_t)k * n_local + i];
            DSub& S = m->lv[k][i];
            S.gid = local_ids[i];
            rav_opts ol = o;
            ol.n_vel = D.n_vel;
            int64_t bp = -1;
            st = rav_setup(&D.A, &D.P, &ol, &S.sm, &bp);
            if (st != RAV_OK) break;
            S.n = D.A.n_rows;
            if (o.variant == RAV_VARIANT_MV) {
                if (D.n_colors < 1 || !D.color_offs || !D.color_ids) {
                    set_error("mgd_setup: RAV_VARIANT_MV needs the colouring of every subdomain");
                    st = RAV_ERR_ARG;
                    break;
                }
                if (i == 0) m->ncolors[k] = D.n_colors;
                else if (m->ncolors[k] != D.n_colors) {
                    set_error("mgd_setup: every subdomain of a level needs the same number of colours");
                    st = RAV_ERR_ARG;
                    break;
                }
                st = rav_set_colors(S.sm, D.n_colors, D.color_offs, D.color_ids);
                if (st != RAV_OK) break;
                m->coffs[k][i] = S.sm->coffs;
                m->plist[k][i] = S.sm->plist;
                S.sm->plist = nullptr;   // owned by the mgd context now
            }
            for (int q = 0; q < 2; ++q)
                if (D.owned[2 * q] < 0 || D.owned[2 * q + 1] < D.owned[2 * q] || D.owned[2 * q + 1] > S.n) {
                    set_error("mgd_setup: owned range %d of level %d subdomain %d outside [0, n]", q, k, S.gid);
                    st = RAV_ERR_ARG;
                }
            for (int q = 0; q < 4; ++q) S.own[q] = D.owned[q];
            if (st != RAV_OK) break;
            std::vector<void*> tmp;
            st = upload_idx(D.ghost_written, D.n_ghost_written, &S.gw, tmp);
            S.ngw = D.n_ghost_written;
            if (st != RAV_OK) break;
            S.nb.resize(D.n_neighbors);
            for (int j = 0; j < D.n_neighbors && st == RAV_OK; ++j) {
                const rav_neighbor& N = D.neighbors[j];
                DNb& B = S.nb[j];
                if (N.peer < 0 || N.peer >= n_sub_total || N.peer == S.gid) {
                    set_error("mgd_setup: bad neighbour id %d", N.peer);
                    st = RAV_ERR_ARG;
                    break;
                }
                B.peer = N.peer;
                auto it = local_of.find(N.peer);
                B.peer_local = it == local_of.end() ? -1 : it->second;
                B.remote = B.peer_local < 0 || m->via_comm || m->peer;
                B.ncs = N.n_corr_send; B.ncr = N.n_corr_recv; B.nhs = N.n_halo_send; B.nhr = N.n_halo_recv;
                if (st == RAV_OK) st = upload_idx(N.corr_send, B.ncs, &B.cs, B.allocs);
                if (st == RAV_OK) st = upload_idx(N.corr_recv, B.ncr, &B.cr, B.allocs);
                if (st == RAV_OK) st = upload_idx(N.halo_send, B.nhs, &B.hs, B.allocs);
                if (st == RAV_OK) st = upload_idx(N.halo_recv, B.nhr, &B.hr, B.allocs);
                if (st == RAV_OK) st = alloc_buf(B.ncs, &B.cs_buf, B.allocs);
                if (st == RAV_OK) st = alloc_buf(B.nhs, &B.hs_buf, B.allocs);
                if (st == RAV_OK) st = alloc_buf(B.nhr, &B.rs_buf, B.allocs);
                if (st == RAV_OK && B.remote && !m->peer) {   // peer transport: in the peer block
                    st = alloc_buf(B.ncr, &B.cr_in, B.allocs);
                    if (st == RAV_OK) st = alloc_buf(B.nhr, &B.hr_in, B.allocs);
                    if (st == RAV_OK) st = alloc_buf(B.nhs, &B.rr_in, B.allocs);
                }
            }
            if (st != RAV_OK) break;
            // duplicate targets of the additions: plain adds when the union is unique
            std::vector<std::pair<const int32_t*, int64_t>> lc, lr;
            for (int j = 0; j < D.n_neighbors; ++j) {
                lc.push_back({D.neighbors[j].corr_recv, D.neighbors[j].n_corr_recv});
                lr.push_back({D.neighbors[j].halo_send, D.neighbors[j].n_halo_send});
            }
            S.add_atomic_c = !unique_union(lc);
            S.add_atomic_r = !unique_union(lr);
            if (m->fused) {   // the ghost-written DoFs' slots in the consumers' receive buffers
                if (!schur_fusable(S.sm->P, S.sm->F) || S.nb.size() > 2) {
                    set_error("mgd_setup: level %d subdomain %d: the fused exchange needs the Schur sweep kernels "
                              "and at most two neighbours", k, S.gid);
                    st = RAV_ERR_ARG;
                    break;
                }
                std::vector<int32_t> rm((size_t)std::max<int64_t>(1, S.n), -1);
                int q = 0;
                for (int j = 0; j < D.n_neighbors; ++j) {
                    const rav_neighbor& N = D.neighbors[j];
                    if (N.n_corr_send <= 0) continue;
                    if (N.n_corr_send >= (1 << 24)) { set_error("mgd_setup: message too long for the fused exchange"); st = RAV_ERR_ARG; break; }
                    for (int64_t u = 0; u < N.n_corr_send; ++u) rm[N.corr_send[u]] = (q << 24) | (int32_t)u;
                    ++q;
                }
                if (st != RAV_OK) break;
                cudaError_t e = cudaMalloc(&S.rmap, sizeof(int32_t) * rm.size());
                if (e == cudaSuccess) e = cudaMemcpy(S.rmap, rm.data(), sizeof(int32_t) * rm.size(), cudaMemcpyHostToDevice);
                if (e == cudaSuccess) e = cudaDeviceSynchronize();   // the DMA of a pageable copy, before m->stream reads it
                if (e == cudaSuccess) e = cudaMalloc(&S.pflag, std::max<int64_t>(1, S.sm->P.n_patches));
                if (e != cudaSuccess) { set_error("mgd_setup: %s", cudaGetErrorString(e)); st = RAV_ERR_OOM; break; }
                const int64_t np = S.sm->P.n_patches;
                pflag_kernel<<<(int)std::max<int64_t>(1, std::min<int64_t>(cdiv(np, 256), 4096)), 256, 0, m->stream>>>(
                    np, S.sm->P.offs, S.sm->P.dofs, S.sm->P.w, S.rmap, S.pflag);
                count_launch();
                if (cudaGetLastError() != cudaSuccess) { set_error("mgd_setup: pflag kernel failed"); st = RAV_ERR_CUDA; break; }
                // writers per launch: chunks of 32 patches (thread layout) or patches (per-patch layout)
                std::vector<uint8_t> hf((size_t)std::max<int64_t>(1, np));
                // on the setup stream (may be non-blocking: a legacy-stream cudaMemcpy would not wait
                // for pflag_kernel and read uninitialised flags -- wrong writer counts, hung releases)
                if (cudaMemcpyAsync(hf.data(), S.pflag, (size_t)np, cudaMemcpyDeviceToHost, m->stream) != cudaSuccess ||
                    cudaStreamSynchronize(m->stream) != cudaSuccess) { st = RAV_ERR_CUDA; break; }
                unsigned int nw = 0;
                if (S.sm->F.layout == 4) {
                    const int64_t nch = (np + 31) / 32;
                    std::vector<uint8_t> cw((size_t)nch, 0);
                    for (int64_t c = 0; c < nch; ++c) {
                        for (int64_t u = c * 32; u < std::min<int64_t>(np, c * 32 + 32); ++u) cw[c] |= hf[u];
                        nw += cw[c];
                    }
                    // rotate the trailing run of writer chunks (the slab's last vertex layers) to the front
                    int64_t first = nch;
                    for (int64_t c = nch - 1; c >= 0 && (cw[c] || nch - c <= 64); --c)
                        if (cw[c]) first = c;
                    S.ob.rot = first < nch && first > nch / 2 ? nch - first : 0;
                } else {
                    for (int64_t u = 0; u < np; ++u) nw += hf[u] != 0;
                }
                S.ob.nflag = nw;
            }
            // transfer to the next level (levels < K-1: its windows; last: the agglomerated level)
            if (D.P_coarse.n_rows > 0) {
                if (D.P_coarse.n_rows != S.n) {
                    set_error("mgd_setup: P_coarse of level %d subdomain %d must have n rows", k, S.gid);
                    st = RAV_ERR_ARG;
                    break;
                }
                st = csr_upload(&D.P_coarse, S.P, m->stream);
                if (st == RAV_OK) st = csr_transpose(S.P, S.PT, m->stream);
                if (st == RAV_OK && D.grid_fine && D.grid_coarse) {   // stencil form, verified against P
                    XStruct X;
                    if (xs_build(D.grid_fine, D.grid_coarse, S.P.n_rows, S.P.n_cols, X) == RAV_OK &&
                        xs_verify(X, S.P, S.PT, m->stream) == RAV_OK)
                        S.xs = X;
                    set_error("");
                }
            } else if (k + 1 < n_levels || coarse) {
                set_error("mgd_setup: level %d subdomain %d needs P_coarse", k, S.gid);
                st = RAV_ERR_ARG;
            }
            if (st != RAV_OK) break;
            cudaError_t e = cudaMalloc(&S.r, sizeof(double) * std::max<int64_t>(1, S.n));
            if (e == cudaSuccess && k > 0) e = cudaMalloc(&S.x, sizeof(double) * std::max<int64_t>(1, S.n));
            if (e == cudaSuccess && k > 0) e = cudaMalloc(&S.b, sizeof(double) * std::max<int64_t>(1, S.n));
            if (e != cudaSuccess) { set_error("mgd_setup: %s", cudaGetErrorString(e)); st = RAV_ERR_OOM; }
        }
    }
    // match local neighbours (receive = the sender's packed buffer) and check message sizes
    for (int k = 0; k < n_levels && st == RAV_OK; ++k)
        for (int i = 0; i < n_local && st == RAV_OK; ++i)
            for (auto& B : m->lv[k][i].nb) {
                if (B.peer_local < 0) continue;
                DSub& Q = m->lv[k][B.peer_local];
                DNb* R = nullptr;
                for (auto& c : Q.nb)
                    if (c.peer == m->lv[k][i].gid) R = &c;
                if (!R || R->ncr != B.ncs || R->ncs != B.ncr || R->nhr != B.nhs || R->nhs != B.nhr) {
                    set_error("mgd_setup: level %d: the lists of subdomains %d and %d do not match", k,
                              m->lv[k][i].gid, B.peer);
                    st = RAV_ERR_ARG;
                    break;
                }
                if (!B.remote) {
                    B.cr_in = R->cs_buf;   // its corrections for me
                    B.hr_in = R->hs_buf;   // its owned values for my ghosts
                    B.rr_in = R->rs_buf;   // its ghost partials for my owned DoFs
                }
            }
    if (st == RAV_OK && m->peer) st = peer_setup(m);
    if (st == RAV_OK && m->fused) {   // outboxes: consumers = neighbours receiving corrections
        unsigned int* tmo = nullptr;
        if (cudaGetSymbolAddress(reinterpret_cast<void**>(&tmo), g_peer_timeout) != cudaSuccess) {
            set_error("mgd_setup: cudaGetSymbolAddress failed");
            st = RAV_ERR_CUDA;
        }
        const size_t nsub = (size_t)m->K * m->nl;
        if (st == RAV_OK && cudaMalloc(&m->ob_block, 16 * std::max<size_t>(1, nsub)) != cudaSuccess) st = RAV_ERR_OOM;
        if (st == RAV_OK && cudaMemset(m->ob_block, 0, 16 * std::max<size_t>(1, nsub)) != cudaSuccess) st = RAV_ERR_CUDA;
        auto* seqs = static_cast<unsigned long long*>(m->ob_block);
        auto* dones = reinterpret_cast<unsigned int*>(seqs + std::max<size_t>(1, nsub));
        for (int k = 0; k < m->K && st == RAV_OK; ++k)
            for (int i = 0; i < m->nl; ++i) {
                DSub& S = m->lv[k][i];
                Outbox& O = S.ob;
                O.rmap = S.rmap;
                O.pflag = S.pflag;
                O.nq = 0;
                for (DNb& B : S.nb) {
                    if (!B.ncs) continue;
                    O.buf[O.nq] = B.out_buf[0];
                    O.sig[O.nq] = B.out_sig[0];
                    O.ack[O.nq] = B.my_ack[0];
                    O.sys[O.nq] = B.peer_local < 0;
                    ++O.nq;
                }
                if (O.nq > 0 && O.nflag == 0) {
                    set_error("mgd_setup: level %d subdomain %d sends corrections but no patch writes a ghost DoF", k, S.gid);
                    st = RAV_ERR_ARG;
                }
                O.seq = seqs + (size_t)k * m->nl + i;
                O.done = dones + (size_t)k * m->nl + i;
                O.timeout = tmo;
            }
    }
    // phases and NCCL messages
    for (int k = 0; k < n_levels && st == RAV_OK; ++k) {
        auto& P = m->ph[k];
        std::map<std::tuple<int64_t, int64_t, int64_t>, Msg> mc, mh, mr;
        for (int i = 0; i < n_local; ++i) {
            DSub& S = m->lv[k][i];
            if (S.ngw) P.zero_gw.h.push_back({OP_ZERO, i, S.gw, S.ngw, nullptr});
            for (auto& B : S.nb) {
                const int pp = m->sub_proc[B.peer];
                if (m->peer) {   // producers write the consumers' buffers; no NCCL messages
                    auto prod = [&](int t) {
                        return Step{OP_GATHER, i, t == 0 ? B.cs : t == 1 ? B.hs : B.hr, B.n_out(t), B.out_buf[t],
                                    ROLE_PRODUCER, B.out_sig[t], B.my_ack[t], B.seq_p[t], B.done_p[t],
                                    B.peer_local < 0};
                    };
                    auto cons = [&](int t, int op) {
                        return Step{op, i, t == 0 ? B.cr : t == 1 ? B.hr : B.hs, B.n_in(t), B.in_buf(t),
                                    ROLE_CONSUMER, B.my_flag[t], B.peer_ack[t], B.seq_c[t], B.done_c[t],
                                    B.peer_local < 0};
                    };
                    if (B.ncs && !m->fused) P.pack_c.h.push_back(prod(0));   // fused: the sweep produces
                    if (B.ncr)
                        P.add_c.h.push_back(cons(0, m->fused ? (S.add_atomic_c ? OP_ADD_ATOMIC_CLEAR : OP_ADD_CLEAR)
                                                             : (S.add_atomic_c ? OP_ADD_ATOMIC : OP_ADD)));
                    if (B.nhs) P.pack_h.h.push_back(prod(1));
                    if (B.nhr) P.unpack_h.h.push_back(cons(1, OP_SCATTER));
                    if (B.nhr) P.pack_r.h.push_back(prod(2));
                    if (B.nhs) P.add_r.h.push_back(cons(2, S.add_atomic_r ? OP_ADD_ATOMIC : OP_ADD));
                    continue;
                }
                if (B.ncs) {
                    P.pack_c.h.push_back({OP_GATHER, i, B.cs, B.ncs, B.cs_buf});
                    P.diff_c.h.push_back({OP_DIFF, i, B.cs, B.ncs, B.cs_buf});
                }
                if (B.ncr) P.add_c.h.push_back({S.add_atomic_c ? OP_ADD_ATOMIC : OP_ADD, i, B.cr, B.ncr, B.cr_in});
                if (B.nhs) P.pack_h.h.push_back({OP_GATHER, i, B.hs, B.nhs, B.hs_buf});
                if (B.nhr) P.unpack_h.h.push_back({OP_SCATTER, i, B.hr, B.nhr, B.hr_in});
                if (B.nhr) P.pack_r.h.push_back({OP_GATHER, i, B.hr, B.nhr, B.rs_buf});
                if (B.nhs) P.add_r.h.push_back({S.add_atomic_r ? OP_ADD_ATOMIC : OP_ADD, i, B.hs, B.nhs, B.rr_in});
                if (!B.remote) continue;
                // ordering key (source subdomain, destination subdomain): equal at both ends
                if (B.ncs) mc[{0, S.gid, B.peer}] = Msg{S.gid, B.peer, 0, pp, B.cs_buf, B.ncs, true};
                if (B.ncr) mc[{1, B.peer, S.gid}] = Msg{B.peer, S.gid, 1, pp, B.cr_in, B.ncr, false};
                if (B.nhs) mh[{0, S.gid, B.peer}] = Msg{S.gid, B.peer, 0, pp, B.hs_buf, B.nhs, true};
                if (B.nhr) mh[{1, B.peer, S.gid}] = Msg{B.peer, S.gid, 1, pp, B.hr_in, B.nhr, false};
                if (B.nhr) mr[{0, S.gid, B.peer}] = Msg{S.gid, B.peer, 0, pp, B.rs_buf, B.nhr, true};
                if (B.nhs) mr[{1, B.peer, S.gid}] = Msg{B.peer, S.gid, 1, pp, B.rr_in, B.nhs, false};
            }
        }
        // sends in (source, destination) order, then receives in (source, destination) order: the
        // n-th send from process p to process q meets the n-th receive of q from p
        for (auto& kv : mc) P.m_corr.push_back(kv.second);
        for (auto& kv : mh) P.m_halo.push_back(kv.second);
        for (auto& kv : mr) P.m_rev.push_back(kv.second);
        for (Phase* q : {&P.zero_gw, &P.pack_c, &P.add_c, &P.pack_h, &P.unpack_h, &P.pack_r, &P.add_r, &P.diff_c})
            if (st == RAV_OK) st = phase_upload(*q);
    }
    // remote message sizes agree with the peers' lists (one exchange of the counts at setup)
    if (st == RAV_OK && comm->nc) {
        std::vector<std::vector<Msg>*> all;
        for (auto& P : m->ph) all.insert(all.end(), {&P.m_corr, &P.m_halo, &P.m_rev});
        std::vector<int64_t> counts;
        for (auto* v : all)
            for (auto& g : *v) counts.push_back(g.n);
        if (!counts.empty()) {
            int64_t* d = nullptr;
            RAV_CUDA(cudaMalloc(&d, sizeof(int64_t) * counts.size() * 2));
            RAV_CUDA(cudaMemcpy(d, counts.data(), sizeof(int64_t) * counts.size(), cudaMemcpyHostToDevice));
            const NcclApi& N = nccl();
            size_t q = 0;
            ncclResult_t r = N.GroupStart();
            for (auto* v : all)
                for (auto& g : *v) {
                    if (r == ncclSuccess)
                        r = g.send ? N.Send(d + q, 1, ncclInt64, g.peer_proc, comm->nc, m->stream)
                                   : N.Recv(d + counts.size() + q, 1, ncclInt64, g.peer_proc, comm->nc, m->stream);
                    ++q;
                }
            ncclResult_t r2 = N.GroupEnd();
            if (r == ncclSuccess) r = r2;
            std::vector<int64_t> got(counts.size());
            cudaMemcpyAsync(got.data(), d + counts.size(), sizeof(int64_t) * counts.size(), cudaMemcpyDeviceToHost,
                            m->stream);
            cudaStreamSynchronize(m->stream);
            cudaFree(d);
            if (r != ncclSuccess) {
                set_error("mgd_setup: size exchange: %s", N.GetErrorString(r));
                st = RAV_ERR_COMM;
            }
            q = 0;
            for (auto* v : all)
                for (auto& g : *v) {
                    if (st == RAV_OK && !g.send && got[q] != g.n) {
                        set_error("mgd_setup: a message from process %d has %lld entries, the receiver expects %lld",
                                  g.peer_proc, (long long)got[q], (long long)g.n);
                        st = RAV_ERR_ARG;
                    }
                    ++q;
                }
        }
    }
    // agglomerated level and norm buffers
    if (st == RAV_OK) {
        if (coarse) {
            m->nc = coarse->lv[coarse->L - 1].A.n_rows;
            for (int i = 0; i < n_local; ++i)
                if (m->lv[n_levels - 1][i].P.n_cols != m->nc) {
                    set_error("mgd_setup: the last partitioned level's P_coarse needs %lld columns", (long long)m->nc);
                    st = RAV_ERR_ARG;
                }
            if (st == RAV_OK) st = mg_set_stream(coarse, m->stream);
        }
        const int64_t nc = std::max<int64_t>(1, m->nc);
        const int np = comm->nprocs;
        cudaError_t e = cudaSuccess;
        for (auto pr : std::vector<std::pair<double**, int64_t>>{{&m->bc, nc}, {&m->xc, nc}, {&m->bc_part, nc * n_local},
                                                                 {&m->bc_loc, nc}, {&m->bc_all, nc * np},
                                                                 {&m->nrm_part, n_local}, {&m->nrm_loc, 1},
                                                                 {&m->nrm_all, np}, {&m->nrm, 1},
                                                                 {&m->dot_part, residual_norm_blocks()}})
            if (e == cudaSuccess) e = cudaMalloc(pr.first, sizeof(double) * pr.second);
        if (e == cudaSuccess) e = cudaMallocHost(&m->h_nrm, sizeof(double));
        if (e != cudaSuccess) { set_error("mgd_setup: %s", cudaGetErrorString(e)); st = RAV_ERR_OOM; }
    }
    if (st == RAV_OK) {
        for (auto& L : m->lv)
            for (auto& S : L) S.sm->stream = m->stream;
        // every setup upload (legacy-stream copies included) complete before m->stream uses them
        cudaError_t e = cudaDeviceSynchronize();
        if (e != cudaSuccess) { set_error("mgd_setup: %s", cudaGetErrorString(e)); st = RAV_ERR_CUDA; }
    }
    if (st != RAV_OK) {
        mgd_destroy(m);
        return st;
    }
    *out = m;
    return RAV_OK;
}

rav_status mgd_set_stream(mgd_ctx* m, void* stream) {
    if (!m) { set_error("NULL ctx"); return RAV_ERR_ARG; }
    if (m->stream != as_stream(stream)) {
        m->g_smooth.reset();
        m->g_cycle.reset();
    }
    m->stream = as_stream(stream);
    for (auto& L : m->lv)
        for (auto& S : L) S.sm->stream = m->stream;
    if (m->coarse) RAV_TRY(mg_set_stream(m->coarse, stream));
    return RAV_OK;
}

rav_status mgd_smooth(mgd_ctx* m, double* const* x, const double* const* b, int nu, double omega) {
    NvtxRange nvtx_range("mgd_smooth");
    if (!m || nu < 0) { set_error("mgd_smooth: bad argument"); return RAV_ERR_ARG; }
    std::vector<double*> X;
    std::vector<const double*> B;
    RAV_TRY(check_vectors(m, x, b, X, B));
    g_launches = 0;
    if (nu == 0) { m->last_launches = 0; return RAV_OK; }
    if (!m->g_smooth.exec || !same_key(m, X, B) || m->key_nu != nu || m->key_om != omega) {
        m->g_smooth.reset();
        m->g_cycle.reset();
        set_key(m, X, B);
        m->key_nu = nu;
        m->key_om = omega;
        m->key_pre = m->key_post = -1;
    }
    int64_t launches = 0;
    RAV_TRY(run_graph(m->g_smooth, m->stream, m->stream != nullptr, X[0], B[0], nu, 0, 0, omega, launches,
                      [&]() { return dist_sweeps(m, 0, X, B, nu, omega); }));
    m->last_launches = launches;
    return RAV_OK;
}

rav_status mgd_vcycle(mgd_ctx* m, double* const* x, const double* const* b, int pre, int post, double omega) {
    NvtxRange nvtx_range("mgd_vcycle");
    if (!m || pre < 0 || post < 0 || !m->coarse) { set_error("mgd_vcycle: bad argument (or no coarse hierarchy)"); return RAV_ERR_ARG; }
    std::vector<double*> X;
    std::vector<const double*> B;
    RAV_TRY(check_vectors(m, x, b, X, B));
    g_launches = 0;
    RAV_TRY(dist_cycle(m, 0, X, B, pre, post, omega));
    m->last_launches = g_launches;
    return RAV_OK;
}

rav_status mgd_residual_norm(mgd_ctx* m, double* const* x, const double* const* b, double* norm) {
    if (!m || !norm) { set_error("mgd_residual_norm: bad argument"); return RAV_ERR_ARG; }
    std::vector<double*> X;
    std::vector<const double*> B;
    RAV_TRY(check_vectors(m, x, b, X, B));
    g_launches = 0;
    RAV_TRY(dist_norm(m, X, B));
    RAV_CUDA(cudaStreamSynchronize(m->stream));
    *norm = sqrt(*m->h_nrm);
    m->last_launches = g_launches;
    return m->peer ? peer_check() : RAV_OK;
}

rav_status mgd_solve(mgd_ctx* m, double* const* x, const double* const* b, int pre, int post, double omega,
                     double rtol, int maxit, int* iters, double* hist) {
    NvtxRange nvtx_range("mgd_solve");
    if (!m || pre < 0 || post < 0 || maxit < 0 || !m->coarse) {
        set_error("mgd_solve: bad argument (or no coarse hierarchy)");
        return RAV_ERR_ARG;
    }
    std::vector<double*> X;
    std::vector<const double*> B;
    RAV_TRY(check_vectors(m, x, b, X, B));
    g_launches = 0;
    int64_t total = 0;
    RAV_TRY(dist_norm(m, X, B));
    RAV_CUDA(cudaStreamSynchronize(m->stream));
    total += g_launches;
    const double r0 = sqrt(*m->h_nrm);
    if (hist) hist[0] = r0;
    int k = 0;
    rav_status st = RAV_OK;
    if (!(r0 == r0) || isinf(r0)) { set_error("mgd_solve: initial residual is not finite"); st = RAV_ERR_DIVERGED; }
    if (!m->g_cycle.exec || !same_key(m, X, B) || m->key_pre != pre || m->key_post != post || m->key_om != omega) {
        m->g_cycle.reset();
        m->g_smooth.reset();
        set_key(m, X, B);
        m->key_pre = pre;
        m->key_post = post;
        m->key_om = omega;
        m->key_nu = -1;
    }
    m->host_enqueue_s = m->host_wait_s = 0.0;
    m->host_cycles = 0;
    while (st == RAV_OK && r0 > 0.0 && k < maxit) {
        int64_t launches = 0;
        const double t0 = now_s();
        st = run_graph(m->g_cycle, m->stream, m->stream != nullptr, X[0], B[0], pre, post, 1, omega, launches, [&]() {
            RAV_TRY(dist_cycle(m, 0, X, B, pre, post, omega));
            return dist_norm(m, X, B);
        });
        if (st != RAV_OK) break;
        total += launches;
        const double t1 = now_s();
        cudaError_t e = cudaStreamSynchronize(m->stream);
        m->host_enqueue_s += t1 - t0;
        m->host_wait_s += now_s() - t1;
        m->host_cycles++;
        if (e != cudaSuccess) { set_error("mgd_solve: %s", cudaGetErrorString(e)); st = RAV_ERR_CUDA; break; }
        const double rk = sqrt(*m->h_nrm);
        ++k;
        if (hist) hist[k] = rk;
        if (!(rk == rk) || isinf(rk)) { set_error("mgd_solve: residual is not finite at cycle %d", k); st = RAV_ERR_DIVERGED; break; }
        if (rk <= rtol * r0) break;
    }
    if (iters) *iters = k;
    m->last_launches = total;
    if (st == RAV_OK && m->peer) st = peer_check();
    return st;
}

int64_t mgd_last_launches(const mgd_ctx* m) { return m ? m->last_launches : 0; }

rav_status mgd_host_time(const mgd_ctx* m, double* enqueue_s, double* wait_s, int* cycles) {
    if (!m) { set_error("NULL ctx"); return RAV_ERR_ARG; }
    if (enqueue_s) *enqueue_s = m->host_enqueue_s;
    if (wait_s) *wait_s = m->host_wait_s;
    if (cycles) *cycles = m->host_cycles;
    return RAV_OK;
}

}  // extern "C"
