"""The slab-partitioned smoother and V-cycle INSIDE the library (mgd_*, csrc/dist.cu; SURVEY
section 8 rows a11 / b / e).  One GPU is available to the tests, so a multi-GPU run is emulated
by one process driving R subdomains on the same device: the exchanges between them are device
reads of the neighbour's packed buffers (no kernel waits on another).  With via_comm the same
exchanges go through a one-rank NCCL communicator's self sends / receives, i.e. the NCCL code
path of the multi-process run (ordering, sizes, graph capture of NCCL calls).  With via_comm = 2
the exchanges use the peer-memory transport: the pack kernels store into the consumer's receive
buffer and release its flag, the unpack kernels acquire it and release the producer's ack (local
subdomains: plain pointers; between processes the same kernels run on CUDA IPC mappings).
Results are gathered from the owned DoFs and compared with the single-domain oracle entry by
entry."""
import numpy as np
import pytest
import torch

import oracle
import seeded_inputs as si
from _parity import assert_entrywise, sweep_magnitude

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def rg():
    from paper_2103_10127_b200 import ravgmg
    return ravgmg


@pytest.fixture(scope="module")
def rdist():
    from paper_2103_10127_b200 import dist
    return dist


def _comm(rg, via_comm):
    return rg.Comm(1, 0, rg.Comm.unique_id() if via_comm == 1 else None)


def _gather(info, xs, n):
    out = np.full(n, np.nan)
    for s, x in zip(info["slabs"][0], xs):
        own = s.owned_mask()
        out[s.global_ids()[own]] = x.cpu().numpy()[own]
    assert not np.isnan(out).any()
    return out


def _scatter(info, v):
    return [torch.tensor(v[s.global_ids()], device="cuda") for s in info["slabs"][0]]


SMOOTH_CASES = [
    (si.problem(2, (48, 40), si.KIND_MMS, eta="fourier"), "pou", 0, 0.66, 4, False),
    (si.problem(2, (48, 40), si.KIND_MMS, eta="fourier"), "pou", 0, 0.66, 4, True),
    (si.problem(2, (33, 29), si.KIND_CAVITY, eta="fourier"), "own", 0, 0.66, 3, False),
    (si.problem(2, (36, 30), si.KIND_MMS, eta="fourier"), "full", 1, 0.1, 2, True),
    (si.problem(3, (5, 4, 12), si.KIND_CAVITY, eta="fourier"), "pou", 0, 0.66, 3, True),
    (si.problem(2, (48, 40), si.KIND_MMS, eta="fourier"), "pou", 0, 0.66, 4, 2),
    (si.problem(2, (36, 30), si.KIND_MMS, eta="fourier"), "full", 1, 0.1, 2, 2),
    (si.problem(3, (5, 4, 12), si.KIND_CAVITY, eta="fourier"), "pou", 0, 0.66, 3, 2),
]


@pytest.mark.parametrize("case", SMOOTH_CASES, ids=["2d-pou-4", "2d-pou-4-nccl", "2d-own-3", "2d-diag-2-nccl",
                                                    "3d-pou-3-nccl", "2d-pou-4-peer", "2d-diag-2-peer",
                                                    "3d-pou-3-peer"])
def test_mgd_sweeps_match_oracle(rg, rdist, case):
    prob, weights, variant, omega, R, via = case
    comm = _comm(rg, via)
    mgd, info = rdist.build_lib_dist(prob, 1, R, list(range(R)), [0] * R, comm, weights=weights, variant=variant,
                                     smooth_only=True, via_comm=via)
    O = oracle.assemble(prob)
    P = oracle.patches(prob, weights)
    fmt = oracle.FMT_DIAG if variant == 1 else oracle.FMT_ROWS
    F = oracle.factor(O, P, fmt)
    x0 = si.initial_guess(O["n"], seed=19)
    xs = _scatter(info, x0)
    nu = 4
    mgd.smooth(xs, info["b"], nu, omega)
    torch.cuda.synchronize()
    xd = _gather(info, xs, O["n"])
    xo = oracle.additive_sweeps(O, P, F, x0, O["b"], omega, nu)
    if fmt == oracle.FMT_ROWS:
        scale = sweep_magnitude(O, P, F, x0, O["b"], omega).max()
    else:
        scale = np.abs(x0).max() + np.abs(xo).max()
    assert_entrywise(xd, xo, scale, what=f"mgd {R} subdomains, {nu} sweeps")
    # ghosts are current: every copy of a DoF equals its owner's value
    for s, x in zip(info["slabs"][0], xs):
        assert_entrywise(x.cpu().numpy(), xd[s.global_ids()], scale, what="ghost copies")
    assert mgd.last_launches > 0


def test_mgd_multicolor_mv_matches_oracle(rg, rdist):
    prob = si.problem(2, (40, 36), si.KIND_MMS, eta="fourier")
    comm = _comm(rg, True)
    mgd, info = rdist.build_lib_dist(prob, 1, 3, [0, 1, 2], [0, 0, 0], comm, weights="full", variant=2,
                                     smooth_only=True, via_comm=True)
    O = oracle.assemble(prob)
    P = oracle.patches(prob, "full")
    F = oracle.factor(O, P, oracle.FMT_LU)
    x0 = si.initial_guess(O["n"], seed=29)
    xs = _scatter(info, x0)
    mgd.smooth(xs, info["b"], 2, 0.66)
    torch.cuda.synchronize()
    xd = _gather(info, xs, O["n"])
    xo = oracle.mv_sweeps(O, P, F, x0, O["b"], 0.66, 2, order=oracle.multicolor_order(prob))
    assert_entrywise(xd, xo, np.abs(x0).max() + np.abs(xo).max(), what="mgd multicoloured MV")


VC_CASES = [
    (si.problem(2, (64, 64), si.KIND_MMS, eta="fourier"), 5, 3, False, 1e-8, True),
    (si.problem(2, (64, 64), si.KIND_MMS, eta="fourier"), 5, 4, True, 1e-8, False),
    (si.problem(2, (32, 32), si.KIND_CAVITY, eta="fourier"), 4, 2, True, 1e-10, True),
    (si.problem(3, (8, 8, 16), si.KIND_CAVITY, eta="fourier"), 3, 3, True, 1e-8, False),
    (si.problem(2, (64, 64), si.KIND_MMS, eta="fourier"), 5, 3, 2, 1e-8, True),
    (si.problem(3, (8, 8, 16), si.KIND_CAVITY, eta="fourier"), 3, 3, 2, 1e-8, False),
    (si.problem(2, (64, 64), si.KIND_MMS, eta="fourier"), 5, 4, 2, 1e-8, False),
]


@pytest.mark.parametrize("case", VC_CASES, ids=["2d-mms-3-det", "2d-mms-4-nccl", "2d-cav-2-nccl-det", "3d-3-nccl",
                                                "2d-mms-3-peer-det", "3d-3-peer-fused", "2d-mms-4-peer-fused"])
def test_mgd_solve_matches_oracle(rg, rdist, case):
    prob, levels, R, via, rtol, det = case
    comm = _comm(rg, via)
    mgd, info = rdist.build_lib_dist(prob, levels, R, list(range(R)), [0] * R, comm, via_comm=via,
                                     deterministic=det)
    H = oracle.Hierarchy(prob, levels, "rav")
    xo, ko, ho = H.solve(rtol=rtol, omega=0.66, pre=2, post=2, maxit=100)
    xs, kg, hg = mgd.solve(info["x"], info["b"], pre=2, post=2, omega=0.66, rtol=rtol, maxit=100)
    assert kg == ko, (kg, ko, info["K"])
    np.testing.assert_allclose(hg, ho, rtol=1e-6, atol=1e-12 * ho[0])
    xd = _gather(info, xs, H.fine["n"])
    assert_entrywise(xd, xo, np.abs(xo).max(), tol=1e-9, what="mgd V-cycle iterate")
    # the captured cycle replays: to the same bits in deterministic mode (R16), else to rounding
    x1 = [x.clone() for x in xs]
    for x in info["x"]:
        x.zero_()
    mgd.solve(info["x"], info["b"], pre=2, post=2, omega=0.66, rtol=rtol, maxit=100)
    for a, b in zip(info["x"], x1):
        if det:
            assert torch.equal(a, b)
        else:
            assert float((a - b).abs().max()) <= 1e-12 * float(b.abs().max())
    assert mgd.last_launches > 0


def test_mgd_rejects_mismatched_lists(rg, rdist):
    prob = si.problem(2, (24, 24), si.KIND_MMS, eta="fourier")
    comm = _comm(rg, False)
    from paper_2103_10127_b200 import dist as d
    slabs = [d.Slab(prob, 2, r, d.partition_layers(25, 2)) for r in range(2)]
    levels = [rg.gen_level(s.local_problem(), "pou") for s in slabs]
    written = [d.written_local_from_patches(L) for L in levels]
    infos = [d.exchange_info(s, w) for s, w in zip(slabs, written)]
    subs = []
    for s, L, w in zip(slabs, levels, written):
        lists = d._exchange_lists(s, w, infos)
        e = np.zeros(0, np.int64)
        peers = set(lists["corr_send"]) | set(lists["halo_recv"]) | set(lists["halo_send"]) | set(lists["corr_recv"])
        nb = {q: (lists["corr_send"].get(q, e), lists["corr_recv"].get(q, e), lists["halo_send"].get(q, e),
                  lists["halo_recv"].get(q, e)) for q in peers}
        subs.append({"level": L, "neighbors": nb, "ghost_written": lists["ghost_written"],
                     "owned": s.owned_ranges(), "prol": None, "colors": None})
    cs, cr, hs, hr = subs[1]["neighbors"][0]
    subs[1]["neighbors"][0] = (cs, cr[:-1], hs, hr)        # one entry short
    with pytest.raises(rg.RavError) as ei:
        rg.DistMultigrid(comm, [0, 0], [0, 1], [subs])
    assert ei.value.status == 1


def test_mgd_peer_transport_equals_local_exchange(rg, rdist):
    """The peer-memory transport moves the same values in the same order as the local exchange:
    after 3 x 2 sweeps (graph-captured; flags and sequence numbers advance on every replay) the
    iterates are bitwise equal (deterministic mode), and the transport's bounded waits never
    timed out (mgd_residual_norm reports a timeout as an error)."""
    prob = si.problem(2, (40, 48), si.KIND_MMS, eta="fourier")
    n = oracle.assemble(prob)["n"]
    out = []
    for via in (0, 2):
        comm = _comm(rg, via)
        mgd, info = rdist.build_lib_dist(prob, 1, 3, [0, 1, 2], [0, 0, 0], comm, smooth_only=True, via_comm=via,
                                         deterministic=True)
        xs = _scatter(info, si.initial_guess(n, seed=5))
        for _ in range(3):
            mgd.smooth(xs, info["b"], 2, 0.66)
        torch.cuda.synchronize()
        out.append([x.clone() for x in xs])
        assert np.isfinite(mgd.residual_norm(xs, info["b"]))
        mgd.close()
    for a, b in zip(*out):
        assert torch.equal(a, b)


def test_mgd_peer_transport_rejects_mv(rg, rdist):
    prob = si.problem(2, (24, 24), si.KIND_MMS, eta="fourier")
    with pytest.raises(rg.RavError):
        rdist.build_lib_dist(prob, 1, 2, [0, 1], [0, 0], _comm(rg, 0), weights="full", variant=2, smooth_only=True,
                             via_comm=2)


def test_mgd_fused_exchange_matches_local_exchange(rg, rdist):
    """The interface exchange fused into the sweep (peer transport, non-deterministic mode: the
    sweep's scatter adds ghost-written corrections into the owners' receive buffers) gives the
    local exchange's iterate to rounding (the same additions, atomics in another order), through
    graph replays of 3 x 2 sweeps, 2D thread kernel and 3D warp kernel."""
    for prob in (si.problem(2, (40, 48), si.KIND_MMS, eta="fourier"), si.problem(3, (6, 6, 14), si.KIND_CAVITY,
                                                                                   eta="fourier")):
        n = oracle.assemble(prob)["n"]
        out = []
        for via in (0, 2):
            mgd, info = rdist.build_lib_dist(prob, 1, 3, [0, 1, 2], [0, 0, 0], _comm(rg, via), smooth_only=True,
                                             via_comm=via)
            xs = _scatter(info, si.initial_guess(n, seed=7))
            for _ in range(3):
                mgd.smooth(xs, info["b"], 2, 0.66)
            torch.cuda.synchronize()
            out.append(_gather(info, xs, n))
            assert np.isfinite(mgd.residual_norm(xs, info["b"]))
            mgd.close()
        assert_entrywise(out[1], out[0], np.abs(out[0]).max(), tol=1e-13, what="fused vs local exchange")


def test_mgd_fused_exchange_nonblocking_stream(rg, rdist):
    """The fused exchange set up and run on a non-blocking stream (the bench's and the scaling
    model's setting), 2 and 4 subdomains of a slab-stacked 2D grid large enough for the thread
    kernel: the per-patch writer flags must be read after the kernel that computes them (a legacy-
    stream copy raced it and miscounted the writers: hung releases / a setup error).  Fused
    iterate = local exchange's to rounding; a bounded wait that expired would raise."""
    prob = si.problem(2, (96, 192), si.KIND_MMS, eta="fourier")   # >= 4096 patches per subdomain
    n = oracle.assemble(prob)["n"]
    stream = torch.cuda.Stream()
    for N in (2, 4):
        out = []
        for via in (0, 2):
            mgd, info = rdist.build_lib_dist(prob, 1, N, list(range(N)), [0] * N, _comm(rg, via), smooth_only=True,
                                             via_comm=via, stream=stream)
            xs = _scatter(info, si.initial_guess(n, seed=11))
            torch.cuda.synchronize()
            with torch.cuda.stream(stream):
                for _ in range(3):
                    mgd.smooth(xs, info["b"], 2, 0.66)
            torch.cuda.synchronize()
            out.append(_gather(info, xs, n))
            mgd.close()
        assert_entrywise(out[1], out[0], np.abs(out[0]).max(), tol=1e-13, what=f"fused vs local, {N} subdomains")
