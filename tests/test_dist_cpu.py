"""Multi-rank host logic of the slab-partitioned RAV sweep (SURVEY section 8 row
e) on CPU: world_size 2 and 3 over gloo (127.0.0.1), the exchange protocol of
paper_2103_10127_b200/dist.py driven by a numpy backend whose local operators,
patches and factor rows are cut out of the ORACLE's global system.  The
distributed sweeps must reproduce the single-domain oracle sweeps (P:124
Eq. 13; the additive corrections are order independent up to rounding, R16).

This covers the partition, ownership, window sizes (every local row's columns
stay inside its window), the index lists and the message schedule; the GPU
kernels behind the same protocol are covered by tests/test_gpu_dist.py."""
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

import oracle
import seeded_inputs as si
from paper_2103_10127_b200 import dist as rdist


class NumpyBackend:
    """Local compute with the oracle's global system restricted to a slab."""

    def __init__(self, slab, O, P, F, weights_global):
        gids = slab.global_ids()
        g2l = -np.ones(O["n"], np.int64)
        g2l[gids] = np.arange(len(gids))
        w = slab.window
        is_vel, layer = slab.layer_of_global(gids)
        in_rows = np.where(is_vel, (layer >= w["rnode_lo"]) & (layer <= w["rnode_hi"]),
                           (layer >= w["rvert_lo"]) & (layer <= w["rvert_hi"]))
        rp = [0]
        ci, val = [], []
        for l, g in enumerate(gids):
            if in_rows[l]:
                s, e = O["rp"][g], O["rp"][g + 1]
                cols = g2l[O["ci"][s:e]]
                assert np.all(cols >= 0), "row couples outside the window"
                ci.append(cols)
                val.append(O["val"][s:e])
            rp.append(rp[-1] + (len(ci[-1]) if in_rows[l] else 0))
        self.rp = np.array(rp)
        self.ci = np.concatenate(ci) if ci else np.zeros(0, np.int64)
        self.val = np.concatenate(val) if val else np.zeros(0)
        self.b = np.where(in_rows, O["b"][gids], 0.0)
        # own patches = vertices of layers [V0, V1)
        p0, p1 = slab.nlow_vert * slab.V0, slab.nlow_vert * slab.V1
        self.patches = []
        for i in range(p0, p1):
            d = P["dofs"][P["offs"][i]:P["offs"][i + 1]]
            wt = P["w"][P["offs"][i]:P["offs"][i + 1]]
            ld = g2l[d]
            assert np.all(ld >= 0), "patch outside the window"
            k = int((wt > 0).sum())
            rows = F["fac"][F["foffs"][i]:F["foffs"][i + 1]].reshape(k, len(d))
            self.patches.append((ld, k, rows))
        self.written = np.unique(np.concatenate([ld[:k] for ld, k, _ in self.patches]))

    def residual(self, x, b, r):
        xv, rv, bv = x.numpy(), r.numpy(), b.numpy()
        for i in range(len(self.rp) - 1):
            s, e = self.rp[i], self.rp[i + 1]
            rv[i] = bv[i] - np.dot(self.val[s:e], xv[self.ci[s:e]])

    def apply(self, r, x, omega):
        rv, xv = r.numpy(), x.numpy()
        delta = np.zeros_like(xv)
        for ld, k, rows in self.patches:
            c = rows @ rv[ld]
            np.add.at(delta, ld[:k], c)
        xv += omega * delta

    def gather(self, src, idx, out):
        out.numpy()[:] = src.numpy()[idx]

    def scatter(self, src, idx, dst):
        dst.numpy()[idx] = src.numpy()

    def scatter_add(self, src, idx, dst):
        dst.numpy()[idx] += src.numpy()

    def fill(self, dst, idx, value):
        dst.numpy()[idx] = value

    def index(self, a):
        return np.asarray(a, dtype=np.int64)

    def buffer(self, n):
        return torch.zeros(int(n), dtype=torch.float64)


def _worker(rank, world, port, prob, weights, nu, out_q):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        O = oracle.assemble(prob)
        P = oracle.patches(prob, weights)
        F = oracle.factor(O, P, oracle.FMT_ROWS)
        slab = rdist.Slab(prob, world, rank)
        be = NumpyBackend(slab, O, P, F, weights)
        sw = rdist.DistSweeper(slab, be, rdist.TorchComm(), be.written)
        x0 = si.initial_guess(O["n"], seed=17)
        gids = slab.global_ids()
        x = torch.tensor(x0[gids])
        b = torch.tensor(be.b)
        sw.smooth(x, b, nu, 0.66)
        own = slab.owned_mask()
        out_q.put((rank, gids[own], x.numpy()[own].copy(), slab.n_loc, len(be.patches)))
    finally:
        dist.destroy_process_group()


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


CASES = [
    (si.problem(2, (12, 15), si.KIND_MMS, eta="fourier"), "pou", 2),
    (si.problem(2, (10, 17), si.KIND_CAVITY, eta="fourier"), "own", 3),
    (si.problem(2, (9, 11), si.KIND_MMS, eta="fourier"), "full", 2),
    (si.problem(3, (3, 4, 9), si.KIND_CAVITY, eta="fourier"), "pou", 3),
]


@pytest.mark.parametrize("case", CASES, ids=["2d-pou-w2", "2d-own-w3", "2d-av-w2", "3d-pou-w3"])
def test_distributed_sweeps_match_single_domain_oracle(case):
    prob, weights, world = case
    nu = 3
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, prob, weights, nu, q)) for r in range(world)]
    for p in procs:
        p.start()
    res = [q.get(timeout=300) for _ in range(world)]
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    O = oracle.assemble(prob)
    P = oracle.patches(prob, weights)
    F = oracle.factor(O, P, oracle.FMT_ROWS)
    x0 = si.initial_guess(O["n"], seed=17)
    xo = oracle.additive_sweeps(O, P, F, x0, O["b"], 0.66, nu)
    xd = np.full(O["n"], np.nan)
    npatch = 0
    for _, g, v, _, npl in res:
        assert np.all(np.isnan(xd[g])), "a DoF has two owners"
        xd[g] = v
        npatch += npl
    assert not np.isnan(xd).any(), "a DoF has no owner"
    assert npatch == len(P["offs"]) - 1
    assert np.linalg.norm(xd - xo) <= 1e-13 * np.linalg.norm(xo)


def test_partition_and_windows():
    prob = si.problem(2, (16, 40), si.KIND_MMS)
    for world in (1, 2, 4, 8):
        lay = rdist.partition_layers(41, world)
        assert lay[0][0] == 0 and lay[-1][1] == 41
        assert all(b - a >= 3 for a, b in lay)
        assert max(b - a for a, b in lay) - min(b - a for a, b in lay) <= 1
        owned = 0
        for r in range(world):
            s = rdist.Slab(prob, world, r)
            owned += int(s.owned_mask().sum())
            w = s.window
            assert w["node_lo"] <= w["rnode_lo"] and w["rnode_hi"] <= w["node_hi"]
        nglob = 2 * 31 * 79 + 17 * 41
        assert owned == nglob
    with pytest.raises(ValueError):
        rdist.partition_layers(10, 4)


# ---------------------------------------------------------------------------------------------
# distributed V-cycle (SURVEY section 8 rows a9 / e): slab-partitioned levels with
# windowed transfers, agglomerated coarse levels, all-reduced coarse rhs and residual norms
# ---------------------------------------------------------------------------------------------

def window_prolongation(Pg, fine_slab, coarse_slab=None):
    """Rows = the fine slab's OWNED local DoFs (others empty); columns = the coarse
    slab's local DoFs (global ids when coarse_slab is None), cut from the oracle's
    global P."""
    fg = fine_slab.global_ids()
    own = fine_slab.owned_mask()
    if coarse_slab is not None:
        c2l = -np.ones(Pg["nc"], np.int64)
        c2l[coarse_slab.global_ids()] = np.arange(coarse_slab.n_loc)
        nc = coarse_slab.n_loc
    else:
        c2l = np.arange(Pg["nc"])
        nc = Pg["nc"]
    rows, cols, vals = [], [], []
    for l, g in enumerate(fg):
        if not own[l]:
            continue
        s, e = Pg["rp"][g], Pg["rp"][g + 1]
        c = c2l[Pg["ci"][s:e]]
        assert np.all(c >= 0), "owned fine row interpolates from outside the coarse window"
        rows += [l] * (e - s)
        cols += list(c)
        vals += list(Pg["val"][s:e])
    import scipy.sparse as sp
    return sp.csr_matrix((vals, (rows, cols)), shape=(fine_slab.n_loc, nc))


class NumpyCycleBackend(NumpyBackend):
    def __init__(self, slab, O, P, F, coarse=None):
        super().__init__(slab, O, P, F, None)
        self.coarse = coarse

    def restrict(self, T, r, bc):
        bc.numpy()[:] = T.T @ r.numpy()

    def prolong(self, T, xc, x):
        x.numpy()[:] += T @ xc.numpy()

    def zero(self, v):
        v.zero_()

    def dot_owned(self, r, ranges):
        rv = r.numpy()
        return torch.tensor([sum(float(np.dot(rv[a:b], rv[a:b])) for a, b in ranges)], dtype=torch.float64)

    def coarse_vcycle(self, xc, bc, pre, post, omega):
        xc.numpy()[:] = self.coarse.vcycle(np.zeros(len(bc)), bc.numpy(), pre, post, omega)


def build_dist_cycle(prob, n_levels, world, rank, comm, agg_layers=0):
    probs, parts = rdist.plan_levels(prob, n_levels, world, agg_layers=agg_layers)
    K = len(parts)
    coarse = oracle.Hierarchy(probs[K], n_levels - K)
    slabs = [rdist.Slab(probs[k], world, rank, parts[k]) for k in range(K)]
    levels, xfers = [], []
    for k in range(K):
        O = oracle.assemble(probs[k])
        P = oracle.patches(probs[k], "pou")
        F = oracle.factor(O, P, oracle.FMT_ROWS)
        be = NumpyCycleBackend(slabs[k], O, P, F, coarse if k == K - 1 else None)
        sw = rdist.DistSweeper(slabs[k], be, comm, be.written)
        n = slabs[k].n_loc
        levels.append({"slab": slabs[k], "be": be, "sweeper": sw,
                       "b": torch.tensor(be.b) if k == 0 else torch.zeros(n, dtype=torch.float64),
                       "x": torch.zeros(n, dtype=torch.float64)})
        if k + 1 < K:
            xfers.append(window_prolongation(oracle.prolongation(probs[k], probs[k + 1]), slabs[k], slabs[k + 1]))
    agg = window_prolongation(oracle.prolongation(probs[K - 1], probs[K]), slabs[K - 1], None)
    cyc = rdist.DistVCycle(levels, xfers, agg, comm, coarse.fine["n"])
    return cyc, levels, K


def _cycle_worker(rank, world, port, prob, n_levels, agg_layers, out_q):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        cyc, levels, K = build_dist_cycle(prob, n_levels, world, rank, rdist.TorchComm(), agg_layers)
        slab = levels[0]["slab"]
        x = torch.zeros(slab.n_loc, dtype=torch.float64)
        _, k, hist = cyc.solve(x, levels[0]["b"], rtol=1e-10, omega=0.66, maxit=60)
        own = slab.owned_mask()
        out_q.put((rank, slab.global_ids()[own], x.numpy()[own].copy(), k, hist, K))
    finally:
        dist.destroy_process_group()


CYCLE_CASES = [
    (si.problem(2, (16, 24), si.KIND_MMS, eta="fourier"), 4, 2, 0),
    (si.problem(2, (24, 24), si.KIND_CAVITY, eta="fourier"), 4, 3, 0),
    (si.problem(2, (16, 32), si.KIND_MMS, eta="fourier", box=[1.0, 2.0]), 4, 2, 8),
    (si.problem(3, (4, 4, 8), si.KIND_CAVITY, eta="fourier", box=[1.0, 1.0, 2.0]), 2, 2, 0),
]


@pytest.mark.parametrize("case", CYCLE_CASES, ids=["2d-mms-w2", "2d-cavity-w3", "2d-agg8-w2", "3d-cavity-w2"])
def test_distributed_vcycle_matches_single_domain_oracle(case):
    prob, n_levels, world, agg = case
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_cycle_worker, args=(r, world, port, prob, n_levels, agg, q)) for r in range(world)]
    for p in procs:
        p.start()
    res = [q.get(timeout=600) for _ in range(world)]
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    H = oracle.Hierarchy(prob, n_levels)
    xo, ko, ho = H.solve(rtol=1e-10, omega=0.66, maxit=60)
    assert ko < 60, "the reference solve must converge"
    xd = np.full(H.fine["n"], np.nan)
    for _, g, v, k, hist, K in res:
        assert k == ko, f"distributed cycles {k} != oracle {ko}"
        assert K >= 1
        np.testing.assert_allclose(hist, ho, rtol=1e-9, atol=1e-13 * ho[0])   # rounding floor ~ eps ||b||
        xd[g] = v
    assert not np.isnan(xd).any()
    assert np.linalg.norm(xd - xo) <= 1e-10 * np.linalg.norm(xo)


def test_level_plan_nesting():
    prob = si.problem(2, (64, 256), si.KIND_MMS)
    probs, parts = rdist.plan_levels(prob, 7, 4)
    assert [p["ncell"][1] for p in probs] == [256, 128, 64, 32, 16, 8, 4]
    for k, part in enumerate(parts):
        n = probs[k]["ncell"][1]
        assert part[0][0] == 0 and part[-1][1] == n + 1
        assert all(b - a >= 3 for a, b in part)
        assert all(part[r][1] == part[r + 1][0] for r in range(3))
    assert len(parts) == 5      # 257, 129, 65, 33, 17 layers over 4 ranks; 9 layers -> < 3 per rank
    _, parts8 = rdist.plan_levels(prob, 7, 4, agg_layers=8)
    assert len(parts8) == 4


# ---------------------------------------------------------------------------------------------
# comparison smoothers across ranks: multicoloured MV with
# per-colour interface exchanges, additive diagonal Vanka through the additive protocol
# ---------------------------------------------------------------------------------------------

class NumpySmootherBackend(NumpyBackend):
    """Local MV colours / diagonal-Vanka corrections from dense local systems of the
    slab's local rows (plain numpy, written from Eqs. 11 / 12 and R17)."""

    def __init__(self, slab, O, P, F, mode):
        super().__init__(slab, O, P, F, None)
        import scipy.sparse as sp
        self.mode = mode
        self.colors = rdist.local_colors(slab)
        n = len(self.rp) - 1
        self.Lloc = sp.csr_matrix((self.val, self.ci, self.rp), shape=(n, n))
        is_vel = np.arange(n) < slab.nvel_loc
        self.inv = []
        for ld, _, _ in self.patches:
            Li = self.Lloc[ld][:, ld].toarray()          # L_i = R_i L R_i^T
            if mode == "diag":                           # R17: velocity block -> its diagonal
                v = is_vel[ld]
                Li[np.ix_(v, v)] = np.diag(np.diag(Li)[v])
            self.inv.append(np.linalg.inv(Li))

    def apply_color(self, c, x, b, omega):
        offs, ids = self.colors
        xv, bv = x.numpy(), b.numpy()
        for p in ids[offs[c]:offs[c + 1]]:
            ld = self.patches[p][0]
            r = bv[ld] - self.Lloc[ld] @ xv             # fresh local residual (Eq. 15)
            xv[ld] += omega * (self.inv[p] @ r)

    def gather_diff(self, src, idx, buf):
        buf.numpy()[:] = src.numpy()[idx] - buf.numpy()

    def apply(self, r, x, omega):       # additive diagonal Vanka, full prolongation (Eq. 12 with R17)
        rv, xv = r.numpy(), x.numpy()
        delta = np.zeros_like(xv)
        for (ld, _, _), Mi in zip(self.patches, self.inv):
            delta[ld] += Mi @ rv[ld]
        xv += omega * delta


def _smoother_worker(rank, world, port, prob, mode, nu, out_q):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        O = oracle.assemble(prob)
        P = oracle.patches(prob, "full")
        F = oracle.factor(O, P, oracle.FMT_ROWS)
        slab = rdist.Slab(prob, world, rank)
        be = NumpySmootherBackend(slab, O, P, F, mode)
        comm = rdist.TorchComm()
        if mode == "mv":
            sw = rdist.DistMVSweeper(slab, be, comm, be.written, len(be.colors[0]) - 1)
        else:
            sw = rdist.DistSweeper(slab, be, comm, be.written)
        x0 = si.initial_guess(O["n"], seed=23)
        gids = slab.global_ids()
        x = torch.tensor(x0[gids])
        b = torch.tensor(be.b)
        sw.smooth(x, b, nu, 0.66 if mode == "mv" else 0.1)
        own = slab.owned_mask()
        out_q.put((rank, gids[own], x.numpy()[own].copy()))
    finally:
        dist.destroy_process_group()


SMOOTHER_CASES = [
    (si.problem(2, (10, 14), si.KIND_MMS, eta="fourier"), "mv", 2),
    (si.problem(2, (9, 17), si.KIND_CAVITY, eta="fourier"), "mv", 3),
    (si.problem(2, (8, 12), si.KIND_MMS, eta="fourier"), "diag", 2),
    (si.problem(3, (3, 3, 8), si.KIND_CAVITY, eta="fourier"), "mv", 2),
]


@pytest.mark.parametrize("case", SMOOTHER_CASES, ids=["mv-w2", "mv-w3", "diag-w2", "mv-3d-w2"])
def test_distributed_comparison_smoothers_match_oracle(case):
    prob, mode, world = case
    nu = 2
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_smoother_worker, args=(r, world, port, prob, mode, nu, q)) for r in range(world)]
    for p in procs:
        p.start()
    res = [q.get(timeout=600) for _ in range(world)]
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    O = oracle.assemble(prob)
    P = oracle.patches(prob, "full")
    x0 = si.initial_guess(O["n"], seed=23)
    if mode == "mv":
        F = oracle.factor(O, P, oracle.FMT_LU)
        xo = oracle.mv_sweeps(O, P, F, x0, O["b"], 0.66, nu, order=oracle.multicolor_order(prob))
    else:
        F = oracle.factor(O, P, oracle.FMT_DIAG)
        xo = oracle.additive_sweeps(O, P, F, x0, O["b"], 0.1, nu)
    xd = np.full(O["n"], np.nan)
    for _, g, v in res:
        xd[g] = v
    assert not np.isnan(xd).any()
    assert np.linalg.norm(xd - xo) <= 1e-12 * np.linalg.norm(xo)


def _lib_plan_worker(rank, world, port, nsub, q):
    """Planning of the library-driven cycle (dist.neighbor_plan) across processes: 2 processes
    driving nsub // 2 subdomains each, exchange_info all-gathered over gloo."""
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        prob = si.problem(2, (20, 26), si.KIND_MMS, eta="fourier")
        P = oracle.patches(prob, "pou")
        per = nsub // world
        local = list(range(rank * per, (rank + 1) * per))
        parts = rdist.partition_balanced(prob, nsub)
        slabs = [rdist.Slab(prob, nsub, g, parts) for g in local]
        written = []
        for s in slabs:
            gids = s.global_ids()
            g2l = -np.ones(int(gids.max()) + 1 + 10 ** 7, np.int64)
            g2l[gids] = np.arange(len(gids))
            p0, p1 = s.nlow_vert * s.V0, s.nlow_vert * s.V1
            wr = [g2l[P["dofs"][P["offs"][i]:P["offs"][i + 1]][P["w"][P["offs"][i]:P["offs"][i + 1]] > 0]]
                  for i in range(p0, p1)]
            written.append(np.unique(np.concatenate(wr)))
        infos = [rdist.exchange_info(s, w) for s, w in zip(slabs, written)]
        out = [None] * world
        dist.all_gather_object(out, infos)
        infos_all = [i for part in out for i in part]
        plans = {g: rdist.neighbor_plan(s, w, infos_all) for g, s, w in zip(local, slabs, written)}
        sizes = {g: {p: tuple(len(v) for v in lists) for p, lists in pl["neighbors"].items()} for g, pl in plans.items()}
        allsizes = [None] * world
        dist.all_gather_object(allsizes, sizes)
        q.put((rank, {k: v for d in allsizes for k, v in d.items()}))
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("nsub", [2, 4])
def test_lib_plan_lists_match_across_processes(nsub):
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_lib_plan_worker, args=(r, 2, port, nsub, q)) for r in range(2)]
    for p in procs:
        p.start()
    res = dict(q.get(timeout=240) for _ in procs)
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    sizes = res[0]
    assert res[0] == res[1] and sorted(sizes) == list(range(nsub))
    for g, nbs in sizes.items():
        for p, (cs, cr, hs, hr) in nbs.items():
            pcs, pcr, phs, phr = sizes[p][g]      # the peer's lists for me
            assert (cs, cr, hs, hr) == (pcr, pcs, phr, phs), (g, p)
            assert cs + cr > 0 and hs + hr > 0
