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
        xv, rv = x.numpy(), r.numpy()
        for i in range(len(self.rp) - 1):
            s, e = self.rp[i], self.rp[i + 1]
            rv[i] = self.b[i] - np.dot(self.val[s:e], xv[self.ci[s:e]])

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
