"""Comparison smoothers across slab-partitioned ranks on the GPU (SURVEY section 8
rows a6 / d5 / e): multicoloured multiplicative Vanka (dist.DistMVSweeper:
rav_apply_color per colour, changes of ghost DoFs to their owners, halo
refresh) and additive diagonal Vanka (dist.DistSweeper with the closed-form
diagonal kernel).  Ranks are threads of this process on the one GPU
(dist.ThreadComm, host rendezvous only).  The assembled result must match the
single-domain oracle sweep (colour-major order for MV) to 1e-12.  (MV on the
GPU is 2D: its per-patch full rows use one lane per node, <= 32 nodes; the 3D
MV host protocol is covered on CPU in tests/test_dist_cpu.py.)"""
import numpy as np
import pytest
import torch

import oracle
import seeded_inputs as si
from _parity import assert_entrywise

pytestmark = pytest.mark.gpu


def run(prob, world, mode, nu):
    from paper_2103_10127_b200 import dist as rdist
    from paper_2103_10127_b200 import ravgmg as rg
    hub = rdist.ThreadComm.Hub(world)
    n = None

    def rank_fn(r):
        torch.cuda.set_device(0)
        comm = rdist.ThreadComm(hub, r, sync=torch.cuda.synchronize)
        slab = rdist.Slab(prob, world, r)
        L = rg.gen_level(slab.local_problem(), "full")
        variant = rg.VARIANT_MV if mode == "mv" else rg.VARIANT_DIAG
        sm = rg.Smoother(L, L, variant=variant)
        be = rdist.GpuBackend(sm)
        written = rdist.written_local_from_patches(L)
        if mode == "mv":
            offs, ids = rdist.local_colors(slab)
            sm.set_colors(offs, ids)
            sw = rdist.DistMVSweeper(slab, be, comm, written, len(offs) - 1)
        else:
            sw = rdist.DistSweeper(slab, be, comm, written)
        nglob = slab.nvel_glob + slab.nvert_glob
        x0 = si.initial_guess(nglob, seed=29)
        x = torch.tensor(x0[slab.global_ids()], device="cuda")
        sw.smooth(x, L["b"], nu, 0.66 if mode == "mv" else 0.1)
        torch.cuda.synchronize()
        own = slab.owned_mask()
        return slab.global_ids()[own], x.cpu().numpy()[own]

    return rdist.run_threads(world, rank_fn)


CASES = [
    (si.problem(2, (16, 24), si.KIND_MMS, eta="fourier"), 2, "mv"),
    (si.problem(2, (12, 30), si.KIND_CAVITY, eta="fourier"), 3, "mv"),
    (si.problem(2, (16, 24), si.KIND_MMS, eta="fourier"), 2, "diag"),
    (si.problem(3, (3, 4, 9), si.KIND_CAVITY, eta="fourier"), 3, "diag"),
]


@pytest.mark.parametrize("case", CASES, ids=["mv-2d-w2", "mv-2d-w3", "diag-2d-w2", "diag-3d-w3"])
def test_distributed_smoother_matches_oracle(case):
    prob, world, mode = case
    nu = 2
    res = run(prob, world, mode, nu)
    O = oracle.assemble(prob)
    P = oracle.patches(prob, "full")
    x0 = si.initial_guess(O["n"], seed=29)
    if mode == "mv":
        F = oracle.factor(O, P, oracle.FMT_LU)
        xo = oracle.mv_sweeps(O, P, F, x0, O["b"], 0.66, nu, order=oracle.multicolor_order(prob))
    else:
        F = oracle.factor(O, P, oracle.FMT_DIAG)
        xo = oracle.additive_sweeps(O, P, F, x0, O["b"], 0.1, nu)
    xd = np.full(O["n"], np.nan)
    for g, v in res:
        xd[g] = v
    assert not np.isnan(xd).any()
    assert_entrywise(xd, xo, np.abs(xo).max(), tol=1e-12)
