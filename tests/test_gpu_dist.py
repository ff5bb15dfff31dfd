"""Slab-partitioned RAV sweeps on the GPU (SURVEY section 8 row e).

Only one GPU is available to the tests, so R ranks are emulated in ONE process
on one device, driven phase by phase in lock step (dist.DistSweeper phases;
the buffers move between the rank objects with plain device copies) -- no
kernel ever waits on another rank.  Every rank generates its own window with
rav_gen_* (win = 1), builds its own smoother and exchanges through the
rav_index_op pack/unpack kernels.  The result must equal the single-domain
GPU smoother and the oracle.  The NCCL transport of the same protocol is the
torch.distributed path exercised by bench.py under torchrun."""
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


def run_emulated(rg, prob, weights, world, nu, omega=0.66, kernel=0):
    from paper_2103_10127_b200 import dist as rdist
    slabs = [rdist.Slab(prob, world, r) for r in range(world)]
    levels = [rg.gen_level(s.local_problem(), weights) for s in slabs]
    for s, L in zip(slabs, levels):
        assert L["n"] == s.n_loc and len(L["offs"]) - 1 == s.n_patches
    sms = [rg.Smoother(L, L, kernel=kernel) for L in levels]
    written = [rdist.written_local_from_patches(L) for L in levels]
    infos = [rdist.exchange_info(s, w) for s, w in zip(slabs, written)]
    sws = [rdist.DistSweeper(s, rdist.GpuBackend(sm), None, w, all_infos=infos)
           for s, sm, w in zip(slabs, sms, written)]
    n = slabs[0].nvel_glob + slabs[0].nvert_glob
    x0 = si.initial_guess(n, seed=19)
    xs = [torch.tensor(x0[s.global_ids()], device="cuda") for s in slabs]
    for _ in range(nu):
        for sw, x, L in zip(sws, xs, levels):
            sw.phase_compute(x, L["b"], omega)
        for r, sw in enumerate(sws):
            for q, buf in sw.cs_buf.items():
                sws[q].cr_buf[r].copy_(buf)
        for sw, x in zip(sws, xs):
            sw.phase_corrections(x)
        for r, sw in enumerate(sws):
            for q, buf in sw.hs_buf.items():
                sws[q].hr_buf[r].copy_(buf)
        for sw, x in zip(sws, xs):
            sw.phase_halo(x)
    torch.cuda.synchronize()
    out = np.full(n, np.nan)
    for s, x in zip(slabs, xs):
        own = s.owned_mask()
        out[s.global_ids()[own]] = x.cpu().numpy()[own]
    assert not np.isnan(out).any()
    return out, x0


@pytest.mark.parametrize("prob,weights,world", [
    (si.problem(2, (48, 40), si.KIND_MMS, eta="fourier"), "pou", 4),
    (si.problem(2, (33, 29), si.KIND_CAVITY, eta="fourier"), "own", 3),
    (si.problem(3, (5, 4, 12), si.KIND_CAVITY, eta="fourier"), "pou", 3),
], ids=["2d-pou-4", "2d-own-3", "3d-pou-3"])
def test_emulated_ranks_match_single_domain(rg, prob, weights, world):
    nu = 4
    xd, x0 = run_emulated(rg, prob, weights, world, nu)
    G = rg.gen_level(prob, weights)
    sm = rg.Smoother(G, G)
    x = torch.tensor(x0, device="cuda")
    sm.smooth(x, G["b"], nu, 0.66)
    xg = x.cpu().numpy()
    O = oracle.assemble(prob)
    P = oracle.patches(prob, weights)
    F = oracle.factor(O, P, oracle.FMT_ROWS)
    scale = sweep_magnitude(O, P, F, x0, O["b"], 0.66).max()
    assert_entrywise(xd, xg, scale, what="emulated ranks vs single-domain GPU")
    xo = oracle.additive_sweeps(O, P, F, x0, O["b"], 0.66, nu)
    assert_entrywise(xd, xo, scale, what="emulated ranks vs oracle")


def test_window_generator_rows_equal_global_rows(rg):
    from paper_2103_10127_b200 import dist as rdist
    prob = si.problem(2, (20, 24), si.KIND_MMS, eta="fourier")
    G = rg.gen_level(prob, "pou")
    grp, gci, gval = (t.cpu().numpy() for t in (G["rp"], G["ci"], G["val"]))
    for r in range(3):
        s = rdist.Slab(prob, 3, r)
        L = rg.gen_level(s.local_problem(), "pou")
        gids = s.global_ids()
        rp, ci, val, b = (t.cpu().numpy() for t in (L["rp"], L["ci"], L["val"], L["b"]))
        for l in range(0, s.n_loc, 7):
            if rp[l + 1] == rp[l]:
                continue
            g = gids[l]
            assert np.array_equal(gids[ci[rp[l]:rp[l + 1]]], gci[grp[g]:grp[g + 1]])
            assert np.array_equal(val[rp[l]:rp[l + 1]], gval[grp[g]:grp[g + 1]])
            assert b[l] == G["b"][g].item()
