"""The adaptive hierarchy on the GPU (rav_adaptive_*, reading R20)
against the oracle (oracle/adaptive.py) and the paper's Table 1: element and DoF
counts, operator / rhs / patches / prolongation parity (integer data exact,
values 1e-14), RAV sweeps 1e-12, V-cycle counts equal to the oracle."""
import numpy as np
import pytest
import torch

import oracle
import seeded_inputs as si
from _parity import assert_entrywise
from oracle import adaptive as ad

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def rg():
    from paper_2103_10127_b200 import ravgmg
    return ravgmg


def np_(t):
    return t.detach().cpu().numpy()


def test_table1_counts(rg):
    from test_oracle_adaptive import table1
    T = table1()
    levels = rg.gen_adaptive(si.problem(2, (8, 8), si.KIND_CAVITY, elem=si.ELEM_Q1Q1), 7)
    for k, lev in enumerate(levels, start=1):
        npres = lev["n"] - lev["nvel"]
        assert (lev["n_cells"], 3 * npres) == T[k], k


@pytest.mark.parametrize("kind,eta", [(si.KIND_CAVITY, "const"), (si.KIND_MMS, "fourier")])
def test_adaptive_levels_match_oracle(rg, kind, eta):
    prob = si.problem(2, (8, 8), kind, eta=eta, elem=si.ELEM_Q1Q1)
    L = 4
    levels = rg.gen_adaptive(prob, L)
    cells, N = ad.hierarchy_cells(L)
    meshes = [ad.Mesh(c, N) for c in cells]
    for l, (lev, m) in enumerate(zip(levels, meshes)):
        A = ad.assemble(prob, m)
        assert lev["n"] == A["n"] and lev["nvel"] == A["nvel"]
        assert np.array_equal(np_(lev["rp"]), A["rp"]) and np.array_equal(np_(lev["ci"]), A["ci"])
        assert np.abs(np_(lev["val"]) - A["val"]).max() <= 1e-14 * np.abs(A["val"]).max()
        assert np.abs(np_(lev["b"]) - A["b"]).max() <= 1e-13 * max(np.abs(A["b"]).max(), 1e-300)
        P = ad.patches(A, m)
        for k in ("offs", "dofs", "w"):
            assert np.array_equal(np_(lev[k]), P[k]), (l, k)
        if l > 0:
            T = ad.prolongation(m, meshes[l - 1])
            for k in ("rp", "ci", "val"):
                assert np.array_equal(np_(lev["prol"][k]), T[k]), (l, k)


def test_adaptive_rav_sweeps_match_oracle(rg):
    prob = si.problem(2, (8, 8), si.KIND_MMS, eta="fourier", elem=si.ELEM_Q1Q1)
    lev = rg.gen_adaptive(prob, 3)[-1]
    sm = rg.Smoother(lev, lev)
    cells, N = ad.hierarchy_cells(3)
    m = ad.Mesh(cells[-1], N)
    A = ad.assemble(prob, m)
    P = ad.patches(A, m)
    F = oracle.factor(A, P, oracle.FMT_ROWS)
    x0 = si.initial_guess(A["n"], seed=41)
    x = torch.tensor(x0, device="cuda")
    sm.smooth(x, lev["b"], 3, 0.66)
    xo = oracle.additive_sweeps(A, P, F, x0, A["b"], 0.66, 3)
    assert_entrywise(np_(x), xo, np.abs(xo).max(), tol=1e-12)


@pytest.mark.parametrize("smoother,weights,omega", [("rav", "own", 0.66), ("av", "full", 0.1)])
def test_adaptive_vcycle_counts_match_oracle(rg, smoother, weights, omega):
    prob = si.problem(2, (8, 8), si.KIND_CAVITY, elem=si.ELEM_Q1Q1)
    H = ad.AdaptiveHierarchy(prob, 4, smoother)
    xo, ko, _ = H.solve(rtol=1e-8, omega=omega, pre=3, post=3, maxit=300)
    mg, fine = rg.build_adaptive_hierarchy(prob, 4, weights)
    x = torch.zeros(fine["n"], dtype=torch.float64, device="cuda")
    _, kg, _ = mg.solve(x, fine["b"], pre=3, post=3, omega=omega, rtol=1e-8, maxit=300)
    assert kg == ko, (kg, ko)
    assert_entrywise(np_(x), xo, np.abs(xo).max(), tol=1e-9)


def test_greedy_colors_match_oracle_and_mv_vcycle(rg):
    prob = si.problem(2, (8, 8), si.KIND_CAVITY, elem=si.ELEM_Q1Q1)
    levels = rg.gen_adaptive(prob, 3)
    cells, N = ad.hierarchy_cells(3)
    for l in (1, 2):
        m = ad.Mesh(cells[l], N)
        A = ad.assemble(prob, m)
        P = dict(ad.patches(A, m))
        P["w"] = np.ones_like(P["w"])
        order = ad.greedy_colors(A, P)
        offs, ids = rg.color_patches(levels[l], levels[l])
        assert np.array_equal(ids, order)
    H = ad.AdaptiveHierarchy(prob, 3, "mv", mv_order="color")
    xo, ko, _ = H.solve(rtol=1e-8, omega=0.66, pre=3, post=3, maxit=300)
    mg, fine = rg.build_adaptive_hierarchy(prob, 3, "full", variant=rg.VARIANT_MV)
    x = torch.zeros(fine["n"], dtype=torch.float64, device="cuda")
    _, kg, _ = mg.solve(x, fine["b"], pre=3, post=3, omega=0.66, rtol=1e-8, maxit=300)
    assert kg == ko, (kg, ko)
    assert_entrywise(np_(x), xo, np.abs(xo).max(), tol=1e-9)
