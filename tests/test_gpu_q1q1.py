"""GPU parity for the paper's own stabilized Q1-Q1 pair (Eq. 8, reading
R18): the CUDA generator, the smoother kernels and the
V-cycle through the C-ABI against the CPU oracle, with the tolerances of
tests/test_gpu_parity.py (integer data exact, entries 1e-14 max|L|, sweeps
1e-12, identical V-cycle counts)."""
import numpy as np
import pytest
import torch

import oracle
import seeded_inputs as si
from _parity import assert_entrywise

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def rg():
    from paper_2103_10127_b200 import ravgmg
    return ravgmg


def np_(t):
    return t.detach().cpu().numpy()


PROBLEMS = [
    si.problem(2, (8, 8), si.KIND_CAVITY, elem=si.ELEM_Q1Q1),
    si.problem(2, (13, 7), si.KIND_MMS, eta="fourier", elem=si.ELEM_Q1Q1),
    si.problem(3, (3, 4, 2), si.KIND_CAVITY, eta="fourier", elem=si.ELEM_Q1Q1),
]
IDS = ["cav8", "mms13x7", "cav3d"]


@pytest.mark.parametrize("prob", PROBLEMS, ids=IDS)
def test_q1q1_operator_matches_oracle(rg, prob):
    G = rg.gen_level(prob, "pou")
    O = oracle.assemble(prob)
    assert G["n"] == O["n"] and G["nvel"] == O["nvel"]
    assert np.array_equal(np_(G["rp"]), O["rp"])
    assert np.array_equal(np_(G["ci"]), O["ci"])
    assert np.abs(np_(G["val"]) - O["val"]).max() <= 1e-14 * np.abs(O["val"]).max()
    assert np.abs(np_(G["b"]) - O["b"]).max() <= 1e-13 * max(np.abs(O["b"]).max(), 1e-300)


@pytest.mark.parametrize("weights", ["pou", "full"])
@pytest.mark.parametrize("prob", PROBLEMS, ids=IDS)
def test_q1q1_patches_match_oracle(rg, prob, weights):
    G = rg.gen_patches(prob, weights)
    O = oracle.patches(prob, weights)
    for k in ("offs", "dofs", "w"):
        assert np.array_equal(np_(G[k]), O[k])


@pytest.mark.parametrize("dim,nc", [(2, (4, 3)), (3, (2, 2, 3))])
def test_q1q1_prolongation_matches_oracle(rg, dim, nc):
    pc = si.problem(dim, nc, si.KIND_CAVITY, elem=si.ELEM_Q1Q1)
    pf = si.problem(dim, [2 * c for c in nc], si.KIND_CAVITY, elem=si.ELEM_Q1Q1)
    G = rg.gen_prolongation(pf, pc)
    O = oracle.prolongation(pf, pc)
    for k in ("rp", "ci", "val"):
        assert np.array_equal(np_(G[k]), O[k])


@pytest.mark.parametrize("kernel", [0, 1, 2, 4], ids=["auto", "warp", "thread", "schur"])
@pytest.mark.parametrize("weights", ["pou", "full"])
@pytest.mark.parametrize("prob", PROBLEMS[1:], ids=IDS[1:])
def test_q1q1_additive_sweeps_match_oracle(rg, prob, weights, kernel):
    if prob["dim"] == 3 and kernel == 2:
        pytest.skip("thread kernel is 2D-sized")
    G = rg.gen_level(prob, weights)
    sm = rg.Smoother(G, G, kernel=kernel)
    O = oracle.assemble(prob)
    P = oracle.patches(prob, weights)
    F = oracle.factor(O, P, oracle.FMT_ROWS)
    x0 = si.initial_guess(O["n"], seed=11)
    x = torch.tensor(x0, device="cuda")
    om = 0.66 if weights == "pou" else 0.1
    xo = x0
    for nu in (1, 1, 3):          # cumulative 1, 2, 5 sweeps
        sm.smooth(x, G["b"], nu, om)
        xo = oracle.additive_sweeps(O, P, F, xo, O["b"], om, nu)
        torch.cuda.synchronize()
        assert_entrywise(np_(x), xo, np.abs(xo).max(), tol=1e-12)


@pytest.mark.parametrize("variant,smoother,omega", [(0, "rav", 0.66), (0, "av", 0.1), (2, "mv", 0.66)],
                         ids=["rav", "av", "mv-color"])
def test_q1q1_vcycle_counts_match_oracle(rg, variant, smoother, omega):
    """The paper's cavity setting on uniform grids: 8x8 coarse grid, V(3,3)
    (P:136), 1e-8 reduction."""
    prob = si.problem(2, (32, 32), si.KIND_CAVITY, eta="fourier", elem=si.ELEM_Q1Q1)
    weights = {"rav": "pou", "av": "full", "mv": "full"}[smoother]
    H = oracle.Hierarchy(prob, 3, smoother, mv_order="color")
    xo, ko, _ = H.solve(rtol=1e-8, omega=omega, pre=3, post=3, maxit=300)
    mg, fine = rg.build_hierarchy(prob, 3, weights, variant=variant)
    x = torch.zeros(fine["n"], dtype=torch.float64, device="cuda")
    _, kg, hist = mg.solve(x, fine["b"], pre=3, post=3, omega=omega, rtol=1e-8, maxit=300)
    assert kg == ko, (kg, ko)
    assert_entrywise(np_(x), xo, np.abs(xo).max(), tol=1e-9)
