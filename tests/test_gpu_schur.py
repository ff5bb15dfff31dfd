"""GPU parity of the factored (Schur) patch format, RAV_KERNEL_SCHUR
(csrc/schur.cu), against the oracle's explicit rows of L_i^{-1}.

The format stores the restricted rows of A_s^{-1}, g = A_s^{-1} b and 1/S
instead of the rows of L_i^{-1}; the applied operator is the same S_RAV
(Eq. 13), so the same 1e-12 per-sweep bar applies."""
import numpy as np
import pytest
import torch

import oracle
import seeded_inputs as si
from _parity import SweepChecker

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def rg():
    from paper_2103_10127_b200 import ravgmg
    return ravgmg


def np_(t):
    return t.detach().cpu().numpy()


CASES = [
    (si.problem(2, (40, 33), si.KIND_MMS, eta="fourier"), "pou", 0.66),
    (si.problem(2, (31, 40), si.KIND_CAVITY, eta="fourier"), "own", 0.66),
    (si.problem(2, (24, 24), si.KIND_MMS, eta="fourier", box=(1.0, 2.0)), "full", 0.1),
    (si.problem(3, (5, 4, 6), si.KIND_CAVITY, eta="fourier"), "pou", 0.66),
    (si.problem(3, (4, 4, 4), si.KIND_CAVITY, eta="fourier"), "own", 0.66),
]


@pytest.mark.parametrize("case", CASES, ids=["2d-pou", "2d-own", "2d-av", "3d-pou", "3d-own"])
def test_schur_sweeps_match_oracle(rg, case):
    prob, weights, omega = case
    G = rg.gen_level(prob, weights)
    sm = rg.Smoother(G, G, kernel=rg.KERNEL_SCHUR)
    O = oracle.assemble(prob)
    P = oracle.patches(prob, weights)
    F = oracle.factor(O, P, oracle.FMT_ROWS)
    x0 = si.initial_guess(O["n"], seed=5)
    x = torch.tensor(x0, device="cuda")

    def gpu(k):
        sm.smooth(x, G["b"], k, omega)
        return np_(x)

    SweepChecker(O, P, F, O["b"], omega).run(x0, gpu, (1, 3, 20), what=sm.kernel_name)


@pytest.mark.parametrize("dim,n", [(2, (9, 7)), (3, (3, 3, 2))])
def test_schur_rows_match_oracle(rg, dim, n):
    prob = si.problem(dim, n, si.KIND_MMS if dim == 2 else si.KIND_CAVITY, eta="fourier")
    G = rg.gen_level(prob, "pou")
    sm = rg.Smoother(G, G, kernel=rg.KERNEL_SCHUR)
    rows = np_(sm.export_rows())
    O = oracle.assemble(prob)
    P = oracle.patches(prob, "pou")
    F = oracle.factor(O, P, oracle.FMT_ROWS)
    fo = F["foffs"]
    for i in range(len(P["offs"]) - 1):
        ni = P["offs"][i + 1] - P["offs"][i]
        Rg = rows[fo[i]:fo[i + 1]].reshape(-1, ni)
        Ro = F["fac"][fo[i]:fo[i + 1]].reshape(-1, ni)
        for k in range(Ro.shape[0]):
            assert np.abs(Rg[k] - Ro[k]).max() <= 1e-12 * np.abs(Ro[k]).max(), (i, k)


def test_schur_rejects_unstructured_patches(rg):
    # one patch covering everything (many pressure DoFs): SCHUR must refuse, AUTO falls back
    prob = si.problem(2, (3, 3), si.KIND_MMS, eta="fourier")
    G = rg.gen_level(prob, "pou")
    n = G["n"]
    P = {"offs": torch.tensor([0, n], dtype=torch.int64, device="cuda"),
         "dofs": torch.arange(n, dtype=torch.int32, device="cuda"),
         "w": torch.ones(n, dtype=torch.float64, device="cuda")}
    with pytest.raises(rg.RavError):
        rg.Smoother(G, P, kernel=rg.KERNEL_SCHUR)


def test_schur_is_default_and_cuts_bytes(rg):
    prob = si.problem(2, (64, 64), si.KIND_MMS, eta="fourier")
    G = rg.gen_level(prob, "pou")
    auto = rg.Smoother(G, G).sweep_bytes()["sweep"]
    rows = rg.Smoother(G, G, kernel=rg.KERNEL_THREAD).sweep_bytes()["sweep"]
    assert auto < 0.45 * rows


def test_vcycle_3d_schur_counts_match_oracle(rg):
    prob = si.problem(3, (8, 8, 8), si.KIND_CAVITY, eta="fourier")
    H = oracle.Hierarchy(prob, 3, "rav")
    _, ko, ho = H.solve(rtol=1e-8, omega=0.66, pre=2, post=2, maxit=100)
    mg, fine = rg.build_hierarchy(prob, 3, "pou")
    x = torch.zeros(fine["n"], dtype=torch.float64, device="cuda")
    x, kg, hg = mg.solve(x, fine["b"], pre=2, post=2, omega=0.66, rtol=1e-8, maxit=100)
    assert kg == ko, (kg, ko)
