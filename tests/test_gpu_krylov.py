"""FGMRES with the RAV V-cycle as preconditioner on the GPU (mg_fgmres; SURVEY
row f3, reading R19) against the oracle's flexible GMRES
(oracle/krylov.py): identical step counts, residual histories to 1e-7
relative (above the 1e-13 ||r0|| rounding floor; the GPU orthogonalises with
CGS2, the oracle with MGS), solutions to 1e-9."""
import numpy as np
import pytest
import torch

import oracle
import seeded_inputs as si
from _parity import assert_entrywise
from oracle import krylov

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def rg():
    from paper_2103_10127_b200 import ravgmg
    return ravgmg


CASES = [
    (si.problem(2, (64, 64), si.KIND_MMS, eta="fourier"), 5, 2, 30),
    (si.problem(2, (32, 32), si.KIND_CAVITY, eta="fourier", elem=si.ELEM_Q1Q1), 3, 3, 30),
    (si.problem(2, (48, 32), si.KIND_CAVITY, eta="fourier"), 4, 2, 4),       # restarts
    (si.problem(3, (4, 4, 4), si.KIND_CAVITY, eta="fourier"), 2, 2, 30),
]


@pytest.mark.parametrize("case", CASES, ids=["mms64", "q1q1-cav32", "cav-restart4", "cav3d"])
def test_fgmres_matches_oracle(rg, case):
    prob, levels, pre, restart = case
    H = oracle.Hierarchy(prob, levels)
    xo, ko, ho = krylov.mg_fgmres(H, pre=pre, post=pre, omega=0.66, restart=restart, rtol=1e-10, maxit=100)
    mg, fine = rg.build_hierarchy(prob, levels, "pou")
    x = torch.zeros(fine["n"], dtype=torch.float64, device="cuda")
    _, kg, hg = mg.fgmres(x, fine["b"], pre=pre, post=pre, omega=0.66, restart=restart, rtol=1e-10, maxit=100)
    assert kg == ko, (kg, ko)
    np.testing.assert_allclose(hg, ho, rtol=1e-7, atol=1e-13 * ho[0])
    xg = x.cpu().numpy()
    assert_entrywise(xg, xo, np.abs(xo).max(), tol=1e-9)
    # FGMRES does not need more preconditioner applications than stationary MG
    _, ks, _ = H.solve(rtol=1e-10, omega=0.66, pre=pre, post=pre)
    assert kg <= ks
