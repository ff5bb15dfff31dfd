"""GPU parity of the stencil-form transfers (csrc/xfer.cu).

The stencil kernels apply the nested interpolation P of a uniformly refined grid and
R = P^T without a matrix.  Here the transfer object is built from the ORACLE's P
(host CSR), so rav_xfer_set_structured's built-in check compares the stencil form
with an independent assembly of P; the applied results are then compared with
numpy products of the oracle's P.  The weights are dyadic (1, 3/4, 3/8, -1/8,
1/2 and their products), so the only difference is the order of <= 125 fp64
additions: bar 1e-14 relative to max|result|.
"""
import numpy as np
import pytest
import torch

import oracle
import seeded_inputs as si

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def rg():
    from paper_2103_10127_b200 import ravgmg
    return ravgmg


CASES = {
    "q2q1_2d": si.problem(2, (16, 12), si.KIND_MMS, eta="fourier"),
    "q2q1_2d_box": si.problem(2, (10, 6), si.KIND_CAVITY, box=(1.0, 2.0)),
    "q2q1_3d": si.problem(3, (4, 6, 4), si.KIND_CAVITY, eta="fourier"),
    "q1q1_2d": si.problem(2, (16, 16), si.KIND_CAVITY, elem=si.ELEM_Q1Q1),
}


def _dense_apply(Pm, x):
    n = Pm["n"]
    rows = np.repeat(np.arange(n), np.diff(Pm["rp"]))
    return np.bincount(rows, weights=Pm["val"] * x[Pm["ci"]], minlength=n)


def _dense_apply_t(Pm, y):
    return np.bincount(Pm["ci"], weights=Pm["val"] * y[np.repeat(np.arange(Pm["n"]), np.diff(Pm["rp"]))],
                       minlength=Pm["nc"])


@pytest.mark.parametrize("name", list(CASES))
def test_stencil_transfers_match_oracle(rg, name):
    fine = CASES[name]
    coarse = rg.coarsen_problem(fine)
    Pm = oracle.prolongation(fine, coarse)
    t = rg.Transfer(Pm)
    t.set_structured(fine, coarse)     # verified against the oracle's P inside the library
    rng = np.random.default_rng(7)
    xc = rng.standard_normal(Pm["nc"])
    xf0 = rng.standard_normal(Pm["n"])
    rf = rng.standard_normal(Pm["n"])
    xf = torch.tensor(xf0, device="cuda")
    t.prolong(torch.tensor(xc, device="cuda"), xf, alpha=0.7)
    bc = torch.full((Pm["nc"],), np.nan, dtype=torch.float64, device="cuda")
    t.restrict(torch.tensor(rf, device="cuda"), bc)
    torch.cuda.synchronize()
    ref_p = xf0 + 0.7 * _dense_apply(Pm, xc)
    ref_r = _dense_apply_t(Pm, rf)
    assert np.abs(xf.cpu().numpy() - ref_p).max() <= 1e-14 * np.abs(ref_p).max()
    assert np.abs(bc.cpu().numpy() - ref_r).max() <= 1e-14 * np.abs(ref_r).max()
    t.close()


def test_structured_transfer_rejects_non_nested_grids(rg):
    fine = CASES["q2q1_2d"]
    coarse = rg.coarsen_problem(fine)
    Pm = oracle.prolongation(fine, coarse)
    t = rg.Transfer(Pm)
    wrong = dict(coarse, ncell=[coarse["ncell"][0], coarse["ncell"][1] + 1, 1])
    with pytest.raises(rg.RavError):
        t.set_structured(fine, wrong)
    q1 = dict(coarse, vel_order=1, beta=0.01)
    with pytest.raises(rg.RavError):
        t.set_structured(fine, q1)
    # a P that is not the nested interpolation: the numerical check refuses it
    Pbad = {k: (v.copy() if isinstance(v, np.ndarray) else v) for k, v in Pm.items()}
    Pbad["val"][len(Pbad["val"]) // 2] += 0.25
    tb = rg.Transfer(Pbad)
    with pytest.raises(rg.RavError):
        tb.set_structured(fine, coarse)
    t.close()
    tb.close()


@pytest.mark.parametrize("dim,n,levels", [(2, 64, 5), (3, 8, 3)])
def test_vcycle_same_with_stencil_and_csr_transfers(rg, dim, n, levels):
    prob = si.problem(dim, [n] * dim, si.KIND_MMS if dim == 2 else si.KIND_CAVITY, eta="fourier")
    out = []
    for structured in (False, True):
        mg, fine = rg.build_hierarchy(prob, levels, "pou", structured_transfers=structured)
        x = torch.zeros(fine["n"], dtype=torch.float64, device="cuda")
        x, k, hist = mg.solve(x, fine["b"], pre=2, post=2, omega=0.66, rtol=1e-8, maxit=100)
        torch.cuda.synchronize()
        out.append((k, x.cpu().numpy(), hist))
        mg.close()
    assert out[0][0] == out[1][0]
    assert np.abs(out[0][1] - out[1][1]).max() <= 1e-10 * np.abs(out[0][1]).max()
