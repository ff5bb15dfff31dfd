"""GPU parity of the residual r = b - L x (Eq. 10).

rav_residual runs the node-blocked kernel (nb.cu) for Taylor-Hood operators and
the SELL kernel otherwise (the Q1-Q1 pressure rows carry C entries, so the
node-blocked structure check rejects them).  The sizes reach every lane count
the launcher picks by level size (a full warp, 8, 2 and 1 lanes per block row),
ragged slice tails, and 8-byte-aligned (not 16-byte-aligned) vectors, which take
the scalar b / r path of the 2D pair layout.

Bar: |r_gpu - r_oracle|_i <= 1e-14 * (sum_j |L_ij x_j| + |b_i|) + tiny, i.e. the
rounding of a reordered fp64 dot product of <= 100 terms, row by row.  The
oracle assembles its own operator and computes its own residual.
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
    "q2q1_8x8": si.problem(2, (8, 8), si.KIND_CAVITY),                          # 32 lanes per row
    "q2q1_37x29": si.problem(2, (37, 29), si.KIND_MMS, eta="fourier"),          # 8 lanes, ragged
    "q2q1_64x64": si.problem(2, (64, 64), si.KIND_MMS, eta="fourier"),          # 2 lanes
    "q2q1_203x190": si.problem(2, (203, 190), si.KIND_MMS, eta="fourier"),      # 1 lane (c2 path)
    "q2q1_3d_4x3x5": si.problem(3, (4, 3, 5), si.KIND_CAVITY, eta="fourier"),
    "q2q1_3d_12": si.problem(3, (12, 12, 12), si.KIND_CAVITY, eta="fourier"),
    "q1q1_48x40": si.problem(2, (48, 40), si.KIND_CAVITY, elem=si.ELEM_Q1Q1),   # SELL path
}


def _oracle_bound(O, x, b):
    rows = np.repeat(np.arange(O["n"]), np.diff(O["rp"]))
    absax = np.bincount(rows, weights=np.abs(O["val"] * x[O["ci"]]), minlength=O["n"])
    return absax + np.abs(b)


@pytest.mark.parametrize("name", list(CASES))
@pytest.mark.parametrize("aligned", [True, False], ids=["aligned16", "offset8"])
def test_residual_matches_oracle(rg, name, aligned):
    prob = CASES[name]
    L = rg.gen_level(prob, "pou")
    sm = rg.Smoother(L, L)
    n = L["n"]
    O = oracle.assemble(prob)
    assert O["n"] == n
    x_h = si.initial_guess(n, seed=si.X0_SEED)
    b_h = O["b"] + si.initial_guess(n, seed=si.X0_SEED + 1)   # a generic right-hand side
    if aligned:
        x = torch.tensor(x_h, device="cuda")
        b = torch.tensor(b_h, device="cuda")
        r = torch.full((n,), np.nan, dtype=torch.float64, device="cuda")
    else:   # views one double into larger buffers: 8-byte but not 16-byte aligned
        xb = torch.zeros(n + 1, dtype=torch.float64, device="cuda")
        bb = torch.zeros(n + 1, dtype=torch.float64, device="cuda")
        rb = torch.full((n + 1,), np.nan, dtype=torch.float64, device="cuda")
        x, b, r = xb[1:], bb[1:], rb[1:]
        x.copy_(torch.tensor(x_h))
        b.copy_(torch.tensor(b_h))
    sm.residual(x, b, r)
    torch.cuda.synchronize()
    r_gpu = r.cpu().numpy()
    r_ora = oracle.residual(O, x_h, b_h)
    bound = 1e-14 * _oracle_bound(O, x_h, b_h) + 1e-300
    err = np.abs(r_gpu - r_ora)
    assert np.all(np.isfinite(r_gpu))
    worst = int(np.argmax(err / bound))
    assert np.all(err <= bound), (name, worst, err[worst], bound[worst])


def test_residual_is_repeatable_bitwise(rg):
    """No atomics in the residual: two launches give identical bits."""
    prob = CASES["q2q1_203x190"]
    L = rg.gen_level(prob, "pou")
    sm = rg.Smoother(L, L)
    x = torch.tensor(si.initial_guess(L["n"], seed=si.X0_SEED), device="cuda")
    r1 = sm.residual(x, L["b"])
    r2 = sm.residual(x, L["b"])
    torch.cuda.synchronize()
    assert torch.equal(r1, r2)
