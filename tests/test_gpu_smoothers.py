"""GPU comparison smoothers against the oracle:
diagonal Vanka (R17; closed-form kernel and the generic local-solve path) and
multicoloured multiplicative Vanka (Eq. 11 with fresh local residuals,
P:221 Eq. 15; colouring R10) -- the GPU relaxes each colour concurrently, the
oracle runs the patches one after the other in colour-major order."""
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


@pytest.mark.parametrize("block_dim,weights", [(None, "full"), (0, "full"), (None, "pou")],
                         ids=["closed-form", "generic", "closed-form-restricted"])
def test_diag_vanka(rg, block_dim, weights):
    prob = si.problem(2, (33, 26), si.KIND_MMS, eta="fourier")
    G = rg.gen_level(prob, weights)
    sm = rg.Smoother(G, G, variant=rg.VARIANT_DIAG, block_dim=block_dim)
    if block_dim is None:
        assert "diag_sweep" in sm.kernel_name
    O = oracle.assemble(prob)
    P = oracle.patches(prob, weights)
    F = oracle.factor(O, P, oracle.FMT_DIAG)
    x0 = si.initial_guess(O["n"], seed=21)
    x = torch.tensor(x0, device="cuda")
    sm.smooth(x, G["b"], 25, 0.1)
    xo = oracle.additive_sweeps(O, P, F, x0, O["b"], 0.1, 25)
    assert_entrywise(np_(x), xo, np.abs(xo).max())


def test_diag_vanka_3d(rg):
    prob = si.problem(3, (4, 3, 5), si.KIND_CAVITY, eta="fourier")
    G = rg.gen_level(prob, "full")
    sm = rg.Smoother(G, G, variant=rg.VARIANT_DIAG)
    O = oracle.assemble(prob)
    P = oracle.patches(prob, "full")
    F = oracle.factor(O, P, oracle.FMT_DIAG)
    x0 = si.initial_guess(O["n"], seed=22)
    x = torch.tensor(x0, device="cuda")
    sm.smooth(x, G["b"], 10, 0.1)
    xo = oracle.additive_sweeps(O, P, F, x0, O["b"], 0.1, 10)
    assert_entrywise(np_(x), xo, np.abs(xo).max())


@pytest.mark.parametrize("n", [(17, 13), (40, 40)])
def test_multicolor_mv_matches_sequential_oracle(rg, n):
    prob = si.problem(2, n, si.KIND_MMS, eta="fourier")
    G = rg.gen_level(prob, "full")
    sm = rg.Smoother(G, G, variant=rg.VARIANT_MV)
    offs, ids = rg.multicolor(prob)
    sm.set_colors(offs, ids)
    O = oracle.assemble(prob)
    P = oracle.patches(prob, "full")
    F = oracle.factor(O, P, oracle.FMT_LU)
    order = oracle.multicolor_order(prob)
    assert np.array_equal(order, ids)
    x0 = si.initial_guess(O["n"], seed=23)
    x = torch.tensor(x0, device="cuda")
    xo = x0.copy()
    done = 0
    for target in (1, 5):
        sm.smooth(x, G["b"], target - done, 0.66)
        xo = oracle.mv_sweeps(O, P, F, xo, O["b"], 0.66, target - done, order=order)
        done = target
        assert_entrywise(np_(x), xo, np.abs(xo).max(), what=f"after {target} sweeps")


def test_mv_needs_colors(rg):
    prob = si.problem(2, (8, 8), si.KIND_MMS, eta="fourier")
    G = rg.gen_level(prob, "full")
    sm = rg.Smoother(G, G, variant=rg.VARIANT_MV)
    x = torch.zeros(G["n"], dtype=torch.float64, device="cuda")
    with pytest.raises(rg.RavError):
        sm.smooth(x, G["b"], 1, 0.66)
