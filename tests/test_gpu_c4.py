"""BASELINE config 4 (3D 32^3 Q2-Q1 lid-driven cavity, seeded viscosity) at
full size on the GPU: generator parity on sampled rows, a sampled-DoF sweep
against the oracle (which factorizes only the patches it needs), and V-cycle
convergence (5 levels, 2^3 coarsest; reading R14)."""
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


def np_(t):
    return t.detach().cpu().numpy()


def test_c4_full_size_sampled_sweep(rg):
    prob = si.config_problem("c4")
    G = rg.gen_level(prob, "pou")
    sm = rg.Smoother(G, G)
    assert "schur" in sm.kernel_name
    x0 = si.initial_guess(G["n"], seed=7)
    x = torch.tensor(x0, device="cuda")
    sm.smooth(x, G["b"], 1, 0.66)
    O = oracle.assemble(prob)
    assert np.array_equal(np_(G["rp"]), O["rp"]) and np.array_equal(np_(G["ci"]), O["ci"])
    assert np.abs(np_(G["val"]) - O["val"]).max() <= 1e-14 * np.abs(O["val"]).max()
    P = oracle.patches(prob, "pou")
    rng = np.random.Generator(np.random.PCG64(13))
    sample = np.unique(np.concatenate([rng.choice(O["n"], 60, replace=False),
                                       np.arange(O["nvel"] - 6, O["nvel"] + 6), np.arange(O["n"] - 6, O["n"])]))
    xs = oracle.rav_sweep_sampled(O, P, x0, O["b"], 0.66, sample)
    xg = np_(x)[sample]
    assert np.linalg.norm(xg - xs) <= 1e-12 * np.linalg.norm(xs)


def test_c4_vcycle_converges(rg):
    c = si.CONFIGS["c4"]
    mg, fine = rg.build_hierarchy(si.config_problem("c4"), c["levels"], "pou")
    x = torch.zeros(fine["n"], dtype=torch.float64, device="cuda")
    x, k, h = mg.solve(x, fine["b"], pre=c["pre"], post=c["post"], omega=c["omega"], rtol=c["rtol"], maxit=100)
    assert h[-1] <= c["rtol"] * h[0]
    assert k <= 40
