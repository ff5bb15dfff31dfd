"""BASELINE config 4 (3D 32^3 Q2-Q1 lid-driven cavity, seeded viscosity) on the
GPU: generator parity, a sampled-DoF sweep against the oracle (which factorizes
only the patches it needs) checked entry by entry, the 3D warp-per-patch sweep
kernel (the kernel c4's finest level runs: >= 2048 patches) against the oracle
through 1/2/10/100 sweeps, and V-cycle iteration-count parity with the oracle at
16^3 (4 levels) and at full size 32^3 (5 levels, 2^3 coarsest; reading R14)."""
import numpy as np
import pytest
import torch

import oracle
import seeded_inputs as si
from _parity import SweepChecker, assert_entrywise, iterate_tol

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
    xs, ms = oracle.rav_sweep_sampled(O, P, x0, O["b"], 0.66, sample, with_magnitude=True)
    assert_entrywise(np_(x)[sample], xs, ms, what="c4 sampled sweep")


@pytest.mark.parametrize("weights", ["pou", "own"])
def test_3d_warp_kernel_sweeps_match_oracle(rg, weights):
    """14 x 13 x 12 cells: 15 x 14 x 13 = 2,730 patches, above the 2,048 at which the
    per-patch warp kernel (schur_sweep_warp_kernel, c4's finest-level sweep) replaces the
    CTA-per-patch kernel; ragged in every axis."""
    prob = si.problem(3, (14, 13, 12), si.KIND_CAVITY, eta="fourier")
    G = rg.gen_level(prob, weights)
    sm = rg.Smoother(G, G)
    assert "warp" in sm.kernel_name, sm.kernel_name
    O = oracle.assemble(prob)
    P = oracle.patches(prob, weights)
    F = oracle.factor(O, P, oracle.FMT_ROWS)
    x0 = si.initial_guess(O["n"], seed=23)
    x = torch.tensor(x0, device="cuda")

    def gpu(k):
        sm.smooth(x, G["b"], k, 0.66)
        return np_(x)

    SweepChecker(O, P, F, O["b"], 0.66).run(x0, gpu, (1, 2, 10, 100), what=sm.kernel_name)


@pytest.mark.parametrize("n,levels", [(16, 4), (32, 5)])
def test_c4_family_cycle_counts_match_oracle(rg, n, levels):
    """Identical V(2,2)-RAV iteration counts (P:132 stopping rule, R11) and residual
    histories at 16^3 and at c4's full size 32^3 (the oracle factors 35,937 376 x 376
    patches, ~9 GB of rows, on the host)."""
    c = si.CONFIGS["c4"]
    prob = si.problem(3, (n, n, n), si.KIND_CAVITY, eta="fourier")
    mg, fine = rg.build_hierarchy(prob, levels, "pou")
    x = torch.zeros(fine["n"], dtype=torch.float64, device="cuda")
    x, kg, hg = mg.solve(x, fine["b"], pre=c["pre"], post=c["post"], omega=c["omega"], rtol=c["rtol"], maxit=100)
    xg = np_(x)
    mg.close()
    H = oracle.Hierarchy(prob, levels, "rav")
    xo, ko, ho = H.solve(rtol=c["rtol"], omega=c["omega"], pre=c["pre"], post=c["post"], maxit=100)
    assert kg == ko, (kg, ko)
    np.testing.assert_allclose(hg, ho, rtol=1e-6, atol=1e-12 * ho[0])
    assert_entrywise(xg, xo, np.abs(xo).max(), tol=iterate_tol(n), what=f"{n}^3 V-cycle iterate")


def test_c4_vcycle_converges(rg):
    c = si.CONFIGS["c4"]
    mg, fine = rg.build_hierarchy(si.config_problem("c4"), c["levels"], "pou")
    x = torch.zeros(fine["n"], dtype=torch.float64, device="cuda")
    x, k, h = mg.solve(x, fine["b"], pre=c["pre"], post=c["post"], omega=c["omega"], rtol=c["rtol"], maxit=100)
    assert h[-1] <= c["rtol"] * h[0]
    assert k <= 40
