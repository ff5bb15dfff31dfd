"""Deterministic scatter mode (rav_opts.deterministic; reading R16): every
correction goes to its own slot and a second kernel adds them per DoF in
ascending patch order.  Repeated runs must agree bit for bit (the atomic mode
may differ in the last bits), match the oracle to 1e-12 and give the same
V-cycle iteration counts."""
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


PROBLEMS = [si.problem(2, (40, 36), si.KIND_MMS, eta="fourier"),                       # 2D thread layout
            si.problem(2, (12, 10), si.KIND_CAVITY, eta="fourier", elem=si.ELEM_Q1Q1),
            si.problem(3, (6, 5, 4), si.KIND_CAVITY, eta="fourier"),                     # 3D CTA-per-patch
            si.problem(3, (16, 12, 12), si.KIND_CAVITY, eta="fourier")]                  # 3D warp kernel


@pytest.mark.parametrize("prob", PROBLEMS, ids=["2d-q2q1", "2d-q1q1", "3d-small", "3d-warp"])
def test_deterministic_sweeps_are_bitwise_reproducible_and_match_oracle(rg, prob):
    G = rg.gen_level(prob, "pou")
    sm = rg.Smoother(G, G, deterministic=True)
    x0 = si.initial_guess(G["n"], seed=31)
    runs = []
    for _ in range(3):
        x = torch.tensor(x0, device="cuda")
        sm.smooth(x, G["b"], 4, 0.66)
        torch.cuda.synchronize()
        runs.append(x.cpu().numpy())
    for r in runs[1:]:
        assert np.array_equal(r, runs[0])
    O = oracle.assemble(prob)
    P = oracle.patches(prob, "pou")
    F = oracle.factor(O, P, oracle.FMT_ROWS)
    xd = torch.tensor(x0, device="cuda")

    def gpu(k):
        sm.smooth(xd, G["b"], k, 0.66)
        return xd.cpu().numpy()

    SweepChecker(O, P, F, O["b"], 0.66).run(x0, gpu, (1, 4), what="deterministic " + sm.kernel_name)
    sa = rg.Smoother(G, G)
    xa = torch.tensor(x0, device="cuda")
    sa.smooth(xa, G["b"], 4, 0.66)
    assert np.abs(xa.cpu().numpy() - runs[0]).max() <= 1e-13 * np.abs(runs[0]).max()


def test_deterministic_vcycle_same_counts(rg):
    prob = si.problem(2, (64, 64), si.KIND_MMS, eta="fourier")
    H = oracle.Hierarchy(prob, 5)
    _, ko, _ = H.solve(rtol=1e-10, omega=0.66)
    res = []
    for _ in range(2):
        mg, fine = rg.build_hierarchy(prob, 5, "pou", deterministic=True)
        x = torch.zeros(fine["n"], dtype=torch.float64, device="cuda")
        _, k, h = mg.solve(x, fine["b"], rtol=1e-10, omega=0.66)
        assert k == ko
        res.append((x.cpu().numpy(), h))
    assert np.array_equal(res[0][0], res[1][0]) and np.array_equal(res[0][1], res[1][1])


def test_deterministic_mode_rejects_generic_formats(rg):
    prob = si.problem(2, (6, 6), si.KIND_CAVITY)
    G = rg.gen_level(prob, "pou")
    with pytest.raises(rg.RavError):
        rg.Smoother(G, G, kernel=rg.KERNEL_WARP, deterministic=True)
