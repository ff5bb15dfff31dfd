"""Row a10: pressure normalisation after a solve (reading R4; config c1
"pressure pinned at one corner vertex").  The operators keep every pressure DoF and
the constant is fixed only inside the coarsest solve, so the fine-level pressure of
an iterate carries an arbitrary constant; mg_normalize_pressure / rav_pressure_normalize
remove it: mode 0 p <- p - p(vertex 0) (the oracle's pressure_shift), mode 1
p <- p - mean(p)."""
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


def test_c1_normalized_pressure_matches_oracle(rg):
    c = si.CONFIGS["c1"]
    prob = si.problem(2, c["ncell"], c["kind"], eta=c["eta"])
    H = oracle.Hierarchy(prob, c["levels"], "rav")
    xo, ko, _ = H.solve(rtol=c["rtol"], omega=c["omega"], pre=c["pre"], post=c["post"])
    xo = oracle.pressure_shift(H.fine, xo)
    mg, fine = rg.build_hierarchy(prob, c["levels"], "pou")
    x = torch.zeros(fine["n"], dtype=torch.float64, device="cuda")
    x, kg, _ = mg.solve(x, fine["b"], pre=c["pre"], post=c["post"], omega=c["omega"], rtol=c["rtol"])
    assert kg == ko
    x += 0.37 * (torch.arange(fine["n"], device="cuda") >= fine["nvel"])    # any pressure constant
    mg.normalize_pressure(x, mode=0)
    xg = x.cpu().numpy()
    assert xg[fine["nvel"]] == 0.0
    assert_entrywise(xg, xo, np.abs(xo).max(), tol=1e-9, what="c1 normalized solution")


@pytest.mark.parametrize("n_vel,n", [(0, 1), (10, 10 + 4097), (1000, 1000 + 300000)])
def test_pressure_normalize_modes(rg, n_vel, n):
    v = si.random_vector(n, 41)
    x = torch.tensor(v, device="cuda")
    rg.pressure_normalize(x, n_vel, mode=1)
    p = v[n_vel:] - np.sum(v[n_vel:]) / (n - n_vel)
    got = x.cpu().numpy()
    assert np.array_equal(got[:n_vel], v[:n_vel])
    assert np.abs(got[n_vel:] - p).max() <= 1e-13 * np.abs(v).max()
    assert abs(got[n_vel:].mean()) <= 1e-13 * np.abs(v).max()
    x = torch.tensor(v, device="cuda")
    pin = n_vel + (n - n_vel) // 2
    rg.pressure_normalize(x, n_vel, mode=0, pin=pin)
    got = x.cpu().numpy()
    assert np.array_equal(got[:n_vel], v[:n_vel])
    assert np.array_equal(got[n_vel:], v[n_vel:] - v[pin])


def test_pressure_normalize_rejects_bad_arguments(rg):
    x = torch.zeros(10, dtype=torch.float64, device="cuda")
    with pytest.raises(rg.RavError):
        rg.pressure_normalize(x, 4, mode=0, pin=2)      # pin inside the velocity block
    with pytest.raises(rg.RavError):
        rg.pressure_normalize(x, 4, mode=2)
