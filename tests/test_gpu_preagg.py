"""The thread sweep's pre-aggregated scatter (schur.cu PA, RAV_SCHUR_PA; DESIGN 5.1): lanes of a
chunk hold x-neighbouring patches, and a lane adds its right neighbour's correction for a shared
node to its own before the atomic.  That changes the summation order only, so the sweep with it
on and the sweep with the plain scatter must both equal the oracle's sweep (Eq. 13) entry by
entry within the rounding bound of tests/_parity.py, after 1 and after 5 sweeps.  The grid's vertex
rows (91, 131) are no multiple of the 32-patch chunk, so chunks wrap grid rows and boundary
patterns (fewer restricted nodes, other slot orders) sit next to interior ones inside a warp.

The switch is read once per process: each setting runs in its own Python process."""
import os
import subprocess
import sys

import numpy as np
import pytest

import oracle
import seeded_inputs as si
from _parity import assert_entrywise, sweep_magnitude

pytestmark = pytest.mark.gpu

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
SIZES = {"a": (90, 70), "b": (130, 33)}
OMEGA = 0.66

CHILD = r"""
import sys, numpy as np, torch
sys.path.insert(0, {root!r})
import seeded_inputs as si
from paper_2103_10127_b200 import ravgmg as rg
out = {{}}
for name, n in {sizes!r}.items():
    prob = si.problem(2, n, si.KIND_MMS, eta="fourier")
    L = rg.gen_level(prob, "pou")
    sm = rg.Smoother(L, L)
    assert "thread" in sm.kernel_name, sm.kernel_name
    x = torch.tensor(si.initial_guess(L["n"], seed=si.X0_SEED), device="cuda")
    sm.smooth(x, L["b"], 1, {omega})
    torch.cuda.synchronize()
    out[name + "_1"] = x.cpu().numpy()
    sm.smooth(x, L["b"], 4, {omega})
    torch.cuda.synchronize()
    out[name + "_5"] = x.cpu().numpy()
np.savez({path!r}, **out)
"""


def _run(tmp_path, tag, env):
    path = str(tmp_path / f"{tag}.npz")
    e = dict(os.environ)
    e.update(env)
    subprocess.run([sys.executable, "-c", CHILD.format(root=ROOT, path=path, sizes=SIZES, omega=OMEGA)],
                   env=e, check=True, timeout=600)
    return np.load(path)


def test_preaggregated_and_plain_scatter_match_the_oracle(tmp_path):
    on = _run(tmp_path, "pa", {"RAV_SCHUR_PA": "1"})
    off = _run(tmp_path, "plain", {"RAV_SCHUR_PA": "0"})
    for name, n in SIZES.items():
        prob = si.problem(2, n, si.KIND_MMS, eta="fourier")
        A = oracle.assemble(prob)
        P = oracle.patches(prob, "pou")
        F = oracle.factor(A, P, oracle.FMT_ROWS)
        x0 = si.initial_guess(A["n"], seed=si.X0_SEED)
        mag1 = sweep_magnitude(A, P, F, x0, A["b"], OMEGA)
        x1 = oracle.additive_sweeps(A, P, F, x0, A["b"], OMEGA, 1)
        scale5 = mag1.max()
        xk = x1
        for _ in range(4):
            scale5 = max(scale5, sweep_magnitude(A, P, F, xk, A["b"], OMEGA).max())
            xk = oracle.additive_sweeps(A, P, F, xk, A["b"], OMEGA, 1)
        for tag, got in (("pre-aggregated", on), ("plain", off)):
            assert_entrywise(got[name + "_1"], x1, mag1, what=f"{tag} scatter, {n}, 1 sweep")
            assert_entrywise(got[name + "_5"], xk, scale5, what=f"{tag} scatter, {n}, 5 sweeps")
        # the two scatters against each other, entry by entry at the same bar
        assert_entrywise(on[name + "_1"], off[name + "_1"], mag1, what=f"pre-aggregated vs plain, {n}")
