"""Slab-partitioned V-cycle on the GPU (SURVEY section 8 rows a9 / e).

R ranks are emulated as R threads of this process on the one available GPU
(dist.ThreadComm: host-side rendezvous only, no kernel ever waits on another
rank).  Every rank generates its windows of the partitioned levels with
rav_gen_*, builds its smoothers, its windowed transfers (rav_gen_prolongation
with windows + rav_xfer_setup) and the agglomerated coarse hierarchy
(mg_setup), and runs dist.DistVCycle through the C-ABI.  The iteration count
must equal the oracle's single-domain V-cycle and the assembled solution must
match it to 1e-10 relative."""
import numpy as np
import pytest
import torch

import oracle
import seeded_inputs as si
from _parity import assert_entrywise

pytestmark = pytest.mark.gpu


def run(prob, n_levels, world, rtol=1e-10, agg_layers=0, maxit=60):
    from paper_2103_10127_b200 import dist as rdist
    hub = rdist.ThreadComm.Hub(world)

    def rank_fn(r):
        torch.cuda.set_device(0)
        comm = rdist.ThreadComm(hub, r, sync=torch.cuda.synchronize)
        cyc, levels = rdist.build_gpu_cycle(prob, n_levels, world, r, comm, agg_layers=agg_layers)
        x = levels[0]["x"]
        _, k, hist = cyc.solve(x, levels[0]["b"], rtol=rtol, omega=0.66, maxit=maxit)
        torch.cuda.synchronize()
        s = levels[0]["slab"]
        own = s.owned_mask()
        return s.global_ids()[own], x.cpu().numpy()[own], k, hist, len(levels)

    return rdist.run_threads(world, rank_fn)


CASES = [
    (si.problem(2, (32, 32), si.KIND_MMS, eta="fourier"), 4, 2, 0),
    (si.problem(2, (24, 48), si.KIND_CAVITY, eta="fourier", box=[1.0, 2.0]), 4, 3, 0),
    (si.problem(2, (32, 64), si.KIND_MMS, eta="fourier", box=[1.0, 2.0]), 5, 4, 4),
    (si.problem(3, (4, 4, 8), si.KIND_CAVITY, eta="fourier", box=[1.0, 1.0, 2.0]), 2, 2, 0),
]


@pytest.mark.parametrize("case", CASES, ids=["2d-mms-w2", "2d-cavity-w3", "2d-mms-w4-agg4", "3d-cavity-w2"])
def test_distributed_vcycle_matches_oracle(case):
    prob, n_levels, world, agg = case
    res = run(prob, n_levels, world, agg_layers=agg)
    H = oracle.Hierarchy(prob, n_levels)
    xo, ko, ho = H.solve(rtol=1e-10, omega=0.66, maxit=60)
    assert ko < 60
    xd = np.full(H.fine["n"], np.nan)
    for g, v, k, hist, K in res:
        assert k == ko, f"distributed cycles {k} != oracle {ko}"
        np.testing.assert_allclose(hist, ho, rtol=1e-8, atol=1e-12 * ho[0])
        xd[g] = v
    assert not np.isnan(xd).any()
    assert_entrywise(xd, xo, np.abs(xo).max(), tol=1e-10)
    assert max(r[4] for r in res) >= 1
