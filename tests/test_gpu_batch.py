"""rav_smooth_batch: independent problems in host buffers, copies overlapped with the sweeps of
the neighbouring problems (two device staging pairs, a copy stream).  Each problem's result must
be rav_smooth's on it -- bitwise in deterministic mode (fixed scatter order) -- whatever its slot,
for 1, 2 and an odd number of problems, pinned and pageable host memory, shared and distinct
right-hand sides; and the oracle's within the sweep bar."""
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


@pytest.fixture(scope="module")
def level(rg):
    prob = si.problem(2, (40, 36), si.KIND_MMS, eta="fourier")
    return prob, rg.gen_level(prob, "pou")


@pytest.mark.parametrize("nprob", [1, 2, 5])
@pytest.mark.parametrize("pinned", [True, False], ids=["pinned", "pageable"])
def test_batch_equals_single_smooth(rg, level, nprob, pinned):
    prob, G = level
    n = G["n"]
    stream = torch.cuda.Stream()
    sm = rg.Smoother(G, G, deterministic=True, stream=stream)
    b0 = G["b"].cpu()
    xs0 = [torch.tensor(si.initial_guess(n, seed=100 + k)) for k in range(nprob)]
    bs0 = [b0 if k % 2 == 0 else b0 + torch.tensor(si.initial_guess(n, seed=200 + k)) for k in range(nprob)]
    ref = []
    for k in range(nprob):   # rav_smooth on device buffers, one problem at a time
        x = xs0[k].cuda()
        sm.smooth(x, bs0[k].cuda(), 3, 0.66)
        torch.cuda.synchronize()
        ref.append(x.cpu().numpy())
    xs = [x.clone().pin_memory() if pinned else x.clone() for x in xs0]
    bs = [b.clone().pin_memory() if pinned else b.clone() for b in bs0]
    sm.smooth_batch(xs, bs, 3, 0.66)
    for k in range(nprob):
        assert np.array_equal(xs[k].numpy().view(np.int64), ref[k].view(np.int64)), k
    sm.smooth_batch(xs, bs, 3, 0.66)   # graph replay on the same buffers: 6 sweeps in total
    O = oracle.assemble(prob)
    P = oracle.patches(prob, "pou")
    F = oracle.factor(O, P, oracle.FMT_ROWS)
    for k in (0, nprob - 1):
        xo = oracle.additive_sweeps(O, P, F, xs0[k].numpy(), bs0[k].numpy(), 0.66, 6)
        assert_entrywise(xs[k].numpy(), xo, np.abs(xo).max(), what=f"problem {k} after 6 sweeps")
    sm.close()


def test_batch_rejects_device_pointers(rg, level):
    _, G = level
    sm = rg.Smoother(G, G, stream=torch.cuda.Stream())
    x = torch.zeros(G["n"], dtype=torch.float64, device="cuda")
    with pytest.raises(rg.RavError):
        sm.smooth_batch([x], [G["b"]], 1, 0.66)
    sm.close()
