"""CPU checks of the element-wise parity bound (tests/_parity.py): the two
independent computations of mag_j (numpy over the oracle's weighted rows, C in the
sampled oracle sweep) agree, and mag_j bounds the sweep's own update."""
import numpy as np

import oracle
import seeded_inputs as si
from _parity import sweep_magnitude


def test_magnitude_bounds_update_and_matches_sampled_oracle():
    prob = si.problem(2, (9, 7), si.KIND_MMS, eta="fourier")
    A = oracle.assemble(prob)
    P = oracle.patches(prob, "pou")
    F = oracle.factor(A, P, oracle.FMT_ROWS)
    x0 = si.initial_guess(A["n"], seed=3)
    mag = sweep_magnitude(A, P, F, x0, A["b"], 0.66)
    x1 = oracle.additive_sweeps(A, P, F, x0, A["b"], 0.66, 1)
    assert np.all(np.abs(x1) <= mag * (1 + 1e-12))
    sample = np.arange(0, A["n"], 7)
    xs, ms = oracle.rav_sweep_sampled(A, P, x0, A["b"], 0.66, sample, with_magnitude=True)
    np.testing.assert_allclose(xs, x1[sample], rtol=1e-11, atol=1e-12 * np.abs(x1).max())
    np.testing.assert_allclose(ms, mag[sample], rtol=1e-9)
