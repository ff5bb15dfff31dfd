"""Host logic of the byte-balanced slab partition (dist.layer_weights / partition_balanced; SURVEY
section 8 row e): the per-layer factor bytes equal sum n~_i n_i over the oracle's patches, and
the partition is contiguous, covers every layer, respects min_layers and is no worse than the
count-based split."""
import numpy as np
import pytest

import oracle
import seeded_inputs as si
from paper_2103_10127_b200 import dist as rdist


@pytest.mark.parametrize("prob,weights", [(si.problem(2, (7, 9), si.KIND_MMS), "pou"),
                                          (si.problem(2, (6, 5), si.KIND_CAVITY), "own"),
                                          (si.problem(2, (5, 6), si.KIND_CAVITY), "full"),
                                          (si.problem(3, (3, 4, 5), si.KIND_CAVITY), "pou")])
def test_layer_weights_equal_patch_bytes(prob, weights):
    P = oracle.patches(prob, weights)
    ni = np.diff(P["offs"])
    nres = np.add.reduceat((P["w"] > 0).astype(np.int64), P["offs"][:-1])
    dim = prob["dim"]
    nlast = prob["ncell"][dim - 1] + 1
    per = (ni * nres).reshape(nlast, -1).sum(axis=1)
    assert np.array_equal(rdist.layer_weights(prob, weights), per.astype(np.float64))


@pytest.mark.parametrize("prob,R", [(si.problem(3, (32, 32, 32), 0), 8), (si.problem(2, (2048, 2048), 1), 8),
                                    (si.problem(3, (5, 4, 12), 0), 3), (si.problem(2, (20, 30), 1), 5)])
def test_balanced_partition_properties(prob, R):
    w = rdist.layer_weights(prob)
    part = rdist.partition_balanced(prob, R)
    assert part[0][0] == 0 and part[-1][1] == len(w)
    assert all(a < b and b - a >= 3 for a, b in part)
    assert all(part[r][1] == part[r + 1][0] for r in range(R - 1))
    cnt = rdist.partition_layers(len(w), R)
    worst = lambda p: max(w[a:b].sum() for a, b in p)
    assert worst(part) <= worst(cnt) + 1e-9
