"""The band-pipelined sweep chain (csrc/wave.cu, opt-in RAV_WAVE=1) against the default chain.

The pipelined kernels compute the same residual and RAV update; only the order of the
atomic PoU additions differs, as between any two runs of the default chain.  Bars: 20
sweeps on a 512^2 grid (the level size where the chain is used) agree to 1e-13
relative; a V(2,2) solve with a 512^2 finest level (first sweep of each cycle reusing
the stopping test's residual) takes the same number of cycles and agrees to 1e-10.
The environment is read once per process, so each side runs in its own process.
"""
import json
import os
import subprocess
import sys

import numpy as np
import pytest

pytestmark = pytest.mark.gpu
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _run(args, wave, tmp_path, tag, spatial=False):
    env = dict(os.environ)
    env.pop("RAV_WAVE", None)
    env.pop("RAV_WAVE_SPATIAL", None)
    if wave:
        env["RAV_WAVE"] = "1"
    if spatial:
        env["RAV_WAVE_SPATIAL"] = "1"
    out = str(tmp_path / f"{tag}.npy")
    res = subprocess.run([sys.executable] + args + [out], cwd=ROOT, env=env, capture_output=True, text=True,
                         timeout=300)
    assert res.returncode == 0, res.stderr[-2000:]
    return np.load(out), res.stdout


@pytest.mark.parametrize("spatial", [False, True], ids=["slot_order", "spatial_order"])
def test_wave_sweeps_match_default_chain(tmp_path, spatial):
    a, _ = _run(["scripts/wave_check.py", "512", "20"], False, tmp_path, "ref")
    b, _ = _run(["scripts/wave_check.py", "512", "20"], True, tmp_path, "wave", spatial=spatial)
    assert np.abs(a - b).max() <= 1e-13 * np.abs(a).max()


def test_wave_vcycle_matches_default_chain(tmp_path):
    a, oa = _run(["scripts/wave_vcycle.py", "512", "8"], False, tmp_path, "ref")
    b, ob = _run(["scripts/wave_vcycle.py", "512", "8"], True, tmp_path, "wave")
    ra, rb = json.loads(oa.strip().splitlines()[-1]), json.loads(ob.strip().splitlines()[-1])
    assert ra["cycles"] == rb["cycles"]
    assert np.abs(a - b).max() <= 1e-10 * np.abs(a).max()
