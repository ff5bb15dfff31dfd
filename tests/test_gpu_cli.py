"""The command-line driver (python -m paper_2103_10127_b200.solve) end to end."""
import json
import os
import subprocess
import sys

import pytest

pytestmark = pytest.mark.gpu
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def run(*args):
    out = subprocess.run([sys.executable, "-m", "paper_2103_10127_b200.solve", *args], cwd=ROOT,
                         capture_output=True, text=True, timeout=600)
    assert out.returncode == 0, out.stderr[-2000:]
    return json.loads(out.stdout.strip().splitlines()[-1])


@pytest.mark.parametrize("args", [("--config", "c1"),
                                  ("--grid", "64", "--smoother", "mv"),
                                  ("--grid", "32", "--elem", "q1q1", "--kind", "cavity", "--pre", "3", "--post", "3"),
                                  ("--adaptive", "4", "--pre", "3", "--post", "3", "--fgmres"),
                                  ("--grid", "64", "--deterministic")])
def test_cli_solves(args):
    r = run(*args)
    assert r["converged"] and 0.0 < r["avg_reduction_factor"] < 1.0
    assert len(r["residual_history"]) == r["iterations"] + 1
