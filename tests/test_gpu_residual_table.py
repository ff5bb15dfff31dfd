"""The residual's B-value table (nb.cu nb_compress_bvals; DESIGN 5.1), the sweep-stream
prefetch hint (Factors.lead, RAV_XPF_MB), the thread sweep's per-pattern weight table
(Factors.wtab, RAV_SCHUR_WTAB) and MV's colour residuals by the node-blocked kernel (RAV_MV_NB)
change which bytes the kernels stream, not what they compute: the residual with the B / B^T
values read from the table must equal, bit for bit, the residual with the values streamed
(RAV_NB_BVALS=0), and the streamed bytes must drop by the B values; sweeps after residuals that
prefetch the sweep's factors, and sweeps with the weight table, must equal the plain sweeps bit
for bit (deterministic mode, so the scatter order is fixed); MV's two colour-residual paths
agree to rounding.

The switches are read once per process, so each setting runs in its own Python process; the
seeded inputs and the comparison stay here.  2D (pair layout, one lane per row) and 3D (two
lanes per row) fine-level sizes plus a coarse size (full-warp rows).
"""
import os
import subprocess
import sys

import numpy as np
import pytest

pytestmark = pytest.mark.gpu

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))

CHILD = r"""
import sys, numpy as np, torch
sys.path.insert(0, {root!r})
import seeded_inputs as si
from paper_2103_10127_b200 import ravgmg as rg
out = {{}}
for name, prob in (("2d", si.problem(2, (203, 190), si.KIND_MMS, eta="fourier")),
                   ("2d_small", si.problem(2, (24, 20), si.KIND_MMS, eta="fourier")),
                   ("3d", si.problem(3, (14, 12, 13), si.KIND_CAVITY, eta="fourier"))):
    L = rg.gen_level(prob, "pou")
    sm = rg.Smoother(L, L, deterministic=True)
    x = torch.tensor(si.initial_guess(L["n"], seed=si.X0_SEED), device="cuda")
    r = sm.residual(x, L["b"])
    sm.smooth(x, L["b"], 3, 0.66)
    torch.cuda.synchronize()
    out[name + "_r"] = r.cpu().numpy()
    out[name + "_x"] = x.cpu().numpy()
    out[name + "_bytes"] = np.array([sm.sweep_bytes()["residual"]])
np.savez({path!r}, **out)
"""


def _run(tmp_path, tag, env):
    path = str(tmp_path / f"{tag}.npz")
    e = dict(os.environ)
    e.update(env)
    subprocess.run([sys.executable, "-c", CHILD.format(root=ROOT, path=path)], env=e, check=True, timeout=600)
    return np.load(path)


def test_bvalue_table_bitwise_equal_and_fewer_bytes(tmp_path):
    on = _run(tmp_path, "on", {"RAV_NB_BVALS": "1", "RAV_XPF_MB": "0"})
    off = _run(tmp_path, "off", {"RAV_NB_BVALS": "0", "RAV_XPF_MB": "0"})
    for name in ("2d", "2d_small", "3d"):
        assert np.array_equal(on[name + "_r"].view(np.int64), off[name + "_r"].view(np.int64)), name
        assert np.array_equal(on[name + "_x"].view(np.int64), off[name + "_x"].view(np.int64)), name
        # the B / B^T values leave the stream: the 2D / 3D fine levels stream well under 3/4 of the bytes
        ratio = float(on[name + "_bytes"][0]) / float(off[name + "_bytes"][0])
        assert ratio < (0.75 if name != "2d_small" else 1.0), (name, ratio)


def test_sweep_prefetch_hint_bitwise_equal(tmp_path):
    on = _run(tmp_path, "pf", {"RAV_XPF_MB": "48"})
    off = _run(tmp_path, "nopf", {"RAV_XPF_MB": "0"})
    for name in ("2d", "2d_small", "3d"):
        assert np.array_equal(on[name + "_x"].view(np.int64), off[name + "_x"].view(np.int64)), name


def test_sweep_weight_table_bitwise_equal(tmp_path):
    """Per-pattern PoU weights (verified bitwise at setup) give the sweeps of the streamed AUX
    weights bit for bit, and stream fewer bytes."""
    on = _run(tmp_path, "wt", {"RAV_SCHUR_WTAB": "1"})
    off = _run(tmp_path, "nowt", {"RAV_SCHUR_WTAB": "0"})
    for name in ("2d", "2d_small", "3d"):
        assert np.array_equal(on[name + "_x"].view(np.int64), off[name + "_x"].view(np.int64)), name


MV_CHILD = r"""
import sys, numpy as np, torch
sys.path.insert(0, {root!r})
import seeded_inputs as si
from paper_2103_10127_b200 import ravgmg as rg
prob = si.problem(2, (64, 72), si.KIND_MMS, eta="fourier")
G = rg.gen_level(prob, "full")
sm = rg.Smoother(G, G, variant=rg.VARIANT_MV)
offs, ids = rg.multicolor(prob)
sm.set_colors(offs, ids)
x = torch.tensor(si.initial_guess(G["n"], seed=5), device="cuda")
sm.smooth(x, G["b"], 3, 0.66)
torch.cuda.synchronize()
np.save({path!r}, x.cpu().numpy())
"""


def test_mv_colour_residual_paths_agree(tmp_path):
    """MV's colour residual from the node-blocked kernel (default) and from the patch rows of L
    (RAV_MV_NB=0) are the same fresh local residuals (same-colour patches are uncoupled through
    L), so 3 MV sweeps agree to rounding."""
    out = []
    for v in ("1", "0"):
        path = str(tmp_path / f"mv{v}.npy")
        e = dict(os.environ)
        e["RAV_MV_NB"] = v
        subprocess.run([sys.executable, "-c", MV_CHILD.format(root=ROOT, path=path)], env=e, check=True, timeout=600)
        out.append(np.load(path))
    scale = np.abs(out[1]).max()
    assert np.abs(out[0] - out[1]).max() <= 1e-12 * scale
