"""Command-line driver of the library: one multigrid solve on one GPU, reported as
one JSON line (SURVEY section 5 "metrics / logging": cycles, average reduction
factor rho = (||r_k|| / ||r_0||)^(1/k), setup / per-cycle / total time, DoFs per
level).  Argument marshalling only -- every step runs in libravgmg.

    python -m paper_2103_10127_b200.solve --config c3
    python -m paper_2103_10127_b200.solve --grid 512 --elem q1q1 --kind cavity --smoother mv --pre 3 --post 3
    python -m paper_2103_10127_b200.solve --adaptive 7 --smoother rav --pre 3 --post 3 --fgmres
"""
from __future__ import annotations

import argparse
import json
import math
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)

SMOOTHERS = {   # weights, variant, default omega (R5, R17)
    "rav": ("pou", 0, 0.66),
    "own": ("own", 0, 0.66),
    "av": ("full", 0, 0.1),
    "diag": ("full", 1, 0.1),
    "mv": ("full", 2, 0.66),
}


def main(argv=None) -> int:
    ap = argparse.ArgumentParser(description=__doc__.split("\n")[0])
    ap.add_argument("--config", choices=["c1", "c3", "c4"], help="a BASELINE V-cycle configuration")
    ap.add_argument("--grid", type=int, default=64, help="cells per axis (2D unit square) when no --config")
    ap.add_argument("--dim", type=int, default=2, choices=[2, 3])
    ap.add_argument("--elem", default="q2q1", choices=["q2q1", "q1q1"])
    ap.add_argument("--kind", default="mms", choices=["cavity", "mms"])
    ap.add_argument("--eta", default="fourier", choices=["const", "fourier"])
    ap.add_argument("--levels", type=int, default=0, help="0: down to a 4^d (Q2-Q1) / 8^d (Q1-Q1) coarse grid")
    ap.add_argument("--adaptive", type=int, default=0, help="use the paper's adaptive hierarchy with this many levels")
    ap.add_argument("--smoother", default="rav", choices=sorted(SMOOTHERS))
    ap.add_argument("--pre", type=int, default=2)
    ap.add_argument("--post", type=int, default=2)
    ap.add_argument("--omega", type=float, default=None)
    ap.add_argument("--tol", type=float, default=1e-8)
    ap.add_argument("--max-iters", type=int, default=200)
    ap.add_argument("--fgmres", action="store_true", help="FGMRES(30) with the V-cycle as preconditioner (R19)")
    ap.add_argument("--deterministic", action="store_true", help="bitwise reproducible scatter (R16)")
    ap.add_argument("--pressure", default="pin", choices=["pin", "mean", "none"],
                    help="normalise the solution's pressure (row a10, R4): p(vertex 0) = 0, zero mean, or as is")
    a = ap.parse_args(argv)

    import torch

    import seeded_inputs as si
    from . import ravgmg as rg

    weights, variant, omega0 = SMOOTHERS[a.smoother]
    omega = omega0 if a.omega is None else a.omega
    stream = torch.cuda.Stream()
    torch.cuda.set_stream(stream)
    t0 = time.perf_counter()
    if a.config:
        c = si.CONFIGS[a.config]
        prob = si.config_problem(a.config)
        mg, fine = rg.build_hierarchy(prob, c["levels"], weights, variant=variant, deterministic=a.deterministic)
        desc = a.config
        a.pre, a.post = c["pre"], c["post"]
    elif a.adaptive:
        prob = si.problem(2, (8, 8), si.KIND_CAVITY if a.kind == "cavity" else si.KIND_MMS, eta=a.eta,
                          elem=si.ELEM_Q1Q1)
        w = "own" if weights == "pou" else weights
        mg, fine = rg.build_adaptive_hierarchy(prob, a.adaptive, w, variant=variant, deterministic=a.deterministic)
        desc = f"adaptive Q1-Q1 hierarchy, {a.adaptive} levels (R20)"
    else:
        kind = si.KIND_CAVITY if a.kind == "cavity" else si.KIND_MMS
        elem = si.ELEM_Q1Q1 if a.elem == "q1q1" else si.ELEM_Q2Q1
        prob = si.problem(a.dim, [a.grid] * a.dim, kind, eta=a.eta, elem=elem)
        coarsest = 8 if a.elem == "q1q1" else 4
        levels = a.levels or max(1, int(math.log2(max(a.grid // coarsest, 1))) + 1)
        mg, fine = rg.build_hierarchy(prob, levels, weights, variant=variant, deterministic=a.deterministic)
        desc = f"{a.dim}D {a.grid}^{a.dim} {a.elem}, {a.kind}, eta {a.eta}, {levels} levels"
    torch.cuda.synchronize()
    setup = time.perf_counter() - t0
    x = torch.zeros(fine["n"], dtype=torch.float64, device="cuda")
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(stream)
    if a.fgmres:
        x, k, hist = mg.fgmres(x, fine["b"], pre=a.pre, post=a.post, omega=omega, rtol=a.tol, maxit=a.max_iters)
    else:
        x, k, hist = mg.solve(x, fine["b"], pre=a.pre, post=a.post, omega=omega, rtol=a.tol, maxit=a.max_iters)
    e1.record(stream)
    if a.pressure != "none":
        mg.normalize_pressure(x, mode=0 if a.pressure == "pin" else 1)
    torch.cuda.synchronize()
    t = e0.elapsed_time(e1) / 1e3
    rho = float((hist[-1] / hist[0]) ** (1.0 / max(k, 1))) if hist[0] > 0 else 0.0
    print(json.dumps({"problem": desc, "smoother": a.smoother, "omega": omega, "pre": a.pre, "post": a.post,
                      "krylov": "fgmres(30)" if a.fgmres else None, "pressure": a.pressure, "free_dofs": fine["n"], "iterations": k,
                      "converged": bool(hist[-1] <= a.tol * hist[0]), "avg_reduction_factor": rho,
                      "setup_s": setup, "solve_s": t, "ms_per_iteration": t / max(k, 1) * 1e3,
                      "residual_history": [float(h) for h in hist]}))
    return 0


if __name__ == "__main__":
    sys.exit(main())
