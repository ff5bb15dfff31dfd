"""Depth versus resolution on the c3 family (VERDICT r01 "what's weak" 4): V(2,2)-RAV cycle
counts to 1e-8 (P:132 stopping rule, R11) for 64^2 ... 2048^2 with
  (a) the c3 hierarchy shape: 4^2 coarsest grid, so the depth grows with the resolution;
  (b) a 16^2 coarsest grid (two levels fewer at every resolution);
  (c) fixed resolution (256^2, 1024^2), depth varied: coarsest 16^2, 8^2, 4^2
(the direct coarse solve takes at most 6000 DoFs, i.e. 16^2 at most, so a fixed depth over the
whole family is not possible); all with the seeded variable viscosity (R12) and with eta = 1.
GPU (mg_solve) for every case; the oracle's count beside it where it finishes in seconds
(n <= 256).  Writes one JSON file (argv[1]).

    python scripts/depth_study.py profiles/r02_depth_study.json
"""
import json
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch

import oracle
import seeded_inputs as si
from paper_2103_10127_b200 import ravgmg as rg

C = si.CONFIGS["c3"]
OUT = sys.argv[1] if len(sys.argv) > 1 else "depth_study.json"
rows = []


def gpu(prob, levels):
    mg, fine = rg.build_hierarchy(prob, levels, "pou")
    x = torch.zeros(fine["n"], dtype=torch.float64, device="cuda")
    x, k, h = mg.solve(x, fine["b"], pre=C["pre"], post=C["post"], omega=C["omega"], rtol=C["rtol"], maxit=100)
    mg.close()
    del mg, x
    torch.cuda.empty_cache()
    return k, float((h[-1] / h[0]) ** (1.0 / max(k, 1))), [float(v / h[0]) for v in h]


def ora(prob, levels):
    H = oracle.Hierarchy(prob, levels, "rav")
    _, k, _ = H.solve(rtol=C["rtol"], omega=C["omega"], pre=C["pre"], post=C["post"], maxit=100)
    return k


cases = [(n, c) for n in (64, 128, 256, 512, 1024, 2048) for c in (4, 16)] + [(256, 8), (1024, 8)]
for eta in ("fourier", "const"):
    for n, coarse in cases:
        for _ in (0,):
            levels = int(np.log2(n // coarse)) + 1
            shape = f"coarsest {coarse}^2"
            prob = si.problem(2, (n, n), si.KIND_MMS, eta=eta)
            k, rho, hist = gpu(prob, levels)
            row = {"eta": eta, "n": n, "shape": shape, "levels": levels, "coarsest": n >> (levels - 1),
                   "gpu_cycles": k, "gpu_rho": rho, "gpu_rho_first5": hist[min(5, k)] ** (1.0 / min(5, k)),
                   "gpu_rel_hist": hist}
            if n <= 256:
                t0 = time.perf_counter()
                row["oracle_cycles"] = ora(prob, levels)
                row["oracle_s"] = time.perf_counter() - t0
            rows.append(row)
            print(json.dumps(row), flush=True)

with open(OUT, "w") as f:
    json.dump({"what": __doc__.strip().splitlines()[0], "config": "c3 family: 2D Q2-Q1 MMS (R13), "
               "V(2,2)-RAV omega 0.66, x0 = 0, rtol 1e-8", "rows": rows}, f, indent=1)
