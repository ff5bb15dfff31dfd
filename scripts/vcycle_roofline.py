"""HBM roofline of one V(2,2)-RAV cycle of c3 / c4 (BASELINE metric "V-cycle time to 1e-8"):
the algorithmic bytes every kernel of a cycle must move -- per level the sweep kernel's
(rav_sweep_bytes "sweep") x sweeps, the residual kernel's ("residual") x residual launches,
the stencil transfers' vector reads / writes -- against the measured copy peak, next to the
measured cycle time (mg_vcycle, CUDA events).  Residual launches per level, from the launch list
(profiles/r02_launches_*_vcycle.csv): the finest level 5 (4 sweeps + the restriction's residual),
the coarser smoothed levels 4 (their first sweep reads b: x = 0), and 2 + 2 sweeps everywhere.

    python scripts/vcycle_roofline.py c3 [c4]   ->  one JSON line per config
"""
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch

import seeded_inputs as si
from paper_2103_10127_b200 import ravgmg as rg

peaks = json.load(open(os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "MEASURED_PEAKS.json")))
peak_gbs = None
for k, v in peaks.items():
    if "hbm" in k.lower() and isinstance(v, (int, float)):
        peak_gbs = peak_gbs or float(v)
for name in sys.argv[1:] or ["c3"]:
    c = si.CONFIGS[name]
    probs = [si.config_problem(name)]
    for _ in range(c["levels"] - 1):
        probs.append(rg.coarsen_problem(probs[-1]))
    total, per_level = 0.0, []
    for l, p in enumerate(probs[:-1]):          # smoothed levels, finest first (the coarsest is solved)
        L = rg.gen_level(p, "pou")
        sm = rg.Smoother(L, L)
        by = sm.sweep_bytes()
        nres = 5 if l == 0 else 4
        xfer = 8.0 * L["n"] * 3                 # prolongation (read x_c, read + write x) and restriction, ~
        b = 4 * by["sweep"] + nres * by["residual"] + xfer
        per_level.append({"level": l, "n": L["n"], "sweep_gb": by["sweep"] / 1e9, "residual_gb": by["residual"] / 1e9,
                          "cycle_gb": b / 1e9})
        total += b
        sm.close()
        del sm, L
        torch.cuda.empty_cache()
    mg, fine = rg.build_hierarchy(si.config_problem(name), c["levels"], "pou")
    x = torch.zeros(fine["n"], dtype=torch.float64, device="cuda")
    mg.vcycle(x, fine["b"], c["pre"], c["post"], c["omega"])
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(10):
        mg.vcycle(x, fine["b"], c["pre"], c["post"], c["omega"])
    e1.record()
    torch.cuda.synchronize()
    t = e0.elapsed_time(e1) / 10 * 1e-3
    mg.close()
    out = {"config": name, "cycle_s": t, "algorithmic_gb_per_cycle": total / 1e9,
           "achieved_gbs": total / t / 1e9, "peak_gbs": peak_gbs,
           "frac": (total / t / 1e9) / peak_gbs if peak_gbs else None, "levels": per_level}
    print(json.dumps(out), flush=True)
