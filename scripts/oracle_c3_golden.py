"""Write tests/golden/c3_oracle_vcycle.json: the ORACLE's V(2,2)-RAV solve of BASELINE config c3
(2048^2 Q2-Q1 MMS, seeded viscosity, 10 levels, omega 0.66, x0 = 0, relative residual 1e-8,
P:132 stopping rule) -- cycle count, residual history and the final iterate at seeded sampled DoFs.
Calls only oracle/ and the seeded input generators (no GPU, no product code); needs ~40 GB of
host memory and a few minutes of the GPU box's host cores (OpenMP oracle sweeps).

    python scripts/oracle_c3_golden.py [out.json]
"""
import json
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np

import oracle
import seeded_inputs as si

out = sys.argv[1] if len(sys.argv) > 1 else os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))),
                                                          "tests", "golden", "c3_oracle_vcycle.json")
c = si.CONFIGS["c3"]
prob = si.config_problem("c3")
t0 = time.time()
H = oracle.Hierarchy(prob, c["levels"], "rav")
t1 = time.time()
x, k, hist = H.solve(rtol=c["rtol"], omega=c["omega"], pre=c["pre"], post=c["post"], maxit=100)
t2 = time.time()
rng = np.random.default_rng(20260)
sample = np.sort(rng.choice(len(x), size=4096, replace=False))
json.dump({"config": "c3: " + json.dumps({k_: v for k_, v in c.items() if k_ != "ncell"}) + ", ncell 2048 x 2048",
           "source": "scripts/oracle_c3_golden.py (oracle.Hierarchy + Hierarchy.solve only)",
           "n": int(len(x)), "cycles": int(k), "history": [float(v) for v in hist],
           "sample_dofs": [int(i) for i in sample], "sample_x": [float(x[i]) for i in sample],
           "x_absmax": float(np.abs(x).max()), "setup_s": t1 - t0, "solve_s": t2 - t1,
           "host_threads": os.cpu_count()}, open(out, "w"), indent=0)
print(f"c3 oracle: {k} cycles, setup {t1 - t0:.1f} s, solve {t2 - t1:.1f} s -> {out}")
