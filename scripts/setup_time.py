"""Setup time of a BASELINE V-cycle config (generator + factorization + transfers), best of 2."""
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch

import seeded_inputs as si
from paper_2103_10127_b200 import ravgmg as rg

name = sys.argv[1] if len(sys.argv) > 1 else "c4"
c = si.CONFIGS[name]
best = None
for _ in range(int(os.environ.get("RAV_SETUP_REPS", "2"))):
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    mg, fine = rg.build_hierarchy(si.config_problem(name), c["levels"], "pou")
    torch.cuda.synchronize()
    dt = time.perf_counter() - t0
    best = dt if best is None else min(best, dt)
    mg.close()
    del mg, fine
    torch.cuda.empty_cache()
print(f"{name} setup {best:.3f} s")
