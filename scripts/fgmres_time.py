"""FGMRES(30) + V-cycle time to 1e-8 on a BASELINE config (CUDA events, best of 2)."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch

import seeded_inputs as si
from paper_2103_10127_b200 import ravgmg as rg

name = sys.argv[1] if len(sys.argv) > 1 else "c3"
c = si.CONFIGS[name]
stream = torch.cuda.Stream()
torch.cuda.set_stream(stream)
mg, fine = rg.build_hierarchy(si.config_problem(name), c["levels"], "pou")
best = None
for _ in range(3):
    x = torch.zeros(fine["n"], dtype=torch.float64, device="cuda")
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(stream)
    x, k, hist = mg.fgmres(x, fine["b"], pre=c["pre"], post=c["post"], omega=c["omega"], rtol=c["rtol"], maxit=100)
    e1.record(stream)
    torch.cuda.synchronize()
    t = e0.elapsed_time(e1)
    best = t if best is None else min(best, t)
print(f"{name} fgmres {k} applications, {best:.1f} ms, final ratio {hist[-1] / hist[0]:.2e}")
