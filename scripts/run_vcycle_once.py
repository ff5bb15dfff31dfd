"""One timed mg_solve on a BASELINE V-cycle config (for ncu launch lists)."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch

import seeded_inputs as si
from paper_2103_10127_b200 import ravgmg as rg

name = sys.argv[1] if len(sys.argv) > 1 else "c4"
c = si.CONFIGS[name]
stream = torch.cuda.Stream()
torch.cuda.set_stream(stream)
mg, fine = rg.build_hierarchy(si.config_problem(name), c["levels"], "pou")
x = torch.zeros(fine["n"], dtype=torch.float64, device="cuda")
mg.solve(x, fine["b"], pre=c["pre"], post=c["post"], omega=c["omega"], rtol=c["rtol"], maxit=3)
x.zero_()
torch.cuda.synchronize()
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
e0.record(stream)
_, k, h = mg.solve(x, fine["b"], pre=c["pre"], post=c["post"], omega=c["omega"], rtol=c["rtol"], maxit=int(sys.argv[2]) if len(sys.argv) > 2 else 100)
e1.record(stream)
torch.cuda.synchronize()
print(name, "cycles", k, "ms", e0.elapsed_time(e1))
