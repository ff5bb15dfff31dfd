"""One V(2,2)-RAV solve on a 2D MMS hierarchy; prints cycles and the final residual ratio
(run with and without RAV_WAVE=1: the pipelined sweeps must not change the iteration)."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import json

import numpy as np
import torch

import seeded_inputs as si
from paper_2103_10127_b200 import ravgmg as rg

n, levels = int(sys.argv[1]), int(sys.argv[2])
mg, fine = rg.build_hierarchy(si.problem(2, (n, n), si.KIND_MMS, eta="fourier"), levels, "pou")
x = torch.zeros(fine["n"], dtype=torch.float64, device="cuda")
x, k, hist = mg.solve(x, fine["b"], pre=2, post=2, omega=0.66, rtol=1e-8, maxit=100)
torch.cuda.synchronize()
np.save(sys.argv[3], x.cpu().numpy())
print(json.dumps({"cycles": int(k), "ratio": float(hist[-1] / hist[0])}))
