"""Time the residual kernel (rav_residual, CUDA events) on a BASELINE config."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch

import seeded_inputs as si
from paper_2103_10127_b200 import ravgmg as rg

stream = torch.cuda.Stream()
torch.cuda.set_stream(stream)
L = rg.gen_level(si.config_problem(sys.argv[1] if len(sys.argv) > 1 else "c4"), "pou")
sm = rg.Smoother(L, L)
x = torch.tensor(si.initial_guess(L["n"], seed=si.X0_SEED), device="cuda")
r = sm.residual(x, L["b"])
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
for _ in range(5):
    sm.residual(x, L["b"], r)
e0.record(stream)
for _ in range(50):
    sm.residual(x, L["b"], r)
e1.record(stream)
torch.cuda.synchronize()
ms = e0.elapsed_time(e1) / 50
by = sm.sweep_bytes()["residual"]
print(f"residual {ms*1e3:8.1f} us  {by/ms/1e6:8.1f} GB/s  ({by/1e9:.3f} GB)  nnz {L['nnz']}", flush=True)
print("patterns", "n/a")
if len(sys.argv) > 2:
    import numpy as np
    np.save(sys.argv[2], r.cpu().numpy())
