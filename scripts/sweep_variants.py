"""Time the RAV sweep kernel (rav_apply alone, CUDA events) on a BASELINE config
for the current build / environment (e.g. RAV_SCHUR_PF)."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch

import seeded_inputs as si
from paper_2103_10127_b200 import ravgmg as rg

stream = torch.cuda.Stream()
torch.cuda.set_stream(stream)
prob = si.config_problem(sys.argv[1] if len(sys.argv) > 1 else "c2")
L = rg.gen_level(prob, "pou")
x0 = torch.tensor(si.initial_guess(L["n"], seed=si.X0_SEED), device="cuda")
kernels = [("auto", rg.KERNEL_AUTO)] + ([("schur", rg.KERNEL_SCHUR)] if len(sys.argv) > 2 else [])
for name, k in kernels:
    sm = rg.Smoother(L, L, kernel=k)
    r = sm.residual(x0, L["b"])
    x = x0.clone()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    for _ in range(5):
        sm.apply(r, x, 0.66)
    e0.record(stream)
    for _ in range(50):
        sm.apply(r, x, 0.66)
    e1.record(stream)
    torch.cuda.synchronize()
    ms = e0.elapsed_time(e1) / 50
    by = sm.sweep_bytes()["sweep"]
    print(f"{name:6s} {sm.kernel_name:80s} {ms*1e3:8.1f} us  {by/ms/1e6:8.1f} GB/s", flush=True)
    sm.close()
