"""Sweep-kernel and residual time against the grid size (2D Q2-Q1 MMS): separates the
size-independent part of a launch from the bandwidth slope (DESIGN 5.1)."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch

import seeded_inputs as si
from paper_2103_10127_b200 import ravgmg as rg

stream = torch.cuda.Stream()
torch.cuda.set_stream(stream)
rows = []
for n in [int(a) for a in (sys.argv[1:] or ["256", "384", "512", "768", "1024", "1536"])]:
    L = rg.gen_level(si.problem(2, (n, n), si.KIND_MMS, eta="fourier"), "pou")
    sm = rg.Smoother(L, L)
    x = torch.tensor(si.initial_guess(L["n"], seed=si.X0_SEED), device="cuda")
    r = sm.residual(x, L["b"])
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    out = {}
    for name, fn in (("apply", lambda: sm.apply(r, x, 0.66)), ("residual", lambda: sm.residual(x, L["b"], r))):
        for _ in range(5):
            fn()
        e0.record(stream)
        for _ in range(40):
            fn()
        e1.record(stream)
        torch.cuda.synchronize()
        out[name] = e0.elapsed_time(e1) / 40 * 1e3
    by = sm.sweep_bytes()
    rows.append((n, by["sweep"], out["apply"], by["residual"], out["residual"]))
    print(f"{n:5d}  apply {by['sweep']/1e9:7.3f} GB {out['apply']:9.1f} us   residual {by['residual']/1e9:7.3f} GB "
          f"{out['residual']:9.1f} us", flush=True)
    sm.close()
    del L
    torch.cuda.empty_cache()
a = np.array(rows)
for col, name in ((1, "apply"), (3, "residual")):
    slope, icpt = np.polyfit(a[:, col] / 1e9, a[:, col + 1], 1)
    print(f"{name}: {icpt:6.1f} us fixed + {1e3 / slope:6.2f} TB/s")
