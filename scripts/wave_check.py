"""Run nu RAV sweeps on a 2D MMS grid and save x (compare RAV_WAVE=1 against the default chain)."""
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch

import seeded_inputs as si
from paper_2103_10127_b200 import ravgmg as rg

n, nu, out = int(sys.argv[1]), int(sys.argv[2]), sys.argv[3]
timed = os.environ.get("RAV_WAVE_CHECK_TIME", "1") == "1" and not out.endswith("wave.npy") and not out.endswith("ref.npy")
stream = torch.cuda.Stream()
torch.cuda.set_stream(stream)
L = rg.gen_level(si.problem(2, (n, n), si.KIND_MMS, eta="fourier"), "pou")
sm = rg.Smoother(L, L)
x0 = torch.tensor(si.initial_guess(L["n"], seed=si.X0_SEED), device="cuda")
x = x0.clone()
sm.smooth(x, L["b"], nu, 0.66)
torch.cuda.synchronize()
np.save(out, x.cpu().numpy())
if not timed:
    sys.exit(0)
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
for _ in range(3):
    sm.smooth(x, L["b"], 100, 0.66)
e0.record(stream)
for _ in range(5):
    sm.smooth(x, L["b"], 100, 0.66)
e1.record(stream)
torch.cuda.synchronize()
ms = e0.elapsed_time(e1) / 5 / 100
print(f"n={n} nu={nu}: {ms*1e3:.1f} us per sweep, {L['n']/ms/1e3:.0f} MDoF/s, launches {sm.last_launches}", flush=True)
