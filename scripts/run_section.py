"""Run one bench.py section alone on cuda:0 and print its JSON (development aid).
    python scripts/run_section.py q1q1|vcycle_smoothers|c5"""
import json
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import torch

import bench
import seeded_inputs as si
from paper_2103_10127_b200 import ravgmg as rg

stream = torch.cuda.Stream()
torch.cuda.set_stream(stream)
t0 = time.time()
fn = {"q1q1": bench.run_q1q1_studies, "vcycle_smoothers": bench.run_vcycle_smoothers,
      "c5": bench.run_c5_smoothers, "adaptive": bench.run_adaptive_study}[sys.argv[1]]
out = fn(rg, si, stream)
print(json.dumps(out, indent=1))
print("wall", time.time() - t0, file=sys.stderr)
