"""Q1-Q1 stabilization constant study (reading R18): V(3,3) cycle counts of RAV /
MV / AV on the uniform driven cavity for several beta_0."""
import math
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch

import bench
import seeded_inputs as si
from paper_2103_10127_b200 import ravgmg as rg

stream = torch.cuda.Stream()
torch.cuda.set_stream(stream)
for beta in [float(b) for b in sys.argv[1:]]:
    for n in (128, 512, 1024):
        prob = si.problem(2, (n, n), si.KIND_CAVITY, elem=si.ELEM_Q1Q1, beta=beta)
        lv = int(math.log2(n // 8)) + 1
        res = {}
        for name, w, v, om in (("rav", "pou", rg.VARIANT_ROWS, 0.66), ("mv", "full", rg.VARIANT_MV, 0.66),
                               ("av", "full", rg.VARIANT_ROWS, 0.1)):
            r = bench._timed_solve(rg, prob, lv, w, v, om, 3, stream, maxit=200)
            res[name] = (r.get("cycles"), round(r.get("avg_reduction_factor", -1), 3))
        print(f"beta {beta:6.3f} n {n:5d} {res}", flush=True)
