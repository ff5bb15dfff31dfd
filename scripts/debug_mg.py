import faulthandler, sys, time
faulthandler.dump_traceback_later(60, exit=True)
sys.path.insert(0, '.')
import torch, numpy as np
import seeded_inputs as si
from paper_2103_10127_b200 import ravgmg as rg
prob = si.problem(2, (8, 8), si.KIND_CAVITY)
print("gen", flush=True)
probs = [prob, rg.coarsen_problem(prob), rg.coarsen_problem(rg.coarsen_problem(prob))][::-1]
levels = [rg.gen_level(p) for p in probs]
print("levels", [l["n"] for l in levels], flush=True)
prols = [None] + [rg.gen_prolongation(probs[l], probs[l-1]) for l in range(1, 3)]
print("prols", flush=True)
mg = rg.Multigrid(levels, prols, levels[0]["nvel"])
print("mg setup ok", flush=True)
x = torch.zeros(levels[-1]["n"], dtype=torch.float64, device="cuda")
mg.vcycle(x, levels[-1]["b"])
torch.cuda.synchronize()
print("vcycle ok", x.norm().item(), flush=True)
x.zero_()
x, k, h = mg.solve(x, levels[-1]["b"], rtol=1e-10)
print("solve", k, h[-1]/h[0], flush=True)
