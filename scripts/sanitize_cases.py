"""Small end-to-end cases for compute-sanitizer: c1 V-cycle, 64^2
RAV sweeps (Schur / rows / warp / sym formats), deterministic mode, diagonal and MV
smoothers, Q1-Q1, an adaptive hierarchy, a 3D patch set, FGMRES, windowed transfers."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch

import seeded_inputs as si
from paper_2103_10127_b200 import dist as rdist
from paper_2103_10127_b200 import ravgmg as rg

torch.cuda.set_device(0)
c1 = si.problem(2, (8, 8), si.KIND_CAVITY)
mg, fine = rg.build_hierarchy(c1, 3, "pou")
x = torch.zeros(fine["n"], dtype=torch.float64, device="cuda")
print("c1 cycles", mg.solve(x, fine["b"], rtol=1e-10)[1])
x.zero_()
print("c1 fgmres", mg.fgmres(x, fine["b"], rtol=1e-10)[1])
p64 = si.problem(2, (64, 64), si.KIND_MMS, eta="fourier")
G = rg.gen_level(p64, "pou")
x0 = torch.tensor(si.initial_guess(G["n"], seed=3), device="cuda")
for k in (rg.KERNEL_AUTO, rg.KERNEL_WARP, rg.KERNEL_THREAD, rg.KERNEL_SYM):
    sm = rg.Smoother(G, G, kernel=k)
    x = x0.clone()
    sm.smooth(x, G["b"], 3, 0.66)
    print("64^2", sm.kernel_name, float(x.norm()))
sm = rg.Smoother(G, G, deterministic=True)
x = x0.clone()
sm.smooth(x, G["b"], 3, 0.66)
print("det", float(x.norm()))
Gf = rg.gen_level(p64, "full")
for v in (rg.VARIANT_DIAG, rg.VARIANT_MV):
    sm = rg.Smoother(Gf, Gf, variant=v)
    if v == rg.VARIANT_MV:
        sm.set_colors(*rg.multicolor(p64))
    x = x0.clone()
    sm.smooth(x, Gf["b"], 2, 0.1 if v == rg.VARIANT_DIAG else 0.66)
    print("variant", v, float(x.norm()))
q1 = si.problem(2, (16, 16), si.KIND_CAVITY, elem=si.ELEM_Q1Q1)
mg, fine = rg.build_hierarchy(q1, 2, "pou")
x = torch.zeros(fine["n"], dtype=torch.float64, device="cuda")
print("q1q1 cycles", mg.solve(x, fine["b"], pre=3, post=3, rtol=1e-8)[1])
mg, fine = rg.build_adaptive_hierarchy(si.problem(2, (8, 8), si.KIND_CAVITY, elem=si.ELEM_Q1Q1), 3, "own")
x = torch.zeros(fine["n"], dtype=torch.float64, device="cuda")
print("adaptive cycles", mg.solve(x, fine["b"], pre=3, post=3, rtol=1e-8)[1])
mg, fine = rg.build_hierarchy(si.problem(3, (4, 4, 4), si.KIND_CAVITY, eta="fourier"), 2, "pou")
x = torch.zeros(fine["n"], dtype=torch.float64, device="cuda")
print("3d cycles", mg.solve(x, fine["b"], rtol=1e-8)[1])
prob = si.problem(2, (16, 32), si.KIND_MMS)
slab = rdist.Slab(prob, 2, 1)
T = rg.Transfer(rg.gen_prolongation(dict(prob, window=slab.transfer_window()), rg.coarsen_problem(prob)))
print("windowed transfer nc", T.nc)
torch.cuda.synchronize()
print("sanitize cases done")
