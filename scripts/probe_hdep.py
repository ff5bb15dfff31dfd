import sys, time
sys.path.insert(0, '.')
import torch, numpy as np
import seeded_inputs as si, oracle
from paper_2103_10127_b200 import ravgmg as rg
for n in (64, 128, 256, 512, 1024, 2048):
    for coarse in (4, 16):
        lev = int(np.log2(n // coarse)) + 1
        mg, fine = rg.build_hierarchy(si.problem(2, (n, n), si.KIND_MMS, eta="fourier"), lev, "pou")
        x = torch.zeros(fine["n"], dtype=torch.float64, device="cuda")
        x, k, h = mg.solve(x, fine["b"], rtol=1e-8, maxit=100)
        print(f"GPU n={n} levels={lev} coarse={coarse}: cycles {k} rho {(h[-1]/h[0])**(1/k):.3f}", flush=True)
        mg.close(); del mg
    if n <= 256:
        for coarse in (4, 16):
            lev = int(np.log2(n // coarse)) + 1
            H = oracle.Hierarchy(si.problem(2, (n, n), si.KIND_MMS, eta="fourier"), lev, "rav")
            print(f"ORA n={n} levels={lev} coarse={coarse}: cycles {H.solve(rtol=1e-8)[1]}", flush=True)
for n in (64, 256, 1024):
    lev = int(np.log2(n // 4)) + 1
    mg, fine = rg.build_hierarchy(si.problem(2, (n, n), si.KIND_MMS, eta="const"), lev, "pou")
    x = torch.zeros(fine["n"], dtype=torch.float64, device="cuda")
    x, k, h = mg.solve(x, fine["b"], rtol=1e-8, maxit=100)
    print(f"GPU const-eta n={n} levels={lev}: cycles {k}", flush=True)
