"""One V-cycle of a BASELINE config (c3 / c4) for an ncu launch list: builds the hierarchy,
runs mg_vcycle three times (the first captures the cycle graph, then launches it), each inside
the library's NVTX range "mg_vcycle".

    ncu --nvtx --nvtx-include "mg_vcycle/" --metrics gpu__time_duration.sum --clock-control none \
        --csv --log-file out.csv python scripts/cycle_breakdown.py c3
    python scripts/cycle_breakdown.py --summarize out.csv
    (python scripts/cycle_breakdown.py c3 N: the slab-partitioned cycle, N subdomains on this GPU,
     NVTX range "mgd_vcycle")
"""
import csv
import os
import sys
from collections import defaultdict

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

if len(sys.argv) > 2 and sys.argv[1] == "--summarize":
    rows = list(csv.reader(open(sys.argv[2])))
    h = next(i for i, r in enumerate(rows) if "Kernel Name" in r)
    hdr, data = rows[h], rows[h + 1:]
    iN, iG, iV, iM = hdr.index("Kernel Name"), hdr.index("Grid Size"), hdr.index("Metric Value"), hdr.index("Metric Name")
    per = defaultdict(lambda: [0, 0.0])
    tot = 0.0
    for r in data:
        if len(r) <= iV or r[iM] != "gpu__time_duration.sum":
            continue
        v = float(r[iV].replace(",", ""))
        key = (r[iN].split("(")[0].split("<")[0].replace("void ", "").strip(), r[iG])
        per[key][0] += 1
        per[key][1] += v
        tot += v
    print(f"total {tot / 3e6:.3f} ms per cycle (3 cycles profiled), {sum(c for c, _ in per.values()) // 3} launches per cycle")
    for (k, g), (c, v) in sorted(per.items(), key=lambda kv: -kv[1][1])[:40]:
        print(f"{v / 3e3:9.1f} us  {c // 3:4d}x  {k:40s} grid {g}")
    sys.exit(0)

import torch

import seeded_inputs as si
from paper_2103_10127_b200 import ravgmg as rg

name = sys.argv[1] if len(sys.argv) > 1 else "c3"
c = si.CONFIGS[name]
if len(sys.argv) > 2:   # the slab-partitioned cycle with N subdomains on this GPU (NVTX range "mgd_vcycle")
    from paper_2103_10127_b200 import dist as rdist
    N = int(sys.argv[2])
    comm = rg.Comm(1, 0, None)
    mgd, info = rdist.build_lib_dist(si.config_problem(name), c["levels"], N, list(range(N)), [0] * N, comm)
    xs = [torch.zeros_like(v) for v in info["x"]]
    for _ in range(3):
        mgd.vcycle(xs, info["b"], c["pre"], c["post"], c["omega"])
    torch.cuda.synchronize()
    sys.exit(0)
mg, fine = rg.build_hierarchy(si.config_problem(name), c["levels"], "pou")
x = torch.zeros(fine["n"], dtype=torch.float64, device="cuda")
mg.vcycle(x, fine["b"], c["pre"], c["post"], c["omega"])
torch.cuda.synchronize()
for _ in range(2):  # + the first call above: 3 cycles
    mg.vcycle(x, fine["b"], c["pre"], c["post"], c["omega"])
torch.cuda.synchronize()
