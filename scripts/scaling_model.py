"""Parallel-efficiency model for 1 -> 8 GPUs from measured single-GPU times (VERDICT r01 "next
round" 6; SURVEY section 8 row e).  Only one GPU is available to this build, so the N-GPU time of
one rank is assembled from pieces measured on it:

  T_N = (T_emul(N) - T_coarse) / N + T_coarse + T_nccl(N) + T_link(N)

* T_emul(N): the library's slab-partitioned driver (mgd_vcycle / mgd_smooth, csrc/dist.cu) with
  all N subdomains on the one GPU and the exchanges between them as device reads (via_comm = 0).
  The subdomains' kernels run one after another, each on the whole GPU -- as each rank's kernels
  would on its own GPU -- so T_emul(N) / N is one rank's compute (balanced slabs).
* T_coarse: the agglomerated coarse levels, which every rank runs whole (not divided by N):
  mg_vcycle of that sub-hierarchy alone.
* T_nccl(N): T_emul(N, via_comm = 1) - T_emul(N, via_comm = 0): the same run with every exchange
  phase as an NCCL group of self sends / receives (one group per phase, as each rank posts one
  group per phase) -- NCCL's launch and copy cost per phase on this GPU.
* T_link(N): one rank's message bytes per cycle (largest interface lists) / 400 GB/s (NVLink 5,
  900 GB/s per direction nominal; half of it assumed achieved for ~100 KB messages).

Strong scaling (c3, c4 V-cycles): E = T_1 / (N T_N).  Weak scaling (c5 smoothers, c2 sweeps per
GPU): E = T_1 / T_N.  Writes one JSON file (argv[1]).
"""
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch

import seeded_inputs as si
from paper_2103_10127_b200 import dist as rdist
from paper_2103_10127_b200 import ravgmg as rg

OUT = sys.argv[1] if len(sys.argv) > 1 else "scaling_model.json"
STREAM = torch.cuda.Stream()
torch.cuda.set_stream(STREAM)
LINK_GBS = 400.0


def timed(fn, reps):
    fn()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(STREAM)
    for _ in range(reps):
        fn()
    e1.record(STREAM)
    torch.cuda.synchronize()
    return e0.elapsed_time(e1) / reps * 1e-3


def link_bytes(subs, sweeps_per_level):
    """Largest per-subdomain message bytes of one cycle: per level, (interface sums + halo) per
    sweep, both directions counted once (a rank sends and receives concurrently)."""
    worst = 0
    for i in range(len(subs[0])):
        tot = 0
        for k, row in enumerate(subs):
            nb = row[i]["neighbors"]
            per = sum(len(v[0]) + len(v[2]) for v in nb.values()) * 8
            tot += per * sweeps_per_level
        worst = max(worst, tot)
    return worst


def vcycle_case(name, Ns):
    c = si.CONFIGS[name]
    prob = si.config_problem(name)
    pre, post, om = c["pre"], c["post"], c["omega"]
    mg, fine = rg.build_hierarchy(prob, c["levels"], "pou")
    x = torch.zeros(fine["n"], dtype=torch.float64, device="cuda")
    b = fine["b"]
    t1 = timed(lambda: mg.vcycle(x, b, pre, post, om), 10)
    mg.close()
    del mg, x, fine
    torch.cuda.empty_cache()
    out = {"config": name, "T1_s_per_cycle": t1, "N": {}}
    comm0 = rg.Comm(1, 0, None)
    comm1 = rg.Comm(1, 0, rg.Comm.unique_id())
    for N in Ns:
        row = {}
        for via, comm in ((False, comm0), (True, comm1)):
            mgd, info = rdist.build_lib_dist(prob, c["levels"], N, list(range(N)), [0] * N, comm, via_comm=via,
                                             stream=STREAM)
            xs = [torch.zeros_like(v) for v in info["x"]]
            t = timed(lambda: mgd.vcycle(xs, info["b"], pre, post, om), 5)
            row["T_emul_nccl_s" if via else "T_emul_s"] = t
            if not via:
                subs, coarse = mgd._keep
                row["partitioned_levels"] = info["K"]
                row["coarse_levels"] = c["levels"] - info["K"]
                row["link_bytes_per_cycle"] = link_bytes(subs, pre + post + 2)
                row["T_coarse_s"] = 0.0
                if coarse is not None:
                    xc = torch.zeros(coarse.n, dtype=torch.float64, device="cuda")
                    bc = torch.randn(coarse.n, dtype=torch.float64, device="cuda")
                    row["T_coarse_s"] = timed(lambda: coarse.vcycle(xc, bc, pre, post, om), 10)
            mgd.close()
            del mgd, info, xs
            torch.cuda.empty_cache()
        tc = row.get("T_coarse_s") or 0.0
        row["T_nccl_s"] = max(0.0, row["T_emul_nccl_s"] - row["T_emul_s"])
        row["T_link_s"] = row["link_bytes_per_cycle"] / (LINK_GBS * 1e9)
        TN = (row["T_emul_s"] - tc) / N + tc + row["T_nccl_s"] + row["T_link_s"]
        row["T_N_model_s"] = TN
        row["efficiency_strong"] = t1 / (N * TN)
        out["N"][N] = row
        print(name, N, json.dumps(row), flush=True)
    comm0.close()
    comm1.close()
    return out


def smooth_case(name, Ns, sweeps):
    """Weak scaling of RAV sweeps: the config's grid per GPU stacked in y (config_problem scale_y)."""
    out = {"config": f"{name} per GPU stacked in y, seeded eta, RAV omega 0.66", "N": {}}
    prob1 = si.config_problem(name)
    L = rg.gen_level(prob1, "pou")
    sm = rg.Smoother(L, L)
    x = torch.tensor(si.initial_guess(L["n"], seed=si.X0_SEED), device="cuda")
    t1 = timed(lambda: sm.smooth(x, L["b"], sweeps, 0.66), 3) / sweeps
    sm.close()
    del sm, L, x
    torch.cuda.empty_cache()
    out["T1_s_per_sweep"] = t1
    comm0 = rg.Comm(1, 0, None)
    comm1 = rg.Comm(1, 0, rg.Comm.unique_id())
    for N in Ns:
        prob = si.config_problem(name, scale_y=N)
        row = {}
        for via, comm in ((False, comm0), (True, comm1)):
            mgd, info = rdist.build_lib_dist(prob, 1, N, list(range(N)), [0] * N, comm, smooth_only=True,
                                             via_comm=via, stream=STREAM)
            xs = [torch.zeros_like(v) for v in info["x"]]
            t = timed(lambda: mgd.smooth(xs, info["b"], sweeps, 0.66), 3) / sweeps
            row["T_emul_nccl_s" if via else "T_emul_s"] = t
            if not via:
                subs, _ = mgd._keep
                row["link_bytes_per_sweep"] = link_bytes(subs, 1)
            mgd.close()
            del mgd, info, xs
            torch.cuda.empty_cache()
        row["T_nccl_s"] = max(0.0, row["T_emul_nccl_s"] - row["T_emul_s"])
        row["T_link_s"] = row["link_bytes_per_sweep"] / (LINK_GBS * 1e9)
        TN = row["T_emul_s"] / N + row["T_nccl_s"] + row["T_link_s"]
        row["T_N_model_s"] = TN
        row["efficiency_weak"] = t1 / TN
        out["N"][N] = row
        print(name, N, json.dumps(row), flush=True)
    comm0.close()
    comm1.close()
    return out


res = {"model": __doc__.strip(), "gpu": torch.cuda.get_device_name(0)}
res["c2_weak_sweeps"] = smooth_case("c2", (2, 4, 8), 20)
res["c5_weak_sweeps"] = smooth_case("c5", (2, 4), 10)
res["c4_vcycle"] = vcycle_case("c4", (2, 4, 8))
res["c3_vcycle"] = vcycle_case("c3", (2, 4, 8))
with open(OUT, "w") as f:
    json.dump(res, f, indent=1)
