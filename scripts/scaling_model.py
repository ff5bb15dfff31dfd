"""Parallel-efficiency model for 1 -> 8 GPUs from measured single-GPU times (VERDICT r01 "next
round" 6; SURVEY section 8 row e).  Only one GPU is available to this build, so the N-GPU time of
one rank is assembled from pieces measured on it:

  strong (c3, c4 V-cycles):  T_N = (T_emul(N) - T_coarse) / N + T_coarse + T_nccl + T_link(N)
                             (+ (1 - 1/N) T_phase in the conservative form)
  weak (c2, c5 sweeps):      T_N = T_1 + (T_emul(N) - N T_1) + T_nccl + T_link(N)

* T_emul(N): the library's slab-partitioned driver (mgd_vcycle / mgd_smooth, csrc/dist.cu) with
  all N subdomains on the one GPU and the exchanges between them as device reads (via_comm = 0).
  The subdomains' kernels run one after another, each on the whole GPU -- as each rank's kernels
  would on its own GPU -- so T_emul(N) / N is one rank's compute (balanced slabs).
* T_coarse: the agglomerated coarse levels, which every rank runs whole (not divided by N):
  mg_vcycle of that sub-hierarchy alone.
* T_nccl: T_emul(2, via_comm = 1) - T_emul(2, via_comm = 0): the same 2-subdomain run with every
  exchange phase as an NCCL group of self sends / receives.  With two subdomains one group holds
  2 sends + 2 receives, what an interior rank posts per phase (two neighbours); with N
  subdomains the emulated group holds all 2(N - 1) pairs, more than any rank posts, so the
  N = 2 difference is the per-rank estimate (the N > 2 differences are reported too).  NCCL's
  self send is its on-device copy path: NVLink adds its latency (a few us per phase) -- T_link.
* T_emul_peer(N): the same run with the peer-memory transport (mgd via_comm = 2; local
  pointers on one GPU): the cost of its flag / fence protocol inside the pack / unpack kernels.
  With it the per-rank exchange estimate is T_emul_peer(2) - T_emul(2) + T_link (no NCCL).
* T_phase (strong, conservative): the exchange-phase kernels (zero / pack / add / unpack) run once
  per phase for ALL local subdomains in the emulation but once per rank on N GPUs; counted from
  the graph's launch count (mgd_last_launches for N = 2 and 4) at 3 us per launch.
* weak: T_emul(N) - N T_1 is everything the partitioned run adds to N single-GPU sweeps (ghost
  rows, phase kernels); it is charged to every rank in full.
* T_link(N): one rank's message bytes per cycle (largest interface lists) / 400 GB/s (NVLink 5,
  900 GB/s per direction nominal; half of it assumed achieved for ~100 KB messages) + 3 us of
  NVLink latency per exchange phase.

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
LINK_LAT_S = 3e-6
LAUNCH_S = 3e-6


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


def vcycle_case(name, Ns, agg_layers=0):
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
    out = {"config": name, "agg_layers": agg_layers, "T1_s_per_cycle": t1, "N": {}}
    comm0 = rg.Comm(1, 0, None)
    comm1 = rg.Comm(1, 0, rg.Comm.unique_id())
    for N in Ns:
        row = {}
        for via, comm in ((0, comm0), (1, comm1), (2, comm0)):
            mgd, info = rdist.build_lib_dist(prob, c["levels"], N, list(range(N)), [0] * N, comm, via_comm=via,
                                             stream=STREAM, agg_layers=agg_layers)
            xs = [torch.zeros_like(v) for v in info["x"]]
            t = timed(lambda: mgd.vcycle(xs, info["b"], pre, post, om), 5)
            row[("T_emul_s", "T_emul_nccl_s", "T_emul_peer_s")[via]] = t
            if not via:
                subs, coarse = mgd._keep
                row["launches_per_cycle"] = mgd.last_launches
                row["partitioned_levels"] = info["K"]
                row["coarse_levels"] = c["levels"] - info["K"]
                row["link_bytes_per_cycle"] = link_bytes(subs, pre + post + 2)
                row["phases_per_cycle"] = 2 * (pre + post) * info["K"] + 4 * info["K"]
                row["T_coarse_s"] = 0.0
                row["coarse_launches_per_cycle"] = 0
                if coarse is not None:
                    xc = torch.zeros(coarse.n, dtype=torch.float64, device="cuda")
                    bc = torch.randn(coarse.n, dtype=torch.float64, device="cuda")
                    row["T_coarse_s"] = timed(lambda: coarse.vcycle(xc, bc, pre, post, om), 10)
                    row["coarse_launches_per_cycle"] = coarse.last_launches
                    del xc, bc
                del subs, coarse
            mgd.close()
            del mgd, info, xs
            torch.cuda.empty_cache()
        row["T_nccl_s_emulated_group"] = max(0.0, row["T_emul_nccl_s"] - row["T_emul_s"])
        out["N"][N] = row
        print(name, N, json.dumps(row), flush=True)
    comm0.close()
    comm1.close()
    # per-subdomain and shared (phase) launches from N = 2 and N = 4: L(N) = N L_sub + L_phase + L_coarse
    r2, r4 = out["N"][2], out["N"][4]
    l_sub = (r4["launches_per_cycle"] - r2["launches_per_cycle"]) / 2
    l_phase = max(0.0, r2["launches_per_cycle"] - 2 * l_sub - r2["coarse_launches_per_cycle"])
    t_nccl = r2["T_nccl_s_emulated_group"]
    t_peer = max(0.0, r2["T_emul_peer_s"] - r2["T_emul_s"])
    out["per_rank"] = {"launches_per_subdomain": l_sub, "phase_launches": l_phase, "T_nccl_s": t_nccl,
                       "T_peer_protocol_s": t_peer}
    for N, row in out["N"].items():
        tc = row["T_coarse_s"]
        t_link = row["link_bytes_per_cycle"] / (LINK_GBS * 1e9) + row["phases_per_cycle"] * LINK_LAT_S
        TN = (row["T_emul_s"] - tc) / N + tc + t_nccl + t_link
        TNc = TN + (1 - 1 / N) * l_phase * LAUNCH_S
        TNp = (row["T_emul_s"] - tc) / N + tc + t_peer + t_link
        row.update({"T_link_s": t_link, "T_N_model_s": TN, "T_N_model_conservative_s": TNc,
                    "efficiency_strong": t1 / (N * TN), "efficiency_strong_conservative": t1 / (N * TNc),
                    "T_N_model_peer_s": TNp, "efficiency_strong_peer": t1 / (N * TNp)})
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
        for via, comm in ((0, comm0), (1, comm1), (2, comm0)):
            mgd, info = rdist.build_lib_dist(prob, 1, N, list(range(N)), [0] * N, comm, smooth_only=True,
                                             via_comm=via, stream=STREAM)
            xs = [torch.zeros_like(v) for v in info["x"]]
            t = timed(lambda: mgd.smooth(xs, info["b"], sweeps, 0.66), 3) / sweeps
            row[("T_emul_s", "T_emul_nccl_s", "T_emul_peer_s")[via]] = t
            if not via:
                subs, _ = mgd._keep
                row["link_bytes_per_sweep"] = link_bytes(subs, 1)
                del subs
            mgd.close()
            del mgd, info, xs
            torch.cuda.empty_cache()
        row["T_nccl_s_emulated_group"] = max(0.0, row["T_emul_nccl_s"] - row["T_emul_s"])
        out["N"][N] = row
        print(name, N, json.dumps(row), flush=True)
    comm0.close()
    comm1.close()
    t_nccl = out["N"][Ns[0]]["T_nccl_s_emulated_group"]   # N = 2: one interior rank's group
    t_peer = max(0.0, out["N"][Ns[0]]["T_emul_peer_s"] - out["N"][Ns[0]]["T_emul_s"])
    for N, row in out["N"].items():
        t_link = row["link_bytes_per_sweep"] / (LINK_GBS * 1e9) + 2 * LINK_LAT_S
        extra = max(0.0, row["T_emul_s"] - N * t1)
        TN = t1 + extra + t_nccl + t_link
        TNp = t1 + extra + t_peer + t_link
        row.update({"T_extra_s": extra, "T_nccl_s": t_nccl, "T_link_s": t_link, "T_N_model_s": TN,
                    "efficiency_weak": t1 / TN, "T_peer_protocol_s": t_peer, "T_N_model_peer_s": TNp,
                    "efficiency_weak_peer": t1 / TNp})
    return out


res = {"model": __doc__.strip(), "gpu": torch.cuda.get_device_name(0)}
which = sys.argv[2].split(",") if len(sys.argv) > 2 else ["c2", "c5", "c4", "c3"]
if "c2" in which:
    res["c2_weak_sweeps"] = smooth_case("c2", (2, 4, 8), 20)
if "c5" in which:
    res["c5_weak_sweeps"] = smooth_case("c5", (2, 4), 10)
if "c4" in which:
    res["c4_vcycle"] = vcycle_case("c4", (2, 4, 8))
if "c3" in which:
    res["c3_vcycle"] = vcycle_case("c3", (2, 4, 8))
for agg in [int(a) for a in (sys.argv[3].split(",") if len(sys.argv) > 3 else [])]:
    res[f"c3_vcycle_agg{agg}"] = vcycle_case("c3", (2, 4, 8), agg_layers=agg)
with open(OUT, "w") as f:
    json.dump(res, f, indent=1)
