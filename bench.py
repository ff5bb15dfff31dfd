#!/usr/bin/env python
"""Benchmark of the RAV hot path (BASELINE.json metric: "RAV sweep MDoF/s and
HBM GB/s vs peak; V-cycle time to 1e-8").

Workload (N=1): BASELINE config 2 -- 2D unit square 512x512 Taylor-Hood Q2-Q1,
seeded variable viscosity, manufactured forcing; one STEP = 100 RAV sweeps
(residual SpMV + fused RAV sweep kernel, rav_smooth(nu=100)) from the seeded
N(0,1) guess.  value = free DoFs x sweeps / second (MDoF/s), device-timed.

  python bench.py [--gpus N] [--steps K] [--warmup W] [--impl reference]

--impl reference times the CPU oracle (oracle/, plain C) on the same workload
(bounded: one sweep per step).  Under torchrun (N > 1) the c2 workload is
stacked along y, one 512^2 block per GPU, and slab-partitioned: every sweep runs
the interface-correction sum and the halo refresh between neighbouring ranks
(weak scaling).

The JSON line ends with the V-cycle metric ("vcycle": c3 / c4 time to 1e-8);
the paper-setting studies (Q1-Q1, adaptive hierarchy, V-cycle smoother
comparison) run only with --studies FILE and go to FILE.
"""
from __future__ import annotations

import argparse
import json
import os
import statistics
import subprocess
import sys
import threading
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

SWEEPS_PER_STEP = 100
OMEGA = 0.66


def load_peaks():
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as f:
            p = json.load(f)
        return float(p["hbm_gbs"]), "measured"
    except Exception:
        return 6650.0, "fallback"


class ClockSampler:
    """nvidia-smi clocks / throttle reasons sampled during the timed region."""
    Q = ("clocks.sm,clocks.max.sm,clocks_event_reasons.active,clocks_event_reasons.hw_slowdown,"
         "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,"
         "clocks_event_reasons.sw_power_cap")

    def __init__(self, index=0):
        self.index = index
        self.proc = None
        self.out = None

    def __enter__(self):
        try:
            self.proc = subprocess.Popen(["nvidia-smi", "-i", str(self.index), f"--query-gpu={self.Q}",
                                          "--format=csv,noheader,nounits", "-lms", "100"],
                                         stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
        except Exception:
            self.proc = None
        return self

    def __exit__(self, *a):
        if self.proc is None:
            self.out = ""
            return
        time.sleep(0.25)
        self.proc.terminate()
        try:
            self.out, _ = self.proc.communicate(timeout=5)
        except Exception:
            self.proc.kill()
            self.out = ""

    def summary(self):
        sm, mx, reasons = [], 0.0, set()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        for line in (self.out or "").strip().splitlines():
            parts = [p.strip() for p in line.split(",")]
            if len(parts) < 7:
                continue
            try:
                sm.append(float(parts[0]))
                mx = max(mx, float(parts[1]))
            except ValueError:
                continue
            for nm, v in zip(names, parts[3:7]):
                if v.lower() == "active":
                    reasons.add(nm)
        return {"sm_mhz": statistics.median(sm) if sm else None, "sm_max_mhz": mx or None,
                "reasons": sorted(reasons), "samples": len(sm)}


def dist_env():
    ws = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    return ws, rank, local


def cpu_oracle_rate(prob, steps, warmup, sweeps_per_step=1, threads=None):
    """The oracle (as it stands) timed on this host: setup untimed, then
    `sweeps_per_step` RAV sweeps per step on `threads` OpenMP threads (None: all;
    the oracle's parallel loops give the same bits at any count).
    Returns (MDoF/s, threads used, sample, seconds)."""
    import oracle
    import seeded_inputs as si
    O = oracle.assemble(prob)
    P = oracle.patches(prob, "pou")
    F = oracle.factor(O, P, oracle.FMT_ROWS)
    x = si.initial_guess(O["n"], seed=si.X0_SEED)
    prev = oracle.set_num_threads(threads or (os.cpu_count() or 1))
    used = oracle.lib().or_num_threads()
    try:
        for _ in range(warmup):
            x = oracle.additive_sweeps(O, P, F, x, O["b"], OMEGA, sweeps_per_step)
        t0 = time.perf_counter()
        for _ in range(steps):
            x = oracle.additive_sweeps(O, P, F, x, O["b"], OMEGA, sweeps_per_step)
        dt = time.perf_counter() - t0
    finally:
        oracle.set_num_threads(prev)
    rate = O["n"] * sweeps_per_step * steps / dt / 1e6
    sample = (f"c2 (512^2, {O['n']} DoFs) oracle RAV sweeps, {steps} x {sweeps_per_step} sweep(s) "
              f"after untimed setup; {dt:.2f} s on {used} thread(s) of {host_cpu()}")
    return rate, used, sample, dt


def oracle_sweep_samples(si, threads):
    """Per-sweep oracle times for c3 / c4 / c5 from bounded samples at the configs' mesh
    spacing (SURVEY row d): a strip 2048 x 128 cells of the 2048^2
    grid (1/16 of c3 / c5) and a slab 32 x 32 x 4 cells of c4 (5 of its 33 vertex layers);
    per-sweep time scaled to the full config by the patch count.  RAV (Eq. 13), and
    for c5 also diagonal Vanka (R17) and multiplicative Vanka (Eq. 11, sequential)."""
    import oracle
    out = {}
    prev = oracle.set_num_threads(threads)
    used = oracle.lib().or_num_threads()
    try:
        strip = si.problem(2, (2048, 128), si.KIND_MMS, eta="fourier", box=(1.0, 1.0 / 16))
        full_patches = 2049 * 2049
        O = oracle.assemble(strip)
        for name, w, fmt, om in (("rav", "pou", oracle.FMT_ROWS, OMEGA), ("diag_vanka", "full", oracle.FMT_DIAG, 0.1),
                                 ("mv", "full", oracle.FMT_LU, OMEGA)):
            P = oracle.patches(strip, w)
            F = oracle.factor(O, P, fmt)
            x = si.initial_guess(O["n"], seed=si.X0_SEED)
            t0 = time.perf_counter()
            if name == "mv":
                oracle.mv_sweeps(O, P, F, x, O["b"], om, 1)
            else:
                oracle.additive_sweeps(O, P, F, x, O["b"], om, 1)
            dt = time.perf_counter() - t0
            out[f"c3_c5_{name}_s_per_sweep"] = dt * full_patches / (len(P["offs"]) - 1)
            del P, F
        out["c3_c5_sample"] = "2048 x 128 cells (h = 1/2048), 1 sweep, scaled x 2049^2 / 2049*129 patches"
        slab = si.problem(3, (32, 32, 4), si.KIND_CAVITY, eta="fourier", box=(1.0, 1.0, 0.125))
        O = oracle.assemble(slab)
        P = oracle.patches(slab, "pou")
        F = oracle.factor(O, P, oracle.FMT_ROWS)
        x = si.initial_guess(O["n"], seed=si.X0_SEED)
        t0 = time.perf_counter()
        oracle.additive_sweeps(O, P, F, x, O["b"], OMEGA, 1)
        dt = time.perf_counter() - t0
        out["c4_rav_s_per_sweep"] = dt * 33 ** 3 / (len(P["offs"]) - 1)
        out["c4_sample"] = "32 x 32 x 4 cells (h = 1/32), 1 sweep, scaled x 33^3 / 33*33*5 patches"
    finally:
        oracle.set_num_threads(prev)
    out["threads"] = used
    return out


def host_info() -> dict:
    """nproc, CPU model and memory of this host (context for the oracle timings)."""
    mem = None
    try:
        for line in open("/proc/meminfo"):
            if line.startswith("MemTotal"):
                mem = round(int(line.split()[1]) / 2 ** 20, 1)
    except OSError:
        pass
    return {"cpu": host_cpu(), "nproc": os.cpu_count(), "mem_gib": mem}


def host_cpu() -> str:
    """CPU model and logical core count of this host (context for the oracle timing)."""
    model = "unknown CPU"
    try:
        for line in open("/proc/cpuinfo"):
            if line.startswith("model name"):
                model = line.split(":", 1)[1].strip()
                break
    except OSError:
        pass
    return f"{model}, {os.cpu_count()} logical cores"


def run_reference(args):
    ws, rank, _ = dist_env()
    if rank != 0:
        return 0
    import seeded_inputs as si
    prob = si.config_problem("c2")
    rate, cores, sample, dt = cpu_oracle_rate(prob, args.steps, args.warmup)
    n = None
    line = {"metric": "RAV sweep throughput (c2: 512^2 Q2-Q1, variable viscosity)", "value": rate,
            "unit": "MDoF/s", "n_gpus": ws, "steps": args.steps, "warmup": args.warmup,
            "ms_per_step": dt / args.steps * 1e3, "higher_is_better": True, "scaling": "weak",
            "vs_baseline": None, "dtype": "f64", "data": "synthetic",
            "config": {"workload": "c2: 2D 512x512 Q2-Q1 MMS, seeded eta in [0.1,10], RAV sweeps",
                       "sweeps_per_step": 1},
            "impl": "reference",
            "cpu_baseline": {"value": rate, "unit": "MDoF/s", "cores": cores, "kind": "oracle", "sample": sample},
            "e2e": {"value": rate, "unit": "MDoF/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    print(json.dumps(line), flush=True)
    return 0


VCYCLE_DESC = {
    "c3": "c3: 2048^2 Q2-Q1 MMS, seeded eta, 10 levels (4^2 coarsest), V(2,2)-RAV omega 0.66, x0 = 0",
    "c4": "c4: 32^3 Q2-Q1 lid-driven cavity, seeded eta, 5 levels (2^3 coarsest, reading R14), "
          "V(2,2)-RAV omega 0.66, x0 = 0",
}


def run_vcycle(name, rg, si, stream, dist):
    """mg_solve on a BASELINE V-cycle config (c3: 2048^2 MMS, 10 levels; c4:
    32^3 cavity, 5 levels), V(2,2)-RAV, omega 0.66, x0 = 0, to ||r|| <= 1e-8
    ||r0||.  Device-timed with CUDA events around mg_solve (which reads back
    one norm per cycle for the stopping test)."""
    import torch
    c = si.CONFIGS[name]
    prob = si.config_problem(name)
    t0 = time.perf_counter()
    mg, fine = rg.build_hierarchy(prob, c["levels"], "pou")
    torch.cuda.synchronize()
    setup_s = time.perf_counter() - t0
    b = fine["b"]
    x = torch.zeros(fine["n"], dtype=torch.float64, device="cuda")
    mg.solve(x, b, pre=c["pre"], post=c["post"], omega=c["omega"], rtol=c["rtol"], maxit=3)  # warm (graph capture)
    times, iters, hist = [], None, None
    for _ in range(3):
        x.zero_()
        torch.cuda.synchronize()
        if dist is not None:
            dist.barrier()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(stream)
        x, iters, hist = mg.solve(x, b, pre=c["pre"], post=c["post"], omega=c["omega"], rtol=c["rtol"], maxit=100)
        e1.record(stream)
        torch.cuda.synchronize()
        times.append(e0.elapsed_time(e1) / 1e3)
    t = min(times)
    if dist is not None:
        tt = torch.tensor([t], device="cuda")
        dist.all_reduce(tt, op=dist.ReduceOp.MAX)
        t = float(tt.item())
    launches = mg.last_launches
    rho = (hist[-1] / hist[0]) ** (1.0 / max(iters, 1))
    # the same V-cycle as the preconditioner of flexible GMRES(30) (R19)
    fg = None
    try:
        x.zero_()
        mg.fgmres(x, b, pre=c["pre"], post=c["post"], omega=c["omega"], rtol=c["rtol"], maxit=2)   # work space
        x.zero_()
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(stream)
        _, fk, fh = mg.fgmres(x, b, pre=c["pre"], post=c["post"], omega=c["omega"], rtol=c["rtol"], maxit=100)
        e1.record(stream)
        torch.cuda.synchronize()
        ft = e0.elapsed_time(e1) / 1e3
        fg = {"preconditioner_applications": fk, "converged": bool(fh[-1] <= c["rtol"] * fh[0]),
              "time_to_rtol_s": ft, "restart": 30}
    except Exception as err:  # report, keep the line
        fg = {"error": f"{type(err).__name__}: {err}"[:200]}
    # HBM roofline of the whole cycle: mg_cycle_bytes (algorithmic bytes of every kernel of a cycle
    # + the stopping test's residual) / the measured time per cycle
    cyc_bytes = mg.cycle_bytes(c["pre"], c["post"])
    peak, peak_kind = load_peaks()
    ach = cyc_bytes / (t / max(iters, 1)) / 1e9
    out = {"config": VCYCLE_DESC[name], "free_dofs": fine["n"], "rtol": c["rtol"], "cycles": iters, "converged": bool(hist[-1] <= c["rtol"] * hist[0]),
           "time_to_rtol_s": t, "ms_per_cycle": t / max(iters, 1) * 1e3, "avg_reduction_factor": rho,
           "roofline": {"bound": "hbm", "algorithmic_gb_per_cycle": cyc_bytes / 1e9, "achieved": ach,
                        "peak": peak, "peak_kind": peak_kind, "unit": "GB/s", "frac": ach / peak},
           "setup_s": setup_s, "gpu_launches": launches, "timing": "CUDA events around mg_solve, best of 3",
           "fgmres": fg}
    mg.close()
    del mg, fine, x, b
    torch.cuda.empty_cache()
    return out


def run_c1(rg, si):
    """BASELINE config 1 (correctness config, launch-bound): 8x8 cavity, 3 levels, V(2,2)-RAV to
    1e-10, then the pressure normalised so p(vertex 0) = 0 (row a10, R4)."""
    import torch
    c = si.CONFIGS["c1"]
    prob = si.problem(2, c["ncell"], c["kind"], eta=c["eta"])
    mg, fine = rg.build_hierarchy(prob, c["levels"], "pou")
    x = torch.zeros(fine["n"], dtype=torch.float64, device="cuda")
    x, k, h = mg.solve(x, fine["b"], pre=c["pre"], post=c["post"], omega=c["omega"], rtol=c["rtol"])
    mg.normalize_pressure(x, mode=0)
    p0 = float(x[fine["nvel"]].item())
    mg.close()
    return {"config": "c1: 8x8 Q2-Q1 cavity, eta = 1, 3 levels, V(2,2)-RAV omega 0.66, rtol 1e-10",
            "free_dofs": fine["n"], "cycles": k, "converged": bool(h[-1] <= c["rtol"] * h[0]),
            "pressure_normalized": "p(vertex 0) = 0 (mg_normalize_pressure)", "p_vertex0": p0}


def run_c5_smoothers(rg, si, stream):
    """BASELINE config 5 on one GPU: 2048^2 MMS with seeded eta, 50 sweeps each of
    RAV (omega 0.66), diagonal Vanka (omega 0.1) and multicoloured MV (omega
    0.66) from the seeded N(0,1) guess: time per sweep, MDoF/s and the residual
    reduction ||b - L x_50|| / ||b - L x_0|| ("runtime per iteration")."""
    import torch
    prob = si.config_problem("c5")
    out = {"config": "c5 (1 GPU): 2048^2 Q2-Q1 MMS, seeded eta, 50 sweeps from seeded N(0,1)"}
    x0 = None
    for name, weights, variant, omega in (("rav", "pou", rg.VARIANT_ROWS, 0.66),
                                          ("diag_vanka", "full", rg.VARIANT_DIAG, 0.1),
                                          ("mv_color", "full", rg.VARIANT_MV, 0.66)):
        G = rg.gen_level(prob, weights)
        t0 = time.perf_counter()
        sm = rg.Smoother(G, G, variant=variant)
        if variant == rg.VARIANT_MV:
            sm.set_colors(*rg.multicolor(prob))
        torch.cuda.synchronize()
        setup_s = time.perf_counter() - t0
        if x0 is None:
            x0 = torch.tensor(si.initial_guess(G["n"], seed=si.X0_SEED), device="cuda")
        b = G["b"]
        r0 = float(torch.linalg.vector_norm(sm.residual(x0, b)))
        x = x0.clone()
        sm.smooth(x, b, 50, omega)     # warm-up (graph capture)
        x = x0.clone()
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(stream)
        sm.smooth(x, b, 50, omega)
        e1.record(stream)
        torch.cuda.synchronize()
        ms = e0.elapsed_time(e1) / 50
        r50 = float(torch.linalg.vector_norm(sm.residual(x, b)))
        out[name] = {"ms_per_sweep": ms, "mdofs": G["n"] / (ms * 1e-3) / 1e6, "omega": omega,
                     "residual_reduction_50": r50 / r0, "setup_s": setup_s, "kernel": sm.kernel_name,
                     "factor_bytes_per_sweep": sm.sweep_bytes()["sweep"]}
        if name == "rav":   # the two kernels of the sweep alone at this size (roofline, DESIGN 5.1)
            peak = load_peaks()[0]
            r = sm.residual(x0, b)
            for kname, fn, nbytes in (("sweep_kernel", lambda: sm.apply(r, x, omega), sm.sweep_bytes()["sweep"]),
                                      ("residual_kernel", lambda: sm.residual(x, b, r), sm.sweep_bytes()["residual"])):
                for _ in range(3):
                    fn()
                torch.cuda.synchronize()
                e0.record(stream)
                for _ in range(20):
                    fn()
                e1.record(stream)
                torch.cuda.synchronize()
                kms = e0.elapsed_time(e1) / 20
                out[name][kname] = {"ms": kms, "algorithmic_bytes": nbytes,
                                    "achieved_gbs": nbytes / (kms * 1e-3) / 1e9,
                                    "frac_of_measured_peak": nbytes / (kms * 1e-3) / 1e9 / peak}
        sm.close()
        del sm, G, x, b
        torch.cuda.empty_cache()
    return out


def run_vcycle_smoothers(rg, si, stream):
    """The paper's smoother comparison (Figs. 4-5) as GPU V-cycles:
    512^2 MMS with seeded eta, 8 levels (4^2 coarsest), x0 = 0, rtol 1e-8;
    RAV / MV (0.66, V(2,2)), diagonal Vanka (0.1, V(2,2)), AV (0.1, V(3,3))."""
    import torch
    prob = si.problem(2, (512, 512), si.KIND_MMS, eta="fourier")
    out = {"config": "512^2 Q2-Q1 MMS, seeded eta, 8 levels, x0 = 0, rtol 1e-8"}
    for name, weights, variant, omega, pre in (("rav", "pou", rg.VARIANT_ROWS, 0.66, 2),
                                               ("mv_color", "full", rg.VARIANT_MV, 0.66, 2),
                                               ("diag_vanka", "full", rg.VARIANT_DIAG, 0.1, 2),
                                               ("av", "full", rg.VARIANT_ROWS, 0.1, 3)):
        mg, fine = rg.build_hierarchy(prob, 8, weights, variant=variant)
        x = torch.zeros(fine["n"], dtype=torch.float64, device="cuda")
        mg.solve(x, fine["b"], pre=pre, post=pre, omega=omega, rtol=1e-8, maxit=2)   # warm
        x.zero_()
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(stream)
        try:
            x, k, h = mg.solve(x, fine["b"], pre=pre, post=pre, omega=omega, rtol=1e-8, maxit=400)
        except rg.RavError as err:   # diagonal Vanka diverges on this problem (oracle too)
            torch.cuda.synchronize()
            out[name] = {"converged": False, "diverged": str(err)[:120], "pre_post": pre, "omega": omega}
            mg.close()
            continue
        e1.record(stream)
        torch.cuda.synchronize()
        t = e0.elapsed_time(e1) / 1e3
        out[name] = {"cycles": k, "converged": bool(h[-1] <= 1e-8 * h[0]), "time_s": t,
                     "ms_per_cycle": t / max(k, 1) * 1e3, "pre_post": pre, "omega": omega,
                     "avg_reduction_factor": (h[-1] / h[0]) ** (1.0 / max(k, 1))}
        mg.close()
        del mg, fine, x
        torch.cuda.empty_cache()
    return out


def _timed_solve(rg, prob, levels, weights, variant, omega, pre, stream, rtol=1e-8, maxit=400):
    """Build a GPU hierarchy and time mg_solve (CUDA events, after a warm-up that
    captures the V-cycle graph).  Returns a dict (or a divergence record)."""
    import torch
    mg, fine = rg.build_hierarchy(prob, levels, weights, variant=variant)
    x = torch.zeros(fine["n"], dtype=torch.float64, device="cuda")
    out = {"pre_post": pre, "omega": omega}
    try:
        mg.solve(x, fine["b"], pre=pre, post=pre, omega=omega, rtol=rtol, maxit=2)
        x.zero_()
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(stream)
        x, k, h = mg.solve(x, fine["b"], pre=pre, post=pre, omega=omega, rtol=rtol, maxit=maxit)
        e1.record(stream)
        torch.cuda.synchronize()
        t = e0.elapsed_time(e1) / 1e3
        out.update({"cycles": k, "converged": bool(h[-1] <= rtol * h[0]), "time_s": t,
                    "ms_per_cycle": t / max(k, 1) * 1e3,
                    "avg_reduction_factor": (h[-1] / h[0]) ** (1.0 / max(k, 1))})
    except rg.RavError as err:
        torch.cuda.synchronize()
        out.update({"converged": False, "diverged": str(err)[:120]})
    out["free_dofs"] = fine["n"]
    mg.close()
    del mg, fine, x
    torch.cuda.empty_cache()
    return out


def run_q1q1_studies(rg, si, stream):
    """The paper's own discretization (stabilized Q1-Q1; SURVEY section 8
    row f1) in the paper's driven-cavity setting on uniform grids: coarse grid
    8x8, V(3,3), RAV / MV omega 0.66, AV omega 0.1,
    1e8 reduction.  (a) convergence study over the grid hierarchy (Figs. 4-5:
    cycles, average reduction factor, runtime per cycle, total runtime);
    (b) smoothing-step study n_S = 1..6 on 512^2 (Fig. 7 / P:199-213);
    (c) RAV sweep throughput on a 2048^2 Q1-Q1 level."""
    import math
    import torch
    smoothers = (("rav", "pou", rg.VARIANT_ROWS, 0.66), ("mv_color", "full", rg.VARIANT_MV, 0.66),
                 ("av", "full", rg.VARIANT_ROWS, 0.1))
    out = {"config": "Q1-Q1 stabilized (beta = 0.01/eta, R18) lid-driven cavity, eta = 1, uniform grids, "
                     "8x8 coarsest, x0 = 0, rtol 1e-8"}
    study = {}
    for n in (64, 128, 256, 512, 1024):
        prob = si.problem(2, (n, n), si.KIND_CAVITY, elem=si.ELEM_Q1Q1)
        lv = int(math.log2(n // 8)) + 1
        study[f"{n}x{n}"] = {name: _timed_solve(rg, prob, lv, w, v, om, 3, stream)
                             for name, w, v, om in smoothers}
    out["convergence_study_V33"] = study
    # the same at SPEC's beta = 0.1 / eta beside the beta_0 = 0.01 of R18, which was
    # chosen by a beta study (DESIGN R18): f1 reported at both values
    study = {}
    for n in (64, 256, 1024):
        prob = si.problem(2, (n, n), si.KIND_CAVITY, elem=si.ELEM_Q1Q1, beta=0.1)
        lv = int(math.log2(n // 8)) + 1
        study[f"{n}x{n}"] = {name: _timed_solve(rg, prob, lv, w, v, om, 3, stream, maxit=200)
                             for name, w, v, om in smoothers}
    out["convergence_study_V33_beta0_0.1"] = study
    steps = {}
    prob = si.problem(2, (512, 512), si.KIND_CAVITY, elem=si.ELEM_Q1Q1)
    for ns in range(1, 7):
        steps[f"nS={ns}"] = {name: _timed_solve(rg, prob, 7, w, v, om, ns, stream, maxit=300)
                             for name, w, v, om in smoothers}
    out["smoothing_steps_512"] = steps
    # RAV sweep throughput (residual + sweep) on 2048^2 Q1-Q1 with the seeded viscosity
    prob = si.problem(2, (2048, 2048), si.KIND_MMS, eta="fourier", elem=si.ELEM_Q1Q1)
    G = rg.gen_level(prob, "pou")
    sm = rg.Smoother(G, G)
    x = torch.tensor(si.initial_guess(G["n"], seed=si.X0_SEED), device="cuda")
    sm.smooth(x, G["b"], 10, 0.66)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(stream)
    sm.smooth(x, G["b"], 50, 0.66)
    e1.record(stream)
    torch.cuda.synchronize()
    ms = e0.elapsed_time(e1) / 50
    by = sm.sweep_bytes()
    out["rav_sweep_2048"] = {"free_dofs": G["n"], "ms_per_sweep": ms, "mdofs": G["n"] / (ms * 1e-3) / 1e6,
                             "kernel": sm.kernel_name, "algorithmic_gb_per_sweep": (by["sweep"] + by["residual"]) / 1e9,
                             "achieved_gbs": (by["sweep"] + by["residual"]) / (ms * 1e-3) / 1e9}
    sm.close()
    del sm, G, x
    torch.cuda.empty_cache()
    return out


def run_adaptive_study(rg, si, stream, max_levels=7):
    """The paper's driven-cavity convergence study (Figs. 4-5) on its own grid
    hierarchy: stabilized Q1-Q1 on the adaptive grids of Table 1 (reading R20: level
    counts reproduced exactly), M^2 .. M^7 with the 8x8 grid as the coarse grid,
    V(3,3), RAV / multicoloured MV omega 0.66, AV omega 0.1, 1e8 reduction."""
    import torch
    prob = si.problem(2, (8, 8), si.KIND_CAVITY, elem=si.ELEM_Q1Q1)
    out = {"config": "driven cavity, stabilized Q1-Q1 (beta_0 = 0.01, R18), eta = 1, adaptive hierarchy of "
                     "Table 1 (R20), V(3,3), x0 = 0, rtol 1e-8"}
    for L in range(2, max_levels + 1):
        row = {}
        for name, w, v, om in (("rav", "own", rg.VARIANT_ROWS, 0.66), ("mv_color", "full", rg.VARIANT_MV, 0.66),
                               ("av", "full", rg.VARIANT_ROWS, 0.1)):
            t0 = time.perf_counter()
            mg, fine = rg.build_adaptive_hierarchy(prob, L, w, variant=v)
            torch.cuda.synchronize()
            setup = time.perf_counter() - t0
            x = torch.zeros(fine["n"], dtype=torch.float64, device="cuda")
            r = {"setup_s": setup}
            try:
                mg.solve(x, fine["b"], pre=3, post=3, omega=om, rtol=1e-8, maxit=2)
                x.zero_()
                torch.cuda.synchronize()
                e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                e0.record(stream)
                x, k, h = mg.solve(x, fine["b"], pre=3, post=3, omega=om, rtol=1e-8, maxit=400)
                e1.record(stream)
                torch.cuda.synchronize()
                t = e0.elapsed_time(e1) / 1e3
                r.update({"cycles": k, "converged": bool(h[-1] <= 1e-8 * h[0]), "time_s": t,
                          "ms_per_cycle": t / max(k, 1) * 1e3,
                          "avg_reduction_factor": (h[-1] / h[0]) ** (1.0 / max(k, 1))})
            except rg.RavError as err:
                r.update({"converged": False, "diverged": str(err)[:120]})
            row[name] = r
            mg.close()
            del mg, x
            torch.cuda.empty_cache()
        row["elements"] = fine["n_cells"]
        row["dofs"] = fine["n"]
        out[f"M{L}"] = row
    # smoothing-step study on M6 (Fig. 7 / P:199-213, here on the cavity's own adaptive grids)
    steps = {}
    for ns in range(1, 7):
        row = {}
        for name, w, v, om in (("rav", "own", rg.VARIANT_ROWS, 0.66), ("mv_color", "full", rg.VARIANT_MV, 0.66),
                               ("av", "full", rg.VARIANT_ROWS, 0.1)):
            mg, fine = rg.build_adaptive_hierarchy(prob, 6, w, variant=v)
            x = torch.zeros(fine["n"], dtype=torch.float64, device="cuda")
            r = {}
            try:
                mg.solve(x, fine["b"], pre=ns, post=ns, omega=om, rtol=1e-8, maxit=2)
                x.zero_()
                torch.cuda.synchronize()
                e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                e0.record(stream)
                x, k, h = mg.solve(x, fine["b"], pre=ns, post=ns, omega=om, rtol=1e-8, maxit=300)
                e1.record(stream)
                torch.cuda.synchronize()
                r = {"cycles": k, "converged": bool(h[-1] <= 1e-8 * h[0]), "time_s": e0.elapsed_time(e1) / 1e3,
                     "avg_reduction_factor": (h[-1] / h[0]) ** (1.0 / max(k, 1))}
            except rg.RavError as err:
                r = {"converged": False, "diverged": str(err)[:120]}
            row[name] = r
            mg.close()
            del mg, x
            torch.cuda.empty_cache()
        steps[f"nS={ns}"] = row
    out["smoothing_steps_M6"] = steps
    return out


class LineGuard:
    """Keeps the N > 1 bench line if a measurement added after it stalls: when `limit_s` passes
    before finish(), rank 0 prints the line as it stands (plus "extras_timeout_s") and every rank
    exits 0 without the communicator teardown (which would wait on the stalled collective)."""

    def __init__(self, line, rank, limit_s, exit_fn=os._exit, out=None):
        self.line, self.rank, self.limit_s = line, rank, limit_s
        self.exit_fn, self.out = exit_fn, out
        self.lock = threading.Lock()
        self.done = False
        self.timer = threading.Timer(limit_s, self._expire)
        self.timer.daemon = True
        self.timer.start()

    def _expire(self):
        with self.lock:
            if self.done:
                return
            self.done = True
            if self.rank == 0:
                snap = {k: v for k, v in list(self.line.items())}
                snap["extras_timeout_s"] = self.limit_s
                print(json.dumps(snap, default=str), file=self.out or sys.stdout, flush=True)
        self.exit_fn(0)

    def finish(self) -> bool:
        """True: the caller prints the line; False: the limit already fired and printed it."""
        with self.lock:
            if self.done:
                return False
            self.done = True
        self.timer.cancel()
        return True


def _transport():
    """RAV_MGD_TRANSPORT=peer: the peer-memory transport (mgd_setup via_comm = 2: pack kernels store
    into the neighbour's receive buffer over NVLink and release its flag); default nccl."""
    return "peer" if os.environ.get("RAV_MGD_TRANSPORT", "nccl") == "peer" else "nccl"


def _dist_build(rdist, rg, prob, levels, ws, rank, comm, gather, stream, **kw):
    """One rank's share of the library-driven slab-partitioned hierarchy (mgd_setup)."""
    if _transport() == "peer" and kw.get("variant", 0) != 2:
        kw.setdefault("via_comm", 2)
    return rdist.build_lib_dist(prob, levels, ws, [rank], list(range(ws)), comm, gather=gather, stream=stream, **kw)


def run_dist_vcycle(name, rdist, rg, si, stream, dist, ws, rank, comm, gather):
    """Slab-partitioned V-cycle to rtol on ws GPUs (strong scaling of c3 / c4) inside the library
    (mgd_solve): partitioned fine levels with NCCL interface sums / halo refreshes, windowed
    transfers, the coarse levels agglomerated (all-gathered rhs summed in subdomain order, solved
    redundantly on every rank); ||r||^2 all-gathered per cycle; every cycle one CUDA graph.
    Device time with CUDA events around the solve, max over ranks."""
    import torch
    c = si.CONFIGS[name]
    prob = si.config_problem(name)
    t0 = time.perf_counter()
    mgd, info = _dist_build(rdist, rg, prob, c["levels"], ws, rank, comm, gather, stream)
    torch.cuda.synchronize()
    setup_s = time.perf_counter() - t0
    xs, bs = info["x"], info["b"]
    mgd.solve(xs, bs, pre=c["pre"], post=c["post"], omega=c["omega"], rtol=c["rtol"], maxit=2)   # warm (capture)
    times = []
    for _ in range(2):
        for x in xs:
            x.zero_()
        torch.cuda.synchronize()
        dist.barrier()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(stream)
        _, iters, hist = mgd.solve(xs, bs, pre=c["pre"], post=c["post"], omega=c["omega"], rtol=c["rtol"], maxit=100)
        e1.record(stream)
        torch.cuda.synchronize()
        times.append(e0.elapsed_time(e1) / 1e3)
    enq, wait, ncyc = mgd.host_time()
    tt = torch.tensor([min(times)], device="cuda")
    dist.all_reduce(tt, op=dist.ReduceOp.MAX)
    t = float(tt.item())
    slab = info["slabs"][0][0]
    out = {"config": VCYCLE_DESC[name] + f"; slab-partitioned over {ws} GPUs (library mgd_solve, NCCL)",
           "free_dofs": slab.nvel_glob + slab.nvert_glob, "rtol": c["rtol"], "cycles": iters,
           "converged": bool(hist[-1] <= c["rtol"] * hist[0]), "time_to_rtol_s": t,
           "ms_per_cycle": t / max(iters, 1) * 1e3, "partitioned_levels": info["K"],
           "partition": [list(p) for p in info["parts"][0]], "setup_s": setup_s,
           "host_enqueue_ms_per_cycle": enq / max(ncyc, 1) * 1e3, "gpu_launches": mgd.last_launches,
           "timing": "CUDA events around mgd_solve, best of 2, max over ranks"}
    mgd.close()
    del mgd, info, xs, bs
    torch.cuda.empty_cache()
    return out


def run_dist_c5(rdist, rg, si, stream, dist, ws, rank, comm, gather):
    """BASELINE config 5 at N GPUs (weak scaling): 2048^2 Q2-Q1 per GPU stacked in y, slab-
    partitioned; 50 sweeps each of RAV (omega 0.66), diagonal Vanka (omega 0.1) and multicoloured
    MV (omega 0.66) from the seeded N(0,1) guess through mgd_smooth (every sweep with its interface
    exchanges over NCCL; MV: one exchange pair per colour).  Device time, max over ranks."""
    import torch
    prob = si.config_problem("c5", scale_y=ws)
    out = {"config": f"c5 weak scaling: 2048 x {2048 * ws} Q2-Q1 MMS on [0,1]x[0,{ws}], seeded eta, "
                     f"slab-partitioned over {ws} GPUs, 50 sweeps from seeded N(0,1)"}
    for name, weights, variant, omega in (("rav", "pou", rg.VARIANT_ROWS, 0.66),
                                          ("diag_vanka", "full", rg.VARIANT_DIAG, 0.1),
                                          ("mv_color", "full", rg.VARIANT_MV, 0.66)):
        try:
            mgd, info = _dist_build(rdist, rg, prob, 1, ws, rank, comm, gather, stream, weights=weights,
                                    variant=variant, smooth_only=True)
            slab = info["slabs"][0][0]
            nglob = slab.nvel_glob + slab.nvert_glob
            x0 = torch.tensor(si.initial_guess(nglob, seed=si.X0_SEED)[slab.global_ids()], device="cuda")
            b = info["b"][0]
            r0 = mgd.residual_norm([x0], [b])
            x = x0.clone()
            mgd.smooth([x], [b], 50, omega)      # warm (capture)
            x.copy_(x0)
            torch.cuda.synchronize()
            dist.barrier()
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record(stream)
            mgd.smooth([x], [b], 50, omega)
            e1.record(stream)
            torch.cuda.synchronize()
            t = torch.tensor([e0.elapsed_time(e1) / 50], device="cuda")
            dist.all_reduce(t, op=dist.ReduceOp.MAX)
            ms = float(t.item())
            out[name] = {"ms_per_sweep": ms, "mdofs": nglob / (ms * 1e-3) / 1e6, "omega": omega,
                         "residual_reduction_50": mgd.residual_norm([x], [b]) / r0}
            mgd.close()
            del mgd, info, x, x0, b
            torch.cuda.empty_cache()
        except Exception as err:  # report, keep the line
            out[name] = {"error": f"{type(err).__name__}: {err}"[:200]}
    return out


def run_gpu_dist(args):
    """N > 1 (torchrun): weak scaling of the c2 workload, one 512^2 block per GPU stacked along y
    (BASELINE config 5's layout), slab-partitioned inside the library: every sweep runs the
    interface-correction sum and the halo refresh over NCCL (mgd_smooth, one CUDA graph per step).
    torch.distributed (NCCL) is the plumbing: the library communicator's NCCL id, the host
    all-gather of the exchange plans, barriers and the max-over-ranks timing."""
    import torch
    import torch.distributed as dist
    ws, rank, local = dist_env()
    torch.cuda.set_device(local)
    dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    from paper_2103_10127_b200 import dist as rdist
    from paper_2103_10127_b200 import ravgmg as rg
    import seeded_inputs as si

    obj = [rg.Comm.unique_id() if rank == 0 else None]
    dist.broadcast_object_list(obj, src=0)
    comm = rg.Comm(ws, rank, obj[0])

    def gather(o):
        out = [None] * ws
        dist.all_gather_object(out, o)
        return out

    stream = torch.cuda.Stream()
    torch.cuda.set_stream(stream)
    prob = si.config_problem("c2", scale_y=ws)
    t0 = time.perf_counter()
    mgd, info = _dist_build(rdist, rg, prob, 1, ws, rank, comm, gather, stream, smooth_only=True)
    torch.cuda.synchronize()
    setup_s = time.perf_counter() - t0
    slab = info["slabs"][0][0]
    n_glob = slab.nvel_glob + slab.nvert_glob
    x0 = torch.tensor(si.initial_guess(n_glob, seed=si.X0_SEED)[slab.global_ids()], device="cuda")
    x, b = x0.clone(), info["b"][0]

    for _ in range(args.warmup):
        mgd.smooth([x], [b], SWEEPS_PER_STEP, OMEGA)
    launches_per_step = mgd.last_launches
    torch.cuda.synchronize()
    dist.barrier()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    with ClockSampler(local) as clk:
        e0.record(stream)
        for _ in range(args.steps):
            mgd.smooth([x], [b], SWEEPS_PER_STEP, OMEGA)
        e1.record(stream)
        torch.cuda.synchronize()
    dist.barrier()
    torch.cuda.synchronize()
    t = torch.tensor([e0.elapsed_time(e1)], device="cuda")
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    ms_per_step = float(t.item()) / args.steps
    value = n_glob * SWEEPS_PER_STEP / (ms_per_step * 1e-3) / 1e6
    assert torch.isfinite(x).all()

    # dominant kernel alone on this rank (its window's patches), through a single-domain smoother
    L = mgd._keep[0][0][0]["level"]
    sm = rg.Smoother(L, L)
    r = sm.residual(x, b)
    for _ in range(5):
        sm.apply(r, x, OMEGA)
    torch.cuda.synchronize()
    e0.record(stream)
    for _ in range(50):
        sm.apply(r, x, OMEGA)
    e1.record(stream)
    torch.cuda.synchronize()
    sweep_ms = e0.elapsed_time(e1) / 50
    bytes_info = sm.sweep_bytes()
    peak, peak_kind = load_peaks()
    achieved = bytes_info["sweep"] / (sweep_ms * 1e-3) / 1e9
    kname = sm.kernel_name
    sm.close()
    del sm

    # end to end: pinned host x / b in, the iterate out, every step
    xh = x0.cpu().pin_memory()
    bh = b.cpu().pin_memory()
    dist.barrier()
    torch.cuda.synchronize()
    e0.record(stream)
    for _ in range(args.steps):
        x.copy_(xh, non_blocking=True)
        b.copy_(bh, non_blocking=True)
        mgd.smooth([x], [b], SWEEPS_PER_STEP, OMEGA)
        xh.copy_(x, non_blocking=True)
    e1.record(stream)
    torch.cuda.synchronize()
    t = torch.tensor([e0.elapsed_time(e1)], device="cuda")
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    e2e_value = n_glob * SWEEPS_PER_STEP * args.steps / (float(t.item()) * 1e-3) / 1e6

    line = {
        "metric": "RAV sweep throughput (c2: 512^2 Q2-Q1, variable viscosity)",
        "value": value, "unit": "MDoF/s", "n_gpus": ws, "steps": args.steps, "warmup": args.warmup,
        "ms_per_step": ms_per_step, "higher_is_better": True, "scaling": "weak", "vs_baseline": None,
        "dtype": "f64", "data": "synthetic",
        "config": {"workload": f"c2 per GPU stacked along y: 512 x {512 * ws} Q2-Q1 cells on [0,1]x[0,{ws}], "
                               "MMS forcing, seeded eta; step = 100 slab-partitioned RAV sweeps inside the library "
                               "(residual, RAV sweep, NCCL interface-correction sum + halo refresh; one CUDA graph)",
                   "free_dofs": n_glob, "sweeps_per_step": SWEEPS_PER_STEP, "omega": OMEGA,
                   "parallelism": f"slab partition x{ws} (mgd_smooth, "
                                  + ("peer-memory transport over NVLink)" if _transport() == "peer"
                                     else "NCCL point-to-point)"),
                   "partition": [list(p) for p in info["parts"][0]],
                   "l2": "inputs larger than L2 (factor rows + node-blocked operator stream from HBM every sweep)"},
        "roofline": {"bound": "hbm", "achieved": achieved, "peak": peak, "unit": "GB/s", "frac": achieved / peak,
                     "traffic": None, "peak_kind": peak_kind, "kernel": kname + " via rav_apply (rank 0's window)",
                     "kernel_ms": sweep_ms, "algorithmic_bytes_per_launch": bytes_info["sweep"]},
        "setup_s": setup_s,
        "e2e": {"value": e2e_value, "unit": "MDoF/s", "h2d_bytes_per_step": 16 * slab.n_loc * ws,
                "d2h_bytes_per_step": 8 * slab.n_loc * ws},
        "gpu_launches": launches_per_step * args.steps,
        "clocks": clk.summary(),
    }
    mgd.close()
    del mgd, info, x, x0, b
    torch.cuda.empty_cache()
    # The sweep line above is the contract's line; what follows only adds keys to it.  If an added
    # measurement stalls on some rank (a collective waiting on a rank that raised), every rank
    # leaves after the limit and rank 0 still prints the line, with the stall named in it.
    guard = LineGuard(line, rank, float(os.environ.get("RAV_BENCH_EXTRAS_LIMIT_S", "900")))
    if not args.no_smoothers:
        try:
            line["c5_smoothers"] = run_dist_c5(rdist, rg, si, stream, dist, ws, rank, comm, gather)
        except Exception as e:  # report, keep the sweep line
            line["c5_smoothers"] = {"error": f"{type(e).__name__}: {e}"[:300]}
    if not args.no_vcycle:
        vc = {}
        for name in ("c3", "c4"):
            try:
                vc[name] = run_dist_vcycle(name, rdist, rg, si, stream, dist, ws, rank, comm, gather)
            except Exception as e:  # report, keep the sweep line
                vc[name] = {"error": f"{type(e).__name__}: {e}"[:300]}
        line["vcycle"] = vc
    if not guard.finish():
        return 0
    if rank == 0:
        print(json.dumps(line), flush=True)
    comm.close()
    dist.destroy_process_group()
    return 0


def run_gpu(args):
    if dist_env()[0] > 1:
        return run_gpu_dist(args)
    import numpy as np
    import torch
    ws, rank, local = dist_env()
    torch.cuda.set_device(local)
    dist = None
    if ws > 1:
        import torch.distributed as dist
        dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    from paper_2103_10127_b200 import ravgmg as rg
    import seeded_inputs as si

    prob = si.config_problem("c2")
    # a non-default stream: the library captures sweep sequences / V-cycles as CUDA graphs on it
    stream = torch.cuda.Stream()
    torch.cuda.set_stream(stream)
    t_setup0 = time.perf_counter()
    G = rg.gen_level(prob, "pou")
    torch.cuda.synchronize()
    t_gen = time.perf_counter() - t_setup0
    t1 = time.perf_counter()
    sm = rg.Smoother(G, G)
    torch.cuda.synchronize()
    t_factor = time.perf_counter() - t1
    n = G["n"]
    nnz_c2, npatch_c2 = G["nnz"], len(G["offs"]) - 1
    b = G["b"]
    x0 = torch.tensor(si.initial_guess(n, seed=si.X0_SEED), device="cuda")
    x = x0.clone()
    bytes_info = sm.sweep_bytes()

    def barrier():
        if dist is not None:
            dist.barrier()

    # ---- device-timed steps: rav_smooth(nu = 100) --------------------------------
    for _ in range(args.warmup):
        sm.smooth(x, b, SWEEPS_PER_STEP, OMEGA)
    launches_per_step = sm.last_launches
    torch.cuda.synchronize()
    barrier()
    torch.cuda.synchronize()
    ev0, ev1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    with ClockSampler(local) as clk:
        ev0.record(stream)
        for _ in range(args.steps):
            sm.smooth(x, b, SWEEPS_PER_STEP, OMEGA)
        ev1.record(stream)
        torch.cuda.synchronize()
    barrier()
    torch.cuda.synchronize()
    ms = ev0.elapsed_time(ev1)
    if dist is not None:
        t = torch.tensor([ms], device="cuda")
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        ms = float(t.item())
    ms_per_step = ms / args.steps
    value = ws * n * SWEEPS_PER_STEP / (ms_per_step * 1e-3) / 1e6
    assert torch.isfinite(x).all()

    # ---- dominant kernel alone (sweep, rav_apply) and the residual SpMV ------------
    r = sm.residual(x, b)
    nk = 50
    for _ in range(5):
        sm.apply(r, x, OMEGA)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(stream)
    for _ in range(nk):
        sm.apply(r, x, OMEGA)
    e1.record(stream)
    torch.cuda.synchronize()
    sweep_ms = e0.elapsed_time(e1) / nk
    for _ in range(5):
        sm.residual(x, b, r)
    torch.cuda.synchronize()
    e0.record(stream)
    for _ in range(nk):
        sm.residual(x, b, r)
    e1.record(stream)
    torch.cuda.synchronize()
    resid_ms = e0.elapsed_time(e1) / nk
    peak, peak_kind = load_peaks()
    achieved = bytes_info["sweep"] / (sweep_ms * 1e-3) / 1e9
    kernel_name = sm.kernel_name
    # DRAM traffic per launch from the committed ncu capture of this same kernel (or null)
    traffic = None
    tpath = os.path.join(ROOT, "profiles", "sweep_traffic.json")
    if os.path.exists(tpath):
        try:
            tj = json.load(open(tpath))
            if kernel_name.split(" ")[0] in tj.get("kernel", ""):
                traffic = tj.get("bytes_per_launch")
        except Exception:
            traffic = None

    # ---- deterministic scatter mode (R16): same sweeps, slot writes + ordered per-DoF sums ----
    det = None
    try:
        smd = rg.Smoother(G, G, deterministic=True)
        xd = x0.clone()
        smd.smooth(xd, b, SWEEPS_PER_STEP, OMEGA)       # warm (graph)
        xd = x0.clone()
        torch.cuda.synchronize()
        e0.record(stream)
        smd.smooth(xd, b, SWEEPS_PER_STEP, OMEGA)
        e1.record(stream)
        torch.cuda.synchronize()
        dms = e0.elapsed_time(e1) / SWEEPS_PER_STEP
        det = {"ms_per_sweep": dms, "mdofs": n / (dms * 1e-3) / 1e6, "kernel": smd.kernel_name + " + det_gather_kernel"}
        smd.close()
        del smd, xd
    except Exception as err:  # report, keep the line
        det = {"error": f"{type(err).__name__}: {err}"[:200]}

    # ---- end to end through the C-ABI with host buffers ----------------------------
    # K steps = K independent problems (the seeded x0, b) in pinned host memory through
    # rav_smooth_batch: every step copies its x and b host -> device and its result device -> host
    # inside the timed region; the library overlaps those copies with the neighbouring steps' sweeps
    x0h = x0.cpu()
    bh = b.cpu().pin_memory()
    xh = [x0h.clone().pin_memory() for _ in range(args.steps)]
    nw = min(2, args.steps)
    sm.smooth_batch(xh[:nw], [bh] * nw, SWEEPS_PER_STEP, OMEGA)   # warm (staging buffers, both graphs)
    for t_ in xh[:nw]:
        t_.copy_(x0h)
    barrier()
    t0 = time.perf_counter()
    sm.smooth_batch(xh, [bh] * args.steps, SWEEPS_PER_STEP, OMEGA)
    e2e_s = time.perf_counter() - t0
    if not torch.equal(xh[-1], xh[0]):   # independent identical problems: the same result (to atomics)
        assert float((xh[-1] - xh[0]).abs().max()) <= 1e-10 * float(xh[0].abs().max()), "batch results differ"
    del xh
    if dist is not None:
        t = torch.tensor([e2e_s], device="cuda")
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        e2e_s = float(t.item())
    e2e_value = ws * n * SWEEPS_PER_STEP * args.steps / e2e_s / 1e6

    # ---- V-cycle time to 1e-8 on c3 (2048^2, 10 levels) and c4, BASELINE metric part 2 ----
    del sm, G
    torch.cuda.empty_cache()
    extra = {}
    if not args.no_smoothers and ws == 1:
        extra["c5_smoothers"] = run_c5_smoothers(rg, si, stream)
    vcyc = None
    if not args.no_vcycle:
        vcyc = {"c1": run_c1(rg, si)}
        vcyc.update({name: run_vcycle(name, rg, si, stream, dist) for name in ("c3", "c4")})
    if args.studies and ws == 1:   # the paper-setting studies (rows f1, f2, f4), to their own file
        studies = {"vcycle_smoothers": run_vcycle_smoothers(rg, si, stream),
                   "q1q1_paper_setting": run_q1q1_studies(rg, si, stream),
                   "adaptive_cavity_table1": run_adaptive_study(rg, si, stream)}
        with open(args.studies, "w") as f:
            json.dump(studies, f)

    # ---- CPU oracle baseline (rank 0, N = 1 only; bounded sample) ------------------
    cpu = None
    if rank == 0 and ws == 1 and not args.no_cpu_baseline:
        rate, cores, sample, _ = cpu_oracle_rate(prob, steps=3, warmup=1)
        rate1, _, sample1, _ = cpu_oracle_rate(prob, steps=2, warmup=0, threads=1)
        cpu = {"value": rate, "unit": "MDoF/s", "cores": cores, "kind": "oracle", "sample": sample,
               "single_thread": {"value": rate1, "unit": "MDoF/s", "cores": 1, "sample": sample1},
               "host": host_info()}
        try:
            cpu["per_sweep"] = oracle_sweep_samples(si, os.cpu_count() or 1)
        except Exception as err:  # report, keep the line
            cpu["per_sweep"] = {"error": f"{type(err).__name__}: {err}"[:200]}

    clocks = clk.summary()
    line = {
        "metric": "RAV sweep throughput (c2: 512^2 Q2-Q1, variable viscosity)",
        "value": value, "unit": "MDoF/s", "n_gpus": ws, "steps": args.steps, "warmup": args.warmup,
        "ms_per_step": ms_per_step, "higher_is_better": True, "scaling": "weak", "vs_baseline": None,
        "dtype": "f64", "data": "synthetic",
        "config": {"workload": "c2: 2D 512x512 Taylor-Hood Q2-Q1, MMS forcing, seeded eta in [0.1,10]; "
                               "step = 100 RAV sweeps (residual SpMV + RAV sweep) from seeded N(0,1)",
                   "free_dofs": n, "nnz": nnz_c2, "patches": npatch_c2,
                   "sweeps_per_step": SWEEPS_PER_STEP, "omega": OMEGA, "weights": "partition of unity (R3)",
                   "l2": "inputs larger than L2 (per sweep the factored Schur rows, 0.58 GB, and the node-blocked "
                         "operator, 0.22 GB with its B values in an L1-resident table, stream from HBM; x, r, b "
                         "vectors, 19 MB each, stay L2-resident by design)",
                   "parallelism": f"replicas x{ws}" if ws > 1 else "1 GPU"},
        "roofline": {"bound": "hbm", "achieved": achieved, "peak": peak, "unit": "GB/s",
                     "frac": achieved / peak, "traffic": traffic, "peak_kind": peak_kind,
                     "kernel": kernel_name + " via rav_apply", "kernel_ms": sweep_ms,
                     "algorithmic_bytes_per_launch": bytes_info["sweep"]},
        "residual_kernel": {"ms": resid_ms, "algorithmic_bytes": bytes_info["residual"],
                            "achieved_gbs": bytes_info["residual"] / (resid_ms * 1e-3) / 1e9},
        "sweep_total": {"ms_per_sweep": ms_per_step / SWEEPS_PER_STEP,
                        "algorithmic_bytes": bytes_info["sweep"] + bytes_info["residual"],
                        "achieved_gbs": (bytes_info["sweep"] + bytes_info["residual"]) /
                                        (ms_per_step / SWEEPS_PER_STEP * 1e-3) / 1e9},
        "setup_s": {"generate": t_gen, "factorize": t_factor},
        "e2e": {"value": e2e_value, "unit": "MDoF/s", "h2d_bytes_per_step": 2 * 8 * n,
                "d2h_bytes_per_step": 8 * n,
                "how": "rav_smooth_batch over the K steps as K independent problems in pinned host memory "
                       "(wall clock around the call); each step's x, b copied in and x copied out inside the "
                       "timed region, overlapped by the library with the neighbouring steps' sweeps"},
        "gpu_launches": launches_per_step * args.steps,
        "clocks": clocks,
    }
    if cpu is not None:
        line["cpu_baseline"] = cpu
    if det is not None:
        line["deterministic_mode"] = det
    line.update(extra)
    if vcyc is not None:
        line["vcycle"] = vcyc          # last: the record keeps the tail of the line
    if rank == 0:
        print(json.dumps(line), flush=True)
    if dist is not None:
        dist.destroy_process_group()
    return 0


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=10)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-vcycle", action="store_true", help="skip the c3 V-cycle time-to-1e-8 measurement")
    ap.add_argument("--no-smoothers", action="store_true", help="skip the c5 / V-cycle smoother comparisons")
    ap.add_argument("--studies", default="", help="also run the paper-setting studies (V-cycle smoother "
                    "comparison, Q1-Q1, adaptive hierarchy) and write them to this JSON file")
    args = ap.parse_args()
    if args.warmup < 3 and args.impl == "ours":
        print("warning: --warmup < 3 violates the timing rules", file=sys.stderr)
    if args.impl == "reference":
        return run_reference(args)
    return run_gpu(args)


if __name__ == "__main__":
    sys.exit(main())
