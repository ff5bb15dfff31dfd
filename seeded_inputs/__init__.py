"""Seeded synthetic inputs shared by the oracle (``oracle/``) and the CUDA path
(``paper_2103_10127_b200/``).

This module holds NO arithmetic of the method (no assembly, no patches, no
smoother, no multigrid).  It only draws the random numbers the workloads need and
describes the synthetic problems, so that both sides receive identical inputs:

* ``viscosity_params``: the seeded variable-viscosity field of BASELINE.json
  configs 2-5 ("nu = exp(g), g a seeded sum of 8 random Fourier modes scaled to
  [0.1, 10]"), read per SURVEY.md R12.  The field is
  described by mode amplitudes / wave numbers / phases and the min/max of the
  raw sum sampled on a lattice; each side evaluates eta(x) with its own code.
* ``initial_guess``: the seeded N(0,1) initial iterate of configs 2 and 5.
* ``problem``: the named configurations c1..c5 (grid, box, boundary kind,
  viscosity, hierarchy depth, smoother settings) as plain dictionaries.

Seeds: PCG64 (numpy.random.Generator), fixed per config in ``CONFIGS``.
"""
from __future__ import annotations

import math
from typing import Dict, Optional

import numpy as np

# Problem kinds (boundary data / forcing); both sides interpret the integer.
KIND_CAVITY = 0        # lid-driven cavity: u = e_x on the lid, no-slip elsewhere, f = 0
KIND_MMS = 1           # manufactured solution u = curl(sin^2 pi x sin^2 pi y), p = cos pi x cos pi y (2D)
KIND_HOMOGENEOUS = 2   # f = 0, u = 0 on the boundary (b = 0)

ETA_CONST = 0
ETA_FOURIER = 1

VISC_SEED = 20210318
X0_SEED = 1
N_MODES = 8


def _lattice_minmax(dim: int, box, amp, mode, phase, npts: int):
    """min/max of g_raw(x) = sum_k a_k prod_d cos(pi m_kd x_d + phi_kd) on an
    npts^dim lattice over the box (chunked over the last axis)."""
    axes = [np.linspace(0.0, box[d], npts) for d in range(dim)]
    # per mode, per axis 1D factors: shape (K, npts)
    fac = [np.cos(math.pi * mode[:, d][:, None] * axes[d][None, :] + phase[:, d][:, None])
           for d in range(dim)]
    gmin, gmax = np.inf, -np.inf
    if dim == 2:
        g = np.einsum("k,kx,ky->yx", amp, fac[0], fac[1])
        gmin, gmax = float(g.min()), float(g.max())
    else:
        for iz in range(npts):
            w = amp * fac[2][:, iz]
            g = np.einsum("k,kx,ky->yx", w, fac[0], fac[1])
            gmin = min(gmin, float(g.min()))
            gmax = max(gmax, float(g.max()))
    return gmin, gmax


def viscosity_params(dim: int, box=(1.0, 1.0, 1.0), seed: int = VISC_SEED,
                     n_modes: int = N_MODES, lattice: Optional[int] = None) -> Dict:
    """Seeded Fourier-mode viscosity description.

    Draws (PCG64(seed)): amplitudes a_k ~ N(0,1); integer wave numbers
    m_kd in {1..4}; phases phi_kd ~ U[0, 2pi).  The min/max of the raw sum are
    sampled on a 1025^2 lattice (2D) or 257^3 lattice (3D; DESIGN.md reading)
    over the box so that eta = exp(ln 0.1 + (g_raw - gmin)/(gmax - gmin) ln 100)
    spans ~[0.1, 10].
    """
    rng = np.random.Generator(np.random.PCG64(seed + 1000 * dim))
    amp = rng.standard_normal(n_modes)
    mode = rng.integers(1, 5, size=(n_modes, dim))
    phase = rng.uniform(0.0, 2.0 * math.pi, size=(n_modes, dim))
    if lattice is None:
        lattice = 1025 if dim == 2 else 257
    gmin, gmax = _lattice_minmax(dim, box, amp, mode, phase, lattice)
    m3 = np.zeros((n_modes, 3), dtype=np.int32)
    p3 = np.zeros((n_modes, 3), dtype=np.float64)
    m3[:, :dim] = mode
    p3[:, :dim] = phase
    return {"amp": amp.astype(np.float64), "mode": m3, "phase": p3,
            "gmin": gmin, "gmax": gmax, "n_modes": n_modes}


def initial_guess(n: int, seed: int = X0_SEED) -> np.ndarray:
    """Seeded N(0,1) initial iterate (configs 2 and 5), float64, length n."""
    rng = np.random.Generator(np.random.PCG64(seed))
    return rng.standard_normal(n)


def random_vector(n: int, seed: int) -> np.ndarray:
    """Generic seeded N(0,1) vector (test inputs)."""
    return np.random.Generator(np.random.PCG64(seed)).standard_normal(n)


ELEM_Q2Q1 = "q2q1"     # Taylor-Hood, C = 0 (R1; BASELINE configs)
ELEM_Q1Q1 = "q1q1"     # the paper's stabilized equal-order pair (Eq. 8; R18)
BETA0 = 0.01           # R18: beta(x) = BETA0 / eta(x) (chosen by the MMS + multigrid beta study)


def problem(dim: int, ncell, kind: int, eta: str = "const", eta0: float = 1.0,
            box=None, seed: int = VISC_SEED, elem: str = ELEM_Q2Q1, beta: float = BETA0) -> Dict:
    """A problem description dict understood by both the oracle wrapper and the
    CUDA binding: grid cells per axis, box lengths, boundary/forcing kind, the
    viscosity field and the element pair (vel_order 2: Q2-Q1, 1: Q1-Q1 with
    stabilization constant beta)."""
    ncell = list(ncell) + [1] * (3 - len(ncell))
    if box is None:
        box = [1.0, 1.0, 1.0]
    box = list(box) + [1.0] * (3 - len(box))
    d = {"dim": dim, "ncell": ncell[:3], "len": [float(b) for b in box[:3]], "kind": kind,
         "eta_mode": ETA_CONST, "eta0": float(eta0), "n_modes": 0,
         "amp": np.zeros(8), "mode": np.zeros((8, 3), np.int32), "phase": np.zeros((8, 3)),
         "gmin": 0.0, "gmax": 1.0,
         "vel_order": 1 if elem == ELEM_Q1Q1 else 2, "beta": float(beta) if elem == ELEM_Q1Q1 else 0.0}
    if eta == "fourier":
        vp = viscosity_params(dim, box, seed=seed)
        d.update({"eta_mode": ETA_FOURIER, "n_modes": vp["n_modes"], "amp": vp["amp"],
                  "mode": vp["mode"], "phase": vp["phase"], "gmin": vp["gmin"], "gmax": vp["gmax"]})
    return d


def coarsen(desc: Dict, factor: int = 2) -> Dict:
    """Same problem on the grid with ncell/factor cells per axis (the nested
    coarse level; the viscosity field and box are unchanged)."""
    d = dict(desc)
    d["ncell"] = [max(1, c // factor) if i < desc["dim"] else 1 for i, c in enumerate(desc["ncell"])]
    return d


# Named configurations (BASELINE.json "configs", SURVEY.md §8 row d).
CONFIGS = {
    # c1: 8x8 cavity, eta = 1, 3 levels (2x2 coarsest), V(2,2)-RAV, omega 0.66, rtol 1e-10
    "c1": dict(dim=2, ncell=(8, 8), kind=KIND_CAVITY, eta="const", levels=3, pre=2, post=2,
               omega=0.66, rtol=1e-10),
    # c2: 512x512 MMS with seeded variable viscosity, 100 RAV sweeps from N(0,1)
    "c2": dict(dim=2, ncell=(512, 512), kind=KIND_MMS, eta="fourier", sweeps=100, omega=0.66),
    # c3: 2048x2048 MMS, same viscosity, 10 levels (4x4 coarsest), V(2,2)-RAV to 1e-8
    "c3": dict(dim=2, ncell=(2048, 2048), kind=KIND_MMS, eta="fourier", levels=10, pre=2,
               post=2, omega=0.66, rtol=1e-8),
    # c4: 32^3 cavity (lid z = 1), seeded viscosity; 5 levels (2^3 coarsest, reading R14)
    "c4": dict(dim=3, ncell=(32, 32, 32), kind=KIND_CAVITY, eta="fourier", levels=5, pre=2,
               post=2, omega=0.66, rtol=1e-8),
    # c5: weak scaling 2048 x (2048 G), 50 sweeps of RAV / diag-Vanka / MV-color
    "c5": dict(dim=2, ncell=(2048, 2048), kind=KIND_MMS, eta="fourier", sweeps=50, omega=0.66),
}


def config_problem(name: str, scale_y: int = 1) -> Dict:
    c = CONFIGS[name]
    ncell = list(c["ncell"])
    box = [1.0] * c["dim"]
    if scale_y > 1:
        ncell[1] *= scale_y
        box[1] = float(scale_y)
    return problem(c["dim"], ncell, c["kind"], eta=c["eta"], box=box)
