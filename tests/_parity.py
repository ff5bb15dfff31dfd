"""Element-wise parity bounds (test infrastructure).

The GPU path and the oracle differ only by rounding: the order of the sums in
the residual and in each patch product, the local solver (block / Schur form
vs LU), and the order of the <= 2^d partition-of-unity additions per DoF
(DESIGN.md 5.3).  One RAV sweep x_new_j = x_j + omega sum_i (W_i R_i r)_j
therefore agrees per entry to a small multiple of eps times the magnitude of
the terms that make up x_new_j:

    mag_j = |x_j| + omega sum_i sum_k |W_i[j, k]| (|b| + |L||x| + |r|)_{dof k}

(|b| + |L||x| bounds the rounding of r = b - Lx; |W| the amplification through
the local solve).  The bar is |x_gpu - x_ora|_j <= 1e-12 mag_j for EVERY entry
-- no norm averaging, so a single wrong entry (e.g. a ragged boundary patch)
cannot hide among millions of good ones.  After several sweeps the rounding of
earlier sweeps propagates through (I - omega S L), which mixes entries within
patches; there the bar is the same 1e-12 against max_j mag_j, per entry.
"""
from __future__ import annotations

import numpy as np
import scipy.sparse as sp

import oracle

TOL = 1e-12


def _csr(A):
    return sp.csr_matrix((A["val"], A["ci"], A["rp"]), shape=(A["n"], A["n"]))


def sweep_magnitude(A, P, F, x, b, omega, chunk=20000):
    """mag_j (see module doc) for one sweep from x, with the oracle's weighted rows F
    (oracle.factor(..., FMT_ROWS)); computed in chunks of patches."""
    M = _csr(A)
    r = b - M @ x
    rabs = np.abs(b) + abs(M) @ np.abs(x) + np.abs(r)
    offs, dofs, w = P["offs"], P["dofs"], P["w"]
    fo, fac = F["foffs"], F["fac"]
    npatch = len(offs) - 1
    ni = np.diff(offs)
    restricted = w > 0
    rpos = np.nonzero(restricted)[0]                        # restricted entries, patch by patch
    coffs = np.zeros(npatch + 1, np.int64)
    np.cumsum(np.add.reduceat(restricted.astype(np.int64), offs[:-1]) * (ni > 0), out=coffs[1:])
    nres = np.diff(coffs)
    mag = np.zeros(A["n"])
    for p0 in range(0, npatch, chunk):
        p1 = min(npatch, p0 + chunk)
        a, e = fo[p0], fo[p1]
        cnt = nres[p0:p1] * ni[p0:p1]
        pid = np.repeat(np.arange(p0, p1), cnt)
        u = np.arange(a, e) - fo[pid]
        j = u // ni[pid]
        k = u % ni[pid]
        rowdof = dofs[rpos[coffs[pid] + j]]
        coldof = dofs[offs[pid] + k]
        mag += np.bincount(rowdof, weights=np.abs(fac[a:e]) * rabs[coldof], minlength=A["n"])
    return np.abs(x) + omega * mag


def assert_entrywise(got, want, scale, tol=TOL, what=""):
    """|got - want|_j <= tol * scale_j for every j (scale: array or scalar)."""
    got, want = np.asarray(got), np.asarray(want)
    err = np.abs(got - want)
    bound = tol * np.asarray(scale)
    bad = np.nonzero(err > bound)[0]
    if len(bad):
        j = bad[np.argmax((err / np.maximum(bound, 1e-300))[bad])]
        raise AssertionError(f"{what}: {len(bad)} of {len(err)} entries outside the bound; worst entry {j}: "
                             f"|diff| {err[j]:.3e} > {np.broadcast_to(bound, err.shape)[j]:.3e}")


class SweepChecker:
    """Sweeps checked against the oracle at the given targets: target 1 entry by entry
    against mag_j of the first sweep, later targets entry by entry against
    max_j mag_j of the sweeps since the previous target (module doc)."""

    def __init__(self, A, P, F, b, omega):
        self.A, self.P, self.F, self.b, self.omega = A, P, F, b, omega

    def run(self, x0, gpu_sweeps, targets=(1, 2, 10, 100), what=""):
        """gpu_sweeps(k): advance the GPU iterate by k sweeps and return it (numpy)."""
        xo = np.array(x0, dtype=np.float64, copy=True)
        done = 0
        worst = 0.0
        for t in targets:
            mag = sweep_magnitude(self.A, self.P, self.F, xo, self.b, self.omega)
            xo = oracle.additive_sweeps(self.A, self.P, self.F, xo, self.b, self.omega, t - done)
            xg = gpu_sweeps(t - done)
            done = t
            scale = mag if t == 1 else mag.max()
            assert_entrywise(xg, xo, scale, what=f"{what} after {t} sweeps")
            worst = max(worst, float(np.max(np.abs(xg - xo) / (TOL * np.asarray(scale) + 1e-300))))
        return xo, worst


def iterate_tol(ncell_per_axis: int) -> float:
    """Entry-wise bar for a converged V-cycle iterate relative to max |x|: the two paths follow the
    same cycles and differ by rounding of each cycle's residual, ~eps |L| |x|, which the solve maps
    to ~eps cond(L) |x| in x; cond(L) grows like h^-2 = N^2 for the Stokes operator (N cells per
    axis).  20 eps N^2, at least 1e-10 (the coarse-grid cases)."""
    return max(1e-10, 20 * 2.22e-16 * float(ncell_per_axis) ** 2)
