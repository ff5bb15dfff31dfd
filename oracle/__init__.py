"""Parity ORACLE for the RAV-smoothed geometric multigrid hot path.

TEST INFRASTRUCTURE ONLY: only ``tests/``, ``__graft_entry__.smoke()`` and
``bench.py``'s cpu_baseline / ``--impl reference`` legs may import this
package.  It shares no code with the CUDA path (``paper_2103_10127_b200/``) and
imports nothing from it; the only common module is ``seeded_inputs`` (random
draws and problem descriptions, no method arithmetic).

The arithmetic lives in plain C (``ravoracle.c``, compiled with gcc on demand);
this file only marshals numpy arrays.  Citations: P:n = PAPER.md line n,
S:n = SPEC.md line n, R<k> = readings in DESIGN.md.

Pins (tests/test_oracle_*.py) -- what fixes each function other than itself:
  assemble           closed-form Q2 stiffness entries (28/45, 256/45, scaled),
                     zero row sums, L = L^T bitwise, B^T (x,-y) = 0 and
                     B^T (x,0) = -h^2 at interior vertices, Galerkin identity
                     P^T L_f P = L_c (constant eta), MMS convergence rates 8 / 4
  patches            interior sizes 51 / 376, nres 19 / 82, sum of weights = 1
                     exactly, patch = structural support of the B^T row
  factor (rows)      L_i * rows^T = diag(w) (rows are rows of L_i^{-1}),
                     numpy.linalg.inv on random patches
  additive sweeps    dense explicit-matrix Eq. 12 / 13 (oracle/dense.py, brute
                     force), single patch covering all DoFs = exact solve,
                     fixed point, patch-order independence
  MV sweeps          dense sequential Eq. 11 replay, single patch = AV
  diagonal Vanka     closed form (R17) vs the local dense solve
  transfers          exact interpolation of quadratics / bilinears, R = P^T
  coarse solve       round trip L e -> e on the pinned system
  V-cycle / solve    SciPy sparse direct solve of the same system, h-independent
                     cycle counts, smoother effectiveness ordering
  iteration counts vs the paper: parity unpinned (the paper prints none).
"""
from __future__ import annotations

import ctypes as C
import os
import subprocess
import threading
from typing import Dict, Optional

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_SRC = os.path.join(_HERE, "ravoracle.c")
_LIB = os.path.join(_HERE, "liboracle.so")
_lock = threading.Lock()
_lib = None

WEIGHTS = {"pou": 0, "own": 1, "full": 2}
FMT_ROWS, FMT_LU, FMT_DIAG = 0, 1, 2


class SingularLocalSystem(RuntimeError):
    def __init__(self, patch: int):
        super().__init__(f"singular local system in patch {patch}")
        self.patch = patch


class Desc(C.Structure):
    _fields_ = [("dim", C.c_int32), ("ncell", C.c_int32 * 3), ("len", C.c_double * 3),
                ("kind", C.c_int32), ("eta_mode", C.c_int32), ("eta0", C.c_double),
                ("n_modes", C.c_int32), ("amp", C.c_double * 8), ("mode", (C.c_int32 * 3) * 8),
                ("phase", (C.c_double * 3) * 8), ("gmin", C.c_double), ("gmax", C.c_double),
                ("vel_order", C.c_int32), ("beta", C.c_double)]


class Level(C.Structure):
    _fields_ = [("n", C.c_int64), ("nvel", C.c_int64),
                ("rp", C.c_void_p), ("ci", C.c_void_p), ("val", C.c_void_p),
                ("npatch", C.c_int64), ("poffs", C.c_void_p), ("pdofs", C.c_void_p), ("pw", C.c_void_p),
                ("foffs", C.c_void_p), ("fac", C.c_void_p), ("piv", C.c_void_p), ("pivoffs", C.c_void_p),
                ("order", C.c_void_p),
                ("prp", C.c_void_p), ("pci", C.c_void_p), ("pval", C.c_void_p), ("nc", C.c_int64)]


class Coarse(C.Structure):
    _fields_ = [("n", C.c_int64), ("pin", C.c_int64), ("lu", C.c_void_p), ("piv", C.c_void_p)]


def build(force: bool = False) -> str:
    """Compile liboracle.so with gcc (plain -O2, OpenMP over patches).  With
    ORACLE_SANITIZE=1 a separate AddressSanitizer + UBSan build is used instead
    (scripts/oracle_sanitize.sh; the process needs libasan preloaded)."""
    global _LIB
    if os.environ.get("ORACLE_SANITIZE") == "1":
        _LIB = os.path.join(_HERE, "liboracle_asan.so")
        with _lock:
            if force or not os.path.exists(_LIB) or os.path.getmtime(_LIB) < os.path.getmtime(_SRC):
                subprocess.check_call(["gcc", "-O1", "-g", "-fsanitize=address,undefined", "-fno-sanitize-recover=all",
                                       "-fno-omit-frame-pointer", "-fopenmp", "-shared", "-fPIC", "-std=c11",
                                       "-D_GNU_SOURCE", "-o", _LIB, _SRC, "-lm"])
        return _LIB
    with _lock:
        if force or not os.path.exists(_LIB) or os.path.getmtime(_LIB) < os.path.getmtime(_SRC):
            tmp = _LIB + f".tmp{os.getpid()}"
            subprocess.check_call(["gcc", "-O2", "-fopenmp", "-shared", "-fPIC", "-std=c11",
                                   "-D_GNU_SOURCE", "-o", tmp, _SRC, "-lm"])
            os.replace(tmp, _LIB)
    return _LIB


def lib():
    global _lib
    if _lib is None:
        build()
        L = C.CDLL(_LIB)
        i64, i32, dbl, vp = C.c_int64, C.c_int32, C.c_double, C.c_void_p
        pd = C.POINTER(Desc)
        sig = {
            "or_n_dofs": (i64, [pd]), "or_n_velocity": (i64, [pd]), "or_n_vertices": (i64, [pd]),
            "or_n_free_nodes": (i64, [pd]),
            "or_assemble_nnz": (i64, [pd]), "or_assemble": (C.c_int, [pd, vp, vp, vp, vp]),
            "or_residual": (None, [i64, vp, vp, vp, vp, vp, vp]),
            "or_spmv": (None, [i64, vp, vp, vp, vp, vp]),
            "or_spmv_t": (None, [i64, i64, vp, vp, vp, vp, vp]),
            "or_patch_entries": (i64, [pd, C.c_int]), "or_patches": (C.c_int, [pd, C.c_int, vp, vp, vp]),
            "or_lu_factor": (C.c_int, [C.c_int, vp, vp]),
            "or_lu_solve": (None, [C.c_int, vp, vp, vp]), "or_lu_solve_t": (None, [C.c_int, vp, vp, vp]),
            "or_factor": (i64, [i64, i64, vp, vp, vp, i64, vp, vp, vp, C.c_int, vp, vp, vp, vp]),
            "or_additive_sweeps": (None, [i64, vp, vp, vp, i64, vp, vp, vp, vp, vp, vp, vp, dbl, C.c_int]),
            "or_additive_lu_sweeps": (None, [i64, vp, vp, vp, i64, vp, vp, vp, vp, vp, vp, vp, vp, vp,
                                             dbl, C.c_int]),
            "or_mv_sweeps": (None, [i64, vp, vp, vp, i64, vp, vp, vp, vp, vp, vp, vp, vp, vp, dbl, C.c_int]),
            "or_prolongation_nnz": (i64, [pd, pd]), "or_prolongation": (C.c_int, [pd, pd, vp, vp, vp]),
            "or_coarse_factor": (C.c_int, [i64, vp, i64, vp, vp]),
            "or_coarse_solve": (None, [C.POINTER(Coarse), vp, vp]),
            "or_vcycle": (None, [C.POINTER(Level), C.POINTER(Coarse), C.c_int, C.c_int, vp, vp,
                                 C.c_int, C.c_int, dbl]),
            "or_mg_solve": (C.c_int, [C.POINTER(Level), C.POINTER(Coarse), C.c_int, C.c_int, vp, vp,
                                      C.c_int, C.c_int, dbl, dbl, C.c_int, vp]),
            "or_rav_sweep_sampled": (i64, [i64, vp, vp, vp, i64, vp, vp, vp, vp, vp, dbl, vp, vp, vp]),
            "or_mms_errors": (None, [pd, vp, C.POINTER(dbl), C.POINTER(dbl)]),
            "or_eta": (dbl, [pd, dbl, dbl, dbl]),
            "or_element_matrices": (C.c_int, [pd, vp, vp, vp, vp, vp, vp]),
            "or_num_threads": (C.c_int, []),
            "or_set_num_threads": (None, [C.c_int]),
        }
        for name, (res, args) in sig.items():
            f = getattr(L, name)
            f.restype = res
            f.argtypes = args
        _lib = L
    return _lib


def set_num_threads(t: int) -> int:
    """OpenMP threads of the oracle (row-independent loops only; results do not depend
    on it).  Returns the previous value."""
    L = lib()
    prev = L.or_num_threads()
    L.or_set_num_threads(int(t))
    return prev


def _p(a: Optional[np.ndarray]):
    return None if a is None else a.ctypes.data


def desc(problem: Dict) -> Desc:
    d = Desc()
    d.dim = problem["dim"]
    for k in range(3):
        d.ncell[k] = int(problem["ncell"][k])
        d.len[k] = float(problem["len"][k])
    d.kind = problem["kind"]
    d.eta_mode = problem["eta_mode"]
    d.eta0 = problem["eta0"]
    d.n_modes = problem["n_modes"]
    for m in range(8):
        d.amp[m] = float(problem["amp"][m]) if m < len(problem["amp"]) else 0.0
        for k in range(3):
            d.mode[m][k] = int(problem["mode"][m][k])
            d.phase[m][k] = float(problem["phase"][m][k])
    d.gmin = problem["gmin"]
    d.gmax = problem["gmax"]
    d.vel_order = int(problem.get("vel_order", 2))   # 2 Taylor-Hood Q2-Q1 (R1), 1 stabilized Q1-Q1 (R18)
    d.beta = float(problem.get("beta", 0.0))
    if problem["dim"] == 3 and problem["kind"] == 1:
        raise ValueError("manufactured solution is 2D only (R13)")
    return d


def sizes(problem: Dict) -> Dict:
    d = desc(problem)
    L = lib()
    return {"n": L.or_n_dofs(C.byref(d)), "nvel": L.or_n_velocity(C.byref(d)),
            "np": L.or_n_vertices(C.byref(d)), "nfree_nodes": L.or_n_free_nodes(C.byref(d))}


def assemble(problem: Dict) -> Dict:
    """L = [A B; B^T 0] and b on the free DoFs (Eq. 6; R1, R7, R8, R9)."""
    d = desc(problem)
    L = lib()
    n = L.or_n_dofs(C.byref(d))
    nnz = L.or_assemble_nnz(C.byref(d))
    rp = np.zeros(n + 1, np.int64)
    ci = np.zeros(nnz, np.int32)
    val = np.zeros(nnz, np.float64)
    b = np.zeros(n, np.float64)
    L.or_assemble(C.byref(d), _p(rp), _p(ci), _p(val), _p(b))
    return {"n": n, "nvel": L.or_n_velocity(C.byref(d)), "rp": rp, "ci": ci, "val": val, "b": b}


def patches(problem: Dict, weights: str = "pou") -> Dict:
    """One Vanka patch per vertex, restricted DoFs first (R2, R3)."""
    d = desc(problem)
    L = lib()
    mode = WEIGHTS[weights]
    nv = L.or_n_vertices(C.byref(d))
    tot = L.or_patch_entries(C.byref(d), mode)
    offs = np.zeros(nv + 1, np.int64)
    dofs = np.zeros(tot, np.int32)
    w = np.zeros(tot, np.float64)
    L.or_patches(C.byref(d), mode, _p(offs), _p(dofs), _p(w))
    return {"offs": offs, "dofs": dofs, "w": w}


def factor(A: Dict, P: Dict, fmt: int = FMT_ROWS) -> Dict:
    """Local factorizations: ROWS = weighted restricted rows of
    L_i^{-1}, LU = full LU of L_i, DIAG = LU of the diagonal-Vanka
    local matrix (R17)."""
    L = lib()
    offs, w = P["offs"], P["w"]
    ni = np.diff(offs)
    npatch = len(ni)
    if fmt == FMT_ROWS:
        nres = np.add.reduceat((w > 0).astype(np.int64), offs[:-1]) if npatch else np.zeros(0, np.int64)
        nres = np.where(ni > 0, nres, 0)
        sz = nres * ni
    else:
        sz = ni * ni
    foffs = np.zeros(npatch + 1, np.int64)
    np.cumsum(sz, out=foffs[1:])
    fac = np.zeros(int(foffs[-1]), np.float64)
    piv = pivoffs = None
    if fmt != FMT_ROWS:
        pivoffs = offs.copy()
        piv = np.zeros(int(offs[-1]), np.int32)
    bad = L.or_factor(A["n"], A["nvel"], _p(A["rp"]), _p(A["ci"]), _p(A["val"]), npatch,
                      _p(offs), _p(P["dofs"]), _p(w), fmt, _p(foffs), _p(fac), _p(piv), _p(pivoffs))
    if bad >= 0:
        raise SingularLocalSystem(int(bad))
    return {"fmt": fmt, "foffs": foffs, "fac": fac, "piv": piv, "pivoffs": pivoffs}


def residual(A: Dict, x: np.ndarray, b: np.ndarray) -> np.ndarray:
    r = np.zeros(A["n"])
    lib().or_residual(A["n"], _p(A["rp"]), _p(A["ci"]), _p(A["val"]), _p(x), _p(b), _p(r))
    return r


def additive_sweeps(A: Dict, P: Dict, F: Dict, x: np.ndarray, b: np.ndarray, omega: float, nu: int):
    """nu sweeps of RAV (Eq. 13; PoU/own rows) or AV (Eq. 12; full rows)."""
    x = np.array(x, dtype=np.float64, copy=True)
    L = lib()
    if F["fmt"] == FMT_ROWS:
        L.or_additive_sweeps(A["n"], _p(A["rp"]), _p(A["ci"]), _p(A["val"]), len(P["offs"]) - 1,
                             _p(P["offs"]), _p(P["dofs"]), _p(P["w"]), _p(F["foffs"]), _p(F["fac"]),
                             _p(x), _p(b), float(omega), int(nu))
    else:
        L.or_additive_lu_sweeps(A["n"], _p(A["rp"]), _p(A["ci"]), _p(A["val"]), len(P["offs"]) - 1,
                                _p(P["offs"]), _p(P["dofs"]), _p(P["w"]), _p(F["foffs"]), _p(F["fac"]),
                                _p(F["piv"]), _p(F["pivoffs"]), _p(x), _p(b), float(omega), int(nu))
    return x


def mv_sweeps(A: Dict, P: Dict, F: Dict, x: np.ndarray, b: np.ndarray, omega: float, nu: int,
              order: Optional[np.ndarray] = None):
    """nu sweeps of multiplicative Vanka (Eq. 11, fresh residual Eq. 15)."""
    assert F["fmt"] == FMT_LU
    x = np.array(x, dtype=np.float64, copy=True)
    if order is not None:
        order = np.ascontiguousarray(order, dtype=np.int32)
    lib().or_mv_sweeps(A["n"], _p(A["rp"]), _p(A["ci"]), _p(A["val"]), len(P["offs"]) - 1,
                       _p(P["offs"]), _p(P["dofs"]), _p(F["foffs"]), _p(F["fac"]), _p(F["piv"]),
                       _p(F["pivoffs"]), _p(order), _p(x), _p(b), float(omega), int(nu))
    return x


def multicolor_order(problem: Dict) -> np.ndarray:
    """R10: 4^d colors (i mod 4, j mod 4[, k mod 4]), color-major, then ascending."""
    dim = problem["dim"]
    nv = [problem["ncell"][k] + 1 for k in range(dim)]
    idx = np.arange(int(np.prod(nv)))
    coords = []
    r = idx.copy()
    for k in range(dim):
        coords.append(r % nv[k])
        r = r // nv[k]
    color = np.zeros_like(idx)
    mult = 1
    for k in range(dim):
        color += (coords[k] % 4) * mult
        mult *= 4
    return np.lexsort((idx, color)).astype(np.int32)


def prolongation(fine: Dict, coarse: Dict) -> Dict:
    """Nested Q2/Q1 interpolation P (fine free DoFs x coarse free DoFs)."""
    L = lib()
    df, dc = desc(fine), desc(coarse)
    n = L.or_n_dofs(C.byref(df))
    nnz = L.or_prolongation_nnz(C.byref(df), C.byref(dc))
    rp = np.zeros(n + 1, np.int64)
    ci = np.zeros(nnz, np.int32)
    val = np.zeros(nnz)
    L.or_prolongation(C.byref(df), C.byref(dc), _p(rp), _p(ci), _p(val))
    return {"n": n, "nc": L.or_n_dofs(C.byref(dc)), "rp": rp, "ci": ci, "val": val}


def to_dense(A: Dict) -> np.ndarray:
    n = A["n"]
    ncol = A.get("nc", n)
    M = np.zeros((n, ncol))
    rows = np.repeat(np.arange(n), np.diff(A["rp"]))
    M[rows, A["ci"]] = A["val"]
    return M


def lu_factor(M: np.ndarray):
    n = M.shape[0]
    LU = np.ascontiguousarray(M, dtype=np.float64).copy()
    piv = np.zeros(n, np.int32)
    st = lib().or_lu_factor(n, _p(LU), _p(piv))
    if st != 0:
        raise SingularLocalSystem(-1)
    return LU, piv


def lu_solve(LU, piv, rhs, trans=False):
    x = np.array(rhs, dtype=np.float64, copy=True)
    f = lib().or_lu_solve_t if trans else lib().or_lu_solve
    f(LU.shape[0], _p(LU), _p(piv), _p(x))
    return x


class Hierarchy:
    """Level hierarchy for the oracle V-cycle: rediscretized
    operators on ncell/2^k grids ("assembled on all grids"), nested
    transfers, smoother data per level, pinned coarse LU (R4)."""

    SMOOTHERS = {"rav": 0, "av": 0, "mv": 1, "diag": 2}

    def __init__(self, problem: Dict, n_levels: int, smoother: str = "rav", weights: Optional[str] = None,
                 mv_order: str = "ascending"):
        self.problem = problem
        self.smoother = smoother
        if weights is None:       # R3 (RAV), Eq. 12 / Eq. 11 full prolongation, R17
            weights = {"rav": "pou", "av": "full", "mv": "full", "diag": "full"}[smoother]
        self.weights = weights
        probs = [problem]
        for _ in range(n_levels - 1):
            p = dict(probs[-1])
            p["ncell"] = [c // 2 if k < problem["dim"] else c for k, c in enumerate(p["ncell"])]
            probs.append(p)
        probs = probs[::-1]        # coarsest first
        self.probs = probs
        self.A, self.P, self.F, self.T, self.order = [], [], [], [], []
        for l, p in enumerate(probs):
            A = assemble(p)
            self.A.append(A)
            if l == 0:
                self.P.append(None)
                self.F.append(None)
                self.order.append(None)
            else:
                Pt = patches(p, weights)
                fmt = {"rav": FMT_ROWS, "av": FMT_ROWS, "mv": FMT_LU, "diag": FMT_DIAG}[smoother]
                F = factor(A, Pt, fmt)
                self.P.append(Pt)
                self.F.append(F)
                if smoother == "mv" and mv_order == "color":
                    self.order.append(multicolor_order(p))
                else:
                    self.order.append(None)
            self.T.append(None if l == 0 else prolongation(p, probs[l - 1]))
        # coarse pinned LU (R4): pin the pressure DoF of vertex 0
        A0 = self.A[0]
        dense = to_dense(A0)
        self.pin = int(A0["nvel"])
        m = A0["n"] - 1
        self.coarse_lu = np.zeros((m, m))
        self.coarse_piv = np.zeros(m, np.int32)
        st = lib().or_coarse_factor(A0["n"], _p(np.ascontiguousarray(dense)), self.pin,
                                    _p(self.coarse_lu), _p(self.coarse_piv))
        if st != 0:
            raise RuntimeError("singular coarse system")
        self._build_structs()

    def _build_structs(self):
        n = len(self.probs)
        self.levels = (Level * n)()
        for l in range(n):
            A = self.A[l]
            lv = self.levels[l]
            lv.n, lv.nvel = A["n"], A["nvel"]
            lv.rp, lv.ci, lv.val = _p(A["rp"]), _p(A["ci"]), _p(A["val"])
            if l > 0:
                Pt, F, T = self.P[l], self.F[l], self.T[l]
                lv.npatch = len(Pt["offs"]) - 1
                lv.poffs, lv.pdofs, lv.pw = _p(Pt["offs"]), _p(Pt["dofs"]), _p(Pt["w"])
                lv.foffs, lv.fac = _p(F["foffs"]), _p(F["fac"])
                lv.piv, lv.pivoffs = _p(F["piv"]), _p(F["pivoffs"])
                lv.order = _p(self.order[l])
                lv.prp, lv.pci, lv.pval, lv.nc = _p(T["rp"]), _p(T["ci"]), _p(T["val"]), T["nc"]
        self.coarse = Coarse(self.A[0]["n"], self.pin, _p(self.coarse_lu), _p(self.coarse_piv))

    @property
    def fine(self):
        return self.A[-1]

    def vcycle(self, x, b, pre=2, post=2, omega=0.66):
        x = np.array(x, dtype=np.float64, copy=True)
        lib().or_vcycle(self.levels, C.byref(self.coarse), len(self.probs) - 1,
                        self.SMOOTHERS[self.smoother], _p(x), _p(b), pre, post, float(omega))
        return x

    def solve(self, b=None, x0=None, pre=2, post=2, omega=0.66, rtol=1e-8, maxit=200):
        A = self.fine
        if b is None:
            b = A["b"]
        x = np.zeros(A["n"]) if x0 is None else np.array(x0, dtype=np.float64, copy=True)
        hist = np.zeros(maxit + 1)
        k = lib().or_mg_solve(self.levels, C.byref(self.coarse), len(self.probs),
                              self.SMOOTHERS[self.smoother], _p(x), _p(np.ascontiguousarray(b)),
                              pre, post, float(omega), float(rtol), int(maxit), _p(hist))
        return x, k, hist[:k + 1]


def rav_sweep_sampled(A: Dict, P: Dict, x: np.ndarray, b: np.ndarray, omega: float,
                      sample: np.ndarray, with_magnitude: bool = False):
    """One RAV sweep evaluated only at the sampled DoFs (full-size parity).  With
    with_magnitude also the per-entry rounding scale |x_j| + omega sum |w L_i^{-T} e_k|
    (|b| + |L||x| + |r|) of the sampled entries (for element-wise bounds)."""
    mask = np.zeros(A["n"], np.uint8)
    mask[sample] = 1
    xnew = np.full(A["n"], np.nan)
    mag = np.full(A["n"], np.nan) if with_magnitude else None
    bad = lib().or_rav_sweep_sampled(A["n"], _p(A["rp"]), _p(A["ci"]), _p(A["val"]), len(P["offs"]) - 1,
                                     _p(P["offs"]), _p(P["dofs"]), _p(P["w"]), _p(x), _p(b), float(omega),
                                     _p(mask), _p(xnew), _p(mag))
    if bad >= 0:
        raise SingularLocalSystem(int(bad))
    return (xnew[sample], mag[sample]) if with_magnitude else xnew[sample]


def mms_errors(problem: Dict, x: np.ndarray):
    eu, ep = C.c_double(), C.c_double()
    d = desc(problem)
    lib().or_mms_errors(C.byref(d), _p(np.ascontiguousarray(x)), C.byref(eu), C.byref(ep))
    return eu.value, ep.value


def eta(problem: Dict, x: float, y: float, z: float = 0.0) -> float:
    d = desc(problem)
    return lib().or_eta(C.byref(d), x, y, z)


def pressure_shift(A: Dict, x: np.ndarray) -> np.ndarray:
    """a10 / R4: p <- p - p(vertex 0) after the solve."""
    y = np.array(x, copy=True)
    nv = A["nvel"]
    y[nv:] -= y[nv]
    return y
