"""Thin Python binding of libravgmg.so (include/ravgmg.h) -- argument
marshalling only: every step of the hot path runs in the library's CUDA
kernels.  PyTorch provides device memory and streams.

There is no CPU fallback: if the shared library cannot be loaded, importing
this module raises.
"""
from __future__ import annotations

import ctypes as C
import os
from typing import Dict, List, Optional, Sequence

import numpy as np
import torch

_HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(_HERE, "libravgmg.so")

RAV_OK = 0
STATUS = {0: "RAV_OK", 1: "RAV_ERR_ARG", 2: "RAV_ERR_SINGULAR_LOCAL", 3: "RAV_ERR_SINGULAR_COARSE",
          4: "RAV_ERR_OOM", 5: "RAV_ERR_CUDA", 6: "RAV_ERR_COMM", 7: "RAV_ERR_DIVERGED"}
VARIANT_ROWS, VARIANT_DIAG, VARIANT_MV = 0, 1, 2
KERNEL_AUTO, KERNEL_WARP, KERNEL_THREAD, KERNEL_SYM, KERNEL_SCHUR = 0, 1, 2, 3, 4
WEIGHTS = {"pou": 0, "own": 1, "full": 2}


class RavError(RuntimeError):
    def __init__(self, status: int, msg: str, bad_patch: int = -1, bad_level: int = -1):
        super().__init__(f"{STATUS.get(status, status)}: {msg}")
        self.status = status
        self.bad_patch = bad_patch
        self.bad_level = bad_level


class RavGrid(C.Structure):
    _fields_ = [("dim", C.c_int32), ("ncell", C.c_int32 * 3), ("len", C.c_double * 3),
                ("kind", C.c_int32), ("eta_mode", C.c_int32), ("eta0", C.c_double),
                ("n_modes", C.c_int32), ("amp", C.c_double * 8), ("mode", (C.c_int32 * 3) * 8),
                ("phase", (C.c_double * 3) * 8), ("gmin", C.c_double), ("gmax", C.c_double),
                ("win", C.c_int32), ("node_lo", C.c_int32), ("node_hi", C.c_int32), ("vert_lo", C.c_int32),
                ("vert_hi", C.c_int32), ("rnode_lo", C.c_int32), ("rnode_hi", C.c_int32),
                ("rvert_lo", C.c_int32), ("rvert_hi", C.c_int32), ("pvert_lo", C.c_int32), ("pvert_hi", C.c_int32),
                ("vel_order", C.c_int32), ("beta", C.c_double)]

WINDOW_KEYS = ("node_lo", "node_hi", "vert_lo", "vert_hi", "rnode_lo", "rnode_hi", "rvert_lo", "rvert_hi",
               "pvert_lo", "pvert_hi")


class RavAdaptiveDesc(C.Structure):
    _fields_ = [("base", RavGrid), ("n_levels", C.c_int32), ("bands", C.c_int32 * 16), ("uniform", C.c_int32)]


class RavCsr(C.Structure):
    _fields_ = [("n_rows", C.c_int64), ("n_cols", C.c_int64), ("row_ptr", C.c_void_p),
                ("col", C.c_void_p), ("val", C.c_void_p), ("on_device", C.c_int32)]


class RavPatches(C.Structure):
    _fields_ = [("n_patches", C.c_int64), ("offs", C.c_void_p), ("dofs", C.c_void_p),
                ("weight", C.c_void_p), ("on_device", C.c_int32)]


class RavNeighbor(C.Structure):
    _fields_ = [("peer", C.c_int32), ("n_corr_send", C.c_int64), ("n_corr_recv", C.c_int64),
                ("n_halo_send", C.c_int64), ("n_halo_recv", C.c_int64), ("corr_send", C.c_void_p),
                ("corr_recv", C.c_void_p), ("halo_send", C.c_void_p), ("halo_recv", C.c_void_p)]


class RavSubdomain(C.Structure):
    _fields_ = [("A", RavCsr), ("P", RavPatches), ("n_vel", C.c_int64), ("n_neighbors", C.c_int32),
                ("neighbors", C.c_void_p), ("n_ghost_written", C.c_int64), ("ghost_written", C.c_void_p),
                ("owned", C.c_int64 * 4), ("P_coarse", RavCsr), ("n_colors", C.c_int32),
                ("color_offs", C.c_void_p), ("color_ids", C.c_void_p),
                ("grid_fine", C.c_void_p), ("grid_coarse", C.c_void_p)]


class RavOpts(C.Structure):
    _fields_ = [("variant", C.c_int32), ("kernel", C.c_int32), ("deterministic", C.c_int32),
                ("n_vel", C.c_int64), ("stream", C.c_void_p), ("block_dim", C.c_int32)]


def _load():
    from . import build as _build
    if not os.path.exists(LIB_PATH) or (_build.stale() and os.path.exists(_build.NVCC)):
        _build.build()
    L = C.CDLL(LIB_PATH)
    i64, vp, dbl, st = C.c_int64, C.c_void_p, C.c_double, C.c_int
    P = C.POINTER
    sigs = {
        "rav_gen_sizes": [P(RavGrid), C.c_int, vp, P(i64), P(i64), P(i64), P(i64), P(i64)],
        "rav_gen_operator": [P(RavGrid), vp, vp, vp, vp, vp],
        "rav_gen_patches": [P(RavGrid), C.c_int, vp, vp, vp, vp],
        "rav_gen_prolongation_nnz": [P(RavGrid), P(RavGrid), vp, P(i64)],
        "rav_gen_prolongation": [P(RavGrid), P(RavGrid), vp, vp, vp, vp],
        "rav_setup": [P(RavCsr), P(RavPatches), P(RavOpts), P(vp), P(i64)],
        "rav_smooth": [vp, vp, vp, C.c_int, dbl],
        "rav_smooth_batch": [vp, i64, P(vp), P(vp), C.c_int, dbl],
        "rav_residual": [vp, vp, vp, vp],
        "rav_apply": [vp, vp, vp, dbl],
        "rav_rows_size": [vp, P(i64)],
        "rav_export_rows": [vp, vp],
        "rav_sweep_bytes": [vp, P(dbl), P(dbl), P(dbl)],
        "rav_set_stream": [vp, vp],
        "rav_set_colors": [vp, C.c_int, vp, vp],
        "rav_apply_color": [vp, C.c_int, vp, vp, dbl],
        "mg_set_colors": [vp, C.c_int, C.c_int, vp, vp],
        "rav_index_op": [C.c_int, vp, vp, i64, vp, dbl, vp],
        "mg_setup": [C.c_int, P(RavCsr), P(RavPatches), P(RavCsr), P(i64), i64, P(RavOpts), P(vp), P(C.c_int),
                     P(i64)],
        "mg_vcycle": [vp, vp, vp, C.c_int, C.c_int, dbl],
        "mg_solve": [vp, vp, vp, C.c_int, C.c_int, dbl, dbl, C.c_int, P(C.c_int), vp],
        "mg_set_stream": [vp, vp],
        "rav_xfer_setup": [P(RavCsr), vp, P(vp)],
        "rav_prolong": [vp, vp, vp, dbl],
        "rav_restrict": [vp, vp, vp],
        "rav_xfer_set_stream": [vp, vp],
        "rav_xfer_set_structured": [vp, P(RavGrid), P(RavGrid)],
        "mg_set_structured_transfers": [vp, vp],
        "rav_dot": [vp, vp, i64, vp, C.c_int, vp],
        "mg_fgmres": [vp, vp, vp, C.c_int, C.c_int, dbl, C.c_int, dbl, C.c_int, P(C.c_int), vp],
        "rav_adaptive_create": [P(RavAdaptiveDesc), P(vp)],
        "rav_color_patches": [P(RavCsr), P(RavPatches), P(i64), vp, vp],
        "rav_gen_colors": [P(RavGrid), vp, vp],
        "rav_comm_unique_id": [vp],
        "rav_comm_create": [C.c_int, C.c_int, vp, P(vp)],
        "mgd_setup": [vp, C.c_int, vp, C.c_int, vp, C.c_int, vp, vp, P(RavOpts), C.c_int, P(vp)],
        "mgd_smooth": [vp, vp, vp, C.c_int, dbl],
        "mgd_vcycle": [vp, vp, vp, C.c_int, C.c_int, dbl],
        "mgd_solve": [vp, vp, vp, C.c_int, C.c_int, dbl, dbl, C.c_int, P(C.c_int), vp],
        "mgd_residual_norm": [vp, vp, vp, P(dbl)],
        "mgd_set_stream": [vp, vp],
        "mgd_host_time": [vp, P(dbl), P(dbl), P(C.c_int)],
        "rav_pressure_normalize": [vp, i64, i64, C.c_int, i64, vp],
        "mg_normalize_pressure": [vp, vp, C.c_int],
        "mg_cycle_bytes": [vp, C.c_int, C.c_int, P(dbl)],
        "rav_adaptive_sizes": [vp, C.c_int, P(i64), P(i64), P(i64), P(i64), P(i64), P(i64), P(i64)],
        "rav_adaptive_fill": [vp, C.c_int, vp, vp, vp, vp, vp, vp, vp, vp, vp, vp],
    }
    for name, args in sigs.items():
        f = getattr(L, name)
        f.argtypes = args
        f.restype = st
    L.rav_destroy.argtypes = [vp]
    L.rav_destroy.restype = None
    L.mg_destroy.argtypes = [vp]
    L.mg_destroy.restype = None
    L.rav_xfer_destroy.argtypes = [vp]
    L.rav_xfer_destroy.restype = None
    L.rav_adaptive_destroy.argtypes = [vp]
    L.rav_adaptive_destroy.restype = None
    L.rav_kernel_name.argtypes = [vp]
    L.rav_kernel_name.restype = C.c_char_p
    L.rav_last_error.restype = C.c_char_p
    L.rav_version.restype = C.c_char_p
    L.rav_last_launches.argtypes = [vp]
    L.rav_last_launches.restype = i64
    L.mg_last_launches.argtypes = [vp]
    L.mg_last_launches.restype = i64
    L.mgd_last_launches.argtypes = [vp]
    L.mgd_last_launches.restype = i64
    L.mgd_destroy.argtypes = [vp]
    L.mgd_destroy.restype = None
    L.rav_comm_destroy.argtypes = [vp]
    L.rav_comm_destroy.restype = None
    return L


lib = _load()


def _check(status: int, **kw):
    if status != RAV_OK:
        raise RavError(status, lib.rav_last_error().decode(), **kw)


def _stream(stream=None):
    s = stream if stream is not None else torch.cuda.current_stream()
    return C.c_void_p(s.cuda_stream)


def _ptr(t) -> Optional[int]:
    if t is None:
        return None
    if isinstance(t, torch.Tensor):
        return t.data_ptr()
    return t.ctypes.data


def grid(problem: Dict) -> RavGrid:
    g = RavGrid()
    g.dim = problem["dim"]
    for k in range(3):
        g.ncell[k] = int(problem["ncell"][k])
        g.len[k] = float(problem["len"][k])
    g.kind = problem["kind"]
    g.eta_mode = problem["eta_mode"]
    g.eta0 = problem["eta0"]
    g.n_modes = problem["n_modes"]
    for m in range(8):
        g.amp[m] = float(problem["amp"][m]) if m < len(problem["amp"]) else 0.0
        for k in range(3):
            g.mode[m][k] = int(problem["mode"][m][k])
            g.phase[m][k] = float(problem["phase"][m][k])
    g.gmin = problem["gmin"]
    g.gmax = problem["gmax"]
    g.vel_order = int(problem.get("vel_order", 2))
    g.beta = float(problem.get("beta", 0.0))
    win = problem.get("window")
    if win is not None:   # slab window of one rank (dist.py)
        g.win = 1
        for k in WINDOW_KEYS:
            setattr(g, k, int(win[k]))
    return g


def rav_gen_sizes(problem: Dict, weights: str = "pou", stream=None) -> Dict:
    g = grid(problem)
    out = [C.c_int64() for _ in range(5)]
    _check(lib.rav_gen_sizes(C.byref(g), WEIGHTS[weights], _stream(stream), *[C.byref(o) for o in out]))
    return dict(zip(["n", "nvel", "nnz", "npatch", "patch_entries"], [o.value for o in out]))


def gen_level(problem: Dict, weights: str = "pou", device="cuda", stream=None) -> Dict:
    """Operator, right-hand side and patches of one structured level, generated on the GPU."""
    sz = rav_gen_sizes(problem, weights, stream)
    g = grid(problem)
    n, nnz = sz["n"], sz["nnz"]
    rp = torch.empty(n + 1, dtype=torch.int64, device=device)
    ci = torch.empty(nnz, dtype=torch.int32, device=device)
    val = torch.empty(nnz, dtype=torch.float64, device=device)
    b = torch.empty(n, dtype=torch.float64, device=device)
    _check(lib.rav_gen_operator(C.byref(g), _ptr(rp), _ptr(ci), _ptr(val), _ptr(b), _stream(stream)))
    offs = torch.empty(sz["npatch"] + 1, dtype=torch.int64, device=device)
    dofs = torch.empty(sz["patch_entries"], dtype=torch.int32, device=device)
    w = torch.empty(sz["patch_entries"], dtype=torch.float64, device=device)
    _check(lib.rav_gen_patches(C.byref(g), WEIGHTS[weights], _ptr(offs), _ptr(dofs), _ptr(w), _stream(stream)))
    return {"n": n, "nvel": sz["nvel"], "nnz": nnz, "rp": rp, "ci": ci, "val": val, "b": b,
            "offs": offs, "dofs": dofs, "w": w, "problem": problem}


def gen_patches(problem: Dict, weights: str, device="cuda", stream=None) -> Dict:
    sz = rav_gen_sizes(problem, weights, stream)
    g = grid(problem)
    offs = torch.empty(sz["npatch"] + 1, dtype=torch.int64, device=device)
    dofs = torch.empty(sz["patch_entries"], dtype=torch.int32, device=device)
    w = torch.empty(sz["patch_entries"], dtype=torch.float64, device=device)
    _check(lib.rav_gen_patches(C.byref(g), WEIGHTS[weights], _ptr(offs), _ptr(dofs), _ptr(w), _stream(stream)))
    return {"offs": offs, "dofs": dofs, "w": w}


def gen_prolongation(fine: Dict, coarse: Dict, device="cuda", stream=None) -> Dict:
    gf, gc = grid(fine), grid(coarse)
    nnz = C.c_int64()
    _check(lib.rav_gen_prolongation_nnz(C.byref(gf), C.byref(gc), _stream(stream), C.byref(nnz)))
    nf = rav_gen_sizes(fine, stream=stream)["n"]
    nc = rav_gen_sizes(coarse, stream=stream)["n"]
    rp = torch.empty(nf + 1, dtype=torch.int64, device=device)
    ci = torch.empty(nnz.value, dtype=torch.int32, device=device)
    val = torch.empty(nnz.value, dtype=torch.float64, device=device)
    _check(lib.rav_gen_prolongation(C.byref(gf), C.byref(gc), _ptr(rp), _ptr(ci), _ptr(val), _stream(stream)))
    return {"n": nf, "nc": nc, "rp": rp, "ci": ci, "val": val}


def csr(A: Dict, n_cols: Optional[int] = None) -> RavCsr:
    on_dev = int(isinstance(A["rp"], torch.Tensor) and A["rp"].is_cuda)
    n = A["n"]
    return RavCsr(n, n if n_cols is None else n_cols, _ptr(A["rp"]), _ptr(A["ci"]), _ptr(A["val"]), on_dev)


def patches_struct(P: Dict) -> RavPatches:
    on_dev = int(isinstance(P["offs"], torch.Tensor) and P["offs"].is_cuda)
    return RavPatches(len(P["offs"]) - 1, _ptr(P["offs"]), _ptr(P["dofs"]), _ptr(P["w"]), on_dev)


class Smoother:
    """rav_setup / rav_smooth / rav_destroy (Eq. 13)."""

    def __init__(self, A: Dict, P: Dict, variant: int = VARIANT_ROWS, kernel: int = KERNEL_AUTO,
                 stream=None, block_dim: Optional[int] = None, deterministic: bool = False):
        self.n = A["n"]
        self._keep = (A, P)
        if block_dim is None:   # the generator's interleaved velocity numbering (R9)
            block_dim = A["problem"]["dim"] if "problem" in A else 0
        opts = RavOpts(variant, kernel, int(bool(deterministic)), A.get("nvel", 0), _stream(stream), int(block_dim))
        ctx = C.c_void_p()
        bad = C.c_int64(-1)
        st = lib.rav_setup(C.byref(csr(A)), C.byref(patches_struct(P)), C.byref(opts), C.byref(ctx), C.byref(bad))
        _check(st, bad_patch=bad.value)
        self.ctx = ctx

    def smooth(self, x, b, nu: int, omega: float):
        """x <- x + omega S_RAV (b - L x), nu times (x updated in place)."""
        _check(lib.rav_smooth(self.ctx, _ptr(x), _ptr(b), int(nu), float(omega)))
        return x

    def smooth_batch(self, xs, bs, nu: int, omega: float):
        """rav_smooth on independent problems in host buffers (numpy arrays or CPU tensors, pinned
        for overlap): x_k <- nu sweeps from x_k with rhs b_k, in place; copies overlap the sweeps."""
        k = len(xs)
        if len(bs) != k:
            raise ValueError("smooth_batch: one b per x")
        xa = (C.c_void_p * max(1, k))(*[_ptr(x) for x in xs])
        ba = (C.c_void_p * max(1, k))(*[_ptr(b) for b in bs])
        _check(lib.rav_smooth_batch(self.ctx, k, xa, ba, int(nu), float(omega)))
        return xs

    def residual(self, x, b, r=None):
        if r is None:
            r = torch.empty_like(b)
        _check(lib.rav_residual(self.ctx, _ptr(x), _ptr(b), _ptr(r)))
        return r

    def apply(self, r, x, omega: float):
        """x += omega S_RAV r (the sweep kernel alone)."""
        _check(lib.rav_apply(self.ctx, _ptr(r), _ptr(x), float(omega)))
        return x

    def export_rows(self) -> torch.Tensor:
        n = C.c_int64()
        _check(lib.rav_rows_size(self.ctx, C.byref(n)))
        rows = torch.empty(n.value, dtype=torch.float64, device="cuda")
        _check(lib.rav_export_rows(self.ctx, _ptr(rows)))
        return rows

    def sweep_bytes(self) -> Dict:
        a, b, f = C.c_double(), C.c_double(), C.c_double()
        _check(lib.rav_sweep_bytes(self.ctx, C.byref(a), C.byref(b), C.byref(f)))
        return {"sweep": a.value, "residual": b.value, "flops": f.value}

    @property
    def last_launches(self) -> int:
        return int(lib.rav_last_launches(self.ctx))

    @property
    def kernel_name(self) -> str:
        return lib.rav_kernel_name(self.ctx).decode()

    def set_colors(self, offs: np.ndarray, ids: np.ndarray):
        offs = np.ascontiguousarray(offs, dtype=np.int64)
        ids = np.ascontiguousarray(ids, dtype=np.int32)
        self._colors = (offs, ids)
        _check(lib.rav_set_colors(self.ctx, len(offs) - 1, offs.ctypes.data, ids.ctypes.data))

    def apply_color(self, color: int, x, b, omega: float):
        """One colour of multiplicative Vanka (rav_apply_color)."""
        _check(lib.rav_apply_color(self.ctx, int(color), _ptr(x), _ptr(b), float(omega)))
        return x

    def set_stream(self, stream):
        _check(lib.rav_set_stream(self.ctx, _stream(stream)))

    def close(self):
        if getattr(self, "ctx", None):
            lib.rav_destroy(self.ctx)
            self.ctx = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass


class Multigrid:
    """mg_setup / mg_vcycle / mg_solve."""

    def __init__(self, levels: Sequence[Dict], prolongations: Sequence[Optional[Dict]], coarse_pin: int,
                 variant: int = VARIANT_ROWS, kernel: int = KERNEL_AUTO, stream=None,
                 block_dim: Optional[int] = None, deterministic: bool = False):
        L = len(levels)
        self.L = L
        self.n = levels[-1]["n"]
        self._keep = (levels, prolongations)
        As = (RavCsr * L)(*[csr(A) for A in levels])
        Ps = (RavPatches * L)(*[patches_struct(A) for A in levels])
        Pr = (RavCsr * L)()
        for l in range(1, L):
            Pr[l] = csr(prolongations[l], n_cols=prolongations[l]["nc"])
        if block_dim is None:
            block_dim = levels[-1]["problem"]["dim"] if "problem" in levels[-1] else 0
        opts = RavOpts(variant, kernel, int(bool(deterministic)), levels[-1].get("nvel", 0), _stream(stream),
                       int(block_dim))
        nvel = (C.c_int64 * L)(*[int(A.get("nvel", 0)) for A in levels])
        self._keep = (levels, prolongations, nvel)
        ctx = C.c_void_p()
        bl, bp = C.c_int(-1), C.c_int64(-1)
        st = lib.mg_setup(L, As, Ps, Pr, nvel, int(coarse_pin), C.byref(opts), C.byref(ctx), C.byref(bl),
                          C.byref(bp))
        _check(st, bad_patch=bp.value, bad_level=bl.value)
        self.ctx = ctx

    def set_colors(self, level: int, offs: np.ndarray, ids: np.ndarray):
        offs = np.ascontiguousarray(offs, dtype=np.int64)
        ids = np.ascontiguousarray(ids, dtype=np.int32)
        _check(lib.mg_set_colors(self.ctx, int(level), len(offs) - 1, offs.ctypes.data, ids.ctypes.data))

    def set_structured_transfers(self, problems: Sequence[Dict]):
        """mg_set_structured_transfers: stencil-form P / P^T on every level (problems coarsest
        first, each the uniform refinement of the previous; verified against the CSR P)."""
        gs = (RavGrid * self.L)(*[grid(p) for p in problems])
        _check(lib.mg_set_structured_transfers(self.ctx, gs))

    def vcycle(self, x, b, pre=2, post=2, omega=0.66):
        _check(lib.mg_vcycle(self.ctx, _ptr(x), _ptr(b), int(pre), int(post), float(omega)))
        return x

    def solve(self, x, b, pre=2, post=2, omega=0.66, rtol=1e-8, maxit=200):
        hist = np.zeros(maxit + 1)
        it = C.c_int(0)
        st = lib.mg_solve(self.ctx, _ptr(x), _ptr(b), int(pre), int(post), float(omega), float(rtol), int(maxit),
                          C.byref(it), hist.ctypes.data)
        _check(st)
        return x, it.value, hist[:it.value + 1]

    def fgmres(self, x, b, pre=2, post=2, omega=0.66, restart=30, rtol=1e-8, maxit=200):
        """mg_fgmres: FGMRES(restart) preconditioned by one V-cycle (R19)."""
        hist = np.zeros(maxit + 1)
        it = C.c_int(0)
        _check(lib.mg_fgmres(self.ctx, _ptr(x), _ptr(b), int(pre), int(post), float(omega), int(restart),
                             float(rtol), int(maxit), C.byref(it), hist.ctypes.data))
        return x, it.value, hist[:it.value + 1]

    def normalize_pressure(self, x, mode: int = 0):
        """mg_normalize_pressure (row a10, R4): mode 0 p -= p(vertex 0), mode 1 p -= mean(p)."""
        _check(lib.mg_normalize_pressure(self.ctx, _ptr(x), int(mode)))
        return x

    def cycle_bytes(self, pre=2, post=2) -> float:
        """mg_cycle_bytes: algorithmic HBM bytes of one V(pre, post) cycle."""
        out = C.c_double()
        _check(lib.mg_cycle_bytes(self.ctx, int(pre), int(post), C.byref(out)))
        return out.value

    @property
    def last_launches(self) -> int:
        return int(lib.mg_last_launches(self.ctx))

    def close(self):
        if getattr(self, "ctx", None):
            lib.mg_destroy(self.ctx)
            self.ctx = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass


class Transfer:
    """rav_xfer_setup / rav_prolong / rav_restrict: xf += alpha P xc, bc = P^T rf."""

    def __init__(self, Pm: Dict, stream=None):
        self._keep = Pm
        ctx = C.c_void_p()
        _check(lib.rav_xfer_setup(C.byref(csr(Pm, n_cols=Pm["nc"])), _stream(stream), C.byref(ctx)))
        self.ctx = ctx
        self.n, self.nc = Pm["n"], Pm["nc"]

    def prolong(self, xc, xf, alpha: float = 1.0):
        _check(lib.rav_prolong(self.ctx, _ptr(xc), _ptr(xf), float(alpha)))
        return xf

    def restrict(self, rf, bc):
        _check(lib.rav_restrict(self.ctx, _ptr(rf), _ptr(bc)))
        return bc

    def set_stream(self, stream):
        _check(lib.rav_xfer_set_stream(self.ctx, _stream(stream)))

    def set_structured(self, fine_problem: Dict, coarse_problem: Dict):
        """rav_xfer_set_structured: stencil-form transfer (verified against the CSR P)."""
        gf, gc = grid(fine_problem), grid(coarse_problem)
        _check(lib.rav_xfer_set_structured(self.ctx, C.byref(gf), C.byref(gc)))

    def close(self):
        if getattr(self, "ctx", None):
            lib.rav_xfer_destroy(self.ctx)
            self.ctx = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass


def dot(a, b, out, accumulate: bool = False, n: Optional[int] = None, stream=None):
    """rav_dot: out[0] (device) = sum a[i] b[i] (+ out[0] if accumulate)."""
    n = a.numel() if n is None else int(n)
    _check(lib.rav_dot(_ptr(a), _ptr(b), n, _ptr(out), int(bool(accumulate)), _stream(stream)))
    return out


def pressure_normalize(x, n_vel: int, mode: int = 0, pin: Optional[int] = None, stream=None):
    """rav_pressure_normalize (row a10, R4): mode 0 p -= p[pin] (default pin = n_vel, vertex 0),
    mode 1 p -= mean(p), over x[n_vel:] (device tensor, in place)."""
    pin = int(n_vel) if pin is None else int(pin)
    _check(lib.rav_pressure_normalize(_ptr(x), int(n_vel), x.numel(), int(mode), pin, _stream(stream)))
    return x


def index_op(op: int, src, idx, dst, value: float = 0.0, stream=None):
    """rav_index_op: 0 gather dst[k] = src[idx[k]], 1 scatter dst[idx[k]] = src[k],
    2 scatter-add, 3 fill dst[idx[k]] = value, 4 gather-difference
    dst[k] = src[idx[k]] - dst[k] (device tensors)."""
    n = idx.numel()
    _check(lib.rav_index_op(int(op), _ptr(src) if src is not None else None, _ptr(idx), int(n), _ptr(dst),
                            float(value), _stream(stream)))
    return dst


def multicolor(problem: Dict):
    """rav_gen_colors: 4^d colouring of the generated vertex patches (R10) by global
    vertex coordinates (a slab window colours its patches like the whole grid),
    patches ascending inside each colour.  Returns (offs, ids) for rav_set_colors."""
    g = grid(problem)
    sz = rav_gen_sizes(problem) if "window" not in problem else None
    npatch = sz["npatch"] if sz is not None else _window_patches(problem)
    offs = np.zeros(4 ** problem["dim"] + 1, np.int64)
    ids = np.zeros(max(npatch, 1), np.int32)
    _check(lib.rav_gen_colors(C.byref(g), offs.ctypes.data, ids.ctypes.data))
    return offs, ids[:npatch]


def _window_patches(problem: Dict) -> int:
    """Patches of a slab window (vertex layers [pvert_lo, pvert_hi] of the last axis), host arithmetic."""
    dim, w = problem["dim"], problem["window"]
    low = int(np.prod([int(problem["ncell"][k]) + 1 for k in range(dim - 1)]))
    return low * (int(w["pvert_hi"]) - int(w["pvert_lo"]) + 1)


def coarsen_problem(problem: Dict) -> Dict:
    p = dict(problem)
    p["ncell"] = [c // 2 if k < problem["dim"] else c for k, c in enumerate(problem["ncell"])]
    return p


def build_hierarchy(problem: Dict, n_levels: int, weights: str = "pou", variant: int = VARIANT_ROWS,
                    kernel: int = KERNEL_AUTO, free_inputs: bool = True, deterministic: bool = False,
                    structured_transfers: bool = True):
    """Generate every level on the GPU (rediscretized operators) and
    build the multigrid context.  Returns (mg, fine_level_dict).  With
    structured_transfers the V-cycle applies P / P^T in stencil form
    (mg_set_structured_transfers) instead of streaming their CSR."""
    probs = [problem]
    for _ in range(n_levels - 1):
        probs.append(coarsen_problem(probs[-1]))
    probs = probs[::-1]
    levels, prols = [], [None]
    for l, p in enumerate(probs):
        lev = gen_level(p, weights)
        levels.append(lev)
        if l > 0:
            prols.append(gen_prolongation(p, probs[l - 1]))
    pin = levels[0]["nvel"]       # pressure DoF of vertex 0 (R4)
    mg = Multigrid(levels, prols, pin, variant=variant, kernel=kernel, deterministic=deterministic)
    if variant == VARIANT_MV:     # colour every smoothed level (R10)
        for l in range(1, len(probs)):
            mg.set_colors(l, *multicolor(probs[l]))
    nested = all(probs[l]["ncell"][k] == 2 * probs[l - 1]["ncell"][k]
                 for l in range(1, len(probs)) for k in range(problem["dim"]))
    if structured_transfers and nested and len(probs) > 1:
        mg.set_structured_transfers(probs)
    fine = levels[-1]
    if free_inputs:   # the library copied everything it needs
        fine = {k: v for k, v in fine.items() if k in ("n", "nvel", "nnz", "b", "problem")}
        del levels, prols
        torch.cuda.empty_cache()
    return mg, fine


def gen_adaptive(problem: Dict, n_levels: int, bands: Optional[Sequence[int]] = None, uniform: bool = False,
                 device="cuda") -> List[Dict]:
    """rav_adaptive_*: the paper's adaptive hierarchy (R20) -- per level
    (coarsest first) the operator, rhs, patches, and the prolongation from the level
    below ("prol", levels >= 1).  problem: 2D Q1-Q1 on an n0 x n0 grid."""
    d = RavAdaptiveDesc()
    d.base = grid(problem)
    d.n_levels = int(n_levels)
    for k, bk in enumerate(bands or []):
        d.bands[k] = int(bk)
    d.uniform = int(bool(uniform))
    h = C.c_void_p()
    _check(lib.rav_adaptive_create(C.byref(d), C.byref(h)))
    out = []
    try:
        for l in range(n_levels):
            sz = [C.c_int64() for _ in range(7)]
            _check(lib.rav_adaptive_sizes(h, l, *[C.byref(s) for s in sz]))
            n, nvel, nnz, npatch, pe, pnnz, ncell = [s.value for s in sz]
            t = lambda k, dt: torch.empty(max(k, 1), dtype=dt, device=device)
            rp, ci, val, b = t(n + 1, torch.int64), t(nnz, torch.int32), t(nnz, torch.float64), t(n, torch.float64)
            offs, dofs, w = t(npatch + 1, torch.int64), t(pe, torch.int32), t(pe, torch.float64)
            prp, pci, pval = t(n + 1, torch.int64), t(pnnz, torch.int32), t(pnnz, torch.float64)
            _check(lib.rav_adaptive_fill(h, l, _ptr(rp), _ptr(ci), _ptr(val), _ptr(b), _ptr(offs), _ptr(dofs),
                                         _ptr(w), _ptr(prp), _ptr(pci), _ptr(pval)))
            lev = {"n": n, "nvel": nvel, "nnz": nnz, "rp": rp, "ci": ci[:nnz], "val": val[:nnz], "b": b[:n],
                   "offs": offs, "dofs": dofs[:pe], "w": w[:pe], "n_cells": ncell, "problem": problem}
            if l > 0:
                lev["prol"] = {"n": n, "nc": out[-1]["n"], "rp": prp, "ci": pci[:pnnz], "val": pval[:pnnz]}
            out.append(lev)
    finally:
        lib.rav_adaptive_destroy(h)
    return out


def color_patches(A: Dict, P: Dict):
    """rav_color_patches: greedy multicolouring for multiplicative Vanka on any patches.
    Returns (offs, ids) for rav_set_colors."""
    npatch = len(P["offs"]) - 1
    offs = np.zeros(npatch + 1, np.int64)
    ids = np.zeros(max(npatch, 1), np.int32)
    nc = C.c_int64()
    _check(lib.rav_color_patches(C.byref(csr(A)), C.byref(patches_struct(P)), C.byref(nc), offs.ctypes.data,
                                 ids.ctypes.data))
    return offs[:nc.value + 1].copy(), ids[:npatch].copy()


def build_adaptive_hierarchy(problem: Dict, n_levels: int, weights: str = "own", variant: int = VARIANT_ROWS,
                             kernel: int = KERNEL_AUTO, deterministic: bool = False):
    """mg_setup on the adaptive hierarchy.  weights: "own" = the paper's restricted
    prolongation, "full" = additive Vanka (Eq. 12)."""
    levels = gen_adaptive(problem, n_levels)
    if weights == "full":
        for lev in levels:
            lev["w"].fill_(1.0)
    prols = [None] + [lev["prol"] for lev in levels[1:]]
    pin = levels[0]["nvel"]       # pressure DoF of vertex (0, 0) (R4)
    mg = Multigrid(levels, prols, pin, variant=variant, kernel=kernel, deterministic=deterministic)
    if variant == VARIANT_MV:     # greedy colouring of every smoothed level (R10 / R20)
        for l in range(1, n_levels):
            mg.set_colors(l, *color_patches(levels[l], levels[l]))
    fine = {k: v for k, v in levels[-1].items() if k in ("n", "nvel", "nnz", "b", "problem", "n_cells")}
    return mg, fine


# ---------------------------------------------------------------------------------------------
# slab-partitioned smoother / V-cycle in the library (mgd_*; include/ravgmg.h)
# ---------------------------------------------------------------------------------------------

class Comm:
    """rav_comm_create: the library's communicator (NCCL between processes, loaded at run time).
    nccl_id: 128 bytes from unique_id() on process 0, broadcast by the caller; None = no NCCL
    (one process, every subdomain local)."""

    def __init__(self, nprocs: int = 1, proc: int = 0, nccl_id: Optional[bytes] = None):
        h = C.c_void_p()
        idb = None if nccl_id is None else (C.c_ubyte * 128).from_buffer_copy(nccl_id)
        _check(lib.rav_comm_create(int(nprocs), int(proc), idb, C.byref(h)))
        self.ctx, self.nprocs, self.proc = h, nprocs, proc

    @staticmethod
    def unique_id() -> bytes:
        buf = (C.c_ubyte * 128)()
        _check(lib.rav_comm_unique_id(buf))
        return bytes(buf)

    def close(self):
        if getattr(self, "ctx", None):
            lib.rav_comm_destroy(self.ctx)
            self.ctx = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass


def _i32(a) -> np.ndarray:
    return np.ascontiguousarray(np.asarray(a, dtype=np.int64).astype(np.int32))


class DistMultigrid:
    """mgd_setup / mgd_smooth / mgd_vcycle / mgd_solve.  subs[k][i]: dict of partitioned level k,
    local subdomain i with keys level (gen_level dict of the window), neighbors {peer: (corr_send,
    corr_recv, halo_send, halo_recv)}, ghost_written, owned (2 ranges), prol (gen_prolongation dict
    or None), colors ((offs, ids) or None).  Argument marshalling only."""

    def __init__(self, comm: "Comm", sub_proc: Sequence[int], local_ids: Sequence[int], subs, coarse=None,
                 variant: int = VARIANT_ROWS, kernel: int = KERNEL_AUTO, stream=None, via_comm: int = 0,
                 deterministic: bool = False):
        K, nl = len(subs), len(local_ids)
        keep = []
        arr = (RavSubdomain * (K * nl))()
        for k in range(K):
            for i in range(nl):
                d = subs[k][i]
                L = d["level"]
                sd = arr[k * nl + i]
                sd.A = csr(L)
                sd.P = patches_struct(L)
                sd.n_vel = int(L["nvel"])
                peers = sorted(d["neighbors"])
                nbs = (RavNeighbor * max(1, len(peers)))()
                for j, q in enumerate(peers):
                    lists = [_i32(v) for v in d["neighbors"][q]]
                    keep.append(lists)
                    nb = nbs[j]
                    nb.peer = int(q)
                    nb.n_corr_send, nb.n_corr_recv, nb.n_halo_send, nb.n_halo_recv = [len(v) for v in lists]
                    nb.corr_send, nb.corr_recv, nb.halo_send, nb.halo_recv = [v.ctypes.data for v in lists]
                keep.append(nbs)
                sd.n_neighbors = len(peers)
                sd.neighbors = C.cast(nbs, C.c_void_p)
                gw = _i32(d["ghost_written"])
                keep.append(gw)
                sd.n_ghost_written = len(gw)
                sd.ghost_written = gw.ctypes.data
                (a0, b0), (a1, b1) = d["owned"]
                sd.owned[0], sd.owned[1], sd.owned[2], sd.owned[3] = int(a0), int(b0), int(a1), int(b1)
                if d.get("prol") is not None:
                    sd.P_coarse = csr(d["prol"], n_cols=d["prol"]["nc"])
                if d.get("prol_grids") is not None:
                    gf, gc = grid(d["prol_grids"][0]), grid(d["prol_grids"][1])
                    keep.append((gf, gc))
                    sd.grid_fine, sd.grid_coarse = C.addressof(gf), C.addressof(gc)
                if d.get("colors") is not None:
                    offs = np.ascontiguousarray(d["colors"][0], dtype=np.int64)
                    ids = np.ascontiguousarray(d["colors"][1], dtype=np.int32)
                    keep.append((offs, ids))
                    sd.n_colors = len(offs) - 1
                    sd.color_offs, sd.color_ids = offs.ctypes.data, ids.ctypes.data
        sp = _i32(sub_proc)
        li = _i32(local_ids)
        dim = subs[0][0]["level"]["problem"]["dim"] if "problem" in subs[0][0]["level"] else 0
        opts = RavOpts(variant, kernel, int(bool(deterministic)), 0, _stream(stream), int(dim))
        h = C.c_void_p()
        _check(lib.mgd_setup(comm.ctx, len(sp), sp.ctypes.data, nl, li.ctypes.data, K, arr,
                             coarse.ctx if coarse is not None else None, C.byref(opts), int(via_comm),
                             C.byref(h)))
        self.ctx, self.nl, self.comm, self.coarse = h, nl, comm, coarse

    def _vecs(self, xs, bs):
        X = (C.c_void_p * self.nl)(*[_ptr(x) for x in xs])
        B = (C.c_void_p * self.nl)(*[_ptr(b) for b in bs])
        return X, B

    def smooth(self, xs, bs, nu: int, omega: float):
        X, B = self._vecs(xs, bs)
        _check(lib.mgd_smooth(self.ctx, X, B, int(nu), float(omega)))
        return xs

    def vcycle(self, xs, bs, pre=2, post=2, omega=0.66):
        X, B = self._vecs(xs, bs)
        _check(lib.mgd_vcycle(self.ctx, X, B, int(pre), int(post), float(omega)))
        return xs

    def solve(self, xs, bs, pre=2, post=2, omega=0.66, rtol=1e-8, maxit=200):
        X, B = self._vecs(xs, bs)
        hist = np.zeros(maxit + 1)
        it = C.c_int(0)
        _check(lib.mgd_solve(self.ctx, X, B, int(pre), int(post), float(omega), float(rtol), int(maxit), C.byref(it),
                             hist.ctypes.data))
        return xs, it.value, hist[:it.value + 1]

    def residual_norm(self, xs, bs) -> float:
        X, B = self._vecs(xs, bs)
        out = C.c_double()
        _check(lib.mgd_residual_norm(self.ctx, X, B, C.byref(out)))
        return out.value

    def set_stream(self, stream):
        _check(lib.mgd_set_stream(self.ctx, _stream(stream)))

    def host_time(self):
        """(enqueue seconds, wait seconds, cycles) of the last solve (mgd_host_time)."""
        a, b, c = C.c_double(), C.c_double(), C.c_int()
        _check(lib.mgd_host_time(self.ctx, C.byref(a), C.byref(b), C.byref(c)))
        return a.value, b.value, c.value

    @property
    def last_launches(self) -> int:
        return int(lib.mgd_last_launches(self.ctx))

    def close(self):
        if getattr(self, "ctx", None):
            lib.mgd_destroy(self.ctx)
            self.ctx = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass
