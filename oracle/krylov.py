"""Flexible GMRES oracle ("the geometric
multigrid method can also be used as a preconditioner in a Krylov subspace
solver, which typically leads to an improvement in performance").

TEST INFRASTRUCTURE ONLY (see oracle/__init__.py).  Plain right-preconditioned
flexible GMRES(m) written step by step (Saad, "Iterative Methods for Sparse
Linear Systems", Algorithm 9.6): Arnoldi with modified Gram-Schmidt on the
preconditioned directions z_j = M(v_j), the small least-squares problem
min ||beta e_1 - Hbar_j y|| solved afresh at every step with numpy.linalg.lstsq
(no Givens bookkeeping), restarts every m steps.  Stopping (reading R19):
||b - L x_k||_2 (the least-squares residual estimate) <= rtol ||b - L x_0||_2,
x_0 = the initial guess of the whole solve; k counts Arnoldi steps (one
preconditioner application each).
"""
from __future__ import annotations

from typing import Callable

import numpy as np


def csr_matvec(A):
    rp, ci, val = A["rp"], A["ci"], A["val"]
    rows = np.repeat(np.arange(len(rp) - 1), np.diff(rp))

    def mv(v):
        return np.bincount(rows, weights=val * v[ci], minlength=len(rp) - 1)
    return mv


def fgmres(matvec: Callable, b: np.ndarray, precond: Callable, x0=None, restart: int = 30,
           rtol: float = 1e-8, maxit: int = 200):
    """Returns (x, k, hist): hist[j] = least-squares residual norm after j steps
    (hist[0] = ||b - L x0||), the true residual at every restart."""
    x = np.zeros_like(b) if x0 is None else np.array(x0, dtype=np.float64, copy=True)
    r = b - matvec(x)
    r0 = np.linalg.norm(r)
    hist = [r0]
    k = 0
    if r0 == 0.0:
        return x, 0, np.array(hist)
    while k < maxit:
        beta = np.linalg.norm(r)
        V = [r / beta]
        Z = []
        H = np.zeros((restart + 1, restart))
        y = np.zeros(0)
        done = False
        for j in range(restart):
            z = precond(V[j])
            Z.append(z)
            w = matvec(z)
            for i in range(j + 1):                  # modified Gram-Schmidt
                H[i, j] = np.dot(w, V[i])
                w = w - H[i, j] * V[i]
            H[j + 1, j] = np.linalg.norm(w)
            rhs = np.zeros(j + 2)
            rhs[0] = beta
            y = np.linalg.lstsq(H[:j + 2, :j + 1], rhs, rcond=None)[0]
            res = np.linalg.norm(rhs - H[:j + 2, :j + 1] @ y)
            k += 1
            hist.append(res)
            if res <= rtol * r0 or k >= maxit or H[j + 1, j] == 0.0:
                done = True
                break
            V.append(w / H[j + 1, j])
        x = x + np.column_stack(Z[:len(y)]) @ y
        r = b - matvec(x)
        if done:
            break
    return x, k, np.array(hist)


def mg_fgmres(H, b=None, x0=None, pre=2, post=2, omega=0.66, restart=30, rtol=1e-8, maxit=200):
    """FGMRES on the finest level of an oracle Hierarchy, preconditioned by one
    V-cycle from a zero guess."""
    A = H.fine
    if b is None:
        b = A["b"]
    mv = csr_matvec(A)

    def M(v):
        return H.vcycle(np.zeros_like(v), v, pre, post, omega)
    return fgmres(mv, b, M, x0, restart, rtol, maxit)
