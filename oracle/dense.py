"""Brute-force dense oracle (O2) for tiny meshes -- TEST INFRASTRUCTURE ONLY.

Writes Eqs. 11-13 of the paper as explicit
dense matrix products: restriction operators R_i as rows of the identity
(P:114), local systems L_i = R_i L R_i^T, local inverses by numpy.linalg.inv,
the restricted prolongation R~_i^T = R_i^T diag(w_i) (the paper's 0/1
G_i when w is the ownership indicator, R3 otherwise).  Used to pin the C
oracle's sweeps on <= 5x5 meshes (acceptance criterion S:525).
"""
from __future__ import annotations

import numpy as np


def restriction(n: int, dofs: np.ndarray) -> np.ndarray:
    """R_i: rows of the n x n identity for the patch DoFs."""
    R = np.zeros((len(dofs), n))
    R[np.arange(len(dofs)), dofs] = 1.0
    return R


def patch_list(P):
    offs, dofs, w = P["offs"], P["dofs"], P["w"]
    return [(dofs[offs[i]:offs[i + 1]], w[offs[i]:offs[i + 1]]) for i in range(len(offs) - 1)]


def S_additive(L: np.ndarray, patches, omega: float, restricted: bool) -> np.ndarray:
    """S_AV = sum_i R_i^T omega L_i^{-1} R_i (Eq. 12) or, with restricted=True,
    S_RAV = sum_i R~_i^T omega L_i^{-1} R_i (Eq. 13), R~_i^T = R_i^T diag(w_i)."""
    n = L.shape[0]
    S = np.zeros((n, n))
    for dofs, w in patches:
        R = restriction(n, dofs)
        Li = R @ L @ R.T
        Rt = (R.T * w[None, :]) if restricted else R.T
        S += Rt @ (omega * np.linalg.inv(Li)) @ R
    return S


def additive_sweep(L, b, x, patches, omega, restricted):
    """x^{k+1} = x^k + S (b - L x^k)  (Eq. 10)."""
    S = S_additive(L, patches, omega, restricted)
    return x + S @ (b - L @ x)


def mv_sweep(L, b, x, patches, omega, order=None):
    """Multiplicative Vanka (Eq. 11): the patch corrections applied one after
    the other, each from the current residual."""
    n = L.shape[0]
    x = x.copy()
    idx = range(len(patches)) if order is None else order
    for i in idx:
        dofs, _ = patches[i]
        R = restriction(n, dofs)
        Li = R @ L @ R.T
        x = x + R.T @ (omega * np.linalg.inv(Li)) @ R @ (b - L @ x)
    return x


def S_mv_product(L, patches, omega, order=None):
    """Error propagation of one MV sweep: prod_i (I - R_i^T omega L_i^{-1} R_i L)."""
    n = L.shape[0]
    E = np.eye(n)
    idx = range(len(patches)) if order is None else order
    for i in idx:
        dofs, _ = patches[i]
        R = restriction(n, dofs)
        Li = R @ L @ R.T
        E = (np.eye(n) - R.T @ (omega * np.linalg.inv(Li)) @ R @ L) @ E
    return E
