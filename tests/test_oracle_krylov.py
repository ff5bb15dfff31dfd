"""Pins of the flexible GMRES oracle (oracle/krylov.py)
against what the mathematics fixes, not against itself:
* without preconditioning, the residual after k steps is the minimum of
  ||b - L x|| over x0 + K_k(L, r0) -- computed independently from an
  orthonormal basis of the explicit Krylov matrix [r0, L r0, ..., L^{k-1} r0];
* an exact preconditioner (dense inverse) converges in one step;
* restarts: the true residual never increases across a restart (minimal
  residual over a space containing the previous iterate);
* with the RAV V-cycle as preconditioner, FGMRES needs no more iterations
  than the stationary multigrid iteration and reaches the same solution.
"""
import numpy as np
import pytest

import oracle
import seeded_inputs as si
from oracle import krylov


def small_system():
    p = si.problem(2, (3, 3), si.KIND_MMS, eta="fourier")
    A = oracle.assemble(p)
    L = oracle.to_dense(A)
    nu = A["nvel"]
    L[nu, :] = 0.0          # pin one pressure DoF: nonsingular (R4)
    L[:, nu] = 0.0
    L[nu, nu] = 1.0
    b = A["b"].copy()
    b[nu] = 0.0
    return L, b


def test_fgmres_unpreconditioned_is_minimal_residual():
    L, b = small_system()
    mv = lambda v: L @ v
    x, k, hist = krylov.fgmres(mv, b, lambda v: v.copy(), restart=50, rtol=1e-30, maxit=8)
    r0 = b.copy()
    K = np.zeros((len(b), 8))
    v = r0.copy()
    for j in range(8):
        K[:, j] = v
        v = L @ v
    for kk in range(1, 9):
        Q, _ = np.linalg.qr(K[:, :kk])
        AQ = L @ Q
        y = np.linalg.lstsq(AQ, b, rcond=None)[0]
        rmin = np.linalg.norm(b - AQ @ y)
        assert hist[kk] == pytest.approx(rmin, rel=1e-8, abs=1e-12 * np.linalg.norm(b))


def test_fgmres_exact_preconditioner_one_step():
    L, b = small_system()
    Li = np.linalg.inv(L)
    x, k, hist = krylov.fgmres(lambda v: L @ v, b, lambda v: Li @ v, rtol=1e-12)
    assert k == 1
    assert np.linalg.norm(L @ x - b) <= 1e-12 * np.linalg.norm(b)


def test_fgmres_restart_monotone_true_residual():
    L, b = small_system()
    rs = []
    x = np.zeros_like(b)
    for _ in range(5):
        x, k, hist = krylov.fgmres(lambda v: L @ v, b, lambda v: v.copy(), x0=x, restart=4, rtol=1e-30, maxit=4)
        rs.append(np.linalg.norm(b - L @ x))
    assert all(rs[i + 1] <= rs[i] * (1 + 1e-12) for i in range(len(rs) - 1))


@pytest.mark.parametrize("prob,levels", [(si.problem(2, (32, 32), si.KIND_MMS, eta="fourier"), 4),
                                         (si.problem(2, (32, 32), si.KIND_CAVITY, elem=si.ELEM_Q1Q1), 3)])
def test_fgmres_with_rav_vcycle_improves_on_stationary_mg(prob, levels):
    H = oracle.Hierarchy(prob, levels)
    xs, ks, _ = H.solve(rtol=1e-10, omega=0.66)
    xk, kk, hist = krylov.mg_fgmres(H, rtol=1e-10, omega=0.66)
    assert hist[-1] <= 1e-10 * hist[0]
    assert kk <= ks, (kk, ks)
    A = H.fine
    r = A["b"] - krylov.csr_matvec(A)(xk)
    assert np.linalg.norm(r) <= 1.01e-10 * hist[0]
    # same discrete solution up to the pressure constant (R4) and the tolerance
    nu = A["nvel"]
    assert np.linalg.norm(xk[:nu] - xs[:nu]) <= 1e-7 * np.linalg.norm(xs[:nu])
