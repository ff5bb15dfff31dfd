"""Pins of the oracle's local solves and smoothers (Eqs. 10-13)
against brute-force dense algebra (oracle/dense.py: explicit R_i, numpy.linalg.inv)
and against properties the paper/mathematics fix."""
import numpy as np
import pytest

import oracle
from oracle import dense
import seeded_inputs as si


def _setup(n=3, kind=si.KIND_CAVITY, eta="const", weights="pou", dim=2):
    p = si.problem(dim, [n] * dim, kind, eta=eta)
    A = oracle.assemble(p)
    P = oracle.patches(p, weights)
    return p, A, P


@pytest.mark.parametrize("n", [2, 3, 4])
def test_factor_rows_are_weighted_rows_of_local_inverse(n):
    p, A, P = _setup(n, eta="fourier")
    F = oracle.factor(A, P, oracle.FMT_ROWS)
    L = oracle.to_dense(A)
    for i in range(len(P["offs"]) - 1):
        d = P["dofs"][P["offs"][i]:P["offs"][i + 1]]
        w = P["w"][P["offs"][i]:P["offs"][i + 1]]
        Li = L[np.ix_(d, d)]
        k = int((w > 0).sum())
        rows = F["fac"][F["foffs"][i]:F["foffs"][i + 1]].reshape(k, len(d))
        inv = np.linalg.inv(Li)
        np.testing.assert_allclose(rows, w[:k, None] * inv[:k], rtol=1e-10,
                                   atol=1e-12 * np.abs(inv[:k]).max())
        # rows_k L_i = w_k e_k^T  (definition of a row of the inverse)
        np.testing.assert_allclose(rows @ Li, np.diag(w[:k]) @ np.eye(len(d))[:k], atol=1e-11)


@pytest.mark.parametrize("weights,restricted", [("pou", True), ("own", True), ("full", False)])
@pytest.mark.parametrize("n", [2, 3, 5])
def test_additive_sweep_matches_dense_eq12_eq13(weights, restricted, n):
    p, A, P = _setup(n, eta="fourier", weights=weights)
    F = oracle.factor(A, P, oracle.FMT_ROWS)
    L = oracle.to_dense(A)
    b = si.random_vector(A["n"], 7)
    x0 = si.random_vector(A["n"], 8)
    omega = 0.66 if restricted else 0.1
    xo = oracle.additive_sweeps(A, P, F, x0, b, omega, 1)
    xd = dense.additive_sweep(L, b, x0, dense.patch_list(P), omega, restricted)
    assert np.abs(xo - xd).max() <= 1e-12 * max(1.0, np.abs(xd).max())


@pytest.mark.parametrize("n", [2, 3])
def test_mv_sweep_matches_dense_eq11(n):
    p, A, P = _setup(n, eta="fourier", weights="full")
    F = oracle.factor(A, P, oracle.FMT_LU)
    L = oracle.to_dense(A)
    b = si.random_vector(A["n"], 3)
    x0 = si.random_vector(A["n"], 4)
    xo = oracle.mv_sweeps(A, P, F, x0, b, 0.66, 1)
    xd = dense.mv_sweep(L, b, x0, dense.patch_list(P), 0.66)
    assert np.abs(xo - xd).max() <= 1e-12 * max(1.0, np.abs(xd).max())
    # error propagation form of Eq. 11: x* - x1 = E (x* - x0) for any consistent x*
    E = dense.S_mv_product(L, dense.patch_list(P), 0.66)
    xs = si.random_vector(A["n"], 5)
    bs = L @ xs
    x1 = oracle.mv_sweeps(A, P, F, x0, bs, 0.66, 1)
    np.testing.assert_allclose(xs - x1, E @ (xs - x0), atol=1e-11)


def test_mv_order_matters_and_multicolor_equals_parallel_colors():
    p, A, P = _setup(9, eta="fourier", weights="full")
    F = oracle.factor(A, P, oracle.FMT_LU)
    L = oracle.to_dense(A)
    b = si.random_vector(A["n"], 11)
    x0 = si.random_vector(A["n"], 12)
    order = oracle.multicolor_order(p)
    xa = oracle.mv_sweeps(A, P, F, x0, b, 0.66, 1)
    xr = oracle.mv_sweeps(A, P, F, x0, b, 0.66, 1, order=np.arange(len(order))[::-1].copy())
    assert np.abs(xa - xr).max() > 1e-6          # MV depends on the order
    # R10: same-color patches are L-decoupled, so applying each color
    # additively (one residual per color) equals the sequential sweep
    xc = oracle.mv_sweeps(A, P, F, x0, b, 0.66, 1, order=order)
    pl = dense.patch_list(P)
    nv = p["ncell"][0] + 1
    x = x0.copy()
    for col in range(16):
        r = b - L @ x
        dx = np.zeros_like(x)
        for i in range(len(pl)):
            if (i % nv) % 4 + 4 * ((i // nv) % 4) != col:
                continue
            d = pl[i][0]
            dx[d] += 0.66 * np.linalg.solve(L[np.ix_(d, d)], r[d])
        x = x + dx
    assert np.abs(xc - x).max() <= 1e-12 * np.abs(x).max()


def test_diag_vanka_closed_form():
    # R17: local system [diag(A_i) b; b^T 0]; closed form
    # dp = (b^T D^-1 r_u - r_p) / (b^T D^-1 b); du = D^-1 (r_u - b dp)
    p, A, P = _setup(4, eta="fourier", weights="full")
    F = oracle.factor(A, P, oracle.FMT_DIAG)
    L = oracle.to_dense(A)
    b = si.random_vector(A["n"], 21)
    x0 = si.random_vector(A["n"], 22)
    xo = oracle.additive_sweeps(A, P, F, x0, b, 0.1, 1)
    r = b - L @ x0
    dx = np.zeros_like(x0)
    for d, _ in dense.patch_list(P):
        vel, pr = d[:-1], d[-1]
        order = np.argsort(d)
        dd = d[order]
        vel = dd[dd < A["nvel"]]
        pr = dd[dd >= A["nvel"]][0]
        Dg = np.diag(L)[vel]
        bb = L[vel, pr]
        dp = (bb @ (r[vel] / Dg) - r[pr]) / (bb @ (bb / Dg))
        du = (r[vel] - bb * dp) / Dg
        dx[vel] += du
        dx[pr] += dp
    np.testing.assert_allclose(xo, x0 + 0.1 * dx, rtol=1e-12, atol=1e-12)


def test_single_patch_covering_everything_is_exact_solve():
    # Schwarz with one subdomain is a direct solve.  The cavity
    # system is singular (constant pressure), so use the pinned system (R4).
    p = si.problem(2, (3, 3), si.KIND_CAVITY, eta="fourier")
    A = oracle.assemble(p)
    L = oracle.to_dense(A)
    pin = A["nvel"]
    keep = np.array([i for i in range(A["n"]) if i != pin])
    Lp = L[np.ix_(keep, keep)]
    bp = A["b"][keep]
    rp = np.zeros(len(keep) + 1, np.int64)
    rows, cols = np.nonzero(Lp != 0)
    rp[1:] = np.cumsum(np.bincount(rows, minlength=len(keep)))
    Ap = {"n": len(keep), "nvel": A["nvel"], "rp": rp, "ci": cols.astype(np.int32),
          "val": Lp[rows, cols].copy()}
    for fmt in (oracle.FMT_ROWS, oracle.FMT_LU):
        P1 = {"offs": np.array([0, len(keep)], np.int64), "dofs": np.arange(len(keep), dtype=np.int32),
              "w": np.ones(len(keep))}
        F = oracle.factor(Ap, P1, fmt)
        x0 = si.random_vector(len(keep), 5)
        if fmt == oracle.FMT_ROWS:
            x1 = oracle.additive_sweeps(Ap, P1, F, x0, bp, 1.0, 1)
        else:
            x1 = oracle.mv_sweeps(Ap, P1, F, x0, bp, 1.0, 1)
        xs = np.linalg.solve(Lp, bp)
        np.testing.assert_allclose(x1, xs, rtol=1e-10, atol=1e-12)


@pytest.mark.parametrize("weights", ["pou", "own", "full"])
def test_exact_solution_is_fixed_point(weights):
    p, A, P = _setup(6, eta="fourier", weights=weights)
    F = oracle.factor(A, P, oracle.FMT_ROWS)
    L = oracle.to_dense(A)
    xs = si.random_vector(A["n"], 9)
    b = L @ xs
    x1 = oracle.additive_sweeps(A, P, F, xs, b, 0.66, 3)
    assert np.abs(x1 - xs).max() <= 1e-12 * np.abs(xs).max()


def test_rav_independent_of_patch_order():
    p, A, P = _setup(7, eta="fourier")
    F = oracle.factor(A, P, oracle.FMT_ROWS)
    b = si.random_vector(A["n"], 1)
    x0 = si.random_vector(A["n"], 2)
    x1 = oracle.additive_sweeps(A, P, F, x0, b, 0.66, 2)
    # reverse the patch list
    npch = len(P["offs"]) - 1
    perm = np.arange(npch)[::-1]
    sizes = np.diff(P["offs"])[perm]
    offs = np.zeros(npch + 1, np.int64); offs[1:] = np.cumsum(sizes)
    dofs = np.concatenate([P["dofs"][P["offs"][i]:P["offs"][i + 1]] for i in perm])
    w = np.concatenate([P["w"][P["offs"][i]:P["offs"][i + 1]] for i in perm])
    P2 = {"offs": offs, "dofs": dofs, "w": w}
    F2 = oracle.factor(A, P2, oracle.FMT_ROWS)
    x2 = oracle.additive_sweeps(A, P2, F2, x0, b, 0.66, 2)
    assert np.abs(x1 - x2).max() <= 1e-13 * np.abs(x1).max()


def test_rav_3d_matches_dense():
    p, A, P = _setup(2, dim=3, eta="fourier")
    F = oracle.factor(A, P, oracle.FMT_ROWS)
    L = oracle.to_dense(A)
    b = si.random_vector(A["n"], 31)
    x0 = si.random_vector(A["n"], 32)
    xo = oracle.additive_sweeps(A, P, F, x0, b, 0.66, 1)
    xd = dense.additive_sweep(L, b, x0, dense.patch_list(P), 0.66, True)
    assert np.abs(xo - xd).max() <= 1e-12 * np.abs(xd).max()


def test_sampled_sweep_equals_full_sweep():
    p, A, P = _setup(8, kind=si.KIND_MMS, eta="fourier")
    F = oracle.factor(A, P, oracle.FMT_ROWS)
    x0 = si.random_vector(A["n"], 41)
    x1 = oracle.additive_sweeps(A, P, F, x0, A["b"], 0.66, 1)
    sample = np.random.Generator(np.random.PCG64(3)).choice(A["n"], 50, replace=False)
    xs = oracle.rav_sweep_sampled(A, P, x0, A["b"], 0.66, sample)
    np.testing.assert_allclose(xs, x1[sample], rtol=1e-13, atol=1e-13)


def test_lu_pivoting_and_transposed_solve():
    # [[0,1],[1,0]] requires pivoting; S:265 transposed solve = row of inverse
    LU, piv = oracle.lu_factor(np.array([[0.0, 1.0], [1.0, 0.0]]))
    np.testing.assert_allclose(oracle.lu_solve(LU, piv, [3.0, 4.0]), [4.0, 3.0])
    M = np.random.Generator(np.random.PCG64(5)).standard_normal((8, 8))
    LU, piv = oracle.lu_factor(M)
    inv = np.linalg.inv(M)
    for j in range(8):
        e = np.eye(8)[j]
        np.testing.assert_allclose(oracle.lu_solve(LU, piv, e, trans=True), inv[j], rtol=1e-10, atol=1e-12)
    with pytest.raises(oracle.SingularLocalSystem):
        oracle.lu_factor(np.array([[1.0, 2.0], [2.0, 4.0]]))


def test_oracle_sweeps_are_thread_count_independent():
    """The oracle's parallel loops (residual rows, per-patch products / local solves) write
    disjoint slots and the corrections are summed serially in ascending patch order, so 1
    and all threads give the same bits (AV/RAV rows and the LU-based diagonal Vanka)."""
    prob = si.problem(2, (12, 10), si.KIND_MMS, eta="fourier")
    A = oracle.assemble(prob)
    x0 = si.initial_guess(A["n"], seed=5)
    out = {}
    for t in (1, 4):
        prev = oracle.set_num_threads(t)
        for w, fmt, om in (("pou", oracle.FMT_ROWS, 0.66), ("full", oracle.FMT_DIAG, 0.1)):
            P = oracle.patches(prob, w)
            F = oracle.factor(A, P, fmt)
            out[(t, w)] = oracle.additive_sweeps(A, P, F, x0, A["b"], om, 3)
        oracle.set_num_threads(prev)
    for w in ("pou", "full"):
        assert np.array_equal(out[(1, w)], out[(4, w)]), w
