"""Pins of the oracle's discretization (assembly, patches, transfers) against
closed forms that do not come from the oracle itself.

* Constant-eta operators equal Kronecker products of exactly integrated 1D
  Q2/Q1 element matrices (numpy polynomial integration, not the oracle's Gauss
  rule): pins A and B of P:74 Eq. 7 entry by entry, incl. Dirichlet lifting (R8).
* Textbook Q2 stiffness diagonals (28/45 corner, 256/45 centre, 88/45 edge).
* Discrete divergence of linear fields (B^T (x,-y) = 0, B^T (x,0) = -h^2).
* Patches: P:108's algebraic definition (row of B^T + p_i), interior sizes
  51/376, restricted counts 19/82, partition of unity (exact).
* Transfers: exact interpolation of Q2/Q1 functions; Galerkin identity.
"""
import itertools

import numpy as np
import numpy.polynomial.polynomial as npoly
import pytest

import oracle
import seeded_inputs as si

# --- exact 1D element matrices -------------------------------------------------
Q2 = [np.array([1.0, -3.0, 2.0]), np.array([0.0, 4.0, -4.0]), np.array([0.0, -1.0, 2.0])]  # coeffs in t
Q1 = [np.array([1.0, -1.0]), np.array([0.0, 1.0])]


def _int01(c):
    ic = npoly.polyint(c)
    return npoly.polyval(1.0, ic) - npoly.polyval(0.0, ic)


def elem_1d(h):
    K = np.array([[_int01(npoly.polymul(npoly.polyder(a), npoly.polyder(b))) / h for b in Q2] for a in Q2])
    M = np.array([[_int01(npoly.polymul(a, b)) * h for b in Q2] for a in Q2])
    D = np.array([[_int01(npoly.polymul(m, npoly.polyder(a))) for m in Q1] for a in Q2])
    N = np.array([[_int01(npoly.polymul(m, a)) * h for m in Q1] for a in Q2])
    return K, M, D, N


def global_1d(n, h):
    K, M, D, N = elem_1d(h)
    Kg = np.zeros((2 * n + 1, 2 * n + 1)); Mg = np.zeros_like(Kg)
    Dg = np.zeros((2 * n + 1, n + 1)); Ng = np.zeros_like(Dg)
    for e in range(n):
        q = slice(2 * e, 2 * e + 3); v = slice(e, e + 2)
        Kg[q, q] += K; Mg[q, q] += M; Dg[q, v] += D; Ng[q, v] += N
    return Kg, Mg, Dg, Ng


def kron_operator(dim, n, eta=1.0):
    """Full (no elimination) velocity-scalar A and per-component B as Kronecker
    products; index x fastest."""
    h = [1.0 / n] * dim
    G = [global_1d(n, h[k]) for k in range(dim)]
    def kr(mats):  # mats[k] acts on axis k; kron with axis dim-1 outermost
        out = mats[dim - 1]
        for k in range(dim - 2, -1, -1):
            out = np.kron(out, mats[k])
        return out
    A = np.zeros(1)
    terms = []
    for k in range(dim):
        terms.append(kr([G[j][0] if j == k else G[j][1] for j in range(dim)]))
    A = eta * sum(terms)
    B = [-kr([G[j][2] if j == c else G[j][3] for j in range(dim)]) for c in range(dim)]
    return A, B


def expected_L(dim, n, kind):
    A, B = kron_operator(dim, n)
    nn = 2 * n + 1
    nodes = list(itertools.product(*[range(nn)] * dim))  # last axis fastest in product -> reverse
    # lexicographic with x fastest: node id = sum a_k nn^k
    ids = np.arange(nn ** dim)
    coords = np.array([(ids // nn ** k) % nn for k in range(dim)]).T
    interior = np.all((coords > 0) & (coords < 2 * n), axis=1)
    free = ids[interior]
    nf = len(free)
    nv = (n + 1) ** dim
    L = np.zeros((dim * nf + nv, dim * nf + nv))
    for c in range(dim):
        rows = dim * np.arange(nf) + c
        L[np.ix_(rows, rows)] = A[np.ix_(free, free)]
        L[rows, dim * nf:] = B[c][free, :]
        L[dim * nf:, rows] = B[c][free, :].T
    # Dirichlet lift of the cavity lid: u = e_x on the top face interior
    b = np.zeros(dim * nf + nv)
    if kind == si.KIND_CAVITY:
        top = dim - 1
        lid = (coords[:, top] == 2 * n) & np.all(
            [(coords[:, k] > 0) & (coords[:, k] < 2 * n) for k in range(top)], axis=0)
        ud = lid.astype(float)          # component 0 value on all nodes
        b[0:dim * nf:dim] -= A[np.ix_(free, ids)] @ ud
        b[dim * nf:] -= B[0].T @ ud
    return L, b


@pytest.mark.parametrize("dim,n", [(2, 2), (2, 3), (2, 5), (3, 2)])
def test_constant_eta_operator_is_kronecker_of_exact_1d_matrices(dim, n):
    p = si.problem(dim, [n] * dim, si.KIND_CAVITY)
    A = oracle.assemble(p)
    Lo = oracle.to_dense(A)
    Le, be = expected_L(dim, n, si.KIND_CAVITY)
    scale = np.abs(Le).max()
    assert np.abs(Lo - Le).max() <= 1e-13 * scale
    assert np.abs(A["b"] - be).max() <= 1e-13 * max(1.0, np.abs(be).max())


def test_q2_stiffness_diagonals_textbook():
    # 2D Laplacian is h-invariant: a vertex node shared by 4 elements has
    # 4 * 28/45, an edge midpoint 2 * 88/45, a cell centre 256/45.
    p = si.problem(2, (2, 2), si.KIND_HOMOGENEOUS)
    A = oracle.assemble(p)
    Lo = oracle.to_dense(A)
    # free nodes of the 5x5 lattice: interior 3x3, lexicographic
    def vel_row(ax, ay, c=0):
        return 2 * ((ax - 1) + 3 * (ay - 1)) + c
    assert Lo[vel_row(2, 2), vel_row(2, 2)] == pytest.approx(4 * 28 / 45, rel=1e-14)
    assert Lo[vel_row(1, 1), vel_row(1, 1)] == pytest.approx(256 / 45, rel=1e-14)
    assert Lo[vel_row(2, 1), vel_row(2, 1)] == pytest.approx(2 * 88 / 45, rel=1e-14)
    assert Lo[vel_row(2, 1, 1), vel_row(2, 1, 1)] == pytest.approx(2 * 88 / 45, rel=1e-14)


@pytest.mark.parametrize("eta", ["const", "fourier"])
def test_L_symmetric_bitwise(eta):
    p = si.problem(2, (6, 5), si.KIND_MMS, eta=eta)
    A = oracle.assemble(p)
    M = oracle.to_dense(A)
    assert np.array_equal(M, M.T)
    p3 = si.problem(3, (2, 3, 2), si.KIND_CAVITY, eta=eta)
    M3 = oracle.to_dense(oracle.assemble(p3))
    assert np.array_equal(M3, M3.T)


@pytest.mark.parametrize("dim,n", [(2, 8), (3, 5)])
def test_discrete_divergence_of_linear_fields(dim, n):
    p = si.problem(dim, [n] * dim, si.KIND_HOMOGENEOUS, eta="fourier")
    A = oracle.assemble(p)
    M = oracle.to_dense(A)
    nvel, ntot = A["nvel"], A["n"]
    h = 1.0 / n
    nn = 2 * n + 1
    ids = np.arange(nn ** dim)
    coords = np.array([(ids // nn ** k) % nn for k in range(dim)]).T
    interior = np.all((coords > 0) & (coords < 2 * n), axis=1)
    X = coords[interior] * h / 2
    # vertices at least 2 cells from the boundary: their B^T rows see no Dirichlet node
    nv = n + 1
    vid = np.arange(nv ** dim)
    vc = np.array([(vid // nv ** k) % nv for k in range(dim)]).T
    deep = np.all((vc >= 2) & (vc <= n - 2), axis=1)
    rows = nvel + vid[deep]
    assert deep.any()
    # div-free linear field u = (x, -y[, 0])
    u = np.zeros(ntot)
    u[0:nvel:dim] = X[:, 0]
    u[1:nvel:dim] = -X[:, 1]
    assert np.abs(M[rows] @ u).max() <= 1e-15 * 10
    # u = (x, 0[, 0]): -int psi_v div u = -h^dim
    u = np.zeros(ntot)
    u[0:nvel:dim] = X[:, 0]
    np.testing.assert_allclose(M[rows] @ u, -h ** dim, rtol=1e-12)


@pytest.mark.parametrize("dim,n,size,nres", [(2, 6, 51, 19), (3, 4, 376, 82)])
def test_patch_sizes_and_partition_of_unity(dim, n, size, nres):
    p = si.problem(dim, [n] * dim, si.KIND_CAVITY)
    A = oracle.assemble(p)
    for mode in ("pou", "own"):
        P = oracle.patches(p, mode)
        ni = np.diff(P["offs"])
        assert ni.max() == size
        nr = np.add.reduceat((P["w"] > 0).astype(int), P["offs"][:-1])
        if mode == "pou":
            assert nr.max() == nres
        else:
            assert nr.max() == (2 ** dim) * dim + 1
        # sum over patches of the weights of each DoF is exactly 1 (dyadic)
        s = np.zeros(A["n"])
        np.add.at(s, P["dofs"], P["w"])
        assert np.all(s == 1.0)
        # restricted DoFs come first in each patch
        for i in range(len(ni)):
            w = P["w"][P["offs"][i]:P["offs"][i + 1]]
            k = int((w > 0).sum())
            assert np.all(w[:k] > 0) and np.all(w[k:] == 0)


@pytest.mark.parametrize("dim,n", [(2, 5), (3, 3)])
def test_patch_is_structural_Bt_row_support(dim, n):
    # "the degrees of freedom corresponding to the nonzero entries in
    # the i-th row of B^T plus the i-th pressure degree of freedom" (structural
    # pattern, R2)
    p = si.problem(dim, [n] * dim, si.KIND_CAVITY)
    A = oracle.assemble(p)
    P = oracle.patches(p, "pou")
    nvel = A["nvel"]
    for i in range(len(P["offs"]) - 1):
        row = nvel + i
        cols = A["ci"][A["rp"][row]:A["rp"][row + 1]]
        pd = np.sort(P["dofs"][P["offs"][i]:P["offs"][i + 1]])
        assert np.array_equal(pd, np.sort(np.append(cols, row)))


def _nodal(problem, f_vel, f_p):
    """interpolant of (f_vel componentwise, f_p) on the free DoFs"""
    dim, n = problem["dim"], problem["ncell"][0]
    nn = 2 * n + 1
    ids = np.arange(nn ** dim)
    coords = np.array([(ids // nn ** k) % nn for k in range(dim)]).T
    interior = np.all((coords > 0) & (coords < 2 * n), axis=1)
    X = coords[interior] / (2.0 * n)
    nv = n + 1
    vid = np.arange(nv ** dim)
    V = np.array([(vid // nv ** k) % nv for k in range(dim)]).T / n
    u = np.zeros(dim * len(X) + len(V))
    for c in range(dim):
        u[c:dim * len(X):dim] = f_vel(X, c)
    u[dim * len(X):] = f_p(V)
    return u


@pytest.mark.parametrize("dim,n", [(2, 4), (3, 2)])
def test_prolongation_interpolates_q2_q1_exactly(dim, n):
    pf = si.problem(dim, [2 * n] * dim, si.KIND_CAVITY)
    pc = si.problem(dim, [n] * dim, si.KIND_CAVITY)
    T = oracle.prolongation(pf, pc)
    Pm = oracle.to_dense(T)
    # bubble-like Q2 function vanishing on the boundary, bilinear pressure
    fv = lambda X, c: (c + 1) * np.prod(X * (1 - X), axis=1)
    fp = lambda V: np.prod(V + 0.5, axis=1)
    uc = _nodal(pc, fv, fp)
    uf = _nodal(pf, fv, fp)
    np.testing.assert_allclose(Pm @ uc, uf, atol=1e-14)


@pytest.mark.parametrize("dim,n", [(2, 4), (3, 2)])
def test_galerkin_identity_constant_eta(dim, n):
    pf = si.problem(dim, [2 * n] * dim, si.KIND_CAVITY)
    pc = si.problem(dim, [n] * dim, si.KIND_CAVITY)
    Lf = oracle.to_dense(oracle.assemble(pf))
    Lc = oracle.to_dense(oracle.assemble(pc))
    Pm = oracle.to_dense(oracle.prolongation(pf, pc))
    assert np.abs(Pm.T @ Lf @ Pm - Lc).max() <= 1e-13 * np.abs(Lc).max()


def test_viscosity_field_range():
    p = si.problem(2, (4, 4), si.KIND_MMS, eta="fourier")
    xs = np.linspace(0, 1, 201)
    vals = np.array([oracle.eta(p, x, y) for x in xs for y in xs])
    assert 0.0999 <= vals.min() and vals.max() <= 10.001
    assert vals.min() < 0.12 and vals.max() > 8.0
