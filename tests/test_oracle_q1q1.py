"""Pins of the oracle's stabilized Q1-Q1 discretization (the paper's own pair,
P:76-80 Eq. 8; reading R18 in DESIGN.md) against
closed forms that do not come from the oracle:

* constant-eta A, B and C equal Kronecker products of exactly integrated 1D Q1
  element matrices (numpy polynomial integration, not the oracle's 2-point
  Gauss rule), incl. the Dirichlet lift of the cavity lid (R8);
* the textbook Q1 stiffness stencil (8/3 centre, -1/3 neighbours, S:163
  "corner diagonal 2/3 per element"), C 1 = 0 and C <= 0;
* SPEC's sizes: 8x8 cavity -> 98 velocity + 81 pressure DoFs, interior
  patches of 19 DoFs with 3 restricted (velocity on the pressure node + p,
  P:122);
* discrete divergence of constant / linear fields;
* MMS convergence: velocity L2 error ratio ~4 per refinement;
* RAV / AV / MV on Q1-Q1 equal the dense explicit Eqs. 11-13 (brute force);
* V-cycles: the paper's settings (AV omega 0.1, RAV / MV omega 0.66)
  all converge, with MV <= RAV < AV in cycles, h-robust RAV.
"""
import numpy as np
import numpy.polynomial.polynomial as npoly
import pytest

import oracle
import seeded_inputs as si
from oracle import dense

Q1 = [np.array([1.0, -1.0]), np.array([0.0, 1.0])]
BETA0 = si.BETA0


def _int01(c):
    ic = npoly.polyint(c)
    return npoly.polyval(1.0, ic) - npoly.polyval(0.0, ic)


def global_1d(n, h):
    K = np.array([[_int01(npoly.polymul(npoly.polyder(a), npoly.polyder(b))) / h for b in Q1] for a in Q1])
    M = np.array([[_int01(npoly.polymul(a, b)) * h for b in Q1] for a in Q1])
    D = np.array([[_int01(npoly.polymul(m, npoly.polyder(a))) for m in Q1] for a in Q1])   # [a][m]
    Kg = np.zeros((n + 1, n + 1)); Mg = np.zeros_like(Kg); Dg = np.zeros_like(Kg)
    for e in range(n):
        s = slice(e, e + 2)
        Kg[s, s] += K; Mg[s, s] += M; Dg[s, s] += D
    return Kg, Mg, Dg


def expected_L(dim, n, kind, eta=1.0, beta=BETA0):
    h = 1.0 / n
    K, M, D = global_1d(n, h)
    def kr(mats):
        out = mats[dim - 1]
        for k in range(dim - 2, -1, -1):
            out = np.kron(out, mats[k])
        return out
    lap = sum(kr([K if j == k else M for j in range(dim)]) for k in range(dim))
    A = eta * lap
    B = [-kr([D if j == c else M for j in range(dim)]) for c in range(dim)]   # B[c][a][m]
    C = -beta / eta * (dim * h * h) * lap        # h_e^2 = d h^2 (element diameter squared)
    nn = n + 1
    ids = np.arange(nn ** dim)
    coords = np.array([(ids // nn ** k) % nn for k in range(dim)]).T
    free = ids[np.all((coords > 0) & (coords < n), axis=1)]
    nf, nv = len(free), nn ** dim
    L = np.zeros((dim * nf + nv, dim * nf + nv))
    for c in range(dim):
        rows = dim * np.arange(nf) + c
        L[np.ix_(rows, rows)] = A[np.ix_(free, free)]
        L[rows, dim * nf:] = B[c][free, :]
        L[dim * nf:, rows] = B[c][free, :].T
    L[dim * nf:, dim * nf:] = C
    b = np.zeros(dim * nf + nv)
    if kind == si.KIND_CAVITY:
        top = dim - 1
        lid = (coords[:, top] == n) & np.all([(coords[:, k] > 0) & (coords[:, k] < n) for k in range(top)], axis=0)
        ud = lid.astype(float)
        b[0:dim * nf:dim] -= A[np.ix_(free, ids)] @ ud
        b[dim * nf:] -= B[0].T @ ud
    return L, b


@pytest.mark.parametrize("dim,n", [(2, 2), (2, 4), (2, 7), (3, 3)])
def test_q1q1_constant_eta_operator_is_kronecker_of_exact_1d_matrices(dim, n):
    p = si.problem(dim, [n] * dim, si.KIND_CAVITY, elem=si.ELEM_Q1Q1)
    A = oracle.assemble(p)
    Lo = oracle.to_dense(A)
    Le, be = expected_L(dim, n, si.KIND_CAVITY)
    assert Lo.shape == Le.shape
    assert np.abs(Lo - Le).max() <= 1e-13 * np.abs(Le).max()
    assert np.abs(A["b"] - be).max() <= 1e-13 * max(1.0, np.abs(be).max())


def test_q1q1_stencils_and_stabilization_properties():
    n = 6
    h = 1.0 / n
    p = si.problem(2, (n, n), si.KIND_HOMOGENEOUS, elem=si.ELEM_Q1Q1)
    A = oracle.assemble(p)
    Lo = oracle.to_dense(A)
    nu = A["nvel"]
    # interior velocity node (3, 3): 8/3 centre, -1/3 for all 8 neighbours (h-invariant in 2D)
    def vel(ax, ay, c=0):
        return 2 * ((ax - 1) + (n - 1) * (ay - 1)) + c
    assert Lo[vel(3, 3), vel(3, 3)] == pytest.approx(8 / 3, rel=1e-14)
    for dx in (-1, 0, 1):
        for dy in (-1, 0, 1):
            if dx or dy:
                assert Lo[vel(3, 3), vel(3 + dx, 3 + dy)] == pytest.approx(-1 / 3, rel=1e-13)
    assert Lo[vel(3, 3), vel(3, 3, 1)] == 0.0          # no inter-component coupling
    C = Lo[nu:, nu:]
    assert np.abs(C @ np.ones(C.shape[0])).max() <= 1e-12 * np.abs(C).max()   # constants in the kernel
    assert np.linalg.eigvalsh(C).max() <= 1e-12 * np.abs(C).max()            # negative semidefinite
    vc = 3 + 7 * 3                                                           # interior vertex (3, 3)
    assert C[vc, vc] == pytest.approx(-BETA0 * 2 * h * h * 8 / 3, rel=1e-13)
    # B^T applied to the constant field (1, 0) vanishes at deep interior vertices; (x, 0) gives -h^2
    xs = np.zeros(A["n"]); lin = np.zeros(A["n"])
    for ay in range(1, n):
        for ax in range(1, n):
            xs[vel(ax, ay)] = 1.0
            lin[vel(ax, ay)] = ax * h
    BT = Lo[nu:, :nu]
    for vx, vy in [(2, 2), (3, 4)]:
        v = vx + 7 * vy
        assert abs((BT @ xs[:nu])[v]) <= 1e-15
        assert (BT @ lin[:nu])[v] == pytest.approx(-h * h, rel=1e-13)


def test_q1q1_sizes_and_patches_match_spec():
    p = si.problem(2, (8, 8), si.KIND_CAVITY, elem=si.ELEM_Q1Q1)
    s = oracle.sizes(p)
    assert s["nvel"] == 98 and s["np"] == 81 and s["n"] == 179
    A = oracle.assemble(p)
    P = oracle.patches(p, "pou")
    Lo = oracle.to_dense(A)
    nu = A["nvel"]
    for i in range(81):
        d = P["dofs"][P["offs"][i]:P["offs"][i + 1]]
        w = P["w"][P["offs"][i]:P["offs"][i + 1]]
        # the nonzero pattern of row i of B^T plus p_i (structural support)
        support = np.nonzero(Lo[nu + i, :nu])[0]
        assert set(support) <= set(d[d < nu]) and nu + i in set(d)
        vx, vy = i % 9, i // 9
        interior = 0 < vx < 8 and 0 < vy < 8
        if 1 < vx < 7 and 1 < vy < 7:
            assert len(d) == 19
        # restricted = velocity DoFs on the pressure node + p_i (weights 0/1)
        rest = set(d[w > 0])
        exp = {nu + i} | ({2 * ((vx - 1) + 7 * (vy - 1)), 2 * ((vx - 1) + 7 * (vy - 1)) + 1} if interior else set())
        assert rest == exp
        assert set(np.unique(w)) <= {0.0, 1.0}
    F = oracle.factor(A, P, oracle.FMT_ROWS)
    assert F["fac"].size == sum(int((P["w"][P["offs"][i]:P["offs"][i + 1]] > 0).sum()) *
                                int(P["offs"][i + 1] - P["offs"][i]) for i in range(81))   # 3 x 19 rows


def test_q1q1_mms_convergence_rate():
    errs = []
    for n in (8, 16, 32):
        p = si.problem(2, (n, n), si.KIND_MMS, elem=si.ELEM_Q1Q1)
        A = oracle.assemble(p)
        import scipy.sparse as sp
        import scipy.sparse.linalg as spl
        M = sp.csr_matrix((A["val"], A["ci"], A["rp"]), shape=(A["n"], A["n"])).tolil()
        nu = A["nvel"]
        # the stabilized system is nonsingular up to the constant pressure: pin vertex 0 (R4)
        M[nu, :] = 0.0
        M[nu, nu] = 1.0
        b = A["b"].copy()
        b[nu] = 0.0
        x = spl.spsolve(M.tocsc(), b)
        eu, ep = oracle.mms_errors(p, x)
        errs.append((eu, ep))
    ru = [errs[i][0] / errs[i + 1][0] for i in range(2)]
    assert 3.4 < ru[0] < 4.6 and 3.6 < ru[1] < 4.4, ru       # O(h^2) velocity
    rp = [errs[i][1] / errs[i + 1][1] for i in range(2)]
    assert min(rp) > 1.8, rp                                   # pressure converges at least O(h)


@pytest.mark.parametrize("weights", ["pou", "full"])
def test_q1q1_additive_sweep_equals_dense_explicit_operator(weights):
    p = si.problem(2, (4, 5), si.KIND_MMS, eta="fourier", elem=si.ELEM_Q1Q1)
    A = oracle.assemble(p)
    P = oracle.patches(p, weights)
    F = oracle.factor(A, P, oracle.FMT_ROWS)
    x0 = si.initial_guess(A["n"], seed=5)
    xo = oracle.additive_sweeps(A, P, F, x0, A["b"], 0.66, 2)
    L = oracle.to_dense(A)
    xd = x0.copy()
    for _ in range(2):
        xd = dense.additive_sweep(L, A["b"], xd, dense.patch_list(P), 0.66, restricted=weights != "full")
    assert np.linalg.norm(xo - xd) <= 1e-12 * np.linalg.norm(xd)


def test_q1q1_multiplicative_sweep_equals_dense_sequential():
    p = si.problem(2, (4, 4), si.KIND_CAVITY, eta="fourier", elem=si.ELEM_Q1Q1)
    A = oracle.assemble(p)
    P = oracle.patches(p, "full")
    F = oracle.factor(A, P, oracle.FMT_LU)
    x0 = si.initial_guess(A["n"], seed=6)
    xo = oracle.mv_sweeps(A, P, F, x0, A["b"], 0.66, 2)
    L = oracle.to_dense(A)
    xd = x0.copy()
    for _ in range(2):
        xd = dense.mv_sweep(L, A["b"], xd, dense.patch_list(P), 0.66)
    assert np.linalg.norm(xo - xd) <= 1e-12 * np.linalg.norm(xd)


def test_q1q1_vcycle_paper_settings_converge_with_paper_ordering():
    """The paper's driven-cavity setting on uniform grids (coarse grid of
    three uniform refinements = 8x8, V(3,3) P:136, omega 0.66 RAV/MV and 0.1 AV
    P:132, 1e8 reduction): all three smoothers converge and the cycle counts
    order as in Fig. 4 (AV consistently the most; MV <= RAV)."""
    for n in (32, 64):
        p = si.problem(2, (n, n), si.KIND_CAVITY, elem=si.ELEM_Q1Q1)
        nl = int(np.log2(n // 8)) + 1
        cyc = {}
        for sm, om in [("rav", 0.66), ("mv", 0.66), ("av", 0.1)]:
            H = oracle.Hierarchy(p, nl, sm)
            _, k, hist = H.solve(rtol=1e-8, omega=om, pre=3, post=3, maxit=400)
            assert hist[-1] <= 1e-8 * hist[0], (sm, n, k)
            cyc[sm] = k
        assert cyc["mv"] <= cyc["rav"] < cyc["av"], cyc
