"""Dense one-cycle pin of the oracle's V-cycle (or_vcycle, Fig. 1, P:86;
S:406) -- the cycle composition written out as explicit matrices.

A V(pre, post) cycle is an affine map x1 = E x0 + M b.  Built from the level
operators L_l, the prolongations P_l (R = P^T), the dense smoother of
Eqs. 11-13 (oracle/dense.py: inverses of the extracted local systems, P:114,
P:122) and the pinned coarse inverse (R4: the pressure DoF of vertex 0 removed,
set to 0; numpy.linalg.inv of the reduced matrix):

    smoothing sweep   x <- x + S (b - L x)             E <- (I - S L) E,   M <- (I - S L) M + S
    coarse correction x <- x + P M_c P^T (b - L x)     E <- (I - P M_c P^T L) E,
                                                       M <- M + P M_c P^T (I - L M)
    level 0           x = C_pin b                      (E, M) = (0, C_pin)

where M_c is the M of the level below (its cycle starts from x = 0).  For a
smoother written as a product (multiplicative Vanka, Eq. 11) the sweep's
(E_s, M_s) pair is composed patch by patch.  The test compares or_vcycle with
E x0 + M b on 4x4 / 6x6 (two levels) and 8x8 (three levels, config c1) meshes
and checks that the pin is sharp: V(2,1), V(3,0), V(1,2) -- one sweep dropped
or moved -- differ from V(2,2) by far more than the tolerance.
"""
import numpy as np
import pytest

import oracle
from oracle import dense
import seeded_inputs as si


def _sweep_affine(L, patches, omega, smoother):
    """(E_s, M_s) of one smoothing sweep: x <- E_s x + M_s b."""
    n = L.shape[0]
    if smoother in ("rav", "av"):
        S = dense.S_additive(L, patches, omega, restricted=(smoother == "rav"))
        return np.eye(n) - S @ L, S
    assert smoother == "mv"           # Eq. 11, ascending patch order
    E, M = np.eye(n), np.zeros((n, n))
    for dofs, _ in patches:
        K = omega * np.linalg.inv(L[np.ix_(dofs, dofs)])
        # x <- x + R^T K R (b - L x): rows `dofs` change
        dE = K @ (L[dofs, :] @ E)
        dM = K @ (np.eye(n)[dofs, :] - L[dofs, :] @ M)
        E[dofs, :] -= dE
        M[dofs, :] += dM
    return E, M


def _dense_cycle(H, smoother, pre, post, omega):
    """(E, M) of one V(pre, post) cycle on the finest level of oracle Hierarchy H."""
    nl = len(H.probs)
    Ls = [oracle.to_dense(A) for A in H.A]
    # level 0: pinned coarse inverse (R4)
    n0 = Ls[0].shape[0]
    keep = np.array([i for i in range(n0) if i != H.pin])
    C = np.zeros((n0, n0))
    C[np.ix_(keep, keep)] = np.linalg.inv(Ls[0][np.ix_(keep, keep)])
    Mc = C
    E = None
    for l in range(1, nl):
        L = Ls[l]
        n = L.shape[0]
        P = oracle.to_dense(H.T[l])
        Es, Ms = _sweep_affine(L, dense.patch_list(H.P[l]), omega, smoother)
        E, M = np.eye(n), np.zeros((n, n))
        for _ in range(pre):
            E, M = Es @ E, Es @ M + Ms
        Q = P @ Mc @ P.T
        E, M = E - Q @ (L @ E), M + Q @ (np.eye(n) - L @ M)
        for _ in range(post):
            E, M = Es @ E, Es @ M + Ms
        Mc = M
    return E, M


CASES = [((4, 4), 2), ((6, 6), 2), ((8, 8), 3)]


@pytest.mark.parametrize("ncell,levels", CASES)
@pytest.mark.parametrize("smoother,omega", [("rav", 0.66), ("av", 0.1), ("mv", 0.66)])
def test_vcycle_equals_dense_composition(ncell, levels, smoother, omega):
    p = si.problem(2, ncell, si.KIND_CAVITY, eta="fourier")
    H = oracle.Hierarchy(p, levels, smoother)
    n = H.fine["n"]
    x0 = si.random_vector(n, 11)
    b = si.random_vector(n, 12)
    E, M = _dense_cycle(H, smoother, 2, 2, omega)
    want = E @ x0 + M @ b
    got = H.vcycle(x0, b, 2, 2, omega)
    scale = np.abs(want).max()
    assert np.abs(got - want).max() <= 1e-10 * scale, np.abs(got - want).max() / scale
    # sharpness: a cycle with one smoothing sweep dropped or moved is far away
    for pre, post in ((2, 1), (3, 0), (1, 2)):
        Em, Mm = _dense_cycle(H, smoother, pre, post, omega)
        other = Em @ x0 + Mm @ b
        assert np.abs(other - want).max() > 1e-4 * scale, (pre, post)


def test_vcycle_pre_post_counts_are_honoured():
    """V(pre, post) for several (pre, post) -- the oracle takes exactly the sweeps asked for."""
    p = si.problem(2, (4, 4), si.KIND_CAVITY)
    H = oracle.Hierarchy(p, 2, "rav")
    n = H.fine["n"]
    x0 = si.random_vector(n, 21)
    b = si.random_vector(n, 22)
    for pre, post in ((0, 0), (1, 0), (0, 1), (2, 1), (1, 3)):
        E, M = _dense_cycle(H, "rav", pre, post, 0.66)
        want = E @ x0 + M @ b
        got = H.vcycle(x0, b, pre, post, 0.66)
        assert np.abs(got - want).max() <= 1e-10 * np.abs(want).max(), (pre, post)


def test_solve_history_is_iterated_cycle():
    """or_mg_solve = repeated or_vcycle with the R11 stopping test: its residual history
    equals ||b - L x_k|| of x_k = E x_{k-1} + M b (dense), on c1."""
    c = si.CONFIGS["c1"]
    p = si.problem(2, c["ncell"], c["kind"], eta=c["eta"])
    H = oracle.Hierarchy(p, c["levels"], "rav")
    E, M = _dense_cycle(H, "rav", c["pre"], c["post"], c["omega"])
    L = oracle.to_dense(H.fine)
    b = H.fine["b"]
    x, k, hist = H.solve(rtol=c["rtol"], omega=c["omega"], pre=c["pre"], post=c["post"])
    xd = np.zeros(H.fine["n"])
    hd = [np.linalg.norm(b - L @ xd)]
    while hd[-1] > c["rtol"] * hd[0] and len(hd) < 200:
        xd = E @ xd + M @ b
        hd.append(np.linalg.norm(b - L @ xd))
    assert k == len(hd) - 1, (k, len(hd) - 1)
    np.testing.assert_allclose(hist, hd, rtol=1e-6, atol=1e-12 * hd[0])
