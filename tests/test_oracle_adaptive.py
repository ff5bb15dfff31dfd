"""Pins of the adaptive-hierarchy oracle (oracle/adaptive.py; SURVEY section 8 row
f4, reading R20) against what the paper and the mathematics fix:
* the paper's Table 1 (tests/golden/table1_cavity_hierarchy.txt): element and
  DoF counts of levels 1-7 of the driven-cavity hierarchy, exactly;
* 2:1 edge balance and nesting, by brute force;
* with the uniform marker the adaptive code reproduces the structured Q1-Q1
  oracle (operator, rhs, patches, transfers) -- pinned in test_oracle_q1q1.py;
* hanging-node constraints: L = L^T, constants in the kernel of C, the pressure
  prolongation is exact for linear functions, hanging weights 1/2;
* one RAV sweep equals the dense Eq. 13 on an adaptive level (brute force);
* V-cycles in the paper's setting converge with AV the slowest.
"""
import os

import numpy as np
import pytest

import oracle
import seeded_inputs as si
from oracle import adaptive as ad
from oracle import dense

GOLDEN = os.path.join(os.path.dirname(__file__), "golden", "table1_cavity_hierarchy.txt")


def table1():
    rows = [l.split() for l in open(GOLDEN) if l.strip() and not l.startswith("#")]
    return {int(r[0]): (int(r[1]), int(r[2])) for r in rows[1:]}


def test_cavity_hierarchy_reproduces_table1():
    T = table1()
    cells, N = ad.hierarchy_cells(7)
    for k, c in enumerate(cells, start=1):
        m = ad.Mesh(c, N)
        assert (len(c), 3 * len(m.regular)) == T[k], k


def _leaf_at_point(cells, x, y):
    return [c for c in cells if c[0] <= x < c[0] + c[2] and c[1] <= y < c[1] + c[2]]


def test_balance_and_nesting_brute_force():
    cells, N = ad.hierarchy_cells(5)
    for k, c in enumerate(cells):
        # every lattice unit square lies in exactly one leaf; edge neighbours differ by <= one level
        cover = {}
        for (x0, y0, s) in c:
            for i in range(x0, x0 + s):
                for j in range(y0, y0 + s):
                    assert (i, j) not in cover
                    cover[(i, j)] = s
        assert len(cover) == N * N
        for (i, j), s in cover.items():
            for (a, b) in ((i + 1, j), (i, j + 1)):
                if (a, b) in cover:
                    t = cover[(a, b)]
                    assert max(s, t) <= 2 * min(s, t), (k, i, j)
        if k > 0:   # nesting: every leaf lies inside one leaf of the previous level
            prev = cells[k - 1]
            for (x0, y0, s) in c:
                par = _leaf_at_point(prev, x0, y0)
                assert len(par) == 1 and par[0][2] >= s
                px, py, ps = par[0]
                assert px <= x0 and x0 + s <= px + ps and py <= y0 and y0 + s <= py + ps


@pytest.mark.parametrize("kind", [si.KIND_CAVITY, si.KIND_MMS])
def test_uniform_marker_reproduces_structured_q1q1(kind):
    prob = si.problem(2, (32, 32), kind, eta="fourier", elem=si.ELEM_Q1Q1)
    cells, N = ad.hierarchy_cells(3, uniform=True)
    assert N == 32 and all(len(c) == 64 * 4 ** k for k, c in enumerate(cells))
    m = ad.Mesh(cells[-1], N)
    assert not m.hang
    A = ad.assemble(prob, m)
    O = oracle.assemble(prob)
    assert np.array_equal(A["rp"], O["rp"]) and np.array_equal(A["ci"], O["ci"])
    assert np.abs(A["val"] - O["val"]).max() <= 1e-14 * np.abs(O["val"]).max()
    assert np.abs(A["b"] - O["b"]).max() <= 1e-13 * max(np.abs(O["b"]).max(), 1e-300)
    P = ad.patches(A, m)
    Po = oracle.patches(prob, "pou")
    for k in ("offs", "dofs", "w"):
        assert np.array_equal(P[k], Po[k])
    mc = ad.Mesh(cells[-2], N)
    T = ad.prolongation(m, mc)
    To = oracle.prolongation(prob, dict(prob, ncell=[16, 16, 1]))
    for k in ("rp", "ci", "val"):
        assert np.array_equal(T[k], To[k])


def test_hanging_constraints():
    prob = si.problem(2, (32, 32), si.KIND_CAVITY, eta="fourier", elem=si.ELEM_Q1Q1)
    cells, N = ad.hierarchy_cells(4)
    m = ad.Mesh(cells[-1], N)
    assert len(m.hang) > 0
    for v, (a, b) in m.hang.items():          # midpoint of its coarse edge, weights 1/2
        assert 2 * v[0] == a[0] + b[0] and 2 * v[1] == a[1] + b[1]
        e = m.expand(v)
        assert abs(sum(e.values()) - 1.0) == 0.0
    A = ad.assemble(prob, m)
    L = oracle.to_dense(A)
    assert np.array_equal(L, L.T)
    nu = A["nvel"]
    Cp = L[nu:, nu:]
    assert np.abs(Cp @ np.ones(Cp.shape[0])).max() <= 1e-12 * np.abs(Cp).max()
    # pressure prolongation is exact for linear functions
    mc = ad.Mesh(cells[-2], N)
    T = ad.prolongation(m, mc)
    lin = lambda verts: np.array([0.3 + 1.7 * x / N - 0.9 * y / N for (x, y) in verts])
    rows = np.repeat(np.arange(T["n"]), np.diff(T["rp"]))
    y = np.bincount(rows, weights=T["val"] * np.concatenate([np.zeros(mc.nvel), lin(mc.regular)])[T["ci"]],
                    minlength=T["n"])
    assert np.abs(y[m.nvel:] - lin(m.regular)).max() <= 1e-14


def test_rav_sweep_on_adaptive_level_equals_dense_eq13():
    prob = si.problem(2, (16, 16), si.KIND_MMS, eta="fourier", elem=si.ELEM_Q1Q1)
    cells, N = ad.hierarchy_cells(2)
    m = ad.Mesh(cells[-1], N)
    A = ad.assemble(prob, m)
    P = ad.patches(A, m)
    F = oracle.factor(A, P, oracle.FMT_ROWS)
    x0 = si.initial_guess(A["n"], seed=37)
    xo = oracle.additive_sweeps(A, P, F, x0, A["b"], 0.66, 2)
    L = oracle.to_dense(A)
    xd = x0.copy()
    for _ in range(2):
        xd = dense.additive_sweep(L, A["b"], xd, dense.patch_list(P), 0.66, restricted=True)
    assert np.linalg.norm(xo - xd) <= 1e-12 * np.linalg.norm(xd)


def test_vcycle_on_adaptive_hierarchy_paper_setting():
    prob = si.problem(2, (8, 8), si.KIND_CAVITY, elem=si.ELEM_Q1Q1)
    cyc = {}
    for sm, om in [("rav", 0.66), ("mv", 0.66), ("av", 0.1)]:
        H = ad.AdaptiveHierarchy(prob, 4, sm)
        _, k, hist = H.solve(rtol=1e-8, omega=om, pre=3, post=3, maxit=300)
        assert hist[-1] <= 1e-8 * hist[0], (sm, k)
        cyc[sm] = k
    assert cyc["mv"] <= cyc["rav"] < cyc["av"], cyc
