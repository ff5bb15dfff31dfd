"""Adaptive quadtree hierarchies with hanging nodes -- ORACLE (SURVEY section 8 row
f4; reading R20 in DESIGN.md).  TEST INFRASTRUCTURE ONLY (see oracle/__init__.py).

The paper's grids (Table 1): an 8x8 uniform coarse grid of the
unit square ("three levels of uniform refinement"), refined adaptively towards
the boundaries, 2:1 balance between neighbouring cells, hanging nodes "handled as
constraints and removed from the global system of equations".  The
element pair is the paper's stabilized Q1-Q1 (R18).

Written plainly, step by step:
  * cells live on an integer lattice: N = 8 * 2^(L-1) units per side for an
    L-level hierarchy; a cell is (x0, y0, s) with side s units;
  * level 1 = the 8x8 grid; level k+1 = level k with every leaf cell whose
    closure is closer to the boundary than BANDS[k-1] cells of the finest size
    split in 4 (R20), then 2:1 edge balance by closure refinement;
  * hanging vertex = the midpoint of a leaf edge that is a vertex of another
    leaf; its value is the mean of the edge's end points, resolved
    recursively; boundary vertices are Dirichlet (R8);
  * L = C^T L_full C assembled element by element from the oracle's Q1-Q1
    element matrices (or_element_matrices, pinned in test_oracle_q1q1.py),
    structural pattern = every (row, column) pair the expansion touches;
  * patches: per pressure DoF, the velocity columns of its row + itself,
    restricted = the velocity DoFs on its vertex;
  * prolongation: the coarse Q1 function (hanging and Dirichlet constraints
    folded in) evaluated at the fine free vertices.
Numbering (R9 / R20): free velocity vertices sorted by (y, x), components
interleaved; then pressure on all regular vertices sorted by (y, x).
"""
from __future__ import annotations

import ctypes as C
from typing import Dict, List, Tuple

import numpy as np

from . import FMT_ROWS, Coarse, Hierarchy, Level, _p, desc, factor, lib, to_dense


# ---- mesh ------------------------------------------------------------------------------------
# R20: at step k (level k -> k+1) the leaves closer to the boundary than BANDS[k-1] cells of
# the current finest size h_k = N / (8 2^(k-1)) are split.  With 2:1 balance these bands
# reproduce the element counts of the paper's Table 1 (64, 208, 676, 2296, 7672, 25612, 79648).
BANDS = (2, 3, 5, 8, 13, 19)


def refine_step(cells: set, k: int, N: int, uniform: bool = False) -> set:
    """Level k -> k+1: split the leaves within BANDS[k-1] finest cells of the boundary
    (R20), then balance.  uniform=True splits every leaf (the structured grids, a pin)."""
    band = N + 1 if uniform else BANDS[min(k, len(BANDS)) - 1] * (N // (8 << (k - 1)))
    out = set()
    for (x0, y0, s) in cells:
        d = min(x0, y0, N - (x0 + s), N - (y0 + s))
        if d < band and s > 1:
            h = s // 2
            out |= {(x0, y0, h), (x0 + h, y0, h), (x0, y0 + h, h), (x0 + h, y0 + h, h)}
        else:
            out.add((x0, y0, s))
    return balance(out, N)


def leaf_at(cells: set, sizes: List[int], px: int, py: int):
    """The leaf whose half-open square [x0, x0+s) x [y0, y0+s) holds the lattice point."""
    for s in sizes:
        c = ((px // s) * s, (py // s) * s, s)
        if c in cells:
            return c
    return None


def balance(cells: set, N: int) -> set:
    """2:1 edge balance by closure refinement: split every leaf with an edge neighbour
    more than one level finer, until nothing changes."""
    while True:
        sizes = sorted({c[2] for c in cells}, reverse=True)
        split = []
        for (x0, y0, s) in cells:
            if s < 4:
                continue
            q = s // 4
            probes = []
            for t in range(4):
                probes += [(x0 + s, y0 + t * q), (x0 - 1, y0 + t * q), (x0 + t * q, y0 + s), (x0 + t * q, y0 - 1)]
            for (px, py) in probes:
                if 0 <= px < N and 0 <= py < N:
                    nb = leaf_at(cells, sizes, px, py)
                    if nb is not None and nb[2] <= q:
                        split.append((x0, y0, s))
                        break
        if not split:
            return cells
        for (x0, y0, s) in split:
            cells.discard((x0, y0, s))
            h = s // 2
            cells |= {(x0, y0, h), (x0 + h, y0, h), (x0, y0 + h, h), (x0 + h, y0 + h, h)}


def hierarchy_cells(n_levels: int, n0: int = 8, uniform: bool = False) -> Tuple[List[set], int]:
    S1 = 1 << (n_levels - 1)
    N = n0 * S1
    lv = [{(i * S1, j * S1, S1) for j in range(n0) for i in range(n0)}]
    for k in range(1, n_levels):
        lv.append(refine_step(set(lv[-1]), k, N, uniform))
    return lv, N


# ---- DoFs and constraints --------------------------------------------------------------------
class Mesh:
    def __init__(self, cells: set, N: int):
        self.cells, self.N = cells, N
        self.sizes = sorted({c[2] for c in cells}, reverse=True)
        verts = set()
        for (x0, y0, s) in cells:
            verts |= {(x0, y0), (x0 + s, y0), (x0, y0 + s), (x0 + s, y0 + s)}
        self.hang = {}                      # hanging vertex -> (a, b) end points of its coarse edge
        for (x0, y0, s) in cells:
            h = s // 2
            if s % 2:
                continue
            for (m, a, b) in (((x0 + h, y0), (x0, y0), (x0 + s, y0)), ((x0 + h, y0 + s), (x0, y0 + s), (x0 + s, y0 + s)),
                              ((x0, y0 + h), (x0, y0), (x0, y0 + s)), ((x0 + s, y0 + h), (x0 + s, y0), (x0 + s, y0 + s))):
                if m in verts:
                    self.hang[m] = (a, b)
        self.regular = sorted((v for v in verts if v not in self.hang), key=lambda v: (v[1], v[0]))
        bnd = lambda v: v[0] == 0 or v[1] == 0 or v[0] == N or v[1] == N
        self.free = [v for v in self.regular if not bnd(v)]
        self.vel_id = {v: i for i, v in enumerate(self.free)}
        self.p_id = {v: i for i, v in enumerate(self.regular)}
        self.nvel = 2 * len(self.free)
        self.n = self.nvel + len(self.regular)

    def expand(self, v) -> Dict:
        """Regular vertices (with weights) that determine the value at v."""
        if v not in self.hang:
            return {v: 1.0}
        a, b = self.hang[v]
        out = {}
        for u, w in list(self.expand(a).items()) + list(self.expand(b).items()):
            out[u] = out.get(u, 0.0) + 0.5 * w
        return out


def lid_value(v, N: int, kind: int, c: int) -> float:
    """Cavity lid (R8): u = e_x on the top edge, corners excluded."""
    return 1.0 if (kind == 0 and c == 0 and v[1] == N and 0 < v[0] < N) else 0.0


def assemble(problem: Dict, mesh: Mesh) -> Dict:
    """L = C^T L_full C and b (Eq. 6, Eq. 8), element by element."""
    N = mesh.N
    d = desc(problem)
    L = lib()
    Ae, Be, Ce, Fe = np.zeros(16), np.zeros(4 * 3 * 4), np.zeros(16), np.zeros(4 * 3)
    rows: Dict[int, Dict[int, float]] = {i: {} for i in range(mesh.n)}
    b = np.zeros(mesh.n)

    def add(r, c, v):
        rows[r][c] = rows[r].get(c, 0.0) + v

    for (x0, y0, s) in sorted(mesh.cells, key=lambda c: (c[1], c[0], c[2])):
        org = np.array([x0 / N, y0 / N, 0.0])
        hh = np.array([s / N, s / N, 1.0])
        L.or_element_matrices(C.byref(d), _p(org), _p(hh), _p(Ae), _p(Be), _p(Ce), _p(Fe))
        corners = [(x0 + (a & 1) * s, y0 + (a >> 1) * s) for a in range(4)]
        ex = [mesh.expand(v) for v in corners]
        for a in range(4):
            for c in range(2):
                for ua, wa in ex[a].items():
                    if ua not in mesh.vel_id:          # Dirichlet row: nothing assembled
                        continue
                    r = 2 * mesh.vel_id[ua] + c
                    b[r] += wa * Fe[a * 3 + c]
                    for bb in range(4):
                        for ub, wb in ex[bb].items():
                            v = wa * wb * Ae[a * 4 + bb]
                            if ub in mesh.vel_id:
                                add(r, 2 * mesh.vel_id[ub] + c, v)
                            else:
                                b[r] -= v * lid_value(ub, N, problem["kind"], c)
                    for m in range(4):
                        for um, wm in ex[m].items():
                            v = wa * wm * Be[(a * 3 + c) * 4 + m]
                            add(r, mesh.nvel + mesh.p_id[um], v)
                            add(mesh.nvel + mesh.p_id[um], r, v)
                # Dirichlet velocity lifted into the pressure rows (B^T u_D)
                for ua, wa in ex[a].items():
                    if ua in mesh.vel_id:
                        continue
                    g = lid_value(ua, N, problem["kind"], c)
                    for m in range(4):
                        for um, wm in ex[m].items():
                            b[mesh.nvel + mesh.p_id[um]] -= wa * wm * Be[(a * 3 + c) * 4 + m] * g
        for m in range(4):
            for um, wm in ex[m].items():
                for m2 in range(4):
                    for um2, wm2 in ex[m2].items():
                        add(mesh.nvel + mesh.p_id[um], mesh.nvel + mesh.p_id[um2], wm * wm2 * Ce[m * 4 + m2])
    rp = np.zeros(mesh.n + 1, np.int64)
    ci, val = [], []
    for i in range(mesh.n):
        cols = sorted(rows[i])
        ci += cols
        val += [rows[i][c] for c in cols]
        rp[i + 1] = rp[i] + len(cols)
    return {"n": mesh.n, "nvel": mesh.nvel, "rp": rp, "ci": np.array(ci, np.int32), "val": np.array(val), "b": b}


def patches(A: Dict, mesh: Mesh) -> Dict:
    """Vanka patches: p_v + the velocity columns of its row; restricted = the
    velocity DoFs on v, weights 0/1; order: restricted, p, others (ascending)."""
    offs, dofs, w = [0], [], []
    for v in mesh.regular:
        p = mesh.nvel + mesh.p_id[v]
        cols = A["ci"][A["rp"][p]:A["rp"][p + 1]]
        vel = sorted(int(c) for c in cols if c < mesh.nvel)
        rest = [2 * mesh.vel_id[v], 2 * mesh.vel_id[v] + 1] if v in mesh.vel_id else []
        others = [c for c in vel if c not in rest]
        dofs += rest + [p] + others
        w += [1.0] * (len(rest) + 1) + [0.0] * len(others)
        offs.append(len(dofs))
    return {"offs": np.array(offs, np.int64), "dofs": np.array(dofs, np.int32), "w": np.array(w)}


def prolongation(fine: Mesh, coarse: Mesh) -> Dict:
    """Coarse Q1 functions (constraints folded in, Dirichlet dropped) at the fine free
    vertices (velocity, both components) and at the fine regular vertices (pressure)."""
    rows = []

    def interp(v, need_free):
        c = leaf_at(coarse.cells, coarse.sizes, min(v[0], coarse.N - 1), min(v[1], coarse.N - 1))
        x0, y0, s = c
        tx, ty = (v[0] - x0) / s, (v[1] - y0) / s
        out = {}
        for a in range(4):
            wa = (tx if a & 1 else 1.0 - tx) * (ty if a >> 1 else 1.0 - ty)
            if wa == 0.0:
                continue
            for u, wu in coarse.expand((x0 + (a & 1) * s, y0 + (a >> 1) * s)).items():
                if need_free and u not in coarse.vel_id:
                    continue
                out[u] = out.get(u, 0.0) + wa * wu
        return out

    for v in fine.free:
        e = interp(v, True)
        for c in range(2):
            rows.append(sorted((2 * coarse.vel_id[u] + c, w) for u, w in e.items()))
    for v in fine.regular:
        e = interp(v, False)
        rows.append(sorted((coarse.nvel + coarse.p_id[u], w) for u, w in e.items()))
    rp = np.zeros(len(rows) + 1, np.int64)
    for i, r in enumerate(rows):
        rp[i + 1] = rp[i] + len(r)
    ci = np.array([c for r in rows for c, _ in r], np.int32)
    val = np.array([w for r in rows for _, w in r])
    return {"n": fine.n, "nc": coarse.n, "rp": rp, "ci": ci, "val": val}


def greedy_colors(A: Dict, P: Dict) -> np.ndarray:
    """Greedy multicolouring (R10 / R20), written plainly: patch j conflicts with patch i
    when j holds a DoF of patch i or a DoF coupled to one through L; patches in
    ascending order take the smallest colour no conflicting earlier patch has.
    Returns the colour-major order (ascending inside a colour)."""
    npatch = len(P["offs"]) - 1
    holders: Dict[int, List[int]] = {}
    for i in range(npatch):
        for d in P["dofs"][P["offs"][i]:P["offs"][i + 1]]:
            holders.setdefault(int(d), []).append(i)
    color = [-1] * npatch
    for i in range(npatch):
        touched = set()
        for d in P["dofs"][P["offs"][i]:P["offs"][i + 1]]:
            touched.add(int(d))
            touched |= set(int(c) for c in A["ci"][A["rp"][d]:A["rp"][d + 1]])
        taken = {color[j] for d in touched for j in holders.get(d, []) if j < i}
        c = 0
        while c in taken:
            c += 1
        color[i] = c
    return np.array(sorted(range(npatch), key=lambda i: (color[i], i)), np.int32)


class AdaptiveHierarchy(Hierarchy):
    """The oracle V-cycle on the adaptive hierarchy: level operators,
    RAV / AV / MV patch data and transfers from this module, the C oracle's
    factorizations, sweeps, coarse LU (pin: pressure of vertex (0, 0), R4)."""

    def __init__(self, problem: Dict, n_levels: int, smoother: str = "rav", uniform: bool = False, n0: int = 8,
                 mv_order: str = "ascending"):
        from . import FMT_DIAG, FMT_LU
        self.problem = problem
        self.smoother = smoother
        cells, N = hierarchy_cells(n_levels, n0, uniform)
        self.meshes = [Mesh(c, N) for c in cells]
        self.probs = [problem] * n_levels
        self.A, self.P, self.F, self.T, self.order = [], [], [], [], []
        for l, m in enumerate(self.meshes):
            A = assemble(problem, m)
            self.A.append(A)
            if l == 0:
                self.order.append(None)
                self.P.append(None)
                self.F.append(None)
                self.T.append(None)
                continue
            Pt = patches(A, m)
            if smoother in ("av", "mv", "diag"):
                Pt = dict(Pt, w=np.ones_like(Pt["w"]))
            fmt = {"rav": FMT_ROWS, "av": FMT_ROWS, "mv": FMT_LU, "diag": FMT_DIAG}[smoother]
            self.order.append(greedy_colors(A, Pt) if (smoother == "mv" and mv_order == "color") else None)
            self.P.append(Pt)
            self.F.append(factor(A, Pt, fmt))
            self.T.append(prolongation(m, self.meshes[l - 1]))
        A0 = self.A[0]
        dense = to_dense(A0)
        self.pin = int(A0["nvel"])
        mm = A0["n"] - 1
        self.coarse_lu = np.zeros((mm, mm))
        self.coarse_piv = np.zeros(mm, np.int32)
        if lib().or_coarse_factor(A0["n"], _p(np.ascontiguousarray(dense)), self.pin, _p(self.coarse_lu),
                                  _p(self.coarse_piv)) != 0:
            raise RuntimeError("singular coarse system")
        self._build_structs()
