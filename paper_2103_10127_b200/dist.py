"""Slab-partitioned RAV sweeps over several ranks (SURVEY section 8 rows a11 / e).

The finest level is cut into contiguous slabs of vertex layers along the last
axis (y in 2D, z in 3D).  Rank r owns the patches of its vertex layers
[V0, V1) and therefore the additive corrections of Eq. 13 that they
produce; within a sweep every patch is independent, so the only
communication is

  1. the interface-correction sum: the restricted (partition-of-unity) DoFs of
     a rank's outermost patches that another rank owns receive partial
     corrections from both sides; the non-owner sends its partial sum to the
     owner, which adds it (R16);
  2. the halo refresh: after the update every rank receives the current values
     of the ghost DoFs its residual rows (b - L x on its patch DoFs) read.

Ownership: pressure DoFs by vertex layer; velocity node layer a (1..2n-1) by
the rank that owns vertex layer floor((a + 1) / 2).  Each rank's local system
is generated directly on its GPU by rav_gen_* with a window (include/ravgmg.h):
DoFs = node layers [2 V0 - 4, 2 V1 + 2], vertex layers [V0 - 2, V1 + 1]
(clipped), rows assembled on node layers [2 V0 - 2, 2 V1] and vertex layers
[V0, V1 - 1] -- exactly the rows of its patch DoFs, whose columns stay inside
the window (one element = two node layers of coupling).

This module holds only host logic (partition, index lists, message schedule)
and calls a backend for every compute step, so the same protocol runs on the
GPU (C-ABI kernels, NCCL) and in the CPU tests (gloo, numpy backend).
"""
from __future__ import annotations

from typing import Dict, List, Sequence, Tuple

import numpy as np


def partition_layers(n_vertex_layers: int, nranks: int, min_layers: int = 3) -> List[Tuple[int, int]]:
    """Contiguous vertex-layer ranges [V0, V1) with sizes differing by at most one."""
    if n_vertex_layers < nranks * min_layers:
        raise ValueError(f"{n_vertex_layers} vertex layers cannot give {nranks} slabs of >= {min_layers} layers")
    base, extra = divmod(n_vertex_layers, nranks)
    out, v = [], 0
    for r in range(nranks):
        sz = base + (1 if r < extra else 0)
        out.append((v, v + sz))
        v += sz
    return out


class Slab:
    """Geometry of rank `rank`'s window and its local <-> global DoF maps."""

    def __init__(self, problem: Dict, nranks: int, rank: int):
        self.problem = problem
        self.dim = dim = problem["dim"]
        self.nranks, self.rank = nranks, rank
        nc = [int(c) for c in problem["ncell"][:dim]]
        n = nc[-1]
        self.n_last = n
        self.layers = partition_layers(n + 1, nranks)
        V0, V1 = self.layers[rank]
        self.V0, self.V1 = V0, V1
        self.nlow_free = int(np.prod([2 * c - 1 for c in nc[:-1]]))
        self.nlow_vert = int(np.prod([c + 1 for c in nc[:-1]]))
        self.nvel_glob = dim * self.nlow_free * (2 * n - 1)
        self.nvert_glob = self.nlow_vert * (n + 1)
        clip_n = lambda a: min(max(a, 1), 2 * n - 1)
        clip_v = lambda v: min(max(v, 0), n)
        self.window = {
            "node_lo": clip_n(2 * V0 - 4), "node_hi": clip_n(2 * V1 + 2),
            "vert_lo": clip_v(V0 - 2), "vert_hi": clip_v(V1 + 1),
            "rnode_lo": clip_n(2 * V0 - 2), "rnode_hi": clip_n(2 * V1),
            "rvert_lo": V0, "rvert_hi": V1 - 1,
            "pvert_lo": V0, "pvert_hi": V1 - 1,
        }
        w = self.window
        self.vel_off = dim * self.nlow_free * (w["node_lo"] - 1)
        self.nvel_loc = dim * self.nlow_free * (w["node_hi"] - w["node_lo"] + 1)
        self.vert_off = self.nlow_vert * w["vert_lo"]
        self.nvert_loc = self.nlow_vert * (w["vert_hi"] - w["vert_lo"] + 1)
        self.n_loc = self.nvel_loc + self.nvert_loc
        self.n_patches = self.nlow_vert * (V1 - V0)
        # owned node layers [own_lo, own_hi] (inclusive), owned vertex layers [V0, V1 - 1]
        self.own_node = (max(1, 2 * V0 - 1), min(2 * n - 1, 2 * V1 - 2))

    def local_problem(self) -> Dict:
        p = dict(self.problem)
        p["window"] = dict(self.window)
        return p

    # ---- maps --------------------------------------------------------------------------
    def global_ids(self) -> np.ndarray:
        """Global DoF id of every local DoF (velocity block then pressure block)."""
        vel = np.arange(self.nvel_loc, dtype=np.int64) + self.vel_off
        pre = self.nvel_glob + self.vert_off + np.arange(self.nvert_loc, dtype=np.int64)
        return np.concatenate([vel, pre])

    def layer_of_global(self, gid: np.ndarray) -> Tuple[np.ndarray, np.ndarray]:
        """(is_velocity, last-axis layer: node layer for velocity, vertex layer for pressure)."""
        gid = np.asarray(gid, dtype=np.int64)
        is_vel = gid < self.nvel_glob
        layer = np.empty_like(gid)
        layer[is_vel] = gid[is_vel] // (self.dim * self.nlow_free) + 1
        layer[~is_vel] = (gid[~is_vel] - self.nvel_glob) // self.nlow_vert
        return is_vel, layer

    def owner_of_global(self, gid: np.ndarray) -> np.ndarray:
        is_vel, layer = self.layer_of_global(gid)
        vlayer = np.where(is_vel, (layer + 1) // 2, layer)
        starts = np.array([a for a, _ in self.layers])
        return np.searchsorted(starts, vlayer, side="right") - 1

    def owned_mask(self) -> np.ndarray:
        return self.owner_of_global(self.global_ids()) == self.rank


def exchange_info(slab: Slab, written_local: np.ndarray) -> Dict:
    """What this rank will send (ghost-written DoFs) and needs (ghost DoFs), by global id.
    written_local: local indices this rank's patches write (weight > 0)."""
    gids = slab.global_ids()
    owner = slab.owner_of_global(gids)
    ghosts = np.nonzero(owner != slab.rank)[0]
    gw = np.intersect1d(np.asarray(written_local), ghosts)      # ghost-written local indices
    return {"rank": slab.rank,
            "gw_gid": gids[gw], "gw_owner": owner[gw],            # corrections I send
            "ghost_gid": gids[ghosts], "ghost_owner": owner[ghosts]}  # halo values I need


def _exchange_lists(slab: Slab, written_local: np.ndarray, allinfo: Sequence[Dict]) -> Dict:
    """Index lists of the two exchanges, agreed with the other ranks' exchange_info."""
    gids = slab.global_ids()
    owner = slab.owner_of_global(gids)
    ghosts = np.nonzero(owner != slab.rank)[0]
    gw = np.intersect1d(np.asarray(written_local), ghosts)
    g2l = {int(g): i for i, g in enumerate(gids)}
    lists = {"corr_send": {}, "corr_recv": {}, "halo_send": {}, "halo_recv": {}}
    for other in allinfo:
        q = other["rank"]
        if q == slab.rank:
            continue
        # corrections I send to q / receive from q (global-id order on both sides)
        sel = gw[owner[gw] == q]
        if len(sel):
            lists["corr_send"][q] = sel[np.argsort(gids[sel], kind="stable")]
        mine = np.sort(other["gw_gid"][other["gw_owner"] == slab.rank])
        if len(mine):
            lists["corr_recv"][q] = np.array([g2l[int(g)] for g in mine], dtype=np.int64)
        # halo: q needs my owned values at its ghosts owned by me; I need q's at my ghosts owned by q
        need = np.sort(other["ghost_gid"][other["ghost_owner"] == slab.rank])
        if len(need):
            lists["halo_send"][q] = np.array([g2l[int(g)] for g in need], dtype=np.int64)
        sel = ghosts[owner[ghosts] == q]
        if len(sel):
            lists["halo_recv"][q] = sel[np.argsort(gids[sel], kind="stable")]
    lists["ghost_written"] = gw
    return lists


class DistSweeper:
    """Per-sweep protocol of the slab-partitioned RAV smoother.

    backend (device-agnostic) must provide:
      residual(x, b, r), apply(r, x, omega)               -- local compute
      gather(src, idx, out), scatter(src, idx, dst),
      scatter_add(src, idx, dst), fill(dst, idx, value)   -- pack / unpack
      index(np_array) -> backend index array, buffer(n) -> backend float64 buffer
    comm: all_gather_object(obj), exchange(sends: {peer: buf}, recvs: {peer: buf})
      (point-to-point, every rank posts matching sends and receives)."""

    def __init__(self, slab: Slab, backend, comm, written_local: np.ndarray, all_infos=None):
        self.slab, self.be, self.comm = slab, backend, comm
        if all_infos is None:
            all_infos = comm.all_gather_object(exchange_info(slab, written_local))
        L = _exchange_lists(slab, np.asarray(written_local), all_infos)
        self.lists = L
        ix = backend.index
        self.gw = ix(L["ghost_written"])
        self.cs = {q: ix(v) for q, v in L["corr_send"].items()}
        self.cr = {q: ix(v) for q, v in L["corr_recv"].items()}
        self.hs = {q: ix(v) for q, v in L["halo_send"].items()}
        self.hr = {q: ix(v) for q, v in L["halo_recv"].items()}
        self.cs_buf = {q: backend.buffer(len(v)) for q, v in L["corr_send"].items()}
        self.cr_buf = {q: backend.buffer(len(v)) for q, v in L["corr_recv"].items()}
        self.hs_buf = {q: backend.buffer(len(v)) for q, v in L["halo_send"].items()}
        self.hr_buf = {q: backend.buffer(len(v)) for q, v in L["halo_recv"].items()}
        self.r = backend.buffer(slab.n_loc)

    # the sweep in three local phases separated by the two exchanges
    def phase_compute(self, x, b, omega: float):
        be = self.be
        be.residual(x, b, self.r)                      # r = b - L x on the patch rows
        be.fill(x, self.gw, 0.0)                       # ghost-written entries collect corrections
        be.apply(self.r, x, omega)                     # x += omega S_RAV r  (local patches)
        for q, idx in self.cs.items():
            be.gather(x, idx, self.cs_buf[q])

    def phase_corrections(self, x):
        be = self.be
        for q, idx in self.cr.items():
            be.scatter_add(self.cr_buf[q], idx, x)     # interface-correction sum at the owner
        for q, idx in self.hs.items():
            be.gather(x, idx, self.hs_buf[q])

    def phase_halo(self, x):
        for q, idx in self.hr.items():
            self.be.scatter(self.hr_buf[q], idx, x)    # refreshed ghost values

    def sweep(self, x, b, omega: float):
        self.phase_compute(x, b, omega)
        self.comm.exchange(self.cs_buf, self.cr_buf)
        self.phase_corrections(x)
        self.comm.exchange(self.hs_buf, self.hr_buf)
        self.phase_halo(x)

    def smooth(self, x, b, nu: int, omega: float):
        for _ in range(nu):
            self.sweep(x, b, omega)
        return x


class TorchComm:
    """torch.distributed plumbing (NCCL on GPUs, gloo on CPU)."""

    def __init__(self, group=None):
        import torch.distributed as dist
        self.dist = dist
        self.group = group

    def all_gather_object(self, obj):
        out = [None] * self.dist.get_world_size(self.group)
        self.dist.all_gather_object(out, obj, group=self.group)
        return out

    def exchange(self, sends: Dict, recvs: Dict):
        dist = self.dist
        ops = [dist.P2POp(dist.isend, buf, q, group=self.group) for q, buf in sorted(sends.items())]
        ops += [dist.P2POp(dist.irecv, buf, q, group=self.group) for q, buf in sorted(recvs.items())]
        if ops:
            for req in dist.batch_isend_irecv(ops):
                req.wait()


class GpuBackend:
    """Compute steps through the C-ABI (paper_2103_10127_b200.ravgmg)."""

    def __init__(self, smoother, stream=None):
        import torch
        from . import ravgmg as rg
        self.torch, self.rg, self.sm, self.stream = torch, rg, smoother, stream

    def residual(self, x, b, r):
        self.sm.residual(x, b, r)

    def apply(self, r, x, omega):
        self.sm.apply(r, x, omega)

    def gather(self, src, idx, out):
        self.rg.index_op(0, src, idx, out, stream=self.stream)

    def scatter(self, src, idx, dst):
        self.rg.index_op(1, src, idx, dst, stream=self.stream)

    def scatter_add(self, src, idx, dst):
        self.rg.index_op(2, src, idx, dst, stream=self.stream)

    def fill(self, dst, idx, value):
        self.rg.index_op(3, None, idx, dst, value=value, stream=self.stream)

    def index(self, a):
        return self.torch.tensor(np.asarray(a, dtype=np.int32), device="cuda")

    def buffer(self, n):
        return self.torch.zeros(int(n), dtype=self.torch.float64, device="cuda")


def written_local_from_patches(P: Dict) -> np.ndarray:
    """Local DoFs written by the patches (weight > 0)."""
    dofs = np.asarray(P["dofs"].cpu() if hasattr(P["dofs"], "cpu") else P["dofs"])
    w = np.asarray(P["w"].cpu() if hasattr(P["w"], "cpu") else P["w"])
    return np.unique(dofs[w > 0]).astype(np.int64)
