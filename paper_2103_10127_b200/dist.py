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

    def __init__(self, problem: Dict, nranks: int, rank: int, layers: Sequence[Tuple[int, int]] = None):
        self.problem = problem
        self.dim = dim = problem["dim"]
        self.nranks, self.rank = nranks, rank
        nc = [int(c) for c in problem["ncell"][:dim]]
        n = nc[-1]
        self.n_last = n
        self.layers = list(layers) if layers is not None else partition_layers(n + 1, nranks)
        assert len(self.layers) == nranks and self.layers[0][0] == 0 and self.layers[-1][1] == n + 1
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

    def owned_ranges(self) -> List[Tuple[int, int]]:
        """The owned local DoFs as two contiguous ranges [a, b): velocity, pressure."""
        w = self.window
        per = self.dim * self.nlow_free
        lo, hi = self.own_node
        vel = (per * (lo - w["node_lo"]), per * (hi - w["node_lo"] + 1))
        pre = (self.nvel_loc + self.nlow_vert * (self.V0 - w["vert_lo"]),
               self.nvel_loc + self.nlow_vert * (self.V1 - w["vert_lo"]))
        return [vel, pre]

    def transfer_window(self) -> Dict:
        """This rank's window with the row window narrowed to its OWNED layers: the
        fine-grid argument of a windowed rav_gen_prolongation (rows = owned DoFs)."""
        w = dict(self.window)
        w["rnode_lo"], w["rnode_hi"] = self.own_node
        w["rvert_lo"], w["rvert_hi"] = self.V0, self.V1 - 1
        return w


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

    # vector consistency outside the sweep (transfers of the distributed V-cycle)
    def halo(self, v):
        """Owner values -> every ghost copy (the halo refresh of the sweep)."""
        be = self.be
        for q, idx in self.hs.items():
            be.gather(v, idx, self.hs_buf[q])
        self.comm.exchange(self.hs_buf, self.hr_buf)
        self.phase_halo(v)

    def accumulate_ghosts(self, v):
        """Partial sums held at ghost copies -> added into the owner's entry (the
        halo exchange reversed); the ghost entries are left stale."""
        be = self.be
        for q, idx in self.hr.items():
            be.gather(v, idx, self.hr_buf[q])
        self.comm.exchange(self.hr_buf, self.hs_buf)
        for q, idx in self.hs.items():
            be.scatter_add(self.hs_buf[q], idx, v)


def local_colors(slab: Slab) -> Tuple[np.ndarray, np.ndarray]:
    """4^d colouring (R10) of this rank's patches by GLOBAL vertex coordinates,
    so every rank relaxes the same colour at the same time: the library's
    rav_gen_colors on the rank's window.  Returns (offs[4^d + 1], local patch ids)."""
    from . import ravgmg as rg
    return rg.multicolor(slab.local_problem())


class DistMVSweeper(DistSweeper):
    """Slab-partitioned multiplicative Vanka in colours (Eq. 11, R10).

    Per colour every rank relaxes its patches of that colour (fresh local
    residuals, Eq. 15, full prolongation).  Same-colour patches share no
    DoF and are not coupled through L (vertex spacing >= 4), also across ranks,
    so a DoF is changed by at most one patch per colour: the rank that changed
    a ghost DoF sends its change (new - old) to the owner, which adds it; then
    a halo refresh makes the next colour see current values.  The result equals
    the sequential single-domain MV sweep in colour-major order.

    backend additionally: apply_color(c, x, b, omega), gather_diff(src, idx, buf)
    (buf[k] = src[idx[k]] - buf[k])."""

    def __init__(self, slab: Slab, backend, comm, written_local: np.ndarray, n_colors: int, all_infos=None):
        super().__init__(slab, backend, comm, written_local, all_infos)
        self.n_colors = n_colors

    def sweep(self, x, b, omega: float):
        be = self.be
        for c in range(self.n_colors):
            for q, idx in self.cs.items():
                be.gather(x, idx, self.cs_buf[q])          # old values of ghost-written DoFs
            be.apply_color(c, x, b, omega)
            for q, idx in self.cs.items():
                be.gather_diff(x, idx, self.cs_buf[q])     # their changes in this colour
            self.comm.exchange(self.cs_buf, self.cr_buf)
            for q, idx in self.cr.items():
                be.scatter_add(self.cr_buf[q], idx, x)
            self.halo(x)


def nested_layers(fine_layers: Sequence[Tuple[int, int]]) -> List[Tuple[int, int]]:
    """Slab partition of the next coarser level (vertex layer 2c of the fine grid
    is vertex layer c of the coarse grid): interior cuts V -> ceil(V / 2).  With
    it every owned fine row interpolates from DoFs inside the rank's coarse
    window (checked by rav_gen_prolongation)."""
    cuts = [0] + [(b + 1) // 2 for _, b in fine_layers[:-1]] + [(fine_layers[-1][1] - 1) // 2 + 1]
    return [(cuts[r], cuts[r + 1]) for r in range(len(fine_layers))]


def plan_levels(problem: Dict, n_levels: int, nranks: int, min_layers: int = 3,
                agg_layers: int = 0) -> Tuple[List[Dict], List[List[Tuple[int, int]]]]:
    """Problems of the hierarchy (finest first) and the slab partitions of the
    levels that stay partitioned: level k (0 = finest) is partitioned while every
    slab has >= max(min_layers, agg_layers) vertex layers; the levels below are
    agglomerated (every rank holds them whole).  Returns (problems, partitions)
    with len(partitions) = number of partitioned levels (>= 1)."""
    probs = [problem]
    for _ in range(n_levels - 1):
        p = dict(probs[-1])
        p["ncell"] = [c // 2 if k < problem["dim"] else c for k, c in enumerate(p["ncell"])]
        probs.append(p)
    n_last = problem["ncell"][problem["dim"] - 1]
    parts = [partition_layers(n_last + 1, nranks, min_layers)]
    need = max(min_layers, agg_layers)
    while len(parts) < n_levels - 1:   # the coarsest level is never partitioned
        nxt = nested_layers(parts[-1])
        if min(b - a for a, b in nxt) < need:
            break
        parts.append(nxt)
    return probs, parts


class DistVCycle:
    """Slab-partitioned V-cycle (SURVEY section 8 rows a9 / e).

    levels[k], k = 0 (finest) .. K-1: per rank a DistSweeper over the rank's
    window of level k.  xfers[k] (k < K-1): the rank's windowed prolongation
    from level k+1 to level k (rows = owned DoFs of level k, columns = level
    k+1's window).  agg: the prolongation from the agglomerated level (global
    numbering, held whole by every rank) to level K-1 (rows = owned DoFs).
    coarse: the agglomerated hierarchy below (every rank runs it redundantly on
    the same all-reduced right-hand side).

    Per cycle on a partitioned level: pre-smoothing (sweeps with their
    interface sums and halo refresh), residual on the local rows,
    b_c = P_own^T r (partial sums of the rank's owned fine rows), partial sums
    at coarse ghosts -> owners (accumulate_ghosts) and a coarse halo refresh, the
    coarse cycle from x_c = 0, x += P_own x_c on owned rows, a fine halo
    refresh, post-smoothing.  At the agglomeration level the coarse right-hand
    side is all-reduced instead.  ||r||^2 over owned DoFs, all-reduced, for the
    stopping test (R11).

    backend (per level, see DistSweeper) additionally provides
      restrict(xfer, r, bc), prolong(xfer, xc, x), zero(v),
      dot_owned(r, ranges) -> partial ||r||^2 as a backend scalar buffer,
      coarse_vcycle(xc, bc, pre, post, omega), buffer(n)
    comm additionally: allreduce_sum(buf) (in place, identical on every rank)."""

    def __init__(self, levels: Sequence[Dict], xfers: Sequence, agg, comm, n_coarse: int):
        self.levels, self.xfers, self.agg, self.comm = list(levels), list(xfers), agg, comm
        for lv in self.levels:
            be = lv["be"]
            lv.setdefault("r", be.buffer(lv["slab"].n_loc))
        self.bc = self.levels[-1]["be"].buffer(n_coarse)
        self.xc = self.levels[-1]["be"].buffer(n_coarse)

    def _cycle(self, k: int, x, b, pre: int, post: int, omega: float):
        lv = self.levels[k]
        be, sw = lv["be"], lv["sweeper"]
        sw.smooth(x, b, pre, omega)
        be.residual(x, b, lv["r"])
        if k + 1 < len(self.levels):
            c = self.levels[k + 1]
            cbe = c["be"]
            be.restrict(self.xfers[k], lv["r"], c["b"])
            c["sweeper"].accumulate_ghosts(c["b"])
            c["sweeper"].halo(c["b"])
            cbe.zero(c["x"])
            self._cycle(k + 1, c["x"], c["b"], pre, post, omega)
            be.prolong(self.xfers[k], c["x"], x)
        else:
            be.restrict(self.agg, lv["r"], self.bc)
            self.comm.allreduce_sum(self.bc)
            be.zero(self.xc)
            be.coarse_vcycle(self.xc, self.bc, pre, post, omega)
            be.prolong(self.agg, self.xc, x)
        sw.halo(x)
        sw.smooth(x, b, post, omega)

    def vcycle(self, x, b, pre: int = 2, post: int = 2, omega: float = 0.66):
        self._cycle(0, x, b, pre, post, omega)
        return x

    def residual_norm(self, x, b) -> float:
        lv = self.levels[0]
        be = lv["be"]
        be.residual(x, b, lv["r"])
        s = be.dot_owned(lv["r"], lv["slab"].owned_ranges())
        self.comm.allreduce_sum(s)
        return float(s.cpu()[0]) ** 0.5 if hasattr(s, "cpu") else float(s[0]) ** 0.5

    def solve(self, x, b, pre: int = 2, post: int = 2, omega: float = 0.66, rtol: float = 1e-8,
              maxit: int = 200):
        """V-cycles until ||b - L x_k|| <= rtol ||b - L x_0|| (R11).  Returns (x, k, hist)."""
        hist = [self.residual_norm(x, b)]
        k = 0
        while hist[0] > 0 and k < maxit:
            self.vcycle(x, b, pre, post, omega)
            k += 1
            hist.append(self.residual_norm(x, b))
            if not np.isfinite(hist[-1]):
                raise FloatingPointError(f"distributed V-cycle diverged at cycle {k}")
            if hist[-1] <= rtol * hist[0]:
                break
        return x, k, np.array(hist)


class TorchComm:
    """torch.distributed plumbing (NCCL on GPUs, gloo on CPU).  Under gloo, device
    buffers of the point-to-point exchanges are staged through host memory (gloo
    has no CUDA send/recv); this is the debug path that lets several ranks share
    one GPU, never a timed configuration."""

    def __init__(self, group=None):
        import torch.distributed as dist
        self.dist = dist
        self.group = group
        self.stage = dist.get_backend(group) == "gloo"

    def all_gather_object(self, obj):
        out = [None] * self.dist.get_world_size(self.group)
        self.dist.all_gather_object(out, obj, group=self.group)
        return out

    def allreduce_sum(self, buf):
        self.dist.all_reduce(buf, op=self.dist.ReduceOp.SUM, group=self.group)

    def exchange(self, sends: Dict, recvs: Dict):
        dist = self.dist
        staged = {}
        if self.stage:
            sends = {q: (b.cpu() if b.is_cuda else b) for q, b in sends.items()}
            staged = {q: b for q, b in recvs.items() if b.is_cuda}
            recvs = {q: (b.cpu() if b.is_cuda else b) for q, b in recvs.items()}
        ops = [dist.P2POp(dist.isend, buf, q, group=self.group) for q, buf in sorted(sends.items())]
        ops += [dist.P2POp(dist.irecv, buf, q, group=self.group) for q, buf in sorted(recvs.items())]
        if ops:
            for req in dist.batch_isend_irecv(ops):
                req.wait()
        for q, dev in staged.items():
            dev.copy_(recvs[q])


class ThreadComm:
    """In-process transport for R ranks run as threads of one process (the GPU
    tests emulate ranks on the single available GPU this way; the CPU tests use
    it for quick checks).  Each rank holds its own ThreadComm(hub, rank); every
    collective is a host-side rendezvous (no kernel ever waits on another rank),
    received data are copied after the sender's work is complete."""

    class Hub:
        def __init__(self, nranks: int):
            import threading
            self.n = nranks
            self.barrier = threading.Barrier(nranks)
            self.box: Dict = {}

    def __init__(self, hub: "ThreadComm.Hub", rank: int, sync=None):
        self.hub, self.rank = hub, rank
        self.sync = sync or (lambda: None)   # e.g. torch.cuda.current_stream().synchronize

    def all_gather_object(self, obj):
        h = self.hub
        h.box[("obj", self.rank)] = obj
        h.barrier.wait()
        out = [h.box[("obj", r)] for r in range(h.n)]
        h.barrier.wait()
        return out

    def exchange(self, sends: Dict, recvs: Dict):
        h = self.hub
        self.sync()
        for q, buf in sends.items():
            h.box[("p2p", self.rank, q)] = buf
        h.barrier.wait()
        for q, buf in recvs.items():
            buf.copy_(h.box[("p2p", q, self.rank)])
        self.sync()
        h.barrier.wait()
        for q in sends:
            del h.box[("p2p", self.rank, q)]

    def allreduce_sum(self, buf):
        h = self.hub
        self.sync()
        h.box[("ar", self.rank)] = buf.clone()
        h.barrier.wait()
        acc = h.box[("ar", 0)].clone()
        for r in range(1, h.n):       # rank order: identical bits on every rank
            acc += h.box[("ar", r)]
        h.barrier.wait()
        buf.copy_(acc)
        self.sync()


def run_threads(nranks: int, fn):
    """fn(rank) on nranks threads; re-raises the first failure."""
    import threading
    out, err = [None] * nranks, []

    def body(r):
        try:
            out[r] = fn(r)
        except BaseException as e:  # noqa: BLE001
            err.append(e)
            raise

    ts = [threading.Thread(target=body, args=(r,)) for r in range(nranks)]
    for t in ts:
        t.start()
    for t in ts:
        t.join()
    if err:
        raise err[0]
    return out


class GpuBackend:
    """Compute steps through the C-ABI (paper_2103_10127_b200.ravgmg)."""

    def __init__(self, smoother, stream=None, coarse=None):
        import torch
        from . import ravgmg as rg
        self.torch, self.rg, self.sm, self.stream = torch, rg, smoother, stream
        self.coarse = coarse     # ravgmg.Multigrid of the agglomerated levels (last partitioned level)

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

    def apply_color(self, c, x, b, omega):
        self.sm.apply_color(c, x, b, omega)

    def gather_diff(self, src, idx, buf):
        self.rg.index_op(4, src, idx, buf, stream=self.stream)

    def restrict(self, xfer, r, bc):
        xfer.restrict(r, bc)

    def prolong(self, xfer, xc, x):
        xfer.prolong(xc, x)

    def zero(self, v):
        v.zero_()

    def dot_owned(self, r, ranges):
        out = self.torch.zeros(1, dtype=self.torch.float64, device="cuda")
        for k, (a, b) in enumerate(ranges):
            self.rg.dot(r[a:b], r[a:b], out, accumulate=k > 0, stream=self.stream)
        return out

    def coarse_vcycle(self, xc, bc, pre, post, omega):
        self.coarse.vcycle(xc, bc, pre, post, omega)

    def index(self, a):
        return self.torch.tensor(np.asarray(a, dtype=np.int32), device="cuda")

    def buffer(self, n):
        return self.torch.zeros(int(n), dtype=self.torch.float64, device="cuda")


def written_local_from_patches(P: Dict) -> np.ndarray:
    """Local DoFs written by the patches (weight > 0)."""
    dofs = np.asarray(P["dofs"].cpu() if hasattr(P["dofs"], "cpu") else P["dofs"])
    w = np.asarray(P["w"].cpu() if hasattr(P["w"], "cpu") else P["w"])
    return np.unique(dofs[w > 0]).astype(np.int64)


def build_gpu_cycle(problem: Dict, n_levels: int, nranks: int, rank: int, comm, weights: str = "pou",
                    agg_layers: int = 0, kernel: int = 0) -> Tuple["DistVCycle", List[Dict]]:
    """One rank's share of the slab-partitioned V-cycle on its GPU: every
    partitioned level generated directly in the rank's window (rav_gen_*, win =
    1), its smoother (rav_setup), windowed transfers (rav_gen_prolongation +
    rav_xfer_setup) and the agglomerated coarse hierarchy (mg_setup on the whole
    coarse grids, identical on every rank).  Returns (cycle, levels); levels[0]
    holds the rank's fine-level rhs "b" and a zero iterate "x"."""
    import torch
    from . import ravgmg as rg
    probs, parts = plan_levels(problem, n_levels, nranks, agg_layers=agg_layers)
    K = len(parts)
    coarse_mg, coarse_fine = rg.build_hierarchy(probs[K], n_levels - K, weights, kernel=kernel)
    slabs = [Slab(probs[k], nranks, rank, parts[k]) for k in range(K)]
    levels, xfers = [], []
    for k in range(K):
        L = rg.gen_level(slabs[k].local_problem(), weights)
        sm = rg.Smoother(L, L, kernel=kernel)
        be = GpuBackend(sm, coarse=coarse_mg if k == K - 1 else None)
        sw = DistSweeper(slabs[k], be, comm, written_local_from_patches(L))
        n = slabs[k].n_loc
        levels.append({"slab": slabs[k], "be": be, "sweeper": sw, "smoother": sm,
                       "b": L["b"] if k == 0 else torch.zeros(n, dtype=torch.float64, device="cuda"),
                       "x": torch.zeros(n, dtype=torch.float64, device="cuda")})
        del L
    for k in range(K - 1):
        fine = dict(probs[k], window=slabs[k].transfer_window())
        coarse = dict(probs[k + 1], window=dict(slabs[k + 1].window))
        xfers.append(rg.Transfer(rg.gen_prolongation(fine, coarse)))
    fine = dict(probs[K - 1], window=slabs[K - 1].transfer_window())
    agg = rg.Transfer(rg.gen_prolongation(fine, probs[K]))
    cyc = DistVCycle(levels, xfers, agg, comm, coarse_fine["n"])
    cyc.coarse_mg = coarse_mg
    torch.cuda.empty_cache()
    return cyc, levels


# ---------------------------------------------------------------------------------------------
# planning for the library-driven distributed cycle (mgd_* in csrc/dist.cu): this module only
# computes the partition, the windows and the index lists; every compute step and exchange of
# the sweep and the V-cycle runs inside the library, captured as CUDA graphs
# ---------------------------------------------------------------------------------------------

def layer_weights(problem: Dict, weights: str = "pou") -> np.ndarray:
    """Factor bytes of each vertex layer along the last axis, proportional to sum_i n~_i n_i over
    the layer's patches (SURVEY section 8 row e: "balance by sum n~_i n_i bytes, not whole
    layers"): n_i = d prod_k a_k + 1, n~_i = d prod_k t_k + 1 with a_k / t_k the free / restricted
    Q2 node counts of the patch along axis k (host arithmetic on the structured grid, R2 / R3)."""
    dim = problem["dim"]
    nc = [int(c) for c in problem["ncell"][:dim]]
    per_axis = []
    for n in nc:
        v = np.arange(n + 1)
        lo, hi = np.maximum(2 * v - 2, 1), np.minimum(2 * v + 2, 2 * n - 1)     # free nodes of the patch
        a = hi - lo + 1
        if weights == "own":
            t = ((2 * v >= 1) & (2 * v <= 2 * n - 1)).astype(int) + ((2 * v + 1) <= 2 * n - 1).astype(int)
        else:
            rlo, rhi = np.maximum(2 * v - 1, 1), np.minimum(2 * v + 1, 2 * n - 1)
            t = rhi - rlo + 1
        if weights == "full":
            t = a
        per_axis.append((a, t))
    # sum over the other axes of (d prod a + 1)(d prod t + 1), per layer of the last axis
    A = np.ones(1)
    T = np.ones(1)
    for a, t in per_axis[:-1]:
        A = np.outer(A, a).ravel()
        T = np.outer(T, t).ravel()
    a_l, t_l = per_axis[-1]
    n_i = dim * np.outer(A, a_l) + 1
    nt_i = dim * np.outer(T, t_l) + 1
    return (n_i * nt_i).sum(axis=0).astype(np.float64)


def partition_balanced(problem: Dict, nranks: int, min_layers: int = 3, weights: str = "pou") -> List[Tuple[int, int]]:
    """Contiguous vertex-layer slabs [V0, V1) of >= min_layers layers minimising the largest slab's
    factor bytes (layer_weights): bisection on the bottleneck with a greedy feasibility test, then
    the cuts of the smallest feasible bottleneck (whole layers, so the bound is one layer's weight)."""
    w = layer_weights(problem, weights)
    nv = len(w)
    if nv < nranks * min_layers:
        raise ValueError(f"{nv} vertex layers cannot give {nranks} slabs of >= {min_layers} layers")

    def cuts_for(cap):
        cuts, acc, cnt = [0], 0.0, 0
        for v in range(nv):
            left_layers = nv - v
            need = (nranks - len(cuts)) * min_layers       # layers the later slabs still need
            if cnt >= min_layers and (acc + w[v] > cap or left_layers <= need) and len(cuts) < nranks:
                cuts.append(v)
                acc, cnt = 0.0, 0
            acc += w[v]
            cnt += 1
            if acc > cap and cnt > min_layers:
                return None
        if len(cuts) != nranks or acc > cap or cnt < min_layers:
            return None
        return cuts + [nv]

    lo, hi = float(w.max()), float(w.sum())
    best = None
    for _ in range(100):
        mid = 0.5 * (lo + hi)
        c = cuts_for(mid)
        if c is not None:
            best, hi = c, mid
        else:
            lo = mid
        if hi - lo <= 1e-9 * hi:
            break
    if best is None:
        return partition_layers(nv, nranks, min_layers)
    return [(best[r], best[r + 1]) for r in range(nranks)]


def plan_levels_balanced(problem: Dict, n_levels: int, nranks: int, min_layers: int = 3, agg_layers: int = 0,
                         weights: str = "pou"):
    """plan_levels with the finest partition balanced by factor bytes (partition_balanced)."""
    probs, _ = plan_levels(problem, n_levels, 1, min_layers=1)
    parts = [partition_balanced(problem, nranks, min_layers, weights)]
    need = max(min_layers, agg_layers)
    while len(parts) < n_levels - 1:
        nxt = nested_layers(parts[-1])
        if min(b - a for a, b in nxt) < need:
            break
        parts.append(nxt)
    return probs, parts


def neighbor_plan(slab: "Slab", written: np.ndarray, all_infos: Sequence[Dict]) -> Dict:
    """One subdomain's exchange plan for mgd_setup: {peer: (corr_send, corr_recv, halo_send,
    halo_recv)} local index lists, its ghost-written DoFs and owned ranges (from the exchange_info
    of every subdomain)."""
    lists = _exchange_lists(slab, written, all_infos)
    peers = set(lists["corr_send"]) | set(lists["corr_recv"]) | set(lists["halo_send"]) | set(lists["halo_recv"])
    e = np.zeros(0, np.int64)
    nb = {q: (lists["corr_send"].get(q, e), lists["corr_recv"].get(q, e), lists["halo_send"].get(q, e),
              lists["halo_recv"].get(q, e)) for q in peers}
    return {"neighbors": nb, "ghost_written": lists["ghost_written"], "owned": slab.owned_ranges()}


def build_lib_dist(problem: Dict, n_levels: int, nsub: int, local_ids: Sequence[int], sub_proc: Sequence[int],
                   comm, gather=None, weights: str = "pou", variant: int = 0, agg_layers: int = 0,
                   smooth_only: bool = False, via_comm: int = 0, balanced: bool = True, stream=None,
                   deterministic: bool = False):
    """One process's share of the library-driven slab-partitioned hierarchy (mgd_setup).

    nsub subdomains in all; this process drives local_ids (global ids, ascending) on its current
    GPU; sub_proc[g] = process of subdomain g.  gather(obj) -> list over ALL processes of obj (the
    host all-gather of the exchange plans; None when every subdomain is local).  smooth_only: the
    finest level alone, no coarse hierarchy (mgd_smooth).  Returns (DistMultigrid, info) with
    info["b"] / info["x"]: per local subdomain the window's rhs and a zero iterate, and
    info["slabs"]: per level, per local subdomain, its Slab."""
    import torch
    from . import ravgmg as rg
    if smooth_only:
        probs = [problem]
        parts = [partition_balanced(problem, nsub) if balanced else partition_layers(problem["ncell"][problem["dim"] - 1] + 1, nsub)]
    elif balanced:
        probs, parts = plan_levels_balanced(problem, n_levels, nsub, agg_layers=agg_layers, weights=weights)
    else:
        probs, parts = plan_levels(problem, n_levels, nsub, agg_layers=agg_layers)
    K = len(parts)
    coarse = None
    if not smooth_only:
        coarse, _ = rg.build_hierarchy(probs[K], n_levels - K, weights, variant=variant, deterministic=deterministic)
    subs, slabs = [], []
    for k in range(K):
        lev_slabs = [Slab(probs[k], nsub, g, parts[k]) for g in local_ids]
        levels = [rg.gen_level(s.local_problem(), weights) for s in lev_slabs]
        written = [written_local_from_patches(L) for L in levels]
        infos = [exchange_info(s, w) for s, w in zip(lev_slabs, written)]
        if gather is not None:
            infos = [i for part in gather(infos) for i in part]
        row = []
        for s, L, w in zip(lev_slabs, levels, written):
            d = neighbor_plan(s, w, infos)
            d.update({"level": L, "prol": None, "colors": local_colors(s) if variant == 2 else None})
            row.append(d)
        subs.append(row)
        slabs.append(lev_slabs)
    if not smooth_only:
        for k in range(K):
            for i, g in enumerate(local_ids):
                fine = dict(probs[k], window=slabs[k][i].transfer_window())
                crs = dict(probs[k + 1], window=dict(slabs[k + 1][i].window)) if k + 1 < K else probs[K]
                subs[k][i]["prol"] = rg.gen_prolongation(fine, crs)
                subs[k][i]["prol_grids"] = (fine, crs)   # -> the stencil form (mgd_setup verifies it)
    mgd = rg.DistMultigrid(comm, sub_proc, local_ids, subs, coarse=coarse, variant=variant, stream=stream,
                           via_comm=via_comm, deterministic=deterministic)
    mgd._keep = (subs, coarse)
    info = {"b": [d["level"]["b"] for d in subs[0]],
            "x": [torch.zeros(d["level"]["n"], dtype=torch.float64, device="cuda") for d in subs[0]],
            "slabs": slabs, "parts": parts, "K": K}
    return mgd, info
