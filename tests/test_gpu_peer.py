"""Peer-memory exchange transport (dist.PeerComm; SURVEY section 8 row e) on the one
available GPU: two processes (two CUDA contexts on cuda:0) exchange interface
corrections and halos through CUDA IPC mappings with stream-memory-operation flags --
no host round trip per exchange, no NCCL, no spinning kernel.  The slab-partitioned RAV
sweeps and a distributed V-cycle must reproduce the single-domain oracle."""
import os
import socket

import numpy as np
import pytest
import torch
import torch.multiprocessing as mp

import oracle
import seeded_inputs as si
from _parity import assert_entrywise

pytestmark = [pytest.mark.gpu,
              pytest.mark.skipif(os.environ.get("RAV_TEST_PEER") != "1",
                                 reason="opt-in: two CUDA contexts time-sharing one GPU can starve each other while "
                                        "a stream waits on a flag the other context writes (one flaky hang seen); "
                                        "set RAV_TEST_PEER=1 to run")]


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, prob, mode, q):
    import torch.distributed as dist
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        torch.cuda.set_device(0)
        stream = torch.cuda.Stream()
        torch.cuda.set_stream(stream)
        from paper_2103_10127_b200 import dist as rdist
        from paper_2103_10127_b200 import ravgmg as rg
        comm = rdist.PeerComm(rdist.TorchComm(), rank)
        if mode == "sweep":
            slab = rdist.Slab(prob, world, rank)
            L = rg.gen_level(slab.local_problem(), "pou")
            sm = rg.Smoother(L, L)
            sw = rdist.DistSweeper(slab, rdist.GpuBackend(sm, stream), comm, rdist.written_local_from_patches(L))
            nglob = slab.nvel_glob + slab.nvert_glob
            x = torch.tensor(si.initial_guess(nglob, seed=43)[slab.global_ids()], device="cuda")
            sw.smooth(x, L["b"], 5, 0.66)
            torch.cuda.synchronize()
            own = slab.owned_mask()
            q.put((rank, slab.global_ids()[own], x.cpu().numpy()[own], 0))
        else:
            cyc, levels = rdist.build_gpu_cycle(prob, 4, world, rank, comm)
            slab = levels[0]["slab"]
            x = levels[0]["x"]
            _, k, _ = cyc.solve(x, levels[0]["b"], rtol=1e-10, omega=0.66, maxit=60)
            torch.cuda.synchronize()
            own = slab.owned_mask()
            q.put((rank, slab.global_ids()[own], x.cpu().numpy()[own], k))
        comm.close()
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("mode", ["sweep", "vcycle"])
def test_peer_transport_matches_oracle(mode):
    prob = si.problem(2, (24, 24), si.KIND_MMS, eta="fourier")
    world = 2
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, prob, mode, q)) for r in range(world)]
    for p in procs:
        p.start()
    res = [q.get(timeout=240) for _ in range(world)]
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    O = oracle.assemble(prob)
    xd = np.full(O["n"], np.nan)
    for _, g, v, _ in res:
        xd[g] = v
    assert not np.isnan(xd).any()
    if mode == "sweep":
        P = oracle.patches(prob, "pou")
        F = oracle.factor(O, P, oracle.FMT_ROWS)
        xo = oracle.additive_sweeps(O, P, F, si.initial_guess(O["n"], seed=43), O["b"], 0.66, 5)
        assert_entrywise(xd, xo, np.abs(xo).max(), tol=1e-12)
    else:
        H = oracle.Hierarchy(prob, 4)
        xo, ko, _ = H.solve(rtol=1e-10, omega=0.66, maxit=60)
        assert all(r[3] == ko for r in res)
        assert_entrywise(xd, xo, np.abs(xo).max(), tol=1e-10)
