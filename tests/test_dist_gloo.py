"""CPU (gloo, world_size 2-3) tests of the z-slab partition and halo plan of the multi-GPU
path.  Each process builds its host-side plan through the C-ABI
(msp_dist_plan, no GPU), exchanges ghost values of a global vector with its peers over
torch.distributed (gloo) in exactly the plan's send / receive order, and checks
  (1) the received ghost values are those of the named ghost cells (plans of the two
      sides agree),
  (2) a rank-local BSR SpMV over owned rows with owned+ghost columns reproduces the
      global SpMV rows (the ghost set is complete),
  (3) cells are partitioned, and every ABMC block / level-1 aggregate is owned whole."""
import os
import socket
import sys

import numpy as np
import pytest
import torch.multiprocessing as mp

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, cfgname, shape, q):
    sys.path.insert(0, ROOT)
    import torch
    import torch.distributed as dist
    import scipy.sparse as sp
    import gen
    import oracle
    from paper_2208_08594_b200 import HostSetup
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        nx, ny, nz = shape
        p = gen.make_config(cfgname, nx=nx, ny=ny, nz=nz)
        b = p["b"]
        H = HostSetup(p["row_ptr"], p["col"], p["val"], p["nc"], coarsest_max_dof=40)
        owner = H.partition_owner(nx, ny, nz, world)
        plan = H.dist_plan(rank, world, owner)
        x = gen.random_vector(p["n"] * b, 42).reshape(-1, b)
        # (1) halo exchange in plan order
        reqs, bufs = [], {}
        for peer in range(world):
            if peer == rank:
                continue
            sc = plan["send_cells"][plan["send_ptr"][peer]:plan["send_ptr"][peer + 1]]
            nr = plan["recv_ptr"][peer + 1] - plan["recv_ptr"][peer]
            if len(sc):
                reqs.append(dist.isend(torch.from_numpy(np.ascontiguousarray(x[sc])), dst=peer))
            if nr:
                bufs[peer] = torch.zeros((nr, b), dtype=torch.float64)
                reqs.append(dist.irecv(bufs[peer], src=peer))
        for r in reqs:
            r.wait()
        ghost_vals = np.zeros((len(plan["ghosts"]), b))
        for peer, t in bufs.items():
            ghost_vals[plan["recv_ptr"][peer]:plan["recv_ptr"][peer + 1]] = t.numpy()
        ok1 = np.array_equal(ghost_vals, x[plan["ghosts"]])
        # (2) local SpMV over owned rows with owned + ghost columns
        own = plan["owned"]
        lcol = -np.ones(p["n"], dtype=np.int64)
        lcol[own] = np.arange(len(own))
        lcol[plan["ghosts"]] = len(own) + np.arange(len(plan["ghosts"]))
        xl = np.vstack([x[own], ghost_vals])
        yl = np.zeros((len(own), b))
        complete = True
        for li, c in enumerate(own):
            for e in range(p["row_ptr"][c], p["row_ptr"][c + 1]):
                d = p["col"][e]
                if lcol[d] < 0:
                    complete = False
                    continue
                yl[li] += p["val"][e] @ xl[lcol[d]]
        # the same sums over global columns (same order): must be bit-identical
        yg = np.zeros((len(own), b))
        for li, c in enumerate(own):
            for e in range(p["row_ptr"][c], p["row_ptr"][c + 1]):
                yg[li] += p["val"][e] @ x[p["col"][e]]
        yo = oracle.bsr_spmv(p["row_ptr"], p["col"], p["val"], x.reshape(-1)).reshape(-1, b)[own]
        absy = oracle.bsr_spmv(p["row_ptr"], p["col"], np.abs(p["val"]), np.abs(x).reshape(-1)).reshape(-1, b)[own]
        ok2 = complete and np.array_equal(yl, yg) and bool(np.all(np.abs(yl - yo) <= 1e-12 * absy))
        # (3) whole aggregates per rank
        O = oracle.Msp(p["row_ptr"], p["col"], p["val"], coarsest_max_dof=40)
        agg = O.level_agg(0)[1]
        mine = np.zeros(p["n"], bool)
        mine[own] = True
        ok3 = all(mine[agg == I].all() or (~mine[agg == I]).all() for I in np.unique(agg))
        counts = torch.tensor([len(own)], dtype=torch.int64)
        dist.all_reduce(counts)
        q.put((rank, bool(ok1), bool(ok2), bool(ok3), int(counts.item()) == p["n"], len(plan["ghosts"])))
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("world,cfg,shape", [(2, "C2", (14, 12, 9)), (3, "C3", (10, 24, 12))])
def test_gloo_halo_plan(world, cfg, shape):
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, cfg, shape, q)) for r in range(world)]
    for pr in procs:
        pr.start()
    res = [q.get(timeout=300) for _ in range(world)]
    for pr in procs:
        pr.join(timeout=60)
    assert all(pr.exitcode == 0 for pr in procs)
    for rank, ok1, ok2, ok3, ok4, ng in res:
        assert ok1, f"rank {rank}: ghost values differ from the plan"
        assert ok2, f"rank {rank}: local SpMV differs (incomplete ghost set)"
        assert ok3, f"rank {rank}: an aggregate is split across ranks"
        assert ok4 and ng > 0
