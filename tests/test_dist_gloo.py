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


def _exchange(dist, torch, rank, world, send, recv_counts, vec):
    """Send vec[send[q]] to every peer q, receive recv_counts[q] values from q (gloo).
    The send counts are agreed first (all ranks take the same decision), so inconsistent
    plans fail the test instead of hanging it: returns None then."""
    mine = torch.tensor([len(send[t]) if t != rank else 0 for t in range(world)], dtype=torch.int64)
    allc = [torch.zeros(world, dtype=torch.int64) for _ in range(world)]
    dist.all_gather(allc, mine)
    ok = torch.tensor([int(all(int(allc[t][rank]) == recv_counts[t] for t in range(world) if t != rank))])
    dist.all_reduce(ok, op=dist.ReduceOp.MIN)
    if not int(ok.item()):
        return None
    reqs, bufs = [], {}
    for q in range(world):
        if q == rank:
            continue
        if len(send[q]):
            reqs.append(dist.isend(torch.from_numpy(np.ascontiguousarray(vec[send[q]])), dst=q))
        if recv_counts[q]:
            bufs[q] = torch.zeros(recv_counts[q], dtype=torch.float64)
            reqs.append(dist.irecv(bufs[q], src=q))
    for r in reqs:
        r.wait()
    return {q: t.numpy() for q, t in bufs.items()}


def _level_worker(rank, world, port, cfgname, shape, q):
    """Partitioned AMG levels (dist_levels): the host plan of every level >= 1 checked by
    exchanging seeded level vectors over gloo in the plan's order."""
    sys.path.insert(0, ROOT)
    import torch
    import torch.distributed as dist
    import gen
    from paper_2208_08594_b200 import HostSetup
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        nx, ny, nz = shape
        p = gen.make_config(cfgname, nx=nx, ny=ny, nz=nz)
        H = HostSetup(p["row_ptr"], p["col"], p["val"], p["nc"], coarsest_max_dof=20)
        L = H.info()["levels"]
        owner = H.partition_owner(nx, ny, nz, world)
        # effective cell owners (whole ABMC blocks), from every rank's host cell plan
        own = np.full(p["n"], -1)
        for r in range(world):
            own[H.dist_plan(r, world, owner)["owned"]] = r
        results = []
        for l in range(1, L):
            P = H.dist_level_plan(rank, world, l, owner)
            ptr, col, val = H.level_csr(l)
            nl = len(ptr) - 1
            # (0) owners: the owner of the lowest-index member, level by level (independent)
            o_prev = own
            for k in range(l):
                a = H.level_agg(k)
                lo = np.full(a.max() + 1, np.iinfo(np.int64).max)
                np.minimum.at(lo, a, np.arange(len(a)))
                o_prev = o_prev[lo]
            ok0 = np.array_equal(P["owner"], o_prev) and np.array_equal(np.sort(P["rows"]), np.flatnonzero(o_prev == rank))
            ri = P["row_index"]
            ok0 = ok0 and np.array_equal(P["rows"], P["rows"][np.argsort(ri[P["rows"]], kind="stable")])
            # (1) matrix ghosts: values arrive in the receiver's order
            v = gen.random_vector(nl, 100 + l)
            rc = [int(np.sum(P["owner"][P["gx"]] == t)) for t in range(world)]
            got = _exchange(dist, torch, rank, world, P["sendx"], rc, v)
            if got is None:
                results.append((l, bool(ok0), False, False, False, False, False))
                continue
            gx_vals = np.concatenate([got[t] for t in range(world) if t != rank and rc[t]] or [np.zeros(0)])
            ok1 = np.array_equal(gx_vals, v[P["gx"]])
            # (2) complete ghost set: owned rows of the local matrix = global rows (same order)
            loc = -np.ones(nl, np.int64)
            loc[P["rows"]] = np.arange(len(P["rows"]))
            loc[P["gx"]] = len(P["rows"]) + np.arange(len(P["gx"]))
            vl = np.concatenate([v[P["rows"]], gx_vals])
            ok2 = True
            for i in P["rows"]:
                cols = col[ptr[i]:ptr[i + 1]]
                if (loc[cols] < 0).any():
                    ok2 = False
                    break
                a_loc = 0.0
                a_glob = 0.0
                for e in range(ptr[i], ptr[i + 1]):
                    a_loc += val[e] * vl[loc[col[e]]]
                    a_glob += val[e] * v[col[e]]
                ok2 = ok2 and a_loc == a_glob
            # (3) member ghosts: every owned next-level aggregate summed in global row order
            r_l = gen.random_vector(nl, 200 + l)
            rcm = [int(np.sum(P["owner"][P["gm"]] == t)) for t in range(world)]
            got = _exchange(dist, torch, rank, world, P["sendm"], rcm, r_l)
            gm_vals = (np.concatenate([got[t] for t in range(world) if t != rank and rcm[t]] or [np.zeros(0)])
                       if got is not None else np.zeros(len(P["gm"])) + np.nan)
            ok3 = got is not None and np.array_equal(gm_vals, r_l[P["gm"]])
            a = H.level_agg(l)
            lo = np.full(a.max() + 1, np.iinfo(np.int64).max)
            np.minimum.at(lo, a, np.arange(nl))
            own_next = P["owner"][lo]
            rl = dict(zip(P["rows"].tolist(), r_l[P["rows"]]))
            rl.update(zip(P["gm"].tolist(), gm_vals))
            order = np.argsort(ri, kind="stable")
            for J in np.flatnonzero(own_next == rank):
                mem = [i for i in order if a[i] == J]
                ok3 = ok3 and all(i in rl for i in mem)
                if not ok3:
                    break
                s_loc = 0.0
                s_glob = 0.0
                for i in mem:
                    s_loc += rl[i]
                    s_glob += r_l[i]
                ok3 = ok3 and s_loc == s_glob
            # (4) parent ghosts: every owned level-(l-1) row finds its level-l row
            rcp = [int(np.sum(P["owner"][P["gp"]] == t)) for t in range(world)]
            got = _exchange(dist, torch, rank, world, P["sendp"], rcp, v)
            gp_vals = (np.concatenate([got[t] for t in range(world) if t != rank and rcp[t]] or [np.zeros(0)])
                       if got is not None else np.zeros(len(P["gp"])) + np.nan)
            ok4 = got is not None and np.array_equal(gp_vals, v[P["gp"]])
            ap = H.level_agg(l - 1)
            o_up = own if l == 1 else None
            if o_up is None:
                o_up = own
                for k in range(l - 1):
                    ak = H.level_agg(k)
                    lk = np.full(ak.max() + 1, np.iinfo(np.int64).max)
                    np.minimum.at(lk, ak, np.arange(len(ak)))
                    o_up = o_up[lk]
            avail = set(P["rows"].tolist()) | set(P["gp"].tolist())
            ok4 = ok4 and all(ap[i] in avail for i in np.flatnonzero(o_up == rank))
            cnt = torch.tensor([len(P["rows"])], dtype=torch.int64)
            dist.all_reduce(cnt)
            results.append((l, bool(ok0), bool(ok1), bool(ok2), bool(ok3), bool(ok4), int(cnt.item()) == nl))
        q.put((rank, results))
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("world,cfg,shape", [(2, "C2", (24, 20, 9)), (3, "C3", (10, 24, 12))])
def test_gloo_partitioned_level_plans(world, cfg, shape):
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_level_worker, args=(r, world, port, cfg, shape, q)) for r in range(world)]
    for pr in procs:
        pr.start()
    res = [q.get(timeout=600) for _ in range(world)]
    for pr in procs:
        pr.join(timeout=60)
    assert all(pr.exitcode == 0 for pr in procs)
    for rank, results in res:
        assert len(results) >= 2
        for l, ok0, ok1, ok2, ok3, ok4, ok5 in results:
            assert ok0, f"rank {rank} level {l}: owners / row order"
            assert ok1, f"rank {rank} level {l}: matrix ghost values"
            assert ok2, f"rank {rank} level {l}: local rows differ (incomplete ghost set)"
            assert ok3, f"rank {rank} level {l}: member ghosts / restriction sums"
            assert ok4, f"rank {rank} level {l}: parent ghosts / prolongation sources"
            assert ok5, f"level {l}: rows not partitioned"
