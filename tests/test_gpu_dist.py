"""Distributed (z-slab) MSP-GMRES, exercised on ONE GPU through the loopback
harness (virtual ranks = host threads with their own streams; halos and collectives are
device copies ordered by CUDA events).  The partitioned solve performs the single-GPU
operations (same coloring, aggregates, ordering and factors), so iterations must match
the single-GPU solve within 1 (dot-product summation order) and the solution must agree."""
import numpy as np
import pytest
import scipy.sparse as sp

import gen
import oracle

pytestmark = pytest.mark.gpu
torch = pytest.importorskip("torch")


def run(p, nranks, owner=None, **kw):
    from paper_2208_08594_b200 import MspSolver, loopback_solve, HostSetup
    s = MspSolver(p["row_ptr"], p["col"], p["val"], nc=p["nc"], **kw)
    r1 = s.solve(torch.from_numpy(p["rhs"]).cuda())
    if owner == "zslab":
        owner = HostSetup(p["row_ptr"], p["col"], p["val"], p["nc"], **kw).partition_owner(
            p["nx"], p["ny"], p["nz"], nranks)
    rd = loopback_solve(p["row_ptr"], p["col"], p["val"], p["nc"], nranks, p["rhs"], owner=owner, **kw)
    A = sp.bsr_matrix((p["val"], p["col"], p["row_ptr"]), shape=(p["n"] * p["b"],) * 2)
    true = np.linalg.norm(p["rhs"] - A @ rd["x"]) / np.linalg.norm(p["rhs"])
    assert abs(rd["iters"] - r1["iters"]) <= 1, (rd["iters"], r1["iters"])
    assert true <= 1e-6
    x1 = r1["x"].cpu().numpy()
    assert np.linalg.norm(rd["x"] - x1) <= 1e-6 * np.linalg.norm(x1)
    info = rd["rank_info"]
    assert info[:, 0].sum() == p["n"]                    # cells partitioned
    if nranks > 1:
        assert (info[:, 1] > 0).all()                    # every rank has ghosts
    return rd, r1


@pytest.mark.parametrize("nranks", [1, 2, 3])
def test_loopback_zslab_matches_single_gpu(nranks):
    p = gen.make_config("C2", nx=24, ny=20, nz=9)
    run(p, nranks, owner="zslab", coarsest_max_dof=100)


def test_loopback_index_ranges_and_oracle():
    p = gen.make_config("C3", nx=12, ny=30, nz=17)
    rd, r1 = run(p, 4, owner=None, coarsest_max_dof=200)
    o = oracle.Msp(p["row_ptr"], p["col"], p["val"], coarsest_max_dof=200).solve(p["rhs"])
    assert abs(rd["iters"] - o["iters"]) <= 1


def test_loopback_nc6_and_restarts():
    p = gen.make_config("C2", nx=16, ny=14, nz=8, nc=6)
    from paper_2208_08594_b200 import loopback_solve, MspSolver
    rd = loopback_solve(p["row_ptr"], p["col"], p["val"], p["nc"], 2, p["rhs"], restart=6, coarsest_max_dof=60)
    s = MspSolver(p["row_ptr"], p["col"], p["val"], nc=p["nc"], coarsest_max_dof=60)
    r1 = s.solve(torch.from_numpy(p["rhs"]).cuda(), restart=6)
    assert r1["iters"] > 6 and abs(rd["iters"] - r1["iters"]) <= 1


@pytest.mark.parametrize("nograph", ["0", "1"])
def test_nccl_backend_single_rank_matches_single_gpu(nograph, monkeypatch):
    """The NCCL communicator path (ncclCommInitRank, ncclAllReduce, ncclAllGather, empty
    halos) at world size 1 reproduces the single-GPU solve, with the Arnoldi steps
    captured as CUDA graphs (NCCL calls inside) and launched directly."""
    from paper_2208_08594_b200 import DistSolver, MspSolver, nccl_unique_id
    monkeypatch.setenv("MSP_DIST_NOGRAPH", nograph)
    p = gen.make_config("C2", nx=20, ny=16, nz=6)
    uid = nccl_unique_id()
    d = DistSolver(p["row_ptr"], p["col"], p["val"], p["nc"], 0, 1, uid, coarsest_max_dof=80)
    own = d.owned_cells()
    assert np.array_equal(own, np.arange(p["n"]))
    rd = d.solve(torch.from_numpy(p["rhs"]).cuda())
    assert (d.stats()["kernels_per_iter"] > 0) == (nograph == "0")      # graph captured or not
    s = MspSolver(p["row_ptr"], p["col"], p["val"], nc=p["nc"], coarsest_max_dof=80)
    r1 = s.solve(torch.from_numpy(p["rhs"]).cuda())
    assert abs(rd["iters"] - r1["iters"]) <= 1
    x1 = r1["x"].cpu().numpy()
    assert np.linalg.norm(rd["x"].cpu().numpy() - x1) <= 1e-8 * np.linalg.norm(x1)


@pytest.mark.parametrize("nograph", ["0", "1"])
def test_nccl_single_rank_partitioned_levels(nograph, monkeypatch):
    """The NCCL path (graph-captured and direct) with every AMG level partitioned
    (dist_levels clamped; one rank: no ghosts, the hand-over goes straight to the
    coarsest) is bit-identical to the same handle with replicated levels."""
    from paper_2208_08594_b200 import DistSolver, nccl_unique_id
    monkeypatch.setenv("MSP_DIST_NOGRAPH", nograph)
    p = gen.make_config("C2", nx=20, ny=16, nz=6)
    out = []
    for D in (0, 99):
        d = DistSolver(p["row_ptr"], p["col"], p["val"], p["nc"], 0, 1, nccl_unique_id(), coarsest_max_dof=40,
                       dist_levels=D)
        out.append(d.solve(torch.from_numpy(p["rhs"]).cuda()))
        d.close()
    assert out[0]["iters"] == out[1]["iters"]
    assert torch.equal(out[0]["x"], out[1]["x"])


@pytest.mark.parametrize("nranks", [2, 3])
def test_loopback_coarse_root_bit_identical(nranks):
    """coarse_mode=1 (ROOT, north_star's "coarse levels agglomerated onto one GPU"): rank 0
    runs levels >= 1 and the coarsest and broadcasts the level-1 correction; the iterates
    are bit-identical to the replicated mode (same arithmetic on the same data)."""
    from paper_2208_08594_b200 import loopback_solve, HostSetup
    p = gen.make_config("C2", nx=24, ny=20, nz=9)
    owner = HostSetup(p["row_ptr"], p["col"], p["val"], p["nc"], coarsest_max_dof=100).partition_owner(
        p["nx"], p["ny"], p["nz"], nranks)
    r0 = loopback_solve(p["row_ptr"], p["col"], p["val"], p["nc"], nranks, p["rhs"], owner=owner,
                        coarsest_max_dof=100)
    r1 = loopback_solve(p["row_ptr"], p["col"], p["val"], p["nc"], nranks, p["rhs"], owner=owner,
                        coarsest_max_dof=100, coarse_mode=1)
    assert r0["iters"] == r1["iters"]
    assert np.array_equal(r0["x"], r1["x"])


@pytest.mark.parametrize("nranks", [2, 4])
def test_loopback_full_size_c3_zslabs_vs_oracle_golden(nranks):
    """C3 at full size partitioned into z-slabs (§8(e): 85 layers over 2 / 4 ranks), on one
    GPU through the loopback harness, against the ORACLE's committed solve
    (tests/golden/oracle_c3.json): iterations within 1 and the converged true residual."""
    import json
    import os
    from paper_2208_08594_b200 import loopback_solve, HostSetup
    p = gen.make_config("C3")
    owner = HostSetup(p["row_ptr"], p["col"], p["val"], p["nc"]).partition_owner(p["nx"], p["ny"], p["nz"], nranks)
    rd = loopback_solve(p["row_ptr"], p["col"], p["val"], p["nc"], nranks, p["rhs"], owner=owner,
                        coarse_mode=1 if nranks == 4 else 0)
    ref = json.load(open(os.path.join(os.path.dirname(__file__), "golden", "oracle_c3.json")))
    assert abs(rd["iters"] - ref["iters"]) <= 1, (rd["iters"], ref["iters"])
    A = sp.bsr_matrix((p["val"], p["col"], p["row_ptr"]), shape=(p["n"] * p["b"],) * 2)
    assert np.linalg.norm(p["rhs"] - A @ rd["x"]) / np.linalg.norm(p["rhs"]) <= 1e-6
    info = rd["rank_info"]
    assert info[:, 0].sum() == p["n"] and (info[:, 1] > 0).all()


@pytest.mark.parametrize("nranks,owner", [(2, "zslab"), (3, "zslab"), (3, None)])
@pytest.mark.parametrize("coarse_mode", [0, 1])
def test_loopback_distributed_levels_bit_identical(nranks, owner, coarse_mode):
    """dist_levels (NEXT-3): AMG levels 1..D partitioned (rows on the owner of their
    lowest-index member, per-color halos in the sweeps, member / parent halos around the
    transfers) instead of replicated.  Same per-row arithmetic and summation orders ->
    iterates bit-identical to dist_levels=0 for every D (0 < D < levels, and clamped)."""
    from paper_2208_08594_b200 import loopback_solve, HostSetup
    p = gen.make_config("C2", nx=24, ny=20, nz=9)
    kw = dict(coarsest_max_dof=20)
    H = HostSetup(p["row_ptr"], p["col"], p["val"], p["nc"], **kw)
    assert H.info()["levels"] >= 4
    own = H.partition_owner(p["nx"], p["ny"], p["nz"], nranks) if owner == "zslab" else None
    ref = loopback_solve(p["row_ptr"], p["col"], p["val"], p["nc"], nranks, p["rhs"], owner=own,
                         coarse_mode=coarse_mode, **kw)
    for D in (1, 2, 99):
        rd = loopback_solve(p["row_ptr"], p["col"], p["val"], p["nc"], nranks, p["rhs"], owner=own,
                            coarse_mode=coarse_mode, dist_levels=D, **kw)
        assert rd["iters"] == ref["iters"], (D, rd["iters"], ref["iters"])
        assert np.array_equal(rd["x"], ref["x"]), D


def test_loopback_distributed_levels_full_size_c3_vs_oracle_golden():
    """C3 at full size over 2 z-slab ranks with EVERY smoothed level partitioned
    (dist_levels clamped): the oracle's committed iteration count (+-1) and residual."""
    import json
    import os
    from paper_2208_08594_b200 import loopback_solve, HostSetup
    p = gen.make_config("C3")
    owner = HostSetup(p["row_ptr"], p["col"], p["val"], p["nc"]).partition_owner(p["nx"], p["ny"], p["nz"], 2)
    rd = loopback_solve(p["row_ptr"], p["col"], p["val"], p["nc"], 2, p["rhs"], owner=owner, dist_levels=99)
    ref = json.load(open(os.path.join(os.path.dirname(__file__), "golden", "oracle_c3.json")))
    assert abs(rd["iters"] - ref["iters"]) <= 1, (rd["iters"], ref["iters"])
    A = sp.bsr_matrix((p["val"], p["col"], p["row_ptr"]), shape=(p["n"] * p["b"],) * 2)
    assert np.linalg.norm(p["rhs"] - A @ rd["x"]) / np.linalg.norm(p["rhs"]) <= 1e-6


def test_nccl_single_rank_coarse_root():
    from paper_2208_08594_b200 import DistSolver, MspSolver, nccl_unique_id
    p = gen.make_config("C2", nx=20, ny=16, nz=6)
    d = DistSolver(p["row_ptr"], p["col"], p["val"], p["nc"], 0, 1, nccl_unique_id(), coarsest_max_dof=80,
                   coarse_mode=1)
    rd = d.solve(torch.from_numpy(p["rhs"]).cuda())
    s = MspSolver(p["row_ptr"], p["col"], p["val"], nc=p["nc"], coarsest_max_dof=80)
    r1 = s.solve(torch.from_numpy(p["rhs"]).cuda())
    assert abs(rd["iters"] - r1["iters"]) <= 1


@pytest.mark.parametrize("nranks", [2, 3])
def test_loopback_rank_local_bilu_vs_oracle(nranks):
    """bilu_local=1 (NEXT-3): BILU(0) of A with the couplings between ranks removed (block
    Jacobi across the z-slabs), no halo exchange in the substitutions.  Against the oracle's
    MSP whose BILU is refactorized from the same masked values in the same order
    (orc_msp_bilu_refactor): iterations within 1."""
    from paper_2208_08594_b200 import loopback_solve, HostSetup
    p = gen.make_config("C2", nx=24, ny=20, nz=9)
    H = HostSetup(p["row_ptr"], p["col"], p["val"], p["nc"], coarsest_max_dof=100)
    owner_in = H.partition_owner(p["nx"], p["ny"], p["nz"], nranks)
    owner = np.empty(p["n"], np.int32)
    for r in range(nranks):
        owner[H.dist_plan(r, nranks, owner_in)["owned"]] = r
    val = p["val"].copy()
    for c in range(p["n"]):
        for e in range(p["row_ptr"][c], p["row_ptr"][c + 1]):
            if owner[p["col"][e]] != owner[c]:
                val[e] = 0.0
    O = oracle.Msp(p["row_ptr"], p["col"], p["val"], coarsest_max_dof=100)
    O.bilu_refactor(val)
    o = O.solve(p["rhs"])
    rd = loopback_solve(p["row_ptr"], p["col"], p["val"], p["nc"], nranks, p["rhs"], owner=owner_in,
                        coarsest_max_dof=100, bilu_local=1)
    assert abs(rd["iters"] - o["iters"]) <= 1, (rd["iters"], o["iters"])
    A = sp.bsr_matrix((p["val"], p["col"], p["row_ptr"]), shape=(p["n"] * p["b"],) * 2)
    assert np.linalg.norm(p["rhs"] - A @ rd["x"]) / np.linalg.norm(p["rhs"]) <= 1e-6
    full = loopback_solve(p["row_ptr"], p["col"], p["val"], p["nc"], nranks, p["rhs"], owner=owner_in,
                          coarsest_max_dof=100)
    print("iterations: global BILU", full["iters"], "rank-local BILU", rd["iters"])


def test_loopback_gpu_factorization_bit_identical_to_single_gpu():
    """The distributed setup factorizes the GLOBAL matrix on the GPU (like msp_setup) and
    keeps its rows: the loopback solve at 1 rank reproduces the single-GPU solve."""
    from paper_2208_08594_b200 import loopback_solve, MspSolver
    p = gen.make_config("C2", nx=20, ny=16, nz=6)
    rd = loopback_solve(p["row_ptr"], p["col"], p["val"], p["nc"], 1, p["rhs"], coarsest_max_dof=80)
    s = MspSolver(p["row_ptr"], p["col"], p["val"], nc=p["nc"], coarsest_max_dof=80)
    r1 = s.solve(torch.from_numpy(p["rhs"]).cuda())
    assert rd["iters"] == r1["iters"]
    x1 = r1["x"].cpu().numpy()
    assert np.linalg.norm(rd["x"] - x1) <= 1e-9 * np.linalg.norm(x1)


@pytest.mark.parametrize("nranks", [2, 3])
def test_loopback_halo_overlap_bit_identical(nranks, monkeypatch):
    """The z halo of the SpMV / a8 input overlapped with the slab-interior rows (side
    stream, fork/join events) gives the same iterates as exchange-then-compute."""
    from paper_2208_08594_b200 import loopback_solve, HostSetup
    p = gen.make_config("C2", nx=24, ny=20, nz=9)
    owner = HostSetup(p["row_ptr"], p["col"], p["val"], p["nc"], coarsest_max_dof=100).partition_owner(
        p["nx"], p["ny"], p["nz"], nranks)
    out = []
    for v in ("0", "1"):
        monkeypatch.setenv("MSP_DIST_OVERLAP", v)
        out.append(loopback_solve(p["row_ptr"], p["col"], p["val"], p["nc"], nranks, p["rhs"], owner=owner,
                                  coarsest_max_dof=100))
    assert out[0]["iters"] == out[1]["iters"]
    assert np.array_equal(out[0]["x"], out[1]["x"])


@pytest.mark.parametrize("nranks", [2, 3])
def test_loopback_rank0_setup_broadcast_identical(nranks, monkeypatch):
    """Only rank 0 runs S1-S4 and broadcasts the result (default) vs every rank running the
    host setup (MSP_DIST_SETUP_ALL=1): identical plans -> bit-identical iterates."""
    from paper_2208_08594_b200 import loopback_solve, HostSetup
    p = gen.make_config("C2", nx=24, ny=20, nz=9)
    owner = HostSetup(p["row_ptr"], p["col"], p["val"], p["nc"], coarsest_max_dof=100).partition_owner(
        p["nx"], p["ny"], p["nz"], nranks)
    out = []
    for v in ("1", "0"):
        monkeypatch.setenv("MSP_DIST_SETUP_ALL", v)
        out.append(loopback_solve(p["row_ptr"], p["col"], p["val"], p["nc"], nranks, p["rhs"], owner=owner,
                                  coarsest_max_dof=100))
    assert out[0]["iters"] == out[1]["iters"]
    assert np.array_equal(out[0]["x"], out[1]["x"])
    assert np.array_equal(out[0]["rank_info"], out[1]["rank_info"])


def test_loopback_rank0_setup_error_propagates():
    """A setup error on rank 0 (coarsening stall -> MSP_ESTALL there) reaches every rank
    through the broadcast status instead of leaving the others waiting."""
    from paper_2208_08594_b200 import loopback_solve
    from paper_2208_08594_b200._binding import MspError
    p = gen.make_config("C2", nx=12, ny=10, nz=4)
    with pytest.raises(MspError):
        loopback_solve(p["row_ptr"], p["col"], p["val"], p["nc"], 2, p["rhs"], coarsest_max_dof=1, max_levels=2)


@pytest.mark.parametrize("nranks", [2, 3])
def test_loopback_fused_halo_pack_bit_identical(nranks, monkeypatch):
    """Halo packing inside the producer kernels (BILU color phases, level-0 PGS-MC colors,
    a3's fused first color, the prolongation) instead of a separate pack kernel per
    exchange: same send buffers, so bit-identical iterates."""
    from paper_2208_08594_b200 import loopback_solve, HostSetup
    p = gen.make_config("C2", nx=24, ny=20, nz=9)
    owner = HostSetup(p["row_ptr"], p["col"], p["val"], p["nc"], coarsest_max_dof=100).partition_owner(
        p["nx"], p["ny"], p["nz"], nranks)
    out = []
    for v in ("0", "1"):
        monkeypatch.setenv("MSP_DIST_FUSE_PACK", v)
        out.append(loopback_solve(p["row_ptr"], p["col"], p["val"], p["nc"], nranks, p["rhs"], owner=owner,
                                  coarsest_max_dof=100))
    assert out[0]["iters"] == out[1]["iters"]
    assert np.array_equal(out[0]["x"], out[1]["x"])


def test_dist_update_reuses_with_global_sizes():
    """msp_update on a distributed handle compares the GLOBAL size and pattern,
    so an ASMSP step with last_iterations <= mu reuses the preconditioner."""
    from paper_2208_08594_b200 import DistSolver, nccl_unique_id
    p0 = gen.make_config("C2", nx=20, ny=16, nz=6)
    p1 = gen.make_config("C2", nx=20, ny=16, nz=6, newton_step=1)
    d = DistSolver(p0["row_ptr"], p0["col"], p0["val"], p0["nc"], 0, 1, nccl_unique_id(), coarsest_max_dof=80)
    assert d.update(p1["row_ptr"], p1["col"], p1["val"], iota=2, last_iterations=5, mu=10) is False
    assert d.stats()["reuse_calls"] == 1
    r = d.solve(torch.from_numpy(p1["rhs"]).cuda())
    assert r["final_rel"] <= 1e-6
    assert d.update(p1["row_ptr"], p1["col"], p1["val"], iota=3, last_iterations=11, mu=10) is True
