"""GPU parity tests: the CUDA path (through the C-ABI) against the CPU oracle on the same
seeded inputs.  Tolerances:
  - SpMV (a2): componentwise |dy_i| <= 1e-12 (|A||x|)_i, bit-exact on integer inputs;
  - one PGS-MC sweep (a4): ||dx||_inf / ||x||_inf <= 1e-12;
  - V-cycle / BILU / MSP apply: normwise 1e-10 (composites of many kernels plus the
    dense coarsest inverse vs LU: error ~ cond * eps);
  - full solve: iterations within +-1 of the oracle, both true residuals <= tol,
    history agreeing to 1e-6 relative while above 1e-10 (north_star).
"""
import json
import os

import numpy as np
import pytest
import scipy.sparse as sp

import gen
import oracle
from _parity import assert_hist_agree

pytestmark = pytest.mark.gpu

torch = pytest.importorskip("torch")


def solver(p, **kw):
    from paper_2208_08594_b200 import MspSolver
    return MspSolver(p["row_ptr"], p["col"], p["val"], nc=p["nc"], **kw)


def absA_absx(p, x):
    return oracle.bsr_spmv(p["row_ptr"], p["col"], np.abs(p["val"]), np.abs(x))


def to_internal(order, v, b):
    return v.reshape(-1, b)[order].reshape(-1)


def from_internal(order, v, b):
    out = np.empty_like(v.reshape(-1, b))
    out[order] = v.reshape(-1, b)
    return out.reshape(-1)


# ------------------------------------------------------------------ a2 SpMV
@pytest.mark.parametrize("name,kw", [("C1", {}), ("C2", {}), ("C2", dict(nx=17, ny=13, nz=3, nc=6)),
                                     ("C1", dict(nx=1, ny=1, nz=1))])
def test_spmv_parity(name, kw):
    p = gen.make_config(name, **kw)
    s = solver(p, coarsest_max_dof=64)
    order = s.order()
    b = p["b"]
    x = gen.random_vector(p["n"] * b, 11)
    ref = oracle.bsr_spmv(p["row_ptr"], p["col"], p["val"], x)
    xd = torch.from_numpy(to_internal(order, x, b)).cuda()
    yd = torch.zeros_like(xd)
    s.spmv_internal(xd, yd)
    y = from_internal(order, yd.cpu().numpy(), b)
    bound = 1e-12 * absA_absx(p, x)
    assert np.all(np.abs(y - ref) <= bound + 1e-300)
    assert np.linalg.norm(y - ref) <= 1e-12 * np.linalg.norm(ref)


def test_spmv_integer_bit_exact():
    p = gen.make_config("C2", nx=31, ny=29, nz=7)
    rng = np.random.default_rng(5)
    p["val"] = rng.integers(-50, 51, p["val"].shape).astype(np.float64)
    for c in range(p["n"]):
        for e in range(p["row_ptr"][c], p["row_ptr"][c + 1]):
            if p["col"][e] == c:
                p["val"][e] += 400 * np.eye(p["b"])
    s = solver(p, coarsest_max_dof=100000, decoupling=1)
    order = s.order()
    x = gen.integer_vector(p["n"] * p["b"], 3, lim=100)
    ref = oracle.bsr_spmv(p["row_ptr"], p["col"], p["val"], x)
    xd = torch.from_numpy(to_internal(order, x, p["b"])).cuda()
    yd = torch.zeros_like(xd)
    s.spmv_internal(xd, yd)
    assert np.array_equal(from_internal(order, yd.cpu().numpy(), p["b"]), ref)


# ------------------------------------------------------------------ a4 PGS-MC
@pytest.mark.parametrize("asc", [True, False])
def test_pgs_sweep_parity_every_level(asc):
    p = gen.make_config("C2", nx=40, ny=30, nz=6)
    s = solver(p, coarsest_max_dof=200)
    O = oracle.Msp(p["row_ptr"], p["col"], p["val"], coarsest_max_dof=200)
    L = O.info()["levels"]
    assert L >= 2
    for l in range(L):
        ptr, col, val = O.level_csr(l)
        g, color = O.level_colors(l)
        n = len(ptr) - 1
        b = gen.random_vector(n, 100 + l)
        x0 = gen.random_vector(n, 200 + l)
        ref = oracle.pgs_mc(ptr, col, val, color, g, b, x0, asc)
        bd = torch.from_numpy(b).cuda()
        xd = torch.from_numpy(x0.copy()).cuda()
        s.pgs_sweep(l, bd, xd, asc)
        x = xd.cpu().numpy()
        assert np.max(np.abs(x - ref)) <= 1e-12 * np.max(np.abs(ref)), l


# ------------------------------------------------------------------ NEXT-4 smoothers (R13)
@pytest.mark.parametrize("sm,K", [(1, 32), (2, 32), (2, 1), (2, 7), (2, 16), (2, 45), (2, 100000)])
@pytest.mark.parametrize("asc", [True, False])
def test_no_smoother_sweep_parity_every_level(sm, K, asc):
    """One PJAC-NO / PGS-NO sweep per AMG level vs the oracle's definition (R13)."""
    p = gen.make_config("C2", nx=40, ny=30, nz=6)
    s = solver(p, coarsest_max_dof=200, smoother=sm, gs_chunk=K)
    O = oracle.Msp(p["row_ptr"], p["col"], p["val"], coarsest_max_dof=200)
    L = O.info()["levels"]
    assert L >= 2
    for l in range(L):
        ptr, col, val = O.level_csr(l)
        n = len(ptr) - 1
        b = gen.random_vector(n, 100 + l)
        x0 = gen.random_vector(n, 200 + l)
        if sm == 1:
            ref = oracle.jacobi_sweep(ptr, col, val, b, x0)
        else:
            ref = oracle.hybrid_gs_sweep(ptr, col, val, K, b, x0, asc)
        xd = torch.from_numpy(x0.copy()).cuda()
        s.pgs_sweep(l, torch.from_numpy(b).cuda(), xd, asc)
        x = xd.cpu().numpy()
        assert np.max(np.abs(x - ref)) <= 1e-12 * np.max(np.abs(ref)), l


@pytest.mark.parametrize("sm", [1, 2])
def test_no_smoother_vcycle_and_solve_parity(sm):
    """V-cycle and MSP-GMRES with the comparison smoothers vs the oracle (Table 2 analog)."""
    p = gen.make_config("C2", nx=24, ny=20, nz=4)
    s = solver(p, coarsest_max_dof=50, smoother=sm)
    O = oracle.Msp(p["row_ptr"], p["col"], p["val"], coarsest_max_dof=50, smoother=sm)
    r = gen.random_vector(p["n"], 7)
    ref = O.vcycle(r)
    xd = torch.zeros(p["n"], dtype=torch.float64, device="cuda")
    s.vcycle(torch.from_numpy(r).cuda(), xd)
    assert np.linalg.norm(xd.cpu().numpy() - ref) <= 1e-10 * np.linalg.norm(ref)
    ro = O.solve(p["rhs"], tol=1e-8)
    rg = s.solve(torch.from_numpy(p["rhs"]).cuda(), tol=1e-8)
    assert abs(rg["iters"] - ro["iters"]) <= 1, (rg["iters"], ro["iters"])
    assert rg["final_rel"] <= 1e-8


# ------------------------------------------------------------------ V-cycle, BILU, MSP
@pytest.mark.parametrize("kw", [dict(coarsest_max_dof=200), dict(coarsest_max_dof=200, pair_passes=1),
                                dict(), dict(coarsest_max_dof=200, use_graphs=0),
                                dict(coarsest_max_dof=200, pre_sweeps=2, post_sweeps=2)])
def test_vcycle_parity(kw):
    p = gen.make_config("C2", nx=40, ny=30, nz=6)
    s = solver(p, **kw)
    O = oracle.Msp(p["row_ptr"], p["col"], p["val"], **{k: v for k, v in kw.items() if k != "use_graphs"})
    r = gen.random_vector(p["n"], 7)
    ref = O.vcycle(r)
    xd = torch.zeros(p["n"], dtype=torch.float64, device="cuda")
    s.vcycle(torch.from_numpy(r).cuda(), xd)
    x = xd.cpu().numpy()
    assert np.linalg.norm(x - ref) <= 1e-10 * np.linalg.norm(ref)


@pytest.mark.parametrize("nc,dims,orth", [(2, (13, 11, 3), 0), (4, (7, 5, 9), 0), (2, (13, 11, 3), 2),
                                          (4, (7, 5, 9), 2), (2, (13, 11, 3), 1)])
def test_solve_odd_vector_length(nc, dims, orth):
    """N = n*b odd (b = 3, 5 with an odd cell count): the Krylov kernels' 16-byte paths
    must not drop the last entry or misalign the basis slots."""
    p = gen.make_config("C2", nx=dims[0], ny=dims[1], nz=dims[2], nc=nc)
    assert (p["n"] * p["b"]) % 2 == 1
    s = solver(p, coarsest_max_dof=60, orth=orth)
    O = oracle.Msp(p["row_ptr"], p["col"], p["val"], coarsest_max_dof=60, orth=orth)
    ro = O.solve(p["rhs"], tol=1e-8)
    rg = s.solve(torch.from_numpy(p["rhs"]).cuda(), tol=1e-8)
    assert abs(rg["iters"] - ro["iters"]) <= 1, (rg["iters"], ro["iters"])
    A = sp.bsr_matrix((p["val"], p["col"], p["row_ptr"]), shape=(p["n"] * p["b"],) * 2)
    xs = rg["x"].cpu().numpy()
    assert np.linalg.norm(p["rhs"] - A @ xs) / np.linalg.norm(p["rhs"]) <= 1e-8


@pytest.mark.parametrize("name,gkw,kw", [("C2", dict(nx=25, ny=20, nz=5), dict()),
                                         ("C2", dict(nx=12, ny=10, nz=4, nc=6), dict()),
                                         ("C2", dict(nx=13, ny=11, nz=3, nc=2), dict(bilu_order=0))])
def test_gpu_bilu_factorization_bit_exact(name, gkw, kw, monkeypatch):
    """NEXT-2: the BILU(0) factors computed on the GPU per block color are bit-identical to
    the oracle's factorization (L/U blocks) and inverted pivot blocks D~^-1 (R5), and to
    the product's host factorization (MSP_HOST_BILU=1)."""
    p = gen.make_config(name, **gkw)
    s = solver(p, coarsest_max_dof=100, **kw)
    F = s.bilu_factors()
    O = oracle.Msp(p["row_ptr"], p["col"], p["val"], coarsest_max_dof=100, **kw)
    Fo, Do = O.bilu_factors()
    rp, col = p["row_ptr"], p["col"]
    diag = np.zeros(len(col), bool)
    for i in range(p["n"]):
        for e in range(rp[i], rp[i + 1]):
            if col[e] == i:
                diag[e] = True
                assert np.array_equal(F[e], Do[i]), i
    assert np.array_equal(F[~diag], Fo[~diag])
    monkeypatch.setenv("MSP_HOST_BILU", "1")
    assert np.array_equal(solver(p, coarsest_max_dof=100, **kw).bilu_factors(), F)


@pytest.mark.parametrize("kw", [dict(), dict(bilu_order=0), dict(decoupling=1), dict(stages=3)])
def test_bilu_and_msp_apply_parity(kw):
    p = gen.make_config("C2", nx=25, ny=20, nz=5)
    s = solver(p, coarsest_max_dof=100, **kw)
    O = oracle.Msp(p["row_ptr"], p["col"], p["val"], coarsest_max_dof=100, **kw)
    g = gen.random_vector(p["n"] * p["b"], 9)
    out = torch.zeros(p["n"] * p["b"], dtype=torch.float64, device="cuda")
    s.bilu_apply(torch.from_numpy(g).cuda(), out)
    ref = O.bilu_apply(g)
    assert np.linalg.norm(out.cpu().numpy() - ref) <= 1e-10 * np.linalg.norm(ref)
    s.apply(torch.from_numpy(g).cuda(), out)
    ref = O.apply(g)
    assert np.linalg.norm(out.cpu().numpy() - ref) <= 1e-10 * np.linalg.norm(ref)
    # host pointers through the same entry point
    w = np.zeros_like(g)
    s.apply(g, w)
    assert np.linalg.norm(w - ref) <= 1e-10 * np.linalg.norm(ref)


# ------------------------------------------------------------------ full solve
def check_solve(p, tol=1e-6, restart=30, **kw):
    """GPU solve vs the oracle's TEXTBOOK orthogonalisation (CGS2, or MGS when asked): the
    product's DCGS2 (R14) builds the same basis in exact arithmetic."""
    s = solver(p, **kw)
    okw = {k: v for k, v in kw.items() if k not in ("use_graphs", "orth")}
    O = oracle.Msp(p["row_ptr"], p["col"], p["val"], orth=1 if kw.get("orth") == 1 else 0, **okw)
    o = O.solve(p["rhs"], tol=tol, restart=restart)
    r = s.solve(torch.from_numpy(p["rhs"]).cuda(), tol=tol, restart=restart)
    x = r["x"].cpu().numpy()
    assert abs(r["iters"] - o["iters"]) <= 1, (r["iters"], o["iters"])
    A = sp.bsr_matrix((p["val"], p["col"], p["row_ptr"]), shape=(p["n"] * p["b"],) * 2)
    true = np.linalg.norm(p["rhs"] - A @ x) / np.linalg.norm(p["rhs"])
    assert true <= tol and o["final_rel"] <= tol
    assert abs(true - r["final_rel"]) <= 1e-10
    k = assert_hist_agree(r["hist"], r["iters"], o["hist"], o["iters"], restart)
    assert k >= min(r["iters"], o["iters"]) // 2
    return r, o


@pytest.mark.parametrize("name,gkw,kw", [
    ("C1", {}, {}),
    ("C1", {}, dict(coarsest_max_dof=50)),
    ("C1", {}, dict(coarsest_max_dof=50, bilu_order=0)),
    ("C1", {}, dict(coarsest_max_dof=50, use_graphs=0)),
    ("C2", dict(nx=37, ny=23, nz=7), dict(coarsest_max_dof=100, use_graphs=0)),
    ("C2", dict(nx=37, ny=23, nz=7), dict(coarsest_max_dof=100)),
    ("C2", dict(nx=20, ny=20, nz=5, nc=6), dict(coarsest_max_dof=100)),
    ("C3", dict(nx=12, ny=44, nz=17), dict(coarsest_max_dof=300)),
    ("C1", {}, dict(coarsest_max_dof=50, stages=3)),
    ("C2", dict(nx=25, ny=20, nz=5), dict(coarsest_max_dof=100, stages=3)),
    ("C2", dict(nx=20, ny=20, nz=5, nc=6), dict(coarsest_max_dof=100, stages=3)),
    ("C1", {}, dict(coarsest_max_dof=50, orth=2)),
    ("C1", {}, dict(coarsest_max_dof=50, orth=2, use_graphs=0)),
    ("C2", dict(nx=37, ny=23, nz=7), dict(coarsest_max_dof=100, orth=2)),
    ("C2", dict(nx=20, ny=20, nz=5, nc=6), dict(coarsest_max_dof=100, orth=2)),
    ("C3", dict(nx=12, ny=44, nz=17), dict(coarsest_max_dof=300, orth=2)),
])
def test_solve_parity(name, gkw, kw):
    check_solve(gen.make_config(name, **gkw), **kw)


def test_solve_parity_restarts_and_mgs():
    p = gen.make_config("C2", nx=30, ny=30, nz=6)
    r, o = check_solve(p, restart=5, coarsest_max_dof=100)
    assert r["iters"] > 5                                  # several restart cycles
    check_solve(p, coarsest_max_dof=100, orth=1)
    r, o = check_solve(p, restart=5, coarsest_max_dof=100, orth=2)
    r, o = check_solve(p, restart=30, coarsest_max_dof=100, orth=2, tol=1e-10)
    assert r["iters"] > 17                                  # exercises the k > 16 (unfused) pass 2


def test_solve_parity_C2_full():
    check_solve(gen.make_config("C2"))


def test_solve_edge_cases():
    p = gen.make_config("C1", nx=4, ny=3, nz=2)
    s = solver(p)
    r = s.solve(torch.zeros(p["n"] * p["b"], dtype=torch.float64, device="cuda"))
    assert r["iters"] == 0 and float(r["x"].abs().max()) == 0.0
    # one cell: MSP with exact stages is A^-1 -> one iteration
    q = gen.make_config("C1", nx=1, ny=1, nz=1)
    s1 = solver(q)
    r = s1.solve(torch.from_numpy(q["rhs"]).cuda(), tol=1e-10)
    assert r["iters"] == 1
    # x0 = exact solution -> 0 iterations
    r = s.solve(torch.from_numpy(p["rhs"]).cuda(), x=torch.from_numpy(p["xstar"].copy()).cuda(),
                tol=1e-6)
    assert r["iters"] == 0
    # host (numpy) buffers
    r = s.solve(p["rhs"].copy())
    assert isinstance(r["x"], np.ndarray) and r["final_rel"] <= 1e-6
    # maxit reached -> ENOCONV with valid outputs
    r = s.solve(torch.from_numpy(p["rhs"]).cuda(), tol=1e-14, maxit=2)
    assert r["status"] == 3 and r["iters"] == 2


def test_asmsp_update_reuse_and_rebuild():
    p0 = gen.make_config("C2", nx=20, ny=20, nz=4)
    s = solver(p0, coarsest_max_dof=100)
    O = oracle.Msp(p0["row_ptr"], p0["col"], p0["val"], coarsest_max_dof=100)
    p1 = gen.make_config("C2", nx=20, ny=20, nz=4, newton_step=1)
    assert s.update(p1["row_ptr"], p1["col"], p1["val"], iota=2, last_iterations=5, mu=10) is False
    O.update_values(p1["val"])
    o = O.solve(p1["rhs"])
    r = s.solve(torch.from_numpy(p1["rhs"]).cuda())
    assert abs(r["iters"] - o["iters"]) <= 1
    assert s.update(p1["row_ptr"], p1["col"], p1["val"], iota=3, last_iterations=11, mu=10) is True
    st = s.stats()
    assert st["setup_calls"] == 2 and st["reuse_calls"] == 1


def test_full_size_c3_spmv_sampled_and_solve():
    """C3 at full size in the bench's launch configuration: SpMV on sampled rows vs the
    oracle's definition, and the solve against the oracle's committed iteration count
    (tests/golden/oracle_c3.json, written by tests/golden/make_oracle.py)."""
    p = gen.make_config("C3")
    s = solver(p)
    order = s.order()
    b = p["b"]
    x = gen.random_vector(p["n"] * b, 21)
    xd = torch.from_numpy(to_internal(order, x, b)).cuda()
    yd = torch.zeros_like(xd)
    s.spmv_internal(xd, yd)
    y = from_internal(order, yd.cpu().numpy(), b)
    rows = np.random.default_rng(0).choice(p["n"], 2000, replace=False)
    for c in rows:
        ref = np.zeros(b)
        for e in range(p["row_ptr"][c], p["row_ptr"][c + 1]):
            ref += p["val"][e] @ x[p["col"][e] * b:(p["col"][e] + 1) * b]
        absref = sum(np.abs(p["val"][e]) @ np.abs(x[p["col"][e] * b:(p["col"][e] + 1) * b])
                     for e in range(p["row_ptr"][c], p["row_ptr"][c + 1]))
        assert np.all(np.abs(y[c * b:(c + 1) * b] - ref) <= 1e-12 * absref)
    r = s.solve(torch.from_numpy(p["rhs"]).cuda(), tol=1e-6)
    A = sp.bsr_matrix((p["val"], p["col"], p["row_ptr"]), shape=(p["n"] * b,) * 2)
    xs = r["x"].cpu().numpy()
    assert np.linalg.norm(p["rhs"] - A @ xs) / np.linalg.norm(p["rhs"]) <= 1e-6
    gold = os.path.join(os.path.dirname(__file__), "golden", "oracle_c3.json")
    if os.path.exists(gold):
        ref = json.load(open(gold))
        assert abs(r["iters"] - ref["iters"]) <= 1, (r["iters"], ref["iters"])
        _check_hist(r["hist"], ref["hist"], iters=r["iters"], ref_iters=ref["iters"])


def _check_hist(h, ref, n_first=15, rtol=1e-9, iters=None, ref_iters=None):
    """Relative-residual history against the oracle's: the first n_first iterations
    (before rounding differences amplify) agree to rtol, and the whole history obeys the
    north_star rule (1e-6 relative while > 1e-10, tests/_parity.py)."""
    h = np.asarray(h)
    ref = np.asarray(ref)
    k = min(n_first, len(h), len(ref))
    dev = np.abs(h[:k] - ref[:k]) / ref[:k]
    print("hist max rel dev (first %d): %.3e" % (k, dev.max()))
    assert dev.max() <= rtol, dev
    if iters is not None:
        assert_hist_agree(h, iters, ref, ref_iters, 30)


@pytest.mark.parametrize("sm", [1, 2])
def test_full_size_c3_no_smoothers_vs_oracle_golden(sm):
    """Table 2 analog at full C3 size (NEXT-4, R13): MSP-GMRES with PJAC-NO / PGS-NO (K=32)
    against the oracle's committed runs (oracle_c3_sm<k>.json, make_oracle.py C3 <k>)."""
    p = gen.make_config("C3")
    s = solver(p, smoother=sm, gs_chunk=32)
    r = s.solve(torch.from_numpy(p["rhs"]).cuda(), tol=1e-6)
    ref = json.load(open(os.path.join(os.path.dirname(__file__), "golden", f"oracle_c3_sm{sm}.json")))
    assert ref["smoother"] == sm and ref["gs_chunk"] == 32
    assert abs(r["iters"] - ref["iters"]) <= 1, (r["iters"], ref["iters"])
    assert r["final_rel"] <= 1e-6
    _check_hist(r["hist"], ref["hist"], iters=r["iters"], ref_iters=ref["iters"])


def test_full_size_c3_dcgs2_vs_oracle_golden():
    """DCGS2 (orth=2, R14) at full C3 size against the oracle's CGS2 run: the same Arnoldi
    basis in exact arithmetic -> same iterations, early history to rounding level."""
    p = gen.make_config("C3")
    s = solver(p, orth=2)
    r = s.solve(torch.from_numpy(p["rhs"]).cuda(), tol=1e-6)
    ref = json.load(open(os.path.join(os.path.dirname(__file__), "golden", "oracle_c3.json")))
    assert abs(r["iters"] - ref["iters"]) <= 1, (r["iters"], ref["iters"])
    assert r["final_rel"] <= 1e-6
    _check_hist(r["hist"], ref["hist"], iters=r["iters"], ref_iters=ref["iters"])


def test_full_size_c4_solve_vs_oracle_golden():
    """C4 (SPE10-size, 6 components -> 7x7 blocks, the 8-lane kernel variants) at full
    size: converged true residual, iteration count and early residual history against the
    oracle's committed run (tests/golden/oracle_c4.json, make_oracle.py C4)."""
    p = gen.make_config("C4")
    s = solver(p)
    r = s.solve(torch.from_numpy(p["rhs"]).cuda(), tol=1e-6)
    b = p["b"]
    A = sp.bsr_matrix((p["val"], p["col"], p["row_ptr"]), shape=(p["n"] * b,) * 2)
    xs = r["x"].cpu().numpy()
    assert np.linalg.norm(p["rhs"] - A @ xs) / np.linalg.norm(p["rhs"]) <= 1e-6
    ref = json.load(open(os.path.join(os.path.dirname(__file__), "golden", "oracle_c4.json")))
    assert s.stats()["levels"] == ref["levels"]["levels"]
    assert abs(r["iters"] - ref["iters"]) <= 1, (r["iters"], ref["iters"])
    _check_hist(r["hist"], ref["hist"], iters=r["iters"], ref_iters=ref["iters"])


def test_full_size_c5_solve_vs_oracle_golden():
    """C5 (200^3 = 8 M cells, 4x4 blocks, the scaling configuration) at full size: the
    GPU solve against the oracle's committed run (tests/golden/oracle_c5.json, written by
    make_oracle.py C5: 51 iterations, CGS2, ~17 min single-threaded), sampled SpMV rows
    against the definition, and the converged true residual."""
    p = gen.make_config("C5")
    s = solver(p)
    b = p["b"]
    order = s.order()
    x = gen.random_vector(p["n"] * b, 31)
    xd = torch.from_numpy(to_internal(order, x, b)).cuda()
    yd = torch.zeros_like(xd)
    s.spmv_internal(xd, yd)
    y = from_internal(order, yd.cpu().numpy(), b)
    del xd, yd
    for c in np.random.default_rng(1).choice(p["n"], 1000, replace=False):
        e0, e1 = p["row_ptr"][c], p["row_ptr"][c + 1]
        ref = sum(p["val"][e] @ x[p["col"][e] * b:(p["col"][e] + 1) * b] for e in range(e0, e1))
        absref = sum(np.abs(p["val"][e]) @ np.abs(x[p["col"][e] * b:(p["col"][e] + 1) * b]) for e in range(e0, e1))
        assert np.all(np.abs(y[c * b:(c + 1) * b] - ref) <= 1e-12 * absref)
    r = s.solve(torch.from_numpy(p["rhs"]).cuda(), tol=1e-6)
    ref = json.load(open(os.path.join(os.path.dirname(__file__), "golden", "oracle_c5.json")))
    assert s.stats()["levels"] == ref["levels"]["levels"]
    assert s.stats()["n_coarsest"] == ref["levels"]["n_coarsest"]
    assert abs(r["iters"] - ref["iters"]) <= 1, (r["iters"], ref["iters"])
    A = sp.bsr_matrix((p["val"], p["col"], p["row_ptr"]), shape=(p["n"] * b,) * 2)
    xs = r["x"].cpu().numpy()
    assert np.linalg.norm(p["rhs"] - A @ xs) / np.linalg.norm(p["rhs"]) <= 1e-6
    _check_hist(r["hist"], ref["hist"], iters=r["iters"], ref_iters=ref["iters"])


@pytest.mark.parametrize("orth", [0, 2])
def test_cycle_graph_matches_per_step_graphs(orth, monkeypatch):
    """MSP_CYCLE_GRAPH=1: each restart cycle runs as ONE graph of conditional Arnoldi steps
    with the Givens update / convergence test on the device (givens_kernel); same
    iterations, history and solution as the per-step graphs with the host loop."""
    p = gen.make_config("C2", nx=30, ny=30, nz=6)
    out = []
    for v in ("0", "1"):
        monkeypatch.setenv("MSP_CYCLE_GRAPH", v)
        s = solver(p, coarsest_max_dof=100, orth=orth)
        r = s.solve(torch.from_numpy(p["rhs"]).cuda(), restart=7, tol=1e-9)
        out.append(r)
    assert out[0]["iters"] == out[1]["iters"] and out[0]["iters"] > 7
    assert_hist_agree(out[0]["hist"], out[0]["iters"], out[1]["hist"], out[1]["iters"], 7, rtol=1e-7)
    x0, x1 = out[0]["x"].cpu().numpy(), out[1]["x"].cpu().numpy()
    assert np.linalg.norm(x0 - x1) <= 1e-10 * np.linalg.norm(x0)


@pytest.mark.parametrize("orth", [0, 2])
def test_speculative_steps_bit_identical(orth, monkeypatch):
    """Step j+1 enqueued before the host's Givens update of step j (MSP_SPEC_STEPS, on by
    default): bit-identical solution and history to the synchronous loop, over restarts,
    at convergence (a step enqueued past it is discarded) and at maxit."""
    p = gen.make_config("C2", nx=30, ny=30, nz=6)
    for kw in (dict(restart=7, tol=1e-9), dict(restart=30, tol=1e-6), dict(restart=5, tol=1e-12, maxit=12)):
        out = []
        for v in ("0", "1"):
            monkeypatch.setenv("MSP_SPEC_STEPS", v)
            s = solver(p, coarsest_max_dof=100, orth=orth)
            out.append(s.solve(torch.from_numpy(p["rhs"]).cuda(), **kw))
        assert out[0]["iters"] == out[1]["iters"], kw
        assert np.array_equal(out[0]["hist"], out[1]["hist"]), kw
        assert torch.equal(out[0]["x"], out[1]["x"]), kw


def test_device_bsr_input_matches_host():
    """msp_bsr with device pointers (include/msp.h: device >= 0; the binding passes CUDA
    tensors through): the same SETUP and solve as from host arrays, bit for bit, and the
    ASMSP reuse path refreshing values straight from device memory."""
    p = gen.make_config("C2", nx=20, ny=18, nz=6)
    q = gen.make_config("C2", nx=20, ny=18, nz=6, newton_step=1)
    b = torch.from_numpy(p["rhs"]).cuda()
    hs = solver(p, coarsest_max_dof=80)
    dev = lambda a, dt: torch.from_numpy(np.ascontiguousarray(a)).to(dt).cuda()
    ds = solver(dict(p, row_ptr=dev(p["row_ptr"], torch.int32), col=dev(p["col"], torch.int32),
                     val=dev(p["val"], torch.float64)), coarsest_max_dof=80)
    r0, r1 = hs.solve(b), ds.solve(b)
    assert r0["iters"] == r1["iters"] and torch.equal(r0["x"], r1["x"])
    assert not hs.update(q["row_ptr"], q["col"], q["val"], 2, 5, 50)
    assert not ds.update(dev(q["row_ptr"], torch.int32), dev(q["col"], torch.int32), dev(q["val"], torch.float64),
                         2, 5, 50)
    r0, r1 = hs.solve(b), ds.solve(b)
    assert r0["iters"] == r1["iters"] and torch.equal(r0["x"], r1["x"])
    assert ds.update(dev(q["row_ptr"], torch.int32), dev(q["col"], torch.int32), dev(q["val"], torch.float64),
                     3, 100, 50)                               # rebuild from device values
    assert hs.update(q["row_ptr"], q["col"], q["val"], 3, 100, 50)
    r0, r1 = hs.solve(b), ds.solve(b)
    assert r0["iters"] == r1["iters"] and torch.equal(r0["x"], r1["x"])


@pytest.mark.parametrize("orth", [0, 1, 2])
def test_zbasis_cycle_end_matches_b_of_v_y(orth, monkeypatch):
    """zbasis mode (default): the cycle end forms x += Z y' from the z_j = B v_j the steps
    computed (DCGS2: y' = T y maps the provisional vectors the steps saw to the final
    basis) instead of applying B to V y.  Same iterations, histories within the parity
    rule, solutions equal to rounding, over several restarts."""
    p = gen.make_config("C2", nx=30, ny=30, nz=6)
    out = []
    for v in ("0", "1"):
        monkeypatch.setenv("MSP_ZBASIS", v)
        s = solver(p, coarsest_max_dof=100, orth=orth)
        out.append(s.solve(torch.from_numpy(p["rhs"]).cuda(), restart=7, tol=1e-9))
    assert out[0]["iters"] == out[1]["iters"] and out[0]["iters"] > 14
    assert_hist_agree(out[0]["hist"], out[0]["iters"], out[1]["hist"], out[1]["iters"], 7, rtol=1e-7)
    x0, x1 = out[0]["x"].cpu().numpy(), out[1]["x"].cpu().numpy()
    assert np.linalg.norm(x0 - x1) <= 1e-9 * np.linalg.norm(x0)


def test_time_kernel_per_level_vcycle():
    """msp_time_kernel kinds 16 + l (the V-cycle from level l down; 16 + L = the coarsest
    solve alone, the same piece as kind 5): positive, monotone in l (each level adds its
    sweeps and transfers), and the last one matches the coarsest-GEMV kind."""
    p = gen.make_config("C2", nx=30, ny=30, nz=8)
    s = solver(p, coarsest_max_dof=60)
    L = s.stats()["levels"]
    assert L >= 2
    t = [s.time_kernel(16 + l, reps=5)[0] for l in range(L + 1)]
    assert all(x > 0 for x in t)
    assert all(t[l] > t[l + 1] for l in range(L)), t
    c = s.time_kernel("a6_coarse_gemv", reps=5)[0]
    assert 0.5 * c < t[L] < 2.0 * c, (t[L], c)
    with pytest.raises(Exception):
        s.time_kernel(17 + L, reps=1)


def test_caller_stream_ordering():
    """the library orders its work after the caller's stream.  b is produced by
    a kernel on a torch side stream that the solver was told about (set_stream), with no
    host synchronisation in between; the solve must see the finished b."""
    p = gen.make_config("C2", nx=20, ny=16, nz=6)
    s = solver(p, coarsest_max_dof=80)
    side = torch.cuda.Stream()
    b0 = torch.from_numpy(p["rhs"]).cuda()
    torch.cuda.synchronize()
    s.set_stream(side.cuda_stream)
    with torch.cuda.stream(side):
        b = torch.empty_like(b0)
        torch.cuda._sleep(50_000_000)                   # keep the side stream busy
        b.copy_(b0)
        x = torch.zeros_like(b)
        r = s.solve(b, x, tol=1e-8)
    assert r["final_rel"] <= 1e-8
    ref = s.solve(b0.clone(), tol=1e-8)
    assert r["iters"] == ref["iters"]


def test_failed_rebuild_invalidates_handle():
    """a rebuild that fails after the old device state was released (here: a
    singular pivot / coarsest matrix) leaves the handle unusable (MSP_EINVAL) instead of
    running kernels on freed memory; a good rebuild revives it.  (A failure in the host
    steps before the release keeps the previous preconditioner.)"""
    from paper_2208_08594_b200 import MspSolver
    from paper_2208_08594_b200._binding import MspError
    ptr, col = np.array([0, 1], np.int32), np.array([0], np.int32)
    good = np.array([[[2.0, 1.0], [1.0, 2.0]]])
    bad = np.array([[[1.0, 1.0], [1.0, 1.0]]])           # singular; C_NN fine, A_PP = 0
    s = MspSolver(ptr, col, good, nc=1)
    rhs = torch.tensor([1.0, 2.0], dtype=torch.float64, device="cuda")
    assert s.solve(rhs, tol=1e-12)["final_rel"] <= 1e-12
    with pytest.raises(MspError):
        s.update(ptr, col, bad, iota=1, last_iterations=0, mu=0)
    with pytest.raises(MspError) as ei:
        s.solve(rhs)
    assert ei.value.status == 1
    assert s.update(ptr, col, good, iota=1, last_iterations=0, mu=0) is True
    assert s.solve(rhs, tol=1e-12)["final_rel"] <= 1e-12
