"""Pins of the CPU oracle against what the paper and mathematics fix.

No test here compares the oracle with itself or re-types its formula: each check
is a worked example (tests/golden, cited), a closed form, an invariant, a special
case that reduces to a textbook/library routine (numpy/scipy), or brute force.
"""
import json
import os

import numpy as np
import pytest
import scipy.linalg as sla
import scipy.sparse as sp

import gen
import oracle

GOLD = json.load(open(os.path.join(os.path.dirname(__file__), "golden", "spec_examples.json")))


def csr_of(A):
    M = sp.csr_matrix(np.asarray(A, dtype=float))
    M.sort_indices()
    return M.indptr.astype(np.int32), M.indices.astype(np.int32), M.data.astype(float)


def csr_struct(A):
    """CSR keeping explicit zeros of a dense pattern where A != 0 OR on the diagonal."""
    A = np.asarray(A, dtype=float)
    n = A.shape[0]
    ptr, col, val = [0], [], []
    for i in range(n):
        for j in range(n):
            if A[i, j] != 0 or i == j:
                col.append(j); val.append(A[i, j])
        ptr.append(len(col))
    return np.array(ptr, np.int32), np.array(col, np.int32), np.array(val)


def graph_of(n, edges):
    adj = [set() for _ in range(n)]
    for a, b in edges:
        adj[a].add(b); adj[b].add(a)
    ptr = [0]; col = []
    for i in range(n):
        col += sorted(adj[i]); ptr.append(len(col))
    return np.array(ptr, np.int32), np.array(col, np.int32)


def groups_of(g, color):
    return [sorted(np.flatnonzero(color == k).tolist()) for k in range(g)]


def bsr_dense(p):
    n, b = p["n"], p["b"]
    return sp.bsr_matrix((p["val"], p["col"], p["row_ptr"]), shape=(n * b, n * b)).toarray()


def rand_sparse(n, density, rng, diag=4.0, integer=False, sym_pattern=False):
    M = sp.random(n, n, density=density, random_state=rng).toarray()
    if integer:
        M = np.round(M * 8) - 0.0
    M[M != 0] -= 0.5 if not integer else 0
    if sym_pattern:
        M = M + M.T
    np.fill_diagonal(M, diag + np.abs(M).sum(1))
    return M


# ------------------------------------------------------------------ c-1 SpMV
def test_spmv_golden():
    e = GOLD["spmv_2x2"]
    A = np.array(e["A"], float).reshape(1, 2, 2)
    y = oracle.bsr_spmv(np.array([0, 1]), np.array([0]), A, np.array(e["x"], float))
    assert y.tolist() == e["y"]


def test_spmv_vs_dense_integer_exact():
    p = gen.make_config("C1")
    rng = np.random.default_rng(3)
    val = rng.integers(-9, 10, p["val"].shape).astype(float)
    x = gen.integer_vector(p["n"] * p["b"], 4)
    q = dict(p, val=val)
    y = oracle.bsr_spmv(p["row_ptr"], p["col"], val, x)
    assert np.array_equal(y, bsr_dense(q) @ x)          # integer sums are exact in FP64


def test_generator_manufactured_solution():
    """||A x* - b|| <= 1e-13 ||b|| (b is generated as A x*)."""
    for name, kw in (("C1", {}), ("C2", dict(nx=20, ny=20, nz=4))):
        p = gen.make_config(name, **kw)
        y = oracle.bsr_spmv(p["row_ptr"], p["col"], p["val"], p["xstar"])
        assert np.linalg.norm(y - p["rhs"]) <= 1e-13 * np.linalg.norm(p["rhs"])


# ------------------------------------------------------------------ c-3 adjacency
def test_adjacency_golden():
    for key in ("adjacency_tridiag", "adjacency_nonsym"):
        e = GOLD[key]
        ptr, col, val = csr_of(e["A"])
        gp, gc = oracle.csr_adjacency(ptr, col, val)
        edges = {(i, int(j)) for i in range(len(gp) - 1) for j in gc[gp[i]:gp[i + 1]] if i < j}
        assert edges == {tuple(x) for x in e["edges"]}
        if "degrees" in e:
            assert np.diff(gp).tolist() == e["degrees"]


def test_adjacency_by_value_symmetric_and_transpose_invariant():
    rng = np.random.default_rng(0)
    for _ in range(20):
        A = rand_sparse(30, 0.1, rng)
        A[0, 5] = -0.0                                     # explicit -0.0 is not an edge
        ptr, col, val = csr_struct(A)
        gp, gc = oracle.csr_adjacency(ptr, col, val)
        D = np.zeros_like(A, dtype=bool)
        for i in range(30):
            D[i, gc[gp[i]:gp[i + 1]]] = True
        ref = ((A != 0) | (A.T != 0)) & ~np.eye(30, dtype=bool)
        assert np.array_equal(D, ref)
        tp, tc, tv = csr_struct(A.T)
        gp2, gc2 = oracle.csr_adjacency(tp, tc, tv)
        assert np.array_equal(gp, gp2) and np.array_equal(gc, gc2)


# ------------------------------------------------------------------ c-4 coloring
def test_splitting_and_grouping_golden():
    e = GOLD["splitting_path"]
    gp, gc = graph_of(e["n"], e["edges"])
    W, Wb = oracle.splitting(gp, gc, np.arange(e["n"]))
    assert W.tolist() == e["W"] and Wb.tolist() == e["Wbar"]
    for key in ("grouping_path", "grouping_edgeless", "grouping_K3"):
        e = GOLD[key]
        gp, gc = graph_of(e["n"], e["edges"])
        g, color = oracle.grouping(gp, gc)
        if "groups" in e:
            assert groups_of(g, color) == e["groups"]
        else:
            assert g == e["ngroups"]


def test_grouping_complete_graph_n_colors():
    n = 7
    gp, gc = graph_of(n, [(i, j) for i in range(n) for j in range(i + 1, n)])
    g, color = oracle.grouping(gp, gc)
    assert g == n and sorted(color.tolist()) == list(range(n))


@pytest.mark.parametrize("shape", [(10, 10, 10), (3, 3, 3), (6, 22, 9), (8, 8, 1)])
def test_grouping_grid_closed_form(shape):
    """SURVEY c-4 closed form: full 7/5-point grids give g=2 and V_1 is the parity
    class of the lowest-index maximum-degree vertex (red-black)."""
    nx, ny, nz = shape
    n, ptr, col, val = gen.tpfa_laplacian_csr(nx, ny, nz)
    g, color = oracle.csr_grouping(ptr, col, val)
    deg = np.diff(ptr) - 1
    v0 = int(np.flatnonzero(deg == deg.max())[0])
    par = lambda c: (c % nx + (c // nx) % ny + c // (nx * ny)) % 2
    assert g == 2
    for c in range(n):
        assert (color[c] == 0) == (par(c) == par(v0))


def test_grouping_validity_random_200():
    """Principles (i)-(iii) by O(n^2) brute force; g <= Delta+1; determinism."""
    rng = np.random.default_rng(1)
    for t in range(200):
        n = int(rng.integers(1, 60))
        A = rand_sparse(n, float(rng.uniform(0.02, 0.3)), rng)
        ptr, col, val = csr_struct(A)
        g, color = oracle.csr_grouping(ptr, col, val)
        assert color.min() >= 0 and color.max() == g - 1                 # partition, no empty group
        S = ((A != 0) | (A.T != 0)) & ~np.eye(n, dtype=bool)
        for i in range(n):
            for j in range(n):
                if S[i, j]:
                    assert color[i] != color[j]                           # independence
        assert g <= S.sum(1).max(initial=0) + 1
        g2, color2 = oracle.csr_grouping(ptr, col, val)
        assert g2 == g and np.array_equal(color, color2)


def test_splitting_is_maximal_independent():
    """Each Alg. 2 result W is independent and maximal within V (greedy MIS, SURVEY c-4)."""
    rng = np.random.default_rng(5)
    for _ in range(50):
        n = 40
        A = rand_sparse(n, 0.08, rng)
        ptr, col, val = csr_struct(A)
        gp, gc = oracle.csr_adjacency(ptr, col, val)
        W, Wb = oracle.splitting(gp, gc, np.arange(n))
        Ws = set(W.tolist())
        assert sorted(W.tolist() + Wb.tolist()) == list(range(n))
        for v in range(n):
            nb = set(gc[gp[v]:gp[v + 1]].tolist())
            if v in Ws:
                assert not (nb & Ws)
            else:
                assert nb & Ws                                            # maximality


# ------------------------------------------------------------------ c-6 PGS-MC
def test_gs_golden():
    e = GOLD["gs_2x2"]
    ptr, col, val = csr_of(e["A"])
    color = np.zeros(2, np.int32)
    for k, grp in enumerate(e["groups"]):
        color[grp] = k
    x = oracle.pgs_mc(ptr, col, val, color, 2, np.array(e["b"], float), np.zeros(2))
    assert x.tolist() == e["x"]


def test_pgs_mc_equals_sequential_gs_in_color_order():
    """Paper claim P:23/P:434/P:491: PGS-MC == sequential GS in order V_1||...||V_g.
    Brute force: a plain sequential GS over that order, on integer data (exact)."""
    rng = np.random.default_rng(2)
    for _ in range(30):
        n = 25
        A = rand_sparse(n, 0.15, rng, integer=True)
        ptr, col, val = csr_struct(A)
        g, color = oracle.csr_grouping(ptr, col, val)
        b = rng.integers(-20, 20, n).astype(float)
        x0 = rng.integers(-5, 5, n).astype(float)
        for asc in (True, False):
            x = oracle.pgs_mc(ptr, col, val, color, g, b, x0, asc)
            order = [i for k in (range(g) if asc else range(g - 1, -1, -1))
                     for i in np.flatnonzero(color == k)]
            y = x0.copy()
            for i in order:
                s = sum(A[i, j] * y[j] for j in range(n) if j != i and A[i, j] != 0)
                y[i] = (b[i] - s) / A[i, i]
            assert np.allclose(x, y, rtol=1e-14, atol=0)


def test_pgs_mc_diagonal_exact_and_converges_to_solution():
    rng = np.random.default_rng(3)
    d = rng.uniform(1, 3, 10)
    ptr, col, val = csr_of(np.diag(d))
    b = rng.normal(size=10)
    x = oracle.pgs_mc(ptr, col, val, np.zeros(10, np.int32), 1, b, np.zeros(10))
    assert np.allclose(x, b / d, rtol=1e-15)
    n, ptr, col, val = gen.tpfa_laplacian_csr(6, 5, 1)
    A = sp.csr_matrix((val, col, ptr)).toarray()
    g, color = oracle.csr_grouping(ptr, col, val)
    b = rng.normal(size=n)
    xs = np.linalg.solve(A, b)
    x = np.zeros(n)
    errs = []
    for _ in range(400):
        x = oracle.pgs_mc(ptr, col, val, color, g, b, x)
        errs.append(np.linalg.norm(x - xs))
    assert errs[-1] < 1e-10 * np.linalg.norm(xs)
    assert all(errs[i + 1] <= errs[i] * (1 + 1e-12) for i in range(len(errs) - 1))


# ------------------------------------------------------------------ NEXT-4 smoothers (R13)
def test_jacobi_closed_form_modes_and_fixed_point():
    """PJAC-NO: on tridiag(-1, 2, -1) the sine modes are eigenvectors of the Jacobi
    iteration matrix D^-1 (L + U) with eigenvalue cos(k pi / (n + 1)) (textbook closed form);
    the exact solution is a fixed point."""
    n = 15
    ptr, col, val = csr_of(poisson1d(n))
    i = np.arange(1, n + 1)
    for k in (1, 4, 9, 15):
        v = np.sin(k * np.pi * i / (n + 1))
        x = oracle.jacobi_sweep(ptr, col, val, np.zeros(n), v)
        assert np.allclose(x, np.cos(k * np.pi / (n + 1)) * v, rtol=0, atol=1e-14)
        # K = 1: every coupling is to another chunk -> the same Jacobi mode factor
        x1 = oracle.hybrid_gs_sweep(ptr, col, val, 1, np.zeros(n), v)
        assert np.allclose(x1, np.cos(k * np.pi / (n + 1)) * v, rtol=0, atol=1e-14)
    rng = np.random.default_rng(5)
    A = rand_sparse(40, 0.1, rng)
    ptr, col, val = csr_of(A)
    b = rng.normal(size=40)
    xs = np.linalg.solve(A, b)
    assert np.allclose(oracle.jacobi_sweep(ptr, col, val, b, xs), xs, rtol=1e-12, atol=1e-13)


@pytest.mark.parametrize("K", [1, 3, 5, 8, 23, 100])
def test_hybrid_gs_is_chunkwise_triangular_solve(K):
    """PGS-NO (R13): one sweep is x' = M^-1 (b - (A - M) x) with M = D + the couplings to
    earlier rows of the same chunk (descending: later rows), i.e. a sparse triangular
    solve (scipy); K >= n is sequential natural-order forward / backward GS."""
    from scipy.sparse.linalg import spsolve_triangular
    rng = np.random.default_rng(11 + K)
    n = 23
    A = rand_sparse(n, 0.2, rng)
    ptr, col, val = csr_of(A)
    b, x0 = rng.normal(size=n), rng.normal(size=n)
    chunk = np.arange(n) // K
    same = chunk[:, None] == chunk[None, :]
    for asc in (True, False):
        tri = np.tril(A, -1) if asc else np.triu(A, 1)
        M = np.diag(np.diag(A)) + np.where(same, tri, 0.0)
        ref = spsolve_triangular(sp.csr_matrix(M), b - (A - M) @ x0, lower=asc)
        x = oracle.hybrid_gs_sweep(ptr, col, val, K, b, x0, asc)
        assert np.allclose(x, ref, rtol=1e-12, atol=1e-12)
        if K >= n:                                          # plain sequential GS
            ref2 = spsolve_triangular(sp.csr_matrix(np.tril(A) if asc else np.triu(A)),
                                      b - (np.triu(A, 1) if asc else np.tril(A, -1)) @ x0, lower=asc)
            assert np.allclose(x, ref2, rtol=1e-12, atol=1e-12)


def test_smoothers_in_msp_gmres_converge_and_order():
    """MSP-GMRES with each pressure smoother (Table 2 analog) reaches the
    tolerance (true residual), and on this generated problem the iteration counts keep
    the paper's order PGS-MC <= PGS-NO <= PJAC-NO (measured property, R13)."""
    p = gen.make_config("C2", nx=24, ny=20, nz=4)
    A = bsr_dense(p)
    its = {}
    for sm in (0, 2, 1):
        M = oracle.Msp(p["row_ptr"], p["col"], p["val"], coarsest_max_dof=50, smoother=sm)
        r = M.solve(p["rhs"], tol=1e-8)
        assert np.linalg.norm(p["rhs"] - A @ r["x"]) <= 1.01e-8 * np.linalg.norm(p["rhs"])
        its[sm] = r["iters"]
    assert its[0] <= its[2] <= its[1], its


# ------------------------------------------------------------------ c-5 NPAIR + Galerkin
def poisson1d(n):
    return np.diag(2.0 * np.ones(n)) - np.diag(np.ones(n - 1), 1) - np.diag(np.ones(n - 1), -1)


def test_npair_and_galerkin_golden():
    e = GOLD["npair_poisson4"]
    ptr, col, val = csr_of(e["A"])
    na, agg = oracle.npair(ptr, col, val)
    assert na == 2 and groups_of(na, agg) == e["aggregates"]
    cp, cc, cv = oracle.galerkin(ptr, col, val, agg, na)
    Ac = sp.csr_matrix((cv, cc, cp), shape=(2, 2)).toarray()
    assert Ac.tolist() == GOLD["galerkin_poisson4"]["Ac"]


def test_hierarchy_poisson16_sizes():
    A = poisson1d(16)
    ptr, col, val = csr_of(A)
    M = oracle.Msp(ptr, col, val.reshape(-1, 1, 1), coarsest_max_dof=4, pair_passes=1)
    info = M.info()
    sizes = [M.level_sizes(l)[0] for l in range(info["levels"] + 1)]
    assert sizes == GOLD["hierarchy_poisson16"]["sizes"]


def test_npair_partition_properties_random():
    rng = np.random.default_rng(4)
    for _ in range(100):
        n = int(rng.integers(2, 50))
        A = rand_sparse(n, 0.1, rng)
        ptr, col, val = csr_struct(A)
        na, agg = oracle.npair(ptr, col, val)
        S = ((A != 0) | (A.T != 0)) & ~np.eye(n, dtype=bool)
        assert sorted(set(agg.tolist())) == list(range(na))
        for I in range(na):
            m = np.flatnonzero(agg == I)
            assert 1 <= len(m) <= 2
            if len(m) == 2:
                assert S[m[0], m[1]]                      # pairs are graph edges
        # maximality: no two adjacent singletons remain unpaired... (greedy matching is maximal)
        singles = [int(np.flatnonzero(agg == I)[0]) for I in range(na) if (agg == I).sum() == 1]
        for a in singles:
            for c in singles:
                assert not S[a, c]


def test_npair_diagonal_singletons():
    ptr, col, val = csr_of(np.diag([1.0, 2.0, 3.0, 4.0]))
    na, agg = oracle.npair(ptr, col, val)
    assert na == 4 and sorted(agg.tolist()) == [0, 1, 2, 3]


def test_galerkin_equals_dense_PtAP_exact():
    rng = np.random.default_rng(6)
    for _ in range(50):
        n = 30
        A = rand_sparse(n, 0.15, rng, integer=True)
        ptr, col, val = csr_struct(A)
        na, agg = oracle.npair(ptr, col, val)
        P = np.zeros((n, na)); P[np.arange(n), agg] = 1
        cp, cc, cv = oracle.galerkin(ptr, col, val, agg, na)
        Ac = sp.csr_matrix((cv, cc, cp), shape=(na, na)).toarray()
        assert np.array_equal(Ac, P.T @ A @ P)
        assert np.array_equal(Ac.sum(1), P.T @ A.sum(1))             # row-sum identity


# ------------------------------------------------------------------ c-2 decoupling
def test_ti_weights_closed_form_on_generator():
    """SURVEY c-2: on the Eq.17/18 generator, C_NN = I/dt and C_0N = -alpha/dt, so y = alpha;
    A_PP row sums = alpha_P/dt; off-diagonals <= 0 (M-matrix)."""
    acc = 1e-2
    p = gen.make_config("C2", nx=12, ny=10, nz=4, acc=acc, with_alpha=True)
    M = oracle.Msp(p["row_ptr"], p["col"], p["val"], coarsest_max_dof=100000)
    W = M.weights()
    assert np.all(W[:, 0] == 1.0)
    eps = np.finfo(float).eps
    assert np.max(np.abs(W[:, 1:] - p["alpha"][:, 1:]) / p["alpha"][:, 1:]) <= 50 * eps / acc
    ptr, col, val = M.level_csr(0)
    n = p["n"]
    A = sp.csr_matrix((val, col, ptr), shape=(n, n)).toarray()
    rs = A.sum(1)
    ref = p["alpha"][:, 0] / p["dt"]
    scale = np.abs(A).sum(1)
    assert np.max(np.abs(rs - ref) / scale) <= 1e-12
    off = A - np.diag(np.diag(A))
    assert off.max() <= 1e-12 * np.abs(A).max()


def test_pressure_matrix_dense_WtAPi_and_none_golden():
    p = gen.make_config("C1", nx=3, ny=3, nz=3)
    n, b = p["n"], p["b"]
    Ad = bsr_dense(p)
    for mode in (0, 1, 2):
        M = oracle.Msp(p["row_ptr"], p["col"], p["val"], decoupling=mode)
        W = M.weights()
        Wt = np.zeros((n, n * b)); Pi = np.zeros((n * b, n))
        for c in range(n):
            Wt[c, c * b:(c + 1) * b] = W[c]
            Pi[c * b, c] = 1
        ptr, col, val = M.level_csr(0)
        App = sp.csr_matrix((val, col, ptr), shape=(n, n)).toarray()
        assert np.allclose(App, Wt @ Ad @ Pi, rtol=1e-13, atol=1e-13 * np.abs(Ad).max())
    # S:384 example (NONE): block-diagonal [[p,q],[r,s]] -> diag(p,p)
    e = GOLD["extract_pressure_blockdiag"]
    blk = np.array(e["block"], float)
    val = np.stack([blk, blk])
    M = oracle.Msp(np.array([0, 1, 2]), np.array([0, 1]), val, decoupling=0)
    ptr, col, v = M.level_csr(0)
    assert v.tolist() == e["App_diag"]


# ------------------------------------------------------------------ dense LU, V-cycle
def test_dense_lu_residual():
    rng = np.random.default_rng(7)
    A = rng.normal(size=(40, 40)) + 10 * np.eye(40)
    b = rng.normal(size=40)
    x = oracle.dense_lu_solve(A, b)
    assert np.linalg.norm(A @ x - b) <= 1e-12 * np.linalg.norm(b)
    assert np.allclose(x, sla.lu_solve(sla.lu_factor(A), b), rtol=1e-12)
    assert oracle.dense_lu_solve(np.diag([2.0, 4.0]), np.array([2.0, 4.0])).tolist() == [1.0, 1.0]


def scalar_msp(ptr, col, val, **kw):
    return oracle.Msp(ptr, col, np.asarray(val, float).reshape(-1, 1, 1), **kw)


def test_vcycle_single_level_exact_and_linear():
    n, ptr, col, val = gen.tpfa_laplacian_csr(8, 8, 1)
    A = sp.csr_matrix((val, col, ptr)).toarray()
    r = np.random.default_rng(8).normal(size=n)
    M = scalar_msp(ptr, col, val)                              # 64 <= 10000: direct only
    assert np.allclose(M.vcycle(r), np.linalg.solve(A, r), rtol=1e-12)
    M = scalar_msp(ptr, col, val, coarsest_max_dof=4)
    assert M.info()["levels"] >= 2
    v1, v2 = M.vcycle(r), M.vcycle(3.5 * r)
    assert np.allclose(v2, 3.5 * v1, rtol=1e-13, atol=1e-13 * np.abs(v2).max())


def test_vcycle_contraction_poisson32():
    """S:336 asks >= 2x error reduction per V-cycle on 2D Poisson 32^2.  That holds for a
    two-level UA-AMG cycle (1 pass, coarsest 256 rows); deep unsmoothed-aggregation
    V-cycles are known to contract more slowly (reading R11), so the deep
    hierarchy is pinned to a monotone contraction with rate < 0.8."""
    n, ptr, col, val = gen.tpfa_laplacian_csr(32, 32, 1)
    A = sp.csr_matrix((val, col, ptr))
    for kw, bound in ((dict(coarsest_max_dof=256, pair_passes=1), 0.5),
                      (dict(coarsest_max_dof=16, pair_passes=2), 0.8)):
        M = scalar_msp(ptr, col, val, **kw)
        rng = np.random.default_rng(9)
        xs = rng.normal(size=n)
        b = A @ xs
        x = np.zeros(n)
        e0 = np.linalg.norm(xs)
        for k in range(10):
            x = x + M.vcycle(b - A @ x)
            e1 = np.linalg.norm(x - xs)
            assert e1 <= bound * e0
            e0 = e1


# ------------------------------------------------------------------ c-9 BILU
def dense_blocks(n, b, ptr, col, val):
    return sp.bsr_matrix((val, col, ptr), shape=(n * b, n * b)).toarray()


def test_bilu_ilu0_pattern_property():
    """Defining property of ILU(0): in the elimination order, (L U)_ij = A_ij on every
    stored block (i,j) (L unit block-lower, U block-upper with D~ on the diagonal)."""
    for order_kind in (0, 1):
        p = gen.make_config("C2", nx=5, ny=4, nz=3, nc=2)
        n, b = p["n"], p["b"]
        M = oracle.Msp(p["row_ptr"], p["col"], p["val"], bilu_order=order_kind, coarsest_max_dof=8)
        F, Dinv = M.bilu_factors()
        order = M.order()
        pos = np.empty(n, int); pos[order] = np.arange(n)
        L = np.zeros((n * b, n * b)); U = np.zeros((n * b, n * b))
        for c in range(n):
            pc = pos[c]
            L[pc * b:(pc + 1) * b, pc * b:(pc + 1) * b] = np.eye(b)
            for e in range(p["row_ptr"][c], p["row_ptr"][c + 1]):
                d = p["col"][e]; pd = pos[d]
                blk = F[e]
                if pd < pc:
                    L[pc * b:(pc + 1) * b, pd * b:(pd + 1) * b] = blk
                elif pd > pc:
                    U[pc * b:(pc + 1) * b, pd * b:(pd + 1) * b] = blk
                else:
                    U[pc * b:(pc + 1) * b, pc * b:(pc + 1) * b] = np.linalg.inv(Dinv[c])
        LU = L @ U
        Ad = dense_blocks(n, b, p["row_ptr"], p["col"], p["val"])
        for c in range(n):
            for e in range(p["row_ptr"][c], p["row_ptr"][c + 1]):
                d = p["col"][e]
                blkA = Ad[c * b:(c + 1) * b, d * b:(d + 1) * b]
                blkLU = LU[pos[c] * b:(pos[c] + 1) * b, pos[d] * b:(pos[d] + 1) * b]
                assert np.allclose(blkLU, blkA, rtol=1e-11, atol=1e-11 * np.abs(blkA).max())
        # apply = (LU)^-1 r in the permuted ordering
        r = np.random.default_rng(1).normal(size=n * b)
        Pm = np.zeros((n * b, n * b))
        for c in range(n):
            Pm[pos[c] * b:(pos[c] + 1) * b, c * b:(c + 1) * b] = np.eye(b)
        ref = Pm.T @ np.linalg.solve(LU, Pm @ r)
        assert np.allclose(M.bilu_apply(r), ref, rtol=1e-10, atol=1e-12 * np.abs(ref).max())


def test_bilu_exact_on_block_diagonal_and_triangular():
    rng = np.random.default_rng(10)
    n, b = 6, 3
    # block diagonal: pattern is diagonal only
    val = rng.normal(size=(n, b, b)) + 4 * np.eye(b)
    ptr = np.arange(n + 1); col = np.arange(n)
    M = oracle.Msp(ptr, col, val, decoupling=0, coarsest_max_dof=100)
    r = rng.normal(size=n * b)
    Ad = dense_blocks(n, b, ptr, col, val)
    assert np.allclose(M.bilu_apply(r), np.linalg.solve(Ad, r), rtol=1e-12)


def test_bilu_rb_closed_form_black_pivot():
    """RB on a 2-color graph: D~_black = D_b - sum_k A_bk D_k^-1 A_kb (red pivots unchanged)."""
    p = gen.make_config("C1", nx=4, ny=3, nz=2, nc=1)
    n, b = p["n"], p["b"]
    M = oracle.Msp(p["row_ptr"], p["col"], p["val"], bilu_order=0)
    F, Dinv = M.bilu_factors()
    order = M.order()
    Ad = dense_blocks(n, b, p["row_ptr"], p["col"], p["val"])
    blk = lambda i, j: Ad[i * b:(i + 1) * b, j * b:(j + 1) * b]
    nred = n // 2
    red = set(order[:nred].tolist())
    for c in range(n):
        if c in red:
            ref = blk(c, c)
        else:
            ref = blk(c, c) - sum(blk(c, k) @ np.linalg.inv(blk(k, k)) @ blk(k, c)
                                  for k in p["col"][p["row_ptr"][c]:p["row_ptr"][c + 1]] if k != c)
        assert np.allclose(np.linalg.inv(Dinv[c]), ref, rtol=1e-11)


# ------------------------------------------------------------------ c-8 MSP
def test_msp_operator_identity_eq21():
    """Eq. 21 with stages PR: I - B A == (I - R A)(I - Pi_P B_P W^T A), assembled
    column by column from msp_apply, vcycle and bilu_apply, dim 12."""
    p = gen.make_config("C1", nx=3, ny=2, nz=1, nc=1)        # 6 cells, b=2 -> 12 unknowns
    n, b = p["n"], p["b"]
    N = n * b
    M = oracle.Msp(p["row_ptr"], p["col"], p["val"], coarsest_max_dof=2)
    assert M.info()["levels"] >= 1
    A = bsr_dense(p)
    W = M.weights()
    Wt = np.zeros((n, N)); Pi = np.zeros((N, n))
    for c in range(n):
        Wt[c, c * b:(c + 1) * b] = W[c]; Pi[c * b, c] = 1
    B = np.column_stack([M.apply(e) for e in np.eye(N)])
    R = np.column_stack([M.bilu_apply(e) for e in np.eye(N)])
    BP = np.column_stack([M.vcycle(e) for e in np.eye(n)])
    I = np.eye(N)
    lhs = I - B @ A
    rhs = (I - R @ A) @ (I - Pi @ BP @ Wt @ A)
    assert np.allclose(lhs, rhs, atol=1e-12 * max(1, np.abs(rhs).max()))
    assert np.array_equal(M.apply(np.zeros(N)), np.zeros(N))
    g1, g2 = np.random.default_rng(2).normal(size=(2, N))
    assert np.allclose(M.apply(2 * g1 - g2), 2 * M.apply(g1) - M.apply(g2), atol=1e-12)


def test_msp_operator_identity_eq21_three_stages():
    """Full Eq. 21 with stages NPR: I - BA == (I - RA)(I - Pi_P B_P W^T A)(I - Pi_N B_N Pi_N^T A)."""
    p = gen.make_config("C1", nx=2, ny=2, nz=1, nc=2)        # 4 cells, b=3 -> 12 unknowns
    n, b = p["n"], p["b"]
    N, nc = n * b, b - 1
    M = oracle.Msp(p["row_ptr"], p["col"], p["val"], coarsest_max_dof=2, stages=3)
    A = bsr_dense(p)
    W = M.weights()
    Wt = np.zeros((n, N)); Pi = np.zeros((N, n)); PiN = np.zeros((N, n * nc))
    for c in range(n):
        Wt[c, c * b:(c + 1) * b] = W[c]; Pi[c * b, c] = 1
        for i in range(nc):
            PiN[c * b + 1 + i, c * nc + i] = 1
    I = np.eye(N)
    B = np.column_stack([M.apply(e) for e in I])
    R = np.column_stack([M.bilu_apply(e) for e in I])
    BP = np.column_stack([M.vcycle(e) for e in np.eye(n)])
    BN = np.column_stack([M.bgs_apply(PiN @ e) for e in np.eye(n * nc)])   # B_N on Pi_N^T r
    rhs = (I - R @ A) @ (I - Pi @ BP @ Wt @ A) @ (I - PiN @ BN @ PiN.T @ A)
    assert np.allclose(I - B @ A, rhs, atol=1e-12 * max(1, np.abs(rhs).max()))


def test_bgs_is_block_forward_substitution_in_order():
    """B_N = one forward block GS sweep on A_NN from zero in the BILU order: equals the
    exact solve of the block-lower-triangular part (in that order) of A_NN (brute force)."""
    p = gen.make_config("C2", nx=4, ny=3, nz=2, nc=2)
    n, b = p["n"], p["b"]
    nc = b - 1
    M = oracle.Msp(p["row_ptr"], p["col"], p["val"], stages=3)
    order = M.order()
    pos = np.empty(n, int); pos[order] = np.arange(n)
    A = bsr_dense(p)
    idxN = [c * b + 1 + i for c in range(n) for i in range(nc)]
    ANN = A[np.ix_(idxN, idxN)]
    Lw = np.zeros_like(ANN)
    for c in range(n):
        for d in range(n):
            if pos[d] <= pos[c]:
                Lw[c * nc:(c + 1) * nc, d * nc:(d + 1) * nc] = ANN[c * nc:(c + 1) * nc, d * nc:(d + 1) * nc]
    r = np.random.default_rng(3).normal(size=n * b)
    ref = np.linalg.solve(Lw, r[idxN])
    assert np.allclose(M.bgs_apply(r), ref, rtol=1e-11, atol=1e-12 * np.abs(ref).max())


def test_msp_exact_on_one_cell():
    rng = np.random.default_rng(11)
    blk = rng.normal(size=(4, 4)) + 5 * np.eye(4)
    M = oracle.Msp(np.array([0, 1]), np.array([0]), blk.reshape(1, 4, 4))
    g = rng.normal(size=4)
    assert np.allclose(M.apply(g), np.linalg.solve(blk, g), rtol=1e-12)
    r = M.solve(g, tol=1e-10)
    assert r["iters"] == 1


# ------------------------------------------------------------------ c-11 GMRES
def test_gmres_golden_and_identity():
    e = GOLD["gmres_diag124"]
    ptr, col, val = csr_of(np.diag(e["diag"]))
    r = oracle.gmres_csr(ptr, col, val, np.array(e["b"], float), tol=1e-12)
    assert r["iters"] <= e["max_iters"] and np.allclose(r["x"], e["x"], rtol=1e-10)
    ptr, col, val = csr_of(np.eye(5))
    b = np.arange(1.0, 6.0)
    r = oracle.gmres_csr(ptr, col, val, b)
    assert r["iters"] == 1 and np.allclose(r["x"], b)
    r = oracle.gmres_csr(ptr, col, val, np.zeros(5))
    assert r["iters"] == 0 and np.all(r["x"] == 0)


def test_gmres_exact_preconditioner_one_iteration():
    rng = np.random.default_rng(12)
    A = rng.normal(size=(20, 20)) + 6 * np.eye(20)
    ptr, col, val = csr_of(A)
    r = oracle.gmres_csr(ptr, col, val, rng.normal(size=20), tol=1e-10, Minv=np.linalg.inv(A))
    assert r["iters"] == 1


@pytest.mark.parametrize("orth", [0, 1, 2])
def test_gmres_vs_scipy_random30(orth):
    """Same Krylov method as scipy's GMRES (restart 30, identity preconditioner):
    iteration counts agree within 1 and solutions match the dense solve."""
    import scipy.sparse.linalg as spla
    rng = np.random.default_rng(13)
    for t in range(5):
        A = rng.normal(size=(30, 30)) + 8 * np.eye(30)
        b = rng.normal(size=30)
        ptr, col, val = csr_of(A)
        r = oracle.gmres_csr(ptr, col, val, b, tol=1e-8, orth=orth)
        cnt = [0]
        spla.gmres(A, b, rtol=1e-8, restart=30, maxiter=50,
                   callback=lambda pr: cnt.__setitem__(0, cnt[0] + 1), callback_type="pr_norm")
        assert abs(r["iters"] - cnt[0]) <= 1
        assert np.allclose(r["x"], np.linalg.solve(A, b), rtol=1e-6)
        assert abs(r["final_rel"] - np.linalg.norm(b - A @ r["x"]) / np.linalg.norm(b)) <= 1e-12


@pytest.mark.parametrize("orth", [0, 1, 2])
def test_gmres_residuals_are_krylov_minima(orth):
    """Brute force: the k-th GMRES residual estimate equals min over x in K_k(A, b) of
    ||b - A x|| / ||b|| (numpy least squares on a QR basis of [b, Ab, ...]); identity
    preconditioner, no restart.  Checks CGS2, MGS and DCGS2 (R14) Arnoldi alike, including
    the DCGS2 Hessenberg correction and its one-step-delayed reorthogonalisation."""
    rng = np.random.default_rng(21)
    n = 40
    A = rng.normal(size=(n, n)) / np.sqrt(n) + 1.5 * np.eye(n)
    b = rng.normal(size=n)
    ptr, col, val = csr_of(A)
    r = oracle.gmres_csr(ptr, col, val, b, tol=1e-13, m=40, maxit=40, orth=orth)
    Q = (b / np.linalg.norm(b))[:, None]                  # orthonormal basis of K_k (Householder QR)
    for k in range(1, 16):
        y, *_ = np.linalg.lstsq(A @ Q, b, rcond=None)
        ref = np.linalg.norm(b - A @ Q @ y) / np.linalg.norm(b)
        assert abs(r["hist"][k - 1] - ref) <= 1e-9 * ref + 1e-15, (k, r["hist"][k - 1], ref)
        Q, _ = np.linalg.qr(np.column_stack([Q, A @ Q[:, -1]]))


@pytest.mark.parametrize("orth", [0, 1, 2])
def test_gmres_terminates_at_minimal_polynomial_degree(orth):
    """Closed form (Krylov theory): unrestarted GMRES reaches the exact solution in
    exactly deg(minimal polynomial of A w.r.t. b) steps.  (1) A = S diag(λ) S⁻¹, nonsymmetric,
    with 4 distinct eigenvalues of multiplicity 5 each (n = 20): 4 iterations. (2) A Jordan
    block I + N (N the upper shift) with b = e_n: the Krylov space grows one unit vector per
    step, so exactly n iterations; before that the k-th relative residual is 1/sqrt(k+1):
    A K_k ⊂ span(e_{n-k}..e_n), whose unit vector orthogonal to A K_k is the alternating
    (±1, ..., ±1)/sqrt(k+1) (w_j + w_{j-1} = 0), and its e_n component is the residual."""
    rng = np.random.default_rng(31)
    n = 20
    S = rng.normal(size=(n, n)) + 4 * np.eye(n)
    lam = np.repeat([1.0, 2.0, 3.5, 5.0], 5)
    A = S @ np.diag(lam) @ np.linalg.inv(S)
    b = rng.normal(size=n)
    ptr, col, val = csr_of(A)
    r = oracle.gmres_csr(ptr, col, val, b, tol=1e-9, m=n, maxit=n, orth=orth)
    assert r["iters"] == 4, r["iters"]
    assert np.allclose(r["x"], np.linalg.solve(A, b), rtol=1e-7)
    n = 8
    J = np.eye(n) + np.eye(n, k=1)
    e = np.zeros(n)
    e[-1] = 1.0
    ptr, col, val = csr_of(J)
    r = oracle.gmres_csr(ptr, col, val, e, tol=1e-12, m=n, maxit=n, orth=orth)
    assert r["iters"] == n, r["iters"]
    assert np.allclose(r["x"], np.linalg.solve(J, e), rtol=1e-10)
    for k in range(1, n):
        assert abs(r["hist"][k - 1] - 1 / np.sqrt(k + 1)) <= 1e-12, (k, r["hist"][k - 1])


@pytest.mark.parametrize("m", [5, 30])
def test_dcgs2_restarted_matches_cgs2(m):
    """DCGS2 (R14) computes the same Arnoldi basis as CGS2 in exact arithmetic: with
    restarts, MSP preconditioning and a nonsymmetric system its residual history agrees
    with the (scipy-pinned) CGS2 history to rounding level."""
    p = gen.make_config("C2", nx=12, ny=10, nz=3)
    out = []
    for orth in (0, 2):
        M = oracle.Msp(p["row_ptr"], p["col"], p["val"], orth=orth, coarsest_max_dof=40)
        out.append(M.solve(p["rhs"], tol=1e-10, restart=m))
    assert out[0]["iters"] == out[1]["iters"]
    h0, h1 = out[0]["hist"], out[1]["hist"]
    assert len(h0) == len(h1)
    # rounding differences, amplified through restarts: relative 1e-7 plus 1e-13 of ||b||
    assert np.all(np.abs(h0 - h1) <= 1e-7 * h0 + 1e-13)
    k = min(m, out[0]["iters"])                                      # first-cycle estimates
    assert np.max(np.abs(h0[:k] - h1[:k]) / h0[:k]) <= 1e-10
    assert np.linalg.norm(out[0]["x"] - out[1]["x"]) <= 1e-8 * np.linalg.norm(out[0]["x"])


def test_msp_gmres_3cube_vs_dense_lu():
    """3^3 cells, b=4 (N=108): MSP-GMRES solution vs dense LU (cond * tol bound) and to
    1e-10 at tol 1e-14; reported residual equals the recomputed one."""
    p = gen.make_config("C2", nx=3, ny=3, nz=3)
    A = bsr_dense(p)
    xs = np.linalg.solve(A, p["rhs"])
    for kw in (dict(), dict(coarsest_max_dof=4), dict(coarsest_max_dof=4, bilu_order=0),
               dict(stages=3)):
        M = oracle.Msp(p["row_ptr"], p["col"], p["val"], **kw)
        r = M.solve(p["rhs"], tol=1e-14, maxit=300)
        assert np.linalg.norm(r["x"] - xs) <= 1e-10 * np.linalg.norm(xs)
        r = M.solve(p["rhs"], tol=1e-6)
        true = np.linalg.norm(p["rhs"] - A @ r["x"]) / np.linalg.norm(p["rhs"])
        assert true <= 1e-6 and abs(true - r["final_rel"]) <= 1e-12
        cond = np.linalg.cond(A)
        assert np.linalg.norm(r["x"] - xs) <= cond * 1e-6 * np.linalg.norm(xs)


def test_cgs2_and_mgs_same_iterations_C1():
    p = gen.make_config("C1")
    its = []
    for orth in (0, 1, 2):
        M = oracle.Msp(p["row_ptr"], p["col"], p["val"], orth=orth, coarsest_max_dof=50)
        its.append(M.solve(p["rhs"])["iters"])
    assert abs(its[0] - its[1]) <= 1 and abs(its[0] - its[2]) <= 1


# ------------------------------------------------------------------ c-12 ASMSP
def test_asmsp_decisions_golden():
    for c in GOLD["asmsp"]["cases"]:
        assert oracle.asmsp_decide(c["iota"], c["last_it"], c["mu"], c["dims_changed"]) == c["setup"]


# ------------------------------------------------------------------ round 2 pins
# c-9 (R5): the ABMC ordering itself, the forward/backward halves of Alg. 1 line 6, and the
# "parallel by color" equivalence.
ABMC_CASES = [("C2", dict(nx=9, ny=7, nz=4), dict()),
              ("C2", dict(nx=9, ny=7, nz=4), dict(pair_passes=1)),
              ("C2", dict(nx=9, ny=7, nz=4), dict(bilu_order=0)),
              ("C2", dict(nx=6, ny=5, nz=4, nc=2), dict(decoupling=1)),
              ("C1", dict(nx=6, ny=5, nz=3), dict(decoupling=0)),      # A_PP diagonal: cell Laplacian
              ("C3", dict(nx=6, ny=11, nz=6), dict())]


def block_nonzero(p):
    """Z[c, d] = block (c, d) stored with a nonzero entry (c != d), dense n x n."""
    n = p["n"]
    Z = np.zeros((n, n), bool)
    for c in range(n):
        for e in range(p["row_ptr"][c], p["row_ptr"][c + 1]):
            d = p["col"][e]
            if d != c and np.any(p["val"][e] != 0):
                Z[c, d] = True
    return Z | Z.T


@pytest.mark.parametrize("name,gkw,kw", ABMC_CASES)
def test_abmc_order_validity_bruteforce(name, gkw, kw):
    """P:332-334 principles for the block coloring of R5, by O(n^2) brute force over all
    cell pairs: (i) two cells of DIFFERENT blocks of the SAME color are never coupled;
    (ii) every block of color c > 0 is coupled to some block of every earlier color (each
    color class is a maximal independent set of the blocks left, Alg. 2); the order is
    (color, block, cell) ascending; blocks are connected in the cell graph with <= 2^passes
    cells."""
    p = gen.make_config(name, **gkw)
    n = p["n"]
    M = oracle.Msp(p["row_ptr"], p["col"], p["val"], coarsest_max_dof=30, **kw)
    g, color, blk = M.bilu_blocks()
    Z = block_nonzero(p)
    same_color = color[:, None] == color[None, :]
    diff_blk = blk[:, None] != blk[None, :]
    assert not np.any(Z & same_color & diff_blk)
    # maximality: block I of color c touches a block of every color c' < c
    nb = blk.max() + 1
    bcol = np.zeros(nb, int)
    bcol[blk] = color
    Q = np.zeros((nb, nb), bool)
    cc, dd = np.nonzero(Z)
    Q[blk[cc], blk[dd]] = True
    np.fill_diagonal(Q, False)
    for I in range(nb):
        seen = set(bcol[np.flatnonzero(Q[I])].tolist())
        assert all(c in seen for c in range(bcol[I])), I
    order = M.order()
    key = sorted(range(n), key=lambda c: (color[c], blk[c], c))
    assert order.tolist() == key
    passes = kw.get("pair_passes", 2)
    for I in range(nb):
        m = np.flatnonzero(blk == I)
        assert 1 <= len(m) <= (1 if kw.get("bilu_order", 1) == 0 else 2 ** passes)
        # connected inside the cell graph
        reach = {m[0]}
        stack = [m[0]]
        while stack:
            a = stack.pop()
            for c in m:
                if c not in reach and Z[a, c]:
                    reach.add(c); stack.append(c)
        assert len(reach) == len(m)
    assert g == color.max() + 1


@pytest.mark.parametrize("name,gkw,kw", ABMC_CASES)
def test_bilu_parallel_by_color_equals_sequential(name, gkw, kw):
    """Sequential-equivalent parallelism for the block smoother: the BILU
    substitutions executed color by color (other blocks read from the snapshot before the
    color phase) equal the sequential substitutions in the elimination order BIT FOR BIT."""
    p = gen.make_config(name, **gkw)
    M = oracle.Msp(p["row_ptr"], p["col"], p["val"], coarsest_max_dof=30, **kw)
    r = gen.random_vector(p["n"] * p["b"], 5)
    assert np.array_equal(M.bilu_apply_by_color(r), M.bilu_apply(r))


def test_bilu_coupled_cells_get_distinct_colors():
    """Two coupled cells (RB): distinct colors, and the by-color substitution equals the
    sequential one."""
    rng = np.random.default_rng(2)
    n, b = 2, 2
    ptr = np.array([0, 2, 4]); col = np.array([0, 1, 0, 1])
    val = rng.normal(size=(4, b, b)) + 5 * np.eye(b)
    M = oracle.Msp(ptr, col, val, decoupling=0, bilu_order=0, coarsest_max_dof=100)
    g, color, blk = M.bilu_blocks()
    assert g == 2 and color[0] != color[1]             # coupled cells get different colors
    r = rng.normal(size=n * b)
    assert np.array_equal(M.bilu_apply_by_color(r), M.bilu_apply(r))


def _lu_dense(M, p):
    n, b = p["n"], p["b"]
    F, Dinv = M.bilu_factors()
    order = M.order()
    pos = np.empty(n, int); pos[order] = np.arange(n)
    L = np.eye(n * b); U = np.zeros((n * b, n * b))
    for c in range(n):
        for e in range(p["row_ptr"][c], p["row_ptr"][c + 1]):
            d = p["col"][e]
            sl = (slice(c * b, (c + 1) * b), slice(d * b, (d + 1) * b))
            if pos[d] < pos[c]:
                L[sl] = F[e]
            elif pos[d] > pos[c]:
                U[sl] = F[e]
            else:
                U[sl] = np.linalg.inv(Dinv[c])
    return L, U


@pytest.mark.parametrize("kw", [dict(), dict(bilu_order=0)])
def test_bilu_forward_backward_are_triangular_solves(kw):
    """Alg. 1 line 6 split in its two halves (R5): forward = (unit block-lower L)^-1 r,
    backward = (block-upper U incl. D~)^-1 y, against dense scipy triangular solves in
    natural numbering (L, U permuted by the elimination order); the abs-mode recurrences
    bound |L^-1 r| and |U^-1 y| componentwise."""
    p = gen.make_config("C2", nx=6, ny=5, nz=3, nc=2)
    M = oracle.Msp(p["row_ptr"], p["col"], p["val"], coarsest_max_dof=20, **kw)
    L, U = _lu_dense(M, p)
    r = gen.random_vector(p["n"] * p["b"], 8)
    y = M.bilu_forward(r)
    yref = np.linalg.solve(L, r)
    assert np.max(np.abs(y - yref)) <= 1e-12 * np.max(np.abs(yref))
    x = M.bilu_backward(y)
    xref = np.linalg.solve(U, y)
    assert np.max(np.abs(x - xref)) <= 1e-11 * np.max(np.abs(xref))
    assert np.array_equal(M.bilu_backward(M.bilu_forward(r)), M.bilu_apply(r))
    ya = M.bilu_forward(r, absmode=True)
    assert np.all(ya >= np.abs(y) * (1 - 1e-14))
    xa = M.bilu_backward(ya, absmode=True)
    assert np.all(xa >= np.abs(x) * (1 - 1e-14))


def test_vcycle_transfers_dense():
    """a5 / a7 (P:459 UA-AMG): residual + restriction = P^T (b - A_l x) and
    prolongation + correction = x + P e, against dense products with P from the aggregates."""
    p = gen.make_config("C2", nx=12, ny=10, nz=3)
    M = oracle.Msp(p["row_ptr"], p["col"], p["val"], coarsest_max_dof=40)
    L = M.info()["levels"]
    assert L >= 2
    for l in range(L):
        ptr, col, val = M.level_csr(l)
        n = len(ptr) - 1
        A = sp.csr_matrix((val, col, ptr), shape=(n, n)).toarray()
        nn, agg = M.level_agg(l)
        P = np.zeros((n, nn)); P[np.arange(n), agg] = 1
        b = gen.random_vector(n, 30 + l); x = gen.random_vector(n, 40 + l)
        bc = M.residual_restrict(l, b, x)
        ref = P.T @ (b - A @ x)
        assert np.max(np.abs(bc - ref)) <= 1e-12 * (P.T @ (np.abs(b) + np.abs(A) @ np.abs(x))).max()
        e = gen.random_vector(nn, 50 + l)
        assert np.array_equal(M.prolong(l, e, x), x + P @ e)
        # integer inputs: exact
        bi = gen.integer_vector(n, 60 + l); xi = gen.integer_vector(n, 70 + l)
        Ai = np.round(A)
        if np.array_equal(Ai, A):
            assert np.array_equal(M.residual_restrict(l, bi, xi), P.T @ (bi - A @ xi))


def test_restrict_pressure_dense_and_dots():
    """a3: r_p = W^T g (R4) against the dense block-row product of the weights; a10 dots
    against numpy."""
    p = gen.make_config("C1", nx=4, ny=3, nz=2)
    n, b = p["n"], p["b"]
    for mode in (0, 1, 2):
        M = oracle.Msp(p["row_ptr"], p["col"], p["val"], decoupling=mode)
        W = M.weights()
        Wt = np.zeros((n, n * b))
        for c in range(n):
            Wt[c, c * b:(c + 1) * b] = W[c]
        g = gen.random_vector(n * b, 3)
        rp = M.restrict_pressure(g)
        assert np.max(np.abs(rp - Wt @ g)) <= 1e-14 * (np.abs(Wt) @ np.abs(g)).max()
        if mode == 0:
            assert np.array_equal(rp, g[0::b])               # NONE: the pressure slots
    rng = np.random.default_rng(0)
    V = rng.normal(size=(7, 1001)); w = rng.normal(size=1001)
    assert np.allclose(oracle.dots(V, w), V @ w, rtol=1e-13, atol=1e-13)
    Vi = rng.integers(-20, 20, size=(5, 333)).astype(float); wi = rng.integers(-20, 20, size=333).astype(float)
    assert np.array_equal(oracle.dots(Vi, wi), Vi @ wi)


def test_qi_weights_closed_form():
    """R4 QI: w_c = [1, y], D_NN^T y = -D_0N^T with D the diagonal block.  Diagonal blocks
    built with D_NN = d I and D_0N = -d a (d a power of two) give y = a exactly; on random
    blocks the defining equation holds to rounding (numpy solve of each nc x nc system)."""
    p = gen.make_config("C2", nx=5, ny=4, nz=3)
    n, b = p["n"], p["b"]
    rng = np.random.default_rng(12)
    val = p["val"].copy()
    alpha = rng.uniform(0.5, 1.5, size=(n, b - 1))
    for c in range(n):
        for e in range(p["row_ptr"][c], p["row_ptr"][c + 1]):
            if p["col"][e] == c:
                d = 2.0 ** int(rng.integers(-4, 8))
                val[e, 1:, 1:] = d * np.eye(b - 1)
                val[e, 0, 1:] = -d * alpha[c]
    M = oracle.Msp(p["row_ptr"], p["col"], val, decoupling=1, coarsest_max_dof=100000)
    W = M.weights()
    assert np.all(W[:, 0] == 1.0) and np.array_equal(W[:, 1:], alpha)
    M2 = oracle.Msp(p["row_ptr"], p["col"], p["val"], decoupling=1, coarsest_max_dof=100000)
    W2 = M2.weights()
    for c in range(n):
        e = [e for e in range(p["row_ptr"][c], p["row_ptr"][c + 1]) if p["col"][e] == c][0]
        D = p["val"][e]
        y = np.linalg.solve(D[1:, 1:].T, -D[0, 1:])
        assert np.allclose(W2[c, 1:], y, rtol=1e-12, atol=1e-14)


@pytest.mark.parametrize("passes,expect", [(1, [[0, 1], [2, 3]]), (2, [[0, 1, 2, 3]])])
def test_none_decoupling_cell_laplacian_blocks_chain(passes, expect):
    """R5 with NONE decoupling on the Eq. 17 generator (A_PP diagonal): the ABMC blocks are
    the NPAIR aggregates of the cell-graph Laplacian.  On a 4-cell chain the Laplacian is
    [[1,-1],[-1,2,-1],[-1,2,-1],[-1,1]]: pass 1 pairs (0,1) (fewest neighbours, lowest
    index) then (2,3); its Galerkin matrix [[1,-1],[-1,1]] pairs the two in pass 2."""
    p = gen.make_config("C1", nx=4, ny=1, nz=1)
    M = oracle.Msp(p["row_ptr"], p["col"], p["val"], decoupling=0, pair_passes=passes)
    assert M.info()["coarse_diag"] or M.info()["levels"] == 0
    ptr, col, val = M.level_csr(0)
    A = sp.csr_matrix((val, col, ptr), shape=(4, 4)).toarray()
    assert np.count_nonzero(A - np.diag(np.diag(A))) == 0          # A_PP diagonal (Eq. 17)
    g, color, blk = M.bilu_blocks()
    assert groups_of(blk.max() + 1, blk) == expect


def test_stall_and_max_levels_give_estall():
    """R11 stop rules ("coarsest ... 10000"): coarsening that keeps > 0.9 n on
    a non-diagonal level -> MSP_ESTALL (5); reaching max_levels above coarsest_max_dof ->
    MSP_ESTALL; a diagonal stalled level becomes the (exact, diagonal) coarsest."""
    n = 100
    A = np.diag(4.0 * np.ones(n))
    A[0, 1] = A[1, 0] = -1.0                                 # one coupling: 99 aggregates
    ptr, col, val = csr_of(A)
    with pytest.raises(oracle.OracleError) as ei:
        scalar_msp(ptr, col, val, coarsest_max_dof=10)
    assert "(5)" in str(ei.value)
    ptr, col, val = csr_of(poisson1d(64))
    with pytest.raises(oracle.OracleError) as ei:
        scalar_msp(ptr, col, val, coarsest_max_dof=1, max_levels=3)
    assert "(5)" in str(ei.value)
    ptr, col, val = csr_of(np.diag(np.arange(1.0, n + 1)))
    M = scalar_msp(ptr, col, val, coarsest_max_dof=10)
    assert M.info()["coarse_diag"]
    r = gen.random_vector(n, 1)
    assert np.allclose(M.vcycle(r), r / np.arange(1.0, n + 1), rtol=1e-15)


def test_omp_mode_bit_identical():
    """the oracle's OpenMP switch is for timing only -- a full MSP-GMRES
    solve (PGS-MC, ABMC BILU, CGS2) gives bit-identical iterates with 1 and 4 threads."""
    p = gen.make_config("C2", nx=24, ny=20, nz=5)
    out = []
    try:
        for t in (1, 4):
            assert oracle.set_threads(t) == t
            M = oracle.Msp(p["row_ptr"], p["col"], p["val"], coarsest_max_dof=60)
            r = M.solve(p["rhs"], tol=1e-8)
            out.append((r["iters"], r["hist"], r["x"]))
    finally:
        oracle.set_threads(1)
    assert out[0][0] == out[1][0]
    assert np.array_equal(out[0][1], out[1][1])
    assert np.array_equal(out[0][2], out[1][2])
