"""Per-kernel GPU parity (SURVEY §8(c)-15 "FP64 kernels <= 1e-12 per SpMV or sweep"): every
single step of the hot path, run through its own C-ABI entry point with the SAME kernel the
solve runs, against the oracle's step on identical inputs.

Pass rule (componentwise, relative to the magnitude of what is summed):
    |y_gpu - y_oracle|_i <= 1e-12 * bound_i
with bound = (|A||x| + |b|) for products and residuals, the abs-mode recurrences of the
oracle for the triangular substitutions of a9 (applied twice: the growth of rounding
errors through the recurrence), and sum |v||w| for the a10 dots; plus
the normwise ||dy|| <= 1e-12 ||y|| where no cancellation makes it meaningless.  Integer-
valued inputs are bit-exact (a4 with a power-of-two diagonal, a8, a9 with integer
factors).
"""
import numpy as np
import pytest
import scipy.sparse as sp

import gen
import oracle

pytestmark = pytest.mark.gpu

torch = pytest.importorskip("torch")

TOL = 1e-12


def solver(p, **kw):
    from paper_2208_08594_b200 import MspSolver
    return MspSolver(p["row_ptr"], p["col"], p["val"], nc=p["nc"], **kw)


def dev(a):
    return torch.from_numpy(np.ascontiguousarray(a)).cuda()


def check(y, ref, bound, normwise=True):
    y = np.asarray(y)
    assert np.all(np.abs(y - ref) <= TOL * bound + 1e-300), np.max(np.abs(y - ref) / (bound + 1e-300))
    if normwise:
        assert np.linalg.norm(y - ref) <= TOL * np.linalg.norm(ref), np.linalg.norm(y - ref) / np.linalg.norm(ref)


CASES = [("C2", dict(nx=25, ny=20, nz=5), dict()),
         ("C2", dict(nx=25, ny=20, nz=5), dict(decoupling=1)),
         ("C2", dict(nx=25, ny=20, nz=5), dict(decoupling=0)),
         ("C2", dict(nx=25, ny=20, nz=5), dict(bilu_order=0)),
         ("C2", dict(nx=12, ny=10, nz=4, nc=6), dict()),
         ("C3", dict(nx=12, ny=44, nz=17), dict()),
         ("C2", dict(nx=13, ny=11, nz=3, nc=2), dict(pair_passes=1))]


# ------------------------------------------------------------------ a3
@pytest.mark.parametrize("name,gkw,kw", CASES)
def test_a3_restrict_pressure(name, gkw, kw):
    p = gen.make_config(name, **gkw)
    s = solver(p, coarsest_max_dof=100, **kw)
    O = oracle.Msp(p["row_ptr"], p["col"], p["val"], coarsest_max_dof=100, **kw)
    g = gen.random_vector(p["n"] * p["b"], 3)
    ref = O.restrict_pressure(g)
    out = torch.zeros(p["n"], dtype=torch.float64, device="cuda")
    s.restrict_pressure(dev(g), out)
    W = O.weights()
    bound = (np.abs(W) * np.abs(g.reshape(-1, p["b"]))).sum(1)
    check(out.cpu().numpy(), ref, bound, normwise=False)


# ------------------------------------------------------------------ a5, a7
@pytest.mark.parametrize("name,gkw,kw", CASES[:1] + CASES[4:6])
def test_a5_residual_restrict_and_a7_prolong_every_level(name, gkw, kw):
    p = gen.make_config(name, **gkw)
    s = solver(p, coarsest_max_dof=60, **kw)
    O = oracle.Msp(p["row_ptr"], p["col"], p["val"], coarsest_max_dof=60, **kw)
    L = O.info()["levels"]
    assert L >= 2
    for l in range(L):
        ptr, col, val = O.level_csr(l)
        n = len(ptr) - 1
        A = sp.csr_matrix((val, col, ptr), shape=(n, n))
        nn, agg = O.level_agg(l)
        b = gen.random_vector(n, 10 + l)
        x = gen.random_vector(n, 20 + l)
        ref = O.residual_restrict(l, b, x)
        out = torch.zeros(nn, dtype=torch.float64, device="cuda")
        s.residual_restrict(l, dev(b), dev(x), out)
        P = sp.csr_matrix((np.ones(n), (np.arange(n), agg)), shape=(n, nn))
        bound = P.T @ (np.abs(b) + abs(A) @ np.abs(x))
        check(out.cpu().numpy(), ref, bound, normwise=False)
        e = gen.random_vector(nn, 30 + l)
        xd = dev(x.copy())
        s.prolong(l, dev(e), xd)
        assert np.array_equal(xd.cpu().numpy(), O.prolong(l, e, x))          # one add: exact


# ------------------------------------------------------------------ a8
@pytest.mark.parametrize("name,gkw,kw", CASES)
def test_a8_pcol_residual(name, gkw, kw):
    p = gen.make_config(name, **gkw)
    s = solver(p, coarsest_max_dof=100, **kw)
    n, b = p["n"], p["b"]
    g = gen.random_vector(n * b, 4)
    xp = gen.random_vector(n, 5)
    w = np.zeros(n * b)
    w[0::b] = xp                                                    # Pi_P x_p
    ref = g - oracle.bsr_spmv(p["row_ptr"], p["col"], p["val"], w)     # Alg. 1 line 5
    out = torch.zeros(n * b, dtype=torch.float64, device="cuda")
    s.pcol_residual(dev(g), dev(xp), out)
    bound = np.abs(g) + oracle.bsr_spmv(p["row_ptr"], p["col"], np.abs(p["val"]), np.abs(w))
    check(out.cpu().numpy(), ref, bound, normwise=False)


@pytest.mark.parametrize("ell", ["1", "0"])
def test_a8_both_layouts(monkeypatch, ell):
    """a8 through the ELL copy of the pressure columns (default for 4x4 blocks, rows of
    <= 8 blocks) and through the BSR layout (MSP_A8_ELL=0; the kernel rows wider than 8
    blocks use): same componentwise bound against the oracle's Alg. 1 line 5."""
    monkeypatch.setenv("MSP_A8_ELL", ell)
    p = gen.make_config("C3", nx=21, ny=44, nz=9)
    s = solver(p, coarsest_max_dof=100)
    n, b = p["n"], p["b"]
    g = gen.random_vector(n * b, 14)
    xp = gen.random_vector(n, 15)
    w = np.zeros(n * b)
    w[0::b] = xp
    ref = g - oracle.bsr_spmv(p["row_ptr"], p["col"], p["val"], w)
    out = torch.zeros(n * b, dtype=torch.float64, device="cuda")
    s.pcol_residual(dev(g), dev(xp), out)
    bound = np.abs(g) + oracle.bsr_spmv(p["row_ptr"], p["col"], np.abs(p["val"]), np.abs(w))
    check(out.cpu().numpy(), ref, bound, normwise=False)


# ------------------------------------------------------------------ a9 halves
@pytest.mark.parametrize("name,gkw,kw", CASES)
def test_a9_bilu_forward_and_backward(name, gkw, kw):
    p = gen.make_config(name, **gkw)
    s = solver(p, coarsest_max_dof=100, **kw)
    O = oracle.Msp(p["row_ptr"], p["col"], p["val"], coarsest_max_dof=100, **kw)
    N = p["n"] * p["b"]
    r = gen.random_vector(N, 6)
    yref = O.bilu_forward(r)
    y = torch.zeros(N, dtype=torch.float64, device="cuda")
    s.bilu_forward(dev(r), y)
    bound_f = O.bilu_forward(O.bilu_forward(r, absmode=True), absmode=True)
    check(y.cpu().numpy(), yref, bound_f)
    xref = O.bilu_backward(yref)                                   # identical input y
    x = torch.zeros(N, dtype=torch.float64, device="cuda")
    s.bilu_backward(dev(yref), x)
    bound_b = O.bilu_backward(O.bilu_backward(yref, absmode=True), absmode=True)
    check(x.cpu().numpy(), xref, bound_b)


# ------------------------------------------------------------------ a10
def test_a10_multidot():
    p = gen.make_config("C1")
    s = solver(p)
    rng = np.random.default_rng(0)
    N = p["n"] * p["b"]                 # the kernel strides vectors by the handle's n*b
    for k in (1, 3, 4, 8, 13, 16, 17, 25, 32):
        V = rng.normal(size=(k, N))
        w = rng.normal(size=N)
        ref = oracle.dots(V, w)
        out = s.multidot(dev(V), dev(w))
        bound = np.abs(V) @ np.abs(w)
        check(out, ref, bound, normwise=False)
        Vi = rng.integers(-1000, 1000, size=(k, N)).astype(float)
        wi = rng.integers(-1000, 1000, size=N).astype(float)
        assert np.array_equal(s.multidot(dev(Vi), dev(wi)), oracle.dots(Vi, wi))


@pytest.mark.parametrize("dims", [(13, 11, 3), (20, 20, 10)])
def test_a10_multidot_sizes(dims):
    """Odd and large vector lengths (8-byte vs 16-byte kernel paths, many CTAs)."""
    p = gen.make_config("C2", nx=dims[0], ny=dims[1], nz=dims[2], nc=2)
    s = solver(p, coarsest_max_dof=100)
    N = p["n"] * p["b"]
    rng = np.random.default_rng(1)
    for k in (2, 16, 30):
        V = rng.normal(size=(k, N)); w = rng.normal(size=N)
        check(s.multidot(dev(V), dev(w)), oracle.dots(V, w), np.abs(V) @ np.abs(w), normwise=False)


# ------------------------------------------------------------------ integer bit-exact
def integer_system(nx, ny, nz, seed, diag=64.0):
    """Integer BSR on a 7-point grid with a power-of-two pressure diagonal: A_PP (NONE
    decoupling) has integer off-diagonals and diagonal `diag`, so a GS sweep from integer
    data produces dyadic numbers and every product/sum is exact in FP64."""
    p = gen.make_config("C2", nx=nx, ny=ny, nz=nz)
    rng = np.random.default_rng(seed)
    val = rng.integers(-3, 4, p["val"].shape).astype(np.float64)
    for c in range(p["n"]):
        for e in range(p["row_ptr"][c], p["row_ptr"][c + 1]):
            if p["col"][e] == c:
                val[e] += 64 * np.eye(p["b"])
                val[e][0, 0] = diag
            else:
                if val[e][0, 0] == 0:
                    val[e][0, 0] = -1.0                  # keep the pressure graph connected
    p["val"] = val
    return p


@pytest.mark.parametrize("asc", [True, False])
def test_a4_pgs_sweep_integer_bit_exact(asc):
    p = integer_system(20, 16, 4, 3)
    s = solver(p, coarsest_max_dof=60, decoupling=0)
    O = oracle.Msp(p["row_ptr"], p["col"], p["val"], coarsest_max_dof=60, decoupling=0)
    ptr, col, val = O.level_csr(0)
    assert np.all(np.round(val) == val)
    g, color = O.level_colors(0)
    n = len(ptr) - 1
    b = gen.integer_vector(n, 7, lim=1000)
    x0 = gen.integer_vector(n, 8, lim=1000)
    ref = oracle.pgs_mc(ptr, col, val, color, g, b, x0, asc)
    xd = dev(x0.copy())
    s.pgs_sweep(0, dev(b), xd, asc)
    assert np.array_equal(xd.cpu().numpy(), ref)


def test_a8_integer_bit_exact():
    p = integer_system(20, 16, 4, 4)
    s = solver(p, coarsest_max_dof=60, decoupling=0)
    n, b = p["n"], p["b"]
    g = gen.integer_vector(n * b, 1, lim=1000)
    xp = gen.integer_vector(n, 2, lim=1000)
    w = np.zeros(n * b); w[0::b] = xp
    ref = g - oracle.bsr_spmv(p["row_ptr"], p["col"], p["val"], w)
    out = torch.zeros(n * b, dtype=torch.float64, device="cuda")
    s.pcol_residual(dev(g), dev(xp), out)
    assert np.array_equal(out.cpu().numpy(), ref)


@pytest.mark.parametrize("kw", [dict(), dict(bilu_order=0), dict(pair_passes=1)])
def test_a9_bilu_integer_factors_bit_exact(kw):
    """Both substitution kernels on INTEGER factors (L, U entries in {-1, 0, 1}, D~^-1 = I,
    set through the test hooks of both sides): every intermediate is an integer below
    2^53, so forward and backward must agree bit for bit."""
    p = gen.make_config("C2", nx=14, ny=12, nz=4)
    s = solver(p, coarsest_max_dof=60, **kw)
    O = oracle.Msp(p["row_ptr"], p["col"], p["val"], coarsest_max_dof=60, **kw)
    n, b = p["n"], p["b"]
    rng = np.random.default_rng(9)
    F = rng.choice([-1.0, 0.0, 0.0, 0.0, 1.0], size=p["val"].shape)
    Dinv = np.broadcast_to(np.eye(b), (n, b, b)).copy()
    for c in range(n):
        for e in range(p["row_ptr"][c], p["row_ptr"][c + 1]):
            if p["col"][e] == c:
                F[e] = Dinv[c]
    O.set_bilu_factors(F, Dinv)
    s.set_bilu_factors(F)
    assert np.array_equal(s.bilu_factors(), F)
    r = gen.integer_vector(n * b, 3, lim=50)
    y = O.bilu_forward(r)
    ya = O.bilu_backward(O.bilu_forward(r, absmode=True), absmode=True)
    assert ya.max() < 2.0 ** 52                     # exactness of the integer arithmetic
    yd = torch.zeros(n * b, dtype=torch.float64, device="cuda")
    s.bilu_forward(dev(r), yd)
    assert np.array_equal(yd.cpu().numpy(), y)
    xd = torch.zeros(n * b, dtype=torch.float64, device="cuda")
    s.bilu_backward(dev(y), xd)
    assert np.array_equal(xd.cpu().numpy(), O.bilu_backward(y))
    # and the fused apply (the solve's launch sequence, last color fused)
    zd = torch.zeros(n * b, dtype=torch.float64, device="cuda")
    s.bilu_apply(dev(r), zd)
    assert np.array_equal(zd.cpu().numpy(), O.bilu_apply(r))
