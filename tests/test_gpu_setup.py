"""NEXT-2: the GPU SETUP steps -- S1 decoupling weights and A_PP (block
column sums / diagonal blocks, the small eliminations, the pressure-matrix products) and
the S3 Galerkin products P^T A P of every AMG level -- are BIT-IDENTICAL to the host
setup and to the oracle (explicitly rounded operations in the specified orders, R4/R3),
so every integer decision downstream (NPAIR, colorings, ABMC order) is unchanged."""
import numpy as np
import pytest

import gen
import oracle

pytestmark = pytest.mark.gpu

torch = pytest.importorskip("torch")

CASES = [("C2", dict(nx=25, ny=20, nz=5), dict()),
         ("C2", dict(nx=25, ny=20, nz=5), dict(decoupling=1)),
         ("C2", dict(nx=25, ny=20, nz=5), dict(decoupling=0)),
         ("C2", dict(nx=12, ny=10, nz=4, nc=6), dict()),
         ("C2", dict(nx=13, ny=11, nz=3, nc=1), dict()),
         ("C3", dict(nx=24, ny=88, nz=17), dict(coarsest_max_dof=500)),
         ("C2", dict(nx=30, ny=30, nz=6), dict(pair_passes=1, coarsest_max_dof=100))]


def host_setup(p, gpu, monkeypatch, **kw):
    from paper_2208_08594_b200._binding import HostSetup
    if gpu:
        monkeypatch.setenv("MSP_HOST_SETUP_GPU", "1")
    else:
        monkeypatch.delenv("MSP_HOST_SETUP_GPU", raising=False)
    return HostSetup(p["row_ptr"], p["col"], p["val"], nc=p["nc"], **kw)


@pytest.mark.parametrize("name,gkw,kw", CASES)
def test_gpu_s1_and_galerkin_bit_exact(name, gkw, kw, monkeypatch):
    p = gen.make_config(name, **gkw)
    kw = dict(dict(coarsest_max_dof=60), **kw)
    G = host_setup(p, True, monkeypatch, **kw)
    H = host_setup(p, False, monkeypatch, **kw)
    O = oracle.Msp(p["row_ptr"], p["col"], p["val"], **kw)
    assert np.array_equal(G.weights(), H.weights())
    assert np.array_equal(G.weights(), O.weights())
    gi, hi = G.info(), H.info()
    assert gi == hi and gi["levels"] == O.info()["levels"]
    for l in range(gi["levels"] + 1):
        for a, b in zip(G.level_csr(l), H.level_csr(l)):
            assert np.array_equal(a, b), l
        for a, b in zip(G.level_csr(l), O.level_csr(l)):
            assert np.array_equal(a, b), l
        if l < gi["levels"]:
            assert np.array_equal(G.level_colors(l)[1], H.level_colors(l)[1])
            assert np.array_equal(G.level_agg(l), H.level_agg(l))
    assert np.array_equal(G.order(), H.order())
    assert np.array_equal(G.order(), O.order())


@pytest.mark.parametrize("name,gkw,kw", CASES[:4])
def test_solver_setup_uses_gpu_s1(name, gkw, kw, monkeypatch):
    """msp_setup runs S1 on the GPU by default; its weights and A_PP equal the host path's."""
    from paper_2208_08594_b200 import MspSolver
    p = gen.make_config(name, **gkw)
    s = MspSolver(p["row_ptr"], p["col"], p["val"], nc=p["nc"], coarsest_max_dof=60, **kw)
    W, App, on_gpu = s.s1()
    assert on_gpu
    H = host_setup(p, False, monkeypatch, coarsest_max_dof=60, **kw)
    assert np.array_equal(W, H.weights())
    assert np.array_equal(App, H.level_csr(0)[2])
