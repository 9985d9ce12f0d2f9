"""ctypes wrapper of the CPU oracle (oracle/oracle.cpp).

TEST INFRASTRUCTURE ONLY: only tests/, __graft_entry__.smoke() and bench.py's
cpu_baseline / ``--impl reference`` legs may import this package.  The product
package (paper_2208_08594_b200) never imports it.
"""
from __future__ import annotations

import ctypes
import os
import subprocess

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_SRC = os.path.join(_HERE, "oracle.cpp")
_LIB = os.path.join(_HERE, "liboracle.so")

I32 = np.int32
F64 = np.float64


def build(force: bool = False) -> str:
    if force or not os.path.exists(_LIB) or os.path.getmtime(_LIB) < os.path.getmtime(_SRC):
        subprocess.check_call(["g++", "-O2", "-fPIC", "-shared", "-ffp-contract=off", "-std=c++17",
                               "-fopenmp", "-o", _LIB, _SRC])
    return _LIB


_lib = None


def lib():
    global _lib
    if _lib is None:
        _lib = ctypes.CDLL(build())
        _lib.orc_last_error.restype = ctypes.c_char_p
        _lib.orc_msp_setup.restype = ctypes.c_void_p
        for name in ("orc_msp_update_values", "orc_msp_destroy", "orc_msp_info", "orc_msp_level_n",
                     "orc_msp_level_csr", "orc_msp_level_colors", "orc_msp_level_agg",
                     "orc_msp_weights", "orc_msp_order", "orc_msp_bilu_factors", "orc_msp_vcycle",
                     "orc_msp_bilu_apply", "orc_msp_apply", "orc_msp_solve", "orc_msp_bgs_apply",
                     "orc_msp_restrict_pressure", "orc_msp_level_resid_restrict",
                     "orc_msp_level_prolong", "orc_msp_bilu_forward", "orc_msp_bilu_backward",
                     "orc_msp_bilu_apply_by_color", "orc_msp_bilu_blocks", "orc_msp_bilu_set_factors", "orc_msp_bilu_refactor"):
            getattr(_lib, name).argtypes = None
    return _lib


def _p(a):
    return a.ctypes.data_as(ctypes.c_void_p) if a is not None else None


def _c(a, dt):
    return np.ascontiguousarray(a, dtype=dt)


class OracleError(RuntimeError):
    pass


def last_error() -> str:
    return lib().orc_last_error().decode()


class Config(ctypes.Structure):
    _fields_ = [(k, ctypes.c_int32) for k in ("coarsest_max_dof", "max_levels", "pre_sweeps",
                                              "post_sweeps", "pair_passes", "decoupling",
                                              "bilu_order", "stages", "orth", "smoother",
                                              "gs_chunk")]

    @classmethod
    def make(cls, coarsest_max_dof=10000, max_levels=20, pre_sweeps=1, post_sweeps=1, pair_passes=2,
             decoupling=2, bilu_order=1, stages=2, orth=0, smoother=0, gs_chunk=32):
        return cls(coarsest_max_dof, max_levels, pre_sweeps, post_sweeps, pair_passes, decoupling,
                   bilu_order, stages, orth, smoother, gs_chunk)


# ---------------------------------------------------------------- primitives
def set_threads(n: int) -> int:
    """Timing switch: run the oracle's independent loops on n OpenMP threads (0 = all
    cores); results are bit-identical for any n.  Returns the thread count in use."""
    return int(lib().orc_set_threads(int(n)))


def bsr_spmv(row_ptr, col, val, x):
    n = len(row_ptr) - 1
    b = val.shape[-1]
    y = np.zeros(n * b)
    lib().orc_bsr_spmv(n, b, _p(_c(row_ptr, I32)), _p(_c(col, I32)), _p(_c(val, F64)),
                       _p(_c(x, F64)), _p(y))
    return y


def _graph_out(fn, n, nnz_cap, *args):
    optr = np.zeros(n + 1, dtype=I32)
    ocol = np.zeros(max(nnz_cap, 1), dtype=I32)
    m = fn(*args, _p(optr), _p(ocol))
    return optr, ocol[:m].copy()


def csr_adjacency(ptr, col, val):
    n = len(ptr) - 1
    return _graph_out(lib().orc_csr_adjacency, n, 2 * len(col), n, _p(_c(ptr, I32)),
                      _p(_c(col, I32)), _p(_c(val, F64)))


def cell_graph(row_ptr, col, val):
    n = len(row_ptr) - 1
    b = val.shape[-1]
    return _graph_out(lib().orc_cell_graph, n, 2 * len(col), n, b, _p(_c(row_ptr, I32)),
                      _p(_c(col, I32)), _p(_c(val, F64)))


def grouping(gptr, gcol):
    n = len(gptr) - 1
    color = np.zeros(n, dtype=I32)
    g = lib().orc_grouping(n, _p(_c(gptr, I32)), _p(_c(gcol, I32)), _p(color))
    return g, color


def splitting(gptr, gcol, V):
    n = len(gptr) - 1
    V = _c(V, I32)
    W = np.zeros(len(V), dtype=I32)
    Wb = np.zeros(len(V), dtype=I32)
    k = lib().orc_splitting(n, _p(_c(gptr, I32)), _p(_c(gcol, I32)), len(V), _p(V), _p(W), _p(Wb))
    return W[:k].copy(), Wb[:len(V) - k].copy()


def csr_grouping(ptr, col, val):
    n = len(ptr) - 1
    color = np.zeros(n, dtype=I32)
    g = lib().orc_csr_grouping(n, _p(_c(ptr, I32)), _p(_c(col, I32)), _p(_c(val, F64)), _p(color))
    return g, color


def npair(ptr, col, val):
    n = len(ptr) - 1
    agg = np.zeros(n, dtype=I32)
    na = lib().orc_npair(n, _p(_c(ptr, I32)), _p(_c(col, I32)), _p(_c(val, F64)), _p(agg))
    return na, agg


def galerkin(ptr, col, val, agg, nagg):
    n = len(ptr) - 1
    optr = np.zeros(nagg + 1, dtype=I32)
    ocol = np.zeros(len(col), dtype=I32)
    oval = np.zeros(len(col), dtype=F64)
    m = lib().orc_galerkin(n, _p(_c(ptr, I32)), _p(_c(col, I32)), _p(_c(val, F64)),
                           _p(_c(agg, I32)), nagg, _p(optr), _p(ocol), _p(oval))
    return optr, ocol[:m].copy(), oval[:m].copy()


def pgs_mc(ptr, col, val, color, g, b, x, ascending=True):
    n = len(ptr) - 1
    x = _c(x, F64).copy()
    rc = lib().orc_pgs_mc(n, _p(_c(ptr, I32)), _p(_c(col, I32)), _p(_c(val, F64)),
                          _p(_c(color, I32)), g, _p(_c(b, F64)), _p(x), 1 if ascending else 0)
    if rc:
        raise OracleError(last_error())
    return x


def jacobi_sweep(ptr, col, val, b, x):
    """One PJAC-NO sweep (R13)."""
    n = len(ptr) - 1
    x = _c(x, F64).copy()
    if lib().orc_jacobi(n, _p(_c(ptr, I32)), _p(_c(col, I32)), _p(_c(val, F64)), _p(_c(b, F64)), _p(x)):
        raise OracleError(last_error())
    return x


def hybrid_gs_sweep(ptr, col, val, K, b, x, ascending=True):
    """One PGS-NO sweep: chunks of K natural-order rows, GS inside, Jacobi across (R13)."""
    n = len(ptr) - 1
    x = _c(x, F64).copy()
    if lib().orc_hybrid_gs(n, _p(_c(ptr, I32)), _p(_c(col, I32)), _p(_c(val, F64)), int(K),
                           _p(_c(b, F64)), _p(x), 1 if ascending else 0):
        raise OracleError(last_error())
    return x


def dense_lu_solve(M, b):
    M = _c(M, F64)
    n = M.shape[0]
    x = np.zeros(n)
    if lib().orc_dense_lu_solve(n, _p(M), _p(_c(b, F64)), _p(x)):
        raise OracleError(last_error())
    return x


def blk_inv(D):
    D = _c(D, F64)
    out = np.zeros_like(D)
    if lib().orc_blk_inv(D.shape[0], _p(D), _p(out)):
        raise OracleError("singular block")
    return out


def gmres_csr(ptr, col, val, b, x0=None, tol=1e-6, m=30, maxit=1000, orth=0, Minv=None):
    n = len(ptr) - 1
    x = np.zeros(n) if x0 is None else _c(x0, F64).copy()
    it = ctypes.c_int(0)
    fr = ctypes.c_double(0)
    hl = ctypes.c_int(0)
    hist = np.zeros(maxit + 200)
    st = lib().orc_gmres_csr(n, _p(_c(ptr, I32)), _p(_c(col, I32)), _p(_c(val, F64)), _p(_c(b, F64)),
                             _p(x), ctypes.c_double(tol), m, maxit, orth,
                             _p(_c(Minv, F64)) if Minv is not None else None, ctypes.byref(it),
                             ctypes.byref(fr), _p(hist), len(hist), ctypes.byref(hl))
    return dict(x=x, iters=it.value, final_rel=fr.value, hist=hist[:hl.value].copy(), status=st)


def dots(V, w):
    """a10: V[i]^T w for the rows of V (k x N), plain index-ascending sums."""
    V = _c(V, F64)
    k, N = V.shape
    out = np.zeros(k)
    lib().orc_dots(ctypes.c_longlong(N), k, _p(V), _p(_c(w, F64)), _p(out))
    return out


def asmsp_decide(iota, last_it, mu, dims_changed=False):
    return bool(lib().orc_asmsp_decide(iota, last_it, mu, 1 if dims_changed else 0))


# ---------------------------------------------------------------- full MSP
class Msp:
    """Oracle MSP preconditioner + GMRES on a BSR system (natural cell order)."""

    def __init__(self, row_ptr, col, val, cfg: Config | None = None, **kw):
        self.n = len(row_ptr) - 1
        self.b = val.shape[-1]
        self.nnzb = len(col)
        self.cfg = cfg if cfg is not None else Config.make(**kw)
        st = ctypes.c_int(0)
        self._h = lib().orc_msp_setup(self.n, self.b, _p(_c(row_ptr, I32)), _p(_c(col, I32)),
                                      _p(_c(val, F64)), ctypes.byref(self.cfg), ctypes.byref(st))
        self.status = st.value
        if not self._h:
            raise OracleError(f"oracle setup failed ({st.value}): {last_error()}")

    def __del__(self):
        if getattr(self, "_h", None):
            lib().orc_msp_destroy(ctypes.c_void_p(self._h))
            self._h = None

    @property
    def h(self):
        return ctypes.c_void_p(self._h)

    def update_values(self, val):
        lib().orc_msp_update_values(self.h, _p(_c(val, F64)))

    def info(self):
        a = np.zeros(3, dtype=I32)
        lib().orc_msp_info(self.h, _p(a))
        return dict(levels=int(a[0]), n_coarsest=int(a[1]), coarse_diag=bool(a[2]))

    def level_sizes(self, l):
        n, nnz, g = ctypes.c_int(), ctypes.c_int(), ctypes.c_int()
        lib().orc_msp_level_n(self.h, l, ctypes.byref(n), ctypes.byref(nnz), ctypes.byref(g))
        return n.value, nnz.value, g.value

    def level_csr(self, l):
        n, nnz, _ = self.level_sizes(l)
        ptr = np.zeros(n + 1, dtype=I32); col = np.zeros(nnz, dtype=I32); val = np.zeros(nnz)
        lib().orc_msp_level_csr(self.h, l, _p(ptr), _p(col), _p(val))
        return ptr, col, val

    def level_colors(self, l):
        n, _, _ = self.level_sizes(l)
        c = np.zeros(n, dtype=I32)
        g = lib().orc_msp_level_colors(self.h, l, _p(c))
        return g, c

    def level_agg(self, l):
        n, _, _ = self.level_sizes(l)
        a = np.zeros(n, dtype=I32)
        nn = lib().orc_msp_level_agg(self.h, l, _p(a))
        return nn, a

    def weights(self):
        W = np.zeros((self.n, self.b))
        lib().orc_msp_weights(self.h, _p(W))
        return W

    def order(self):
        o = np.zeros(self.n, dtype=I32)
        lib().orc_msp_order(self.h, _p(o))
        return o

    def bilu_factors(self):
        F = np.zeros((self.nnzb, self.b, self.b)); D = np.zeros((self.n, self.b, self.b))
        lib().orc_msp_bilu_factors(self.h, _p(F), _p(D))
        return F, D

    def vcycle(self, r):
        x = np.zeros(self.n)
        if lib().orc_msp_vcycle(self.h, _p(_c(r, F64)), _p(x)):
            raise OracleError(last_error())
        return x

    def bilu_apply(self, r):
        x = np.zeros(self.n * self.b)
        lib().orc_msp_bilu_apply(self.h, _p(_c(r, F64)), _p(x))
        return x

    def restrict_pressure(self, g):
        """a3: r_p = W^T g (natural cell order)."""
        rp = np.zeros(self.n)
        lib().orc_msp_restrict_pressure(self.h, _p(_c(g, F64)), _p(rp))
        return rp

    def residual_restrict(self, l, b, x):
        """a5 on level l: r_{l+1}[I] = sum_{i in I} (b - A_l x)_i."""
        nn, _ = self.level_agg(l)
        bc = np.zeros(nn)
        if lib().orc_msp_level_resid_restrict(self.h, l, _p(_c(b, F64)), _p(_c(x, F64)), _p(bc)):
            raise OracleError("bad level")
        return bc

    def prolong(self, l, e, x):
        """a7 on level l: returns x + P e."""
        x = _c(x, F64).copy()
        if lib().orc_msp_level_prolong(self.h, l, _p(_c(e, F64)), _p(x)):
            raise OracleError("bad level")
        return x

    def bilu_forward(self, r, absmode=False):
        y = np.zeros(self.n * self.b)
        lib().orc_msp_bilu_forward(self.h, _p(_c(r, F64)), _p(y), 1 if absmode else 0)
        return y

    def bilu_backward(self, y, absmode=False):
        x = np.zeros(self.n * self.b)
        lib().orc_msp_bilu_backward(self.h, _p(_c(y, F64)), _p(x), 1 if absmode else 0)
        return x

    def set_bilu_factors(self, F, Dinv):
        """Test hook: replace the BILU factors (natural storage, row-major) and D~^-1."""
        lib().orc_msp_bilu_set_factors(self.h, _p(_c(F, F64)), _p(_c(Dinv, F64)))

    def bilu_refactor(self, val):
        """Test hook: refactorize BILU(0) in the same order from other values (natural BSR)."""
        if lib().orc_msp_bilu_refactor(self.h, _p(_c(val, F64))):
            raise OracleError(last_error())

    def bilu_apply_by_color(self, r):
        x = np.zeros(self.n * self.b)
        lib().orc_msp_bilu_apply_by_color(self.h, _p(_c(r, F64)), _p(x))
        return x

    def bilu_blocks(self):
        """(g, color[n], blk[n]): ABMC block color and block (aggregate) id of every cell."""
        color = np.zeros(self.n, dtype=I32)
        blk = np.zeros(self.n, dtype=I32)
        g = lib().orc_msp_bilu_blocks(self.h, _p(color), _p(blk))
        return g, color, blk

    def bgs_apply(self, r):
        wN = np.zeros(self.n * (self.b - 1))
        if lib().orc_msp_bgs_apply(self.h, _p(_c(r, F64)), _p(wN)):
            raise OracleError("bgs_apply needs stages=3")
        return wN

    def apply(self, g):
        w = np.zeros(self.n * self.b)
        if lib().orc_msp_apply(self.h, _p(_c(g, F64)), _p(w)):
            raise OracleError(last_error())
        return w

    def solve(self, b, x0=None, tol=1e-6, restart=30, maxit=1000):
        N = self.n * self.b
        x = np.zeros(N) if x0 is None else _c(x0, F64).copy()
        it = ctypes.c_int(0); fr = ctypes.c_double(0); hl = ctypes.c_int(0)
        hist = np.zeros(maxit + maxit // max(restart, 1) + 8)
        st = lib().orc_msp_solve(self.h, _p(_c(b, F64)), _p(x), ctypes.c_double(tol), restart, maxit,
                                 ctypes.byref(it), ctypes.byref(fr), _p(hist), len(hist),
                                 ctypes.byref(hl))
        return dict(x=x, iters=it.value, final_rel=fr.value, hist=hist[:hl.value].copy(), status=st)
