"""Seeded synthetic inputs: FIM compositional Jacobians with the
block structure of PAPER.md Eq. 17/18, TPFA transmissibilities (Eq. 13,
P:150-155), manufactured RHS, and the drifted Newton sequence for ASMSP.

This module is the ONLY code shared by the oracle side and the CUDA side, and it is
an input source only: it contains none of the method's arithmetic.
"""
from __future__ import annotations

import ctypes
import os
import subprocess

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_SRC = os.path.join(_HERE, "gen.cpp")
_LIB = os.path.join(_HERE, "libgen.so")


def build(force: bool = False) -> str:
    if force or not os.path.exists(_LIB) or os.path.getmtime(_LIB) < os.path.getmtime(_SRC):
        subprocess.check_call(["g++", "-O2", "-fPIC", "-shared", "-ffp-contract=off",
                               "-o", _LIB, _SRC])
    return _LIB


class _Params(ctypes.Structure):
    _fields_ = [("nx", ctypes.c_int32), ("ny", ctypes.c_int32), ("nz", ctypes.c_int32),
                ("nc", ctypes.c_int32), ("dx", ctypes.c_double), ("dy", ctypes.c_double),
                ("dz", ctypes.c_double), ("perm_kind", ctypes.c_int32), ("sigma", ctypes.c_double),
                ("acc", ctypes.c_double), ("seed", ctypes.c_uint64), ("newton_step", ctypes.c_int32),
                ("drift", ctypes.c_double), ("kz_ratio_x10", ctypes.c_int32)]


_lib = None


def _load():
    global _lib
    if _lib is None:
        _lib = ctypes.CDLL(build())
        _lib.gen_nnzb.restype = ctypes.c_int64
        _lib.gen_nnzb.argtypes = [ctypes.c_int32] * 3
        _lib.gen_jacobian.restype = ctypes.c_int
    return _lib


# Default accumulation ratio; recorded in DESIGN.md.
ACC_DEFAULT = 1e-2

# The BASELINE.json configs.  C1 is the oracle-sized case.
CONFIGS = {
    "C1": dict(nx=10, ny=10, nz=10, nc=3, dx=1.0, dy=1.0, dz=1.0, perm_kind=0, sigma=0.0, seed=1),
    "C2": dict(nx=100, ny=100, nz=10, nc=3, dx=10.0, dy=10.0, dz=2.0, perm_kind=1, sigma=2.0, seed=2),
    "C3": dict(nx=60, ny=220, nz=85, nc=3, dx=20.0, dy=10.0, dz=2.0, perm_kind=2, sigma=0.0, seed=3,
               kz_ratio_x10=1),
    "C4": dict(nx=60, ny=220, nz=85, nc=6, dx=20.0, dy=10.0, dz=2.0, perm_kind=2, sigma=0.0, seed=4,
               kz_ratio_x10=1),
    "C5": dict(nx=200, ny=200, nz=200, nc=3, dx=1.0, dy=1.0, dz=1.0, perm_kind=1, sigma=2.0, seed=5),
}


def make_problem(nx, ny, nz, nc=3, dx=1.0, dy=1.0, dz=1.0, perm_kind=0, sigma=0.0,
                 acc=ACC_DEFAULT, seed=1, newton_step=0, drift=1e-2, kz_ratio_x10=10,
                 with_alpha=False):
    """Return dict(n, b, row_ptr, col, val (nnzb,b,b row-major), xstar, rhs, [alpha, dt])."""
    lib = _load()
    b = nc + 1
    n = nx * ny * nz
    nnzb = int(lib.gen_nnzb(nx, ny, nz))
    row_ptr = np.zeros(n + 1, dtype=np.int32)
    col = np.zeros(nnzb, dtype=np.int32)
    val = np.zeros(nnzb * b * b, dtype=np.float64)
    xstar = np.zeros(n * b, dtype=np.float64)
    rhs = np.zeros(n * b, dtype=np.float64)
    alpha = np.zeros(n * b, dtype=np.float64) if with_alpha else None
    dt = ctypes.c_double(0.0)
    p = _Params(nx, ny, nz, nc, dx, dy, dz, perm_kind, sigma, acc, seed, newton_step, drift,
                kz_ratio_x10)
    P = lambda a: a.ctypes.data_as(ctypes.c_void_p) if a is not None else None
    rc = lib.gen_jacobian(ctypes.byref(p), P(row_ptr), P(col), P(val), P(xstar), P(rhs),
                          P(alpha), ctypes.byref(dt))
    if rc != 0:
        raise ValueError("gen_jacobian failed")
    out = dict(n=n, b=b, nc=nc, nx=nx, ny=ny, nz=nz, row_ptr=row_ptr, col=col,
               val=val.reshape(nnzb, b, b), xstar=xstar, rhs=rhs, dt=dt.value)
    if with_alpha:
        out["alpha"] = alpha.reshape(n, b)
    return out


def make_config(name, **over):
    kw = dict(CONFIGS[name])
    kw.update(over)
    return make_problem(**kw)


def random_vector(n, seed):
    """Seeded U(-1,1) vector for kernel parity inputs."""
    return np.random.default_rng(seed).uniform(-1.0, 1.0, n)


def integer_vector(n, seed, lim=8):
    """Seeded integer-valued vector (exact FP64 sums -> bit-exact parity pins)."""
    return np.random.default_rng(seed).integers(-lim, lim + 1, n).astype(np.float64)


def tpfa_laplacian_csr(nx, ny, nz=1):
    """Scalar 5/7-point Laplacian (2D/3D Poisson) in CSR, for smoother/AMG pins."""
    n = nx * ny * nz
    rows, cols, vals = [], [], []
    for k in range(nz):
        for j in range(ny):
            for i in range(nx):
                c = i + nx * (j + ny * k)
                ent = []
                if k > 0: ent.append((c - nx * ny, -1.0))
                if j > 0: ent.append((c - nx, -1.0))
                if i > 0: ent.append((c - 1, -1.0))
                deg = 0
                for (di, dj, dk) in ((1, 0, 0), (0, 1, 0), (0, 0, 1), (-1, 0, 0), (0, -1, 0), (0, 0, -1)):
                    if 0 <= i + di < nx and 0 <= j + dj < ny and 0 <= k + dk < nz:
                        deg += 1
                ent.append((c, float(2 * (3 if nz > 1 else 2))))
                if i + 1 < nx: ent.append((c + 1, -1.0))
                if j + 1 < ny: ent.append((c + nx, -1.0))
                if k + 1 < nz: ent.append((c + nx * ny, -1.0))
                for cc, v in ent:
                    rows.append(c); cols.append(cc); vals.append(v)
    rows = np.array(rows); cols = np.array(cols, dtype=np.int32); vals = np.array(vals)
    ptr = np.zeros(n + 1, dtype=np.int32)
    np.add.at(ptr, rows + 1, 1)
    ptr = np.cumsum(ptr).astype(np.int32)
    return n, ptr, cols, vals
