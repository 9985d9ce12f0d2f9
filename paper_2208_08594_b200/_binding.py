"""ctypes marshalling for libmsp.so.  Names follow include/msp.h."""
from __future__ import annotations

import ctypes
import os

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
lib_path = os.path.join(_HERE, "libmsp.so")

if not os.path.exists(lib_path):
    raise ImportError(f"{lib_path} is missing: run `python __graft_entry__.py build` "
                      "(the MSP solve path has no CPU fallback)")
_lib = ctypes.CDLL(lib_path)

STATUS = {0: "MSP_OK", 1: "MSP_EINVAL", 2: "MSP_ESINGULAR", 3: "MSP_ENOCONV", 4: "MSP_EBREAKDOWN",
          5: "MSP_ESTALL", 6: "MSP_ECUDA", 7: "MSP_ENCCL", 8: "MSP_ENOMEM"}

ALLOC_FN = ctypes.CFUNCTYPE(ctypes.c_void_p, ctypes.c_size_t, ctypes.c_void_p, ctypes.c_void_p)
FREE_FN = ctypes.CFUNCTYPE(None, ctypes.c_void_p, ctypes.c_void_p)


class Bsr(ctypes.Structure):
    _fields_ = [("n_cells", ctypes.c_int64), ("block", ctypes.c_int32),
                ("row_ptr", ctypes.c_void_p), ("col_idx", ctypes.c_void_p),
                ("values", ctypes.c_void_p), ("device", ctypes.c_int32)]


class Config(ctypes.Structure):
    _fields_ = [("coarsest_max_dof", ctypes.c_int32), ("max_levels", ctypes.c_int32),
                ("pre_sweeps", ctypes.c_int32), ("post_sweeps", ctypes.c_int32),
                ("pair_passes", ctypes.c_int32), ("decoupling", ctypes.c_int32),
                ("bilu_order", ctypes.c_int32), ("stages", ctypes.c_int32),
                ("orth", ctypes.c_int32), ("use_graphs", ctypes.c_int32),
                ("use_coop", ctypes.c_int32), ("smoother", ctypes.c_int32),
                ("gs_chunk", ctypes.c_int32),
                ("alloc", ALLOC_FN), ("free_fn", FREE_FN), ("alloc_ctx", ctypes.c_void_p),
                ("coarse_mode", ctypes.c_int32), ("bilu_local", ctypes.c_int32),
                ("dist_levels", ctypes.c_int32)]

    @classmethod
    def make(cls, **kw):
        c = cls()
        _lib.msp_config_default(ctypes.byref(c))
        for k, v in kw.items():
            if not hasattr(c, k):
                raise TypeError(f"unknown msp_config field {k}")
            setattr(c, k, v)
        return c


class Stats(ctypes.Structure):
    _fields_ = [("setup_calls", ctypes.c_int32), ("reuse_calls", ctypes.c_int32),
                ("setup_seconds", ctypes.c_double), ("last_setup_seconds", ctypes.c_double),
                ("solve_seconds", ctypes.c_double), ("levels", ctypes.c_int32),
                ("n_coarsest", ctypes.c_int32), ("bilu_colors", ctypes.c_int32),
                ("level_n", ctypes.c_int32 * 24), ("level_nnz", ctypes.c_int64 * 24),
                ("level_colors", ctypes.c_int32 * 24), ("device_bytes", ctypes.c_int64),
                ("kernels_per_iter", ctypes.c_int32), ("fused_a8", ctypes.c_int32)]


_lib.msp_last_error.restype = ctypes.c_char_p
_lib.msp_last_error.argtypes = [ctypes.c_void_p]
for _n in ("msp_setup", "msp_update", "msp_solve", "msp_apply", "msp_get_stats", "msp_spmv",
           "msp_pgs_sweep", "msp_vcycle", "msp_bilu_apply", "msp_bilu_factors", "msp_get_order", "msp_host_setup_run",
           "msp_host_setup_info", "msp_host_setup_level_dims", "msp_host_setup_level_csr",
           "msp_host_setup_level_colors", "msp_host_setup_level_agg", "msp_host_setup_weights",
           "msp_host_setup_order", "msp_partition_owner", "msp_nccl_unique_id", "msp_setup_dist",
           "msp_dist_owned_cells", "msp_loopback_solve", "msp_dist_plan", "msp_restrict_pressure",
           "msp_residual_restrict", "msp_prolong", "msp_pcol_residual", "msp_bilu_forward",
           "msp_bilu_backward", "msp_multidot", "msp_bilu_set_factors", "msp_set_stream", "msp_get_s1"):
    getattr(_lib, _n).restype = ctypes.c_int
_lib.msp_destroy.argtypes = [ctypes.c_void_p]
_lib.msp_time_kernel.restype = ctypes.c_int
_lib.msp_dist_n_owned.restype = ctypes.c_int32
_lib.msp_dist_n_owned.argtypes = [ctypes.c_void_p]
_lib.msp_kernel_launches.restype = ctypes.c_int64
_lib.msp_kernel_launches.argtypes = [ctypes.c_void_p]

KERNEL_KINDS = {"a2_bsr_spmv": 0, "a4_pgs_sweep_l0": 1, "a8_pcol_residual": 2, "a9_bilu_apply": 3,
                "a10_multidot16": 4, "a6_coarse_gemv": 5, "msp_apply": 6, "vcycle": 7,
                "bilu": 8, "arnoldi_step15": 9, "cgs2_step15": 10, "arnoldi_step25": 11,
                "cgs2_step25": 12,
                # the configured orthogonalisation (DCGS2 by default) at steps 15 / 25
                "orth_step15": 10, "orth_step25": 12, "bilu_spmv": 13, "msp_apply_spmv": 14,
                "spmv_orth15": 15}
_lib.msp_host_setup_free.argtypes = [ctypes.c_void_p]


class MspError(RuntimeError):
    def __init__(self, status, msg):
        super().__init__(f"{STATUS.get(status, status)}: {msg}")
        self.status = status


def _ptr(a):
    """Raw pointer of a numpy array or torch tensor (contiguous, no copy)."""
    if isinstance(a, np.ndarray):
        assert a.flags.c_contiguous
        return ctypes.c_void_p(a.ctypes.data)
    assert a.is_contiguous()
    return ctypes.c_void_p(a.data_ptr())


def _bsr(row_ptr, col, val, device=-1):
    n = len(row_ptr) - 1
    b = int(val.shape[-1])
    keep = (row_ptr, col, val)
    return Bsr(n, b, _ptr(row_ptr).value, _ptr(col).value, _ptr(val).value, device), keep


def _np(a, dt):
    return np.ascontiguousarray(a, dtype=dt)


def _bsr_any(row_ptr, col, val):
    """msp_bsr from numpy arrays (host) or CUDA torch tensors (device pointers, no copy):
    all three on the same side; device arrays must already be int32 / int32 / float64."""
    if _is_cuda(val):
        if not (_is_cuda(row_ptr) and _is_cuda(col)):
            raise ValueError("row_ptr, col and val must all be CUDA tensors (or all host arrays)")
        import torch
        if row_ptr.dtype != torch.int32 or col.dtype != torch.int32 or val.dtype != torch.float64:
            raise ValueError("device BSR arrays must be int32, int32, float64")
        rp, ci, v = row_ptr.contiguous(), col.contiguous(), val.contiguous()
        dev = v.device.index if v.device.index is not None else 0
        return _bsr(rp, ci, v, device=dev)
    return _bsr(_np(row_ptr, np.int32), _np(col, np.int32), _np(val, np.float64))


def _is_cuda(a):
    return hasattr(a, "is_cuda") and bool(a.is_cuda)


class _TorchAllocator:
    """Routes the library's device allocations through PyTorch's caching allocator."""

    def __init__(self):
        import torch
        self.torch = torch
        self.alloc = ALLOC_FN(self._alloc)
        self.free = FREE_FN(self._free)

    def _alloc(self, size, stream, ctx):
        try:
            return self.torch.cuda.caching_allocator_alloc(int(size), stream=int(stream or 0))
        except Exception:
            return None

    def _free(self, ptr, ctx):
        try:
            self.torch.cuda.caching_allocator_delete(int(ptr))
        except Exception:          # interpreter teardown: torch already unloaded
            pass


def _caller_stream(stream):
    """The stream the library orders its work after: the given one, else PyTorch's current
    stream (so tensors written by torch are complete before the library reads them)."""
    if stream:
        return int(stream)
    try:
        import torch
        if torch.cuda.is_available():
            return int(torch.cuda.current_stream().cuda_stream)
    except ImportError:
        pass
    return 0


class MspSolver:
    """msp_setup / msp_solve handle.  A given as BSR arrays (natural cell order, row-major
    b x b blocks, unknown 0 = pressure).  Vectors may be numpy arrays (host) or torch
    tensors (host or CUDA)."""

    def __init__(self, row_ptr, col, val, nc, stream=None, torch_allocator=True, **cfg):
        self.n = len(row_ptr) - 1
        self.b = int(val.shape[-1])
        self.nnzb = len(col)
        self.nc = nc
        self.N = self.n * self.b
        self._keep_alloc = None
        c = Config.make(**cfg)
        if torch_allocator:
            try:
                import torch
                if torch.cuda.is_available():
                    self._keep_alloc = _TorchAllocator()
                    c.alloc = self._keep_alloc.alloc
                    c.free_fn = self._keep_alloc.free
            except ImportError:
                pass
        self.cfg = c
        A, keep = _bsr_any(row_ptr, col, val)
        h = ctypes.c_void_p()
        st = _lib.msp_setup(ctypes.byref(A), nc, ctypes.byref(c), ctypes.c_void_p(_caller_stream(stream)),
                            ctypes.byref(h))
        if st:
            raise MspError(st, _lib.msp_last_error(None).decode())
        self._h = h

    def _check(self, st, ok=(0,)):
        if st not in ok:
            raise MspError(st, _lib.msp_last_error(self._h).decode())
        return st

    def close(self):
        if getattr(self, "_h", None):
            _lib.msp_destroy(self._h)
            self._h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    def update(self, row_ptr, col, val, iota, last_iterations, mu):
        """ASMSP: returns True when SETUP was executed."""
        A, keep = _bsr_any(row_ptr, col, val)
        did = ctypes.c_int(0)
        self._check(_lib.msp_update(self._h, ctypes.byref(A), iota, last_iterations, mu,
                                    ctypes.byref(did)))
        return bool(did.value)

    def solve(self, b, x=None, tol=1e-6, restart=30, maxit=1000, hist_cap=None):
        """Restarted GMRES; b, x natural order.  Returns dict(x, iters, final_rel, hist, status)."""
        import torch
        if isinstance(b, np.ndarray):
            b = _np(b, np.float64)
            if x is None:
                x = np.zeros_like(b)
        else:
            b = b.contiguous()
            if x is None:
                x = torch.zeros_like(b)
        it = ctypes.c_int(0)
        fr = ctypes.c_double(0)
        cap = hist_cap or (maxit + maxit // restart + 8)
        hist = np.zeros(cap)
        hl = ctypes.c_int(0)
        st = _lib.msp_solve(self._h, _ptr(b), _ptr(x), ctypes.c_double(tol), restart, maxit,
                            ctypes.byref(it), ctypes.byref(fr), _ptr(hist), cap, ctypes.byref(hl))
        self._check(st, ok=(0, 3))
        return dict(x=x, iters=it.value, final_rel=fr.value, hist=hist[:hl.value].copy(), status=st)

    def apply(self, g, w):
        self._check(_lib.msp_apply(self._h, _ptr(g), _ptr(w)))
        return w

    def spmv_internal(self, x, y):
        self._check(_lib.msp_spmv(self._h, _ptr(x), _ptr(y)))
        return y

    def pgs_sweep(self, level, b, x, ascending=True):
        self._check(_lib.msp_pgs_sweep(self._h, level, _ptr(b), _ptr(x), 1 if ascending else 0))
        return x

    def vcycle(self, r, x):
        self._check(_lib.msp_vcycle(self._h, _ptr(r), _ptr(x)))
        return x

    def bilu_apply(self, r, x):
        self._check(_lib.msp_bilu_apply(self._h, _ptr(r), _ptr(x)))
        return x

    # single hot-path steps (per-kernel parity tests); device tensors, natural order
    def restrict_pressure(self, g, rp):
        """a3: rp = W^T g."""
        self._check(_lib.msp_restrict_pressure(self._h, _ptr(g), _ptr(rp)))
        return rp

    def residual_restrict(self, level, b, x, bc):
        """a5 on AMG level `level`: bc = P^T (b - A x)."""
        self._check(_lib.msp_residual_restrict(self._h, level, _ptr(b), _ptr(x), _ptr(bc)))
        return bc

    def prolong(self, level, e, x):
        """a7: x += P e (in place)."""
        self._check(_lib.msp_prolong(self._h, level, _ptr(e), _ptr(x)))
        return x

    def pcol_residual(self, g, xp, r):
        """a8: r = g - A Pi_P xp."""
        self._check(_lib.msp_pcol_residual(self._h, _ptr(g), _ptr(xp), _ptr(r)))
        return r

    def bilu_forward(self, r, y):
        self._check(_lib.msp_bilu_forward(self._h, _ptr(r), _ptr(y)))
        return y

    def bilu_backward(self, y, x):
        self._check(_lib.msp_bilu_backward(self._h, _ptr(y), _ptr(x)))
        return x

    def multidot(self, V, w):
        """a10: V_i^T w for the k rows of V (k x N device tensor); returns numpy (k,)."""
        k = int(V.shape[0])
        out = np.zeros(k)
        self._check(_lib.msp_multidot(self._h, k, _ptr(V), _ptr(w), _ptr(out)))
        return out

    def set_bilu_factors(self, F):
        """Test hook: replace the BILU factors (natural entry order, row-major, D~^-1 on the
        diagonal slots; the layout bilu_factors() returns)."""
        F = _np(F, np.float64)
        self._check(_lib.msp_bilu_set_factors(self._h, _ptr(F)))

    def s1(self):
        """(W (n, b), A_PP values (nnzb,), computed_on_gpu) of the last SETUP (natural order)."""
        W = np.zeros((self.n, self.b))
        App = np.zeros(self.nnzb)
        g = ctypes.c_int32(0)
        self._check(_lib.msp_get_s1(self._h, _ptr(W), _ptr(App), ctypes.byref(g)))
        return W, App, bool(g.value)

    def set_stream(self, stream):
        """Order every later call after the work queued on `stream` (a cudaStream_t int)."""
        self._check(_lib.msp_set_stream(self._h, ctypes.c_void_p(stream or 0)))

    def bilu_factors(self):
        """(nnzb, b, b) BILU(0) factors, natural entry order; diagonal slots hold D~^-1."""
        F = np.zeros((self.nnzb, self.b, self.b))
        self._check(_lib.msp_bilu_factors(self._h, _ptr(F)))
        return F

    def order(self):
        o = np.zeros(self.n, dtype=np.int32)
        self._check(_lib.msp_get_order(self._h, _ptr(o)))
        return o

    def time_kernel(self, kind, reps=10, flush=True):
        """(ms per launch, algorithmic bytes per launch) of one hot-path kernel, L2 flushed
        before each launch (CUDA events on the solver's stream)."""
        k = KERNEL_KINDS[kind] if isinstance(kind, str) else int(kind)
        if not flush:
            k |= 0x100
        ms = ctypes.c_double(0)
        by = ctypes.c_double(0)
        self._check(_lib.msp_time_kernel(self._h, k, reps, ctypes.byref(ms), ctypes.byref(by)))
        return ms.value, by.value

    def kernel_launches(self):
        return int(_lib.msp_kernel_launches(self._h))

    def stats(self):
        s = Stats()
        self._check(_lib.msp_get_stats(self._h, ctypes.byref(s)))
        L = s.levels
        return dict(setup_calls=s.setup_calls, reuse_calls=s.reuse_calls,
                    setup_seconds=s.setup_seconds, last_setup_seconds=s.last_setup_seconds,
                    solve_seconds=s.solve_seconds, levels=L, n_coarsest=s.n_coarsest,
                    bilu_colors=s.bilu_colors, level_n=list(s.level_n[:L + 1]),
                    level_nnz=list(s.level_nnz[:L + 1]), level_colors=list(s.level_colors[:L]),
                    device_bytes=s.device_bytes, kernels_per_iter=s.kernels_per_iter,
                    fused_a8=bool(s.fused_a8))


def nccl_unique_id() -> bytes:
    """128-byte ncclUniqueId (rank 0); broadcast it to the other ranks."""
    buf = (ctypes.c_char * 128)()
    st = _lib.msp_nccl_unique_id(buf)
    if st:
        raise MspError(st, _lib.msp_last_error(None).decode())
    return bytes(buf)


class DistSolver(MspSolver):
    """One rank of the z-slab distributed solver (msp_setup_dist, NCCL).  Vectors passed
    to solve/apply are this rank's owned cells (ascending natural id: owned_cells())."""

    def __init__(self, row_ptr, col, val, nc, rank, nranks, unique_id, owner=None, stream=None,
                 torch_allocator=True, **cfg):
        self.n_global = len(row_ptr) - 1
        self.b = int(val.shape[-1])
        self.nc = nc
        self._keep_alloc = None
        c = Config.make(**cfg)
        if torch_allocator:
            import torch
            if torch.cuda.is_available():
                self._keep_alloc = _TorchAllocator()
                c.alloc = self._keep_alloc.alloc
                c.free_fn = self._keep_alloc.free
        self.cfg = c
        rp, ci, v = _np(row_ptr, np.int32), _np(col, np.int32), _np(val, np.float64)
        A, keep = _bsr(rp, ci, v)
        own = None if owner is None else _np(owner, np.int32)
        uid = ctypes.create_string_buffer(bytes(unique_id), 128)
        h = ctypes.c_void_p()
        st = _lib.msp_setup_dist(ctypes.byref(A), nc, ctypes.byref(c), _ptr(own) if own is not None else None,
                                 uid, rank, nranks, ctypes.c_void_p(_caller_stream(stream)), ctypes.byref(h))
        if st:
            raise MspError(st, _lib.msp_last_error(None).decode())
        self._h = h
        self.n = int(_lib.msp_dist_n_owned(h))
        self.N = self.n * self.b

    def owned_cells(self):
        o = np.zeros(self.n, dtype=np.int32)
        self._check(_lib.msp_dist_owned_cells(self._h, _ptr(o)))
        return o


def loopback_solve(row_ptr, col, val, nc, nranks, b, x0=None, owner=None, tol=1e-6, restart=30, maxit=1000,
                   **cfg):
    """Distributed path on ONE GPU: nranks virtual ranks (threads), event-ordered copies."""
    c = Config.make(**cfg)
    rp, ci, v = _np(row_ptr, np.int32), _np(col, np.int32), _np(val, np.float64)
    A, keep = _bsr(rp, ci, v)
    b = _np(b, np.float64)
    x = np.zeros_like(b) if x0 is None else _np(x0, np.float64).copy()
    own = None if owner is None else _np(owner, np.int32)
    it = ctypes.c_int(0)
    fr = ctypes.c_double(0)
    info = np.zeros(4 * nranks, dtype=np.int32)
    st = _lib.msp_loopback_solve(ctypes.byref(A), nc, ctypes.byref(c), _ptr(own) if own is not None else None,
                                 nranks, _ptr(b), _ptr(x), ctypes.c_double(tol), restart, maxit,
                                 ctypes.byref(it), ctypes.byref(fr), _ptr(info))
    if st not in (0, 3):
        raise MspError(st, _lib.msp_last_error(None).decode())
    return dict(x=x, iters=it.value, final_rel=fr.value, status=st, rank_info=info.reshape(nranks, 4))


class HostSetup:
    """Host-only SETUP (S1-S4) introspection: integer structures and Galerkin values, no GPU."""

    def __init__(self, row_ptr, col, val, nc, **cfg):
        self.n = len(row_ptr) - 1
        self.b = int(val.shape[-1])
        c = Config.make(**cfg)
        rp, ci, v = _np(row_ptr, np.int32), _np(col, np.int32), _np(val, np.float64)
        A, keep = _bsr(rp, ci, v)
        h = ctypes.c_void_p()
        st = _lib.msp_host_setup_run(ctypes.byref(A), nc, ctypes.byref(c), ctypes.byref(h))
        if st:
            raise MspError(st, _lib.msp_last_error(None).decode())
        self._h = h

    def __del__(self):
        if getattr(self, "_h", None):
            _lib.msp_host_setup_free(self._h)
            self._h = None

    def info(self):
        o = np.zeros(4, dtype=np.int32)
        _lib.msp_host_setup_info(self._h, _ptr(o))
        return dict(levels=int(o[0]), n_coarsest=int(o[1]), coarse_diag=bool(o[2]),
                    bilu_colors=int(o[3]))

    def level_dims(self, l):
        n, nnz, g = ctypes.c_int32(), ctypes.c_int64(), ctypes.c_int32()
        st = _lib.msp_host_setup_level_dims(self._h, l, ctypes.byref(n), ctypes.byref(nnz),
                                            ctypes.byref(g))
        if st:
            raise MspError(st, "bad level")
        return n.value, nnz.value, g.value

    def level_csr(self, l):
        n, nnz, _ = self.level_dims(l)
        ptr = np.zeros(n + 1, np.int32); col = np.zeros(nnz, np.int32); val = np.zeros(nnz)
        _lib.msp_host_setup_level_csr(self._h, l, _ptr(ptr), _ptr(col), _ptr(val))
        return ptr, col, val

    def level_colors(self, l):
        n, _, g = self.level_dims(l)
        c = np.zeros(n, np.int32)
        _lib.msp_host_setup_level_colors(self._h, l, _ptr(c))
        return g, c

    def level_agg(self, l):
        n, _, _ = self.level_dims(l)
        a = np.zeros(n, np.int32)
        _lib.msp_host_setup_level_agg(self._h, l, _ptr(a))
        return a

    def weights(self):
        W = np.zeros((self.n, self.b))
        _lib.msp_host_setup_weights(self._h, _ptr(W))
        return W

    def order(self):
        o = np.zeros(self.n, np.int32)
        _lib.msp_host_setup_order(self._h, _ptr(o))
        return o

    def dist_plan(self, rank, nranks, owner=None):
        """Host-only cell-space halo plan of `rank` (see msp_dist_plan)."""
        n = self.n
        no, ng = ctypes.c_int32(), ctypes.c_int32()
        owned = np.zeros(n, np.int32); ghosts = np.zeros(n, np.int32)
        sp_ = np.zeros(nranks + 1, np.int32); rp_ = np.zeros(nranks + 1, np.int32)
        sc = np.zeros(max(n * nranks, 1), np.int32)
        own = None if owner is None else _np(owner, np.int32)
        st = _lib.msp_dist_plan(self._h, _ptr(own) if own is not None else None, rank, nranks, ctypes.byref(no),
                                _ptr(owned), ctypes.byref(ng), _ptr(ghosts), _ptr(sp_), _ptr(sc), _ptr(rp_))
        if st:
            raise MspError(st, _lib.msp_last_error(None).decode())
        return dict(owned=owned[:no.value].copy(), ghosts=ghosts[:ng.value].copy(), send_ptr=sp_,
                    send_cells=sc[:sp_[-1]].copy(), recv_ptr=rp_)

    def dist_level_plan(self, rank, nranks, level, owner=None):
        """Host-only plan of a partitioned AMG level (msp_dist_level_plan), parsed."""
        own = None if owner is None else _np(owner, np.int32)
        op = _ptr(own) if own is not None else None
        ln = ctypes.c_int64(0)
        st = _lib.msp_dist_level_plan(self._h, op, rank, nranks, level, None, ctypes.c_int64(0), ctypes.byref(ln))
        if st:
            raise MspError(st, _lib.msp_last_error(None).decode())
        buf = np.zeros(ln.value, np.int32)
        st = _lib.msp_dist_level_plan(self._h, op, rank, nranks, level, _ptr(buf), ctypes.c_int64(ln.value),
                                      ctypes.byref(ln))
        if st:
            raise MspError(st, _lib.msp_last_error(None).decode())
        k = 4
        cnt = buf[:4]
        out = {}
        for name, c in zip(("rows", "gx", "gp", "gm"), cnt):
            out[name] = buf[k:k + c].copy()
            k += c
        for name in ("sendx", "sendp", "sendm"):
            out[name] = []
        for q in range(nranks):
            for name in ("sendx", "sendp", "sendm"):
                c = buf[k]
                out[name].append(buf[k + 1:k + 1 + c].copy())
                k += 1 + c
        m = buf[k]
        out["owner"] = buf[k + 1:k + 1 + m].copy()
        out["row_index"] = buf[k + 1 + m:k + 1 + 2 * m].copy()
        return out

    def partition_owner(self, nx, ny, nz, nranks):
        o = np.zeros(self.n, np.int32)
        st = _lib.msp_partition_owner(self._h, nx, ny, nz, nranks, _ptr(o))
        if st:
            raise MspError(st, "partition")
        return o
