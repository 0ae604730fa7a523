"""Thin Python binding of the C ABI in include/te.h (argument marshalling only).

Every step of the method runs inside libtimeevolver.so (CUDA kernels for sm_100a + the
host restart loop in C++).  There is no Python or CPU fallback: if the library is missing
or no CUDA device is present, calls raise ``TEError``.  PyTorch is only used by callers
for device memory / streams (``te_evolve_dev`` takes tensors' data pointers).
"""
from __future__ import annotations

import ctypes as C
import os

import numpy as np

from . import build as _build

_LIB = None

TE_OK = 0
STATUS = {0: "TE_OK", 1: "TE_ERR_ARG", 2: "TE_ERR_CSR", 3: "TE_ERR_NOT_HERMITIAN", 4: "TE_ERR_NOT_NORMALIZED",
          5: "TE_ERR_STEP_COLLAPSE", 6: "TE_ERR_NUMERICAL", 7: "TE_ERR_OOM", 8: "TE_ERR_CUDA", 9: "TE_ERR_NCCL",
          10: "TE_ERR_UNSUPPORTED"}
TE_WARN_ROUNDOFF = 1
TE_WARN_QUADRATURE = 2
TE_OPT_PROFILE = 1
TE_OPT_GRAPH = 2
TE_INFO_XS_GLOBAL, TE_INFO_XS_GLOBAL_TILES, TE_INFO_XS_X_PER_ENTRY, TE_INFO_SW_FILL = 101, 102, 103, 104
TE_INFO_SW_PANEL, TE_INFO_SW_FAR = 105, 106
TE_OPT_KERNELS = 3
TE_OPT_PREFETCH = 4
TE_OPT_SPMV = 5
TE_OPT_ORTHO = 6
TE_OPT_INTEGRATOR = 7
TE_OPT_HALO = 8
KERNELS = {0: "spmv", 1: "update_proj", 2: "update_norm", 3: "combine", 4: "halo_pack", 5: "proj_dots",
           6: "host_step"}


class TEError(RuntimeError):
    def __init__(self, status: int, msg: str):
        super().__init__(f"{STATUS.get(status, status)}: {msg}")
        self.status = status


class Stats(C.Structure):
    _fields_ = [("err_bound", C.c_double), ("n_restarts", C.c_int64), ("n_krylov_steps", C.c_int64),
                ("n_breakdowns", C.c_int64), ("roundoff_step", C.c_double), ("roundoff_total", C.c_double),
                ("warnings", C.c_uint32), ("_pad", C.c_uint32), ("t_step_min", C.c_double),
                ("t_step_max", C.c_double), ("one_norm", C.c_double)]

    def as_dict(self):
        return {k: getattr(self, k) for k, _ in self._fields_ if k != "_pad"}


class KernelProfile(C.Structure):
    _fields_ = [("launches", C.c_int64), ("total_ms", C.c_double), ("alg_bytes", C.c_double)]


def lib_path() -> str:
    return _build.LIB


def load():
    """Load libtimeevolver.so (built in-tree by ``python -m paper_2205_15346_b200.build``)."""
    global _LIB
    if _LIB is not None:
        return _LIB
    if not os.path.exists(_build.LIB):
        raise TEError(8, f"{_build.LIB} is not built (run __graft_entry__.build())")
    L = C.CDLL(_build.LIB)
    P, I64, I32, D, V = C.POINTER, C.c_int64, C.c_int32, C.c_double, C.c_void_p
    L.te_create_csr.restype = V
    L.te_create_csr.argtypes = [I64, V, V, V]
    L.te_create_csr_real.restype = V
    L.te_create_csr_real.argtypes = [I64, V, V, V]
    L.te_evolve.restype = C.c_int
    L.te_evolve.argtypes = [V, V, D, D, C.c_int, V, P(Stats)]
    L.te_evolve_dev.restype = C.c_int
    L.te_evolve_dev.argtypes = [V, V, D, D, C.c_int, V, P(Stats), V]
    L.te_evolve_schedule.restype = C.c_int
    L.te_evolve_schedule.argtypes = [V, V, I64, V, D, C.c_int, V, P(Stats)]
    L.te_evolve_sampled.restype = C.c_int
    L.te_evolve_sampled.argtypes = [V, V, D, D, C.c_int, I64, V, V, V, V, P(Stats)]
    L.te_get_schedule.restype = I64
    L.te_get_schedule.argtypes = [V, I64, V, V, V]
    L.te_krylov_basis.restype = C.c_int
    L.te_krylov_basis.argtypes = [V, V, C.c_int, D, V, V, P(C.c_int), P(C.c_int), V]
    L.te_destroy.restype = None
    L.te_destroy.argtypes = [V]
    L.te_set_option.restype = C.c_int
    L.te_set_option.argtypes = [V, C.c_int, D]
    L.te_small_eig.restype = C.c_int
    L.te_small_eig.argtypes = [C.c_int, V, V, V, V]
    L.te_step_search.restype = C.c_int
    L.te_step_search.argtypes = [C.c_int, V, V, D, C.c_int, C.c_int, D, D, D, D, C.c_int, P(D), P(D), P(C.c_int)]
    L.te_get_option.restype = C.c_int
    L.te_get_option.argtypes = [V, C.c_int, P(D)]
    L.te_get_profile.restype = C.c_int
    L.te_get_profile.argtypes = [V, C.c_int, P(KernelProfile)]
    L.te_launch_count.restype = I64
    L.te_launch_count.argtypes = [V]
    L.te_one_norm.restype = D
    L.te_one_norm.argtypes = [V]
    L.te_last_status.restype = C.c_int
    L.te_last_error.restype = C.c_char_p
    L.te_version.restype = C.c_char_p
    L.te_nccl_unique_id.restype = C.c_int
    L.te_nccl_unique_id.argtypes = [V]
    L.te_dist_init.restype = V
    L.te_dist_init.argtypes = [C.c_int, C.c_int, V]
    L.te_dist_destroy.restype = None
    L.te_dist_destroy.argtypes = [V]
    L.te_create_csr_dist.restype = V
    L.te_create_csr_dist.argtypes = [V, I64, I64, I64, V, V, V, C.c_int]
    L.te_halo_plan.restype = I64
    L.te_halo_plan.argtypes = [C.c_int, C.c_int, V, I64, V, V, V, V, I64]
    _LIB = L
    return L


def _err(L):
    return TEError(L.te_last_status(), (L.te_last_error() or b"").decode())


def _check(L, rc):
    if rc != TE_OK:
        raise TEError(rc, (L.te_last_error() or b"").decode())


def _ptr(a: np.ndarray):
    return a.ctypes.data_as(C.c_void_p)


def _vec_in(v, n: int, what: str) -> np.ndarray:
    """Host input vector: converted to contiguous complex128; must hold exactly n entries."""
    v = np.ascontiguousarray(v, dtype=np.complex128)
    if v.shape != (n,):
        raise ValueError(f"{what}: expected shape ({n},), got {v.shape}")
    return v


def _vec_out(out, n: int, what: str) -> np.ndarray:
    """Caller-supplied host output: must be a writeable C-contiguous complex128 array of n entries
    (the library writes exactly n * 16 bytes into it)."""
    if out is None:
        return np.empty(n, dtype=np.complex128)
    if not isinstance(out, np.ndarray) or out.dtype != np.complex128 or out.shape != (n,) \
            or not out.flags.c_contiguous or not out.flags.writeable:
        raise ValueError(f"{what}: expected a writeable C-contiguous complex128 array of shape ({n},)")
    return out


def _dev_ptr(t, n: int, what: str) -> int:
    """Device vector: a CUDA tensor (complex128, contiguous, n entries) or a raw device pointer
    (unchecked: the caller guarantees n complex128 entries)."""
    if hasattr(t, "data_ptr"):
        import torch
        if not t.is_cuda or t.dtype != torch.complex128 or t.numel() != n or not t.is_contiguous():
            raise ValueError(f"{what}: expected a contiguous complex128 CUDA tensor of {n} entries, got "
                             f"{t.dtype} numel={t.numel()} cuda={t.is_cuda} contiguous={t.is_contiguous()}")
        return t.data_ptr()
    return int(t)


def _csr_in(n: int, rowptr, col, val):
    rowptr = np.ascontiguousarray(rowptr, dtype=np.int64)
    if rowptr.shape != (int(n) + 1,):
        raise ValueError(f"rowptr: expected shape ({int(n) + 1},), got {rowptr.shape}")
    nnz = int(rowptr[-1]) if rowptr.shape[0] else 0
    if np.shape(col)[0] < nnz or np.shape(val)[0] < nnz:
        raise ValueError(f"col/val hold fewer than rowptr[-1] = {nnz} entries")
    return rowptr


class Handle:
    """Owns a te_handle*; te_destroy on close()/GC."""

    def __init__(self, ptr, n, cplx, dist=None):
        self.ptr = ptr
        self.n = n
        self.cplx = cplx
        self.dist = dist

    def close(self):
        if self.ptr:
            load().te_destroy(self.ptr)
            self.ptr = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass


def te_create_csr(n, rowptr, col, val) -> Handle:
    L = load()
    rowptr = _csr_in(n, rowptr, col, val)
    col = np.ascontiguousarray(col, dtype=np.int32)
    if np.iscomplexobj(val):
        val = np.ascontiguousarray(val, dtype=np.complex128)
        p = L.te_create_csr(int(n), _ptr(rowptr), _ptr(col), _ptr(val))
    else:
        val = np.ascontiguousarray(val, dtype=np.float64)
        p = L.te_create_csr_real(int(n), _ptr(rowptr), _ptr(col), _ptr(val))
    if not p:
        raise _err(L)
    return Handle(p, int(n), np.iscomplexobj(val))


def te_destroy(h: Handle):
    h.close()


def te_evolve(h: Handle, v0, t, tol, m_max, out=None):
    L = load()
    v0 = _vec_in(v0, h.n, "v0")
    vo = _vec_out(out, h.n, "out")
    st = Stats()
    _check(L, L.te_evolve(h.ptr, _ptr(v0), float(t), float(tol), int(m_max), _ptr(vo), C.byref(st)))
    return vo, st.as_dict()


def te_evolve_dev(h: Handle, d_v0, t, tol, m_max, d_vout, stream=None):
    """d_v0 / d_vout: CUDA tensors (complex128, contiguous) or raw device pointers."""
    L = load()
    p0 = _dev_ptr(d_v0, h.n, "d_v0")
    p1 = _dev_ptr(d_vout, h.n, "d_vout")
    s = None
    if stream is not None:
        s = stream.cuda_stream if hasattr(stream, "cuda_stream") else int(stream)
    st = Stats()
    _check(L, L.te_evolve_dev(h.ptr, C.c_void_p(p0), float(t), float(tol), int(m_max), C.c_void_p(p1),
                              C.byref(st), C.c_void_p(s) if s else None))
    return st.as_dict()


def te_evolve_schedule(h: Handle, v0, t_steps, tol, m_max):
    L = load()
    v0 = _vec_in(v0, h.n, "v0")
    ts = np.ascontiguousarray(t_steps, dtype=np.float64)
    vo = np.empty_like(v0)
    st = Stats()
    _check(L, L.te_evolve_schedule(h.ptr, _ptr(v0), ts.shape[0], _ptr(ts), float(tol), int(m_max), _ptr(vo),
                                   C.byref(st)))
    return vo, st.as_dict()


def te_evolve_sampled(h: Handle, v0, t, tol, m_max, sample_times):
    """Returns (v(t), samples [n_samples x n], sample_bounds, stats)."""
    L = load()
    v0 = _vec_in(v0, h.n, "v0")
    ts = np.ascontiguousarray(sample_times, dtype=np.float64)
    out = np.zeros((ts.shape[0], v0.shape[0]), dtype=np.complex128)
    sb = np.zeros(ts.shape[0])
    vo = np.empty_like(v0)
    st = Stats()
    _check(L, L.te_evolve_sampled(h.ptr, _ptr(v0), float(t), float(tol), int(m_max), ts.shape[0], _ptr(ts),
                                  _ptr(out), _ptr(sb), _ptr(vo), C.byref(st)))
    return vo, out, sb, st.as_dict()


def te_get_schedule(h: Handle):
    L = load()
    k = L.te_get_schedule(h.ptr, 0, None, None, None)
    ts = np.zeros(k)
    me = np.zeros(k, dtype=np.int32)
    es = np.zeros(k)
    L.te_get_schedule(h.ptr, k, _ptr(ts), _ptr(me), _ptr(es))
    return [(float(a), int(b), float(c)) for a, b, c in zip(ts, me, es)]


def te_krylov_basis(h: Handle, v1, m, tol_rate, want_V=True):
    L = load()
    v1 = _vec_in(v1, h.n, "v1")
    a = np.zeros(m)
    b = np.zeros(m)
    me = C.c_int(0)
    bk = C.c_int(0)
    V = np.zeros((m, h.n), dtype=np.complex128) if want_V else None
    _check(L, L.te_krylov_basis(h.ptr, _ptr(v1), int(m), float(tol_rate), _ptr(a), _ptr(b), C.byref(me),
                                C.byref(bk), _ptr(V) if want_V else None))
    k = me.value
    out = dict(alpha=a[:k], beta=b[:k], m_eff=k, breakdown=bool(bk.value), h=float(b[k - 1]))
    if want_V:
        out["V"] = V[:k].T.copy()
    return out


def te_set_option(h: Handle, option: int, value: float):
    L = load()
    _check(L, L.te_set_option(h.ptr, int(option), float(value)))


def te_small_eig(alpha, beta):
    """Host eigensolver of the library (no GPU needed): returns (lam, U), U[:, k] eigenvectors."""
    L = load()
    a = np.ascontiguousarray(alpha, dtype=np.float64)
    m = a.shape[0]
    b = np.zeros(max(1, m), dtype=np.float64)
    b[: max(0, m - 1)] = np.asarray(beta, dtype=np.float64)[: max(0, m - 1)]
    lam = np.zeros(m)
    U = np.zeros((m, m))
    _check(L, L.te_small_eig(m, _ptr(a), _ptr(b), _ptr(lam), _ptr(U)))
    return lam, U


def te_step_search(alpha, beta, h, breakdown, first, tau_prev, rem, tol_rate, t_total, integrator=0):
    """Host step search of the library (no GPU needed): returns (tau, err, quad_ok)."""
    L = load()
    a = np.ascontiguousarray(alpha, dtype=np.float64)
    m = a.shape[0]
    b = np.zeros(max(1, m), dtype=np.float64)
    b[: max(0, m - 1)] = np.asarray(beta, dtype=np.float64)[: max(0, m - 1)]
    tau, err, ok = C.c_double(0), C.c_double(0), C.c_int(0)
    _check(L, L.te_step_search(m, _ptr(a), _ptr(b), float(h), int(bool(breakdown)), int(bool(first)), float(tau_prev),
                               float(rem), float(tol_rate), float(t_total), int(integrator), C.byref(tau),
                               C.byref(err), C.byref(ok)))
    return tau.value, err.value, bool(ok.value)


def te_get_option(h: Handle, option: int) -> float:
    L = load()
    v = C.c_double(0.0)
    _check(L, L.te_get_option(h.ptr, int(option), C.byref(v)))
    return v.value


def te_get_profile(h: Handle):
    L = load()
    out = {}
    for k, name in KERNELS.items():
        p = KernelProfile()
        _check(L, L.te_get_profile(h.ptr, k, C.byref(p)))
        out[name] = dict(launches=p.launches, total_ms=p.total_ms, alg_bytes=p.alg_bytes)
    return out


def te_launch_count(h: Handle) -> int:
    return int(load().te_launch_count(h.ptr))


def te_one_norm(h: Handle) -> float:
    return float(load().te_one_norm(h.ptr))


def te_version() -> str:
    return load().te_version().decode()


# ---------------------------------------------------------------- distributed

def te_nccl_unique_id() -> bytes:
    L = load()
    buf = C.create_string_buffer(128)
    _check(L, L.te_nccl_unique_id(buf))
    return buf.raw


class Dist:
    def __init__(self, ptr, nranks, rank):
        self.ptr, self.nranks, self.rank = ptr, nranks, rank

    def close(self):
        if self.ptr:
            load().te_dist_destroy(self.ptr)
            self.ptr = None


def te_dist_init(nranks: int, rank: int, uid: bytes) -> Dist:
    L = load()
    buf = C.create_string_buffer(bytes(uid), 128)
    p = L.te_dist_init(int(nranks), int(rank), buf)
    if not p:
        raise _err(L)
    return Dist(p, nranks, rank)


def te_create_csr_dist(d: Dist, n_global, row_begin, row_end, rowptr_local, col_global, val) -> Handle:
    L = load()
    rp = _csr_in(int(row_end) - int(row_begin), rowptr_local, col_global, val)
    cg = np.ascontiguousarray(col_global, dtype=np.int64)
    cplx = np.iscomplexobj(val)
    v = np.ascontiguousarray(val, dtype=np.complex128 if cplx else np.float64)
    p = L.te_create_csr_dist(d.ptr, int(n_global), int(row_begin), int(row_end), _ptr(rp), _ptr(cg), _ptr(v),
                             1 if cplx else 0)
    if not p:
        raise _err(L)
    return Handle(p, int(row_end - row_begin), cplx, dist=d)


def te_halo_plan(nranks: int, rank: int, row_starts, col_global):
    """Host-only (no GPU): returns (col_local int32, recv_counts int64[nranks], halo_global int64)."""
    L = load()
    rs = np.ascontiguousarray(row_starts, dtype=np.int64)
    cg = np.ascontiguousarray(col_global, dtype=np.int64)
    cl = np.zeros(max(1, cg.shape[0]), dtype=np.int32)
    rc = np.zeros(nranks, dtype=np.int64)
    halo = np.zeros(max(1, cg.shape[0]), dtype=np.int64)
    nh = L.te_halo_plan(int(nranks), int(rank), _ptr(rs), cg.shape[0], _ptr(cg), _ptr(cl), _ptr(rc), _ptr(halo),
                        halo.shape[0])
    if nh < 0:
        raise _err(L)
    return cl[: cg.shape[0]], rc, halo[:nh]
