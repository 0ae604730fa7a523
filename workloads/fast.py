"""Fast host builders (C, OpenMP) for the largest configs — input generators only.

xxz_csr_fast(L, J1, delta, h, J2) returns exactly the arrays of models.xxz_csr (bit-identical;
tests/test_workloads.py checks it) in O(nnz) C instead of numpy, for L = 26 (1.8e9 nnz)."""
from __future__ import annotations

import ctypes as C
import os
import subprocess

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
SRC = os.path.join(HERE, "cbuild", "xxz.c")
LIB = os.path.join(HERE, "cbuild", "libwlbuild.so")
_lib = None


def build(force=False):
    if force or not os.path.exists(LIB) or os.path.getmtime(LIB) < os.path.getmtime(SRC):
        subprocess.check_call(["gcc", "-O2", "-ffp-contract=off", "-fno-fast-math", "-fopenmp", "-shared", "-fPIC",
                               "-o", LIB + ".tmp", SRC])
        os.replace(LIB + ".tmp", LIB)
    return LIB


def _load():
    global _lib
    if _lib is None:
        build()
        _lib = C.CDLL(LIB)
        _lib.xxz_rowptr.argtypes = [C.c_int, C.c_double, C.c_double, C.c_int64, C.c_int64, C.c_void_p]
        _lib.xxz_fill.argtypes = [C.c_int, C.c_double, C.c_double, C.c_double, C.c_void_p, C.c_int64, C.c_int64,
                                  C.c_void_p, C.c_void_p, C.c_void_p]
    return _lib


def xxz_csr_fast(L, J1, delta, h, J2=0.0, r0=0, r1=None):
    """CSR of rows [r0, r1) (default: all rows); rowptr local (starts at 0), columns global."""
    lib = _load()
    n = 1 << L
    r1 = n if r1 is None else r1
    rowptr = np.empty(r1 - r0 + 1, dtype=np.int64)
    lib.xxz_rowptr(L, float(J1), float(J2), r0, r1, rowptr.ctypes.data)
    nnz = int(rowptr[-1])
    col = np.empty(nnz, dtype=np.int32)
    val = np.empty(nnz, dtype=np.float64)
    hh = np.ascontiguousarray(h, dtype=np.float64)
    lib.xxz_fill(L, float(J1), float(J2), float(delta), hh.ctypes.data, r0, r1, rowptr.ctypes.data,
                 col.ctypes.data, val.ctypes.data)
    return rowptr, col, val
