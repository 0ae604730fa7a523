"""Row-parallel build of the involution matrices (configs 1 and 4) — input generation only.

``models.involution_csr`` is row-local (every candidate of row r depends only on r and the seed),
so rows can be built in independent chunks by a process pool and concatenated; the result is
byte-identical to the single-process build (tests/test_workloads.py).  Config 4 (2^24 rows,
5.4e8 entries) takes ~6 min single-threaded."""
from __future__ import annotations

import multiprocessing as mp
import os

import numpy as np

from . import models


def _chunk(args):
    n, seed, n_uniform, n_band, diagonal, a, b = args
    return models.involution_csr(n, seed, n_uniform=n_uniform, n_band=n_band, diagonal=diagonal,
                                 rows=np.arange(a, b, dtype=np.int64))


def involution_csr_parallel(n: int, seed: int, n_uniform: int, n_band: int = 0, diagonal: bool = True,
                            nproc: int | None = None, chunk: int = 1 << 19):
    nproc = nproc or min(32, os.cpu_count() or 1)
    bounds = [(a, min(n, a + chunk)) for a in range(0, n, chunk)]
    jobs = [(n, seed, n_uniform, n_band, diagonal, a, b) for a, b in bounds]
    if nproc <= 1 or len(jobs) == 1:
        parts = [_chunk(j) for j in jobs]
    else:
        with mp.get_context("forkserver").Pool(nproc) as pool:  # no fork of a threaded parent
            parts = pool.map(_chunk, jobs, chunksize=1)
    nnz = sum(int(p[0][-1]) for p in parts)
    rowptr = np.empty(n + 1, dtype=np.int64)
    col = np.empty(nnz, dtype=np.int32)
    val = np.empty(nnz, dtype=parts[0][2].dtype)
    rowptr[0] = 0
    off = 0
    for (a, b), (rp, c, v) in zip(bounds, parts):
        k = int(rp[-1])
        rowptr[a + 1: b + 1] = rp[1:] + off
        col[off: off + k] = c
        val[off: off + k] = v
        off += k
    return rowptr, col, val
