"""C-ABI library checks that need no GPU: the library loads, exports every symbol that
include/te.h declares, fails loudly without a device, and the host-only halo plan is
bit-exact against an independent numpy construction."""
import ctypes
import os
import re

import numpy as np
import pytest

from paper_2205_15346_b200 import build as B
from paper_2205_15346_b200 import te

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


@pytest.fixture(scope="module")
def lib():
    B.build()
    return te.load()


def declared_symbols():
    src = open(os.path.join(ROOT, "include", "te.h")).read()
    src = re.sub(r"/\*.*?\*/", "", src, flags=re.S)
    return sorted(set(re.findall(r"\b(te_[a-z0-9_]+)\s*\(", src)))


def test_header_declares_core_three():
    syms = declared_symbols()
    for s in ("te_create_csr", "te_evolve", "te_destroy"):
        assert s in syms


def test_library_exports_every_declared_symbol(lib):
    raw = ctypes.CDLL(B.LIB)
    missing = [s for s in declared_symbols() if not hasattr(raw, s)]
    assert not missing, missing


def test_version_and_no_device_behaviour(lib):
    assert "sm_100a" in te.te_version()
    import torch
    if torch.cuda.is_available():
        pytest.skip("device present")
    with pytest.raises(te.TEError) as ei:
        te.te_create_csr(2, np.array([0, 1, 2]), np.array([1, 0]), np.array([1.0, 1.0]))
    assert ei.value.status == 8  # TE_ERR_CUDA: no silent CPU fallback


def test_bad_csr_rejected_on_host(lib):
    with pytest.raises(te.TEError) as ei:
        te.te_create_csr(2, np.array([1, 1, 2]), np.array([1, 0]), np.array([1.0, 1.0]))
    assert ei.value.status == 2
    with pytest.raises(te.TEError) as ei:
        te.te_create_csr(2, np.array([0, 2, 1]), np.array([1, 0]), np.array([1.0, 1.0]))
    assert ei.value.status == 2


def numpy_halo_plan(P, rank, row_starts, cols):
    rb, re_ = row_starts[rank], row_starts[rank + 1]
    remote = np.unique(cols[(cols < rb) | (cols >= re_)])
    owner = np.searchsorted(row_starts, remote, side="right") - 1
    counts = np.bincount(owner, minlength=P).astype(np.int64)
    local = np.where((cols >= rb) & (cols < re_), cols - rb,
                     (re_ - rb) + np.searchsorted(remote, cols)).astype(np.int32)
    return local, counts, remote


@pytest.mark.parametrize("P", [2, 3, 4, 8])
def test_halo_plan_bit_exact(lib, P):
    from workloads import models
    L = 10
    n = 1 << L
    rp, col, _ = models.xxz_csr(L, 1.0, 0.5, models.xxz_fields(L, 2), J2=0.5)
    row_starts = np.array([(q * n) // P for q in range(P + 1)], dtype=np.int64)
    for rank in range(P):
        a, b = row_starts[rank], row_starts[rank + 1]
        cols = col[rp[a]: rp[b]].astype(np.int64)
        cl, rc, halo = te.te_halo_plan(P, rank, row_starts, cols)
        ncl, nrc, nhalo = numpy_halo_plan(P, rank, row_starts, cols)
        assert np.array_equal(cl, ncl) and np.array_equal(rc, nrc) and np.array_equal(halo, nhalo)
        assert rc[rank] == 0


def test_halo_plan_rejects_out_of_range(lib):
    with pytest.raises(te.TEError):
        te.te_halo_plan(2, 0, np.array([0, 4, 8]), np.array([0, 9], dtype=np.int64))
