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


def test_binding_rejects_bad_buffers_before_the_c_call(lib):
    """The binding checks every buffer it hands to C (the library copies n * 16 bytes each way):
    wrong length, dtype, strides or a read-only output raise ValueError before any C call, so a
    short vector can never be read or written past its end."""
    h = te.Handle(None, 4, True)  # never reaches C: validation comes first
    good = np.zeros(4, dtype=np.complex128)
    good[0] = 1
    with pytest.raises(ValueError):
        te.te_evolve(h, np.zeros(3, complex), 1.0, 1e-8, 4)
    for out in (np.zeros(4), np.zeros(3, complex), np.zeros(8, complex)[::2], np.zeros((2, 2), complex)):
        with pytest.raises(ValueError):
            te.te_evolve(h, good, 1.0, 1e-8, 4, out=out)
    ro = np.zeros(4, complex)
    ro.flags.writeable = False
    with pytest.raises(ValueError):
        te.te_evolve(h, good, 1.0, 1e-8, 4, out=ro)
    with pytest.raises(ValueError):
        te.te_evolve_schedule(h, np.zeros(5, complex), [0.1], 1e-8, 4)
    with pytest.raises(ValueError):
        te.te_evolve_sampled(h, np.zeros(2, complex), 1.0, 1e-8, 4, [0.5])
    with pytest.raises(ValueError):
        te.te_krylov_basis(h, np.zeros(6, complex), 3, 1e-9)
    import torch
    for bad in (torch.zeros(4, dtype=torch.complex64), torch.zeros(4, dtype=torch.complex128),  # not on CUDA
                torch.zeros(5, dtype=torch.complex128)):
        with pytest.raises(ValueError):
            te.te_evolve_dev(h, bad, 1.0, 1e-8, 4, bad)
    with pytest.raises(ValueError):
        te.te_create_csr(2, np.array([0, 1]), np.array([1, 0]), np.array([1.0, 1.0]))      # rowptr too short
    with pytest.raises(ValueError):
        te.te_create_csr(2, np.array([0, 1, 3]), np.array([1, 0]), np.array([1.0, 1.0]))   # col shorter than nnz


@pytest.mark.parametrize("m", [1, 2, 3, 8, 40, 64])
def test_host_eigensolver_against_numpy(lib, m):
    """The library's host tridiagonal eigensolver (te_small_eig, implicit symmetric QR)
    against numpy.linalg.eigh: eigenvalues, T U = U diag(lam), U orthogonal; also a matrix with
    negligible couplings (deflation), a zero matrix and repeated eigenvalues."""
    g = np.random.default_rng(m)
    cases = [(g.standard_normal(m), np.abs(g.standard_normal(max(0, m - 1))) + 0.1)]
    if m > 2:
        b = np.abs(g.standard_normal(m - 1)) + 0.1
        b[m // 2] = 1e-300
        cases += [(g.standard_normal(m), b), (np.zeros(m), np.zeros(m - 1)), (np.ones(m), np.zeros(m - 1) + 1e-17)]
    for a, b in cases:
        T = np.diag(a) + np.diag(b, 1) + np.diag(b, -1) if m > 1 else np.diag(a)
        lam, U = te.te_small_eig(a, b)
        assert np.allclose(np.sort(lam), np.linalg.eigvalsh(T), atol=1e-13 * max(1, np.abs(T).max()), rtol=0)
        assert np.abs(T @ U - U * lam).max() <= 1e-13 * max(1, np.abs(T).max()) * m
        assert np.abs(U.T @ U - np.eye(m)).max() <= 1e-13 * m


@pytest.mark.parametrize("first", [True, False])
@pytest.mark.parametrize("integrator", [0, 1])
def test_host_step_search_matches_oracle(lib, first, integrator):
    """The library's host step search (te_step_search: Eq. 16 integral + Alg. 1 step 2) against the
    oracle's find_step on the same T: the same step (both follow reading O-6 with the same
    decisions) and error integrals within the quadrature tolerance 1e-3 max(e, tol_rate tau)."""
    from oracle import krylov as K
    for seed in range(6):
        g = np.random.default_rng(100 + seed)
        m = 8 + seed
        a = g.standard_normal(m)
        b = np.abs(g.standard_normal(m)) + 0.3
        h = b[m - 1] * 1e-3
        tol_rate, t = 1e-6, 3.0
        lam, U = K.small_eig(a, b[: m - 1])
        f = lambda x: K.integrand(lam, U, h, x)  # noqa: E731
        integ = (lambda lo, hi: K.tanh_sinh(f, lo, hi, floor=tol_rate * (hi - lo))[0]) if integrator == 0 else \
            (lambda lo, hi: K.gauss_legendre(f, lo, hi)[0])
        to, eo = K.find_step(integ, False, first, 0.4, t, tol_rate, t)
        tg, eg, ok = te.te_step_search(a, b[: m - 1], h, False, first, 0.4, t, tol_rate, t, integrator)
        assert ok
        assert abs(tg - to) <= 1e-12 * t
        assert abs(eg - eo) <= 1e-3 * max(eo, tol_rate * to) + 1e-18
        assert eg <= tol_rate * tg * (1 + 1e-12)
    # breakdown: the remaining time in one step
    tg, eg, _ = te.te_step_search(a, b[: m - 1], 0.0, True, first, 0.4, t, tol_rate, t, integrator)
    assert tg == t and eg == 0.0
