"""GPU parity: the CUDA path (through the C ABI) against the oracle, element by element on
the same seeded inputs, plus full-size properties.  Tolerances (BASELINE.json north star):
||dv||_2 <= 1e-10 with the step schedule forced identical; <= tol + 1e-12 with adaptive
stepping (both runs individually satisfy their bound, reading C16/C18)."""
import math

import numpy as np
import pytest
import scipy.linalg as sl
import scipy.sparse as sp

from oracle import krylov as K
from workloads import configs, models

pytestmark = pytest.mark.gpu


def csr_from_dense(A):
    S = sp.csr_matrix(A)
    S.sort_indices()
    return S.indptr.astype(np.int64), S.indices.astype(np.int32), S.data


def small_cases():
    return [
        ("cfg1_n4096", configs.build(1)),
        ("xxz_L12", configs.build(2, L=12)),
        ("bh_L6_N6_ragged", configs.build(3, L=6, N=6)),
        ("xxznnn_L12", configs.build(5, L=12)),
        ("banded_n8192", configs.build(4, n=8192)),
        ("cfg1_n1000_ragged", configs.build(1, n=1000)),
    ]


CASES = small_cases()


KERNEL_SETS = [(2, 8), (2, 7), (2, 6), (3, 7), (5, 7)]
KERNEL_IDS = ["hybrid-spmvxs", "hybrid-spmvring", "hybrid-spmvsell", "tma", "regacc"]


@pytest.mark.parametrize("kset", KERNEL_SETS, ids=KERNEL_IDS)
@pytest.mark.parametrize("name,c", CASES, ids=[x[0] for x in CASES])
def test_krylov_basis_matches_oracle(gpu_lib, name, c, kset):
    te = gpu_lib
    h = te.te_create_csr(c["n"], c["rowptr"], c["col"], c["val"])
    te.te_set_option(h, te.TE_OPT_KERNELS, kset[0])
    te.te_set_option(h, te.TE_OPT_SPMV, kset[1])
    m = min(c["m"], c["n"])
    tol_rate = c["tol"] / c["t"]
    g = te.te_krylov_basis(h, c["v0"], m, tol_rate, want_V=True)
    o = K.arnoldi(lambda x: K.spmv(c["rowptr"], c["col"], c["val"], x), c["v0"], m, tol_rate)
    assert g["m_eff"] == o["m_eff"] and g["breakdown"] == o["breakdown"]
    k = g["m_eff"]
    scale = max(1.0, np.abs(o["alpha"]).max(), np.abs(o["beta"]).max())
    assert np.abs(g["alpha"] - o["alpha"]).max() <= 1e-12 * scale
    assert np.abs(g["beta"] - o["beta"]).max() <= 1e-12 * scale
    assert np.linalg.norm(g["V"] - o["V"]) <= 1e-10
    # CGS2 orthonormality of the GPU basis itself
    V = g["V"]
    assert np.abs(V.conj().T @ V - np.eye(k)).max() <= 1e-13
    h.close()


PIPE_CASES = [("xxznnn_L12", configs.build(5, L=12)), ("s5_K4_N20", configs.build(6, K=4, K1=4, Nm=2, N0=20, Nc=20)),
              ("cfg1_n1000_ragged", configs.build(1, n=1000))]


RING_CASES = PIPE_CASES + [("long_rows", None)]


def _long_row_case():
    """Rows longer than one ring SpMV tile (2816-5632 entries) next to short ones."""
    n = 3000
    g = np.random.default_rng(11)
    A = np.zeros((n, n), complex)
    A[np.arange(n), np.arange(n)] = g.standard_normal(n)
    for r in (5, 1700):
        cols = g.choice(n, 1500, replace=False)
        A[r, cols] = g.standard_normal(1500) + 1j * g.standard_normal(1500)
    A = (A + A.conj().T) / 2
    rp, col, val = csr_from_dense(A)
    v0 = g.standard_normal(n) + 1j * g.standard_normal(n)
    return dict(n=n, rowptr=rp, col=col, val=val, v0=v0 / np.linalg.norm(v0), t=1.0, tol=1e-8, m=12)


@pytest.mark.parametrize("stages", [3, 4])
@pytest.mark.parametrize("tpr", [1, 2, 4, 8])
@pytest.mark.parametrize("halo", [0, 1])
@pytest.mark.parametrize("name,c", RING_CASES, ids=[x[0] for x in RING_CASES])
def test_spmv_ring_variants(gpu_lib, name, c, tpr, halo, stages, monkeypatch):
    """Warp-specialised ring SpMV (TE_OPT_SPMV = 7) for every lanes-per-row choice and both ring
    depths, plain and halo-aware, including rows longer than a tile (one warp from global memory),
    vs the oracle."""
    te = gpu_lib
    if c is None:
        c = _long_row_case()
    monkeypatch.setenv("TE_SPMV_RING_STAGES", str(stages))
    monkeypatch.setenv("TE_SPMV_RING_TPR", str(tpr))
    monkeypatch.setenv("TE_SPMV_FORCE_HALO", str(halo))
    h = te.te_create_csr(c["n"], c["rowptr"], c["col"], c["val"])
    te.te_set_option(h, te.TE_OPT_SPMV, 7)
    g = te.te_krylov_basis(h, c["v0"], 12, c["tol"] / c["t"], want_V=True)
    o = K.arnoldi(lambda x: K.spmv(c["rowptr"], c["col"], c["val"], x), c["v0"], 12, c["tol"] / c["t"])
    scale = max(1.0, np.abs(o["alpha"]).max(), np.abs(o["beta"]).max())
    assert g["m_eff"] == o["m_eff"]
    assert np.abs(g["alpha"] - o["alpha"]).max() <= 1e-12 * scale
    assert np.linalg.norm(g["V"] - o["V"]) <= 1e-10
    h.close()


def _complex_dict_case():
    """XXZ+NNN at L=10 with complex couplings: off-diagonal entries times e^{+-i phi} (Hermitian),
    so the value dictionary holds complex values."""
    c = dict(configs.build(5, L=10))
    rows = np.repeat(np.arange(c["n"]), np.diff(c["rowptr"]))
    ph = np.where(c["col"] > rows, np.exp(0.7j), np.exp(-0.7j))
    c["val"] = np.where(c["col"] == rows, c["val"] + 0j, c["val"] * ph)
    return c


XS_CASES = RING_CASES + [("xxz_L14", configs.build(2, L=14)), ("bh_L7_N7", configs.build(3, L=7, N=7)),
                         ("banded_n8192", configs.build(4, n=8192)), ("xxznnn_L10_cplx", _complex_dict_case())]


@pytest.mark.parametrize("ecap", [0, 256])
@pytest.mark.parametrize("tpr", [1, 2, 4, 8])
@pytest.mark.parametrize("halo", [0, 1])
@pytest.mark.parametrize("name,c", XS_CASES, ids=[x[0] for x in XS_CASES])
def test_spmv_xs_variants(gpu_lib, name, c, tpr, halo, ecap, monkeypatch):
    """Staged-x ring SpMV (TE_OPT_SPMV = 8) for every lanes-per-row choice, plain and halo-aware,
    with the default tile size and with 256-entry tiles (many tiles per CTA: the 2-stage ring wraps,
    ranges cut by the slot budget), on matrices whose x windows are fully staged (spin chains,
    bosons), partly staged (banded + uniform) and hardly at all (uniform random columns, long
    rows: the global-gather path), real and complex values, vs the oracle's Arnoldi basis."""
    te = gpu_lib
    if c is None:
        c = _long_row_case()
    monkeypatch.setenv("TE_SPMV_XS_TPR", str(tpr))
    monkeypatch.setenv("TE_SPMV_FORCE_HALO", str(halo))
    if ecap:
        monkeypatch.setenv("TE_SPMV_XS_ECAP", str(ecap))
    h = te.te_create_csr(c["n"], c["rowptr"], c["col"], c["val"])
    te.te_set_option(h, te.TE_OPT_SPMV, 8)
    assert te.te_get_option(h, te.TE_OPT_SPMV) == 8
    g = te.te_krylov_basis(h, c["v0"], 12, c["tol"] / c["t"], want_V=True)
    o = K.arnoldi(lambda x: K.spmv(c["rowptr"], c["col"], c["val"], x), c["v0"], 12, c["tol"] / c["t"])
    scale = max(1.0, np.abs(o["alpha"]).max(), np.abs(o["beta"]).max())
    assert g["m_eff"] == o["m_eff"]
    assert np.abs(g["alpha"] - o["alpha"]).max() <= 1e-12 * scale
    assert np.abs(g["beta"] - o["beta"]).max() <= 1e-12 * scale
    assert np.linalg.norm(g["V"] - o["V"]) <= 1e-10
    h.close()


def _principal_submatrix(c, m):
    """Rows/columns [0, m) of a CSR matrix (Hermitian stays Hermitian): ragged slices, rows that
    lose entries."""
    rp, col, val = c["rowptr"], c["col"], c["val"]
    keep = np.zeros(len(col), dtype=bool)
    keep[: rp[m]] = col[: rp[m]] < m
    rows = np.repeat(np.arange(m), np.diff(rp[: m + 1]))
    nrp = np.zeros(m + 1, dtype=np.int64)
    np.add.at(nrp, rows[keep[: rp[m]]] + 1, 1)
    v0 = c["v0"][:m] / np.linalg.norm(c["v0"][:m]) if np.linalg.norm(c["v0"][:m]) > 0 else np.ones(m, complex) / np.sqrt(m)
    return dict(c, n=m, rowptr=np.cumsum(nrp), col=col[keep].astype(np.int32), val=val[keep], v0=v0.astype(np.complex128))


def _no_diag_case():
    """XXZ L=10 without its diagonal (rows with no diagonal entry, some rows empty)."""
    c = dict(configs.build(2, L=10))
    rows = np.repeat(np.arange(c["n"]), np.diff(c["rowptr"]))
    keep = c["col"] != rows
    nrp = np.zeros(c["n"] + 1, dtype=np.int64)
    np.add.at(nrp, rows[keep] + 1, 1)
    v0 = np.random.default_rng(3).standard_normal(c["n"]) + 0j
    return dict(c, rowptr=np.cumsum(nrp), col=c["col"][keep], val=c["val"][keep], v0=v0 / np.linalg.norm(v0))


SW_CASES = [("xxz_L12", configs.build(2, L=12)), ("xxznnn_L12", configs.build(5, L=12)), ("xxz_L14", configs.build(2, L=14)),
            ("xxznnn_L10_cplx", _complex_dict_case()), ("xxz_L12_ragged1000", _principal_submatrix(configs.build(2, L=12), 1000)),
            ("xxz_L10_nodiag", _no_diag_case()), ("bh_L7_N7", configs.build(3, L=7, N=7)),
            ("xxz_L5", configs.build(2, L=5))]


@pytest.mark.parametrize("panel", [0, 1, 3, 4])
@pytest.mark.parametrize("bits", [8, 16])
@pytest.mark.parametrize("name,c", SW_CASES, ids=[x[0] for x in SW_CASES])
def test_spmv_sw_variants(gpu_lib, name, c, bits, panel, monkeypatch):
    """Slot-window SELL-32 SpMV (TE_OPT_SPMV = 9) vs the oracle's Arnoldi basis: spin chains (real
    and complex dictionary values), a ragged last slice, rows without a diagonal and empty rows, a
    single slice (n = 32), and a boson matrix whose windows align poorly (the padding check is
    overridden for all of these small matrices); 8-bit entries (3-bit code, dictionaries of <= 7
    values: the spin chains) and 16-bit entries; one pass, and the two-pass panel sweep (panels of
    2^panel slices: near windows in row order, far windows added in the permuted slice order)."""
    te = gpu_lib
    monkeypatch.setenv("TE_SPMV_SW_FORCE", "1")  # small chains: more slices straddle the window edges
    monkeypatch.setenv("TE_SPMV_SW_BITS", str(bits))  # 8-bit entries apply to dictionaries of <= 7 values
    monkeypatch.setenv("TE_SPMV_SW_PANEL", str(panel))
    h = te.te_create_csr(c["n"], c["rowptr"], c["col"], c["val"])
    te.te_set_option(h, te.TE_OPT_SPMV, 9)
    assert te.te_get_option(h, te.TE_OPT_SPMV) == 9
    assert te.te_get_option(h, te.TE_INFO_SW_FILL) > 0
    nsl = (c["n"] + 31) // 32
    two_pass = panel > 0 and (1 << panel) < nsl
    assert te.te_get_option(h, te.TE_INFO_SW_PANEL) == (panel if two_pass else 0)
    if two_pass and name.startswith("xxz"):
        assert 0 < te.te_get_option(h, te.TE_INFO_SW_FAR) < 1
    m = min(12, c["n"] - 1)
    g = te.te_krylov_basis(h, c["v0"], m, c["tol"] / c["t"], want_V=True)
    o = K.arnoldi(lambda x: K.spmv(c["rowptr"], c["col"], c["val"], x), c["v0"], m, c["tol"] / c["t"])
    scale = max(1.0, np.abs(o["alpha"]).max(), np.abs(o["beta"]).max())
    assert g["m_eff"] == o["m_eff"]
    assert np.abs(g["alpha"] - o["alpha"]).max() <= 1e-12 * scale
    assert np.abs(g["beta"] - o["beta"]).max() <= 1e-12 * scale
    assert np.linalg.norm(g["V"] - o["V"]) <= 1e-10
    h.close()


CB_CASES = [("cfg1_n4096", configs.build(1)), ("banded_n8192", configs.build(4, n=8192)),
            ("bh_L6_N6_ragged", configs.build(3, L=6, N=6)), ("cfg1_n1000_ragged", configs.build(1, n=1000)),
            ("xxz_L10_nodiag", _no_diag_case())]


@pytest.mark.parametrize("kb", [1, 2])
@pytest.mark.parametrize("name,c", CB_CASES, ids=[x[0] for x in CB_CASES])
def test_spmv_colblk_variants(gpu_lib, name, c, kb, monkeypatch):
    """Column-blocked ring SpMV (TE_OPT_SPMV = 10): one ring pass per column block of x (kb KB of x
    per block: 4-128 blocks), passes > 0 accumulating into W, lanes per row chosen per block; rows
    with no entry in a block, empty rows, a ragged last block; vs the oracle's Arnoldi basis and a
    forced-schedule evolution."""
    te = gpu_lib
    monkeypatch.setenv("TE_SPMV_COLBLK_MB", str(kb / 1024.0))
    h = te.te_create_csr(c["n"], c["rowptr"], c["col"], c["val"])
    te.te_set_option(h, te.TE_OPT_SPMV, 10)
    assert te.te_get_option(h, te.TE_OPT_SPMV) == 10
    g = te.te_krylov_basis(h, c["v0"], 12, c["tol"] / c["t"], want_V=True)
    o = K.arnoldi(lambda x: K.spmv(c["rowptr"], c["col"], c["val"], x), c["v0"], 12, c["tol"] / c["t"])
    scale = max(1.0, np.abs(o["alpha"]).max(), np.abs(o["beta"]).max())
    assert g["m_eff"] == o["m_eff"]
    assert np.abs(g["alpha"] - o["alpha"]).max() <= 1e-12 * scale
    assert np.abs(g["beta"] - o["beta"]).max() <= 1e-12 * scale
    assert np.linalg.norm(g["V"] - o["V"]) <= 1e-10
    # a forced-schedule evolution through the same kernel matches the oracle
    t = min(c["t"], 1.0)
    v, st = te.te_evolve(h, c["v0"], t, c["tol"], 12)
    sched = te.te_get_schedule(h)
    ref = K.evolve(c["rowptr"], c["col"], c["val"], c["v0"], t, c["tol"], 12, schedule=[x[0] for x in sched])
    assert np.linalg.norm(v - ref["v"]) <= 1e-10
    h.close()


def test_spmv_sw_not_applicable(gpu_lib):
    """More than 255 distinct off-diagonal values: TE_OPT_SPMV 9 is refused (TE_ERR_ARG) and the
    handle keeps its SpMV."""
    te = gpu_lib
    c = configs.build(1, n=2048)
    h = te.te_create_csr(c["n"], c["rowptr"], c["col"], c["val"])
    before = te.te_get_option(h, te.TE_OPT_SPMV)
    with pytest.raises(te.TEError):
        te.te_set_option(h, te.TE_OPT_SPMV, 9)
    assert te.te_get_option(h, te.TE_OPT_SPMV) == before
    h.close()


def test_spmv_default_choice(gpu_lib):
    """At create: the slot-window SELL-32 for spin chains (dictionary + aligned windows, padding
    <= 2.0x with 8-bit entries), the staged-x ring when its plan stages >= 95 % of the entries
    (bosons, n >= 65536), the plain ring otherwise (uniform random columns, small n); TE_OPT_SPMV
    switches either way with the same result."""
    te = gpu_lib
    # (a random matrix must be large enough that a tile's uniform columns are isolated in x)
    for c, want in ((configs.build(5, L=18), 9), (configs.build(2, L=12), None), (configs.build(3, L=10, N=10), 8),
                    (configs.build(3, L=7, N=7), 7), (configs.build(1, n=1 << 18), 7)):
        h = te.te_create_csr(c["n"], c["rowptr"], c["col"], c["val"])
        fill = te.te_get_option(h, te.TE_INFO_SW_FILL)
        if want is None:  # small chain: the slot-window format iff its padding is within the limit
            assert fill > 0
            want = 9 if fill <= 2.0 else (8 if c["n"] >= 65536 else 7)
        assert te.te_get_option(h, te.TE_OPT_SPMV) == want, fill
        if c["cfg"] in (2, 5):
            assert (want == 9) == (0 < fill <= 2.0)
        other = 7 if want in (8, 9) else 8
        v1, _ = te.te_evolve(h, c["v0"], 0.5, 1e-9, 16)
        te.te_set_option(h, te.TE_OPT_SPMV, other)
        assert te.te_get_option(h, te.TE_OPT_SPMV) == other
        v2, _ = te.te_evolve(h, c["v0"], 0.5, 1e-9, 16)
        assert np.linalg.norm(v1 - v2) <= 1e-12
        h.close()


@pytest.mark.parametrize("halo", [0, 1])
@pytest.mark.parametrize("name,c", PIPE_CASES, ids=[x[0] for x in PIPE_CASES])
def test_spmv_sell_halo_variants(gpu_lib, name, c, halo, monkeypatch):
    """SELL-32-sigma SpMV (TE_OPT_SPMV = 6), plain and halo-aware instantiation, vs the oracle."""
    te = gpu_lib
    monkeypatch.setenv("TE_SPMV_FORCE_HALO", str(halo))
    h = te.te_create_csr(c["n"], c["rowptr"], c["col"], c["val"])
    te.te_set_option(h, te.TE_OPT_SPMV, 6)
    g = te.te_krylov_basis(h, c["v0"], 12, c["tol"] / c["t"], want_V=True)
    o = K.arnoldi(lambda x: K.spmv(c["rowptr"], c["col"], c["val"], x), c["v0"], 12, c["tol"] / c["t"])
    scale = max(1.0, np.abs(o["alpha"]).max(), np.abs(o["beta"]).max())
    assert g["m_eff"] == o["m_eff"]
    assert np.abs(g["alpha"] - o["alpha"]).max() <= 1e-12 * scale
    assert np.linalg.norm(g["V"] - o["V"]) <= 1e-10
    h.close()


def test_spmv_sell_refuses_uneven_rows(gpu_lib):
    """A few rows much longer than the rest would make the padded SELL copy several times the
    CSR: selecting it fails with TE_ERR_ARG and the handle keeps working on its previous SpMV."""
    te = gpu_lib
    c = _long_row_case()
    h = te.te_create_csr(c["n"], c["rowptr"], c["col"], c["val"])
    with pytest.raises(te.TEError):
        te.te_set_option(h, te.TE_OPT_SPMV, 6)
    v, st = te.te_evolve(h, c["v0"], 0.5, 1e-8, 12)
    assert st["err_bound"] <= 1e-8
    h.close()


@pytest.mark.parametrize("name,c", CASES, ids=[x[0] for x in CASES])
def test_evolve_forced_and_adaptive(gpu_lib, name, c):
    te = gpu_lib
    h = te.te_create_csr(c["n"], c["rowptr"], c["col"], c["val"])
    t, tol, m = c["t"], c["tol"], c["m"]
    if c["n"] > 5000:
        t = min(t, 2.0)
    v, st = te.te_evolve(h, c["v0"], t, tol, m)
    sched = te.te_get_schedule(h)
    assert st["n_restarts"] == len(sched) and st["err_bound"] <= tol
    assert math.fsum(s[0] for s in sched) == pytest.approx(t, abs=1e-12)
    # forced identical schedule -> 1e-10
    ref = K.evolve(c["rowptr"], c["col"], c["val"], c["v0"], t, tol, m, schedule=[s[0] for s in sched])
    assert np.linalg.norm(v - ref["v"]) <= 1e-10
    assert [s[1] for s in ref["schedule"]] == [s[1] for s in sched]
    # per-step bounds agree within the quadrature's own tolerance (rel. 1e-3) plus the
    # absolute floor of the integrand: f = h |sum_k c_k e^{-i lam_k tau}| is a small matrix
    # element formed with cancellation, accurate to ~ h m eps absolute (h <= ||H||_1)
    for (tg, _, eg), (to, _, eo) in zip(sched, ref["schedule"]):
        floor = 10.0 * tg * st["one_norm"] * m * 2.0 ** -52
        assert abs(eg - eo) <= 1e-3 * eo + floor
    # adaptive vs adaptive -> tol + 1e-12
    ada = K.evolve(c["rowptr"], c["col"], c["val"], c["v0"], t, tol, m)
    assert np.linalg.norm(v - ada["v"]) <= tol + 1e-12
    # schedule of the GPU and of the oracle coincide (same algorithm; equal decisions)
    assert len(ada["schedule"]) == len(sched)
    assert max(abs(a[0] - b[0]) for a, b in zip(ada["schedule"], sched)) <= 1e-12 * t
    # the explicitly forced path of the library reproduces the adaptive result
    vf, stf = te.te_evolve_schedule(h, c["v0"], [s[0] for s in sched], tol, m)
    assert np.linalg.norm(vf - v) <= 1e-13
    h.close()


def test_dense_exponential_and_bound(gpu_lib):
    te = gpu_lib
    c = configs.build(1)
    h = te.te_create_csr(c["n"], c["rowptr"], c["col"], c["val"])
    v, st = te.te_evolve(h, c["v0"], c["t"], c["tol"], c["m"])
    H = sp.csr_matrix((c["val"], c["col"], c["rowptr"])).toarray()
    lam, U = np.linalg.eigh(H)
    ve = U @ (np.exp(-1j * lam * c["t"]) * (U.conj().T @ c["v0"]))
    err = np.linalg.norm(v - ve)
    assert err <= st["err_bound"] + 10 * st["roundoff_total"]
    assert st["err_bound"] <= c["tol"]


@pytest.mark.parametrize("kset,ortho", [((2, 7), 0), ((3, 7), 0), ((5, 7), 0), ((2, 6), 0), ((2, 7), 2), ((2, 7), 1),
                                        ((3, 7, "runtime-R"), 0), ((3, 7, "runtime-R"), 2), ((2, 7, "norm-tma"), 0),
                                        ((3, 7, "norm-tma-runtime-R"), 0)],
                         ids=["hybrid-ring", "tma", "regacc", "hybrid-sell", "cgs2gram", "lanczos3", "tma-runtimeR",
                              "cgs2gram-runtimeR", "norm-tma", "norm-tma-runtimeR"])
def test_maximum_krylov_dimension(gpu_lib, kset, ortho, monkeypatch):
    """m = TE_M_MAX = 64: every column group of the projection kernels (register partials and the
    16-wide butterflies up to column 63, the 64 x 64 Gram matrix of f2; the TMA kernels' builds with
    a compile-time sub-tile count for 9-14 / 15-16 / 17-30 / 31-64 columns, and their runtime-R
    fallback) against the oracle; one adaptive evolution at m = 64; m = 65 is rejected."""
    te = gpu_lib
    monkeypatch.setenv("TE_PROJ_CONST_R", "0" if len(kset) > 2 and "runtime-R" in kset[2] else "1")
    # K3 (update + norm) on the TMA ring (k_proj_tma<4>; the default from 2^22 rows) at every column count
    monkeypatch.setenv("TE_NORM_TMA", "1" if len(kset) > 2 and "norm-tma" in kset[2] else "0")
    c = configs.build(1)
    h = te.te_create_csr(c["n"], c["rowptr"], c["col"], c["val"])
    te.te_set_option(h, te.TE_OPT_KERNELS, kset[0])
    te.te_set_option(h, te.TE_OPT_SPMV, kset[1])
    te.te_set_option(h, te.TE_OPT_ORTHO, ortho)
    mode = ["cgs2", "lanczos3", "cgs2gram"][ortho]
    g = te.te_krylov_basis(h, c["v0"], 64, 1e-14, want_V=True)
    o = K.arnoldi(lambda x: K.spmv(c["rowptr"], c["col"], c["val"], x), c["v0"], 64, 1e-14, ortho=mode)
    assert g["m_eff"] == o["m_eff"] == 64
    scale = max(1.0, np.abs(o["alpha"]).max(), np.abs(o["beta"]).max())
    # the paper-literal recurrence loses orthogonality over 64 steps; both sides follow it alike
    tolr = 1e-12 if ortho != 1 else 1e-9
    assert np.abs(g["alpha"] - o["alpha"]).max() <= tolr * scale
    assert np.abs(g["beta"] - o["beta"]).max() <= tolr * scale
    if ortho != 1:
        assert np.linalg.norm(g["V"] - o["V"]) <= 1e-10
    v, st = te.te_evolve(h, c["v0"], 2.0, 1e-8, 64)
    r = K.evolve(c["rowptr"], c["col"], c["val"], c["v0"], 2.0, 1e-8, 64, ortho=mode)
    assert st["err_bound"] <= 1e-8 and np.linalg.norm(v - r["v"]) <= 1e-8 + 1e-12
    with pytest.raises(te.TEError):
        te.te_evolve(h, c["v0"], 2.0, 1e-8, 65)
    h.close()


@pytest.mark.parametrize("spmv", [7, 6])
def test_fresh_handles_bitwise_reproducible(gpu_lib, spmv):
    """Every kernel is deterministic, so the same decomposition / evolution on freshly created handles
    (allocations recycled back to back) must agree bit for bit.  This is what exposed workspace
    initialisation that was not ordered with the handle's stream."""
    te = gpu_lib
    for c in (configs.build(5, L=12), configs.build(1, n=3001)):
        ref = None
        for _ in range(25):
            h = te.te_create_csr(c["n"], c["rowptr"], c["col"], c["val"])
            te.te_set_option(h, te.TE_OPT_SPMV, spmv)
            g = te.te_krylov_basis(h, c["v0"], 16, 1e-12, want_V=False)
            v, _ = te.te_evolve(h, c["v0"], 0.7, 1e-9, 16)
            h.close()
            key = np.concatenate([g["alpha"], g["beta"], v.view(np.float64)])
            if ref is None:
                ref = key
            else:
                assert np.array_equal(key.view(np.uint64), ref.view(np.uint64))


def test_option_validation(gpu_lib):
    """Out-of-range option values are rejected (TE_ERR_ARG) and leave the handle usable; the halo
    mode is accepted on a single-rank handle and has no effect there."""
    te = gpu_lib
    c = configs.build(1, n=600)
    h = te.te_create_csr(c["n"], c["rowptr"], c["col"], c["val"])
    v_ref, _ = te.te_evolve(h, c["v0"], 0.5, 1e-9, 20)
    for opt, bad in ((te.TE_OPT_SPMV, 9), (te.TE_OPT_SPMV, 4), (te.TE_OPT_SPMV, -1), (te.TE_OPT_KERNELS, 0), (te.TE_OPT_HALO, 2), (te.TE_OPT_ORTHO, 3),
                     (te.TE_OPT_KERNELS, 4), (te.TE_OPT_KERNELS, 6), (te.TE_OPT_INTEGRATOR, 2), (te.TE_OPT_SPMV, 4.5)):
        with pytest.raises(te.TEError):
            te.te_set_option(h, opt, bad)
    te.te_set_option(h, te.TE_OPT_HALO, 1)
    v, _ = te.te_evolve(h, c["v0"], 0.5, 1e-9, 20)
    assert np.array_equal(v, v_ref)
    h.close()


def test_edge_cases(gpu_lib):
    te = gpu_lib
    # Pauli X, t = pi -> -e1 (exp(-i X pi) = -I); breakdown at j = 1 (m_eff = 2)
    rp, cl, vl = csr_from_dense(np.array([[0, 1], [1, 0]], dtype=complex))
    h = te.te_create_csr(2, rp, cl, vl)
    v, st = te.te_evolve(h, np.array([1, 0], complex), math.pi, 1e-10, 10)
    assert np.abs(v - np.array([-1, 0])).max() < 1e-12
    assert st["n_breakdowns"] == st["n_restarts"] == 1
    # t = 0 returns v0
    v0 = np.array([0.6, 0.8j])
    v, st = te.te_evolve(h, v0, 0.0, 1e-10, 10)
    assert np.array_equal(v, v0) and st["n_restarts"] == 0 and st["err_bound"] == 0.0
    # not normalised
    with pytest.raises(te.TEError) as ei:
        te.te_evolve(h, np.array([1, 1], complex), 1.0, 1e-8, 5)
    assert ei.value.status == 4
    # bad args
    with pytest.raises(te.TEError) as ei:
        te.te_evolve(h, np.array([1, 0], complex), 1.0, 0.0, 5)
    assert ei.value.status == 1
    with pytest.raises(te.TEError):
        te.te_evolve(h, np.array([1, 0], complex), -1.0, 1e-8, 5)
    with pytest.raises(te.TEError):
        te.te_evolve(h, np.array([1, 0], complex), 1.0, 1e-8, 65)
    h.close()
    # eigenvector input: breakdown at j = 0, exact phase
    rp, cl, vl = csr_from_dense(np.diag([1.0, 2.0, 3.0]))
    h = te.te_create_csr(3, rp, cl, vl)
    v, st = te.te_evolve(h, np.array([0, 1, 0], complex), 3.0, 1e-8, 5)
    assert abs(v[1] - np.exp(-6j)) < 1e-14 and st["n_breakdowns"] == 1
    h.close()
    # invalid CSR / non-Hermitian
    with pytest.raises(te.TEError) as ei:
        te.te_create_csr(2, np.array([0, 2, 3]), np.array([1, 0, 0]), np.array([1.0, 1.0, 2.0]))
    assert ei.value.status == 2
    with pytest.raises(te.TEError) as ei:
        te.te_create_csr(2, np.array([0, 1, 2]), np.array([1, 0]), np.array([1.0, 2.0]))
    assert ei.value.status == 3
    with pytest.raises(te.TEError) as ei:
        te.te_create_csr(2, np.array([0, 1, 2]), np.array([1, 0]), np.array([1 + 1j, 1 + 1j]))
    assert ei.value.status == 3
    # m_max = 1 on a non-trivial problem -> step collapse (reading C17)
    A = np.array([[0.0, 1.0, 0.0], [1.0, 0.5, 1.0], [0.0, 1.0, -0.3]])
    rp, cl, vl = csr_from_dense(A)
    h = te.te_create_csr(3, rp, cl, vl)
    with pytest.raises(te.TEError) as ei:
        te.te_evolve(h, np.array([1, 0, 0], complex), 1.0, 1e-10, 1)
    assert ei.value.status == 5
    # m_max > n: capped at n, exact
    v, st = te.te_evolve(h, np.array([1, 0, 0], complex), 1.0, 1e-10, 40)
    assert np.linalg.norm(v - sl.expm(-1j * A) @ np.array([1, 0, 0])) < 1e-12
    h.close()


def test_determinism_and_device_path(gpu_lib):
    import torch
    te = gpu_lib
    c = configs.build(2, L=14)
    h = te.te_create_csr(c["n"], c["rowptr"], c["col"], c["val"])
    v1, s1 = te.te_evolve(h, c["v0"], 3.0, 1e-10, 40)
    v2, s2 = te.te_evolve(h, c["v0"], 3.0, 1e-10, 40)
    assert np.array_equal(v1, v2) and s1 == s2
    d0 = torch.from_numpy(c["v0"]).cuda()
    d1 = torch.empty_like(d0)
    s3 = te.te_evolve_dev(h, d0, 3.0, 1e-10, 40, d1, stream=torch.cuda.current_stream())
    torch.cuda.synchronize()
    assert np.array_equal(d1.cpu().numpy(), v1)
    # in-place (v_out aliases v0)
    v = c["v0"].copy()
    te.te_evolve(h, v, 3.0, 1e-10, 40, out=v)
    assert np.array_equal(v, v1)
    # direct launches (no CUDA graph replay) and profiling events give the same bits
    te.te_set_option(h, te.TE_OPT_GRAPH, 0)
    v4, s4 = te.te_evolve(h, c["v0"], 3.0, 1e-10, 40)
    assert np.array_equal(v4, v1) and s4 == s1
    te.te_set_option(h, te.TE_OPT_GRAPH, 1)
    te.te_set_option(h, te.TE_OPT_PROFILE, 1)
    v5, s5 = te.te_evolve(h, c["v0"], 3.0, 1e-10, 40)
    assert np.array_equal(v5, v1)
    prof = te.te_get_profile(h)
    assert prof["spmv"]["launches"] == s5["n_krylov_steps"] and prof["combine"]["launches"] == s5["n_restarts"]
    assert all(p["total_ms"] > 0 for k, p in prof.items() if p["launches"] and k != "host_step")
    h.close()


def test_full_size_xxz_L20_one_magnon_pin(gpu_lib):
    """Full config-2 size (n = 2^20), launch configuration of bench.py: a one-magnon initial
    state evolves inside the L x L one-magnon block, computed exactly."""
    te = gpu_lib
    c = configs.build(2)
    L = 20
    h_f = c["fields"]
    J, Dl = 1.0, 0.5
    E_ref = J * L * Dl / 4 - 0.5 * h_f.sum()
    M = np.zeros((L, L))
    for k in range(L):
        M[k, k] = E_ref - J * Dl + h_f[k]
        M[k, (k + 1) % L] = M[(k + 1) % L, k] = J / 2
    g = np.random.default_rng(5)
    a = g.standard_normal(L) + 1j * g.standard_normal(L)
    a /= np.linalg.norm(a)
    v0 = np.zeros(1 << L, complex)
    idx = [1 << k for k in range(L)]
    v0[idx] = a
    h = te.te_create_csr(c["n"], c["rowptr"], c["col"], c["val"])
    t = c["t"]
    v, st = te.te_evolve(h, v0, t, c["tol"], c["m"])
    exact = sl.expm(-1j * M * t) @ a
    assert np.linalg.norm(v[idx] - exact) <= st["err_bound"] + 1e-12
    mask = np.ones(1 << L, bool)
    mask[idx] = False
    assert np.all(v[mask] == 0)
    h.close()


def test_full_size_xxz_L20_neel(gpu_lib):
    """Config 2 at full size: Sz-sector exact zeros, norm, bound, partition of t; the first
    restart against the oracle with the schedule forced identical (sampled at full size)."""
    te = gpu_lib
    c = configs.build(2)
    h = te.te_create_csr(c["n"], c["rowptr"], c["col"], c["val"])
    v, st = te.te_evolve(h, c["v0"], c["t"], c["tol"], c["m"])
    sched = te.te_get_schedule(h)
    assert st["err_bound"] <= c["tol"]
    assert math.fsum(s[0] for s in sched) == pytest.approx(c["t"], abs=1e-12)
    pop = np.array([bin(i).count("1") for i in range(c["n"])])
    assert np.all(v[pop != 10] == 0)
    assert abs(np.linalg.norm(v) - 1) <= st["err_bound"] + 10 * st["roundoff_total"]
    tau1 = sched[0][0]
    v1, _ = te.te_evolve_schedule(h, c["v0"], [tau1], c["tol"], c["m"])
    r1 = K.evolve(c["rowptr"], c["col"], c["val"], c["v0"], tau1, c["tol"], c["m"], schedule=[tau1])
    assert np.linalg.norm(v1 - r1["v"]) <= 1e-10
    h.close()


def test_full_size_paper_s5_benchmark(gpu_lib):
    """Config 6, the paper's own benchmark: d = 1,565,904, t = 10, err_max = 1e-7, m = 40.
    The bound is met; the norm holds; the forward-backward round trip of P:509 at the P:527 size,
    using exp(+iHt) w = conj(exp(-iHt) conj(w)) for real H, returns to v0 within the two
    bounds; one forced restart (m = 8) against the oracle element by element."""
    te = gpu_lib
    c = configs.build(6)
    h = te.te_create_csr(c["n"], c["rowptr"], c["col"], c["val"])
    v, st = te.te_evolve(h, c["v0"], c["t"], c["tol"], c["m"])
    assert st["err_bound"] <= c["tol"] and st["one_norm"] == pytest.approx(171.515, abs=5e-4)
    assert abs(np.linalg.norm(v) - 1) <= st["err_bound"] + 1e-9
    w, st2 = te.te_evolve(h, np.conj(v), c["t"], c["tol"], c["m"])
    assert np.linalg.norm(np.conj(w) - c["v0"]) <= st["err_bound"] + st2["err_bound"] + 1e-9
    tau, m = 0.02, 8
    v1, _ = te.te_evolve_schedule(h, c["v0"], [tau], c["tol"], m)
    r1 = K.evolve(c["rowptr"], c["col"], c["val"], c["v0"], tau, c["tol"], m, schedule=[tau])
    assert np.linalg.norm(v1 - r1["v"]) <= 1e-10
    h.close()


def _sampled_arnoldi_relation(te, c, m=4, nsample=300, seed=0):
    """Full-size check of one Krylov decomposition in bench.py's launch configuration (default
    kernels): orthonormal basis (all n rows) and the three-term Arnoldi relation of Eq. 8,
    H V_k = beta_{k-1} V_{k-1} + alpha_k V_k + beta_k V_{k+1}, on sampled rows with (H V_k)_r
    from the oracle's row-restricted product (reading C2: CGS2's off-tridiagonal coefficients
    vanish for Hermitian H up to rounding)."""
    h = te.te_create_csr(c["n"], c["rowptr"], c["col"], c["val"])
    g = te.te_krylov_basis(h, c["v0"], m, c["tol"] / c["t"], want_V=True)
    nrm = te.te_one_norm(h) if hasattr(te, "te_one_norm") else None
    h.close()
    V, a, b, k = g["V"], g["alpha"], g["beta"], g["m_eff"]
    assert k == m
    G = V.conj().T @ V
    assert np.abs(G - np.eye(k)).max() <= 1e-12
    n = c["n"]
    rows = np.unique(np.concatenate([[0, n - 1], np.random.default_rng(seed).integers(0, n, nsample)]))
    scale = nrm if nrm else max(1.0, np.abs(a).max() + 2 * np.abs(b).max())
    for j in range(k - 1):
        hv = K.spmv_rows(c["rowptr"], c["col"], c["val"], V[:, j], rows)
        rhs = a[j] * V[rows, j] + b[j] * V[rows, j + 1]
        if j > 0:
            rhs = rhs + b[j - 1] * V[rows, j - 1]
        assert np.abs(hv - rhs).max() <= 1e-12 * scale
    return g


def test_full_size_config3_bose_hubbard(gpu_lib):
    """Config 3 at full size (n = 1,352,078): one forced restart against the oracle element by
    element; the adaptive evolution meets its bound, keeps the norm, and the forward-backward
    round trip (real H: exp(+iHt) w = conj(exp(-iHt) conj(w))) returns to v0 within the bounds."""
    te = gpu_lib
    c = configs.build(3)
    h = te.te_create_csr(c["n"], c["rowptr"], c["col"], c["val"])
    v, st = te.te_evolve(h, c["v0"], c["t"], c["tol"], c["m"])
    assert st["err_bound"] <= c["tol"]
    assert abs(np.linalg.norm(v) - 1) <= st["err_bound"] + 1e-9
    w, st2 = te.te_evolve(h, np.conj(v), c["t"], c["tol"], c["m"])
    assert np.linalg.norm(np.conj(w) - c["v0"]) <= st["err_bound"] + st2["err_bound"] + 1e-9
    tau, m = 0.05, 10
    v1, _ = te.te_evolve_schedule(h, c["v0"], [tau], c["tol"], m)
    r1 = K.evolve(c["rowptr"], c["col"], c["val"], c["v0"], tau, c["tol"], m, schedule=[tau])
    assert np.linalg.norm(v1 - r1["v"]) <= 1e-10
    h.close()
    _sampled_arnoldi_relation(te, c)


def test_full_size_config4_random_banded(gpu_lib):
    """Config 4 at full size (n = 2^24, 5.4e8 complex entries): sampled Arnoldi relation and
    orthonormality; the adaptive evolution meets its bound and keeps the norm."""
    te = gpu_lib
    c = configs.build(4)
    _sampled_arnoldi_relation(te, c)
    h = te.te_create_csr(c["n"], c["rowptr"], c["col"], c["val"])
    v, st = te.te_evolve(h, c["v0"], c["t"], c["tol"], c["m"])
    assert st["err_bound"] <= c["tol"]
    assert abs(np.linalg.norm(v) - 1) <= st["err_bound"] + 1e-9
    h.close()


def test_full_size_config5_xxz_nnn_L26(gpu_lib):
    """Config 5 at full size (n = 2^26, 1.8e9 entries): sampled Arnoldi relation and
    orthonormality; the adaptive evolution meets its bound, keeps the norm and the total S^z
    (the Hamiltonian conserves it; the product state's S^z distribution must not change)."""
    te = gpu_lib
    c = configs.build(5)
    _sampled_arnoldi_relation(te, c, m=3, nsample=200)
    h = te.te_create_csr(c["n"], c["rowptr"], c["col"], c["val"])
    del c["rowptr"], c["col"], c["val"]
    v, st = te.te_evolve(h, c["v0"], c["t"], c["tol"], c["m"])
    h.close()
    assert st["err_bound"] <= c["tol"]
    assert abs(np.linalg.norm(v) - 1) <= st["err_bound"] + 1e-9
    L = 26
    pop = np.zeros(c["n"], dtype=np.int8)
    idx = np.arange(c["n"], dtype=np.int64)
    for b in range(L):
        pop += ((idx >> b) & 1).astype(np.int8)
    w0 = np.bincount(pop, weights=np.abs(c["v0"]) ** 2, minlength=L + 1)
    w1 = np.bincount(pop, weights=np.abs(v) ** 2, minlength=L + 1)
    assert np.abs(w1 - w0).max() <= 2 * st["err_bound"] + 1e-9


def _forced_wrap_parity(te, c, sched, m, ring_min_wraps=4, spmv=None):
    """Forced-schedule evolution vs the oracle element by element (<= 1e-10, north star) at a
    size where every CTA of the ring SpMV takes many tiles (the ring wraps, the mbarrier phase
    flips many times).  The SpMV instantiation (value type, lanes per row, ring depth) depends only
    on the value type and the mean row length, so it is the one the full-size config launches."""
    h = te.te_create_csr(c["n"], c["rowptr"], c["col"], c["val"])
    if spmv is not None:
        te.te_set_option(h, te.TE_OPT_SPMV, spmv)
    v, st = te.te_evolve_schedule(h, c["v0"], sched, c["tol"], m)
    h.close()
    ref = K.evolve(c["rowptr"], c["col"], c["val"], c["v0"], float(sum(sched)), c["tol"], m, schedule=sched)
    tiles_per_cta = c["rowptr"][-1] / (5632 if c["val"].dtype == np.float64 else 2816) / 148
    assert tiles_per_cta >= ring_min_wraps * 4
    assert [s[1] for s in ref["schedule"]] == [m] * len(sched)
    err = np.linalg.norm(v - ref["v"])
    assert err <= 1e-10, err
    assert st["n_krylov_steps"] == ref["krylov_steps"]
    return err


@pytest.mark.parametrize("spmv", [7, 8, 10])
def test_forced_parity_complex_ring_wraps_config4_n2e20(gpu_lib, spmv, monkeypatch):
    """Complex H through the ring SpMV at a wrapping size: config 4's model at n = 2^20 (32
    complex entries per row, the k_spmv_ring<complex, TPR 4, 3 stages> instantiation of the full
    2^24 config), m = 8, two forced restarts, element by element against the oracle.  spmv 10: the
    column-blocked ring as config 4 runs it (6 blocks of 2.7 MB here; 16 entries per row per pass
    in the diagonal block, the rest uniform: TPR 1-2 per pass)."""
    if spmv == 10:
        monkeypatch.setenv("TE_SPMV_COLBLK_MB", "2.7")
    c = configs.build(4, n=1 << 20)
    _forced_wrap_parity(gpu_lib, c, [0.05, 0.05], 8, spmv=spmv)


@pytest.mark.parametrize("spmv", [7, 8, 9, "9-panel"])
def test_forced_parity_config5_instantiation_L22(gpu_lib, spmv, monkeypatch):
    """Config 5's model at L = 22 (n = 4,194,304, 23 entries per row on average: the TPR 2 /
    3-stage real ring instantiation of the full L = 26 config; spmv 9: the slot-window SELL-32 that
    config 5 runs by default, with the same dictionary and window structure; "9-panel": its two-pass
    panel sweep with 6 outer slice bits as at L = 26 — panels of 2^11 slices here, 2^15 there), m = 10,
    one forced restart, element by element against the oracle."""
    monkeypatch.setenv("TE_SPMV_SW_PANEL", "11" if spmv == "9-panel" else "0")
    c = configs.build(5, L=22)
    _forced_wrap_parity(gpu_lib, c, [0.1], 10, spmv=9 if isinstance(spmv, str) else spmv)


def test_sw_panel_sweep_lanczos_and_breakdown(gpu_lib, monkeypatch):
    """The far-window pass of the panel sweep under the non-deferred step gate (f1 Lanczos: the SpMV
    applies s_j itself; the second pass reads the gate without writing it) and through a lucky
    breakdown (an eigenvector of S^z-conserving XXZ: |all up> stops at j = 0)."""
    te = gpu_lib
    monkeypatch.setenv("TE_SPMV_SW_FORCE", "1")
    monkeypatch.setenv("TE_SPMV_SW_PANEL", "2")
    c = configs.build(5, L=12)
    h = te.te_create_csr(c["n"], c["rowptr"], c["col"], c["val"])
    te.te_set_option(h, te.TE_OPT_SPMV, 9)
    assert te.te_get_option(h, te.TE_INFO_SW_PANEL) == 2
    te.te_set_option(h, te.TE_OPT_ORTHO, 1)
    tol_rate = c["tol"] / c["t"]
    g = te.te_krylov_basis(h, c["v0"], 16, tol_rate, want_V=True)
    o = K.arnoldi(lambda x: K.spmv(c["rowptr"], c["col"], c["val"], x), c["v0"], 16, tol_rate, ortho="lanczos3")
    scale = max(1.0, np.abs(o["alpha"]).max(), np.abs(o["beta"]).max())
    assert g["m_eff"] == o["m_eff"]
    assert np.abs(g["alpha"] - o["alpha"]).max() <= 1e-10 * scale
    assert np.abs(g["beta"] - o["beta"]).max() <= 1e-10 * scale
    assert np.linalg.norm(g["V"] - o["V"]) <= 1e-8
    for ortho in (0, 1, 2):
        te.te_set_option(h, te.TE_OPT_ORTHO, ortho)
        e = np.zeros(c["n"], dtype=np.complex128)
        e[c["n"] - 1] = 1.0  # all spins up: an eigenvector
        gb = te.te_krylov_basis(h, e, 8, tol_rate, want_V=False)
        ob = K.arnoldi(lambda x: K.spmv(c["rowptr"], c["col"], c["val"], x), e, 8, tol_rate)
        assert gb["m_eff"] == ob["m_eff"] == 1
        assert abs(gb["alpha"][0] - ob["alpha"][0]) <= 1e-12 * scale
    h.close()


def test_distributed_api_single_rank(gpu_lib):
    """te_dist_init / te_create_csr_dist on one rank (global columns, halo plan, no NCCL
    traffic) gives the same evolution as the plain handle."""
    te = gpu_lib
    c = configs.build(3, L=8, N=8)
    h = te.te_create_csr(c["n"], c["rowptr"], c["col"], c["val"])
    v1, s1 = te.te_evolve(h, c["v0"], 2.0, 1e-9, 30)
    D = te.te_dist_init(1, 0, b"\0" * 128)
    hd = te.te_create_csr_dist(D, c["n"], 0, c["n"], c["rowptr"], c["col"].astype(np.int64), c["val"])
    v2, s2 = te.te_evolve(hd, c["v0"], 2.0, 1e-9, 30)
    assert np.array_equal(v1, v2) and s1["n_restarts"] == s2["n_restarts"]
    assert s1["one_norm"] == s2["one_norm"]
    hd.close()
    h.close()
    D.close()


@pytest.mark.parametrize("name,c", CASES[:4], ids=[x[0] for x in CASES[:4]])
def test_lanczos3_mode_matches_oracle(gpu_lib, name, c):
    """the paper-literal 3-term recurrence (TE_OPT_ORTHO=1) against the oracle's
    ortho='lanczos3' — same recurrence, same arithmetic up to summation order."""
    te = gpu_lib
    h = te.te_create_csr(c["n"], c["rowptr"], c["col"], c["val"])
    te.te_set_option(h, te.TE_OPT_ORTHO, 1)
    m = min(20, c["n"])
    tol_rate = c["tol"] / c["t"]
    g = te.te_krylov_basis(h, c["v0"], m, tol_rate, want_V=True)
    o = K.arnoldi(lambda x: K.spmv(c["rowptr"], c["col"], c["val"], x), c["v0"], m, tol_rate, ortho="lanczos3")
    assert g["m_eff"] == o["m_eff"]
    scale = max(1.0, np.abs(o["alpha"]).max(), np.abs(o["beta"]).max())
    assert np.abs(g["alpha"] - o["alpha"]).max() <= 1e-10 * scale
    assert np.abs(g["beta"] - o["beta"]).max() <= 1e-10 * scale
    assert np.linalg.norm(g["V"] - o["V"]) <= 1e-8
    t, tol = min(c["t"], 2.0), c["tol"]
    v, st = te.te_evolve(h, c["v0"], t, tol, c["m"])
    sched = te.te_get_schedule(h)
    ref = K.evolve(c["rowptr"], c["col"], c["val"], c["v0"], t, tol, c["m"], ortho="lanczos3",
                   schedule=[s[0] for s in sched])
    assert np.linalg.norm(v - ref["v"]) <= 1e-9
    assert st["err_bound"] <= tol
    h.close()


def test_sampling_and_gauss_integrator(gpu_lib):
    """P:335 intermediate-time sampling and the P:406 Gauss-Legendre option against the oracle."""
    te = gpu_lib
    c = configs.build(1, n=2000)
    h = te.te_create_csr(c["n"], c["rowptr"], c["col"], c["val"])
    ts = [0.0, 0.25, 0.8, 1.5, 2.0]
    v, S, sb, st = te.te_evolve_sampled(h, c["v0"], 2.0, 1e-9, 30, ts)
    sched = te.te_get_schedule(h)
    ref = K.evolve(c["rowptr"], c["col"], c["val"], c["v0"], 2.0, 1e-9, 30, schedule=[s[0] for s in sched], samples=ts)
    for i in range(len(ts)):
        assert np.linalg.norm(S[i] - ref["samples"][i]) <= 1e-10
        assert abs(sb[i] - ref["sample_bounds"][i]) <= 1e-3 * ref["sample_bounds"][i] + 1e-15
    assert np.array_equal(S[0], c["v0"])
    assert np.linalg.norm(S[-1] - v) <= 1e-13
    te.te_set_option(h, te.TE_OPT_INTEGRATOR, 1)
    vg, stg = te.te_evolve(h, c["v0"], 2.0, 1e-9, 30)
    sg = te.te_get_schedule(h)
    refg = K.evolve(c["rowptr"], c["col"], c["val"], c["v0"], 2.0, 1e-9, 30, schedule=[s[0] for s in sg], integrator="gauss")
    assert np.linalg.norm(vg - refg["v"]) <= 1e-10
    assert stg["err_bound"] == pytest.approx(refg["bound"], rel=1e-6)
    ada = K.evolve(c["rowptr"], c["col"], c["val"], c["v0"], 2.0, 1e-9, 30, integrator="gauss")
    assert np.linalg.norm(vg - ada["v"]) <= 1e-9 + 1e-12
    h.close()


@pytest.mark.parametrize("name,c", CASES, ids=[x[0] for x in CASES])
def test_cgs2gram_mode_matches_oracle(gpu_lib, name, c):
    """SURVEY f2 (TE_OPT_ORTHO=2): against the oracle's 'cgs2gram' (same recurrence) and its
    plain CGS2 (equal in exact arithmetic): basis and the evolved state at 1e-10."""
    te = gpu_lib
    h = te.te_create_csr(c["n"], c["rowptr"], c["col"], c["val"])
    te.te_set_option(h, te.TE_OPT_ORTHO, 2)
    m = min(c["m"], c["n"])
    tol_rate = c["tol"] / c["t"]
    g = te.te_krylov_basis(h, c["v0"], m, tol_rate, want_V=True)
    mv = lambda x: K.spmv(c["rowptr"], c["col"], c["val"], x)  # noqa: E731
    for ortho in ("cgs2gram", "cgs2"):
        o = K.arnoldi(mv, c["v0"], m, tol_rate, ortho=ortho)
        assert g["m_eff"] == o["m_eff"]
        scale = max(1.0, np.abs(o["alpha"]).max(), np.abs(o["beta"]).max())
        assert np.abs(g["alpha"] - o["alpha"]).max() <= 1e-12 * scale
        assert np.abs(g["beta"] - o["beta"]).max() <= 1e-12 * scale
        assert np.linalg.norm(g["V"] - o["V"]) <= 1e-10
    k = g["m_eff"]
    assert np.abs(g["V"].conj().T @ g["V"] - np.eye(k)).max() <= 1e-13
    t, tol = (min(c["t"], 2.0) if c["n"] > 5000 else c["t"]), c["tol"]
    v, st = te.te_evolve(h, c["v0"], t, tol, c["m"])
    sched = te.te_get_schedule(h)
    ref = K.evolve(c["rowptr"], c["col"], c["val"], c["v0"], t, tol, c["m"], schedule=[s[0] for s in sched])
    assert np.linalg.norm(v - ref["v"]) <= 1e-10
    assert st["err_bound"] <= tol
    h.close()
