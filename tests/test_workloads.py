"""Input generators: closed forms and bit-exactness of the fast C builder."""
import math

import numpy as np
import pytest

from workloads import configs, fast, models


@pytest.mark.parametrize("L,J2", [(8, 0.0), (10, 0.5), (12, 0.5), (13, 0.0)])
def test_fast_xxz_builder_bit_exact(L, J2):
    h = models.xxz_fields(L, 7)
    a = models.xxz_csr(L, 1.0, 0.7, h, J2=J2)
    b = fast.xxz_csr_fast(L, 1.0, 0.7, h, J2=J2)
    for x, y in zip(a, b):
        assert x.dtype == y.dtype and np.array_equal(x.view(np.uint8), y.view(np.uint8))


def test_closed_form_sizes():
    c = configs.build(2, L=14)
    assert c["rowptr"][-1] == (1 << 14) * (1 + 14 // 2)            # 2^L (1 + L/2)
    c = configs.build(5, L=12)
    assert c["rowptr"][-1] == (1 << 12) * (1 + 12)                 # 2^L (1 + L) with NNN
    occ = models.bh_basis(6, 6)
    assert occ.shape[0] == math.comb(11, 6)                        # C(N+L-1, N)
    c = configs.build(3, L=6, N=6)
    d = math.comb(11, 6)
    assert c["rowptr"][-1] == d * (1 + 2 * 5 * 6 / 11)            # d (1 + 2 (L-1) N / (N+L-1))
    assert int(np.nonzero(c["v0"])[0][0]) == int(np.searchsorted(models.bh_keys(occ), models.bh_keys(np.ones((1, 6), np.uint8))[0]))


def test_full_size_closed_forms():
    """BASELINE sizes, integer setup bit-exact against closed forms (SURVEY.md App. A,
    north_star "Integer setup ... must be bit-exact"):
      config 2  XXZ L=20:     nnz = 2^L (1 + L/2) = 11,534,336;  Neel (even sites up) -> 349,525
      config 5  XXZ+NNN L=26: nnz = 2^L (1 + L)   = 1,811,939,328 (C rowptr builder, all rows)
      config 3  BH L=N=12:    d = C(23,12) = 1,352,078;  nnz = d (1 + 2 (L-1) N/(N+L-1)) =
                              16,871,582;  |1,...,1> -> 873,885;  first (0,..,0,12), last (12,0,..,0)."""
    assert models.neel_index(20) == 349525 == sum(1 << i for i in range(0, 20, 2))
    lib = fast._load()
    for L, J2, nnz in [(20, 0.0, 11534336), (26, 0.5, 1811939328)]:
        n = 1 << L
        rp = np.empty(n + 1, dtype=np.int64)
        lib.xxz_rowptr(L, 1.0, J2, 0, n, rp.ctypes.data)
        assert rp[0] == 0 and int(rp[-1]) == nnz
        assert nnz == (1 << L) * (1 + (L if J2 else L // 2))
        del rp
    c = configs.build(3)
    d = math.comb(23, 12)
    assert c["n"] == d == 1352078
    assert int(c["rowptr"][-1]) == 16871582 == d * (23 + 2 * 11 * 12) // 23
    assert int(np.nonzero(c["v0"])[0][0]) == 873885
    assert tuple(c["occ"][0]) == (0,) * 11 + (12,) and tuple(c["occ"][-1]) == (12,) + (0,) * 11


def test_bh_hash_index_map_bit_exact():
    """The hash-table ind^-1 and the sorted-key search give bit-identical Bose-Hubbard CSR
    arrays at the full config-3 size, and the table round-trips every basis key (exhaustive,
    SURVEY §8(c) BH pin) and rejects keys outside the sector."""
    L, N = 12, 12
    mu = models.bh_mu(L, 3)
    a = models.bose_hubbard_csr(L, N, 1.0, 2.0, mu, index="search")
    b = models.bose_hubbard_csr(L, N, 1.0, 2.0, mu, index="hash")
    for x, y in zip(a, b):
        assert x.dtype == y.dtype and np.array_equal(x.view(np.uint8), y.view(np.uint8))
    keys = models.bh_keys(a[0])
    T = models.BHIndexHash(keys)
    assert T.slot_key.shape[0] == 1 << 22
    assert np.array_equal(T.lookup(keys), np.arange(keys.shape[0]))
    bad = keys[:1000] + 1  # sum of occupations N+1: not in the fixed-N sector
    assert np.all(T.lookup(bad) == -1)


def test_hermitian_and_sorted():
    import scipy.sparse as sp
    for c in (configs.build(1, n=512), configs.build(4, n=4096), configs.build(3, L=5, N=5), configs.build(5, L=9)):
        rp, col = c["rowptr"], c["col"]
        H = sp.csr_matrix((c["val"], col, rp), shape=(c["n"], c["n"]))
        assert abs(H - H.getH()).max() == 0
        for r in range(0, c["n"], max(1, c["n"] // 50)):
            seg = col[rp[r]: rp[r + 1]]
            assert np.all(np.diff(seg) > 0)
        assert abs(np.linalg.norm(c["v0"]) - 1) < 1e-12


def test_band_involutions_within_band():
    rows = np.arange(1 << 14, dtype=np.int64)
    for k in range(16):
        p, pair, ok = models.band_involution(1 << 14, 4, k, rows)
        assert np.all(np.abs(p - rows) <= 255) and np.all(p != rows)
        q, _, _ = models.band_involution(1 << 14, 4, k, p)
        assert np.array_equal(q, rows)                               # involution
    ds = np.stack([models.band_involution(1 << 14, 4, k, rows)[0] ^ rows for k in range(16)])
    assert np.all(np.sort(ds, axis=0)[1:] != np.sort(ds, axis=0)[:-1])  # 16 distinct offsets per row


def test_uniform_involution_is_matching():
    n = 1 << 12
    rows = np.arange(n, dtype=np.int64)
    p, pair, ok = models.uniform_involution(n, 1, 100, rows)
    assert ok.all() and np.all(p != rows)
    assert np.array_equal(p[p], rows)


def test_fast_xxz_row_range():
    L, h = 11, models.xxz_fields(11, 3)
    rp, col, val = models.xxz_csr(L, 1.0, 0.5, h, J2=0.5)
    r0, r1 = 300, 1500
    lrp, lcol, lval = fast.xxz_csr_fast(L, 1.0, 0.5, h, J2=0.5, r0=r0, r1=r1)
    assert np.array_equal(lrp, rp[r0:r1 + 1] - rp[r0])
    assert np.array_equal(lcol, col[rp[r0]:rp[r1]]) and np.array_equal(lval, val[rp[r0]:rp[r1]])


@pytest.mark.parametrize("p", [None, dict(K=6, K1=6, Nm=3, N0=30, Nc=30), dict(K=5, K1=3, Nm=4, N0=7, Nc=9, dNc=2),
                               dict(K=3, K1=4, Nm=1, N0=0, Nc=5)], ids=["default", "K6", "asym", "N0_0"])
def test_memory_burden_fast_builder_bit_exact(p):
    """The vectorised §5 builder equals the per-row loop builder bit for bit."""
    from workloads import memory_burden as mb
    a, b = mb.hamiltonian(p), mb.hamiltonian_fast(p)
    assert a["n"] == b["n"] and a["init_index"] == b["init_index"]
    for k in ("rowptr", "col", "val"):
        assert a[k].dtype == b[k].dtype and np.array_equal(a[k].view(np.uint8), b[k].view(np.uint8))


def test_paper_s5_instance_config6():
    """Config 6 = the P:527 benchmark matrix: d = 1,565,904 (printed); 122,109,000 nonzeros
     plus 504 explicit zero diagonals: the diagonal eps(1-n0/Nc)qa + eps(1-n0/(Nc-dNc))qb
     vanishes at n0 = Nc-dNc = 88 with qa = 0 and at n0 = Nc = 100 with qb = 0, C(10,5) = 252
    rows each; 76 memory-sector entries (diagonal + 5*15 hops) + 1 or 2 C0 terms per row;
    v0 = |N0,0,1^5,0^15>, the lexicographically largest tuple of the N0 block."""
    c = configs.build(6)
    rp, col, val = c["rowptr"], c["col"], c["val"]
    assert c["n"] == 1565904
    assert rp[-1] == 122109504 and int(np.count_nonzero(val)) == 122109000
    w = np.diff(rp)
    d2 = math.comb(20, 5)
    assert np.all(w[:d2] == 77) and np.all(w[-d2:] == 77) and np.all(w[d2:-d2] == 78)
    assert np.array_equal(np.nonzero(c["v0"])[0], [100 * d2 + d2 - 1])
    zpos = np.nonzero(val == 0)[0]
    zrows = np.searchsorted(rp, zpos, side="right") - 1
    assert np.all(col[zpos] == zrows)                                  # every zero is a diagonal entry
    blk, cnt = np.unique(zrows // d2, return_counts=True)
    assert blk.tolist() == [88, 100] and cnt.tolist() == [252, 252]


@pytest.mark.parametrize("diag,band", [(True, 0), (False, 16)])
def test_parallel_involution_builder_bit_exact(diag, band):
    """Chunked process-pool build == single-process build, byte for byte (ragged last chunk)."""
    from workloads import parallel_build
    n = 70000
    a = models.involution_csr(n, 4, n_uniform=16, n_band=band, diagonal=diag)
    b = parallel_build.involution_csr_parallel(n, 4, n_uniform=16, n_band=band, diagonal=diag, nproc=3, chunk=1 << 14)
    for x, y in zip(a, b):
        assert x.dtype == y.dtype and np.array_equal(x.view(np.uint8), y.view(np.uint8))
