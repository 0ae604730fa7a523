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
