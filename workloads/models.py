"""Synthetic Hamiltonians and initial states for the BASELINE.json configs.

Input generators only: sparse Hermitian matrices in CSR form (int64 rowptr,
int32 col, float64 or complex128 val, columns strictly increasing per row) and
normalised complex128 initial vectors.  Nothing here implements the Krylov
method; the oracle and the CUDA library both consume these arrays.

Models (recipe in DESIGN.md "Input recipe", after SURVEY.md §8(d) and App. B):

* ``xxz_csr``        spin-1/2 XXZ chain, S = sigma/2, bit i of the row index is
                     spin i (1 = up).  H = sum_bonds J (SxSx + SySy + Delta SzSz)
                     + sum_i h_i Sz_i.  Off-diagonal J/2 on antiparallel bonds.
* ``bose_hubbard``   fixed-N Bose-Hubbard chain, lexicographic basis (site 0
                     most significant), H = -J sum (b_i^+ b_{i+1} + h.c.)
                     + U/2 sum n_i(n_i-1) - sum mu_i n_i.
* ``involution_csr`` random sparse Hermitian matrix as a sum of random
                     involutions (perfect matchings): every row gets one
                     partner per involution, H_{i,pi(i)} = z, H_{pi(i),i} = conj z.
"""
from __future__ import annotations

import math

import numpy as np

from . import rng

# ----------------------------------------------------------------------------
# CSR assembly helper (per-row candidate lists -> sorted, merged CSR)
# ----------------------------------------------------------------------------


def _assemble(cols: np.ndarray, vals: np.ndarray, valid: np.ndarray, ncols: int):
    """cols/vals/valid are (m, K) per-row candidate arrays (m rows, global
    column indices < ncols).  Each row's valid candidates are sorted by column
    (stable, so equal columns keep candidate order) and duplicate columns are
    merged by summing left to right (runs are short, so numpy's reduceat sums
    them sequentially)."""
    m, K = cols.shape
    big = np.int64(ncols)  # sentinel sorts last
    c = np.where(valid, cols.astype(np.int64), big)
    order = np.argsort(c, axis=1, kind="stable")
    c = np.take_along_axis(c, order, axis=1)
    v = np.take_along_axis(vals, order, axis=1)
    ok = c < big
    rows = np.broadcast_to(np.arange(m, dtype=np.int64)[:, None], (m, K))[ok]
    cf = c[ok]
    vf = v[ok]
    if cf.size:
        head = np.ones(cf.size, dtype=bool)
        head[1:] = (rows[1:] != rows[:-1]) | (cf[1:] != cf[:-1])
        starts = np.nonzero(head)[0]
        if starts.size != cf.size:
            vf = np.add.reduceat(vf, starts)
            cf = cf[starts]
            rows = rows[starts]
    counts = np.bincount(rows, minlength=m).astype(np.int64)
    rowptr = np.zeros(m + 1, dtype=np.int64)
    np.cumsum(counts, out=rowptr[1:])
    return rowptr, cf.astype(np.int32), vf


# ----------------------------------------------------------------------------
# spin chains
# ----------------------------------------------------------------------------


def xxz_bonds(L: int, J1: float, J2: float = 0.0, periodic: bool = True):
    """Bond list [(a, b, J)]: NN bonds i=0..L-1 then NNN bonds i=0..L-1."""
    bonds = []
    nn = L if periodic else L - 1
    for i in range(nn):
        bonds.append((i, (i + 1) % L, float(J1)))
    if J2 != 0.0:
        nnn = L if periodic else L - 2
        for i in range(nnn):
            bonds.append((i, (i + 2) % L, float(J2)))
    return bonds


def xxz_csr(L: int, J1: float, delta: float, h: np.ndarray, J2: float = 0.0,
            periodic: bool = True, rows: np.ndarray | None = None):
    """Real CSR of the XXZ(+NNN) chain on 2^L states.

    The diagonal is always stored (so nnz = sum_r (1 + #antiparallel bonds)).
    Diagonal accumulation order (fixed, FMA-free): start at 0.0, add
    J*Delta/4 * (+1 parallel / -1 antiparallel) for bonds in ``xxz_bonds``
    order, then +-h_i/2 for i = 0..L-1.

    ``rows`` restricts the build to a subset of rows (returns local CSR whose
    columns stay global) -- used for sampled checks at full size.
    """
    n = 1 << L
    r = np.arange(n, dtype=np.int64) if rows is None else np.asarray(rows, dtype=np.int64)
    bonds = xxz_bonds(L, J1, J2, periodic)
    nb = len(bonds)
    diag = np.zeros(r.shape[0], dtype=np.float64)
    cols = np.empty((r.shape[0], nb + 1), dtype=np.int64)
    vals = np.empty((r.shape[0], nb + 1), dtype=np.float64)
    valid = np.zeros((r.shape[0], nb + 1), dtype=bool)
    for k, (a, b, J) in enumerate(bonds):
        ba = (r >> a) & 1
        bb = (r >> b) & 1
        anti = ba != bb
        zz = J * delta * 0.25
        diag = diag + np.where(anti, -zz, zz)
        cols[:, k + 1] = r ^ ((1 << a) | (1 << b))
        vals[:, k + 1] = 0.5 * J
        valid[:, k + 1] = anti
    hv = np.asarray(h, dtype=np.float64)
    for i in range(L):
        bi = (r >> i) & 1
        half = 0.5 * hv[i]
        diag = diag + np.where(bi == 1, half, -half)
    cols[:, 0] = r
    vals[:, 0] = diag
    valid[:, 0] = True
    return _assemble(cols, vals, valid, n)


def xxz_fields(L: int, seed: int) -> np.ndarray:
    """h_i ~ U[-1, 1] as 2u - 1 (exact) from tag 10."""
    return 2.0 * rng.uniform(seed, 10, np.arange(L)) - 1.0


def neel_index(L: int) -> int:
    """Neel state with even sites up: bits 0, 2, 4, ... set."""
    return sum(1 << i for i in range(0, L, 2))


def product_state(L: int, seed: int) -> np.ndarray:
    """tensor_i (a_i |down> + b_i |up>) with cos(theta_i) ~ U[-1,1], phi_i ~ U[0, 2pi).

    a = cos(theta/2) = sqrt((1+c)/2), b = e^{i phi} sin(theta/2) = e^{i phi} sqrt((1-c)/2).
    Amplitude of index r is the product over sites in site order (site 0 first).
    """
    c = 2.0 * rng.uniform(seed, 20, np.arange(L)) - 1.0
    phi = 2.0 * math.pi * rng.uniform(seed, 21, np.arange(L))
    a = np.sqrt((1.0 + c) / 2.0).astype(np.complex128)
    b = np.exp(1j * phi) * np.sqrt((1.0 - c) / 2.0)
    v = np.ones(1, dtype=np.complex128)
    # index r = sum_i bit_i 2^i  ->  v_new[r + bit*2^i] = v[r] * f_i(bit)
    for i in range(L):
        v = np.concatenate([v * a[i], v * b[i]])
    return v


# ----------------------------------------------------------------------------
# Bose-Hubbard
# ----------------------------------------------------------------------------


def bh_basis(L: int, N: int) -> np.ndarray:
    """All occupation tuples with sum N, lexicographic (site 0 most significant,
    ascending): first (0,..,0,N), last (N,0,..,0).  Returns (d, L) uint8."""
    assert N <= 15 and L <= 16
    occ = np.zeros((1, 0), dtype=np.uint8)
    rem = np.array([N], dtype=np.int64)
    for site in range(L - 1):
        reps = rem + 1
        idx = np.repeat(np.arange(occ.shape[0]), reps)
        starts = np.cumsum(reps) - reps
        v = np.arange(idx.shape[0]) - np.repeat(starts, reps)
        occ = np.concatenate([occ[idx], v[:, None].astype(np.uint8)], axis=1)
        rem = rem[idx] - v
    occ = np.concatenate([occ, rem[:, None].astype(np.uint8)], axis=1)
    keys = bh_keys(occ)
    order = np.argsort(keys, kind="stable")
    return occ[order]


def bh_keys(occ: np.ndarray) -> np.ndarray:
    """4 bits per site, site 0 most significant (48-bit key for L = 12)."""
    L = occ.shape[1]
    k = np.zeros(occ.shape[0], dtype=np.int64)
    for i in range(L):
        k = (k << 4) | occ[:, i].astype(np.int64)
    return k


class BHIndexHash:
    """ind^-1 of the Bose-Hubbard basis as an open-addressing hash table (TimeEvolver
    indexes its basis with a hash map): slot = splitmix64 finaliser of
    the 48-bit occupation key, masked to a power-of-two capacity (2^22 for d = 1,352,078, load
    0.32), linear probing.  Built and queried with vectorised probe rounds (every still-unplaced
    key tries its next slot; the lowest basis index wins a contested empty slot, so the layout is
    deterministic).  Independent of ``searchsorted``;
    tests/test_workloads.py checks the two give bit-identical CSR arrays."""

    EMPTY = np.int64(-1)

    def __init__(self, keys: np.ndarray, capacity: int | None = None):
        d = keys.shape[0]
        cap = capacity or (1 << max(4, int(math.ceil(math.log2(max(2, 3 * d))))))
        assert cap & (cap - 1) == 0 and cap > d
        self.mask = np.uint64(cap - 1)
        self.slot_key = np.full(cap, -1, dtype=np.int64)
        self.slot_idx = np.full(cap, -1, dtype=np.int64)
        pend = np.arange(d, dtype=np.int64)
        pos = self._home(keys)
        while pend.size:
            s = pos[pend].astype(np.int64)
            free = self.slot_key[s] < 0
            # one winner per free slot: the smallest pending basis index (pend is ascending)
            cand = pend[free]
            cs = s[free]
            _, first = np.unique(cs, return_index=True)
            win = cand[first]
            self.slot_key[cs[first]] = keys[win]
            self.slot_idx[cs[first]] = win
            placed = np.zeros(d, dtype=bool)
            placed[win] = True
            pend = pend[~placed[pend]]
            pos[pend] = (pos[pend] + np.uint64(1)) & self.mask
        self.d = d

    def _home(self, keys):
        return rng.mix64(np.asarray(keys, dtype=np.int64).astype(np.uint64)) & self.mask

    def lookup(self, q: np.ndarray) -> np.ndarray:
        """Basis index of every key in q (-1 where the key is not in the basis)."""
        q = np.asarray(q, dtype=np.int64)
        out = np.full(q.shape[0], -1, dtype=np.int64)
        pend = np.arange(q.shape[0], dtype=np.int64)
        pos = self._home(q)
        while pend.size:
            s = pos[pend].astype(np.int64)
            k = self.slot_key[s]
            hit = k == q[pend]
            out[pend[hit]] = self.slot_idx[s[hit]]
            go = (~hit) & (k >= 0)            # occupied by another key: probe on
            pend = pend[go]
            pos[pend] = (pos[pend] + np.uint64(1)) & self.mask
        return out


def bh_mu(L: int, seed: int) -> np.ndarray:
    """mu_i ~ U[-0.5, 0.5] as u - 0.5 (exact) from tag 30."""
    return rng.uniform(seed, 30, np.arange(L)) - 0.5


def bose_hubbard_csr(L: int, N: int, J: float, U: float, mu: np.ndarray,
                     periodic: bool = False, index: str = "search"):
    """Real CSR of the Bose-Hubbard chain in the fixed-N sector.

    Diagonal order: 0.0, += (U/2) n_i (n_i - 1) for i ascending, then
    -= mu_i n_i for i ascending.  Hop amplitudes -J sqrt(n_s (n_t + 1)).
    Row/column index = position in ``bh_basis``; the inverse map ind^-1 is a
    sorted-key search (``index="search"``) or the open-addressing hash table of
    P:412 (``index="hash"``, ``BHIndexHash``) — bit-identical results.
    """
    occ = bh_basis(L, N)
    d = occ.shape[0]
    keys = bh_keys(occ)
    table = BHIndexHash(keys) if index == "hash" else None
    o = occ.astype(np.int64)
    diag = np.zeros(d, dtype=np.float64)
    for i in range(L):
        diag = diag + (0.5 * U) * (o[:, i] * (o[:, i] - 1)).astype(np.float64)
    for i in range(L):
        diag = diag - mu[i] * o[:, i].astype(np.float64)
    nbond = L if periodic else L - 1
    K = 1 + 2 * nbond
    cols = np.zeros((d, K), dtype=np.int64)
    vals = np.zeros((d, K), dtype=np.float64)
    valid = np.zeros((d, K), dtype=bool)
    cols[:, 0] = np.arange(d)
    vals[:, 0] = diag
    valid[:, 0] = True
    q = 1
    for bnd in range(nbond):
        i, j = bnd, (bnd + 1) % L
        si = np.int64(4 * (L - 1 - i))
        sj = np.int64(4 * (L - 1 - j))
        # b_i^+ b_j : needs n_j > 0
        for (a, b, sa, sb) in ((i, j, si, sj), (j, i, sj, si)):
            ok = o[:, b] > 0
            newkey = keys + (np.int64(1) << sa) - (np.int64(1) << sb)
            if table is None:
                tgt = np.searchsorted(keys, np.where(ok, newkey, keys))
            else:
                tgt = table.lookup(np.where(ok, newkey, keys))
                assert np.all(tgt >= 0)
            amp = -J * np.sqrt((o[:, b] * (o[:, a] + 1)).astype(np.float64))
            cols[:, q] = tgt
            vals[:, q] = amp
            valid[:, q] = ok
            q += 1
    rowptr, col, val = _assemble(cols, vals, valid, d)
    return occ, rowptr, col, val


# ----------------------------------------------------------------------------
# random Hermitian matrices from involutions
# ----------------------------------------------------------------------------


def _feistel_bits(n: int) -> int:
    b = max(2, (n - 1).bit_length())
    return b + (b & 1)


def feistel(x: np.ndarray, nbits: int, seed: int, tag: int, inverse: bool = False):
    """Keyed 4-round balanced Feistel bijection on [0, 2^nbits) (nbits even)."""
    half = nbits // 2
    mask = np.uint64((1 << half) - 1)
    x = np.asarray(x, dtype=np.uint64)
    hi = x >> np.uint64(half)
    lo = x & mask
    rounds = range(4) if not inverse else range(3, -1, -1)
    for r in rounds:
        if not inverse:
            f = rng.bits(seed, tag + r, lo) & mask
            hi, lo = lo, hi ^ f
        else:
            f = rng.bits(seed, tag + r, hi) & mask
            hi, lo = lo ^ f, hi
    return (hi << np.uint64(half)) | lo


def perm(x, n: int, seed: int, tag: int, inverse: bool = False) -> np.ndarray:
    """Bijection on [0, n) by cycle-walking the Feistel network."""
    nb = _feistel_bits(n)
    y = feistel(x, nb, seed, tag, inverse)
    while True:
        bad = y >= np.uint64(n)
        if not bad.any():
            return y
        y = np.where(bad, feistel(y, nb, seed, tag, inverse), y)


def uniform_involution(n: int, seed: int, tag: int, rows: np.ndarray):
    """pi(i) = sigma^-1(sigma(i) xor 1) and the pair id sigma(i) >> 1.
    Rows whose partner falls outside [0, n) (odd n) have no partner."""
    s = perm(rows, n, seed, tag)
    t = s ^ np.uint64(1)
    ok = t < np.uint64(n)
    p = perm(np.where(ok, t, s), n, seed, tag, inverse=True)
    return p.astype(np.int64), (s >> np.uint64(1)).astype(np.int64), ok


def band_involution(n: int, seed: int, k: int, rows: np.ndarray):
    """i -> i xor d_k(i >> 8) with 16 distinct d_k in [1, 255] per 256-block:
    d_k = 1 + ((r_blk + 15 k + u_{blk,k}) mod 255), u in [0, 15)."""
    blk = (rows >> 8).astype(np.uint64)
    r = (rng.bits(seed, 60, blk) % np.uint64(255)).astype(np.int64)
    u = (rng.bits(seed, 61, blk * np.uint64(16) + np.uint64(k)) % np.uint64(15)).astype(np.int64)
    d = 1 + ((r + 15 * k + u) % 255)
    p = rows ^ d
    ok = p < n
    pair = np.minimum(rows, p)
    return p, pair, ok


def involution_csr(n: int, seed: int, n_uniform: int, n_band: int = 0,
                   diagonal: bool = True, rows: np.ndarray | None = None):
    """Complex CSR sum of ``n_band`` band and ``n_uniform`` uniform involutions.

    Candidate order per row: diagonal (real N(0,1), tag 50), band involutions
    k = 0..n_band-1 (values tag 2000+2k), uniform involutions k = 0..n_uniform-1
    (Feistel tags 100+8k.., values tag 1000+2k).  Duplicate columns are summed
    in that order.  H_{i,j} = z for i < j and conj(z) for i > j.
    """
    r = np.arange(n, dtype=np.int64) if rows is None else np.asarray(rows, dtype=np.int64)
    K = (1 if diagonal else 0) + n_band + n_uniform
    cols = np.zeros((r.shape[0], K), dtype=np.int64)
    vals = np.zeros((r.shape[0], K), dtype=np.complex128)
    valid = np.zeros((r.shape[0], K), dtype=bool)
    q = 0
    if diagonal:
        cols[:, q] = r
        vals[:, q] = rng.normal(seed, 50, r)
        valid[:, q] = True
        q += 1
    for k in range(n_band):
        p, pair, ok = band_involution(n, seed, k, r)
        z = rng.complex_normal(seed, 2000 + 2 * k, pair)
        cols[:, q] = p
        vals[:, q] = np.where(r < p, z, np.conj(z))
        valid[:, q] = ok
        q += 1
    for k in range(n_uniform):
        p, pair, ok = uniform_involution(n, seed, 100 + 8 * k, r)
        z = rng.complex_normal(seed, 1000 + 2 * k, pair)
        cols[:, q] = p
        vals[:, q] = np.where(r < p, z, np.conj(z))
        valid[:, q] = ok
        q += 1
    return _assemble(cols, vals, valid, n)


def complex_gaussian_state(n: int, seed: int, tag: int = 70) -> np.ndarray:
    v = rng.complex_normal(seed, tag, np.arange(n))
    return v / np.linalg.norm(v)
