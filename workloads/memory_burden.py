"""The paper's own example system, §5 "Exemplary System".

Input generator only (no Krylov arithmetic).  Modes |n0, m0, n_1..n_K, n'_1..n'_K'>
(Eq. genericStateExample); a0, b0 bosonic with N0 = n0 + m0 conserved,
the K + K' memory modes are qubits with N_m = sum n_k + sum n'_k' conserved
(P:431-435).  Hamiltonian Eq. fullHamiltonianSimple with the
couplings f_i.  Basis order: sector {a0, b0} slowest, each sector
lexicographic ascending in its occupation tuple (SPEC fock-basis reading).
Normalised ladder factors sqrt(n), sqrt(n+1); qubit creation on |1> vanishes.
"""
from __future__ import annotations

import itertools
import math

import numpy as np

DEFAULTS = dict(eps_m=math.sqrt(20.0), N0=20, Nc=20, dNc=12, K=4, K1=4, C0=1.0, Cm=1.0, Nm=2)


def coupling(i: int, k: int, l: int, K: int) -> float:
    """f_i(k, l) with F_i = (sqrt2 (k+dk_i)^3 + sqrt7 (l+dl_i)^5) mod 1."""
    dk = {1: 1, 2: 1, 3: K + 1}[i]
    dl = {1: K + 1, 2: 1, 3: K + 1}[i]
    F = (math.sqrt(2.0) * (k + dk) ** 3 + math.sqrt(7.0) * (l + dl) ** 5) % 1.0
    return F - 1.0 if F < 0.5 else F


def basis(p: dict):
    """(d, 2 + K + K') int array of occupation tuples in basis order."""
    N0, K, K1, Nm = p["N0"], p["K"], p["K1"], p["Nm"]
    s1 = [(n0, N0 - n0) for n0 in range(N0 + 1)]                      # lexicographic (n0, m0)
    q = K + K1
    s2 = sorted(t for t in itertools.product((0, 1), repeat=q) if sum(t) == Nm)
    occ = np.array([a + b for a in s1 for b in s2], dtype=np.int64)
    return occ, len(s1), len(s2)


def dimension(p: dict) -> int:
    return (p["N0"] + 1) * math.comb(p["K"] + p["K1"], p["Nm"])


def hamiltonian(p: dict | None = None):
    """Real CSR (rowptr, col, val), the basis and the initial state index
    |N0, 0, 1..1 (N_m), 0..0> (Eq. initialStateSimple)."""
    p = dict(DEFAULTS, **(p or {}))
    occ, d1, d2 = basis(p)
    K, K1 = p["K"], p["K1"]
    index = {tuple(r): i for i, r in enumerate(occ)}   # ind^-1 by hash table
    d = occ.shape[0]
    rows, cols, vals = [], [], []
    for i in range(d):
        s = occ[i]
        n0, m0 = s[0], s[1]
        qa = s[2: 2 + K]
        qb = s[2 + K:]
        ent = {}
        diag = p["eps_m"] * (1.0 - n0 / p["Nc"]) * float(qa.sum()) \
            + p["eps_m"] * (1.0 - n0 / (p["Nc"] - p["dNc"])) * float(qb.sum())
        ent[i] = diag
        # C0 (a0^+ b0 + b0^+ a0)
        if m0 > 0:
            t = s.copy(); t[0] += 1; t[1] -= 1
            j = index[tuple(t)]
            ent[j] = ent.get(j, 0.0) + p["C0"] * math.sqrt((n0 + 1) * m0)
        if n0 > 0:
            t = s.copy(); t[0] -= 1; t[1] += 1
            j = index[tuple(t)]
            ent[j] = ent.get(j, 0.0) + p["C0"] * math.sqrt(n0 * (m0 + 1))

        def hop(a, b, c):  # c (a_a^+ a_b + a_b^+ a_a) on qubit positions a, b
            for x, y in ((a, b), (b, a)):
                if s[y] == 1 and s[x] == 0:
                    t = s.copy(); t[x] = 1; t[y] = 0
                    j = index[tuple(t)]
                    ent[j] = ent.get(j, 0.0) + c

        for k in range(1, K + 1):
            for k1 in range(1, K1 + 1):
                hop(1 + k, 1 + K + k1, p["Cm"] * coupling(1, k, k1, K))
        for k in range(1, K + 1):
            for l in range(k + 1, K + 1):
                hop(1 + k, 1 + l, p["Cm"] * coupling(2, k, l, K))
        for k1 in range(1, K1 + 1):
            for l1 in range(k1 + 1, K1 + 1):
                hop(1 + K + k1, 1 + K + l1, p["Cm"] * coupling(3, k1, l1, K))
        for j in sorted(ent):
            rows.append(i); cols.append(j); vals.append(ent[j])
    rowptr = np.zeros(d + 1, dtype=np.int64)
    np.cumsum(np.bincount(np.array(rows), minlength=d), out=rowptr[1:])
    init = np.zeros(2 + K + K1, dtype=np.int64)
    init[0] = p["N0"]
    init[2: 2 + p["Nm"]] = 1
    return dict(rowptr=rowptr, col=np.array(cols, dtype=np.int32), val=np.array(vals),
                occ=occ, init_index=index[tuple(init)], n=d)


def _pair_couplings(p: dict) -> np.ndarray:
    """q x q symmetric table of the hop amplitude between qubit positions (0-based within the
    memory sector), same three loops and the same coupling() calls as hamiltonian()."""
    K, K1 = p["K"], p["K1"]
    q = K + K1
    C = np.zeros((q, q))
    for k in range(1, K + 1):
        for k1 in range(1, K1 + 1):
            C[k - 1, K + k1 - 1] = C[K + k1 - 1, k - 1] = p["Cm"] * coupling(1, k, k1, K)
    for k in range(1, K + 1):
        for l in range(k + 1, K + 1):
            C[k - 1, l - 1] = C[l - 1, k - 1] = p["Cm"] * coupling(2, k, l, K)
    for k1 in range(1, K1 + 1):
        for l1 in range(k1 + 1, K1 + 1):
            C[K + k1 - 1, K + l1 - 1] = C[K + l1 - 1, K + k1 - 1] = p["Cm"] * coupling(3, k1, l1, K)
    return C


def hamiltonian_fast(p: dict | None = None):
    """Same CSR as hamiltonian(), bit for bit, built with numpy for the paper-size instance
    (K=K'=10, N_m=5, N0=Nc=100, d=1,565,904, ~78 entries per row).

    Structure used: the basis is the product sector1 x sector2 (index i1*d2 + i2);
    each row holds the two C0 terms of sector 1 (columns (i1 -+ 1)*d2 + i2), the diagonal and
    N_m (q - N_m) memory-sector hops (columns i1*d2 + i2').  Every qubit pair belongs to exactly
    one of the three coupling loops, so each hop target is reached once and no entries sum."""
    p = dict(DEFAULTS, **(p or {}))
    N0, K, K1, Nm = p["N0"], p["K"], p["K1"], p["Nm"]
    q = K + K1
    # sector 2: tuples with sum N_m in lexicographic order == integers with popcount N_m
    # ascending, tuple position x <-> bit (q-1-x)
    r = np.arange(1 << q, dtype=np.int64)
    pc = np.zeros_like(r)
    for b in range(q):
        pc += (r >> b) & 1
    s2 = r[pc == Nm]
    d2 = s2.shape[0]
    rank2 = np.full(1 << q, -1, dtype=np.int64)
    rank2[s2] = np.arange(d2)
    bits = ((s2[:, None] >> (q - 1 - np.arange(q))[None, :]) & 1).astype(np.int64)   # (d2, q)
    C = _pair_couplings(p)
    # memory-sector hops: for each occupied y and empty x, target s ^ bit(x) ^ bit(y)
    src, dst, amp = [], [], []
    for x in range(q):
        for y in range(q):
            if x == y:
                continue
            sel = np.nonzero((bits[:, y] == 1) & (bits[:, x] == 0))[0]
            tgt = s2[sel] ^ (1 << (q - 1 - x)) ^ (1 << (q - 1 - y))
            src.append(sel); dst.append(rank2[tgt]); amp.append(np.full(sel.shape[0], C[x, y]))
    src, dst, amp = np.concatenate(src), np.concatenate(dst), np.concatenate(amp)
    # add the diagonal slot (value filled per i1) and sort every sector-2 row by column
    src = np.concatenate([src, np.arange(d2)])
    dst = np.concatenate([dst, np.arange(d2)])
    amp = np.concatenate([amp, np.zeros(d2)])
    isdiag = np.concatenate([np.zeros(src.shape[0] - d2, bool), np.ones(d2, bool)])
    o = np.lexsort((dst, src))
    src, dst, amp, isdiag = src[o], dst[o], amp[o], isdiag[o]
    per = np.bincount(src, minlength=d2)
    assert np.all(per == per[0]) and per[0] == 1 + Nm * (q - Nm)
    w = int(per[0])
    cols2 = dst.reshape(d2, w)
    amps2 = amp.reshape(d2, w)
    dpos = np.nonzero(isdiag.reshape(d2, w))[1]
    qa = bits[:, :K].sum(axis=1)
    qb = bits[:, K:].sum(axis=1)
    d1 = N0 + 1
    d = d1 * d2
    rows_nnz = np.empty(d, dtype=np.int64)
    col_blocks, val_blocks = [], []
    for i1 in range(d1):
        n0, m0 = np.int64(i1), np.int64(N0 - i1)
        left, right = n0 > 0, m0 > 0
        width = w + int(left) + int(right)
        cb = np.empty((d2, width), dtype=np.int64)
        vb = np.empty((d2, width))
        c = 0
        if left:   # (n0-1, m0+1) sits one sector-1 block lower
            cb[:, 0] = (i1 - 1) * d2 + np.arange(d2)
            vb[:, 0] = p["C0"] * math.sqrt(n0 * (m0 + 1))
            c = 1
        cb[:, c: c + w] = i1 * d2 + cols2
        diag = p["eps_m"] * (1.0 - n0 / p["Nc"]) * qa.astype(np.float64) \
            + p["eps_m"] * (1.0 - n0 / (p["Nc"] - p["dNc"])) * qb.astype(np.float64)
        blk = amps2.copy()
        blk[np.arange(d2), dpos] = diag
        vb[:, c: c + w] = blk
        if right:  # (n0+1, m0-1)
            cb[:, c + w] = (i1 + 1) * d2 + np.arange(d2)
            vb[:, c + w] = p["C0"] * math.sqrt((n0 + 1) * m0)
        rows_nnz[i1 * d2: (i1 + 1) * d2] = width
        col_blocks.append(cb.ravel().astype(np.int32))
        val_blocks.append(vb.ravel())
    rowptr = np.zeros(d + 1, dtype=np.int64)
    np.cumsum(rows_nnz, out=rowptr[1:])
    init_bits = np.zeros(q, dtype=np.int64)
    init_bits[:Nm] = 1
    init2 = int(rank2[int((init_bits << (q - 1 - np.arange(q))).sum())])
    return dict(rowptr=rowptr, col=np.concatenate(col_blocks), val=np.concatenate(val_blocks),
                init_index=N0 * d2 + init2, n=d)
