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
