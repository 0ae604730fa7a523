"""The five BASELINE.json configs as concrete seeded synthetic inputs.

``build(i, **scale)`` returns a dict with the CSR (rowptr int64, col int32,
val float64|complex128), ``v0`` (complex128, normalised), ``t``, ``tol``, ``m``
and a ``name``.  Seeds are the config index.  Keyword
overrides shrink a config for tests (same model, smaller L / n), e.g.
``build(2, L=12)`` or ``build(3, L=6, N=6)``.

Config strings (BASELINE.json "configs"):
 1 random sparse Hermitian n=4096 complex, ~16 nnz/row uniform, real diag; t=10 tol=1e-8 m=40
 2 XXZ periodic L=20, J=1, Delta=0.5, h_i~U[-1,1], Neel v0; t=20 tol=1e-10 m=40
 3 Bose-Hubbard L=12 N=12 (n=1,352,078), J=1 U=2 mu_i~U[-.5,.5], v0=|1..1>; t=5 tol=1e-8 m=50
 4 random n=2^24 complex, 32 nnz/row (16 band within +-255, 16 uniform); t=2 tol=1e-8 m=30
 5 XXZ+NNN periodic L=26, J1=1 J2=0.5 Delta=1, h_i~U[-1,1], product v0; t=10 tol=1e-10 m=40
 6 (not in BASELINE.json) the paper's own benchmark, §5 memory-burden model at
   K=K'=10, N_m=5, N0=Nc=100 (d=1,565,904), initial state Eq. initialStateSimple; t=10
   err_max=1e-7 m=40.  Deterministic (no random draws): the couplings f_i are P:452-460.
"""
from __future__ import annotations

import numpy as np

from . import fast, memory_burden, models, parallel_build

NAMES = {
    1: "random_herm_n4096",
    2: "xxz_L20",
    3: "bose_hubbard_L12_N12",
    4: "random_banded_n2^24",
    5: "xxz_nnn_L26",
    6: "paper_s5_memory_burden_d1565904",
}

LABELS = {i: f"BASELINE configs[{i - 1}]" for i in range(1, 6)}
LABELS[6] = "paper §5 P:527 benchmark (353 s on 1 CPU thread in the paper)"


def params(i: int, **ov):
    if i == 1:
        p = dict(n=4096, t=10.0, tol=1e-8, m=40)
    elif i == 2:
        p = dict(L=20, J=1.0, delta=0.5, t=20.0, tol=1e-10, m=40)
    elif i == 3:
        p = dict(L=12, N=12, J=1.0, U=2.0, t=5.0, tol=1e-8, m=50)
    elif i == 4:
        p = dict(n=1 << 24, t=2.0, tol=1e-8, m=30)
    elif i == 5:
        p = dict(L=26, J1=1.0, J2=0.5, delta=1.0, t=10.0, tol=1e-10, m=40)
    elif i == 6:
        p = dict(K=10, K1=10, Nm=5, N0=100, Nc=100, t=10.0, tol=1e-7, m=40)
    else:
        raise ValueError(i)
    p.update(ov)
    return p


def build(i: int, with_matrix: bool = True, **ov):
    p = params(i, **ov)
    seed = i
    out = dict(cfg=i, name=NAMES[i], t=p["t"], tol=p["tol"], m=p["m"], params=p)
    if i == 1:
        n = p["n"]
        if with_matrix:
            build_inv = parallel_build.involution_csr_parallel if n >= (1 << 20) else models.involution_csr
            out["rowptr"], out["col"], out["val"] = build_inv(n, seed, n_uniform=16, diagonal=True)
        out["v0"] = models.complex_gaussian_state(n, seed)
    elif i == 4:
        n = p["n"]
        if with_matrix:
            build_inv = parallel_build.involution_csr_parallel if n >= (1 << 20) else models.involution_csr
            out["rowptr"], out["col"], out["val"] = build_inv(n, seed, n_uniform=16, n_band=16, diagonal=False)
        out["v0"] = models.complex_gaussian_state(n, seed)
    elif i == 2:
        L = p["L"]
        n = 1 << L
        h = models.xxz_fields(L, seed)
        out["fields"] = h
        if with_matrix:
            build_xxz = fast.xxz_csr_fast if L > 22 else models.xxz_csr
            out["rowptr"], out["col"], out["val"] = build_xxz(L, p["J"], p["delta"], h)
        v0 = np.zeros(n, dtype=np.complex128)
        v0[models.neel_index(L)] = 1.0
        out["v0"] = v0
    elif i == 5:
        L = p["L"]
        n = 1 << L
        h = models.xxz_fields(L, seed)
        out["fields"] = h
        if with_matrix:
            build_xxz = fast.xxz_csr_fast if L > 20 else models.xxz_csr
            out["rowptr"], out["col"], out["val"] = build_xxz(L, p["J1"], p["delta"], h, J2=p["J2"])
        out["v0"] = models.product_state(L, seed)
    elif i == 3:
        L, N = p["L"], p["N"]
        mu = models.bh_mu(L, seed)
        out["mu"] = mu
        occ, rp, c, v = models.bose_hubbard_csr(L, N, p["J"], p["U"], mu)
        n = occ.shape[0]
        if with_matrix:
            out["rowptr"], out["col"], out["val"] = rp, c, v
        keys = models.bh_keys(occ)
        target = models.bh_keys(np.ones((1, L), dtype=np.uint8))[0] if N == L else None
        v0 = np.zeros(n, dtype=np.complex128)
        if target is not None:
            v0[int(np.searchsorted(keys, target))] = 1.0
        else:  # uniform filling not possible: put the bosons as evenly as possible
            occ0 = np.zeros((1, L), dtype=np.uint8)
            for b in range(N):
                occ0[0, b % L] += 1
            v0[int(np.searchsorted(keys, models.bh_keys(occ0)[0]))] = 1.0
        out["v0"] = v0
        out["occ"] = occ
    elif i == 6:
        mp = {k: p[k] for k in p if k not in ("t", "tol", "m")}
        H = memory_burden.hamiltonian_fast(mp)
        if with_matrix:
            out["rowptr"], out["col"], out["val"] = H["rowptr"], H["col"], H["val"]
        v0 = np.zeros(H["n"], dtype=np.complex128)
        v0[H["init_index"]] = 1.0
        out["v0"] = v0
    out["n"] = out["v0"].shape[0]
    return out
