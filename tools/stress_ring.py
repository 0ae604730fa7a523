"""Race detector for the SpMV kernels: the same Krylov decomposition, repeated, must be bitwise
identical (every kernel is deterministic).  Prints mismatch counts per (case, SpMV variant)."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
from paper_2205_15346_b200 import te
from workloads import configs

def long_rows():
    import scipy.sparse as sp
    n = 3000
    g = np.random.default_rng(11)
    A = np.zeros((n, n), complex)
    A[np.arange(n), np.arange(n)] = g.standard_normal(n)
    for r in (5, 1700):
        cols = g.choice(n, 1500, replace=False)
        A[r, cols] = g.standard_normal(1500) + 1j * g.standard_normal(1500)
    A = (A + A.conj().T) / 2
    S = sp.csr_matrix(A); S.sort_indices()
    v0 = g.standard_normal(n) + 1j * g.standard_normal(n)
    return dict(n=n, rowptr=S.indptr.astype(np.int64), col=S.indices.astype(np.int32), val=S.data, v0=v0 / np.linalg.norm(v0))

cases = {"xxznnn_L12": configs.build(5, L=12), "long_rows": long_rows(), "cfg1": configs.build(1),
         "xxz_L16": configs.build(2, L=16)}
reps = int(sys.argv[1]) if len(sys.argv) > 1 else 50
envsets = [dict(), dict(TE_SPMV_TPR="4", TE_SPMV_FORCE_HALO="1"), dict(TE_SPMV_RING_TPR="8"), dict(TE_SPMV_RING_STAGES="3")]
for name, c in cases.items():
    for env in envsets:
        for k, v in env.items(): os.environ[k] = v
        for spmv in (7, 4):
            ref = None; bad = 0
            for r in range(reps):
                h = te.te_create_csr(c["n"], c["rowptr"], c["col"], c["val"])   # fresh handle each time
                te.te_set_option(h, te.TE_OPT_SPMV, spmv)
                g = te.te_krylov_basis(h, c["v0"], 12, 1e-12, want_V=False)
                h.close()
                a = np.concatenate([g["alpha"], g["beta"]])
                if ref is None: ref = a
                elif not np.array_equal(a.view(np.uint64), ref.view(np.uint64)): bad += 1
            print(f"{name:12s} env={env} spmv={spmv} mismatches={bad}/{reps-1}", flush=True)
        for k in env: del os.environ[k]
