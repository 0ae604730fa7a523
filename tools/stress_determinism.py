"""Race detector without compute-sanitizer (the GPU pool refuses it): every kernel of the path is
deterministic, so the same Krylov decomposition repeated on fresh handles must be bitwise identical —
alpha, beta and the whole basis V.  A data race in an mbarrier ring, a missing fence before a
last-block reduction or an unordered workspace initialisation shows up as a mismatch (round 1 found
two bugs this way).  Runs every shipped SpMV format (slot-window one-pass and panel sweep, staged-x
with small tiles so that its ring wraps, column-blocked ring, ring, SELL), projection kernel set
and orthogonalisation mode; m = 40 reaches every instantiation of the TMA projection kernels.

  python tools/stress_determinism.py [reps]     # prints mismatches per (case, configuration)"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
from paper_2205_15346_b200 import te  # noqa: E402
from workloads import configs  # noqa: E402

reps = int(sys.argv[1]) if len(sys.argv) > 1 else 20
cases = {"xxznnn_L14": configs.build(5, L=14), "xxz_L16": configs.build(2, L=16), "bh_L8_N8": configs.build(3, L=8, N=8),
         "cfg1_n4096": configs.build(1), "banded_n65536": configs.build(4, n=65536)}
# (label, environment read at create, SpMV option or None for the default, kernel set, ortho)
runs = [("default", {}, None, 2, 0),
        ("sw one pass", {"TE_SPMV_SW_FORCE": "1", "TE_SPMV_SW_PANEL": "0"}, 9, 2, 0),
        ("sw panel sweep", {"TE_SPMV_SW_FORCE": "1", "TE_SPMV_SW_PANEL": "5"}, 9, 2, 0),
        ("sw panel sweep, lanczos", {"TE_SPMV_SW_FORCE": "1", "TE_SPMV_SW_PANEL": "5"}, 9, 2, 1),
        ("staged-x small tiles", {"TE_SPMV_XS_ECAP": "256"}, 8, 2, 0),
        ("column-blocked ring", {"TE_SPMV_COLBLK_MB": "0.05"}, 10, 2, 0),
        ("ring tpr 4 halo-aware", {"TE_SPMV_RING_TPR": "4", "TE_SPMV_FORCE_HALO": "1"}, 7, 2, 0),
        ("ring 3 stages", {"TE_SPMV_RING_STAGES": "3"}, 7, 2, 0),
        ("sell", {}, 6, 2, 0),
        ("tma projections only", {}, 7, 3, 0),
        ("tma projections, runtime R", {"TE_PROJ_CONST_R": "0"}, 7, 3, 0),
        ("register projections only", {}, 7, 5, 0),
        ("cgs2gram", {}, 7, 2, 2)]
total_bad = 0
for name, c in cases.items():
    for label, env, spmv, kset, ortho in runs:
        for k, v in env.items():
            os.environ[k] = v
        ref, bad, skipped = None, 0, False
        for r in range(reps):
            h = te.te_create_csr(c["n"], c["rowptr"], c["col"], c["val"])  # fresh handle each time
            try:
                if spmv is not None:
                    te.te_set_option(h, te.TE_OPT_SPMV, spmv)
            except te.TEError:
                skipped = True
                h.close()
                break
            te.te_set_option(h, te.TE_OPT_KERNELS, kset)
            te.te_set_option(h, te.TE_OPT_ORTHO, ortho)
            g = te.te_krylov_basis(h, c["v0"], 40, 1e-14, want_V=True)
            h.close()
            a = np.concatenate([g["alpha"], g["beta"], g["V"].view(np.float64).ravel()])
            if ref is None:
                ref = a
            elif not np.array_equal(a.view(np.uint64), ref.view(np.uint64)):
                bad += 1
        for k in env:
            del os.environ[k]
        total_bad += bad
        print(f"{name:14s} {label:28s} " + ("not applicable" if skipped else f"mismatches={bad}/{reps - 1}"), flush=True)
print("total mismatches", total_bad)
sys.exit(1 if total_bad else 0)
