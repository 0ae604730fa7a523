"""Small evolutions through every shipped SpMV format (slot-window SELL-32, column-blocked ring,
staged-x, ring, SELL-sigma), projection kernel set and
orthogonalisation mode, for compute-sanitizer (memcheck / racecheck / synccheck;
tools/sanitize.sh).  Sizes span several tiles per CTA: the staged-x SpMV runs with small tiles
(TE_SPMV_XS_ECAP=256) so its mbarrier ring wraps; the column-blocked ring with 1 KB column blocks;
the slot-window format with the padding check overridden (small chains), as one pass and as the
two-pass panel sweep (panels of 4 slices)."""
import os
import sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
os.environ.setdefault("TE_SPMV_XS_ECAP", "256")
os.environ.setdefault("TE_SPMV_COLBLK_MB", str(1.0 / 1024))
os.environ.setdefault("TE_SPMV_SW_FORCE", "1")
from paper_2205_15346_b200 import te  # noqa: E402
from workloads import configs  # noqa: E402

cases = [configs.build(2, L=12), configs.build(3, L=6, N=6), configs.build(1, n=1000), configs.build(5, L=11)]
# (kernel set, SpMV, ortho)
runs = [(2, 9, 0), (2, "9-panel", 0), (2, "9-panel", 1), (2, 10, 0), (2, 8, 0), (2, 7, 0), (2, 6, 0), (3, 7, 0), (5, 7, 0),
        (2, 8, 2), (2, 8, 1)]
for c in cases:
    for kset, spmv, ortho in runs:
        os.environ["TE_SPMV_SW_PANEL"] = "2" if spmv == "9-panel" else "0"
        spmv = 9 if spmv == "9-panel" else spmv
        h = te.te_create_csr(c["n"], c["rowptr"], c["col"], c["val"])
        te.te_set_option(h, te.TE_OPT_KERNELS, kset)
        try:
            te.te_set_option(h, te.TE_OPT_SPMV, spmv)
        except te.TEError:  # SELL refuses very uneven rows; the slot-window format needs a dictionary
            pass
        te.te_set_option(h, te.TE_OPT_ORTHO, ortho)
        v, st = te.te_evolve(h, c["v0"], 0.5, 1e-8, 24)
        h.close()
    print(c["name"], c["n"], "ok", st["n_restarts"], flush=True)
print("sanitize run done")
