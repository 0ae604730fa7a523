"""Small evolutions through every kernel set / SpMV variant / ortho mode, for compute-sanitizer."""
import os
import sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
from paper_2205_15346_b200 import te
from workloads import configs

cases = [configs.build(2, L=12), configs.build(3, L=6, N=6), configs.build(1, n=1000), configs.build(5, L=11)]
for c in cases:
    for kset, spmv, ortho in [(2, 4, 0), (3, 4, 0), (4, 4, 0), (0, 4, 0), (1, 4, 0), (2, 3, 0), (2, 2, 0), (2, 1, 0),
                              (2, 0, 0), (2, 4, 1)]:
        h = te.te_create_csr(c["n"], c["rowptr"], c["col"], c["val"])
        te.te_set_option(h, te.TE_OPT_KERNELS, kset)
        te.te_set_option(h, te.TE_OPT_SPMV, spmv)
        te.te_set_option(h, te.TE_OPT_ORTHO, ortho)
        v, st = te.te_evolve(h, c["v0"], 0.5, 1e-8, 24)
        h.close()
    print(c["name"], c["n"], "ok", st["n_restarts"], flush=True)
print("sanitize run done")
