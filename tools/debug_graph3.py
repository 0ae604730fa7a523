import sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
from paper_2205_15346_b200 import te
from workloads import configs
torch.cuda.set_device(0)
c = configs.build(2, L=14)
def run(tag, opts, dev=True):
    h = te.te_create_csr(c["n"], c["rowptr"], c["col"], c["val"])
    for o, v in opts:
        te.te_set_option(h, o, v)
    d0 = torch.from_numpy(c["v0"]).cuda(); d1 = torch.empty_like(d0)
    try:
        if dev:
            st = te.te_evolve_dev(h, d0, 3.0, 1e-10, 40, d1, stream=torch.cuda.current_stream())
        else:
            v, st = te.te_evolve(h, c["v0"], 3.0, 1e-10, 40)
        print(tag, "ok", flush=True)
    except Exception as e:
        print(tag, "FAIL", e, flush=True)
    h.close()
run("kernels2", [(te.TE_OPT_KERNELS, 2)])
run("kernels3", [(te.TE_OPT_KERNELS, 3)])
run("profile", [(te.TE_OPT_PROFILE, 1)], dev=False)
run("profile-nograph", [(te.TE_OPT_GRAPH, 0), (te.TE_OPT_PROFILE, 1)], dev=False)
run("graph0", [(te.TE_OPT_GRAPH, 0)])
run("spmv1", [(te.TE_OPT_SPMV, 1)])
