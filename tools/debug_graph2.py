import sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
from paper_2205_15346_b200 import te
from workloads import configs
torch.cuda.set_device(0)
for L in (14, 16, 18, 20):
    c = configs.build(2, L=L)
    for graph in (1, 0):
        h = te.te_create_csr(c["n"], c["rowptr"], c["col"], c["val"])
        te.te_set_option(h, te.TE_OPT_GRAPH, graph)
        d0 = torch.from_numpy(c["v0"]).cuda(); d1 = torch.empty_like(d0)
        try:
            st = te.te_evolve_dev(h, d0, 20.0, 1e-10, 40, d1, stream=torch.cuda.current_stream())
            print(L, "graph", graph, "ok", st["n_restarts"], flush=True)
        except Exception as e:
            print(L, "graph", graph, "FAIL", e, flush=True)
        h.close()
