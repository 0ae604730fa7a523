import sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
from paper_2205_15346_b200 import te
from workloads import configs
c = configs.build(2, L=14)
s = torch.cuda.current_stream()
print("torch stream", s.cuda_stream, flush=True)
for graph in (1, 0):
    for first in ("dev", "host"):
        h = te.te_create_csr(c["n"], c["rowptr"], c["col"], c["val"])
        te.te_set_option(h, te.TE_OPT_GRAPH, graph)
        d0 = torch.from_numpy(c["v0"]).cuda(); d1 = torch.empty_like(d0)
        try:
            if first == "host":
                te.te_evolve(h, c["v0"], 3.0, 1e-10, 40)
            st = te.te_evolve_dev(h, d0, 3.0, 1e-10, 40, d1, stream=s)
            st = te.te_evolve_dev(h, d0, 3.0, 1e-10, 40, d1, stream=None)
            print("graph", graph, first, "ok", st["n_restarts"], flush=True)
        except Exception as e:
            print("graph", graph, first, "FAIL", e, flush=True)
        h.close()
