"""Small driver for ncu: one short evolution of a BASELINE config through the C ABI."""
import argparse
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))


def main():
    from paper_2205_15346_b200 import te
    from workloads import configs
    ap = argparse.ArgumentParser()
    ap.add_argument("--config", type=int, default=2)
    ap.add_argument("--t", type=float, default=None)
    ap.add_argument("--kernels", type=int, default=2)
    ap.add_argument("--spmv", type=int, default=None)
    a = ap.parse_args()
    c = configs.build(a.config)
    h = te.te_create_csr(c["n"], c["rowptr"], c["col"], c["val"])
    te.te_set_option(h, te.TE_OPT_KERNELS, a.kernels)
    if a.spmv is not None:
        te.te_set_option(h, te.TE_OPT_SPMV, a.spmv)
    t = a.t if a.t is not None else c["t"] / 8
    v, st = te.te_evolve(h, c["v0"], t, c["tol"] * t / c["t"], c["m"])
    print("restarts", st["n_restarts"], "steps", st["n_krylov_steps"], "bound", st["err_bound"])


if __name__ == "__main__":  # the config-4 builder starts a forkserver pool: guarded main
    main()
