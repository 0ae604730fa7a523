"""SpMV variant sweep on one BASELINE config (GPU): the matrix is built once, then for every variant
(environment settings read at create + TE_OPT_SPMV) a handle is created, a short Krylov basis is
run with per-launch CUDA events (TE_OPT_PROFILE) and the SpMV's time per launch is printed with
its algorithmic GB/s and the staged-x plan statistics.

  python tools/spmv_sweep.py --config 5 --m 6 --reps 2 \
      --variant "9:" --variant "8:" --variant "8:TE_SPMV_XS_STAGES=3" --variant "7:"
A variant is "<spmv>:<ENV=VAL,ENV=VAL,...>" (spmv: 10 column-blocked ring, 9 slot-window SELL-32,
8 staged-x, 7 ring, 6 SELL-sigma)."""
from __future__ import annotations

import argparse
import json
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import numpy as np  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--config", type=int, default=5)
    ap.add_argument("--m", type=int, default=6)
    ap.add_argument("--reps", type=int, default=2)
    ap.add_argument("--variant", action="append", default=[])
    a = ap.parse_args()
    from paper_2205_15346_b200 import te
    from workloads import configs
    t0 = time.time()
    c = configs.build(a.config)
    print(f"# config {a.config}: n={c['n']} nnz={int(c['rowptr'][-1])} built in {time.time() - t0:.1f}s", flush=True)
    base_env = dict(os.environ)
    for var in a.variant or ["8:", "7:"]:
        spmv, _, envs = var.partition(":")
        os.environ.clear()
        os.environ.update(base_env)
        for kv in filter(None, envs.split(",")):
            k, _, v = kv.partition("=")
            os.environ[k] = v
        t1 = time.time()
        h = te.te_create_csr(c["n"], c["rowptr"], c["col"], c["val"])
        tc = time.time() - t1
        try:
            te.te_set_option(h, te.TE_OPT_SPMV, int(spmv))
        except te.TEError as e:
            print(json.dumps({"variant": var, "error": str(e)}), flush=True)
            h.close()
            continue
        info = {k: te.te_get_option(h, getattr(te, k)) for k in ("TE_INFO_XS_GLOBAL", "TE_INFO_XS_GLOBAL_TILES", "TE_INFO_XS_X_PER_ENTRY", "TE_INFO_SW_FILL", "TE_INFO_SW_PANEL", "TE_INFO_SW_FAR")}
        te.te_krylov_basis(h, c["v0"], a.m, 0.0, want_V=False)  # warm-up
        te.te_set_option(h, te.TE_OPT_PROFILE, 1)
        for _ in range(a.reps):
            te.te_krylov_basis(h, c["v0"], a.m, 0.0, want_V=False)
        p = te.te_get_profile(h)["spmv"]
        ms = p["total_ms"] / max(1, p["launches"])
        out = {"variant": var, "spmv_ran": te.te_get_option(h, te.TE_OPT_SPMV), "ms_per_launch": ms,
               "alg_gbs": p["alg_bytes"] / max(1, p["launches"]) / ms / 1e6, "alg_gb_per_launch": p["alg_bytes"] / max(1, p["launches"]) / 1e9,
               "create_s": tc, **{k.lower(): v for k, v in info.items()}}
        print(json.dumps(out), flush=True)
        h.close()


if __name__ == "__main__":
    main()
