"""Projection-kernel variant sweep on one BASELINE config (GPU): for every variant (environment
settings read when the library configures its kernels: one process per variant) a full Krylov basis
of m columns is built with per-launch CUDA events (TE_OPT_PROFILE) and the time and algorithmic
GB/s of the proj_dots / update_proj / update_norm classes are printed.

  python tools/proj_sweep.py --config 5 --variant "" --variant "TE_PROJ_CONST_R=0" """
from __future__ import annotations

import argparse
import json
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def one(cfg, m, reps):
    from paper_2205_15346_b200 import te
    from workloads import configs
    c = configs.build(cfg)
    h = te.te_create_csr(c["n"], c["rowptr"], c["col"], c["val"])
    te.te_krylov_basis(h, c["v0"], m, 0.0, want_V=False)
    te.te_set_option(h, te.TE_OPT_PROFILE, 1)
    for _ in range(reps):
        te.te_krylov_basis(h, c["v0"], m, 0.0, want_V=False)
    p = te.te_get_profile(h)
    out = {}
    for k in ("spmv", "proj_dots", "update_proj", "update_norm"):
        q = p[k]
        ms = q["total_ms"] / max(1, q["launches"])
        out[k] = {"ms": round(ms, 4), "gbs": round(q["alg_bytes"] / max(1, q["launches"]) / ms / 1e6, 1)}
    print(json.dumps(out), flush=True)
    h.close()


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--config", type=int, default=5)
    ap.add_argument("--m", type=int, default=40)
    ap.add_argument("--reps", type=int, default=2)
    ap.add_argument("--variant", action="append", default=[])
    ap.add_argument("--child", action="store_true")
    a = ap.parse_args()
    if a.child:
        one(a.config, a.m, a.reps)
        return
    for var in a.variant or [""]:
        env = dict(os.environ)
        for kv in filter(None, var.split(",")):
            k, _, v = kv.partition("=")
            env[k] = v
        r = subprocess.run([sys.executable, os.path.abspath(__file__), "--child", "--config", str(a.config), "--m", str(a.m),
                            "--reps", str(a.reps)], env=env, capture_output=True, text=True)
        line = [l for l in r.stdout.splitlines() if l.startswith("{")]
        print(json.dumps({"variant": var, **(json.loads(line[-1]) if line else {"error": r.stderr[-400:]})}), flush=True)


if __name__ == "__main__":
    main()
