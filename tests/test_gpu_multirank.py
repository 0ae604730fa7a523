"""The multi-rank device path on ONE GPU: 2 and 3 ranks run as
threads of one process, each with its own handle and stream, through te_dist_init /
te_create_csr_dist / te_evolve, with an NCCL-compatible stand-in (tests/support/fake_nccl.cu,
loaded through TE_NCCL_LIB) doing the exchanges as stream-ordered device copies.  This runs the
library's real halo plan, need-list exchange, halo pack kernel, halo-aware SpMV instantiation and
allreduce placement; only the transport differs from NCCL over NVLink.  Checked against the oracle:
the Krylov basis (rows gathered over ranks), one evolution with the oracle's own step schedule
forced (<= 1e-10), and the adaptive evolution (<= tol + 1e-12)."""
import json
import os
import subprocess
import sys

import pytest

pytestmark = pytest.mark.gpu
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))

SCRIPT = r'''
import faulthandler, json, sys, threading
faulthandler.dump_traceback_later(int(__import__("os").environ.get("MR_DUMP_AFTER", "240")), exit=True)
import numpy as np
sys.path.insert(0, sys.argv[3])
from paper_2205_15346_b200 import te
from oracle import krylov as K
from workloads import configs
ws, case, halo_mode = int(sys.argv[1]), sys.argv[2], int(sys.argv[4])
def blockdiag():
    # two independent Hermitian blocks of 1000 rows: split at 1000 (2 ranks) there is no halo at all
    a, b = configs.build(1, n=1000), configs.build(1, n=1000)
    rp = np.concatenate([a["rowptr"], b["rowptr"][1:] + a["rowptr"][-1]])
    col = np.concatenate([a["col"], b["col"] + 1000]).astype(np.int32)
    v0 = np.concatenate([a["v0"], b["v0"]]) / np.sqrt(2.0)
    return dict(n=2000, rowptr=rp, col=col, val=np.concatenate([a["val"], b["val"]]), v0=v0)
c = {"xxz": lambda: configs.build(5, L=12), "bh": lambda: configs.build(3, L=7, N=7),
     "random": lambda: configs.build(1, n=3001), "blockdiag": blockdiag}[case]()
n, m, t, tol = c["n"], 16, 1.0, 1e-9
rp, col, val, v0 = c["rowptr"], c["col"], c["val"], c["v0"]
tol_rate = tol / t
ob = K.arnoldi(lambda x: K.spmv(rp, col, val, x), v0, m, tol_rate)
oe = K.evolve(rp, col, val, v0, t, tol, m)
sched = [float(s[0]) if isinstance(s, (tuple, list)) else float(s) for s in oe["schedule"]]
rs = [(q * n) // ws for q in range(ws + 1)]
uid = te.te_nccl_unique_id()
res, errs = [None] * ws, []

def worker(r):
    try:
        D = te.te_dist_init(ws, r, uid)
        rb, re_ = rs[r], rs[r + 1]
        h = te.te_create_csr_dist(D, n, rb, re_, (rp[rb:re_ + 1] - rp[rb]).astype(np.int64),
                                  col[rp[rb]:rp[re_]].astype(np.int64), val[rp[rb]:rp[re_]])
        te.te_set_option(h, te.TE_OPT_HALO, halo_mode)
        # a first evolution with a smaller basis: the m = 16 calls below reallocate V, and every
        # rank must rebuild its peer table (halo mode 1) even if cudaMalloc returns the same address
        te.te_evolve(h, v0[rb:re_], 0.2, tol, 8)
        g = te.te_krylov_basis(h, v0[rb:re_], m, tol_rate, want_V=True)
        vf = None
        if sched is not None:
            vf, _ = te.te_evolve_schedule(h, v0[rb:re_], sched, tol, m)
        va, st = te.te_evolve(h, v0[rb:re_], t, tol, m)
        res[r] = dict(V=g["V"], alpha=g["alpha"], beta=g["beta"], m_eff=g["m_eff"], vf=vf, va=va, st=st,
                      norm1=te.te_one_norm(h))
        h.close()
        D.close()
    except Exception as e:
        errs.append(f"rank {r}: {e!r}")
        print(f"rank {r} failed: {e!r}", file=sys.stderr, flush=True)

th = [threading.Thread(target=worker, args=(r,)) for r in range(ws)]
for x in th: x.start()
for x in th: x.join(timeout=600)
out = {"errors": errs}
if not errs:
    k = ob["m_eff"]
    V = np.concatenate([res[r]["V"] for r in range(ws)], axis=0)
    scale = max(1.0, np.abs(ob["alpha"]).max(), np.abs(ob["beta"]).max())
    out["m_eff_ok"] = all(res[r]["m_eff"] == k for r in range(ws))
    out["alpha_err"] = max(float(np.abs(res[r]["alpha"] - ob["alpha"]).max()) for r in range(ws)) / scale
    out["beta_err"] = max(float(np.abs(res[r]["beta"] - ob["beta"]).max()) for r in range(ws)) / scale
    out["V_err"] = float(np.linalg.norm(V - ob["V"]))
    if sched is not None:
        out["forced_err"] = float(np.linalg.norm(np.concatenate([res[r]["vf"] for r in range(ws)]) - oe["v"]))
    va = np.concatenate([res[r]["va"] for r in range(ws)])
    out["adaptive_err"] = float(np.linalg.norm(va - oe["v"]))
    out["bound"] = float(res[0]["st"]["err_bound"])
    out["norm1"] = [float(res[r]["norm1"]) for r in range(ws)]
    out["norm1_oracle"] = float(K.one_norm(rp, col, val, n))
import ctypes, os
out["fake_calls"] = int(ctypes.CDLL(os.environ["TE_NCCL_LIB"]).fake_nccl_calls())
print("RESULT " + json.dumps(out))
'''


@pytest.fixture(scope="module")
def fake_nccl(tmp_path_factory):
    from paper_2205_15346_b200 import build as B
    lib = str(tmp_path_factory.mktemp("fakenccl") / "libfakenccl.so")
    src = os.path.join(ROOT, "tests", "support", "fake_nccl.cu")
    subprocess.run([B.nvcc(), "-O2", "-std=c++17", "-shared", "-Xcompiler", "-fPIC", "-gencode",
                    "arch=compute_100a,code=sm_100a", "-I", B.nccl_include(), "-o", lib, src], check=True)
    return lib


FORMATS = {"auto": {}, "slotwindow": {"TE_SPMV_SW_FORCE": "1"},
           "colblk": {"TE_SPMV_DEFAULT": "10", "TE_SPMV_COLBLK_MB": "0.002"}}


@pytest.mark.parametrize("fmt", list(FORMATS))
@pytest.mark.parametrize("halo", [0, 1], ids=["nccl_exchange", "peer_loads"])
@pytest.mark.parametrize("ws", [2, 3])
@pytest.mark.parametrize("case", ["xxz", "bh", "random", "blockdiag"])
def test_multirank_device_path_on_one_gpu(gpu_lib, fake_nccl, ws, case, halo, fmt):
    """halo 0: staged NCCL send/recv exchange before each SpMV; halo 1 (TE_OPT_HALO): the
    SpMV reads halo columns directly from the owning rank's V column (same address space here).
    fmt: each rank's local SpMV format as chosen at create ("auto"), the slot-window SELL-32 forced
    on every rank whose local values fit the dictionary, or the column-blocked ring (128-column
    blocks) — the halo entries are added by k_spmv_halo after the local format's passes."""
    env = dict(os.environ, TE_NCCL_LIB=fake_nccl, **FORMATS[fmt])
    p = subprocess.run([sys.executable, "-c", SCRIPT, str(ws), case, ROOT, str(halo)], env=env, capture_output=True,
                       text=True, timeout=300)
    line = [l for l in p.stdout.splitlines() if l.startswith("RESULT ")]
    assert p.returncode == 0 and line, p.stdout[-2000:] + p.stderr[-4000:]
    r = json.loads(line[0][7:])
    assert not r["errors"], r["errors"]
    assert r["fake_calls"] > 0                       # the exchanges went through the stand-in
    assert r["m_eff_ok"]
    assert r["alpha_err"] <= 1e-12 and r["beta_err"] <= 1e-12
    assert r["V_err"] <= 1e-10
    if "forced_err" in r:
        assert r["forced_err"] <= 1e-10
    assert r["adaptive_err"] <= 1e-9 + 1e-12
    assert all(abs(x - r["norm1_oracle"]) <= 1e-12 * r["norm1_oracle"] for x in r["norm1"])
