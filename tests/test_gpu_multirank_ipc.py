"""The distributed path across PROCESSES on one GPU: 2 and 3
ranks as separate processes, each with its own CUDA context, talking through an NCCL-compatible
host-staged stand-in (tests/support/shm_nccl.cu, POSIX shared memory; NCCL refuses two ranks on
one device).  With TE_OPT_HALO = 1 every rank maps the other ranks' Krylov bases through CUDA IPC
(cudaIpcGetMemHandle / cudaIpcOpenMemHandle, the mapping NVLink peer access uses across GPUs) and
k_spmv_halo reads their V columns directly; with TE_OPT_HALO = 0 the halo goes through grouped
send/recv on the side stream.  Each rank's rows of the Krylov basis, a forced-schedule evolution
(<= 1e-10) and an adaptive one (<= tol) are compared with the oracle; a second evolution with a
larger basis reallocates V and must rebuild the peer mappings on every rank."""
import json
import os
import subprocess
import sys
import uuid

import numpy as np
import pytest

pytestmark = pytest.mark.gpu
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))

RANK_SCRIPT = r'''
import faulthandler, json, os, sys
faulthandler.dump_traceback_later(240, exit=True)
import numpy as np
sys.path.insert(0, sys.argv[1])
from paper_2205_15346_b200 import te
from oracle import krylov as K
from workloads import configs
ws, r, case, halo_mode, out = int(sys.argv[2]), int(sys.argv[3]), sys.argv[4], int(sys.argv[5]), sys.argv[6]
c = {"xxz": lambda: configs.build(5, L=11), "bh": lambda: configs.build(3, L=6, N=6),
     "random": lambda: configs.build(1, n=1500)}[case]()
n, t, tol = c["n"], 1.0, 1e-9
rp, col, val, v0 = c["rowptr"], c["col"], c["val"], c["v0"]
rs = [(q * n) // ws for q in range(ws + 1)]
rb, re_ = rs[r], rs[r + 1]
D = te.te_dist_init(ws, r, te.te_nccl_unique_id())
h = te.te_create_csr_dist(D, n, rb, re_, (rp[rb:re_ + 1] - rp[rb]).astype(np.int64),
                          col[rp[rb]:rp[re_]].astype(np.int64), val[rp[rb]:rp[re_]])
te.te_set_option(h, te.TE_OPT_HALO, halo_mode)
te.te_evolve(h, v0[rb:re_], 0.2, tol, 8)                 # V allocated for 8 columns ...
sched = json.loads(os.environ["TE_TEST_SCHED"])
g = te.te_krylov_basis(h, v0[rb:re_], 16, tol / t, want_V=True)   # ... then reallocated for 16
vf, _ = te.te_evolve_schedule(h, v0[rb:re_], sched, tol, 16)
va, st = te.te_evolve(h, v0[rb:re_], t, tol, 16)
np.savez(out, V=g["V"], alpha=g["alpha"], beta=g["beta"], m_eff=g["m_eff"], vf=vf, va=va,
         bound=st["err_bound"], norm1=te.te_one_norm(h))
h.close()
D.close()
print("RANK_OK", r)
'''


@pytest.fixture(scope="module")
def shm_nccl(tmp_path_factory):
    from paper_2205_15346_b200 import build as B
    lib = str(tmp_path_factory.mktemp("shmnccl") / "libshmnccl.so")
    src = os.path.join(ROOT, "tests", "support", "shm_nccl.cu")
    subprocess.run([B.nvcc(), "-O2", "-std=c++17", "-shared", "-Xcompiler", "-fPIC", "-gencode",
                    "arch=compute_100a,code=sm_100a", "-I", B.nccl_include(), "-o", lib, src, "-lrt"], check=True)
    return lib


@pytest.mark.parametrize("halo", [1, 0], ids=["ipc_peer_loads", "nccl_exchange"])
@pytest.mark.parametrize("ws", [2, 3])
@pytest.mark.parametrize("case", ["xxz", "bh", "random"])
def test_multiprocess_distributed_path(gpu_lib, shm_nccl, tmp_path, ws, case, halo):
    from oracle import krylov as K
    from workloads import configs
    c = {"xxz": lambda: configs.build(5, L=11), "bh": lambda: configs.build(3, L=6, N=6),
         "random": lambda: configs.build(1, n=1500)}[case]()
    n, t, tol, m = c["n"], 1.0, 1e-9, 16
    rp, col, val, v0 = c["rowptr"], c["col"], c["val"], c["v0"]
    ob = K.arnoldi(lambda x: K.spmv(rp, col, val, x), v0, m, tol / t)
    oe = K.evolve(rp, col, val, v0, t, tol, m)
    sched = [float(s[0]) for s in oe["schedule"]]
    env = dict(os.environ, TE_NCCL_LIB=shm_nccl, TE_SHM_NAME="/te_test_" + uuid.uuid4().hex[:12],
               TE_TEST_SCHED=json.dumps(sched))
    procs = [subprocess.Popen([sys.executable, "-c", RANK_SCRIPT, ROOT, str(ws), str(r), case, str(halo),
                               str(tmp_path / f"r{r}.npz")], env=env, stdout=subprocess.PIPE,
                              stderr=subprocess.PIPE, text=True) for r in range(ws)]
    outs = [p.communicate(timeout=300) for p in procs]
    for p, (so, se) in zip(procs, outs):
        assert p.returncode == 0 and "RANK_OK" in so, so[-2000:] + se[-4000:]
    parts = [np.load(tmp_path / f"r{r}.npz") for r in range(ws)]
    k = ob["m_eff"]
    scale = max(1.0, np.abs(ob["alpha"]).max(), np.abs(ob["beta"]).max())
    for p in parts:
        assert int(p["m_eff"]) == k
        assert np.abs(p["alpha"] - ob["alpha"]).max() <= 1e-12 * scale
        assert np.abs(p["beta"] - ob["beta"]).max() <= 1e-12 * scale
        assert abs(float(p["norm1"]) - K.one_norm(rp, col, val, n)) <= 1e-12 * float(p["norm1"])
    assert np.linalg.norm(np.concatenate([p["V"] for p in parts], axis=0) - ob["V"]) <= 1e-10
    assert np.linalg.norm(np.concatenate([p["vf"] for p in parts]) - oe["v"]) <= 1e-10
    assert np.linalg.norm(np.concatenate([p["va"] for p in parts]) - oe["v"]) <= tol + 1e-12
