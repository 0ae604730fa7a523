"""Multi-process CPU test (torch.distributed, gloo, world_size 2 and 3) of the row-sharded
protocol that te_create_csr_dist / the NCCL path implement:

  create:  row partition -> te_halo_plan (library, host-only) -> counts matrix (all_gather)
           -> need lists exchanged with grouped send/recv -> send index lists
  step j:  pack V_j[send_idx] -> send/recv into the halo -> local SpMV w' = H V_j (unscaled)
           CGS2: allreduce([||p''_{j-1}||^2, g1 = V^H w']) -> gate (s_j, breakdown)
                 -> p' = s_j (w' - V e1) -> allreduce(g2) -> p'' -> V_{j+1}
           f2:   allreduce([||p''_{j-1}||^2, g1, Gram dots of step j-1]) -> gate, Gram row j
                 -> p'' = s_j (w' - V (c1 + c2)), c2 = c1 - G c1 -> V_{j+1}, dots, ||p''||^2
           per restart: allreduce(||p''_{m-1}||^2)
  i.e. 2 allreduces per Krylov step for CGS2 and 1 for f2 (the library's defer mode).

Each rank runs one Arnoldi decomposition on its rows with numpy arithmetic (columns stored
unnormalised with scales s_k, as in the library); the gathered
result must equal the single-process oracle (alpha, beta to 1e-12 relative, V to 1e-10).  The
library's kernels are not involved (no GPU here); what is tested is the partition, the halo
plan and the communication pattern the CUDA path follows."""
import os
import socket

import numpy as np
import pytest
import torch.distributed as dist
import torch.multiprocessing as mp

from oracle import krylov as K
from paper_2205_15346_b200 import build as B
from paper_2205_15346_b200 import te
from workloads import configs


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _case(name):
    if name == "xxz":
        return configs.build(5, L=10)
    if name == "bh":
        return configs.build(3, L=6, N=6)
    return configs.build(1, n=700)


def _worker(rank, ws, port, name, m, out_dir, mode):
    import torch
    dist.init_process_group("gloo", rank=rank, world_size=ws, init_method=f"tcp://127.0.0.1:{port}")
    c = _case(name)
    n = c["n"]
    rp, col, val = c["rowptr"], c["col"], c["val"]
    row_starts = np.array([(q * n) // ws for q in range(ws + 1)], dtype=np.int64)
    rb, re_ = int(row_starts[rank]), int(row_starts[rank + 1])
    nloc = re_ - rb
    lrp = rp[rb: re_ + 1] - rp[rb]
    cols_g = col[rp[rb]: rp[re_]].astype(np.int64)
    lval = val[rp[rb]: rp[re_]]
    col_loc, recv_counts, halo = te.te_halo_plan(ws, rank, row_starts, cols_g)
    # counts matrix M[q][p] = entries rank q needs from rank p
    rc = torch.from_numpy(recv_counts.copy())
    allc = [torch.zeros_like(rc) for _ in range(ws)]
    dist.all_gather(allc, rc)
    send_counts = np.array([0 if q == rank else int(allc[q][rank]) for q in range(ws)])
    # need lists: send my need list segment to its owner, receive the peers' needs of my rows
    offs = np.concatenate([[0], np.cumsum(recv_counts)])
    reqs = []
    give = {}
    for q in range(ws):
        if q == rank:
            continue
        if recv_counts[q] > 0:
            reqs.append(dist.isend(torch.from_numpy(halo[offs[q]: offs[q + 1]].copy()), q))
        if send_counts[q] > 0:
            buf = torch.zeros(int(send_counts[q]), dtype=torch.int64)
            reqs.append(dist.irecv(buf, q))
            give[q] = buf
    for r in reqs:
        r.wait()
    send_idx = {q: (give[q].numpy() - rb).astype(np.int64) for q in give}
    assert all(((s >= 0) & (s < nloc)).all() for s in send_idx.values())
    # one Arnoldi decomposition, distributed (defer-mode protocol of the library)
    tol_rate = c["tol"] / c["t"]
    V = np.zeros((nloc, m), dtype=np.complex128)   # stored columns: V_0 = v0, V_{j+1} = p''_j
    V[:, 0] = c["v0"][rb:re_]
    s = np.zeros(m + 1)
    s[0] = 1.0
    alpha, beta = np.zeros(m), np.zeros(m)
    G = np.zeros((m, m), dtype=np.complex128)
    m_eff = m
    rows = np.repeat(np.arange(nloc), np.diff(lrp))
    calls = [0]

    def allreduce(a):
        calls[0] += 1
        t = torch.from_numpy(np.ascontiguousarray(a).view(np.float64).copy())
        dist.all_reduce(t)
        return t.numpy().view(a.dtype)

    nrm_prev = 0.0
    g2_prev = np.zeros(0, dtype=np.complex128)
    for j in range(m):
        x = V[:, j]
        hbuf = np.zeros(len(halo), dtype=np.complex128)
        reqs = []
        for q in range(ws):
            if q == rank:
                continue
            if send_counts[q] > 0:
                reqs.append(dist.isend(torch.from_numpy(x[send_idx[q]].view(np.float64).copy()), q))
            if recv_counts[q] > 0:
                buf = torch.zeros(2 * int(recv_counts[q]), dtype=torch.float64)
                reqs.append((dist.irecv(buf, q), q, buf))
        for r in reqs:
            if isinstance(r, tuple):
                r[0].wait()
                q, buf = r[1], r[2]
                hbuf[offs[q]: offs[q + 1]] = buf.numpy().view(np.complex128)
            else:
                r.wait()
        xe = np.concatenate([x, hbuf])
        w = np.zeros(nloc, dtype=np.complex128)
        np.add.at(w, rows, lval * xe[col_loc])        # H V_j, unscaled
        Vj = V[:, : j + 1]
        g1 = Vj.conj().T @ w
        if mode == "cgs2":
            red = allreduce(np.concatenate([[nrm_prev + 0j], g1]))
        else:
            red = allreduce(np.concatenate([[nrm_prev + 0j], g1, g2_prev]))
        nrm_g, g1 = red[0].real, red[1: j + 2]
        if j > 0:                                      # the deferred gate of step j
            b = float(np.sqrt(nrm_g))
            beta[j - 1] = b
            if b < tol_rate:
                m_eff = j
                break
            s[j] = 1.0 / b
        sj = s[j]
        sk = s[: j + 1]
        if mode == "cgs2":
            p = sj * (w - Vj @ (sk ** 2 * g1))
            g2 = allreduce(Vj.conj().T @ p)
            alpha[j] = sj * (sj * g1[j].real + g2[j].real)
            p = p - Vj @ (sk ** 2 * g2)
        else:
            if j > 0:
                gp = red[j + 2:]
                G[:j, j] = sk[:j] * sj * gp
                G[j, :j] = np.conj(G[:j, j])
            G[j, j] = 1.0
            c1 = sk * g1
            cc = c1 + (c1 - G[: j + 1, : j + 1] @ c1)
            alpha[j] = sj * cc[j].real
            p = sj * (w - Vj @ (sk * cc))
            g2_prev = Vj.conj().T @ p
        nrm_prev = float(np.vdot(p, p).real)
        if j < m - 1:
            V[:, j + 1] = p
    else:
        b = float(np.sqrt(allreduce(np.array([nrm_prev]))[0]))
        beta[m - 1] = b
        if b < tol_rate:
            m_eff = m
    n_steps = m_eff
    V = V[:, :m_eff] * s[:m_eff]
    assert calls[0] == (2 if mode == "cgs2" else 1) * n_steps + (1 if m_eff == m else 0)
    np.savez(os.path.join(out_dir, f"r{rank}.npz"), alpha=alpha[:m_eff], beta=beta[:m_eff], V=V[:, :m_eff],
             rb=rb, re=re_)
    dist.barrier()
    dist.destroy_process_group()


@pytest.mark.parametrize("mode", ["cgs2", "cgs2gram"])
@pytest.mark.parametrize("ws", [2, 3])
@pytest.mark.parametrize("name", ["xxz", "bh", "random"])
def test_row_sharded_arnoldi_matches_oracle(tmp_path, ws, name, mode):
    B.build()
    te.load()
    m = 12
    mp.start_processes(_worker, args=(ws, _free_port(), name, m, str(tmp_path), mode), nprocs=ws, join=True,
                       start_method="spawn")
    c = _case(name)
    o = K.arnoldi(lambda x: K.spmv(c["rowptr"], c["col"], c["val"], x), c["v0"], m, c["tol"] / c["t"], ortho=mode)
    parts = [np.load(tmp_path / f"r{r}.npz") for r in range(ws)]
    for p in parts:
        assert np.allclose(p["alpha"], o["alpha"], rtol=0, atol=1e-12 * max(1, np.abs(o["alpha"]).max()))
        assert np.allclose(p["beta"], o["beta"], rtol=0, atol=1e-12 * max(1, np.abs(o["beta"]).max()))
    Vg = np.concatenate([p["V"] for p in parts], axis=0)
    assert np.linalg.norm(Vg - o["V"]) <= 1e-10
