#!/usr/bin/env python
"""bench.py — Krylov steps/s and achieved HBM GB/s (fraction of roofline) of the restarted
Krylov exp(-iHt) v engine on 1..8 B200 (BASELINE.json metric).

A bench "step" is one full te_evolve of the workload (all hot-path rows: SpMV+projection,
CGS2 sweeps, norm, host eigensolve + error integral + step search, V.omega) from v0 to t.
value = Krylov steps (Arnoldi iterations of the global problem) / device time, max over
ranks, inputs resident in HBM (te_evolve_dev).  e2e = the same through te_evolve with host
buffers (pinned), H2D of v0 and D2H of v(t) inside the timed region.

  python bench.py [--gpus N] [--steps K] [--warmup W] [--config 5] [--impl ours|reference]
  N > 1: python -m torch.distributed.run --nproc-per-node N ... bench.py --gpus N
         (run without WORLD_SIZE in the environment, bench.py re-launches itself that way)

Default workload: BASELINE configs[4] (XXZ+NNN, L = 26, n = 2^26, 1.8e9 nnz), the largest
configuration that fits one B200 and the one the north star's targets are stated on; configs[0]
is the oracle-size case and the other configs are parity-test / --config cases.
"""
from __future__ import annotations

import argparse
import json
import math
import os
import statistics
import subprocess
import sys
import threading
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

import numpy as np  # noqa: E402

WORKLOAD_DEFAULT = 5  # BASELINE.json configs[4] (XXZ+NNN L=26, n=2^26): largest single-GPU config


def parse():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=5)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--config", type=int, default=WORKLOAD_DEFAULT,
                    help="workload: 1-5 BASELINE.json configs (default 5, XXZ+NNN L=26), 6 the paper's P:527 benchmark")
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--cpu-sample-steps", type=int, default=None,
                    help="oracle Krylov steps timed for cpu_baseline (default: 1 for n >= 2^24, else 8)")
    ap.add_argument("--prof-steps", type=int, default=3, help="evolutions in the per-kernel (roofline) pass")
    ap.add_argument("--e2e-steps", type=int, default=5, help="evolutions in the e2e (host buffers) pass")
    ap.add_argument("--kernels", type=int, default=2, help="projection kernels: 2 hybrid (register accumulators up to 8 columns, TMA ring above; default), 3 TMA only, 5 register accumulators only")
    ap.add_argument("--prefetch", type=int, default=None, help="L2 bulk-prefetch distance (library default if unset)")
    ap.add_argument("--spmv", type=int, default=None, help="SpMV kernel (library default if unset): 10 column-blocked ring, 9 slot-window SELL-32, 8 staged-x ring, 7 warp-specialised ring, 6 SELL-32-sigma")
    ap.add_argument("--force-dist", action="store_true",
                    help="single rank through the distributed API (te_dist_init/te_create_csr_dist), for testing")
    ap.add_argument("--halo", type=int, default=0, help="N>1: 0 NCCL halo exchange (default), 1 SpMV reads peer memory (f4)")
    ap.add_argument("--ortho", type=int, default=0, help="0 CGS2 (north star), 1 paper-literal Lanczos (f1), 2 CGS2 with Gram second sweep (f2)")
    return ap.parse_args()


def load_peaks():
    p = os.path.join(ROOT, "MEASURED_PEAKS.json")
    if os.path.exists(p):
        d = json.load(open(p))
        return float(d["hbm_gbs"]), "measured (MEASURED_PEAKS.json hbm_gbs, copy)"
    return 6650.0, "fallback (B200_PROFILING.md 6.65 TB/s)"


def load_traffic(cfg_name):
    """Per-launch DRAM bytes of each kernel from the committed ncu --set full capture."""
    p = os.path.join(ROOT, "profiles", "ncu_traffic.json")
    if not os.path.exists(p):
        return None
    d = json.load(open(p))
    return d.get(cfg_name)


class ClockSampler:
    """nvidia-smi clocks/throttle reasons sampled every 100 ms during the timed region."""
    FIELDS = ["clocks.sm", "clocks.max.sm", "clocks_event_reasons.sw_power_cap",
              "clocks_event_reasons.hw_slowdown", "clocks_event_reasons.hw_thermal_slowdown",
              "clocks_event_reasons.sw_thermal_slowdown"]

    def __init__(self, index):
        self.index = index
        self.rows = []
        self.proc = None

    def start(self):
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", "-i", str(self.index), "--query-gpu=" + ",".join(self.FIELDS),
                 "--format=csv,noheader,nounits", "-lms", "100"],
                stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self.t = threading.Thread(target=self._read, daemon=True)
            self.t.start()
        except Exception:
            self.proc = None

    def _read(self):
        for line in self.proc.stdout:
            parts = [x.strip() for x in line.split(",")]
            if len(parts) == len(self.FIELDS):
                self.rows.append(parts)

    def stop(self):
        if self.proc is None:
            return None
        self.proc.terminate()
        try:
            self.proc.wait(timeout=5)
        except Exception:
            self.proc.kill()
        self.t.join(timeout=2)
        if not self.rows:
            return None
        sm = [float(r[0]) for r in self.rows if r[0].replace(".", "").isdigit()]
        mx = [float(r[1]) for r in self.rows if r[1].replace(".", "").isdigit()]
        names = ["sw_power_cap", "hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown"]
        reasons = sorted({names[i] for r in self.rows for i in range(4) if r[2 + i].lower().startswith("active")})
        return {"sm_mhz": statistics.median(sm) if sm else None, "sm_max_mhz": max(mx) if mx else None,
                "reasons": reasons, "samples": len(self.rows)}


def dist_env():
    ws = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    return ws, rank, local


def build_workload(cfg, ws, rank):
    from workloads import configs, fast
    if ws > 1 and cfg in (2, 5):  # XXZ configs: each rank builds only its own rows (C builder)
        c = configs.build(cfg, with_matrix=False)
        p = c["params"]
        n = c["n"]
        rb, re_ = (rank * n) // ws, ((rank + 1) * n) // ws
        J1 = p.get("J", p.get("J1"))
        rp, col, val = fast.xxz_csr_fast(p["L"], J1, p["delta"], c["fields"], J2=p.get("J2", 0.0), r0=rb, r1=re_)
        c["rowptr_local"], c["col_local_global"], c["val_local"] = rp, col.astype(np.int64), val
        c["nnz_global"] = None
        return c, rb, re_
    c = configs.build(cfg)
    n = c["n"]
    if ws == 1:
        return c, 0, n
    rb, re_ = (rank * n) // ws, ((rank + 1) * n) // ws
    rp = c["rowptr"]
    c["rowptr_local"] = (rp[rb: re_ + 1] - rp[rb]).astype(np.int64)
    c["col_local_global"] = c["col"][rp[rb]: rp[re_]].astype(np.int64)
    c["val_local"] = c["val"][rp[rb]: rp[re_]]
    return c, rb, re_


# ------------------------------------------------------------------------------------------
# CPU baseline: the oracle as it stands, single thread, bounded sample
# ------------------------------------------------------------------------------------------
def step_bytes(n, nnz, val_bytes, j):
    """SURVEY.md §8(d) analytic bytes of one Krylov step at basis size j: B_H + n (96 + 48 j)."""
    return nnz * (val_bytes + 4) + 8 * (n + 1) + n * (96 + 48 * j)


BIG = 1 << 24  # n at and above which the oracle's basis is a stand-in (configs 4, 5)


def oracle_sample(c, steps, warmup=0, standin=None):
    """The oracle as it stands (oracle.krylov.arnoldi_step, CGS2, 1 thread) timed for `steps` Krylov
    steps at the mean basis size j = m/2 of the workload (the step cost is linear in j).  Setup is
    untimed: for n < 2^24 the first j columns come from the oracle's own arnoldi; for the 2^24 and
    2^26 configs the basis is a stand-in (every column = v0; the timing does not depend on the
    values) because building it with the oracle would take j times the timed step.
    Returns (steps/s, seconds per step, sample description, per-step times)."""
    from oracle import krylov as K
    m = c["m"]
    j = m // 2
    n = c["n"]
    tol_rate = c["tol"] / c["t"]

    def mv(x):
        return K.spmv(c["rowptr"], c["col"], c["val"], x)

    if standin is None:
        standin = n >= BIG
    if standin:
        V = np.empty((n, j + 1), dtype=np.complex128)
        for k in range(j + 1):
            V[:, k] = c["v0"]
        beta = np.ones(j + 1)
        basis = "stand-in basis (every column = v0)"
    else:
        kr = K.arnoldi(mv, c["v0"], j + 1, tol_rate)
        V = np.zeros((n, j + 1), dtype=np.complex128)
        V[:, : kr["V"].shape[1]] = kr["V"]
        beta = kr["beta"]
        basis = "basis from the oracle's arnoldi"
    times = []
    for it in range(warmup + steps):
        t0 = time.perf_counter()
        K.arnoldi_step(mv, V, beta, j)
        dt = time.perf_counter() - t0
        if it >= warmup:
            times.append(dt)
    del V
    per = sum(times) / len(times)
    sample = (f"{len(times)} oracle Arnoldi/CGS2 step(s) (oracle.krylov.arnoldi_step) at j={j} (mean basis size "
              f"of an m={m} restart) on the {c['name']} model at n={n}, nnz={int(c['rowptr'][-1])}, {basis}, 1 thread")
    return 1.0 / per, per, sample, times


def oracle_ram_ok(c):
    """The oracle's step at j = m/2 holds V (n (j+1) complex), its conjugate copy and the SpMV's
    temporaries (rows int64, x[col] and the products, complex: 40 B per entry).  Returns
    (fits, bytes needed, bytes available)."""
    j = c["m"] // 2
    need = 2 * 16 * c["n"] * (j + 1) + 40 * int(c["rowptr"][-1]) + 64 * c["n"]
    try:
        import psutil
        avail = psutil.virtual_memory().available
    except Exception:
        avail = 0
    return avail > 1.15 * need, need, avail


def reduced_for_reference(cfg):
    """The --impl reference arm times K oracle steps; at 2^24 / 2^26 rows one oracle step takes
    minutes, so each step runs on the same model at 1/16 of the rows (config 4: n = 2^20; config 5:
    L = 22) and the rate is scaled to the full workload by the §8(d) analytic bytes per step."""
    from workloads import configs
    if cfg == 5:
        return configs.build(5, L=22)
    if cfg == 4:
        return configs.build(4, n=1 << 20)
    return None


def set_single_thread():
    for k in ("OMP_NUM_THREADS", "OPENBLAS_NUM_THREADS", "MKL_NUM_THREADS"):
        os.environ[k] = "1"
    try:
        from threadpoolctl import threadpool_limits
        threadpool_limits(1)
    except Exception:
        pass


def config_dict(c, args, ws, nloc):
    """The workload description shared by both arms (the driver compares them)."""
    from workloads import configs
    return {"workload": f"{c['name']} ({configs.LABELS[args.config]})", "n": c["n"],
            "nnz": int(c["nnz"]), "m": c["m"], "t": c["t"], "tol": c["tol"],
            "l2": "inputs larger than L2 (V = %.0f MB > 126 MB)" % (16 * nloc * c["m"] / 1e6),
            "parallelism": f"rows{ws}", "kernels": {2: "hybrid", 3: "tma", 5: "regacc"}[args.kernels],
            "spmv": {None: "library default", 6: "sell", 7: "ring", 8: "staged-x ring", 9: "slot-window sell",
                     10: "column-blocked ring"}[args.spmv],
            "ortho": ["cgs2", "lanczos3", "cgs2gram"][args.ortho],
            "halo": (["nccl_exchange", "peer_loads"][args.halo] if ws > 1 else None)}


def run_reference(args):
    ws, rank, _ = dist_env()
    if ws > 1 and rank != 0:
        return 0
    set_single_thread()
    from workloads import configs
    c = configs.build(args.config, with_matrix=False)
    c["nnz"] = full_nnz(args.config, c)
    small = reduced_for_reference(args.config)
    if small is None:
        src = configs.build(args.config)
        rate, per, sample, times = oracle_sample(src, args.steps, args.warmup)
    else:
        r_small, per_small, sample, times = oracle_sample(small, args.steps, args.warmup, standin=True)
        j = c["m"] // 2
        vb = 16 if np.iscomplexobj(small["val"]) else 8
        ratio = step_bytes(small["n"], int(small["rowptr"][-1]), vb, j) / step_bytes(c["n"], c["nnz"], vb, j)
        rate = r_small * ratio
        per = 1.0 / rate
        sample += (f"; scaled to the full workload (n={c['n']}) by the SURVEY §8(d) analytic bytes per step "
                   f"(x{ratio:.4f}); extrapolated, the oracle at the full size needs minutes per step")
    line = {
        "impl": "reference", "metric": "Krylov steps/s", "value": rate, "unit": "krylov_steps/s",
        "n_gpus": args.gpus, "steps": args.steps, "warmup": args.warmup, "ms_per_step": per * 1e3,
        "higher_is_better": True, "scaling": "strong", "vs_baseline": None, "dtype": "c128",
        "data": "synthetic", "config": config_dict(c, args, args.gpus, c["n"] // max(1, args.gpus)),
        "cpu_baseline": {"value": rate, "unit": "krylov_steps/s", "cores": 1, "kind": "oracle", "sample": sample},
        "e2e": {"value": rate, "unit": "krylov_steps/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line))
    return 0


def full_nnz(cfg, c):
    """nnz of the full workload without building it where a closed form exists."""
    if "rowptr" in c:
        return int(c["rowptr"][-1])
    p = c["params"]
    if cfg == 5:
        return (1 << p["L"]) * (1 + p["L"])
    if cfg == 2:
        return (1 << p["L"]) * (1 + p["L"] // 2)
    from workloads import configs
    return int(configs.build(cfg)["rowptr"][-1])


# ------------------------------------------------------------------------------------------
# our arm
# ------------------------------------------------------------------------------------------
def run_ours(args):
    import torch
    from paper_2205_15346_b200 import build as B
    from paper_2205_15346_b200 import te
    from workloads import configs

    ws, rank, local = dist_env()
    if ws > 1:
        import torch.distributed as dist
        torch.cuda.set_device(local)
        dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    else:
        torch.cuda.set_device(0)
    if rank == 0:
        B.build()
    if ws > 1:
        torch.distributed.barrier()
    te.load()
    dev = torch.device("cuda", local if ws > 1 else 0)

    c, rb, re_ = build_workload(args.config, ws, rank)
    c["nnz"] = full_nnz(args.config, c)
    n_glob, nloc = c["n"], re_ - rb
    t, tol, m = c["t"], c["tol"], c["m"]
    D = None
    if ws == 1 and args.force_dist:
        D = te.te_dist_init(1, 0, b"\0" * 128)
        h = te.te_create_csr_dist(D, n_glob, 0, n_glob, c["rowptr"], c["col"].astype(np.int64), c["val"])
        v0_loc = c["v0"]
    elif ws == 1:
        h = te.te_create_csr(n_glob, c["rowptr"], c["col"], c["val"])
        v0_loc = c["v0"]
    else:
        import torch.distributed as dist
        uid = [te.te_nccl_unique_id() if rank == 0 else None]
        dist.broadcast_object_list(uid, src=0)
        D = te.te_dist_init(ws, rank, uid[0])
        h = te.te_create_csr_dist(D, n_glob, rb, re_, c["rowptr_local"], c["col_local_global"], c["val_local"])
        v0_loc = c["v0"][rb:re_]
    te.te_set_option(h, te.TE_OPT_KERNELS, args.kernels)
    if args.prefetch is not None:
        te.te_set_option(h, te.TE_OPT_PREFETCH, args.prefetch)
    if args.spmv is not None:
        te.te_set_option(h, te.TE_OPT_SPMV, args.spmv)
    te.te_set_option(h, te.TE_OPT_ORTHO, args.ortho)
    te.te_set_option(h, te.TE_OPT_HALO, args.halo)
    stream = torch.cuda.current_stream(dev)
    d_v0 = torch.from_numpy(np.ascontiguousarray(v0_loc)).to(dev)
    d_out = torch.empty_like(d_v0)

    def barrier():
        if ws > 1:
            torch.distributed.barrier()

    def one_step():
        return te.te_evolve_dev(h, d_v0, t, tol, m, d_out, stream=stream)

    for _ in range(args.warmup):
        st = one_step()
    torch.cuda.synchronize()
    # ---- timed region (device-resident inputs), CUDA events on the launching stream.
    # The library replays each restart as a CUDA graph here (no per-kernel events).
    l0 = te.te_launch_count(h)
    clk = ClockSampler(local if ws > 1 else 0) if rank == 0 else None
    if clk:
        clk.start()
    barrier()
    torch.cuda.synchronize()
    e0 = torch.cuda.Event(enable_timing=True)
    e1 = torch.cuda.Event(enable_timing=True)
    e0.record(stream)
    ksteps = 0
    stats = []
    for _ in range(args.steps):
        st = one_step()
        stats.append(st)
        ksteps += st["n_krylov_steps"]
    e1.record(stream)
    torch.cuda.synchronize()
    barrier()
    ms = e0.elapsed_time(e1)
    clocks = clk.stop() if clk else None
    launches = te.te_launch_count(h) - l0
    if ws > 1:
        tt = torch.tensor([ms], device=dev, dtype=torch.float64)
        torch.distributed.all_reduce(tt, op=torch.distributed.ReduceOp.MAX)
        ms = float(tt.item())
    # ---- per-kernel timed region: the same K steps with a CUDA event pair around every launch
    # (direct launches), for the roofline of the dominant kernel
    te.te_set_option(h, te.TE_OPT_PROFILE, 1)
    torch.cuda.synchronize()
    p0 = torch.cuda.Event(enable_timing=True)
    p1 = torch.cuda.Event(enable_timing=True)
    prof_steps = max(1, min(args.steps, args.prof_steps))
    p0.record(stream)
    for _ in range(prof_steps):
        one_step()
    p1.record(stream)
    torch.cuda.synchronize()
    ms_prof = p0.elapsed_time(p1)
    prof = te.te_get_profile(h)
    te.te_set_option(h, te.TE_OPT_PROFILE, 0)

    # ---- e2e through the public host-buffer API (pinned host memory), wall clock
    hv0 = torch.from_numpy(np.ascontiguousarray(v0_loc)).pin_memory()
    hout = torch.empty_like(hv0).pin_memory()
    v0n, outn = hv0.numpy(), hout.numpy()
    te.te_evolve(h, v0n, t, tol, m, out=outn)
    barrier()
    e2e_n = max(1, min(args.steps, args.e2e_steps))
    w0 = time.perf_counter()
    e2e_steps = 0
    for _ in range(e2e_n):
        _, st2 = te.te_evolve(h, v0n, t, tol, m, out=outn)
        e2e_steps += st2["n_krylov_steps"]
    w1 = time.perf_counter()
    e2e_s = w1 - w0
    if ws > 1:
        tt = torch.tensor([e2e_s], device=dev, dtype=torch.float64)
        torch.distributed.all_reduce(tt, op=torch.distributed.ReduceOp.MAX)
        e2e_s = float(tt.item())

    if rank != 0:
        h.close()
        if D is not None:
            D.close()
        if ws > 1:
            torch.distributed.destroy_process_group()
        return 0

    peak, peak_src = load_peaks()
    # dominant kernel = largest share of device time in the timed region
    dom = max((k for k in prof if prof[k]["launches"] > 0), key=lambda k: prof[k]["total_ms"])
    p = prof[dom]
    achieved = p["alg_bytes"] / (p["total_ms"] * 1e-3) / 1e9
    traffic_tab = load_traffic(c["name"])
    traffic = None
    if traffic_tab and dom in traffic_tab:
        traffic = traffic_tab[dom].get("dram_bytes_per_launch")
    all_ms = sum(prof[k]["total_ms"] for k in prof)
    all_bytes = sum(prof[k]["alg_bytes"] for k in prof)
    value = ksteps / (ms * 1e-3)
    line = {
        "metric": "Krylov steps/s", "value": value, "unit": "krylov_steps/s", "n_gpus": ws,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": ms / args.steps,
        "higher_is_better": True, "scaling": "strong", "vs_baseline": None, "dtype": "c128",
        "data": "synthetic",
        "config": {**config_dict(c, args, ws, nloc),
                   "spmv_ran": {6: "sell", 7: "ring", 8: "staged-x ring", 9: "slot-window sell", 10: "column-blocked ring"}
                   .get(int(te.te_get_option(h, te.TE_OPT_SPMV)), "?")},
        "krylov_steps_per_step": ksteps / args.steps,
        "restarts_per_step": stats[-1]["n_restarts"],
        "achieved_hbm_gbs": all_bytes / (all_ms * 1e-3) / 1e9 if all_ms > 0 else None,
        "step_hbm_gbs": (all_bytes / prof_steps) / (ms / args.steps * 1e-3) / 1e9,
        "profiled_region_ms_per_step": ms_prof / prof_steps,
        "evolved_time_per_s": t * args.steps / (ms * 1e-3),
        **({"paper_context": {"paper_wall_s": 353.0, "paper_hw": "i9-9900K, 1 thread (P:527-529)",
                              "ours_wall_s": ms / args.steps * 1e-3,
                              "err_bound": stats[-1]["err_bound"], "roundoff_total": stats[-1]["roundoff_total"]}}
           if args.config == 6 else {}),
        "roofline": {"bound": "hbm", "kernel": dom, "achieved": achieved, "peak": peak, "unit": "GB/s",
                     "frac": achieved / peak, "traffic": traffic, "peak_source": peak_src,
                     "alg_bytes_per_launch": p["alg_bytes"] / p["launches"],
                     "avg_launch_ms": p["total_ms"] / p["launches"],
                     "share_of_kernel_time": p["total_ms"] / all_ms if all_ms else None,
                     "timing": f"CUDA events on the launching stream around every launch of a second timed pass "
                               f"of {prof_steps} of the same steps (direct launches; the headline pass replays CUDA "
                               f"graphs)"},
        "kernels": {k: {"launches": prof[k]["launches"], "ms": prof[k]["total_ms"],
                        "gbs": (prof[k]["alg_bytes"] / (prof[k]["total_ms"] * 1e-3) / 1e9) if prof[k]["total_ms"] else None}
                    for k in prof if prof[k]["launches"]},
        "e2e": {"value": e2e_steps / e2e_s, "unit": "krylov_steps/s", "h2d_bytes_per_step": 16 * nloc,
                "d2h_bytes_per_step": 16 * nloc, "steps": e2e_n,
                "timing": "wall clock around te_evolve (host buffers, pinned), max over ranks"},
        "gpu_launches": launches,
        "clocks": clocks,
        "err_bound": stats[-1]["err_bound"],
    }
    if not args.no_cpu_baseline and ws == 1:
        set_single_thread()
        h.close()
        torch.cuda.empty_cache()
        steps = args.cpu_sample_steps or (1 if c["n"] >= BIG else 8)
        fits, need, avail = oracle_ram_ok(c)
        if fits:
            rate, per, sample, _ = oracle_sample(c, steps)
        else:  # not enough host RAM for the oracle's temporaries at this size: same model, 1/16 rows
            small = reduced_for_reference(args.config)
            r_small, _, sample, _ = oracle_sample(small, steps, standin=True)
            j = c["m"] // 2
            vb = 16 if np.iscomplexobj(small["val"]) else 8
            ratio = step_bytes(small["n"], int(small["rowptr"][-1]), vb, j) / step_bytes(c["n"], c["nnz"], vb, j)
            rate = r_small * ratio
            sample += (f"; scaled to n={c['n']} by the §8(d) bytes per step (x{ratio:.4f}): host RAM "
                       f"{avail / 1e9:.0f} GB < {need / 1e9:.0f} GB the full-size oracle step needs")
        line["cpu_baseline"] = {"value": rate, "unit": "krylov_steps/s", "cores": 1, "kind": "oracle",
                                "sample": sample}
    print(json.dumps(line))
    h.close()
    if D is not None:
        D.close()
    if ws > 1:
        torch.distributed.destroy_process_group()
    return 0


def free_port():
    import socket
    with socket.socket() as so:
        so.bind(("127.0.0.1", 0))
        return so.getsockname()[1]


def self_launch(args):
    """--gpus N > 1 without a torch.distributed environment: re-run this command as N ranks (one
    process per GPU) under torch.distributed.run on this node; rank 0 prints the JSON line.  Fails
    loudly when fewer than N GPUs are visible (a 1-GPU timing must never pass as N GPUs)."""
    import torch
    have = torch.cuda.device_count() if args.impl == "ours" else args.gpus
    if have < args.gpus:
        sys.stderr.write(f"bench.py: --gpus {args.gpus} requested but only {have} CUDA device(s) visible\n")
        return 2
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={args.gpus}",
           "--master-addr=127.0.0.1", f"--master-port={free_port()}", os.path.abspath(__file__)] + sys.argv[1:]
    return subprocess.call(cmd)


def main():
    args = parse()
    if args.gpus > 1 and "WORLD_SIZE" not in os.environ:
        return self_launch(args)
    if args.impl == "reference":
        return run_reference(args)
    ws = dist_env()[0]
    if ws != args.gpus:
        sys.stderr.write(f"bench.py: --gpus {args.gpus} but WORLD_SIZE={ws}\n")
        return 2
    return run_ours(args)


if __name__ == "__main__":
    sys.exit(main())
