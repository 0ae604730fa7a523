"""Rebuild profiles/<round>_summary.md from the committed bench lines profiles/<round>_bench_*.json.
Usage: python tools/make_summary.py [round]   (default r02)"""
import glob
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
RND = sys.argv[1] if len(sys.argv) > 1 else "r02"
LABEL = {1: "1 random n=4096", 2: "2 XXZ L=20", 3: "3 Bose-Hubbard 12/12", 4: "4 random banded n=2^24",
         5: "5 XXZ+NNN L=26", 6: "6 paper §5 model d=1,565,904 (P:527)"}


def main():
    rows, ref = [], None
    for f in sorted(glob.glob(os.path.join(ROOT, "profiles", f"{RND}_bench_*.json"))):
        d = json.load(open(f))
        if d.get("impl") == "reference":
            ref = d
            continue
        cfg = int(os.path.basename(f).split("config")[1].split("_")[0].split(".")[0])
        rows.append((cfg, d))
    rows.sort(key=lambda x: (x[0], x[1]["config"].get("ortho", "")))
    out = [f"# Bench summary ({RND}, one B200, bench.py lines in profiles/{RND}_bench_*.json)", "",
           "value = Krylov steps / device time (CUDA events, inputs resident, restart graphs); e2e = the same "
           "through te_evolve with host buffers; roofline = the kernel class with the largest device time "
           "(algorithmic bytes of §6 / its event time, peak = measured 6536 GB/s copy); traffic = its DRAM "
           "bytes per call from ncu over one restart (profiles/ncu_traffic.json).", "",
           "| config | ortho | SpMV | Krylov steps/s | e2e | roofline kernel | frac | traffic / alg | SpMV / dots / update / norm GB/s | SM MHz (reasons) | oracle steps/s |",
           "|---|---|---|---|---|---|---|---|---|---|---|"]
    for cfg, d in rows:
        r, k = d["roofline"], d["kernels"]
        tr = f"{r['traffic'] / r['alg_bytes_per_launch']:.2f}" if r.get("traffic") else "—"
        g = lambda name: f"{k[name]['gbs']:.0f}" if name in k else "—"  # noqa: E731
        cl = d.get("clocks") or {}
        cpu = d.get("cpu_baseline", {}).get("value")
        out.append(f"| {LABEL[cfg]} | {d['config'].get('ortho')} | {d['config'].get('spmv_ran', '?')} | {d['value']:.1f} | "
                   f"{d['e2e']['value']:.1f} | {r['kernel']} | {r['frac']:.3f} | {tr} | "
                   f"{g('spmv')} / {g('proj_dots')} / {g('update_proj')} / {g('update_norm')} | "
                   f"{cl.get('sm_mhz')} ({', '.join(cl.get('reasons', [])) or '-'}) | "
                   f"{'%.3g' % cpu if cpu else '—'} |")
    if ref:
        out += ["", f"Reference arm (`bench.py --impl reference`, the oracle as it stands, 1 thread): "
                    f"{ref['value']:.4g} {ref['unit']} on {ref['config']['workload']}; sample: {ref['cpu_baseline']['sample']}."]
    path = os.path.join(ROOT, "profiles", f"{RND}_summary.md")
    open(path, "w").write("\n".join(out) + "\n")
    print("\n".join(out))


if __name__ == "__main__":
    main()
