"""Summarise ncu CSV captures into profiles/: per-kernel-class DRAM traffic per launch (for
bench.py's roofline.traffic) and launch-list shares.  Usage:
  python tools/ncu_summarize.py <restart_metrics.csv> <launches.csv> <workload-name> <out-prefix>"""
import collections
import csv
import json
import os
import re
import sys

CLASS = [(r"k_spmv", "spmv"), (r"k_proj_tma<0[,>]|k_proj_r<0", "proj_dots"), (r"k_proj_tma<[13][,>]|k_proj_r<1", "update_proj"),
         (r"k_update_norm|k_proj_tma<4[,>]", "update_norm"), (r"k_combine", "combine")]


def cls(name):
    for pat, c in CLASS:
        if re.search(pat, name):
            return c
    return None


def rows_of(path):
    rows = [r for r in csv.reader(open(path)) if len(r) > 10]
    hdr = rows[0]
    return hdr, rows[1:]


def main():
    mpath, lpath, wl, prefix = sys.argv[1:5]
    hdr, rows = rows_of(mpath)
    ik, iv, im, iid = hdr.index("Kernel Name"), hdr.index("Metric Value"), hdr.index("Metric Name"), hdr.index("ID")
    per = collections.defaultdict(dict)
    for r in rows:
        per[(r[iid], r[ik])][r[im]] = float(r[iv].replace(",", ""))
    agg = collections.defaultdict(lambda: {"launches": 0, "dram": 0.0, "ns": 0.0, "kernels": set()})
    for (i, name), m in per.items():
        c = cls(name)
        if not c:
            continue
        a = agg[c]
        a["launches"] += 1
        a["dram"] += m.get("dram__bytes_read.sum", 0) + m.get("dram__bytes_write.sum", 0)
        a["ns"] += m.get("gpu__time_duration.sum", 0)
        a["kernels"].add(re.sub(r"\(.*", "", name).strip())
    out = {}
    # one SpMV call may be several launches (the column-blocked ring: one pass per column block);
    # per-call figures use the number of Krylov steps (one proj_dots launch each)
    steps = agg["proj_dots"]["launches"] if "proj_dots" in agg else None
    for c, a in agg.items():
        calls = a["launches"]
        if c == "spmv" and steps and a["launches"] > steps and a["launches"] % steps == 0:
            calls = steps
        out[c] = {"launches_captured": calls, "dram_bytes_per_launch": a["dram"] / calls,
                  "ncu_time_us_per_launch": a["ns"] / calls / 1e3, "kernels": sorted(a["kernels"])}
        if calls != a["launches"]:
            out[c]["kernel_launches_per_call"] = a["launches"] // calls
    tpath = os.path.join("profiles", "ncu_traffic.json")
    tab = json.load(open(tpath)) if os.path.exists(tpath) else {}
    tab[wl] = out
    json.dump(tab, open(tpath, "w"), indent=1, sort_keys=True)
    hdr, rows = rows_of(lpath)
    ik, iv, im = hdr.index("Kernel Name"), hdr.index("Metric Value"), hdr.index("Metric Name")
    tot = collections.defaultdict(lambda: [0, 0.0])
    for r in rows:
        if r[im] != "gpu__time_duration.sum":
            continue
        name = re.sub(r"\(.*", "", r[ik]).strip()
        tot[name][0] += 1
        tot[name][1] += float(r[iv].replace(",", ""))
    S = sum(v[1] for v in tot.values())
    with open(prefix + "_launches.md", "w") as f:
        f.write(f"# ncu launch list ({wl}): gpu__time_duration.sum per launch, --clock-control none\n\n")
        f.write("cold-cache, serialised replay: compare shares, not absolute times\n\n")
        f.write("| kernel | launches | total us | share |\n|---|---|---|---|\n")
        for k, v in sorted(tot.items(), key=lambda x: -x[1][1]):
            f.write(f"| {k} | {v[0]} | {v[1] / 1e3:.1f} | {v[1] / S:.3f} |\n")
    with open(prefix + "_traffic.md", "w") as f:
        f.write(f"# DRAM traffic per launch by kernel class ({wl}), one full restart (ncu --metrics)\n\n")
        f.write("| class | calls | DRAM MB/call | ncu us/call | DRAM GB/s (ncu) | kernels |\n|---|---|---|---|---|---|\n")
        for c, o in out.items():
            f.write(f"| {c} | {o['launches_captured']} | {o['dram_bytes_per_launch'] / 1e6:.1f} | "
                    f"{o['ncu_time_us_per_launch']:.1f} | {o['dram_bytes_per_launch'] / o['ncu_time_us_per_launch'] / 1e3:.0f} | "
                    f"{', '.join(o['kernels'])} |\n")
    print(json.dumps(out, indent=1))


if __name__ == "__main__":
    main()
