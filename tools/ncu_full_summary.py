"""Summarise an `ncu --set full` report into a markdown table (one row per captured launch).
Usage: python tools/ncu_full_summary.py <report.ncu-rep> <out.md> <title> [raw_out.csv]"""
import csv
import io
import subprocess
import sys

rep, out, title = sys.argv[1:4]
raw = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
if len(sys.argv) > 4:
    open(sys.argv[4], "w").write(raw)
rows = list(csv.reader(io.StringIO(raw)))
hdr, units, data = rows[0], rows[1], rows[2:]
col = {k: i for i, k in enumerate(hdr)}


def g(r, k):
    i = col.get(k)
    return r[i] if i is not None else ""


lines = [f"# {title}", "",
         "ncu --set full --clock-control none --import-source on (one capture per listed launch; cold caches,",
         "serialised replay).", "",
         "| kernel | time (us) | DRAM read (MB) | DRAM write (MB) | DRAM % peak | L2 hit % | L1 hit % | warps active % | regs | "
         "grid | block | top stalls (samples) |", "|" + "---|" * 12]
for r in data:
    stalls = []
    for k, i in col.items():
        if k.startswith("smsp__pcsamp_warps_issue_stalled_") and not k.endswith("not_issued"):
            try:
                stalls.append((float(r[i]), k.replace("smsp__pcsamp_warps_issue_stalled_", "")))
            except ValueError:
                pass
    stalls.sort(reverse=True)
    tot = sum(s for s, _ in stalls) or 1.0
    top = ", ".join(f"{n} {100 * s / tot:.0f}%" for s, n in stalls[:4])
    rd = float(g(r, "dram__bytes_read.sum") or 0)
    wr = float(g(r, "dram__bytes_write.sum") or 0)
    scale = {"byte": 1e-6, "Kbyte": 1e-3, "Mbyte": 1.0, "Gbyte": 1e3}
    ur, uw = units[col["dram__bytes_read.sum"]], units[col["dram__bytes_write.sum"]]
    tus = float(g(r, "gpu__time_duration.sum") or 0)
    ut = units[col["gpu__time_duration.sum"]]
    tus = tus / 1e3 if ut == "nsecond" else (tus * 1e3 if ut == "msecond" else tus)
    lines.append(f"| {g(r, 'Kernel Name')[:60]} | {tus:.1f} | {rd * scale.get(ur, 1):.1f} | {wr * scale.get(uw, 1):.1f} | "
                 f"{float(g(r, 'gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed') or 0):.1f} | "
                 f"{float(g(r, 'lts__t_sector_hit_rate.pct') or 0):.1f} | {float(g(r, 'l1tex__t_sector_hit_rate.pct') or 0):.1f} | "
                 f"{float(g(r, 'sm__warps_active.avg.pct_of_peak_sustained_active') or 0):.1f} | "
                 f"{g(r, 'launch__registers_per_thread')} | {g(r, 'launch__grid_size')} | {g(r, 'launch__block_size')} | {top} |")
sass = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "sass"], capture_output=True,
                      text=True).stdout
marks = [m for m in ("UTMALDG", "UBLKCP", "SYNCS.PHASECHK", "SYNCS.ARRIVE", "LDG.E.128.CONSTANT", "LDG.E.EF")
         if m in sass]
lines += ["", f"SASS of the captured kernels contains: {', '.join(marks)}."]
open(out, "w").write("\n".join(lines) + "\n")
print("\n".join(lines))
