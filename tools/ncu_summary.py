"""Key --set full metrics of every launch in an ncu report (one line per launch):
duration, DRAM bytes and throughput, SM / memory throughput, issue-slot use,
achieved occupancy, registers, top warp-stall reasons.
    python tools/ncu_summary.py REPORT.ncu-rep > summary.txt"""
import csv
import io
import subprocess
import sys

rep = sys.argv[1]
out = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(out)))
hdr = rows[0]
col = {h: i for i, h in enumerate(hdr)}


units = rows[1]
SCALE = {"nsecond": 1e-3, "usecond": 1.0, "msecond": 1e3, "second": 1e6,            # -> us
         "byte": 1e-6, "Kbyte": 1e-3, "Mbyte": 1.0, "Gbyte": 1e3}                     # -> MB


def g(r, name):
    try:
        i = col[name]
        return float(r[i].replace(",", "")) * SCALE.get(units[i], 1.0)
    except (KeyError, ValueError):
        return float("nan")


stall_cols = [h for h in hdr if h.startswith("smsp__pcsamp_warps_issue_stalled_") and not h.endswith("_not_issued")]
print(f"{'#':>2} {'kernel':34s} {'us':>8s} {'DRAM MB':>8s} {'DRAM%':>6s} {'SM%':>6s} {'issue%':>7s} {'occ%':>6s} "
      f"{'regs':>5s}  top stalls")
for i, r in enumerate(rows[2:]):
    name = r[col["Kernel Name"]].split("(")[0].replace("void ", "").replace("lf::", "")[:34]
    dur = g(r, "gpu__time_duration.sum")
    dram = (g(r, "dram__bytes_read.sum") + g(r, "dram__bytes_write.sum"))
    stalls = sorted(((g(r, h), h.replace("smsp__pcsamp_warps_issue_stalled_", "")) for h in stall_cols), reverse=True)
    tot = sum(v for v, _ in stalls if v == v) or 1.0
    top = ", ".join(f"{n} {100 * v / tot:.0f}%" for v, n in stalls[:3])
    print(f"{i:2d} {name:34s} {dur:8.1f} {dram:8.1f} {g(r, 'gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed'):6.1f} "
          f"{g(r, 'sm__throughput.avg.pct_of_peak_sustained_elapsed'):6.1f} "
          f"{g(r, 'sm__inst_issued.avg.pct_of_peak_sustained_active'):7.1f} "
          f"{g(r, 'sm__warps_active.avg.pct_of_peak_sustained_active'):6.1f} "
          f"{g(r, 'launch__registers_per_thread'):5.0f}  {top}")
