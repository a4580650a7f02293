"""Top stall lines of one kernel from an ncu report's SASS source page.
    python tools/ncu_src_top.py REPORT.ncu-rep KERNEL_REGEX [N]"""
import csv
import io
import subprocess
import sys

rep, kre = sys.argv[1], sys.argv[2]
n = int(sys.argv[3]) if len(sys.argv) > 3 else 20
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "-k", f"regex:{kre}", "--print-source", "sass"],
                     capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(out)))
hdrs = [i for i, r in enumerate(rows) if r and r[0] == "Address"]
hi = hdrs[-1]
hdr = rows[hi]
data = [r for r in rows[hi + 1:] if len(r) == len(hdr)]
ai, si = hdr.index("Address"), hdr.index("Source")
wi, ei = hdr.index("Warp Stall Sampling (All Samples)"), hdr.index("Instructions Executed")
tot = sum(float(r[wi] or 0) for r in data)
print(f"{rows[hi - 1][1][:100]}\nsamples {tot:.0f}")
for idx, r in sorted(enumerate(data), key=lambda x: -float(x[1][wi] or 0))[:n]:
    ctx = " <- " + data[idx - 1][si][:40] if idx else ""
    print(f"{float(r[wi]) / tot * 100:5.1f}% #{idx:5d} {r[si][:70]:70s} exec={r[ei]}{ctx}")
