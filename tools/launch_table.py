"""Per-kernel device time and DRAM bytes from an ncu --csv launch list captured with
--metrics gpu__time_duration.sum[,dram__bytes_read.sum]."""
import collections
import csv
import sys

rows = [r for r in csv.reader(open(sys.argv[1])) if len(r) > 10]
hdr = rows[0]
ik, im, iv = hdr.index("Kernel Name"), hdr.index("Metric Name"), hdr.index("Metric Value")
agg = collections.defaultdict(lambda: [0.0, 0.0, 0])
for r in rows[1:]:
    name = r[ik].split("(")[0].replace("void ", "")[:34]
    val = float(r[iv].replace(",", ""))
    if "time" in r[im]:
        agg[name][0] += val
        agg[name][2] += 1
    else:
        agg[name][1] += val
tot = sum(a[0] for a in agg.values())
print(f"{'kernel':36s} {'n':>4s} {'us':>9s} {'share':>6s} {'GB':>7s} {'GB/s':>7s}")
for k, (t, b, n) in sorted(agg.items(), key=lambda x: -x[1][0]):
    print(f"{k:36s} {n:4d} {t / 1e3:9.1f} {100 * t / tot:5.1f}% {b / 1e9:7.3f} {b / t if t else 0:7.0f}")
print(f"{'total':36s} {'':4s} {tot / 1e3:9.1f}")
