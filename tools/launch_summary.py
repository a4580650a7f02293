"""Summarise an ncu launch list (--metrics gpu__time_duration.sum --csv) per kernel."""
import csv
import sys

path = sys.argv[1] if len(sys.argv) > 1 else "gpurun_out/launches.csv"
lines = [l for l in open(path) if l.startswith('"')]
rows = list(csv.DictReader(lines))
tot = sum(float(r["Metric Value"]) for r in rows)
agg = {}
for r in rows:
    n = r["Kernel Name"].split("(")[0].replace("void ", "")
    a = agg.setdefault(n, [0, 0.0])
    a[0] += 1
    a[1] += float(r["Metric Value"])
print(f"{'kernel':72s} {'launches':>8s} {'ms':>9s} {'share':>7s}")
for n, (c, t) in sorted(agg.items(), key=lambda x: -x[1][1]):
    print(f"{n[:72]:72s} {c:8d} {t / 1e6:9.3f} {100 * t / tot:6.2f}%")
print(f"{'total':72s} {len(rows):8d} {tot / 1e6:9.3f}")
