"""Build profiles/scan_kernel_ncu.json (bench.py's roofline.traffic) from the
scan-kernel DRAM capture of tools/ncu_capture.sh: measured DRAM bytes of every
leaf-scan launch of one timed step next to the algorithmic bytes bench.py
counted for the same step."""
import csv
import json
import sys

csv_path = sys.argv[1] if len(sys.argv) > 1 else "gpurun_out/scan_dram.csv"
bench_path = sys.argv[2] if len(sys.argv) > 2 else "gpurun_out/ncu_dram_bench.json"
out_path = sys.argv[3] if len(sys.argv) > 3 else "profiles/scan_kernel_ncu.json"
rows = list(csv.DictReader([l for l in open(csv_path) if l.startswith('"')]))
per = {}
for r in rows:
    per.setdefault(r["ID"], {"kernel": r["Kernel Name"].split("(")[0]})[r["Metric Name"]] = (
        float(r["Metric Value"].replace(",", "")), r["Metric Unit"])


def to_bytes(v):
    val, unit = v
    return val * {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}.get(unit, 1)


def to_ns(v):
    val, unit = v
    return val * {"nsecond": 1, "usecond": 1e3, "msecond": 1e6}.get(unit, 1)


launches = []
for k, v in per.items():
    launches.append({"id": int(k), "kernel": v["kernel"],
                     "dram_read_bytes": to_bytes(v["dram__bytes_read.sum"]),
                     "dram_write_bytes": to_bytes(v["dram__bytes_write.sum"]),
                     "ns": to_ns(v["gpu__time_duration.sum"])})
b = json.loads([l for l in open(bench_path) if l.startswith("{")][-1])
alg = b["roofline"]["algorithmic_bytes_per_step"]
n = len(launches)
# one scan phase per round: its streaming kernel (scan_q8 / scan_pq) plus, after scan_pq,
# the survivor re-read and selection kernels -- bench.py's "achieved" and "traffic" are per phase
rounds = sum(1 for x in launches if "scan_q8" in x["kernel"] or "scan_pq" in x["kernel"])
tot = sum(x["dram_read_bytes"] + x["dram_write_bytes"] for x in launches)
out = {
    "source": "ncu --metrics dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum, every scan "
              "launch of one timed bench step (tools/ncu_capture.sh)",
    "launches_per_step": n,
    "scan_phases_per_step": rounds,
    "dram_bytes_per_step": tot,
    "dram_bytes_per_launch": tot / max(rounds, 1),
    "dram_bytes_per_launch_definition": "per scan phase (round): streaming kernel + survivor re-read / selection kernels",
    "algorithmic_bytes_per_step": alg,
    "algorithmic_bytes_per_launch": alg / max(rounds, 1),
    "traffic_over_algorithmic": tot / alg if alg else None,
    "scan_ns_serialised_per_step": sum(x["ns"] for x in launches),
    "launches": launches,
}
json.dump(out, open(out_path, "w"), indent=1)
print(json.dumps({k: v for k, v in out.items() if k != "launches"}, indent=1))
