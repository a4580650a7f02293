"""Print the headline fields of a bench.py JSON line."""
import json
import sys

d = json.loads([l for l in open(sys.argv[1] if len(sys.argv) > 1 else "gpurun_out/bench.json") if l.startswith("{")][-1])
for k in ("value", "ms_per_step", "recall_at_1", "leaves_pruned_pct", "e2e", "roofline", "filter_kernel",
          "train_data_gen", "cpu_baseline", "clocks", "gpu_launches"):
    print(k, json.dumps(d.get(k)))
