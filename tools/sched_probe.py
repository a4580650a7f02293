"""Round-schedule probe on the bench workload through the graph plans: for each
(growth g, cap R) leaves per query per round grow as 2^(round * g) up to R; device
time per batch (CUDA events over 20 plan launches), series scanned, recall; plus the
sequential schedule's counters (the reference's one-leaf-at-a-time walk)."""
import os
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
import numpy as np
import torch

import bench
from paper_2502_01836_b200.pipeline import search_queries

args = bench.make_parser().parse_args(sys.argv[1:] + ["--tdg-queries", "0"])
w = bench.setup_workload(args, torch.device("cuda", 0))
e, Q = w["eidx"], w["Q"]
seq = search_queries(e, Q, 1, target=0.99, sequential=True)
print(f"sequential: leaves_searched {seq.stats[:, 1].mean():.2f} scanned {int(seq.stats[:, 5].sum())} "
      f"recall {bench.recall_of(seq, w['exact']):.3f}", flush=True)
configs = [tuple(map(int, c.split(":"))) for c in os.environ.get("SCHED", "2:256,3:256,1:256,2:64,3:512").split(",")]
for g, R in configs:
    os.environ["LF_ROUND_GROWTH_LOG2"] = str(g)
    e.__dict__.pop("_plans", None)
    r = search_queries(e, Q, 1, target=0.99, max_round_leaves=R)
    s = torch.cuda.current_stream()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(s)
    for _ in range(20):
        search_queries(e, Q, 1, target=0.99, max_round_leaves=R, copy_out=False)
    e1.record(s)
    torch.cuda.synchronize()
    print(f"g={g} R={R:4d} ms={e0.elapsed_time(e1) / 20:7.3f} leaves_searched={r.stats[:, 1].mean():6.2f} "
          f"scanned={int(r.stats[:, 5].sum()):11d} recall={bench.recall_of(r, w['exact']):.3f}", flush=True)
