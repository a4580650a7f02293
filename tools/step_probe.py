"""Median search time of the bench workload (1K queries) through search_queries, with
the per-phase profile: for quick A/B of kernel variants on one box."""
import sys
import time
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
import numpy as np
import torch

import bench
from paper_2502_01836_b200 import _lib
from paper_2502_01836_b200.pipeline import search_queries

tag = sys.argv[1] if len(sys.argv) > 1 else ""
args = bench.make_parser().parse_args(sys.argv[2:])
w = bench.setup_workload(args, torch.device("cuda", 0))
e, Q = w["eidx"], w["Q"]
search_queries(e, Q, 1, target=0.99)
ts, profs = [], []
for _ in range(7):
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    prof = np.zeros(_lib.N_PROF)
    r = search_queries(e, Q, 1, target=0.99, profile=prof)
    torch.cuda.synchronize()
    ts.append(time.perf_counter() - t0)
    profs.append(prof.copy())
p = np.median(np.array(profs), axis=0)
print(f"{tag} total_ms={1e3 * np.median(ts):.3f} lf_search={p[6]:.3f} bounds={p[0]:.3f} plan={p[1]:.3f} "
      f"scan={p[2]:.3f} merge={p[3]:.3f} recall={bench.recall_of(r, w['exact']):.3f}", flush=True)
