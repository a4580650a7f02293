"""Round schedule probe on the bench workload: leaves per query per round grow as
2^(round * g) up to max_round_leaves; total search time, rounds, scanned series."""
import os
import sys
import time
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
import numpy as np
import torch

import bench
from paper_2502_01836_b200 import _lib
from paper_2502_01836_b200.pipeline import search_queries

args = bench.make_parser().parse_args(sys.argv[1:])
w = bench.setup_workload(args, torch.device("cuda", 0))
e, Q = w["eidx"], w["Q"]
for g, R in ((1, 64), (2, 128), (2, 256), (2, 512), (3, 512), (4, 256), (2, 1024), (3, 4096)):
    os.environ["LF_ROUND_GROWTH_LOG2"] = str(g)
    search_queries(e, Q, 1, target=0.99, max_round_leaves=R)
    ts = []
    for _ in range(5):
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        prof = np.zeros(_lib.N_PROF)
        r = search_queries(e, Q, 1, target=0.99, max_round_leaves=R, profile=prof)
        torch.cuda.synchronize()
        ts.append(time.perf_counter() - t0)
    print(f"g={g} R={R:4d} total_ms={1e3 * np.median(ts):7.3f} lf_search_ms={prof[6]:7.3f} rounds={int(prof[4])} "
          f"scanned={int(r.stats[:, 5].sum()):11d} recall={bench.recall_of(r, w['exact']):.3f}", flush=True)
