"""Scan variant x round schedule on the bench workload: scanned volume, early-abandon
survivors, scan time, recall.  One setup, many configurations."""
import argparse
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

ap = argparse.ArgumentParser()
ap.add_argument("--n", type=int, default=25_000_000)
ap.add_argument("--leaf-cap", type=int, default=10_000)
ap.add_argument("--max-epochs", type=int, default=1000)
a = ap.parse_args()
args = bench.make_parser().parse_args(["--n", str(a.n), "--leaf-cap", str(a.leaf_cap), "--max-epochs", str(a.max_epochs)])
w = bench.setup_workload(args, torch.device("cuda", 0))
e, Q = w["eidx"], w["Q"]
configs = [("q8", dict(max_round_leaves=64)), ("ea2", dict(max_round_leaves=64)), ("full", dict(max_round_leaves=64)),
           ("q8", dict(max_round_leaves=16)), ("q8", dict(max_round_leaves=256))]
for var, kw in configs:
    os.environ["LF_SCAN_VARIANT"] = var
    search_queries(e, Q, 1, target=0.99, **kw)
    torch.cuda.synchronize()
    prof = np.zeros(_lib.N_PROF)
    t0 = time.perf_counter()
    r = search_queries(e, Q, 1, target=0.99, profile=prof, **kw)
    dt = time.perf_counter() - t0
    surv = prof[9] / prof[8] if prof[8] else float("nan")
    print(f"{var:4s} {str(kw):28s} scanned={int(r.stats[:, 5].sum()):11d} leaves={r.stats[:, 1].mean():6.2f} "
          f"recall={bench.recall_of(r, w['exact']):.3f} rounds={int(prof[4]):3d} scan_ms={prof[2]:7.2f} "
          f"total_ms={dt * 1e3:7.2f} survivors={surv:.3f}", flush=True)
