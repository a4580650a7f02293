"""Visit-order build (fused bounds + block radix sort + records) on the bench
workload for each LF_SORT_RB digit width: profile slot 0 (bounds+sort ms)."""
import argparse
import os
import sys
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
ap.add_argument("--max-epochs", type=int, default=50)
a = ap.parse_args()
args = bench.make_parser().parse_args(["--n", str(a.n), "--leaf-cap", str(a.leaf_cap), "--max-epochs", str(a.max_epochs)])
w = bench.setup_workload(args, torch.device("cuda", 0))
e, Q = w["eidx"], w["Q"]
ref = None
for rb in ("4", "5", "6", "7", "4"):
    os.environ["LF_SORT_RB"] = rb
    search_queries(e, Q, 1, target=0.99)
    ts = []
    for _ in range(5):
        prof = np.zeros(_lib.N_PROF)
        r = search_queries(e, Q, 1, target=0.99, profile=prof)
        ts.append(prof[0])
    ids = r.ids.cpu().numpy() if hasattr(r.ids, "cpu") else np.asarray(r.ids)
    same = ref is None or np.array_equal(ids, ref)
    ref = ids if ref is None else ref
    print(f"RB={rb} bounds+sort ms: median {np.median(ts):.3f} min {min(ts):.3f}  ids identical={same}", flush=True)
