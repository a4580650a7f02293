"""How much leaf data do the queries of one round share?  Runs the bench workload
with the batched trace, assigns each query's scanned leaves to rounds (doubling
schedule 1, 2, 4, .., 64 leaves per query per round) and compares the rows the
per-query scan reads with the rows a leaf-major scan (each (leaf, round) read
once for all its queries) would read."""
import argparse
import sys
from collections import Counter
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
import numpy as np
import torch

import bench
from paper_2502_01836_b200.pipeline import search_queries

ap = argparse.ArgumentParser()
ap.add_argument("--n", type=int, default=25_000_000)
ap.add_argument("--leaf-cap", type=int, default=10_000)
ap.add_argument("--max-epochs", type=int, default=1000)
a = ap.parse_args()
args = bench.make_parser().parse_args(["--n", str(a.n), "--leaf-cap", str(a.leaf_cap), "--max-epochs", str(a.max_epochs)])
w = bench.setup_workload(args, torch.device("cuda", 0))
e, Q, tree = w["eidx"], w["Q"], w["tree"]
di = tree.device()
size = {int(l): int(di.leaf_ptr_host[j + 1] - di.leaf_ptr_host[j]) for j, l in enumerate(di.leaf_ids)}
for exact in (False, True):
    r = search_queries(e, Q, 1, target=0.99, exact=exact, want_trace=True)
    tr = r.trace
    per_round = {}
    for qi in range(Q.shape[0]):
        n = int(tr["len"][qi])
        sl = [int(tr["leaf"][qi, j]) for j in range(n) if tr["searched"][qi, j]]
        j, rnd, R = 0, 0, 1
        while j < len(sl):
            per_round.setdefault(rnd, []).extend(sl[j:j + R])
            j += R
            rnd += 1
            R = min(2 * R, 64)
    tot_rows = tot_distinct = 0
    print(f"== {'exact' if exact else 'LeaFi 0.99'}: scanned rows {int(r.stats[:, 5].sum())}")
    for rnd in sorted(per_round):
        c = Counter(per_round[rnd])
        rows = sum(size[l] * k for l, k in c.items())
        distinct = sum(size[l] for l in c)
        tot_rows += rows
        tot_distinct += distinct
        print(f"round {rnd:2d}: (query, leaf) pairs {len(per_round[rnd]):6d}  leaves {len(c):5d}  rows {rows:11d}  "
              f"distinct rows {distinct:10d}  sharing x{rows / max(distinct, 1):.2f}")
    print(f"total rows {tot_rows}  distinct-per-round {tot_distinct}  sharing x{tot_rows / max(tot_distinct, 1):.2f}",
          flush=True)
