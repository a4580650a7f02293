"""How many (query, filtered leaf) pairs can the walk reach once round 0's best-so-far
is known?  Counts, per query, the leaves with lb <= bsf0 (bsf0 = exact best in the
query's first leaf) and lb <= bsf_final, on the bench workload (25M x 256, cap 10K)."""
import sys, time
from pathlib import Path
sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
import numpy as np
import torch

from paper_2502_01836_b200 import build_index_device, search_batch
from paper_2502_01836_b200.engine import query_bounds
from paper_2502_01836_b200.synth import queries_device, randwalk_device

n = int(sys.argv[1]) if len(sys.argv) > 1 else 25_000_000
X = randwalk_device(n, 256, 1234)
tree = build_index_device(X, max_leaf_size=10_000)
di = tree.device()
Q = torch.cat([queries_device(X, 250, nz, 1234 + int(10 * nz)) for nz in (0.1, 0.2, 0.3, 0.4)]).contiguous()
ex = search_batch(tree, Q, 1)
_, lb = query_bounds(Q.cpu().numpy().astype(np.float64), tree.env_min, tree.env_max, tree.starts, tree.widths)
leaves = tree.leaf_ids
lbl = lb[:, leaves]                                   # [Q, L] in leaf-slot order
first = np.lexsort((np.broadcast_to(np.arange(len(leaves)), lbl.shape), lbl), axis=1)[:, 0] if False else None
order = np.argsort(lbl, axis=1, kind="stable")
first = order[:, 0]
ptr = di.leaf_ptr_host
bsf0 = np.empty(Q.shape[0])
for s in np.unique(first):
    qs = np.nonzero(first == s)[0]
    rows = di.X[ptr[s]:ptr[s + 1]].double()
    d = torch.cdist(Q[torch.from_numpy(qs).cuda()].double(), rows).min(1).values
    bsf0[qs] = d.cpu().numpy()
fin = ex.dists[:, 0]
r0 = (lbl <= bsf0[:, None]).sum(1)
rf = (lbl <= fin[:, None]).sum(1)
for i, nz in enumerate((0.1, 0.2, 0.3, 0.4)):
    sl = slice(250 * i, 250 * (i + 1))
    print(f"noise {nz}: reach(bsf0) mean {r0[sl].mean():.0f} max {r0[sl].max()}  reach(final) mean {rf[sl].mean():.0f}"
          f"  bsf0/final {np.mean(bsf0[sl] / fin[sl]):.3f}")
print(f"total pairs reach(bsf0) {r0.sum()}  reach(final) {rf.sum()}  dense {lbl.size}")
