"""Feasibility probe: if the rows of every leaf were ordered along the leaf's own
principal direction (in the projected space), how many 512-row chunks of the leaves a
query can reach (lb <= its exact 1-NN distance) could be skipped whole by a chunk bound
(||y_q - c|| - rho, plus the residual-norm interval) at the query's final best-so-far?
Compared with the rows' current order."""
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
import numpy as np
import torch

import bench
from paper_2502_01836_b200.engine import query_bounds

args = bench.make_parser().parse_args(sys.argv[1:] + ["--tdg-queries", "0"])
w = bench.setup_workload(args, torch.device("cuda", 0))
tree, di, Q, exact = w["tree"], w["di"], w["Q"], w["exact"]
P, mu = di.P, di.mu
L = di.n_leaves
ptr = di.leaf_ptr_host
bsf = torch.from_numpy(exact.dists[:, 0]).cuda()
Qd = Q.double()
yq = (Qd - mu) @ P.T
rq = ((Qd - mu) - yq @ P).norm(dim=1)
_, lb = query_bounds(Q.cpu().numpy().astype(np.float64), tree.env_min, tree.env_max, tree.starts, tree.widths)
lbl = torch.from_numpy(lb[:, tree.leaf_ids]).cuda()
CH = 512
tot = {"sorted": [0, 0], "original": [0, 0]}
for s in range(L):
    X = di.X[ptr[s]:ptr[s + 1]].double()
    y = (X - mu) @ P.T
    r = ((X - mu) - y @ P).norm(dim=1)
    qs = torch.nonzero(lbl[:, s] <= bsf).flatten()
    if qs.numel() == 0:
        continue
    yc = y - y.mean(0)
    _, _, V = torch.linalg.svd(yc, full_matrices=False)
    orders = {"sorted": torch.argsort(yc @ V[0]), "original": torch.arange(y.shape[0], device=y.device)}
    for name, o in orders.items():
        ys, rs = y[o], r[o]
        for c0 in range(0, ys.shape[0], CH):
            cy, cr = ys[c0:c0 + CH], rs[c0:c0 + CH]
            c = cy.mean(0)
            rho = (cy - c).norm(dim=1).max()
            dproj = ((yq[qs] - c).norm(dim=1) - rho).clamp(min=0)
            dres = torch.maximum(cr.min() - rq[qs], rq[qs] - cr.max()).clamp(min=0)
            skip = (dproj ** 2 + dres ** 2).sqrt() > bsf[qs] * (1 + 1e-6)
            tot[name][0] += int(skip.sum()) * cy.shape[0]
            tot[name][1] += qs.numel() * cy.shape[0]
for name, (sk, all_) in tot.items():
    print(f"{name}: rows in reachable chunks {all_}, skippable {sk} ({100.0 * sk / max(all_, 1):.1f}%)", flush=True)
