"""Small end-to-end workload for compute-sanitizer (tools/sanitize.sh): every kernel
family of the library once, at sizes the sanitizer finishes in minutes.  Results are
checked against the oracle so a silent corruption also fails the run."""
import os
import sys
import tempfile
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))

import numpy as np
import torch

from oracle import leafi_oracle as lo
from paper_2502_01836_b200 import build_index, load_index, save_dataset, search_batch
from paper_2502_01836_b200.filters import FilterPack
from paper_2502_01836_b200.targets import leaf_min_distances

m = 256
data = lo.randwalk(6000, m, 5)
t = build_index(data, 400)
di = t.device()
di.ensure_pca(32)                     # projected shadow (pq scans, seeded round 0)
Q = np.concatenate([lo.noisy_queries(data, 12, nz, 7 + int(10 * nz)) for nz in (0.1, 0.4)])
qd = torch.from_numpy(Q.astype(np.float32)).cuda()
ot = lo.build_tree(data, 400)

for k, seq in ((1, False), (3, False), (1, True)):
    r = search_batch(t, qd, k, sequential=seq)
    for i in range(0, len(Q), 5):
        assert r.ids[i].tolist() == [a for a, _ in lo.search(ot, Q[i], k).results], (k, seq, i)

rng = np.random.default_rng(3)
leaves = [int(l) for l in t.leaf_ids]
F = len(leaves)
pack = FilterPack(leaves, rng.normal(0, 0.05, (F, m, m)), rng.normal(0, 0.05, (F, m)),
                  rng.normal(0, 0.05, (F, m)), rng.uniform(1.0, 6.0, F), path="tc16")
offs = rng.uniform(0.0, 1.0, F)
lf = pack.leaf_filter(di)
dense = search_batch(t, qd, 1, predictions=pack.predict(qd), offsets=offs, leaf_filter=lf)
reach = search_batch(t, qd, 1, filters=pack, offsets=offs, leaf_filter=lf)
assert np.array_equal(dense.ids, reach.ids) and np.array_equal(dense.stats, reach.stats)

from paper_2502_01836_b200.engine import SearchPlan

# the CUDA-graph path (conditional WHILE node set from the device).  racecheck and
# synccheck abort on device-updated conditional graphs, so only memcheck / initcheck
# run it; the kernels inside are the ones search_batch launched above.
if os.environ.get("SAN_TOOL", "memcheck") in ("memcheck", "initcheck"):
    plan = SearchPlan(t, Q.shape[0], 1, filters=pack, offsets=offs, leaf_filter=lf)
    for _ in range(2):
        g = plan.run(qd)
        assert np.array_equal(g.ids, reach.ids) and np.array_equal(g.stats, reach.stats)
    plan.close()
big = build_index(lo.randwalk(60000, 32, 9), 18)                   # > 8,192 nodes: the big leaf order
Qb = lo.noisy_queries(lo.randwalk(60000, 32, 9), 8, 0.3, 5)
rb = search_batch(big, Qb, 3)
for i in range(0, 8, 3):
    assert rb.ids[i].tolist() == [a for a, _ in lo.linear_scan(lo.randwalk(60000, 32, 9), Qb[i], 3)]

dl = leaf_min_distances(t, qd, list(range(di.n_leaves))).cpu().numpy()
for i in range(0, len(Q), 6):
    for j in (0, di.n_leaves - 1):
        rows = data[t.leaf_members(int(t.leaf_ids[j]))]
        assert abs(dl[i, j] - np.sqrt(((rows - Q[i]) ** 2).sum(1)).min()) <= 1e-9 * max(1.0, dl[i, j])

with tempfile.TemporaryDirectory() as d:
    p = Path(d) / "c.bin"
    save_dataset(torch.from_numpy(data.astype(np.float32)).cuda(), p)
    t2 = load_index(p, 400)
    assert torch.equal(t2.device().X, di.X)
torch.cuda.synchronize()
print("sanitize driver ok")
