import sys; sys.path.insert(0, "/root/repo")
import numpy as np, torch
from oracle import leafi_oracle as lo
from paper_2502_01836_b200 import build_index, search_batch
from paper_2502_01836_b200.filters import FilterPack
data = lo.randwalk(30000, 64, 91)
t = build_index(data, 150)
rng = np.random.default_rng(3)
leaves = [int(l) for l in t.leaf_ids]
sel = sorted(set(leaves[::2] + leaves[1::7]))
F, m = len(sel), 64
pack = FilterPack(sel, rng.normal(0, 0.08, (F, m, m)), rng.normal(0, 0.05, (F, m)), rng.normal(0, 0.08, (F, m)), rng.uniform(1.0, 9.0, F), path="tc")
Q = np.concatenate([lo.noisy_queries(data, 70, nz, 40 + int(10 * nz)) for nz in (0.1, 0.3, 0.6)])
qd = torch.from_numpy(Q.astype(np.float32)).cuda()
di = t.device()
offs = rng.uniform(0.0, 1.5, F)
lf = pack.leaf_filter(di)
P = pack.predict(qd)
dense = search_batch(t, qd, 1, predictions=P, offsets=offs, leaf_filter=lf, want_trace=True)
lazy = search_batch(t, qd, 1, filters=pack, offsets=offs, leaf_filter=lf, want_trace=True)
bad = np.nonzero(dense.ids[:, 0] != lazy.ids[:, 0])[0]
print("bad", bad, "nodes", t.n_nodes, "F", F)
Ph = P.cpu().numpy()
slot = {l: i for i, l in enumerate(sel)}
for qi in bad[:2]:
    td, tl = dense.trace_of(qi), lazy.trace_of(qi)
    print("query", qi, "len", len(td), len(tl))
    for j, (a, b) in enumerate(zip(td, tl)):
        if a.leaf_id != b.leaf_id or a.searched != b.searched:
            l = a.leaf_id
            s = slot.get(l)
            print(" first diff at", j, a, b, "pred", None if s is None else (Ph[qi, s], Ph[qi, s] - offs[s]))
            break
prof = np.zeros(16)
lazy2 = search_batch(t, qd, 1, filters=pack, offsets=offs, leaf_filter=lf, profile=prof)
ot = lo.build_tree(data, 150)
exp = 0
per_q = []
for qi in range(Q.shape[0]):
    qs = lo.paa(Q[qi], ot.starts, ot.widths)
    lbs = np.array([lo.node_lb(qs, ot.env_min[n], ot.env_max[n], ot.widths) for n in range(t.n_nodes)])
    order = np.lexsort((np.arange(t.n_nodes), lbs))
    first = next(n for n in order if ot.is_leaf(n))
    d = lo.row_dist(Q[qi], data[ot.members[first]]).min()
    c = sum(1 for n in order if lbs[n] <= d and ot.is_leaf(n) and n in slot and n != first)
    c += 1 if first in slot else 0
    per_q.append(c)
    exp += c
print("pairs expected", exp, "(includes the first leaf)", "got", prof[11], "predict_ms", prof[10])
# pair predictions vs dense
pq = np.repeat(np.arange(Q.shape[0]), F)
pf = np.tile(np.arange(F), Q.shape[0])
pp = pack.predict_pairs(qd, pq, pf).cpu().numpy().reshape(Q.shape[0], F)
print("pairs vs dense: max abs diff", np.abs(pp - Ph.astype(np.float64)).max(), "n diff", int((pp != Ph.astype(np.float64)).sum()))
