"""CPU oracle for the LeaFi hot path -- TEST INFRASTRUCTURE ONLY.

This module is a numpy restatement of the reference package `leafsearch`
(arXiv 2502.01836 companion code, /root/reference/pkg/src/leafsearch) for the
functions on the query-time and training-data hot path.  Every function cites
the reference file:line it follows.  It exists to CHECK the CUDA path:

* only `tests/`, `__graft_entry__.smoke()` and the `cpu_baseline` /
  `--impl reference` legs of `bench.py` may import it;
* the product package `paper_2502_01836_b200` never imports it and has no CPU
  fallback.

Parity is pinned: `tests/test_oracle_golden.py` checks this restatement
bit-for-bit against golden vectors produced by running the real reference
(`tests/golden/make_golden.py`, committed together with its outputs).

Numerics follow the reference exactly: series are fp32-exact values held in
fp64, segment means use `np.add.reduceat`, the lower bound uses `np.dot`
(one fp64 FMA chain on x86 OpenBLAS), leaf scans use the direct
subtract-square-sum form in fp64, filters run in fp32.
"""

from __future__ import annotations

import heapq
import math
from dataclasses import dataclass, field

import numpy as np

RECALL_REL_TOL = 1e-6  # conformal.py:20, cli.py:34


# ---------------------------------------------------------------------------
# seeds and synthetic data (series.py, traingen.py, enhanced.py)
# ---------------------------------------------------------------------------

def derive_seed(master: int, tag: int) -> int:
    """enhanced.py:66-67."""
    return (master * 1_000_003 + tag) % (2**31 - 1)


def to_f32_exact(a) -> np.ndarray:
    """series.py:48-50 (`quantize32`)."""
    return np.asarray(a, dtype=np.float64).astype(np.float32).astype(np.float64)


def randwalk(n: int, m: int, seed: int) -> np.ndarray:
    """series.py:161-171: cumulative N(0,1) steps, z-normalised (ddof=1), fp32-exact."""
    g = np.random.default_rng(seed)
    w = np.cumsum(g.standard_normal((n, m)), axis=1)
    mu = w.mean(axis=1, keepdims=True)
    sd = w.std(axis=1, ddof=1, keepdims=True)
    if not (sd > 0).all():
        raise ValueError("degenerate random walk")
    return to_f32_exact((w - mu) / sd)


def noisy_queries(values: np.ndarray, count: int, noise: float, seed: int) -> np.ndarray:
    """series.py:174-187 (`make_queries`): uniform source row + N(0, noise^2)."""
    g = np.random.default_rng(seed)
    src = g.integers(0, values.shape[0], size=count)
    eps = g.standard_normal((count, values.shape[1])) * noise
    return to_f32_exact(values[src] + eps)


def _levelled_noise(rows: np.ndarray, lo: float, hi: float, g) -> tuple:
    """traingen.py:100-107: per-row uniform noise level in [lo, hi]."""
    if not 0.0 <= lo <= hi <= 1.0:
        raise ValueError("bad noise range")
    lv = g.uniform(lo, hi, size=rows.shape[0])
    eps = g.standard_normal(rows.shape) * lv[:, None]
    return to_f32_exact(rows + eps), lv


def global_queries(values: np.ndarray, n: int, noise_range, seed: int) -> tuple:
    """traingen.py:110-117."""
    g = np.random.default_rng(seed)
    src = g.integers(0, values.shape[0], size=n)
    return _levelled_noise(values[src], float(noise_range[0]), float(noise_range[1]), g)


def local_queries(tree: "OracleTree", leaf_id: int, n: int, noise_range, seed: int) -> tuple:
    """traingen.py:120-132: returns (queries, levels, source_ids)."""
    ids = tree.members[leaf_id]
    g = np.random.default_rng(seed)
    pick = g.integers(0, ids.shape[0], size=n)
    rows = tree.values[ids[pick]]
    q, lv = _levelled_noise(rows, float(noise_range[0]), float(noise_range[1]), g)
    return q, lv, ids[pick]


# ---------------------------------------------------------------------------
# summaries and bounds (summarize.py)
# ---------------------------------------------------------------------------

def seg_layout(m: int, l: int) -> tuple:
    """summarize.py:27-37: equal widths, leading segments take the remainder."""
    if not 1 <= l <= m:
        raise ValueError("bad segment count")
    q, r = divmod(m, l)
    widths = np.array([q + (1 if i < r else 0) for i in range(l)], dtype=np.int64)
    starts = np.concatenate(([0], np.cumsum(widths)[:-1])).astype(np.int64)
    return starts, widths


def paa(values: np.ndarray, starts: np.ndarray, widths: np.ndarray) -> np.ndarray:
    """summarize.py:44-56: per-segment means (np.add.reduceat, then / width)."""
    v = np.asarray(values, dtype=np.float64)
    if v.ndim == 1:
        return np.add.reduceat(v, starts) / widths
    return np.add.reduceat(v, starts, axis=1) / widths


def node_lb(qsumm: np.ndarray, mn: np.ndarray, mx: np.ndarray, widths: np.ndarray) -> float:
    """summarize.py:97-107: sqrt(sum_i w_i * gap_i^2) via np.dot (search path)."""
    gap = np.maximum(mn - qsumm, qsumm - mx)
    gap = np.maximum(gap, 0.0)
    return math.sqrt(float(np.dot(widths * gap, gap)))


def lb_matrix(qsumms: np.ndarray, mins: np.ndarray, maxs: np.ndarray, widths: np.ndarray) -> np.ndarray:
    """summarize.py:114-122: all (query, node) bounds via einsum (traingen path)."""
    qs = np.atleast_2d(qsumms)
    gap = np.maximum(mins[None] - qs[:, None], qs[:, None] - maxs[None])
    gap = np.maximum(gap, 0.0)
    return np.sqrt(np.einsum("qns,qns,s->qn", gap, gap, widths.astype(np.float64)))


# ---------------------------------------------------------------------------
# EAPCA bound (north_star "EAPCA/SAX summarisation bounds").
# PARITY UNPINNED: the reference has no EAPCA code (its envelopes keep segment
# means only, summarize.py:59-107).  This is the repository's
# own CPU restatement of the DSTree EAPCA bound in the shape of
# summarize.py:97-107, defined so the GPU can reproduce it bit for bit:
#   per segment i (start s_i, width w_i):
#     mean_i = the reference segment mean (paa: np.add.reduceat / w_i);
#     sd_i   = sqrt(S_i / w_i), S_i = sum over t of (x_t - mean_i)^2 added LEFT
#              TO RIGHT in fp64 (population stdev);
#   node envelope: [min, max] of the members' means (the reference envelope)
#   and of their sds;
#   lb^2 = sum_i w_i * (gm_i^2 + gs_i^2), left to right, no fused multiply-add,
#   gm_i = max(mean_min - mu_q, mu_q - mean_max, 0), gs_i likewise for sd.
# Sound: per segment, ||q - x||^2 = w (mu_q - mu_x)^2 + ||q~ - x~||^2 and
# ||q~ - x~|| >= | ||q~|| - ||x~|| | = sqrt(w) |sd_q - sd_x|.
# ---------------------------------------------------------------------------

def eapca(values: np.ndarray, starts: np.ndarray, widths: np.ndarray) -> tuple:
    """(means, sds), each [n, l] (or [l] for one series)."""
    v = np.asarray(values, dtype=np.float64)
    one = v.ndim == 1
    v = np.atleast_2d(v)
    mu = paa(v, starts, widths)
    sd = np.empty_like(mu)
    for i, (s, w) in enumerate(zip(starts, widths)):
        acc = np.zeros(v.shape[0])
        for t in range(int(s), int(s + w)):
            d = v[:, t] - mu[:, i]
            acc = acc + d * d
        sd[:, i] = np.sqrt(acc / float(w))
    return (mu[0], sd[0]) if one else (mu, sd)


def eapca_envelopes(t: "OracleTree") -> tuple:
    """Per node [min, max] of the members' segment sds (internal nodes: all descendants)."""
    _, sd = eapca(t.values, t.starts, t.widths)
    l = t.widths.shape[0]
    smin = [np.full(l, math.inf) for _ in range(t.n_nodes)]
    smax = [np.full(l, -math.inf) for _ in range(t.n_nodes)]
    for nid in reversed(range(t.n_nodes)):          # children have larger ids than parents
        if t.is_leaf(nid):
            ids = t.members[nid]
            if ids.size:
                smin[nid] = sd[ids].min(axis=0)
                smax[nid] = sd[ids].max(axis=0)
        else:
            for c in (t.left[nid], t.right[nid]):
                smin[nid] = np.minimum(smin[nid], smin[c])
                smax[nid] = np.maximum(smax[nid], smax[c])
    return smin, smax


def node_lb_eapca(qmu, qsd, mn, mx, smn, smx, widths) -> float:
    """The EAPCA bound of one node (definition above)."""
    return float(lb_matrix_eapca(np.atleast_2d(qmu), np.atleast_2d(qsd), np.atleast_2d(mn), np.atleast_2d(mx),
                                 np.atleast_2d(smn), np.atleast_2d(smx), widths)[0, 0])


def lb_matrix_eapca(qmu, qsd, mins, maxs, smins, smaxs, widths) -> np.ndarray:
    """All (query, node) EAPCA bounds [Q, nodes]."""
    qmu, qsd = np.atleast_2d(qmu), np.atleast_2d(qsd)
    acc = np.zeros((qmu.shape[0], mins.shape[0]))
    for i in range(widths.shape[0]):
        gm = np.maximum(mins[None, :, i] - qmu[:, None, i], qmu[:, None, i] - maxs[None, :, i])
        gm = np.maximum(gm, 0.0)
        gs = np.maximum(smins[None, :, i] - qsd[:, None, i], qsd[:, None, i] - smaxs[None, :, i])
        gs = np.maximum(gs, 0.0)
        acc = acc + float(widths[i]) * (gm * gm + gs * gs)
    return np.sqrt(acc)


# ---------------------------------------------------------------------------
# distances (series.py)
# ---------------------------------------------------------------------------

def row_dist(q: np.ndarray, block: np.ndarray) -> np.ndarray:
    """series.py:142-146: one query vs every row, direct form, fp64."""
    d = np.asarray(block, dtype=np.float64) - q
    return np.sqrt(np.einsum("ij,ij->i", d, d))


def pair_dist(queries: np.ndarray, block: np.ndarray, chunk: int = 64) -> np.ndarray:
    """series.py:127-139: (q, b) matrix, direct form, chunked over queries."""
    Q = np.atleast_2d(np.asarray(queries, dtype=np.float64))
    B = np.atleast_2d(np.asarray(block, dtype=np.float64))
    out = np.empty((Q.shape[0], B.shape[0]))
    for s in range(0, Q.shape[0], chunk):
        d = Q[s:s + chunk, None, :] - B[None]
        out[s:s + chunk] = np.einsum("qbm,qbm->qb", d, d)
    return np.sqrt(out)


# ---------------------------------------------------------------------------
# the tree (tree.py:125-189)
# ---------------------------------------------------------------------------

@dataclass
class OracleTree:
    """Flat node table of the reference tree; node ids are list positions."""

    values: np.ndarray            # (n, m) fp64, fp32-exact
    starts: np.ndarray
    widths: np.ndarray
    max_leaf_size: int
    env_min: list = field(default_factory=list)
    env_max: list = field(default_factory=list)
    left: list = field(default_factory=list)
    right: list = field(default_factory=list)
    split_seg: list = field(default_factory=list)
    split_thr: list = field(default_factory=list)
    member_lists: list = field(default_factory=list)   # list[int] or None (internal)
    size: list = field(default_factory=list)
    oversized: list = field(default_factory=list)
    members: dict = field(default_factory=dict)        # leaf id -> int64 ids (after freeze)

    @property
    def n_nodes(self) -> int:
        return len(self.left)

    def is_leaf(self, nid: int) -> bool:
        return self.member_lists[nid] is not None

    @property
    def leaf_ids(self) -> list:
        return [i for i in range(self.n_nodes) if self.is_leaf(i)]

    def _new_node(self, l: int) -> int:
        self.env_min.append(np.full(l, math.inf))
        self.env_max.append(np.full(l, -math.inf))
        self.left.append(-1)
        self.right.append(-1)
        self.split_seg.append(-1)
        self.split_thr.append(math.nan)
        self.member_lists.append([])
        self.size.append(0)
        self.oversized.append(False)
        return len(self.left) - 1

    def freeze(self) -> "OracleTree":
        self.members = {
            i: np.asarray(self.member_lists[i], dtype=np.int64) for i in self.leaf_ids
        }
        return self


def _split(t: OracleTree, nid: int, summs: np.ndarray) -> None:
    """tree.py:125-161: widest-envelope segment, split at the member median."""
    width = t.env_max[nid] - t.env_min[nid]
    seg = int(np.argmax(width))
    if not width[seg] > 0.0:
        t.oversized[nid] = True
        return
    ids = np.asarray(t.member_lists[nid], dtype=np.int64)
    col = summs[ids, seg]
    thr = float(np.median(col))
    go_left = col <= thr
    if go_left.all() or not go_left.any():
        thr = float((col.min() + col.max()) / 2.0)
        go_left = col <= thr
        if go_left.all() or not go_left.any():
            t.oversized[nid] = True
            return
    l = width.shape[0]
    a = t._new_node(l)
    b = t._new_node(l)
    for child, mask in ((a, go_left), (b, ~go_left)):
        sel = ids[mask]
        t.member_lists[child] = [int(i) for i in sel]
        t.size[child] = int(sel.shape[0])
        t.env_min[child] = summs[sel].min(axis=0)
        t.env_max[child] = summs[sel].max(axis=0)
    t.member_lists[nid] = None
    t.split_seg[nid] = seg
    t.split_thr[nid] = thr
    t.left[nid] = a
    t.right[nid] = b


def build_tree(values: np.ndarray, max_leaf_size: int = 1000, segments: int = 8) -> OracleTree:
    """tree.py:164-189: insert rows in id order, split on overflow."""
    if max_leaf_size < 2:
        raise ValueError("max_leaf_size must be >= 2")
    values = np.ascontiguousarray(values, dtype=np.float64)
    starts, widths = seg_layout(values.shape[1], segments)
    summs = paa(values, starts, widths)
    t = OracleTree(values, starts, widths, max_leaf_size)
    t._new_node(segments)
    for sid in range(values.shape[0]):
        s = summs[sid]
        nid = 0
        while t.member_lists[nid] is None:
            t.size[nid] += 1
            np.minimum(t.env_min[nid], s, out=t.env_min[nid])
            np.maximum(t.env_max[nid], s, out=t.env_max[nid])
            nid = t.left[nid] if s[t.split_seg[nid]] <= t.split_thr[nid] else t.right[nid]
        t.member_lists[nid].append(sid)
        t.size[nid] += 1
        np.minimum(t.env_min[nid], s, out=t.env_min[nid])
        np.maximum(t.env_max[nid], s, out=t.env_max[nid])
        if t.size[nid] > max_leaf_size:
            _split(t, nid, summs)
    return t.freeze()


def tree_from_reference(index) -> OracleTree:
    """Adopt a reference `tree.Index` (tests only, when the reference is importable)."""
    cfg = index.cfg
    t = OracleTree(np.asarray(index.dataset.values), np.asarray(cfg.starts), np.asarray(cfg.widths),
                   index.max_leaf_size)
    for nd in index.nodes:
        t.env_min.append(np.array(nd.envelope.mean_min))
        t.env_max.append(np.array(nd.envelope.mean_max))
        t.left.append(-1 if nd.left is None else nd.left.node_id)
        t.right.append(-1 if nd.right is None else nd.right.node_id)
        t.split_seg.append(-1 if nd.split_segment is None else nd.split_segment)
        t.split_thr.append(math.nan if nd.split_threshold is None else nd.split_threshold)
        t.member_lists.append(None if nd.members is None else list(nd.members))
        t.size.append(nd.size)
        t.oversized.append(nd.oversized)
    return t.freeze()


# ---------------------------------------------------------------------------
# search (tree.py:192-315)
# ---------------------------------------------------------------------------

class KBest:
    """tree.py:192-217: k smallest (distance, id); ties rank by smaller id."""

    def __init__(self, k: int):
        self.k = k
        self.d = np.empty(0)
        self.i = np.empty(0, dtype=np.int64)

    @property
    def bsf(self) -> float:
        return float(self.d[-1]) if self.d.shape[0] == self.k else math.inf

    def offer(self, d: np.ndarray, ids: np.ndarray) -> None:
        keep = d <= self.bsf
        if not keep.any():
            return
        dd = np.concatenate((self.d, d[keep]))
        ii = np.concatenate((self.i, ids[keep]))
        o = np.lexsort((ii, dd))[: self.k]
        self.d, self.i = dd[o], ii[o]

    def results(self) -> list:
        return [(int(a), float(b)) for a, b in zip(self.i, self.d)]


STAT_KEYS = (
    "leaves_visited",
    "leaves_searched",
    "leaves_lb_pruned",
    "leaves_filter_pruned",
    "filter_inferences",
    "series_scanned",
)


@dataclass
class OracleOutcome:
    results: list
    stats: dict
    trace: list | None = None   # (leaf_id, lb, searched, leaf_nn or None, bsf_before)


def search(t: OracleTree, q, k: int = 1, bsf_factor: float = 1.0, predictors=None,
           offsets=None, want_trace: bool = False, eapca_env=None) -> OracleOutcome:
    """tree.py:220-297: best-first traversal, cascade lb -> filter -> scan.
    eapca_env=(sd_min, sd_max) (eapca_envelopes): the EAPCA bound replaces the
    reference's mean-only bound (same traversal, unpinned extension)."""
    q = np.ascontiguousarray(q, dtype=np.float64)
    if q.ndim != 1 or q.shape[0] != t.values.shape[1]:
        raise ValueError("query length mismatch")
    if not 1 <= k <= t.values.shape[0]:
        raise ValueError("k out of range")
    predictors = predictors or {}
    offsets = offsets or {}
    if any(lid not in offsets for lid in predictors):
        raise ValueError("missing offsets")
    qs = paa(q, t.starts, t.widths)
    if eapca_env is not None:
        qmu, qsd = eapca(q, t.starts, t.widths)

        def bound(nid):
            return node_lb_eapca(qmu, qsd, t.env_min[nid], t.env_max[nid], eapca_env[0][nid], eapca_env[1][nid],
                                 t.widths)
    else:
        def bound(nid):
            return node_lb(qs, t.env_min[nid], t.env_max[nid], t.widths)
    best = KBest(k)
    st = dict.fromkeys(STAT_KEYS, 0)
    trace = [] if want_trace else None
    heap = [(bound(0), 0)]
    while heap:
        lb, nid = heapq.heappop(heap)
        bsf = best.bsf
        leaf = t.is_leaf(nid)
        if lb > bsf * bsf_factor:
            if leaf:
                st["leaves_visited"] += 1
                st["leaves_lb_pruned"] += 1
                if want_trace:
                    trace.append((nid, lb, False, None, bsf))
            break
        if not leaf:
            for c in (t.left[nid], t.right[nid]):
                heapq.heappush(heap, (bound(c), c))
            continue
        st["leaves_visited"] += 1
        f = predictors.get(nid)
        if f is not None:
            st["filter_inferences"] += 1
            if float(f(q)) - offsets[nid] > bsf * bsf_factor:
                st["leaves_filter_pruned"] += 1
                if want_trace:
                    trace.append((nid, lb, False, None, bsf))
                continue
        ids = t.members[nid]
        d = row_dist(q, t.values[ids])
        st["leaves_searched"] += 1
        st["series_scanned"] += int(ids.shape[0])
        if want_trace:
            trace.append((nid, lb, True, float(d.min()), bsf))
        best.offer(d, ids)
    return OracleOutcome(best.results(), st, trace)


def linear_scan(values: np.ndarray, q, k: int = 1) -> list:
    """tree.py:310-315: brute-force top-k by (distance, id)."""
    d = row_dist(np.asarray(q, dtype=np.float64), values)
    o = np.lexsort((np.arange(values.shape[0]), d))[:k]
    return [(int(i), float(d[i])) for i in o]


def pruning_ratio(stats: dict, n: int) -> float:
    """tree.py:305-307."""
    return 1.0 - stats["series_scanned"] / n


def recall_at_1(result: list, oracle_id: int, oracle_dist: float) -> float:
    """cli.py:83-88."""
    rid, rd = result[0]
    if rid == oracle_id:
        return 1.0
    return 1.0 if abs(rd - oracle_dist) <= RECALL_REL_TOL * max(oracle_dist, 1e-300) else 0.0


# ---------------------------------------------------------------------------
# filters (mlp.py:90-95)
# ---------------------------------------------------------------------------

def mlp_forward(W1, b1, W2, b2, x) -> float:
    """mlp.py:90-95: fp32 y = b2 + W2 . relu(x W1 + b1)."""
    W1 = np.asarray(W1, dtype=np.float32)
    x = np.asarray(x, dtype=np.float32)
    h = np.maximum(x @ W1 + np.asarray(b1, dtype=np.float32), 0)
    return float(h @ np.asarray(W2, dtype=np.float32) + np.float32(b2))


# ---------------------------------------------------------------------------
# training-data generation (traingen.py:135-220)
# ---------------------------------------------------------------------------

def local_targets(t: OracleTree, leaf_id: int, queries: np.ndarray) -> tuple:
    """traingen.py:135-144: (leaf-wise NN distance, lb vs own envelope)."""
    tg = pair_dist(queries, t.values[t.members[leaf_id]]).min(axis=1)
    qs = paa(queries, t.starts, t.widths)
    lbs = lb_matrix(qs, t.env_min[leaf_id][None], t.env_max[leaf_id][None], t.widths)[:, 0]
    return tg, lbs


@dataclass
class OracleTargets:
    selected: list
    dl_selected: np.ndarray
    nn_distance: np.ndarray
    leaf_ids: np.ndarray
    lb_matrix: np.ndarray
    visit_order: np.ndarray
    calibration_count: int
    dl_calib_full: np.ndarray


def collect_targets(t: OracleTree, selected, queries: np.ndarray, calibration_count: int) -> OracleTargets:
    """traingen.py:147-220: pass 1 (selected x all queries, all x calib tail), pass 2 walk."""
    Q = np.atleast_2d(np.asarray(queries, dtype=np.float64))
    nq = Q.shape[0]
    if not 1 <= calibration_count < nq:
        raise ValueError("calibration_count must be in [1, n_queries)")
    sel = sorted(int(s) for s in selected)
    leaf_ids = np.asarray(t.leaf_ids, dtype=np.int64)
    if set(sel) - set(int(i) for i in leaf_ids):
        raise ValueError("unknown leaf ids")
    qs = paa(Q, t.starts, t.widths)
    mins = np.stack([t.env_min[i] for i in leaf_ids])
    maxs = np.stack([t.env_max[i] for i in leaf_ids])
    lbm = lb_matrix(qs, mins, maxs, t.widths)
    order = np.argsort(lbm, axis=1, kind="stable").astype(np.int32)
    dsel = np.empty((nq, len(sel)))
    for c, lid in enumerate(sel):
        dsel[:, c] = pair_dist(Q, t.values[t.members[lid]]).min(axis=1)
    c0 = nq - calibration_count
    dcal = np.empty((calibration_count, leaf_ids.shape[0]))
    col_of = {lid: c for c, lid in enumerate(sel)}
    for p, lid in enumerate(leaf_ids):
        lid = int(lid)
        if lid in col_of:
            dcal[:, p] = dsel[c0:, col_of[lid]]
        else:
            dcal[:, p] = pair_dist(Q[c0:], t.values[t.members[lid]]).min(axis=1)
    nn = np.empty(nq)
    nn[c0:] = dcal.min(axis=1)
    pos_col = {p: col_of[int(l)] for p, l in enumerate(leaf_ids) if int(l) in col_of}
    for qi in range(c0):
        bsf = float(dsel[qi].min()) if sel else math.inf
        for p in order[qi]:
            p = int(p)
            if lbm[qi, p] >= bsf:
                break
            c = pos_col.get(p)
            d = (float(dsel[qi, c]) if c is not None
                 else float(pair_dist(Q[qi:qi + 1], t.values[t.members[int(leaf_ids[p])]]).min()))
            bsf = min(bsf, d)
        nn[qi] = bsf
    return OracleTargets(sel, dsel, nn, leaf_ids, lbm, order, calibration_count, dcal)


# ---------------------------------------------------------------------------
# conformal calibration (conformal.py) and selection (select.py)
# ---------------------------------------------------------------------------

def alphas_desc(pred, target) -> np.ndarray:
    """conformal.py:25-31."""
    return np.sort(np.abs(np.asarray(target, float) - np.asarray(pred, float)))[::-1].copy()


def replay(lb_v, dl_v, pred_v, slot_v, offsets) -> np.ndarray:
    """conformal.py:171-198 over visit-ordered (c, L) matrices; returns achieved bsf."""
    off = np.asarray(offsets, dtype=np.float64)
    offm = np.where(slot_v >= 0, off[np.maximum(slot_v, 0)] if off.size else 0.0, 0.0)
    bsf = np.full(lb_v.shape[0], math.inf)
    for p in range(lb_v.shape[1]):
        alive = lb_v[:, p] <= bsf
        if not alive.any():
            break
        pr = pred_v[:, p]
        filt = alive & ~np.isnan(pr) & (pr - offm[:, p] > bsf)
        np.minimum(bsf, np.where(alive & ~filt, dl_v[:, p], math.inf), out=bsf)
    return bsf


def select_threshold(t_series: float, t_filter: float, a: float) -> int:
    """select.py:100-102."""
    return math.ceil(a * t_filter / t_series)


def select_leaves(leaf_sizes, threshold: int, capacity: int, filter_bytes: int) -> list:
    """select.py:113-131: largest first (ties: smaller id), size >= th, within budget."""
    out, used = [], 0
    for lid, sz in sorted(leaf_sizes, key=lambda p: (-p[1], p[0])):
        if sz < threshold or used + filter_bytes > capacity:
            break
        out.append(lid)
        used += filter_bytes
    return out
