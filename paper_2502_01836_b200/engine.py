"""Batched GPU search behind the reference's search seam.

Reference seam: ``search_engine(index, q, k=1, *, bsf_factor=1.0,
predictors=None, offsets=None, want_trace=False) -> SearchOutcome``
(tree.py:220-297) and its callers ``exact_search`` (tree.py:300-302),
``epsilon_search`` (cli.py:57-65).  The same names, argument meaning,
validation errors (ValueError, tree.py:239-248) and result types are kept
here; the work runs in one ``lf_search`` call (include/leafi_b200.h) per
query batch.

Two schedules:

* ``sequential=True``: one scanned leaf per query per round.  Bit-for-bit the
  reference traversal (same results, counters and trace); used by the
  single-query seam.
* ``sequential=False`` (batch default): rounds of 1, 4, 16, ... leaves per
  query.  Same exact-mode answers; the best-so-far is refreshed
  between rounds only, so a query may scan a few extra leaves (F3).
"""

from __future__ import annotations

import math
import time
import weakref
from dataclasses import dataclass, field

import numpy as np

from . import _lib
from .index import DeviceIndex, TreeIndex

STAT_NAMES = ("leaves_visited", "leaves_searched", "leaves_lb_pruned", "leaves_filter_pruned",
              "filter_inferences", "series_scanned")


@dataclass
class SearchStats:
    """tree.py:65-74."""

    n: int
    leaves_visited: int = 0
    leaves_searched: int = 0
    leaves_lb_pruned: int = 0
    leaves_filter_pruned: int = 0
    filter_inferences: int = 0
    series_scanned: int = 0
    wall_time_s: float = 0.0


@dataclass(frozen=True)
class TraceEntry:
    """tree.py:77-83."""

    leaf_id: int
    lower_bound: float
    searched: bool
    leaf_nn_distance: float | None
    bsf_before: float


@dataclass
class SearchOutcome:
    """tree.py:86-90: results ascending by (distance, id)."""

    results: list
    stats: SearchStats
    trace: list | None = None


def pruning_ratio(stats) -> float:
    """tree.py:305-307."""
    return 1.0 - stats.series_scanned / stats.n


# ----------------------------------------------------------------- index --
_adopted = weakref.WeakKeyDictionary()


def as_tree(index) -> TreeIndex:
    """Accept our TreeIndex, a DeviceIndex, or a reference tree.Index (adopted once)."""
    if isinstance(index, TreeIndex):
        return index
    if isinstance(index, DeviceIndex):
        return index.tree
    try:
        t = _adopted.get(index)
    except TypeError:
        t = None
    if t is None:
        t = TreeIndex.from_reference(index)
        try:
            _adopted[index] = t
        except TypeError:
            pass
    return t


@dataclass
class BatchResult:
    """Device results of one lf_search call, copied to host."""

    n: int
    ids: np.ndarray            # int64 [Q, k], -1 where fewer than k were found
    dists: np.ndarray          # fp64 [Q, k]
    stats: np.ndarray          # int64 [Q, 6] in STAT_NAMES order
    trace: dict | None = None
    wall_time_s: float = 0.0
    extra: dict = field(default_factory=dict)

    def __len__(self) -> int:
        return self.ids.shape[0]

    def results(self, i: int) -> list:
        return [(int(a), float(b)) for a, b in zip(self.ids[i], self.dists[i]) if a >= 0]

    def stats_of(self, i: int) -> SearchStats:
        return SearchStats(self.n, *(int(x) for x in self.stats[i]), wall_time_s=self.wall_time_s)

    def trace_of(self, i: int) -> list | None:
        if self.trace is None:
            return None
        t = self.trace
        n = int(t["len"][i])
        out = []
        for j in range(n):
            nn = float(t["leaf_nn"][i, j])
            out.append(TraceEntry(int(t["leaf"][i, j]), float(t["lb"][i, j]), bool(t["searched"][i, j]),
                                  None if math.isnan(nn) else nn, float(t["bsf"][i, j])))
        return out

    def outcome(self, i: int) -> SearchOutcome:
        return SearchOutcome(self.results(i), self.stats_of(i), self.trace_of(i))

    def pruning_ratios(self) -> np.ndarray:
        return 1.0 - self.stats[:, 5] / self.n


def _queries_device(queries, m: int, dev):
    """fp32 device copy of fp32-exact queries (the reference quantizes, series.py:187)."""
    import torch

    if isinstance(queries, torch.Tensor):
        q = queries.to(device=dev, dtype=torch.float32)
    else:
        q = torch.from_numpy(np.ascontiguousarray(np.atleast_2d(queries), dtype=np.float32)).to(dev)
    if q.ndim != 2 or q.shape[1] != m:
        raise ValueError(f"query length {q.shape[-1]} does not match dataset length {m}")
    return q.contiguous()


def _search_options(t, di, Q: int, k: int, *, bsf_factor: float = 1.0, predictions=None, offsets=None,
                    leaf_filter=None, sequential: bool = False, max_round_leaves: int = 256,
                    want_trace: bool = False, profile=None, early_abandon: bool = True, filters=None):
    """lf_search_opts + lf_index of one batched search, and the tensors they point into."""
    torch = _lib.require_cuda()
    dev = di.device
    if not 1 <= k <= t.n:
        raise ValueError(f"k must be in [1, {t.n}], got {k}")
    opts = _lib.LfSearchOpts()
    opts.k = int(k)
    opts.bsf_factor = float(bsf_factor)
    opts.sequential = 1 if sequential else 0
    opts.max_round_leaves = int(max_round_leaves)
    opts.want_trace = 1 if want_trace else 0
    opts.early_abandon = 1 if early_abandon else 0
    if profile is not None:
        if profile.dtype != np.float64 or profile.shape[0] < _lib.N_PROF:
            raise ValueError("profile must be a float64 array of at least N_PROF entries")
        opts.h_profile = profile.ctypes.data
    keep = []
    if filters is not None:
        if predictions is not None:
            raise ValueError("pass predictions or filters, not both")
        if offsets is None or leaf_filter is None:
            raise ValueError("filters need offsets and a leaf->filter map")
        if filters.path != "tc16":
            raise ValueError("in-search filter inference needs the fp16 tensor-core filter pack (path 'tc16')")
        off = torch.as_tensor(np.asarray(offsets, dtype=np.float64) if not isinstance(offsets, torch.Tensor)
                              else offsets, dtype=torch.float64).to(dev).contiguous()
        lf = leaf_filter.to(device=dev, dtype=torch.int32).contiguous()
        if off.shape[0] != filters.n_filters or lf.shape != (di.n_leaves,):
            raise ValueError("filter / offset / leaf map shapes do not agree")
        keep += [off, lf, filters]
        opts.d_W1T_h, opts.d_wexp = filters.W1T_h.data_ptr(), filters.wexp.data_ptr()
        opts.d_b1 = filters.h_b1.data_ptr()
        opts.d_W2, opts.d_b2 = filters.h_W2.data_ptr(), filters.b2.data_ptr()
        opts.filter_m = filters.mp if filters.mp != filters.m else 0
        opts.d_offset, opts.n_filters = off.data_ptr(), int(off.shape[0])
        ist = di.struct(lf)
    elif predictions is not None:
        if offsets is None or leaf_filter is None:
            raise ValueError("filter predictions need offsets and a leaf->filter map")
        pdt = torch.float64 if predictions.dtype == torch.float64 else torch.float32
        pr = predictions.to(device=dev, dtype=pdt).contiguous()
        off = torch.as_tensor(np.asarray(offsets, dtype=np.float64) if not isinstance(offsets, torch.Tensor)
                              else offsets, dtype=torch.float64).to(dev).contiguous()
        lf = leaf_filter.to(device=dev, dtype=torch.int32).contiguous()
        if pr.shape != (Q, off.shape[0]) or lf.shape != (di.n_leaves,):
            raise ValueError("prediction / offset / leaf map shapes do not agree")
        keep += [pr, off, lf]
        if pdt == torch.float64:
            opts.d_pred_f64 = pr.data_ptr()
        else:
            opts.d_pred = pr.data_ptr()
        opts.d_offset, opts.n_filters = off.data_ptr(), int(off.shape[0])
        ist = di.struct(lf)
    else:
        ist = di.struct(None)
    return opts, ist, keep


class SearchPlan:
    """A batched search captured once as a CUDA graph (lf_search_plan_*) for a fixed
    index, batch size Q, k and filter set; `run` launches it for a new query batch.
    Results and counters equal search_batch's with the same arguments.  Predictions
    passed here are fixed for the plan's life (use `filters` -- the fp16 pack, predicted
    inside the search -- for per-batch filtering)."""

    def __init__(self, index, Q: int, k: int = 1, *, stream=None, **kw):
        torch = _lib.require_cuda()
        t = as_tree(index)
        self.di = index if isinstance(index, DeviceIndex) else t.device()
        self.tree, self.Q, self.k = t, int(Q), int(k)
        opts, ist, self._keep = _search_options(t, self.di, self.Q, self.k, **kw)
        self._opts, self._ist = opts, ist
        self._h = None
        with torch.cuda.device(self.di.device):
            h = _lib.lib().lf_search_plan_create(ist, self.Q, opts, _lib.stream_ptr(stream))
        if not h:
            _lib.check(_lib.LF_ECUDA)
        self._h = h

    def run(self, queries, stream=None, copy_out: bool = True, outputs=None):
        """outputs: optional preallocated device (ids [Q, k] int64, dists [Q, k] fp64,
        stats [Q, N_STATS] int64) the results are copied into (copy_out=False returns them)."""
        torch = _lib.require_cuda()
        q = _queries_device(queries, self.tree.m, self.di.device)
        if q.shape[0] != self.Q:
            raise ValueError(f"plan was built for {self.Q} queries, got {q.shape[0]}")
        dev = self.di.device
        if outputs is not None:
            ids, dists, stats = outputs
            if (tuple(ids.shape) != (self.Q, self.k) or tuple(dists.shape) != (self.Q, self.k)
                    or tuple(stats.shape) != (self.Q, _lib.N_STATS) or ids.dtype != torch.int64
                    or dists.dtype != torch.float64 or stats.dtype != torch.int64
                    or not all(x.is_cuda and x.is_contiguous() for x in (ids, dists, stats))):
                raise ValueError("outputs must be contiguous device (int64 [Q, k], fp64 [Q, k], int64 [Q, N_STATS])")
        else:
            ids = torch.empty((self.Q, self.k), dtype=torch.int64, device=dev)
            dists = torch.empty((self.Q, self.k), dtype=torch.float64, device=dev)
            stats = torch.empty((self.Q, _lib.N_STATS), dtype=torch.int64, device=dev)
        with torch.cuda.device(dev):
            _lib.check(_lib.lib().lf_search_plan_run(self._h, q.data_ptr(), ids.data_ptr(), dists.data_ptr(),
                                                     stats.data_ptr(), _lib.stream_ptr(stream)))
        if not copy_out:
            return ids, dists, stats
        # results to pinned host buffers, stream-ordered, one synchronisation for all three
        if getattr(self, "_host", None) is None:
            self._host = tuple(torch.empty(x.shape, dtype=x.dtype, pin_memory=True) for x in (ids, dists, stats))
        st = stream if stream is not None else torch.cuda.current_stream(dev)
        with torch.cuda.stream(st):
            for h, x in zip(self._host, (ids, dists, stats)):
                h.copy_(x, non_blocking=True)
        st.synchronize()
        return BatchResult(self.tree.n, *(h.numpy().copy() for h in self._host))

    def close(self) -> None:
        """Free the graph, its streams and scratch now (also done on garbage collection)."""
        h, self._h = getattr(self, "_h", None), None
        if h:
            _lib.lib().lf_search_plan_free(h)

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass



def search_batch(index, queries, k: int = 1, *, bsf_factor: float = 1.0, predictions=None,
                 offsets=None, leaf_filter=None, sequential: bool = False,
                 max_round_leaves: int = 256, want_trace: bool = False, stream=None,
                 copy_out: bool = True, profile: np.ndarray | None = None, early_abandon: bool = True,
                 filters=None):
    """Search a batch of queries in one lf_search call.

    predictions: device fp32 [Q, F] filter outputs (FilterPack.predict), with
    offsets [F] (fp64) and leaf_filter int32 [n_leaves] (filter slot per leaf
    slot, -1 for unfiltered leaves).
    filters: an fp16 tensor-core FilterPack (path "tc16") INSTEAD of predictions
    (in-search inference: one pass right after round 0 predicts only the (query, leaf)
    pairs the walk can still reach, with the dense kernel's arithmetic, so results and
    counters equal the predictions path bit for bit).
    """
    torch = _lib.require_cuda()
    t = as_tree(index)
    di = index if isinstance(index, DeviceIndex) else t.device()
    dev = di.device
    q = _queries_device(queries, t.m, dev)
    Q = q.shape[0]
    opts, ist, keep = _search_options(t, di, Q, k, bsf_factor=bsf_factor, predictions=predictions,
                                      offsets=offsets, leaf_filter=leaf_filter, sequential=sequential,
                                      max_round_leaves=max_round_leaves, want_trace=want_trace,
                                      profile=profile, early_abandon=early_abandon, filters=filters)
    ids = torch.empty((Q, k), dtype=torch.int64, device=dev)
    dists = torch.empty((Q, k), dtype=torch.float64, device=dev)
    stats = torch.empty((Q, _lib.N_STATS), dtype=torch.int64, device=dev)
    tr = None
    trs = None
    if want_trace:
        L = di.n_leaves
        tr = {
            "len": torch.zeros(Q, dtype=torch.int32, device=dev),
            "leaf": torch.full((Q, L), -1, dtype=torch.int32, device=dev),
            "lb": torch.zeros((Q, L), dtype=torch.float64, device=dev),
            "searched": torch.zeros((Q, L), dtype=torch.int8, device=dev),
            "leaf_nn": torch.full((Q, L), float("nan"), dtype=torch.float64, device=dev),
            "bsf": torch.zeros((Q, L), dtype=torch.float64, device=dev),
        }
        trs = _lib.LfTrace(*(tr[key].data_ptr() for key in ("len", "leaf", "lb", "searched", "leaf_nn", "bsf")))
    t0 = time.perf_counter()
    with torch.cuda.device(dev):
        sp = _lib.stream_ptr(stream)
        _lib.check(_lib.lib().lf_search(ist, q.data_ptr(), Q, opts, ids.data_ptr(), dists.data_ptr(),
                                        stats.data_ptr(), trs, sp))
    if not copy_out:
        return ids, dists, stats
    res = BatchResult(t.n, ids.cpu().numpy(), dists.cpu().numpy(), stats.cpu().numpy(),
                      {key: v.cpu().numpy() for key, v in tr.items()} if tr is not None else None)
    res.wall_time_s = time.perf_counter() - t0
    return res


def _eval_predictors(t: TreeIndex, q: np.ndarray, predictors: dict, offsets: dict):
    """Host callables (reference predictor dict, tests' lambdas) -> one prediction row."""
    import torch

    slots = sorted(predictors)
    di = t.device()
    leaf_filter = torch.full((di.n_leaves,), -1, dtype=torch.int32)
    for s, lid in enumerate(slots):
        j = di.slot_of_leaf.get(int(lid))
        if j is None:
            raise ValueError(f"predictor for unknown leaf {lid}")
        leaf_filter[j] = s
    # fp64: a host callable may return any Python float (tree.py:281 float(predictor(q)))
    pred = torch.tensor([[float(predictors[l](q)) for l in slots]], dtype=torch.float64)
    off = np.array([float(offsets[l]) for l in slots], dtype=np.float64)
    return pred, off, leaf_filter


def search_engine(index, q, k: int = 1, *, bsf_factor: float = 1.0, predictors=None,
                  offsets=None, want_trace: bool = False) -> SearchOutcome:
    """Drop-in for tree.search_engine (tree.py:220-297), exact reference semantics."""
    t0 = time.perf_counter()
    t = as_tree(index)
    qa = np.asarray(q, dtype=np.float64)
    if qa.ndim != 1:
        raise ValueError(f"expected a 1-d series, got shape {qa.shape}")
    if qa.shape[0] != t.m:
        raise ValueError(f"query length {qa.shape[0]} does not match dataset length {t.m}")
    if not 1 <= k <= t.n:
        raise ValueError(f"k must be in [1, {t.n}], got {k}")
    predictors = predictors or {}
    offsets = offsets or {}
    missing = [lid for lid in predictors if lid not in offsets]
    if missing:
        raise ValueError(f"missing offsets for filtered leaves {missing}")
    kw = {}
    if predictors:
        pred, off, lf = _eval_predictors(t, qa, predictors, offsets)
        kw = dict(predictions=pred, offsets=off, leaf_filter=lf)
    res = search_batch(t, qa[None, :], k, bsf_factor=bsf_factor, sequential=True, want_trace=want_trace, **kw)
    out = res.outcome(0)
    out.stats.wall_time_s = time.perf_counter() - t0
    return out


def exact_search(index, q, k: int = 1, want_trace: bool = False) -> SearchOutcome:
    """tree.py:300-302."""
    return search_engine(index, q, k, want_trace=want_trace)


def epsilon_search(index, q, k: int, epsilon: float) -> SearchOutcome:
    """cli.py:57-65: prune when lb > bsf / (1 + eps)."""
    if epsilon < 0:
        raise ValueError(f"epsilon must be >= 0, got {epsilon}")
    return search_engine(index, q, k, bsf_factor=1.0 / (1.0 + epsilon))


def batch_distances(queries, block) -> np.ndarray:
    """series.batch_distances (series.py:127-139) on the GPU, fp64 direct form."""
    torch = _lib.require_cuda()
    qv = np.atleast_2d(np.asarray(queries, dtype=np.float64))
    bv = np.atleast_2d(np.asarray(block, dtype=np.float64))
    if qv.shape[1] != bv.shape[1]:
        raise ValueError("queries and block must have the same series length")
    dq = torch.from_numpy(qv.astype(np.float32)).cuda()
    db = torch.from_numpy(bv.astype(np.float32)).cuda()
    out = torch.empty((qv.shape[0], bv.shape[0]), dtype=torch.float64, device=dq.device)
    _lib.check(_lib.lib().lf_batch_distances(dq.data_ptr(), qv.shape[0], db.data_ptr(), bv.shape[0],
                                             qv.shape[1], out.data_ptr(), _lib.stream_ptr()))
    return out.cpu().numpy()


def linear_scan(index_or_values, q, k: int = 1) -> list:
    """tree.linear_scan (tree.py:310-315): brute-force top-k by (distance, id) on the GPU."""
    vals = index_or_values.values if isinstance(index_or_values, TreeIndex) else np.asarray(
        getattr(index_or_values, "values", index_or_values))
    d = batch_distances(np.asarray(q, dtype=np.float64)[None, :], vals)[0]
    o = np.lexsort((np.arange(d.shape[0]), d))[:k]
    return [(int(i), float(d[i])) for i in o]


def query_bounds(queries, env_min, env_max, starts, widths, mode: int = 0):
    """Segment means and node lower bounds on the GPU (lf_bounds).

    env_min / env_max are [nodes, segments] (reference orientation); mode 0 is
    the search bound (summarize.py:97-107), mode 1 the batched traingen bound
    (summarize.py:114-122).  Returns (qsumm [Q, segments], lb [Q, nodes]).
    """
    torch = _lib.require_cuda()
    qv = np.atleast_2d(np.asarray(queries, dtype=np.float64))
    mn = np.atleast_2d(np.asarray(env_min, dtype=np.float64))
    mx = np.atleast_2d(np.asarray(env_max, dtype=np.float64))
    nseg = int(len(widths))
    s = _lib.LfIndex()
    s.m = qv.shape[1]
    s.n_seg = nseg
    for i in range(nseg):
        s.seg_start[i] = int(starts[i])
        s.seg_width[i] = int(widths[i])
    dq = torch.from_numpy(qv.astype(np.float32)).cuda()
    dmn = torch.from_numpy(np.ascontiguousarray(mn.T)).cuda()
    dmx = torch.from_numpy(np.ascontiguousarray(mx.T)).cuda()
    qs = torch.empty((qv.shape[0], nseg), dtype=torch.float64, device=dq.device)
    lb = torch.empty((qv.shape[0], mn.shape[0]), dtype=torch.float64, device=dq.device)
    _lib.check(_lib.lib().lf_bounds(dq.data_ptr(), qv.shape[0], s, dmn.data_ptr(), dmx.data_ptr(),
                                    mn.shape[0], mode, qs.data_ptr(), lb.data_ptr(), _lib.stream_ptr()))
    return qs.cpu().numpy(), lb.cpu().numpy()
