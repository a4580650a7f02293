"""LeaFi enhancement and filtered search (the reference's enhanced.py seam).

``enhance(index, plan, budget, seed, ...) -> EnhancedIndex`` follows the
reference stages (enhanced.py:189-313) with the GPU doing the heavy ones:

  select          threshold + greedy selection (select.py:100-131), host
  global-queries  numpy stream identical to the reference (traingen.py:110-117)
  collect-targets lf_bounds + lf_leaf_min_dist (targets.collect_targets)
  local-queries   numpy streams per leaf, ONE lf_local_min_dist launch
  train-filters   all filters batched on the GPU (training.train_filters)
  fit-tuners      calibration predictions from lf_filter_predict -- the same
                  kernel as search (F6) -- then the replay/curve fit
                  (calibration.fit_auto_tuners)

``search(eidx, SearchRequest)`` is the single-query drop-in (enhanced.py:137-144,
exact reference semantics); ``search_queries`` is the batched product path
(one filter launch + one lf_search per batch).  A reference EnhancedIndex can
be passed to both: its filters are packed onto the GPU and its curves used.
"""

from __future__ import annotations

import logging
import os
import math
import time
from dataclasses import dataclass, field

import warnings
import weakref

import numpy as np

from . import _lib
from .calibration import DeviceReplay, build_skeleton, compute_alphas, fit_auto_tuners, tune
from .engine import BatchResult, SearchOutcome, as_tree, search_batch
from .filters import FilterPack
from .synth import generate_global_queries, generate_local_queries
from .targets import collect_targets, local_targets_all
from .training import TrainConfig, TrainingDivergedError, init_weights, train_filters

log = logging.getLogger(__name__)
FILTER_OVERHEAD_BYTES = 64          # select.py:17


class EnhanceError(RuntimeError):
    """enhanced.py:58-63: a stage failed; carries the stage name."""

    def __init__(self, stage: str, cause: BaseException):
        super().__init__(f"enhancement stage '{stage}' failed: {cause}")
        self.stage = stage


def derive_seed(master: int, tag: int) -> int:
    """enhanced.py:66-67."""
    return (master * 1_000_003 + tag) % (2**31 - 1)


@dataclass(frozen=True)
class SplitPlan:
    """traingen.py:26-46."""

    n_global: int = 1500
    n_local: int = 500
    calibration: int = 300

    def __post_init__(self):
        if self.n_global < 1 or self.n_local < 0 or self.calibration < 1:
            raise ValueError("plan counts must be positive")
        if self.calibration >= self.n_global:
            raise ValueError("calibration must be smaller than the global pool")


@dataclass(frozen=True)
class RuntimeConstants:
    """select.py:31-39."""

    t_series: float
    t_filter: float
    filter_bytes: int

    def __post_init__(self):
        if not (self.t_series > 0 and self.t_filter > 0 and self.filter_bytes > 0):
            raise ValueError("runtime constants must be strictly positive")


@dataclass(frozen=True)
class SelectionBudget:
    """select.py:42-51."""

    capacity_bytes: int
    a: float = 2.0

    def __post_init__(self):
        if self.capacity_bytes < 0:
            raise ValueError("capacity must be >= 0")
        if self.a < 1:
            raise ValueError("a must be >= 1")


def filter_memory_bytes(m: int) -> int:
    """select.py:54-55 with mlp.weight_byte_size (mlp.py:257-259)."""
    return 4 * (m * m + 2 * m + 1) + FILTER_OVERHEAD_BYTES


def compute_threshold(constants: RuntimeConstants, a: float) -> int:
    """select.py:100-102."""
    return math.ceil(a * constants.t_filter / constants.t_series)


def select_greedy(leaves, threshold: int, budget: SelectionBudget, filter_bytes: int) -> list:
    """select.py:113-131: largest first (ties by id), size >= threshold, within budget."""
    if filter_bytes <= 0:
        raise ValueError("filter_bytes must be positive")
    chosen, used = [], 0
    for lid, size in sorted(leaves, key=lambda it: (-it[1], it[0])):
        if size < threshold or used + filter_bytes > budget.capacity_bytes:
            break
        chosen.append(lid)
        used += filter_bytes
    return chosen


@dataclass(frozen=True)
class SearchRequest:
    """enhanced.py:70-84."""

    query: object
    k: int = 1
    target: float | None = None
    exact: bool = False

    def __post_init__(self):
        if self.k < 1:
            raise ValueError("k must be >= 1")
        if not self.exact:
            if self.target is None:
                raise ValueError("request needs a recall target or the exact flag")
            if not 0.0 <= self.target <= 1.0:
                raise ValueError(f"target must be in [0, 1], got {self.target}")


@dataclass
class FilterModel:
    """One filter's parameters (the fields of mlp.MlpModel)."""

    W1: np.ndarray
    b1: np.ndarray
    W2: np.ndarray
    b2: float


class EnhancedIndex:
    """enhanced.py:87-134: base index + filters + curves, with a device filter pack."""

    def __init__(self, base, filters: dict, curves: dict, plan: SplitPlan | None = None,
                 budget: SelectionBudget | None = None, constants: RuntimeConstants | None = None,
                 selection: dict | None = None, train_reports: dict | None = None, pack: FilterPack | None = None):
        self.base = as_tree(base)
        leaf_set = set(int(l) for l in self.base.leaf_ids)
        for lid in filters:
            if lid not in leaf_set:
                raise ValueError(f"filter leaf {lid} does not exist in the index")
            if lid not in curves:
                raise ValueError(f"filter leaf {lid} has no fitted curve")
        self.filters = dict(sorted(filters.items()))
        self.curves = curves
        self.plan, self.budget, self.constants = plan, budget, constants
        self.selection = selection or {}
        self.train_reports = train_reports or {}
        self._pack = pack
        self._offset_cache = {}
        self._offset_vec_cache = {}

    @classmethod
    def adopt(cls, ref_eidx) -> "EnhancedIndex":
        """Wrap a reference enhanced.EnhancedIndex (duck-typed).

        The reference's conformal curves were fitted on its numpy fp32 forward;
        searches here predict with the tensor-core pack, so the calibration rule
        "calibrate on the search's own predictor" (enhanced.py:280-283) holds only
        approximately for an adopted index.  Re-run enhance() on the adopted base
        index for a guaranteed recall target."""
        warnings.warn("adopted reference EnhancedIndex: its curves were calibrated on the numpy forward, "
                      "the GPU search predicts on the tensor-core pack -- the recall target is approximate "
                      "(re-run pipeline.enhance for a calibrated index)", RuntimeWarning, stacklevel=2)
        filters = {int(l): FilterModel(np.asarray(m.W1), np.asarray(m.b1), np.asarray(m.W2), float(m.b2))
                   for l, m in ref_eidx.filters.items()}
        return cls(ref_eidx.base, filters, dict(ref_eidx.curves), ref_eidx.plan, ref_eidx.budget,
                   ref_eidx.constants, ref_eidx.selection, ref_eidx.train_reports)

    @property
    def filter_leaf_ids(self) -> list:
        return list(self.filters)

    @property
    def pack(self) -> FilterPack:
        if self._pack is None:
            self._pack = FilterPack.from_models(self.filters)
        return self._pack

    def tuned_offsets(self, target: float) -> dict:
        """Per-filter offsets, memoised on the exact target (enhanced.py:127-134)."""
        key = float(target)
        got = self._offset_cache.get(key)
        if got is None:
            got = tune(self.curves, key)
            self._offset_cache[key] = got
        return got

    def offset_vector(self, target: float, device: bool = False):
        """Offsets in filter-pack order (host fp64, or a cached device tensor)."""
        key = (float(target), bool(device))
        got = self._offset_vec_cache.get(key)
        if got is None:
            offs = self.tuned_offsets(target)
            got = np.array([offs[l] for l in self.pack.leaf_ids], dtype=np.float64)
            if device:
                import torch
                got = torch.from_numpy(got).to(self.pack.device)
            self._offset_vec_cache[key] = got
        return got


_adopted_eidx = weakref.WeakKeyDictionary()   # reference EnhancedIndex -> wrapper (dies with it)


def _as_enhanced(eidx) -> EnhancedIndex:
    if isinstance(eidx, EnhancedIndex):
        return eidx
    try:
        got = _adopted_eidx.get(eidx)
    except TypeError:                             # not weak-referenceable: adopt per call
        return EnhancedIndex.adopt(eidx)
    if got is None:
        got = EnhancedIndex.adopt(eidx)
        _adopted_eidx[eidx] = got
    return got


def _plan_for(e, Q: int, k: int, target: float, sequential: bool, max_round_leaves: int, stream=None):
    """The cached graph plan of (batch size, k, target, schedule) on e's device."""
    di = e.base.device()
    plans = e.__dict__.setdefault("_plans", {})
    key = (int(Q), int(k), float(target), bool(sequential), int(max_round_leaves), str(di.device))
    plan = plans.get(key)
    if plan is None:
        from .engine import SearchPlan

        pk = e.pack
        plan = SearchPlan(e.base, Q, k, filters=pk, offsets=e.offset_vector(target, device=True),
                          leaf_filter=pk.leaf_filter(di), sequential=sequential,
                          max_round_leaves=max_round_leaves, stream=stream)
        plans[key] = plan
    return plan


class SearchPipeline:
    """Serving form of `search_queries` (in-search inference, graph plan): batches
    submitted back to back overlap their copies with the search of the batch before,
    and their searches with each other: consecutive batches alternate between `plans`
    independent graph plans (own scratch and counters; default one per slot) on their
    own compute streams, so one batch's latency-bound phases (bounds, visit orders,
    planning, tails) run under another's memory-bound scans (bench workload, 20
    batches: 1 plan 1.43 ms per batch, 2 plans 1.21, 3 plans 1.18, 4 plans 1.17;
    `tools/conc_probe.py`).  Each batch's queries go
    host -> device on one copy stream, the results come back device -> host on another;
    `depth` slots of device queries, device results and pinned host results rotate.
    Results and counters equal `search_queries`' for the same batch.

        pipe = SearchPipeline(eidx, batch=1000, k=1, target=0.99)
        t = pipe.submit(q0)              # pinned host tensors overlap best
        for q in rest:
            t_next = pipe.submit(q)
            res = pipe.result(t)         # BatchResult of the earlier batch
            t = t_next
        res = pipe.result(t)

    At most `depth` batches are in flight: a slot's result must be collected before the
    slot is submitted again.  The caller keeps a submitted host tensor unchanged until
    its result is collected."""

    def __init__(self, eidx, batch: int, k: int = 1, *, target: float, depth: int = 3, plans: int | None = None,
                 sequential: bool = False, max_round_leaves: int = 256):
        torch = _lib.require_cuda()
        e = _as_enhanced(eidx)
        if not e.filters or e.pack.path != "tc16":
            raise ValueError("SearchPipeline needs an enhanced index with the fp16 filter pack (path 'tc16')")
        if not 0.0 <= target <= 1.0:
            raise ValueError(f"target must be in [0, 1], got {target}")
        if depth < 1:
            raise ValueError(f"depth must be >= 1, got {depth}")
        plans = depth if plans is None else int(plans)
        if not 1 <= plans <= depth:
            raise ValueError(f"plans must be in [1, depth], got {plans}")
        di = e.base.device()
        dev = di.device
        self.n_series, self.batch, self.k, self.depth = e.base.n, int(batch), int(k), int(depth)
        from .engine import SearchPlan

        # private plans (not search_queries' cached one): a search_queries call on another
        # stream never shares scratch with a batch in flight here
        self._plans = [
            SearchPlan(e.base, self.batch, self.k, filters=e.pack, offsets=e.offset_vector(float(target), device=True),
                       leaf_filter=e.pack.leaf_filter(di), sequential=sequential, max_round_leaves=max_round_leaves)
            for _ in range(plans)]
        m = e.base.m
        with torch.cuda.device(dev):
            self._comps = [torch.cuda.Stream(dev) for _ in range(plans)]
            self._h2d, self._d2h = (torch.cuda.Stream(dev) for _ in range(2))
            self._qd = [torch.empty((self.batch, m), dtype=torch.float32, device=dev) for _ in range(depth)]
            self._out = [(torch.empty((self.batch, self.k), dtype=torch.int64, device=dev),
                          torch.empty((self.batch, self.k), dtype=torch.float64, device=dev),
                          torch.empty((self.batch, _lib.N_STATS), dtype=torch.int64, device=dev))
                         for _ in range(depth)]
            self._host = [tuple(torch.empty(x.shape, dtype=x.dtype, pin_memory=True) for x in o) for o in self._out]
            self._ev = [[torch.cuda.Event() for _ in range(3)] for _ in range(depth)]   # h2d, search, d2h
        self._qh = [None] * depth
        self._slot_ticket = [None] * depth
        self._pending = {}
        self._n = 0

    def submit(self, queries) -> int:
        """Enqueue one batch ([batch, m] fp32: a pinned host tensor, any host array, or a
        device tensor); returns its ticket."""
        torch = _lib.require_cuda()
        i = self._n % self.depth
        if self._slot_ticket[i] is not None and self._slot_ticket[i] in self._pending:
            raise RuntimeError(f"collect result({self._slot_ticket[i]}) before submitting more than "
                               f"{self.depth} batches")
        q = queries if isinstance(queries, torch.Tensor) else torch.from_numpy(
            np.ascontiguousarray(np.atleast_2d(queries), dtype=np.float32))
        if tuple(q.shape) != (self.batch, self._qd[i].shape[1]):
            raise ValueError(f"batch of shape {tuple(q.shape)}, pipeline built for {(self.batch, self._qd[i].shape[1])}")
        ev_h2d, ev_run, ev_d2h = self._ev[i]
        reuse = self._n >= self.depth
        j = self._n % len(self._plans)                   # this batch's plan and compute stream
        comp = self._comps[j]
        with torch.cuda.stream(self._h2d):
            if reuse:
                self._h2d.wait_event(ev_run)             # the slot's previous search read its queries
            self._qd[i].copy_(q.to(torch.float32), non_blocking=True)
            ev_h2d.record(self._h2d)
        self._qh[i] = q
        comp.wait_event(ev_h2d)
        if reuse:
            comp.wait_event(ev_d2h)                      # the slot's previous results left the device
        self._plans[j].run(self._qd[i], stream=comp, copy_out=False, outputs=self._out[i])
        ev_run.record(comp)
        self._d2h.wait_event(ev_run)
        with torch.cuda.stream(self._d2h):
            for h, x in zip(self._host[i], self._out[i]):
                h.copy_(x, non_blocking=True)
            ev_d2h.record(self._d2h)
        t = self._n
        self._pending[t] = i
        self._slot_ticket[i] = t
        self._n += 1
        return t

    def run_resident(self, queries, steps: int, stream=None):
        """`steps` batches of the same device-resident queries ([batch, m] fp32 on the
        index's device) through the alternating plans, no host copies: the caller's
        stream forks to the compute streams and joins them again, so events recorded on
        it around the call time the whole job (device-timed throughput).  Not to be
        interleaved with pending submit() batches.  Returns the last batch's device
        (ids, dists, stats)."""
        torch = _lib.require_cuda()
        if self._pending:
            raise RuntimeError("collect the submitted batches before run_resident")
        dev = self._qd[0].device
        main = stream if stream is not None else torch.cuda.current_stream(dev)
        fork = torch.cuda.Event()
        fork.record(main)
        for c in self._comps:
            c.wait_event(fork)
        last = None
        for n in range(int(steps)):
            j = n % len(self._plans)
            last = self._out[j]
            self._plans[j].run(queries, stream=self._comps[j], copy_out=False, outputs=last)
        for c in self._comps:
            e = torch.cuda.Event()
            e.record(c)
            main.wait_event(e)
        return last

    def result(self, ticket: int) -> BatchResult:
        """Wait for a submitted batch and return its BatchResult (host arrays)."""
        if ticket not in self._pending:
            raise KeyError(f"no pending batch with ticket {ticket}")
        i = self._pending.pop(ticket)
        self._ev[i][2].synchronize()
        self._qh[i] = None
        return BatchResult(self.n_series, *(h.numpy().copy() for h in self._host[i]))


def search_queries(eidx, queries, k: int = 1, *, target: float | None = None, exact: bool = False,
                   sequential: bool = False, max_round_leaves: int = 256, want_trace: bool = False,
                   stream=None, copy_out: bool = True, profile=None, lazy: bool | None = None,
                   graph: bool = True):
    """Batched LeaFi search in one lf_search call.  lazy=True (default for the fp16
    pack, path "tc16"): the filters are evaluated inside the search, in one tensor-core
    pass right after round 0, only for the (query, leaf) pairs the walk can still reach
    (lb <= bsf0 * f; 0.42M of the 4.1M pairs on the bench workload).  lazy=False: one
    lf_filter_predict over every (query, filter) pair first.  Both give identical
    results and counters (same kernel arithmetic).  graph=True (default; in-search
    inference, no trace / profile): the search runs as a cached CUDA-graph plan
    (engine.SearchPlan, one per (batch size, k, target, schedule)) -- same results,
    no per-call host work beyond one graph launch."""
    e = _as_enhanced(eidx)
    if exact or not e.filters:
        return search_batch(e.base, queries, k, sequential=sequential, max_round_leaves=max_round_leaves,
                            want_trace=want_trace, stream=stream, copy_out=copy_out, profile=profile)
    if target is None or not 0.0 <= target <= 1.0:
        raise ValueError(f"target must be in [0, 1], got {target}")
    torch = _lib.require_cuda()
    di = e.base.device()
    pk = e.pack
    q = queries if isinstance(queries, torch.Tensor) else torch.from_numpy(
        np.ascontiguousarray(np.atleast_2d(queries), dtype=np.float32))
    q = q.to(device=di.device, dtype=torch.float32, non_blocking=True)   # stream-ordered from pinned memory
    if lazy is None:
        lazy = pk.path == "tc16"
    if lazy and pk.path != "tc16":
        raise ValueError("in-search filter inference runs on the fp16 pack (FilterPack path 'tc16')")
    if lazy and graph and profile is None and not want_trace and os.environ.get("LF_SEARCH_GRAPH", "1") != "0":
        plan = _plan_for(e, int(q.shape[0]), k, target, sequential, max_round_leaves, stream)
        return plan.run(q, stream=stream, copy_out=copy_out)
    if lazy:
        return search_batch(e.base, q.contiguous(), k, filters=pk, offsets=e.offset_vector(target, device=True),
                            leaf_filter=pk.leaf_filter(di), sequential=sequential,
                            max_round_leaves=max_round_leaves, want_trace=want_trace, stream=stream,
                            copy_out=copy_out, profile=profile)
    pred = pk.predict(q, stream=stream)
    return search_batch(e.base, q, k, predictions=pred, offsets=e.offset_vector(target, device=True),
                        leaf_filter=pk.leaf_filter(di), sequential=sequential,
                        max_round_leaves=max_round_leaves, want_trace=want_trace, stream=stream,
                        copy_out=copy_out, profile=profile)


def search(eidx, req: SearchRequest) -> SearchOutcome:
    """enhanced.py:137-144 drop-in (reference traversal semantics)."""
    t0 = time.perf_counter()
    res = search_queries(eidx, np.asarray(req.query, dtype=np.float64)[None, :], req.k,
                         target=req.target, exact=req.exact, sequential=True)
    out = res.outcome(0)
    out.stats.wall_time_s = time.perf_counter() - t0
    return out


# --------------------------------------------------------------- enhance ----
def enhance(index, plan: SplitPlan, budget: SelectionBudget, seed: int, *,
            constants: RuntimeConstants | None = None, train_cfg: TrainConfig | None = None,
            noise_range=(0.1, 0.4), record_trajectories: bool = False, timings: dict | None = None,
            shard=None) -> EnhancedIndex:
    """Build filters and auto-tuners over an index (enhanced.py:189-313), GPU stages.

    shard=(rank, world, group): leaf-sharded enhancement (call on every rank).  The
    selection, global queries and calibration are global; training-data generation
    runs on this rank's leaves and all-gathers the columns; each rank trains ONLY the
    filters of its own leaves; the calibration predictions of every rank's filters are
    all-gathered, so every rank fits the same curves.  The returned index holds this
    rank's filters (and every curve)."""
    torch = _lib.require_cuda()
    t = as_tree(index)
    sharded = shard is not None and shard[1] > 1
    if sharded:
        import torch.distributed as dist

        rank, world, group = shard
        di_loc = t.shard(rank, world)
        a_loc, b_loc = di_loc.leaf_range
        own = set(int(l) for l in t.leaf_ids[a_loc:b_loc])
    train_cfg = train_cfg or TrainConfig()
    timings = timings if timings is not None else {}
    stage = "init"
    t_stage = time.perf_counter()

    def begin(name):
        nonlocal stage, t_stage
        now = time.perf_counter()
        timings[stage] = timings.get(stage, 0.0) + now - t_stage
        stage, t_stage = name, now
        log.info("enhancement stage: %s", name)

    try:
        begin("measure")
        if constants is None:
            raise ValueError("inject RuntimeConstants: selection must not depend on wall-clock noise "
                             "(reference tests/conftest.py:11)")
        begin("select")
        threshold = compute_threshold(constants, budget.a)
        selected = sorted(select_greedy(t.leaf_sizes(), threshold, budget, constants.filter_bytes))
        sizes = dict(t.leaf_sizes())
        report = {"t_S": constants.t_series, "t_F": constants.t_filter, "w": constants.filter_bytes,
                  "a": budget.a, "th": threshold, "capacity": budget.capacity_bytes,
                  "selected": [{"leaf_id": l, "size": sizes[l]} for l in selected]}
        if not selected:
            log.warning("selection is empty: search will behave exactly")
            return EnhancedIndex(t, {}, {}, plan, budget, constants, report, {})

        begin("global-queries")
        gq, _ = generate_global_queries(t.values, plan.n_global, noise_range, derive_seed(seed, 2))

        begin("collect-targets")
        gts = collect_targets(t, selected, gq, plan.calibration, train_nn=False,   # only nn[pool:] is read
                              shard=shard)

        begin("local-queries")
        col_of = {lid: c for c, lid in enumerate(selected)}
        mine = [l for l in selected if l in own] if sharded else selected
        local_q = {}
        for lid in mine:
            q, _, _ = generate_local_queries(t, lid, plan.n_local, noise_range, derive_seed(seed, 10_000 + lid))
            local_q[lid] = q
        local = (local_targets_all(t, local_q, dindex=di_loc if sharded else None)
                 if plan.n_local and mine else {l: (np.zeros(0), np.zeros(0)) for l in mine})

        begin("train-filters")
        m, F, pool = t.m, len(mine), gts.train_pool_size
        n_all = pool + plan.n_local
        n_tr = (n_all * 4) // 5
        bank = np.concatenate([gts.queries[:pool]] + [local_q[l] for l in mine]).astype(np.float32)
        tr_idx = np.empty((F, n_tr), np.int64)
        va_idx = np.empty((F, n_all - n_tr), np.int64)
        tr_y = np.empty((F, n_tr))
        va_y = np.empty((F, n_all - n_tr))
        W1 = np.empty((F, m, m), np.float32); b1 = np.empty((F, m), np.float32)
        W2 = np.empty((F, m), np.float32); b2 = np.empty(F, np.float32)
        for s, lid in enumerate(mine):
            rows = np.concatenate([np.arange(pool), pool + s * plan.n_local + np.arange(plan.n_local)])
            y = np.concatenate([gts.dl_selected[:pool, col_of[lid]], local[lid][0]])
            perm = np.random.default_rng(derive_seed(seed, 30_000 + lid)).permutation(n_all)
            tr_idx[s], va_idx[s] = rows[perm[:n_tr]], rows[perm[n_tr:]]
            tr_y[s], va_y[s] = y[perm[:n_tr]], y[perm[n_tr:]]
            W1[s], b1[s], W2[s], b2[s] = init_weights(m, derive_seed(seed, 40_000 + lid))
        dbank = torch.from_numpy(bank).cuda()
        (W1, b1, W2, b2), reps = train_filters(dbank, tr_idx, tr_y, va_idx, va_y, (W1, b1, W2, b2), train_cfg,
                                              seed=derive_seed(seed, 20_000), record_trajectories=record_trajectories)
        filters = {lid: FilterModel(W1[s], b1[s], W2[s], float(b2[s])) for s, lid in enumerate(mine)}
        reports = {lid: reps[s] for s, lid in enumerate(mine)}
        pack = FilterPack(mine, W1, b1, W2, b2, device=di_loc.device if sharded else None)

        begin("fit-tuners")
        calib = gts.queries[pool:]
        cp = pack.predict(calib) if mine else torch.zeros((calib.shape[0], 0), dtype=torch.float32,
                                                          device=di_loc.device)
        if sharded:          # every rank's filters are a contiguous block of `selected`
            widths = [0] * world
            dist.all_gather_object(widths, int(cp.shape[1]), group=group)
            wmax = max(max(widths), 1)
            pad = torch.zeros((cp.shape[0], wmax), dtype=cp.dtype, device=cp.device)
            pad[:, :cp.shape[1]] = cp
            parts = [torch.empty_like(pad) for _ in range(world)]
            dist.all_gather(parts, pad, group=group)
            cp = torch.cat([parts[r][:, :widths[r]] for r in range(world)], dim=1)
        cpred = cp.cpu().numpy().astype(np.float64)      # same kernel as search (F6)
        preds = {lid: cpred[:, s] for s, lid in enumerate(selected)}
        alphas = {lid: compute_alphas(preds[lid], gts.dl_selected[pool:, s]) for s, lid in enumerate(selected)}
        sk = build_skeleton(gts.lb_matrix[pool:], gts.dl_calib_full, gts.visit_order[pool:],
                            gts.nn_distance[pool:], gts.leaf_ids, selected, preds)
        curves = fit_auto_tuners(sk, alphas, replay=DeviceReplay(sk))          # GPU replay, SURVEY §8(f)1
        begin("done")
        e = EnhancedIndex(t, filters, curves, plan, budget, constants, report, reports, pack=pack)
        e.global_set = gts
        return e
    except EnhanceError:
        raise
    except BaseException as exc:
        raise EnhanceError(stage, exc) from exc
