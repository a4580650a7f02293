"""Leaf-sharded multi-GPU search: one process per GPU.

Each rank holds a contiguous range of leaves (balanced by series count,
`index.shard_leaf_ranges`), its rows and its filters; queries are
replicated.  Every rank walks the SAME global visit order (bounds cover the
whole tree) but scans only its own leaves.  After every round the ranks
exchange, in ONE collective, the per-query best-so-far (allreduce MIN over
NVLink/NVSwitch with NCCL) together with the "any query still active" flag
(encoded as -active in the same MIN).  The min over ranks of their local
k-th best is >= the global k-th best, so pruning with it stays exact.  At the
end the per-rank top-k lists are all-gathered and merged by (distance, id),
and the counters are summed.

The round loop is written against a small engine protocol so the collective
logic can be tested on CPU with gloo (tests/test_sharded_cpu.py) while the GPU
engine drives lf_search_begin / lf_search_round / lf_search_end.
"""

from __future__ import annotations

import ctypes as C
import math
from dataclasses import dataclass

import numpy as np

from . import _lib


class GpuRoundEngine:
    """lf_search session over one device (leaf shard) index."""

    def __init__(self, dindex, queries, k: int, *, predictions=None, offsets=None, leaf_filter=None,
                 bsf_factor: float = 1.0, max_round_leaves: int = 256, early_abandon: bool = True,
                 stream=None, profile=None, filters=None):
        import torch

        self.torch = torch
        self.di = dindex
        self.device = dindex.device
        self.k = int(k)
        q = queries.to(device=self.device, dtype=torch.float32).contiguous()
        self.Q = q.shape[0]
        self._keep = [q]
        o = _lib.LfSearchOpts()
        o.k = self.k
        o.bsf_factor = float(bsf_factor)
        o.sequential = 0
        o.max_round_leaves = int(max_round_leaves)
        o.early_abandon = 1 if early_abandon else 0
        lf = None
        if filters is not None:                      # in-search inference (fp16 pack)
            if filters.path != "tc16":
                raise ValueError("in-search filter inference needs the fp16 tensor-core filter pack (path 'tc16')")
            off = torch.as_tensor(offsets, dtype=torch.float64).to(self.device).contiguous()
            lf = leaf_filter.to(device=self.device, dtype=torch.int32).contiguous()
            self._keep += [off, lf, filters]
            o.d_W1T_h, o.d_wexp = filters.W1T_h.data_ptr(), filters.wexp.data_ptr()
            o.d_b1 = filters.h_b1.data_ptr()
            o.d_W2, o.d_b2 = filters.h_W2.data_ptr(), filters.b2.data_ptr()
            o.filter_m = filters.mp if filters.mp != filters.m else 0
            o.d_offset = off.data_ptr()
            o.n_filters = int(off.shape[0])
        elif predictions is not None:
            pr = predictions.to(self.device).contiguous()
            off = torch.as_tensor(offsets, dtype=torch.float64).to(self.device).contiguous()
            lf = leaf_filter.to(device=self.device, dtype=torch.int32).contiguous()
            self._keep += [pr, off, lf]
            if pr.dtype == torch.float64:
                o.d_pred_f64 = pr.data_ptr()
            else:
                o.d_pred = pr.data_ptr()
            o.d_offset = off.data_ptr()
            o.n_filters = int(off.shape[0])
        if profile is not None:
            o.h_profile = profile.ctypes.data
        self._opts = o
        self._ist = dindex.struct(lf)
        self.stats = torch.zeros((self.Q, _lib.N_STATS), dtype=torch.int64, device=self.device)
        self.sess = _lib.lib().lf_search_begin(self._ist, q.data_ptr(), self.Q, o, None, self.stats.data_ptr(),
                                               _lib.stream_ptr(stream))
        if not self.sess:
            _lib.check(_lib.LF_ECUDA)
        self.stream = stream

    def round(self, bound, bsf_out) -> int:
        act = C.c_int32(0)
        _lib.check(_lib.lib().lf_search_round(self.sess, bound.data_ptr(), bsf_out.data_ptr(), C.byref(act)))
        return int(act.value)

    @property
    def async_rounds(self) -> bool:
        return True                              # every round decision stays on the device

    def enqueue(self, bound, bsf_out, active_dev) -> None:
        """Enqueue one round without a host sync; its active count lands in active_dev (int32 [1])."""
        _lib.check(_lib.lib().lf_search_round_async(self.sess, bound.data_ptr(), bsf_out.data_ptr(),
                                                    active_dev.data_ptr()))

    def wait(self) -> int:
        """Wait for the oldest enqueued round; its active count."""
        act = C.c_int32(0)
        _lib.check(_lib.lib().lf_search_round_wait(self.sess, C.byref(act)))
        return int(act.value)

    def end(self):
        torch = self.torch
        ids = torch.empty((self.Q, self.k), dtype=torch.int64, device=self.device)
        d = torch.empty((self.Q, self.k), dtype=torch.float64, device=self.device)
        try:
            _lib.check(_lib.lib().lf_search_end(self.sess, ids.data_ptr(), d.data_ptr()))
        finally:
            _lib.lib().lf_search_free(self.sess)
            self.sess = None
        return ids, d, self.stats


def merge_topk(ids, dists, k: int):
    """[Q, W*k] candidates (id -1 = empty) -> k smallest by (distance, id)."""
    import torch

    d = torch.where(ids < 0, torch.full_like(dists, math.inf), dists)
    o1 = torch.argsort(ids, dim=1, stable=True)
    d1 = torch.gather(d, 1, o1)
    o2 = torch.argsort(d1, dim=1, stable=True)
    order = torch.gather(o1, 1, o2)[:, :k]
    return torch.gather(ids, 1, order), torch.gather(d, 1, order)


def run_rounds(engine, group=None, max_rounds: int = 1 << 20) -> tuple:
    """Drive an engine's rounds with one MIN-allreduce per round; returns merged
    (ids [Q,k], dists [Q,k], stats [Q,6]) on every rank, and the round count."""
    import torch
    import torch.distributed as dist

    world = dist.get_world_size(group) if dist.is_initialized() else 1
    if world > 1 and getattr(engine, "async_rounds", False):
        return _run_rounds_pipelined(engine, group, world, max_rounds)
    Q, k, dev = engine.Q, engine.k, engine.device
    buf = torch.full((Q + 1,), math.inf, dtype=torch.float64, device=dev)
    bound = torch.full((Q,), math.inf, dtype=torch.float64, device=dev)
    local = torch.empty((Q,), dtype=torch.float64, device=dev)
    rounds = 0
    while rounds < max_rounds:
        act = engine.round(bound, local)
        rounds += 1
        if world == 1:
            bound.copy_(local)
            if act == 0:
                break
            continue
        buf[:Q].copy_(local)
        buf[Q] = -float(act)
        dist.all_reduce(buf, op=dist.ReduceOp.MIN, group=group)
        bound.copy_(buf[:Q])
        if float(buf[Q]) == 0.0:          # no rank has an active query
            break
    ids, d, stats = engine.end()
    if world > 1:
        gi = [torch.empty_like(ids) for _ in range(world)]
        gd = [torch.empty_like(d) for _ in range(world)]
        dist.all_gather(gi, ids, group=group)
        dist.all_gather(gd, d, group=group)
        ids, d = merge_topk(torch.cat(gi, dim=1), torch.cat(gd, dim=1), k)
        dist.all_reduce(stats, op=dist.ReduceOp.SUM, group=group)
    return ids, d, stats, rounds


def _finish(engine, group, world: int):
    import torch
    import torch.distributed as dist

    ids, d, stats = engine.end()
    gi = [torch.empty_like(ids) for _ in range(world)]
    gd = [torch.empty_like(d) for _ in range(world)]
    dist.all_gather(gi, ids, group=group)
    dist.all_gather(gd, d, group=group)
    ids, d = merge_topk(torch.cat(gi, dim=1), torch.cat(gd, dim=1), engine.k)
    dist.all_reduce(stats, op=dist.ReduceOp.SUM, group=group)
    return ids, d, stats


def _run_rounds_pipelined(engine, group, world: int, max_rounds: int) -> tuple:
    """One round in flight ahead of the host, like lf_search: round r's exchange
    (MIN-allreduce of [bsf..., -active], stream-ordered after the round) and round
    r+1 are enqueued before the host reads round r's global active flag -- ONE
    host synchronisation per round, and the GPU never idles on it.  A round
    enqueued after the last active one finds every query done on every rank."""
    import torch
    import torch.distributed as dist

    Q, dev = engine.Q, engine.device
    buf = torch.full((Q + 1,), math.inf, dtype=torch.float64, device=dev)
    bound = torch.full((Q,), math.inf, dtype=torch.float64, device=dev)
    locs = [torch.empty((Q,), dtype=torch.float64, device=dev) for _ in range(2)]
    acts = [torch.zeros((1,), dtype=torch.int32, device=dev) for _ in range(2)]
    flag = torch.empty((2,), dtype=torch.float64, pin_memory=True)
    evs = [torch.cuda.Event() for _ in range(2)]
    engine.enqueue(bound, locs[0], acts[0])
    inflight, rounds, r = 1, 0, 0
    while True:
        s = r & 1
        buf[:Q].copy_(locs[s])
        buf[Q:].copy_(acts[s].to(torch.float64).neg_())
        dist.all_reduce(buf, op=dist.ReduceOp.MIN, group=group)
        bound.copy_(buf[:Q])
        flag[s:s + 1].copy_(buf[Q:], non_blocking=True)
        evs[s].record()
        rounds += 1
        if rounds < max_rounds:
            engine.enqueue(bound, locs[s ^ 1], acts[s ^ 1])
            inflight += 1
        engine.wait()
        inflight -= 1
        evs[s].synchronize()
        if float(flag[s]) == 0.0 or rounds >= max_rounds:       # no rank has an active query
            break
        r += 1
    while inflight:
        engine.wait()
        inflight -= 1
    ids, d, stats = _finish(engine, group, world)
    return ids, d, stats, rounds


@dataclass
class ShardedResult:
    ids: np.ndarray
    dists: np.ndarray
    stats: np.ndarray
    rounds: int
    n: int

    def pruning_ratios(self) -> np.ndarray:
        return 1.0 - self.stats[:, 5] / self.n


def search_sharded(tree, queries, k: int = 1, *, rank: int, world: int, pack=None, offsets=None,
                   bsf_factor: float = 1.0, max_round_leaves: int = 256, group=None, copy_out: bool = True,
                   profile=None, lazy: bool | None = None):
    """Leaf-sharded batched search on this rank's GPU (call on every rank).

    pack: this rank's FilterPack (its local filters only) with `offsets` in pack
    order; predictions are computed for the local filters only.  lazy (default: when
    the pack is fp16, path "tc16"): in-search inference after round 0 instead of a
    dense pass over every (query, filter) pair; results are identical.
    """
    torch = _lib.require_cuda()
    di = tree.shard(rank, world)
    q = queries if isinstance(queries, torch.Tensor) else torch.from_numpy(
        np.ascontiguousarray(np.atleast_2d(queries), dtype=np.float32))
    q = q.to(device=di.device, dtype=torch.float32).contiguous()
    kw = {}
    if pack is not None and pack.n_filters:
        if lazy is None:
            lazy = pack.path == "tc16"
        if lazy:
            kw = dict(filters=pack, offsets=offsets, leaf_filter=pack.leaf_filter(di))
        else:
            kw = dict(predictions=pack.predict(q), offsets=offsets, leaf_filter=pack.leaf_filter(di))
    eng = GpuRoundEngine(di, q, k, bsf_factor=bsf_factor, max_round_leaves=max_round_leaves, profile=profile, **kw)
    ids, d, stats, rounds = run_rounds(eng, group)
    if not copy_out:
        return ids, d, stats, rounds
    return ShardedResult(ids.cpu().numpy(), d.cpu().numpy(), stats.cpu().numpy(), rounds, tree.n)
