"""Training-data generation on the GPU: exact query x leaf minimum distances.

Mirrors the reference build seam:

* ``collect_targets(index, selected_leaves, queries, calibration_count) ->
  GlobalTrainSet`` (traingen.py:147-220) -- lower-bound matrix (bit-exact,
  lf_bounds mode 1), stable visit order, pass 1 (every selected leaf x every
  query, lf_leaf_min_dist), calibration tail against every leaf, and the
  pass-2 nearest-neighbour walk (break on lb >= bsf, traingen.py:193-208);
* ``collect_local_targets(index, local) -> LocalQueries`` (traingen.py:135-144);
* ``local_targets_all`` -- every selected leaf's local queries in ONE launch
  (the reference loops leaf by leaf, enhanced.py:258-262).
"""

from __future__ import annotations

from dataclasses import dataclass

import numpy as np

from . import _lib
from .engine import as_tree
from .index import shard_leaf_ranges


@dataclass
class GlobalTrainSet:
    """traingen.py:59-97 (same fields, shapes and column conventions)."""

    queries: np.ndarray
    selected_leaves: list
    dl_selected: np.ndarray        # (n_global, n_selected)
    nn_distance: np.ndarray
    leaf_ids: np.ndarray
    lb_matrix: np.ndarray          # (n_global, n_leaves)
    visit_order: np.ndarray        # (n_global, n_leaves) int32 column positions
    calibration_count: int
    dl_calib_full: np.ndarray      # (calibration_count, n_leaves)

    @property
    def n_global(self) -> int:
        return self.queries.shape[0]

    @property
    def train_pool_size(self) -> int:
        return self.n_global - self.calibration_count

    def leaf_column(self, leaf_id: int) -> int:
        pos = int(np.searchsorted(self.leaf_ids, leaf_id))
        if pos >= self.leaf_ids.shape[0] or self.leaf_ids[pos] != leaf_id:
            raise KeyError(f"unknown leaf id {leaf_id}")
        return pos

    def selected_column(self, leaf_id: int) -> int:
        try:
            return self.selected_leaves.index(leaf_id)
        except ValueError:
            raise KeyError(f"leaf {leaf_id} was not selected") from None


@dataclass
class LocalQueries:
    """traingen.py:49-56."""

    leaf_id: int
    queries: np.ndarray
    levels: np.ndarray
    source_ids: np.ndarray
    targets: np.ndarray | None = None
    lbs: np.ndarray | None = None


_QCHUNK = 64 * 65535   # lf_leaf_min_dist query-tile grid limit


def tc_ok(m: int) -> bool:
    """The tensor-core (tcgen05 tf32 + exact fp64 re-check) path covers m in {32, ..., 256}."""
    return m % 32 == 0 and 32 <= m <= 256


def default_path(t, di) -> str:
    """int8 tensor cores over the int8 shadow when it exists (m in {128, 256}), else
    tf32 tensor cores (m in {32, ..., 256}), else fp64 CUDA cores."""
    if getattr(di, "X8", None) is not None and t.m in (128, 256):
        return "q8"
    return "tc" if tc_ok(t.m) else "simt"


def leaf_min_distances(index, queries, leaf_slots, path: str | None = None, dindex=None) -> "torch.Tensor":
    """Device fp64 [Q, S]: exact min distance from each query to each leaf slot.

    path "q8" (default when the int8 shadow exists): lf_leaf_min_dist_q8; "tc":
    lf_leaf_min_dist_tc (tf32); "simt": lf_leaf_min_dist (fp64 CUDA cores).  All
    return the exact fp64 minima (to ~1 ulp: different summation orders).
    dindex: a DeviceIndex (e.g. a leaf shard) whose slots `leaf_slots` refer to."""
    torch = _lib.require_cuda()
    t = as_tree(index)
    di = dindex if dindex is not None else t.device()
    path = path or default_path(t, di)
    q = queries if isinstance(queries, torch.Tensor) else torch.from_numpy(
        np.ascontiguousarray(np.atleast_2d(queries), dtype=np.float32))
    q = q.to(device=di.device, dtype=torch.float32).contiguous()
    sel = torch.as_tensor(np.asarray(leaf_slots, dtype=np.int32)).to(di.device)
    Q, S = q.shape[0], sel.shape[0]
    out = torch.empty((Q, S), dtype=torch.float64, device=di.device)
    st = di.struct(None)
    if path in ("tc", "q8") and Q and S:
        hsel = np.ascontiguousarray(np.asarray(leaf_slots, dtype=np.int32))
        fn = _lib.lib().lf_leaf_min_dist_q8 if path == "q8" else _lib.lib().lf_leaf_min_dist_tc
        _lib.check(fn(q.data_ptr(), Q, st, _lib.ptr(hsel), S, out.data_ptr(), S, _lib.stream_ptr()))
        return out
    for s0 in range(0, S, 65535):
        s1 = min(S, s0 + 65535)
        for q0 in range(0, Q, _QCHUNK):
            q1 = min(Q, q0 + _QCHUNK)
            _lib.check(_lib.lib().lf_leaf_min_dist(
                q[q0:q1].data_ptr(), q1 - q0, st, sel[s0:s1].data_ptr(), s1 - s0,
                out[q0:q1, s0:s1].data_ptr(), S, _lib.stream_ptr()))
    return out


def sharded_leaf_min_distances(index, queries, rank: int, world: int, *, gather: bool = True, group=None,
                               path: str | None = None):
    """Training-data generation sharded like the search: this rank
    computes the min distances to ITS leaf shard only (contiguous leaves balanced by
    series count, queries replicated); with gather=True the columns of every rank are
    all-gathered into the full [Q, n_leaves] matrix (leaf slots in ascending node id).
    Returns (local [Q, L_r], full or None, (a, b) = this rank's leaf-slot range)."""
    torch = _lib.require_cuda()
    import torch.distributed as dist

    t = as_tree(index)
    di = t.shard(rank, world)
    a, b = di.leaf_range
    local = leaf_min_distances(t, queries, list(range(b - a)), path=path, dindex=di)
    if not gather:
        return local, None, (a, b)
    if world == 1:
        return local, local, (a, b)
    sizes = t.size[t.leaf_ids]
    ranges = shard_leaf_ranges(sizes, world)
    width = max(r1 - r0 for r0, r1 in ranges)
    pad = torch.full((local.shape[0], width), float("inf"), dtype=local.dtype, device=local.device)
    pad[:, :b - a] = local
    parts = [torch.empty_like(pad) for _ in range(world)]
    dist.all_gather(parts, pad, group=group)
    full = torch.cat([parts[r][:, :r1 - r0] for r, (r0, r1) in enumerate(ranges)], dim=1)
    return local, full, (a, b)


def leaf_bounds(index, queries, mode: int = 1, dindex=None):
    """(qsumm, lb) of queries against every LEAF envelope, columns in ascending leaf id.
    dindex: the DeviceIndex whose device runs it (a leaf shard is enough: the
    envelopes of every leaf are host data)."""
    torch = _lib.require_cuda()
    t = as_tree(index)
    di = dindex if dindex is not None else t.device()
    leaf_ids = t.leaf_ids
    eapca = t.sd_min is not None                  # the index searches with the EAPCA bound: so does TDG
    if not hasattr(di, "_leaf_env"):
        env = [t.env_min, t.env_max] + ([t.sd_min, t.sd_max] if eapca else [])
        di._leaf_env = tuple(torch.from_numpy(np.ascontiguousarray(a[leaf_ids].T)).to(di.device) for a in env)
    mn, mx = di._leaf_env[:2]
    q = queries if isinstance(queries, torch.Tensor) else torch.from_numpy(
        np.ascontiguousarray(np.atleast_2d(queries), dtype=np.float32))
    q = q.to(device=di.device, dtype=torch.float32).contiguous()
    Q = q.shape[0]
    qs = torch.empty((Q, t.n_seg * (2 if eapca else 1)), dtype=torch.float64, device=di.device)
    lb = torch.empty((Q, leaf_ids.shape[0]), dtype=torch.float64, device=di.device)
    if eapca:
        smn, smx = di._leaf_env[2:]
        _lib.check(_lib.lib().lf_bounds_eapca(q.data_ptr(), Q, di.struct(None), mn.data_ptr(), mx.data_ptr(),
                                              smn.data_ptr(), smx.data_ptr(), leaf_ids.shape[0], qs.data_ptr(),
                                              lb.data_ptr(), _lib.stream_ptr()))
    else:
        _lib.check(_lib.lib().lf_bounds(q.data_ptr(), Q, di.struct(None), mn.data_ptr(), mx.data_ptr(),
                                        leaf_ids.shape[0], mode, qs.data_ptr(), lb.data_ptr(),
                                        _lib.stream_ptr()))
    return qs, lb


def collect_targets(index, selected_leaves, queries, calibration_count: int, *,
                    train_nn: bool = True, shard=None) -> GlobalTrainSet:
    """GPU twin of traingen.collect_targets (traingen.py:147-220).

    train_nn=False skips the pass-2 walk for the training rows (nn_distance[:c0]
    is then NaN): enhance() reads only the calibration rows' nn_distance, and the
    walk needs distances to every non-selected leaf it reaches.
    shard=(rank, world, group): leaf-sharded -- this rank computes
    every query's minimum distance to ITS leaves only; the columns of all ranks are
    all-gathered (same kernel per column, so the matrices equal the unsharded ones)."""
    torch = _lib.require_cuda()
    t = as_tree(index)
    if shard is not None and shard[1] > 1:
        if not train_nn:
            return _collect_targets_sharded(t, selected_leaves, queries, calibration_count, *shard)
        raise ValueError("the sharded collection computes the calibration rows' nn_distance only (train_nn=False)")
    di = t.device()
    Qh = np.atleast_2d(np.asarray(queries, dtype=np.float64))
    n_q = Qh.shape[0]
    if not 1 <= calibration_count < n_q:
        raise ValueError("calibration_count must be in [1, n_queries)")
    selected = sorted(int(s) for s in selected_leaves)
    leaf_ids = t.leaf_ids.astype(np.int64)
    unknown = set(selected) - set(int(i) for i in leaf_ids)
    if unknown:
        raise ValueError(f"unknown leaf ids in selection: {sorted(unknown)}")
    q = torch.from_numpy(Qh.astype(np.float32)).to(di.device)
    _, lb = leaf_bounds(t, q, mode=1)
    # stable sort: ties resolve to the smaller column = smaller leaf id (traingen.py:170-171)
    order = torch.sort(lb, dim=1, stable=True).indices.to(torch.int32)
    sel_slots = [di.slot_of_leaf[l] for l in selected]
    dl_sel = leaf_min_distances(t, q, sel_slots) if selected else torch.empty((n_q, 0), dtype=torch.float64,
                                                                              device=di.device)
    c0 = n_q - calibration_count
    L = leaf_ids.shape[0]
    dcal = torch.empty((calibration_count, L), dtype=torch.float64, device=di.device)
    sel_set = set(selected)
    col_of = {l: c for c, l in enumerate(selected)}
    sel_pos = [p for p, l in enumerate(leaf_ids) if int(l) in sel_set]
    other_pos = [p for p, l in enumerate(leaf_ids) if int(l) not in sel_set]
    if sel_pos:
        dcal[:, sel_pos] = dl_sel[c0:, [col_of[int(leaf_ids[p])] for p in sel_pos]]
    if other_pos:
        dcal[:, other_pos] = leaf_min_distances(t, q[c0:], other_pos)
    # pass 2 (traingen.py:190-208): walk the visit order, break on lb >= bsf
    lbh = lb.cpu().numpy()
    orh = order.cpu().numpy()
    dsel_h = dl_sel.cpu().numpy()
    nn = np.empty(n_q)
    dcal_h = dcal.cpu().numpy()
    nn[c0:] = dcal_h.min(axis=1)
    if c0 > 0 and not train_nn:
        nn[:c0] = np.nan
    elif c0 > 0:
        d_other = None
        if other_pos:
            d_other = np.full((c0, L), np.inf)
            d_other[:, other_pos] = leaf_min_distances(t, q[:c0], other_pos).cpu().numpy()
        dfull = np.full((c0, L), np.inf)
        if sel_pos:
            dfull[:, sel_pos] = dsel_h[:c0, [col_of[int(leaf_ids[p])] for p in sel_pos]]
        if d_other is not None:
            dfull[:, other_pos] = d_other[:, other_pos]
        bsf = dsel_h[:c0].min(axis=1) if selected else np.full(c0, np.inf)
        alive = np.ones(c0, dtype=bool)
        rows = np.arange(c0)
        for p in range(L):
            col = orh[:c0, p]
            lbp = lbh[rows, col]
            alive &= ~(lbp >= bsf)
            if not alive.any():
                break
            np.minimum(bsf, np.where(alive, dfull[rows, col], np.inf), out=bsf)
        nn[:c0] = bsf
    return GlobalTrainSet(Qh, selected, dsel_h, nn, leaf_ids, lbh, orh, calibration_count, dcal_h)


def _collect_targets_sharded(t, selected_leaves, queries, calibration_count: int, rank: int, world: int,
                             group=None) -> GlobalTrainSet:
    torch = _lib.require_cuda()
    di = t.shard(rank, world)
    Qh = np.atleast_2d(np.asarray(queries, dtype=np.float64))
    n_q = Qh.shape[0]
    if not 1 <= calibration_count < n_q:
        raise ValueError("calibration_count must be in [1, n_queries)")
    selected = sorted(int(s) for s in selected_leaves)
    leaf_ids = t.leaf_ids.astype(np.int64)
    unknown = set(selected) - set(int(i) for i in leaf_ids)
    if unknown:
        raise ValueError(f"unknown leaf ids in selection: {sorted(unknown)}")
    q = torch.from_numpy(Qh.astype(np.float32)).to(di.device)
    _, lb = leaf_bounds(t, q, mode=1, dindex=di)
    order = torch.sort(lb, dim=1, stable=True).indices.to(torch.int32)
    _, full, _ = sharded_leaf_min_distances(t, q, rank, world, gather=True, group=group)
    sel_cols = np.searchsorted(leaf_ids, np.asarray(selected, dtype=np.int64))
    c0 = n_q - calibration_count
    dsel_h = full[:, torch.as_tensor(sel_cols, device=full.device)].cpu().numpy()
    dcal_h = full[c0:].cpu().numpy()
    nn = np.full(n_q, np.nan)
    nn[c0:] = dcal_h.min(axis=1)
    return GlobalTrainSet(Qh, selected, dsel_h, nn, leaf_ids, lb.cpu().numpy(), order.cpu().numpy(),
                          calibration_count, dcal_h)


def collect_local_targets(index, local: LocalQueries) -> LocalQueries:
    """GPU twin of traingen.collect_local_targets (traingen.py:135-144)."""
    t = as_tree(index)
    res = local_targets_all(t, {local.leaf_id: local.queries})
    local.targets, local.lbs = res[local.leaf_id]
    return local


def own_leaf_bounds(t, leaf_id: int, queries: np.ndarray) -> np.ndarray:
    """lb of each query against one leaf envelope, in the einsum order of
    lower_bounds_batch (summarize.py:114-122): sum_s (g_s * g_s) * w_s, s ascending."""
    from .index import segment_means

    qs = segment_means(queries, t.n_seg)
    g = np.maximum(t.env_min[leaf_id][None, :] - qs, qs - t.env_max[leaf_id][None, :])
    g = np.maximum(g, 0.0)
    acc = np.zeros(qs.shape[0])
    w = t.widths.astype(np.float64)
    for s in range(t.n_seg):
        acc = acc + (g[:, s] * g[:, s]) * w[s]
    return np.sqrt(acc)


def local_targets_all(index, queries_by_leaf: dict, path: str | None = None, dindex=None) -> dict:
    """{leaf_id: queries} -> {leaf_id: (targets, lbs)} in one lf_local_min_dist launch per 65535 leaves.
    dindex: a DeviceIndex (e.g. this rank's leaf shard) holding every leaf asked for."""
    torch = _lib.require_cuda()
    t = as_tree(index)
    di = dindex if dindex is not None else t.device()
    path = path or default_path(t, di)
    fn = {"q8": _lib.lib().lf_local_min_dist_q8,
          "tc": _lib.lib().lf_local_min_dist_tc}.get(path, _lib.lib().lf_local_min_dist)
    st = di.struct(None)
    leaves = list(queries_by_leaf)
    out = {}
    for g0 in range(0, len(leaves), 65535):
        grp = leaves[g0:g0 + 65535]
        qs = [np.atleast_2d(np.asarray(queries_by_leaf[l], dtype=np.float64)) for l in grp]
        qptr = np.zeros(len(grp) + 1, dtype=np.int64)
        qptr[1:] = np.cumsum([a.shape[0] for a in qs])
        allq = torch.from_numpy(np.concatenate(qs).astype(np.float32)).to(di.device)
        gleaf = np.array([di.slot_of_leaf[int(l)] for l in grp], dtype=np.int32)
        dl = torch.empty(int(qptr[-1]), dtype=torch.float64, device=di.device)
        _lib.check(fn(allq.data_ptr(), st, _lib.ptr(qptr), _lib.ptr(gleaf), len(grp),
                      dl.data_ptr(), _lib.stream_ptr()))
        dlh = dl.cpu().numpy()
        for gi, l in enumerate(grp):
            out[l] = (dlh[qptr[gi]:qptr[gi + 1]], own_leaf_bounds(t, l, qs[gi]))
    return out
