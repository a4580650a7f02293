"""Host image of the summarization tree and its HBM layout.

`TreeIndex` carries the same node table as the reference `tree.Index`
(tree.py:93-122): envelopes over segment means, split rules, leaf members.
It is produced by the native builder (`build_index`, bit-identical to
tree.build_index, tree.py:164-189) or adopted from a reference Index object
(`TreeIndex.from_reference`, duck-typed; the drop-in path).

`DeviceIndex` is the HBM layout the kernels read:

* ``X``        fp32 [n, m], LEAF-CONTIGUOUS: leaves in ascending node id,
               members in ascending series id (tree.py:102-106);
* ``row_id``   int64 [n]: original series id of every row;
* ``leaf_ptr`` int64 [L+1]: row range of leaf slot j;
* ``node_leaf`` int32 [nodes]: leaf slot of a node, -1 for internal nodes;
* ``env_min`` / ``env_max`` fp64 [segments][nodes], structure-of-arrays so
  one warp reads one segment of 32 consecutive nodes in one transaction.
"""

from __future__ import annotations

import ctypes as C
import os
from dataclasses import dataclass, field

import numpy as np

from . import _lib


def segment_layout(m: int, n_seg: int) -> tuple:
    """Equal widths, leading segments +1 (summarize.py:27-37)."""
    if not 1 <= n_seg <= m:
        raise ValueError(f"num_segments must be in [1, length], got {n_seg} for length {m}")
    base, rem = divmod(m, n_seg)
    widths = np.full(n_seg, base, dtype=np.int64)
    widths[:rem] += 1
    starts = np.zeros(n_seg, dtype=np.int64)
    starts[1:] = np.cumsum(widths)[:-1]
    return starts, widths


def as_f32_rows(values) -> np.ndarray:
    """fp32 storage of a collection; the reference keeps fp32-exact values (series.py:48-50)."""
    v = np.asarray(values)
    if v.ndim != 2:
        raise ValueError(f"dataset values must be 2-d, got shape {v.shape}")
    if v.dtype == np.float32:
        return np.ascontiguousarray(v)
    v32 = np.ascontiguousarray(v, dtype=np.float32)
    if not np.array_equal(v32.astype(v.dtype), v):
        raise ValueError("dataset values are not fp32-exact (quantize with series.quantize32 first)")
    return v32



PCA_MIN_ENERGY = 0.9     # default projected-shadow gate (random walks: ~0.98 in 32 directions)

class DeviceRows:
    """Row access to a device-resident collection with numpy semantics (rows -> host fp32)."""

    def __init__(self, tensor):
        self.tensor = tensor
        self.shape = tuple(tensor.shape)
        self.dtype = np.float32

    def __getitem__(self, ids):
        import torch

        idx = torch.as_tensor(np.asarray(ids, dtype=np.int64)).to(self.tensor.device)
        return self.tensor.index_select(0, idx.reshape(-1)).cpu().numpy().reshape(*np.shape(ids), self.shape[1])

    def __len__(self) -> int:
        return self.shape[0]


class ReleasedRows:
    """Stand-in for a collection whose rows were dropped (a leaf-sharded rank keeps
    only its shard's rows): the shape stays known, any row access raises."""

    def __init__(self, shape):
        self.shape = tuple(shape)
        self.dtype = np.float32

    def __getitem__(self, ids):
        raise RuntimeError("the collection rows were released on this rank (leaf shard only)")

    def __len__(self) -> int:
        return self.shape[0]


@dataclass
class TreeIndex:
    values: object                  # fp32 [n, m] host ndarray, or DeviceRows (original row order)
    starts: np.ndarray
    widths: np.ndarray
    max_leaf_size: int
    env_min: np.ndarray             # fp64 [nodes, segments]
    env_max: np.ndarray
    left: np.ndarray                # int32 [nodes], -1 for leaves
    right: np.ndarray
    split_seg: np.ndarray
    split_thr: np.ndarray
    size: np.ndarray                # int64 [nodes]
    oversized: np.ndarray           # bool [nodes]
    member_ptr: np.ndarray          # int64 [nodes + 1]; internal nodes have empty ranges
    members: np.ndarray             # int64 [n]
    _device: dict = field(default_factory=dict, repr=False, compare=False)
    sd_min: np.ndarray | None = None  # fp64 [nodes, segments]: EAPCA envelopes (use_eapca), else None
    sd_max: np.ndarray | None = None

    def use_eapca(self) -> "TreeIndex":
        """Switch the index to the EAPCA bound (mean + stdev per segment,
        include/leafi_b200.h lf_bounds_eapca): per node the [min, max] of its members'
        segment stdevs, computed on the GPU (lf_eapca_device) in row chunks.  The tree
        (the reference's mean-based splits) is unchanged; search and training-data
        generation then use the EAPCA bound.  Call before the first device image."""
        torch = _lib.require_cuda()
        if self.sd_min is not None:
            return self
        if self._device:
            raise RuntimeError("use_eapca() must precede the first device image of the index")
        n, l = self.n, self.n_seg
        sd = np.empty((n, l))
        src = self.values.tensor if isinstance(self.values, DeviceRows) else None
        step = 1 << 20
        for r0 in range(0, n, step):
            r1 = min(n, r0 + step)
            x = src[r0:r1] if src is not None else torch.from_numpy(
                np.ascontiguousarray(self.values[r0:r1], dtype=np.float32)).cuda()
            out = torch.empty((r1 - r0, 2 * l), dtype=torch.float64, device=x.device)
            _lib.check(_lib.lib().lf_eapca_device(x.data_ptr(), r1 - r0, self.m, l, out.data_ptr(), _lib.stream_ptr()))
            sd[r0:r1] = out[:, l:].cpu().numpy()
        nn = self.n_nodes
        smin = np.full((nn, l), np.inf)
        smax = np.full((nn, l), -np.inf)
        for nid in range(nn - 1, -1, -1):                 # children have larger ids than parents
            if self.left[nid] < 0:
                ids = self.members[self.member_ptr[nid]:self.member_ptr[nid + 1]]
                if ids.size:
                    smin[nid] = sd[ids].min(axis=0)
                    smax[nid] = sd[ids].max(axis=0)
            else:
                for c in (self.left[nid], self.right[nid]):
                    np.minimum(smin[nid], smin[c], out=smin[nid])
                    np.maximum(smax[nid], smax[c], out=smax[nid])
        self.sd_min, self.sd_max = smin, smax
        return self

    def release_rows(self) -> None:
        """Drop the full collection (e.g. after a rank built its leaf shard); the
        device images already built keep their own rows."""
        self.values = ReleasedRows(self.values.shape)

    # ------------------------------------------------------------- shape --
    @property
    def n(self) -> int:
        return int(self.values.shape[0])

    @property
    def m(self) -> int:
        return int(self.values.shape[1])

    @property
    def n_seg(self) -> int:
        return int(self.widths.shape[0])

    @property
    def n_nodes(self) -> int:
        return int(self.left.shape[0])

    @property
    def is_leaf(self) -> np.ndarray:
        return self.left < 0

    @property
    def leaf_ids(self) -> np.ndarray:
        return np.nonzero(self.is_leaf)[0].astype(np.int64)

    @property
    def n_leaves(self) -> int:
        return int(self.is_leaf.sum())

    def leaf_members(self, leaf_id: int) -> np.ndarray:
        return self.members[self.member_ptr[leaf_id]:self.member_ptr[leaf_id + 1]]

    def leaf_sizes(self) -> list:
        """(leaf id, size) pairs in ascending leaf id (tree.py:112-113)."""
        return [(int(l), int(self.size[l])) for l in self.leaf_ids]

    def has_oversized_leaves(self) -> bool:
        return bool(self.oversized[self.is_leaf].any())

    # ------------------------------------------------------ constructors --
    @classmethod
    def from_reference(cls, index) -> "TreeIndex":
        """Adopt a reference `tree.Index` (duck-typed) without copying its tree logic."""
        nodes = index.nodes
        l = int(index.cfg.num_segments)
        nn = len(nodes)
        members = [nd.members if nd.members is not None else [] for nd in nodes]
        ptr = np.zeros(nn + 1, dtype=np.int64)
        ptr[1:] = np.cumsum([len(mm) for mm in members])
        flat = np.fromiter((i for mm in members for i in mm), dtype=np.int64, count=int(ptr[-1]))
        t = cls(
            values=as_f32_rows(index.dataset.values),
            starts=np.asarray(index.cfg.starts, dtype=np.int64),
            widths=np.asarray(index.cfg.widths, dtype=np.int64),
            max_leaf_size=int(index.max_leaf_size),
            env_min=np.stack([np.asarray(nd.envelope.mean_min, dtype=np.float64) for nd in nodes]).reshape(nn, l),
            env_max=np.stack([np.asarray(nd.envelope.mean_max, dtype=np.float64) for nd in nodes]).reshape(nn, l),
            left=np.array([-1 if nd.left is None else nd.left.node_id for nd in nodes], dtype=np.int32),
            right=np.array([-1 if nd.right is None else nd.right.node_id for nd in nodes], dtype=np.int32),
            split_seg=np.array([-1 if nd.split_segment is None else nd.split_segment for nd in nodes], dtype=np.int32),
            split_thr=np.array([np.nan if nd.split_threshold is None else nd.split_threshold for nd in nodes]),
            size=np.array([nd.size for nd in nodes], dtype=np.int64),
            oversized=np.array([bool(nd.oversized) for nd in nodes]),
            member_ptr=ptr,
            members=flat,
        )
        return t

    # ------------------------------------------------------------ device --
    def device(self, device=None, leaf_range=None) -> "DeviceIndex":
        torch = _lib.require_cuda()
        dev = torch.device(device if device is not None else "cuda")
        if dev.index is None:
            dev = torch.device("cuda", torch.cuda.current_device())
        key = (str(dev), tuple(leaf_range) if leaf_range is not None else None)
        if key not in self._device:
            self._device[key] = DeviceIndex(self, dev, leaf_range)
        return self._device[key]

    def shard(self, rank: int, world: int, device=None) -> "DeviceIndex":
        """This rank's leaf shard (contiguous leaves, balanced by series count)."""
        sizes = self.size[self.leaf_ids]
        return self.device(device, shard_leaf_ranges(sizes, world)[rank])


def build_index(values, max_leaf_size: int = 1000, segments: int = 8,
                n_threads: int | None = None) -> TreeIndex:
    """Native tree build, bit-identical to tree.build_index (tree.py:164-189)."""
    if max_leaf_size < 2:
        raise ValueError(f"max_leaf_size must be >= 2, got {max_leaf_size}")
    v = as_f32_rows(values)
    n, m = v.shape
    if n < 1 or m < 2:
        raise ValueError(f"dataset needs n >= 1 and m >= 2, got {v.shape}")
    if not np.isfinite(v).all():
        raise ValueError("dataset contains non-finite values")
    starts, widths = segment_layout(m, segments)
    L = _lib.lib()
    h = L.lf_tree_build(_lib.ptr(v), n, m, segments, max_leaf_size, n_threads or _lib.threads())
    if not h:
        _lib.check(_lib.LF_EINVAL)
    try:
        arrays = _export(L, h, n, segments)
    finally:
        L.lf_tree_free(h)
    return TreeIndex(v, starts, widths, int(max_leaf_size), *arrays)


def build_index_device(X, max_leaf_size: int = 1000, segments: int = 8) -> TreeIndex:
    """Tree build for a DEVICE collection (fp32 [n, m] torch tensor): segment means on
    the GPU (lf_paa_device, numpy order), insertion/split loop on the host from the
    means alone (lf_tree_build_from_summaries) -- the rows never visit the host."""
    import torch

    if max_leaf_size < 2:
        raise ValueError(f"max_leaf_size must be >= 2, got {max_leaf_size}")
    n, m = int(X.shape[0]), int(X.shape[1])
    starts, widths = segment_layout(m, segments)
    summ = torch.empty((n, segments), dtype=torch.float64, device=X.device)
    _lib.check(_lib.lib().lf_paa_device(X.data_ptr(), n, m, segments, summ.data_ptr(), _lib.stream_ptr()))
    hs = summ.cpu().numpy()
    del summ
    L = _lib.lib()
    h = L.lf_tree_build_from_summaries(_lib.ptr(hs), n, segments, max_leaf_size)
    if not h:
        _lib.check(_lib.LF_EINVAL)
    try:
        arrays = _export(L, h, n, segments)
    finally:
        L.lf_tree_free(h)
    return TreeIndex(DeviceRows(X), starts, widths, int(max_leaf_size), *arrays)


def _export(L, h, n: int, segments: int) -> tuple:
    nn, nl = C.c_int32(), C.c_int32()
    _lib.check(L.lf_tree_info(h, C.byref(nn), C.byref(nl)))
    k = nn.value
    env_min = np.empty((k, segments)); env_max = np.empty((k, segments))
    left = np.empty(k, np.int32); right = np.empty(k, np.int32)
    sseg = np.empty(k, np.int32); sthr = np.empty(k)
    size = np.empty(k, np.int64); over = np.empty(k, np.int8)
    mptr = np.empty(k + 1, np.int64); mem = np.empty(n, np.int64)
    _lib.check(L.lf_tree_export(h, *(_lib.ptr(a) for a in (env_min, env_max, left, right, sseg,
                                                          sthr, size, over, mptr, mem))))
    return env_min, env_max, left, right, sseg, sthr, size, over.astype(bool), mptr, mem


def segment_means(values, segments: int = 8) -> np.ndarray:
    """Host segment means in numpy's reduceat order (summarize.py:52-56)."""
    v = as_f32_rows(np.atleast_2d(values))
    out = np.empty((v.shape[0], segments))
    _lib.check(_lib.lib().lf_paa_host(_lib.ptr(v), v.shape[0], v.shape[1], segments, _lib.ptr(out),
                                      _lib.threads()))
    return out


def shard_leaf_ranges(sizes, world: int) -> list:
    """Cut leaves (ascending node id) into `world` contiguous ranges of about equal
    series count: range r ends at the first leaf whose cumulative
    size reaches (r+1)/world of the total."""
    sizes = np.asarray(sizes, dtype=np.int64)
    if world < 1:
        raise ValueError("world must be >= 1")
    csum = np.cumsum(sizes)
    total = int(csum[-1]) if csum.size else 0
    bounds = [0]
    for r in range(1, world):
        cut = int(np.searchsorted(csum, total * r / world, side="left")) + 1
        bounds.append(min(max(cut, bounds[-1]), sizes.shape[0]))
    bounds.append(sizes.shape[0])
    return [(bounds[r], bounds[r + 1]) for r in range(world)]


class DeviceIndex:
    """The tree in HBM (see module docstring for the layout).

    leaf_range=(a, b) keeps only leaf slots a..b-1 (a leaf shard): their rows,
    and a node->leaf map in which every other leaf reads as "not mine" (-1),
    so the kernels skip it exactly like an internal node.  Visit order and
    bounds still cover the whole tree, so every shard agrees on the break point.
    """

    def __init__(self, t: TreeIndex, dev, leaf_range=None):
        import torch

        self.tree = t
        self.device = dev
        all_leaves = t.leaf_ids
        a, b = leaf_range if leaf_range is not None else (0, all_leaves.shape[0])
        self.leaf_range = (int(a), int(b))
        leaf_ids = all_leaves[a:b]
        sizes = t.member_ptr[leaf_ids + 1] - t.member_ptr[leaf_ids]
        leaf_ptr = np.zeros(leaf_ids.shape[0] + 1, dtype=np.int64)
        leaf_ptr[1:] = np.cumsum(sizes)
        order = np.concatenate([t.leaf_members(l) for l in leaf_ids]) if leaf_ids.size else np.zeros(0, np.int64)
        node_leaf = np.full(t.n_nodes, -1, dtype=np.int32)
        node_leaf[leaf_ids] = np.arange(leaf_ids.shape[0], dtype=np.int32)
        with torch.cuda.device(dev):
            rid = torch.from_numpy(order).to(dev)
            from .leafio import FileRows, load_rows_to

            if isinstance(t.values, DeviceRows):
                self.X = t.values.tensor.index_select(0, rid).contiguous()
            elif isinstance(t.values, FileRows):
                # LEAF file: rows streamed straight into their leaf-contiguous slots
                pos = np.full(t.n, -1, dtype=np.int64)
                pos[order] = np.arange(order.shape[0], dtype=np.int64)
                self.X = torch.empty((order.shape[0], t.m), dtype=torch.float32, device=dev)
                load_rows_to(t.values, torch.from_numpy(pos).to(dev), self.X)
            else:
                src = torch.from_numpy(t.values).to(dev)
                self.X = src.index_select(0, rid).contiguous()
                del src
            self.row_id = rid
            self.leaf_ptr = torch.from_numpy(leaf_ptr).to(dev)
            self.node_leaf = torch.from_numpy(node_leaf).to(dev)
            self.env_min = torch.from_numpy(np.ascontiguousarray(t.env_min.T)).to(dev)
            self.env_max = torch.from_numpy(np.ascontiguousarray(t.env_max.T)).to(dev)
            self.sd_min = self.sd_max = None
            if t.sd_min is not None:                  # EAPCA envelopes, SoA like the means
                self.sd_min = torch.from_numpy(np.ascontiguousarray(t.sd_min.T)).to(dev)
                self.sd_max = torch.from_numpy(np.ascontiguousarray(t.sd_max.T)).to(dev)
            # int8 shadow for the bounded scan (scan_q8_kernel), when the layout allows it
            self.X8 = self.qmeta = None
            n_rows, m = int(self.X.shape[0]), int(self.X.shape[1])
            if m % 4 == 0 and m <= 512 and n_rows:     # codes zero-padded to a multiple of 32
                self.X8 = torch.empty((n_rows, (m + 31) // 32 * 32), dtype=torch.int8, device=dev)
                self.qmeta = torch.empty((n_rows, 4), dtype=torch.float32, device=dev)
                _lib.check(_lib.lib().lf_quantize_rows(self.X.data_ptr(), n_rows, m, self.X8.data_ptr(),
                                                       self.qmeta.data_ptr(), _lib.stream_ptr()))
            self.pca_k = 0
            self.P = self.mu = self.Xp = self.pmeta = None
            self.pca_energy = None
            variant = os.environ.get("LF_SCAN_VARIANT") or None
            if m % 4 == 0 and 64 <= m <= 512 and n_rows >= 256 and variant in (None, "pq"):
                # projected shadow for the two-stage scan: by default only when the leading
                # directions hold most of the energy (else the projected bound prunes little)
                self.ensure_pca(int(os.environ.get("LF_PCA_K", "32")),
                                min_energy=None if variant == "pq" else PCA_MIN_ENERGY)
        self.leaf_ids = leaf_ids
        self.leaf_ptr_host = leaf_ptr
        self.slot_of_leaf = {int(l): j for j, l in enumerate(leaf_ids)}
        self.max_leaf_rows = int(sizes.max()) if sizes.size else 0

    @property
    def n_leaves(self) -> int:
        return int(self.leaf_ids.shape[0])

    def ensure_pca(self, k: int = 32, sample: int = 200_000, seed: int = 0, min_energy: float | None = None) -> bool:
        """Projected shadow for the two-stage scan (lf_index.d_Xp): the top-k principal
        directions of a row sample (fp64 SVD, orthonormal rows), and per row the int8
        codes of y = P (x - mu) with {scale, ||scale * code||^2, code error (rounded
        up), residual norm}.  Index-build plumbing in torch; the search reads it in the
        scan kernel.  With min_energy, the shadow is built only when the k directions
        hold at least that fraction of the sample's centred energy (self.pca_energy).
        Returns whether the shadow exists."""
        import torch

        if k not in (32, 64):
            raise ValueError("pca_k must be 32 or 64")
        X = self.X
        n, m = int(X.shape[0]), int(X.shape[1])
        with torch.cuda.device(self.device):
            g = torch.Generator(device=self.device)
            g.manual_seed(seed)
            pick = torch.randint(0, n, (min(sample, n),), generator=g, device=self.device)
            S = X[pick].double()
            mu = S.mean(0)
            _, sv, V = torch.linalg.svd(S - mu, full_matrices=False)
            e2 = sv * sv
            self.pca_energy = float(e2[:k].sum() / e2.sum()) if float(e2.sum()) > 0 else 1.0
            if min_energy is not None and self.pca_energy < min_energy:
                return False
            P = V[:k].contiguous()
            codes = torch.empty((n, k), dtype=torch.int8, device=self.device)
            # 8 B of fp16 metadata per row (+ 2 rows of padding: the scan's bulk copies
            # round a piece's metadata up to 16 bytes)
            meta = torch.zeros((n + 2, 4), dtype=torch.float16, device=self.device)
            inf16 = torch.tensor(float("inf"), dtype=torch.float16, device=self.device)
            for r0 in range(0, n, 1 << 20):
                A = X[r0:r0 + (1 << 20)].double() - mu
                y = A @ P.T
                r = (A - y @ P).norm(dim=1)
                s = y.abs().amax(1) / 127
                s16 = torch.where(s > 0, s, torch.ones_like(s)).half()
                s16 = torch.where(s16.double() < s, torch.nextafter(s16, inf16), s16)   # up: |y| / s <= 127
                sd = s16.double()
                c = torch.round(y / sd[:, None]).clamp(-127, 127)
                e = ((c * sd[:, None] - y).norm(dim=1) * (1 + 1e-9) + 1e-30)
                e16 = e.half()
                e16 = torch.where(e16.double() < e, torch.nextafter(e16, inf16), e16)   # rounded up
                codes[r0:r0 + (1 << 20)] = c.to(torch.int8)
                meta[r0:r0 + A.shape[0]] = torch.stack([s16, e16, r.half(), torch.zeros_like(s16)], dim=1)
        self.pca_k, self.P, self.mu, self.Xp, self.pmeta = k, P, mu.contiguous(), codes, meta
        return True

    def struct(self, leaf_filter=None) -> _lib.LfIndex:
        t = self.tree
        s = _lib.LfIndex()
        s.n_series = t.n
        s.m = t.m
        s.n_seg = t.n_seg
        s.n_nodes = t.n_nodes
        s.n_leaves = self.n_leaves
        s.max_leaf_rows = self.max_leaf_rows
        for i in range(t.n_seg):
            s.seg_start[i] = int(t.starts[i])
            s.seg_width[i] = int(t.widths[i])
        s.d_X = self.X.data_ptr()
        s.d_row_id = self.row_id.data_ptr()
        s.d_leaf_ptr = self.leaf_ptr.data_ptr()
        s.d_node_leaf = self.node_leaf.data_ptr()
        s.d_env_min = self.env_min.data_ptr()
        s.d_env_max = self.env_max.data_ptr()
        s.d_leaf_filter = None if leaf_filter is None else leaf_filter.data_ptr()
        if self.X8 is not None:
            s.d_X8, s.d_qmeta = self.X8.data_ptr(), self.qmeta.data_ptr()
        if self.sd_min is not None:
            s.d_sd_min, s.d_sd_max = self.sd_min.data_ptr(), self.sd_max.data_ptr()
        if getattr(self, "Xp", None) is not None:
            s.pca_k = self.pca_k
            s.d_P, s.d_mu = self.P.data_ptr(), self.mu.data_ptr()
            s.d_Xp, s.d_pmeta = self.Xp.data_ptr(), self.pmeta.data_ptr()
        return s
