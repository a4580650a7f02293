"""iSAX index (BASELINE config 3: "iSAX + LeaFi"), built into the same node table
as the DSTree-style `TreeIndex`, so the whole GPU path (bounds, visit order,
filters, leaf scan, training-data generation) runs on it unchanged.

The reference package has no iSAX (parity unpinned); this follows
the iSAX definition: a node is a SAX word -- per segment a symbol at some
cardinality 2^b over the standard-normal breakpoints of the segment means -- so
its region on segment i is the breakpoint interval [beta_lo, beta_hi].  The
search bound is MINDIST_PAA_iSAX, which is exactly the envelope bound the
kernels already evaluate (summarize.py:97-107 shape) with the interval as the
envelope:  lb = sqrt(sum_i w_i * max(beta_lo_i - mu_i, mu_i - beta_hi_i, 0)^2).
It is sound because every member's segment means lie in its node's intervals.

Splits are binary (iSAX 2.0 style): a full leaf raises the cardinality of one
segment by one bit -- the segment whose new breakpoint splits the members most
evenly.  A split that would leave one side empty refines the node's interval in
place instead (the region shrinks, the bound tightens), so no empty leaves are
created.  Children get larger node ids than their parent and their regions are
nested in the parent's, so the best-first heap still pops in (lb, id) order
 and the batched GPU walk applies as is.
"""

from __future__ import annotations

from statistics import NormalDist

import numpy as np

from .index import DeviceRows, TreeIndex, as_f32_rows, segment_layout, segment_means

_ND = NormalDist()


def breakpoint(bits: int, j: int) -> float:
    """j-th boundary of the 2^bits equiprobable N(0, 1) symbols (j = 0 .. 2^bits)."""
    if j <= 0:
        return -np.inf
    if j >= (1 << bits):
        return np.inf
    return _ND.inv_cdf(j / float(1 << bits))


def build_isax_from_summaries(summ: np.ndarray, values, max_leaf_size: int, segments: int,
                              max_bits: int = 8) -> TreeIndex:
    """iSAX tree over precomputed segment means summ [n, segments] (fp64)."""
    if max_leaf_size < 2:
        raise ValueError(f"max_leaf_size must be >= 2, got {max_leaf_size}")
    if not 1 <= max_bits <= 16:
        raise ValueError("max_bits must be in [1, 16]")
    n, l = summ.shape
    m = int(values.shape[1])
    starts, widths = segment_layout(m, segments)
    env_min, env_max, left, right, sseg, sthr, size, over, members = [], [], [], [], [], [], [], [], []

    def new_node(bits, syms, ids):
        env_min.append(np.array([breakpoint(b, s) for b, s in zip(bits, syms)]))
        env_max.append(np.array([breakpoint(b, s + 1) for b, s in zip(bits, syms)]))
        left.append(-1); right.append(-1); sseg.append(-1); sthr.append(np.nan)
        size.append(int(ids.shape[0])); over.append(False); members.append(ids)
        return len(left) - 1

    root = new_node([0] * l, [0] * l, np.arange(n, dtype=np.int64))
    stack = [(root, [0] * l, [0] * l)]
    while stack:
        nid, bits, syms = stack.pop()
        ids = members[nid]
        if ids.shape[0] <= max_leaf_size:
            continue
        while True:
            cand = [i for i in range(l) if bits[i] < max_bits]
            if not cand:
                over[nid] = True
                break
            bounds = np.array([breakpoint(bits[i] + 1, 2 * syms[i] + 1) for i in cand])
            low = (summ[ids][:, cand] < bounds[None, :]).sum(axis=0)
            bal = np.minimum(low, ids.shape[0] - low)
            k = int(np.argmax(bal))
            i = cand[k]
            if bal[k] == 0:
                # one-sided: refine this node's interval on segment i in place
                side = 0 if low[k] == ids.shape[0] else 1
                bits[i] += 1
                syms[i] = 2 * syms[i] + side
                env_min[nid][i] = breakpoint(bits[i], syms[i])
                env_max[nid][i] = breakpoint(bits[i], syms[i] + 1)
                continue
            go_low = summ[ids, i] < bounds[k]
            lb_, ls_ = list(bits), list(syms)
            rb_, rs_ = list(bits), list(syms)
            lb_[i] += 1; rb_[i] += 1
            ls_[i] = 2 * syms[i]; rs_[i] = 2 * syms[i] + 1
            a = new_node(lb_, ls_, ids[go_low])
            b = new_node(rb_, rs_, ids[~go_low])
            left[nid], right[nid], sseg[nid], sthr[nid] = a, b, i, float(bounds[k])
            members[nid] = None
            stack.append((b, rb_, rs_))
            stack.append((a, lb_, ls_))
            break
    nn = len(left)
    counts = [0 if mm is None else mm.shape[0] for mm in members]
    ptr = np.zeros(nn + 1, dtype=np.int64)
    ptr[1:] = np.cumsum(counts)
    flat = np.concatenate([mm for mm in members if mm is not None]) if n else np.zeros(0, np.int64)
    return TreeIndex(values, starts, widths, int(max_leaf_size),
                     np.stack(env_min), np.stack(env_max),
                     np.array(left, np.int32), np.array(right, np.int32), np.array(sseg, np.int32),
                     np.array(sthr), np.array(size, np.int64), np.array(over, bool), ptr, flat)


def build_isax_index(values, max_leaf_size: int = 1000, segments: int = 8, max_bits: int = 8) -> TreeIndex:
    """iSAX index over host rows (fp32-exact) or a device fp32 tensor (segment means on
    the GPU, rows stay in HBM)."""
    if hasattr(values, "data_ptr") and getattr(values, "is_cuda", False):
        import torch

        from . import _lib

        n, m = int(values.shape[0]), int(values.shape[1])
        summ = torch.empty((n, segments), dtype=torch.float64, device=values.device)
        _lib.check(_lib.lib().lf_paa_device(values.data_ptr(), n, m, segments, summ.data_ptr(), _lib.stream_ptr()))
        return build_isax_from_summaries(summ.cpu().numpy(), DeviceRows(values), max_leaf_size, segments, max_bits)
    v = as_f32_rows(values)
    if not np.isfinite(v).all():
        raise ValueError("dataset contains non-finite values")
    return build_isax_from_summaries(segment_means(v, segments), v, max_leaf_size, segments, max_bits)
