"""iSAX index builder (BASELINE config 3) on the host: structure invariants that make
the GPU engine's assumptions hold (nested regions, child ids > parent id, members
inside their node's SAX intervals, leaves partition the collection), and the CPU
oracle search over it equals a linear scan (the bound is sound)."""

import numpy as np
import pytest

from oracle import leafi_oracle as lo


def _tree(n=6000, m=64, cap=100, seed=3):
    from paper_2502_01836_b200.isax import build_isax_index

    data = lo.randwalk(n, m, seed)
    return data, build_isax_index(data, cap)


def _oracle_tree(t):
    ot = lo.OracleTree(t.values.astype(np.float64), t.starts, t.widths, t.max_leaf_size)
    for i in range(t.n_nodes):
        ot.env_min.append(t.env_min[i]); ot.env_max.append(t.env_max[i])
        ot.left.append(int(t.left[i])); ot.right.append(int(t.right[i]))
        ot.split_seg.append(int(t.split_seg[i])); ot.split_thr.append(float(t.split_thr[i]))
        ot.member_lists.append(None if t.left[i] >= 0 else [])
        ot.size.append(int(t.size[i])); ot.oversized.append(bool(t.oversized[i]))
    ot.members = {int(l): t.leaf_members(int(l)) for l in t.leaf_ids}
    return ot


def test_isax_structure():
    from paper_2502_01836_b200.index import segment_means

    data, t = _tree()
    summ = segment_means(data, 8)
    seen = np.concatenate([t.leaf_members(int(l)) for l in t.leaf_ids])
    assert np.array_equal(np.sort(seen), np.arange(data.shape[0]))
    for nid in range(t.n_nodes):
        if t.left[nid] >= 0:
            for c in (t.left[nid], t.right[nid]):
                assert c > nid
                assert (t.env_min[c] >= t.env_min[nid]).all() and (t.env_max[c] <= t.env_max[nid]).all()
        else:
            mem = t.leaf_members(nid)
            assert (np.diff(mem) > 0).all()
            assert t.size[nid] == mem.shape[0] and (mem.shape[0] <= t.max_leaf_size or t.oversized[nid])
            s = summ[mem]
            assert (s >= t.env_min[nid]).all() and (s <= t.env_max[nid]).all()
    # SAX intervals: every finite envelope bound is a standard-normal breakpoint
    from paper_2502_01836_b200.isax import breakpoint

    bps = {breakpoint(b, j) for b in range(1, 9) for j in range(1, 1 << b)}
    fin = t.env_min[np.isfinite(t.env_min)]
    assert all(float(x) in bps for x in np.unique(fin))


def test_isax_oracle_search_exact():
    data, t = _tree()
    ot = _oracle_tree(t)
    Q = lo.noisy_queries(data, 12, 0.3, 9)
    for q in Q:
        o = lo.search(ot, q, 3)
        ls = lo.linear_scan(data, q, 3)
        assert [a for a, _ in o.results] == [a for a, _ in ls]
        assert o.stats["series_scanned"] < data.shape[0]


def test_isax_degenerate_rows_terminate():
    from paper_2502_01836_b200.isax import build_isax_index

    data = np.repeat(lo.randwalk(3, 32, 1), 200, axis=0)      # 3 distinct rows, 200 copies each
    t = build_isax_index(data, 50, max_bits=4)
    assert t.has_oversized_leaves()
    assert sum(int(t.size[l]) for l in t.leaf_ids) == data.shape[0]


def test_gaussian_mixture_and_recall():
    from paper_2502_01836_b200.synth import gaussian_mixture, recall_at_k

    a = gaussian_mixture(5000, 96, 7, n_centers=20)
    b = gaussian_mixture(5000, 96, 7, n_centers=20)
    assert np.array_equal(a, b) and a.shape == (5000, 96)
    assert np.array_equal(a.astype(np.float32).astype(np.float64), a)
    assert recall_at_k(np.array([[1, 2, 3]]), np.array([[3, 2, 9]]))[0] == pytest.approx(2 / 3)
