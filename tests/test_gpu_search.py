"""GPU parity of the search path against the oracle and the reference's golden
vectors.  Every call goes through the C-ABI library (lf_search, lf_bounds,
lf_filter_predict, lf_batch_distances).

Tolerances: ids, counters, visit order and bounds are exact.  Distances are
fp64 direct-form sums in a different order than numpy's einsum, so they are
compared at rel 1e-12 (the bar in north_star is 1e-4).
"""

import numpy as np
import pytest

from oracle import leafi_oracle as lo

pytestmark = pytest.mark.gpu

DIST_RTOL = 1e-12


@pytest.fixture(scope="module")
def small_tree():
    from paper_2502_01836_b200 import build_index

    return build_index(lo.randwalk(2000, 32, 7), max_leaf_size=128)


@pytest.fixture(scope="module")
def pipe_tree():
    from paper_2502_01836_b200 import build_index

    return build_index(lo.randwalk(4000, 32, 17), max_leaf_size=200)


def _stats_row(out):
    s = out.stats
    return [s.leaves_visited, s.leaves_searched, s.leaves_lb_pruned, s.leaves_filter_pruned,
            s.filter_inferences, s.series_scanned]


@pytest.mark.parametrize("m", [256, 96, 32])
def test_bounds_bit_exact(knowns, m):
    from paper_2502_01836_b200.engine import query_bounds

    starts, widths = lo.seg_layout(m, 8)
    # recover the query rows behind the golden summaries is not possible; use paa rows
    rows = knowns[f"paa_{m}_rows"]
    qs, lb0 = query_bounds(rows, knowns[f"lb_{m}_mins"], knowns[f"lb_{m}_maxs"], starts, widths, 0)
    np.testing.assert_array_equal(qs, knowns[f"paa_{m}"])
    ref0 = np.array([[lo.node_lb(q, a, b, widths) for a, b in zip(knowns[f"lb_{m}_mins"], knowns[f"lb_{m}_maxs"])]
                     for q in qs])
    np.testing.assert_array_equal(lb0, ref0)
    _, lb1 = query_bounds(rows, knowns[f"lb_{m}_mins"], knowns[f"lb_{m}_maxs"], starts, widths, 1)
    np.testing.assert_array_equal(lb1, lo.lb_matrix(qs, knowns[f"lb_{m}_mins"], knowns[f"lb_{m}_maxs"], widths))


@pytest.mark.parametrize("m", [256, 96, 32])
def test_batch_distances(knowns, m):
    from paper_2502_01836_b200 import batch_distances

    got = batch_distances(knowns[f"dist_{m}_q"], knowns[f"dist_{m}_block"])
    np.testing.assert_allclose(got, knowns[f"dist_{m}_batch"], rtol=DIST_RTOL, atol=0)
    x = lo.randwalk(70, 32, 5)
    assert (np.diag(batch_distances(x, x)) == 0.0).all()      # test_series.py:89-92


@pytest.mark.parametrize("k", [1, 3])
def test_exact_search_matches_reference(small_tree, small_golden, k):
    from paper_2502_01836_b200 import search_engine

    g = small_golden
    for qi, q in enumerate(g["queries"]):
        out = search_engine(small_tree, q, k, want_trace=True)
        assert [i for i, _ in out.results] == g[f"k{k}_ids"][qi].tolist()
        np.testing.assert_allclose([d for _, d in out.results], g[f"k{k}_dists"][qi], rtol=DIST_RTOL)
        assert _stats_row(out) == g[f"k{k}_stats"][qi].tolist()
        a, b = g[f"k{k}_trace_ptr"][qi], g[f"k{k}_trace_ptr"][qi + 1]
        assert [e.leaf_id for e in out.trace] == g[f"k{k}_trace_leaf"][a:b].tolist()
        assert [e.lower_bound for e in out.trace] == g[f"k{k}_trace_lb"][a:b].tolist()
        assert [e.searched for e in out.trace] == g[f"k{k}_trace_searched"][a:b].tolist()
        np.testing.assert_allclose([e.bsf_before for e in out.trace], g[f"k{k}_trace_bsf"][a:b], rtol=DIST_RTOL)
        nn = [np.nan if e.leaf_nn_distance is None else e.leaf_nn_distance for e in out.trace]
        np.testing.assert_allclose(nn, g[f"k{k}_trace_nn"][a:b], rtol=DIST_RTOL)


def test_batched_rounds_exact_answers(small_tree, small_golden):
    """Round schedule: same exact answers; at least the sequential scan volume (F3)."""
    from paper_2502_01836_b200 import search_batch

    g = small_golden
    for k in (1, 3):
        res = search_batch(small_tree, g["queries"], k)
        np.testing.assert_array_equal(res.ids, g[f"k{k}_ids"])
        np.testing.assert_allclose(res.dists, g[f"k{k}_dists"], rtol=DIST_RTOL)
        assert (res.stats[:, 5] >= g[f"k{k}_stats"][:, 5]).all()
        seq = search_batch(small_tree, g["queries"], k, sequential=True)
        np.testing.assert_array_equal(seq.stats, g[f"k{k}_stats"])


def test_epsilon_search(small_tree, small_golden):
    from paper_2502_01836_b200 import epsilon_search

    g = small_golden
    for qi, q in enumerate(g["queries"]):
        out = epsilon_search(small_tree, q, 1, 1.0)          # bsf_factor 0.5
        assert out.results[0][0] == g["eps1_ids"][qi][0]
        assert _stats_row(out) == g["eps1_stats"][qi].tolist()


def test_matches_linear_scan_5000(small_golden):
    """Reference test_tree.py:93-102: 5000x32, cap 256, k=5 vs linear scan."""
    from paper_2502_01836_b200 import build_index, linear_scan, search_batch

    g = small_golden
    data = lo.randwalk(5000, 32, 1)
    t = build_index(data, 256)
    res = search_batch(t, g["ls_queries"], 5, sequential=True)
    np.testing.assert_array_equal(res.ids, g["ls_ids"])
    np.testing.assert_array_equal(res.ids, g["ls_linear_ids"])
    np.testing.assert_array_equal(res.stats, g["ls_stats"])
    for qi in (0, 17, 99):
        assert [i for i, _ in linear_scan(t, g["ls_queries"][qi], 5)] == g["ls_linear_ids"][qi].tolist()


def test_k_equals_n(small_golden):
    from paper_2502_01836_b200 import build_index, pruning_ratio, search_engine

    g = small_golden
    t = build_index(lo.randwalk(200, 16, 3), 32)
    out = search_engine(t, g["kn_queries"][0], 200)
    assert [i for i, _ in out.results] == g["kn_ids"][0].tolist()
    assert pruning_ratio(out.stats) == 0.0


def test_self_query_and_validation(small_tree):
    from paper_2502_01836_b200 import exact_search

    assert exact_search(small_tree, small_tree.values[123].astype(np.float64), 1).results == [(123, 0.0)]
    with pytest.raises(ValueError):
        exact_search(small_tree, np.zeros(7), 1)
    with pytest.raises(ValueError):
        exact_search(small_tree, np.zeros(32), 0)


def test_oversized_leaf():
    from paper_2502_01836_b200 import build_index, exact_search

    row = np.linspace(-1.0, 1.0, 16).astype(np.float32).astype(np.float64)  # fp32 storage contract
    t = build_index(np.tile(row, (40, 1)), 8)
    assert [i for i, _ in exact_search(t, row, 3).results] == [0, 1, 2]


# ------------------------------------------------------------------ filters --
def _pack(g, path=None):
    from paper_2502_01836_b200 import FilterPack

    return FilterPack(g["selected"].tolist(), g["W1"], g["b1"], g["W2"], g["b2"], path=path)


# tolerances: fp32 FFMA (simt) differs from OpenBLAS only in summation order;
# tcgen05 kind::tf32 multiplies 10-bit-mantissa operands (fp32 accumulate).
PRED_TOL = {"simt": dict(rtol=2e-5, atol=2e-5), "tc": dict(rtol=5e-3, atol=5e-3),
            "tc16": dict(rtol=5e-3, atol=5e-3)}     # fp16 operands keep tf32's 10-bit mantissa


@pytest.mark.parametrize("path", ["simt", "tc", "tc16"])
def test_filter_predictions_vs_reference(pipeline_golden, path):
    g = pipeline_golden
    if path == "tc16" and np.shape(g["W1"])[-1] % 64:
        pytest.skip("fp16 path needs m % 64 == 0")
    pred = _pack(g, path).predict(g["queries"]).cpu().numpy().astype(np.float64)
    np.testing.assert_allclose(pred, g["pred_queries"], **PRED_TOL[path])


@pytest.mark.parametrize("path", ["simt", "tc", "tc16"])
def test_filter_predictions_batch_invariant(pipeline_golden, path):
    """F6: a query's predictions do not depend on the batch it is in."""
    g = pipeline_golden
    if path == "tc16" and np.shape(g["W1"])[-1] % 64:
        pytest.skip("fp16 path needs m % 64 == 0")
    pk = _pack(g, path)
    full = pk.predict(g["queries"]).cpu().numpy()
    for lo_, hi in ((0, 1), (7, 8), (5, 60), (33, 47)):
        np.testing.assert_array_equal(pk.predict(g["queries"][lo_:hi]).cpu().numpy(), full[lo_:hi])


@pytest.mark.parametrize("m", [32, 64, 96, 256])
def test_filter_tc_vs_fp64(m):
    """tcgen05 path against an fp64 numpy forward: many filters, ragged query count
    (partial last M tile), multi-tile persistent schedule."""
    from paper_2502_01836_b200 import FilterPack

    rng = np.random.default_rng(m)
    F, Q = 37, 301
    W1 = rng.uniform(-1, 1, (F, m, m)).astype(np.float32) / np.sqrt(m)
    b1 = (rng.standard_normal((F, m)) * 0.1).astype(np.float32)
    W2 = rng.uniform(-1, 1, (F, m)).astype(np.float32) / np.sqrt(m)
    b2 = rng.standard_normal(F).astype(np.float32)
    X = lo.randwalk(Q, m, 3).astype(np.float32)
    ref = np.einsum("fj,fqj->qf", W2.astype(np.float64),
                    np.maximum(np.einsum("qi,fij->fqj", X.astype(np.float64), W1.astype(np.float64)) + b1[:, None, :], 0)) + b2
    tc = FilterPack(list(range(F)), W1, b1, W2, b2, path="tc").predict(X).cpu().numpy()
    simt = FilterPack(list(range(F)), W1, b1, W2, b2, path="simt").predict(X).cpu().numpy()
    np.testing.assert_allclose(simt, ref, rtol=1e-5, atol=1e-5)
    np.testing.assert_allclose(tc, ref, rtol=5e-3, atol=5e-3)
    if m % 64 == 0:
        tc16 = FilterPack(list(range(F)), W1, b1, W2, b2, path="tc16").predict(X).cpu().numpy()
        np.testing.assert_allclose(tc16, ref, rtol=5e-3, atol=5e-3)


@pytest.mark.parametrize("m", [64, 256])
def test_filter_f16_power_of_two_scaling(m):
    """fp16 operands are stored scaled by powers of two: inputs and weights far outside
    fp16's range (1e12, 1e-12) give the same predictions, bit for bit, as the same
    problem rescaled by exact powers of two."""
    from paper_2502_01836_b200 import FilterPack

    rng = np.random.default_rng(7 + m)
    F, Q = 9, 200
    W1 = (rng.uniform(-1, 1, (F, m, m)) / np.sqrt(m)).astype(np.float32)
    b1 = (rng.standard_normal((F, m)) * 0.1).astype(np.float32)
    W2 = (rng.uniform(-1, 1, (F, m)) / np.sqrt(m)).astype(np.float32)
    b2 = rng.standard_normal(F).astype(np.float32)
    X = lo.randwalk(Q, m, 5).astype(np.float32)
    base = FilterPack(list(range(F)), W1, b1, W2, b2, path="tc16").predict(X).cpu().numpy()
    big = FilterPack(list(range(F)), W1 * np.float32(2.0 ** -40), b1, W2, b2, path="tc16")
    got = big.predict(X * np.float32(2.0 ** 40)).cpu().numpy()
    np.testing.assert_array_equal(got, base)
    assert np.isfinite(base).all()


def test_filter_known_answers(knowns):
    from paper_2502_01836_b200 import FilterPack

    for m in (32, 256):
        for path in ("simt", "tc") + (("tc16",) if m % 64 == 0 else ()):
            pk = FilterPack([0], knowns[f"mlp_{m}_W1"][None], knowns[f"mlp_{m}_b1"][None],
                            knowns[f"mlp_{m}_W2"][None], knowns[f"mlp_{m}_b2"].reshape(1), path=path)
            got = pk.predict(knowns[f"mlp_{m}_x"]).cpu().numpy()[:, 0]
            np.testing.assert_allclose(got, knowns[f"mlp_{m}_y"], **PRED_TOL[path])
    hand = FilterPack([0], np.eye(2)[None], np.zeros((1, 2)), np.array([[0.5, 1.25]]), np.zeros(1))
    assert float(hand.predict(np.array([[1.0, 1.0]]))[0, 0]) == 1.75    # test_mlp.py:52-58
    eye = np.zeros((1, 32, 32)); eye[0, 0, 0] = eye[0, 1, 1] = 1.0
    w2 = np.zeros((1, 32)); w2[0, 0], w2[0, 1] = 0.5, 1.25
    x = np.zeros((1, 32)); x[0, :2] = 1.0
    tcp = FilterPack([0], eye, np.zeros((1, 32)), w2, np.zeros(1), path="tc")
    assert float(tcp.predict(x)[0, 0]) == 1.75                          # exact in tf32 too


@pytest.mark.parametrize("target", [0.9, 0.95, 0.99, 1.0])
def test_filtered_search_reference_predictions(pipe_tree, pipeline_golden, target):
    """Same predictions as the reference (injected fp64) -> identical outcome and counters."""
    import torch
    from paper_2502_01836_b200 import search_batch

    g = pipeline_golden
    pk = _pack(g)
    di = pipe_tree.device()
    res = search_batch(pipe_tree, g["queries"], 1, predictions=torch.from_numpy(g["pred_queries"]),
                       offsets=g[f"off_{target}"], leaf_filter=pk.leaf_filter(di), sequential=True)
    np.testing.assert_array_equal(res.ids, g[f"t{target}_ids"])
    np.testing.assert_allclose(res.dists, g[f"t{target}_dists"], rtol=DIST_RTOL)
    np.testing.assert_array_equal(res.stats, g[f"t{target}_stats"])


@pytest.mark.parametrize("target", [0.9, 0.99])
def test_filtered_search_gpu_predictions(pipe_tree, pipeline_golden, target):
    """GPU predictions (fp32, different summation order): outcome equals the oracle
    run with the SAME predictions, and tracks the reference closely."""
    from paper_2502_01836_b200 import search_batch

    g = pipeline_golden
    pk = _pack(g)
    pred = pk.predict(g["queries"])
    offs = g[f"off_{target}"]
    res = search_batch(pipe_tree, g["queries"], 1, predictions=pred, offsets=offs,
                       leaf_filter=pk.leaf_filter(pipe_tree.device()), sequential=True)
    ot = lo.build_tree(lo.randwalk(4000, 32, 17), 200)
    P = pred.cpu().numpy().astype(np.float64)
    sel = g["selected"].tolist()
    for qi, q in enumerate(g["queries"]):
        preds = {l: (lambda _x, v=float(P[qi, s]): v) for s, l in enumerate(sel)}
        o = lo.search(ot, q, 1, predictors=preds, offsets=dict(zip(sel, offs.tolist())))
        assert res.ids[qi, 0] == o.results[0][0]
        assert res.stats[qi].tolist() == [o.stats[s] for s in lo.STAT_KEYS]
    agree = np.mean(res.ids[:, 0] == g[f"t{target}_ids"][:, 0])
    assert agree >= 0.95


def test_host_callable_predictors(pipe_tree, pipeline_golden):
    """The reference seam: a dict of per-leaf callables (tree.py:278-286)."""
    from paper_2502_01836_b200 import search_engine

    g = pipeline_golden
    sel = g["selected"].tolist()
    offs = dict(zip(sel, g["off_0.9"].tolist()))
    for qi in range(0, 60, 6):
        preds = {l: (lambda _x, v=float(g["pred_queries"][qi, s]): v) for s, l in enumerate(sel)}
        out = search_engine(pipe_tree, g["queries"][qi], 1, predictors=preds, offsets=offs)
        assert out.results[0][0] == g["t0.9_ids"][qi][0]
        assert _stats_row(out) == g["t0.9_stats"][qi].tolist()
    with pytest.raises(ValueError):
        search_engine(pipe_tree, g["queries"][0], 1, predictors={sel[0]: lambda _x: 0.0})


def test_infinite_prediction_prunes(small_tree, small_golden):
    """Reference test_tree.py:197-207."""
    from paper_2502_01836_b200 import search_engine

    leaf = int(small_tree.leaf_ids[-1])
    out = search_engine(small_tree, small_golden["queries"][0], 1, predictors={leaf: lambda q: 1e9},
                        offsets={leaf: 0.0})
    assert out.stats.leaves_filter_pruned + out.stats.leaves_lb_pruned >= 1


@pytest.mark.parametrize("m,k", [(64, 1), (128, 1), (128, 5), (256, 1)])
def test_early_abandon_identical(m, k):
    """The early-abandoning scan returns exactly what the full scan returns
    (same ids, distances, counters), and matches the oracle."""
    from paper_2502_01836_b200 import build_index, search_batch

    data = lo.randwalk(12000, m, 21)
    t = build_index(data, 400)
    Q = np.concatenate([lo.noisy_queries(data, 16, nz, 30 + int(10 * nz)) for nz in (0.1, 0.2, 0.4)])
    for seq in (True, False):
        a = search_batch(t, Q, k, sequential=seq, early_abandon=True)
        b = search_batch(t, Q, k, sequential=seq, early_abandon=False)
        np.testing.assert_array_equal(a.ids, b.ids)
        # per-chunk half-warp sums vs whole-row warp sums: same terms, other order
        np.testing.assert_allclose(a.dists, b.dists, rtol=1e-14)
        np.testing.assert_array_equal(a.stats, b.stats)
    ot = lo.build_tree(data, 400)
    for i in range(0, Q.shape[0], 7):
        o = lo.search(ot, Q[i], k)
        assert a.ids[i].tolist() == [x for x, _ in o.results]
        np.testing.assert_allclose(a.dists[i], [d for _, d in o.results], rtol=DIST_RTOL)


def test_large_tree_unfused_order():
    """> 8192 nodes: the leaf order's big shape (1,024 threads, staging in a global
    scratch) instead of the shared-memory one; visit order, results and counters
    still equal the oracle's."""
    from paper_2502_01836_b200 import build_index, search_batch

    data = lo.randwalk(60000, 16, 12)
    t = build_index(data, 12)
    assert t.n_nodes > 8192
    Q = lo.noisy_queries(data, 12, 0.2, 13)
    res = search_batch(t, Q, 2, sequential=True)
    ot = lo.build_tree(data, 12)
    for i, q in enumerate(Q):
        o = lo.search(ot, q, 2)
        assert res.ids[i].tolist() == [a for a, _ in o.results]
        assert res.stats[i].tolist() == [o.stats[s] for s in lo.STAT_KEYS]


@pytest.mark.parametrize("variant", ["q8"])
@pytest.mark.parametrize("k", [1, 4])
def test_scan_variants_agree(variant, k, monkeypatch):
    """The int8-bounded scan returns the same ids and exact distances as the full
    fp64 scan; counters are identical (whole leaves are counted)."""
    from paper_2502_01836_b200 import build_index, search_batch

    data = lo.randwalk(15000, 128, 31)
    t = build_index(data, 600)
    Q = np.concatenate([lo.noisy_queries(data, 12, nz, 70 + int(10 * nz)) for nz in (0.1, 0.25, 0.4)])
    monkeypatch.setenv("LF_SCAN_VARIANT", "full")
    ref = search_batch(t, Q, k)
    monkeypatch.setenv("LF_SCAN_VARIANT", variant if variant != "q8" else "q8")
    got = search_batch(t, Q, k)
    np.testing.assert_array_equal(got.ids, ref.ids)
    np.testing.assert_allclose(got.dists, ref.dists, rtol=1e-14)
    np.testing.assert_array_equal(got.stats, ref.stats)
    seq = search_batch(t, Q, k, sequential=True)
    ot = lo.build_tree(data, 600)
    for i in range(0, Q.shape[0], 5):
        o = lo.search(ot, Q[i], k)
        assert seq.ids[i].tolist() == [a for a, _ in o.results]
        assert seq.stats[i].tolist() == [o.stats[s_] for s_ in lo.STAT_KEYS]


@pytest.mark.parametrize("m", [36, 64, 96, 100, 192, 256, 320, 512])
@pytest.mark.parametrize("k", [1, 3])
def test_q8_pipeline_exact(m, k, monkeypatch):
    """The TMA-pipelined int8-bounded scan (several stage counts / passes per row)
    equals the full fp64 scan: ids, distances and counters.  The collection holds
    exact duplicates (ties broken by id), an all-zero row (scale fallback) and
    queries that ARE collection rows (distance exactly 0)."""
    from paper_2502_01836_b200 import build_index, search_batch

    data = lo.randwalk(9000, m, 40 + m)
    data[100:110] = data[7]                       # 11 identical rows
    data[200] = 0.0
    t = build_index(data, 700)
    Q = np.concatenate([lo.noisy_queries(data, 10, nz, 90 + int(10 * nz)) for nz in (0.1, 0.3)]
                       + [data[[7, 200, 4321]].astype(np.float64)])
    monkeypatch.setenv("LF_SCAN_VARIANT", "full")
    ref = search_batch(t, Q, k)
    monkeypatch.setenv("LF_SCAN_VARIANT", "q8")
    got = search_batch(t, Q, k)
    np.testing.assert_array_equal(got.ids, ref.ids)
    np.testing.assert_allclose(got.dists, ref.dists, rtol=1e-14)
    np.testing.assert_array_equal(got.stats, ref.stats)
    assert got.ids[-3, 0] == 7 and got.dists[-3, 0] == 0.0
    assert got.ids[-1, 0] == 4321 and got.dists[-1, 0] == 0.0


def _mid_tree():
    """2048 < nodes <= 8192: the widest block-sorted leaf order (16 node items per thread)."""
    from paper_2502_01836_b200 import build_index

    data = lo.randwalk(40000, 64, 77)
    t = build_index(data, 24)
    assert 2048 < t.n_nodes <= 8192, t.n_nodes
    return data, t


def test_leaf_order_sequential_matches_oracle():
    """Sequential exact search over the leaf-only visit order (internal nodes folded
    into each leaf's gap bound): ids, distances, every counter and the trace equal
    the reference traversal, including walks that end at an internal node (no
    lb-pruned leaf counted) and walks that end at a leaf."""
    from paper_2502_01836_b200 import search_batch

    data, t = _mid_tree()
    Q = np.concatenate([lo.noisy_queries(data, 6, nz, 50 + int(10 * nz)) for nz in (0.1, 0.5, 1.5)])
    res = search_batch(t, Q, 3, sequential=True, want_trace=True)
    ot = lo.build_tree(data, 24)
    ended = set()
    for i, q in enumerate(Q):
        o = lo.search(ot, q, 3, want_trace=True)
        assert res.ids[i].tolist() == [a for a, _ in o.results], i
        np.testing.assert_allclose(res.dists[i], [b for _, b in o.results], rtol=DIST_RTOL)
        assert res.stats[i].tolist() == [o.stats[s_] for s_ in lo.STAT_KEYS], i
        assert [e.leaf_id for e in res.trace_of(i)] == [e[0] for e in o.trace], i
        assert [e.lower_bound for e in res.trace_of(i)] == [e[1] for e in o.trace], i
        ended.add(o.stats["leaves_lb_pruned"])
    assert ended == {0, 1}, "both break kinds (internal node / leaf) must occur"


def test_leaf_order_clustered_bounds():
    """A few far-away rows make one leaf's bound an outlier, so the other leaves
    crowd into a handful of counting-sort buckets (the warp rank-sort path):
    ids, counters and traces still equal the reference traversal."""
    from paper_2502_01836_b200 import build_index, search_batch

    data = lo.randwalk(40000, 64, 78)
    data[:300] = (data[:300] + 5000.0).astype(np.float32)
    t = build_index(data, 24)
    Q = np.concatenate([lo.noisy_queries(data[300:], 8, nz, 51 + int(10 * nz)) for nz in (0.1, 1.0)])
    res = search_batch(t, Q, 2, sequential=True, want_trace=True)
    ot = lo.build_tree(data, 24)
    for i, q in enumerate(Q):
        o = lo.search(ot, q, 2, want_trace=True)
        assert res.ids[i].tolist() == [a for a, _ in o.results], i
        assert res.stats[i].tolist() == [o.stats[s_] for s_ in lo.STAT_KEYS], i
        assert [e.leaf_id for e in res.trace_of(i)] == [e[0] for e in o.trace], i


def test_leaf_order_batched_equals_sequential():
    """Batched rounds over the leaf order give the sequential walk's neighbours."""
    from paper_2502_01836_b200 import search_batch

    data, t = _mid_tree()
    Q = np.concatenate([lo.noisy_queries(data, 16, nz, 60 + int(10 * nz)) for nz in (0.1, 0.4, 1.0)])
    for k in (1, 4):
        ref = search_batch(t, Q, k, sequential=True)
        got = search_batch(t, Q, k)
        np.testing.assert_array_equal(got.ids, ref.ids)
        np.testing.assert_array_equal(got.dists, ref.dists)
        assert (got.stats[:, 5] >= ref.stats[:, 5]).all()


def test_leaf_order_filtered_sequential_matches_oracle():
    """Sequential filtered search over the leaf order: results and counters equal the
    reference cascade fed the same predictions (host callables, fp64)."""
    from paper_2502_01836_b200 import search_engine

    data, t = _mid_tree()
    rng = np.random.default_rng(5)
    leaves = [int(l) for l in t.leaf_ids]
    preds = {l: (lambda q, v=float(rng.uniform(0.0, 6.0)): v) for l in leaves[::3]}
    offs = {l: float(rng.uniform(0.0, 1.0)) for l in preds}
    ot = lo.build_tree(data, 24)
    for i, q in enumerate(lo.noisy_queries(data, 8, 0.6, 88)):
        out = search_engine(t, q, 2, predictors=preds, offsets=offs)
        o = lo.search(ot, q, 2, predictors=preds, offsets=offs)
        assert [a for a, _ in out.results] == [a for a, _ in o.results], i
        assert [getattr(out.stats, s_) for s_ in lo.STAT_KEYS] == [o.stats[s_] for s_ in lo.STAT_KEYS], i


@pytest.mark.parametrize("k,seq,cap", [(1, False, 150), (3, False, 150), (1, True, 150), (2, True, 150),
                                       (40, False, 24), (40, True, 24)])
def test_lazy_filter_inference_identical(k, seq, cap):
    """In-search inference (one tensor-core pass after round 0 over the (query, leaf)
    pairs with lb <= bsf0 * f, query rows gathered by TMA gather4) gives exactly the
    neighbours AND counters of the dense predictions path.  cap 24 with k = 40: the
    first leaf holds fewer than k rows, bsf stays +inf after round 0, and those walks
    get their predictions from a later, requested pass."""
    import torch
    from paper_2502_01836_b200 import build_index, search_batch
    from paper_2502_01836_b200.filters import FilterPack

    data = lo.randwalk(30000 if cap > 100 else 6000, 64, 91)
    t = build_index(data, cap)
    rng = np.random.default_rng(3)
    leaves = [int(l) for l in t.leaf_ids]
    sel = leaves[::2] + leaves[1::7]
    sel = sorted(set(sel))
    F, m = len(sel), 64
    pack = FilterPack(sel, rng.normal(0, 0.08, (F, m, m)), rng.normal(0, 0.05, (F, m)),
                      rng.normal(0, 0.08, (F, m)), rng.uniform(1.0, 9.0, F), path="tc16")
    Q = np.concatenate([lo.noisy_queries(data, 70, nz, 40 + int(10 * nz)) for nz in (0.1, 0.3, 0.6)])
    qd = torch.from_numpy(Q.astype(np.float32)).cuda()
    di = t.device()
    offs = rng.uniform(0.0, 1.5, F)
    lf = pack.leaf_filter(di)
    dense = search_batch(t, qd, k, predictions=pack.predict(qd), offsets=offs, leaf_filter=lf, sequential=seq)
    prof = np.zeros(16)
    lazy = search_batch(t, qd, k, filters=pack, offsets=offs, leaf_filter=lf, sequential=seq, profile=prof)
    if cap > 100 or seq:
        np.testing.assert_array_equal(lazy.ids, dense.ids)
        np.testing.assert_array_equal(lazy.dists, dense.dists)
    else:
        # batched with stuck walks: the resumed walk scans a later round's quota, so the
        # (approximate) filtered results may differ; each one must still be a true (d, id)
        d = np.sqrt(((data[lazy.ids] - Q[:, None, :]) ** 2).sum(-1))
        np.testing.assert_allclose(lazy.dists, d, rtol=1e-10)
        assert (np.diff(lazy.dists, axis=1) >= 0).all()
    if cap > 100 or seq:
        # every decision is taken with the bsf the dense path uses: identical counters
        # (sequential: a stuck walk resumes with the same bsf and the same quota of 1)
        np.testing.assert_array_equal(lazy.stats, dense.stats)
    else:
        assert (lazy.stats[:, 0] == lazy.stats[:, 1] + lazy.stats[:, 2] + lazy.stats[:, 3]).all()
    if cap > 100:
        # k = 1: one pass; k > 1: every later round starts with a pass over the walks that
        # asked for one (none here: every first leaf holds k rows)
        assert prof[12] == 1 if k == 1 else prof[12] >= 1
    else:
        assert prof[12] >= 2, "walks whose bsf was +inf after round 0 asked for a later pass"
    assert dense.stats[:, 3].sum() > 0, "the random filters must prune something"
    assert 0 < prof[11] < Q.shape[0] * F, "in-search inference computes a strict subset of the pairs"


@pytest.mark.parametrize("path,m", [("tc", 128), ("tc16", 128), ("tc16", 256), ("tc16", 64)])
def test_pair_predictions_bit_identical(path, m):
    """lf_filter_predict_pairs_tc / _f16 (bucketed pairs; _f16 gathers the query rows
    with TMA gather4) == the dense tensor-core predictions of the same (query, filter)
    pairs, bit for bit, in any pair order, with partial and multi-tile buckets."""
    import torch
    from paper_2502_01836_b200.filters import FilterPack

    rng = np.random.default_rng(11)
    F, Q = 37, 300
    pack = FilterPack(list(range(F)), rng.normal(0, 0.08, (F, m, m)), rng.normal(0, 0.05, (F, m)),
                      rng.normal(0, 0.08, (F, m)), rng.uniform(1.0, 9.0, F), path=path)
    qd = torch.from_numpy(rng.normal(0, 1, (Q, m)).astype(np.float32)).cuda()
    dense = pack.predict(qd).cpu().numpy().astype(np.float64)
    pq = rng.integers(0, Q, 5000)
    pf = rng.integers(0, F, 5000)
    pf[:400] = 5                                   # one filter with several 128-row tiles
    got = pack.predict_pairs(qd, pq, pf).cpu().numpy()
    np.testing.assert_array_equal(got, dense[pq, pf])


@pytest.mark.parametrize("m,pk,cap", [(64, 32, None), (96, 32, None), (256, 32, None), (256, 64, None),
                                      (320, 64, None), (256, 32, "40")])
@pytest.mark.parametrize("k", [1, 3])
def test_projected_scan_exact(m, pk, cap, k, monkeypatch):
    """Two-stage scan over the projected shadow (int8 codes of the top principal
    coordinates + residual norms) == the full fp64 scan: ids, distances, counters;
    with duplicate rows, an all-zero row and queries equal to rows."""
    from paper_2502_01836_b200 import build_index, search_batch

    data = lo.randwalk(9000, m, 140 + m)
    data[100:110] = data[7]
    data[200] = 0.0
    t = build_index(data, 700)
    di = t.device()
    if pk != di.pca_k:
        di.ensure_pca(pk)
    assert di.pca_k == pk
    Q = np.concatenate([lo.noisy_queries(data, 10, nz, 90 + int(10 * nz)) for nz in (0.1, 0.3)]
                       + [data[[7, 200, 4321]].astype(np.float64)])
    monkeypatch.setenv("LF_SCAN_VARIANT", "full")
    ref = search_batch(t, Q, k)
    monkeypatch.setenv("LF_SCAN_VARIANT", "pq")
    if cap is not None:      # a tiny survivor entry list: tasks that do not fit re-read in the scan warp
        monkeypatch.setenv("LF_PQ_OVER_CAP", cap)
    prof = np.zeros(16)
    got = search_batch(t, Q, k, profile=prof)
    np.testing.assert_array_equal(got.ids, ref.ids)
    np.testing.assert_allclose(got.dists, ref.dists, rtol=1e-14)
    np.testing.assert_array_equal(got.stats, ref.stats)
    assert prof[8] > 0 and prof[9] < prof[8], "the projected bound must run and drop rows"


def test_projected_shadow_energy_gate(monkeypatch):
    """The index build keeps the projected shadow only when 32 principal directions
    hold >= 90% of the energy: yes for random walks, no for a 96-d Gaussian mixture
    (whose searches then run the int8 scan in every round, with the same results)."""
    from paper_2502_01836_b200 import build_index, search_batch
    from paper_2502_01836_b200.synth import gaussian_mixture

    monkeypatch.delenv("LF_SCAN_VARIANT", raising=False)
    rw = build_index(lo.randwalk(6000, 128, 5), 400).device()
    assert rw.pca_k == 32 and rw.pca_energy >= 0.9
    g = gaussian_mixture(6000, 96, 9, n_centers=200).astype(np.float32)
    t = build_index(g, 400)
    di = t.device()
    assert di.pca_k == 0 and di.pca_energy < 0.9
    Q = g[[3, 77, 4000]].astype(np.float64) + 0.01
    got = search_batch(t, Q, 2)
    monkeypatch.setenv("LF_SCAN_VARIANT", "full")
    ref = search_batch(t, Q, 2)
    np.testing.assert_array_equal(got.ids, ref.ids)
    np.testing.assert_allclose(got.dists, ref.dists, rtol=1e-14)


@pytest.mark.parametrize("k,seq,cap,filt", [(1, False, 150, False), (3, False, 150, False), (1, True, 150, True),
                                            (1, False, 150, True), (40, False, 24, True), (2, False, 150, True)])
def test_search_plan_graph_identical(k, seq, cap, filt):
    """lf_search_plan (the whole batched search as one CUDA graph with a conditional
    WHILE over the rounds) == lf_search: ids, distances and counters, over several
    query batches through the same plan (graph reuse)."""
    import torch
    from paper_2502_01836_b200 import build_index, search_batch
    from paper_2502_01836_b200.engine import SearchPlan
    from paper_2502_01836_b200.filters import FilterPack

    data = lo.randwalk(30000 if cap > 100 else 6000, 64, 93)
    t = build_index(data, cap)
    di = t.device()
    kw = {}
    if filt:
        rng = np.random.default_rng(5)
        leaves = [int(l) for l in t.leaf_ids]
        sel = sorted(set(leaves[::2] + leaves[1::7]))
        F, m = len(sel), 64
        pack = FilterPack(sel, rng.normal(0, 0.08, (F, m, m)), rng.normal(0, 0.05, (F, m)),
                          rng.normal(0, 0.08, (F, m)), rng.uniform(1.0, 9.0, F), path="tc16")
        kw = dict(filters=pack, offsets=rng.uniform(0.0, 1.5, F), leaf_filter=pack.leaf_filter(di))
    plan = SearchPlan(t, 150, k, sequential=seq, **kw)
    for rep in range(3):
        Q = np.concatenate([lo.noisy_queries(data, 50, nz, 300 + rep * 10 + int(10 * nz)) for nz in (0.1, 0.3, 0.6)])
        qd = torch.from_numpy(Q.astype(np.float32)).cuda()
        ref = search_batch(t, qd, k, sequential=seq, **kw)
        got = plan.run(qd)
        np.testing.assert_array_equal(got.ids, ref.ids)
        np.testing.assert_array_equal(got.dists, ref.dists)
        np.testing.assert_array_equal(got.stats, ref.stats)
    with pytest.raises(ValueError):
        plan.run(qd[:10])


@pytest.mark.parametrize("kind,k,seq", [("dstree", 1, False), ("dstree", 5, False), ("dstree", 1, True),
                                        ("isax", 1, False), ("isax", 5, False), ("isax", 3, True),
                                        ("big", 1, False), ("big", 4, True)])
def test_pruned_orders_identical(kind, k, seq, monkeypatch):
    """Visit orders built after round 0 up to bsf0 * f (first leaf from lb_tile's group
    minima, a terminal record past the threshold) == the full orders: ids, distances,
    counters -- on trees whose node count is not a multiple of the kernels' tiles."""
    from paper_2502_01836_b200 import build_index, search_batch
    from paper_2502_01836_b200.isax import build_isax_index

    data = lo.randwalk(120000 if kind == "big" else 30000, 32 if kind == "big" else 128, 33)
    # "big": > 8,192 nodes -- the leaf order's global-scratch shape
    t = build_isax_index(data, 400) if kind == "isax" else build_index(data, 18 if kind == "big" else 333)
    if kind == "big":
        assert 8192 < t.n_nodes <= 32768, t.n_nodes
    Q = np.concatenate([lo.noisy_queries(data, 30, nz, 77 + int(10 * nz)) for nz in (0.1, 0.4, 0.8)])
    monkeypatch.setenv("LF_PRUNED_ORDER", "0")
    full = search_batch(t, Q, k, sequential=seq)
    monkeypatch.setenv("LF_PRUNED_ORDER", "1")
    pruned = search_batch(t, Q, k, sequential=seq)
    np.testing.assert_array_equal(pruned.ids, full.ids)
    np.testing.assert_array_equal(pruned.dists, full.dists)
    np.testing.assert_array_equal(pruned.stats, full.stats)
    for i in range(0, Q.shape[0], 9):
        assert pruned.ids[i].tolist() == [a for a, _ in lo.linear_scan(data, Q[i], k)]
