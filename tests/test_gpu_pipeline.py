"""GPU parity of training-data generation (lf_bounds mode 1, lf_leaf_min_dist,
lf_local_min_dist) and of the LeaFi pipeline (batched training + calibration
with the search kernel) against the reference's golden vectors / outcomes."""

import json

import numpy as np
import pytest

from oracle import leafi_oracle as lo

pytestmark = pytest.mark.gpu
RTOL = 1e-12


@pytest.fixture(scope="module")
def small_tree():
    from paper_2502_01836_b200 import build_index

    return build_index(lo.randwalk(2000, 32, 7), max_leaf_size=128)


def test_collect_targets_small(small_tree, small_golden):
    from paper_2502_01836_b200.targets import collect_targets

    g = small_golden
    gts = collect_targets(small_tree, g["tg_selected"].tolist(), g["tg_queries"], 30)
    np.testing.assert_array_equal(gts.leaf_ids, g["tg_leaf_ids"])
    np.testing.assert_array_equal(gts.lb_matrix, g["tg_lb_matrix"])           # bit-exact bounds
    np.testing.assert_array_equal(gts.visit_order, g["tg_visit_order"])
    np.testing.assert_allclose(gts.dl_selected, g["tg_dl_selected"], rtol=RTOL)
    np.testing.assert_allclose(gts.dl_calib_full, g["tg_dl_calib_full"], rtol=RTOL)
    np.testing.assert_allclose(gts.nn_distance, g["tg_nn_distance"], rtol=RTOL)


def test_member_query_zero_target(small_tree):
    """Reference test_traingen.py:76-82."""
    from paper_2502_01836_b200.targets import collect_targets

    lid = int(small_tree.leaf_ids[0])
    row = small_tree.values[small_tree.leaf_members(lid)[0]].astype(np.float64)
    gts = collect_targets(small_tree, [lid], np.stack([row] * 3), 1)
    assert gts.dl_selected[0, 0] == 0.0


def test_local_targets(small_tree, small_golden):
    from paper_2502_01836_b200.synth import generate_local_queries
    from paper_2502_01836_b200.targets import LocalQueries, collect_local_targets

    g = small_golden
    lid = int(g["lq_leaf"])
    q, lv, src = generate_local_queries(small_tree, lid, 40, (0.1, 0.4), 4)
    np.testing.assert_array_equal(q, g["lq_queries"])
    np.testing.assert_array_equal(src, g["lq_sources"])
    loc = collect_local_targets(small_tree, LocalQueries(lid, q, lv, src))
    np.testing.assert_allclose(loc.targets, g["lq_targets"], rtol=RTOL)
    np.testing.assert_array_equal(loc.lbs, g["lq_lbs"])
    # zero noise -> exactly 0.0 (test_traingen.py:53-57)
    l0 = int(small_tree.leaf_ids[0])
    q0, lv0, s0 = generate_local_queries(small_tree, l0, 20, (0.0, 0.0), 5)
    assert (collect_local_targets(small_tree, LocalQueries(l0, q0, lv0, s0)).targets == 0.0).all()


def test_collect_targets_pipeline(pipeline_golden):
    from paper_2502_01836_b200 import build_index
    from paper_2502_01836_b200.targets import collect_targets

    g = pipeline_golden
    t = build_index(lo.randwalk(4000, 32, 17), 200)
    gts = collect_targets(t, g["selected"].tolist(), g["gq"], 60)
    np.testing.assert_array_equal(gts.lb_matrix, g["tg_lb_matrix"])
    np.testing.assert_array_equal(gts.visit_order, g["tg_visit_order"])
    np.testing.assert_allclose(gts.dl_selected, g["tg_dl_selected"], rtol=RTOL)
    np.testing.assert_allclose(gts.nn_distance, g["tg_nn_distance"], rtol=RTOL)


def test_collect_targets_m256_int8_vs_oracle():
    """Training-data generation at m = 256, where the int8 tensor-core kernel
    (lf_leaf_min_dist_q8 / lf_local_min_dist_q8) is the default path, against the
    CPU oracle's collect_targets (traingen.py:147-220) on the same tree: bounds and
    visit order bit-exact, every minimum distance within 1e-12 relative (fp64 direct
    form, another summation order), member queries exactly 0."""
    from paper_2502_01836_b200 import build_index
    from paper_2502_01836_b200.targets import collect_targets, default_path, local_targets_all

    data = lo.randwalk(24000, 256, 21)
    t = build_index(data, 600)
    assert default_path(t, t.device()) == "q8"
    gq, _ = lo.global_queries(data, 220, (0.1, 0.4), 5)
    gq = np.concatenate([gq, data[[5, 777, 23000]].astype(np.float64)])    # member queries
    ot = lo.build_tree(data, 600)
    sel = [int(l) for l in t.leaf_ids[::2]]
    got = collect_targets(t, sel, gq, 60)
    ref = lo.collect_targets(ot, sel, gq, 60)
    np.testing.assert_array_equal(got.lb_matrix, ref.lb_matrix)
    np.testing.assert_array_equal(got.visit_order, ref.visit_order)
    np.testing.assert_allclose(got.dl_selected, ref.dl_selected, rtol=1e-12, atol=0)
    np.testing.assert_allclose(got.dl_calib_full, ref.dl_calib_full, rtol=1e-12, atol=0)
    np.testing.assert_allclose(got.nn_distance, ref.nn_distance, rtol=1e-12, atol=0)
    assert (got.dl_calib_full[-3:].min(axis=1) == 0.0).all()
    lids = [int(l) for l in t.leaf_ids[:4]]
    qs = {l: lo.noisy_queries(data[ot.members[l]], 50, 0.2, 30 + l) for l in lids}
    loc = local_targets_all(t, qs)
    for l in lids:
        tg, lbs = lo.local_targets(ot, l, qs[l])
        np.testing.assert_allclose(loc[l][0], tg, rtol=1e-12, atol=0)
        np.testing.assert_array_equal(loc[l][1], lbs)


# -------------------------------------------------------------- pipeline --
FIXED = dict(t_series=2e-7, t_filter=6e-6, filter_bytes=5 * 1024)   # reference tests/conftest.py:11


@pytest.fixture(scope="module")
def pipe(pipeline_golden):
    """The reference conftest `pipeline` configuration, enhanced on the GPU."""
    from paper_2502_01836_b200 import build_index
    from paper_2502_01836_b200 import pipeline as pl
    from paper_2502_01836_b200.training import TrainConfig

    data = lo.randwalk(4000, 32, 17)
    t = build_index(data, 200)
    e = pl.enhance(t, pl.SplitPlan(240, 80, 60), pl.SelectionBudget(16 * 1024 * 1024), seed=23,
                   constants=pl.RuntimeConstants(**FIXED), train_cfg=TrainConfig(max_epochs=150))
    return {"data": data, "tree": t, "eidx": e, "queries": pipeline_golden["queries"]}


def test_pipeline_selection_matches_reference(pipe, pipeline_golden):
    assert pipe["eidx"].filter_leaf_ids == pipeline_golden["selected"].tolist()


def test_pipeline_exact_mode_equivalence(pipe):
    from paper_2502_01836_b200 import exact_search
    from paper_2502_01836_b200.pipeline import SearchRequest, search

    for q in pipe["queries"][:25]:
        a = search(pipe["eidx"], SearchRequest(query=q, k=1, exact=True))
        b = exact_search(pipe["tree"], q, 1)
        assert a.results == b.results and a.stats.series_scanned == b.stats.series_scanned


def test_pipeline_recall_and_pruning(pipe, pipeline_golden):
    """Recall at target and pruning comparable to the reference's own filters."""
    from paper_2502_01836_b200 import search_batch
    from paper_2502_01836_b200.pipeline import search_queries

    g = pipeline_golden
    Q = pipe["queries"]
    ex = search_batch(pipe["tree"], Q, 1)
    for target in (0.9, 0.99):
        res = search_queries(pipe["eidx"], Q, 1, target=target, sequential=True)
        hits = [lo.recall_at_1(res.results(i), int(ex.ids[i, 0]), float(ex.dists[i, 0])) for i in range(len(Q))]
        ours = float(np.mean(res.pruning_ratios()))
        ref = float(np.mean(1.0 - g[f"t{target}_stats"][:, 5] / 4000))
        ref_hits = np.mean(g[f"t{target}_ids"][:, 0] == g["exact_ids"][:, 0])
        assert np.mean(hits) >= min(target, ref_hits) - 0.05
        assert ours >= ref - 0.10
        assert (res.dists[:, 0] >= ex.dists[:, 0] - 1e-12).all()          # never beats exact


def test_pipeline_target_monotone(pipe):
    from paper_2502_01836_b200.pipeline import search_queries

    lo_ = search_queries(pipe["eidx"], pipe["queries"], 1, target=0.9, sequential=True)
    hi = search_queries(pipe["eidx"], pipe["queries"], 1, target=1.0, sequential=True)
    assert (hi.dists[:, 0] <= lo_.dists[:, 0]).all()


def test_pipeline_max_offset_coverage(pipe):
    """Offsets at alpha_max: recall 1.0 on the calibration queries (criterion 4),
    with the GPU search itself (not the replay)."""
    import torch
    from paper_2502_01836_b200 import search_batch

    e = pipe["eidx"]
    gts = e.global_set
    calib = gts.queries[gts.train_pool_size:]
    amax = np.array([e.curves[l].alpha_max for l in e.pack.leaf_ids])
    pred = e.pack.predict(calib)
    res = search_batch(e.base, calib, 1, predictions=pred, offsets=amax, leaf_filter=e.pack.leaf_filter(e.base.device()),
                       sequential=True)
    ex = search_batch(e.base, calib, 1)
    hits = [lo.recall_at_1(res.results(i), int(ex.ids[i, 0]), float(ex.dists[i, 0])) for i in range(len(calib))]
    assert np.mean(hits) == 1.0


def test_reference_filters_adopted(pipeline_golden):
    """A reference-trained filter set on the GPU path: predictions from lf_filter_predict,
    offsets from the reference curves; outcome equals the reference in >= 95% of queries."""
    from paper_2502_01836_b200 import build_index
    from paper_2502_01836_b200.calibration import QualityOffsetCurve
    from paper_2502_01836_b200.pipeline import EnhancedIndex, FilterModel, search_queries

    g = pipeline_golden
    t = build_index(lo.randwalk(4000, 32, 17), 200)
    sel = g["selected"].tolist()
    filters = {l: FilterModel(g["W1"][s], g["b1"][s], g["W2"][s], float(g["b2"][s])) for s, l in enumerate(sel)}
    curves = {l: QualityOffsetCurve(l, g[f"curve_{l}_alphas"], g[f"curve_{l}_kq"], g[f"curve_{l}_ko"],
                                    bool(g[f"curve_{l}_deg"])) for l in sel}
    e = EnhancedIndex(t, filters, curves)
    for target in (0.9, 0.99):
        np.testing.assert_array_equal(e.offset_vector(target), g[f"off_{target}"])
        res = search_queries(e, g["queries"], 1, target=target, sequential=True)
        assert np.mean(res.ids[:, 0] == g[f"t{target}_ids"][:, 0]) >= 0.95


@pytest.mark.parametrize("m,cap", [(32, 90), (64, 300), (256, 700)])
def test_mindist_tc_bit_identical(m, cap):
    """tcgen05 tf32 bound + exact fp64 re-check == fp64 SIMT kernel (same exact
    terms, other summation order: rel 1e-13), including ragged leaves, partial
    query tiles and member queries (exact zeros)."""
    from paper_2502_01836_b200 import build_index
    from paper_2502_01836_b200.targets import leaf_min_distances, local_targets_all

    data = lo.randwalk(9000, m, 4 + m)
    t = build_index(data, cap)
    Q = np.concatenate([lo.noisy_queries(data, 150, 0.2, 5), data[:37]])      # 187 queries
    slots = list(range(t.n_leaves))
    a = leaf_min_distances(t, Q, slots, path="tc").cpu().numpy()
    b = leaf_min_distances(t, Q, slots, path="simt").cpu().numpy()
    np.testing.assert_allclose(a, b, rtol=1e-13, atol=0)
    assert (a[150:].min(axis=1) == 0.0).all()
    lids = [int(l) for l in t.leaf_ids[:5]]
    qs = {l: lo.noisy_queries(data, 130 + l % 3, 0.3, l) for l in lids}
    ta = local_targets_all(t, qs, path="tc")
    tb = local_targets_all(t, qs, path="simt")
    for l in lids:
        np.testing.assert_allclose(ta[l][0], tb[l][0], rtol=1e-13, atol=0)


@pytest.mark.parametrize("path", ["q8"])
@pytest.mark.parametrize("m,cap", [(128, 300), (256, 700), (256, 3000)])
def test_mindist_q8_exact(m, cap, path):
    """int8 tensor-core bound + exact fp64 re-check == fp64 SIMT kernel (rel 1e-13),
    with ragged leaves (partial 256-row chunks), partial 128-query tiles, member
    queries (exact zeros), far queries and the local (grouped) variant."""
    from paper_2502_01836_b200 import build_index
    from paper_2502_01836_b200.targets import leaf_min_distances, local_targets_all

    data = lo.randwalk(12000, m, 9 + m)
    t = build_index(data, cap)
    assert t.device().X8 is not None
    Q = np.concatenate([lo.noisy_queries(data, 150, 0.2, 5), lo.noisy_queries(data, 40, 2.0, 6), data[:37]])
    slots = list(range(t.n_leaves))
    a = leaf_min_distances(t, Q, slots, path=path).cpu().numpy()
    b = leaf_min_distances(t, Q, slots, path="simt").cpu().numpy()
    np.testing.assert_allclose(a, b, rtol=1e-13, atol=0)
    assert (a[190:].min(axis=1) == 0.0).all()
    lids = [int(l) for l in t.leaf_ids[:6]]
    qs = {l: lo.noisy_queries(data, 130 + l % 3, 0.3, l) for l in lids}
    ta = local_targets_all(t, qs, path=path)
    tb = local_targets_all(t, qs, path="simt")
    for l in lids:
        np.testing.assert_allclose(ta[l][0], tb[l][0], rtol=1e-13, atol=0)


def test_sharded_tdg_columns_concatenate():
    """Training-data generation on leaf shards: the ranks' local column blocks, in
    rank order, are exactly the unsharded [Q, n_leaves] min-distance matrix."""
    import torch
    from paper_2502_01836_b200 import build_index
    from paper_2502_01836_b200.targets import leaf_min_distances, sharded_leaf_min_distances

    data = lo.randwalk(15000, 128, 17)
    t = build_index(data, 400)
    Q = np.concatenate([lo.noisy_queries(data, 100, 0.3, 8), data[5:9]])
    full = leaf_min_distances(t, Q, list(range(t.n_leaves))).cpu().numpy()
    for world in (2, 3):
        parts, prev = [], 0
        for r in range(world):
            loc, _, (a, b) = sharded_leaf_min_distances(t, Q, r, world, gather=False)
            assert a == prev and loc.shape == (Q.shape[0], b - a)
            parts.append(loc.cpu().numpy())
            prev = b
        assert prev == t.n_leaves
        np.testing.assert_array_equal(np.concatenate(parts, axis=1), full)
    _, g1, _ = sharded_leaf_min_distances(t, Q, 0, 1)
    np.testing.assert_array_equal(g1.cpu().numpy(), full)


def test_device_replay_bit_identical():
    """lf_replay_offsets == the host replay (conformal.py:171-198 twin) for many offset
    vectors (including an all-infinite one), and GPU-fitted curves equal host-fitted ones."""
    from paper_2502_01836_b200 import calibration as cal

    rng = np.random.default_rng(0)
    nq, L, F = 60, 40, 12
    lb = np.sort(rng.uniform(0, 5, (nq, L)), axis=1)
    dl = lb + rng.uniform(0, 3, (nq, L))
    slot = rng.integers(-1, F, (nq, L)).astype(np.int32)
    pred = np.where(slot >= 0, dl + rng.normal(0, 1, (nq, L)), np.nan)
    sk = cal.CalibrationSkeleton(lb, dl, pred, slot, dl.min(axis=1))
    rows = rng.uniform(0, 2, (97, F))
    rows[3] = np.inf
    dev = cal.DeviceReplay(sk)
    np.testing.assert_array_equal(dev(rows), cal.replay_many(sk, rows))
    alphas = {l: np.sort(rng.uniform(0, 2, nq))[::-1] for l in range(F)}
    a = cal.fit_auto_tuners(sk, alphas)
    b = cal.fit_auto_tuners(sk, alphas, replay=dev)
    for l in a:
        np.testing.assert_array_equal(a[l].knot_quality, b[l].knot_quality)
        np.testing.assert_array_equal(a[l].knot_offset, b[l].knot_offset)


@pytest.fixture(scope="module")
def pipe64():
    """A small m = 64 collection enhanced on the GPU: the fp16 pack (in-search inference)."""
    from paper_2502_01836_b200 import build_index
    from paper_2502_01836_b200 import pipeline as pl
    from paper_2502_01836_b200.training import TrainConfig

    data = lo.randwalk(6000, 64, 29)
    t = build_index(data, 200)
    e = pl.enhance(t, pl.SplitPlan(240, 80, 60), pl.SelectionBudget(16 * 1024 * 1024), seed=31,
                   constants=pl.RuntimeConstants(**FIXED), train_cfg=TrainConfig(max_epochs=60))
    return {"tree": t, "eidx": e, "queries": lo.noisy_queries(data, 96, 0.2, 37)}


def test_search_pipeline_matches_search_queries(pipe64):
    """pipeline.SearchPipeline (copies on their own streams, rotating slots) returns
    exactly search_queries' results and counters, batch by batch."""
    import torch

    from paper_2502_01836_b200.pipeline import SearchPipeline, search_queries

    e = pipe64["eidx"]
    assert e.pack.path == "tc16"
    Q = np.asarray(pipe64["queries"], dtype=np.float32)
    Qr = np.ascontiguousarray(Q[::-1])
    refs = [search_queries(e, Q, 1, target=0.99), search_queries(e, Qr, 1, target=0.99)]
    sp = SearchPipeline(e, Q.shape[0], 1, target=0.99, depth=2)
    batches = [torch.from_numpy(b).pin_memory() for b in (Q, Qr, Q, Qr, Q)]
    pending, outs = [], []
    for b in batches:
        pending.append(sp.submit(b))
        if len(pending) == 2:
            outs.append(sp.result(pending.pop(0)))
    outs.append(sp.result(pending.pop(0)))
    for j, r in enumerate(outs):
        ref = refs[j % 2]
        np.testing.assert_array_equal(r.ids, ref.ids)
        np.testing.assert_array_equal(r.dists, ref.dists)
        np.testing.assert_array_equal(r.stats, ref.stats)
    t0, t1 = sp.submit(Q), sp.submit(Qr)
    with pytest.raises(RuntimeError):
        sp.submit(Q)                                # both slots still hold uncollected batches
    assert np.array_equal(sp.result(t0).ids, refs[0].ids)
    assert np.array_equal(sp.result(t1).ids, refs[1].ids)
    with pytest.raises(KeyError):
        sp.result(t1)
    # device-resident batches through the alternating plans (bench.py's device-timed form)
    ids, dists, stats = sp.run_resident(torch.from_numpy(Q).cuda(), 3)
    torch.cuda.synchronize()
    np.testing.assert_array_equal(ids.cpu().numpy(), refs[0].ids)
    np.testing.assert_array_equal(stats.cpu().numpy(), refs[0].stats)


def test_search_pipeline_k3_plans(pipe64):
    """k > 1 (a prediction pass inside the graph body) with 1, 2 and 3 plans in flight:
    every batch equals search_queries'."""
    import torch

    from paper_2502_01836_b200.pipeline import SearchPipeline, search_queries

    e = pipe64["eidx"]
    Q = np.asarray(pipe64["queries"], dtype=np.float32)
    ref = search_queries(e, Q, 3, target=0.95)
    for plans in (1, 2, 3):
        sp = SearchPipeline(e, Q.shape[0], 3, target=0.95, depth=3, plans=plans)
        ts = [sp.submit(torch.from_numpy(Q).pin_memory()) for _ in range(3)]
        for t in ts:
            r = sp.result(t)
            np.testing.assert_array_equal(r.ids, ref.ids)
            np.testing.assert_array_equal(r.dists, ref.dists)
            np.testing.assert_array_equal(r.stats, ref.stats)
        ids = sp.run_resident(torch.from_numpy(Q).cuda(), 4)[0]
        torch.cuda.synchronize()
        np.testing.assert_array_equal(ids.cpu().numpy(), ref.ids)
