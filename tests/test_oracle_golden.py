"""Pin the CPU oracle against golden vectors produced by the real reference.

Every assertion here is bit-exact (array_equal / ==) unless a tolerance is
written next to it.  CPU only.
"""

import math

import numpy as np
import pytest

from oracle import leafi_oracle as lo
from conftest import oracle_tree_from_table


def _tree_equal(t: "lo.OracleTree", g: dict, prefix: str = "nt_") -> None:
    n = g[prefix + "left"].shape[0]
    assert t.n_nodes == n
    np.testing.assert_array_equal(np.stack(t.env_min), g[prefix + "env_min"])
    np.testing.assert_array_equal(np.stack(t.env_max), g[prefix + "env_max"])
    np.testing.assert_array_equal(np.array(t.left), g[prefix + "left"])
    np.testing.assert_array_equal(np.array(t.right), g[prefix + "right"])
    np.testing.assert_array_equal(np.array(t.size), g[prefix + "size"])
    np.testing.assert_array_equal(np.array(t.split_seg), g[prefix + "split_seg"])
    np.testing.assert_array_equal(np.array(t.split_thr), g[prefix + "split_thr"])
    ptr, mem = g[prefix + "member_ptr"], g[prefix + "members"]
    for i in range(n):
        if g[prefix + "is_leaf"][i]:
            np.testing.assert_array_equal(t.members[i], mem[ptr[i]:ptr[i + 1]])
        else:
            assert not t.is_leaf(i)


class TestKnownAnswers:
    @pytest.mark.parametrize("m,l", [(30, 4), (256, 8), (96, 8), (10, 3), (7, 7)])
    def test_segments(self, knowns, m, l):
        s, w = lo.seg_layout(m, l)
        np.testing.assert_array_equal(s, knowns[f"seg_{m}_{l}_starts"])
        np.testing.assert_array_equal(w, knowns[f"seg_{m}_{l}_widths"])

    def test_segment_example(self):
        # reference test_summarize.py:27-30
        s, w = lo.seg_layout(30, 4)
        assert w.tolist() == [8, 8, 7, 7] and s.tolist() == [0, 8, 16, 23]

    @pytest.mark.parametrize("m", [256, 96, 32])
    def test_paa_bits(self, knowns, m):
        s, w = lo.seg_layout(m, 8)
        rows = knowns[f"paa_{m}_rows"]
        np.testing.assert_array_equal(lo.paa(rows, s, w), knowns[f"paa_{m}"])
        np.testing.assert_array_equal(np.stack([lo.paa(r, s, w) for r in rows]), knowns[f"paa1_{m}"])

    @pytest.mark.parametrize("m", [256, 96, 32])
    def test_lower_bounds_bits(self, knowns, m):
        s, w = lo.seg_layout(m, 8)
        mins, maxs, qs = knowns[f"lb_{m}_mins"], knowns[f"lb_{m}_maxs"], knowns[f"lb_{m}_qs"]
        got = np.array([[lo.node_lb(q, a, b, w) for a, b in zip(mins, maxs)] for q in qs])
        np.testing.assert_array_equal(got, knowns[f"lb_{m}_dot"])
        np.testing.assert_array_equal(lo.lb_matrix(qs, mins, maxs, w), knowns[f"lb_{m}_batch"])

    @pytest.mark.parametrize("m", [256, 96, 32])
    def test_distances_bits(self, knowns, m):
        blk, qq = knowns[f"dist_{m}_block"], knowns[f"dist_{m}_q"]
        np.testing.assert_array_equal(np.stack([lo.row_dist(q, blk) for q in qq]), knowns[f"dist_{m}_scan"])
        np.testing.assert_array_equal(lo.pair_dist(qq, blk), knowns[f"dist_{m}_batch"])

    def test_distance_examples(self):
        # reference test_series.py:33-37, 89-92
        assert lo.row_dist(np.zeros(3), np.zeros((1, 3)))[0] == 0.0
        assert lo.row_dist(np.array([1.0, 2, 3]), np.array([[1.0, 2, 4]]))[0] == 1.0
        x = lo.randwalk(5, 16, 0)
        assert (np.diag(lo.pair_dist(x, x)) == 0.0).all()

    def test_generators_bits(self, knowns):
        np.testing.assert_array_equal(lo.randwalk(100, 256, 1234).astype(np.float32), knowns["rw_100_256"])
        import hashlib
        h = hashlib.sha256(lo.randwalk(5000, 32, 1).tobytes()).hexdigest()
        assert h == str(knowns["rw_5000_32_sha"])
        d = lo.randwalk(500, 64, 3)
        np.testing.assert_array_equal(lo.noisy_queries(d, 30, 0.3, 4).astype(np.float32), knowns["mq_500_64"])
        gq, lv = lo.global_queries(d, 25, (0.1, 0.4), 5)
        np.testing.assert_array_equal(gq.astype(np.float32), knowns["gq_500_64"])
        np.testing.assert_array_equal(lv, knowns["gq_500_64_levels"])

    @pytest.mark.parametrize("m", [32, 256])
    def test_mlp_forward_bits(self, knowns, m):
        W1, b1, W2, b2 = (knowns[f"mlp_{m}_{k}"] for k in ("W1", "b1", "W2", "b2"))
        got = np.array([lo.mlp_forward(W1, b1, W2, b2, x) for x in knowns[f"mlp_{m}_x"]])
        np.testing.assert_array_equal(got, knowns[f"mlp_{m}_y"])

    def test_mlp_hand_computed(self):
        # reference test_mlp.py:52-58 style: W1 = I, b1 = 0, W2 = [0.5, 1.25], b2 = 0
        y = lo.mlp_forward(np.eye(2, dtype=np.float32), np.zeros(2), np.array([0.5, 1.25]), 0.0, [1.0, 1.0])
        assert y == 1.75
        assert lo.mlp_forward(np.eye(2), np.zeros(2), np.ones(2), 0.0, [-1.0, 3.0]) == 3.0


class TestSmallIndex:
    @pytest.fixture(scope="class")
    def tree(self, small_golden):
        return lo.build_tree(lo.randwalk(2000, 32, 7), max_leaf_size=128)

    def test_build_matches_reference(self, tree, small_golden):
        _tree_equal(tree, small_golden)

    def test_table_roundtrip(self, small_golden):
        t = oracle_tree_from_table(lo.randwalk(2000, 32, 7), small_golden)
        _tree_equal(t, small_golden)

    @pytest.mark.parametrize("k", [1, 3])
    def test_exact_search_bits(self, tree, small_golden, k):
        g = small_golden
        for qi, q in enumerate(g["queries"]):
            out = lo.search(tree, q, k, want_trace=True)
            assert [i for i, _ in out.results] == g[f"k{k}_ids"][qi].tolist()
            assert [d for _, d in out.results] == g[f"k{k}_dists"][qi].tolist()
            assert [out.stats[s] for s in lo.STAT_KEYS] == g[f"k{k}_stats"][qi].tolist()
            a, b = g[f"k{k}_trace_ptr"][qi], g[f"k{k}_trace_ptr"][qi + 1]
            assert [e[0] for e in out.trace] == g[f"k{k}_trace_leaf"][a:b].tolist()
            assert [e[1] for e in out.trace] == g[f"k{k}_trace_lb"][a:b].tolist()
            assert [e[4] for e in out.trace] == g[f"k{k}_trace_bsf"][a:b].tolist()
            nn = [np.nan if e[3] is None else e[3] for e in out.trace]
            np.testing.assert_array_equal(nn, g[f"k{k}_trace_nn"][a:b])

    def test_epsilon_mode(self, tree, small_golden):
        g = small_golden
        for qi, q in enumerate(g["queries"]):
            out = lo.search(tree, q, 1, bsf_factor=0.5)
            assert out.results[0][0] == g["eps1_ids"][qi][0]
            assert [out.stats[s] for s in lo.STAT_KEYS] == g["eps1_stats"][qi].tolist()

    def test_linear_scan_config(self, small_golden):
        g = small_golden
        data = lo.randwalk(5000, 32, 1)
        t = lo.build_tree(data, 256)
        for qi in range(0, 100, 9):
            q = g["ls_queries"][qi]
            out = lo.search(t, q, 5)
            assert [i for i, _ in out.results] == g["ls_ids"][qi].tolist()
            assert [i for i, _ in lo.linear_scan(data, q, 5)] == g["ls_linear_ids"][qi].tolist()
            assert [out.stats[s] for s in lo.STAT_KEYS] == g["ls_stats"][qi].tolist()

    def test_collect_targets_bits(self, tree, small_golden):
        g = small_golden
        gq, _ = lo.global_queries(tree.values, 120, (0.1, 0.4), 41)
        np.testing.assert_array_equal(gq, g["tg_queries"])
        tg = lo.collect_targets(tree, g["tg_selected"].tolist(), gq, 30)
        for f in ("dl_selected", "nn_distance", "leaf_ids", "lb_matrix", "visit_order", "dl_calib_full"):
            np.testing.assert_array_equal(getattr(tg, f), g[f"tg_{f}"], err_msg=f)

    def test_local_targets_bits(self, tree, small_golden):
        g = small_golden
        lid = int(g["lq_leaf"])
        q, _, src = lo.local_queries(tree, lid, 40, (0.1, 0.4), 4)
        np.testing.assert_array_equal(q, g["lq_queries"])
        np.testing.assert_array_equal(src, g["lq_sources"])
        tg, lbs = lo.local_targets(tree, lid, q)
        np.testing.assert_array_equal(tg, g["lq_targets"])
        np.testing.assert_array_equal(lbs, g["lq_lbs"])


class TestPipeline:
    """The reference conftest `pipeline` (4000x32, trained filters, fitted curves)."""

    @pytest.fixture(scope="class")
    def tree(self, pipeline_golden):
        t = lo.build_tree(lo.randwalk(4000, 32, 17), 200)
        _tree_equal(t, pipeline_golden)
        return t

    def _predictors(self, g):
        sel = g["selected"].tolist()
        return {lid: (lambda x, i=i: lo.mlp_forward(g["W1"][i], g["b1"][i], g["W2"][i], g["b2"][i], x))
                for i, lid in enumerate(sel)}

    def test_predictions_bits(self, tree, pipeline_golden):
        g = pipeline_golden
        p = self._predictors(g)
        sel = g["selected"].tolist()
        got = np.array([[p[l](q) for l in sel] for q in g["queries"]])
        np.testing.assert_array_equal(got, g["pred_queries"])

    @pytest.mark.parametrize("target", [0.9, 0.95, 0.99, 1.0])
    def test_filtered_search_bits(self, tree, pipeline_golden, target):
        g = pipeline_golden
        sel = g["selected"].tolist()
        offs = dict(zip(sel, g[f"off_{target}"].tolist()))
        p = self._predictors(g)
        for qi, q in enumerate(g["queries"]):
            out = lo.search(tree, q, 1, predictors=p, offsets=offs)
            assert [i for i, _ in out.results] == g[f"t{target}_ids"][qi].tolist()
            assert [d for _, d in out.results] == g[f"t{target}_dists"][qi].tolist()
            assert [out.stats[s] for s in lo.STAT_KEYS] == g[f"t{target}_stats"][qi].tolist()

    def test_calibration_replay_covers(self, tree, pipeline_golden):
        """Max-offset coverage (reference test_enhanced.py:214-221) on the oracle replay."""
        g = pipeline_golden
        sel = g["selected"].tolist()
        lbm, order = g["tg_lb_matrix"], g["tg_visit_order"]
        c = g["tg_dl_calib_full"].shape[0]
        tail = slice(lbm.shape[0] - c, None)
        leaf_ids = np.array(tree.leaf_ids)
        slot_of = {l: s for s, l in enumerate(sel)}
        slots = np.array([slot_of.get(int(l), -1) for l in leaf_ids], np.int32)
        predc = np.full((c, leaf_ids.shape[0]), np.nan)
        for s, l in enumerate(sel):
            predc[:, int(np.searchsorted(leaf_ids, l))] = g["calib_pred"][:, s]
        o = order[tail]
        lb_v = np.take_along_axis(lbm[tail], o, 1)
        dl_v = np.take_along_axis(g["tg_dl_calib_full"], o, 1)
        pr_v = np.take_along_axis(predc, o, 1)
        alphas = [lo.alphas_desc(g["calib_pred"][:, s], g["tg_dl_selected"][tail, s]) for s in range(len(sel))]
        amax = np.array([a[0] for a in alphas])
        np.testing.assert_array_equal(amax, [g[f"curve_{l}_alphas"][0] for l in sel])
        ach = lo.replay(lb_v, dl_v, pr_v, slots[o], amax)
        nn = g["tg_nn_distance"][tail]
        assert np.mean(ach <= nn * (1 + lo.RECALL_REL_TOL)) == 1.0
