"""Host-side conformal calibration (paper_2502_01836_b200.calibration) against the
reference's fitted curves and tuned offsets (pipeline golden).  CPU only."""

import numpy as np
import pytest

from paper_2502_01836_b200 import calibration as cal
from paper_2502_01836_b200 import pipeline as pl


@pytest.fixture(scope="module")
def fitted(pipeline_golden):
    g = pipeline_golden
    sel = g["selected"].tolist()
    c = g["tg_dl_calib_full"].shape[0]
    tail = slice(g["tg_lb_matrix"].shape[0] - c, None)
    leaf_ids = np.flatnonzero(g["nt_is_leaf"]).astype(np.int64)
    preds = {l: g["calib_pred"][:, s] for s, l in enumerate(sel)}
    alphas = {l: cal.compute_alphas(preds[l], g["tg_dl_selected"][tail, s]) for s, l in enumerate(sel)}
    sk = cal.build_skeleton(g["tg_lb_matrix"][tail], g["tg_dl_calib_full"], g["tg_visit_order"][tail],
                            g["tg_nn_distance"][tail], leaf_ids, sel, preds)
    return sk, alphas, cal.fit_auto_tuners(sk, alphas)


def test_curves_match_reference(pipeline_golden, fitted):
    g = pipeline_golden
    _, alphas, curves = fitted
    for l in g["selected"].tolist():
        np.testing.assert_array_equal(alphas[l], g[f"curve_{l}_alphas"])
        np.testing.assert_array_equal(curves[l].knot_quality, g[f"curve_{l}_kq"])
        np.testing.assert_array_equal(curves[l].knot_offset, g[f"curve_{l}_ko"])
        assert curves[l].degenerate == bool(g[f"curve_{l}_deg"])


@pytest.mark.parametrize("target", [0.9, 0.95, 0.99, 1.0])
def test_tuned_offsets_match_reference(pipeline_golden, fitted, target):
    g = pipeline_golden
    _, _, curves = fitted
    offs = cal.tune(curves, target)
    np.testing.assert_array_equal([offs[l] for l in g["selected"].tolist()], g[f"off_{target}"])


def test_max_offset_coverage(fitted):
    """Reference test_enhanced.py:214-221 / criterion 4 (exact property)."""
    sk, alphas, curves = fitted
    amax = np.array([curves[l].alpha_max for l in sorted(curves)])
    assert cal.replay_recall(sk, cal.simulate_search(sk, amax)) == 1.0


def test_replay_offset_monotone(fitted):
    """Reference test_enhanced.py:202-212."""
    sk, _, curves = fitted
    rng = np.random.default_rng(62)
    base = rng.uniform(0.0, 1.5, len(curves))
    for bump in (0.25, 1.0, 3.0):
        assert (cal.simulate_search(sk, base + bump) <= cal.simulate_search(sk, base) + 1e-12).all()


def test_replay_many_equals_single(fitted):
    sk, _, curves = fitted
    rng = np.random.default_rng(3)
    rows = rng.uniform(0, 2, (5, len(curves)))
    many = cal.replay_many(sk, rows)
    for r in range(5):
        np.testing.assert_array_equal(many[r], cal.simulate_search(sk, rows[r]))


def test_steffen_properties():
    s = cal.SteffenInterpolator([0.0, 1.0], [0.0, 2.0])
    assert s(0.5) == 1.0 and s(-1) == 0.0 and s(3) == 2.0
    x = np.array([0.1, 0.3, 0.5, 0.9]); y = np.array([0.0, 0.2, 0.25, 1.0])
    s = cal.SteffenInterpolator(x, y)
    v = [s(t) for t in np.linspace(0, 1, 101)]
    assert all(a <= b + 1e-15 for a, b in zip(v, v[1:]))
    with pytest.raises(ValueError):
        cal.SteffenInterpolator([0.0, 0.0], [1.0, 2.0])


def test_selection_contract():
    """select.py:100-131 and the reference acceptance criterion 7 shape."""
    c = pl.RuntimeConstants(t_series=2e-7, t_filter=6e-6, filter_bytes=5 * 1024)
    assert pl.compute_threshold(c, 2.0) == 61   # fp: 2*6e-6/2e-7 = 60.000000000000014
    leaves = [(3, 100), (1, 100), (2, 50), (7, 59), (9, 61)]
    assert pl.select_greedy(leaves, 60, pl.SelectionBudget(3 * 5 * 1024), 5 * 1024) == [1, 3, 9]
    assert pl.select_greedy(leaves, 60, pl.SelectionBudget(0), 5 * 1024) == []
    assert pl.derive_seed(1234, 2) == (1234 * 1_000_003 + 2) % (2**31 - 1)
    with pytest.raises(ValueError):
        pl.SplitPlan(100, 10, 100)
    with pytest.raises(ValueError):
        pl.SearchRequest(query=np.zeros(4), k=1)
    with pytest.raises(ValueError):
        pl.SearchRequest(query=np.zeros(4), k=1, target=1.5)
