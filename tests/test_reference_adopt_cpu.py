"""Drop-in of real reference objects (build container only: needs the reference
package, marker `reference`).  A reference `tree.Index` and `EnhancedIndex`
(tree.py:164-189, enhanced.py:189-313) are built with the reference's own code,
then adopted by the B200 host layer (`TreeIndex.from_reference`,
`EnhancedIndex.adopt`): the node table, the leaf order, the filters and the
conformal offsets must be the reference's, unchanged.  No GPU compute."""

import sys
import warnings

import numpy as np
import pytest

from conftest import REFERENCE_SRC

pytestmark = pytest.mark.reference


@pytest.fixture(scope="module")
def ref(tmp_path_factory):
    if REFERENCE_SRC not in sys.path:
        sys.path.insert(0, REFERENCE_SRC)
    from leafsearch import enhanced as ren
    from leafsearch.mlp import TrainConfig
    from leafsearch.select import RuntimeConstants, SelectionBudget
    from leafsearch.series import generate_randwalk
    from leafsearch.traingen import SplitPlan
    from leafsearch.tree import build_index

    data = generate_randwalk(3000, 32, seed=7)
    index = build_index(data, 150)
    eidx = ren.enhance(index, SplitPlan(80, 20, 30), SelectionBudget(1 << 20), 11, tmp_path_factory.mktemp("enh"),
                       constants=RuntimeConstants(2e-7, 6e-6, 5 * 1024), train_cfg=TrainConfig(max_epochs=5))
    return index, eidx


def test_adopt_reference_tree(ref):
    from paper_2502_01836_b200.engine import as_tree

    index, _ = ref
    t = as_tree(index)
    assert t is as_tree(index), "adoption is cached per reference object"
    assert t.n_nodes == len(index.nodes) and t.n == index.n
    for nd in index.nodes:
        np.testing.assert_array_equal(t.env_min[nd.node_id], nd.envelope.mean_min)
        np.testing.assert_array_equal(t.env_max[nd.node_id], nd.envelope.mean_max)
        assert t.left[nd.node_id] == (-1 if nd.left is None else nd.left.node_id)
        assert t.right[nd.node_id] == (-1 if nd.right is None else nd.right.node_id)
        if nd.members is not None:
            np.testing.assert_array_equal(t.leaf_members(nd.node_id), np.sort(np.asarray(nd.members)))
    assert [int(l) for l in t.leaf_ids] == sorted(leaf.node_id for leaf in index.leaves)
    np.testing.assert_array_equal(t.values, index.dataset.values.astype(np.float32))


def test_adopt_reference_enhanced_index(ref):
    from paper_2502_01836_b200.pipeline import EnhancedIndex, _as_enhanced

    _, reidx = ref
    with pytest.warns(RuntimeWarning, match="calibrated on the numpy forward"):
        e = EnhancedIndex.adopt(reidx)
    assert reidx.filters, "the reference run must have trained filters"
    assert e.filter_leaf_ids == reidx.filter_leaf_ids
    for lid, m in reidx.filters.items():
        f = e.filters[lid]
        np.testing.assert_array_equal(f.W1, m.W1)
        np.testing.assert_array_equal(f.b1, m.b1)
        np.testing.assert_array_equal(f.W2, m.W2)
        assert float(f.b2) == float(m.b2)
    for target in (0.9, 0.95, 0.99):
        assert e.tuned_offsets(target) == reidx.tuned_offsets(target)
    with warnings.catch_warnings():
        warnings.simplefilter("ignore", RuntimeWarning)
        w1 = _as_enhanced(reidx)
        assert _as_enhanced(reidx) is w1, "the adopted wrapper is cached (weakly) per reference object"
