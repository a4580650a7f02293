"""EAPCA bound on the GPU (include/leafi_b200.h lf_bounds_eapca)
against the oracle's restatement (oracle/leafi_oracle.py eapca; parity
unpinned: the reference has no EAPCA code)."""

import numpy as np
import pytest

from oracle import leafi_oracle as lo

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def eap():
    from paper_2502_01836_b200 import build_index

    data = lo.randwalk(30000, 64, 41)
    t = build_index(data, 40).use_eapca()
    ot = lo.build_tree(data, 40)
    env = lo.eapca_envelopes(ot)
    return data, t, ot, env


def test_eapca_summaries_and_bounds_bit_exact(eap):
    import torch

    from paper_2502_01836_b200 import _lib

    data, t, ot, env = eap
    np.testing.assert_array_equal(t.sd_min, np.stack(env[0]))
    np.testing.assert_array_equal(t.sd_max, np.stack(env[1]))
    Q = np.concatenate([lo.noisy_queries(data, 40, nz, 3 + int(10 * nz)) for nz in (0.1, 0.6)] + [data[:3]])
    qd = torch.from_numpy(Q.astype(np.float32)).cuda()
    out = torch.empty((Q.shape[0], 2 * t.n_seg), dtype=torch.float64, device="cuda")
    _lib.check(_lib.lib().lf_eapca_device(qd.data_ptr(), Q.shape[0], t.m, t.n_seg, out.data_ptr(), _lib.stream_ptr()))
    mu, sd = lo.eapca(Q, ot.starts, ot.widths)
    np.testing.assert_array_equal(out[:, :t.n_seg].cpu().numpy(), mu)
    np.testing.assert_array_equal(out[:, t.n_seg:].cpu().numpy(), sd)
    di = t.device()
    lb = torch.empty((Q.shape[0], t.n_nodes), dtype=torch.float64, device="cuda")
    qs = torch.empty((Q.shape[0], 2 * t.n_seg), dtype=torch.float64, device="cuda")
    _lib.check(_lib.lib().lf_bounds_eapca(qd.data_ptr(), Q.shape[0], di.struct(None), di.env_min.data_ptr(),
                                          di.env_max.data_ptr(), di.sd_min.data_ptr(), di.sd_max.data_ptr(),
                                          t.n_nodes, qs.data_ptr(), lb.data_ptr(), _lib.stream_ptr()))
    ref = lo.lb_matrix_eapca(mu, sd, np.stack(ot.env_min), np.stack(ot.env_max), np.stack(env[0]),
                             np.stack(env[1]), ot.widths)
    np.testing.assert_array_equal(lb.cpu().numpy(), ref)


@pytest.mark.parametrize("k", [1, 3])
def test_eapca_sequential_search_matches_oracle(eap, k):
    """The search on the EAPCA bound (visit order, break rule, gap bounds of the
    internal nodes) walks exactly like the oracle: ids, counters, traces."""
    from paper_2502_01836_b200 import search_batch

    data, t, ot, env = eap
    Q = np.concatenate([lo.noisy_queries(data, 8, nz, 13 + int(10 * nz)) for nz in (0.1, 0.4, 1.2)])
    res = search_batch(t, Q, k, sequential=True, want_trace=True)
    for i, q in enumerate(Q):
        o = lo.search(ot, q, k, want_trace=True, eapca_env=env)
        assert res.ids[i].tolist() == [a for a, _ in o.results], i
        np.testing.assert_allclose(res.dists[i], [b for _, b in o.results], rtol=1e-12)
        assert res.stats[i].tolist() == [o.stats[s] for s in lo.STAT_KEYS], i
        assert [e.leaf_id for e in res.trace_of(i)] == [e[0] for e in o.trace], i


def test_eapca_exact_and_tighter(eap):
    """Exact results do not depend on the bound; the EAPCA walk visits no more leaves."""
    from paper_2502_01836_b200 import build_index, search_batch

    data, t, _, _ = eap
    tm = build_index(data, 40)
    Q = np.concatenate([lo.noisy_queries(data, 30, nz, 23 + int(10 * nz)) for nz in (0.1, 0.4)])
    a = search_batch(t, Q, 2)
    b = search_batch(tm, Q, 2)
    np.testing.assert_array_equal(a.ids, b.ids)
    np.testing.assert_array_equal(a.dists, b.dists)
    sa = search_batch(t, Q, 2, sequential=True)
    sb = search_batch(tm, Q, 2, sequential=True)
    assert (sa.stats[:, 0] <= sb.stats[:, 0]).all()
    assert sa.stats[:, 5].sum() < sb.stats[:, 5].sum()


def test_eapca_training_data_bounds(eap):
    from paper_2502_01836_b200.targets import collect_targets

    data, t, ot, env = eap
    gq, _ = lo.global_queries(data, 60, (0.1, 0.4), 8)
    g = collect_targets(t, [int(l) for l in t.leaf_ids[:20]], gq, 20)
    mu, sd = lo.eapca(gq, ot.starts, ot.widths)
    lids = ot.leaf_ids
    ref = lo.lb_matrix_eapca(mu, sd, np.stack([ot.env_min[i] for i in lids]), np.stack([ot.env_max[i] for i in lids]),
                             np.stack([env[0][i] for i in lids]), np.stack([env[1][i] for i in lids]), ot.widths)
    np.testing.assert_array_equal(g.lb_matrix, ref)
