"""EAPCA bound -- the oracle restatement on CPU.  Parity
unpinned (no reference code); these check the definition's soundness and that
it is at least as tight as the reference's mean-only bound."""

import numpy as np

from oracle import leafi_oracle as lo


def test_eapca_bound_sound_and_tighter():
    data = lo.randwalk(3000, 64, 3)
    t = lo.build_tree(data, 60)
    smin, smax = lo.eapca_envelopes(t)
    Q = np.concatenate([lo.noisy_queries(data, 20, nz, 4 + int(10 * nz)) for nz in (0.1, 0.5, 2.0)])
    qmu, qsd = lo.eapca(Q, t.starts, t.widths)
    mins, maxs = np.stack(t.env_min), np.stack(t.env_max)
    lbe = lo.lb_matrix_eapca(qmu, qsd, mins, maxs, np.stack(smin), np.stack(smax), t.widths)
    lbm = lo.lb_matrix(lo.paa(Q, t.starts, t.widths), mins, maxs, t.widths)
    assert (lbe >= lbm * (1 - 1e-12)).all()
    assert (lbe > lbm * 1.05).mean() > 0.2, "the stdev term must tighten a good share of the bounds"
    for lid in t.leaf_ids[::7]:
        d = lo.pair_dist(Q, data[t.members[lid]]).min(axis=1)
        assert (lbe[:, lid] <= d * (1 + 1e-12)).all()


def test_eapca_search_exact_and_prunes_more():
    data = lo.randwalk(4000, 64, 5)
    t = lo.build_tree(data, 80)
    env = lo.eapca_envelopes(t)
    for q in lo.noisy_queries(data, 12, 0.3, 6):
        a = lo.search(t, q, 2)
        b = lo.search(t, q, 2, eapca_env=env)
        assert a.results == b.results
        assert b.stats["leaves_visited"] <= a.stats["leaves_visited"]
        assert b.stats["series_scanned"] <= a.stats["series_scanned"]


def test_eapca_stdev_definition():
    x = np.array([1.0, 2.0, 4.0, 7.0, -1.0, 0.5], dtype=np.float64)
    starts, widths = np.array([0, 3]), np.array([3, 3])
    mu, sd = lo.eapca(x, starts, widths)
    np.testing.assert_allclose(mu, [7 / 3, 6.5 / 3])
    np.testing.assert_allclose(sd, [np.std(x[:3]), np.std(x[3:])], rtol=1e-15)
