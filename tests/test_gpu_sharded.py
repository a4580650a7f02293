"""Leaf-sharded search on ONE GPU: two shard engines (disjoint leaf ranges)
driven round by round with the bound exchange done in-process (the MIN the
NCCL allreduce computes across GPUs).  Exact answers must equal the
unsharded search; counters must add up."""

import math

import numpy as np
import pytest

from oracle import leafi_oracle as lo

pytestmark = pytest.mark.gpu


@pytest.mark.parametrize("k,world", [(1, 2), (3, 2), (1, 3)])
def test_shards_on_one_gpu_exact(k, world):
    import torch
    from paper_2502_01836_b200 import build_index, search_batch
    from paper_2502_01836_b200.sharded import GpuRoundEngine, merge_topk

    data = lo.randwalk(20000, 64, 8)
    t = build_index(data, 500)
    Q = np.concatenate([lo.noisy_queries(data, 20, nz, 60 + int(10 * nz)) for nz in (0.1, 0.3)])
    qd = torch.from_numpy(Q.astype(np.float32)).cuda()
    engines = [GpuRoundEngine(t.shard(r, world), qd, k) for r in range(world)]
    bound = torch.full((Q.shape[0],), math.inf, dtype=torch.float64, device="cuda")
    locs = [torch.empty_like(bound) for _ in engines]
    while True:
        act = sum(e.round(bound, l) for e, l in zip(engines, locs))
        bound = torch.stack(locs).min(dim=0).values
        if act == 0:
            break
    outs = [e.end() for e in engines]
    ids, d = merge_topk(torch.cat([o[0] for o in outs], 1), torch.cat([o[1] for o in outs], 1), k)
    stats = sum(o[2] for o in outs).cpu().numpy()
    ref = search_batch(t, Q, k)
    np.testing.assert_array_equal(ids.cpu().numpy(), ref.ids)
    np.testing.assert_array_equal(d.cpu().numpy(), ref.dists)
    assert (stats[:, 0] == stats[:, 1] + stats[:, 2] + stats[:, 3]).all()
    seq = search_batch(t, Q, k, sequential=True)
    assert (stats[:, 5] >= seq.stats[:, 5]).all()


def test_search_sharded_world1_matches_batch():
    from paper_2502_01836_b200 import build_index, search_batch
    from paper_2502_01836_b200.sharded import search_sharded

    data = lo.randwalk(20000, 64, 8)
    t = build_index(data, 500)
    Q = lo.noisy_queries(data, 30, 0.2, 77)
    r = search_sharded(t, Q, 2, rank=0, world=1)
    ref = search_batch(t, Q, 2)
    np.testing.assert_array_equal(r.ids, ref.ids)
    np.testing.assert_array_equal(r.stats, ref.stats)
