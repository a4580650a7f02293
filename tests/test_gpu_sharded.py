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


def _enhance_worker(rank, world, port, q):
    import os

    import torch
    import torch.distributed as dist

    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        torch.cuda.set_device(0)
        from paper_2502_01836_b200 import build_index
        from paper_2502_01836_b200 import pipeline as pl
        from paper_2502_01836_b200.sharded import search_sharded
        from paper_2502_01836_b200.targets import collect_targets
        from paper_2502_01836_b200.training import TrainConfig

        data = lo.randwalk(8000, 64, 3)
        t = build_index(data, 300)
        e = pl.enhance(t, pl.SplitPlan(200, 60, 60), pl.SelectionBudget(64 << 20), 5,
                       constants=pl.RuntimeConstants(2e-7, 6e-6, 5 * 1024),
                       train_cfg=TrainConfig(initial_lr=1e-3, max_epochs=40), shard=(rank, world, None))
        g = e.global_set
        offs = e.tuned_offsets(0.99)
        Q = np.concatenate([lo.noisy_queries(data, 30, nz, 90 + int(10 * nz)) for nz in (0.1, 0.3)])
        lo_ = np.array([offs[l] for l in e.pack.leaf_ids], dtype=np.float64)
        res = search_sharded(t, Q, 1, rank=rank, world=world, pack=e.pack, offsets=lo_)
        ex = search_sharded(t, Q, 1, rank=rank, world=world)
        out = {"rank": rank, "filters": sorted(e.filters), "offs": offs, "ids": res.ids, "ex": ex.ids,
               "exd": ex.dists, "d": res.dists, "shard": t.shard(rank, world).leaf_range}
        if rank == 0:          # the unsharded collection of the same queries, for comparison
            ref = collect_targets(t, g.selected_leaves, g.queries, 60, train_nn=False)
            out["eq"] = {name: (bool(np.array_equal(a, b)), float(np.nanmax(np.abs(a - b))) if a.shape == b.shape
                                else str((a.shape, b.shape))) for name, a, b in (
                ("lb", g.lb_matrix, ref.lb_matrix), ("order", g.visit_order, ref.visit_order),
                ("dsel", g.dl_selected, ref.dl_selected), ("dcal", g.dl_calib_full, ref.dl_calib_full),
                ("nn", g.nn_distance[-60:], ref.nn_distance[-60:]))}
            out["selected"] = list(g.selected_leaves)
            out["leaf_ids"] = [int(l) for l in t.leaf_ids]
        q.put(out)
    finally:
        dist.destroy_process_group()


def test_sharded_enhance_two_ranks_gloo():
    """Leaf-sharded enhancement, 2 ranks on one GPU over gloo: the training-data
    matrices equal the unsharded ones bit for bit, each rank trains exactly the
    selected filters of its own leaves, both ranks fit the same offsets, and the
    sharded LeaFi search reaches the target on held-out queries."""
    import multiprocessing as mp
    import socket

    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        port = s.getsockname()[1]
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    ps = [ctx.Process(target=_enhance_worker, args=(r, 2, port, q)) for r in range(2)]
    for p in ps:
        p.start()
    outs = sorted((q.get(timeout=600) for _ in ps), key=lambda o: o["rank"])
    for p in ps:
        p.join(timeout=60)
        assert p.exitcode == 0
    o0, o1 = outs
    assert all(v[0] for v in o0["eq"].values()), o0["eq"]
    assert o0["offs"] == o1["offs"]
    for o in outs:
        a, b = o["shard"]
        own = set(o0["leaf_ids"][a:b])
        assert o["filters"] == [l for l in o0["selected"] if l in own]
    assert sorted(o0["filters"] + o1["filters"]) == o0["selected"]
    np.testing.assert_array_equal(o0["ids"], o1["ids"])
    hits = (o0["ids"][:, 0] == o0["ex"][:, 0]) | (np.abs(o0["d"][:, 0] - o0["exd"][:, 0]) <= 1e-6 * o0["exd"][:, 0])
    assert hits.mean() >= 0.95, hits.mean()
