"""Generate golden vectors by running the REAL reference package.

Run in the build container (the reference is importable there, not on the GPU
box):

    PYTHONPATH=/root/reference/pkg/src python tests/golden/make_golden.py [--c1] [--c1-leafi]

Outputs (committed, small): tests/golden/*.npz and *.json.  The oracle
(`oracle/leafi_oracle.py`) is checked bit-for-bit against these in
`tests/test_oracle_golden.py`; the GPU parity tests compare the CUDA path with
the same vectors.  Nothing here is imported at run time by the product.
"""

from __future__ import annotations

import argparse
import dataclasses
import hashlib
import json
import os
import sys
import tempfile
import time
from pathlib import Path

import numpy as np

REF_SRC = "/root/reference/pkg/src"
OUT = Path(__file__).resolve().parent
sys.path.insert(0, REF_SRC)

from leafsearch import conformal, mlp, series, summarize, traingen, tree  # noqa: E402
from leafsearch.enhanced import SearchRequest, derive_seed, enhance, search  # noqa: E402
from leafsearch.select import RuntimeConstants, SelectionBudget  # noqa: E402

# tests/conftest.py:11 of the reference
FIXED_CONSTANTS = RuntimeConstants(t_series=2e-7, t_filter=6e-6, filter_bytes=5 * 1024)
STAT_KEYS = ("leaves_visited", "leaves_searched", "leaves_lb_pruned", "leaves_filter_pruned",
             "filter_inferences", "series_scanned")


def sha(a: np.ndarray) -> str:
    return hashlib.sha256(np.ascontiguousarray(a).tobytes()).hexdigest()


def node_table(index) -> dict:
    nodes = index.nodes
    members = [nd.members if nd.is_leaf else [] for nd in nodes]
    ptr = np.cumsum([0] + [len(m) for m in members]).astype(np.int64)
    return {
        "env_min": np.stack([nd.envelope.mean_min for nd in nodes]),
        "env_max": np.stack([nd.envelope.mean_max for nd in nodes]),
        "left": np.array([-1 if nd.left is None else nd.left.node_id for nd in nodes], np.int64),
        "right": np.array([-1 if nd.right is None else nd.right.node_id for nd in nodes], np.int64),
        "is_leaf": np.array([nd.is_leaf for nd in nodes]),
        "split_seg": np.array([-1 if nd.split_segment is None else nd.split_segment for nd in nodes], np.int64),
        "split_thr": np.array([np.nan if nd.split_threshold is None else nd.split_threshold for nd in nodes]),
        "size": np.array([nd.size for nd in nodes], np.int64),
        "oversized": np.array([nd.oversized for nd in nodes]),
        "member_ptr": ptr,
        "members": np.concatenate([np.asarray(m, np.int64) for m in members]) if ptr[-1] else np.zeros(0, np.int64),
    }


def outcomes(index, queries, k, want_trace=False, **kw) -> dict:
    ids, dists, stats, tr = [], [], [], []
    for q in queries:
        out = tree.search_engine(index, q, k, want_trace=want_trace, **kw)
        ids.append([i for i, _ in out.results])
        dists.append([d for _, d in out.results])
        st = dataclasses.asdict(out.stats)
        stats.append([st[key] for key in STAT_KEYS])
        if want_trace:
            tr.append([(e.leaf_id, e.lower_bound, e.searched,
                        np.nan if e.leaf_nn_distance is None else e.leaf_nn_distance, e.bsf_before)
                       for e in out.trace])
    res = {"ids": np.array(ids, np.int64), "dists": np.array(dists), "stats": np.array(stats, np.int64)}
    if want_trace:
        ptr = np.cumsum([0] + [len(t) for t in tr]).astype(np.int64)
        flat = [e for t in tr for e in t]
        res["trace_ptr"] = ptr
        res["trace_leaf"] = np.array([e[0] for e in flat], np.int64)
        res["trace_lb"] = np.array([e[1] for e in flat])
        res["trace_searched"] = np.array([e[2] for e in flat])
        res["trace_nn"] = np.array([e[3] for e in flat])
        res["trace_bsf"] = np.array([e[4] for e in flat])
    return res


def prefixed(prefix: str, d: dict) -> dict:
    return {f"{prefix}{k}": v for k, v in d.items()}


def make_knowns() -> None:
    rng = np.random.default_rng(20250203)
    out = {}
    for m, l in ((30, 4), (256, 8), (96, 8), (10, 3), (7, 7)):
        cfg = summarize.segment_config(m, l)
        out[f"seg_{m}_{l}_starts"] = cfg.starts
        out[f"seg_{m}_{l}_widths"] = cfg.widths
    for m in (256, 96, 32):
        cfg = summarize.segment_config(m, 8)
        rows = series.quantize32(rng.standard_normal((64, m)) * 2.0)
        out[f"paa_{m}_rows"] = rows
        out[f"paa_{m}"] = summarize.summarize_matrix(rows, cfg)
        out[f"paa1_{m}"] = np.stack([summarize.summarize_series(r, cfg) for r in rows])
        mins = np.sort(rng.standard_normal((200, 8)), axis=0) - 0.5
        maxs = mins + np.abs(rng.standard_normal((200, 8)))
        qs = summarize.summarize_matrix(series.quantize32(rng.standard_normal((50, m))), cfg)
        out[f"lb_{m}_mins"], out[f"lb_{m}_maxs"], out[f"lb_{m}_qs"] = mins, maxs, qs
        out[f"lb_{m}_dot"] = np.array([[summarize.lower_bound_from_summary(
            q, summarize.NodeEnvelope(mn, mx), cfg) for mn, mx in zip(mins, maxs)] for q in qs])
        out[f"lb_{m}_batch"] = summarize.lower_bounds_batch(qs, mins, maxs, cfg)
        blk = series.quantize32(rng.standard_normal((300, m)))
        qq = series.quantize32(rng.standard_normal((20, m)))
        out[f"dist_{m}_block"], out[f"dist_{m}_q"] = blk, qq
        out[f"dist_{m}_scan"] = np.stack([series.scan_distances(q, blk) for q in qq])
        out[f"dist_{m}_batch"] = series.batch_distances(qq, blk)
    out["rw_100_256"] = series.generate_randwalk(100, 256, 1234).values.astype(np.float32)
    out["rw_5000_32_sha"] = np.array(sha(series.generate_randwalk(5000, 32, 1).values))
    d = series.generate_randwalk(500, 64, 3)
    out["mq_500_64"] = series.make_queries(d, 30, 0.3, 4).values.astype(np.float32)
    gq, glv = traingen.generate_global_queries(d, 25, (0.1, 0.4), 5)
    out["gq_500_64"], out["gq_500_64_levels"] = gq.astype(np.float32), glv
    for m in (32, 256):
        model = mlp.init_model(m, seed=m + 1)
        model.b1 = (rng.standard_normal(m) * 0.1).astype(np.float32)
        model.b2 = np.float32(0.37)
        xs = series.quantize32(rng.standard_normal((40, m)))
        out[f"mlp_{m}_W1"], out[f"mlp_{m}_b1"], out[f"mlp_{m}_W2"] = model.W1, model.b1, model.W2
        out[f"mlp_{m}_b2"] = np.array(model.b2)
        out[f"mlp_{m}_x"] = xs
        out[f"mlp_{m}_y"] = np.array([model.forward(x) for x in xs])
    np.savez_compressed(OUT / "knowns.npz", **out)


def make_small() -> None:
    """Reference conftest fixtures small_data / small_index / small_queries (conftest.py:14-26)."""
    data = series.generate_randwalk(2000, 32, seed=7)
    index = tree.build_index(data, max_leaf_size=128)
    queries = series.make_queries(data, 40, 0.2, seed=31).values
    out = {"data_sha": np.array(sha(data.values)), "queries": queries}
    out.update(prefixed("nt_", node_table(index)))
    out.update(prefixed("k1_", outcomes(index, queries, 1, want_trace=True)))
    out.update(prefixed("k3_", outcomes(index, queries, 3, want_trace=True)))
    out.update(prefixed("eps1_", outcomes(index, queries, 1, bsf_factor=0.5)))
    # 5000x32 vs linear scan (test_tree.py:93-102)
    d2 = series.generate_randwalk(5000, 32, seed=1)
    i2 = tree.build_index(d2, max_leaf_size=256)
    q2 = series.make_queries(d2, 100, 0.3, seed=2).values
    out["ls_queries"] = q2
    out.update(prefixed("ls_", outcomes(i2, q2, 5)))
    out["ls_linear_ids"] = np.array([[i for i, _ in tree.linear_scan(d2, q, 5)] for q in q2], np.int64)
    # k = n (test_tree.py:104-112)
    d3 = series.generate_randwalk(200, 16, seed=3)
    i3 = tree.build_index(d3, max_leaf_size=32)
    q3 = series.make_queries(d3, 1, 0.2, seed=4).values
    out["kn_queries"] = q3
    out.update(prefixed("kn_", outcomes(i3, q3, 200)))
    # training-data generation (test_traingen.py:21-26)
    gq, _ = traingen.generate_global_queries(data, 120, (0.1, 0.4), seed=41)
    sel = [leaf.node_id for leaf in index.leaves[:6]]
    gts = traingen.collect_targets(index, sel, gq, calibration_count=30)
    out["tg_queries"], out["tg_selected"] = gq, np.array(sel, np.int64)
    for f in ("dl_selected", "nn_distance", "leaf_ids", "lb_matrix", "visit_order", "dl_calib_full"):
        out[f"tg_{f}"] = getattr(gts, f)
    lid = index.leaves[2].node_id
    local = traingen.generate_local_queries(index, lid, 40, (0.1, 0.4), seed=4)
    traingen.collect_local_targets(index, local)
    out["lq_leaf"] = np.array(lid)
    out["lq_queries"], out["lq_sources"] = local.queries, local.source_ids
    out["lq_targets"], out["lq_lbs"] = local.targets, local.lbs
    np.savez_compressed(OUT / "small.npz", **out)


def make_pipeline() -> None:
    """Reference conftest `pipeline` fixture (conftest.py:29-46) + filtered outcomes."""
    data = series.generate_randwalk(4000, 32, seed=17)
    index = tree.build_index(data, max_leaf_size=200)
    plan = traingen.SplitPlan(n_global=240, n_local=80, calibration=60)
    with tempfile.TemporaryDirectory() as tmp:
        eidx = enhance(index, plan, SelectionBudget(capacity_bytes=16 * 1024 * 1024), seed=23,
                       out_dir=tmp, constants=FIXED_CONSTANTS,
                       train_cfg=mlp.TrainConfig(max_epochs=150), workers=1)
    queries = series.make_queries(data, 60, 0.25, seed=71).values
    sel = sorted(eidx.filters)
    out = {"data_sha": np.array(sha(data.values)), "queries": queries,
           "selected": np.array(sel, np.int64)}
    out.update(prefixed("nt_", node_table(index)))
    out["W1"] = np.stack([eidx.filters[l].W1 for l in sel])
    out["b1"] = np.stack([eidx.filters[l].b1 for l in sel])
    out["W2"] = np.stack([eidx.filters[l].W2 for l in sel])
    out["b2"] = np.array([eidx.filters[l].b2 for l in sel], np.float32)
    for l in sel:
        c = eidx.curves[l]
        out[f"curve_{l}_alphas"] = c.alphas_desc
        out[f"curve_{l}_kq"] = c.knot_quality
        out[f"curve_{l}_ko"] = c.knot_offset
        out[f"curve_{l}_deg"] = np.array(c.degenerate)
    targets = (0.9, 0.95, 0.99, 1.0)
    out["targets"] = np.array(targets)
    preds = {l: eidx.filters[l].forward for l in sel}
    out["pred_queries"] = np.array([[preds[l](q) for l in sel] for q in queries])
    for t in targets:
        offs = eidx.tuned_offsets(t)
        out[f"off_{t}"] = np.array([offs[l] for l in sel])
        res = {"ids": [], "dists": [], "stats": []}
        for q in queries:
            o = search(eidx, SearchRequest(query=q, k=1, target=t))
            st = dataclasses.asdict(o.stats)
            res["ids"].append([i for i, _ in o.results])
            res["dists"].append([d for _, d in o.results])
            res["stats"].append([st[k] for k in STAT_KEYS])
        out.update({f"t{t}_{k}": np.array(v) for k, v in res.items()})
    out.update(prefixed("k3t09_", outcomes(index, queries, 3, predictors=preds, offsets=eidx.tuned_offsets(0.9))))
    out.update(prefixed("exact_", outcomes(index, queries, 1)))
    # the calibration skeleton exactly as the fit stage saw it (test_enhanced.py:155-181)
    gq, _ = traingen.generate_global_queries(data, plan.n_global, (0.1, 0.4), derive_seed(23, 2))
    gts = traingen.collect_targets(index, sel, gq, plan.calibration)
    out["gq"] = gq
    for f in ("dl_selected", "nn_distance", "lb_matrix", "visit_order", "dl_calib_full"):
        out[f"tg_{f}"] = getattr(gts, f)
    calib = gq[gts.train_pool_size:]
    out["calib_pred"] = np.array([[eidx.filters[l].forward(q) for l in sel] for q in calib])
    np.savez_compressed(OUT / "pipeline.npz", **out)


def make_c1(leafi: bool) -> None:
    """BASELINE config 1: 100K x 256 random walk, cap 1000."""
    t0 = time.perf_counter()
    data = series.generate_randwalk(100_000, 256, seed=1234)
    index = tree.build_index(data, max_leaf_size=1000)
    nt = node_table(index)
    doc = {"data_sha": sha(data.values), "build_s": time.perf_counter() - t0,
           "n_nodes": len(index.nodes), "n_leaves": len(index.leaves),
           "members_sha": sha(nt["members"]), "member_ptr_sha": sha(nt["member_ptr"]),
           "env_min_sha": sha(nt["env_min"]), "env_max_sha": sha(nt["env_max"])}
    out = {"leaf_sizes": np.array([leaf.size for leaf in index.leaves], np.int64)}
    out.update(prefixed("nt_", {k: v for k, v in nt.items() if k != "members"}))
    levels = (0.1, 0.2, 0.3, 0.4)
    for nz in levels:
        qs = series.make_queries(data, 100, nz, seed=1234 + int(10 * nz)).values
        doc[f"queries_{nz}_sha"] = sha(qs)
        out.update(prefixed(f"n{nz}_", outcomes(index, qs, 1)))
    np.savez_compressed(OUT / "c1.npz", **out)
    if leafi:
        from leafsearch.cli import run_bench
        from leafsearch.traingen import SplitPlan
        t1 = time.perf_counter()
        with tempfile.TemporaryDirectory() as tmp:
            eidx = enhance(index, SplitPlan(1500, 500, 300), SelectionBudget(64 * 1024 * 1024, a=2.0),
                           seed=1234, out_dir=tmp, constants=FIXED_CONSTANTS,
                           train_cfg=mlp.TrainConfig(initial_lr=1e-3), workers=os.cpu_count() or 1)
        doc["enhance_s"] = time.perf_counter() - t1
        doc["selected"] = sorted(eidx.filters)
        sets = [(nz, series.make_queries(data, 100, nz, seed=1234 + int(10 * nz)).values) for nz in levels]
        rep = run_bench(index, eidx, sets, targets=[0.99], methods=["exact", "filtered"], seed=1234)
        doc["bench_rows"] = rep["rows"]
    with open(OUT / "c1.json", "w") as fh:
        json.dump(doc, fh, indent=1)


def main() -> None:
    ap = argparse.ArgumentParser()
    ap.add_argument("--c1", action="store_true")
    ap.add_argument("--c1-leafi", action="store_true")
    ap.add_argument("--skip-small", action="store_true")
    a = ap.parse_args()
    if not a.skip_small:
        make_knowns()
        make_small()
        make_pipeline()
    if a.c1 or a.c1_leafi:
        make_c1(a.c1_leafi)


if __name__ == "__main__":
    main()
