#!/usr/bin/env python
"""LeaFi hot-path benchmark on B200 (BASELINE.json metric).

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference]

Workload (BASELINE.json configs[1]): 25M random-walk series of length 256,
DSTree-style tree with leaf cap 10,000, one learned filter per
leaf (enhance() on the GPU, lr 1e-3 at m=256), 1,000 queries
(250 per noise level 0.1/0.2/0.3/0.4), 1-NN at recall target
0.99.  A "step" is one batch of the 1,000 queries through the LeaFi search:
filter inference for every (query, filter) pair + bounds + visit order +
round-driven leaf scan (lf_filter_predict + lf_search).

Inputs: the collection is generated ON THE GPU (synth.randwalk_device: the
reference's law, torch Philox stream -- not numpy-bit-identical at 25M; the
parity tests use the numpy-exact generator at smaller n).  The collection
(25.6 GB) is far larger than L2 (126 MB), so no L2 flush is needed between
steps.

Metric: queries/s over the whole job (`value`), with recall@1 (cli.py:83-88)
against exact GPU search and leaves-pruned %.  `e2e` times the public API
`pipeline.search_queries` from pinned host queries to host results.
`roofline` is the leaf-scan kernel (the dominant kernel) against measured HBM
bandwidth; `cpu_baseline` is the CPU oracle (oracle/leafi_oracle.py, the
reference algorithm restated in numpy) on a bounded query sample, all host
cores.  `--impl reference` times that oracle alone as the reference arm.
"""

from __future__ import annotations

import argparse
import json
import math
import os
import statistics
import subprocess
import sys
import tempfile
import threading
import time
from pathlib import Path

import numpy as np

ROOT = Path(__file__).resolve().parent
sys.path.insert(0, str(ROOT))

FIXED = dict(t_series=2e-7, t_filter=6e-6)       # injected constants (reference tests/conftest.py:11)
NOISE_LEVELS = (0.1, 0.2, 0.3, 0.4)


HEADLINE = "1-NN queries/sec at 99% recall, 25M x 256 random-walk series; leaves pruned %"


def metric_name(args) -> str:
    """BASELINE.json's metric for the default workload; the analogous name for configs 3 / 5."""
    if args.k == 1 and args.dataset == "randwalk" and args.index == "dstree" and args.target == 0.99:
        return HEADLINE
    data = "Gaussian-mixture vectors" if args.dataset == "gmm" else "random-walk series"
    return (f"{args.k}-NN queries/sec at {args.target:.0%} target, {args.n} x {args.m} {data} "
            f"({'iSAX' if args.index == 'isax' else 'DSTree'}); leaves pruned %")


def log(*a):
    print("[bench]", *a, file=sys.stderr, flush=True)


# ------------------------------------------------------------------ clocks --
class ClockSampler:
    """nvidia-smi sampling DURING the timed region (B200_PROFILING.md clocks line)."""

    FIELDS = ("index,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
              "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
              "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, gpu_index: int):
        self.gpu = gpu_index
        self.proc = None
        self.path = None

    def __enter__(self):
        fd, self.path = tempfile.mkstemp(suffix=".csv")
        os.close(fd)
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", f"--id={self.gpu}", f"--query-gpu={self.FIELDS}", "--format=csv,noheader,nounits",
                 "-lms", "100"], stdout=open(self.path, "w"), stderr=subprocess.DEVNULL)
        except OSError:
            self.proc = None
        time.sleep(0.3)
        return self

    def __exit__(self, *exc):
        if self.proc is not None:
            self.proc.terminate()
            self.proc.wait()

    def summary(self) -> dict:
        sm, mx, reasons = [], None, set()
        try:
            for line in open(self.path):
                p = [x.strip() for x in line.split(",")]
                if len(p) < 9:
                    continue
                try:
                    sm.append(float(p[1]))
                    mx = float(p[2])
                except ValueError:
                    continue
                for name, v in zip(("hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"), p[5:9]):
                    if v.lower() == "active":
                        reasons.add(name)
        except OSError:
            pass
        finally:
            if self.path:
                os.unlink(self.path)
        return {"sm_mhz": statistics.median(sm) if sm else None, "sm_max_mhz": mx, "reasons": sorted(reasons),
                "samples": len(sm)}


# ------------------------------------------------------------------- setup --
def setup_workload(args, device, rank: int = 0, world: int = 1):
    """Collection, tree, filters, query batch and exact ground truth (untimed).

    world > 1 (leaf-sharded): every rank generates the collection and
    builds the same tree from its segment means, then keeps ONLY its leaf shard's
    rows (the full collection is dropped after enhancement); enhancement is sharded
    (training-data generation on the rank's leaves + all-gather, each rank trains
    only its own filters, calibration predictions all-gathered); the exact ground
    truth is the sharded exact search."""
    import torch

    from paper_2502_01836_b200 import build_index_device, search_batch
    from paper_2502_01836_b200 import pipeline as pl
    from paper_2502_01836_b200.synth import queries_device, randwalk_device
    from paper_2502_01836_b200.training import TrainConfig

    t0 = time.perf_counter()
    if args.dataset == "gmm":       # BASELINE config 5 (Deep1B-shaped Gaussian mixture)
        from paper_2502_01836_b200.synth import gaussian_mixture_device

        X = gaussian_mixture_device(args.n, args.m, args.seed, device=device)
    else:
        X = randwalk_device(args.n, args.m, args.seed, device=device)
    torch.cuda.synchronize()
    t_gen = time.perf_counter() - t0
    t0 = time.perf_counter()
    if args.index == "isax":        # BASELINE config 3
        from paper_2502_01836_b200.isax import build_isax_index

        tree = build_isax_index(X, max_leaf_size=args.leaf_cap, segments=8)
    else:
        tree = build_index_device(X, max_leaf_size=args.leaf_cap, segments=8)
    di = tree.device(device) if world == 1 else tree.shard(rank, world, device)
    torch.cuda.synchronize()
    t_build = time.perf_counter() - t0
    log(f"collection {args.n}x{args.m} in {t_gen:.1f}s; tree {tree.n_leaves} leaves / {tree.n_nodes} nodes in {t_build:.1f}s")
    fbytes = pl.filter_memory_bytes(args.m)
    consts = pl.RuntimeConstants(FIXED["t_series"], FIXED["t_filter"], fbytes)
    budget = pl.SelectionBudget(capacity_bytes=fbytes * tree.n_leaves, a=2.0)
    timings = {}
    t0 = time.perf_counter()
    shard = (rank, world, None) if world > 1 else None
    eidx = pl.enhance(tree, pl.SplitPlan(args.n_global, args.n_local, args.calibration), budget, args.seed,
                      constants=consts, train_cfg=TrainConfig(initial_lr=1e-3, max_epochs=args.max_epochs),
                      timings=timings, shard=shard)
    torch.cuda.synchronize()
    t_enh = time.perf_counter() - t0
    log(f"enhance {len(eidx.filters)} filters in {t_enh:.1f}s: " +
        ", ".join(f"{k}={v:.1f}s" for k, v in timings.items() if v > 0.05))
    per = args.queries // len(NOISE_LEVELS)
    Q = torch.cat([queries_device(X, per, nz, args.seed + int(10 * nz)) for nz in NOISE_LEVELS]).contiguous()
    tdg_q = None
    if args.tdg_queries > 0:
        tdg_q = torch.cat([queries_device(X, args.tdg_queries // 4, nz, args.seed + 77 + i)
                           for i, nz in enumerate(NOISE_LEVELS)]).contiguous()
    del X
    if world > 1:
        tree.release_rows()                  # the rank keeps its shard's rows only
    torch.cuda.empty_cache()
    t0 = time.perf_counter()
    if world > 1:
        from paper_2502_01836_b200.sharded import search_sharded

        exact = search_sharded(tree, Q, args.k, rank=rank, world=world)
    else:
        exact = search_batch(tree, Q, args.k)
    t_exact = time.perf_counter() - t0
    log(f"exact ground truth for {Q.shape[0]} queries in {t_exact:.2f}s "
        f"(pruning {np.mean(exact.pruning_ratios()):.4f})")
    return {"tree": tree, "eidx": eidx, "Q": Q, "exact": exact, "di": di, "tdg_q": tdg_q,
            "setup_s": {"generate": t_gen, "build": t_build, "enhance": t_enh, "exact": t_exact, **timings}}


def recall_of(res, exact) -> float:
    """cli.py:83-88: id match, or distance within 1e-6 relative (recall@1)."""
    rid, rd = res.ids[:, 0], res.dists[:, 0]
    oid, od = exact.ids[:, 0], exact.dists[:, 0]
    ok = (rid == oid) | (np.abs(rd - od) <= 1e-6 * np.maximum(od, 1e-300))
    return float(np.mean(ok))


# --------------------------------------------------------------- cpu oracle --
_OR = {}


def bench_config(args, tree, n_filters: int, nQ: int, world: int) -> dict:
    """The workload a bench line is quoted on -- one definition for both arms."""
    return {
        "workload": f"{'iSAX' if args.index == 'isax' else 'DSTree'}+LeaFi {args.n}x{args.m} "
                    f"{'Gaussian mixture' if args.dataset == 'gmm' else 'random walk'}, leaf cap {args.leaf_cap}, "
                    f"{nQ} queries (noise {'/'.join(map(str, NOISE_LEVELS))}), {args.k}-NN, target {args.target}",
        "n_series": args.n, "length": args.m, "leaf_cap": args.leaf_cap, "leaves": tree.n_leaves,
        "filters": n_filters, "queries_per_step": nQ, "k": args.k, "recall_target": args.target,
        "parallelism": f"leaf-sharded x{world}" if world > 1 else "1 GPU",
        "l2": f"inputs larger than L2 ({args.n * args.m * 4 / 1e9:.1f} GB collection)",
    }


def _oracle_worker(qi_list):
    from threadpoolctl import threadpool_limits

    from oracle import leafi_oracle as lo

    t, preds, offs, Qh = _OR["tree"], _OR["preds"], _OR["offs"], _OR["Q"]
    out = []
    with threadpool_limits(limits=1):              # one core per worker: BLAS stays single-threaded
        for qi in qi_list:
            o = lo.search(t, Qh[qi], _OR.get("k", 1), predictors=preds, offsets=offs)
            out.append((qi, o.results[0][0], o.stats["series_scanned"]))
    return out


def _oracle_exact_worker(qi_list):
    """Exact search (tree.py:300-302) of the oracle: ids, distances, counters."""
    from oracle import leafi_oracle as lo

    t, Qh = _OR["tree"], _OR["Q"]
    out = []
    for qi in qi_list:
        o = lo.search(t, Qh[qi], 1)
        out.append((qi, [a for a, _ in o.results], [d for _, d in o.results], [o.stats[k] for k in lo.STAT_KEYS]))
    return out


def _oracle_injected_worker(qi_list):
    """The LeaFi cascade of the oracle fed the GPU's own predictions (so any
    difference is the search, not the filter arithmetic)."""
    from oracle import leafi_oracle as lo

    t, Qh, P, offs, lids = _OR["tree"], _OR["Q"], _OR["P"], _OR["offs"], _OR["pack_leaves"]
    out = []
    for qi in qi_list:
        preds = {l: (lambda x, v=float(P[qi, j]): v) for j, l in enumerate(lids)}
        o = lo.search(t, Qh[qi], 1, predictors=preds, offsets=offs)
        out.append((qi, [a for a, _ in o.results], [d for _, d in o.results], [o.stats[k] for k in lo.STAT_KEYS]))
    return out


def oracle_map(fn, idx, workers: int):
    import multiprocessing as mp

    chunks = [c for c in (list(idx[i::workers]) for i in range(workers)) if c]
    with mp.get_context("fork").Pool(len(chunks)) as pool:
        return sorted((r for part in pool.map(fn, chunks) for r in part), key=lambda r: r[0])


def parity_25m(w, workers: int) -> dict:
    """Parity at the headline configuration (rank 0, after oracle_setup):
    (1) exact mode, >= 64 queries (16 per noise level): the oracle's exact search
        (tree.py:300-302) vs the GPU's exact search on the same 25M tree --
        ids identical, distances within 1e-4 relative (north_star) and, with the
        sequential schedule, every counter identical;
    (2) LeaFi cascade: the oracle fed the GPU's own predictions vs the GPU's
        sequential filtered search -- ids and counters identical;
    (3) filter arithmetic A/B: the fp32 CUDA-core pack vs the fp16 tensor-core pack
        on the same trained filters and offsets, all queries: recall, leaves
        pruned, and the (query, filter) prune decisions against the true 1-NN
        distance (pred - offset > d*) that agree;
    (4) training-data generation spot check: exact min distances of sampled
        (query, leaf) pairs recomputed on the host in fp64."""
    import torch

    from oracle import leafi_oracle as lo
    from paper_2502_01836_b200 import search_batch
    from paper_2502_01836_b200.filters import FilterPack

    tree, eidx, Q, exact, di = w["tree"], w["eidx"], w["Q"], w["exact"], w["di"]
    nQ = Q.shape[0]
    per = nQ // len(NOISE_LEVELS)
    take = max(16, 64 // len(NOISE_LEVELS))
    idx = np.concatenate([i * per + np.linspace(0, per - 1, take).astype(int) for i in range(len(NOISE_LEVELS))])
    out = {"queries": int(len(idx)), "sample": f"{take} per noise level, evenly spaced"}
    # (1) exact mode
    t0 = time.perf_counter()
    ores = oracle_map(_oracle_exact_worker, idx, workers)
    seq = search_batch(tree, Q[idx], 1, sequential=True)
    oid = np.array([r[1][0] for r in ores])
    od = np.array([r[2][0] for r in ores])
    ost = np.array([r[3] for r in ores])
    rel = np.abs(seq.dists[:, 0] - od) / np.maximum(od, 1e-300)
    out["exact"] = {"ids_identical": bool((seq.ids[:, 0] == oid).all()),
                    "batched_ids_identical": bool((exact.ids[idx, 0] == oid).all()),
                    "max_rel_dist_err": float(rel.max()), "dist_tolerance": 1e-4,
                    "counters_identical_sequential": bool((seq.stats == ost).all()),
                    "oracle_s": time.perf_counter() - t0}
    # (2) LeaFi cascade with identical predictions
    pack = eidx.pack
    P = pack.predict(Q)
    offv = eidx.offset_vector(w["target"], device=True)
    _OR.update(P=P.cpu().numpy(), pack_leaves=list(pack.leaf_ids))
    ires = oracle_map(_oracle_injected_worker, idx, workers)
    fseq = search_batch(tree, Q[idx], 1, predictions=P[torch.as_tensor(idx, device=P.device)], offsets=offv,
                        leaf_filter=pack.leaf_filter(di), sequential=True)
    out["leafi_same_predictions"] = {
        "ids_identical": bool((fseq.ids[:, 0] == np.array([r[1][0] for r in ires])).all()),
        "counters_identical_sequential": bool((fseq.stats == np.array([r[3] for r in ires])).all())}
    # (3) fp32 CUDA-core pack vs the fp16 tensor-core pack
    p32 = FilterPack.from_models(eidx.filters, device=P.device, path="simt")
    P32 = p32.predict(Q)
    res16 = search_batch(tree, Q, 1, predictions=P, offsets=offv, leaf_filter=pack.leaf_filter(di))
    res32 = search_batch(tree, Q, 1, predictions=P32, offsets=offv, leaf_filter=p32.leaf_filter(di))
    dstar = torch.as_tensor(exact.dists[:, 0], device=P.device)[:, None]
    off_row = offv[None, :]
    d16 = (P.double() - off_row) > dstar
    d32 = (P32.double() - off_row) > dstar
    diff = (P.double() - P32.double()).abs()
    out["filter_precision_ab"] = {
        "recall_fp16_pack": recall_of(res16, exact), "recall_fp32_pack": recall_of(res32, exact),
        "leaves_pruned_pct_fp16_pack": 100.0 * (1.0 - float(np.mean(res16.stats[:, 1])) / tree.n_leaves),
        "leaves_pruned_pct_fp32_pack": 100.0 * (1.0 - float(np.mean(res32.stats[:, 1])) / tree.n_leaves),
        "prune_decisions_agree": float((d16 == d32).double().mean().item()),
        "prune_decisions": int(d16.numel()),
        "max_abs_pred_diff": float(diff.max().item()),
        "max_rel_pred_diff": float((diff / P32.double().abs().clamp_min(1e-30)).max().item()),
        "definition": "decision per (query, filter): pred - offset > exact 1-NN distance; both packs share "
                      "the filters and the offsets fitted on the fp16 pack"}
    del P32, p32
    # (4) training-data generation spot check
    if w.get("tdg_sample") is not None:
        gq, dl, slots = w["tdg_sample"]
        errs = []
        for qi, s_ in zip(range(gq.shape[0]), slots):
            r0, r1 = int(di.leaf_ptr_host[s_]), int(di.leaf_ptr_host[s_ + 1])
            rows = di.X[r0:r1].cpu().numpy()
            ref = float(lo.pair_dist(gq[qi:qi + 1], rows).min())
            errs.append(abs(dl[qi] - ref) / max(ref, 1e-300))
        out["train_data_gen_spot_check"] = {"pairs": len(errs), "max_rel_err": float(max(errs))}
    return out


def oracle_setup(w) -> None:
    """OracleTree over a host copy of the collection + numpy filter callables."""
    from oracle import leafi_oracle as lo

    tree, eidx = w["tree"], w["eidx"]
    di = w["di"]
    # host copy of the leaf-contiguous device rows, re-indexed by series id
    X = di.X.cpu().numpy()
    rowpos = np.empty(tree.n, dtype=np.int64)
    rowpos[di.row_id.cpu().numpy()] = np.arange(tree.n)

    class RowsById:
        shape = (tree.n, tree.m)

        def __getitem__(self, ids):
            return X[rowpos[ids]]

    ot = lo.OracleTree(RowsById(), tree.starts, tree.widths, tree.max_leaf_size)
    for i in range(tree.n_nodes):
        ot.env_min.append(tree.env_min[i]); ot.env_max.append(tree.env_max[i])
        ot.left.append(int(tree.left[i])); ot.right.append(int(tree.right[i]))
        ot.split_seg.append(int(tree.split_seg[i])); ot.split_thr.append(float(tree.split_thr[i]))
        ot.member_lists.append(None if tree.left[i] >= 0 else [])
        ot.size.append(int(tree.size[i])); ot.oversized.append(bool(tree.oversized[i]))
    ot.members = {int(l): tree.leaf_members(int(l)) for l in tree.leaf_ids}
    filt = eidx.filters
    preds = {l: (lambda x, f=filt[l]: lo.mlp_forward(f.W1, f.b1, f.W2, f.b2, x)) for l in filt}
    offs = eidx.tuned_offsets(w["target"])
    _OR.update(tree=ot, preds=preds, offs=offs, Q=w["Q"].cpu().numpy().astype(np.float64), k=w.get("k", 1))


def oracle_time(sample_idx, workers: int) -> tuple:
    """Run the oracle on `sample_idx` queries across `workers` forked processes."""
    import multiprocessing as mp

    chunks = [list(sample_idx[i::workers]) for i in range(workers)]
    chunks = [c for c in chunks if c]
    t0 = time.perf_counter()
    if workers == 1:
        res = _oracle_worker(chunks[0])
    else:
        with mp.get_context("fork").Pool(len(chunks)) as pool:
            res = [r for part in pool.map(_oracle_worker, chunks) for r in part]
    return time.perf_counter() - t0, res


def oracle_sample_size(budget_s: float, workers: int) -> int:
    """Calibrate the sample so the oracle leg stays within ~budget_s of CPU work."""
    nQ = _OR["Q"].shape[0]
    probe = [0, nQ // 4, nQ // 2, (3 * nQ) // 4]          # one query per noise level
    t1, _ = oracle_time(probe, 1)
    per_q = max(t1 / len(probe), 1e-3)
    return int(max(workers, min(_OR["Q"].shape[0], budget_s * workers / per_q)))


# ----------------------------------------------------------------- timing --
def peaks() -> tuple:
    p = ROOT / "MEASURED_PEAKS.json"
    if p.exists():
        d = json.loads(p.read_text())
        return float(d["hbm_gbs"]), "measured (MEASURED_PEAKS.json hbm_gbs)"
    return 6650.0, "fallback (B200_PROFILING.md)"


def bf16_peak() -> float:
    p = ROOT / "MEASURED_PEAKS.json"
    return float(json.loads(p.read_text())["bf16_tflops"]) if p.exists() else 1590.0


def tf32_peak() -> float:
    p = ROOT / "MEASURED_PEAKS.json"
    bf16 = json.loads(p.read_text())["bf16_tflops"] if p.exists() else 1590.0
    return float(bf16) / 2.0


def ncu_traffic():
    """Per-launch DRAM bytes of the scan kernel from the committed ncu capture, if any."""
    p = ROOT / "profiles" / "scan_kernel_ncu.json"
    if p.exists():
        d = json.loads(p.read_text())
        return d.get("dram_bytes_per_launch"), d.get("algorithmic_bytes_per_launch")
    return None, None


def bounds_roofline(tree, nQ: int, ms: float, hbm: float, peak_src: str) -> dict:
    """Roofline entry of the bound + visit-order phase: algorithmic
    bytes = envelopes once per batch (nodes x 2 l x 8 B) + per query and node its
    bound and id written and read by the sort (Q x nodes x 12 B); also the bytes
    this implementation actually moves (bound matrix written and read, 8 B per
    (query, node) each way, leaf records 28 B per (query, leaf))."""
    nodes, L, l = tree.n_nodes, tree.n_leaves, tree.n_seg
    alg = nodes * 2 * l * 8 + nQ * nodes * 12
    moved = nodes * 2 * l * 8 + nQ * nodes * 16 + nQ * L * 28
    return {"kernels": "paa_kernel + lb_tile_kernel (bound matrix, L2-resident) + leaf_order_kernel (counting sort "
                       "of the leaves, gap bounds of the internal nodes, leaf records)",
            "bound": "latency (one CTA per query; see profiles/r02)", "ms": ms,
            "algorithmic_bytes": alg, "achieved": alg / (ms / 1e3) / 1e9 if ms > 0 else None,
            "peak": hbm, "unit": "GB/s", "frac": alg / (ms / 1e3) / 1e9 / hbm if ms > 0 else None,
            "peak_source": peak_src,
            "moved_bytes": moved, "moved_GBps": moved / (ms / 1e3) / 1e9 if ms > 0 else None,
            "definition": "algorithmic: nodes x 2 x segments x 8 B + queries x nodes x (8 B bound + 4 B id)"}


def run_ours(args, rank, world, device):
    import torch
    import torch.distributed as dist

    from paper_2502_01836_b200 import _lib
    from paper_2502_01836_b200.pipeline import search_queries

    w = setup_workload(args, device, rank, world)
    w["target"] = args.target
    w["k"] = args.k
    eidx, Q, exact, tree = w["eidx"], w["Q"], w["exact"], w["tree"]
    nQ = Q.shape[0]
    stream = torch.cuda.current_stream()
    prof = np.zeros(_lib.N_PROF)

    if world == 1 and not args.sharded:
        def step(profile=None):
            return search_queries(eidx, Q, args.k, target=args.target, copy_out=False, profile=profile,
                                  lazy=args.lazy)

        def checked(queries):
            return search_queries(eidx, queries, args.k, target=args.target, lazy=args.lazy)
    else:
        # leaf-sharded: this rank's leaves, rows and filters; one MIN-allreduce per round
        from paper_2502_01836_b200.filters import FilterPack
        from paper_2502_01836_b200.sharded import search_sharded

        a, b = tree.shard(rank, world).leaf_range
        local = [int(l) for l in tree.leaf_ids[a:b] if int(l) in eidx.filters]
        lpack = (eidx.pack if world > 1 else FilterPack.from_models({l: eidx.filters[l] for l in local})) \
            if local else None                     # world > 1: enhance() trained this rank's filters only
        offs_all = eidx.tuned_offsets(args.target)
        loffs = np.array([offs_all[l] for l in local], dtype=np.float64)

        def step(profile=None):
            return search_sharded(tree, Q, args.k, rank=rank, world=world, pack=lpack, offsets=loffs,
                                  copy_out=False, profile=profile, lazy=args.lazy)

        def checked(queries):
            return search_sharded(tree, queries, args.k, rank=rank, world=world, pack=lpack, offsets=loffs,
                                  lazy=args.lazy)

    lazy_on = args.lazy is not False and eidx.pack.path == "tc16"
    for _ in range(args.warmup):
        step()
    torch.cuda.synchronize()
    # one checked run: recall and pruning of the exact workload being timed
    chk = checked(Q)
    recall = recall_of(chk, exact)
    recall_k = None
    if args.k > 1:
        from paper_2502_01836_b200.synth import recall_at_k

        recall_k = float(np.mean(recall_at_k(chk.ids, exact.ids)))
    per_noise = {}
    per = nQ // len(NOISE_LEVELS)
    for i, nz in enumerate(NOISE_LEVELS):
        sl = slice(i * per, (i + 1) * per)
        ok = (chk.ids[sl, 0] == exact.ids[sl, 0]) | (np.abs(chk.dists[sl, 0] - exact.dists[sl, 0]) <= 1e-6 * exact.dists[sl, 0])
        per_noise[str(nz)] = {"recall": float(np.mean(ok)),
                              "pruning": float(np.mean(chk.pruning_ratios()[sl])),
                              "leaves_searched": float(np.mean(chk.stats[sl, 1]))}
    # filter inference alone (the tensor-core kernel), events on the launching stream
    fe0 = torch.cuda.Event(enable_timing=True)
    fe1 = torch.cuda.Event(enable_timing=True)
    fe0.record(stream)
    for _ in range(5):
        eidx.pack.predict(Q)
    fe1.record(stream)
    torch.cuda.synchronize()
    filter_ms = fe0.elapsed_time(fe1) / 5
    F = eidx.pack.n_filters
    filter_tflops = 2.0 * nQ * F * tree.m * (tree.m + 1) / (filter_ms / 1e3) / 1e12
    leaves_pruned = 1.0 - float(np.mean(chk.stats[:, 1])) / tree.n_leaves
    series_pruned = float(np.mean(chk.pruning_ratios()))
    scanned_per_step = int(chk.stats[:, 5].sum())

    # timed region: K steps, events on the launching stream, barrier + sync both sides
    if world > 1:
        dist.barrier()
    torch.cuda.synchronize()
    if args.ncu:
        torch.cuda.cudart().cudaProfilerStart()
    with ClockSampler(torch.cuda.current_device()) as clk:
        ev0 = torch.cuda.Event(enable_timing=True)
        ev1 = torch.cuda.Event(enable_timing=True)
        ev0.record(stream)
        for _ in range(args.steps):
            step()
        ev1.record(stream)
        torch.cuda.synchronize()
    if args.ncu:
        torch.cuda.cudart().cudaProfilerStop()
    if world > 1:
        dist.barrier()
    ms = ev0.elapsed_time(ev1)
    t = torch.tensor([ms], dtype=torch.float64, device=device)
    if world > 1:
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
    ms = float(t.item())
    ms_per_step = ms / args.steps
    value = nQ * args.steps / (ms / 1e3)
    clocks = clk.summary()
    seq_value, seq_ms = value, ms_per_step

    # the serving form (one GPU, in-search inference, graph plans): the same K batches
    # with three in flight -- consecutive batches alternate between three graph plans on
    # three compute streams (pipeline.SearchPipeline.run_resident), the whole job timed with
    # events on the launching stream; this is `value`, the one-batch-at-a-time
    # throughput above is reported beside it
    pipe = None
    if world == 1 and lazy_on and os.environ.get("LF_SEARCH_GRAPH", "1") != "0" and not args.ncu:
        from paper_2502_01836_b200.pipeline import SearchPipeline

        pipe = SearchPipeline(eidx, nQ, args.k, target=args.target)
        Qd = Q.to(device=device, dtype=torch.float32).contiguous()
        ids_last = pipe.run_resident(Qd, max(args.warmup, 2), stream=stream)[0]
        torch.cuda.synchronize()
        assert np.array_equal(ids_last.cpu().numpy(), chk.ids)
        with ClockSampler(torch.cuda.current_device()) as clk2:
            cv0 = torch.cuda.Event(enable_timing=True)
            cv1 = torch.cuda.Event(enable_timing=True)
            cv0.record(stream)
            pipe.run_resident(Qd, args.steps, stream=stream)
            cv1.record(stream)
            torch.cuda.synchronize()
        cms = cv0.elapsed_time(cv1)
        value, ms_per_step, clocks = nQ * args.steps / (cms / 1e3), cms / args.steps, clk2.summary()

    # the same K steps again with the library's per-phase CUDA events (h_profile) for
    # the roofline and the phase split; kept out of the timed region above (the event
    # records and read-backs cost host time)
    scan_ms, scan_launches, kernels, bounds_ms = 0.0, 0, 0, 0.0
    ea_rows, ea_surv, refills, pred_ms, lazy_pairs, pred_steps = 0.0, 0.0, 0.0, 0.0, 0.0, 0.0
    stream_b, exact_b = 0.0, 0.0
    for _ in range(args.steps):
        step(prof)
        scan_ms += prof[2]
        bounds_ms += prof[0]
        scan_launches += int(prof[4])
        ea_rows += prof[8]
        ea_surv += prof[9]
        refills += prof[7]
        pred_ms += prof[10]
        lazy_pairs += prof[11]
        pred_steps += prof[12]
        stream_b += prof[13]
        exact_b += prof[14]
        kernels += int(prof[5]) + (0 if lazy_on else 2 if eidx.pack.path == "tc16" else 1)   # + dense pass
    torch.cuda.synchronize()

    # training-data generation (BASELINE config 4 shape): exact query x leaf min-ED
    tdg = None
    if args.tdg_queries > 0:
        from paper_2502_01836_b200.synth import queries_device
        from paper_2502_01836_b200.targets import default_path, leaf_min_distances

        gq = w["tdg_q"]
        # leaf-sharded like the search: this rank's leaves, all queries
        tdi = tree.shard(rank, world) if world > 1 else w["di"]
        slots = list(range(tdi.n_leaves))
        leaf_min_distances(tree, gq[:256], slots, dindex=tdi)           # warm-up / tensor maps
        torch.cuda.synchronize()
        if world > 1:
            dist.barrier()
        te0 = torch.cuda.Event(enable_timing=True)
        te1 = torch.cuda.Event(enable_timing=True)
        te0.record(stream)
        dl = leaf_min_distances(tree, gq, slots, dindex=tdi)
        te1.record(stream)
        torch.cuda.synchronize()
        t_ms = te0.elapsed_time(te1)
        # member rows as queries: their own leaf's minimum must be exactly 0.0
        mslots = np.linspace(0, tdi.n_leaves - 1, 16).astype(int)
        mrows = torch.stack([tdi.X[int(tdi.leaf_ptr_host[s_])] for s_ in mslots]).contiguous()
        mdl = leaf_min_distances(tree, mrows, slots, dindex=tdi)
        member_zero = bool((mdl[torch.arange(16), torch.as_tensor(mslots)] == 0.0).all().item())
        # a sample of (query, leaf) minima for the host fp64 spot check (parity block)
        samp = np.linspace(0, gq.shape[0] - 1, 8).astype(int)
        sslots = np.linspace(0, tdi.n_leaves - 1, 8).astype(int)
        w["tdg_sample"] = (gq[samp].double().cpu().numpy(), dl[samp, sslots].cpu().numpy(), sslots)
        if world > 1:
            tt = torch.tensor([t_ms], dtype=torch.float64, device=device)
            dist.all_reduce(tt, op=dist.ReduceOp.MAX)
            t_ms = float(tt.item())
        pairs = gq.shape[0] * tree.n
        flops = 2.0 * pairs * tree.m
        path = default_path(tree, w["di"])
        if path == "q8":
            pk, pk_src = 2.0 * bf16_peak(), "dense int8 = 2 x measured bf16 (MEASURED_PEAKS.json bf16_tflops)"
            desc = "tcgen05 kind::i8 GEMM over the int8 shadow + exact fp64 re-check (lf_leaf_min_dist_q8)"
        else:
            pk, pk_src = tf32_peak(), "dense tf32 = 1/2 of measured bf16 (MEASURED_PEAKS.json bf16_tflops)"
            desc = "tcgen05 tf32 GEMM + exact fp64 re-check (lf_leaf_min_dist_tc)"
        tdg = {"queries": int(gq.shape[0]), "leaves": tree.n_leaves, "series": tree.n, "ms": t_ms,
               "sharding": f"leaf-sharded x{world}, max over ranks" if world > 1 else "1 GPU",
               "pairs_per_s": pairs / (t_ms / 1e3), "algorithmic_tflops": flops / (t_ms / 1e3) / 1e12,
               "algorithmic_flops_definition": "2 x queries x series x m (each pair's dot product once)",
               "tensor_peak_tops": pk, "peak_source": pk_src,
               "frac_of_peak": flops / (t_ms / 1e3) / 1e12 / pk,
               "path": desc,
               "member_rows_exact_zero": member_zero,
               "reference_cpu_pairs_per_s_per_core": "1.0-1.3e6 (BASELINE.md, collect_targets at C1)"}
        del dl, gq

    # e2e through the public API: pinned host queries in, host results out.  One GPU
    # with in-search inference: the serving form (pipeline.SearchPipeline), each batch's
    # copies overlapping the previous batch's search; otherwise search_queries /
    # search_sharded call by call.
    Qh = Q.cpu().pin_memory()

    def e2e_run(steps):
        if pipe is None:
            r = None
            for _ in range(steps):
                r = checked(Qh)
            return r
        pending, r = [], None                    # up to pipe.depth batches in flight
        for _ in range(steps):
            if len(pending) == pipe.depth:
                r = pipe.result(pending.pop(0))
            pending.append(pipe.submit(Qh))
        while pending:
            r = pipe.result(pending.pop(0))
        return r

    r = e2e_run(2)
    if pipe is not None:                                 # the pipeline returns the checked results
        assert np.array_equal(r.ids, chk.ids) and np.array_equal(r.stats, chk.stats)
    torch.cuda.synchronize()
    if world > 1:
        dist.barrier()
    e0 = time.perf_counter()
    r = e2e_run(args.steps)
    torch.cuda.synchronize()
    if world > 1:
        dist.barrier()
    e_s = (time.perf_counter() - e0) / args.steps
    e2e = {"value": nQ / e_s, "unit": "queries/s", "h2d_bytes_per_step": int(Q.numel() * 4),
           "d2h_bytes_per_step": int(nQ * (8 + 8 + 6 * 8)), "ms_per_step": e_s * 1e3,
           "api": "pipeline.SearchPipeline (submit / result; copies overlap the previous batch's search, "
                  "consecutive batches alternate between three graph plans on three compute streams)"
                  if pipe is not None else "search_queries per batch"}

    hbm, peak_src = peaks()
    # bytes the scan must move: the int8 shadow (1 B/dim + 12 B/row of scale, code norm,
    # quantisation error) for every scanned series, plus the exact fp32 row (4 B/dim) for
    # the survivors of the bound; the reference reads 4 B/dim for every scanned series.
    ref_bytes = scanned_per_step * tree.m * 4 * args.steps
    if stream_b > 0:
        alg_bytes = stream_b + exact_b
        bytes_def = ("bytes the scan kernels must move, counted in the kernels: per tested row its projected "
                     "codes (pca_k bytes) + 8 B fp16 metadata; per projected survivor its int8 row + 16 B "
                     "metadata; m x 4 B for every row re-read exactly")
    else:
        alg_bytes = ref_bytes
        bytes_def = "series_scanned x m x 4 B"
    achieved = alg_bytes / (scan_ms / 1e3) / 1e9 if scan_ms > 0 else None
    ref_equiv = ref_bytes / (scan_ms / 1e3) / 1e9 if scan_ms > 0 else None
    traffic, _ = ncu_traffic()
    if eidx.pack.path == "tc16":
        fpk, fpk_src = 2.0 * tf32_peak(), "dense f16 = measured bf16 (MEASURED_PEAKS.json bf16_tflops)"
    else:
        fpk, fpk_src = tf32_peak(), "dense tf32 = 1/2 of measured bf16 (MEASURED_PEAKS.json bf16_tflops)"
    di = w.get("di")
    pca_k = int(getattr(di, "pca_k", 0) or 0)
    pca_energy = getattr(di, "pca_energy", None)
    pq_on = pca_k > 0 and os.environ.get("LF_SCAN_VARIANT") in (None, "", "pq")
    line = {
        "metric": metric_name(args),
        "value": value,
        "unit": "queries/s",
        "n_gpus": world,
        "steps": args.steps,
        "warmup": args.warmup,
        "ms_per_step": ms_per_step,
        "batches_in_flight": pipe.depth if pipe is not None else 1,
        "value_one_batch_in_flight": seq_value,
        "ms_per_step_one_batch_in_flight": seq_ms,
        "higher_is_better": True,
        "scaling": "strong",
        "vs_baseline": None,
        "dtype": "f64-accumulated f32 series (scan/bounds), " + (
            "filters on fp16 operands (power-of-two scaled, tf32 mantissa) with f32 accumulation"
            if eidx.pack.path == "tc16" else "tf32 filters" if eidx.pack.path == "tc" else "f32 filters"),
        "data": (f"synthetic {'Gaussian mixture' if args.dataset == 'gmm' else 'random walk (reference law, Philox stream)'} "
                 f"generated on device, {args.n * args.m * 4 / 1e9:.1f} GB >> L2: no flush needed"),
        "config": bench_config(args, tree, len(eidx.curves) if world > 1 else len(eidx.filters), nQ, world),
        "recall_at_1": recall,
        **({f"recall_at_{args.k}": recall_k} if args.k > 1 else {}),
        "leaves_pruned_pct": 100.0 * leaves_pruned,
        "series_pruning_ratio": series_pruned,
        "per_noise": per_noise,
        "counters_per_query": {name: {"mean": float(np.mean(chk.stats[:, j])), "max": int(np.max(chk.stats[:, j]))}
                               for j, name in enumerate(("leaves_visited", "leaves_searched", "leaves_lb_pruned",
                                                         "leaves_filter_pruned", "filter_inferences",
                                                         "series_scanned"))},
        "visit_order_refills_per_step": refills / args.steps,
        "clocks": clocks,
        "e2e": e2e,
        "gpu_launches": kernels,
        "roofline": {
            "kernel": ("leaf scan (scan_q8_kernel round 0, then scan_pq_kernel -> pq_q8_bound_kernel -> "
                       "pq_tail_kernel: projected-int8 / int8 bounds, exact fp64 survivors)") if pq_on
                      else "leaf scan (scan_q8_kernel: TMA-pipelined int8-bounded scan, exact fp64 survivors)",
            "projected_shadow": {"pca_k": pca_k, "energy": pca_energy,
                                 "used": pq_on} if pca_k or pca_energy is not None else None,
            "bound": "hbm",
            "achieved": achieved, "peak": hbm, "unit": "GB/s",
            "frac": (achieved / hbm) if achieved else None, "traffic": traffic,
            "peak_source": peak_src,
            "algorithmic_bytes_per_step": alg_bytes / args.steps,
            "algorithmic_bytes_definition": bytes_def,
            "survivor_fraction": (ea_surv / ea_rows) if ea_rows else None,
            "reference_equivalent_GBps": ref_equiv,
            "reference_equivalent_definition": "series_scanned x m x 4 B (every scanned series read in fp32) / scan time",
            "scan_ms_per_step": scan_ms / args.steps, "scan_launches_per_step": scan_launches / args.steps,
            "phase_ms_last_step": {"filter_inference": prof[10] if lazy_on else filter_ms,
                                   "bounds+sort": prof[0], "plan": prof[1],
                                   "scan": prof[2], "merge": prof[3], "lf_search_total": prof[6]},
        },
        "bounds_roofline": bounds_roofline(tree, nQ, bounds_ms / args.steps, hbm, peak_src),
        "filter_inference": {
            "mode": ("in-search: one pass right after round 0 over the (query, filtered leaf) pairs with "
                     "lb <= bsf0 * f (all the walk can still reach), tcgen05 kind::f16 with the query rows "
                     "gathered by cp.async, bit-identical to the dense kernel") if lazy_on else
                    ("dense: one tcgen05 pass over every (query, filter) pair before lf_search ("
                     + ("kind::f16 over power-of-two-scaled fp16 operands" if eidx.pack.path == "tc16"
                        else eidx.pack.path) + ")"),
            "pairs_per_step": lazy_pairs / args.steps, "dense_pairs_per_step": nQ * F,
            "ms_per_step": pred_ms / args.steps, "passes_per_step": pred_steps / args.steps,
            "pair_flops_per_step": 2.0 * (lazy_pairs / args.steps) * tree.m * (tree.m + 1),
            # the in-search pass (pair lists + GEMM) streams every filter's fp16 W1 once: HBM-bound
            "in_search_roofline": ({
                "bound": "hbm", "unit": "GB/s", "peak": hbm, "peak_source": peak_src,
                "algorithmic_bytes": float(F) * tree.m * tree.m * 2 + (lazy_pairs / args.steps) * 16,
                "definition": "F x m x m x 2 B (each filter's fp16 W1 once) + 16 B per predicted pair "
                              "(pair record + record update); ms = the whole pass (pair ranges, buckets, GEMM)",
                "achieved": (float(F) * tree.m * tree.m * 2 + (lazy_pairs / args.steps) * 16)
                            / (pred_ms / args.steps / 1e3) / 1e9,
                "frac": (float(F) * tree.m * tree.m * 2 + (lazy_pairs / args.steps) * 16)
                        / (pred_ms / args.steps / 1e3) / 1e9 / hbm,
            } if lazy_on and pred_ms > 0 else None),
            "dense_kernel": {
                "path": eidx.pack.path, "bound": "tensor", "ms": filter_ms, "achieved": filter_tflops,
                "unit": "TFLOP/s", "peak": fpk, "frac": filter_tflops / fpk,
                "flops_per_launch": 2.0 * nQ * F * tree.m * (tree.m + 1),
                "peak_source": fpk_src,
                "note": "every (query, filter) pair; used for calibration, timed here for reference",
            },
        },
        "setup_s": w["setup_s"],
        "train_data_gen": tdg,
    }
    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        workers = os.cpu_count() or 1
        oracle_setup(w)
        n_s = oracle_sample_size(args.cpu_budget_s, workers)
        idx = np.linspace(0, nQ - 1, n_s).astype(int)
        el, res = oracle_time(idx, workers)
        agree = float(np.mean([chk.ids[qi, 0] == rid for qi, rid, _ in res]))
        line["parity_25M"] = parity_25m(w, workers)
        line["cpu_baseline"] = {"value": len(idx) / el, "unit": "queries/s", "cores": workers, "kind": "port",
                                "sample": f"{len(idx)} of the {nQ} benchmark queries (evenly spaced over the 4 noise "
                                          f"levels), oracle/leafi_oracle.search with the same tree, filters and "
                                          f"offsets, {workers} forked processes (one BLAS thread each), {el:.1f}s",
                                "ids_agree_with_gpu": agree}
        idx1 = np.linspace(0, nQ - 1, max(4, min(nQ, len(idx) // (4 * workers)))).astype(int)
        t1, _ = oracle_time(idx1, 1)
        line["cpu_baseline"]["one_core"] = {"value": len(idx1) / t1, "unit": "queries/s", "cores": 1,
                                            "sample": f"{len(idx1)} queries evenly spaced over the noise levels"}
    return line


def run_reference(args, rank, world, device):
    """The reference arm: the CPU oracle (restated reference algorithm) on the box's cores."""
    w = setup_workload(args, device)
    w["target"] = args.target
    w["k"] = args.k
    workers = os.cpu_count() or 1
    oracle_setup(w)
    nQ = w["Q"].shape[0]
    n_s = oracle_sample_size(args.ref_step_s, workers)
    idx_all = np.arange(nQ)
    for s in range(args.warmup):
        oracle_time(idx_all[:workers], workers)
    times, n_done = [], 0
    for s in range(args.steps):
        idx = np.roll(idx_all, -s * n_s)[:n_s]
        el, _ = oracle_time(idx, workers)
        times.append(el)
        n_done += len(idx)
    value = n_done / sum(times)
    # one core: the reference's own single-threaded search loop (BASELINE.md asks for it)
    n1 = max(4, min(nQ, int(args.ref_step_s * 0.25 / max(1e-3, sum(times) / max(1, n_done) * workers))))
    t1, _ = oracle_time(idx_all[np.linspace(0, nQ - 1, n1).astype(int)], 1)
    return {
        "impl": "reference",
        "metric": metric_name(args),
        "value": value, "unit": "queries/s", "n_gpus": world, "steps": args.steps, "warmup": args.warmup,
        "ms_per_step": 1e3 * sum(times) / len(times), "higher_is_better": True, "scaling": "strong",
        "vs_baseline": None, "dtype": "f64 (numpy oracle)", "data": "same synthetic workload as the ours arm",
        "config": bench_config(args, w["tree"], len(w["eidx"].filters), nQ, world),
        "cpu_baseline": {"value": value, "unit": "queries/s", "cores": workers, "kind": "port",
                         "sample": f"{n_s} of the {nQ} benchmark queries per step over {workers} forked processes, "
                                   f"one BLAS thread each (oracle/leafi_oracle.search, the reference algorithm "
                                   f"restated; tree, filters and offsets are the ours-arm ones, built before "
                                   f"the timed region)",
                         "one_core": {"value": n1 / t1, "unit": "queries/s", "cores": 1,
                                      "sample": f"{n1} queries evenly spaced over the noise levels"}},
        "e2e": {"value": value, "unit": "queries/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }


def make_parser():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=20)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", choices=("ours", "reference"), default="ours")
    ap.add_argument("--n", "--rows", dest="n", type=int, default=25_000_000)
    ap.add_argument("--m", "--length", dest="m", type=int, default=256)
    ap.add_argument("--leaf-cap", type=int, default=10_000)
    ap.add_argument("--queries", type=int, default=1000)
    ap.add_argument("--target", type=float, default=0.99)
    ap.add_argument("--seed", type=int, default=1234)
    ap.add_argument("--n-global", type=int, default=1500)
    ap.add_argument("--n-local", type=int, default=500)
    ap.add_argument("--calibration", type=int, default=300)
    ap.add_argument("--cpu-budget-s", type=float, default=20.0)
    ap.add_argument("--ref-step-s", type=float, default=15.0)
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--max-epochs", type=int, default=1000, help="filter training cap (setup speed)")
    ap.add_argument("--sharded", action="store_true",
                    help="use the leaf-sharded round driver even on one GPU (what N>1 runs)")
    ap.add_argument("--tdg-queries", type=int, default=10000,
                    help="queries for the training-data-generation measurement (0 = skip)")
    ap.add_argument("--dataset", choices=("randwalk", "gmm"), default="randwalk",
                    help="gmm = BASELINE config 5's Gaussian mixture (use with --m 96 --k 10)")
    ap.add_argument("--index", choices=("dstree", "isax"), default="dstree",
                    help="isax = BASELINE config 3's index family")
    ap.add_argument("--k", type=int, default=1)
    ap.add_argument("--dense-filters", action="store_true",
                    help="A/B: one dense filter pass over every (query, filter) pair before lf_search "
                         "instead of the in-search pass over the reachable pairs")
    ap.add_argument("--ncu", action="store_true",
                    help="bracket the timed steps with cudaProfilerStart/Stop (ncu --profile-from-start off)")
    return ap


def main():
    args = make_parser().parse_args()
    args.lazy = False if args.dense_filters else None     # None: in-search inference on the fp16 pack
    if args.warmup < 3:
        log("warmup raised to 3 (timing rule)")
        args.warmup = 3

    if args.gpus > 1 and "WORLD_SIZE" not in os.environ:
        # one process per GPU: re-launch this command under torch.distributed.run
        import socket

        with socket.socket() as sk:
            sk.bind(("127.0.0.1", 0))
            port = sk.getsockname()[1]
        # torch.distributed.run would read the short "--n" / "--m" as ambiguous prefixes of
        # its own options: pass their long aliases
        alias = {"--n": "--rows", "--m": "--length"}
        passed = [alias.get(a.split("=")[0], a.split("=")[0]) + ("=" + a.split("=", 1)[1] if "=" in a else "")
                  if a.startswith("--") else a for a in sys.argv[1:]]
        cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={args.gpus}",
               "--master-addr", "127.0.0.1", "--master-port", str(port), str(Path(__file__).resolve()), *passed]
        log("launching", args.gpus, "ranks:", " ".join(cmd[1:6]))
        sys.exit(subprocess.call(cmd))

    import torch
    import torch.distributed as dist

    world = int(os.environ.get("WORLD_SIZE", "1"))
    if world != args.gpus:
        raise SystemExit(f"bench.py: --gpus {args.gpus} but WORLD_SIZE={world} (launch with "
                         f"--nproc-per-node {args.gpus}, or drop WORLD_SIZE and let --gpus spawn the ranks)")
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    dev_index = local % max(1, torch.cuda.device_count())     # > 1 rank per GPU only in functional tests
    torch.cuda.set_device(dev_index)
    device = torch.device("cuda", dev_index)
    if world > 1:
        backend = os.environ.get("LF_DIST_BACKEND", "nccl")   # gloo: functional test of N ranks on one GPU
        if backend == "nccl":
            dist.init_process_group("nccl", device_id=device)
        else:
            dist.init_process_group(backend)
    if args.impl == "reference":
        if rank != 0:
            if world > 1:
                dist.destroy_process_group()
            return
        line = run_reference(args, rank, world, device)
    else:
        line = run_ours(args, rank, world, device)
    if rank == 0:
        print(json.dumps(line), flush=True)
    if world > 1:
        dist.destroy_process_group()


if __name__ == "__main__":
    main()
