"""A/B of run-time switches on the bench workload, one setup: for each config
("VAR=VAL[,VAR=VAL...]", or "-" for the defaults) the plan cache is dropped, the
environment set, and 20 graph-plan launches timed with CUDA events; recall and
series scanned are checked on every config.
    CONFIGS="-;LF_PQB_R=4" python tools/ab_probe.py [bench args]"""
import os
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
import torch

import bench
from paper_2502_01836_b200.pipeline import search_queries

args = bench.make_parser().parse_args(sys.argv[1:] + ["--tdg-queries", "0"])
w = bench.setup_workload(args, torch.device("cuda", 0))
e, Q = w["eidx"], w["Q"]
configs = os.environ.get("CONFIGS", "-").split(";")
base_env = dict(os.environ)
for rep in range(2):
    for cfg in configs:
        os.environ.clear()
        os.environ.update(base_env)
        if cfg != "-":
            for kv in cfg.split(","):
                k, v = kv.split("=")
                os.environ[k] = v
        e.__dict__.pop("_plans", None)
        r = search_queries(e, Q, args.k, target=0.99)
        s = torch.cuda.current_stream()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(s)
        for _ in range(20):
            search_queries(e, Q, args.k, target=0.99, copy_out=False)
        e1.record(s)
        torch.cuda.synchronize()
        print(f"[{rep}] {cfg:40s} ms={e0.elapsed_time(e1) / 20:7.3f} scanned={int(r.stats[:, 5].sum())} "
              f"recall={bench.recall_of(r, w['exact']):.3f}", flush=True)
