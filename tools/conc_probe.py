"""Batches in flight on the bench workload: pipeline.SearchPipeline.run_resident with
1, 2, 3 and 4 graph plans (one compute stream each), 20 device-resident batches timed
with CUDA events; results checked against search_queries.
    python tools/conc_probe.py [bench args]"""
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
import numpy as np
import torch

import bench
from paper_2502_01836_b200.pipeline import SearchPipeline, search_queries

args = bench.make_parser().parse_args(sys.argv[1:] + ["--tdg-queries", "0"])
w = bench.setup_workload(args, torch.device("cuda", 0))
e, Q = w["eidx"], w["Q"]
ref = search_queries(e, Q, args.k, target=args.target)
Qd = Q.to("cuda", torch.float32).contiguous()
for plans in (1, 2, 3, 4):
    sp = SearchPipeline(e, Qd.shape[0], args.k, target=args.target, depth=plans, plans=plans)
    ids = sp.run_resident(Qd, 3)[0]
    torch.cuda.synchronize()
    assert np.array_equal(ids.cpu().numpy(), ref.ids)
    for rep in range(2):
        s = torch.cuda.current_stream()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(s)
        sp.run_resident(Qd, 20)
        e1.record(s)
        torch.cuda.synchronize()
        ms = e0.elapsed_time(e1) / 20
        print(f"plans={plans} ms/batch={ms:.3f} QPS={Qd.shape[0] / ms * 1e3:,.0f}", flush=True)
    del sp
