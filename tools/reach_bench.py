"""Microbenchmark of the in-search inference kernel (lf_filter_predict_pairs_f16):
F filters at m = 256, Q queries, ~P/F pairs per filter; CUDA-event time per call.
LF_REACH_DBG bits isolate parts of the pipeline (see filters_tc.cu PairArgs.dbg)."""
import sys
from pathlib import Path
sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
import numpy as np
import torch

from paper_2502_01836_b200.filters import FilterPack

F, m, Q = 4096, 256, 1000
P = int(sys.argv[1]) if len(sys.argv) > 1 else 415_000
g = torch.Generator(device="cuda").manual_seed(0)
W1 = torch.randn((F, m, m), device="cuda", generator=g) * 0.05
pack = FilterPack(list(range(F)), W1, torch.randn((F, m), device="cuda") * 0.05,
                  torch.randn((F, m), device="cuda") * 0.05, torch.rand(F, device="cuda"), path="tc16")
q = torch.randn((Q, m), device="cuda")
pq = torch.randint(0, Q, (P,), device="cuda", dtype=torch.int32)
pf = torch.randint(0, F, (P,), device="cuda", dtype=torch.int32)
out = pack.predict_pairs(q, pq, pf)
if P <= 2_000_000:
    dense = pack.predict(q)
    ref = dense[pq.long(), pf.long()].double()
    print("max |pairs - dense|:", float((out - ref).abs().max()))
for rep in range(2):
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(10):
        pack.predict_pairs(q, pq, pf)
    e1.record()
    torch.cuda.synchronize()
    print(f"P={P}: {e0.elapsed_time(e1) / 10:.3f} ms per call (incl. bucketing)")
if len(sys.argv) > 2:
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(10):
        pack.predict(q)
    e1.record()
    torch.cuda.synchronize()
    print(f"dense {Q} x {F}: {e0.elapsed_time(e1) / 10:.3f} ms per call")
