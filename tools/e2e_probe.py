"""Time the pieces of one LeaFi batch through the public API (device vs host inputs)."""
import sys, time
from pathlib import Path
sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
import numpy as np
import torch
from paper_2502_01836_b200 import build_index_device, search_batch
from paper_2502_01836_b200 import pipeline as pl
from paper_2502_01836_b200.synth import randwalk_device, queries_device
from paper_2502_01836_b200.training import TrainConfig

n = int(sys.argv[1]) if len(sys.argv) > 1 else 2_000_000
X = randwalk_device(n, 256, 1)
t = build_index_device(X, 2000)
t.device()
fb = pl.filter_memory_bytes(256)
e = pl.enhance(t, pl.SplitPlan(300, 50, 100), pl.SelectionBudget(fb * t.n_leaves), 1,
               constants=pl.RuntimeConstants(2e-7, 6e-6, fb), train_cfg=TrainConfig(initial_lr=1e-3, max_epochs=5))
Q = torch.cat([queries_device(X, 250, nz, 7) for nz in (0.1, 0.2, 0.3, 0.4)])
Qh = Q.cpu().pin_memory()

def timeit(label, fn, reps=5):
    fn(); torch.cuda.synchronize()
    t0 = time.perf_counter()
    for _ in range(reps):
        fn()
    torch.cuda.synchronize()
    print(f"{label:40s} {1e3 * (time.perf_counter() - t0) / reps:8.2f} ms", flush=True)

timeit("search_queries(device Q, copy_out=False)", lambda: pl.search_queries(e, Q, 1, target=0.99, copy_out=False))
timeit("search_queries(device Q)", lambda: pl.search_queries(e, Q, 1, target=0.99))
timeit("search_queries(pinned host Q)", lambda: pl.search_queries(e, Qh, 1, target=0.99))
timeit("search_queries(numpy Q)", lambda: pl.search_queries(e, Qh.numpy(), 1, target=0.99))
timeit("pack.predict(device)", lambda: e.pack.predict(Q))
timeit("offset_vector", lambda: e.offset_vector(0.99))
timeit("Qh.to(cuda)", lambda: Qh.to("cuda"))
pred = e.pack.predict(Q); off = e.offset_vector(0.99); lf = e.pack.leaf_filter(t.device())
timeit("search_batch(pred given)", lambda: search_batch(t, Q, 1, predictions=pred, offsets=off, leaf_filter=lf, copy_out=False))
timeit("search_batch exact", lambda: search_batch(t, Q, 1, copy_out=False))
