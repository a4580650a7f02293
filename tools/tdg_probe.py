"""Training-data-generation kernel probe: exact query x leaf minimum distances
(targets.leaf_min_distances, lf_leaf_min_dist_q8) on an n x 256 random walk with
leaf cap 10K; CUDA-event time per call and the algorithmic int8 TOPS.
    python tools/tdg_probe.py [n] [queries] [path]"""
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
import torch

from paper_2502_01836_b200 import build_index_device
from paper_2502_01836_b200.synth import queries_device, randwalk_device
from paper_2502_01836_b200.targets import leaf_min_distances

n = int(sys.argv[1]) if len(sys.argv) > 1 else 2_000_000
nq = int(sys.argv[2]) if len(sys.argv) > 2 else 1024
path = sys.argv[3] if len(sys.argv) > 3 else None
X = randwalk_device(n, 256, 1234)
t = build_index_device(X, max_leaf_size=10_000)
di = t.device()
Q = torch.cat([queries_device(X, nq // 4, nz, 7 + i) for i, nz in enumerate((0.1, 0.2, 0.3, 0.4))]).contiguous()
slots = list(range(di.n_leaves))
out = leaf_min_distances(t, Q, slots, path=path)
torch.cuda.synchronize()
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
e0.record()
for _ in range(3):
    leaf_min_distances(t, Q, slots, path=path)
e1.record()
torch.cuda.synchronize()
ms = e0.elapsed_time(e1) / 3
print(f"n={n} queries={Q.shape[0]} leaves={di.n_leaves} path={path or 'default'}: {ms:.2f} ms, "
      f"{2.0 * Q.shape[0] * n * 256 / (ms / 1e3) / 1e12:.1f} algorithmic TOPS")
