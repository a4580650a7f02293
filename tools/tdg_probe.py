"""Time (and optionally ncu-profile: the q8 call is bracketed by cudaProfilerStart/Stop)
the training-data-generation kernels alone, and check the paths agree."""
import sys
import time
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
import torch

from paper_2502_01836_b200 import build_index_device
from paper_2502_01836_b200.synth import queries_device, randwalk_device
from paper_2502_01836_b200.targets import leaf_min_distances

n = int(sys.argv[1]) if len(sys.argv) > 1 else 2_000_000
nq = int(sys.argv[2]) if len(sys.argv) > 2 else 1024
paths = sys.argv[3].split(",") if len(sys.argv) > 3 else ["q8", "q82", "tc", "simt"]
X = randwalk_device(n, 256, 3)
t = build_index_device(X, 10000)
t.device()
Q = torch.cat([queries_device(X, nq // 4, nz, 4 + i) for i, nz in enumerate((0.1, 0.2, 0.3, 0.4))]).contiguous()
slots = list(range(t.n_leaves))
ref = None
for path in paths:
    leaf_min_distances(t, Q[:128], slots, path=path)
    torch.cuda.synchronize()
    if path.startswith("q8"):
        torch.cuda.cudart().cudaProfilerStart()
    t0 = time.perf_counter()
    out = leaf_min_distances(t, Q, slots, path=path)
    torch.cuda.synchronize()
    dt = time.perf_counter() - t0
    if path.startswith("q8"):
        torch.cuda.cudart().cudaProfilerStop()
    if ref is None:
        ref = out.clone()
    else:
        print("max rel diff vs", paths[0], float(((ref - out).abs() / out.clamp_min(1e-300)).max()))
    print(f"{path}: {dt*1e3:.1f} ms, {Q.shape[0] * n / dt:.3e} pairs/s, "
          f"{2 * Q.shape[0] * n * 256 / dt / 1e12:.1f} TFLOP/s (algorithmic)", flush=True)
