"""Time (and optionally ncu-profile) the training-data-generation kernels alone."""
import sys, time
from pathlib import Path
sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
import torch
from paper_2502_01836_b200 import build_index_device
from paper_2502_01836_b200.synth import randwalk_device, queries_device
from paper_2502_01836_b200.targets import leaf_min_distances

n = int(sys.argv[1]) if len(sys.argv) > 1 else 2_000_000
nq = int(sys.argv[2]) if len(sys.argv) > 2 else 512
X = randwalk_device(n, 256, 3)
t = build_index_device(X, 10000)
t.device()
Q = queries_device(X, nq, 0.25, 4)
slots = list(range(t.n_leaves))
for path in ("tc", "simt"):
    leaf_min_distances(t, Q[:128], slots, path=path)
    torch.cuda.synchronize()
    if path == "tc":
        torch.cuda.cudart().cudaProfilerStart()
    t0 = time.perf_counter()
    out = leaf_min_distances(t, Q, slots, path=path)
    torch.cuda.synchronize()
    dt = time.perf_counter() - t0
    if path == "tc":
        torch.cuda.cudart().cudaProfilerStop()
        ref = out.clone()
    else:
        print("max rel diff tc vs simt:", float(((ref - out).abs() / out.clamp_min(1e-300)).max()))
    print(f"{path}: {dt*1e3:.1f} ms, {nq * n / dt:.3e} pairs/s, {2 * nq * n * 256 / dt / 1e12:.1f} TFLOP/s", flush=True)
