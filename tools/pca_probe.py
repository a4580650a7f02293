"""Feasibility probe: how many rows would a projected (PCA, k dims, int8) + residual-norm
lower bound leave for exact re-reads, vs the full-length int8 bound (the q8 scan)?
Random-walk collection on the GPU, rows of each query's lowest-bound leaves, threshold
= the query's exact NN distance (the late-round best-so-far)."""
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
import torch

from paper_2502_01836_b200 import build_index_device
from paper_2502_01836_b200.synth import queries_device, randwalk_device

n, m = 2_000_000, 256
X = randwalk_device(n, m, 7)
Q = torch.cat([queries_device(X, 250, nz, 3 + i) for i, nz in enumerate((0.1, 0.2, 0.3, 0.4))])
# exact NN distance by brute force
best = torch.full((Q.shape[0],), float("inf"), device="cuda", dtype=torch.float64)
for r0 in range(0, n, 200_000):
    d = torch.cdist(Q.double(), X[r0:r0 + 200_000].double())
    best = torch.minimum(best, d.min(dim=1).values)
# PCA basis from a sample
S = X[torch.randint(0, n, (100_000,), device="cuda")].double()
mu = S.mean(0)
_, _, V = torch.linalg.svd(S - mu, full_matrices=False)
for k in (16, 32, 48, 64):
    P = V[:k]                                             # k x m, orthonormal rows (fp64)
    def split(A):
        y = (A.double() - mu) @ P.T
        r = (A.double() - mu) - y @ P
        return y, r.norm(dim=1)
    # sample rows near each query: 4096 random rows + its true NN band (use all rows of a random 50K slab)
    Y, R = split(X[:400_000])
    yq, rq = split(Q)
    # int8 quantisation of y (per row scale) and its error
    def q8(y):
        s = y.abs().amax(1, keepdim=True) / 127
        c = torch.round(y / s).clamp(-127, 127)
        return c * s, (c * s - y).norm(dim=1)
    Yh, ey = q8(Y)
    yqh, eyq = q8(yq)
    surv = 0
    tot = 0
    for i in range(0, Q.shape[0], 50):
        a = torch.cdist(yqh[i:i + 50], Yh)                # projected distance of the codes
        lo_a = (a - ey[None, :] - eyq[i:i + 50, None]).clamp_min(0)
        lo_r = (R[None, :] - rq[i:i + 50, None]).abs()
        lo = (lo_a ** 2 + lo_r ** 2).sqrt()
        surv += (lo <= best[i:i + 50, None]).sum().item()
        tot += lo.numel()
    print(f"k={k:3d}: residual norm mean {R.mean():.3f} (row norm ~{X[:1000].norm(dim=1).mean():.1f}); "
          f"rows surviving the projected bound at the NN distance: {surv / tot:.5f}", flush=True)
# the full-length int8 bound for comparison
def q8full(A):
    s = A.abs().amax(1, keepdim=True) / 127
    c = torch.round(A / s).clamp(-127, 127)
    return c * s, (c * s - A.double()).norm(dim=1)
Xh, ex = q8full(X[:400_000].double())
Qh, eq = q8full(Q.double())
surv = 0; tot = 0
for i in range(0, Q.shape[0], 50):
    a = torch.cdist(Qh[i:i + 50], Xh)
    lo = (a - ex[None, :] - eq[i:i + 50, None]).clamp_min(0)
    surv += (lo <= best[i:i + 50, None]).sum().item(); tot += lo.numel()
print(f"full int8 bound: {surv / tot:.6f}")
