"""Synthetic collections and training queries.

The host generators consume numpy `default_rng` streams in exactly the order
the reference does, so every array is bit-identical to the reference's:

* random walks: series.py:161-171 (generated in row chunks -- the stream is
  consumed row-major, so chunking is bit-exact and keeps fp64 temporaries
  small at 25M rows);
* noisy queries: series.py:174-187;
* global / local training queries: traingen.py:100-132.

`randwalk_device` is the fast GPU generator used for 25M-row benchmark
collections: the same distribution (cumulative N(0,1) steps, z-normalised with
ddof=1, rounded to fp32) from torch's Philox stream -- not bit-identical to
numpy, and said so wherever it is used.
"""

from __future__ import annotations

import numpy as np


def _f32_exact(a) -> np.ndarray:
    return np.asarray(a, dtype=np.float64).astype(np.float32).astype(np.float64)


def generate_randwalk(n: int, m: int, seed: int, chunk_rows: int = 1 << 16,
                      dtype=np.float64) -> np.ndarray:
    """Bit-identical to series.generate_randwalk(n, m, seed).values (fp32 storage if dtype=float32)."""
    if n < 1 or m < 2:
        raise ValueError(f"need n >= 1 and m >= 2, got n={n} m={m}")
    rng = np.random.default_rng(seed)
    out = np.empty((n, m), dtype=dtype)
    for r0 in range(0, n, chunk_rows):
        r1 = min(n, r0 + chunk_rows)
        w = np.cumsum(rng.standard_normal((r1 - r0, m)), axis=1)
        mu = w.mean(axis=1, keepdims=True)
        sd = w.std(axis=1, ddof=1, keepdims=True)
        if not (sd > 0).all():
            raise ValueError("degenerate random walk (zero variance)")
        out[r0:r1] = ((w - mu) / sd).astype(np.float32)
    return out


def make_queries(values: np.ndarray, count: int, noise_level: float, seed: int) -> np.ndarray:
    """Bit-identical to series.make_queries(...).values."""
    if count < 1:
        raise ValueError(f"count must be >= 1, got {count}")
    if not 0.0 <= noise_level <= 1.0:
        raise ValueError(f"noise_level must be in [0, 1], got {noise_level}")
    rng = np.random.default_rng(seed)
    src = rng.integers(0, values.shape[0], size=count)
    noise = rng.standard_normal((count, values.shape[1])) * noise_level
    return _f32_exact(np.asarray(values[src], dtype=np.float64) + noise)


def _noisy(rows: np.ndarray, noise_range, rng) -> tuple:
    lo, hi = float(noise_range[0]), float(noise_range[1])
    if not 0.0 <= lo <= hi <= 1.0:
        raise ValueError(f"noise range must satisfy 0 <= lo <= hi <= 1, got {noise_range}")
    levels = rng.uniform(lo, hi, size=rows.shape[0])
    noise = rng.standard_normal(rows.shape) * levels[:, None]
    return _f32_exact(np.asarray(rows, dtype=np.float64) + noise), levels


def generate_global_queries(values: np.ndarray, n: int, noise_range=(0.1, 0.4), seed: int = 0):
    """Bit-identical to traingen.generate_global_queries."""
    if n < 1:
        raise ValueError("n must be >= 1")
    rng = np.random.default_rng(seed)
    src = rng.integers(0, values.shape[0], size=n)
    return _noisy(values[src], noise_range, rng)


def generate_local_queries(tree, leaf_id: int, n: int, noise_range=(0.1, 0.4), seed: int = 0):
    """Bit-identical to traingen.generate_local_queries: (queries, levels, source_ids)."""
    if n < 1:
        raise ValueError("n must be >= 1")
    if not (0 <= leaf_id < tree.n_nodes) or tree.left[leaf_id] >= 0:
        raise ValueError(f"unknown leaf id {leaf_id}")
    ids = tree.leaf_members(leaf_id)
    rng = np.random.default_rng(seed)
    pick = rng.integers(0, ids.shape[0], size=n)
    q, lv = _noisy(tree.values[ids[pick]], noise_range, rng)
    return q, lv, ids[pick]


def randwalk_device(n: int, m: int, seed: int, device="cuda", chunk_rows: int = 1 << 20):
    """GPU random-walk collection (same law as series.py:161-171, torch Philox stream)."""
    import torch

    g = torch.Generator(device=device)
    g.manual_seed(seed)
    out = torch.empty((n, m), dtype=torch.float32, device=device)
    for r0 in range(0, n, chunk_rows):
        r1 = min(n, r0 + chunk_rows)
        w = torch.randn((r1 - r0, m), generator=g, device=device, dtype=torch.float64).cumsum_(1)
        mu = w.mean(dim=1, keepdim=True)
        sd = w.std(dim=1, keepdim=True, unbiased=True)
        out[r0:r1] = ((w - mu) / sd).to(torch.float32)
    return out


def queries_device(values, count: int, noise_level: float, seed: int):
    """GPU noisy queries (series.py:174-187 law) over a device collection; fp32-exact."""
    import torch

    g = torch.Generator(device=values.device)
    g.manual_seed(seed)
    src = torch.randint(0, values.shape[0], (count,), generator=g, device=values.device)
    noise = torch.randn((count, values.shape[1]), generator=g, device=values.device, dtype=torch.float64)
    return (values[src].to(torch.float64) + noise * noise_level).to(torch.float32)


# --------------------------------------------------------------------------
# BASELINE config 5 (Deep1B-shaped): Gaussian-mixture vectors.  No reference
# generator exists (parity unpinned): K centers ~ N(0, 1)^m,
# points = center + N(0, sigma^2)^m, rounded to fp32.  Fixed seed.
# --------------------------------------------------------------------------
def gaussian_mixture(n: int, m: int, seed: int, n_centers: int = 1000, sigma: float = 0.25,
                     chunk_rows: int = 1 << 16) -> np.ndarray:
    """Host fp64 (fp32-exact) [n, m] Gaussian mixture."""
    if n < 1 or m < 2 or n_centers < 1:
        raise ValueError(f"need n >= 1, m >= 2, n_centers >= 1, got {n}, {m}, {n_centers}")
    rng = np.random.default_rng(seed)
    centers = rng.standard_normal((n_centers, m))
    out = np.empty((n, m), dtype=np.float64)
    for r0 in range(0, n, chunk_rows):
        r1 = min(n, r0 + chunk_rows)
        c = rng.integers(0, n_centers, size=r1 - r0)
        out[r0:r1] = _f32_exact(centers[c] + sigma * rng.standard_normal((r1 - r0, m)))
    return out


def gaussian_mixture_device(n: int, m: int, seed: int, n_centers: int = 1000, sigma: float = 0.25,
                            device="cuda", chunk_rows: int = 1 << 22):
    """GPU Gaussian mixture (same law as gaussian_mixture, torch Philox stream)."""
    import torch

    g = torch.Generator(device=device)
    g.manual_seed(seed)
    centers = torch.randn((n_centers, m), generator=g, device=device, dtype=torch.float32)
    out = torch.empty((n, m), dtype=torch.float32, device=device)
    for r0 in range(0, n, chunk_rows):
        r1 = min(n, r0 + chunk_rows)
        c = torch.randint(0, n_centers, (r1 - r0,), generator=g, device=device)
        out[r0:r1] = centers[c] + sigma * torch.randn((r1 - r0, m), generator=g, device=device)
    return out


def recall_at_k(ids: np.ndarray, exact_ids: np.ndarray) -> np.ndarray:
    """Per-query recall@k = |returned ids ∩ exact top-k ids| / k (the reference defines
    recall@1 only, cli.py:83-88; this is its k-NN generalisation for config 5)."""
    ids = np.atleast_2d(ids)
    exact_ids = np.atleast_2d(exact_ids)
    k = exact_ids.shape[1]
    return np.array([len(set(a.tolist()) & set(b.tolist())) / k for a, b in zip(ids, exact_ids)])
