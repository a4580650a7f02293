"""Filter training: every selected leaf's MLP trained at once on the GPU.

The reference trains one `MlpModel` per leaf in a process pool
(enhanced.py:147-186 -> mlp.train, mlp.py:145-221).  Here the F filters are
one batched model (W1 [F, m, m], ...) stepped together with torch.bmm, with
the reference's schedule applied per filter:

* SGD, batch 32, MSE on raw distances (mlp.py:116-137, 185-194);
* the learning rate divides by `lr_decay_factor` after `plateau_patience`
  epochs without a `plateau_min_delta` relative improvement of the validation
  loss, and a filter stops once its next rate would fall below `min_lr` or at
  `max_epochs` (mlp.py:196-212);
* the returned parameters are each filter's best-validation epoch
  (mlp.py:200-202);
* a non-finite loss raises TrainingDivergedError (mlp.py:188-189), which the
  pipeline reports as the failing stage.

Initial weights and the 4:1 train/validation split use the reference's numpy
seeds (init_model, mlp.py:105-113; assemble_filter_training,
traingen.py:234-266).  Minibatch shuffles come from torch's generator and
arithmetic is fp32 (the reference accumulates gradients in fp64), so trained
weights are statistically -- not bitwise -- equivalent.
"""

from __future__ import annotations

import math
from dataclasses import dataclass, field

import numpy as np


class TrainingDivergedError(RuntimeError):
    pass


@dataclass
class TrainConfig:
    """mlp.py:25-40."""

    initial_lr: float = 0.01
    lr_decay_factor: float = 10.0
    min_lr: float = 1e-5
    max_epochs: int = 1000
    batch_size: int = 32
    plateau_patience: int = 20
    plateau_min_delta: float = 1e-3
    seed: int = 0

    def __post_init__(self):
        if not self.initial_lr > self.min_lr > 0:
            raise ValueError("require initial_lr > min_lr > 0")
        if self.max_epochs < 1:
            raise ValueError("max_epochs must be >= 1")


@dataclass
class TrainReport:
    epochs_run: int
    final_train_loss: float
    final_val_loss: float
    lr_trajectory: list = field(default_factory=list)
    val_trajectory: list = field(default_factory=list)


def init_weights(m: int, seed: int) -> tuple:
    """init_model (mlp.py:105-113): U(-1/sqrt(m), 1/sqrt(m)) weights, zero biases, fp32."""
    rng = np.random.default_rng(seed)
    bound = 1.0 / math.sqrt(m)
    W1 = rng.uniform(-bound, bound, size=(m, m)).astype(np.float32)
    W2 = rng.uniform(-bound, bound, size=m).astype(np.float32)
    return W1, np.zeros(m, np.float32), W2, np.float32(0.0)


def train_filters(bank, train_idx, train_y, val_idx, val_y, init, cfg: TrainConfig, seed: int = 0,
                  device="cuda", record_trajectories: bool = False, tf32: bool = True) -> tuple:
    """Train F filters together.

    bank:      fp32 [n_rows, m] (device) -- every training/validation input row
    train_idx: int64 [F, n_tr] rows of `bank` per filter; train_y fp64 [F, n_tr]
    val_idx:   int64 [F, n_va];                            val_y   fp64 [F, n_va]
    init:      (W1 [F,m,m], b1 [F,m], W2 [F,m], b2 [F]) fp32 numpy
    Returns ((W1, b1, W2, b2) best-validation parameters as fp32 numpy, [TrainReport]).
    """
    import torch

    dev = torch.device(device)
    bank = bank.to(dev)
    tidx = torch.as_tensor(train_idx, dtype=torch.int64, device=dev)
    vidx = torch.as_tensor(val_idx, dtype=torch.int64, device=dev)
    ty = torch.as_tensor(train_y, dtype=torch.float32, device=dev)
    vy = torch.as_tensor(val_y, dtype=torch.float32, device=dev)
    F, n_tr = tidx.shape
    if F == 0:
        return tuple(np.asarray(a) for a in init), []
    if not (torch.isfinite(ty).all() and (ty >= 0).all()):
        raise ValueError("targets must be finite and non-negative")
    W1 = torch.as_tensor(init[0], dtype=torch.float32, device=dev).clone()
    b1 = torch.as_tensor(init[1], dtype=torch.float32, device=dev).clone()
    W2 = torch.as_tensor(init[2], dtype=torch.float32, device=dev).clone()
    b2 = torch.as_tensor(init[3], dtype=torch.float32, device=dev).clone()
    best = [W1.clone(), b1.clone(), W2.clone(), b2.clone()]
    best_val = torch.full((F,), math.inf, dtype=torch.float64, device=dev)
    plateau_best = torch.full((F,), math.inf, dtype=torch.float64, device=dev)
    wait = torch.zeros(F, dtype=torch.int64, device=dev)
    lr = torch.full((F,), cfg.initial_lr, dtype=torch.float64, device=dev)
    active = torch.ones(F, dtype=torch.bool, device=dev)
    epochs = torch.zeros(F, dtype=torch.int64, device=dev)
    lr_hist, val_hist = [], []
    g = torch.Generator(device=dev)
    g.manual_seed(int(seed) & 0x7FFFFFFF)
    Xv = bank[vidx]                                                    # [F, n_va, m]
    bs = cfg.batch_size
    prev_tf32 = torch.backends.cuda.matmul.allow_tf32
    torch.backends.cuda.matmul.allow_tf32 = tf32        # batched GEMMs on the tensor cores
    try:
        return _train_loop(torch, dev, bank, tidx, vidx, ty, vy, F, n_tr, W1, b1, W2, b2, best, best_val,
                           plateau_best, wait, lr, active, epochs, lr_hist, val_hist, g, Xv, bs, cfg,
                           record_trajectories)
    finally:
        torch.backends.cuda.matmul.allow_tf32 = prev_tf32


def _train_loop(torch, dev, bank, tidx, vidx, ty, vy, F, n_tr, W1, b1, W2, b2, best, best_val, plateau_best,
                wait, lr, active, epochs, lr_hist, val_hist, g, Xv, bs, cfg, record_trajectories):
    with torch.no_grad():
        for epoch in range(cfg.max_epochs):
            if not bool(active.any()):
                break
            if record_trajectories:
                lr_hist.append(lr.cpu().numpy().copy())
            epochs += active.to(torch.int64)
            step_lr = torch.where(active, lr, torch.zeros_like(lr)).to(torch.float32)
            perm = torch.argsort(torch.rand((F, n_tr), generator=g, device=dev), dim=1)
            bad_epoch = torch.zeros(F, dtype=torch.bool, device=dev)
            for s in range(0, n_tr, bs):
                sel = perm[:, s:s + bs]                                # [F, b]
                b = sel.shape[1]
                X = bank[torch.gather(tidx, 1, sel)]                   # [F, b, m]
                y = torch.gather(ty, 1, sel)                           # [F, b]
                Z = torch.baddbmm(b1[:, None, :], X, W1)               # [F, b, m]
                H = torch.relu(Z)
                pred = torch.bmm(H, W2[:, :, None])[:, :, 0] + b2[:, None]
                err = pred - y
                loss = (err * err).mean(dim=1)
                bad_epoch |= ~torch.isfinite(loss) & active   # checked once per epoch (no per-step sync)
                gr = err * (2.0 / b)                                   # [F, b]
                gW2 = torch.bmm(H.transpose(1, 2), gr[:, :, None])[:, :, 0]
                gb2 = gr.sum(dim=1)
                dZ = (gr[:, :, None] * W2[:, None, :]) * (Z > 0)
                gW1 = torch.bmm(X.transpose(1, 2), dZ)
                gb1 = dZ.sum(dim=1)
                W1.sub_(step_lr[:, None, None] * gW1)
                b1.sub_(step_lr[:, None] * gb1)
                W2.sub_(step_lr[:, None] * gW2)
                b2.sub_(step_lr * gb2)
            if bool(bad_epoch.any()):
                f = int(torch.nonzero(bad_epoch)[0, 0])
                raise TrainingDivergedError(
                    f"non-finite loss at epoch {epoch} (lr={float(lr[f]):g}) for filter slot {f}")
            Hv = torch.relu(torch.baddbmm(b1[:, None, :], Xv, W1))
            pv = torch.bmm(Hv, W2[:, :, None])[:, :, 0] + b2[:, None]
            ev = (pv.double() - vy.double())
            val = (ev * ev).mean(dim=1)
            if bool((~torch.isfinite(val) & active).any()):
                raise TrainingDivergedError(f"non-finite validation loss at epoch {epoch}")
            if record_trajectories:
                val_hist.append(val.cpu().numpy().copy())
            improved = active & (val < best_val)
            best_val = torch.where(improved, val, best_val)
            for dst, src in zip(best, (W1, b1, W2, b2)):
                mask = improved.view(-1, *([1] * (src.dim() - 1)))
                dst.copy_(torch.where(mask, src, dst))
            plat = active & (val < plateau_best * (1.0 - cfg.plateau_min_delta))
            plateau_best = torch.where(plat, val, plateau_best)
            wait = torch.where(plat, torch.zeros_like(wait), wait + active.to(torch.int64))
            decay = active & (wait >= cfg.plateau_patience)
            wait = torch.where(decay, torch.zeros_like(wait), wait)
            lr = torch.where(decay, lr / cfg.lr_decay_factor, lr)
            active = active & ~(decay & (lr < cfg.min_lr))
        # final train loss of the best parameters (mlp.py:216)
        tr_loss = torch.empty(F, dtype=torch.float64, device=dev)
        for f0 in range(0, F, 256):
            f1 = min(F, f0 + 256)
            Xt = bank[tidx[f0:f1]]
            Ht = torch.relu(torch.baddbmm(best[1][f0:f1, None, :], Xt, best[0][f0:f1]))
            pt = torch.bmm(Ht, best[2][f0:f1, :, None])[:, :, 0] + best[3][f0:f1, None]
            et = pt.double() - ty[f0:f1].double()
            tr_loss[f0:f1] = (et * et).mean(dim=1)
    ep = epochs.cpu().numpy()
    bv = best_val.cpu().numpy()
    tl = tr_loss.cpu().numpy()
    reports = []
    for f in range(F):
        lrs = [float(h[f]) for h in lr_hist[: int(ep[f])]] if record_trajectories else []
        vals = [float(h[f]) for h in val_hist[: int(ep[f])]] if record_trajectories else []
        reports.append(TrainReport(int(ep[f]), float(tl[f]), float(bv[f]), lrs, vals))
    params = tuple(p.cpu().numpy() for p in best)
    return params, reports
