"""The learned filters of an index as one device pack, and their inference.

Reference: one `MlpModel` per selected leaf (mlp.py:52-102), wired into the
search as a dict of per-leaf callables (enhanced.py:120, tree.py:278-286).
Here all F filters live in stacked HBM tensors (W1 [F, m, m] in the
reference's `x @ W1` layout, b1 [F, m], W2 [F, m], b2 [F], fp32) and one
`lf_filter_predict` launch evaluates every (query, filter) pair.  The kernel
is batch-invariant, so the predictions used to calibrate offsets and the
ones used to search are bit-identical (enhanced.py:283-285).
"""

from __future__ import annotations

import os
import weakref

import numpy as np

from . import _lib


class FilterPack:
    """path: "tc16" (tcgen05 kind::f16 over power-of-two-scaled fp16 operands --
    tf32's mantissa at twice its rate; default for m up to 256 that is a multiple of 64
    or above 64 -- the operands are then zero-padded to the next multiple of 64; the
    in-search inference runs on it), "tc" (tcgen05 tf32; default for m = 32) or
    "simt" (fp32 CUDA-core FFMA).  LF_FILTER_PATH overrides
    the default.  Calibration and search must use the same pack (same path) --
    predictions are then bit-identical (F6)."""

    def __init__(self, leaf_ids, W1, b1, W2, b2, device=None, path: str | None = None):
        torch = _lib.require_cuda()
        dev = torch.device(device if device is not None else "cuda")
        self.leaf_ids = [int(l) for l in leaf_ids]
        if sorted(self.leaf_ids) != self.leaf_ids:
            raise ValueError("filter leaf ids must be ascending")

        def t(a, shape):
            x = torch.as_tensor(np.asarray(a, dtype=np.float32) if not isinstance(a, torch.Tensor) else a,
                                dtype=torch.float32).to(dev).contiguous()
            if tuple(x.shape) != shape:
                raise ValueError(f"filter tensor shape {tuple(x.shape)} != {shape}")
            return x

        F = len(self.leaf_ids)
        m = int(np.shape(W1)[-1]) if F else 0
        self.m = m
        self.W1 = t(W1, (F, m, m))
        self.b1 = t(b1, (F, m))
        self.W2 = t(W2, (F, m))
        self.b2 = t(b2, (F,))
        self.device = dev
        self._slot_maps = weakref.WeakKeyDictionary()   # DeviceIndex -> leaf->filter map
        tc_ok = F > 0 and m % 32 == 0 and 32 <= m <= 256
        # fp16 path: m a multiple of 64, or 64 < m <= 256 with the operands zero-padded to
        # the next multiple of 64 (exact: padded inputs, hidden units and weights are 0)
        tc16_ok = tc_ok and (m % 64 == 0 or m > 64)
        self.path = path or os.environ.get("LF_FILTER_PATH") or ("tc16" if tc16_ok else "tc" if tc_ok else "simt")
        if self.path in ("tc", "tc16"):
            if not tc_ok:
                raise ValueError("tensor-core filter path needs m in {32, 64, ..., 256}")
            if self.path == "tc16" and not tc16_ok:
                raise ValueError("fp16 tensor-core filter path needs m a multiple of 64, or 64 < m <= 256")
            self.W1T = self.W1.transpose(1, 2).contiguous()     # K-major B operand [F][hidden][in]
            if self.path == "tc16":
                mp = (m + 63) // 64 * 64
                pad = mp - m
                W1T = self.W1T if not pad else torch.nn.functional.pad(self.W1T, (0, pad, 0, pad)).contiguous()
                self.mp = mp
                self.h_b1 = self.b1 if not pad else torch.nn.functional.pad(self.b1, (0, pad)).contiguous()
                self.h_W2 = self.W2 if not pad else torch.nn.functional.pad(self.W2, (0, pad)).contiguous()
                self.W1T_h = torch.empty((F, mp, mp), dtype=torch.float16, device=dev)
                self.wexp = torch.empty(F, dtype=torch.int32, device=dev)
                _lib.check(_lib.lib().lf_filter_rows_to_f16(W1T.data_ptr(), F, mp * mp, self.W1T_h.data_ptr(),
                                                           self.wexp.data_ptr(), _lib.stream_ptr()))
        elif self.path != "simt":
            raise ValueError(f"unknown filter path {self.path!r}")
        if self.path != "tc16":
            self.mp, self.h_b1, self.h_W2 = m, self.b1, self.W2

    @property
    def n_filters(self) -> int:
        return len(self.leaf_ids)

    @classmethod
    def from_models(cls, models: dict, device=None, path: str | None = None) -> "FilterPack":
        """From {leaf_id: model} where model has W1, b1, W2, b2 (reference MlpModel)."""
        ids = sorted(int(l) for l in models)
        if not ids:
            return cls([], np.zeros((0, 0, 0)), np.zeros((0, 0)), np.zeros((0, 0)), np.zeros(0), device)
        W1 = np.stack([np.asarray(models[l].W1, dtype=np.float32) for l in ids])
        b1 = np.stack([np.asarray(models[l].b1, dtype=np.float32) for l in ids])
        W2 = np.stack([np.asarray(models[l].W2, dtype=np.float32) for l in ids])
        b2 = np.array([np.float32(models[l].b2) for l in ids], dtype=np.float32)
        return cls(ids, W1, b1, W2, b2, device, path)

    def predict(self, queries, stream=None):
        """fp32 [Q, F] predictions for device (or host) queries."""
        torch = _lib.require_cuda()
        if isinstance(queries, torch.Tensor):
            q = queries.to(device=self.device, dtype=torch.float32).contiguous()
        else:
            q = torch.from_numpy(np.ascontiguousarray(np.atleast_2d(queries), dtype=np.float32)).to(self.device)
        Q = q.shape[0]
        out = torch.empty((Q, self.n_filters), dtype=torch.float32, device=self.device)
        if Q and self.n_filters:
            if q.shape[1] != self.m:
                raise ValueError(f"input shape {tuple(q.shape)} does not match model dim {self.m}")
            if self.path == "tc16":
                qp = self._pad_rows(q)
                _lib.check(_lib.lib().lf_filter_predict_f16(qp.data_ptr(), Q, self.mp, self.W1T_h.data_ptr(),
                                                            self.wexp.data_ptr(), self.h_b1.data_ptr(),
                                                            self.h_W2.data_ptr(), self.b2.data_ptr(), self.n_filters,
                                                            out.data_ptr(), _lib.stream_ptr(stream)))
                return out
            fn = _lib.lib().lf_filter_predict_tc if self.path == "tc" else _lib.lib().lf_filter_predict
            w = self.W1T if self.path == "tc" else self.W1
            _lib.check(fn(q.data_ptr(), Q, self.m, w.data_ptr(), self.b1.data_ptr(), self.W2.data_ptr(),
                          self.b2.data_ptr(), self.n_filters, out.data_ptr(), _lib.stream_ptr(stream)))
        return out

    def predict_pairs(self, queries, pair_q, pair_f, stream=None):
        """fp64 [P] predictions of filter pair_f[i] for query pair_q[i] (tensor-core
        paths; bit-identical to the same entries of predict())."""
        torch = _lib.require_cuda()
        if self.path not in ("tc", "tc16"):
            raise ValueError("pair predictions need a tensor-core filter path")
        q = queries.to(device=self.device, dtype=torch.float32).contiguous() if isinstance(queries, torch.Tensor) \
            else torch.from_numpy(np.ascontiguousarray(np.atleast_2d(queries), dtype=np.float32)).to(self.device)
        pq = torch.as_tensor(pair_q, dtype=torch.int32).to(self.device).contiguous()
        pf = torch.as_tensor(pair_f, dtype=torch.int32).to(self.device).contiguous()
        out = torch.empty(pq.shape[0], dtype=torch.float64, device=self.device)
        if self.path == "tc16":
            qp = self._pad_rows(q)
            _lib.check(_lib.lib().lf_filter_predict_pairs_f16(
                qp.data_ptr(), q.shape[0], self.mp, self.W1T_h.data_ptr(), self.wexp.data_ptr(), self.h_b1.data_ptr(),
                self.h_W2.data_ptr(), self.b2.data_ptr(), self.n_filters, pq.data_ptr(), pf.data_ptr(), pq.shape[0],
                out.data_ptr(), _lib.stream_ptr(stream)))
            return out
        _lib.check(_lib.lib().lf_filter_predict_pairs_tc(q.data_ptr(), self.m, self.W1T.data_ptr(), self.b1.data_ptr(),
                                                         self.W2.data_ptr(), self.b2.data_ptr(), self.n_filters,
                                                         pq.data_ptr(), pf.data_ptr(), pq.shape[0], out.data_ptr(),
                                                         _lib.stream_ptr(stream)))
        return out

    def _pad_rows(self, q):
        """[Q, m] fp32 -> [Q, mp] with zero columns (the fp16 pack's padded width)."""
        torch = _lib.require_cuda()
        return q if self.mp == self.m else torch.nn.functional.pad(q, (0, self.mp - self.m)).contiguous()

    def leaf_filter(self, dindex):
        """int32 [n_leaves]: filter slot of each leaf slot of a DeviceIndex, -1 if none."""
        torch = _lib.require_cuda()
        key = dindex
        if key not in self._slot_maps:
            m = np.full(dindex.n_leaves, -1, dtype=np.int32)
            for s, lid in enumerate(self.leaf_ids):
                j = dindex.slot_of_leaf.get(lid)
                if j is None:
                    raise ValueError(f"filter leaf {lid} does not exist in the index")
                m[j] = s
            self._slot_maps[key] = torch.from_numpy(m).to(self.device)
        return self._slot_maps[key]
