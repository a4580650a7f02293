"""LEAF-format collections straight into HBM (reference
series.py:190-239 `_save_matrix` / `_load_matrix` / `load_dataset`).

The reference loads a file with `read_bytes` and widens it to fp64, so a 25M x 256
collection needs the 25.6 GB payload plus a 51 GB fp64 copy in host RAM (F7).
Here the payload never sits in host memory as a whole:

* `load_index(path, ...)` reads the file twice through the native streaming
  loader (a few pinned 16 MB buffers, `lf_leaf_paa_file` / `lf_leaf_load`):
  pass 1 computes the segment means on the GPU and the host builds the tree from
  them alone (`lf_tree_build_from_summaries`, bit-identical to tree.build_index);
  pass 2 scatters every row to its leaf-contiguous slot in HBM -- the layout the
  kernels read -- so the collection is resident once, already permuted (a leaf
  shard loads only its own rows).
* `load_dataset_device(path)` is `load_dataset` into an fp32 device tensor.
* Row access on the host (query generation picks source rows) goes through a
  read-only memory map of the payload (`FileRows`), never a full copy.

Errors follow the reference: `FormatError(ValueError)` with the byte offset of
the failure (series.py:25-31), `ValueError` for non-finite values
(series.py:65-66).
"""

from __future__ import annotations

import ctypes as C
import os

import numpy as np

from . import _lib

HEADER_SIZE = 16        # series.py:22


class FormatError(ValueError):
    """Malformed dataset file; carries the byte offset of the failure (series.py:25-31)."""

    def __init__(self, message: str, offset: int):
        super().__init__(message)
        self.offset = offset


def _fspath(path) -> bytes:
    return os.fsencode(os.fspath(path))


def read_header(path) -> tuple:
    """(n, m) of a LEAF file, validated like `_load_matrix` (series.py:198-212)."""
    n, m, off = C.c_int64(), C.c_int32(), C.c_int64(-1)
    L = _lib.lib()
    rc = L.lf_leaf_header(_fspath(path), C.byref(n), C.byref(m), C.byref(off))
    if rc == _lib.LF_EFORMAT:
        raise FormatError(L.lf_last_error().decode(errors="replace"), int(off.value))
    _lib.check(rc)
    return int(n.value), int(m.value)


class FileRows:
    """Host row access to a LEAF payload through a read-only memory map (fp32 rows,
    original series order); the index keeps this instead of a host copy."""

    def __init__(self, path):
        self.path = os.fspath(path)
        n, m = read_header(path)
        self.shape = (n, m)
        self.dtype = np.float32
        self._map = np.memmap(self.path, dtype="<f4", mode="r", offset=HEADER_SIZE, shape=(n, m))

    def __getitem__(self, ids):
        return np.asarray(self._map[ids], dtype=np.float32)

    def __len__(self) -> int:
        return self.shape[0]


def save_dataset(values, path, stream=None) -> None:
    """`_save_matrix` (series.py:190-195) from a device fp32 tensor or host array."""
    torch = _lib.require_cuda()
    from .index import as_f32_rows

    if isinstance(values, torch.Tensor):
        if values.dtype != torch.float32 or values.dim() != 2:
            raise ValueError("save_dataset needs an fp32 [n, m] tensor")
        X = values.contiguous()
        if not X.is_cuda:
            X = X.cuda()
    else:
        X = torch.from_numpy(as_f32_rows(values)).cuda()
    n, m = int(X.shape[0]), int(X.shape[1])
    if n < 1 or m < 2:
        raise ValueError(f"dataset needs n >= 1 and m >= 2, got {(n, m)}")
    _lib.check(_lib.lib().lf_leaf_save(_fspath(path), X.data_ptr(), n, m, _lib.stream_ptr(stream)))


def load_dataset_device(path, device=None, threads: int | None = None):
    """`load_dataset` (series.py:218-219) into an fp32 [n, m] device tensor (original order)."""
    torch = _lib.require_cuda()
    n, m = read_header(path)
    if n < 1 or m < 2:
        raise ValueError(f"dataset needs n >= 1 and m >= 2, got {(n, m)}")
    dev = torch.device(device if device is not None else "cuda")
    with torch.cuda.device(dev):
        X = torch.empty((n, m), dtype=torch.float32, device=dev)
        _lib.check(_lib.lib().lf_leaf_load(_fspath(path), n, m, None, X.data_ptr(),
                                           threads or default_threads(), _lib.stream_ptr()))
    return X


def default_threads() -> int:
    return max(1, min(8, os.cpu_count() or 1))


def load_rows_to(path, pos, out, threads: int | None = None) -> None:
    """Pass 2: row i of the file -> out[pos[i]] (pos[i] < 0: skipped).  `pos` is an
    int64 device tensor [n]; `out` an fp32 device tensor [rows, m]."""
    rows = FileRows(path) if not isinstance(path, FileRows) else path
    n, m = rows.shape
    if pos.shape[0] != n or out.shape[1] != m:
        raise ValueError("load_rows_to: pos / out shape mismatch")
    _lib.check(_lib.lib().lf_leaf_load(_fspath(rows.path), n, m, pos.data_ptr(), out.data_ptr(),
                                       threads or default_threads(), _lib.stream_ptr()))


def load_index(path, max_leaf_size: int = 1000, segments: int = 8, device=None,
               threads: int | None = None):
    """`build_index(load_dataset(path), ...)` without a host copy of the collection:
    segment means streamed on the GPU (pass 1), tree built from them on the host, and
    the rows loaded into the leaf-contiguous layout when the device image is made
    (`TreeIndex.device` / `.shard`, pass 2)."""
    torch = _lib.require_cuda()
    from .index import TreeIndex, _export, segment_layout

    if max_leaf_size < 2:
        raise ValueError(f"max_leaf_size must be >= 2, got {max_leaf_size}")
    rows = FileRows(path)
    n, m = rows.shape
    if n < 1 or m < 2:
        raise ValueError(f"dataset needs n >= 1 and m >= 2, got {(n, m)}")
    starts, widths = segment_layout(m, segments)
    dev = torch.device(device if device is not None else "cuda")
    with torch.cuda.device(dev):
        summ = torch.empty((n, segments), dtype=torch.float64, device=dev)
        _lib.check(_lib.lib().lf_leaf_paa_file(_fspath(path), n, m, segments, summ.data_ptr(),
                                               threads or default_threads(), _lib.stream_ptr()))
        hs = summ.cpu().numpy()
        del summ
    L = _lib.lib()
    h = L.lf_tree_build_from_summaries(_lib.ptr(hs), n, segments, max_leaf_size)
    if not h:
        _lib.check(_lib.LF_EINVAL)
    try:
        arrays = _export(L, h, n, segments)
    finally:
        L.lf_tree_free(h)
    return TreeIndex(rows, starts, widths, int(max_leaf_size), *arrays)
