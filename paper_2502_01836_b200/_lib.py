"""ctypes binding of the C-ABI in include/leafi_b200.h.

The product path has NO CPU fallback: if the shared library is missing or no
CUDA device is present, every compute entry point raises.  Host-only entry
points (the native tree builder, segment means) work without a GPU.
"""

from __future__ import annotations

import ctypes as C
import os
from pathlib import Path

LIB_PATH = Path(__file__).resolve().parent / "_lib" / "libleafi_b200.so"
MAX_SEG = 64
N_STATS = 6

LF_OK, LF_EINVAL, LF_ECUDA, LF_ENOMEM, LF_EFORMAT = 0, 1, 2, 3, 4


class LfIndex(C.Structure):
    _fields_ = [
        ("n_series", C.c_int64),
        ("m", C.c_int32),
        ("n_seg", C.c_int32),
        ("n_nodes", C.c_int32),
        ("n_leaves", C.c_int32),
        ("max_leaf_rows", C.c_int64),
        ("seg_start", C.c_int32 * MAX_SEG),
        ("seg_width", C.c_int32 * MAX_SEG),
        ("d_X", C.c_void_p),
        ("d_row_id", C.c_void_p),
        ("d_leaf_ptr", C.c_void_p),
        ("d_node_leaf", C.c_void_p),
        ("d_env_min", C.c_void_p),
        ("d_env_max", C.c_void_p),
        ("d_leaf_filter", C.c_void_p),
        ("d_X8", C.c_void_p),
        ("d_qmeta", C.c_void_p),
        ("pca_k", C.c_int32),
        ("d_P", C.c_void_p),
        ("d_mu", C.c_void_p),
        ("d_Xp", C.c_void_p),
        ("d_pmeta", C.c_void_p),
        ("d_sd_min", C.c_void_p),
        ("d_sd_max", C.c_void_p),
    ]


class LfSearchOpts(C.Structure):
    _fields_ = [
        ("k", C.c_int32),
        ("bsf_factor", C.c_double),
        ("d_pred", C.c_void_p),
        ("d_pred_f64", C.c_void_p),
        ("d_offset", C.c_void_p),
        ("n_filters", C.c_int32),
        ("sequential", C.c_int32),
        ("max_round_leaves", C.c_int32),
        ("want_trace", C.c_int32),
        ("early_abandon", C.c_int32),
        ("h_profile", C.c_void_p),
        ("d_W1T_h", C.c_void_p),
        ("d_wexp", C.c_void_p),
        ("d_b1", C.c_void_p),
        ("d_W2", C.c_void_p),
        ("d_b2", C.c_void_p),
        ("filter_m", C.c_int32),
    ]


N_PROF = 15
PROF_NAMES = ("bounds_ms", "plan_ms", "scan_ms", "merge_ms", "rounds", "kernels", "total_ms", "refills",
              "ea_rows", "ea_survivors", "predict_ms", "pairs", "predict_steps", "scan_stream_bytes",
              "scan_exact_bytes")


class LfTrace(C.Structure):
    _fields_ = [
        ("d_len", C.c_void_p),
        ("d_leaf", C.c_void_p),
        ("d_lb", C.c_void_p),
        ("d_searched", C.c_void_p),
        ("d_leaf_nn", C.c_void_p),
        ("d_bsf_before", C.c_void_p),
    ]


_P = C.c_void_p
_I64 = C.c_int64
_I32 = C.c_int32

# symbol -> (restype, argtypes); mirrors include/leafi_b200.h one to one
SIGNATURES = {
    "lf_last_error": (C.c_char_p, []),
    "lf_version": (C.c_int, []),
    "lf_device_sm_count": (C.c_int, [C.c_int]),
    "lf_abi_sizeof": (C.c_int64, [C.c_char_p]),
    "lf_abi_offsetof": (C.c_int64, [C.c_char_p, C.c_char_p]),
    "lf_bounds": (C.c_int, [_P, _I64, C.POINTER(LfIndex), _P, _P, _I32, _I32, _P, _P, _P]),
    "lf_search": (C.c_int, [C.POINTER(LfIndex), _P, _I64, C.POINTER(LfSearchOpts), _P, _P, _P,
                            C.POINTER(LfTrace), _P]),
    "lf_search_plan_create": (_P, [C.POINTER(LfIndex), _I64, C.POINTER(LfSearchOpts), _P]),
    "lf_search_plan_run": (C.c_int, [_P, _P, _P, _P, _P, _P]),
    "lf_search_plan_free": (None, [_P]),
    "lf_search_begin": (_P, [C.POINTER(LfIndex), _P, _I64, C.POINTER(LfSearchOpts), C.POINTER(LfTrace), _P, _P]),
    "lf_search_round": (C.c_int, [_P, _P, _P, C.POINTER(_I32)]),
    "lf_search_round_async": (C.c_int, [_P, _P, _P, _P]),
    "lf_search_round_wait": (C.c_int, [_P, C.POINTER(_I32)]),
    "lf_search_end": (C.c_int, [_P, _P, _P]),
    "lf_search_free": (None, [_P]),
    "lf_filter_predict": (C.c_int, [_P, _I64, _I32, _P, _P, _P, _P, _I32, _P, _P]),
    "lf_filter_predict_tc": (C.c_int, [_P, _I64, _I32, _P, _P, _P, _P, _I32, _P, _P]),
    "lf_filter_predict_f16": (C.c_int, [_P, _I64, _I32, _P, _P, _P, _P, _P, _I32, _P, _P]),
    "lf_filter_rows_to_f16": (C.c_int, [_P, _I64, _I32, _P, _P, _P]),
    "lf_filter_predict_pairs_tc": (C.c_int, [_P, _I32, _P, _P, _P, _P, _I32, _P, _P, _I64, _P, _P]),
    "lf_filter_predict_pairs_f16": (C.c_int, [_P, _I64, _I32, _P, _P, _P, _P, _P, _I32, _P, _P, _I64, _P, _P]),
    "lf_leaf_min_dist": (C.c_int, [_P, _I64, C.POINTER(LfIndex), _P, _I32, _P, _I64, _P]),
    "lf_local_min_dist": (C.c_int, [_P, C.POINTER(LfIndex), _P, _P, _I32, _P, _P]),
    "lf_batch_distances": (C.c_int, [_P, _I64, _P, _I64, _I32, _P, _P]),
    "lf_leaf_min_dist_tc": (C.c_int, [_P, _I64, C.POINTER(LfIndex), _P, _I32, _P, _I64, _P]),
    "lf_local_min_dist_tc": (C.c_int, [_P, C.POINTER(LfIndex), _P, _P, _I32, _P, _P]),
    "lf_leaf_min_dist_q8": (C.c_int, [_P, _I64, C.POINTER(LfIndex), _P, _I32, _P, _I64, _P]),
    "lf_local_min_dist_q8": (C.c_int, [_P, C.POINTER(LfIndex), _P, _P, _I32, _P, _P]),
    "lf_tree_build": (_P, [_P, _I64, _I32, _I32, _I64, _I32]),
    "lf_tree_info": (C.c_int, [_P, C.POINTER(_I32), C.POINTER(_I32)]),
    "lf_tree_export": (C.c_int, [_P, _P, _P, _P, _P, _P, _P, _P, _P, _P, _P]),
    "lf_tree_free": (None, [_P]),
    "lf_paa_host": (C.c_int, [_P, _I64, _I32, _I32, _P, _I32]),
    "lf_tree_build_from_summaries": (_P, [_P, _I64, _I32, _I64]),
    "lf_paa_device": (C.c_int, [_P, _I64, _I32, _I32, _P, _P]),
    "lf_eapca_device": (C.c_int, [_P, _I64, _I32, _I32, _P, _P]),
    "lf_bounds_eapca": (C.c_int, [_P, _I64, C.POINTER(LfIndex), _P, _P, _P, _P, _I32, _P, _P, _P]),
    "lf_leaf_header": (C.c_int, [C.c_char_p, C.POINTER(_I64), C.POINTER(_I32), C.POINTER(_I64)]),
    "lf_leaf_paa_file": (C.c_int, [C.c_char_p, _I64, _I32, _I32, _P, _I32, _P]),
    "lf_leaf_load": (C.c_int, [C.c_char_p, _I64, _I32, _P, _P, _I32, _P]),
    "lf_leaf_save": (C.c_int, [C.c_char_p, _P, _I64, _I32, _P]),
    "lf_quantize_rows": (C.c_int, [_P, _I64, _I32, _P, _P, _P]),
    "lf_replay_offsets": (C.c_int, [_P, _P, _P, _P, _I64, _I32, _P, _I64, _I32, _P, _P]),
}

_lib = None


def lib():
    """Load (once) the in-tree library; raise loudly when it is absent."""
    global _lib
    if _lib is None:
        if not LIB_PATH.exists():
            raise RuntimeError(
                f"{LIB_PATH} is missing: build it with `python -m paper_2502_01836_b200._build` "
                "(there is no CPU fallback)")
        h = C.CDLL(str(LIB_PATH))
        for name, (res, args) in SIGNATURES.items():
            fn = getattr(h, name)
            fn.restype = res
            fn.argtypes = args
        _lib = h
        check_abi()          # a stale library with another struct layout fails here, not in a kernel
    return _lib


STRUCTS = {"lf_index": LfIndex, "lf_search_opts": LfSearchOpts, "lf_trace": LfTrace}


def check_abi() -> None:
    """Assert that every ctypes mirror matches the compiled struct: sizeof and the
    offset of each field (lf_abi_sizeof / lf_abi_offsetof)."""
    h = lib()
    for name, cls in STRUCTS.items():
        size = h.lf_abi_sizeof(name.encode())
        if size != C.sizeof(cls):
            raise RuntimeError(f"{name}: ctypes sizeof {C.sizeof(cls)} != compiled {size}")
        for fname, _ in cls._fields_:
            off = h.lf_abi_offsetof(name.encode(), fname.encode())
            if off != getattr(cls, fname).offset:
                raise RuntimeError(f"{name}.{fname}: ctypes offset {getattr(cls, fname).offset} != compiled {off}")


def check(rc: int) -> None:
    if rc == LF_OK:
        return
    msg = lib().lf_last_error().decode(errors="replace")
    if rc == LF_EINVAL:
        raise ValueError(msg)
    raise RuntimeError(f"leafi_b200 error {rc}: {msg}")


def require_cuda():
    import torch

    if not torch.cuda.is_available():
        raise RuntimeError("paper_2502_01836_b200 needs a CUDA device (no CPU fallback)")
    return torch


def stream_ptr(stream=None) -> int:
    import torch

    s = stream if stream is not None else torch.cuda.current_stream()
    return int(s.cuda_stream)


def ptr(t) -> int | None:
    """Device (or host) address of a tensor / ndarray, None for None."""
    if t is None:
        return None
    if hasattr(t, "data_ptr"):
        return int(t.data_ptr())
    return int(t.ctypes.data)


def threads() -> int:
    return max(1, min(32, os.cpu_count() or 1))
