"""B200-native LeaFi hot path (arXiv 2502.01836).

Query-time search (bounds -> learned filters -> leaf scan) and build-time
training-data generation run as hand-written sm_100a CUDA kernels behind the
C-ABI in include/leafi_b200.h (library: _lib/libleafi_b200.so).  The Python
layer mirrors the reference package's seams (`leafsearch`: search_engine,
exact_search, search, SearchRequest, collect_targets, ...) so callers switch
by changing the import.  There is no CPU fallback.
"""

from .index import DeviceIndex, DeviceRows, TreeIndex, build_index, build_index_device, segment_layout, segment_means
from .engine import (
    BatchResult,
    SearchOutcome,
    SearchStats,
    TraceEntry,
    batch_distances,
    epsilon_search,
    exact_search,
    linear_scan,
    pruning_ratio,
    search_batch,
    search_engine,
)
from .filters import FilterPack
from .isax import build_isax_index
from .leafio import FileRows, FormatError, load_dataset_device, load_index, read_header, save_dataset

__version__ = "0.1.0"

__all__ = [
    "BatchResult",
    "DeviceIndex",
    "FileRows",
    "FilterPack",
    "FormatError",
    "SearchOutcome",
    "SearchStats",
    "TraceEntry",
    "TreeIndex",
    "batch_distances",
    "build_index",
    "build_index_device",
    "build_isax_index",
    "DeviceRows",
    "epsilon_search",
    "exact_search",
    "linear_scan",
    "load_dataset_device",
    "load_index",
    "pruning_ratio",
    "read_header",
    "save_dataset",
    "search_batch",
    "search_engine",
    "segment_layout",
    "segment_means",
]
