import os
import sys
from pathlib import Path

import numpy as np
import pytest

ROOT = Path(__file__).resolve().parent.parent
GOLDEN = ROOT / "tests" / "golden"
sys.path.insert(0, str(ROOT))

REFERENCE_SRC = "/root/reference/pkg/src"


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a B200 (runs under gpurun / the round-end GPU tier)")
    config.addinivalue_line("markers", "reference: needs the reference package (build container only)")
    config.addinivalue_line("markers", "slow: minutes-long parity case")


def pytest_collection_modifyitems(config, items):
    have_ref = os.path.isdir(REFERENCE_SRC)
    skip_ref = pytest.mark.skip(reason="reference package not present on this host")
    for item in items:
        if "reference" in item.keywords and not have_ref:
            item.add_marker(skip_ref)


def load_golden(name: str) -> dict:
    with np.load(GOLDEN / name, allow_pickle=False) as z:
        return {k: z[k] for k in z.files}


@pytest.fixture(scope="session")
def knowns():
    return load_golden("knowns.npz")


@pytest.fixture(scope="session")
def small_golden():
    return load_golden("small.npz")


@pytest.fixture(scope="session")
def pipeline_golden():
    return load_golden("pipeline.npz")


def oracle_tree_from_table(values: np.ndarray, g: dict, prefix: str = "nt_", segments: int = 8):
    """Rebuild an oracle tree from a golden node table (no reference needed)."""
    from oracle import leafi_oracle as lo

    starts, widths = lo.seg_layout(values.shape[1], segments)
    t = lo.OracleTree(values, starts, widths, 0)
    ptr = g[prefix + "member_ptr"]
    mem = g[prefix + "members"]
    n = g[prefix + "left"].shape[0]
    for i in range(n):
        t.env_min.append(g[prefix + "env_min"][i].copy())
        t.env_max.append(g[prefix + "env_max"][i].copy())
        t.left.append(int(g[prefix + "left"][i]))
        t.right.append(int(g[prefix + "right"][i]))
        t.split_seg.append(int(g[prefix + "split_seg"][i]))
        t.split_thr.append(float(g[prefix + "split_thr"][i]))
        leaf = bool(g[prefix + "is_leaf"][i])
        t.member_lists.append([int(x) for x in mem[ptr[i]:ptr[i + 1]]] if leaf else None)
        t.size.append(int(g[prefix + "size"][i]))
        t.oversized.append(bool(g[prefix + "oversized"][i]))
    return t.freeze()
