"""CPU-side checks of the product: the C-ABI library loads, exports every
declared symbol, and its host-only entry points (native tree build, segment
means) reproduce the reference bit-for-bit.  No GPU compute here."""

import re
from pathlib import Path

import numpy as np
import pytest

from oracle import leafi_oracle as lo

ROOT = Path(__file__).resolve().parent.parent


def declared_symbols():
    text = (ROOT / "include" / "leafi_b200.h").read_text()
    text = re.sub(r"/\*.*?\*/", "", text, flags=re.S)
    return sorted(set(re.findall(r"\b(lf_[a-z0-9_]+)\s*\(", text)))


def test_header_declares_the_path():
    syms = declared_symbols()
    for s in ("lf_search", "lf_bounds", "lf_filter_predict", "lf_leaf_min_dist", "lf_local_min_dist",
              "lf_batch_distances", "lf_tree_build"):
        assert s in syms


def test_library_exports_every_declared_symbol():
    from paper_2502_01836_b200 import _lib

    h = _lib.lib()
    for s in declared_symbols():
        assert hasattr(h, s), s
        assert s in _lib.SIGNATURES, f"{s} has no ctypes signature"
    assert h.lf_version() == 1


def _header_fields(struct: str) -> list:
    text = (ROOT / "include" / "leafi_b200.h").read_text()
    body = re.search(r"typedef struct %s \{(.*?)\} %s;" % (struct, struct), text, re.S).group(1)
    body = re.sub(r"/\*.*?\*/", "", body, flags=re.S)
    return [re.search(r"(\w+)\s*(\[[^\]]*\])?$", d.strip()).group(1) for d in body.split(";") if d.strip()]


def test_struct_layouts_match_header():
    """ctypes structs mirror the compiled C structs: the same fields in header order,
    and sizeof / every offsetof equal to what the library reports (lf_abi_*)."""
    from paper_2502_01836_b200 import _lib

    h = _lib.lib()
    for name, cls in _lib.STRUCTS.items():
        assert [f for f, _ in cls._fields_] == _header_fields(name), name
    _lib.check_abi()
    assert h.lf_abi_sizeof(b"nope") == -1
    assert h.lf_abi_offsetof(b"lf_index", b"nope") == -1
    assert h.lf_abi_offsetof(b"lf_index", b"n_series") == 0


def test_integration_stub_matches_header():
    """INTEGRATION.md's ctypes mirrors are the generator's output for the current header."""
    import sys

    sys.path.insert(0, str(ROOT / "tools"))
    import gen_ctypes_stub

    assert gen_ctypes_stub.doc_block() in (ROOT / "INTEGRATION.md").read_text()
    ns = {}
    exec(gen_ctypes_stub.stub().split("lib = C.CDLL")[0].replace("```python", ""), ns)
    from paper_2502_01836_b200 import _lib
    for name, cls in _lib.STRUCTS.items():
        stub_cls = ns[cls.__name__]
        assert [f for f, _ in stub_cls._fields_] == [f for f, _ in cls._fields_], name
        import ctypes as C
        assert C.sizeof(stub_cls) == _lib.lib().lf_abi_sizeof(name.encode()), name


def _table_equal(t, g, prefix="nt_"):
    np.testing.assert_array_equal(t.env_min, g[prefix + "env_min"])
    np.testing.assert_array_equal(t.env_max, g[prefix + "env_max"])
    np.testing.assert_array_equal(t.left, g[prefix + "left"])
    np.testing.assert_array_equal(t.right, g[prefix + "right"])
    np.testing.assert_array_equal(t.split_seg, g[prefix + "split_seg"])
    np.testing.assert_array_equal(t.split_thr, g[prefix + "split_thr"])
    np.testing.assert_array_equal(t.size, g[prefix + "size"])
    np.testing.assert_array_equal(t.oversized, g[prefix + "oversized"])
    np.testing.assert_array_equal(t.member_ptr, g[prefix + "member_ptr"])
    if prefix + "members" in g:
        np.testing.assert_array_equal(t.members, g[prefix + "members"])


def test_native_build_small(small_golden):
    from paper_2502_01836_b200 import build_index

    t = build_index(lo.randwalk(2000, 32, 7), max_leaf_size=128)
    _table_equal(t, small_golden)


def test_native_build_pipeline(pipeline_golden):
    from paper_2502_01836_b200 import build_index

    t = build_index(lo.randwalk(4000, 32, 17), max_leaf_size=200)
    _table_equal(t, pipeline_golden)


def test_native_build_c1():
    """BASELINE config 1 (100K x 256, cap 1000): identical node table (hashes from the reference)."""
    import hashlib, json
    from conftest import GOLDEN, load_golden
    from paper_2502_01836_b200 import build_index

    doc = json.loads((GOLDEN / "c1.json").read_text())
    g = load_golden("c1.npz")
    v = lo.randwalk(100_000, 256, 1234)
    assert hashlib.sha256(v.tobytes()).hexdigest() == doc["data_sha"]
    t = build_index(v, max_leaf_size=1000)
    assert t.n_nodes == doc["n_nodes"] and t.n_leaves == doc["n_leaves"]
    assert hashlib.sha256(t.members.tobytes()).hexdigest() == doc["members_sha"]
    assert hashlib.sha256(t.env_min.tobytes()).hexdigest() == doc["env_min_sha"]
    assert hashlib.sha256(t.env_max.tobytes()).hexdigest() == doc["env_max_sha"]
    _table_equal(t, g)


def test_native_build_oversized():
    """Identical series cannot be split (reference test_tree.py:64-72)."""
    from paper_2502_01836_b200 import build_index

    row = np.linspace(-1.0, 1.0, 16).astype(np.float32).astype(np.float64)  # fp32 storage contract
    t = build_index(np.tile(row, (40, 1)), max_leaf_size=8)
    assert t.has_oversized_leaves() and t.n_leaves == 1 and t.size[0] == 40


def test_native_build_validation():
    from paper_2502_01836_b200 import build_index

    with pytest.raises(ValueError):
        build_index(lo.randwalk(50, 16, 0), max_leaf_size=1)
    with pytest.raises(ValueError):
        build_index(np.array([[0.1, 0.2]]) / 3.0)   # not fp32-exact


@pytest.mark.parametrize("m", [256, 96, 32])
def test_segment_means_host(knowns, m):
    from paper_2502_01836_b200 import segment_means

    np.testing.assert_array_equal(segment_means(knowns[f"paa_{m}_rows"], 8), knowns[f"paa_{m}"])


def test_single_leaf_and_reference_adoption():
    from paper_2502_01836_b200 import TreeIndex, build_index

    t = build_index(lo.randwalk(10, 16, 0), max_leaf_size=16)
    assert t.n_leaves == 1 and t.leaf_members(0).tolist() == list(range(10))
    with pytest.raises(Exception):
        TreeIndex.from_reference(object())


def test_product_has_no_oracle_dependency():
    """The shipped package never imports the test oracle."""
    pkg = ROOT / "paper_2502_01836_b200"
    for p in pkg.rglob("*.py"):
        src = p.read_text()
        assert "oracle" not in re.findall(r"^\s*(?:from|import)\s+(\S+)", src, flags=re.M), p
        assert "leafi_oracle" not in src, p
