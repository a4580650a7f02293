"""LEAF-format header checks of the native loader (lf_leaf_header) against the
reference's `_load_matrix` rules and its persistence tests (series.py:198-212,
tests/test_series.py:181-231).  No GPU needed: the header pass is host-only."""

import struct

import numpy as np
import pytest

from oracle import leafi_oracle as lo


def _write(path, values, version=1):
    v = np.asarray(values, dtype="<f4")
    with open(path, "wb") as fh:
        fh.write(b"LEAF")
        fh.write(struct.pack("<III", version, v.shape[0], v.shape[1]))
        fh.write(v.tobytes())


def test_header_ok(tmp_path):
    from paper_2502_01836_b200 import read_header

    p = tmp_path / "d.bin"
    _write(p, lo.randwalk(10, 16, 16))
    assert read_header(p) == (10, 16)


def test_bad_magic(tmp_path):
    from paper_2502_01836_b200 import FormatError, read_header

    p = tmp_path / "bad.bin"
    _write(p, lo.randwalk(4, 8, 18))
    raw = bytearray(p.read_bytes())
    raw[:4] = b"XXXX"
    p.write_bytes(bytes(raw))
    with pytest.raises(FormatError) as err:
        read_header(p)
    assert err.value.offset == 0
    assert "bad magic b'XXXX'" in str(err.value)


def test_truncated_payload(tmp_path):
    from paper_2502_01836_b200 import FormatError, read_header

    p = tmp_path / "trunc.bin"
    _write(p, lo.randwalk(4, 8, 19))
    raw = p.read_bytes()
    p.write_bytes(raw[:-5])
    with pytest.raises(FormatError) as err:
        read_header(p)
    assert err.value.offset == len(raw) - 5
    assert f"file length {len(raw) - 5} does not match header-implied {len(raw)}" in str(err.value)


def test_truncated_header(tmp_path):
    from paper_2502_01836_b200 import FormatError, read_header

    p = tmp_path / "short.bin"
    p.write_bytes(b"LEAF\x01")
    with pytest.raises(FormatError) as err:
        read_header(p)
    assert err.value.offset == 5


def test_bad_version(tmp_path):
    from paper_2502_01836_b200 import FormatError, read_header

    p = tmp_path / "ver.bin"
    _write(p, lo.randwalk(4, 8, 20))
    raw = bytearray(p.read_bytes())
    raw[4] = 99
    p.write_bytes(bytes(raw))
    with pytest.raises(FormatError) as err:
        read_header(p)
    assert err.value.offset == 4
    assert "unsupported format version 99" in str(err.value)


def test_missing_file(tmp_path):
    from paper_2502_01836_b200 import read_header

    with pytest.raises(ValueError):
        read_header(tmp_path / "absent.bin")


def test_file_rows_memmap(tmp_path):
    from paper_2502_01836_b200 import FileRows

    v = lo.randwalk(50, 12, 3)
    p = tmp_path / "d.bin"
    _write(p, v)
    rows = FileRows(p)
    assert rows.shape == (50, 12) and len(rows) == 50
    assert np.array_equal(rows[[3, 7]], v[[3, 7]].astype(np.float32))
    assert np.array_equal(rows[10:20], v[10:20].astype(np.float32))


@pytest.mark.reference
def test_messages_match_reference(tmp_path):
    """The same malformed files raise the reference's FormatError messages and offsets."""
    import sys

    sys.path.insert(0, "/root/reference/pkg/src")
    from leafsearch import series as rs

    from paper_2502_01836_b200 import FormatError, read_header

    good = tmp_path / "g.bin"
    rs.save_dataset(rs.generate_randwalk(6, 8, seed=5), good)
    raw = good.read_bytes()
    cases = {"magic": b"ABCD" + raw[4:], "short": raw[:7], "trunc": raw[:-3],
             "ver": raw[:4] + struct.pack("<I", 7) + raw[8:], "long": raw + b"\0\0"}
    for name, blob in cases.items():
        p = tmp_path / f"{name}.bin"
        p.write_bytes(blob)
        with pytest.raises(rs.FormatError) as ref_err:
            rs.load_dataset(p)
        with pytest.raises(FormatError) as our_err:
            read_header(p)
        assert our_err.value.offset == ref_err.value.offset, name
        assert str(our_err.value) == str(ref_err.value), name
    assert read_header(good) == (6, 8)
    assert np.array_equal(np.asarray(np.memmap(good, "<f4", "r", 16, (6, 8)), np.float64),
                          rs.load_dataset(good).values)
