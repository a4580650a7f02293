"""Memory-lean LEAF loader on the GPU: file -> HBM round trips,
the two-pass load_index (device segment means, host tree from them, rows
scattered into the leaf-contiguous layout) against the host build and the
oracle, shard loads, and the reference's error behaviour."""

import struct

import numpy as np
import pytest

from oracle import leafi_oracle as lo

pytestmark = pytest.mark.gpu


def _write(path, values):
    v = np.asarray(values, dtype="<f4")
    with open(path, "wb") as fh:
        fh.write(b"LEAF" + struct.pack("<III", 1, v.shape[0], v.shape[1]) + v.tobytes())


def test_save_load_round_trip(tmp_path):
    import torch

    from paper_2502_01836_b200 import load_dataset_device, save_dataset

    v = lo.randwalk(70_001, 48, 3).astype(np.float32)     # several 16 MB chunks, ragged tail
    X = torch.from_numpy(v).cuda()
    p = tmp_path / "d.bin"
    save_dataset(X, p)
    assert p.stat().st_size == 16 + v.nbytes
    raw = p.read_bytes()
    assert raw[:4] == b"LEAF" and struct.unpack("<III", raw[4:16]) == (1, 70_001, 48)
    assert np.array_equal(np.frombuffer(raw, "<f4", offset=16).reshape(v.shape), v)
    for threads in (1, 3, 8):
        Y = load_dataset_device(p, threads=threads)
        assert torch.equal(Y.cpu(), X.cpu())


def test_load_index_matches_host_build(tmp_path):
    import torch

    from paper_2502_01836_b200 import build_index, load_index, search_batch

    v = lo.randwalk(30_000, 64, 21)
    p = tmp_path / "c.bin"
    _write(p, v)
    a = build_index(v, max_leaf_size=500)
    b = load_index(p, max_leaf_size=500)
    for f in ("env_min", "env_max", "left", "right", "split_seg", "size", "member_ptr", "members"):
        assert np.array_equal(getattr(a, f), getattr(b, f)), f
    assert np.array_equal(np.nan_to_num(a.split_thr, nan=-7), np.nan_to_num(b.split_thr, nan=-7))
    da, db = a.device(), b.device()
    assert torch.equal(da.X, db.X) and torch.equal(da.row_id, db.row_id)
    q = lo.noisy_queries(v, 24, 0.2, 5)
    ra = search_batch(a, q, 3)
    rb = search_batch(b, q, 3)
    assert np.array_equal(ra.ids, rb.ids) and np.array_equal(ra.dists, rb.dists)
    ot = lo.build_tree(v, 500)
    for i in range(0, 24, 5):
        o = lo.search(ot, q[i], 3)
        assert rb.ids[i].tolist() == [x for x, _ in o.results]


def test_load_index_shards(tmp_path):
    import torch

    from paper_2502_01836_b200 import build_index, load_index

    v = lo.randwalk(20_000, 32, 8)
    p = tmp_path / "s.bin"
    _write(p, v)
    a = build_index(v, max_leaf_size=300)
    b = load_index(p, max_leaf_size=300)
    for rank in range(3):
        sa, sb = a.shard(rank, 3), b.shard(rank, 3)
        assert sb.X.shape[0] == sa.X.shape[0] < v.shape[0]
        assert torch.equal(sa.X, sb.X)


def test_rejects_non_finite_and_malformed(tmp_path):
    from paper_2502_01836_b200 import FormatError, load_dataset_device, load_index

    v = lo.randwalk(5000, 16, 4).astype(np.float32)
    v[4321, 7] = np.nan
    p = tmp_path / "nan.bin"
    _write(p, v)
    with pytest.raises(ValueError, match="non-finite"):
        load_dataset_device(p)
    with pytest.raises(ValueError, match="non-finite"):
        load_index(p, max_leaf_size=100)
    q = tmp_path / "bad.bin"
    q.write_bytes(b"LEAF\x01\x00\x00\x00\x02\x00\x00\x00\x02\x00\x00\x00" + b"\0" * 12)
    with pytest.raises(FormatError) as err:
        load_dataset_device(q)
    assert err.value.offset == 28
