""".dsta matrix files (cli.py:60-116): every rank reads / writes its own column block.

Mirrors the reference's test_cli.py:24-73 (round trip for p in {1, 4}, bad magic,
truncated payload, no implicit casts) and pins the byte format against files the
reference's own writer produced (tests/golden/make_golden.py).  The CPU tests run
the in-process backend on host blocks; the gpu test streams device shards through
the pinned staging buffers in several chunks.
"""

import struct

import numpy as np
import pytest
import torch

import paper_2010_16114_b200 as bs
from paper_2010_16114_b200 import io as bio


@pytest.mark.parametrize("tag", ["f32", "f64", "i64"])
def test_reader_and_writer_match_reference_bytes(golden, tmp_path, tag):
    ref_bytes = golden[f"dsta_{tag}_bytes"].tobytes()
    data = golden[f"dsta_{tag}_data"]
    path = tmp_path / "ref.dsta"
    path.write_bytes(ref_bytes)
    out = tmp_path / "ours.dsta"

    def fn(comm):
        a = bio.read_matrix(path, comm)
        bio.write_matrix(out, a)
        comm.barrier()
        return bs.gather_full(a)

    for p in (1, 3):
        for full in bs.run_inproc(p, fn):
            np.testing.assert_array_equal(full, data)
            assert full.dtype == data.dtype
        assert out.read_bytes() == ref_bytes
    bio.write_matrix(out, data)  # plain (non-distributed) array
    assert out.read_bytes() == ref_bytes


@pytest.mark.parametrize("dtype", [np.float32, np.float64, np.int64, np.int8])
@pytest.mark.parametrize("p", [1, 4])
def test_matrix_roundtrip(tmp_path, dtype, p):
    gen = np.random.Generator(np.random.Philox(5))
    data = (gen.random((3, 7)) * 10).astype(dtype)
    path = tmp_path / "m.dsta"

    def fn(comm):
        a = bs.distribute(data if comm.rank == 0 else None, comm)
        bio.write_matrix(path, a)
        comm.barrier()
        return bs.gather_full(bio.read_matrix(path, comm))

    for full in bs.run_inproc(p, fn):
        np.testing.assert_array_equal(full, data)


def test_matrix_more_ranks_than_columns(tmp_path):
    data = np.arange(6.0).reshape(3, 2, order="F")
    path = tmp_path / "m.dsta"
    bio.write_matrix(path, data)
    for full in bs.run_inproc(4, lambda c: bs.gather_full(bio.read_matrix(path, c))):
        np.testing.assert_array_equal(full, data)


def test_matrix_bad_magic(tmp_path):
    path = tmp_path / "bad.dsta"
    path.write_bytes(b"NOPE" + b"\x00" * 32)
    with pytest.raises(bio.FormatError):
        bs.run_inproc(2, lambda c: bio.read_matrix(path, c))


def test_matrix_truncated_payload(tmp_path):
    path = tmp_path / "short.dsta"
    body = b"DSTA" + struct.pack("<B", 1) + struct.pack("<Q", 2) + struct.pack("<QQ", 2, 2)
    path.write_bytes(body + b"\x00" * 8)  # needs 32 payload bytes
    with pytest.raises(bio.FormatError):
        bs.run_inproc(1, lambda c: bio.read_matrix(path, c))


def test_matrix_dtype_mismatch_no_cast(tmp_path):
    path = tmp_path / "f32.dsta"
    bio.write_matrix(path, np.ones((2, 2), dtype=np.float32))
    with pytest.raises(bio.FormatError):
        bs.run_inproc(1, lambda c: bio.read_matrix(path, c, dtype=np.float64))


def test_unknown_dtype_code_and_missing_file(tmp_path):
    path = tmp_path / "code9.dsta"
    path.write_bytes(b"DSTA" + struct.pack("<B", 9) + struct.pack("<Q", 1) + struct.pack("<Q", 1) + b"\x00" * 8)
    with pytest.raises(bio.FormatError):
        bs.run_inproc(2, lambda c: bio.read_matrix(path, c))
    with pytest.raises(bio.FormatError):
        bs.run_inproc(2, lambda c: bio.read_matrix(tmp_path / "nope.dsta", c))


@pytest.mark.gpu
def test_device_shards_stream_in_chunks(tmp_path, monkeypatch):
    """Device blocks larger than one staging buffer: several pread -> pinned -> H2D rounds
    (and D2H -> pwrite on the way out), with uneven column blocks."""
    monkeypatch.setattr(bio, "_CHUNK", 4096)
    data = np.random.Generator(np.random.Philox(6)).random((257, 61)).astype(np.float32)
    path = tmp_path / "big.dsta"
    out = tmp_path / "big2.dsta"
    bio.write_matrix(path, data)

    def fn(comm):
        a = bio.read_matrix(path, comm, dtype=np.float32)
        assert a.local.is_cuda
        a.local.mul_(2.0)
        bio.write_matrix(out, a)
        comm.barrier()
        return bs.gather_full(bio.read_matrix(out, comm))

    for p in (1, 3):
        for full in bs.run_inproc(p, fn):
            np.testing.assert_array_equal(full, data * 2)
    assert torch.cuda.is_available()
