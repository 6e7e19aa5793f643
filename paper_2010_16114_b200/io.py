"""``.dsta`` matrix files read into / written from device shards (cli.py:60-116).

Format (cli.py:14-17, README.md:110-113): magic ``DSTA``, one dtype byte
(0 = f32, 1 = f64, 2 = i64), the number of dimensions as a little-endian u64,
one u64 extent per dimension, then the payload as column-major little-endian
scalars.  This build adds dtype code 3 = int8 (genotype matrices); files with
codes 0-2 are byte-identical to the reference's.

The reference reads the whole file on rank 0 and scatters it (``read_matrix``:
rank 0 ``fh.read()`` + ``distribute``), and writes by gathering to rank 0
(``write_matrix``).  Because the payload is column-major and arrays are split
on the last dimension, every rank's block is one contiguous byte range of the
file.  Here each rank reads (``os.pread``) / writes (``os.pwrite``) its own
range directly, staged through two pinned host buffers so the file I/O of one
chunk overlaps the host<->device copy of the previous one; no payload crosses
ranks.  Errors keep the reference's behaviour: any rank's failure raises
``FormatError`` on every rank (the status is all-reduced before use).
"""

from __future__ import annotations

import os
import struct

import numpy as np

from .comm import ReduceOp
from .distarray import DistArray, partition_of

_MAGIC = b"DSTA"
_DTYPE_BY_CODE = {0: np.dtype(np.float32), 1: np.dtype(np.float64), 2: np.dtype(np.int64),
                  3: np.dtype(np.int8)}
_CODE_BY_DTYPE = {v: k for k, v in _DTYPE_BY_CODE.items()}
_CHUNK = 64 << 20  # bytes per staging buffer


class FormatError(ValueError):
    """Matrix file violates the on-disk format (cli.py:57-58)."""


def _torch():
    import torch

    return torch


def header_bytes(ndim):
    return 4 + 1 + 8 + 8 * ndim


def _encode_header(dtype, shape):
    return (_MAGIC + struct.pack("<B", _CODE_BY_DTYPE[np.dtype(dtype)]) + struct.pack("<Q", len(shape)) +
            struct.pack(f"<{len(shape)}Q", *shape))


def read_header(path):
    """(dtype, shape, payload offset) of a .dsta file (cli.py:81-90)."""
    with open(path, "rb") as fh:
        magic = fh.read(4)
        if magic != _MAGIC:
            raise FormatError(f"bad magic {magic!r}")
        raw = fh.read(1)
        if len(raw) != 1:
            raise FormatError("truncated header")
        (code,) = struct.unpack("<B", raw)
        if code not in _DTYPE_BY_CODE:
            raise FormatError(f"unknown dtype code {code}")
        raw = fh.read(8)
        if len(raw) != 8:
            raise FormatError("truncated header")
        (ndim,) = struct.unpack("<Q", raw)
        if ndim > 64:
            raise FormatError(f"implausible number of dimensions {ndim}")
        raw = fh.read(8 * ndim)
        if len(raw) != 8 * ndim:
            raise FormatError("truncated header")
        shape = struct.unpack(f"<{ndim}Q", raw)
    return _DTYPE_BY_CODE[code], tuple(int(s) for s in shape), header_bytes(ndim)


class _Stager:
    """Two pinned host buffers alternating between file I/O and async H2D/D2H copies."""

    def __init__(self, device, nbytes):
        torch = _torch()
        self.torch = torch
        self.cuda = device.type == "cuda"
        size = max(1, min(_CHUNK, nbytes))
        self.bufs = [torch.empty(size, dtype=torch.uint8, pin_memory=self.cuda) for _ in range(2)]
        self.events = [None, None]
        self.stream = torch.cuda.Stream(device) if self.cuda else None
        self.size = size

    def wait(self, i):
        if self.events[i] is not None:
            self.events[i].synchronize()
            self.events[i] = None

    def record(self, i):
        if self.cuda:
            ev = self.torch.cuda.Event()
            ev.record(self.stream)
            self.events[i] = ev

    def finish(self):
        for i in range(2):
            self.wait(i)


def _read_block(fd, offset, nbytes, dst_bytes):
    """Stream file bytes [offset, offset + nbytes) into the flat uint8 device view ``dst_bytes``."""
    torch = _torch()
    st = _Stager(dst_bytes.device, nbytes)
    done, i = 0, 0
    while done < nbytes:
        n = min(st.size, nbytes - done)
        st.wait(i)
        view = st.bufs[i][:n].numpy()
        got = 0
        while got < n:
            chunk = os.pread(fd, n - got, offset + done + got)
            if not chunk:
                raise FormatError(f"payload ends after {done + got} of {nbytes} bytes of this block")
            view[got:got + len(chunk)] = np.frombuffer(chunk, dtype=np.uint8)
            got += len(chunk)
        if st.cuda:
            with torch.cuda.stream(st.stream):
                dst_bytes[done:done + n].copy_(st.bufs[i][:n], non_blocking=True)
            st.record(i)
        else:
            dst_bytes[done:done + n].copy_(st.bufs[i][:n])
        done += n
        i ^= 1
    st.finish()


def _write_block(fd, offset, src_bytes):
    torch = _torch()
    nbytes = src_bytes.numel()
    st = _Stager(src_bytes.device, nbytes)
    pending = [None, None]  # (n, file offset) staged in buffer i

    def flush(i):
        if pending[i] is not None:
            st.wait(i)
            n, off = pending[i]
            view = memoryview(st.bufs[i][:n].numpy())
            put = 0
            while put < n:
                put += os.pwrite(fd, view[put:], off + put)
            pending[i] = None

    done, i = 0, 0
    if st.cuda:
        torch.cuda.current_stream(src_bytes.device).synchronize()  # producer kernels done
    while done < nbytes:
        n = min(st.size, nbytes - done)
        flush(i)
        if st.cuda:
            with torch.cuda.stream(st.stream):
                st.bufs[i][:n].copy_(src_bytes[done:done + n], non_blocking=True)
            st.record(i)
        else:
            st.bufs[i][:n].copy_(src_bytes[done:done + n])
        pending[i] = (n, offset + done)
        done += n
        i ^= 1
    flush(i)
    flush(i ^ 1)


def _bytes_view(t):
    """Flat uint8 view of a column-major (Fortran-strided) block's storage."""
    from .comm import fortran_flat

    flat, _ = fortran_flat(t)
    return flat.view(_torch().uint8)


def _agree(comm, failed, message):
    """All ranks learn whether any rank failed (the reference broadcasts rank 0's status)."""
    status = np.array([1.0 if failed else 0.0])
    comm.allreduce(status, ReduceOp.MAX)
    if status[0]:
        raise FormatError(message or "another rank failed to read or write its block of the matrix file")


def read_matrix(path, comm, dtype=None):
    """Read a .dsta file into a DistArray, each rank loading its own column block (cli.py:93-116).

    No implicit casts: ``dtype`` must match the file (FormatError otherwise).
    """
    failed, message, arr = False, "", None
    try:
        fdt, shape, off = read_header(path)
        if dtype is not None and fdt != np.dtype(dtype):
            raise FormatError(f"file holds {fdt}, run expects {np.dtype(dtype)}")
        if not shape:
            raise FormatError("zero-dimensional matrix")
        want = int(np.prod(shape, dtype=np.int64)) * fdt.itemsize
        have = os.path.getsize(path) - off
        if have != want:
            raise FormatError(f"payload is {have} bytes, expected {want}")
    except (OSError, FormatError) as exc:
        failed, message = True, str(exc)
    _agree(comm, failed, message)
    try:
        arr = DistArray(comm, shape, fdt)
        col_bytes = int(np.prod(shape[:-1], dtype=np.int64)) * fdt.itemsize
        part = partition_of(shape[-1], comm.size)
        nbytes = col_bytes * part.width(comm.rank)
        if nbytes:
            fd = os.open(path, os.O_RDONLY)
            try:
                _read_block(fd, off + col_bytes * part.lo(comm.rank), nbytes, _bytes_view(arr.local))
            finally:
                os.close(fd)
    except (OSError, FormatError) as exc:
        failed, message = True, str(exc)
    _agree(comm, failed, message)
    return arr


def write_matrix(path, array):
    """Write a DistArray (every rank writes its own byte range) or a plain array (cli.py:63-78).

    PackedGenotypes are written as the int8 matrix they hold (dtype code 3)."""
    if getattr(array, "packed", False):
        from .distarray import unpack_genotypes

        array = unpack_genotypes(array)
    if not isinstance(array, DistArray):
        data = np.asarray(array)
        if data.dtype not in _CODE_BY_DTYPE:
            raise FormatError(f"unsupported dtype {data.dtype}")
        with open(path, "wb") as fh:
            fh.write(_encode_header(data.dtype, data.shape))
            fh.write(np.ravel(data, order="F").tobytes())
        return
    comm = array.comm
    failed, message = False, ""
    if array.dtype not in _CODE_BY_DTYPE:
        raise FormatError(f"unsupported dtype {array.dtype}")
    hdr = _encode_header(array.dtype, array.shape)
    total = len(hdr) + int(np.prod(array.shape, dtype=np.int64)) * array.dtype.itemsize
    if comm.rank == 0:
        try:
            with open(path, "wb") as fh:  # create / truncate, then size the file
                fh.write(hdr)
                fh.truncate(total)
        except OSError as exc:
            failed, message = True, str(exc)
    _agree(comm, failed, message)  # also orders the header before the payload writes
    try:
        col_bytes = int(np.prod(array.shape[:-1], dtype=np.int64)) * array.dtype.itemsize
        if array.local.numel():
            fd = os.open(path, os.O_WRONLY)
            try:
                _write_block(fd, len(hdr) + col_bytes * array.lo, _bytes_view(array.local))
            finally:
                os.close(fd)
    except OSError as exc:
        failed, message = True, str(exc)
    _agree(comm, failed, message)
