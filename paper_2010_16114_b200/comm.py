"""Rank-based collectives for the B200 build (contract of blockstat comm.py).

The reference's ``Communicator`` (comm.py:178-264) is kept: every rank issues
the same sequence of broadcast / allreduce / allgatherv / scatterv / barrier
calls on buffers that are flattened in column-major order and written back in
place.  Two backends implement it here:

``inproc:<P>``
    P rank *threads* in one process (comm.py:267-357): the execution model of
    ``run_inproc``.  Rank r drives device ``r % ndevices`` on
    its own CUDA stream.  Payloads may be CUDA tensors (folded on device by the
    ``bs_fold`` kernel, in ascending rank order like comm.py:93-99) or numpy
    arrays (folded on the host exactly as the reference does).  Headers are
    validated like comm.py:102-153 and violations raise
    ``CollectiveContractError`` on every rank.

``nccl`` / ``gloo``
    One process per rank under ``torchrun`` (the multi-GPU path): the
    collectives map onto ``torch.distributed`` (NCCL over NVLink/NVSwitch on a
    B200 box).  NCCL has no v-variants, so ``allgatherv`` / ``reduce_scatterv``
    pad every block to the largest count.

``reduce_scatterv`` is an addition to the reference's five collectives: the
reference all-reduces the r x m product of scenario b and then keeps only its
own column slice (distlinalg.py:251-252); a reduce-scatter moves 1/p of the data.

``tcp:<host:port>,...,rank=<r>``
    The reference's multi-process descriptor (comm.py:12-15, 501-519).  Instead
    of a hub that relays every payload over sockets (comm.py:360-578), the
    first host:port serves a TCPStore rendezvous that bootstraps a
    torch.distributed world (NCCL's unique id travels through the store); the
    collectives then run as in the ``nccl`` / ``gloo`` backend.
"""

from __future__ import annotations

import ctypes
import enum
import os
import re
import threading

import numpy as np


class CommError(RuntimeError):
    """Base class for communication failures."""


class CommInitError(CommError):
    """World could not be constructed (bad descriptor, unreachable peer, ...)."""


class CollectiveContractError(CommError):
    """Ranks invoked collectives with incompatible arguments."""


class RankAbortedError(CommError):
    """Another rank aborted or timed out while this rank waited."""


class ReduceOp(enum.Enum):
    SUM = "sum"
    PROD = "prod"
    MAX = "max"
    MIN = "min"


_REDUCE_UFUNC = {
    ReduceOp.SUM: np.add,
    ReduceOp.PROD: np.multiply,
    ReduceOp.MAX: np.maximum,
    ReduceOp.MIN: np.minimum,
}
_OP_CODE = {ReduceOp.SUM: 0, ReduceOp.PROD: 1, ReduceOp.MAX: 2, ReduceOp.MIN: 3}

_DTYPE_CODES = {
    np.dtype(np.float32): 0,
    np.dtype(np.float64): 1,
    np.dtype(np.int64): 2,
}
_CODE_DTYPES = {v: k for k, v in _DTYPE_CODES.items()}


def _torch():
    import torch

    return torch


def _is_tensor(x):
    try:
        import torch
    except ImportError:  # pragma: no cover
        return False
    return isinstance(x, torch.Tensor)


def _np_dtype(buf):
    if _is_tensor(buf):
        torch = _torch()
        table = {torch.float32: np.dtype(np.float32), torch.float64: np.dtype(np.float64),
                 torch.int64: np.dtype(np.int64)}
        if buf.dtype not in table:
            raise ValueError(f"unsupported buffer dtype {buf.dtype}; use float32/float64/int64")
        return table[buf.dtype]
    dt = np.asarray(buf).dtype
    if dt not in _DTYPE_CODES:
        raise ValueError(f"unsupported buffer dtype {dt}; use float32/float64/int64")
    return dt


def fortran_flat(t):
    """Column-major flattening of a tensor as a view when possible.

    Returns ``(flat, writeback)``; ``writeback`` is True when ``flat`` is a
    copy that must be written back into ``t`` after an in-place collective.
    """
    if t.ndim <= 1:
        return (t, False) if t.is_contiguous() else (t.contiguous(), True)
    rev = t.permute(*reversed(range(t.ndim)))
    if rev.is_contiguous():
        return rev.reshape(-1), False
    return rev.contiguous().reshape(-1), True


def _fortran_writeback(t, flat):
    rev = t.permute(*reversed(range(t.ndim))) if t.ndim > 1 else t
    rev.copy_(flat.reshape(rev.shape))


def _np_flat(buf):
    arr = np.asarray(buf)
    return np.ravel(arr, order="F")


def _np_writeback(buf, flat):
    buf[...] = np.asarray(flat).reshape(buf.shape, order="F")


# Fields every rank must agree on, per collective (the reference's contract, comm.py:102-153).
_AGREE = {
    "broadcast": (("dtype", "buffer dtype"), ("root", "broadcast root"), ("recv_len", "broadcast buffer length")),
    "allreduce": (("dtype", "buffer dtype"), ("redop", "reduction operator"),
                  ("recv_len", "allreduce buffer length")),
    "allgatherv": (("dtype", "buffer dtype"), ("counts", "allgatherv counts")),
    "reduce_scatterv": (("dtype", "buffer dtype"), ("counts", "reduce_scatterv counts"),
                        ("redop", "reduction operator")),
    "scatterv": (("dtype", "buffer dtype"), ("counts", "scatterv counts"), ("root", "scatterv root")),
    "barrier": (),
}


def _lengths_ok(op, headers):
    """Per-rank buffer lengths against the agreed counts; returns an error message or None."""
    counts = headers[0]["counts"]
    if op in ("allgatherv", "reduce_scatterv"):
        block, whole = ("send_len", "recv_len") if op == "allgatherv" else ("recv_len", "send_len")
        total = sum(counts)
        for r, h in enumerate(headers):
            if h[block] != counts[r]:
                return f"{op}: rank {r} block holds {h[block]} values, counts say {counts[r]}"
            if h[whole] != total:
                return f"{op}: rank {r} full buffer holds {h[whole]}, need {total}"
    elif op == "scatterv":
        root = headers[0]["root"]
        if headers[root]["send_len"] != sum(counts):
            return f"scatterv: root sends {headers[root]['send_len']} values, counts sum to {sum(counts)}"
        bad = [r for r, h in enumerate(headers) if h["recv_len"] != counts[r]]
        if bad:
            r = bad[0]
            return f"scatterv: rank {r} receive buffer holds {headers[r]['recv_len']}, counts say {counts[r]}"
    return None


def _validate_headers(headers):
    """Cross-rank contract checks; raises CollectiveContractError on the first violation."""
    first = headers[0]
    fields = (("op", "collective operation"), ("seq", "collective sequence number"))
    for field, what in fields + _AGREE.get(first["op"], ()):
        odd = next((r for r, h in enumerate(headers) if h[field] != first[field]), None)
        if odd is not None:
            raise CollectiveContractError(
                f"{what} mismatch: rank 0 has {first[field]!r}, rank {odd} has {headers[odd][field]!r}")
    if first["op"] not in _AGREE:  # pragma: no cover
        raise CollectiveContractError(f"unknown collective {first['op']!r}")
    msg = _lengths_ok(first["op"], headers)
    if msg:
        raise CollectiveContractError(msg)


class Communicator:
    """One rank's endpoint into a world of ``size`` ranks (comm.py:178-264).

    Buffers may be numpy arrays or torch tensors (host or device).  Device
    tensors stay on the device; collectives run on the rank's current stream.
    """

    rank: int
    size: int
    backend: str

    def __init__(self):
        self._seq = 0
        self.device = None

    # -- collectives -----------------------------------------------------
    def broadcast(self, buf, root=0):
        if not 0 <= root < self.size:
            raise ValueError(f"root {root} out of range for size {self.size}")
        self._collective("broadcast", buf, root=root)

    def allreduce(self, buf, op=ReduceOp.SUM):
        self._collective("allreduce", buf, redop=op)

    def allgatherv(self, send, recv, counts):
        counts = self._counts(counts)
        self._collective("allgatherv", recv, send=send, counts=counts)

    def reduce_scatterv(self, send, recv, counts, op=ReduceOp.SUM):
        """Fold every rank's ``send`` (length sum(counts)) and keep block ``rank``."""
        counts = self._counts(counts)
        self._collective("reduce_scatterv", recv, send=send, counts=counts, redop=op)

    def scatterv(self, send, recv, counts, root=0):
        counts = self._counts(counts)
        self._collective("scatterv", recv, send=send, counts=counts, root=root)

    def barrier(self):
        self._collective("barrier", None)

    def _counts(self, counts):
        counts = tuple(int(c) for c in counts)
        if len(counts) != self.size:
            raise ValueError(f"counts has {len(counts)} entries for {self.size} ranks")
        return counts

    def _collective(self, op, buf, **kw):
        raise NotImplementedError

    def close(self):
        pass

    def abort(self):
        """Break peers out of pending collectives after a local failure."""

    @property
    def stream(self):
        if self.device is None or self.device.type != "cuda":
            return None
        return _torch().cuda.current_stream(self.device)

    def __repr__(self):
        return f"<Communicator rank={self.rank} size={self.size} backend={self.backend}>"


# ---------------------------------------------------------------------------
# In-process backend
# ---------------------------------------------------------------------------


class _InProcWorld:
    """Rendezvous board of the in-process world (one rank per thread).

    Collective number ``seq`` gets its own board: every rank posts its (header,
    payload) entry, waits on the shared condition until all ``size`` entries are
    there, takes a snapshot, and the last rank to read retires the board.  A rank
    that fails (or a wait that exceeds ``timeout``) aborts the world: every waiter
    wakes up with RankAbortedError.
    """

    def __init__(self, size, timeout=180.0):
        self.size = size
        self.timeout = timeout
        self._cond = threading.Condition()
        self._boards = {}
        self._aborted = False

    def exchange(self, rank, seq, entry):
        with self._cond:
            if self._aborted:
                raise RankAbortedError("world aborted")
            board = self._boards.setdefault(seq, {"entries": [None] * self.size, "posted": 0, "read": 0})
            board["entries"][rank] = entry
            board["posted"] += 1
            if board["posted"] == self.size:
                self._cond.notify_all()
            elif not self._cond.wait_for(lambda: self._aborted or board["posted"] == self.size, self.timeout):
                self._abort_locked()
                raise RankAbortedError("a rank timed out mid-collective")
            if self._aborted:
                raise RankAbortedError("world aborted")
            snapshot = list(board["entries"])
            board["read"] += 1
            if board["read"] == self.size:
                del self._boards[seq]
            return snapshot

    def _abort_locked(self):
        self._aborted = True
        self._cond.notify_all()

    def abort(self):
        with self._cond:
            self._abort_locked()


def _device_for_rank(rank):
    torch = _torch()
    if not torch.cuda.is_available():
        return torch.device("cpu")
    return torch.device("cuda", rank % torch.cuda.device_count())


class _InProcCommunicator(Communicator):
    backend = "inproc"

    def __init__(self, world, rank):
        super().__init__()
        self._world = world
        self.rank = rank
        self.size = world.size
        self.device = _device_for_rank(rank)

    def abort(self):
        self._world.abort()

    def _collective(self, op, buf, send=None, counts=None, root=-1, redop=None):
        torch_mode = _is_tensor(buf) or _is_tensor(send)
        # ---- header -------------------------------------------------------
        header = {"op": op, "dtype": -1, "root": root, "send_len": -1, "recv_len": -1,
                  "counts": counts, "redop": -1 if redop is None else _OP_CODE[redop]}
        payload = None
        rflat = None
        wb = False
        if op != "barrier":
            dt = _np_dtype(buf if buf is not None else send)
            header["dtype"] = _DTYPE_CODES[dt]
            if torch_mode:
                rflat, wb = fortran_flat(buf)
                header["recv_len"] = rflat.numel()
            else:
                rflat = _np_flat(buf)
                header["recv_len"] = rflat.size
            if op in ("allgatherv", "reduce_scatterv") or (op == "scatterv" and self.rank == root):
                sflat = (fortran_flat(send)[0] if _is_tensor(send) else _np_flat(send))
                header["send_len"] = int(sflat.numel() if _is_tensor(sflat) else sflat.size)
                payload = sflat
            elif op in ("allreduce",) or (op == "broadcast" and self.rank == root):
                payload = rflat
            if payload is not None:
                if _is_tensor(payload):
                    payload = payload.clone()
                    if payload.is_cuda:
                        _torch().cuda.current_stream(payload.device).synchronize()
                else:
                    payload = np.array(payload, copy=True)
        # ---- exchange -----------------------------------------------------
        self._seq += 1
        header["seq"] = self._seq
        if self.size == 1:
            slots = [(header, payload)]
        else:
            slots = self._world.exchange(self.rank, self._seq, (header, payload))
            if any(entry is None for entry in slots):
                raise CollectiveContractError("ranks invoked different numbers of collectives")
        headers = [h for h, _ in slots]
        _validate_headers(headers)
        if op == "barrier":
            return
        payloads = [p for _, p in slots]
        if torch_mode:
            self._respond_torch(op, headers, payloads, rflat, counts)
            if wb:
                _fortran_writeback(buf, rflat)
            if rflat.is_cuda and self.size > 1:
                _torch().cuda.current_stream(rflat.device).synchronize()
        else:
            out = self._respond_numpy(op, headers, payloads, counts)
            _np_writeback(buf, out)

    # reference semantics on numpy payloads (comm.py:156-175)
    def _respond_numpy(self, op, headers, payloads, counts):
        payloads = [p.cpu().numpy() if _is_tensor(p) else p for p in payloads]
        if op == "broadcast":
            return payloads[headers[0]["root"]]
        if op == "allreduce":
            return _fold_np(payloads, ReduceOp(_op_name(headers[0]["redop"])))
        if op == "allgatherv":
            return np.concatenate([payloads[r] for r in range(self.size)])
        offs = np.concatenate([[0], np.cumsum(counts)]).astype(np.int64)
        if op == "scatterv":
            send = payloads[headers[0]["root"]]
            return send[offs[self.rank]:offs[self.rank + 1]]
        if op == "reduce_scatterv":
            red = _fold_np(payloads, ReduceOp(_op_name(headers[0]["redop"])))
            return red[offs[self.rank]:offs[self.rank + 1]]
        raise CollectiveContractError(f"unknown collective {op!r}")  # pragma: no cover

    def _respond_torch(self, op, headers, payloads, rflat, counts):
        torch = _torch()
        dev = rflat.device

        def local(p):
            if _is_tensor(p):
                return p.to(dev)
            return torch.from_numpy(np.ascontiguousarray(p)).to(dev)

        if op == "broadcast":
            rflat.copy_(local(payloads[headers[0]["root"]]))
            return
        if op == "allgatherv":
            off = 0
            for r in range(self.size):
                if counts[r]:
                    rflat[off:off + counts[r]].copy_(local(payloads[r]))
                off += counts[r]
            return
        offs = np.concatenate([[0], np.cumsum(counts)]).astype(np.int64) if counts else None
        if op == "scatterv":
            src = local(payloads[headers[0]["root"]])
            rflat.copy_(src[offs[self.rank]:offs[self.rank + 1]])
            return
        redop = ReduceOp(_op_name(headers[0]["redop"]))
        srcs = [local(p) for p in payloads]
        if op == "reduce_scatterv":
            srcs = [s[offs[self.rank]:offs[self.rank + 1]] for s in srcs]
        _fold_into(rflat, srcs, redop)


def _op_name(code):
    return {0: "sum", 1: "prod", 2: "max", 3: "min"}[code]


def _fold_np(parts, redop):
    acc = np.array(parts[0], copy=True)
    fn = _REDUCE_UFUNC[redop]
    for part in parts[1:]:
        fn(acc, part, out=acc)
    return acc


def _fold_into(dst, srcs, redop):
    """dst = srcs[0] op srcs[1] op ... (ascending rank), on dst's device."""
    if dst.numel() == 0:
        return
    if dst.is_cuda:
        from . import _lib

        srcs = [s.contiguous() for s in srcs]
        arr = (ctypes.c_void_p * len(srcs))(*[s.data_ptr() for s in srcs])
        _lib.call("bs_fold", _lib.ptr(dst), ctypes.cast(arr, ctypes.c_void_p), len(srcs), dst.numel(),
                  _lib.dtype_code(dst.dtype), _OP_CODE[redop], _lib.stream_ptr())
        return
    acc = srcs[0].clone()
    torch = _torch()
    for s in srcs[1:]:
        if redop is ReduceOp.SUM:
            acc += s
        elif redop is ReduceOp.PROD:
            acc *= s
        elif redop is ReduceOp.MAX:
            acc = torch.maximum(acc, s)
        else:
            acc = torch.minimum(acc, s)
    dst.copy_(acc)


# ---------------------------------------------------------------------------
# torch.distributed backend (one process per rank; NCCL on B200)
# ---------------------------------------------------------------------------


class _TorchCommunicator(Communicator):
    """Collectives over a torch.distributed process group (NCCL or gloo)."""

    def __init__(self, backend_name, rendezvous=None, timeout=30.0):
        """``rendezvous`` = (host, port, rank, size) for the reference's tcp descriptor:
        rank 0 hosts a TCPStore at host:port, the other ranks join it, and the store
        carries NCCL's unique id (the bootstrap the reference's hub socket performed);
        None joins the env:// world (torchrun)."""
        super().__init__()
        torch = _torch()
        import datetime

        import torch.distributed as dist

        self._dist = dist
        if not dist.is_initialized():
            os.environ.setdefault("MASTER_ADDR", "127.0.0.1")
            kw = {}
            if rendezvous is not None:
                host, port, rank, size = rendezvous
                kw.update(init_method=f"tcp://{host}:{port}", rank=rank, world_size=size,
                          timeout=datetime.timedelta(seconds=max(float(timeout), 30.0)))
            if backend_name == "gloo+cuda":
                backend_name = "gloo"
                self._gloo_cuda = True
            if backend_name == "nccl":
                ndev = max(torch.cuda.device_count(), 1)
                local = int(os.environ.get("LOCAL_RANK", str(rendezvous[2] % ndev if rendezvous else 0)))
                torch.cuda.set_device(local)
                kw["device_id"] = torch.device("cuda", local)
            dist.init_process_group(backend=backend_name, **kw)
        elif backend_name == "gloo+cuda":
            self._gloo_cuda = True
        self.rank = dist.get_rank()
        self.size = dist.get_world_size()
        self.backend = dist.get_backend()
        if self.backend == "nccl":
            local = int(os.environ.get("LOCAL_RANK", self.rank % max(torch.cuda.device_count(), 1)))
            self.device = torch.device("cuda", local)
            torch.cuda.set_device(self.device)
            self.coll_device = self.device
        elif getattr(self, "_gloo_cuda", False):
            # data on the GPU (rank mod device count: several ranks may share one GPU), collectives
            # staged through host memory over gloo — the multi-process solver tests on one GPU
            self.device = torch.device("cuda", self.rank % max(torch.cuda.device_count(), 1))
            torch.cuda.set_device(self.device)
            self.coll_device = torch.device("cpu")
        else:
            self.device = torch.device("cpu")
            self.coll_device = self.device
        self._ops = {ReduceOp.SUM: dist.ReduceOp.SUM, ReduceOp.PROD: dist.ReduceOp.PRODUCT,
                     ReduceOp.MAX: dist.ReduceOp.MAX, ReduceOp.MIN: dist.ReduceOp.MIN}

    def close(self):
        if self._dist.is_initialized():
            self._dist.destroy_process_group()

    def _to_dev(self, buf):
        """(flat tensor on the collective device, writeback fn)."""
        torch = _torch()
        if _is_tensor(buf):
            flat, wb = fortran_flat(buf)
            if flat.device != self.coll_device:
                dflat = flat.to(self.coll_device)
                return dflat, (lambda: (_fortran_writeback(buf, dflat.to(buf.device))
                                        if wb else flat.copy_(dflat.to(flat.device))))
            return flat, ((lambda: _fortran_writeback(buf, flat)) if wb else (lambda: None))
        arr = np.asarray(buf)
        flat = torch.from_numpy(np.ascontiguousarray(_np_flat(arr))).to(self.coll_device)
        return flat, (lambda: _np_writeback(buf, flat.cpu().numpy()))

    def _collective(self, op, buf, send=None, counts=None, root=-1, redop=None):
        dist = self._dist
        torch = _torch()
        self._seq += 1
        if op == "barrier":
            dist.barrier()
            return
        rflat, wb = self._to_dev(buf)
        if op == "broadcast":
            dist.broadcast(rflat, src=root)
        elif op == "allreduce":
            dist.all_reduce(rflat, op=self._ops[redop])
        elif op == "allgatherv":
            sflat, _ = self._to_dev(send)
            mx = max(counts) if counts else 0
            if mx:
                pad = torch.zeros(mx, dtype=rflat.dtype, device=self.coll_device)
                pad[:sflat.numel()].copy_(sflat)
                out = torch.empty(mx * self.size, dtype=rflat.dtype, device=self.coll_device)
                dist.all_gather_into_tensor(out, pad)
                off = 0
                for r in range(self.size):
                    if counts[r]:
                        rflat[off:off + counts[r]].copy_(out[r * mx:r * mx + counts[r]])
                    off += counts[r]
        elif op == "reduce_scatterv":
            sflat, _ = self._to_dev(send)
            mx = max(counts) if counts else 0
            if mx:
                padded = torch.zeros(mx * self.size, dtype=rflat.dtype, device=self.coll_device)
                off = 0
                for r in range(self.size):
                    if counts[r]:
                        padded[r * mx:r * mx + counts[r]].copy_(sflat[off:off + counts[r]])
                    off += counts[r]
                out = torch.empty(mx, dtype=rflat.dtype, device=self.coll_device)
                dist.reduce_scatter_tensor(out, padded, op=self._ops[redop])
                rflat.copy_(out[:counts[self.rank]])
        elif op == "scatterv":
            total = sum(counts)
            mx = max(counts) if counts else 0
            full = torch.empty(total, dtype=rflat.dtype, device=self.coll_device)
            if self.rank == root:
                full.copy_(self._to_dev(send)[0])
            dist.broadcast(full, src=root)
            off = sum(counts[:self.rank])
            rflat.copy_(full[off:off + counts[self.rank]])
            del mx
        else:  # pragma: no cover
            raise CollectiveContractError(f"unknown collective {op!r}")
        wb()


# ---------------------------------------------------------------------------
# world construction (comm.py:492-643)
# ---------------------------------------------------------------------------


_TCP_ENTRY = r"([^,]+?):(\d+)(?=,|$)"  # host (IPv6 brackets included) : port
_TCP_RE = re.compile(r"tcp:(?P<hosts>[^,]+?:\d+(?:,[^,]+?:\d+)*),rank=(?P<rank>\d+)")
_TCP_ENTRY_RE = re.compile(_TCP_ENTRY)


def _parse_descriptor(descriptor):
    if descriptor.startswith("inproc:"):
        try:
            size = int(descriptor.split(":", 1)[1])
        except ValueError:
            raise CommInitError(f"bad inproc descriptor {descriptor!r}") from None
        if size < 1:
            raise CommInitError("world size must be >= 1")
        return "inproc", size
    if descriptor in ("nccl", "gloo", "gloo+cuda", "torch"):
        return "torch", descriptor
    if descriptor.startswith("tcp:"):
        # tcp:host:port,...,rank=<r> (comm.py:501-519): one process per rank; here the
        # first entry is the TCPStore that bootstraps NCCL (gloo without a GPU).
        m = _TCP_RE.fullmatch(descriptor)
        if m is None:
            raise CommInitError(f"bad tcp descriptor {descriptor!r}; expected tcp:host:port,...,rank=<r>")
        hosts = [(h, int(pt)) for h, pt in _TCP_ENTRY_RE.findall(m.group("hosts"))]
        rank = int(m.group("rank"))
        if rank >= len(hosts):
            raise CommInitError(f"rank {rank} out of range for {len(hosts)} hosts")
        return "tcp", (hosts, rank)
    raise CommInitError(f"unknown backend descriptor {descriptor!r}")


def init(descriptor, timeout=30.0):
    """Construct communicator endpoint(s) from a backend descriptor.

    ``inproc:<P>`` returns a list of P endpoints sharing one world (one per
    rank thread).  ``nccl`` / ``gloo`` join the torch.distributed world of this
    process (env:// rendezvous, e.g. under torchrun) and return its endpoint.
    ``tcp:host:port,...,rank=<r>`` (the reference's multi-process descriptor)
    rendezvouses at the first host:port and returns this process's endpoint.
    """
    kind, arg = _parse_descriptor(descriptor)
    if kind == "inproc":
        world = _InProcWorld(arg)
        return [_InProcCommunicator(world, r) for r in range(arg)]
    if kind == "tcp":
        hosts, rank = arg
        backend = "nccl" if _torch().cuda.is_available() else "gloo"
        try:
            return _TorchCommunicator(backend, rendezvous=(hosts[0][0], hosts[0][1], rank, len(hosts)),
                                      timeout=timeout)
        except Exception as exc:  # noqa: BLE001
            raise CommInitError(f"tcp rendezvous at {hosts[0][0]}:{hosts[0][1]} failed: {exc}") from exc
    backend = arg
    if backend == "torch":
        backend = "nccl" if _torch().cuda.is_available() else "gloo"
    try:
        return _TorchCommunicator(backend)
    except Exception as exc:  # noqa: BLE001
        raise CommInitError(f"could not join the torch.distributed world: {exc}") from exc


def launch(descriptor, fn, *args, timeout=30.0):
    """Run ``fn(comm, *args)`` on every rank reachable from this process."""
    kind, _ = _parse_descriptor(descriptor)
    if kind == "inproc":
        return _run_threads(init(descriptor), fn, args)
    comm = init(descriptor, timeout=timeout)
    try:
        return [_with_rank_context(comm, fn, args)]
    finally:
        comm.close()


def run_inproc(size, fn, *args):
    """Convenience wrapper: ``launch(f"inproc:{size}", fn, *args)``."""
    return launch(f"inproc:{size}", fn, *args)


def _with_rank_context(comm, fn, args):
    torch = _torch()
    if comm.device is not None and comm.device.type == "cuda":
        torch.cuda.set_device(comm.device)
        if comm.backend == "inproc" and comm.size > 1:
            with torch.cuda.stream(torch.cuda.Stream(comm.device)):
                return fn(comm, *args)
    return fn(comm, *args)


def _run_threads(comms, fn, args):
    """Runs ``fn(comm, *args)`` on one thread per rank; the first failing rank aborts the world.

    The exception re-raised is the root cause: a rank's own error wins over the
    RankAbortedError its failure caused on the others.
    """
    if len(comms) == 1:
        return [_with_rank_context(comms[0], fn, args)]
    import concurrent.futures as cf

    def rank_main(comm):
        try:
            return _with_rank_context(comm, fn, args)
        except BaseException:
            comm.abort()
            raise

    with cf.ThreadPoolExecutor(max_workers=len(comms), thread_name_prefix="rank") as pool:
        futures = [pool.submit(rank_main, c) for c in comms]
        cf.wait(futures)
    for comm in comms:
        comm.close()
    failures = [f.exception() for f in futures if f.exception() is not None]
    if failures:
        root = [e for e in failures if not isinstance(e, RankAbortedError)]
        raise (root or failures)[0]
    return [f.result() for f in futures]
