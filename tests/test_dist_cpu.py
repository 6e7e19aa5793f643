"""CPU (gloo, world_size 2): the torch.distributed Communicator's padded v-collectives and host-side helpers.

The multi-GPU path runs one process per GPU with NCCL; the same Communicator code
runs here over gloo on CPU tensors, so the padding / slicing logic of
allgatherv, reduce_scatterv and scatterv is exercised without a GPU.
"""

import os
import socket

import numpy as np
import pytest
import torch
import torch.multiprocessing as mp

import paper_2010_16114_b200 as bs
from paper_2010_16114_b200.comm import fortran_flat
from paper_2010_16114_b200.distarray import fortran_empty, partition_of


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _worker(rank, world, port, q):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port), RANK=str(rank), WORLD_SIZE=str(world))
    try:
        comm = bs.init("gloo")
        out = {}
        # allgatherv with uneven counts (partition_of semantics)
        counts = list(partition_of(7, world).counts())
        send = torch.arange(counts[rank], dtype=torch.float64) + 10 * rank
        recv = torch.empty(sum(counts), dtype=torch.float64)
        comm.allgatherv(send, recv, counts)
        out["allgatherv"] = recv.numpy().tolist()
        # reduce_scatterv: every rank contributes arange(total) * (rank + 1)
        full = torch.arange(sum(counts), dtype=torch.float64) * (rank + 1)
        part = torch.empty(counts[rank], dtype=torch.float64)
        comm.reduce_scatterv(full, part, counts)
        out["reduce_scatterv"] = part.numpy().tolist()
        # allreduce MIN / SUM on a column-major (Fortran-strided) tensor
        t = fortran_empty((3, 2), torch.float64, "cpu")
        t.copy_(torch.tensor([[1.0, 2.0], [3.0, 4.0], [5.0, 6.0]]) * (rank + 1))
        comm.allreduce(t, bs.ReduceOp.SUM)
        out["allreduce"] = t.numpy().tolist()
        # numpy buffers travel too (host-side values of the reference API)
        a = np.array([float(rank)])
        comm.allreduce(a, bs.ReduceOp.MAX)
        out["np_max"] = a.tolist()
        # scatterv from root 1
        counts2 = [2, 3]
        src = torch.arange(5, dtype=torch.float64) if rank == 1 else None
        dst = torch.empty(counts2[rank], dtype=torch.float64)
        comm.scatterv(src, dst, counts2, root=1)
        out["scatterv"] = dst.numpy().tolist()
        comm.barrier()
        q.put((rank, out))
    except Exception as exc:  # pragma: no cover - surfaced by the parent
        q.put((rank, repr(exc)))
    finally:
        import torch.distributed as dist

        if dist.is_initialized():
            dist.destroy_process_group()


def test_gloo_world2_collectives():
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, 2, port, q)) for r in range(2)]
    for p in procs:
        p.start()
    res = dict(q.get(timeout=120) for _ in procs)
    for p in procs:
        p.join(timeout=60)
    for r in range(2):
        assert isinstance(res[r], dict), res[r]
    counts = [4, 3]
    want_ag = [0.0, 1.0, 2.0, 3.0, 10.0, 11.0, 12.0]
    for r in range(2):
        out = res[r]
        assert out["allgatherv"] == want_ag
        lo = sum(counts[:r])
        assert out["reduce_scatterv"] == [3.0 * i for i in range(lo, lo + counts[r])]
        assert out["allreduce"] == [[3.0, 6.0], [9.0, 12.0], [15.0, 18.0]]
        assert out["np_max"] == [1.0]
    assert res[0]["scatterv"] == [0.0, 1.0] and res[1]["scatterv"] == [2.0, 3.0, 4.0]


def test_partition_and_fortran_views():
    assert partition_of(7, 4).counts() == (2, 2, 2, 1)
    assert partition_of(2, 4).counts() == (1, 1, 0, 0)
    with pytest.raises(ValueError):
        partition_of(-1, 2)
    t = fortran_empty((3, 5), torch.float32, "cpu")
    flat, wb = fortran_flat(t)
    assert not wb and flat.data_ptr() == t.data_ptr() and flat.numel() == 15


def test_inproc_numpy_collectives_and_contract_cpu():
    """The in-process backend's host (numpy) path runs without a GPU."""

    def fn(comm):
        a = np.array([1.0, 2.0]) * (comm.rank + 1)
        comm.allreduce(a)
        recv = np.empty(3)
        comm.allgatherv(np.arange(comm.rank + 1, dtype=np.float64), recv, [1, 2])
        return a.tolist(), recv.tolist()

    res = bs.run_inproc(2, fn)
    assert res[0] == ([3.0, 6.0], [0.0, 0.0, 1.0])

    def bad(comm):
        comm.allreduce(np.zeros(2 + comm.rank))

    with pytest.raises(bs.CollectiveContractError):
        bs.run_inproc(2, bad)


def test_abi_library_exports_every_header_symbol():
    from paper_2010_16114_b200 import _lib

    lib = _lib.load()
    syms = _lib.header_symbols()
    assert len(syms) >= 30
    for name in syms:
        assert hasattr(lib, name), name
    assert set(syms) == set(_lib.SIGNATURES)
    assert lib.bs_abi_version() == 1


def _tcp_worker(rank, port, q):
    """One rank of the reference's multi-process descriptor (comm.py:12-15)."""
    try:
        desc = f"tcp:127.0.0.1:{port},127.0.0.1:{port + 1},rank={rank}"

        def fn(comm):
            a = np.array([1.0, 2.0]) * (comm.rank + 1)
            comm.allreduce(a)
            recv = torch.empty(3, dtype=torch.float64)
            comm.allgatherv(torch.arange(2 - comm.rank, dtype=torch.float64) + 10 * comm.rank, recv, [2, 1])
            return comm.rank, comm.size, a.tolist(), recv.tolist()

        q.put((rank, bs.launch(desc, fn)))
    except Exception as exc:  # pragma: no cover - surfaced by the parent
        q.put((rank, repr(exc)))


def test_tcp_descriptor_world2():
    """tcp:host:port,...,rank=<r> rendezvouses at the first entry and runs the collectives
    (NCCL on a GPU box, gloo here); launch returns the local rank's result only."""
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_tcp_worker, args=(r, port, q)) for r in range(2)]
    for p in procs:
        p.start()
    res = dict(q.get(timeout=120) for _ in procs)
    for p in procs:
        p.join(timeout=60)
    for r in range(2):
        assert isinstance(res[r], list) and len(res[r]) == 1, res[r]
        rank, size, a, ag = res[r][0]
        assert (rank, size) == (r, 2)
        assert a == [3.0, 6.0]
        assert ag == [0.0, 1.0, 10.0]


def test_tcp_descriptor_validation():
    for bad in ("tcp:", "tcp:127.0.0.1:1", "tcp:127.0.0.1:x,rank=0", "tcp:127.0.0.1:1,rank=3", "bogus"):
        with pytest.raises(bs.CommInitError):
            bs.init(bad)


@pytest.mark.parametrize("dtype", [np.float32, np.float64])
def test_standard_normal_chunked_stream_cpu(monkeypatch, dtype):
    """standard_normal is drawn on the host in bounded chunks and scattered chunk by chunk;
    the content equals one numpy call (chunk-invariant stream), for any rank count."""
    from oracle import blockstat_oracle as orc
    from paper_2010_16114_b200 import distarray as bda

    monkeypatch.setattr(bda, "_NORMAL_CHUNK", 7)
    shape = (5, 11)
    want = orc.rand_fill_common(shape, 21, dtype, "standard_normal")

    def fn(comm):
        a = bs.empty(shape, comm, dtype)
        bs.rand_fill(a, seed=21, common_init=True, dist="standard_normal")
        b = bs.empty(shape, comm, dtype)
        bs.rand_fill(b, seed=30, dist="standard_normal")  # per-rank stream seed + rank
        return bs.gather_full(a), b.lo, fortran_flat(b.local)[0].cpu().numpy()

    for p in (1, 3, 4):
        for rank, (full, lo, blk) in enumerate(bs.run_inproc(p, fn)):
            np.testing.assert_array_equal(full, want)
            own = np.random.Generator(np.random.Philox(30 + rank)).standard_normal(blk.size, dtype=dtype)
            np.testing.assert_array_equal(blk, own)
