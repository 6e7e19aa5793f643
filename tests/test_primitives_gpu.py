"""GPU: L1 primitives against numpy / the oracle (rand_fill, distribute/gather, reductions, collectives)."""

import numpy as np
import pytest

import paper_2010_16114_b200 as bs
from oracle import blockstat_oracle as orc

pytestmark = pytest.mark.gpu


@pytest.mark.parametrize("dt", [np.float64, np.float32])
@pytest.mark.parametrize("p", [1, 2, 3])
@pytest.mark.parametrize("shape", [(5, 7), (1, 33), (64, 3), (2, 3, 11)])
def test_rand_fill_matches_numpy_stream(dt, p, shape):
    def fn(comm):
        a = bs.empty(shape, comm, dt)
        bs.rand_fill(a, seed=3, common_init=True)
        return bs.gather_full(a)

    want = orc.rand_fill_common(shape, 3, dt)
    for got in bs.run_inproc(p, fn):
        np.testing.assert_array_equal(got, want)


@pytest.mark.parametrize("dt", [np.float64, np.float32])
def test_rand_fill_per_rank_streams(dt):
    def fn(comm):
        a = bs.empty((4, 9), comm, dt)
        bs.rand_fill(a, seed=10, common_init=False)
        return a.local.cpu().numpy()

    for r, loc in enumerate(bs.run_inproc(3, fn)):
        want = np.random.Generator(np.random.Philox(10 + r)).random(loc.size, dtype=dt)
        np.testing.assert_array_equal(loc, want.reshape(loc.shape, order="F"))


def test_rand_fill_large_offset_block():
    """A block deep inside a long stream (first >> 0) matches numpy."""
    def fn(comm):
        a = bs.empty((1000, 41), comm, np.float32)
        bs.rand_fill(a, seed=99, common_init=True)
        return bs.gather_full(a)

    got = bs.run_inproc(4, fn)[0]
    np.testing.assert_array_equal(got, orc.rand_fill_common((1000, 41), 99, np.float32))


def test_rand_fill_standard_normal_host_stream():
    def fn(comm):
        a = bs.empty((6, 10), comm)
        bs.rand_fill(a, seed=5, common_init=True, dist="standard_normal")
        return bs.gather_full(a)

    for got in bs.run_inproc(3, fn):
        np.testing.assert_array_equal(got, orc.rand_fill_common((6, 10), 5, np.float64, "standard_normal"))


@pytest.mark.parametrize("p", [1, 2, 4, 8])
def test_distribute_gather_roundtrip(p):
    gen = np.random.Generator(np.random.Philox(2000 + p))
    data = [gen.random((3, 17)), gen.random(9), gen.integers(-5, 5, size=(2, 2, 6)).astype(np.int64),
            gen.random((4, 2)).astype(np.float32)]

    def fn(comm):
        return [bs.gather_full(bs.distribute(d if comm.rank == 0 else None, comm)) for d in data]

    for back in bs.run_inproc(p, fn):
        for b, d in zip(back, data):
            np.testing.assert_array_equal(b, d)


@pytest.mark.parametrize("p", [1, 3])
def test_reduce_all_ops(p):
    gen = np.random.Generator(np.random.Philox(77))
    d = gen.standard_normal((5, 11))

    def fn(comm):
        a = bs.distribute(d if comm.rank == 0 else None, comm)
        return (bs.reduce_all(a), bs.reduce_all(a, bs.ReduceOp.MIN), bs.reduce_all(a, bs.ReduceOp.MAX),
                bs.reduce_all(a, transform=np.abs), bs.reduce_all(a, bs.ReduceOp.MAX, transform=np.abs))

    s, mn, mx, l1, linf = bs.run_inproc(p, fn)[0]
    assert abs(s - d.sum()) <= 1e-12 * np.abs(d).sum()
    assert mn == d.min() and mx == d.max() and linf == np.abs(d).max()
    assert abs(l1 - np.abs(d).sum()) <= 1e-12 * l1


@pytest.mark.parametrize("p", [2, 3, 4])
def test_device_collectives_fold_in_rank_order(p):
    import torch

    def fn(comm):
        dev = comm.device
        x = torch.full((5,), float(comm.rank + 1), dtype=torch.float64, device=dev)
        comm.allreduce(x, bs.ReduceOp.SUM)
        counts = [r + 1 for r in range(comm.size)]
        send = torch.full((comm.rank + 1,), float(comm.rank), dtype=torch.float64, device=dev)
        recv = torch.empty(sum(counts), dtype=torch.float64, device=dev)
        comm.allgatherv(send, recv, counts)
        full = torch.arange(sum(counts), dtype=torch.float64, device=dev)
        part = torch.empty(counts[comm.rank], dtype=torch.float64, device=dev)
        comm.reduce_scatterv(full, part, counts)
        return x.cpu().numpy(), recv.cpu().numpy(), part.cpu().numpy()

    res = bs.run_inproc(p, fn)
    counts = [r + 1 for r in range(p)]
    offs = np.cumsum([0] + counts)
    for r, (x, recv, part) in enumerate(res):
        np.testing.assert_array_equal(x, np.full(5, p * (p + 1) / 2))
        np.testing.assert_array_equal(recv, np.concatenate([np.full(c, float(q)) for q, c in enumerate(counts)]))
        np.testing.assert_array_equal(part, p * np.arange(offs[r], offs[r + 1], dtype=np.float64))


def test_contract_violation_raises_everywhere():
    import torch

    def fn(comm):
        x = torch.zeros(3 + comm.rank, dtype=torch.float64, device=comm.device)
        comm.allreduce(x)

    with pytest.raises(bs.CollectiveContractError):
        bs.run_inproc(2, fn)


def test_pairwise_euclidean_matches_oracle():
    gen = np.random.Generator(np.random.Philox(8))
    x = gen.random((7, 53))

    def fn(comm):
        xd = bs.distribute(x if comm.rank == 0 else None, comm)
        y = bs.empty((53, 53), comm)
        bs.pairwise_euclidean(y, xd)
        return bs.gather_full(y)

    want = orc.pairwise_euclidean(x)
    for p in (1, 3):
        got = bs.run_inproc(p, fn)[0]
        np.testing.assert_allclose(got, want, rtol=1e-13, atol=1e-15)
        np.testing.assert_array_equal(got, got.T)
        assert np.all(np.diag(got) == 0)


@pytest.mark.parametrize("p", [1, 3])
def test_opnorm_power_matches_reference(golden, p):
    a = golden["opnorm_a"]

    def fn(comm):
        return bs.opnorm(bs.distribute(a if comm.rank == 0 else None, comm))

    got = bs.run_inproc(p, fn)[0]
    assert abs(got - golden["opnorm_l2"][0]) <= 1e-12 * got
    sv = np.linalg.svd(a, compute_uv=False)[0]
    assert abs(got - sv) <= 1e-5 * sv


@pytest.mark.parametrize("p", [1, 3])
def test_genotype_fill_matches_oracle_and_is_rank_independent(p):
    """Counter-based genotypes (the C5 input): every element depends only on (seed, i, j)."""
    m, n, seed = 37, 23, 77

    def fn(comm):
        x = bs.empty((m, n), comm, np.int8)
        bs.genotype_fill(x, seed)
        return bs.gather_full(x)

    want = orc.genotype_fill(m, n, seed)
    for got in bs.run_inproc(p, fn):
        np.testing.assert_array_equal(got, want)
    assert set(np.unique(want)) <= {0, 1, 2}


def test_genotype_fill_frequencies():
    m, n = 20000, 40

    def fn(comm):
        x = bs.empty((m, n), comm, np.int8)
        bs.genotype_fill(x, 5, maf_range=(0.1, 0.4))
        return bs.gather_full(x)

    x = bs.run_inproc(1, fn)[0].astype(np.float64)
    p = 0.1 + 0.3 * np.random.Generator(np.random.Philox(6)).random(n)
    np.testing.assert_allclose(x.mean(axis=0), 2 * p, atol=0.03)   # Bin(2, p) means


@pytest.mark.parametrize("dt", [np.float32, np.float64])
def test_normal_fill_is_rank_count_independent_and_normal(dt):
    """normal_fill (bs_philox_normal): Box-Muller on Philox words keyed by the global index."""

    def fn(comm):
        a = bs.empty((333, 201), comm, dt)
        bs.normal_fill(a, 77)
        return bs.gather_full(a)

    ref = bs.run_inproc(1, fn)[0]
    for p in (2, 3):
        np.testing.assert_array_equal(bs.run_inproc(p, fn)[0], ref)
    # host restatement (oracle.philox_normal): Box-Muller on Philox block (e // 2 + 1, 1, 0, 0)
    from oracle import blockstat_oracle as orc

    flat = ref.ravel(order="F")
    for e in (0, 1, 2, 12345, flat.size - 1):
        z = orc.philox_normal(77, e, 1)[0]
        assert abs(float(flat[e]) - z) <= (1e-6 if dt == np.float32 else 1e-12) * max(1.0, abs(z))
    assert abs(flat.mean()) < 0.02 and abs(flat.std() - 1.0) < 0.02


@pytest.mark.parametrize("p", [1, 3])
def test_transposed_view_is_a_lazy_row_split_transpose(p):
    """transpose / TransposedView (distarray.py:111-136): shape swapped, the parent's partition
    (rows of the view), no copy, and transposing twice gives the parent back."""
    x = np.arange(7 * 11, dtype=np.float64).reshape((7, 11), order="F")

    def fn(comm):
        a = bs.distribute(x if comm.rank == 0 else None, comm)
        t = bs.transpose(a)
        assert isinstance(t, bs.TransposedView)
        assert t.shape == (11, 7) and t.dtype == a.dtype and t.comm is comm
        assert t.partition.counts() == a.partition.counts()  # the view's rows = the parent's columns
        assert bs.transpose(t) is a
        with pytest.raises(TypeError):
            bs.transpose(np.zeros((2, 2)))
        # the rank's rows of the view are its columns of the parent, no copy
        return a.local.data_ptr(), t.parent.local.data_ptr(), bs.gather_full(t.parent)

    for ptr_a, ptr_t, full in bs.run_inproc(p, fn):
        assert ptr_a == ptr_t
        np.testing.assert_array_equal(full, x)
