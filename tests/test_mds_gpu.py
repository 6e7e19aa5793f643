"""GPU: MDS (solvers.py:209-305) against the reference's golden vectors and the oracle."""

import numpy as np
import pytest

import paper_2010_16114_b200 as bs
from oracle import blockstat_oracle as orc

pytestmark = pytest.mark.gpu


def _run(comm, y, th0, iters, perturb=False, trace_every=1):
    yd = bs.distribute(y if comm.rank == 0 else None, comm)
    st = bs.mds_init(yd, th0.shape[0], seed=1, perturb=perturb)
    st.theta.local[...] = bs.distribute(th0 if comm.rank == 0 else None, comm).local
    bs.mds_fit(st, iters, trace_every=trace_every)
    return np.asarray(st.trace), bs.gather_full(st.theta)


@pytest.mark.parametrize("name", ["d5_n12_q2", "d8_n40_q3", "d6_n30_q2_f32"])
@pytest.mark.parametrize("p", [1, 2, 3])
def test_mds_matches_reference_golden(golden, name, p):
    d, n, q, seed, iters, _ = golden[f"mds_{name}_meta"]
    y = golden[f"mds_{name}_y"]
    tr, th = bs.run_inproc(p, _run, y, golden[f"mds_{name}_theta0"], int(iters))[0]
    tol = 1e-9 if y.dtype == np.float64 else 1e-4
    np.testing.assert_allclose(tr, golden[f"mds_{name}_trace"], rtol=tol)
    np.testing.assert_allclose(th, golden[f"mds_{name}_theta"], rtol=tol, atol=tol)


def test_mds_pipeline_from_points_matches_reference(golden):
    """rand_fill -> pairwise_euclidean -> mds_init -> mds_fit through the public API."""
    name = "d8_n40_q3"
    d, n, q, seed, iters, _ = (int(v) for v in golden[f"mds_{name}_meta"])

    def fn(comm):
        x = bs.empty((d, n), comm)
        bs.rand_fill(x, seed=seed, common_init=True)
        y = bs.empty((n, n), comm)
        bs.pairwise_euclidean(y, x)
        st = bs.mds_init(y, q, seed=seed + 1)
        th0 = bs.gather_full(st.theta)
        bs.mds_fit(st, iters)
        return bs.gather_full(y), th0, np.asarray(st.trace), bs.gather_full(st.theta)

    for p in (1, 4):
        y, th0, tr, th = bs.run_inproc(p, fn)[0]
        np.testing.assert_allclose(y, golden[f"mds_{name}_y"], rtol=1e-13, atol=1e-14)
        np.testing.assert_array_equal(th0, golden[f"mds_{name}_theta0"])
        np.testing.assert_allclose(tr, golden[f"mds_{name}_trace"], rtol=1e-9)
        np.testing.assert_allclose(th, golden[f"mds_{name}_theta"], rtol=1e-9, atol=1e-12)


@pytest.mark.parametrize("n,q,p", [(200, 2, 1), (333, 20, 3), (257, 5, 2), (128, 30, 1), (96, 40, 2)])
def test_mds_matches_oracle(n, q, p):
    x = orc.rand_fill_common((10, n), 50 + q, np.float64)
    y = orc.pairwise_euclidean(x)
    th0 = orc.mds_init(y, q, 60 + q)
    tr, th = bs.run_inproc(p, _run, y, th0, 12)[0]
    oth, otr = orc.mds_fit(y, th0, 12)
    np.testing.assert_allclose(tr, otr, rtol=1e-10)
    np.testing.assert_allclose(th, oth, rtol=1e-9, atol=1e-12)


def test_mds_f32_matches_oracle():
    x = orc.rand_fill_common((10, 400), 71, np.float32)
    y = orc.pairwise_euclidean(x)
    th0 = orc.mds_init(y, 20, 72)
    tr, th = bs.run_inproc(1, _run, y, th0, 10)[0]
    oth, otr = orc.mds_fit(y.astype(np.float64), th0.astype(np.float64), 10)
    np.testing.assert_allclose(tr, otr, rtol=1e-4)
    assert np.abs(th - oth).max() <= 1e-4 * np.abs(oth).max()


@pytest.mark.parametrize("n,q,p", [(400, 20, 1), (1000, 20, 3), (516, 8, 2), (300, 30, 1), (260, 3, 2), (200, 32, 1),
                                   (772, 17, 4)])
def test_mds_f32_tensor_core_pass_matches_oracle(n, q, p):
    """float32 with n % 4 == 0 and n >= 64 takes the tcgen05 pass (mds_tc.cu): 3xTF32 Gram and
    T products, ragged 64-row chunk tails, uneven column blocks and ranks with lo > 0."""
    x = orc.rand_fill_common((12, n), 80 + q, np.float32)
    y = orc.pairwise_euclidean(x)
    th0 = orc.mds_init(y, q, 90 + q)
    tr, th = bs.run_inproc(p, _run, y, th0, 6)[0]
    oth, otr = orc.mds_fit(y.astype(np.float64), th0.astype(np.float64), 6)
    np.testing.assert_allclose(tr, otr, rtol=2e-5)
    assert np.abs(th - oth).max() <= 2e-5 * np.abs(oth).max()


@pytest.mark.parametrize("scale", [0.05, 1.0, 30.0, 100.0])
def test_mds_f32_tensor_core_gram_split_ranges(scale):
    """MMA1 (the Gram product) runs on an f16 hi/lo split when 1 <= max |theta|^2 < 2^14 and on
    3xTF32 otherwise (mds_tc.cu f16_range): scales 0.05 and 100 take tf32, 1 and 30 f16.  MDS is
    scale-equivariant, so every case must match the oracle at the same relative tolerance."""
    n, q = 516, 20
    x = orc.rand_fill_common((12, n), 180, np.float32)
    y = (orc.pairwise_euclidean(x) * scale).astype(np.float32)
    th0 = (orc.mds_init(y, q, 190) * scale).astype(np.float32)
    tr, th = bs.run_inproc(2, _run, y, th0, 6)[0]
    oth, otr = orc.mds_fit(y.astype(np.float64), th0.astype(np.float64), 6)
    np.testing.assert_allclose(tr, otr, rtol=2e-5)
    assert np.abs(th - oth).max() <= 2e-5 * np.abs(oth).max()


def test_mds_f32_tensor_core_coincident_points():
    """Exactly coincident embedding points give d = 0 exactly on the tcgen05 path too
    (cancellation guard): the reference raises, or perturbs d to 1e-10 (solvers.py:290-296)."""
    n, q = 128, 4
    x = orc.rand_fill_common((6, n), 5, np.float32)
    y = orc.pairwise_euclidean(x)
    th0 = orc.mds_init(y, q, 6).astype(np.float32)
    th0[:, 77] = th0[:, 3]
    with pytest.raises(bs.DegenerateConfigError):
        bs.run_inproc(2, _run, y, th0, 1, False)
    for tr, th in bs.run_inproc(2, _run, y, th0, 2, True):
        assert np.all(np.isfinite(tr))
    tr1, _ = bs.run_inproc(1, _run, y, th0, 1, True)[0]
    np.testing.assert_allclose(tr1[0], orc.mds_stress(th0.astype(np.float64), y.astype(np.float64)), rtol=1e-5)


def test_mds_stress_examples_and_bruteforce():
    def fn(comm):
        theta = bs.distribute(np.array([[0.0, 1.0]]) if comm.rank == 0 else None, comm)
        y = bs.distribute(np.array([[0.0, 2.0], [2.0, 0.0]]) if comm.rank == 0 else None, comm)
        y_exact = bs.distribute(np.array([[0.0, 1.0], [1.0, 0.0]]) if comm.rank == 0 else None, comm)
        return bs.mds_stress(theta, y), bs.mds_stress(theta, y_exact)

    for two, exact in bs.run_inproc(2, fn):
        assert two == pytest.approx(2.0) and exact == 0.0

    gen = np.random.Generator(np.random.Philox(41))
    theta_d = gen.standard_normal((2, 6))
    y_d = np.abs(gen.standard_normal((6, 6)))
    y_d = (y_d + y_d.T) / 2
    np.fill_diagonal(y_d, 0.0)
    want = sum((y_d[i, j] - np.linalg.norm(theta_d[:, i] - theta_d[:, j])) ** 2
               for i in range(6) for j in range(6) if i != j)

    def fn2(comm):
        return bs.mds_stress(bs.distribute(theta_d if comm.rank == 0 else None, comm),
                             bs.distribute(y_d if comm.rank == 0 else None, comm))

    for p in (1, 2):
        for got in bs.run_inproc(p, fn2):
            assert abs(got - want) <= 1e-12 * max(1.0, want)


def test_mds_345_triangle_is_bitwise_fixed_point():
    pts = np.array([[0.0, 3.0, 3.0], [0.0, 0.0, 4.0]])
    y_d = np.array([[0.0, 3.0, 5.0], [3.0, 0.0, 4.0], [5.0, 4.0, 0.0]])
    for p in (1, 2, 3):
        tr, th = bs.run_inproc(p, _run, y_d, pts, 5)[0]
        np.testing.assert_array_equal(th, pts)
        assert list(tr) == [0.0] * 5


def test_mds_coincident_points_raise_or_perturb():
    y_d = np.array([[0.0, 1.0], [1.0, 0.0]])
    coincident = np.array([[0.5, 0.5]])
    with pytest.raises(bs.DegenerateConfigError):
        bs.run_inproc(2, _run, y_d, coincident, 1, False)
    for tr, th in bs.run_inproc(2, _run, y_d, coincident, 3, True):
        assert np.all(np.isfinite(tr))


def test_mds_degenerate_keeps_trace_and_theta():
    """The raise happens after the entering stress is traced and before theta moves."""
    y_d = np.array([[0.0, 1.0, 2.0], [1.0, 0.0, 1.0], [2.0, 1.0, 0.0]])
    th0 = np.array([[0.2, 0.2, 0.9]])

    def fn(comm):
        yd = bs.distribute(y_d if comm.rank == 0 else None, comm)
        st = bs.mds_init(yd, 1, seed=1)
        st.theta.local[...] = bs.distribute(th0 if comm.rank == 0 else None, comm).local
        try:
            bs.mds_fit(st, 4)
        except bs.DegenerateConfigError:
            return list(st.trace), bs.gather_full(st.theta)
        return None

    tr, th = bs.run_inproc(1, fn)[0]
    _, otr = orc.mds_fit(y_d, th0, 0)
    assert len(tr) == 1
    np.testing.assert_allclose(tr[0], orc.mds_stress(th0, y_d), rtol=1e-14)
    np.testing.assert_array_equal(th, th0)


def test_mds_descent_and_p_independence():
    traces = {}
    for p in (1, 2, 4):
        def fn(comm):
            x = bs.empty((5, 12), comm)
            bs.rand_fill(x, seed=6000, common_init=True)
            y = bs.empty((12, 12), comm)
            bs.pairwise_euclidean(y, x)
            st = bs.mds_init(y, 2, seed=6001)
            bs.mds_fit(st, 200)
            return np.asarray(st.trace)

        traces[p] = bs.run_inproc(p, fn)[0]
        assert np.all(np.diff(traces[p]) <= 1e-10)
    for p in (2, 4):
        np.testing.assert_allclose(traces[p], traces[1], rtol=1e-10)


def test_mds_init_rejects_bad_targets():
    def nonsquare(comm):
        bs.mds_init(bs.zeros((3, 4), comm), 2)

    def diag(comm):
        bs.mds_init(bs.distribute(np.eye(3) if comm.rank == 0 else None, comm), 2)

    for fn in (nonsquare, diag):
        with pytest.raises(ValueError):
            bs.run_inproc(2, fn)
