"""GPU: NMF (solvers.py:97-185) against the reference's golden vectors and the oracle."""

import numpy as np
import pytest

import paper_2010_16114_b200 as bs
from oracle import blockstat_oracle as orc

pytestmark = pytest.mark.gpu

NMF_CASES = ["mu_16x16_r2", "apg_16x16_r4", "mu_60x44_r6", "apg_60x44_r6", "mu_50x30_r5_f32", "apg_50x30_r5_f32"]


def _run(comm, x, vt0, w0, iters, algo, eps=1e-10, trace_every=1):
    xd = bs.distribute(x if comm.rank == 0 else None, comm)
    st = bs.nmf_init(xd, vt0.shape[0], seed=1, eps=eps)
    st.Vt.local[...] = bs.distribute(vt0 if comm.rank == 0 else None, comm).local
    st.W.local[...] = bs.distribute(w0 if comm.rank == 0 else None, comm).local
    (bs.nmf_multiplicative if algo == 0 else bs.nmf_apg)(st, iters, trace_every=trace_every)
    return np.asarray(st.trace), bs.gather_full(st.Vt), bs.gather_full(st.W)


@pytest.mark.parametrize("name", NMF_CASES)
@pytest.mark.parametrize("p", [1, 2, 3])
def test_nmf_matches_reference_golden(golden, name, p):
    m, n, r, seed, iters, algo, _ = golden[f"nmf_{name}_meta"]
    x = golden[f"nmf_{name}_x"]
    tr, vt, w = bs.run_inproc(p, _run, x, golden[f"nmf_{name}_vt0"], golden[f"nmf_{name}_w0"], int(iters), algo)[0]
    tol = 1e-9 if x.dtype == np.float64 else 1e-5
    np.testing.assert_allclose(tr, golden[f"nmf_{name}_trace"], rtol=tol)
    np.testing.assert_allclose(vt, golden[f"nmf_{name}_vt"], rtol=tol * 10, atol=tol)
    np.testing.assert_allclose(w, golden[f"nmf_{name}_w"], rtol=tol * 10, atol=tol)


@pytest.mark.parametrize("p", [1, 2, 4])
def test_nmf_init_draws_reference_factors(golden, p):
    name = "apg_60x44_r6"
    m, n, r, seed, iters, algo, _ = golden[f"nmf_{name}_meta"]

    def fn(comm):
        x = bs.empty((int(m), int(n)), comm)
        bs.rand_fill(x, seed=int(seed), common_init=True)
        st = bs.nmf_init(x, int(r), seed=int(seed) + 1)
        return bs.gather_full(x), bs.gather_full(st.Vt), bs.gather_full(st.W)

    x, vt, w = bs.run_inproc(p, fn)[0]
    np.testing.assert_array_equal(x, golden[f"nmf_{name}_x"])
    np.testing.assert_array_equal(vt, golden[f"nmf_{name}_vt0"])
    np.testing.assert_array_equal(w, golden[f"nmf_{name}_w0"])


@pytest.mark.parametrize("algo", [0, 1])
@pytest.mark.parametrize("shape,r,p", [((300, 200), 20, 1), ((257, 131), 7, 3), ((129, 380), 33, 2),
                                       ((512, 64), 60, 1), ((40, 700), 64, 4), ((90, 75), 100, 1)])
def test_nmf_matches_oracle_f64(algo, shape, r, p):
    m, n = shape
    x = orc.rand_fill_common(shape, 400 + r, np.float64)
    vt0, w0 = orc.nmf_init(x, r, 500 + r)
    iters = 25
    tr, vt, w = bs.run_inproc(p, _run, x, vt0, w0, iters, algo)[0]
    fn = orc.nmf_multiplicative if algo == 0 else orc.nmf_apg
    ovt, ow, otr = fn(x, vt0, w0, iters)
    np.testing.assert_allclose(tr, otr, rtol=1e-9)
    np.testing.assert_allclose(vt, ovt, rtol=1e-7, atol=1e-10)
    np.testing.assert_allclose(w, ow, rtol=1e-7, atol=1e-10)


@pytest.mark.parametrize("algo", [0, 1])
@pytest.mark.parametrize("shape,r", [((700, 600), 20, ), ((1000, 300), 60), ((333, 517), 13)])
def test_nmf_matches_oracle_f32(algo, shape, r):
    """float32 storage: the oracle runs the same float32 inputs in float64 arithmetic; 1e-4 relative."""
    x = orc.rand_fill_common(shape, 600 + r, np.float32)
    vt0, w0 = orc.nmf_init(x, r, 700 + r)
    iters = 20
    tr, vt, w = bs.run_inproc(1, _run, x, vt0, w0, iters, algo)[0]
    fn = orc.nmf_multiplicative if algo == 0 else orc.nmf_apg
    ovt, ow, otr = fn(x.astype(np.float64), vt0.astype(np.float64), w0.astype(np.float64), iters)
    np.testing.assert_allclose(tr, otr, rtol=1e-4)
    scale_v, scale_w = np.abs(ovt).max(), np.abs(ow).max()
    assert np.abs(vt - ovt).max() <= 1e-4 * scale_v
    assert np.abs(w - ow).max() <= 1e-4 * scale_w


def test_nmf_trace_every_and_objective_api():
    x = orc.rand_fill_common((64, 48), 9, np.float64)
    vt0, w0 = orc.nmf_init(x, 5, 10)

    def fn(comm):
        tr, vt, w = _run(comm, x, vt0, w0, 9, 1, trace_every=4)
        xd = bs.distribute(x if comm.rank == 0 else None, comm)
        v = bs.distribute(vt if comm.rank == 0 else None, comm)
        ww = bs.distribute(w if comm.rank == 0 else None, comm)
        return tr, bs.nmf_objective(xd, v, ww), vt, w

    tr, obj, vt, w = bs.run_inproc(2, fn)[0]
    ovt, ow, otr = orc.nmf_apg(x, vt0, w0, 9, trace_every=4)
    assert len(tr) == 3
    np.testing.assert_allclose(tr, otr, rtol=1e-10)
    assert abs(obj - orc.nmf_objective(x, vt, w)) <= 1e-12 * obj


def test_nmf_objective_examples():
    def fn(comm):
        vt = bs.distribute(np.array([[1.0, 2.0], [0.5, 1.0]]) if comm.rank == 0 else None, comm)
        w = bs.distribute(np.array([[1.0, 0.0], [2.0, 1.0]]) if comm.rank == 0 else None, comm)
        prod = bs.gather_full(vt).T @ bs.gather_full(w)
        x_exact = bs.distribute(prod if comm.rank == 0 else None, comm)
        eye = bs.distribute(np.eye(2) if comm.rank == 0 else None, comm)
        return bs.nmf_objective(x_exact, vt, w), bs.nmf_objective(eye, bs.zeros((2, 2), comm), bs.zeros((2, 2), comm))

    for exact, against_zero in bs.run_inproc(2, fn):
        assert exact == 0.0 and against_zero == 2.0


def test_nmf_zero_data_fixed_point():
    def fn(comm):
        st = bs.nmf_init(bs.zeros((3, 3), comm), 2, seed=5)
        bs.nmf_multiplicative(st, 1)
        return st.trace[-1], bs.gather_full(st.Vt), bs.gather_full(st.W)

    for obj, vt, w in bs.run_inproc(2, fn):
        assert obj == 0.0
        np.testing.assert_array_equal(vt, np.zeros((2, 3)))
        np.testing.assert_array_equal(w, np.zeros((2, 3)))


def test_nmf_apg_exact_factorization_is_bitwise_fixed():
    gen = np.random.Generator(np.random.Philox(33))
    vt_d = gen.integers(1, 4, size=(2, 5)).astype(np.float64)
    w_d = gen.integers(1, 4, size=(2, 6)).astype(np.float64)
    x_d = vt_d.T @ w_d
    for p in (1, 2):
        tr, vt, w = bs.run_inproc(p, _run, x_d, vt_d, w_d, 3, 1)[0]
        np.testing.assert_array_equal(vt, vt_d)
        np.testing.assert_array_equal(w, w_d)
        assert list(tr) == [0.0, 0.0, 0.0]


def test_nmf_rejects_negative_data():
    def fn(comm):
        bs.nmf_init(bs.distribute(np.array([[1.0, -0.5], [0.0, 2.0]]) if comm.rank == 0 else None, comm), 1)

    with pytest.raises(ValueError):
        bs.run_inproc(2, fn)


def test_nmf_check_runs_every_call():
    """_nmf_check (solvers.py:147): data made negative after init is caught on the next call."""
    def fn(comm):
        x = bs.empty((8, 8), comm)
        bs.rand_fill(x, seed=4, common_init=True)
        st = bs.nmf_init(x, 2, seed=5)
        bs.nmf_apg(st, 2)
        if comm.rank == 0:
            x.local[0, 0] = -1.0
        bs.nmf_apg(st, 1)

    with pytest.raises(ValueError):
        bs.run_inproc(2, fn)


@pytest.mark.parametrize("algo", [0, 1])
def test_nmf_descent_nonnegativity_and_p_independence(algo):
    traces = {}
    for p in (1, 2, 4):
        def fn(comm):
            x = bs.empty((16, 16), comm)
            bs.rand_fill(x, seed=5000, common_init=True)
            st = bs.nmf_init(x, 4, seed=5001)
            (bs.nmf_multiplicative if algo == 0 else bs.nmf_apg)(st, 200)
            nonneg = bool((bs.gather_full(st.Vt) >= 0).all() and (bs.gather_full(st.W) >= 0).all())
            return np.asarray(st.trace), nonneg

        tr, nonneg = bs.run_inproc(p, fn)[0]
        assert nonneg and len(tr) == 200
        assert np.all(np.diff(tr) <= 1e-10)
        traces[p] = tr
    for p in (2, 4):
        np.testing.assert_allclose(traces[p], traces[1], rtol=1e-10)


def test_nmf_more_ranks_than_columns():
    """Empty blocks (p > extent) are legal (distarray.py:55-65)."""
    x = orc.rand_fill_common((5, 3), 12, np.float64)
    vt0, w0 = orc.nmf_init(x, 2, 13)
    tr, vt, w = bs.run_inproc(6, _run, x, vt0, w0, 10, 1)[0]
    ovt, ow, otr = orc.nmf_apg(x, vt0, w0, 10)
    np.testing.assert_allclose(tr, otr, rtol=1e-10)
    np.testing.assert_allclose(vt, ovt, rtol=1e-9, atol=1e-12)


_DMMA_SCRIPT = r"""
import sys, numpy as np
import paper_2010_16114_b200 as bs
from oracle import blockstat_oracle as orc
out = {}
for i, (m, n, r) in enumerate([(1000, 777, 20), (257, 131, 7), (129, 380, 30), (3000, 2001, 24)]):
    x = orc.rand_fill_common((m, n), 400 + r, np.float64)
    vt0, w0 = orc.nmf_init(x, r, 500 + r)
    def fn(comm):
        xd = bs.distribute(x if comm.rank == 0 else None, comm)
        st = bs.nmf_init(xd, r, seed=1)
        st.Vt.local[...] = bs.distribute(vt0 if comm.rank == 0 else None, comm).local
        st.W.local[...] = bs.distribute(w0 if comm.rank == 0 else None, comm).local
        bs.nmf_multiplicative(st, 5, trace_every=1)
        return np.asarray(st.trace), bs.gather_full(st.Vt), bs.gather_full(st.W)
    tr, vt, w = bs.run_inproc(1 + i % 2, fn)[0]
    out[f"tr{i}"], out[f"vt{i}"], out[f"w{i}"] = tr, vt, w
np.savez(sys.argv[1], **out)
"""


def test_dmma_cp_async_pipeline_is_bitwise_equal_to_register_pipeline(tmp_path):
    """The cp.async-staged float64 DMMA GEMM (BS_DMMA_STAGES = 3 / 4) keeps the tile, fragment
    mapping and k order of the register double-buffered one (BS_DMMA_STAGES = 0): same bits
    for the same split count (pinned, since the default count follows each kernel's occupancy)."""
    import os
    import subprocess
    import sys
    from pathlib import Path

    root = Path(__file__).resolve().parents[1]
    res = {}
    for ns in ("0", "2", "3", "4"):
        f = tmp_path / f"ns{ns}.npz"
        env = dict(os.environ, BS_DMMA_STAGES=ns, BS_DMMA_SPLITS="5", PYTHONPATH=str(root))  # same splits
        subprocess.run([sys.executable, "-c", _DMMA_SCRIPT, str(f)], check=True, env=env, cwd=root, timeout=600)
        res[ns] = np.load(f)
    for ns in ("2", "3", "4"):
        for k in res["0"].files:
            np.testing.assert_array_equal(res[ns][k], res["0"][k], err_msg=f"stages={ns} {k}")
