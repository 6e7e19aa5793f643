"""Solver-level C ABI (bs_ctx_* / bs_cox_*): the native cox_fit loop must produce the
traces and coefficients of the Python loop over the same kernels.

Multi-rank (NCCL) coverage is in tests/nccl_parity.py (one process per GPU)."""

import numpy as np
import pytest

import paper_2010_16114_b200 as bs
from paper_2010_16114_b200 import runtime
from oracle import blockstat_oracle as orc

pytestmark = pytest.mark.gpu


def _dist(comm, a):
    return bs.distribute(a if comm.rank == 0 else None, comm)


@pytest.mark.parametrize("dt,ties,m,n", [(np.float64, "none", 600, 80), (np.float32, "none", 8000, 700),
                                         (np.float64, "breslow", 500, 60), (np.float32, "breslow", 6000, 300)])
def test_native_cox_run_matches_cox_fit(dt, ties, m, n):
    gen = np.random.Generator(np.random.Philox(m + n))
    x = gen.standard_normal((m, n)).astype(dt)
    delta = (gen.random(m) < 0.5).astype(np.float64)
    y = np.floor(np.arange(m, 0, -1) / (3.0 if ties == "breslow" else 1.0))
    lam, sigma = 1e-4, 2e-5

    def fn(comm, native):
        st = bs.cox_init(_dist(comm, x), y, delta, lam=lam, sigma=sigma, ties=ties)
        if native:
            with runtime.Context(comm) as ctx:
                runtime.cox_run(ctx, st, 6)
                runtime.cox_run(ctx, st, 6, trace_every=2)
        else:
            bs.cox_fit(st, 6)
            bs.cox_fit(st, 6, trace_every=2)
        return np.asarray(st.trace), bs.gather_full(st.beta)

    py = bs.run_inproc(1, fn, False)[0]
    nat = bs.run_inproc(1, fn, True)[0]
    assert len(nat[0]) == len(py[0]) == 9
    # float32 (fused pass): cox_fit's second call reuses the last pass's X beta while a
    # fresh native state recomputes it with the scn m kernel -- same value to ~1e-10
    tol = 1e-12 if dt == np.float64 else 1e-9
    np.testing.assert_allclose(nat[0], py[0], rtol=tol)
    np.testing.assert_allclose(nat[1], py[1], rtol=1e-10 if dt == np.float64 else 1e-5, atol=1e-12 if dt == np.float64 else 1e-9)
    assert np.count_nonzero(py[1]) > 0
    cuts = orc.tie_cuts(y) if ties == "breslow" else np.arange(m)
    _, _, otr = orc.cox_fit(x.astype(np.float64), delta, cuts, lam, sigma, 6)
    np.testing.assert_allclose(nat[0][:6], otr, rtol=1e-10 if dt == np.float64 else 2e-5)


def test_native_cox_run_monitor_and_numeric_error():
    gen = np.random.Generator(np.random.Philox(5))
    m, n = 3000, 200
    x = gen.standard_normal((m, n))
    delta = (gen.random(m) < 0.5).astype(np.float64)
    y = np.arange(m, 0, -1, dtype=np.float64)

    def fn(comm, native):
        st = bs.cox_init(_dist(comm, x), y, delta, lam=1e-4, sigma=1e-6)
        mon = bs.ConvergenceMonitor(window=3, rel_tol=1e-3)
        if native:
            with runtime.Context(comm) as ctx:
                runtime.cox_run(ctx, st, 300, monitor=mon)
        else:
            bs.cox_fit(st, 300, monitor=mon)
        return np.asarray(st.trace)

    py = bs.run_inproc(1, fn, False)[0]
    nat = bs.run_inproc(1, fn, True)[0]
    assert len(nat) == len(py) < 300
    np.testing.assert_allclose(nat, py, rtol=1e-12)

    def bad(comm):
        xb = x.copy()
        xb[7, 3] = np.nan
        st = bs.cox_init(_dist(comm, xb), y, delta, lam=1e-4, sigma=1e-6)
        with runtime.Context(comm) as ctx:
            with pytest.raises(bs.NumericError):
                runtime.cox_run(ctx, st, 5)
        return True

    assert bs.run_inproc(1, bad)[0]


@pytest.mark.parametrize("algo", ["mu", "apg"])
@pytest.mark.parametrize("dt,m,n,r", [(np.float64, 300, 200, 7), (np.float32, 2048, 1500, 20)])
def test_native_nmf_run_matches_python_loop(algo, dt, m, n, r):
    x = orc.rand_fill_common((m, n), 3, dt)

    def fn(comm, native):
        xd = _dist(comm, x)
        st = bs.nmf_init(xd, r, seed=4)
        if native:
            with runtime.Context(comm) as ctx:
                runtime.nmf_run(ctx, st, 5, algo=algo)
                runtime.nmf_run(ctx, st, 4, algo=algo, trace_every=2)
        else:
            fit = bs.nmf_apg if algo == "apg" else bs.nmf_multiplicative
            fit(st, 5)
            fit(st, 4, trace_every=2)
        return np.asarray(st.trace), bs.gather_full(st.Vt), bs.gather_full(st.W)

    py = bs.run_inproc(1, fn, False)[0]
    nat = bs.run_inproc(1, fn, True)[0]
    assert len(nat[0]) == len(py[0]) == 7
    for a, b in zip(nat, py):
        np.testing.assert_array_equal(a, b)  # same kernels, same order, one rank


def test_native_nmf_rejects_negative_data():
    x = orc.rand_fill_common((64, 40), 3, np.float64)
    x[5, 7] = -1.0

    def fn(comm):
        st = bs.nmf_init(_dist(comm, np.abs(x)), 3, seed=4)
        st.X.local[5, 7] = -1.0
        with runtime.Context(comm) as ctx:
            with pytest.raises(ValueError):
                runtime.nmf_run(ctx, st, 2)
        return True

    assert bs.run_inproc(1, fn)[0]


@pytest.mark.parametrize("dt,n,q", [(np.float64, 200, 3), (np.float32, 516, 8)])
def test_native_mds_run_matches_mds_fit(dt, n, q):
    x = orc.rand_fill_common((6, n), 9, dt)
    y = orc.pairwise_euclidean(x).astype(dt)

    def fn(comm, native):
        st = bs.mds_init(_dist(comm, y), q, seed=10)
        if native:
            with runtime.Context(comm) as ctx:
                runtime.mds_run(ctx, st, 5)
                runtime.mds_run(ctx, st, 4, trace_every=2)
        else:
            bs.mds_fit(st, 5)
            bs.mds_fit(st, 4, trace_every=2)
        return np.asarray(st.trace), bs.gather_full(st.theta)

    py = bs.run_inproc(1, fn, False)[0]
    nat = bs.run_inproc(1, fn, True)[0]
    assert len(nat[0]) == len(py[0]) == 7
    np.testing.assert_array_equal(nat[0], py[0])
    np.testing.assert_array_equal(nat[1], py[1])


def test_native_mds_degenerate_raises():
    pts = np.zeros((2, 6))
    pts[:, 1] = pts[:, 0] = 0.5  # points 0 and 1 coincide
    pts[:, 2:] = np.arange(8, dtype=np.float64).reshape(2, 4)
    y = orc.pairwise_euclidean(pts)
    y[0, 1] = y[1, 0] = 1.0  # target distance nonzero, embedding distance zero

    def fn(comm, native):
        st = bs.mds_init(_dist(comm, y), 2, seed=1)
        st.theta.local[:, 1] = st.theta.local[:, 0]
        with pytest.raises(bs.DegenerateConfigError):
            if native:
                with runtime.Context(comm) as ctx:
                    runtime.mds_run(ctx, st, 3)
            else:
                bs.mds_fit(st, 3)
        return np.asarray(st.trace)

    py = bs.run_inproc(1, fn, False)[0]
    nat = bs.run_inproc(1, fn, True)[0]
    assert 1 <= len(py) < 3
    np.testing.assert_array_equal(nat, py)


def test_native_and_python_cox_calls_interleave():
    """cox_fit and runtime.cox_run on one state, alternating: each must notice that the
    other moved beta (neither may reuse a cached X beta) and the trace must equal one
    long cox_fit."""
    gen = np.random.Generator(np.random.Philox(21))
    m, n = 8000, 400
    x = gen.standard_normal((m, n)).astype(np.float32)
    delta = (gen.random(m) < 0.5).astype(np.float64)
    y = np.arange(m, 0, -1, dtype=np.float64)

    def fn(comm, mixed):
        st = bs.cox_init(_dist(comm, x), y, delta, lam=1e-4, sigma=2e-5)
        if mixed:
            with runtime.Context(comm) as ctx:
                runtime.cox_run(ctx, st, 3)
                bs.cox_fit(st, 3)
                runtime.cox_run(ctx, st, 3)
                bs.cox_fit(st, 3)
        else:
            bs.cox_fit(st, 12)
        return np.asarray(st.trace)

    one = bs.run_inproc(1, fn, False)[0]
    mixed = bs.run_inproc(1, fn, True)[0]
    np.testing.assert_allclose(mixed, one, rtol=1e-9)


def test_c_host_program_matches_cox_fit(tmp_path):
    """examples/cox_host.c (plain C, no Python) drives a fit through the solver-level ABI;
    its trace equals cox_fit on the same inputs."""
    import pathlib
    import subprocess

    from paper_2010_16114_b200.distarray import philox_key

    root = pathlib.Path(__file__).resolve().parents[1]
    exe = tmp_path / "cox_host"
    lib = root / "paper_2010_16114_b200"
    subprocess.run(["gcc", "-O2", "-I", str(root / "include"), "-I", "/usr/local/cuda/include",
                    str(root / "examples" / "cox_host.c"), "-o", str(exe), "-L", str(lib), "-lbsb200",
                    "-L/usr/local/cuda/lib64", "-lcudart", f"-Wl,-rpath,{lib}", "-Wl,-rpath,/usr/local/cuda/lib64"],
                   check=True)
    k0, k1 = philox_key(1234)
    out = subprocess.run([str(exe), str(k0), str(k1), "8"], check=True, capture_output=True, text=True).stdout
    got = np.array([float(v) for v in out.split()])
    m, n = 4096, 256
    x = orc.rand_fill_common((m, n), 1234, np.float32)
    delta = np.array([float((i * 7919) % 10 < 6) for i in range(m)])
    y = np.arange(m, 0, -1, dtype=np.float64)

    def fn(comm):
        st = bs.cox_init(_dist(comm, x), y, delta, lam=1e-4, sigma=1e-5)
        bs.cox_fit(st, 8)
        return np.asarray(st.trace)

    want = bs.run_inproc(1, fn)[0]
    assert len(got) == 8
    np.testing.assert_allclose(got, want, rtol=1e-9)
