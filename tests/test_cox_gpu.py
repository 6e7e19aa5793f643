"""GPU: l1-Cox (solvers.py:337-450) against the reference's golden vectors and the oracle."""

import warnings

import numpy as np
import pytest
import torch

import paper_2010_16114_b200 as bs
from oracle import blockstat_oracle as orc

pytestmark = pytest.mark.gpu

COX_CASES = ["m40_n12_lam01", "m40_n12_powersigma", "m40_n12_f32", "m40_n12_breslow"]


def _dist(comm, a):
    return bs.distribute(a if comm.rank == 0 else None, comm)


@pytest.mark.parametrize("name", COX_CASES)
@pytest.mark.parametrize("p", [1, 2, 3])
def test_cox_matches_reference_golden(golden, name, p):
    x = golden[f"cox_{name}_x"]
    y = golden[f"cox_{name}_y"]
    delta = golden[f"cox_{name}_delta"]
    lam, sigma, iters, breslow, _ = golden[f"cox_{name}_meta"]

    def fn(comm):
        st = bs.cox_init(_dist(comm, x), y, delta, lam=lam, sigma=None if sigma < 0 else sigma,
                         ties="breslow" if breslow else "none")
        bs.cox_fit(st, int(iters))
        return (np.asarray(st.trace), bs.gather_full(st.beta), bs.gather_full(st.grad), st.sigma,
                st.w.cpu().numpy(), st.W.cpu().numpy(), st.pd.cpu().numpy())

    tr, beta, grad, sig, w, W, pd = bs.run_inproc(p, fn)[0]
    tol = 1e-10 if x.dtype == np.float64 else 1e-4
    np.testing.assert_allclose(sig, golden[f"cox_{name}_sigma"][0], rtol=1e-12 if x.dtype == np.float64 else 1e-6)
    np.testing.assert_allclose(tr, golden[f"cox_{name}_trace"], rtol=tol)
    np.testing.assert_allclose(beta, golden[f"cox_{name}_beta"], rtol=tol * 10, atol=tol)
    np.testing.assert_allclose(grad, golden[f"cox_{name}_grad"], rtol=tol * 10, atol=tol)
    np.testing.assert_allclose(W, golden[f"cox_{name}_W"], rtol=tol)
    np.testing.assert_allclose(pd, golden[f"cox_{name}_pd"], rtol=tol * 10, atol=tol)


@pytest.mark.parametrize("m,n,p,breslow", [(500, 300, 1, False), (777, 129, 3, True), (1000, 2000, 2, False),
                                          (64, 1500, 4, False), (2048, 8, 1, True)])
def test_cox_matches_oracle(m, n, p, breslow):
    bt = np.zeros(n)
    bt[: min(5, n)] = 0.3
    x, y, delta = orc.survival_data(900 + n, m, n, bt)
    if breslow:
        y = -np.sort(-np.round(y * 4) / 4)
    cuts = orc.tie_cuts(y) if breslow else np.arange(m)
    lam, sigma, iters = 0.02, 0.5 / (np.linalg.norm(x, 2) ** 2), 30

    def fn(comm):
        st = bs.cox_init(_dist(comm, x), y, delta, lam=lam, sigma=sigma, ties="breslow" if breslow else "none")
        bs.cox_fit(st, iters)
        return np.asarray(st.trace), bs.gather_full(st.beta), bs.gather_full(st.grad)

    tr, beta, grad = bs.run_inproc(p, fn)[0]
    ob, og, otr = orc.cox_fit(x, delta, cuts, lam, sigma, iters)
    np.testing.assert_allclose(tr, otr, rtol=1e-10)
    np.testing.assert_allclose(beta, ob, rtol=1e-8, atol=1e-12)
    np.testing.assert_allclose(grad, og, rtol=1e-8, atol=1e-9)


def test_cox_int8_genotypes_widen_exactly():
    """int8 {0,1,2} storage computes the same iterates as float64 storage of the same values."""
    gen = np.random.Generator(np.random.Philox(5))
    m, n = 600, 400
    maf = gen.uniform(0.05, 0.5, size=n)
    g = gen.binomial(2, maf, size=(m, n)).astype(np.int8)
    eta = g[:, :3].astype(np.float64) @ np.array([0.4, -0.3, 0.2])
    t = gen.exponential(1.0 / np.exp(eta))
    order = np.argsort(-t)
    g, t = g[order], t[order]
    delta = (gen.random(m) < 0.3).astype(np.float64)
    sigma = 0.5 / np.linalg.norm(g.astype(np.float64), 2) ** 2

    def fn(comm, arr):
        st = bs.cox_init(_dist(comm, arr), t, delta, lam=0.01, sigma=sigma)
        bs.cox_fit(st, 20)
        return np.asarray(st.trace), bs.gather_full(st.beta)

    for p in (1, 3):
        tr8, b8 = bs.run_inproc(p, fn, g)[0]
        tr64, b64 = bs.run_inproc(p, fn, g.astype(np.float64))[0]
        np.testing.assert_allclose(tr8, tr64, rtol=1e-13)
        np.testing.assert_allclose(b8, b64, rtol=1e-12, atol=1e-15)
    ob, _, otr = orc.cox_fit(g.astype(np.float64), delta, np.arange(m), 0.01, sigma, 20)
    np.testing.assert_allclose(tr8, otr, rtol=1e-10)


def test_cox_loglik_zero_beta_and_single_subject():
    x, y, delta = orc.survival_data(70, 8, 3)
    want = -float(np.sum(delta * np.log(np.arange(1, 9))))

    def fn(comm):
        st = bs.cox_init(_dist(comm, x), y, delta, lam=0.0, sigma=0.01)
        one = bs.cox_init(_dist(comm, np.array([[1.5, -2.0]])), np.array([3.0]), np.array([1.0]), lam=0.0, sigma=0.01)
        one.beta.local[...] = _dist(comm, np.array([0.3, 0.7])).local
        return bs.cox_partial_loglik(st), bs.cox_partial_loglik(one)

    for ll, single in bs.run_inproc(2, fn):
        assert ll == pytest.approx(want, rel=1e-12)
        assert single == pytest.approx(0.0, abs=1e-14)


def test_pi_delta_examples_and_rank_partials(golden):
    def two(comm):
        out = np.empty(2)
        bs.pi_delta(out, np.ones(2), np.cumsum(np.ones(2)), np.ones(2), comm.rank, comm.rank + 1, comm)
        return out

    for out in bs.run_inproc(2, two):
        np.testing.assert_array_equal(out, [1.5, 0.5])

    w, W, d, cuts = golden["pid_w"], golden["pid_W"], golden["pid_delta"], golden["pid_cuts"]
    for p in (1, 3):
        def fn(comm):
            part = bs.partition_of(23, comm.size)
            out = np.empty(23)
            bs.pi_delta(out, w, W, d, part.lo(comm.rank), part.hi(comm.rank), comm, cuts=cuts)
            return out

        for out in bs.run_inproc(p, fn):
            np.testing.assert_allclose(out, golden[f"pid_out_p{p}"], rtol=1e-13, atol=1e-15)

    def zero_events(comm):
        out = np.empty(4)
        lo, hi = [(0, 2), (2, 4)][comm.rank]
        bs.pi_delta(out, np.ones(4), np.cumsum(np.ones(4)), np.zeros(4), lo, hi, comm)
        return out

    for out in bs.run_inproc(2, zero_events):
        np.testing.assert_array_equal(out, np.zeros(4))


def test_cox_gradient_matches_dense_and_finite_differences():
    x, y, delta = orc.survival_data(74, 12, 4)
    beta_d = np.random.Generator(np.random.Philox(74)).standard_normal(4) * 0.2

    def dense(b):
        eta = x @ b
        risk = y[:, None] >= y[None, :]
        big_w = (risk * np.exp(eta)[:, None]).sum(axis=0)
        ll = float(np.sum(delta * (eta - np.log(big_w))))
        p_mat = risk * np.exp(eta)[:, None] / big_w[None, :]
        return ll, x.T @ (delta - p_mat @ delta)

    _, gwant = dense(beta_d)
    h = 1e-6
    fd = np.array([(dense(beta_d + h * e)[0] - dense(beta_d - h * e)[0]) / (2 * h) for e in np.eye(4)])

    def fn(comm):
        st = bs.cox_init(_dist(comm, x), y, delta, lam=0.0, sigma=0.01)
        st.beta.local[...] = _dist(comm, beta_d).local
        bs.cox_fit(st, 1, trace_every=0)
        return bs.gather_full(st.grad), bs.gather_full(st.beta)

    for p in (1, 2, 3):
        grad, beta = bs.run_inproc(p, fn)[0]
        np.testing.assert_allclose(grad, gwant, rtol=1e-10)
        np.testing.assert_allclose(grad, fd, rtol=1e-5)
        np.testing.assert_allclose(beta, beta_d + 0.01 * gwant, rtol=1e-10)


def test_cox_lambda_dominant_keeps_beta_exactly_zero():
    x, y, delta = orc.survival_data(75, 10, 3)

    def fn(comm):
        st = bs.cox_init(_dist(comm, x), y, delta, lam=1e9, sigma=0.01)
        bs.cox_fit(st, 5)
        return bs.gather_full(st.beta)

    for beta in bs.run_inproc(2, fn):
        np.testing.assert_array_equal(beta, np.zeros(3))


def test_cox_monitor_stops_early_like_reference():
    x, y, delta = orc.survival_data(78, 10, 2, np.array([0.5, -0.5]))
    sigma = 1.0 / (2.0 * orc.opnorm_l2_power(x) ** 2)
    _, _, otr = orc.cox_fit(x, delta, np.arange(10), 0.1, sigma, 10_000, window=10)

    def fn(comm):
        st = bs.cox_init(_dist(comm, x), y, delta, lam=0.1)
        mon = bs.ConvergenceMonitor()
        bs.cox_fit(st, 10_000, monitor=mon)
        return np.asarray(st.trace), len(mon.history)

    tr, nh = bs.run_inproc(2, fn)[0]
    assert len(tr) < 10_000 and len(tr) == len(otr) == nh
    np.testing.assert_allclose(tr, otr, rtol=1e-9)


def test_cox_overflow_clamps_with_warning():
    def fn(comm):
        st = bs.cox_init(_dist(comm, np.array([[400.0], [-400.0]])), np.array([2.0, 1.0]), np.array([1.0, 1.0]),
                         lam=0.0, sigma=1e-9)
        st.beta.local[...] = _dist(comm, np.array([10.0])).local
        with pytest.warns(RuntimeWarning):
            val = bs.cox_partial_loglik(st)
        return val

    assert np.isfinite(bs.run_inproc(1, fn)[0])


def test_cox_nonfinite_input_raises():
    def fn(comm):
        st = bs.cox_init(_dist(comm, np.array([[np.nan], [0.0]])), np.array([2.0, 1.0]), np.array([1.0, 1.0]),
                         lam=0.0, sigma=0.1)
        bs.cox_partial_loglik(st)

    with pytest.raises(bs.NumericError):
        bs.run_inproc(1, fn)

    def fit(comm):
        st = bs.cox_init(_dist(comm, np.array([[np.nan], [0.0]])), np.array([2.0, 1.0]), np.array([1.0, 1.0]),
                         lam=0.0, sigma=0.1)
        try:
            bs.cox_fit(st, 3)
        except bs.NumericError:
            return st.trace
        return None

    assert bs.run_inproc(1, fit)[0] == []


def test_cox_init_validation():
    bad = [
        (np.array([1.0, 2.0, 3.0]), np.array([1.0, 0.0, 1.0]), "none"),    # unsorted
        (np.array([3.0, 2.0, 1.0]), np.array([1.0, 0.5, 1.0]), "none"),    # bad delta
        (np.array([2.0, 2.0, 1.0]), np.array([1.0, 0.0, 1.0]), "none"),    # ties need breslow
        (np.array([3.0, 2.0, 1.0]), np.array([1.0, 0.0, 1.0]), "efron"),   # unknown mode
    ]
    for y, d, ties in bad:
        def fn(comm):
            bs.cox_init(bs.zeros((3, 2), comm), y, d, lam=0.0, sigma=0.1, ties=ties)

        with pytest.raises(ValueError):
            bs.run_inproc(2, fn)


def test_cox_unpenalized_gradient_vanishes_at_optimum():
    bt = np.array([0.8, -0.6, 0.0, 0.0, 0.4])
    x, y, delta = orc.survival_data(76, 20, 5, bt)

    def fn(comm):
        st = bs.cox_init(_dist(comm, x), y, delta, lam=0.0)
        bs.cox_fit(st, 800, trace_every=0)
        bs.cox_fit(st, 1, trace_every=0)
        return np.linalg.norm(bs.gather_full(st.grad))

    for g in bs.run_inproc(2, fn):
        assert g <= 1e-4


@pytest.mark.parametrize("xdt,bdt,m,n", [(torch.float32, torch.float32, 4004, 777), (torch.float64, torch.float64, 3002, 301),
                                         (torch.int8, torch.float32, 8000, 250), (torch.float32, torch.float64, 5000, 33),
                                         (torch.float32, torch.float32, 20004, 3001),
                                         (torch.float32, torch.float32, 100000, 1999)])
def test_fused_grad_xbeta_pass_matches_two_pass(xdt, bdt, m, n):
    """bs_cox_grad_xbeta: the cooperative one-stream pass (allow_fused=1) gives the same
    grad, prox step, ||beta||_1 and X beta_new as bs_cox_grad_step + bs_cox_xbeta."""
    from paper_2010_16114_b200 import _lib

    g = torch.Generator(device="cuda")
    g.manual_seed(11)
    if xdt == torch.int8:
        X = torch.randint(0, 3, (n, m), generator=g, device="cuda", dtype=torch.int8)
    else:
        X = torch.randn(n, m, generator=g, device="cuda", dtype=xdt)  # column j = X[j]
    v = torch.randn(m, generator=g, device="cuda", dtype=torch.float64)
    beta0 = torch.randn(n, generator=g, device="cuda", dtype=bdt) * 0.1
    flags = torch.zeros(1, dtype=torch.int32, device="cuda")
    xc, bc = _lib.dtype_code(X.dtype), _lib.dtype_code(bdt)
    ws = torch.zeros(_lib.query("bs_cox_grad_xbeta_workspace", xc, m, n), dtype=torch.uint8, device="cuda")
    out = {}
    for fused in (0, 1):
        beta = beta0.clone()
        grad = torch.empty_like(beta)
        xb = torch.full((m + 1,), float("nan"), dtype=torch.float64, device="cuda")
        _lib.call("bs_cox_grad_xbeta", _lib.ptr(X), xc, _lib.ptr(v), bc, m, n, _lib.ptr(grad), _lib.ptr(beta),
                  1e-4, 0.1, _lib.ptr(xb), _lib.ptr(flags), fused, _lib.ptr(ws), ws.numel(), _lib.stream_ptr())
        torch.cuda.synchronize()
        out[fused] = (grad.double().cpu().numpy(), beta.double().cpu().numpy(), xb.cpu().numpy())
    tol = 1e-12 if bdt == torch.float64 else 1e-5
    for a, b in zip(out[0], out[1]):
        np.testing.assert_allclose(b, a, rtol=tol, atol=tol * max(1.0, np.abs(a).max()))
    assert np.count_nonzero(out[1][1]) < n  # the threshold zeroed some coordinates


def test_cox_int8_genotypes_float32_arithmetic():
    """int8 X with float32 arithmetic (the C5 configuration) runs the conversion-free int8
    kernels; iterates match float32 storage of the same values to float32 accuracy."""
    gen = np.random.Generator(np.random.Philox(9))
    m, n = 4096, 700
    maf = gen.uniform(0.05, 0.5, size=n)
    g = gen.binomial(2, maf, size=(m, n)).astype(np.int8)
    eta = g[:, :3].astype(np.float64) @ np.array([0.4, -0.3, 0.2])
    t = gen.exponential(1.0 / np.exp(eta))
    order = np.argsort(-t)
    g, t = g[order], t[order]
    delta = (gen.random(m) < 0.3).astype(np.float64)
    sigma = 0.5 / np.linalg.norm(g.astype(np.float64), 2) ** 2

    def fn(comm, arr):
        st = bs.cox_init(_dist(comm, arr), t, delta, lam=0.01, sigma=sigma, dtype=np.float32)
        bs.cox_fit(st, 20)
        return np.asarray(st.trace), bs.gather_full(st.beta)

    for p in (1, 2):
        tr8, b8 = bs.run_inproc(p, fn, g)[0]
        tr32, b32 = bs.run_inproc(p, fn, g.astype(np.float32))[0]
        np.testing.assert_allclose(tr8, tr32, rtol=2e-5)
        assert np.abs(b8 - b32).max() <= 1e-4 * max(np.abs(b32).max(), 1e-30)


@pytest.mark.parametrize("p", [1, 2])
def test_cox_fit_split_calls_match_one_call(p):
    """float32 fits run the fused one-stream pass; a fit split over several calls reuses the
    last pass's X beta (no extra pass) and must equal one long call, including after beta is
    changed between calls (the reuse is then skipped)."""
    gen = np.random.Generator(np.random.Philox(41))
    m, n = 8000, 900
    x = gen.standard_normal((m, n)).astype(np.float32)
    delta = (gen.random(m) < 0.5).astype(np.float64)
    y = np.arange(m, 0, -1, dtype=np.float64)

    def fn(comm, splits, poke):
        st = bs.cox_init(_dist(comm, x), y, delta, lam=1e-4, sigma=2e-5)
        for k in splits:
            bs.cox_fit(st, k)
            if poke:
                st.beta.local.mul_(1.0)  # same values: reuse stays valid
        return np.asarray(st.trace), bs.gather_full(st.beta)

    one = bs.run_inproc(p, fn, [12], False)[0]
    split = bs.run_inproc(p, fn, [5, 4, 3], False)[0]
    poked = bs.run_inproc(p, fn, [5, 7], True)[0]
    assert 0 < np.count_nonzero(one[1]) < n
    for got in (split, poked):
        np.testing.assert_allclose(got[0], one[0], rtol=1e-6)
        np.testing.assert_allclose(got[1], one[1], rtol=1e-5, atol=1e-7)

    def changed(comm):
        st = bs.cox_init(_dist(comm, x), y, delta, lam=1e-4, sigma=2e-5)
        bs.cox_fit(st, 3)
        st.beta.local.zero_()  # restart from zero: the cached X beta must not be used
        bs.cox_fit(st, 4)
        return np.asarray(st.trace)

    tr = bs.run_inproc(p, changed)[0]
    fresh = bs.run_inproc(p, fn, [4], False)[0][0]
    np.testing.assert_allclose(tr[3:], fresh, rtol=1e-6)


@pytest.mark.parametrize("m,n", [(8002, 300), (8000, 40)])
def test_cox_float32_shapes_outside_the_fused_plan(m, n):
    """m % 4 != 0 or fewer than 64 local columns: bs_cox_grad_xbeta takes the two-pass path;
    cox_fit results are unchanged against the oracle."""
    gen = np.random.Generator(np.random.Philox(m + n))
    x = gen.standard_normal((m, n)).astype(np.float32)
    delta = (gen.random(m) < 0.5).astype(np.float64)
    y = np.arange(m, 0, -1, dtype=np.float64)

    def fn(comm):
        st = bs.cox_init(_dist(comm, x), y, delta, lam=1e-4, sigma=2e-5)
        bs.cox_fit(st, 6)
        return np.asarray(st.trace)

    tr = bs.run_inproc(1, fn)[0]
    _, _, otr = orc.cox_fit(x.astype(np.float64), delta, np.arange(m), 1e-4, 2e-5, 6)
    np.testing.assert_allclose(tr, otr, rtol=2e-5)


@pytest.mark.parametrize("dtype", [np.float64, np.float32])
@pytest.mark.parametrize("ties", ["none", "breslow"])
def test_long_risk_and_suffix_scans_match_single_cta(dtype, ties):
    """m >= 8 scan tiles: bs_cox_risk / bs_cox_pi_delta run the multi-CTA scans; W, pd and
    loglik equal the single-CTA kernels' (workspace-less call) bit for bit / to rounding."""
    from paper_2010_16114_b200 import _lib

    m = 70_001
    dev = torch.device("cuda:0")
    gen = np.random.Generator(np.random.Philox(91))
    xb = torch.from_numpy(np.r_[gen.standard_normal(m) * 0.5, 0.0]).to(dev)
    delta_h = (gen.random(m) < 0.3).astype(dtype)
    delta = torch.from_numpy(delta_h).to(dev)
    y = np.floor(np.arange(m, 0, -1) / 3.0)
    cuts = None
    if ties == "breslow":
        cuts = torch.from_numpy(np.searchsorted(-y, -y, side="right").astype(np.int64) - 1).to(dev)
    code = _lib.dtype_code(dtype)
    tdt = torch.float64 if dtype == np.float64 else torch.float32
    out = {}
    for multi in (0, 1):
        Xb, w, W, pd = (torch.empty(m, dtype=tdt, device=dev) for _ in range(4))
        dmpd = torch.empty(m, dtype=torch.float64, device=dev)
        ll = torch.zeros(1, dtype=torch.float64, device=dev)
        flags = torch.zeros(1, dtype=torch.int32, device=dev)
        nb = _lib.query("bs_cox_risk_workspace", m)
        assert nb > 0
        ws = torch.zeros(nb, dtype=torch.uint8, device=dev)
        cp = _lib.ptr(cuts) if cuts is not None else None
        _lib.call("bs_cox_risk", _lib.ptr(xb), _lib.ptr(delta), cp, code, m, 700.0, _lib.ptr(Xb), _lib.ptr(w),
                  _lib.ptr(W), _lib.ptr(ll), _lib.ptr(flags), _lib.ptr(ws) if multi else None, nb if multi else 0,
                  _lib.stream_ptr())
        pw = torch.zeros(_lib.query("bs_cox_pi_delta_workspace", m), dtype=torch.uint8, device=dev)
        pw_n = pw.numel() if multi else 8 * m  # single-CTA: S only, no room for the tile totals
        _lib.call("bs_cox_pi_delta", _lib.ptr(w), _lib.ptr(W), _lib.ptr(delta), cp, code, m, 0, m, _lib.ptr(pd),
                  _lib.ptr(dmpd), _lib.ptr(flags), _lib.ptr(pw), pw_n, _lib.stream_ptr())
        torch.cuda.synchronize()
        out[multi] = (W.cpu().numpy(), pd.cpu().numpy(), float(ll.item()), int(flags.item()))
    np.testing.assert_array_equal(out[1][0], out[0][0])
    np.testing.assert_array_equal(out[1][1], out[0][1])
    np.testing.assert_allclose(out[1][2], out[0][2], rtol=1e-12)
    assert out[1][3] == out[0][3] == 0


def test_fused_float32_with_monitor_matches_two_pass(monkeypatch):
    """A convergence monitor stops before stepping; the fused path (default for float32)
    must stop at the same iteration with the same trace as the two-pass path, and a
    follow-up call must not reuse a stale X beta."""
    gen = np.random.Generator(np.random.Philox(77))
    m, n = 8000, 600
    x = gen.standard_normal((m, n)).astype(np.float32)
    delta = (gen.random(m) < 0.5).astype(np.float64)
    y = np.arange(m, 0, -1, dtype=np.float64)

    def fn(comm):
        st = bs.cox_init(_dist(comm, x), y, delta, lam=1e-4, sigma=2e-6)
        mon = bs.ConvergenceMonitor(window=3, rel_tol=1e-3)
        bs.cox_fit(st, 200, monitor=mon)
        first = len(st.trace)
        bs.cox_fit(st, 3)
        return np.asarray(st.trace), first, bs.gather_full(st.beta)

    fused = bs.run_inproc(1, fn)[0]
    monkeypatch.setenv("BS_COX_FUSION", "0")
    two = bs.run_inproc(1, fn)[0]
    assert fused[1] == two[1] < 200
    np.testing.assert_allclose(fused[0], two[0], rtol=1e-6)
    np.testing.assert_allclose(fused[2], two[2], rtol=1e-4, atol=1e-8)
