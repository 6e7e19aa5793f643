"""GPU: parity at BASELINE scale against fixtures produced by the reference itself.

The fixtures (tests/golden/golden_scale.npz) come from tests/golden/make_golden_scale.py,
which runs blockstat (the reference) on seeded inputs.  The inputs are regenerated
here on the device with the bit-exact Philox ``rand_fill`` (distarray.py:170-208), so
nothing large is stored.

Tolerances (north star: 1e-5 relative in emulated-f32/f64 mode over a fixed iteration
count):
  float64 traces 1e-9 relative; float64 iterates 1e-8 normwise (max|a-b| / max|b|).
  float32 traces: 2e-5 relative against the reference's OWN float32 trace, whose error
  against a float64 re-evaluation of its own iterates is up to 7.9e-6 (c2k_slice 5.6e-6,
  planted MU 7.9e-6 — recorded in the fixture), plus 1e-5 relative between our final
  trace value and a float64 direct residual of OUR final iterates (the objective check
  the reference's ``nmf_objective`` (solvers.py:124-136) defines).
  float32 iterates: 1e-4 normwise (both sides round every operation to float32).
"""

import numpy as np
import pytest
import torch

import paper_2010_16114_b200 as bs

pytestmark = pytest.mark.gpu

@pytest.fixture(scope="module")
def gs():
    from pathlib import Path

    with np.load(Path(__file__).resolve().parent / "golden" / "golden_scale.npz") as g:
        return {k: g[k] for k in g.files}


def normwise(a, b):
    a = np.asarray(a, dtype=np.float64)
    b = np.asarray(b, dtype=np.float64)
    return float(np.abs(a - b).max() / np.abs(b).max())


def obj64_dev(x_local, vt_full, w_full):
    """float64 direct residual ||X - Vt^T W||^2 of a device block (checker, torch on cuda)."""
    vt = torch.as_tensor(np.asarray(vt_full, dtype=np.float64), device="cuda")
    w = torch.as_tensor(np.asarray(w_full, dtype=np.float64), device="cuda")
    tot = 0.0
    n = x_local.shape[1]
    for j0 in range(0, n, 256):
        j1 = min(n, j0 + 256)
        d = x_local[:, j0:j1].to(torch.float64) - vt.t() @ w[:, j0:j1]
        tot += float((d * d).sum())
    return tot


def _nmf(comm, m, n, r, xseed, fseed, dt, algo, iters, every, want_obj64=False):
    x = bs.empty((m, n), comm, dt)
    bs.rand_fill(x, seed=xseed, common_init=True)
    st = bs.nmf_init(x, r, seed=fseed)
    (bs.nmf_multiplicative if algo == 0 else bs.nmf_apg)(st, iters, trace_every=every)
    vt, w = bs.gather_full(st.Vt), bs.gather_full(st.W)
    o64 = obj64_dev(x.local, vt, w[:, x.lo:x.hi]) if want_obj64 else None  # this rank's block
    return np.asarray(st.trace), vt, w, o64


def test_c1_full_nmf_mu_f64_1000_iterations(gs):
    """BASELINE configs[0] exactly: 10k x 10k, r = 20, 1,000 MU iterations (solvers.py:144-162)."""
    m, n, r, xs, fs, iters, every, _ = (int(v) for v in gs["c1_full_meta"])
    tr, vt, w, _ = bs.run_inproc(1, _nmf, m, n, r, xs, fs, np.float64, 0, iters, every)[0]
    ref = gs["c1_full_trace"]
    assert len(tr) == len(ref) == iters // every
    np.testing.assert_allclose(tr, ref, rtol=1e-9)
    assert normwise(vt, gs["c1_full_vt"]) <= 1e-8
    assert normwise(w, gs["c1_full_w"]) <= 1e-8


@pytest.mark.parametrize("p", [1, 2])
def test_c2_k_slice_apg_f32_long_reduction(gs, p):
    """C2's reduction length: scn a over K = m = 200,000 (distlinalg.py:239-243) through the tensor cores."""
    m, n, r, xs, fs, iters, every, _ = (int(v) for v in gs["c2k_slice_meta"])
    bs.gemm_path_counts(reset=True)
    res = bs.run_inproc(p, _nmf, m, n, r, xs, fs, np.float32, 1, iters, every, True)
    tr, vt, w, _ = res[0]
    o64 = sum(q[3] for q in res)  # each rank's local block
    counts = bs.gemm_path_counts()
    assert counts["tensor"] > 0 and counts["cuda_core"] == 0, counts
    np.testing.assert_allclose(tr, gs["c2k_slice_trace"], rtol=2e-5)
    assert abs(tr[-1] - o64) <= 1e-5 * o64, (tr[-1], o64)
    assert normwise(w, gs["c2k_slice_w"]) <= 1e-4
    assert normwise(vt[:, ::50], gs["c2k_slice_vt_sample"]) <= 1e-4
    np.testing.assert_allclose(vt.astype(np.float64).sum(axis=1), gs["c2k_slice_vt_rowsum"], rtol=1e-5)


def test_nmf_mu_f32_100_iterations(gs):
    m, n, r, xs, fs, iters, every, _ = (int(v) for v in gs["nmf_mu_f32_meta"])
    # trace every 10: the last value belongs to iteration 90, not to the final iterate
    tr, vt, w, _ = bs.run_inproc(2, _nmf, m, n, r, xs, fs, np.float32, 0, iters, every)[0]
    np.testing.assert_allclose(tr, gs["nmf_mu_f32_trace"], rtol=2e-5)
    assert normwise(vt, gs["nmf_mu_f32_vt"]) <= 1e-4
    assert normwise(w, gs["nmf_mu_f32_w"]) <= 1e-4


def planted(m, n, r, seed, noise):
    """Same generator as tests/golden/make_golden_scale.py:planted."""
    g = np.random.Generator(np.random.Philox(seed))
    vt = g.random((r, m))
    w = g.random((r, n))
    x = (vt.T @ w + noise * g.random((m, n))).astype(np.float32)
    vt0 = (vt * (1.0 + 0.01 * g.random((r, m)))).astype(np.float32)
    w0 = (w * (1.0 + 0.01 * g.random((r, n)))).astype(np.float32)
    return np.asfortranarray(x), vt0, w0


@pytest.mark.parametrize("algo", ["mu", "apg"])
def test_planted_low_rank_objective_is_a_direct_residual(gs, algo):
    """obj / ||X||^2 ~ 2e-7 (MU): the trace must still match a float64 direct residual at 1e-5."""
    name = f"nmf_planted_{algo}"
    m, n, r, seed, fseed, iters, every, a = (int(v) for v in gs[f"{name}_meta"])
    x, vt0, w0 = planted(m, n, r, seed, 1e-3)

    def fn(comm):
        xd = bs.distribute(x if comm.rank == 0 else None, comm)
        st = bs.nmf_init(xd, r, seed=fseed)
        st.Vt.local[...] = bs.distribute(vt0 if comm.rank == 0 else None, comm).local
        st.W.local[...] = bs.distribute(w0 if comm.rank == 0 else None, comm).local
        (bs.nmf_multiplicative if a == 0 else bs.nmf_apg)(st, iters, trace_every=every)
        vt, w = bs.gather_full(st.Vt), bs.gather_full(st.W)
        return np.asarray(st.trace), vt, w, obj64_dev(xd.local, vt, w)

    tr, vt, w, o64 = bs.run_inproc(1, fn)[0]
    assert abs(tr[-1] - o64) <= 1e-5 * o64, (tr[-1], o64)
    np.testing.assert_allclose(tr, gs[f"{name}_trace"], rtol=2e-5)
    assert normwise(vt, gs[f"{name}_vt"]) <= 1e-4
    assert normwise(w, gs[f"{name}_w"]) <= 1e-4


@pytest.mark.parametrize("tag", ["f64", "f32"])
def test_mds_n2000_q20_100_iterations(gs, tag):
    d, n, q, xs, ts, iters = (int(v) for v in gs[f"mds_n2000_{tag}_meta"])
    dt = np.float64 if tag == "f64" else np.float32

    def fn(comm):
        x = bs.empty((d, n), comm, dt)
        bs.rand_fill(x, seed=xs, common_init=True)
        y = bs.empty((n, n), comm, dt)
        bs.pairwise_euclidean(y, x)
        st = bs.mds_init(y, q, seed=ts)
        bs.mds_fit(st, iters)
        return np.asarray(st.trace), bs.gather_full(st.theta)

    tr, th = bs.run_inproc(2, fn)[0]
    if tag == "f64":
        np.testing.assert_allclose(tr, gs["mds_n2000_f64_trace"], rtol=1e-9)
        assert normwise(th, gs["mds_n2000_f64_theta"]) <= 1e-8
    else:
        np.testing.assert_allclose(tr, gs["mds_n2000_f32_trace"], rtol=2e-5)
        assert normwise(th, gs["mds_n2000_f32_theta"]) <= 1e-4


def cox_inputs(m, n, seed):
    """Same data as tests/golden/make_golden_scale.py:cox_inputs (host side: y, delta)."""
    y = np.floor(np.arange(m, 0, -1) / 3.0)
    delta = (np.random.Generator(np.random.Philox(seed + 1)).random(m) > 0.3).astype(np.float64)
    return y, delta


@pytest.mark.parametrize("name", ["cox_breslow_f64", "cox_f32"])
def test_cox_4000x3000_breslow_100_iterations(gs, name):
    m, n, seed, lam, sigma, iters = gs[f"{name}_meta"]
    m, n, seed, iters = int(m), int(n), int(seed), int(iters)
    dt = np.float64 if name.endswith("f64") else np.float32
    y, delta = cox_inputs(m, n, seed)

    def fn(comm):
        x64 = bs.empty((m, n), comm, np.float64)  # X = U(0,1) - 0.5 drawn from the float64 stream
        bs.rand_fill(x64, seed=seed, common_init=True)
        x = bs.empty((m, n), comm, dt)
        x.local.copy_(x64.local - 0.5)
        del x64
        st = bs.cox_init(x, y, delta, lam=float(lam), sigma=None if sigma < 0 else float(sigma), ties="breslow")
        bs.cox_fit(st, iters)
        return np.asarray(st.trace), bs.gather_full(st.beta), st.sigma

    tr, beta, sig = bs.run_inproc(2, fn)[0]
    np.testing.assert_allclose(sig, gs[f"{name}_sigma"][0], rtol=1e-9)
    ref_beta = gs[f"{name}_beta"]
    if dt == np.float64:
        np.testing.assert_allclose(tr, gs[f"{name}_trace"], rtol=1e-9)
        assert normwise(beta, ref_beta) <= 1e-8
        np.testing.assert_array_equal(beta == 0, ref_beta == 0)
    else:
        np.testing.assert_allclose(tr, gs[f"{name}_trace"], rtol=2e-5)
        assert normwise(beta, ref_beta) <= 1e-4


@pytest.mark.parametrize("storage,p", [("packed", 1), ("packed", 2), ("int8", 2)])
def test_cox_genotypes_float64_against_reference(gs, storage, p):
    """Genotype Cox in float64 against the reference run on the same 0/1/2 matrix as float64
    (make_golden_scale.py cox_geno_f64): packed storage takes both passes on the tensor cores
    (kind::mxf4 with 32 digits), int8 storage the exact CUDA-core kernels."""
    m, n, seed, lam, _, iters = gs["cox_geno_f64_meta"]
    m, n, seed, iters = int(m), int(n), int(seed), int(iters)
    y = np.floor(np.arange(m, 0, -1) / 4.0)
    delta = (np.random.Generator(np.random.Philox(seed + 7)).random(m) < 0.4).astype(np.float64)

    def fn(comm):
        if storage == "packed":
            x = bs.genotype_fill(bs.PackedGenotypes(comm, (m, n)), seed)
        else:
            x = bs.genotype_fill(bs.empty((m, n), comm, np.int8), seed)
        bs.gemm_path_counts(reset=True)
        st = bs.cox_init(x, y, delta, lam=float(lam), ties="breslow", dtype=np.float64)
        bs.cox_fit(st, iters)
        return np.asarray(st.trace), bs.gather_full(st.beta), st.sigma, bs.gemm_path_counts()["cox_packed_tensor"]

    tr, beta, sig, passes = bs.run_inproc(p, fn)[0]
    if storage == "packed":
        assert passes >= 2 * iters
    ref_beta = gs["cox_geno_f64_beta"]
    np.testing.assert_allclose(sig, gs["cox_geno_f64_sigma"][0], rtol=1e-9)
    np.testing.assert_allclose(tr, gs["cox_geno_f64_trace"], rtol=1e-9)
    assert normwise(beta, ref_beta) <= 1e-8
    np.testing.assert_array_equal(beta == 0, ref_beta == 0)


@pytest.mark.parametrize("p", [1, 2])
def test_cox_genotypes_float32_against_reference(gs, p):
    """The C5 setting (packed genotypes, float32 arithmetic, both passes on the tensor cores)
    against the reference's float32 run on the same matrix: traces at 2e-5 (the reference's own
    float32 rounding), beta at 1e-4 normwise."""
    m, n, seed, lam, _, iters = gs["cox_geno_f64_meta"]
    m, n, seed, iters = int(m), int(n), int(seed), int(iters)
    y = np.floor(np.arange(m, 0, -1) / 4.0)
    delta = (np.random.Generator(np.random.Philox(seed + 7)).random(m) < 0.4).astype(np.float64)
    sigma = float(gs["cox_geno_f32_sigma"][0])

    def fn(comm):
        x = bs.genotype_fill(bs.PackedGenotypes(comm, (m, n)), seed)
        st = bs.cox_init(x, y, delta, lam=float(lam), sigma=sigma, ties="breslow", dtype=np.float32)
        bs.cox_fit(st, iters)
        return np.asarray(st.trace), bs.gather_full(st.beta)

    tr, beta = bs.run_inproc(p, fn)[0]
    np.testing.assert_allclose(tr, gs["cox_geno_f32_trace"], rtol=2e-5)
    assert normwise(beta, gs["cox_geno_f32_beta"]) <= 1e-4


@pytest.mark.parametrize("p", [1, 2])
def test_mds_n8000_f32_20_iterations(gs, p):
    """MDS with 8,000 points through the tcgen05 pass (several row segments and column blocks
    per rank) against the reference's float32 run.  The reference's float32 stress is a float32
    dot over n^2 = 64M terms, 1.5e-4 low at theta0 against a float64 sum of the same float32 terms
    (make_golden_scale.py): our first trace entry is checked against that float64 sum at 1e-5,
    the trace against the reference at 5e-4, the final theta at 1e-4 normwise."""
    d, n, q, xs, ts, iters = (int(v) for v in gs["mds_n8000_f32_meta"])

    def fn(comm):
        x = bs.empty((d, n), comm, np.float32)
        bs.rand_fill(x, seed=xs, common_init=True)
        y = bs.empty((n, n), comm, np.float32)
        bs.pairwise_euclidean(y, x)
        st = bs.mds_init(y, q, seed=ts)
        bs.gemm_path_counts(reset=True)
        bs.mds_fit(st, iters)
        return np.asarray(st.trace), bs.gather_full(st.theta), bs.gemm_path_counts()["mds_tensor"]

    tr, th, passes = bs.run_inproc(p, fn)[0]
    assert passes >= iters
    np.testing.assert_allclose(tr[0], gs["mds_n8000_f32_stress0_f64"][0], rtol=1e-5)
    np.testing.assert_allclose(tr, gs["mds_n8000_f32_trace"], rtol=5e-4)
    assert normwise(th, gs["mds_n8000_f32_theta"]) <= 1e-4


@pytest.mark.parametrize("p", [1, 2])
def test_cox_f32_fused_pass_against_reference(gs, p):
    """float32 Cox large enough for the one-stream fused pass (bs_cox_grad_xbeta, C4's kernel:
    m >= 4096, n_loc >= 128) against the reference's float32 run: traces at 2e-5, beta 1e-4."""
    from paper_2010_16114_b200 import _lib

    m, n, seed, lam, sigma, iters = gs["cox_f32_fused_meta"]
    m, n, seed, iters = int(m), int(n), int(seed), int(iters)
    y, delta = cox_inputs(m, n, seed)

    def fn(comm):
        x64 = bs.empty((m, n), comm, np.float64)
        bs.rand_fill(x64, seed=seed, common_init=True)
        x = bs.empty((m, n), comm, np.float32)
        x.local.copy_(x64.local - 0.5)
        del x64
        st = bs.cox_init(x, y, delta, lam=float(lam), sigma=float(sigma), ties="breslow")
        with _lib.profile(["bs_cox_grad_xbeta"]) as prof:
            bs.cox_fit(st, iters)
            torch.cuda.synchronize()
        return np.asarray(st.trace), bs.gather_full(st.beta), len(prof.elapsed_ms().get("bs_cox_grad_xbeta", []))

    tr, beta, fused = bs.run_inproc(p, fn)[0]
    if p == 1:  # (the profile hook is process-wide: rank threads would share it)
        assert fused >= iters - 1  # every iteration after the first takes the one-stream pass
    np.testing.assert_allclose(tr, gs["cox_f32_fused_trace"], rtol=2e-5)
    assert normwise(beta, gs["cox_f32_fused_beta"]) <= 1e-4


@pytest.mark.parametrize("p", [1, 2])
def test_nmf_apg_f64_rank60_against_reference(gs, p):
    """C2's rank in float64 (the cp.async m16n8k16 DMMA kernel at RP = 64) against the reference:
    trace 1e-9, iterates 1e-8 normwise."""
    m, n, r, xs, fs, iters, every, _ = (int(v) for v in gs["nmf_apg_f64_r60_meta"])
    tr, vt, w, _ = bs.run_inproc(p, _nmf, m, n, r, xs, fs, np.float64, 1, iters, every)[0]
    np.testing.assert_allclose(tr, gs["nmf_apg_f64_r60_trace"], rtol=1e-9)
    assert normwise(vt[:, ::20], gs["nmf_apg_f64_r60_vt_sample"]) <= 1e-8
    np.testing.assert_allclose(vt.sum(axis=1), gs["nmf_apg_f64_r60_vt_rowsum"], rtol=1e-9)
    assert normwise(w, gs["nmf_apg_f64_r60_w"]) <= 1e-8


@pytest.mark.parametrize("p", [1, 2])
def test_cox_genotypes_long_k_float64(gs, p):
    """200,000 samples x 1,024 packed variants in float64 (the tensor-core passes over 98
    scale groups) against the reference: sigma, trace 1e-9, beta 1e-8, zero pattern."""
    m, n, seed, lam, _, iters = gs["cox_geno_long_f64_meta"]
    m, n, seed, iters = int(m), int(n), int(seed), int(iters)
    y = np.floor(np.arange(m, 0, -1) / 4.0)
    delta = (np.random.Generator(np.random.Philox(seed + 7)).random(m) < 0.3).astype(np.float64)

    def fn(comm):
        x = bs.genotype_fill(bs.PackedGenotypes(comm, (m, n)), seed)
        st = bs.cox_init(x, y, delta, lam=float(lam), ties="breslow", dtype=np.float64)
        bs.cox_fit(st, iters)
        return np.asarray(st.trace), bs.gather_full(st.beta), st.sigma

    tr, beta, sig = bs.run_inproc(p, fn)[0]
    ref = gs["cox_geno_long_f64_beta"]
    np.testing.assert_allclose(sig, gs["cox_geno_long_f64_sigma"][0], rtol=1e-9)
    np.testing.assert_allclose(tr, gs["cox_geno_long_f64_trace"], rtol=1e-9)
    assert normwise(beta, ref) <= 1e-8
    np.testing.assert_array_equal(beta == 0, ref == 0)
