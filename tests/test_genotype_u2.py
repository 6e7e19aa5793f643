"""2-bit packed genotypes: the packed block feeds the same Cox / opnorm
kernels as int8 X and must give the int8 results.

CPU tests pin the oracle's packing against a per-element loop; the gpu tests check the
device pack / unpack / fill against it, and the packed scn-m / scn-p kernels and full
cox_fit traces against the int8 path and the oracle.
"""

import numpy as np
import pytest
import torch

import paper_2010_16114_b200 as bs
from paper_2010_16114_b200 import _lib
from oracle import blockstat_oracle as orc


def _loop_pack(x):
    m, n = x.shape
    ld = ((m + 63) // 64) * 16
    out = np.zeros((ld, n), dtype=np.uint8)
    for j in range(n):
        for i in range(m):
            out[i // 4, j] |= (int(x[i, j]) & 3) << (2 * (i % 4))
    return out


@pytest.mark.parametrize("m", [1, 3, 64, 65, 130])
def test_oracle_packing_matches_loop(m):
    x = np.random.Generator(np.random.Philox(m)).integers(0, 3, size=(m, 5)).astype(np.int8)
    np.testing.assert_array_equal(orc.pack_genotypes_u2(x), _loop_pack(x))
    assert bs.packed_bytes_per_column(m) == orc.pack_genotypes_u2(x).shape[0]


def _device_block(p):
    return p.local.cpu().numpy()


@pytest.mark.gpu
@pytest.mark.parametrize("m,n", [(1, 3), (15, 4), (64, 7), (65, 9), (1000, 33), (8193, 5)])
def test_pack_unpack_match_oracle(m, n):
    x = np.random.Generator(np.random.Philox(m + n)).integers(0, 3, size=(m, n)).astype(np.int8)
    want = orc.pack_genotypes_u2(x)

    def fn(comm):
        a = bs.distribute(x if comm.rank == 0 else None, comm)
        p = bs.pack_genotypes(a)
        assert p.local.shape == (want.shape[0], p.hi - p.lo)
        np.testing.assert_array_equal(_device_block(p), want[:, p.lo:p.hi])
        assert np.array_equal(bs.gather_full(p), bs.gather_full(bs.unpack_genotypes(p)))
        return bs.gather_full(bs.unpack_genotypes(p))

    for p in (1, 3):
        for got in bs.run_inproc(p, fn):
            np.testing.assert_array_equal(got, x)


@pytest.mark.gpu
@pytest.mark.parametrize("m", [37, 64, 131])
def test_fill_packed_matches_int8_fill(m):
    """Packed fill = pack(int8 fill) for odd m (Philox blocks straddling columns) and p ranks."""
    n, seed = 23, 77
    want = orc.pack_genotypes_u2(orc.genotype_fill(m, n, seed))

    def fn(comm):
        p = bs.genotype_fill(bs.PackedGenotypes(comm, (m, n)), seed)
        return p.lo, _device_block(p)

    for ranks in (1, 3):
        for lo, blk in bs.run_inproc(ranks, fn):
            np.testing.assert_array_equal(blk, want[:, lo:lo + blk.shape[1]])


def _xbeta_grad(X, code, beta, v, dtype):
    """Raw C-ABI calls: xb = X beta and g = X^T v for one local block."""
    m, n_loc = v.numel(), beta.numel()
    dev = beta.device
    tcode = _lib.dtype_code(dtype)
    xb = torch.zeros(m + 1, dtype=torch.float64, device=dev)
    ws = torch.zeros(max(_lib.query("bs_cox_xbeta_workspace", code, m, n_loc), 256), dtype=torch.uint8, device=dev)
    _lib.call("bs_cox_xbeta", _lib.ptr(X), code, _lib.ptr(beta), tcode, m, n_loc, _lib.ptr(xb), _lib.ptr(ws),
              ws.numel(), _lib.stream_ptr())
    grad = torch.zeros(n_loc, dtype=dtype, device=dev)
    dummy = torch.zeros(n_loc, dtype=dtype, device=dev)
    l1 = torch.zeros(1, dtype=torch.float64, device=dev)
    wg = torch.zeros(max(_lib.query("bs_cox_grad_workspace", code, m, n_loc), 256), dtype=torch.uint8, device=dev)
    _lib.call("bs_cox_grad_step", _lib.ptr(X), code, _lib.ptr(v), tcode, m, n_loc, _lib.ptr(grad), _lib.ptr(dummy),
              0.0, 0.0, 0, _lib.ptr(l1), None, _lib.ptr(wg), wg.numel(), _lib.stream_ptr())
    return xb[:m].cpu().numpy(), grad.cpu().numpy()


@pytest.mark.gpu
@pytest.mark.parametrize("dtype", [torch.float32, torch.float64])
@pytest.mark.parametrize("m,n", [(100, 7), (4096, 65), (20000, 300), (9000, 1)])
def test_packed_scans_match_int8(dtype, m, n):
    gen = np.random.Generator(np.random.Philox(3 * m + n))
    x = gen.integers(0, 3, size=(m, n)).astype(np.int8)
    beta = gen.standard_normal(n)
    v = gen.standard_normal(m)
    dev = torch.device("cuda:0")
    X8 = torch.from_numpy(np.asfortranarray(x).ravel(order="F")).to(dev)
    XP = torch.from_numpy(orc.pack_genotypes_u2(x).ravel(order="F")).to(dev)
    b = torch.from_numpy(beta).to(dev, dtype)
    vd = torch.from_numpy(v).to(dev)
    xb8, g8 = _xbeta_grad(X8, _lib.BS_I8, b, vd, dtype)
    xbp, gp = _xbeta_grad(XP, _lib.BS_U2, b, vd, dtype)
    bh = b.double().cpu().numpy()
    want_xb = x.astype(np.float64) @ bh
    want_g = x.astype(np.float64).T @ v
    rtol = 1e-12 if dtype == torch.float64 else 2e-5
    scale_xb = np.abs(x).astype(np.float64) @ np.abs(bh) + 1e-300
    scale_g = np.abs(x).astype(np.float64).T @ np.abs(v) + 1e-300
    for got, ref, sc in ((xbp, want_xb, scale_xb), (xb8, want_xb, scale_xb), (gp, want_g, scale_g),
                         (g8, want_g, scale_g)):
        assert np.max(np.abs(got - ref) / sc) < rtol
    np.testing.assert_allclose(xbp, xb8, rtol=0, atol=rtol * scale_xb.max())


@pytest.mark.gpu
@pytest.mark.parametrize("p", [1, 2])
def test_cox_fit_packed_matches_int8_and_oracle(p):
    m, n, seed, iters = 3000, 257, 11, 12
    x = orc.genotype_fill(m, n, seed)
    y = np.floor(np.arange(m, 0, -1) / 4.0)
    delta = (np.random.Generator(np.random.Philox(2)).random(m) < 0.6).astype(np.float64)
    lam = 1e-6

    def fn(comm, packed):
        if packed:
            a = bs.genotype_fill(bs.PackedGenotypes(comm, (m, n)), seed)
        else:
            a = bs.genotype_fill(bs.empty((m, n), comm, np.int8), seed)
        st = bs.cox_init(a, y, delta, lam, ties="breslow", dtype=np.float32)
        bs.cox_fit(st, iters)
        return np.asarray(st.trace, dtype=np.float64), bs.gather_full(st.beta), st.sigma

    int8_runs = bs.run_inproc(p, lambda c: fn(c, False))  # packed: both passes on the tensor cores
    packed_runs = bs.run_inproc(p, lambda c: fn(c, True))
    (t8, b8, s8), (tp, bp, sp) = int8_runs[0], packed_runs[0]
    np.testing.assert_allclose(sp, s8, rtol=1e-10)  # opnorm through the packed kernels
    assert 0 < np.count_nonzero(b8) < n  # the step moved and the threshold zeroed some
    np.testing.assert_allclose(tp, t8, rtol=2e-5)
    np.testing.assert_allclose(bp, b8, rtol=2e-3, atol=2e-5 * np.abs(b8).max())
    _, _, otr = orc.cox_fit(x.astype(np.float64), delta, orc.tie_cuts(y), lam, sp, iters)
    np.testing.assert_allclose(tp, otr, rtol=5e-5)


@pytest.mark.gpu
@pytest.mark.parametrize("scale", [1e-35, 1e-12, 1.0, 1e20])
def test_packed_grad_any_v_scale(scale):
    """The packed scn-p kernel rescales each lane's v by a power of two (subnormal widening);
    results must keep float32 accuracy for tiny and huge v, and with mixed magnitudes."""
    m, n = 20000, 70
    gen = np.random.Generator(np.random.Philox(17))
    x = gen.integers(0, 3, size=(m, n)).astype(np.int8)
    v = gen.standard_normal(m) * scale
    v[::7] *= 1e-6  # mixed magnitudes inside one lane's rows
    v[5::97] = 0.0
    dev = torch.device("cuda:0")
    XP = torch.from_numpy(orc.pack_genotypes_u2(x).ravel(order="F")).to(dev)
    vd = torch.from_numpy(v).to(dev)
    b = torch.zeros(n, dtype=torch.float32, device=dev)
    _, gp = _xbeta_grad(XP, _lib.BS_U2, b, vd, torch.float32)
    want = x.astype(np.float64).T @ v.astype(np.float32).astype(np.float64)
    sc = np.abs(x).astype(np.float64).T @ np.abs(v)
    assert np.all(np.isfinite(gp))
    assert np.max(np.abs(gp - want) / sc) < 2e-5


@pytest.mark.gpu
@pytest.mark.parametrize("scale", [1e-38, 1e-20, 1.0, 1e25])
def test_packed_xbeta_any_beta_scale(scale):
    """The packed scn-m kernel scales beta by a power of two per CTA (subnormal widening)."""
    m, n = 9000, 300
    gen = np.random.Generator(np.random.Philox(19))
    x = gen.integers(0, 3, size=(m, n)).astype(np.int8)
    beta = (gen.standard_normal(n) * scale).astype(np.float32)
    beta[::5] *= np.float32(1e-5)
    beta[3::11] = 0.0
    dev = torch.device("cuda:0")
    XP = torch.from_numpy(orc.pack_genotypes_u2(x).ravel(order="F")).to(dev)
    b = torch.from_numpy(beta).to(dev)
    xbp, _ = _xbeta_grad(XP, _lib.BS_U2, b, torch.zeros(m, dtype=torch.float64, device=dev), torch.float32)
    bh = beta.astype(np.float64)
    want = x.astype(np.float64) @ bh
    sc = np.abs(x).astype(np.float64) @ np.abs(bh) + 1e-300
    assert np.all(np.isfinite(xbp))
    if scale > 1e-30:
        assert np.max(np.abs(xbp - want) / sc) < 2e-5
    else:  # |beta| below 2^-104: subnormal products, absolute error <= 2^-127 per product
        assert np.max(np.abs(xbp - want)) < n * 2.0 ** -127


@pytest.mark.gpu
def test_packed_more_ranks_than_columns():
    """Ranks that own no columns (partition_of gives them empty blocks) still join every
    collective; the fit equals the one-rank fit."""
    m, n, seed = 2000, 3, 5
    y = np.floor(np.arange(m, 0, -1) / 4.0)
    delta = (np.random.Generator(np.random.Philox(8)).random(m) < 0.5).astype(np.float64)

    def fn(comm):
        a = bs.genotype_fill(bs.PackedGenotypes(comm, (m, n)), seed)
        st = bs.cox_init(a, y, delta, lam=1e-6, sigma=1e-5, ties="breslow", dtype=np.float32)
        bs.cox_fit(st, 5)
        return np.asarray(st.trace), bs.gather_full(st.beta), bs.gather_full(a)

    one = bs.run_inproc(1, fn)[0]
    for got in bs.run_inproc(5, fn):
        np.testing.assert_allclose(got[0], one[0], rtol=1e-6)
        np.testing.assert_allclose(got[1], one[1], rtol=1e-5, atol=1e-9)
        np.testing.assert_array_equal(got[2], orc.genotype_fill(m, n, seed))


@pytest.mark.gpu
def test_packed_genotypes_write_as_int8_dsta(tmp_path):
    from paper_2010_16114_b200 import io as bio

    m, n = 301, 17
    path = tmp_path / "g.dsta"

    def fn(comm):
        p = bs.genotype_fill(bs.PackedGenotypes(comm, (m, n)), 9)
        bio.write_matrix(path, p)
        comm.barrier()
        return bs.gather_full(bio.read_matrix(path, comm, dtype=np.int8))

    for got in bs.run_inproc(3, fn):
        np.testing.assert_array_equal(got, orc.genotype_fill(m, n, 9))


def _transpose_dev(XP, m, n):
    ldt = bs.packed_bytes_per_column(n)
    Q = torch.full((ldt * m,), 0xAA, dtype=torch.uint8, device=XP.device)  # pad bytes must come out zero
    _lib.call("bs_genotype_transpose_packed", _lib.ptr(XP), m, n, _lib.ptr(Q), _lib.stream_ptr())
    return Q


@pytest.mark.gpu
@pytest.mark.parametrize("m,n", [(1, 3), (15, 4), (65, 9), (130, 129), (1000, 33), (8193, 5), (300, 1000)])
def test_transpose_packed_matches_oracle(m, n):
    """bs_genotype_transpose_packed: the packed block of X^T, byte for byte (pad bits zero)."""
    x = np.random.Generator(np.random.Philox(5 * m + n)).integers(0, 3, size=(m, n)).astype(np.int8)
    XP = torch.from_numpy(orc.pack_genotypes_u2(x).ravel(order="F")).to("cuda:0")
    got = _transpose_dev(XP, m, n).cpu().numpy()
    np.testing.assert_array_equal(got, orc.pack_genotypes_u2(np.ascontiguousarray(x.T)).ravel(order="F"))


@pytest.mark.gpu
@pytest.mark.parametrize("m,n", [(100, 7), (4096, 65), (20000, 300), (9000, 1), (700, 5000)])
def test_packed_transpose_xbeta_float64(m, n):
    """X beta from the packed transpose with float64 beta: 32 base-8 digits (94 bits of each
    2048-column group's maximum), i.e. float64 accuracy even with a 1e9 spread inside a group."""
    gen = np.random.Generator(np.random.Philox(13 * m + n))
    x = gen.integers(0, 3, size=(m, n)).astype(np.int8)
    beta = gen.standard_normal(n)
    beta[::3] *= 1e-9
    dev = torch.device("cuda:0")
    Q = _transpose_dev(torch.from_numpy(orc.pack_genotypes_u2(x).ravel(order="F")).to(dev), m, n)
    b = torch.from_numpy(beta).to(dev)
    ws = torch.zeros(max(_lib.query("bs_cox_xbeta_workspace", _lib.BS_U2T, m, n), 256), dtype=torch.uint8, device=dev)
    xb = torch.zeros(m, dtype=torch.float64, device=dev)
    _lib.call("bs_cox_xbeta", _lib.ptr(Q), _lib.BS_U2T, _lib.ptr(b), _lib.BS_F64, m, n, _lib.ptr(xb), _lib.ptr(ws),
              ws.numel(), _lib.stream_ptr())
    got = xb.cpu().numpy()
    want = x.astype(np.float64) @ beta
    sc = np.abs(x).astype(np.float64) @ np.abs(beta) + 1e-300
    assert np.max(np.abs(got - want) / sc) < 1e-14


@pytest.mark.gpu
@pytest.mark.parametrize("m,n", [(100, 7), (4096, 65), (20000, 300), (9000, 1), (700, 5000)])
def test_packed_transpose_xbeta_tensor_cores(m, n):
    """X beta from the packed transpose (BS_U2T) on the tensor cores (kind::mxf4, exact sums of
    46-bit beta digits): 1e-9 of sum |x beta| against a float64 X beta, and the packed
    float32 ring kernel within its 2e-5."""
    gen = np.random.Generator(np.random.Philox(7 * m + n))
    x = gen.integers(0, 3, size=(m, n)).astype(np.int8)
    beta = gen.standard_normal(n).astype(np.float32)
    beta[::3] *= np.float32(1e-4)
    dev = torch.device("cuda:0")
    XP = torch.from_numpy(orc.pack_genotypes_u2(x).ravel(order="F")).to(dev)
    Q = _transpose_dev(XP, m, n)
    b = torch.from_numpy(beta).to(dev)
    v = torch.zeros(m, dtype=torch.float64, device=dev)
    bs.gemm_path_counts(reset=True)
    ws = torch.zeros(max(_lib.query("bs_cox_xbeta_workspace", _lib.BS_U2T, m, n), 256), dtype=torch.uint8, device=dev)
    xb = torch.zeros(m + 1, dtype=torch.float64, device=dev)
    _lib.call("bs_cox_xbeta", _lib.ptr(Q), _lib.BS_U2T, _lib.ptr(b), _lib.BS_F32, m, n, _lib.ptr(xb), _lib.ptr(ws),
              ws.numel(), _lib.stream_ptr())
    assert bs.gemm_path_counts()["cox_packed_tensor"] == 1
    xbt = xb[:m].cpu().numpy()
    xbp, _ = _xbeta_grad(XP, _lib.BS_U2, b, v, torch.float32)
    bh = beta.astype(np.float64)
    want = x.astype(np.float64) @ bh
    sc = np.abs(x).astype(np.float64) @ np.abs(bh) + 1e-300
    assert np.max(np.abs(xbt - want) / sc) < 1e-9  # beta rounded to 46 bits of its 2048-column group max
    assert np.max(np.abs(xbp - xbt) / sc) < 2e-5


@pytest.mark.gpu
@pytest.mark.parametrize("scale", [1e-38, 1e-20, 1.0, 1e25])
def test_packed_transpose_xbeta_any_beta_scale(scale):
    """The tensor-core X beta scales each 2048-column group of beta by a power of two in float64,
    so tiny and huge beta keep the 46-bit digits."""
    m, n = 9000, 300
    gen = np.random.Generator(np.random.Philox(19))
    x = gen.integers(0, 3, size=(m, n)).astype(np.int8)
    beta = (gen.standard_normal(n) * scale).astype(np.float32)
    beta[::5] *= np.float32(1e-5)
    beta[3::11] = 0.0
    dev = torch.device("cuda:0")
    Q = _transpose_dev(torch.from_numpy(orc.pack_genotypes_u2(x).ravel(order="F")).to(dev), m, n)
    b = torch.from_numpy(beta).to(dev)
    ws = torch.zeros(max(_lib.query("bs_cox_xbeta_workspace", _lib.BS_U2T, m, n), 256), dtype=torch.uint8, device=dev)
    xb = torch.zeros(m, dtype=torch.float64, device=dev)
    _lib.call("bs_cox_xbeta", _lib.ptr(Q), _lib.BS_U2T, _lib.ptr(b), _lib.BS_F32, m, n, _lib.ptr(xb), _lib.ptr(ws),
              ws.numel(), _lib.stream_ptr())
    got = xb.cpu().numpy()
    bh = beta.astype(np.float64)
    want = x.astype(np.float64) @ bh
    sc = np.abs(x).astype(np.float64) @ np.abs(bh) + 1e-300
    assert np.all(np.isfinite(got))
    assert np.max(np.abs(got - want) / sc) < 1e-9


@pytest.mark.gpu
def test_cox_fit_packed_uses_transposed_xbeta():
    """cox_init keeps a packed transpose for float32 packed X, and cox_fit's X beta then takes
    the tensor-core pass (two packed tensor-core passes per iteration)."""
    m, n, seed, iters = 3000, 257, 11, 6
    y = np.floor(np.arange(m, 0, -1) / 4.0)
    delta = (np.random.Generator(np.random.Philox(2)).random(m) < 0.6).astype(np.float64)

    def fn(comm):
        a = bs.genotype_fill(bs.PackedGenotypes(comm, (m, n)), seed)
        st = bs.cox_init(a, y, delta, 1e-6, ties="breslow", dtype=np.float32)
        assert st._dev.get("xt") is not None
        bs.gemm_path_counts(reset=True)
        bs.cox_fit(st, iters)
        return bs.gemm_path_counts()["cox_packed_tensor"]

    assert bs.run_inproc(1, fn)[0] >= 2 * iters


@pytest.mark.gpu
@pytest.mark.parametrize("m", [5000, 20000])
def test_packed_tensor_core_grad_46_bits(m):
    """The packed gradient on the tensor cores (kind::mxf4) rounds v only to 46 bits of its
    2048-row group maximum: mixed magnitudes inside a group stay far below float32 error."""
    n = 300
    gen = np.random.Generator(np.random.Philox(23 + m))
    x = gen.integers(0, 3, size=(m, n)).astype(np.int8)
    v = gen.standard_normal(m)
    v[::3] *= 1e-6
    dev = torch.device("cuda:0")
    XP = torch.from_numpy(orc.pack_genotypes_u2(x).ravel(order="F")).to(dev)
    b = torch.zeros(n, dtype=torch.float32, device=dev)
    bs.gemm_path_counts(reset=True)
    _, gp = _xbeta_grad(XP, _lib.BS_U2, b, torch.from_numpy(v).to(dev), torch.float32)
    assert bs.gemm_path_counts()["cox_packed_tensor"] == 1
    want = x.astype(np.float64).T @ v
    sc = np.abs(x).astype(np.float64).T @ np.abs(v)
    assert np.max(np.abs(gp.astype(np.float64) - want) / sc) < 1e-7  # float32 output rounding dominates


@pytest.mark.gpu
def test_partial_loglik_float64_beta_on_packed_float32_state():
    """A float64 beta on a float32 packed state takes the packed ring kernel (the transpose
    pass takes float32 beta only) and agrees with the float32 beta."""
    m, n, seed = 2000, 65, 4
    y = np.floor(np.arange(m, 0, -1) / 4.0)
    delta = (np.random.Generator(np.random.Philox(6)).random(m) < 0.5).astype(np.float64)

    def fn(comm):
        a = bs.genotype_fill(bs.PackedGenotypes(comm, (m, n)), seed)
        st = bs.cox_init(a, y, delta, 1e-6, sigma=1e-5, ties="breslow", dtype=np.float32)
        bs.cox_fit(st, 3)
        b64 = bs.empty((n,), comm, np.float64)
        b64.local.copy_(st.beta.local.double())
        return bs.cox_partial_loglik(st), bs.cox_partial_loglik(st, b64)

    l32, l64 = bs.run_inproc(1, fn)[0]
    assert np.isfinite(l64)
    np.testing.assert_allclose(l64, l32, rtol=1e-5)


@pytest.mark.gpu
def test_packed_tensor_core_passes_propagate_nan():
    """A NaN in beta (X beta from the transpose) or in v (the gradient) gives NaN outputs, as
    float arithmetic would, not finite digits of a non-finite value."""
    m, n = 3000, 40
    gen = np.random.Generator(np.random.Philox(31))
    x = gen.integers(1, 3, size=(m, n)).astype(np.int8)  # no zero genotypes: every sum sees the NaN
    dev = torch.device("cuda:0")
    XP = torch.from_numpy(orc.pack_genotypes_u2(x).ravel(order="F")).to(dev)
    Q = _transpose_dev(XP, m, n)
    beta = torch.ones(n, dtype=torch.float32, device=dev)
    beta[7] = float("nan")
    ws = torch.zeros(max(_lib.query("bs_cox_xbeta_workspace", _lib.BS_U2T, m, n), 256), dtype=torch.uint8, device=dev)
    xb = torch.zeros(m, dtype=torch.float64, device=dev)
    _lib.call("bs_cox_xbeta", _lib.ptr(Q), _lib.BS_U2T, _lib.ptr(beta), _lib.BS_F32, m, n, _lib.ptr(xb), _lib.ptr(ws),
              ws.numel(), _lib.stream_ptr())
    assert torch.isnan(xb).all()


@pytest.mark.gpu
@pytest.mark.parametrize("p", [1, 2])
def test_cox_fit_packed_float64_matches_int8(p):
    """Packed genotypes in float64 arithmetic (both passes on the tensor cores with 32 digits)
    against int8 storage (exact CUDA-core float64 kernels): float64-level agreement, also with
    the columns split over two ranks (each rank's X beta partial from its own packed transpose)."""
    m, n, seed, iters = 3000, 257, 11, 12
    y = np.floor(np.arange(m, 0, -1) / 4.0)
    delta = (np.random.Generator(np.random.Philox(2)).random(m) < 0.6).astype(np.float64)

    def fn(comm, packed):
        a = bs.genotype_fill(bs.PackedGenotypes(comm, (m, n)) if packed else bs.empty((m, n), comm, np.int8), seed)
        st = bs.cox_init(a, y, delta, 1e-6, sigma=1e-5, ties="breslow", dtype=np.float64)
        if packed:
            assert st._dev.get("xt") is not None
        bs.gemm_path_counts(reset=True)
        bs.cox_fit(st, iters)
        return np.asarray(st.trace), bs.gather_full(st.beta), bs.gemm_path_counts()["cox_packed_tensor"]

    t8, b8, _ = bs.run_inproc(p, lambda c: fn(c, False))[0]
    tp, bp, passes = bs.run_inproc(p, lambda c: fn(c, True))[0]
    if p == 1:  # the path counter is process-wide, shared by the rank threads
        assert passes >= 2 * iters
    np.testing.assert_allclose(tp, t8, rtol=1e-12)
    np.testing.assert_allclose(bp, b8, rtol=1e-9, atol=1e-12 * np.abs(b8).max())


_NO_TC_SCRIPT = r"""
import sys, numpy as np, torch
import paper_2010_16114_b200 as bs
from paper_2010_16114_b200 import _lib
from oracle import blockstat_oracle as orc
m, n = 3000, 301
x = np.random.Generator(np.random.Philox(41)).integers(0, 3, size=(m, n)).astype(np.int8)
dev = torch.device("cuda:0")
XP = torch.from_numpy(orc.pack_genotypes_u2(x).ravel(order="F")).to(dev)
Q = torch.zeros(bs.packed_bytes_per_column(n) * m, dtype=torch.uint8, device=dev)
_lib.call("bs_genotype_transpose_packed", _lib.ptr(XP), m, n, _lib.ptr(Q), _lib.stream_ptr())
out = {}
for dt, code in ((torch.float32, _lib.BS_F32), (torch.float64, _lib.BS_F64)):
    beta = torch.from_numpy(np.random.Generator(np.random.Philox(42)).standard_normal(n)).to(dev, dt)
    ws = torch.zeros(_lib.query("bs_cox_xbeta_workspace", _lib.BS_U2T, m, n), dtype=torch.uint8, device=dev)
    xb = torch.zeros(m, dtype=torch.float64, device=dev)
    bs.gemm_path_counts(reset=True)
    _lib.call("bs_cox_xbeta", _lib.ptr(Q), _lib.BS_U2T, _lib.ptr(beta), code, m, n, _lib.ptr(xb), _lib.ptr(ws),
              ws.numel(), _lib.stream_ptr())
    out[str(dt)] = (xb.cpu().numpy(), beta.double().cpu().numpy(), bs.gemm_path_counts()["cox_packed_tensor"])
np.savez(sys.argv[1], x=x, **{k + "_xb": v[0] for k, v in out.items()}, **{k + "_b": v[1] for k, v in out.items()},
         **{k + "_tc": np.array(v[2]) for k, v in out.items()})
"""


@pytest.mark.gpu
def test_transposed_xbeta_without_tcgen05(tmp_path):
    """BS_DISABLE_TCGEN05=1: X beta from the packed transpose falls back to the CUDA-core packed
    kernel (same sums), in float32 and float64."""
    import os
    import subprocess
    import sys
    from pathlib import Path

    root = Path(__file__).resolve().parents[1]
    f = tmp_path / "notc.npz"
    env = dict(os.environ, BS_DISABLE_TCGEN05="1", PYTHONPATH=str(root))
    subprocess.run([sys.executable, "-c", _NO_TC_SCRIPT, str(f)], check=True, env=env, cwd=root, timeout=600)
    r = np.load(f)
    x = r["x"].astype(np.float64)
    for dt, tol in (("torch.float32", 2e-6), ("torch.float64", 1e-13)):
        b = r[dt + "_b"]
        want = x @ b
        sc = np.abs(x) @ np.abs(b)
        assert int(r[dt + "_tc"]) == 0  # the tensor-core path did not run
        assert np.max(np.abs(r[dt + "_xb"] - want) / sc) < tol
