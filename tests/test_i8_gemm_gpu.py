"""GPU: the integer digit-slice tcgen05 GEMMs (nmf_i8.cu) — accuracy, bias, path selection.

Float32 NMF GEMMs run as exact int32 accumulations of 8-bit digit products of
block-scaled operands (3 digits each, 512-wide scale groups).  The only rounding is
each value's round-to-nearest to 24 bits relative to its block maximum and the
float32 fold of the group partials, so the error is unbiased; the bar below is
float32-level: 2e-6 of the output magnitude (the reference's own float32 sgemm error
is of the same order), and the mean signed error is checked to be ~0.
"""

import numpy as np
import pytest
import torch

import paper_2010_16114_b200 as bs
from paper_2010_16114_b200 import _lib

pytestmark = pytest.mark.gpu


def _t(a):
    return torch.from_numpy(np.ascontiguousarray(a)).cuda()


def _prepare(X, m, n):
    stats = torch.zeros(6, dtype=torch.float64, device="cuda")
    xs = torch.empty(max(_lib.query("bs_nmf_xscale_bytes", m, n), 16), dtype=torch.uint8, device="cuda")
    ws = torch.zeros(_lib.query("bs_nmf_prepare_workspace", m, n), dtype=torch.uint8, device="cuda")
    _lib.call("bs_nmf_prepare", _lib.ptr(X), _lib.BS_F32, m, n, _lib.ptr(stats), _lib.ptr(xs), _lib.ptr(ws),
              ws.numel(), _lib.stream_ptr())
    return stats.cpu().numpy(), xs


def wxt_i8(x, w):
    """P (r x m) = W X^T through bs_nmf_wxt with prepared scales; x is m x n, w is r x n."""
    m, n = x.shape
    r = w.shape[0]
    X = _t(x.T)
    W = _t(w.T)
    stats, xs = _prepare(X, m, n)
    P = torch.empty(m * r, dtype=torch.float32, device="cuda")
    ws = torch.zeros(_lib.query("bs_nmf_wxt_workspace", _lib.BS_F32, m, n, r), dtype=torch.uint8, device="cuda")
    _lib.call("bs_nmf_wxt", _lib.ptr(X), _lib.ptr(W), _lib.BS_F32, m, n, r, _lib.ptr(P), _lib.ptr(xs), _lib.ptr(ws),
              ws.numel(), _lib.stream_ptr())
    return P.cpu().numpy().reshape(m, r).T, stats


def vtx_i8(x, vt):
    """C (r x n) = Vt X through the W half-step's GEMM (bs_nmf_w_step with MU and a zero W: returns VtX)."""
    m, n = x.shape
    r = vt.shape[0]
    X = _t(x.T)
    stats, xs = _prepare(X, m, n)
    # APG with W = 0, VtV = 0 and eps = 1: tau = 1 and W_new = max(0, 0 - (0 - VtX)) = VtX.
    W = torch.zeros(n * r, dtype=torch.float32, device="cuda")
    VtV = torch.zeros(r * r, dtype=torch.float64, device="cuda")
    red = torch.zeros(r * r + 1, dtype=torch.float64, device="cuda")
    ws = torch.zeros(_lib.query("bs_nmf_w_step_workspace", _lib.BS_F32, m, n, r), dtype=torch.uint8, device="cuda")
    eps = 1.0
    _lib.call("bs_nmf_w_step", _lib.BS_NMF_APG, _lib.ptr(X), _lib.ptr(_t(vt.T)), _lib.ptr(W), _lib.ptr(VtV),
              _lib.BS_F32, m, n, r, eps, _lib.ptr(red), _lib.ptr(xs), _lib.ptr(ws), ws.numel(), _lib.stream_ptr())
    return W.cpu().numpy().reshape(n, r).T


DISTS = ["uniform", "loguniform", "sparse", "integers"]


def _data(kind, shape, gen):
    if kind == "uniform":
        return gen.random(shape, dtype=np.float32)
    if kind == "loguniform":  # values over 2^-20 .. 1 inside every scale group
        return np.exp2(-20.0 * gen.random(shape)).astype(np.float32)
    if kind == "sparse":
        a = gen.random(shape, dtype=np.float32)
        a[gen.random(shape) < 0.9] = 0.0
        return a
    return np.floor(gen.random(shape) * 256.0).astype(np.float32)  # exact ties everywhere


@pytest.mark.parametrize("kind", DISTS)
@pytest.mark.parametrize("m,n,r", [(128, 32, 4), (1000, 777, 60), (4096, 96, 64), (131072, 40, 32), (200, 1500, 36)])
def test_wxt_integer_path_accuracy(kind, m, n, r):
    gen = np.random.Generator(np.random.Philox(m * 7 + n + r))
    x = _data(kind, (m, n), gen)
    w = gen.random((r, n), dtype=np.float32)
    bs.gemm_path_counts(reset=True)
    got, stats = wxt_i8(x, w)
    assert bs.gemm_path_counts()["integer"] == 1
    want = w.astype(np.float64) @ x.astype(np.float64).T
    err = np.abs(got - want).max() / np.abs(want).max()
    assert err < 2e-6, err
    assert stats[0] == x.min()
    np.testing.assert_allclose(stats[1], np.sum(x.astype(np.float64) ** 2), rtol=1e-7)  # float32 partials of 32 squares
    assert stats[2] == 0.0 and stats[3] == 1.0


@pytest.mark.parametrize("kind", DISTS)
@pytest.mark.parametrize("m,n,r", [(1000, 777, 60), (70000, 200, 64), (512, 4096, 20)])
def test_vtx_integer_path_accuracy(kind, m, n, r):
    gen = np.random.Generator(np.random.Philox(m + 3 * n + r))
    x = _data(kind, (m, n), gen)
    vt = gen.random((r, m), dtype=np.float32)
    bs.gemm_path_counts(reset=True)
    got = vtx_i8(x, vt)
    assert bs.gemm_path_counts()["integer"] == 1
    want = vt.astype(np.float64) @ x.astype(np.float64)
    err = np.abs(got - want).max() / np.abs(want).max()
    assert err < 2e-6, err


def test_integer_path_is_unbiased():
    """Mean signed relative error over many outputs ~0 (the 3xTF32 accumulator truncates: ~-1e-6)."""
    gen = np.random.Generator(np.random.Philox(99))
    m, n, r = 8192, 20000, 64
    x = gen.random((m, n), dtype=np.float32)
    w = gen.random((r, n), dtype=np.float32)
    got, _ = wxt_i8(x, w)
    want = w.astype(np.float64) @ x.astype(np.float64).T
    rel = (got - want) / want
    assert abs(rel.mean()) < 2e-8, rel.mean()
    assert np.abs(rel).max() < 1e-6


def test_prepare_flags_nonfinite_and_negative():
    m, n = 512, 600
    x = np.random.Generator(np.random.Philox(5)).random((m, n), dtype=np.float32)
    x[7, 9] = np.inf
    stats, _ = _prepare(_t(x.T), m, n)
    assert stats[2] == 1.0
    x[7, 9] = -2.0
    stats, _ = _prepare(_t(x.T), m, n)
    assert stats[0] == -2.0 and stats[2] == 0.0


def test_supported_shapes_take_the_integer_path():
    """float32 NMF with r <= 64 and m % 4 == 0 runs both GEMMs on the integer tensor-core path."""
    from oracle import blockstat_oracle as orc

    x = orc.rand_fill_common((2048, 1024), 5, np.float32)

    def fn(comm):
        xd = bs.distribute(x if comm.rank == 0 else None, comm)
        st = bs.nmf_init(xd, 60, seed=6)
        bs.gemm_path_counts(reset=True)
        bs.nmf_apg(st, 3)
        return bs.gemm_path_counts()

    c = bs.run_inproc(1, fn)[0]
    assert c["integer"] == 6 and c["tf32"] == 0 and c["cuda_core"] == 0, c


def test_negative_initial_factor_falls_back_to_tf32():
    from oracle import blockstat_oracle as orc

    x = orc.rand_fill_common((1024, 512), 7, np.float32)
    vt0, w0 = orc.nmf_init(x, 20, 8)
    w0[3, 5] = -0.25

    def fn(comm):
        xd = bs.distribute(x if comm.rank == 0 else None, comm)
        st = bs.nmf_init(xd, 20, seed=1)
        st.Vt.local[...] = bs.distribute(vt0 if comm.rank == 0 else None, comm).local
        st.W.local[...] = bs.distribute(w0 if comm.rank == 0 else None, comm).local
        bs.gemm_path_counts(reset=True)
        bs.nmf_apg(st, 2)
        return bs.gemm_path_counts(), np.asarray(st.trace), bs.gather_full(st.Vt), bs.gather_full(st.W)

    c, tr, vt, w = bs.run_inproc(1, fn)[0]
    assert c["integer"] == 0 and c["tf32"] == 4, c
    ovt, ow, otr = orc.nmf_apg(x.astype(np.float64), vt0.astype(np.float64), w0.astype(np.float64), 2)
    np.testing.assert_allclose(tr, otr, rtol=1e-5)
