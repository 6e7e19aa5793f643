"""GPU: the tcgen05 3xTF32 skinny GEMMs (nmf_tc.cu) against float64 numpy products.

3xTF32 keeps hi*hi + hi*lo + lo*hi of the tf32 split, so the products must land
at float32-level accuracy (not tf32's 1e-3): checked at 2e-6 relative to the
magnitude of the output (measured ~2e-6 with two-block TMEM groups).
"""

import ctypes

import numpy as np
import pytest

import paper_2010_16114_b200 as bs
from paper_2010_16114_b200 import _lib

pytestmark = pytest.mark.gpu


def _t(a):
    import torch

    return torch.from_numpy(np.ascontiguousarray(a)).cuda()


def _wxt(x, w):
    """P (r x m) = W X^T via bs_nmf_wxt; x is m x n (column-major block), w is r x n."""
    import torch

    m, n = x.shape
    r = w.shape[0]
    X = _t(x.T)            # memory [j][i] = column-major m x n
    W = _t(w.T)            # memory [j][k]
    P = torch.empty(m * r, dtype=torch.float32, device="cuda")
    ws = torch.zeros(_lib.query("bs_nmf_wxt_workspace", _lib.BS_F32, m, n, r), dtype=torch.uint8, device="cuda")
    _lib.call("bs_nmf_wxt", _lib.ptr(X), _lib.ptr(W), _lib.BS_F32, m, n, r, _lib.ptr(P), None, _lib.ptr(ws),
              ws.numel(), _lib.stream_ptr())
    return P.cpu().numpy().reshape(m, r).T


@pytest.mark.parametrize("m,n,r", [(128, 32, 4), (256, 64, 20), (1000, 777, 60), (4096, 96, 64), (384, 5000, 96),
                                   (520, 300, 128), (131072, 40, 32), (200, 33, 36)])
def test_wxt_3xtf32_accuracy(m, n, r):
    gen = np.random.Generator(np.random.Philox(m + n + r))
    x = gen.random((m, n), dtype=np.float32)
    w = gen.random((r, n), dtype=np.float32)
    got = _wxt(x, w)
    want = w.astype(np.float64) @ x.astype(np.float64).T
    err = np.abs(got - want).max() / np.abs(want).max()
    assert err < 4e-6, err


@pytest.mark.parametrize("m,n,r,algo", [(2048, 1024, 60, 1), (1000, 600, 20, 0), (4000, 130, 32, 1), (512, 4096, 64, 0)])
def test_nmf_f32_tcgen05_path_matches_float64(m, n, r, algo):
    """Both tcgen05 GEMMs inside full NMF iterations vs the float64 oracle on the same float32 data."""
    from oracle import blockstat_oracle as orc

    x = orc.rand_fill_common((m, n), 31 + r, np.float32)
    vt0, w0 = orc.nmf_init(x, r, 32 + r)

    def fn(comm):
        xd = bs.distribute(x if comm.rank == 0 else None, comm)
        st = bs.nmf_init(xd, r, seed=1)
        st.Vt.local[...] = bs.distribute(vt0 if comm.rank == 0 else None, comm).local
        st.W.local[...] = bs.distribute(w0 if comm.rank == 0 else None, comm).local
        (bs.nmf_multiplicative if algo == 0 else bs.nmf_apg)(st, 5)
        return np.asarray(st.trace), bs.gather_full(st.Vt), bs.gather_full(st.W)

    tr, vt, w = bs.run_inproc(1, fn)[0]
    f = orc.nmf_multiplicative if algo == 0 else orc.nmf_apg
    ovt, ow, otr = f(x.astype(np.float64), vt0.astype(np.float64), w0.astype(np.float64), 5)
    np.testing.assert_allclose(tr, otr, rtol=2e-5)
    assert np.abs(vt - ovt).max() <= 2e-5 * np.abs(ovt).max()
    assert np.abs(w - ow).max() <= 2e-5 * np.abs(ow).max()
