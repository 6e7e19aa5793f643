"""Debug probe for the tcgen05 GEMM: structured inputs reveal layout errors."""
import sys
import numpy as np
import torch
sys.path.insert(0, ".")
from paper_2010_16114_b200 import _lib

def wxt(x, w):
    m, n = x.shape; r = w.shape[0]
    X = torch.from_numpy(np.ascontiguousarray(x.T)).cuda()
    W = torch.from_numpy(np.ascontiguousarray(w.T)).cuda()
    P = torch.full((m * r,), -7.0, dtype=torch.float32, device="cuda")
    ws = torch.zeros(_lib.query("bs_nmf_wxt_workspace", 0, m, n, r), dtype=torch.uint8, device="cuda")
    _lib.call("bs_nmf_wxt", _lib.ptr(X), _lib.ptr(W), 0, m, n, r, _lib.ptr(P), _lib.ptr(ws), ws.numel(), _lib.stream_ptr())
    torch.cuda.synchronize()
    return P.cpu().numpy().reshape(m, r).T

np.set_printoptions(linewidth=200, precision=1, suppress=True)
m, n, r = 128, 32, 32
i = np.arange(m)[:, None]; j = np.arange(n)[None, :]
x = (i + 1000 * j).astype(np.float32)        # X[i, j]
w = np.eye(r, n, dtype=np.float32)            # W[k, j] = [k == j]
got = wxt(x, w)                                # want P[k, i] = X[i, k] = i + 1000 k
want = w @ x.T
print("max err", np.abs(got - want).max())
print("got[:4,:8]\n", got[:4, :8]); print("want[:4,:8]\n", want[:4, :8])
print("got[:4, 32:40]\n", got[:4, 32:40])
print("got col0 rows 0..8 (k):", got[:8, 0])
# second probe: X = ones, W = ones -> every entry = n
got2 = wxt(np.ones((m, n), np.float32), np.ones((r, n), np.float32))
print("ones probe unique:", np.unique(got2)[:10])
# third probe: W = ones, X[i,j] = 1 only for j == 0
x3 = np.zeros((m, n), np.float32); x3[:, 0] = np.arange(m)
got3 = wxt(x3, np.ones((r, n), np.float32))
print("probe3 (P[k,i]=i):", got3[0, :16], got3[5, 100:108])
