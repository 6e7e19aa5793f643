import sys, os
import numpy as np
import torch
sys.path.insert(0, ".")
from paper_2010_16114_b200 import _lib
def wxt(x, w):
    m, n = x.shape; r = w.shape[0]
    X = torch.from_numpy(np.ascontiguousarray(x.T)).cuda(); W = torch.from_numpy(np.ascontiguousarray(w.T)).cuda()
    P = torch.full((m * r,), -7.0, dtype=torch.float32, device="cuda")
    ws = torch.zeros(_lib.query("bs_nmf_wxt_workspace", 0, m, n, r), dtype=torch.uint8, device="cuda")
    _lib.call("bs_nmf_wxt", _lib.ptr(X), _lib.ptr(W), 0, m, n, r, _lib.ptr(P), _lib.ptr(ws), ws.numel(), _lib.stream_ptr())
    torch.cuda.synchronize()
    return P.cpu().numpy().reshape(m, r).T
for (m, n, r) in [(128, 64, 32), (128, 96, 32), (128, 160, 32), (128, 320, 32), (128, 1024, 32), (256, 1024, 32), (128, 64, 64), (128, 64, 60), (128, 320, 64), (1000, 777, 60)]:
    gen = np.random.Generator(np.random.Philox(1))
    x = gen.random((m, n), dtype=np.float32); w = gen.random((r, n), dtype=np.float32)
    got = wxt(x, w); want = w.astype(np.float64) @ x.astype(np.float64).T
    err = np.abs(got - want) / np.abs(want).max()
    bad = np.argwhere(err > 1e-5)
    print(f"m={m} n={n} r={r}: maxrel={err.max():.3e} nbad={len(bad)} first={bad[:3].tolist()} ratio={np.median(got/want):.4f}", flush=True)
