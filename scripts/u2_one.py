"""Time the Cox passes on the same 400,000 x 100,000 genotype matrix stored int8 (40 GB)
and 2-bit packed (10 GB), float32 arithmetic; prints genotypes/s and GB/s per pass."""
import sys
import numpy as np
import torch
sys.path.insert(0, ".")
import paper_2010_16114_b200 as bs
from paper_2010_16114_b200 import _lib
m, n = 400000, int(sys.argv[1]) if len(sys.argv) > 1 else 100000
which = sys.argv[2] if len(sys.argv) > 2 else "both"
comm = bs.init("inproc:1")[0]
v = torch.randn(m, device="cuda", dtype=torch.float64)
beta = torch.randn(n, device="cuda") * 1e-3
grad = torch.empty_like(beta)
xb = torch.empty(m + 1, dtype=torch.float64, device="cuda")
flags = torch.zeros(1, dtype=torch.int32, device="cuda")
for code, name in ((_lib.BS_U2, "u2"), (_lib.BS_I8, "int8")):
    if which not in ("both", name):
        continue
    x = bs.PackedGenotypes(comm, (m, n)) if code == _lib.BS_U2 else bs.empty((m, n), comm, np.int8)
    bs.genotype_fill(x, 2016)
    X = x.local
    wg = torch.zeros(_lib.query("bs_cox_grad_workspace", code, m, n), dtype=torch.uint8, device="cuda")
    wx = torch.zeros(_lib.query("bs_cox_xbeta_workspace", code, m, n), dtype=torch.uint8, device="cuda")
    ev = [torch.cuda.Event(enable_timing=True) for _ in range(3)]
    for it in range(3):
        ev[0].record()
        _lib.call("bs_cox_grad_step", _lib.ptr(X), code, _lib.ptr(v), 0, m, n, _lib.ptr(grad), _lib.ptr(beta), 1e-6,
                  0.0, 0, _lib.ptr(xb[m:]), _lib.ptr(flags), _lib.ptr(wg), wg.numel(), _lib.stream_ptr())
        ev[1].record()
        _lib.call("bs_cox_xbeta", _lib.ptr(X), code, _lib.ptr(beta), 0, m, n, _lib.ptr(xb), _lib.ptr(wx), wx.numel(),
                  _lib.stream_ptr())
        ev[2].record()
    torch.cuda.synchronize()
    gb = X.numel() / 1e9
    tg, tx = ev[0].elapsed_time(ev[1]), ev[1].elapsed_time(ev[2])
    gg = m * n / 1e9
    print(f"{name}: grad {tg:.2f} ms ({gb / tg:.2f} TB/s, {gg / tg:.2f} Tgeno/s), "
          f"xbeta {tx:.2f} ms ({gb / tx:.2f} TB/s, {gg / tx:.2f} Tgeno/s)", flush=True)
    del x, X, wg, wx
    torch.cuda.empty_cache()
