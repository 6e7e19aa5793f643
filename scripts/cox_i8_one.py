"""Time the int8 Cox passes (float32 arithmetic) at 400,000 x 100,000 (40 GB) on one GPU."""
import sys
import torch
sys.path.insert(0, ".")
from paper_2010_16114_b200 import _lib
m, n = 400000, 100000
g = torch.Generator(device="cuda"); g.manual_seed(1)
X = torch.empty(n, m, dtype=torch.int8, device="cuda")
for c in range(0, n, 4096):
    X[c:c + 4096] = torch.randint(0, 3, (min(4096, n - c), m), generator=g, device="cuda", dtype=torch.int8)
v = torch.randn(m, generator=g, device="cuda", dtype=torch.float64)
beta = torch.randn(n, generator=g, device="cuda") * 1e-3
grad = torch.empty_like(beta)
xb = torch.empty(m + 1, dtype=torch.float64, device="cuda")
flags = torch.zeros(1, dtype=torch.int32, device="cuda")
wg = torch.zeros(_lib.query("bs_cox_grad_workspace", 3, m, n), dtype=torch.uint8, device="cuda")
wx = torch.zeros(_lib.query("bs_cox_xbeta_workspace", 3, m, n), dtype=torch.uint8, device="cuda")
ev = [torch.cuda.Event(enable_timing=True) for _ in range(3)]
for it in range(3):
    ev[0].record()
    _lib.call("bs_cox_grad_step", _lib.ptr(X), 3, _lib.ptr(v), 0, m, n, _lib.ptr(grad), _lib.ptr(beta), 1e-6, 0.0, 0,
              _lib.ptr(xb[m:]), _lib.ptr(flags), _lib.ptr(wg), wg.numel(), _lib.stream_ptr())
    ev[1].record()
    _lib.call("bs_cox_xbeta", _lib.ptr(X), 3, _lib.ptr(beta), 0, m, n, _lib.ptr(xb), _lib.ptr(wx), wx.numel(),
              _lib.stream_ptr())
    ev[2].record()
torch.cuda.synchronize()
gb = m * n / 1e9
tg, tx = ev[0].elapsed_time(ev[1]), ev[1].elapsed_time(ev[2])
print(f"int8 grad {tg:.2f} ms ({gb / tg:.2f} TB/s), xbeta {tx:.2f} ms ({gb / tx:.2f} TB/s)")
