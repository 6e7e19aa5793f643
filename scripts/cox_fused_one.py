"""One fused Cox pass (bs_cox_grad_xbeta, allow_fused=1) at 100000 x 20000 fp32, for ncu."""
import sys
import torch
sys.path.insert(0, ".")
from paper_2010_16114_b200 import _lib
m, n = 100000, 20000
g = torch.Generator(device="cuda"); g.manual_seed(1)
X = torch.randn(n, m, generator=g, device="cuda")
v = torch.randn(m, generator=g, device="cuda", dtype=torch.float64)
beta = torch.randn(n, generator=g, device="cuda") * 0.01
grad = torch.empty_like(beta)
xb = torch.empty(m + 1, dtype=torch.float64, device="cuda")
flags = torch.zeros(1, dtype=torch.int32, device="cuda")
ws = torch.zeros(_lib.query("bs_cox_grad_xbeta_workspace", 0, m, n), dtype=torch.uint8, device="cuda")
fused = int(sys.argv[1]) if len(sys.argv) > 1 else 1
ev = [torch.cuda.Event(enable_timing=True) for _ in range(2)]
for it in range(4):
    if it == 3: ev[0].record()
    _lib.call("bs_cox_grad_xbeta", _lib.ptr(X), 0, _lib.ptr(v), 0, m, n, _lib.ptr(grad), _lib.ptr(beta), 1e-6, 1e-8,
              _lib.ptr(xb), _lib.ptr(flags), fused, _lib.ptr(ws), ws.numel(), _lib.stream_ptr())
ev[1].record(); torch.cuda.synchronize()
print("fused" if fused else "two-pass", f"{ev[0].elapsed_time(ev[1]):.3f} ms for {m * n * 4 / 1e9:.1f} GB")
