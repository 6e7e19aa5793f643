"""One wxt (or w_step) GEMM launch at a C2-like size, for ncu."""
import sys
import torch
sys.path.insert(0, ".")
from paper_2010_16114_b200 import _lib
which = sys.argv[1] if len(sys.argv) > 1 else "wxt"
m, n, r = 200000, 12500, 60
g = torch.Generator(device="cuda"); g.manual_seed(1)
X = torch.rand(n, m, generator=g, device="cuda")
if which == "wxt":
    W = torch.rand(n, r, generator=g, device="cuda")
    P = torch.empty(m * r, device="cuda")
    ws = torch.zeros(_lib.query("bs_nmf_wxt_workspace", 0, m, n, r), dtype=torch.uint8, device="cuda")
    for _ in range(3):
        _lib.call("bs_nmf_wxt", _lib.ptr(X), _lib.ptr(W), 0, m, n, r, _lib.ptr(P), _lib.ptr(ws), ws.numel(), _lib.stream_ptr())
else:
    Vt = torch.rand(m, r, generator=g, device="cuda")
    W = torch.rand(n, r, generator=g, device="cuda")
    VtV = torch.rand(r * r, dtype=torch.float64, device="cuda")
    red = torch.zeros(r * r + 1, dtype=torch.float64, device="cuda")
    ws = torch.zeros(_lib.query("bs_nmf_w_step_workspace", 0, m, n, r), dtype=torch.uint8, device="cuda")
    for _ in range(3):
        _lib.call("bs_nmf_w_step", 1, _lib.ptr(X), _lib.ptr(Vt), _lib.ptr(W), _lib.ptr(VtV), 0, m, n, r, 1e-10,
                  _lib.ptr(red), _lib.ptr(ws), ws.numel(), _lib.stream_ptr())
torch.cuda.synchronize()
print("ok")
