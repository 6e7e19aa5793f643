"""Time bs_reduce / bs_nmf_scan over an 80 GB fp32 block (the nmf_init / _nmf_check passes)."""
import sys
import torch
sys.path.insert(0, ".")
from paper_2010_16114_b200 import _lib
n = 20_000_000_000
x = torch.empty(n, dtype=torch.float32, device="cuda").uniform_()
out = torch.zeros(2, dtype=torch.float64, device="cuda")
ws = torch.zeros(1 << 20, dtype=torch.uint8, device="cuda")
ev = [torch.cuda.Event(enable_timing=True) for _ in range(3)]
for _ in range(2):
    ev[0].record()
    _lib.call("bs_reduce", _lib.ptr(x), 0, n, 3, 0, _lib.ptr(out), _lib.ptr(ws), ws.numel(), _lib.stream_ptr())
    ev[1].record()
    _lib.call("bs_nmf_scan", _lib.ptr(x), 0, n, _lib.ptr(out), _lib.ptr(ws), ws.numel(), _lib.stream_ptr())
    ev[2].record()
torch.cuda.synchronize()
print(f"reduce {ev[0].elapsed_time(ev[1]):.2f} ms ({80 / ev[0].elapsed_time(ev[1]):.2f} TB/s), "
      f"scan {ev[1].elapsed_time(ev[2]):.2f} ms ({80 / ev[1].elapsed_time(ev[2]):.2f} TB/s)")
