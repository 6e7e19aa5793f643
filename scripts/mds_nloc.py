"""Time bs_mds_pass (tcgen05, float32) at n = 100,000 for several local column counts
(the per-GPU block at 1, 2, 4, 8 GPUs), with random Y / theta (timing only)."""
import sys
import torch
sys.path.insert(0, ".")
from paper_2010_16114_b200 import _lib

n, q = 100_000, 20
theta = torch.rand(n, q, device="cuda") * 2 - 1   # column i of theta = theta[i] (q contiguous)
for n_loc in (100_000, 50_000, 25_000, 12_500):
    Y = torch.rand(n_loc, n, device="cuda") + 0.5    # column j of Y contiguous
    red = torch.zeros(2, dtype=torch.float64, device="cuda")
    zsum = torch.zeros(n_loc, dtype=torch.float32, device="cuda")
    T = torch.zeros(n_loc, q, dtype=torch.float32, device="cuda")
    ws = torch.zeros(_lib.query("bs_mds_pass_workspace", 0, n, n_loc, q), dtype=torch.uint8, device="cuda")
    lo = 0
    ev = [torch.cuda.Event(enable_timing=True) for _ in range(2)]
    for it in range(4):
        if it == 1:
            ev[0].record()
        _lib.call("bs_mds_pass", _lib.ptr(Y), _lib.ptr(theta), 0, n, lo, n_loc, q, 0, 0, _lib.ptr(red), _lib.ptr(zsum),
                  _lib.ptr(T), _lib.ptr(ws), ws.numel(), _lib.stream_ptr())
    ev[1].record()
    torch.cuda.synchronize()
    ms = ev[0].elapsed_time(ev[1]) / 3
    print(f"n_loc={n_loc}: {ms:.3f} ms per pass, {n * n_loc * 4 / ms / 1e9:.2f} TB/s", flush=True)
    del Y, ws
    torch.cuda.empty_cache()
