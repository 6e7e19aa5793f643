"""Time bs_pairwise_euclidean at C3 scale (1000-dim points, n = 100,000) and check a sample vs fp64."""
import sys
import numpy as np
import torch
sys.path.insert(0, ".")
from paper_2010_16114_b200 import _lib
d, n = 1000, int(sys.argv[1]) if len(sys.argv) > 1 else 100000
g = torch.Generator(device="cuda"); g.manual_seed(3)
x = torch.rand(n, d, generator=g, device="cuda")  # point i = row i (x[i*d + k])
Y = torch.empty(n, n, device="cuda")
ev = [torch.cuda.Event(enable_timing=True) for _ in range(2)]
ev[0].record()
_lib.call("bs_pairwise_euclidean", _lib.ptr(x), 0, d, n, 0, n, _lib.ptr(Y), _lib.stream_ptr())
ev[1].record(); torch.cuda.synchronize()
idx = torch.randint(0, n, (2000,), generator=g, device="cuda")
jdx = torch.randint(0, n, (2000,), generator=g, device="cuda")
ref = (x[idx].double() - x[jdx].double()).norm(dim=1)
got = Y.view(-1)[jdx * n + idx].double()
ref[idx == jdx] = 0
print(f"pairwise n={n} d={d}: {ev[0].elapsed_time(ev[1]):.1f} ms, max rel err {((got - ref).abs() / ref.clamp_min(1e-30)).max().item():.2e}")
