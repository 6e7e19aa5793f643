"""Per-entry-point device time of C2 NMF-APG iterations (CUDA events around every C-ABI call)."""
import sys
import numpy as np
import torch
sys.path.insert(0, ".")
import paper_2010_16114_b200 as bs
from paper_2010_16114_b200 import _lib
m, n, r = (int(a) for a in sys.argv[1:4]) if len(sys.argv) > 3 else (200000, 100000, 60)
comm = bs.init("inproc:1")[0]
x = bs.empty((m, n), comm, np.float32)
bs.rand_fill(x, seed=2010, common_init=True)
st = bs.nmf_init(x, r, seed=2011)
bs.nmf_apg(st, 3)
names = [k for k in _lib.SIGNATURES if not k.endswith("_workspace")]
ev = [torch.cuda.Event(enable_timing=True) for _ in range(2)]
with _lib.profile(names) as prof:
    ev[0].record()
    bs.nmf_apg(st, 5)
    ev[1].record()
torch.cuda.synchronize()
tot = ev[0].elapsed_time(ev[1]) / 5
print(f"{tot:.2f} ms per iteration")
for k, v in sorted(prof.elapsed_ms().items(), key=lambda kv: -sum(kv[1])):
    if v:
        print(f"  {k:28s} {len(v):3d} calls  {np.sum(v) / 5:8.3f} ms/iter")
