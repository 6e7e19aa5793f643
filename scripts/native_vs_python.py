"""C1 (NMF-MU 10k x 10k r=20 float64) and C4-shaped Cox: the Python host loop vs the
native solver loop (runtime.*_run) over the same kernels; device time per iteration."""
import sys
import time
import numpy as np
import torch
sys.path.insert(0, ".")
import paper_2010_16114_b200 as bs
from paper_2010_16114_b200 import runtime

comm = bs.init("inproc:1")[0]
x = bs.empty((10_000, 10_000), comm, np.float64)
bs.rand_fill(x, seed=2010, common_init=True)
st = bs.nmf_init(x, 20, seed=2011)
ctx = runtime.Context(comm)
for name, fn in (("python", lambda k: bs.nmf_multiplicative(st, k)), ("native", lambda k: runtime.nmf_run(ctx, st, k, algo="mu")),
                 ("python", lambda k: bs.nmf_multiplicative(st, k)), ("native", lambda k: runtime.nmf_run(ctx, st, k, algo="mu"))):
    fn(3)
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    fn(200)
    e1.record()
    torch.cuda.synchronize()
    print(f"C1 NMF-MU f64 {name}: {200 / (time.perf_counter() - t0):.1f} it/s (device {200 / e0.elapsed_time(e1) * 1e3:.1f})",
          flush=True)
ctx.close()
