"""Time cox_fit(st, 10) calls at C4 size with the X beta reuse on / off (host and device clocks)."""
import os
import sys
import time
import numpy as np
import torch
sys.path.insert(0, ".")
import paper_2010_16114_b200 as bs

comm = bs.init("inproc:1")[0]
m, n = 100_000, 200_000
x = bs.empty((m, n), comm, np.float32)
g = torch.Generator(device="cuda"); g.manual_seed(2012)
x.local.normal_(generator=g)
y = np.arange(m, 0, -1, dtype=np.float64)
delta = (np.random.Generator(np.random.Philox(2013)).random(m) > 0.3).astype(np.float64)
st = bs.cox_init(x, y, delta, lam=1e-8, sigma=1e-7)
bs.cox_fit(st, 3)
for mode in ("1", "0", "1", "0"):
    os.environ["BS_COX_REUSE"] = mode
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    t0 = time.perf_counter()
    e0.record()
    bs.cox_fit(st, 10)
    e1.record()
    torch.cuda.synchronize()
    print(f"reuse={mode}: device {e0.elapsed_time(e1):.1f} ms, host {1e3 * (time.perf_counter() - t0):.1f} ms", flush=True)
