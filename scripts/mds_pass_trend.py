"""Per-pass time of bs_mds_pass over a C3 fit (theta evolving), to see whether the pass slows as
the embedding spreads (more 16-pair slices on the out-of-line cancellation path)."""
import os
import sys

import numpy as np
import torch

sys.path.insert(0, ".")
import paper_2010_16114_b200 as bs  # noqa: E402
from paper_2010_16114_b200 import _lib  # noqa: E402

n = int(os.environ.get("MDS_N", "100000"))
iters = int(os.environ.get("MDS_ITERS", "60"))
comm = bs.init("inproc:1")[0]
torch.cuda.set_device(comm.device)
pts = bs.empty((1000, n), comm, np.float32)
bs.rand_fill(pts, seed=2014, common_init=True)
y = bs.empty((n, n), comm, np.float32)
bs.pairwise_euclidean(y, pts)
del pts
st = bs.mds_init(y, 20, seed=2015)
reset = os.environ.get("MDS_RESET_AT")  # restore theta of this iteration before every pass
saved = None
times = []
for it in range(iters):
    if reset is not None and it == int(reset):
        saved = st.theta.local.clone()
    if saved is not None:
        st.theta.local.copy_(saved)
    if os.environ.get("MDS_IDLE_AT") and it == int(os.environ["MDS_IDLE_AT"]):
        import time
        time.sleep(float(os.environ.get("MDS_IDLE_S", "5")))  # let the device idle
    with _lib.profile(["bs_mds_pass"]) as prof:
        bs.mds_fit(st, 1)
        torch.cuda.synchronize()
    times += prof.elapsed_ms()["bs_mds_pass"]
    if it % 5 == 0:
        th = st.theta.local.float()
        nrm = (th * th).sum(0)
        print(f"iter {it:3d} pass {times[-1]:.3f} ms  stress {st.trace[-1]:.6g}  max|theta|^2 {nrm.max().item():.4g}",
              flush=True)
t = np.array(times)
print("mean by decile:", " ".join(f"{x:.2f}" for x in [t[i * len(t) // 10:(i + 1) * len(t) // 10].mean() for i in range(10)]))
