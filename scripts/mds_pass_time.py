"""Debug-build experiment: time bs_mds_pass at C3 with theta reset before every iteration, so
work-skipping modes that corrupt the update (BS_MDS_TC_MODE) still time a realistic pass."""
import os
import sys

import numpy as np
import torch

sys.path.insert(0, ".")
import paper_2010_16114_b200 as bs  # noqa: E402
from paper_2010_16114_b200 import _lib  # noqa: E402

n = int(os.environ.get("MDS_N", "100000"))
comm = bs.init("inproc:1")[0]
torch.cuda.set_device(comm.device)
pts = bs.empty((1000, n), comm, np.float32)
bs.rand_fill(pts, seed=2014, common_init=True)
y = bs.empty((n, n), comm, np.float32)
bs.pairwise_euclidean(y, pts)
del pts
st = bs.mds_init(y, 20, seed=2015)
saved = st.theta.local.clone()
times = []
for it in range(8):
    st.theta.local.copy_(saved)
    with _lib.profile(["bs_mds_pass"]) as prof:
        try:
            bs.mds_fit(st, 1)
        except Exception:  # noqa: BLE001 - modes that skip work may produce degenerate updates
            pass
        torch.cuda.synchronize()
    if it >= 2:
        times += prof.elapsed_ms()["bs_mds_pass"]
print(f"mode={os.environ.get('BS_MDS_TC_MODE', '0')} pass={np.mean(times):.2f} ms", flush=True)
