"""Debug-build experiment: C3 MDS pass time and SM clock with parts of mds_tc_kernel skipped.

BS_MDS_TC_MODE bits (only honoured by a -DBS_DEBUG_MODES build): 1 no pair math, 2 no MMAs.
Prints ms per bs_mds_pass launch and the median SM clock."""
import os
import sys

import numpy as np
import torch

sys.path.insert(0, ".")
import paper_2010_16114_b200 as bs  # noqa: E402
from paper_2010_16114_b200 import _lib  # noqa: E402
from bench import Clocks  # noqa: E402

n = int(os.environ.get("MDS_N", "100000"))
comm = bs.init("inproc:1")[0]
torch.cuda.set_device(comm.device)
pts = bs.empty((1000, n), comm, np.float32)
bs.rand_fill(pts, seed=2014, common_init=True)
y = bs.empty((n, n), comm, np.float32)
bs.pairwise_euclidean(y, pts)
del pts
st = bs.mds_init(y, 20, seed=2015)
try:
    bs.mds_fit(st, 2)
except Exception as exc:  # noqa: BLE001 - modes that skip work may produce degenerate updates
    print("warm-up:", type(exc).__name__)
with Clocks(0) as clk, _lib.profile(["bs_mds_pass"]) as prof:
    try:
        bs.mds_fit(st, 6)
    except Exception as exc:  # noqa: BLE001
        print("run:", type(exc).__name__)
    torch.cuda.synchronize()
el = prof.elapsed_ms()
print(f"mode={os.environ.get('BS_MDS_TC_MODE', '0')} pass={np.mean(el['bs_mds_pass']):.2f} ms "
      f"({40e9 * (n / 1e5) ** 2 / (np.mean(el['bs_mds_pass']) * 1e-3) / 1e12:.2f} TB/s) clocks={clk.summary()}",
      flush=True)
