"""Debug-build experiment: C2 GEMM launch time and SM clock with parts of the i8 kernel skipped.

BS_I8_MODE bits (only honoured by a -DBS_DEBUG_MODES build): 1 no conversion, 2 no MMAs,
4 no factor-image loads, 8 no X loads.  Prints ms per bs_nmf_wxt / bs_nmf_w_step launch and
the median SM clock while they run."""
import os
import sys
import time

import numpy as np
import torch

sys.path.insert(0, ".")
import paper_2010_16114_b200 as bs  # noqa: E402
from paper_2010_16114_b200 import _lib  # noqa: E402
from bench import Clocks  # noqa: E402

comm = bs.init("inproc:1")[0]
torch.cuda.set_device(comm.device)
x = bs.empty((200000, 100000), comm, np.float32)
bs.rand_fill(x, seed=2010, common_init=True)
st = bs.nmf_init(x, 60, seed=2011)
bs.nmf_apg(st, 2)
with Clocks(0) as clk, _lib.profile(["bs_nmf_wxt", "bs_nmf_w_step"]) as prof:
    bs.nmf_apg(st, 6)
    torch.cuda.synchronize()
el = prof.elapsed_ms()
print(f"mode={os.environ.get('BS_I8_MODE', '0')} wxt={np.mean(el['bs_nmf_wxt']):.2f} ms "
      f"w_step={np.mean(el['bs_nmf_w_step']):.2f} ms clocks={clk.summary()}", flush=True)
