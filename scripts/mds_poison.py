"""Run the tcgen05 MDS parity case after filling the caching allocator's free blocks with a
pattern (uninitialized-read check): traces must not depend on what memory held before."""
import sys
import numpy as np
import torch
sys.path.insert(0, ".")
sys.path.insert(0, "tests")
import paper_2010_16114_b200 as bs
from oracle import blockstat_oracle as orc
from test_mds_gpu import _run

n, q, p = (int(a) for a in (sys.argv[1:4] if len(sys.argv) > 3 else (516, 8, 2)))
x = orc.rand_fill_common((12, n), 80 + q, np.float32)
y = orc.pairwise_euclidean(x)
th0 = orc.mds_init(y, q, 90 + q)
oth, otr = orc.mds_fit(y.astype(np.float64), th0.astype(np.float64), 6)
for pat in (None, 0.0, 1.0e20, float("nan"), 3.7):
    if pat is not None:
        blocks = [torch.full((1 << 24,), pat, device="cuda") for _ in range(16)]
        del blocks
    tr, th = bs.run_inproc(p, _run, y, th0, 6)[0]
    print(pat, "max trace rel err", np.max(np.abs(np.asarray(tr) - otr) / np.abs(otr)), flush=True)
