"""One MDS pass at n=20000, q=20 float32 (for ncu)."""
import sys
import numpy as np
import torch
sys.path.insert(0, ".")
import paper_2010_16114_b200 as bs
comm = bs.init("inproc:1")[0]
n, q = 20000, 20
pts = bs.empty((50, n), comm, np.float32)
bs.rand_fill(pts, seed=1, common_init=True)
y = bs.empty((n, n), comm, np.float32)
bs.pairwise_euclidean(y, pts)
st = bs.mds_init(y, q, seed=2)
bs.mds_fit(st, 3)
torch.cuda.synchronize()
print("ok", st.trace[-1])
