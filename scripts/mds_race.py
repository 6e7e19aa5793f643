"""Repeat the tcgen05 MDS parity case many times; any run-to-run difference is a race."""
import sys
import numpy as np
sys.path.insert(0, ".")
sys.path.insert(0, "tests")
import paper_2010_16114_b200 as bs
from oracle import blockstat_oracle as orc
from test_mds_gpu import _run

n, q, p, reps = (int(a) for a in (sys.argv[1:5] if len(sys.argv) > 4 else (516, 8, 2, 40)))
x = orc.rand_fill_common((12, n), 80 + q, np.float32)
y = orc.pairwise_euclidean(x)
th0 = orc.mds_init(y, q, 90 + q)
oth, otr = orc.mds_fit(y.astype(np.float64), th0.astype(np.float64), 6)
ref = None
errs = []
diff = 0
for r in range(reps):
    tr, th = bs.run_inproc(p, _run, y, th0, 6)[0]
    tr = np.asarray(tr)
    errs.append(np.max(np.abs(tr - otr) / np.abs(otr)))
    if ref is None:
        ref = (tr, th)
    elif not (np.array_equal(tr, ref[0]) and np.array_equal(th, ref[1])):
        diff += 1
print(f"n={n} q={q} p={p}: {diff}/{reps - 1} runs differ from run 0; max rel err {max(errs):.3g}, "
      f"median {np.median(errs):.3g}", flush=True)
