"""Debug: per-tile error of the integer wxt GEMM at a multi-unit shape."""
import sys
import numpy as np
sys.path.insert(0, ".")
sys.path.insert(0, "tests")
from test_i8_gemm_gpu import wxt_i8, vtx_i8

m, n, r = [int(a) for a in sys.argv[1:4]]
gen = np.random.Generator(np.random.Philox(1))
x = gen.random((m, n), dtype=np.float32)
w = gen.random((r, n), dtype=np.float32)
got, st = wxt_i8(x, w)
want = w.astype(np.float64) @ x.astype(np.float64).T
err = np.abs(got - want) / np.abs(want).max()
tiles = (m + 127) // 128
pt = err.max(axis=0)[: tiles * 128].reshape(-1, 128).max(axis=1) if m % 128 == 0 else None
bad = np.nonzero(pt > 1e-5)[0]
print("max err", err.max(), "bad tiles", len(bad), "of", tiles, bad[:40])
print("bad tile -> cta", (bad % 148)[:40], "unit idx in cta", (bad // 148)[:40])
cols = err.max(axis=1)
print("per-k max err", np.round(cols[:8], 6))
