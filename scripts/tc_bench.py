"""Accuracy + speed of bs_nmf_wxt / w_step GEMMs at a realistic size (env: BS_TC_GROUP, BS_DISABLE_TCGEN05)."""
import os, sys, json
import numpy as np
import torch
sys.path.insert(0, ".")
from paper_2010_16114_b200 import _lib

def run(m, n, r, reps=5):
    g = torch.Generator(device="cuda"); g.manual_seed(1)
    X = torch.rand(n, m, generator=g, device="cuda")       # memory [j][i]: column-major m x n
    W = torch.rand(n, r, generator=g, device="cuda")       # memory [j][k]
    P = torch.empty(m * r, device="cuda")
    ws = torch.zeros(_lib.query("bs_nmf_wxt_workspace", 0, m, n, r), dtype=torch.uint8, device="cuda")
    args = (_lib.ptr(X), _lib.ptr(W), 0, m, n, r, _lib.ptr(P), _lib.ptr(ws), ws.numel(), _lib.stream_ptr())
    _lib.call("bs_nmf_wxt", *args); torch.cuda.synchronize()
    # accuracy on a row sample
    rows = torch.arange(0, m, max(1, m // 512), device="cuda")
    want = (W.double().t() @ X[:, rows].double())            # r x rows
    got = P.view(m, r)[rows].t().double()
    err = ((got - want).abs().max() / want.abs().max()).item()
    e0, e1 = torch.cuda.Event(True), torch.cuda.Event(True)
    e0.record()
    for _ in range(reps): _lib.call("bs_nmf_wxt", *args)
    e1.record(); torch.cuda.synchronize()
    ms = e0.elapsed_time(e1) / reps
    gbs = m * n * 4 / (ms * 1e-3) / 1e9
    return dict(m=m, n=n, r=r, err=err, ms=ms, GBs=gbs)

out = {"group": os.environ.get("BS_TC_GROUP", "2"), "tc": os.environ.get("BS_DISABLE_TCGEN05", "0") != "1"}
out["cases"] = [run(*c) for c in [(200000, 12500, 60), (200000, 100000, 60), (10000, 10000, 20), (100000, 20000, 20)]]
print(json.dumps(out), flush=True)
