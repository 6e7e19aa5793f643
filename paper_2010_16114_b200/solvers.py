"""NMF, MDS and l1-Cox solvers on B200 (drop-in for blockstat solvers.py).

Same entry points, state dataclasses, trace semantics and exceptions as the
reference (solvers.py:40-450).  Every per-iteration flop runs in the fused
CUDA kernels of ``libbsb200.so`` on the data blocks resident in HBM; the host
only sequences kernels and the few small collectives the algorithms need:

NMF per iteration (solvers.py:144-185)
    bs_nmf_wxt (X pass 1) -> reduce-scatter(r*m) -> bs_nmf_vt_step
    -> allgather(Vt), allreduce(r^2) -> bs_nmf_w_step (X pass 2; also forms the
    next iteration's W W^T and the objective cross term) -> allreduce(r^2+1)
    -> bs_nmf_objective.  The m x n residual buffer of the reference
    (solvers.py:91, 131) is never allocated: the objective uses the Gram
    identity ||X - V^T W||^2 = ||X||^2 - 2<VtX, W> + <VtV, WWt>.
MDS per iteration (solvers.py:269-305)
    allgather(theta) -> bs_mds_pass (single pass over Y) -> allreduce(2)
    -> bs_mds_update.  No n x n temporary.
Cox per iteration (solvers.py:422-450)
    bs_cox_xbeta (X pass 1) -> allreduce(m+1, packs ||beta||_1) -> bs_cox_risk
    -> bs_cox_objective -> bs_cox_pi_delta (computed redundantly, no
    allreduce) -> bs_cox_grad_step (X pass 2 + prox).

Traces are accumulated on the device and copied to the host once per call,
except when a ConvergenceMonitor needs each value (solvers.py:443).  Error
conditions (negative NMF data, coincident MDS points, nonfinite Cox weights)
are detected on the device and raised with the reference's exception types and
trace contents.
"""

from __future__ import annotations

import ctypes
from dataclasses import dataclass, field
import os
import warnings

import numpy as np

from . import _lib
from .comm import ReduceOp
from .distarray import (
    DistArray,
    _flat_local,
    empty,
    local_reduce,
    partition_of,
    rand_fill,
    to_fortran_tensor,
    torch_dtype,
    zeros,
)


class DegenerateConfigError(RuntimeError):
    """An embedding update hit coincident points (zero pairwise distance)."""


class NumericError(RuntimeError):
    """A solver produced nonfinite intermediate values."""


def _torch():
    import torch

    return torch


def soft_threshold(x, lam):
    """Shrink toward zero by ``lam``, zeroing the interval [-lam, lam] (solvers.py:48-51)."""
    torch = _torch()
    if isinstance(x, torch.Tensor):
        return torch.sign(x) * torch.clamp(torch.abs(x) - lam, min=0)
    x = np.asarray(x)
    return np.sign(x) * np.maximum(np.abs(x) - lam, 0)


@dataclass
class ConvergenceMonitor:
    """Windowed relative-change stopping rule over an objective trace (solvers.py:54-60)."""

    window: int = 10
    rel_tol: float = 1e-5
    history: list = field(default_factory=list)


def converged(monitor, f_new):
    """Record ``f_new``; True once the window-lagged relative change drops below ``rel_tol``."""
    h = monitor.history
    h.append(float(f_new))
    if len(h) <= monitor.window:
        return False
    return abs(h[-1] - h[-1 - monitor.window]) / (abs(h[-1]) + 1.0) < monitor.rel_tol


# ---------------------------------------------------------------------------
# helpers
# ---------------------------------------------------------------------------


class _Work:
    """Per-state device scratch, one zeroed slice per entry point (counters live inside)."""

    def __init__(self, device):
        self.device = device
        self.bufs = {}

    def get(self, name, nbytes):
        torch = _torch()
        nbytes = max(int(nbytes), 256)
        b = self.bufs.get(name)
        if b is None or b.numel() < nbytes:
            b = torch.zeros(nbytes, dtype=torch.uint8, device=self.device)
            self.bufs[name] = b
        return b

    def args(self, name, nbytes):
        b = self.get(name, nbytes)
        return _lib.ptr(b), b.numel()


def _at(t, index):
    """Pointer to element ``index`` of a contiguous device tensor."""
    return ctypes.c_void_p(t.data_ptr() + int(index) * t.element_size())


def _dev_f64(n, device):
    torch = _torch()
    return torch.zeros(max(int(n), 1), dtype=torch.float64, device=device)


# ---------------------------------------------------------------------------
# Nonnegative matrix factorization
# ---------------------------------------------------------------------------


@dataclass
class NmfState:
    """Factors (stored as Vt, W) plus the device workspaces (solvers.py:78-94).

    ``WWt``/``VtV`` are float64 device r x r Grams.  ``WWtVt``, ``VtVW`` and
    ``resid`` exist in the reference as materialized buffers; here they are
    fused into the half-step kernels and stay ``None``.  ``tmp`` is the
    gathered r x m factor (the all-gather target of scenario a).
    """

    X: DistArray
    Vt: DistArray
    W: DistArray
    WXt: DistArray
    WWt: object
    WWtVt: object
    VtX: object
    VtV: object
    VtVW: object
    resid: object
    tmp: object
    eps: float
    trace: list = field(default_factory=list)
    _dev: dict = field(default_factory=dict, repr=False)
    _work: object = field(default=None, repr=False)


def nmf_init(x, rank, seed=None, eps=1e-10):
    """Allocate NMF state with uniform(0, 1) factors (solvers.py:97-121)."""
    from .distarray import reduce_all

    if x.ndim != 2:
        raise ValueError("NMF expects a 2-D data matrix")
    if x.dtype.kind != "f":
        raise ValueError("NMF expects float32 or float64 data")
    if reduce_all(x, ReduceOp.MIN) < 0:
        raise ValueError("NMF requires nonnegative data")
    m, n = x.shape
    comm = x.comm
    dt = x.dtype
    vt = empty((rank, m), comm, dt)
    w = empty((rank, n), comm, dt)
    rand_fill(vt, seed=seed, common_init=True)
    rand_fill(w, seed=None if seed is None else seed + 1, common_init=True)
    dev = comm.device
    torch = _torch()
    red = _dev_f64(rank * rank + 1, dev)
    state = NmfState(
        X=x, Vt=vt, W=w,
        WXt=empty((rank, m), comm, dt),
        WWt=red[:rank * rank].view(rank, rank),
        WWtVt=None,
        VtX=None,
        VtV=_dev_f64(rank * rank, dev).view(rank, rank),
        VtVW=None,
        resid=None,
        tmp=(torch.empty((rank, m), dtype=torch_dtype(dt), device=dev).t().contiguous().t()
             if comm.size > 1 else None),
        eps=eps,
    )
    state._dev = {"red": red, "scan": _dev_f64(6, dev)}
    state._work = _Work(dev)
    return state


def _gather_factor(a, out):
    """All-gather a column-split r x k factor into the r x k buffer ``out``."""
    rows = a.shape[0]
    counts = [rows * c for c in a.partition.counts()]
    a.comm.allgatherv(_flat_local(a), out.t().reshape(-1) if out.ndim == 2 else out, counts)


# Cancellation guard of the Gram-identity objective (bs_nmf_objective): when
# ||X||^2 / obj exceeds kappa, the trace value is replaced by the reference's own
# direct residual (solvers.py:124-136).  The bound follows each GEMM path's error:
# the integer digit-slice path (exact int32 accumulation, symmetric rounding,
# ~1e-7 relative) and float64 stay within 1e-6 of the direct value up to these
# ratios; the 3xTF32 path's accumulator truncates (biased ~2e-6), so it always
# takes the direct residual.
_KAPPA_I8 = 16.0
_GRAPHS = os.environ.get("BS_NMF_GRAPH", "1") != "0"  # A/B switch: replay NMF iterations as CUDA graphs
_KAPPA_F64 = 1e6
_KAPPA_ALWAYS = -1.0


def _path_counts():
    buf = (ctypes.c_int64 * 8)()
    _lib.call("bs_gemm_path_counts", buf, 0)
    return list(buf)


def gemm_path_counts(reset=False):
    """How many NMF GEMMs (scn a / scn b) ran on each path since the last reset (bs_gemm_path_counts).

    Keys: ``integer`` (tcgen05 kind::i8 digit slices), ``tf32`` (tcgen05 3xTF32),
    ``cuda_core`` (float32 CUDA cores), ``float64`` (DMMA / CUDA cores); ``tensor`` = the
    first two together; ``mds_tensor`` / ``mds_cuda_core``: MDS passes (bs_mds_pass);
    ``cox_packed_tensor``: packed-genotype Cox passes (gradient, X beta) on the tensor cores (kind::mxf4).
    """
    import ctypes as C

    buf = (C.c_int64 * 8)()
    _lib.call("bs_gemm_path_counts", buf, 1 if reset else 0)
    d = {"integer": buf[0], "tf32": buf[1], "cuda_core": buf[2], "float64": buf[3], "mds_tensor": buf[4],
         "mds_cuda_core": buf[5], "cox_packed_tensor": buf[6]}
    d["tensor"] = d["integer"] + d["tf32"]
    return d


def _nmf_prepare(s):
    """The call's X pass (_nmf_check, solvers.py:139-141) + ||X||^2 + the integer GEMMs' block scales.

    Returns True when the float32 GEMMs may run on the integer digit-slice path:
    scales prepared, X finite and both factors nonnegative (the solver keeps them so).
    """
    torch = _torch()
    x = s.X
    comm = x.comm
    m = x.shape[0]
    n_loc = x.local.shape[1]
    flat = _flat_local(x)
    stats = s._dev["scan"]
    xs = None
    if x.dtype == np.float32:
        nb = _lib.query("bs_nmf_xscale_bytes", m, n_loc)
        xs = s._dev.get("xscale")
        if xs is None or xs.numel() < nb:
            xs = torch.empty(max(nb, 16), dtype=torch.uint8, device=comm.device)
            s._dev["xscale"] = xs
    wp, wn = s._work.args("prep", _lib.query("bs_nmf_prepare_workspace", m, n_loc))
    _lib.call("bs_nmf_prepare", _lib.ptr(flat), _lib.dtype_code(flat.dtype), m, n_loc, _lib.ptr(stats),
              _lib.ptr(xs), wp, wn, _lib.stream_ptr())
    local_reduce(s.Vt.local, ReduceOp.MIN, out=stats[4:5])
    local_reduce(s.W.local, ReduceOp.MIN, out=stats[5:6])
    if comm.size > 1:
        mins = torch.stack([stats[0], stats[4], stats[5], -stats[2]])
        comm.allreduce(mins, ReduceOp.MIN)
        sq = stats[1:2].clone()
        comm.allreduce(sq, ReduceOp.SUM)
        stats[0], stats[4], stats[5], stats[2] = mins[0], mins[1], mins[2], -mins[3]
        stats[1:2].copy_(sq)
    host = stats.cpu().numpy()
    if not (x.local.numel() == 0 and comm.size == 1) and host[0] < 0:
        raise ValueError("NMF requires nonnegative data")
    return bool(host[3] == 1.0 and host[2] == 0.0 and host[4] >= 0.0 and host[5] >= 0.0)


def _nmf_run(s, iters, trace_every, algo):
    torch = _torch()
    x = s.X
    comm = x.comm
    m, n = x.shape
    r = s.Vt.shape[0]
    code = _lib.dtype_code(x.dtype)
    m_loc = s.Vt.local.shape[1]
    n_loc = x.local.shape[1]
    use_i8 = _nmf_prepare(s)
    if iters <= 0:
        return s
    st = _lib.stream_ptr()
    dev = comm.device
    red = s._dev["red"]
    xsq = s._dev["scan"][1:2]
    xs = s._dev.get("xscale") if use_i8 else None
    VtV = s.VtV.reshape(-1)
    Xf = _flat_local(x)
    Wl = _flat_local(s.W)
    Vtl = _flat_local(s.Vt)
    # WWt of the entering W (scn d, solvers.py:151); later iterations reuse the
    # Gram the W half-step produces for its updated W.
    gp, gn = s._work.args("gram", _lib.query("bs_gram_workspace", r, n_loc))
    _lib.call("bs_gram", _lib.ptr(Wl), code, r, n_loc, _lib.ptr(red), gp, gn, st)
    if comm.size > 1:
        comm.allreduce(red[:r * r], ReduceOp.SUM)
    mcounts = [r * c for c in partition_of(m, comm.size).counts()]
    if comm.size > 1:
        P = s._dev.get("P")
        if P is None or P.numel() < r * m:
            P = torch.empty(r * m, dtype=torch_dtype(x.dtype), device=dev)
            s._dev["P"] = P
        tmp = s.tmp.t().reshape(-1)
    else:
        P = _flat_local(s.WXt)
        tmp = Vtl
    WXt_loc = _flat_local(s.WXt)
    trace_dev = _dev_f64(iters, dev)
    guard = s._dev.get("guard")
    if guard is None:
        guard = torch.zeros(2, dtype=torch.int32, device=dev)
        s._dev["guard"] = guard
    direct = s._dev["direct"] if "direct" in s._dev else _dev_f64(1, dev)
    s._dev["direct"] = direct
    if x.dtype == np.float64:
        kappa = _KAPPA_F64
    elif use_i8 and r <= 64:
        kappa = _KAPPA_I8
    else:
        kappa = _KAPPA_ALWAYS
    xp, xn = s._work.args("wxt", _lib.query("bs_nmf_wxt_workspace", code, m, n_loc, r))
    vp, vn = s._work.args("vt", _lib.query("bs_nmf_vt_step_workspace", r, m_loc))
    wp, wn = s._work.args("w", _lib.query("bs_nmf_w_step_workspace", code, m, n_loc, r))
    rp, rn = s._work.args("resid", _lib.query("bs_nmf_residual_workspace", m, n_loc))
    eps = float(s.eps)

    def iteration(tr, st):
        """One NMF iteration on stream `st`; the objective goes to device slot `tr` (None: no trace)."""
        # WXt = W X^T (scn b) and its reduce-scatter (distlinalg.py:246-252)
        _lib.call("bs_nmf_wxt", _lib.ptr(Xf), _lib.ptr(Wl), code, m, n_loc, r, _lib.ptr(P), _lib.ptr(xs), xp, xn, st)
        if comm.size > 1:
            comm.reduce_scatterv(P[:r * m], WXt_loc, mcounts)
        # Vt half-step (solvers.py:152-156 / 173-176)
        _lib.call("bs_nmf_vt_step", algo, _lib.ptr(Vtl), _lib.ptr(WXt_loc), _lib.ptr(red), code, r, m_loc, eps,
                  _lib.ptr(VtV), None, vp, vn, st)
        if comm.size > 1:
            comm.allreduce(VtV, ReduceOp.SUM)
            comm.allgatherv(Vtl, tmp, mcounts)
        # W half-step + next WWt + objective cross term (solvers.py:155-159 / 177-182)
        _lib.call("bs_nmf_w_step", algo, _lib.ptr(Xf), _lib.ptr(tmp), _lib.ptr(Wl), _lib.ptr(VtV), code, m,
                  n_loc, r, eps, _lib.ptr(red), _lib.ptr(xs), wp, wn, st)
        if comm.size > 1:
            comm.allreduce(red, ReduceOp.SUM)
        if tr is not None:
            _lib.call("bs_nmf_objective", _lib.ptr(xsq), _lib.ptr(red), _lib.ptr(VtV), r, tr, _lib.ptr(guard),
                      kappa, st)
            # cancellation regime: the reference's direct residual (solvers.py:124-136), skipped on the
            # device when the guard is clear
            _lib.call("bs_nmf_residual", _lib.ptr(Xf), _lib.ptr(tmp), _lib.ptr(Wl), code, m, n_loc, r,
                      _lib.ptr(direct), _lib.ptr(guard), rp, rn, st)
            if comm.size > 1:
                comm.allreduce(direct, ReduceOp.SUM)
            _lib.call("bs_nmf_objective_select", _lib.ptr(guard), _lib.ptr(direct), tr, st)

    # One rank, X under 4 GiB: after a first eager iteration (which also sets up kernel attributes
    # and tensor maps), the iteration is captured once as a CUDA graph (with / without the trace)
    # and replayed — C1's iteration is ~0.5 ms of ~10 launches, so launch gaps matter.  The traced
    # graph writes the objective to a fixed slot that is copied into the call's trace.
    # Only where launches matter: a C2-sized iteration (80 GB of X, ~30 ms) gains nothing.
    use_graph = comm.size == 1 and iters >= 3 and _GRAPHS and Xf.numel() * Xf.element_size() < (4 << 30)
    graphs = s._dev.setdefault("graphs", {})
    slot = s._dev.get("slot")
    if slot is None:
        slot = s._dev["slot"] = _dev_f64(1, dev)
    for it in range(iters):
        want = bool(trace_every and it % trace_every == 0)
        if not use_graph or it == 0:
            iteration(_at(trace_dev, it) if want else None, st)
            continue
        # every pointer and scalar the captured launches bake in
        key = (want, algo, kappa, eps, xp.value, vp.value, wp.value, rp.value,
               *(t.data_ptr() if t is not None else 0 for t in (Xf, Wl, Vtl, xs, P, tmp, red, VtV, direct, guard)))
        entry = graphs.get(key)
        if entry is None:
            g = torch.cuda.CUDAGraph()
            lib = _lib.load()
            n0, p0 = lib.bs_launch_count(), _path_counts()
            with torch.cuda.graph(g):
                iteration(_lib.ptr(slot) if want else None, _lib.stream_ptr())
            n, dp = lib.bs_launch_count() - n0, (ctypes.c_int64 * 8)(*(b - a for a, b in zip(p0, _path_counts())))
            lib.bs_note_replayed_launches(-n)  # captured, not run
            lib.bs_add_gemm_path_counts((ctypes.c_int64 * 8)(*(-v for v in dp)))
            entry = graphs[key] = (g, n, dp)
        entry[0].replay()
        _lib.load().bs_note_replayed_launches(entry[1])
        _lib.load().bs_add_gemm_path_counts(entry[2])
        if want:
            trace_dev[it:it + 1].copy_(slot)
    if trace_every:
        vals = trace_dev.cpu().numpy()
        s.trace.extend(float(vals[it]) for it in range(iters) if it % trace_every == 0)
    return s


def nmf_multiplicative(state, iters, trace_every=1):
    """Multiplicative updates; the objective is nonincreasing (solvers.py:144-162)."""
    return _nmf_run(state, iters, trace_every, _lib.BS_NMF_MU)


def nmf_apg(state, iters, trace_every=1):
    """Alternating projected gradient with Frobenius-norm step sizes (solvers.py:165-185)."""
    return _nmf_run(state, iters, trace_every, _lib.BS_NMF_APG)


def nmf_objective(x, vt, w, state=None):
    """Squared Frobenius norm of ``X - V W`` (V given transposed), direct residual (solvers.py:124-136)."""
    torch = _torch()
    comm = x.comm
    m, n = x.shape
    r = vt.shape[0]
    dev = comm.device
    code = _lib.dtype_code(x.dtype)
    if comm.size > 1:
        full = torch.empty(r * m, dtype=torch_dtype(vt.dtype), device=dev)
        comm.allgatherv(_flat_local(vt), full, [r * c for c in vt.partition.counts()])
    else:
        full = _flat_local(vt)
    out = _dev_f64(1, dev)
    work = state._work if state is not None else _Work(dev)
    n_loc = x.local.shape[1]
    wp, wn = work.args("resid", _lib.query("bs_nmf_residual_workspace", m, n_loc))
    _lib.call("bs_nmf_residual", _lib.ptr(_flat_local(x)), _lib.ptr(full), _lib.ptr(_flat_local(w)), code, m, n_loc,
              r, _lib.ptr(out), None, wp, wn, _lib.stream_ptr())
    if comm.size > 1:
        comm.allreduce(out, ReduceOp.SUM)
    return float(out.item())


# ---------------------------------------------------------------------------
# Multidimensional scaling
# ---------------------------------------------------------------------------


@dataclass
class MdsState:
    """Embedding (one point per column) plus the MM workspaces (solvers.py:193-206).

    ``theta_distances`` (the reference's second n x n buffer) is never
    allocated; ``d_dist`` holds the Z column sums and ``theta_WmZ`` the
    theta (W - Z) product of the last update, as in the reference.
    """

    Y: DistArray
    theta: DistArray
    theta_distances: object
    theta_WmZ: DistArray
    d_dist: DistArray
    d_local: np.ndarray
    W_sums: float
    tmp: object
    perturb: bool = False
    trace: list = field(default_factory=list)
    _dev: dict = field(default_factory=dict, repr=False)
    _work: object = field(default=None, repr=False)


def _replicated_diag(y):
    """diag_get into a replicated host vector (distlinalg.py:102-122)."""
    torch = _torch()
    n = y.shape[0]
    own = torch.empty(y.hi - y.lo, dtype=y.local.dtype, device=y.local.device)
    if own.numel():
        _lib.call("bs_diag_get", _lib.ptr(_flat_local(y)), _lib.dtype_code(y.dtype), n, y.lo, own.numel(),
                  _lib.ptr(own), _lib.stream_ptr())
    if y.comm.size > 1:
        full = torch.empty(n, dtype=own.dtype, device=own.device)
        y.comm.allgatherv(own, full, y.partition.counts())
        own = full
    return own.cpu().numpy().reshape(n, 1)


def mds_init(y, ndim, seed=None, perturb=False):
    """Allocate MDS state with a uniform embedding rescaled into (-1, 1) (solvers.py:209-234)."""
    if y.ndim != 2 or y.shape[0] != y.shape[1]:
        raise ValueError("MDS expects a square distance matrix")
    n = y.shape[0]
    if n < 2:
        raise ValueError("MDS needs at least two points")
    if y.dtype.kind != "f":
        raise ValueError("MDS expects float32 or float64 distances")
    comm = y.comm
    dt = y.dtype
    d_local = _replicated_diag(y)
    if np.any(d_local != 0):
        raise ValueError("target distance matrix must have a zero diagonal")
    theta = empty((ndim, n), comm, dt)
    rand_fill(theta, seed=seed, common_init=True)
    theta.local.mul_(2.0).sub_(1.0)  # solvers.py:224
    torch = _torch()
    dev = comm.device
    state = MdsState(
        Y=y, theta=theta,
        theta_distances=None,
        theta_WmZ=empty((ndim, n), comm, dt),
        d_dist=empty((1, n), comm, dt),
        d_local=d_local,
        W_sums=float(n - 1),
        tmp=(torch.empty((ndim, n), dtype=torch_dtype(dt), device=dev).t().contiguous().t()
             if comm.size > 1 else None),
        perturb=perturb,
    )
    state._dev = {"red": _dev_f64(2, dev), "flags": torch.zeros(1, dtype=torch.int32, device=dev)}
    state._work = _Work(dev)
    return state


def _theta_full(theta, tmp):
    if theta.comm.size == 1:
        return _flat_local(theta)
    flat = tmp.t().reshape(-1)
    theta.comm.allgatherv(_flat_local(theta), flat, [theta.shape[0] * c for c in theta.partition.counts()])
    return flat


def mds_stress(theta, y, state=None):
    """Weighted squared misfit between target and embedding distances (solvers.py:250-266)."""
    torch = _torch()
    comm = y.comm
    n = y.shape[0]
    q = theta.shape[0]
    dev = comm.device
    tmp = state.tmp if state is not None else (
        torch.empty((q, n), dtype=torch_dtype(theta.dtype), device=dev).t().contiguous().t()
        if comm.size > 1 else None)
    full = _theta_full(theta, tmp)
    red = _dev_f64(2, dev)
    work = state._work if state is not None else _Work(dev)
    n_loc = y.local.shape[1]
    wp, wn = work.args("mds", _lib.query("bs_mds_pass_workspace", _lib.dtype_code(y.dtype), n, n_loc, q))
    _lib.call("bs_mds_pass", _lib.ptr(_flat_local(y)), _lib.ptr(full), _lib.dtype_code(y.dtype), n, y.lo, n_loc, q,
              0, 1, _lib.ptr(red), None, None, wp, wn, _lib.stream_ptr())
    if comm.size > 1:
        comm.allreduce(red, ReduceOp.SUM)
    return float(red[0].item())


def mds_fit(state, iters, trace_every=1):
    """Majorization-minimization updates; stress is nonincreasing (solvers.py:269-305).

    The trace records the stress of the iterate entering each update.
    """
    s = state
    torch = _torch()
    y = s.Y
    comm = y.comm
    n = y.shape[0]
    q = s.theta.shape[0]
    if iters <= 0:
        return s
    dev = comm.device
    code = _lib.dtype_code(y.dtype)
    n_loc = y.local.shape[1]
    st = _lib.stream_ptr()
    red = s._dev["red"]
    flags = s._dev["flags"]
    flags.zero_()
    hist = _dev_f64(2 * iters, dev)
    Yf = _flat_local(y)
    th = _flat_local(s.theta)
    zsum = _flat_local(s.d_dist)
    T = _flat_local(s.theta_WmZ)
    wp, wn = s._work.args("mds", _lib.query("bs_mds_pass_workspace", code, n, n_loc, q))
    perturb = 1 if s.perturb else 0
    for it in range(iters):
        full = _theta_full(s.theta, s.tmp)
        _lib.call("bs_mds_pass", _lib.ptr(Yf), _lib.ptr(full), code, n, y.lo, n_loc, q, perturb, 0, _lib.ptr(red),
                  _lib.ptr(zsum), _lib.ptr(T), wp, wn, st)
        if comm.size > 1:
            comm.allreduce(red, ReduceOp.SUM)
        hist[2 * it:2 * it + 2].copy_(red)
        _lib.call("bs_mds_update", _lib.ptr(th), _lib.ptr(zsum), _lib.ptr(T), code, q, n_loc, s.W_sums,
                  _lib.ptr(red), perturb, _lib.ptr(flags), st)
    h = hist.cpu().numpy().reshape(iters, 2)
    failed = bool(int(flags.item()) & _lib.BS_FLAG_DEGENERATE)
    last = iters
    if failed:
        last = int(np.nonzero(h[:, 1] > 0)[0][0]) + 1
    if trace_every:
        s.trace.extend(float(h[it, 0]) for it in range(last) if it % trace_every == 0)
    if failed:
        raise DegenerateConfigError("coincident embedding points; rerun with perturb=True")
    return s


# ---------------------------------------------------------------------------
# L1-regularized Cox proportional hazards
# ---------------------------------------------------------------------------


@dataclass
class CoxState:
    """Covariates, survival outcome and proximal-gradient workspaces (solvers.py:313-329).

    ``y`` stays a host array; ``delta``, ``Xbeta``, ``w``, ``W``, ``pd`` and
    ``cuts`` are replicated device vectors.  ``X`` may hold float32, float64 or
    int8 (genotype) data; the solver arithmetic runs in ``beta``'s dtype.
    """

    X: DistArray
    y: np.ndarray
    delta: object
    beta: DistArray
    lam: float
    sigma: float
    Xbeta: object
    w: object
    W: object
    pd: object
    grad: DistArray
    cuts: object
    trace: list = field(default_factory=list)
    _dev: dict = field(default_factory=dict, repr=False)
    _work: object = field(default=None, repr=False)


def _tie_cuts(y):
    neg = -np.asarray(y, dtype=np.float64)
    return np.searchsorted(neg, neg, side="right").astype(np.int64) - 1


def cox_init(x, y, delta, lam, sigma=None, ties="none", dtype=None):
    """Allocate Cox state; the step size defaults to 1 / (2 ||X||_2^2) (solvers.py:337-373).

    ``dtype`` (an addition) selects the arithmetic dtype for int8 genotype X;
    it defaults to X's dtype for float X and float64 for int8.
    """
    from .distlinalg import opnorm

    torch = _torch()
    if x.ndim != 2:
        raise ValueError("Cox expects a 2-D covariate matrix")
    m, n = x.shape
    sdt = np.dtype(dtype) if dtype is not None else (x.dtype if x.dtype.kind == "f" else np.dtype(np.float64))
    y = np.asarray(y.cpu().numpy() if isinstance(y, torch.Tensor) else y, dtype=np.float64)
    delta_h = np.asarray(delta.cpu().numpy() if isinstance(delta, torch.Tensor) else delta, dtype=sdt)
    if y.shape != (m,) or delta_h.shape != (m,):
        raise ValueError("y and delta must have one entry per sample")
    if np.any(np.diff(y) > 0):
        raise ValueError("samples must be ordered by nonincreasing observed time")
    if not np.all((delta_h == 0) | (delta_h == 1)):
        raise ValueError("event indicators must be 0 or 1")
    if ties == "none":
        if np.any(np.diff(y) == 0):
            raise ValueError("tied observed times need ties='breslow'")
        cuts = np.arange(m, dtype=np.int64)
    elif ties == "breslow":
        cuts = _tie_cuts(y)
    else:
        raise ValueError(f"unknown tie mode {ties!r}")
    if sigma is None:
        norm2 = opnorm(x, "l2_power")
        sigma = 1.0 / (2.0 * norm2 * norm2)
    if sigma <= 0:
        raise ValueError("step size must be positive")
    comm = x.comm
    dev = comm.device
    tdt = torch_dtype(sdt)
    state = CoxState(
        X=x, y=y, delta=torch.from_numpy(delta_h).to(dev),
        beta=zeros((n,), comm, sdt),
        lam=float(lam), sigma=float(sigma),
        Xbeta=torch.empty(m, dtype=tdt, device=dev),
        w=torch.empty(m, dtype=tdt, device=dev),
        W=torch.empty(m, dtype=tdt, device=dev),
        pd=torch.empty(m, dtype=tdt, device=dev),
        grad=empty((n,), comm, sdt),
        cuts=torch.from_numpy(cuts).to(dev),
    )
    state._dev = {"xb": _dev_f64(m + 1, dev), "dmpd": _dev_f64(m, dev), "loglik": _dev_f64(1, dev),
                  "flags": torch.zeros(1, dtype=torch.int32, device=dev),
                  "no_ties": ties == "none"}
    state._work = _Work(dev)
    xt = _packed_transpose(x, sdt)
    if xt is not None:
        state._dev["xt"] = xt
    return state


_U2_XT = os.environ.get("BS_U2_XT", "1") != "0"  # A/B switch: X beta from a packed transpose


def _packed_transpose(x, sdt):
    """The packed transpose of a PackedGenotypes block (float32 / float64 arithmetic), or None.

    X beta then runs on the tensor cores (kind::mxf4) as the same K-major pass as the gradient
    (bs_genotype_transpose_packed).  It costs a second copy of the packed block, taken here
    (later in-place changes to X are not seen), so it is made only when the device keeps
    4 GiB free beside it; otherwise X beta stays on the CUDA-core ring kernel.
    """
    if not (_U2_XT and getattr(x, "packed", False) and sdt in (np.dtype(np.float32), np.dtype(np.float64))):
        return None
    torch = _torch()
    m, n_loc = x.shape[0], x.local.shape[1]
    if m == 0 or n_loc == 0 or x.comm.device.type != "cuda":
        return None
    ldt = _lib.query("bs_genotype_packed_bytes", n_loc)
    free, _ = torch.cuda.mem_get_info(x.comm.device)
    if ldt * m + (4 << 30) > free:
        return None
    xt = torch.empty(ldt * m, dtype=torch.uint8, device=x.comm.device)
    _lib.call("bs_genotype_transpose_packed", _lib.ptr(_flat_local(x)), m, n_loc, _lib.ptr(xt), _lib.stream_ptr())
    return xt


_EXP_CLAMP = {np.dtype(np.float64): 700.0, np.dtype(np.float32): 85.0}


def _cuts_ptr(s):
    return None if s._dev.get("no_ties") else _lib.ptr(s.cuts)


def _xbeta(s, beta_local):
    """xb[0:m] = X beta (reduced over ranks), xb[m] = ||beta||_1 (reduced)."""
    x = s.X
    comm = x.comm
    m = x.shape[0]
    n_loc = x.local.shape[1]
    xb = s._dev["xb"]
    st = _lib.stream_ptr()
    s._dev.pop("xb_beta", None)  # xb no longer holds a fused pass's partial
    local_reduce(beta_local, ReduceOp.SUM, _lib.BS_T_ABS, out=xb[m:m + 1])
    xt = s._dev.get("xt") if beta_local.dtype == s.beta.local.dtype else None  # the state's arithmetic
    xptr, xcode = (_lib.ptr(xt), _lib.BS_U2T) if xt is not None else (_lib.ptr(_flat_local(x)), _lib.xcode(x))
    wp, wn = s._work.args("xbeta", _lib.query("bs_cox_xbeta_workspace", xcode, m, n_loc))
    _lib.call("bs_cox_xbeta", xptr, xcode, _lib.ptr(beta_local), _lib.dtype_code(beta_local.dtype), m, n_loc,
              _lib.ptr(xb), wp, wn, st)
    if comm.size > 1:
        comm.allreduce(xb, ReduceOp.SUM)


def _risk(s):
    m = s.X.shape[0]
    clamp = _EXP_CLAMP[np.dtype(s.beta.dtype)]
    rp, rn = s._work.args("risk", _lib.query("bs_cox_risk_workspace", m))
    _lib.call("bs_cox_risk", _lib.ptr(s._dev["xb"]), _lib.ptr(s.delta), _cuts_ptr(s), _lib.dtype_code(s.beta.dtype),
              m, clamp, _lib.ptr(s.Xbeta), _lib.ptr(s.w), _lib.ptr(s.W), _lib.ptr(s._dev["loglik"]),
              _lib.ptr(s._dev["flags"]), rp, rn, _lib.stream_ptr())


def _raise_flags(flags_value):
    if flags_value & _lib.BS_FLAG_CLAMPED:
        warnings.warn("linear predictor clamped before exponentiation", RuntimeWarning, stacklevel=3)
    if flags_value & _lib.BS_FLAG_NONFINITE:
        raise NumericError("nonfinite risk weights; rescale X or lower sigma")


def cox_partial_loglik(state, beta=None):
    """Log partial likelihood at ``beta`` (defaults to the state's) (solvers.py:393-398)."""
    s = state
    b = s.beta if beta is None else beta
    s._dev["flags"].zero_()
    _xbeta(s, _flat_local(b))
    _risk(s)
    _raise_flags(int(s._dev["flags"].item()))
    return float(s._dev["loglik"].item())


def pi_delta(out, w, W, delta, lo, hi, comm, cuts=None):
    """Fused ``P @ delta`` over the owned range [lo, hi), then allreduce (solvers.py:401-419).

    Inputs may be host arrays or device tensors; ``out`` is written in place.
    """
    torch = _torch()
    dev = comm.device
    is_t = isinstance(w, torch.Tensor)
    tdt = w.dtype if is_t else torch_dtype(np.asarray(w).dtype)

    def dvec(v, dt):
        if isinstance(v, torch.Tensor):
            return v.to(device=dev, dtype=dt).contiguous()
        return torch.from_numpy(np.ascontiguousarray(np.asarray(v))).to(device=dev, dtype=dt)

    m = len(delta)
    wd, Wd, dd = dvec(w, tdt), dvec(W, tdt), dvec(delta, tdt)
    cd = dvec(cuts, torch.int64) if cuts is not None else None
    pd = torch.zeros(m, dtype=tdt, device=dev)
    if m:
        ws = torch.zeros(_lib.query("bs_cox_pi_delta_workspace", m), dtype=torch.uint8, device=dev)
        _lib.call("bs_cox_pi_delta", _lib.ptr(wd), _lib.ptr(Wd), _lib.ptr(dd), _lib.ptr(cd) if cd is not None else None,
                  _lib.dtype_code(tdt), m, int(lo), int(hi), _lib.ptr(pd), None, None, _lib.ptr(ws), ws.numel(),
                  _lib.stream_ptr())
    comm.allreduce(pd, ReduceOp.SUM)
    if isinstance(out, torch.Tensor):
        out.copy_(pd)
    else:
        out[...] = pd.cpu().numpy()
    return out


def cox_fit(state, iters, monitor=None, trace_every=1):
    """Proximal-gradient iterations for the L1-penalized partial likelihood (solvers.py:422-450).

    Each iteration records the penalized objective at the current iterate,
    checks the optional convergence monitor (which may stop before stepping),
    then takes one soft-thresholded step.
    """
    s = state
    if iters <= 0:
        return s
    s._dev["py_epoch"] = s._dev.get("py_epoch", 0) + 1  # a native state's cached X beta is stale now
    torch = _torch()
    x = s.X
    m = x.shape[0]
    n_loc = x.local.shape[1]
    dev = x.comm.device
    st = _lib.stream_ptr()
    code = _lib.dtype_code(s.beta.dtype)
    xcode = _lib.xcode(x)
    sigma, lam = float(s.sigma), float(s.lam)
    xb = s._dev["xb"]
    dmpd = s._dev["dmpd"]
    flags = s._dev["flags"]
    flags.zero_()
    trace_dev = _dev_f64(iters, dev)
    fhist = torch.zeros(iters, dtype=torch.int32, device=dev)
    beta = _flat_local(s.beta)
    grad = _flat_local(s.grad)
    Xf = _flat_local(x)
    pp, pn = s._work.args("pd", _lib.query("bs_cox_pi_delta_workspace", m))
    gp, gn = s._work.args("grad", _lib.query("bs_cox_grad_workspace", xcode, m, n_loc))
    comm = x.comm
    # The fused pass (one X stream per iteration, bs_cox_grad_xbeta) is the default for
    # float32 X with float32 arithmetic, where its 2-D grid kernel (cox_fused2.cu) beats
    # the two passes; BS_COX_FUSION=1 forces it for every dtype, =0 disables it.  It spins
    # on per-group counters, so never with other ranks' kernels sharing this GPU.
    mode = os.environ.get("BS_COX_FUSION", "auto")
    want = mode == "1" or (mode == "auto" and xcode == _lib.BS_F32 and code == _lib.BS_F32)
    fuse = int(want and dev.type == "cuda"
               and (comm.backend != "inproc" or comm.size <= torch.cuda.device_count()))
    if fuse:
        fp, fn_ = s._work.args("grad_xbeta", _lib.query("bs_cox_grad_xbeta_workspace", xcode, m, n_loc))
    host_trace = []
    ran = iters
    # A previous call's last fused pass left xb = (local X beta, ||beta||_1) for the beta it
    # produced; reuse it when beta is untouched since (same storage, and torch's in-place
    # version counter unchanged: any torch write to st.beta.local bumps it).  Saves a pass
    # over X per call.
    snap = s._dev.pop("xb_beta", None)
    reuse = bool(fuse and snap is not None and os.environ.get("BS_COX_REUSE", "1") != "0"
                 and snap == (s.beta.local.data_ptr(), s.beta.local._version))
    if fuse and not reuse:
        _xbeta(s, beta)                                         # the fused pass supplies the later ones
    for it in range(iters):
        if not fuse:
            _xbeta(s, beta)                                     # scn m + ||beta||_1 (solvers.py:436)
        elif (it > 0 or reuse) and comm.size > 1:
            comm.allreduce(xb, ReduceOp.SUM)                    # X beta partials of the fused pass
        _risk(s)                                                # solvers.py:437
        fhist[it:it + 1].copy_(flags)
        if trace_every and it % trace_every == 0:
            _lib.call("bs_cox_objective", _lib.ptr(s._dev["loglik"]), _at(xb, m), lam, _at(trace_dev, it), st)
            if monitor is not None:
                fl = int(flags.item())
                if fl & _lib.BS_FLAG_NONFINITE:
                    ran = it
                    break
                obj = float(trace_dev[it].item())
                host_trace.append(obj)
                if converged(monitor, obj):
                    ran = it + 1
                    break
        _lib.call("bs_cox_pi_delta", _lib.ptr(s.w), _lib.ptr(s.W), _lib.ptr(s.delta), _cuts_ptr(s), code, m, 0, m,
                  _lib.ptr(s.pd), _lib.ptr(dmpd), _lib.ptr(flags), pp, pn, st)
        if fuse:  # scn p + prox step and scn m of the next iteration in one pass over X
            _lib.call("bs_cox_grad_xbeta", _lib.ptr(Xf), xcode, _lib.ptr(dmpd), code, m, n_loc, _lib.ptr(grad),
                      _lib.ptr(beta), sigma, lam, _lib.ptr(xb), _lib.ptr(flags), 1, fp, fn_, st)
        else:     # scn p + prox (solvers.py:443-449)
            _lib.call("bs_cox_grad_step", _lib.ptr(Xf), xcode, _lib.ptr(dmpd), code, m, n_loc, _lib.ptr(grad),
                      _lib.ptr(beta), sigma, lam, 1, _at(xb, m), _lib.ptr(flags), gp, gn, st)
    fl_all = fhist[:max(ran, 1)].cpu().numpy() if ran else np.zeros(0, dtype=np.int32)
    bad = np.nonzero(fl_all & _lib.BS_FLAG_NONFINITE)[0] if fl_all.size else []
    if fuse and ran == iters and not len(bad) and not (int(flags.item()) & _lib.BS_FLAG_NONFINITE):
        s._dev["xb_beta"] = (s.beta.local.data_ptr(), s.beta.local._version)  # xb: last fused pass's partial
    stop = int(bad[0]) if len(bad) else ran
    if monitor is not None:
        s.trace.extend(host_trace[:len([it for it in range(stop) if trace_every and it % trace_every == 0])])
    elif trace_every:
        vals = trace_dev.cpu().numpy()
        s.trace.extend(float(vals[it]) for it in range(stop) if it % trace_every == 0)
    final = int(flags.item())
    if fl_all.size and (fl_all & _lib.BS_FLAG_CLAMPED).any():
        final |= _lib.BS_FLAG_CLAMPED
    if len(bad):
        final |= _lib.BS_FLAG_NONFINITE
    _raise_flags(final)
    return s
