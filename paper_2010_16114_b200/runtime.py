"""Python handle on the solver-level C ABI (bs_ctx_* / bs_cox_*; include/bsb200.h).

``Context(comm)`` creates the per-rank native context: its stream is the current
torch stream, and for more than one rank an NCCL communicator whose unique id rank 0
draws and ships over ``comm`` (one process per GPU, as under torchrun; NCCL does not
put two ranks on one GPU, so in-process multi-rank worlds are refused).
``cox_run(ctx, state, iters, ...)`` runs ``cox_fit``'s loop (solvers.py:422-450) inside
the library on a ``CoxState`` made by ``cox_init`` and appends to ``state.trace`` like
``cox_fit`` does; ``nmf_run(ctx, state, iters, algo)`` does the same for
``nmf_multiplicative`` / ``nmf_apg`` (solvers.py:144-185) on an ``NmfState`` and
``mds_run`` for ``mds_fit`` (solvers.py:269-305) on an ``MdsState``.
"""

from __future__ import annotations

import ctypes as C
import warnings

import numpy as np

from . import _lib
from .distarray import _flat_local
from .solvers import DegenerateConfigError, NumericError, _cuts_ptr


class Context:
    def __init__(self, comm):
        import torch

        self.comm = comm
        if comm.size > 1 and getattr(comm, "backend", None) == "inproc":
            raise ValueError("the native runtime needs one process per GPU for more than one rank")
        uid = np.zeros(16, dtype=np.int64)  # 128-byte ncclUniqueId
        if comm.size > 1:
            if comm.rank == 0:
                _lib.call("bs_nccl_unique_id", uid.ctypes.data_as(C.c_void_p))
            comm.broadcast(uid, root=0)
        dev = comm.device.index if comm.device.index is not None else torch.cuda.current_device()
        h = C.c_void_p()
        _lib.call("bs_ctx_create", comm.rank, comm.size, dev, uid.ctypes.data_as(C.c_void_p) if comm.size > 1 else None,
                  _lib.stream_ptr(), C.byref(h))
        self.handle = h
        self._states = []  # (python state, destroy fn name, handle): native states cached per solver state

    def _native(self, state, kind, create, tensors):
        """The native state for ``state``, created on first use and kept until close().

        It holds raw pointers to ``tensors`` (and, for Cox, a cached X beta for the
        current beta), so it is rebuilt when any of them was replaced or written by
        torch since the last call (storage pointer or in-place version changed)."""
        key = ("native", kind, id(self))
        # py_epoch: bumped by the Python cox_fit, which moves beta through raw pointers
        sig = tuple((t.data_ptr(), t._version) for t in tensors) + (state._dev.get("py_epoch", 0),)
        entry = state._dev.get(key)
        if entry is not None and entry[1] != sig:
            self._drop(state, key)
            entry = None
        if entry is None:
            entry = (create(), sig, f"bs_{kind}_state_destroy")
            state._dev[key] = entry
            self._states.append((state, key))
        return entry[0]

    def _drop(self, state, key):
        entry = state._dev.pop(key, None)
        if entry is not None:
            _lib.call(entry[2], entry[0])
        self._states = [(s, k) for s, k in self._states if not (s is state and k == key)]

    def close(self):
        for state, key in list(self._states):
            self._drop(state, key)
        self._states = []
        if self.handle:
            _lib.call("bs_ctx_destroy", self.handle)
            self.handle = None

    def __enter__(self):
        return self

    def __exit__(self, *exc):
        self.close()
        return False


def cox_run(ctx, state, iters, trace_every=1, monitor=None):
    """``cox_fit(state, iters, monitor, trace_every)`` with the loop in native code."""
    s = state
    x = s.X
    m, n_loc = x.shape[0], x.local.shape[1]
    xcode = _lib.xcode(x)
    code = _lib.dtype_code(s.beta.dtype)
    def create():
        h = C.c_void_p()
        _lib.call("bs_cox_state_create", ctx.handle, _lib.ptr(_flat_local(x)) if n_loc else None, xcode, code, m,
                  n_loc, _lib.ptr(s.delta), _cuts_ptr(s), float(s.lam), float(s.sigma),
                  _lib.ptr(_flat_local(s.beta)) if n_loc else None, _lib.ptr(_flat_local(s.grad)) if n_loc else None,
                  C.byref(h))
        return h

    h = ctx._native(s, "cox", create, [x.local, s.beta.local, s.grad.local, s.delta])
    s._dev.pop("xb_beta", None)  # the native loop moves beta: cox_fit's X beta reuse no longer applies
    ntr = (iters + trace_every - 1) // trace_every if trace_every else 0
    trace = np.zeros(max(ntr, 1), dtype=np.float64)
    nt, ran, flags = C.c_int(), C.c_int(), C.c_int()
    window = monitor.window if monitor is not None else 0
    tol = monitor.rel_tol if monitor is not None else 0.0
    rc = _lib.load().bs_cox_run(h, int(iters), int(trace_every), int(window), float(tol),
                                trace.ctypes.data_as(C.c_void_p), C.byref(nt), C.byref(ran), C.byref(flags))
    s.trace.extend(float(v) for v in trace[:nt.value])
    if monitor is not None:
        monitor.history.extend(float(v) for v in trace[:nt.value])
    if flags.value & _lib.BS_FLAG_CLAMPED:
        warnings.warn("linear predictor clamped before exponentiation", RuntimeWarning, stacklevel=2)
    if rc == _lib.BS_ENUMERIC:
        raise NumericError("nonfinite risk weights; rescale X or lower sigma")
    if rc != _lib.BS_OK:
        raise _lib.BsError("bs_cox_run", rc, _lib.load().bs_last_error().decode(errors="replace"))
    return s


def nmf_run(ctx, state, iters, algo="apg", trace_every=1):
    """``nmf_apg`` / ``nmf_multiplicative(state, iters, trace_every)`` with the loop in native code."""
    s = state
    x = s.X
    m, n_loc = x.shape[0], x.local.shape[1]
    r = s.Vt.shape[0]
    code = _lib.dtype_code(x.dtype)
    a = _lib.BS_NMF_APG if algo == "apg" else _lib.BS_NMF_MU
    vt = _flat_local(s.Vt)

    def create():
        h = C.c_void_p()
        _lib.call("bs_nmf_state_create", ctx.handle, _lib.ptr(_flat_local(x)) if n_loc else None, code, m, n_loc, r,
                  float(s.eps), _lib.ptr(vt) if vt.numel() else None, _lib.ptr(_flat_local(s.W)) if n_loc else None,
                  C.byref(h))
        return h

    h = ctx._native(s, "nmf", create, [x.local, s.Vt.local, s.W.local])
    ntr = (iters + trace_every - 1) // trace_every if trace_every else 0
    trace = np.zeros(max(ntr, 1), dtype=np.float64)
    nt = C.c_int()
    rc = _lib.load().bs_nmf_run(h, a, int(iters), int(trace_every), trace.ctypes.data_as(C.c_void_p), C.byref(nt))
    if rc == _lib.BS_EINVAL:
        raise ValueError(_lib.load().bs_last_error().decode(errors="replace"))
    if rc != _lib.BS_OK:
        raise _lib.BsError("bs_nmf_run", rc, _lib.load().bs_last_error().decode(errors="replace"))
    s.trace.extend(float(v) for v in trace[:nt.value])
    return s


def mds_run(ctx, state, iters, trace_every=1):
    """``mds_fit(state, iters, trace_every)`` with the loop in native code."""
    s = state
    y = s.Y
    n, n_loc = y.shape[0], y.local.shape[1]
    q = s.theta.shape[0]
    code = _lib.dtype_code(y.dtype)
    def create():
        h = C.c_void_p()
        _lib.call("bs_mds_state_create", ctx.handle, _lib.ptr(_flat_local(y)) if n_loc else None, code, n, n_loc, q,
                  1 if s.perturb else 0, _lib.ptr(_flat_local(s.theta)) if n_loc else None, C.byref(h))
        return h

    h = ctx._native(s, "mds", create, [y.local, s.theta.local])
    ntr = (iters + trace_every - 1) // trace_every if trace_every else 0
    trace = np.zeros(max(ntr, 1), dtype=np.float64)
    nt = C.c_int()
    rc = _lib.load().bs_mds_run(h, int(iters), int(trace_every), trace.ctypes.data_as(C.c_void_p), C.byref(nt))
    s.trace.extend(float(v) for v in trace[:nt.value])
    if rc == _lib.BS_EDEGEN:
        raise DegenerateConfigError("coincident embedding points; rerun with perturb=True")
    if rc != _lib.BS_OK:
        raise _lib.BsError("bs_mds_run", rc, _lib.load().bs_last_error().decode(errors="replace"))
    return s
