"""Distributed linear algebra used by the hot path (blockstat distlinalg.py subset).

The solvers never call a generic ``matmul``: scenarios b/a/d/j (NMF), f/a
(MDS) and m/p (Cox) are fused into the solver kernels (see solvers.py).  This
module keeps the reference entry points the solvers and their callers need:

* ``opnorm(.., "l2_power")`` — the default Cox step size (distlinalg.py:375-423),
  power iteration on the Cox GEMV kernels (scn n = bs_cox_xbeta, scn q =
  bs_cox_grad_step without the prox), same seed, start vector and stopping rule
  so the stopping step and therefore sigma match the reference;
* ``diag_get`` / ``diag_fill`` (distlinalg.py:97-130);
* ``pairwise_euclidean`` (distlinalg.py:442-468) — the MDS input builder, a
  tiled CUDA kernel over the gathered points;
* ``dot`` (distlinalg.py:83-94).

``matmul`` and its 17 scenarios are not part of this build (no solver issues
them: SURVEY.md §2 row 6); calling it raises ``ScenarioError``.
"""

from __future__ import annotations

import numpy as np

from . import _lib
from .comm import ReduceOp
from .distarray import DistArray, TransposedView, _flat_local, torch_dtype

SCENARIOS = {
    "a": ("dist", "dist", "dist"),
    "b": ("dist", "tdist", "dist"),
    "c": ("dist", "tdist", "tdist"),
    "d": ("dist", "tdist", "repl"),
    "e": ("dist", "repl", "repl"),
    "f": ("tdist", "dist", "dist"),
    "g": ("tdist", "dist", "tdist"),
    "h": ("tdist", "tdist", "tdist"),
    "i": ("tdist", "repl", "tdist"),
    "j": ("repl", "dist", "dist"),
    "k": ("repl", "tdist", "repl"),
    "l": ("dist", "dvec", "dvec"),
    "m": ("dist", "dvec", "rvec"),
    "n": ("dist", "rvec", "rvec"),
    "o": ("tdist", "dvec", "dvec"),
    "p": ("tdist", "rvec", "dvec"),
    "q": ("tdist", "rvec", "rvec"),
}


class ScenarioError(TypeError):
    """The (A, B, C) kind combination is not an admissible scenario."""


class ShapeError(ValueError):
    """Operand extents do not agree."""


def _torch():
    import torch

    return torch


def matmul(c, a, b, tmp=None):
    """Generic distributed matmul is outside the B200 hot path (fused into the solvers)."""
    raise ScenarioError("generic matmul scenarios are not part of the B200 build; the solvers use fused kernels")


def dot(a, b):
    """Sum of the elementwise product of two identically distributed arrays (distlinalg.py:83-94)."""
    if not isinstance(a, DistArray) or not isinstance(b, DistArray):
        raise TypeError("dot expects two DistArrays")
    if a.shape != b.shape:
        raise ShapeError(f"dot shapes differ: {a.shape} vs {b.shape}")
    if a.partition != b.partition:
        raise ShapeError("dot operands must share the partition")
    torch = _torch()
    part = (_flat_local(a).double() * _flat_local(b).double()).sum().reshape(1)
    if a.comm.size > 1:
        a.comm.allreduce(part, ReduceOp.SUM)
    del torch
    return float(part.item())


def diag_get(dest, m):
    """Copy the main diagonal of a square distributed matrix into ``dest`` (distlinalg.py:102-122)."""
    torch = _torch()
    if m.ndim != 2 or m.shape[0] != m.shape[1]:
        raise ShapeError(f"diagonal of a non-square matrix {m.shape}")
    n = m.shape[0]
    own = torch.empty(m.hi - m.lo, dtype=m.local.dtype, device=m.local.device)
    if own.numel():
        _lib.call("bs_diag_get", _lib.ptr(_flat_local(m)), _lib.dtype_code(m.dtype), n, m.lo, own.numel(),
                  _lib.ptr(own), _lib.stream_ptr())
    if isinstance(dest, DistArray):
        if dest.shape != (1, n) or dest.partition != m.partition:
            raise ShapeError(f"distributed dest must be 1 x {n} with the same partition")
        dest.local[0, :] = own
        return
    if tuple(np.shape(dest)) not in ((n,), (n, 1)):
        raise ShapeError(f"replicated dest must have length {n}")
    full = own
    if m.comm.size > 1:
        full = torch.empty(n, dtype=own.dtype, device=own.device)
        m.comm.allgatherv(own, full, m.partition.counts())
    if isinstance(dest, torch.Tensor):
        dest.copy_(full.reshape(dest.shape))
    else:
        dest[...] = full.cpu().numpy().reshape(np.shape(dest))


def diag_fill(m, value):
    """Set the main diagonal of a square distributed matrix to ``value`` (distlinalg.py:125-130)."""
    torch = _torch()
    if m.ndim != 2 or m.shape[0] != m.shape[1]:
        raise ShapeError(f"diagonal of a non-square matrix {m.shape}")
    w = m.hi - m.lo
    if w:
        idx = torch.arange(w, device=m.local.device)
        m.local[idx + m.lo, idx] = value


def opnorm(a, which="l2_power", tol=1e-6, maxiter=1000, seed=95376):
    """Matrix operator norm of a 2-D distributed matrix (distlinalg.py:375-423).

    ``l2_power`` runs on the device GEMV kernels; ``l1``/``linf``/``l2_quick``
    are exact reductions (not on the hot path).
    """
    torch = _torch()
    packed = getattr(a, "packed", False)
    if not (isinstance(a, DistArray) or packed) or a.ndim != 2:
        raise TypeError("opnorm expects a 2-D DistArray")
    m, n = a.shape
    if m == 0 or n == 0:
        raise ShapeError("opnorm of an empty matrix")
    if packed and which != "l2_power":
        raise TypeError("packed genotypes support opnorm(..., 'l2_power') only; unpack_genotypes first")
    comm = a.comm
    if which == "l1":
        local = a.local.double().abs().sum(dim=0).max().reshape(1) if a.local.numel() else \
            torch.full((1,), -np.inf, dtype=torch.float64, device=a.local.device)
        comm.allreduce(local, ReduceOp.MAX)
        return float(local.item())
    if which == "linf":
        rows = a.local.double().abs().sum(dim=1).contiguous() if a.local.numel() else \
            torch.zeros(m, dtype=torch.float64, device=a.local.device)
        comm.allreduce(rows, ReduceOp.SUM)
        return float(rows.max().item())
    if which == "l2_quick":
        return float(np.sqrt(opnorm(a, "l1") * opnorm(a, "linf")))
    if which != "l2_power":
        raise ValueError(f"unknown norm {which!r}")
    if tol <= 0 or maxiter < 1:
        raise ValueError("power iteration needs tol > 0 and maxiter >= 1")
    dev = comm.device
    gen = np.random.Generator(np.random.Philox(seed))
    v = gen.random(n)
    v /= np.linalg.norm(v)
    v_loc = torch.from_numpy(np.ascontiguousarray(v[a.lo:a.hi])).to(dev)
    n_loc = a.hi - a.lo
    xcode = _lib.xcode(a)
    single = a.dtype == np.dtype(np.float32)
    u = torch.zeros(m + 1, dtype=torch.float64, device=dev)
    w_loc = torch.zeros(max(n_loc, 1), dtype=torch.float64, device=dev)
    dummy = torch.zeros(max(n_loc, 1), dtype=torch.float64, device=dev)
    l1 = torch.zeros(1, dtype=torch.float64, device=dev)
    ws_x = torch.zeros(max(_lib.query("bs_cox_xbeta_workspace", xcode, m, n_loc), 256), dtype=torch.uint8,
                       device=dev)
    ws_g = torch.zeros(max(_lib.query("bs_cox_grad_workspace", xcode, m, n_loc), 256), dtype=torch.uint8,
                       device=dev)
    Xf = _flat_local(a)
    estimate = 0.0
    previous = np.inf
    for _ in range(maxiter):
        # u = A v (scn n)
        _lib.call("bs_cox_xbeta", _lib.ptr(Xf), xcode, _lib.ptr(v_loc), _lib.BS_F64, m, n_loc, _lib.ptr(u),
                  _lib.ptr(ws_x), ws_x.numel(), _lib.stream_ptr())
        if comm.size > 1:
            comm.allreduce(u[:m], ReduceOp.SUM)
        if single:  # u is an a.dtype buffer in the reference (distlinalg.py:408)
            u[:m] = u[:m].float().double()
        estimate = float(torch.linalg.vector_norm(u[:m]).item())
        if abs(estimate - previous) <= tol * max(estimate, np.finfo(float).tiny):
            break
        previous = estimate
        # w = A^T u (scn q)
        _lib.call("bs_cox_grad_step", _lib.ptr(Xf), xcode, _lib.ptr(u), _lib.BS_F64, m, n_loc, _lib.ptr(w_loc),
                  _lib.ptr(dummy), 0.0, 0.0, 0, _lib.ptr(l1), None, _lib.ptr(ws_g), ws_g.numel(), _lib.stream_ptr())
        wl = w_loc[:n_loc]
        if single:
            wl = wl.float().double()
        sq = (wl * wl).sum().reshape(1)
        if comm.size > 1:
            comm.allreduce(sq, ReduceOp.SUM)
        norm_w = float(np.sqrt(sq.item()))
        if norm_w == 0:
            return 0.0
        v_loc = wl / norm_w
    return estimate


def pairwise_euclidean(y, x, chunk=64):
    """Pairwise Euclidean distances between the columns of ``x`` (distlinalg.py:442-468).

    ``x`` holds one point per column ((d, n) distributed); ``y`` receives the
    n x n distance matrix with zero diagonal.  The points are all-gathered
    once (the reference streams them in ``chunk``-column pieces to bound host
    memory; the result does not depend on ``chunk``).
    """
    torch = _torch()
    if x.ndim != 2 or y.ndim != 2:
        raise ShapeError("pairwise_euclidean expects 2-D arrays")
    n = x.shape[1]
    if y.shape != (n, n):
        raise ShapeError(f"distance matrix must be {n} x {n}, got {y.shape}")
    if chunk < 1:
        raise ValueError("chunk width must be >= 1")
    d = x.shape[0]
    comm = x.comm
    if comm.size > 1:
        full = torch.empty(d * n, dtype=torch_dtype(x.dtype), device=comm.device)
        comm.allgatherv(_flat_local(x), full, [d * c for c in x.partition.counts()])
    else:
        full = _flat_local(x)
    if full.dtype != y.local.dtype:
        full = full.to(y.local.dtype)
    _lib.call("bs_pairwise_euclidean", _lib.ptr(full), _lib.dtype_code(y.dtype), d, n, y.lo, y.hi - y.lo,
              _lib.ptr(_flat_local(y)), _lib.stream_ptr())
