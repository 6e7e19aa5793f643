"""ctypes binding of ``libbsb200.so`` (declared in ``include/bsb200.h``).

There is no fallback: if the shared library is missing, fails to load, or no
CUDA device is visible when a kernel is requested, the call raises.  The
library takes raw device pointers, sizes and a ``cudaStream_t``; the helpers
below turn torch tensors into those arguments.
"""

from __future__ import annotations

import ctypes as C
import os
import re
import threading
from pathlib import Path

PKG = Path(__file__).resolve().parent
LIB_PATH = Path(os.environ.get("BS_LIB_PATH", str(PKG / "libbsb200.so")))
HEADER = PKG.parent / "include" / "bsb200.h"

# status codes (bsb200.h)
BS_OK, BS_EINVAL, BS_ECUDA, BS_EWORK, BS_ENUMERIC, BS_ENCCL, BS_EDEGEN = 0, 1, 2, 3, 4, 5, 6
# dtype codes (comm.py:68-72 + int8)
BS_F32, BS_F64, BS_I64, BS_I8, BS_U2, BS_U2T = 0, 1, 2, 3, 4, 5
# ReduceOp codes (comm.py:54-58 order)
BS_SUM, BS_PROD, BS_MAX, BS_MIN = 0, 1, 2, 3
BS_T_NONE, BS_T_ABS, BS_T_SQUARE = 0, 1, 2
BS_NMF_MU, BS_NMF_APG = 0, 1
BS_FLAG_CLAMPED, BS_FLAG_NONFINITE, BS_FLAG_DEGENERATE = 1, 2, 4

_p = C.c_void_p
_i = C.c_int
_i64 = C.c_int64
_u64 = C.c_uint64
_d = C.c_double

# name -> (restype, argtypes); mirrors include/bsb200.h one to one.
SIGNATURES = {
    "bs_last_error": (C.c_char_p, []),
    "bs_abi_version": (_i, []),
    "bs_num_sms": (_i, []),
    "bs_launch_count": (_i64, []),
    "bs_note_replayed_launches": (None, [_i64]),
    "bs_philox_uniform": (_i, [_p, _i, _i64, _i64, _u64, _u64, _p]),
    "bs_philox_normal": (_i, [_p, _i, _i64, _i64, _u64, _u64, _p]),
    "bs_genotype_fill": (_i, [_p, _p, _i64, _i64, _i64, _u64, _u64, _p]),
    "bs_genotype_packed_bytes": (_i64, [_i64]),
    "bs_nccl_unique_id": (_i, [_p]),
    "bs_ctx_create": (_i, [_i, _i, _i, _p, _p, _p]),
    "bs_ctx_destroy": (_i, [_p]),
    "bs_cox_state_create": (_i, [_p, _p, _i, _i, _i64, _i64, _p, _p, _d, _d, _p, _p, _p]),
    "bs_cox_state_destroy": (_i, [_p]),
    "bs_cox_run": (_i, [_p, _i, _i, _i, _d, _p, _p, _p, _p]),
    "bs_nmf_state_create": (_i, [_p, _p, _i, _i64, _i64, _i, _d, _p, _p, _p]),
    "bs_nmf_state_destroy": (_i, [_p]),
    "bs_nmf_run": (_i, [_p, _i, _i, _i, _p, _p]),
    "bs_mds_state_create": (_i, [_p, _p, _i, _i64, _i64, _i, _i, _p, _p]),
    "bs_mds_state_destroy": (_i, [_p]),
    "bs_mds_run": (_i, [_p, _i, _i, _p, _p]),
    "bs_genotype_pack": (_i, [_p, _i64, _i64, _p, _p]),
    "bs_genotype_unpack": (_i, [_p, _i64, _i64, _p, _p]),
    "bs_genotype_fill_packed": (_i, [_p, _p, _i64, _i64, _i64, _u64, _u64, _p]),
    "bs_genotype_transpose_packed": (_i, [_p, _i64, _i64, _p, _p]),
    "bs_reduce_workspace": (_i64, [_i64]),
    "bs_reduce": (_i, [_p, _i, _i64, _i, _i, _p, _p, _i64, _p]),
    "bs_fold": (_i, [_p, _p, _i, _i64, _i, _i, _p]),
    "bs_diag_get": (_i, [_p, _i, _i64, _i64, _i64, _p, _p]),
    "bs_gram_workspace": (_i64, [_i, _i64]),
    "bs_gram": (_i, [_p, _i, _i, _i64, _p, _p, _i64, _p]),
    "bs_pairwise_euclidean": (_i, [_p, _i, _i64, _i64, _i64, _i64, _p, _p]),
    "bs_nmf_scan": (_i, [_p, _i, _i64, _p, _p, _i64, _p]),
    "bs_nmf_wxt_workspace": (_i64, [_i, _i64, _i64, _i]),
    "bs_nmf_wxt": (_i, [_p, _p, _i, _i64, _i64, _i, _p, _p, _p, _i64, _p]),
    "bs_nmf_xscale_bytes": (_i64, [_i64, _i64]),
    "bs_nmf_prepare_workspace": (_i64, [_i64, _i64]),
    "bs_nmf_prepare": (_i, [_p, _i, _i64, _i64, _p, _p, _p, _i64, _p]),
    "bs_gemm_path_counts": (_i, [_p, _i]),
    "bs_add_gemm_path_counts": (None, [_p]),
    "bs_nmf_wxt_scan_workspace": (_i64, [_i, _i64, _i64, _i]),
    "bs_nmf_wxt_scan": (_i, [_p, _p, _i, _i64, _i64, _i, _p, _p, _p, _i64, _p]),
    "bs_nmf_vt_step_workspace": (_i64, [_i, _i64]),
    "bs_nmf_vt_step": (_i, [_i, _p, _p, _p, _i, _i, _i64, _d, _p, _p, _p, _i64, _p]),
    "bs_nmf_w_step_workspace": (_i64, [_i, _i64, _i64, _i]),
    "bs_nmf_w_step": (_i, [_i, _p, _p, _p, _p, _i, _i64, _i64, _i, _d, _p, _p, _p, _i64, _p]),
    "bs_nmf_objective": (_i, [_p, _p, _p, _i, _p, _p, _d, _p]),
    "bs_nmf_objective_select": (_i, [_p, _p, _p, _p]),
    "bs_nmf_residual_workspace": (_i64, [_i64, _i64]),
    "bs_nmf_residual": (_i, [_p, _p, _p, _i, _i64, _i64, _i, _p, _p, _p, _i64, _p]),
    "bs_mds_pass_workspace": (_i64, [_i, _i64, _i64, _i]),
    "bs_mds_pass": (_i, [_p, _p, _i, _i64, _i64, _i64, _i, _i, _i, _p, _p, _p, _p, _i64, _p]),
    "bs_mds_update": (_i, [_p, _p, _p, _i, _i, _i64, _d, _p, _i, _p, _p]),
    "bs_cox_xbeta_workspace": (_i64, [_i, _i64, _i64]),
    "bs_cox_xbeta": (_i, [_p, _i, _p, _i, _i64, _i64, _p, _p, _i64, _p]),
    "bs_cox_risk_workspace": (_i64, [_i64]),
    "bs_cox_risk": (_i, [_p, _p, _p, _i, _i64, _d, _p, _p, _p, _p, _p, _p, _i64, _p]),
    "bs_cox_pi_delta_workspace": (_i64, [_i64]),
    "bs_cox_pi_delta": (_i, [_p, _p, _p, _p, _i, _i64, _i64, _i64, _p, _p, _p, _p, _i64, _p]),
    "bs_cox_grad_workspace": (_i64, [_i, _i64, _i64]),
    "bs_cox_grad_step": (_i, [_p, _i, _p, _i, _i64, _i64, _p, _p, _d, _d, _i, _p, _p, _p, _i64, _p]),
    "bs_cox_grad_xbeta_workspace": (_i64, [_i, _i64, _i64]),
    "bs_cox_grad_xbeta": (_i, [_p, _i, _p, _i, _i64, _i64, _p, _p, _d, _d, _p, _p, _i, _p, _i64, _p]),
    "bs_cox_objective": (_i, [_p, _p, _d, _p, _p]),
}


class BsError(RuntimeError):
    """A C-ABI call returned a nonzero status."""

    def __init__(self, name, code, msg):
        super().__init__(f"{name} failed (status {code}): {msg}")
        self.code = code


def header_symbols(path: Path = HEADER):
    """Function names declared in include/bsb200.h."""
    text = path.read_text()
    return sorted(set(re.findall(r"^\s*(?:const\s+)?[a-z_0-9]+\s*\*?\s*(bs_[a-z0-9_]+)\s*\(", text, re.M)))


_lib = None
_lock = threading.Lock()


def load():
    """Loads the shared library (no CUDA call is made)."""
    global _lib
    if _lib is not None:
        return _lib
    with _lock:
        if _lib is not None:
            return _lib
        if not LIB_PATH.exists():
            raise RuntimeError(
                f"{LIB_PATH} is missing: build it with `python -m paper_2010_16114_b200._build` "
                "(there is no CPU fallback)")
        lib = C.CDLL(str(LIB_PATH))
        for name, (res, args) in SIGNATURES.items():
            fn = getattr(lib, name)
            fn.restype = res
            fn.argtypes = args
        _lib = lib
    return _lib


class _Profile(threading.local):
    names = None
    events = None


_profile = _Profile()


class profile:
    """Context manager recording CUDA events around the named entry points.

    The events are recorded on the current stream (the stream the kernels are
    launched on), so ``elapsed()`` gives each call's device time.
    """

    def __init__(self, names):
        self.names = set(names)
        self.events = {n: [] for n in self.names}

    def __enter__(self):
        _profile.names, _profile.events = self.names, self.events
        return self

    def __exit__(self, *exc):
        _profile.names, _profile.events = None, None
        return False

    def elapsed_ms(self):
        """name -> list of per-call device milliseconds (synchronizes)."""
        out = {}
        for n, pairs in self.events.items():
            if pairs:
                pairs[-1][1].synchronize()
            out[n] = [a.elapsed_time(b) for a, b in pairs]
        return out


def call(name, *args):
    """Calls ``name`` and raises BsError on a nonzero status."""
    lib = load()
    prof = _profile.names is not None and name in _profile.names
    if prof:
        import torch

        prof = not torch.cuda.is_current_stream_capturing()  # graph captures are timed by their replays
    if prof:
        ev0 = torch.cuda.Event(enable_timing=True)
        ev1 = torch.cuda.Event(enable_timing=True)
        ev0.record()
    rc = getattr(lib, name)(*args)
    if prof:
        ev1.record()
        _profile.events[name].append((ev0, ev1))
    if rc != BS_OK:
        msg = lib.bs_last_error().decode(errors="replace")
        raise BsError(name, rc, msg)
    return rc


def query(name, *args):
    """Calls a *_workspace query (returns bytes)."""
    return int(getattr(load(), name)(*args))


# ---------------------------------------------------------------------------
# torch helpers
# ---------------------------------------------------------------------------

def dtype_code(dt):
    import numpy as np
    import torch

    if isinstance(dt, torch.dtype):
        table = {torch.float32: BS_F32, torch.float64: BS_F64, torch.int64: BS_I64, torch.int8: BS_I8}
    else:
        dt = np.dtype(dt)
        table = {np.dtype(np.float32): BS_F32, np.dtype(np.float64): BS_F64,
                 np.dtype(np.int64): BS_I64, np.dtype(np.int8): BS_I8}
    if dt not in table:
        raise ValueError(f"unsupported dtype {dt}")
    return table[dt]


def xcode(x):
    """Matrix code of a covariate block: BS_U2 for 2-bit packed genotypes, else its dtype's."""
    return BS_U2 if getattr(x, "packed", False) else dtype_code(x.dtype)


def ptr(t):
    """Device pointer of a CUDA tensor (None for nothing)."""
    if t is None:
        return None
    if not t.is_cuda:
        raise RuntimeError("the B200 kernels need CUDA tensors (no CPU fallback)")
    return C.c_void_p(t.data_ptr())


def stream_ptr(stream=None):
    import torch

    s = stream if stream is not None else torch.cuda.current_stream()
    return C.c_void_p(s.cuda_stream)
