"""ctypes binding of the in-tree native library (include/tds_b200.h).

There is no fallback: if `_lib/libtds_b200.so` is missing the import of any
solver entry point raises. Device memory, streams and collectives come from
PyTorch (plumbing); every kernel on the solve path lives in the .so.
"""

import ctypes
import os
import threading

import numpy as np

from . import errors

_LIB_PATH = os.path.join(os.path.dirname(os.path.abspath(__file__)), "_lib", "libtds_b200.so")
_lib = None
_lock = threading.Lock()

ABI_VERSION = 2
TDS_OK = 0
TDS_ERR_INVALID = 1
TDS_ERR_SINGULAR_PIVOT = 2
TDS_ERR_SINGULAR_PAIR = 3
TDS_ERR_SINGULAR_CORRECTION = 4
TDS_ERR_CUDA = 5
TDS_ERR_UNSUPPORTED = 6

TDS_FLAG_STRICT = 1
TDS_FLAG_STAGED = 2
TDS_FLAG_CHUNK16 = 4
TDS_PATH_FAST = 0
TDS_PATH_STAGED = 1

_P = ctypes.c_void_p
_D = ctypes.c_double
_I = ctypes.c_int
_LL = ctypes.c_longlong
_DP = ctypes.POINTER(ctypes.c_double)
_IP = ctypes.POINTER(ctypes.c_int)


class PlanInfo(ctypes.Structure):
    _fields_ = [("n", _I), ("rank_count", _I), ("rank", _I), ("block_rows", _I),
                ("path", _I), ("strict", _I), ("chunk_rows", _I), ("chunks", _I),
                ("uniform", _I), ("periodic", _I), ("max_dropped", _D),
                ("dominance_margin", _D)]


# exported symbol -> (restype, argtypes); the CPU test suite checks that this
# table covers every function declared in include/tds_b200.h
SIGNATURES = {
    "tds_abi_version": (_I, []),
    "tds_last_error": (ctypes.c_char_p, []),
    "tds_last_error_rank": (_I, []),
    "tds_plan_create": (_I, [_DP, _DP, _DP, _I, _DP, _IP, _I, _IP, _I, _I, _I,
                             ctypes.POINTER(_P)]),
    "tds_plan_create_local": (_I, [_DP, _DP, _DP, _DP, _IP, _I, _I, _I, _D, _D, _I,
                                   ctypes.POINTER(_P)]),
    "tds_plan_destroy": (_I, [_P]),
    "tds_plan_query": (_I, [_P, ctypes.POINTER(PlanInfo)]),
    "tds_plan_rank_coeffs": (_I, [_P, _I, _DP, _DP, _DP, _DP, _DP, _DP]),
    "tds_preprocess": (_I, [_DP, _DP, _DP, _I, _D, _DP, _DP, _DP, _DP, _DP, _DP]),
    "tds_solve": (_I, [_P, _P, _P, _LL, _I, _P]),
    "tds_halo_rows": (_I, [_P, _P, _P, _P, _LL, _I, _P]),
    "tds_boundary_rows": (_I, [_P, _P, _P, _P, _P, _P, _P, _LL, _I, _P]),
    "tds_finish": (_I, [_P, _P, _P, _P, _P, _P, _P, _P, _P, _LL, _I, _P]),
    "tds_decouple_fused": (_I, [_P, _P, _IP, _P, _P, _P, _P, _I, _LL, _P]),
    "tds_substitute": (_I, [_P, _P, _P, _P, _P, _P, _I, _LL, _P]),
    "tds_boundary_pair": (_I, [_P, _P, _D, _D, _P, _P, _LL, _P]),
    "tds_thomas": (_I, [_DP, _DP, _DP, _I, _P, _P, _I, _LL, _I, _D, _P]),
    "tds_mailbox_words": (_LL, [_LL, _I]),
    "tds_fused_eligible": (_I, [_P, _LL, _I]),
    "tds_plan_restrict_fused": (_I, [_P, _I]),
    "tds_fused_grid": (_LL, [_P, _LL, _I, _I]),
    "tds_mailbox_init": (_I, [_P, _LL, _P]),
    "tds_mailbox_status": (_I, [_P, _LL, _P, _P]),
    "tds_peer_access": (_I, [_I]),
    "tds_fused_solve": (_I, [_P, _P, _P, _LL, _I, _P, _P, _P, ctypes.c_ulonglong, _I, _P]),
    "tds_mailbox_error": (_I, [_P, _LL, _I, _IP]),
    "tds_ipc_alloc": (_I, [_LL, ctypes.POINTER(_P), ctypes.c_char_p]),
    "tds_ipc_open": (_I, [ctypes.c_char_p, ctypes.POINTER(_P)]),
    "tds_ipc_close": (_I, [_P]),
    "tds_ipc_free": (_I, [_P]),
    "tds_transport_contribution": (_I, [_P, _P, _P, _P, _P, _D, _I, _LL, _I, _P]),
    "tds_transport_combine": (_I, [_P, _P, _P, _P, _D, _P, _LL, _I, _P]),
    "tds_reorder": (_I, [_P, _P, _I, _I, _I, _I, _I, _P]),
    "tds_transport_contribution_in_x": (_I, [_P, _P, _P, _P, _P, _D, _I, _I, _I, _I, _I, _P]),
    "tds_transport_direction": (_I, [_P, _P, _P, _P, _P, _P, _P, _P, _D, _I, _I, _I, _I, _I, _P]),
    "tds_transport_mailbox_words": (_LL, [_LL, _I]),
    "tds_transport_mailbox_error": (_I, [_P, _LL, _I, ctypes.POINTER(_I)]),
    "tds_fused_transport": (_I, [_P, _P, _P, _P, _P, _D, _LL, _I, _P, _P, _P,
                                 ctypes.c_ulonglong, _I, _P]),
    "tds_fused_transport_in_x": (_I, [_P, _P, _P, _P, _P, _D, _I, _I, _I, _I, _P, _P, _P,
                                      ctypes.c_ulonglong, _I, _P]),
    "tds_fused_transport_direction": (_I, [_P, _P, _P, _P, _P, _P, _P, _P, _D, _I, _I, _I, _I,
                                           _P, _P, _P, ctypes.c_ulonglong, _I, _P]),
    "tds_euler_update": (_I, [_P, _P, _D, _P, _LL, _P]),
    "tds_multiply": (_I, [_P, _P, _P, _LL, _P]),
    "tds_reorder3": (_I, [_P, _P, _I, _I, _I, _I, _I, _I, _I, _P]),
    "tds_pack": (_I, [_P, _P, _I, _I, _I, _I, _I, _LL, _P]),
    "tds_unpack": (_I, [_P, _P, _I, _I, _I, _I, _I, _LL, _P]),
}


def library_path():
    return _LIB_PATH


def lib():
    """Load the native library once; raise loudly if it was not built."""
    global _lib
    if _lib is not None:
        return _lib
    with _lock:
        if _lib is None:
            if not os.path.exists(_LIB_PATH):
                raise RuntimeError(
                    f"native library {_LIB_PATH} is missing: run "
                    "`python -m paper_2411_13532_b200.build` (or __graft_entry__.build()); "
                    "there is no CPU fallback")
            h = ctypes.CDLL(_LIB_PATH)
            for name, (res, args) in SIGNATURES.items():
                fn = getattr(h, name)
                fn.restype = res
                fn.argtypes = args
            if h.tds_abi_version() != ABI_VERSION:
                raise RuntimeError("libtds_b200.so ABI version mismatch")
            _lib = h
    return _lib


def dptr(arr):
    """Pointer to a C-contiguous float64 NumPy array (kept alive by caller)."""
    return arr.ctypes.data_as(_DP)


def f64(x):
    return np.ascontiguousarray(x, dtype=np.float64)


def iptr(arr):
    """Pointer to a C-contiguous int32 NumPy array, or None."""
    if arr is None:
        return None
    return arr.ctypes.data_as(_IP)


_EXC = {
    TDS_ERR_INVALID: ValueError,
    TDS_ERR_SINGULAR_PIVOT: errors.SingularPivot,
    TDS_ERR_SINGULAR_PAIR: errors.SingularPair,
    TDS_ERR_SINGULAR_CORRECTION: errors.SingularCorrection,
    TDS_ERR_CUDA: RuntimeError,
    TDS_ERR_UNSUPPORTED: NotImplementedError,
}


def check(rc, rank_count=1):
    """Map a TDS_ERR_* status to the reference's exception types. Errors of a
    per-rank stage are wrapped in RankPanic as transport.spawn_ranks does
    (reference transport.py:126-138)."""
    if rc == TDS_OK:
        return
    h = lib()
    msg = h.tds_last_error().decode(errors="replace")
    exc = _EXC.get(rc, RuntimeError)(msg)
    rank = h.tds_last_error_rank()
    if rank_count > 1 and rank >= 0:
        raise errors.RankPanic({rank: exc})
    raise exc
