"""Serial (single-subdomain) solvers on the GPU, reference arithmetic:
thomas_solve / periodic_thomas_solve (reference serial.py:26-90). They are
the P=1 semantics of run_distd2; here an RhsBatch (m, n) is solved as a
(m, n, 1) field by the `k_thomas` kernel, bit-identical to the reference.
`pivot_floor` is honoured as in the reference (|pivot| <= floor raises
SingularPivot; the correction denominator raises SingularCorrection)."""

import ctypes

import numpy as np

from . import _native as N
from .distributed import _Field, _stream_handle
from .system import RhsBatch

PIVOT_FLOOR = 1e-300
PAIR_DET_FLOOR = 1e-12
DEFAULT_TRUNCATION_THRESHOLD = 1e-14


def _solve(sys, rhs, periodic, pivot_floor):
    if rhs.n != sys.n:
        raise ValueError(f"rhs length {rhs.n} does not match system size {sys.n}")
    lo, di, up = (N.f64(x) for x in (sys.lower, sys.diag, sys.upper))
    fld = _Field(rhs.values)
    out = fld.empty_like()
    N.check(N.lib().tds_thomas(N.dptr(lo), N.dptr(di), N.dptr(up), int(periodic), fld.ptr,
                               ctypes.c_void_p(out.data_ptr()), sys.n, rhs.m, 1,
                               float(pivot_floor), _stream_handle()))
    return RhsBatch(np.asarray(fld.give(out)) if fld.host else out.cpu().numpy())


def thomas_solve(sys, rhs, pivot_floor=PIVOT_FLOOR):
    """Open system; serial.py:26-56."""
    if sys.periodic:
        raise ValueError("thomas_solve handles open systems; use periodic_thomas_solve")
    return _solve(sys, rhs, False, pivot_floor)


def periodic_thomas_solve(sys, rhs, pivot_floor=PIVOT_FLOOR):
    """Cyclic system via Sherman-Morrison; serial.py:59-90."""
    if not sys.periodic:
        raise ValueError("periodic_thomas_solve requires a periodic system")
    return _solve(sys, rhs, True, pivot_floor)
