"""DistD2 operator API, B200-native: same names, arguments, return types and
errors as the reference's distributed.py (/root/reference/pkg/src/tds/
distributed.py:1-449), computed by the sm_100a kernels in `_lib`.

Field arguments may be NumPy arrays (host; copied to the current CUDA device
and back, like a drop-in for the reference) or CUDA torch tensors (device
resident, result returned on the device). There is no CPU path: every call
below that touches field data launches a kernel from libtds_b200.so.

Arithmetic modes (keyword-only `arithmetic=`):
  "fast"   -- default. Single-pass chunked kernel; FMA; exact reduced system
              between chunks; the reference's truncation only at rank
              boundaries. Agrees with the reference to ~1e-15 relative.
  "strict" -- staged kernels in the reference's operation order, no FMA;
              bit-identical to the reference on the same inputs.
"""

import ctypes
import warnings
from dataclasses import dataclass

import numpy as np

from . import _native as N
from .errors import NotDominantWarning, SingularPair
from .system import SubdomainPartition, TridiagonalSystem, is_diagonally_dominant

HALO_DEPTH = 2
PIVOT_FLOOR = 1e-300
PAIR_DET_FLOOR = 1e-12


# ------------------------------------------------------------------ types

@dataclass(frozen=True)
class DistCoeffs:
    """Preprocessed per-row coefficients of one subdomain (distributed.py:43-68)."""

    s_a: np.ndarray
    s_c: np.ndarray
    w: np.ndarray
    f: np.ndarray
    r: np.ndarray
    n_loc: int
    cyclic_global: bool
    position: str
    dropped_first: float
    dropped_last: float

    @property
    def max_dropped(self):
        return max(self.dropped_first, self.dropped_last)


@dataclass(frozen=True)
class StencilCoeffs:
    """Per-row width-5 RHS weights, offsets -2..+2 (distributed.py:71-86).

    `shift` (extension, default None): per-row window shift s_j, row j's
    weights then apply to u[j + o + s_j], o = -2..2. It carries one-sided
    closures that need points beyond the width-5 window (the open d2/dx2
    operator, assemble(..., closure="one-sided")); only rows 0, 1 (0..2)
    and n-2, n-1 (-2..0) of an open line may be shifted."""

    c: np.ndarray
    halo_depth: int = HALO_DEPTH
    shift: np.ndarray = None

    def __post_init__(self):
        arr = np.ascontiguousarray(self.c, dtype=np.float64)
        if arr.ndim != 2 or arr.shape[1] != 5:
            raise ValueError(f"stencil must be (n, 5), got {arr.shape}")
        object.__setattr__(self, "c", arr)
        if self.shift is not None:
            sh = np.ascontiguousarray(self.shift, dtype=np.int32)
            if sh.shape != (arr.shape[0],):
                raise ValueError(f"stencil shift must be ({arr.shape[0]},), got {sh.shape}")
            if np.any(np.abs(sh) > 2):
                raise ValueError("stencil shifts must lie in -2..2")
            object.__setattr__(self, "shift", sh if np.any(sh) else None)

    @property
    def n(self):
        return self.c.shape[0]

    def rows(self, start, stop):
        """The stencil of rows [start, stop) (a rank's local stencil)."""
        sh = None if self.shift is None else self.shift[start:stop]
        return StencilCoeffs(self.c[start:stop], self.halo_depth, sh)

    def shift4(self):
        """Window shifts of rows 0, 1, n-2, n-1 (int32), or None."""
        if self.shift is None:
            return None
        n = self.n
        return np.ascontiguousarray(self.shift[[0, 1, n - 2, n - 1]], dtype=np.int32)


@dataclass(frozen=True)
class BoundaryPair:
    """Inputs of one cross-boundary 2x2 solve (distributed.py:89-101)."""

    d_last_local: object
    d_first_remote: object
    s_c_last: float
    s_a_first_remote: float


@dataclass(frozen=True)
class PairCoeffs:
    """Cached neighbour couplings, exchanged once (distributed.py:104-109)."""

    prev_s_c_last: float | None
    next_s_a_first: float | None


def identity_stencil(n):
    c = np.zeros((n, 5))
    c[:, 2] = 1.0
    return StencilCoeffs(c)


def local_slice(sys, part, rank_id):
    """Rank `rank_id`'s block with its external couplings (distributed.py:119-133)."""
    off = part.offsets()[rank_id]
    m = part.local_sizes[rank_id]
    a = sys.effective_lower()[off:off + m].copy()
    c = sys.effective_upper()[off:off + m].copy()
    if rank_id == 0:
        a[0] = sys.lower[0] if sys.periodic else 0.0
    if rank_id == part.rank_count - 1:
        c[-1] = sys.upper[-1] if sys.periodic else 0.0
    return TridiagonalSystem(a, sys.diag[off:off + m].copy(), c, periodic=False)


def rank_position(rank_id, rank_count):
    if rank_id == 0:
        return "first"
    if rank_id == rank_count - 1:
        return "last"
    return "interior"


def preprocess(local_sys, position, cyclic, pivot_floor=PIVOT_FLOOR, warn_not_dominant=True):
    """Alg. 5 (distributed.py:144-199), computed by the native plan builder
    (tds_preprocess) with the reference's rounding: bit-identical values."""
    m = local_sys.n
    if m < 4:
        raise ValueError(f"local block needs at least 4 rows, got {m}")
    if warn_not_dominant and not is_diagonally_dominant(local_sys):
        warnings.warn("local block is not strictly diagonally dominant",
                      NotDominantWarning, stacklevel=2)
    a, b, c = (N.f64(x) for x in (local_sys.lower, local_sys.diag, local_sys.upper))
    out = [np.empty(m) for _ in range(5)]
    dropped = np.empty(2)
    N.check(N.lib().tds_preprocess(N.dptr(a), N.dptr(b), N.dptr(c), m, float(pivot_floor),
                                   *[N.dptr(o) for o in out], N.dptr(dropped)))
    sa, sc, w, f, r = out
    return DistCoeffs(sa, sc, w, f, r, m, bool(cyclic), position,
                      abs(float(dropped[0])), abs(float(dropped[1])))


# ------------------------------------------------------------- plumbing

def _torch():
    import torch
    return torch


def _stream_handle(stream=None):
    torch = _torch()
    s = stream if stream is not None else torch.cuda.current_stream()
    return ctypes.c_void_p(s.cuda_stream)


class _Field:
    """A fp64 operand on the current CUDA device. Remembers where the caller's
    data lives: NumPy array or CPU tensor (host: copied in, result copied
    back; pinned CPU tensors copy asynchronously) or CUDA tensor (device)."""

    def __init__(self, x):
        torch = _torch()
        if isinstance(x, torch.Tensor):
            self.numpy = False
            if x.is_cuda:
                self.host = False
                self.t = x.to(torch.float64).contiguous()
                return
            _need_cuda()
            self.host = True
            self.t = x.to(torch.float64).contiguous().to("cuda", non_blocking=x.is_pinned())
        else:
            _need_cuda()
            self.host = True
            self.numpy = True
            arr = np.ascontiguousarray(x, dtype=np.float64)
            if not arr.flags.writeable:          # torch cannot wrap read-only buffers
                arr = arr.copy()
            self.t = torch.from_numpy(arr).to("cuda", non_blocking=False)

    @property
    def ptr(self):
        return ctypes.c_void_p(self.t.data_ptr())

    def empty_like(self, shape=None):
        torch = _torch()
        return torch.empty(self.t.shape if shape is None else shape,
                           dtype=torch.float64, device=self.t.device)

    def give(self, t, out=None):
        """Hand the result back where the input came from (into `out` if given)."""
        torch = _torch()
        if not self.host:
            if out is not None:
                out.copy_(t)
                return out
            return t
        if out is not None:
            out.copy_(t, non_blocking=bool(getattr(out, "is_pinned", lambda: False)()))
            torch.cuda.current_stream().synchronize()
            return out
        if self.numpy:
            return t.cpu().numpy()
        return t.cpu()


def _need_cuda():
    torch = _torch()
    if not torch.cuda.is_available():
        raise RuntimeError("paper_2411_13532_b200 needs a CUDA device; there is no CPU "
                           "fallback")


class Plan:
    """Owns one native tds_plan (coefficient tables on one device)."""

    def __init__(self, handle, rank_count, device):
        self.handle = handle
        self.rank_count = rank_count
        self.device = device
        info = N.PlanInfo()
        N.check(N.lib().tds_plan_query(handle, ctypes.byref(info)))
        self.info = info

    @property
    def path(self):
        return "fast" if self.info.path == N.TDS_PATH_FAST else "staged"

    def __del__(self):
        try:
            if self.handle:
                N.lib().tds_plan_destroy(self.handle)
                self.handle = None
        except Exception:   # interpreter shutdown
            pass

    @classmethod
    def create(cls, sys, stencil_c, sizes, rank=-1, flags=0, shift=None):
        torch = _torch()
        lo, di, up = (N.f64(x) for x in (sys.lower, sys.diag, sys.upper))
        st = None if stencil_c is None else N.f64(stencil_c)
        sh = None if shift is None else np.ascontiguousarray(shift, dtype=np.int32)
        sz = (ctypes.c_int * len(sizes))(*sizes)
        h = ctypes.c_void_p()
        N.check(N.lib().tds_plan_create(
            N.dptr(lo), N.dptr(di), N.dptr(up), int(bool(sys.periodic)),
            None if st is None else N.dptr(st), N.iptr(sh), sys.n, sz, len(sizes), rank, flags,
            ctypes.byref(h)), rank_count=len(sizes))
        return cls(h, len(sizes), torch.cuda.current_device())

    @classmethod
    def create_local(cls, local_sys, stencil_c, has_prev, has_next, prev_sc_last,
                     next_sa_first, flags=0, shift=None):
        torch = _torch()
        a, b, c = (N.f64(x) for x in (local_sys.lower, local_sys.diag, local_sys.upper))
        st = None if stencil_c is None else N.f64(stencil_c)
        sh = None if shift is None else np.ascontiguousarray(shift, dtype=np.int32)
        h = ctypes.c_void_p()
        N.check(N.lib().tds_plan_create_local(
            N.dptr(a), N.dptr(b), N.dptr(c), None if st is None else N.dptr(st), N.iptr(sh),
            local_sys.n, int(has_prev), int(has_next), float(prev_sc_last or 0.0),
            float(next_sa_first or 0.0), flags, ctypes.byref(h)))
        return cls(h, 2, torch.cuda.current_device())


_PLAN_CACHE = {}
_PLAN_CACHE_MAX = 32


def _flags(arithmetic):
    if arithmetic == "fast":
        return 0
    if arithmetic == "strict":
        return N.TDS_FLAG_STRICT
    if arithmetic == "staged":
        return N.TDS_FLAG_STAGED
    raise ValueError(f"arithmetic must be 'fast', 'strict' or 'staged', got {arithmetic!r}")


def get_plan(sys, stencil, part, rank=-1, arithmetic="fast", chunk_rows=None):
    """Cached plan for (operator, partition, rank, arithmetic, device).
    chunk_rows=16 asks for 16-row chunks (TDS_FLAG_CHUNK16)."""
    torch = _torch()
    st = None if stencil is None else stencil.c
    sh = None if stencil is None else stencil.shift
    key = (sys.lower.tobytes(), sys.diag.tobytes(), sys.upper.tobytes(), bool(sys.periodic),
           None if st is None else st.tobytes(), None if sh is None else sh.tobytes(),
           part.local_sizes, rank, arithmetic, chunk_rows, torch.cuda.current_device())
    plan = _PLAN_CACHE.get(key)
    if plan is None:
        if len(_PLAN_CACHE) >= _PLAN_CACHE_MAX:
            _PLAN_CACHE.pop(next(iter(_PLAN_CACHE)))
        flags = _flags(arithmetic) | (N.TDS_FLAG_CHUNK16 if chunk_rows == 16 else 0)
        plan = Plan.create(sys, st, part.local_sizes, rank, flags, shift=sh)
        _PLAN_CACHE[key] = plan
    return plan


# ------------------------------------------------------------- operator

class _RankGroup:
    """P DistD2 ranks of one operator inside this process: one
    LocalRankContext + DistD2Rank per rank, each on its device with its own
    stream (several ranks may share a device; transport.spawn_ranks). The
    per-rank kernels and neighbour rounds are the ones a torchrun rank runs
    (rank.py): the fused k_dd / k_dd2 exchange through device mailboxes
    (NVLink peer stores between B200s), the two-pass path through the
    contexts' device-to-device messages. Replaces the reference's threaded
    run_distd2 body (distributed.py:417-441)."""

    def __init__(self, sys, stencil, part, devices, arithmetic, warn_not_dominant):
        from .rank import DistD2Rank
        from .transport import make_contexts, run_on
        self.part = part
        self.contexts = make_contexts(part.rank_count, sys.periodic, devices)
        self.ranks = run_on(self.contexts, lambda ctx: DistD2Rank(
            sys, stencil, part, ctx, arithmetic=arithmetic, warn_not_dominant=warn_not_dominant))
        self._streams = None
        self._bufs = {}

    def _rank_streams(self):
        torch = _torch()
        if self._streams is None:
            self._streams = [torch.cuda.Stream(c.device) for c in self.contexts]
        return self._streams

    def solve(self, field, out):
        """field, out: (groups, n, sz) CUDA tensors (any device)."""
        from .transport import run_on
        torch = _torch()
        groups, n, sz = field.shape
        offs, sizes = self.part.offsets(), self.part.local_sizes
        if all(r.fused_eligible(groups, sz) for r in self.ranks):
            run_on(self.contexts, lambda ctx: self.ranks[ctx.rank_id].mailbox(groups, sz))
            caller = torch.cuda.current_stream(field.device)
            streams = self._rank_streams()
            key = (groups, sz)
            bufs = self._bufs.get(key)
            if bufs is None:
                bufs = [(torch.empty((groups, m, sz), dtype=torch.float64, device=c.device),
                         torch.empty((groups, m, sz), dtype=torch.float64, device=c.device))
                        for c, m in zip(self.contexts, sizes)]
                self._bufs[key] = bufs
            for k, (rank, s) in enumerate(zip(self.ranks, streams)):
                s.wait_stream(caller)
                with torch.cuda.stream(s):
                    bufs[k][0].copy_(field[:, offs[k]:offs[k] + sizes[k], :], non_blocking=True)
            # every rank's kernel is enqueued before any is waited for: the
            # persistent grids are co-resident (max_ctas splits shared devices)
            for k, (rank, s) in enumerate(zip(self.ranks, streams)):
                with torch.cuda.device(self.contexts[k].device):
                    rank.launch_fused(bufs[k][0], bufs[k][1], s)
            for k, s in enumerate(streams):
                with torch.cuda.stream(s):
                    out[:, offs[k]:offs[k] + sizes[k], :].copy_(bufs[k][1], non_blocking=True)
                caller.wait_stream(s)
            return out
        torch.cuda.current_stream(field.device).synchronize()

        def body(ctx):
            k = ctx.rank_id
            u = field[:, offs[k]:offs[k] + sizes[k], :].to(ctx.device).contiguous()
            res = self.ranks[k].solve(u)
            out[:, offs[k]:offs[k] + sizes[k], :].copy_(res)
            return None

        run_on(self.contexts, body)
        return out

    def check(self):
        """Wait for every rank's last fused solve; TimeoutError if one timed out."""
        from .transport import run_on
        run_on(self.contexts, lambda ctx: self.ranks[ctx.rank_id].check())

    def audit(self, audit, rounds_before):
        self.check()
        audit["rounds_per_rank"] = [c.exchange_rounds - r0
                                    for c, r0 in zip(self.contexts, rounds_before)]
        audit["messages_sent"] = sum(c.messages_sent for c in self.contexts)
        audit["bytes_sent"] = sum(c.bytes_sent for c in self.contexts)
        audit["max_dropped"] = max(r.coeffs.max_dropped for r in self.ranks)

    def close(self):
        for r in self.ranks:
            r.close()


_GROUPS = {}
_GROUPS_MAX = 8


def _rank_group(sys, stencil, part, devices, arithmetic, warn_not_dominant, fresh=False):
    torch = _torch()
    devs = tuple(torch.device("cuda", d) if isinstance(d, int) else torch.device(d)
                 for d in devices)
    if len(devs) != part.rank_count:
        raise ValueError(f"{len(devs)} devices given for {part.rank_count} ranks")
    if fresh:
        return _RankGroup(sys, stencil, part, devs, arithmetic, warn_not_dominant)
    st = None if stencil is None else stencil.c
    sh = None if stencil is None or stencil.shift is None else stencil.shift.tobytes()
    key = (sys.lower.tobytes(), sys.diag.tobytes(), sys.upper.tobytes(), bool(sys.periodic),
           None if st is None else st.tobytes(), sh, part.local_sizes, devs, arithmetic)
    g = _GROUPS.get(key)
    if g is None:
        if len(_GROUPS) >= _GROUPS_MAX:
            _GROUPS.pop(next(iter(_GROUPS))).close()
        g = _GROUPS[key] = _RankGroup(sys, stencil, part, devs, arithmetic, warn_not_dominant)
    return g


class _HostPipe:
    """Per-device staging for host-resident solves: three copy/compute
    streams and a ring of device buffers (allocated once, reused)."""

    def __init__(self, device):
        torch = _torch()
        self.device = device
        self.h2d = torch.cuda.Stream(device)
        self.cmp = torch.cuda.Stream(device)
        self.d2h = torch.cuda.Stream(device)
        self.bufs = []

    def buffers(self, nelem):
        torch = _torch()
        if not self.bufs or self.bufs[0][0].numel() < nelem:
            self.bufs = [(torch.empty(nelem, dtype=torch.float64, device=self.device),
                          torch.empty(nelem, dtype=torch.float64, device=self.device))
                         for _ in range(3)]
        return self.bufs


_PIPES = {}
PIPE_CHUNK_BYTES = 64 << 20


def _pipelined_host_solve(plan, u_host, out_host, groups, sz):
    """Solve a pinned host field chunk by chunk (lines are independent):
    H2D of chunk i+1, the kernel on chunk i and D2H of chunk i-1 overlap, so
    PCIe runs full duplex. Blocks until the result is in out_host."""
    torch = _torch()
    dev = torch.cuda.current_device()
    pipe = _PIPES.get(dev)
    if pipe is None:
        pipe = _PIPES[dev] = _HostPipe(dev)
    per_group = u_host[0].numel()
    import os
    chunk_bytes = int(os.environ.get("TDS_PIPE_MB", "0")) << 20 or PIPE_CHUNK_BYTES
    gchunk = max(1, min(groups, chunk_bytes // (8 * per_group)))
    bufs = pipe.buffers(gchunk * per_group)
    uf = u_host.view(groups, per_group)
    of = out_host.view(groups, per_group)
    cur = torch.cuda.current_stream()
    for s in (pipe.h2d, pipe.cmp, pipe.d2h):
        s.wait_stream(cur)
    free_in = [None] * 3
    free_out = [None] * 3
    lib = N.lib()
    for i, g0 in enumerate(range(0, groups, gchunk)):
        g1 = min(groups, g0 + gchunk)
        k = i % 3
        din, dout = bufs[k][0][:(g1 - g0) * per_group], bufs[k][1][:(g1 - g0) * per_group]
        if free_in[k] is not None:
            pipe.h2d.wait_event(free_in[k])
        with torch.cuda.stream(pipe.h2d):
            din.copy_(uf[g0:g1].reshape(-1), non_blocking=True)
        loaded = torch.cuda.Event()
        loaded.record(pipe.h2d)
        pipe.cmp.wait_event(loaded)
        if free_out[k] is not None:
            pipe.cmp.wait_event(free_out[k])
        N.check(lib.tds_solve(plan.handle, ctypes.c_void_p(din.data_ptr()),
                              ctypes.c_void_p(dout.data_ptr()), g1 - g0, sz,
                              ctypes.c_void_p(pipe.cmp.cuda_stream)), plan.rank_count)
        solved = torch.cuda.Event()
        solved.record(pipe.cmp)
        free_in[k] = solved
        pipe.d2h.wait_event(solved)
        with torch.cuda.stream(pipe.d2h):
            of[g0:g1].reshape(-1).copy_(dout, non_blocking=True)
        drained = torch.cuda.Event()
        drained.record(pipe.d2h)
        free_out[k] = drained
    pipe.d2h.synchronize()


def run_distd2(sys, field_values, part=None, stencil=None, rank_count=None,
               warn_not_dominant=True, audit=None, *, arithmetic="fast", stream=None,
               out=None, devices=None):
    """Solve A u = stencil(field) over P subdomains (distributed.py:399-449).

    field_values: (n_groups, n, sz) NumPy array or CUDA tensor. P=1 gives the
    serial (periodic) Thomas result; P>1 the reference's DistD2 truncation at
    the same subdomain boundaries.

    How P>1 runs:
      * default: one whole-operator kernel on the current GPU, the rank
        boundaries folded into its reduced map (fastest; no messages);
      * `devices=[d_0, ..., d_{P-1}]` (CUDA device per rank, repeats allowed):
        P real ranks in this process (the reference's spawn_ranks shape),
        per-rank kernels with in-kernel neighbour rounds over NVLink peer
        memory (k_dd / k_dd2), or the two-pass path through device messages;
      * `audit=dict`: the real ranks as above (on `devices`, default all on
        the current GPU) with fresh contexts, so rounds / messages / bytes are
        the ones actually exchanged (messages of the fused kernels are counted
        on the device from the words they post).
    One rank per PROCESS (torchrun) is `DistD2Rank`. Keyword extensions:
    `arithmetic` ("fast" | "strict"), `stream` (torch.cuda.Stream), `out`
    (result buffer: a CUDA tensor, or a pinned CPU tensor for host-resident
    pipelines), `devices`."""
    shape = tuple(field_values.shape)
    if len(shape) != 3:
        raise ValueError(f"field must be (n_groups, n, sz), got {shape}")
    groups, n, sz = shape
    if part is None:
        part = SubdomainPartition.balanced(n, 1 if rank_count is None else rank_count)
    if part.n != n:
        raise ValueError(f"partition covers {part.n} positions, field has {n}")
    if stencil is not None and stencil.n != n:
        raise ValueError(f"stencil has {stencil.n} rows, field has {n}")
    if sys.n != n:
        raise ValueError(f"system size {sys.n} does not match field positions {n}")
    if part.rank_count > 1 and warn_not_dominant:
        for k in range(part.rank_count):
            if not is_diagonally_dominant(local_slice(sys, part, k)):
                warnings.warn("local block is not strictly diagonally dominant",
                              NotDominantWarning, stacklevel=2)
    torch = _torch()
    if part.rank_count > 1 and (devices is not None or audit is not None):
        return _run_ranks(sys, field_values, part, stencil, warn_not_dominant, audit,
                          arithmetic, stream, out, devices)
    plan = get_plan(sys, stencil, part, -1, arithmetic)
    if (isinstance(field_values, torch.Tensor) and not field_values.is_cuda
            and field_values.is_pinned() and field_values.dtype == torch.float64
            and field_values.is_contiguous() and groups >= 2):
        res = out if out is not None else torch.empty(shape, dtype=torch.float64,
                                                      pin_memory=True)
        _pipelined_host_solve(plan, field_values, res, groups, sz)
        return res
    fld = _Field(field_values)
    if groups * sz == 0:
        return fld.give(fld.empty_like(), out)
    res = out if (out is not None and not fld.host) else fld.empty_like()
    N.check(N.lib().tds_solve(plan.handle, fld.ptr, ctypes.c_void_p(res.data_ptr()),
                              groups, sz, _stream_handle(stream)), part.rank_count)
    if out is not None and not fld.host:
        return res
    return fld.give(res, out)


def _run_ranks(sys, field_values, part, stencil, warn_not_dominant, audit, arithmetic, stream,
               out, devices):
    """run_distd2 over P real in-process ranks (see run_distd2)."""
    torch = _torch()
    if devices is None:
        _need_cuda()
        devices = [torch.cuda.current_device()] * part.rank_count
    fresh = audit is not None
    group = _rank_group(sys, stencil, part, devices, arithmetic, warn_not_dominant, fresh)
    try:
        rounds_before = [c.exchange_rounds for c in group.contexts]
        fld = _Field(field_values)
        ctx_stream = torch.cuda.stream(stream) if stream is not None else None
        if ctx_stream is not None:
            ctx_stream.__enter__()
        try:
            res = out if (out is not None and not fld.host) else fld.empty_like()
            if fld.t.numel():
                group.solve(fld.t, res)
        finally:
            if ctx_stream is not None:
                ctx_stream.__exit__(None, None, None)
        if audit is not None:
            group.audit(audit, rounds_before)
        if out is not None and not fld.host:
            return res
        return fld.give(res, out)
    finally:
        if fresh:
            group.close()


# ------------------------------------------------------ phase functions

_DEV_COEFFS = {}
_DEV_COEFFS_MAX = 64


def _dev(arr, device):
    """Device copy of a host coefficient array, cached per (array, device):
    the phase kernels take device coefficients (no per-call allocation or
    host synchronisation inside the ABI)."""
    torch = _torch()
    key = (id(arr), str(device))
    hit = _DEV_COEFFS.get(key)
    if hit is not None and hit[0] is arr:
        return hit[1]
    if len(_DEV_COEFFS) >= _DEV_COEFFS_MAX:
        _DEV_COEFFS.pop(next(iter(_DEV_COEFFS)))
    t = torch.from_numpy(np.ascontiguousarray(arr, dtype=np.float64)).to(device)
    _DEV_COEFFS[key] = (arr, t)
    return t


def _lanes_of(shape):
    lanes = 1
    for s in shape[1:]:
        lanes *= s
    return lanes


def decouple_fused(u_ext, coeffs, stencil):
    """Alg. 6 on a halo-extended block (m+4, ...) -> (m, ...), reference
    arithmetic on the GPU (distributed.py:257-276)."""
    m = coeffs.n_loc
    if u_ext.shape[0] != m + 4:
        raise ValueError(f"expected {m + 4} positions incl. halo, got {u_ext.shape[0]}")
    fld = _Field(u_ext)
    d = fld.empty_like((m,) + tuple(u_ext.shape[1:]))
    dev = fld.t.device
    st = _dev(stencil.c, dev)[:m].contiguous()
    w, f, r = (_dev(x, dev) for x in (coeffs.w, coeffs.f, coeffs.r))
    sh4 = stencil.rows(0, m).shift4() if stencil.n != m else stencil.shift4()
    st_p, w_p, f_p, r_p = (ctypes.c_void_p(x.data_ptr()) for x in (st, w, f, r))
    N.check(N.lib().tds_decouple_fused(fld.ptr, st_p, N.iptr(sh4), w_p, f_p, r_p,
                                       ctypes.c_void_p(d.data_ptr()), m,
                                       _lanes_of(u_ext.shape), _stream_handle()))
    return fld.give(d)


def decouple_unfused(d_rhs, coeffs):
    """Sweeps over an already-built RHS (distributed.py:242-254): Alg. 6 with
    the identity stencil on a zero-padded block."""
    torch = _torch()
    m = coeffs.n_loc
    fld = _Field(d_rhs)
    pad = torch.zeros((m + 4,) + tuple(fld.t.shape[1:]), dtype=torch.float64,
                      device=fld.t.device)
    pad[2:m + 2] = fld.t
    d = decouple_fused(pad, coeffs, identity_stencil(m))
    return fld.give(d)


def solve_boundary_pair(pair):
    """Cramer solve of the 2x2 pair (distributed.py:279-293)."""
    det = 1.0 - pair.s_c_last * pair.s_a_first_remote
    if abs(det) < PAIR_DET_FLOOR:
        raise SingularPair(f"boundary determinant {det:.3e}")
    dl = _Field(pair.d_last_local)
    df = _Field(pair.d_first_remote)
    ul, uf = dl.empty_like(), dl.empty_like()
    N.check(N.lib().tds_boundary_pair(dl.ptr, df.ptr, float(pair.s_c_last),
                                      float(pair.s_a_first_remote),
                                      ctypes.c_void_p(ul.data_ptr()),
                                      ctypes.c_void_p(uf.data_ptr()), dl.t.numel(),
                                      _stream_handle()))
    return dl.give(ul), dl.give(uf)


def substitute(d, coeffs, u_start, u_end):
    """Alg. 7 (distributed.py:296-305), reference arithmetic on the GPU."""
    m = coeffs.n_loc
    fd = _Field(d)
    us, ue = _Field(u_start), _Field(u_end)
    out = fd.empty_like()
    sa, sc = (ctypes.c_void_p(_dev(x, fd.t.device).data_ptr()) for x in (coeffs.s_a, coeffs.s_c))
    N.check(N.lib().tds_substitute(fd.ptr, sa, sc, us.ptr, ue.ptr,
                                   ctypes.c_void_p(out.data_ptr()), m, _lanes_of(d.shape),
                                   _stream_handle()))
    return fd.give(out)
