"""Momentum-transport right-hand side on a periodic box, on the GPU: the
consumer of the DistD2 path in the reference (momentum.py:1-222).

    RHS_j of u_i = -1/2 (u_j d(u_i)/dx_j + d(u_j u_i)/dx_j) + nu d2(u_i)/dx_j2

Work is grouped by direction j like the reference, but nothing is re-laid
out: one `k_transport_dir` launch per direction reads u, v, w once (the y / z
lines in place from the x layout), runs the nine compact solves of that
direction and writes (x) or adds (y, z: TMA reduce-add) all three
components' contributions -- 192 B per grid point for the whole RHS.
`SlabTransport` splits the box into z-slabs over the ranks; its z pass is
`k_dd_transport_dir`, the same nine solves with the DistD2 neighbour rounds
in-kernel. Shapes these kernels cannot tile fall back, direction by
direction, to one fused kernel per (i, j) term (`k_transport_tma`) and the
reference-shaped reorder pipeline. Field data stays on the device (CUDA
tensors) for the whole pipeline.
"""

import ctypes
from dataclasses import dataclass

import numpy as np

from . import _native as N
from .compact import assemble, second_derivative_scheme, sixth_order_first_derivative
from .distributed import _stream_handle, get_plan, run_distd2
from .layout import GroupedField, LayoutDescriptor, pack
from .system import SubdomainPartition

import threading

_COMPONENTS = ("u", "v", "w")
_TRUSTED = threading.local()
_DIRECTIONS = ("x", "y", "z")


def _torch():
    import torch
    return torch


def _vp(t):
    return ctypes.c_void_p(t.data_ptr())


@dataclass(frozen=True)
class VelocityField:
    """Three velocity components in one SZ-blocked layout (momentum.py:32-67)."""

    u: GroupedField
    v: GroupedField
    w: GroupedField
    nu: float
    h: float

    def __post_init__(self):
        lay = self.u.layout
        if self.v.layout != lay or self.w.layout != lay:
            raise ValueError("velocity components must share one layout")
        if not (lay.nx == lay.ny == lay.nz):
            raise ValueError("transport demo expects a cubic grid")
        if getattr(_TRUSTED, "on", False):      # re-laid-out copies of checked data
            return
        torch = _torch()
        for f in (self.u, self.v, self.w):
            data = f.data
            finite = (torch.isfinite(data).all().item() if isinstance(data, torch.Tensor)
                      else np.all(np.isfinite(data)))
            if not finite:
                raise ValueError("velocity values must be finite")
        if self.h <= 0:
            raise ValueError("grid spacing must be positive")

    @property
    def layout(self):
        return self.u.layout

    @property
    def n(self):
        return self.layout.nx

    def component(self, i):
        return (self.u, self.v, self.w)[i]

    @classmethod
    def from_arrays(cls, u3, v3, w3, nu, h, sz=8, pad=False):
        """Pack three Cartesian arrays (NumPy or CUDA tensors) for x; the
        packed data lives on the GPU."""
        torch = _torch()

        def dev(a):
            if isinstance(a, torch.Tensor):
                return a.to("cuda", torch.float64)
            return torch.from_numpy(np.ascontiguousarray(a, dtype=np.float64)).cuda()

        u3, v3, w3 = dev(u3), dev(v3), dev(w3)
        lay = LayoutDescriptor(*u3.shape, sz=sz, direction="x", pad=pad)
        return cls(pack(u3, lay), pack(v3, lay), pack(w3, lay), nu, h)


_OPERATOR_CACHE = {}


def _operator(order, h, n):
    key = (order, h, n)
    hit = _OPERATOR_CACHE.get(key)
    if hit is None:
        scheme = sixth_order_first_derivative(h) if order == 1 else second_derivative_scheme(h)
        hit = assemble(scheme, n, periodic=True)
        _OPERATOR_CACHE[key] = hit
    return hit


def _product(a, b):
    """a * b elementwise on the device (k_axpy_mul)."""
    out = _torch().empty_like(a)
    N.check(N.lib().tds_multiply(_vp(a), _vp(b), _vp(out), out.numel(), _stream_handle()))
    return out


def _euler(u, rhs, dt):
    """u + dt * rhs elementwise on the device (k_axpy_mul)."""
    out = _torch().empty_like(u)
    N.check(N.lib().tds_euler_update(_vp(u), _vp(rhs), float(dt), _vp(out), out.numel(),
                                     _stream_handle()))
    return out


def _component_index(i):
    return _COMPONENTS.index(i) if isinstance(i, str) else int(i)


def _direction_name(j):
    return j if isinstance(j, str) else _DIRECTIONS[int(j)]


def _fused_contribution(comp, advect, out, n, h, nu, accumulate):
    """One fused k_transport launch if the shape allows it: the TMA-staged
    16-row-chunk kernel first, then the 32-row kernel. False = not fused."""
    groups, _, sz = comp.shape
    s1, st1 = _operator(1, h, n)
    s2, st2 = _operator(2, h, n)
    part = SubdomainPartition((n,))
    for rows in (16, 32):
        if accumulate and rows == 16:
            continue
        p1 = get_plan(s1, st1, part, chunk_rows=rows)
        if p1.info.chunk_rows != rows:
            continue
        p2 = get_plan(s2, st2, part, chunk_rows=rows) if nu != 0.0 else None
        rc = N.lib().tds_transport_contribution(
            p1.handle, None if p2 is None else p2.handle, _vp(comp), _vp(advect), _vp(out),
            float(nu), int(accumulate), groups, sz, _stream_handle())
        if rc == N.TDS_OK:
            return True
        if rc != N.TDS_ERR_UNSUPPORTED:
            N.check(rc)
    return False


def _contribution_into(ci, dj, fields, out, accumulate, rank_count):
    """out (=|+=) the (ci, dj) contribution, all arrays in the dj layout."""
    n = fields.n
    comp = fields.component(ci).data
    advect = fields.component(_DIRECTIONS.index(dj)).data
    groups, _, sz = comp.shape
    s1, st1 = _operator(1, fields.h, n)
    s2, st2 = _operator(2, fields.h, n)
    if rank_count == 1 and _fused_contribution(comp, advect, out, n, fields.h, fields.nu,
                                                accumulate):
        return
    # general path: three DistD2 solves (any size, emulated ranks) + combine
    d_comp = run_distd2(s1, comp, stencil=st1, rank_count=rank_count)
    d_prod = run_distd2(s1, _product(advect, comp), stencil=st1, rank_count=rank_count)
    d2 = (run_distd2(s2, comp, stencil=st2, rank_count=rank_count)
          if fields.nu != 0.0 else None)
    N.check(N.lib().tds_transport_combine(
        _vp(advect), _vp(d_comp), _vp(d_prod), None if d2 is None else _vp(d2),
        float(fields.nu), _vp(out), out.numel(), int(accumulate), _stream_handle()))


def directional_contribution(i, j, fields, rank_count=1, ledger=None, catalog=None):
    """Direction-j transport contribution to component i, in j layout
    (momentum.py:102-126)."""
    torch = _torch()
    ci = _component_index(i)
    dj = _direction_name(j)
    lay = fields.layout
    if lay.direction != dj:
        raise ValueError(f"fields are packed for {lay.direction!r}, kernel needs {dj!r}")
    out = torch.empty_like(fields.component(ci).data)
    _contribution_into(ci, dj, fields, out, False, rank_count)
    return GroupedField(lay, out)


def _reorder_tensor(data, n, sz, src, dst, out=None, accumulate=False):
    torch = _torch()
    res = torch.empty_like(data) if out is None else out
    N.check(N.lib().tds_reorder(_vp(data), _vp(res), n, sz, _DIRECTIONS.index(src),
                                _DIRECTIONS.index(dst), int(accumulate), _stream_handle()))
    return res


def evaluate_transport_rhs(fields, rank_count=1, ledger=None, catalog=None):
    """Full right-hand side of all three components, x-layout results
    (momentum.py:142-169).

    Default: one `k_transport_dir` launch per direction (x writes the
    accumulators, y / z add into them in place), each reading u, v, w once
    (`tds_transport_direction`). Shapes it cannot tile take the per-term
    kernels below, direction by direction."""
    torch = _torch()
    if fields.layout.direction != "x":
        raise ValueError("inputs must arrive in x layout")
    lay = fields.layout
    n, sz = lay.nx, lay.sz
    if lay.pad:
        raise NotImplementedError("padded layouts are not supported by the GPU transport demo")
    acc = [torch.empty_like(fields.component(i).data) for i in range(3)]
    done = _direction_passes(fields, acc, (0, 1, 2)) if rank_count == 1 else set()
    if 0 not in done:
        for i in range(3):
            _contribution_into(i, "x", fields, acc[i], False, rank_count)
    scratch = None
    # y / z contributions read in place from the x layout and added into the
    # accumulators (k_transport_tma GEOM_XY / GEOM_XZ) when the box allows
    for dj in ("y", "z"):
        if _DIRECTIONS.index(dj) in done:
            continue
        plans = _in_x_plans(fields, dj) if rank_count == 1 else None
        if plans is not None:
            p1, p2 = plans
            adv = fields.component(_DIRECTIONS.index(dj)).data
            ndone = 0
            for i in range(3):
                rc = N.lib().tds_transport_contribution_in_x(
                    p1.handle, None if p2 is None else p2.handle,
                    _vp(fields.component(i).data), _vp(adv), _vp(acc[i]), float(fields.nu), n,
                    n, n, sz, _DIRECTIONS.index(dj), _stream_handle())
                if rc == N.TDS_ERR_UNSUPPORTED and i == 0:
                    break                     # shape not tileable: reorder path below
                N.check(rc)
                ndone += 1
            if ndone == 3:
                continue
        lay_j = LayoutDescriptor(n, n, n, sz, dj)
        _TRUSTED.on = True
        try:
            rot = VelocityField(*(GroupedField(lay_j, _reorder_tensor(fields.component(c).data,
                                                                      n, sz, "x", dj))
                                  for c in range(3)), fields.nu, fields.h)
        finally:
            _TRUSTED.on = False
        if scratch is None:
            scratch = torch.empty_like(acc[0])
        for i in range(3):
            _contribution_into(i, dj, rot, scratch, False, rank_count)
            _reorder_tensor(scratch, n, sz, dj, "x", out=acc[i], accumulate=True)
    return tuple(GroupedField(lay, a) for a in acc)


def _direction_plans(h, nu, rows):
    """16-row-chunk uniform P=1 plans of the d/dx and (nu != 0) d2/dx2
    operators of `rows`-long periodic lines, or None."""
    part = SubdomainPartition((rows,))
    s1, st1 = _operator(1, h, rows)
    p1 = get_plan(s1, st1, part, chunk_rows=16)
    if p1.info.chunk_rows != 16 or p1.info.uniform != 1:
        return None
    p2 = None
    if nu != 0.0:
        s2, st2 = _operator(2, h, rows)
        p2 = get_plan(s2, st2, part, chunk_rows=16)
        if p2.info.chunk_rows != 16 or p2.info.uniform != 1:
            return None
    return p1, p2


def _direction_pass(u, acc, extents, sz, h, nu, dj):
    """One `tds_transport_direction` launch (k_transport_dir: the three
    components' contributions along direction dj, u[0..2] read once) on an
    x-layout (nx, ny, nz) block; dj = 0 writes `acc`, 1 / 2 add into it.
    False when the kernel cannot tile the shape (per-term path instead).
    A/B knob: TDS_TRANSPORT_DIR=0."""
    import os
    if os.environ.get("TDS_TRANSPORT_DIR") == "0":
        return False
    nx, ny, nz = extents
    rows = extents[dj]
    if ny % sz or rows % 16:
        return False
    plans = _direction_plans(h, nu, rows)
    if plans is None:
        return False
    p1, p2 = plans
    rc = N.lib().tds_transport_direction(
        p1.handle, None if p2 is None else p2.handle, _vp(u[0]), _vp(u[1]), _vp(u[2]),
        _vp(acc[0]), _vp(acc[1]), _vp(acc[2]), float(nu), nx, ny, nz, sz, dj,
        _stream_handle())
    if rc == N.TDS_ERR_UNSUPPORTED:
        return False
    N.check(rc)
    return True


def _direction_passes(fields, acc, dirs, extents=None):
    """`_direction_pass` for the directions in `dirs`, in order, stopping at
    the first one the kernel cannot tile (the rest then run per term, in the
    same order, so the accumulation order never changes). Returns the set of
    directions done."""
    lay = fields.layout
    if lay.pad:
        return set()
    ext = extents if extents is not None else (lay.nx, lay.ny, lay.nz)
    u = [fields.component(c).data for c in range(3)]
    done = set()
    for dj in dirs:
        if not _direction_pass(u, acc, ext, lay.sz, fields.h, fields.nu, dj):
            break
        done.add(dj)
    return done


def _in_x_plans(fields, dj):
    """16-row-chunk plans for the in-place y / z contributions
    (k_transport_tma GEOM_XY / GEOM_XZ), or None when the box / layout does
    not allow them. A/B knobs: TDS_TRANSPORT_Y=0, TDS_TRANSPORT_Z=0."""
    import os
    lay = fields.layout
    n, sz = lay.nx, lay.sz
    if lay.pad or n % sz or sz % 8 or n % 16:
        return None
    if os.environ.get("TDS_TRANSPORT_" + dj.upper()) == "0":
        return None
    if dj == "y" and (sz != 32 or n % 32):
        return None
    part = SubdomainPartition((n,))
    s1, st1 = _operator(1, fields.h, n)
    p1 = get_plan(s1, st1, part, chunk_rows=16)
    if p1.info.chunk_rows != 16 or p1.info.uniform != 1:
        return None
    p2 = None
    if fields.nu != 0.0:
        s2, st2 = _operator(2, fields.h, n)
        p2 = get_plan(s2, st2, part, chunk_rows=16)
        if p2.info.chunk_rows != 16 or p2.info.uniform != 1:
            return None
    return p1, p2


def _local_contribution(comp, advect, out, n, h, nu, accumulate):
    """out (=|+=) the contribution along a direction whose lines are whole on
    this device: comp, advect, out are (groups, n, sz) tensors."""
    torch = _torch()
    if _fused_contribution(comp, advect, out, n, h, nu, accumulate):
        return
    s1, st1 = _operator(1, h, n)
    s2, st2 = _operator(2, h, n)
    d_comp = run_distd2(s1, comp, stencil=st1)
    d_prod = run_distd2(s1, _product(advect, comp), stencil=st1)
    d2 = run_distd2(s2, comp, stencil=st2) if nu != 0.0 else None
    N.check(N.lib().tds_transport_combine(
        _vp(advect), _vp(d_comp), _vp(d_prod), None if d2 is None else _vp(d2),
        float(nu), _vp(out), out.numel(), int(accumulate), _stream_handle()))


class SlabTransport:
    """The transport right-hand side (BASELINE config 5) on P GPUs, one
    process per GPU: rank r owns the z-slab [off_r, off_r + m_r) of the
    periodic n^3 box (SubdomainPartition.balanced(n, P), system.py:148-155).

    * x and y lines are whole on every rank: those contributions are local
      (fused k_transport when n <= 512, else three solves + combine);
    * z lines are split across the ranks: each z contribution is three
      DistD2 solves along the rank chain (DistD2Rank: the fused k_dd/k_dd2
      kernels with in-kernel NVLink exchange) + k_transport_combine -- the
      reference's evaluate_transport_rhs (momentum.py:142-169) with its
      rank_count applied to z, the direction the box is decomposed along.
    Local fields are x-layout (n*m/sz, n, sz) tensors of the rank's slab,
    i.e. pack(u3[:, :, off:off+m], LayoutDescriptor(n, n, m, sz, 'x')).
    The layouts of the slab (x, y: whole lines; z: this rank's rows of every
    global z line) are reached with the one-pass k_reorder (tds_reorder3)."""

    def __init__(self, n, sz, nu, h, ctx=None):
        from .rank import DistD2Rank
        self.n, self.sz, self.nu, self.h, self.ctx = n, sz, float(nu), float(h), ctx
        p = 1 if ctx is None else ctx.rank_count
        self.part = SubdomainPartition.balanced(n, p)
        r = 0 if ctx is None else ctx.rank_id
        self.m = self.part.local_sizes[r]
        self.off = self.part.offsets()[r]
        self.lay = {d: LayoutDescriptor(n, n, self.m, sz, d) for d in _DIRECTIONS}
        self._rank = None
        self._marks = None
        if p > 1:
            if not ctx.cyclic:
                raise ValueError("the transport box is periodic: the rank chain must be a ring")
            s1, st1 = _operator(1, self.h, n)
            s2, st2 = _operator(2, self.h, n)
            self._rank = (DistD2Rank(s1, st1, self.part, ctx),
                          DistD2Rank(s2, st2, self.part, ctx) if self.nu != 0.0 else None)
            # fused z terms (k_dd_transport): per-rank 16-row-chunk plans of
            # both operators + one IPC mailbox set per field shape
            from .distributed import Plan
            import os
            self._zfused = None
            # equal blocks on every rank (identical persistent schedules).
            # Measured faster than three k_dd2 solves + combine at every m
            # tried (z phase, 1024^3 on 2 GPUs: 34.7 vs 41.8 ms; 512^3 on 4
            # GPUs: 2.21 vs 2.99 ms). TDS_FUSED_TRANSPORT=0: never.
            knob = os.environ.get("TDS_FUSED_TRANSPORT", "1")
            if knob != "0" and len(set(self.part.local_sizes)) == 1:
                r = ctx.rank_id
                self._zfused = (
                    Plan.create(s1, st1.c, self.part.local_sizes, r, N.TDS_FLAG_CHUNK16),
                    Plan.create(s2, st2.c, self.part.local_sizes, r, N.TDS_FLAG_CHUNK16)
                    if self.nu != 0.0 else None)
            self._zmail = {}
            self._zepoch = 0
            self._zbroken = None
            self._zdir = None          # k_dd_transport_dir usable (None: not tried yet)

    def local_slab(self, u3):
        """Pack this rank's slab of a global Cartesian (n, n, n) array for x."""
        torch = _torch()
        t = u3 if isinstance(u3, torch.Tensor) else torch.from_numpy(np.ascontiguousarray(u3))
        slab = t[:, :, self.off:self.off + self.m].to("cuda", torch.float64).contiguous()
        return pack(slab, self.lay["x"]).data

    def _reorder(self, src, a, b, out=None, accumulate=False):
        torch = _torch()
        dst = self.lay[b]
        res = (torch.empty((dst.n_groups, dst.n, dst.sz), dtype=torch.float64,
                           device=src.device) if out is None else out)
        N.check(N.lib().tds_reorder3(_vp(src), _vp(res), self.n, self.n, self.m, self.sz,
                                     _DIRECTIONS.index(a), _DIRECTIONS.index(b),
                                     int(accumulate), _stream_handle()))
        return res

    def _y_in_place(self, vel, acc):
        """y terms read in place from the slab's x layout and added into acc
        (tds_transport_contribution_in_x, GEOM_XY); False if not tileable."""
        import os
        if os.environ.get("TDS_TRANSPORT_Y") == "0" or self.sz != 32 or self.n % 32:
            return False
        n = self.n
        part = SubdomainPartition((n,))
        s1, st1 = _operator(1, self.h, n)
        p1 = get_plan(s1, st1, part, chunk_rows=16)
        p2 = None
        if self.nu != 0.0:
            s2, st2 = _operator(2, self.h, n)
            p2 = get_plan(s2, st2, part, chunk_rows=16)
        for i in range(3):
            rc = N.lib().tds_transport_contribution_in_x(
                p1.handle, None if p2 is None else p2.handle, _vp(vel[i]), _vp(vel[1]),
                _vp(acc[i]), self.nu, n, n, self.m, self.sz, 1, _stream_handle())
            if rc == N.TDS_ERR_UNSUPPORTED and i == 0:
                return False
            N.check(rc)
        return True

    def _z_fused(self, comp, advect, out):
        """The z term as one k_dd_transport launch per rank; False when the
        plans / shape do not allow it (then three DistD2Rank solves)."""
        if not self._zfused:
            return False
        if self._zbroken is not None:
            raise TimeoutError(str(self._zbroken))
        p1, p2 = self._zfused
        groups, m, sz = comp.shape
        key = (groups, sz)
        mb = self._zmail.get(key)
        if mb is None:
            mb = self.ctx.open_mailboxes(N.lib().tds_transport_mailbox_words(groups, sz))
            self._zmail[key] = mb
        self._poll_z()
        self._zepoch += 1
        stream = _torch().cuda.current_stream()
        rc = N.lib().tds_fused_transport(
            p1.handle, None if p2 is None else p2.handle, _vp(comp), _vp(advect), _vp(out),
            self.nu, groups, sz, mb.own, mb.prev, mb.next, self._zepoch,
            self.ctx.fused_grid_cap, ctypes.c_void_p(stream.cuda_stream))
        if rc == N.TDS_ERR_UNSUPPORTED and self._zepoch == 1:
            self._zfused = None        # same decision on every rank: plans / shape only
            return False
        N.check(rc)
        mb.post_status(stream)
        self.ctx.exchange_rounds += 6
        return True

    def _z_in_x(self, vel, acc):
        """The three z terms read in place from the slab's x layout and added
        into acc (tds_fused_transport_in_x: k_dd_transport on the slab's z
        lines, TMA reduce-add) -- no re-layout passes. False when the plans /
        shape do not allow it (the same decision on every rank: plans and
        shape only). A/B knob: TDS_TRANSPORT_Z=0."""
        import os
        if not self._zfused or os.environ.get("TDS_TRANSPORT_Z") == "0":
            return False
        if self._zbroken is not None:
            raise TimeoutError(str(self._zbroken))
        p1, p2 = self._zfused
        n, sz, m = self.n, self.sz, self.m
        groups = n * n // sz
        key = (groups, sz)
        mb = self._zmail.get(key)
        if mb is None:
            mb = self.ctx.open_mailboxes(N.lib().tds_transport_mailbox_words(groups, sz))
            self._zmail[key] = mb
        self._poll_z()
        stream = _torch().cuda.current_stream()
        if os.environ.get("TDS_TRANSPORT_DIR") != "0" and self._zdir is not False:
            # all three components in one kernel per rank (k_dd_transport_dir)
            self._zepoch += 1
            rc = N.lib().tds_fused_transport_direction(
                p1.handle, None if p2 is None else p2.handle, _vp(vel[0]), _vp(vel[1]),
                _vp(vel[2]), _vp(acc[0]), _vp(acc[1]), _vp(acc[2]), self.nu, n, n, m, sz,
                mb.own, mb.prev, mb.next, self._zepoch, self.ctx.fused_grid_cap,
                ctypes.c_void_p(stream.cuda_stream))
            if rc == N.TDS_OK:
                self._zdir = True
                self.ctx.exchange_rounds += 18       # 9 solves x 2 rounds, as 3 terms
                mb.post_status(stream)
                return True
            if rc != N.TDS_ERR_UNSUPPORTED or self._zdir:
                N.check(rc)
            self._zepoch -= 1
            self._zdir = False             # same decision on every rank: plans / shape only
        for i in range(3):
            self._zepoch += 1
            rc = N.lib().tds_fused_transport_in_x(
                p1.handle, None if p2 is None else p2.handle, _vp(vel[i]), _vp(vel[2]),
                _vp(acc[i]), self.nu, n, n, m, sz, mb.own, mb.prev, mb.next, self._zepoch,
                self.ctx.fused_grid_cap, ctypes.c_void_p(stream.cuda_stream))
            if rc == N.TDS_ERR_UNSUPPORTED and i == 0:
                self._zepoch -= 1
                return False
            N.check(rc)
            self.ctx.exchange_rounds += 6
        mb.post_status(stream)
        return True

    def _poll_z(self, block=False):
        """Fold the fused z kernels' status words into the context: one
        message per field halo (2 L posted words per directed edge: u_i and
        u_j per term, u_0..u_2 per direction kernel) and per boundary row
        (L words per solve); TimeoutError if a wait timed out."""
        from .rank import account_status
        for (groups, sz), mb in self._zmail.items():
            lines = groups * sz
            try:
                account_status(self.ctx, mb, 2 * lines, lines, block)
            except TimeoutError as exc:
                self._zbroken = exc
                raise

    def _z_contribution(self, comp, advect, out):
        torch = _torch()
        if self._rank is None:
            _local_contribution(comp, advect, out, self.m, self.h, self.nu, False)
            return
        if self._z_fused(comp, advect, out):
            return
        r1, r2 = self._rank
        d_comp = r1.solve(comp)
        d_prod = r1.solve(_product(advect, comp))
        d2 = r2.solve(comp) if r2 is not None else None
        N.check(N.lib().tds_transport_combine(
            _vp(advect), _vp(d_comp), _vp(d_prod), None if d2 is None else _vp(d2),
            self.nu, _vp(out), out.numel(), 0, _stream_handle()))

    def rhs(self, u, v, w):
        """Local x-layout slabs of u, v, w -> local x-layout RHS of each
        component (momentum.py:142-169, same per-direction grouping). Local
        directions (x, y; z too on one rank) run as one k_transport_dir
        launch each when the shape allows it."""
        torch = _torch()
        vel = (u, v, w)
        acc = [torch.empty_like(u) for _ in range(3)]
        ext = (self.n, self.n, self.m)
        marks = self._marks
        if marks is not None:
            marks[0].record()
        xdir = _direction_pass(vel, acc, ext, self.sz, self.h, self.nu, 0)
        if not xdir:
            for i in range(3):
                _local_contribution(vel[i], vel[0], acc[i], self.n, self.h, self.nu, False)
        if marks is not None:
            marks[1].record()
        ydir = xdir and _direction_pass(vel, acc, ext, self.sz, self.h, self.nu, 1)
        if not ydir and not self._y_in_place(vel, acc):
            rot = [self._reorder(c, "x", "y") for c in vel]
            scratch = torch.empty_like(rot[0])
            for i in range(3):
                _local_contribution(rot[i], rot[1], scratch, self.n, self.h, self.nu, False)
                self._reorder(scratch, "y", "x", out=acc[i], accumulate=True)
        if marks is not None:
            marks[2].record()
        if self._rank is None:   # one rank: keep evaluate_transport_rhs's order
            zdone = ydir and _direction_pass(vel, acc, ext, self.sz, self.h, self.nu, 2)
        else:
            if self.ctx.fused_grid_cap < 0:
                # ranks sharing a device: a rank's fused z kernel waiting for
                # a neighbour must not hold SMs that the neighbour's
                # persistent x / y kernels still need -- all ranks finish the
                # local passes first
                torch.cuda.current_stream().synchronize()
                self.ctx.barrier()
            zdone = self._z_in_x(vel, acc)
        if not zdone:
            rot = [self._reorder(c, "x", "z") for c in vel]
            scratch = torch.empty_like(rot[0])
            for i in range(3):
                self._z_contribution(rot[i], rot[2], scratch)
                self._reorder(scratch, "z", "x", out=acc[i], accumulate=True)
        if marks is not None:
            marks[3].record()
        return tuple(acc)

    def phase_ms(self):
        """Per-direction device time (x, y, z terms) of the last rhs() call
        when timing was enabled with `timed(True)`."""
        m = self._marks
        return {d: m[k].elapsed_time(m[k + 1]) for k, d in enumerate("xyz")}

    def timed(self, on=True):
        torch = _torch()
        self._marks = ([torch.cuda.Event(enable_timing=True) for _ in range(4)] if on
                       else None)

    def euler_step(self, u, v, w, dt):
        """u <- u + dt * RHS(u) on this rank's slab (momentum.py:216-222)."""
        rhs = self.rhs(u, v, w)
        return tuple(_euler(c, r, dt) for c, r in zip((u, v, w), rhs))

    def check(self):
        """Wait for the last fused kernels' status; TimeoutError if a rank's
        neighbour never arrived (synchronous)."""
        for r in self._rank or ():
            if r is not None:
                r.check()
        if getattr(self, "_zbroken", None) is not None:
            raise TimeoutError(str(self._zbroken))
        if getattr(self, "_zmail", None):
            self._poll_z(block=True)

    @property
    def fused_z(self):
        return bool(getattr(self, "_zfused", None))

    def close(self):
        for r in self._rank or ():
            if r is not None:
                r.close()
        for mb in getattr(self, "_zmail", {}).values():
            mb.close()
        self._zmail = {}


def euler_step(fields, dt, rank_count=1):
    """u <- u + dt * RHS(u) (momentum.py:216-222)."""
    rhs = evaluate_transport_rhs(fields, rank_count=rank_count)
    comps = [GroupedField(fields.layout, _euler(fields.component(i).data, rhs[i].data, dt))
             for i in range(3)]
    return VelocityField(comps[0], comps[1], comps[2], fields.nu, fields.h)
