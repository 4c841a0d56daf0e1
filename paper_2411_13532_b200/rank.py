"""One rank per B200: the per-rank DistD2 solve (reference distributed.py:
327-366 run by transport.spawn_ranks, transport.py:105-139), with the two
neighbour rounds on NCCL (torch.distributed) and the arithmetic in
libtds_b200.so.

DistD2Rank.solve(u_local) for a rank holding rows [off, off+m) of every line:
    tds_halo_rows      -> rows {0,1}, {m-2,m-1}           (K1, tiny)
    ROUND 1            -> halo_lo / halo_hi               (NCCL P2P)
    tds_boundary_rows  -> d[0], d[m-1] of every line      (pass A: reads u)
    ROUND 2            -> prev's d[m-1], next's d[0]      (NCCL P2P)
    tds_finish         -> 2x2 pairs + substitution, out   (pass B: reads u,
                                                           writes out)
The two-pass path recomputes the decoupling in pass B instead of
materialising d: 24 B/point of HBM traffic.

FUSED path (default when every rank holds the same number of rows and the
field is TMA-eligible): ONE kernel per rank per solve, `tds_fused_solve`
(k_dd). Both neighbour rounds are NVLink peer stores into the neighbours'
IPC-mapped mailboxes with per-tile acquire/release flags -- 16 B/point, no
NCCL call and no host synchronisation on the solve path.
"""

import os

import ctypes

from . import _native as N
from .distributed import (Plan, _flags, _stream_handle, decouple_fused, solve_boundary_pair,
                          substitute, BoundaryPair)
from .transport import (BOUNDARY_HIGH, BOUNDARY_LOW, HALO_HIGH, HALO_LOW, exchange_boundary,
                        exchange_halo)


def _vp(t):
    return ctypes.c_void_p(0 if t is None else t.data_ptr())


def open_mailboxes(ctx, words):
    """Allocate this rank's sentinel-filled mailbox of `words` 8-byte slots,
    exchange CUDA IPC handles over the rank group, and map prev's / next's
    mailboxes: returns (own, prev, next, [mapped pointers])."""
    import torch.distributed as dist
    lib = N.lib()
    own = ctypes.c_void_p()
    handle = ctypes.create_string_buffer(64)
    N.check(lib.tds_ipc_alloc(words * 8, ctypes.byref(own), handle))
    handles = [None] * ctx.rank_count
    dist.all_gather_object(handles, handle.raw, group=ctx.group)
    opened = {}

    def open_rank(pos):
        pos %= ctx.rank_count
        if pos not in opened:
            ptr = ctypes.c_void_p()
            N.check(lib.tds_ipc_open(handles[pos], ctypes.byref(ptr)))
            opened[pos] = ptr
        return opened[pos]

    prev = open_rank(ctx.rank_id - 1) if ctx.has_prev else ctypes.c_void_p(0)
    nxt = open_rank(ctx.rank_id + 1) if ctx.has_next else ctypes.c_void_p(0)
    return own, prev, nxt, list(opened.values())


def close_mailboxes(mb):
    lib = N.lib()
    own, _, _, opened = mb
    for ptr in opened:
        lib.tds_ipc_close(ptr)
    lib.tds_ipc_free(own)


class DistD2Rank:
    """Per-rank solver object: plan (coefficient tables on this GPU) and the
    neighbour buffers, reused across solves."""

    def __init__(self, sys, stencil, part, ctx, arithmetic="fast"):
        if part.rank_count != ctx.rank_count:
            raise ValueError("partition and rank context disagree on the rank count")
        if part.rank_count < 2:
            raise ValueError("DistD2Rank needs at least two ranks; use run_distd2 for P=1")
        if sys.periodic != ctx.cyclic:
            raise ValueError("rank topology must be a ring exactly when the system is periodic")
        self.ctx = ctx
        self.part = part
        self.m = part.local_sizes[ctx.rank_id]
        st = None if stencil is None else stencil.c
        self.plan = Plan.create(sys, st, part.local_sizes, ctx.rank_id, _flags(arithmetic))
        self._bufs = {}
        self._mail = {}
        self._epoch = 0
        self.fused = (self.plan.path == "fast" and len(set(part.local_sizes)) == 1
                      and os.environ.get("TDS_FUSED", "1") != "0")

    @property
    def path(self):
        return self.plan.path

    def _buffers(self, groups, sz, device):
        import torch
        key = (groups, sz, str(device))
        b = self._bufs.get(key)
        if b is None:
            def e(*shape):
                return torch.empty(shape, dtype=torch.float64, device=device)
            b = dict(first2=e(groups, 2, sz), last2=e(groups, 2, sz),
                     halo_lo=e(groups, 2, sz) if self.ctx.has_prev else None,
                     halo_hi=e(groups, 2, sz) if self.ctx.has_next else None,
                     d_first=e(groups, sz), d_last=e(groups, sz),
                     prev_last=e(groups, sz) if self.ctx.has_prev else None,
                     next_first=e(groups, sz) if self.ctx.has_next else None)
            self._bufs[key] = b
        return b

    def _mailbox(self, groups, sz):
        """Own mailbox + the neighbours' mailboxes mapped through CUDA IPC
        (one collective handle exchange per field shape)."""
        key = (groups, sz)
        mb = self._mail.get(key)
        if mb is None:
            mb = open_mailboxes(self.ctx, N.lib().tds_mailbox_words(groups, sz))
            self._mail[key] = mb
        return mb

    def check(self):
        """Raise if a fused solve timed out waiting for a neighbour (reads the
        mailbox error words; synchronous)."""
        for (groups, sz), (own, _, _, _) in self._mail.items():
            err = ctypes.c_int(0)
            N.check(N.lib().tds_mailbox_error(own, groups, sz, ctypes.byref(err)))
            if err.value:
                raise TimeoutError(f"rank {self.ctx.rank_id}: fused DistD2 solve timed out "
                                   "waiting for a neighbour")

    def close(self):
        for mb in self._mail.values():
            close_mailboxes(mb)
        self._mail = {}

    def solve(self, u, out=None):
        """u: this rank's (n_groups, m, sz) fp64 CUDA tensor -> out (same shape)."""
        import torch
        groups, m, sz = u.shape
        if m != self.m:
            raise ValueError(f"rank {self.ctx.rank_id} holds {self.m} rows, got {m}")
        u = u.contiguous()
        if u.data_ptr() % 16:
            u = u.clone()
        if out is None:
            out = torch.empty_like(u)
        if self.fused and N.lib().tds_fused_eligible(self.plan.handle, groups, sz):
            own, prev, nxt, _ = self._mailbox(groups, sz)
            self._epoch += 1
            self.ctx.begin_solve()
            self.ctx.exchange_rounds += 2          # both rounds run inside the kernel
            N.check(N.lib().tds_fused_solve(self.plan.handle, _vp(u), _vp(out), groups, sz, own,
                                            prev, nxt, self._epoch, _stream_handle()))
            return out
        b = self._buffers(groups, sz, u.device)
        lib, h, s, ctx = N.lib(), self.plan.handle, _stream_handle(), self.ctx
        ctx.begin_solve()
        N.check(lib.tds_halo_rows(h, _vp(u), _vp(b["first2"]), _vp(b["last2"]), groups, sz, s))
        sends, recvs = [], []
        if ctx.has_next:
            sends.append((HALO_LOW, True, b["last2"]))
        if ctx.has_prev:
            sends.append((HALO_HIGH, False, b["first2"]))
            recvs.append((HALO_LOW, True, b["halo_lo"]))
        if ctx.has_next:
            recvs.append((HALO_HIGH, False, b["halo_hi"]))
        ctx.round(sends, recvs)
        N.check(lib.tds_boundary_rows(h, _vp(u), _vp(b["halo_lo"]), _vp(b["halo_hi"]),
                                      _vp(b["d_first"]), _vp(b["d_last"]), _vp(out),
                                      groups, sz, s))
        sends, recvs = [], []
        if ctx.has_next:
            sends.append((BOUNDARY_LOW, True, b["d_last"]))
        if ctx.has_prev:
            sends.append((BOUNDARY_HIGH, False, b["d_first"]))
            recvs.append((BOUNDARY_LOW, True, b["prev_last"]))
        if ctx.has_next:
            recvs.append((BOUNDARY_HIGH, False, b["next_first"]))
        ctx.round(sends, recvs)
        N.check(lib.tds_finish(h, _vp(u), _vp(b["halo_lo"]), _vp(b["halo_hi"]),
                               _vp(b["d_first"]), _vp(b["d_last"]), _vp(b["prev_last"]),
                               _vp(b["next_first"]), _vp(out), groups, sz, s))
        return out


def distd2_solve(ctx, local_values, coeffs, stencil, pair_coeffs):
    """Reference-shaped per-rank solve (distributed.py:327-366): exactly two
    neighbour rounds, every arithmetic phase a GPU kernel in the reference's
    operation order (bit-identical). local_values: (n_groups, m, sz) tensor."""
    import torch
    ctx.begin_solve()
    groups, m, sz = local_values.shape
    low, high = exchange_halo(ctx, local_values, stencil.halo_depth)
    lanes = groups * sz

    def lanes_of(block):
        return block.permute(1, 0, 2).reshape(block.shape[1], lanes)

    dep = stencil.halo_depth
    u_ext = torch.zeros((m + 2 * dep, lanes), dtype=torch.float64, device=local_values.device)
    if low is not None:
        u_ext[:dep] = lanes_of(low)
    u_ext[dep:dep + m] = lanes_of(local_values)
    if high is not None:
        u_ext[dep + m:] = lanes_of(high)
    d = decouple_fused(u_ext, coeffs, stencil)
    prev_last, next_first = exchange_boundary(ctx, d[0].reshape(groups, sz),
                                              d[m - 1].reshape(groups, sz))
    if prev_last is None:
        u_start = d[0]
    else:
        _, u_start = solve_boundary_pair(BoundaryPair(prev_last.reshape(-1), d[0],
                                                      pair_coeffs.prev_s_c_last,
                                                      coeffs.s_a[0]))
    if next_first is None:
        u_end = d[m - 1]
    else:
        u_end, _ = solve_boundary_pair(BoundaryPair(d[m - 1], next_first.reshape(-1),
                                                    coeffs.s_c[-1],
                                                    pair_coeffs.next_s_a_first))
    u = substitute(d, coeffs, u_start, u_end)
    return u.reshape(m, groups, sz).permute(1, 0, 2).contiguous()
