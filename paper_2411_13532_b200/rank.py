"""The per-rank DistD2 solve (reference distributed.py:308-366 run by
transport.spawn_ranks, transport.py:105-139): one rank per B200 process
(torchrun, `RankContext`) or several ranks in one process (`LocalRankContext`,
one stream per rank; ranks may share a device), arithmetic in libtds_b200.so.

Construction follows the reference's per-rank view: `preprocess` of the
rank's local_slice, the one-time neighbour share of the pair couplings
(share_pair_coeffs, distributed.py:308-324; D16) and a plan built from those
local data only (tds_plan_create_local).

DistD2Rank.solve(u_local) for a rank holding rows [off, off+m) of every line:

FUSED path (default when every rank holds the same number of rows and the
field is TMA-eligible): ONE kernel per rank per solve, `tds_fused_solve`
(k_dd / k_dd2). Both neighbour rounds are NVLink peer stores into the
neighbours' mailboxes -- 16 B/point, no NCCL call and no host
synchronisation on the solve path. The mailbox status words (error, posted
words) are copied back asynchronously and inspected at the next call:
a neighbour that never arrived raises TimeoutError (the kernel poisons the
affected rows with NaN instead of hanging) and the rank refuses further
fused solves; posted words become the context's message accounting.

TWO-PASS path (TDS_FUSED=0, ragged partitions, strict arithmetic):
    tds_halo_rows      -> rows {0,1}, {m-2,m-1}           (K1, tiny)
    ROUND 1            -> halo_lo / halo_hi               (ctx.round)
    tds_boundary_rows  -> d[0], d[m-1] of every line      (pass A: reads u)
    ROUND 2            -> prev's d[m-1], next's d[0]      (ctx.round)
    tds_finish         -> 2x2 pairs + substitution, out   (pass B)
"""

import ctypes
import os

from . import _native as N
from .distributed import (BoundaryPair, Plan, _flags, _stream_handle, decouple_fused,
                          local_slice, preprocess, rank_position, solve_boundary_pair,
                          substitute)
from .transport import (BOUNDARY_HIGH, BOUNDARY_LOW, HALO_HIGH, HALO_LOW, exchange_boundary,
                        exchange_halo, share_scalars)


def _vp(t):
    return ctypes.c_void_p(0 if t is None else t.data_ptr())


def open_mailboxes(ctx, words):
    """This rank's prepared mailbox of `words` slots + the neighbours' mapped
    ones (collective over the rank group); returns a transport.Mailboxes."""
    return ctx.open_mailboxes(words)


def close_mailboxes(mb):
    mb.close()


def account_status(ctx, mb, halo_words_per_msg, bnd_words_per_msg, block=False):
    """Fold the device-side posted-word counters of a mailbox into the
    context's message accounting; raise TimeoutError if the kernel recorded
    a timed-out wait. Returns True if the status was available."""
    st = mb.status(block=block)
    if st is None:
        return False
    err, halo, bnd = st
    dh, db = halo - mb.counted[0], bnd - mb.counted[1]
    if dh or db:
        mb.counted = [halo, bnd]
        ctx.messages_sent += dh // max(1, halo_words_per_msg) + db // max(1, bnd_words_per_msg)
        ctx.bytes_sent += 8 * (dh + db)
    if err:
        raise TimeoutError(f"rank {ctx.rank_id}: fused solve timed out waiting for a neighbour "
                           "(its rows were poisoned with NaN)")
    return True


class DistD2Rank:
    """Per-rank solver object: plan (coefficient tables on this rank's GPU)
    and the neighbour buffers / mailboxes, reused across solves. Collective:
    every rank of the group constructs it (the pair couplings are shared)."""

    def __init__(self, sys, stencil, part, ctx, arithmetic="fast", warn_not_dominant=True):
        if part.rank_count != ctx.rank_count:
            raise ValueError("partition and rank context disagree on the rank count")
        if part.rank_count < 2:
            raise ValueError("DistD2Rank needs at least two ranks; use run_distd2 for P=1")
        if sys.periodic != ctx.cyclic:
            raise ValueError("rank topology must be a ring exactly when the system is periodic")
        self.ctx = ctx
        self.part = part
        k = ctx.rank_id
        self.m = part.local_sizes[k]
        off = part.offsets()[k]
        local_sys = local_slice(sys, part, k)
        self.coeffs = preprocess(local_sys, rank_position(k, part.rank_count), sys.periodic,
                                 warn_not_dominant=warn_not_dominant)
        prev_sc, next_sa = share_scalars(ctx, self.coeffs.s_a[0], self.coeffs.s_c[-1])
        self.pair_coeffs = (prev_sc, next_sa)
        loc_st = None if stencil is None else stencil.rows(off, off + self.m)
        self.plan = Plan.create_local(local_sys, None if loc_st is None else loc_st.c,
                                      ctx.has_prev, ctx.has_next, prev_sc, next_sa,
                                      _flags(arithmetic),
                                      shift=None if loc_st is None else loc_st.shift)
        self._bufs = {}
        self._mail = {}
        self._epoch = 0
        self.broken = None
        self.fused = (self.plan.path == "fast" and len(set(part.local_sizes)) == 1
                      and os.environ.get("TDS_FUSED", "1") != "0")
        # every rank must launch the same fused-kernel variant (persistent
        # schedules must match): agree on the deferral mask (collective)
        lib = N.lib()
        mask = lib.tds_plan_restrict_fused(self.plan.handle, 3)
        agreed = ctx.allreduce_and(mask if self.fused else 3)
        lib.tds_plan_restrict_fused(self.plan.handle, agreed)

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

    def mailbox(self, groups, sz):
        """Own mailbox + the neighbours' and the agreed persistent grid (one
        collective per field shape)."""
        key = (groups, sz)
        mb = self._mail.get(key)
        if mb is None:
            lib = N.lib()
            mb = self.ctx.open_mailboxes(lib.tds_mailbox_words(groups, sz))
            # every rank runs the same persistent schedule: the smallest grid
            # any rank's kernel variant allows (ranks sharing a device split it)
            mine = lib.tds_fused_grid(self.plan.handle, groups, sz, self.ctx.fused_grid_cap)
            mb.grid = self.ctx.allreduce_min(mine if mine > 0 else 1 << 30)
            self._mail[key] = mb
        return mb

    def fused_eligible(self, groups, sz):
        return bool(self.fused and N.lib().tds_fused_eligible(self.plan.handle, groups, sz))

    def _poll(self, block=False):
        for (groups, sz), mb in self._mail.items():
            try:
                account_status(self.ctx, mb, 2 * groups * sz, groups * sz, block)
            except TimeoutError as exc:
                self.broken = exc
                raise

    def check(self):
        """Wait for the last fused solve's status words and raise TimeoutError
        if a wait timed out (synchronous)."""
        if self.broken is not None:
            raise TimeoutError(str(self.broken))
        self._poll(block=True)

    def close(self):
        for mb in self._mail.values():
            mb.close()
        self._mail = {}

    def solve(self, u, out=None, stream=None):
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
        if self.fused_eligible(groups, sz):
            self.launch_fused(u, out, stream)
            return out
        return self._two_pass(u, out, stream)

    def launch_fused(self, u, out, stream=None):
        """Enqueue one fused solve (k_dd / k_dd2) on `stream` (default: the
        current stream). Raises TimeoutError if an earlier solve timed out."""
        import torch
        if self.broken is not None:
            raise TimeoutError(f"rank {self.ctx.rank_id}: an earlier fused solve timed out; "
                               "the mailboxes are no longer usable")
        self._poll()
        groups, _, sz = u.shape
        mb = self.mailbox(groups, sz)
        s = stream if stream is not None else torch.cuda.current_stream()
        self._epoch += 1
        self.ctx.begin_solve()
        self.ctx.exchange_rounds += 2          # both rounds run inside the kernel
        N.check(N.lib().tds_fused_solve(self.plan.handle, _vp(u), _vp(out), groups, sz, mb.own,
                                        mb.prev, mb.next, self._epoch, mb.grid,
                                        ctypes.c_void_p(s.cuda_stream)))
        mb.post_status(s)

    def _two_pass(self, u, out, stream=None):
        groups, m, sz = u.shape
        b = self._buffers(groups, sz, u.device)
        lib, h, ctx = N.lib(), self.plan.handle, self.ctx
        s = _stream_handle(stream)
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
