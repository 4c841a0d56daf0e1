"""Neighbour transport over torch.distributed (NCCL on B200s, gloo on CPU):
the swappable backend of the reference's transport.py (D15,
/root/reference/pkg/src/tds/transport.py:1-230), one process per rank.

The protocol is the reference's: ranks form a path (open) or a ring
(cyclic); a solve is exactly two neighbour rounds -- ROUND 1 the depth-2 halo
of the field, ROUND 2 one decoupled row -- each a single batched group of
point-to-point sends/receives issued in the reference order (send next, send
prev, recv prev, recv next; transport.py:156-169, 181-189), so a P=2 ring
pairs the messages exactly like the reference's FIFO queues.
"""

from dataclasses import dataclass

import numpy as np

from .errors import NoNeighbor

HALO_LOW = "halo_low"
HALO_HIGH = "halo_high"
BOUNDARY_LOW = "boundary_low"
BOUNDARY_HIGH = "boundary_high"
_TAGS = {HALO_LOW: 11, HALO_HIGH: 12, BOUNDARY_LOW: 21, BOUNDARY_HIGH: 22}


def _dist():
    import torch.distributed as dist
    return dist


@dataclass
class RankContext:
    """Per-rank view of the topology plus message accounting (transport.py:38-102).

    rank_id / rank_count are positions in the DistD2 chain; `ranks` maps a
    chain position to the process-group rank (default: identity)."""

    rank_id: int
    rank_count: int
    cyclic: bool
    group: object = None
    ranks: tuple = None
    messages_sent: int = 0
    bytes_sent: int = 0
    exchange_rounds: int = 0
    epoch: int = 0

    @classmethod
    def from_process_group(cls, cyclic, group=None):
        dist = _dist()
        return cls(dist.get_rank(group), dist.get_world_size(group), cyclic, group)

    def _global(self, pos):
        pos %= self.rank_count
        return pos if self.ranks is None else self.ranks[pos]

    @property
    def has_prev(self):
        return self.rank_count > 1 and (self.rank_id > 0 or self.cyclic)

    @property
    def has_next(self):
        return self.rank_count > 1 and (self.rank_id < self.rank_count - 1 or self.cyclic)

    @property
    def prev(self):
        if not self.has_prev:
            raise NoNeighbor(f"rank {self.rank_id} has no previous neighbor")
        return self._global(self.rank_id - 1)

    @property
    def next(self):
        if not self.has_next:
            raise NoNeighbor(f"rank {self.rank_id} has no next neighbor")
        return self._global(self.rank_id + 1)

    def begin_solve(self):
        self.epoch += 1
        return self.epoch

    def round(self, sends, recvs):
        """One neighbour round: sends = [(kind, to_next?, tensor)], recvs =
        [(kind, from_prev?, tensor)], issued as one batched P2P group."""
        dist = _dist()
        ops = []
        for kind, to_next, t in sends:
            peer = self.next if to_next else self.prev
            ops.append(dist.P2POp(dist.isend, t, peer, self.group, _TAGS[kind]))
            self.messages_sent += 1
            self.bytes_sent += t.numel() * t.element_size()
        for kind, from_prev, t in recvs:
            peer = self.prev if from_prev else self.next
            ops.append(dist.P2POp(dist.irecv, t, peer, self.group, _TAGS[kind]))
        if ops:
            for req in dist.batch_isend_irecv(ops):
                req.wait()
        self.exchange_rounds += 1


def exchange_halo(ctx, local, depth):
    """ROUND 1 (transport.py:142-171): send the last `depth` positions to next
    and the first to prev; return (low, high) = prev's last / next's first
    positions, None on open edges. `local` is (n_groups, n_loc, sz)."""
    import torch
    if depth == 0:
        return None, None
    n_loc = local.shape[1]
    if depth > n_loc:
        raise ValueError(f"halo depth {depth} exceeds local size {n_loc}")
    shape = (local.shape[0], depth, local.shape[2])
    sends, recvs = [], []
    low = high = None
    if ctx.has_next:
        sends.append((HALO_LOW, True, local[:, n_loc - depth:, :].contiguous()))
    if ctx.has_prev:
        sends.append((HALO_HIGH, False, local[:, :depth, :].contiguous()))
    if ctx.has_prev:
        low = torch.empty(shape, dtype=local.dtype, device=local.device)
        recvs.append((HALO_LOW, True, low))
    if ctx.has_next:
        high = torch.empty(shape, dtype=local.dtype, device=local.device)
        recvs.append((HALO_HIGH, False, high))
    ctx.round(sends, recvs)
    return low, high


def exchange_boundary(ctx, first_row, last_row):
    """ROUND 2 (transport.py:174-191): first row to prev, last row to next;
    returns (prev_last, next_first), None on open edges."""
    import torch
    sends, recvs = [], []
    prev_last = next_first = None
    if ctx.has_next:
        sends.append((BOUNDARY_LOW, True, last_row.contiguous()))
    if ctx.has_prev:
        sends.append((BOUNDARY_HIGH, False, first_row.contiguous()))
    if ctx.has_prev:
        prev_last = torch.empty_like(last_row)
        recvs.append((BOUNDARY_LOW, True, prev_last))
    if ctx.has_next:
        next_first = torch.empty_like(first_row)
        recvs.append((BOUNDARY_HIGH, False, next_first))
    ctx.round(sends, recvs)
    return prev_last, next_first


def share_scalars(ctx, first_value, last_value):
    """One-time scalar round (share_pair_coeffs, distributed.py:308-324): send
    s_a[0] to prev and s_c[-1] to next; returns (prev's s_c[-1], next's s_a[0])."""
    import torch
    dev = "cuda" if _dist().get_backend(ctx.group) == "nccl" else "cpu"
    first = torch.tensor([float(first_value)], dtype=torch.float64, device=dev)
    last = torch.tensor([float(last_value)], dtype=torch.float64, device=dev)
    prev_sc, next_sa = exchange_boundary(ctx, first, last)
    ctx.exchange_rounds -= 1   # the one-time share is not a solve round
    return (None if prev_sc is None else float(prev_sc.item()),
            None if next_sa is None else float(next_sa.item()))


def gather_to_root(ctx, local):
    """Test-only collective (transport.py:194-212): concatenate position slices
    at chain position 0; returns the full array there and None elsewhere."""
    import torch
    dist = _dist()
    sizes = [None] * ctx.rank_count
    dist.all_gather_object(sizes, tuple(local.shape), group=ctx.group)
    if ctx.rank_id == 0:
        parts = [local.contiguous()]
        for k in range(1, ctx.rank_count):
            buf = torch.empty(sizes[k], dtype=local.dtype, device=local.device)
            dist.recv(buf, ctx._global(k), group=ctx.group)
            parts.append(buf)
        return torch.cat(parts, dim=1)
    dist.send(local.contiguous(), ctx._global(0), group=ctx.group)
    return None


def balanced_rows(n, rank_count, rank_id):
    """Row range of `rank_id` under SubdomainPartition.balanced (system.py:148-155)."""
    base, extra = divmod(n, rank_count)
    sizes = [base + (1 if k < extra else 0) for k in range(rank_count)]
    off = int(np.sum(sizes[:rank_id]))
    return off, sizes[rank_id]
