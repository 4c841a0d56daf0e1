"""Neighbour transport: the swappable backend of the reference's transport.py
(D15, /root/reference/pkg/src/tds/transport.py:1-230), in two forms.

* `RankContext` -- one PROCESS per rank over torch.distributed (NCCL between
  B200s, gloo on CPU): every rank is a torchrun process.
* `LocalRankContext` + `spawn_ranks` -- several ranks in ONE process, one
  thread per rank, like the reference's spawn_ranks (transport.py:105-139):
  per directed edge a FIFO of device tensors, send/recv with kind and tag
  checks (`TagMismatch`), a receive timeout (`TimeoutError`, RECV_TIMEOUT)
  and per-rank failures aggregated into `RankPanic`. Each rank owns a CUDA
  device (several ranks may share one) and a stream of its own; a message is
  a device-to-device copy (NVLink peer copy between B200s) ordered by a CUDA
  event, never a host round trip.

The protocol is the reference's: ranks form a path (open) or a ring
(cyclic); a solve is exactly two neighbour rounds -- ROUND 1 the depth-2 halo
of the field, ROUND 2 one decoupled row -- each issued in the reference order
(send next, send prev, recv prev, recv next; transport.py:156-169, 181-189),
so a P=2 ring pairs the messages exactly like the reference's FIFO queues.

Both contexts also set up the MAILBOXES of the fused per-rank kernels
(`open_mailboxes`): CUDA IPC handles exchanged over the process group, or
plain device pointers shared between the threads of one process.
"""

import ctypes
import queue
import threading
import time
from dataclasses import dataclass

import numpy as np

from .errors import NoNeighbor, RankPanic, TagMismatch

HALO_LOW = "halo_low"
HALO_HIGH = "halo_high"
BOUNDARY_LOW = "boundary_low"
BOUNDARY_HIGH = "boundary_high"
GATHER = "gather"
SCATTER = "scatter"
_TAGS = {HALO_LOW: 11, HALO_HIGH: 12, BOUNDARY_LOW: 21, BOUNDARY_HIGH: 22, GATHER: 31,
         SCATTER: 32}

RECV_TIMEOUT = 60.0          # transport.py:28


def _dist():
    import torch.distributed as dist
    return dist


def _torch():
    import torch
    return torch


# ------------------------------------------------------------------ mailboxes

class Mailboxes:
    """One rank's mailbox (`words` 8-byte slots on its device) plus its
    neighbours' (mapped), for the fused kernels (tds_fused_solve /
    tds_fused_transport). Keeps an asynchronous copy of the three status
    words (error, halo words posted, boundary words posted; include/
    tds_b200.h) so timeouts and message counts are read without stalling the
    solve stream."""

    def __init__(self, own, prev, nxt, words, release):
        self.own, self.prev, self.next = own, prev, nxt      # ctypes.c_void_p
        self.words = words
        self._release = release
        self._host = None
        self._event = None
        self.counted = [0, 0]    # status counts already added to the context

    def post_status(self, stream):
        """Enqueue the async copy of the status words after a launch."""
        from . import _native as N
        torch = _torch()
        if self._host is None:
            self._host = torch.zeros(3, dtype=torch.int64, pin_memory=True)
            self._event = torch.cuda.Event()
        N.check(N.lib().tds_mailbox_status(self.own, self.words,
                                           ctypes.c_void_p(self._host.data_ptr()),
                                           ctypes.c_void_p(stream.cuda_stream)))
        self._event.record(stream)

    def status(self, block=False):
        """(error, halo_words, boundary_words) of the last completed status
        copy, or None if it has not completed (block=False)."""
        if self._event is None:
            return None
        if block:
            self._event.synchronize()
        elif not self._event.query():
            return None
        e, h, b = (int(x) for x in self._host.tolist())
        return e, h, b

    def close(self):
        if self._release is not None:
            self._release()
            self._release = None


def _ipc_mailboxes(ctx, words):
    """Process-group mailboxes: own allocation + CUDA IPC handles exchanged
    over the group (one collective), neighbours mapped (NVLink peer memory)."""
    from . import _native as N
    dist = _dist()
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

    def release():
        for ptr in opened.values():
            lib.tds_ipc_close(ptr)
        lib.tds_ipc_free(own)

    return Mailboxes(own, prev, nxt, words, release)


# ------------------------------------------------------ process-group ranks

@dataclass
class RankContext:
    """Per-rank view of the topology plus message accounting (transport.py:38-102),
    one process per rank over a torch.distributed group.

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

    @property
    def payload_device(self):
        torch = _torch()
        if _dist().get_backend(self.group) == "nccl":
            return torch.device("cuda", torch.cuda.current_device())
        return torch.device("cpu")

    # one process per device: every rank's persistent grid is the device's
    fused_grid_cap = 0

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

    def open_mailboxes(self, words):
        return _ipc_mailboxes(self, words)

    def barrier(self):
        _dist().barrier(group=self.group)

    def allreduce_and(self, mask, bits=8):
        """Bitwise AND of a small non-negative int over the group."""
        torch = _torch()
        dist = _dist()
        t = torch.tensor([(mask >> b) & 1 for b in range(bits)], dtype=torch.int32,
                         device=self.payload_device)
        dist.all_reduce(t, op=dist.ReduceOp.MIN, group=self.group)
        return sum(int(v) << b for b, v in enumerate(t.tolist()))

    def allreduce_min(self, value):
        """Minimum of an int over the group."""
        torch = _torch()
        dist = _dist()
        t = torch.tensor([int(value)], dtype=torch.int64, device=self.payload_device)
        dist.all_reduce(t, op=dist.ReduceOp.MIN, group=self.group)
        return int(t.item())


# ------------------------------------------------------- in-process ranks

@dataclass(frozen=True)
class NeighborMessage:
    """transport.py:31-35; `ready` orders a device payload's producer before
    its consumer (CUDA event on the sender's stream)."""

    kind: str
    payload: object
    tag: int
    ready: object = None


class _World:
    """State shared by the ranks of one spawn_ranks group."""

    def __init__(self, rank_count, devices):
        self.rank_count = rank_count
        self.devices = devices
        self.barrier = threading.Barrier(rank_count)
        self.failed = threading.Event()
        self.boxes = {}
        per_dev = {}
        for d in devices:
            if d is not None and d.type == "cuda":
                per_dev[d.index] = per_dev.get(d.index, 0) + 1
        # ranks sharing a device split its persistent grid (tds_fused_solve
        # max_ctas = -k); the same value on every rank keeps the schedules equal
        k = max(per_dev.values(), default=1)
        self.grid_cap = -k if k > 1 else 0


def _ship(payload, device):
    """Copy a payload to the receiver's device on the sender's stream; the
    returned event marks its completion."""
    torch = _torch()
    if not isinstance(payload, torch.Tensor):
        payload = torch.from_numpy(np.ascontiguousarray(payload, dtype=np.float64))
    if payload.dtype != torch.float64:                 # float64 payloads, as transport.py:63
        payload = payload.to(torch.float64)
    if device is None or device.type != "cuda":
        return payload.detach().to("cpu", copy=True).contiguous(), None
    buf = torch.empty(tuple(payload.shape), dtype=payload.dtype, device=device)
    buf.copy_(payload, non_blocking=True)
    ev = torch.cuda.Event()
    ev.record(torch.cuda.current_stream(payload.device if payload.is_cuda else device))
    return buf, ev


class LocalRankContext:
    """One rank of an in-process group (reference RankContext,
    transport.py:38-102): FIFO per directed edge, send_prev / send_next /
    recv_prev / recv_next with kind + tag checks, message accounting."""

    def __init__(self, rank_id, rank_count, cyclic, device=None, world=None):
        self.rank_id = rank_id
        self.rank_count = rank_count
        self.cyclic = cyclic
        self.device = device
        self.messages_sent = 0
        self.bytes_sent = 0
        self.exchange_rounds = 0
        self.epoch = 0
        self._world = world if world is not None else _World(rank_count, [device] * rank_count)
        self._from_prev = queue.Queue()
        self._from_next = queue.Queue()
        self._prev = None
        self._next = None
        self._boxes_opened = 0

    @property
    def has_prev(self):
        return self._prev is not None

    @property
    def has_next(self):
        return self._next is not None

    @property
    def payload_device(self):
        torch = _torch()
        return self.device if self.device is not None else torch.device("cpu")

    @property
    def fused_grid_cap(self):
        return self._world.grid_cap

    def begin_solve(self):
        self.epoch += 1
        return self.epoch

    def _send(self, dest, inbox_attr, kind, payload, tag, side):
        if dest is None:
            raise NoNeighbor(f"rank {self.rank_id} has no {side} neighbor")
        buf, ev = _ship(payload, dest.device)
        getattr(dest, inbox_attr).put(NeighborMessage(kind, buf, tag, ev))
        self.messages_sent += 1
        self.bytes_sent += buf.numel() * buf.element_size()

    def send_prev(self, kind, payload, tag):
        self._send(self._prev, "_from_next", kind, payload, tag, "previous")

    def send_next(self, kind, payload, tag):
        self._send(self._next, "_from_prev", kind, payload, tag, "next")

    def _recv(self, inbox, expect_kind, expect_tag, side):
        if (side == "prev" and not self.has_prev) or (side == "next" and not self.has_next):
            raise NoNeighbor(f"rank {self.rank_id} has no {side} neighbor")
        deadline = time.monotonic() + RECV_TIMEOUT
        while True:
            try:
                msg = inbox.get(timeout=0.05)
                break
            except queue.Empty:
                if self._world.failed.is_set() or time.monotonic() > deadline:
                    raise TimeoutError(f"rank {self.rank_id} timed out waiting for "
                                       f"{expect_kind} from {side}") from None
        if msg.kind != expect_kind or (expect_tag is not None and msg.tag != expect_tag):
            raise TagMismatch(f"rank {self.rank_id} expected {expect_kind}/tag {expect_tag}, "
                              f"got {msg.kind}/tag {msg.tag}")
        if msg.ready is not None:
            torch = _torch()
            s = torch.cuda.current_stream(msg.payload.device)
            s.wait_event(msg.ready)
            msg.payload.record_stream(s)
        return msg.payload

    def recv_prev(self, expect_kind, expect_tag=None):
        return self._recv(self._from_prev, expect_kind, expect_tag, "prev")

    def recv_next(self, expect_kind, expect_tag=None):
        return self._recv(self._from_next, expect_kind, expect_tag, "next")

    def round(self, sends, recvs):
        """One neighbour round in the reference order, same interface as
        RankContext.round (received payloads are copied into the given
        buffers)."""
        tag = self.epoch
        for kind, to_next, t in sends:
            (self.send_next if to_next else self.send_prev)(kind, t, tag)
        for kind, from_prev, t in recvs:
            got = (self.recv_prev if from_prev else self.recv_next)(kind, tag)
            if tuple(got.shape) != tuple(t.shape):
                raise ValueError(f"{kind} payload shape {tuple(got.shape)}, expected "
                                 f"{tuple(t.shape)}")
            t.copy_(got)
        self.exchange_rounds += 1

    def barrier(self):
        try:
            self._world.barrier.wait(timeout=RECV_TIMEOUT)
        except threading.BrokenBarrierError:
            raise TimeoutError(f"rank {self.rank_id}: barrier broken (a peer failed)") from None

    def _allreduce(self, value, op):
        self._world.boxes[("reduce", self.rank_id)] = int(value)
        self.barrier()
        res = int(value)
        for r in range(self.rank_count):
            res = op(res, self._world.boxes[("reduce", r)])
        self.barrier()
        return res

    def allreduce_and(self, mask, bits=8):
        """Bitwise AND of a small non-negative int over the group (collective)."""
        return self._allreduce(mask, lambda a, b: a & b)

    def allreduce_min(self, value):
        """Minimum of an int over the group (collective)."""
        return self._allreduce(value, min)

    def open_mailboxes(self, words):
        """Collective over the group (every rank calls it in the same
        order): allocate and prepare this rank's mailbox on its device,
        publish it, map the neighbours' (peer access when on another
        device)."""
        from . import _native as N
        torch = _torch()
        lib = N.lib()
        key = self._boxes_opened
        self._boxes_opened += 1
        own = torch.empty(words, dtype=torch.float64, device=self.device)
        stream = torch.cuda.current_stream(self.device)
        N.check(lib.tds_mailbox_init(ctypes.c_void_p(own.data_ptr()), words,
                                     ctypes.c_void_p(stream.cuda_stream)))
        stream.synchronize()                  # prepared before anyone can post
        self._world.boxes[(key, self.rank_id)] = own
        self.barrier()

        def peer(ctx):
            if ctx is None:
                return ctypes.c_void_p(0)
            if ctx.device.index != self.device.index:
                N.check(lib.tds_peer_access(ctx.device.index))
            return ctypes.c_void_p(self._world.boxes[(key, ctx.rank_id)].data_ptr())

        prev, nxt = peer(self._prev), peer(self._next)
        self.barrier()                        # every rank has mapped its neighbours

        def release():
            self._world.boxes.pop((key, self.rank_id), None)

        mb = Mailboxes(ctypes.c_void_p(own.data_ptr()), prev, nxt, words, release)
        mb.tensor = own
        return mb


def _resolve_devices(devices, rank_count):
    torch = _torch()
    if devices is None:
        return [None] * rank_count
    devices = list(devices)
    if len(devices) != rank_count:
        raise ValueError(f"{len(devices)} devices given for {rank_count} ranks")
    out = []
    for d in devices:
        if d is None:
            out.append(None)
        elif isinstance(d, int):
            out.append(torch.device("cuda", d))
        else:
            d = torch.device(d)
            out.append(torch.device("cuda", d.index if d.index is not None else 0)
                       if d.type == "cuda" else d)
    return out


def make_contexts(rank_count, cyclic, devices=None):
    """The linked contexts of an in-process group (spawn_ranks topology)."""
    if rank_count < 1:
        raise ValueError("rank_count must be positive")
    devs = _resolve_devices(devices, rank_count)
    world = _World(rank_count, devs)
    contexts = [LocalRankContext(r, rank_count, cyclic, devs[r], world)
                for r in range(rank_count)]
    if rank_count > 1:
        for r, ctx in enumerate(contexts):
            if r > 0 or cyclic:
                ctx._prev = contexts[(r - 1) % rank_count]
            if r < rank_count - 1 or cyclic:
                ctx._next = contexts[(r + 1) % rank_count]
    return contexts


def _run_rank(ctx, body):
    """body(ctx) on the rank's device and own stream; its device work is
    complete when this returns."""
    torch = _torch()
    if ctx.device is None or ctx.device.type != "cuda":
        return body(ctx)
    torch.cuda.set_device(ctx.device)
    stream = torch.cuda.Stream(ctx.device)
    with torch.cuda.stream(stream):
        res = body(ctx)
    stream.synchronize()
    return res


def run_on(contexts, body):
    """Run body(ctx) on every context of a group, one thread per rank (a
    single rank runs inline); failures are re-raised together as RankPanic
    (transport.py:120-139)."""
    if len(contexts) == 1:
        return [_run_rank(contexts[0], body)]
    results = [None] * len(contexts)
    failures = {}
    world = contexts[0]._world

    def runner(r):
        try:
            results[r] = _run_rank(contexts[r], body)
        except BaseException as exc:  # noqa: BLE001 - aggregated below
            failures[r] = exc
            world.failed.set()
            world.barrier.abort()

    threads = [threading.Thread(target=runner, args=(r,)) for r in range(len(contexts))]
    for t in threads:
        t.start()
    for t in threads:
        t.join()
    if failures:
        world.failed.clear()
        world.barrier.reset()
        raise RankPanic(failures)
    return results


def spawn_ranks(rank_count, cyclic, body, devices=None):
    """Run `body(ctx)` on every rank; return the per-rank results
    (reference transport.py:105-139). `devices` (optional, one per rank,
    repeats allowed) places each rank on a CUDA device with its own stream."""
    return run_on(make_contexts(rank_count, cyclic, devices), body)


# ------------------------------------------------------------ the two rounds

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
    dev = ctx.payload_device
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
    if isinstance(ctx, LocalRankContext):
        # the reference's neighbour relay (transport.py:194-212)
        if ctx.rank_count == 1:
            return local.clone()
        acc = local.contiguous()
        if ctx.rank_id < ctx.rank_count - 1:
            tail = ctx.recv_next(GATHER, ctx.epoch)
            acc = torch.cat([acc, tail], dim=1)
        if ctx.rank_id > 0:
            ctx.send_prev(GATHER, acc, ctx.epoch)
            return None
        return acc
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
