"""Multi-process transport on CPU (gloo, world sizes 2 and 3): the neighbour
rounds deliver exactly what the reference's queues deliver
(reference tests/test_transport.py), on paths and rings, with the
reference's message accounting."""

import os
import socket

import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _worker(rank, world, cyclic, port, q):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        from paper_2411_13532_b200.transport import (RankContext, exchange_boundary,
                                                     exchange_halo, gather_to_root,
                                                     share_scalars)
        ctx = RankContext.from_process_group(cyclic)
        g, m, sz = 3, 6, 4
        local = (torch.arange(g * m * sz, dtype=torch.float64).reshape(g, m, sz)
                 + 1000.0 * rank)
        ctx.begin_solve()
        low, high = exchange_halo(ctx, local, 2)
        first, last = local[:, 0, :].clone(), local[:, m - 1, :].clone()
        prev_last, next_first = exchange_boundary(ctx, first, last)
        sc, sa = share_scalars(ctx, 10.0 + rank, 20.0 + rank)
        full = gather_to_root(ctx, local)
        agreed = ctx.allreduce_and(3 if rank else 1)        # fused-variant agreement
        q.put((rank, agreed, None if low is None else low.numpy(), None if high is None else high.numpy(),
               None if prev_last is None else prev_last.numpy(),
               None if next_first is None else next_first.numpy(), sc, sa,
               ctx.exchange_rounds, ctx.messages_sent,
               None if full is None else full.numpy()))
    finally:
        dist.destroy_process_group()


def _run(world, cyclic):
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, cyclic, port, q)) for r in range(world)]
    for p in procs:
        p.start()
    res = {}
    for _ in range(world):
        item = q.get(timeout=120)
        assert item[1] == 1
        res[item[0]] = item[2:]
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    return res


def _local(rank):
    import numpy as np
    return np.arange(3 * 6 * 4, dtype=np.float64).reshape(3, 6, 4) + 1000.0 * rank


@pytest.mark.parametrize("world,cyclic", [(2, False), (2, True), (3, True), (3, False)])
def test_halo_and_boundary_rounds(world, cyclic):
    import numpy as np
    res = _run(world, cyclic)
    for r in range(world):
        low, high, prev_last, next_first, sc, sa, rounds, msgs, full = res[r]
        has_prev = r > 0 or cyclic
        has_next = r < world - 1 or cyclic
        p, n = (r - 1) % world, (r + 1) % world
        if has_prev:
            np.testing.assert_array_equal(low, _local(p)[:, 4:, :])
            np.testing.assert_array_equal(prev_last, _local(p)[:, 5, :])
            assert sc == 20.0 + p
        else:
            assert low is None and prev_last is None and sc is None
        if has_next:
            np.testing.assert_array_equal(high, _local(n)[:, :2, :])
            np.testing.assert_array_equal(next_first, _local(n)[:, 0, :])
            assert sa == 10.0 + n
        else:
            assert high is None and next_first is None and sa is None
        # two solve rounds; per round one message per existing neighbour, plus
        # the one-time scalar share (reference test_distributed.py:263-286)
        assert rounds == 2
        assert msgs == 3 * (int(has_prev) + int(has_next))
        if r == 0:
            np.testing.assert_array_equal(full, np.concatenate([_local(k) for k in range(world)],
                                                               axis=1))
