"""In-process ranks (transport.LocalRankContext / spawn_ranks) on CPU
tensors: the reference's transport contract (transport.py:38-139 --
send/recv with kind and tag checks, NoNeighbor, TimeoutError, RankPanic,
FIFO per directed edge) and the two solver rounds / gather relay it
carries (transport.py:142-212). The GPU ranks are tests/test_gpu_multirank.py."""

import numpy as np
import pytest

torch = pytest.importorskip("torch")

from paper_2411_13532_b200 import transport as TR  # noqa: E402
from paper_2411_13532_b200.errors import NoNeighbor, RankPanic, TagMismatch  # noqa: E402


def test_topology_path_and_ring():
    def body(ctx):
        return ctx.has_prev, ctx.has_next
    assert TR.spawn_ranks(3, False, body) == [(False, True), (True, True), (True, False)]
    assert TR.spawn_ranks(3, True, body) == [(True, True)] * 3
    assert TR.spawn_ranks(1, True, body) == [(False, False)]


def test_fifo_kind_tag_and_accounting():
    def body(ctx):
        if ctx.rank_id == 0:
            ctx.send_next(TR.HALO_LOW, torch.arange(4.0), 1)
            ctx.send_next(TR.BOUNDARY_LOW, torch.ones(2), 1)
            return ctx.messages_sent, ctx.bytes_sent
        a = ctx.recv_prev(TR.HALO_LOW, 1)
        b = ctx.recv_prev(TR.BOUNDARY_LOW)
        return a.tolist(), b.tolist()
    res = TR.spawn_ranks(2, False, body)
    assert res[0] == (2, 48)
    assert res[1] == ([0.0, 1.0, 2.0, 3.0], [1.0, 1.0])


def test_tag_mismatch_and_no_neighbor_raise_rank_panic():
    def body(ctx):
        if ctx.rank_id == 0:
            ctx.send_next(TR.HALO_LOW, torch.zeros(1), 7)
            return None
        return ctx.recv_prev(TR.HALO_LOW, 8)
    with pytest.raises(RankPanic) as ei:
        TR.spawn_ranks(2, False, body)
    assert isinstance(ei.value.failures[1], TagMismatch)

    def lonely(ctx):
        ctx.send_prev(TR.HALO_HIGH, torch.zeros(1), 0)
    with pytest.raises(RankPanic) as ei:
        TR.spawn_ranks(2, False, lonely)
    assert isinstance(ei.value.failures[0], NoNeighbor)


def test_recv_timeout(monkeypatch):
    monkeypatch.setattr(TR, "RECV_TIMEOUT", 0.2)

    def body(ctx):
        if ctx.rank_id == 1:
            ctx.recv_prev(TR.HALO_LOW)
    with pytest.raises(RankPanic) as ei:
        TR.spawn_ranks(2, False, body)
    assert isinstance(ei.value.failures[1], TimeoutError)


def test_failed_peer_unblocks_receivers():
    def body(ctx):
        if ctx.rank_id == 0:
            raise RuntimeError("boom")
        ctx.recv_prev(TR.HALO_LOW)
    with pytest.raises(RankPanic) as ei:
        TR.spawn_ranks(3, False, body)
    assert isinstance(ei.value.failures[0], RuntimeError)
    assert isinstance(ei.value.failures[1], TimeoutError)     # early, not after 60 s


@pytest.mark.parametrize("cyclic", [False, True])
@pytest.mark.parametrize("p", [2, 3, 5])
def test_rounds_match_reference_semantics(p, cyclic):
    groups, m, sz = 3, 6, 4
    rng = np.random.default_rng(p)
    blocks = [torch.from_numpy(rng.standard_normal((groups, m, sz))) for _ in range(p)]

    def body(ctx):
        ctx.begin_solve()
        low, high = TR.exchange_halo(ctx, blocks[ctx.rank_id], 2)
        pl, nf = TR.exchange_boundary(ctx, blocks[ctx.rank_id][:, 0, :],
                                      blocks[ctx.rank_id][:, -1, :])
        return low, high, pl, nf, ctx.exchange_rounds, ctx.messages_sent

    res = TR.spawn_ranks(p, cyclic, body)
    for k, (low, high, pl, nf, rounds, msgs) in enumerate(res):
        prev, nxt = (k - 1) % p, (k + 1) % p
        has_prev, has_next = cyclic or k > 0, cyclic or k < p - 1
        assert rounds == 2
        assert msgs == 2 * (int(has_prev) + int(has_next))
        if has_prev:
            assert torch.equal(low, blocks[prev][:, m - 2:, :])
            assert torch.equal(pl, blocks[prev][:, -1, :])
        else:
            assert low is None and pl is None
        if has_next:
            assert torch.equal(high, blocks[nxt][:, :2, :])
            assert torch.equal(nf, blocks[nxt][:, 0, :])
        else:
            assert high is None and nf is None


def test_share_scalars_and_gather_relay():
    p = 4

    def body(ctx):
        psc, nsa = TR.share_scalars(ctx, 10.0 + ctx.rank_id, 20.0 + ctx.rank_id)
        full = TR.gather_to_root(ctx, torch.full((1, 2 + ctx.rank_id, 1), float(ctx.rank_id)))
        return psc, nsa, ctx.exchange_rounds, full

    res = TR.spawn_ranks(p, True, body)
    for k, (psc, nsa, rounds, full) in enumerate(res):
        assert psc == 20.0 + (k - 1) % p and nsa == 10.0 + (k + 1) % p
        assert rounds == 0               # the one-time share is not a solve round
        if k == 0:
            want = np.concatenate([np.full(2 + r, float(r)) for r in range(p)])
            assert np.array_equal(full.reshape(-1).numpy(), want)
        else:
            assert full is None


def test_grid_cap_of_shared_devices():
    assert TR.make_contexts(4, True, [0, 0, 1, 1])[0].fused_grid_cap == -2
    assert TR.make_contexts(3, True, [0, 0, 0])[2].fused_grid_cap == -3
    assert TR.make_contexts(2, True, [0, 1])[0].fused_grid_cap == 0
    with pytest.raises(ValueError):
        TR.make_contexts(2, True, [0])


def test_allreduce_and_agrees_on_masks():
    masks = [3, 1, 3, 3]
    assert TR.spawn_ranks(4, True, lambda ctx: ctx.allreduce_and(masks[ctx.rank_id])) == [1] * 4
    assert TR.spawn_ranks(2, False, lambda ctx: [ctx.allreduce_and(2 + ctx.rank_id),
                                                 ctx.allreduce_and(3)]) == [[2, 3]] * 2
