"""torchrun worker: one rank per GPU, DistD2 decomposed along the solve
direction, results gathered to rank 0 and compared with the pinned oracle's
run_distd2 on the same partition (the reference's truncation boundaries).

    python -m torch.distributed.run --nproc-per-node 2 --master-addr 127.0.0.1 \
        --master-port 29533 tests/mgpu_worker.py
"""

import os
import sys
import warnings

import numpy as np
import torch
import torch.distributed as dist

HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, os.path.dirname(HERE))

import paper_2411_13532_b200 as T  # noqa: E402
from oracle import tds_oracle as O  # noqa: E402
from paper_2411_13532_b200.transport import RankContext, gather_to_root, share_scalars  # noqa


def main():
    rank = int(os.environ["RANK"])
    world = int(os.environ["WORLD_SIZE"])
    local = int(os.environ.get("LOCAL_RANK", rank))
    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    dist.init_process_group("nccl", device_id=dev)
    warnings.simplefilter("ignore", T.NotDominantWarning)
    failures = []

    def case(name, lo, di, up, periodic, st, n, sz=32, groups=4, arith="fast", seed=0):
        rng = np.random.default_rng(seed)
        field = rng.standard_normal((groups, n, sz))
        s = T.TridiagonalSystem(lo, di, up, periodic=periodic)
        stc = T.StencilCoeffs(st)
        part = T.SubdomainPartition.balanced(n, world)
        ctx = RankContext.from_process_group(cyclic=periodic)
        off, m = part.offsets()[rank], part.local_sizes[rank]
        u = torch.from_numpy(np.ascontiguousarray(field[:, off:off + m, :])).to(dev)
        solver = T.DistD2Rank(s, stc, part, ctx, arithmetic=arith)
        out = solver.solve(u)
        out2 = solver.solve(u)            # buffers / mailboxes reused, same bits
        torch.cuda.synchronize()
        solver.check()
        same = bool(torch.equal(out, out2))
        full = gather_to_root(ctx, out)
        # reference-shaped per-rank path: preprocess + one-time share + 2 rounds
        local_sys = T.local_slice(s, part, rank)
        co = T.preprocess(local_sys, T.rank_position(rank, world), periodic)
        psc, nsa = share_scalars(ctx, co.s_a[0], co.s_c[-1])
        ref_shaped = T.distd2_solve(ctx, u, co, T.StencilCoeffs(st[off:off + m]),
                                    T.PairCoeffs(psc, nsa))
        full_rs = gather_to_root(ctx, ref_shaped)
        if rank == 0:
            want = O.run_distd2(lo, di, up, periodic, field, st, part.local_sizes)
            got = full.cpu().numpy()
            err = O.rel_linf(got, want)
            exact = np.array_equal(got, want)
            rs_exact = np.array_equal(full_rs.cpu().numpy(), want)
            ok = same and rs_exact and ((exact) if arith == "strict" else (err <= 1e-12))
            print(f"[{name}] P={world} path={solver.path} fused={solver.fused} "
                  f"rel={err:.3e} bitwise={exact} "
                  f"reference_shaped_bitwise={rs_exact} repeat_same={same} "
                  f"{'OK' if ok else 'FAIL'}", flush=True)
            if not ok:
                failures.append(name)

    for n in (1024, 512):
        lo, di, up, st = O.assemble("d1", n, 2 * np.pi / n, True)
        case(f"d1 periodic n={n}", lo, di, up, True, st, n, seed=n)
        lo, di, up, st = O.assemble("d1", n, 2 * np.pi / n, False)
        case(f"d1 open n={n}", lo, di, up, False, st, n, seed=n + 1)
    lo, di, up, st = O.assemble("d2", 256 * world, 0.01, True)
    case("d2 periodic", lo, di, up, True, st, 256 * world, seed=3)
    r = np.random.default_rng(9)
    n = 50 * world + 3
    lo, di, up = 0.3 * (2 * r.random(n) - 1), 2 + r.random(n), 0.3 * (2 * r.random(n) - 1)
    st = r.standard_normal((n, 5))
    case("random dominant, ragged partition (staged path)", lo, di, up, True, st, n, sz=8,
         groups=3, seed=4)
    lo, di, up, st = O.assemble("d1", 1024, 2 * np.pi / 1024, True)
    case("d1 periodic strict", lo, di, up, True, st, 1024, arith="strict", seed=5)

    # config 5: transport RHS on a z-slab decomposition (SlabTransport)
    for nu, sz in ((0.02, 16), (0.0, 16), (0.01, 32), (0.01, 8)):
        n = 128
        rng = np.random.default_rng(77)
        u3, v3, w3 = (rng.standard_normal((n, n, n)) for _ in range(3))
        ctx = RankContext.from_process_group(cyclic=True)
        tr = T.SlabTransport(n, sz, nu, 2 * np.pi / n, ctx)
        loc = [tr.local_slab(a) for a in (u3, v3, w3)]
        rhs = tr.rhs(*loc)
        rhs2 = tr.rhs(*loc)
        torch.cuda.synchronize()
        tr.check()
        same = all(bool(torch.equal(a, b)) for a, b in zip(rhs, rhs2))
        fulls = []
        for comp in rhs:
            cart = T.unpack(T.GroupedField(tr.lay["x"], comp))          # (n, n, m)
            g = gather_to_root(ctx, cart.permute(2, 0, 1).unsqueeze(0).contiguous())
            fulls.append(None if g is None else g[0].permute(1, 2, 0).cpu().numpy())
        tr.close()
        if rank == 0:
            want = O.transport_rhs(u3, v3, w3, nu, 2 * np.pi / n, sz, rank_counts=(1, 1, world))
            errs = [O.rel_linf(g, w) for g, w in zip(fulls, want)]
            ref_p = O.transport_rhs(u3, v3, w3, nu, 2 * np.pi / n, sz,
                                    rank_counts=(world, world, world))
            errs_p = [O.rel_linf(g, w) for g, w in zip(fulls, ref_p)]
            ok = same and max(errs) <= 1e-12 and max(errs_p) <= 1e-12 and tr.fused_z
            print(f"[transport slab nu={nu} sz={sz}] P={world} m={tr.m} fused_z={tr.fused_z} "
                  f"rel(1,1,P)={max(errs):.3e} rel(P,P,P)={max(errs_p):.3e} repeat_same={same} "
                  f"{'OK' if ok else 'FAIL'}", flush=True)
            if not ok:
                failures.append(f"transport nu={nu}")
    dist.barrier()
    dist.destroy_process_group()
    if rank == 0:
        print("MGPU", "FAIL " + ",".join(failures) if failures else "ALL OK", flush=True)
        sys.exit(1 if failures else 0)


if __name__ == "__main__":
    main()
