"""Momentum-transport RHS evaluation time (BASELINE config 5's per-step
kernel pipeline).

Single GPU (default): evaluate_transport_rhs on an n^3 velocity field.
Multi-GPU (under torchrun): SlabTransport, rank r owning the z-slab
[off_r, off_r + m) of the n^3 box; z contributions run DistD2 along the
rank ring (fused k_dd/k_dd2), x/y contributions are local.
CUDA events, best of `--reps`, max over ranks.

Algorithmic traffic of the default pipeline (k_transport_dir, one launch
per direction) per grid point, fp64:
  x:      read u, v, w + write 3 accumulators                         =  48 B
  y, z:   read u, v, w + read-modify-write 3 accumulators             =  72 B
  total                                                               = 192 B
("logical_gbs_432B" keeps the round-1 figure: the reference-shaped pipeline
of reorders + per-term kernels moves 432 B/pt.)

    python tools/bench_transport.py [--grid 512] [--sz 32] [--nu 0.01]
    python -m torch.distributed.run --nproc-per-node 4 --master-addr 127.0.0.1 \
        --master-port 29533 tools/bench_transport.py --grid 1024
"""
import argparse
import json
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2411_13532_b200 as T  # noqa: E402

BYTES_PER_POINT = 432
ALGO_BYTES_PER_POINT = 192


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--grid", type=int, default=512, help="n of the n^3 box")
    ap.add_argument("--sz", type=int, default=32)
    ap.add_argument("--nu", type=float, default=0.01)
    ap.add_argument("--reps", type=int, default=5)
    ap.add_argument("--slab", action="store_true",
                    help="SlabTransport (z-slab decomposition; implied under torchrun)")
    args = ap.parse_args()
    n = args.grid
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    ctx = None
    if world > 1:
        import torch.distributed as dist
        from paper_2411_13532_b200.transport import RankContext
        local = int(os.environ.get("LOCAL_RANK", rank))
        torch.cuda.set_device(local)
        dist.init_process_group("nccl", device_id=torch.device("cuda", local))
        ctx = RankContext.from_process_group(cyclic=True)
    g = torch.Generator(device="cuda")
    g.manual_seed(5 + rank)
    h = 2 * np.pi / n
    if world > 1 or args.slab:
        tr = T.SlabTransport(n, args.sz, args.nu, h, ctx)
        lay = tr.lay["x"]
        vel = [torch.randn((lay.n_groups, lay.n, lay.sz), dtype=torch.float64, device="cuda",
                           generator=g) for _ in range(3)]

        def step():
            return tr.rhs(*vel)
        pts_local = n * n * tr.m
        what = f"SlabTransport z-slabs m={tr.m}, fused_z_kernel={tr.fused_z}"
    else:
        u3, v3, w3 = (torch.randn((n, n, n), dtype=torch.float64, device="cuda", generator=g)
                      for _ in range(3))
        f = T.VelocityField.from_arrays(u3, v3, w3, args.nu, h, sz=args.sz)
        del u3, v3, w3

        def step():
            return T.evaluate_transport_rhs(f)
        pts_local = n ** 3
        what = "evaluate_transport_rhs"
    step()
    torch.cuda.synchronize()
    ev = [torch.cuda.Event(enable_timing=True) for _ in range(2)]
    best = 1e9
    for _ in range(args.reps):
        if world > 1:
            torch.distributed.barrier()
        torch.cuda.synchronize()
        ev[0].record()
        step()
        ev[1].record()
        torch.cuda.synchronize()
        t = ev[0].elapsed_time(ev[1])
        if world > 1:
            tt = torch.tensor([t], device="cuda")
            torch.distributed.all_reduce(tt, op=torch.distributed.ReduceOp.MAX)
            t = float(tt.item())
        best = min(best, t)
    phases = None
    if world > 1 or args.slab:
        tr.timed(True)
        step()
        torch.cuda.synchronize()
        phases = {k: round(v, 3) for k, v in tr.phase_ms().items()}
        tr.timed(False)
    if world > 1:
        tr.check()
        tr.close()
    if rank == 0:
        pts = n ** 3
        print(json.dumps({"workload": f"transport RHS {n}^3 on {world} GPU(s), sz={args.sz}, "
                                      f"nu={args.nu}: {what}",
                          "ms_per_rhs": round(best, 3),
                          "gdof_per_s": round(pts / (best * 1e-3) / 1e9, 2),
                          "gdof_per_s_per_gpu": round(pts_local / (best * 1e-3) / 1e9, 2),
                          "logical_gbs_432B": round(BYTES_PER_POINT * pts / (best * 1e-3) / 1e9, 1),
                          "algorithmic_gbs_192B": round(
                              ALGO_BYTES_PER_POINT * pts_local / (best * 1e-3) / 1e9, 1),
                          "rank0_phase_ms": phases}),
              flush=True)
    if world > 1:
        torch.distributed.barrier()
        torch.distributed.destroy_process_group()


if __name__ == "__main__":
    main()
