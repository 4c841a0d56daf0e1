"""Mailbox wait profile of the fused per-rank kernels over NVLink (debug
build: TDS_NVCC_EXTRA=-DTDS_WAIT_PROF python -m paper_2411_13532_b200.build):
per rank, ns spent polling halo / boundary-row slots per take, over K solves.

    torchrun --nproc-per-node 4 tools/wait_prof.py [--grid 512] [--iters 100]
"""
import argparse
import ctypes
import os
import sys

import numpy as np
import torch
import torch.distributed as dist

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2411_13532_b200 as T  # noqa: E402
from paper_2411_13532_b200 import _native as N  # noqa: E402
from paper_2411_13532_b200.transport import RankContext  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--grid", type=int, default=512)
    ap.add_argument("--iters", type=int, default=100)
    args = ap.parse_args()
    rank, world = int(os.environ["RANK"]), int(os.environ["WORLD_SIZE"])
    local = int(os.environ.get("LOCAL_RANK", rank))
    torch.cuda.set_device(local)
    dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    n = args.grid
    s, st = T.assemble(T.sixth_order_first_derivative(2 * np.pi / n), n)
    part = T.SubdomainPartition.balanced(n, world)
    ctx = RankContext.from_process_group(cyclic=True)
    solver = T.DistD2Rank(s, st, part, ctx)
    m = part.local_sizes[rank]
    u = torch.randn((n * n // 32, m, 32), dtype=torch.float64, device="cuda")
    out = torch.empty_like(u)
    f = N.lib().tds_debug_wait_stats
    f.argtypes = [ctypes.POINTER(ctypes.c_ulonglong)]
    buf = (ctypes.c_ulonglong * 4)()
    for _ in range(5):
        solver.solve(u, out)
    f(buf)
    dist.barrier()
    ev = [torch.cuda.Event(enable_timing=True) for _ in range(2)]
    ev[0].record()
    for _ in range(args.iters):
        solver.solve(u, out)
    ev[1].record()
    f(buf)
    ms = ev[0].elapsed_time(ev[1]) / args.iters
    hn, bn, hk, bk = list(buf)
    print(f"rank {rank}: m={m} {ms:.4f} ms/solve; halo wait {hn / max(hk, 1):.0f} ns/take "
          f"({hk} takes), boundary wait {bn / max(bk, 1):.0f} ns/take ({bk} takes)", flush=True)
    solver.check()
    solver.close()
    dist.destroy_process_group()


if __name__ == "__main__":
    main()
