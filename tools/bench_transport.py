"""Momentum-transport RHS evaluation time on one GPU (BASELINE config 5's
per-step kernel pipeline, single device): evaluate_transport_rhs on an n^3
velocity field, CUDA events, best of 5.

Logical traffic of the pipeline per grid point (fp64, 8 B per access):
  x:      3 contributions, fused (diagonal 16 B, off-diagonal 24 B)  =  64 B
  y, z:   3 one-pass input reorders (16 B each)                       =  48 B
          3 contributions into scratch                                =  64 B
          3 reorder-accumulates into x (24 B each)                    =  72 B
  total   64 + 2 * 184                                                = 432 B

    python tools/bench_transport.py [--n 512] [--sz 32] [--nu 0.01]
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


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--n", type=int, default=512)
    ap.add_argument("--sz", type=int, default=32)
    ap.add_argument("--nu", type=float, default=0.01)
    args = ap.parse_args()
    n = args.n
    g = torch.Generator(device="cuda")
    g.manual_seed(5)
    u3, v3, w3 = (torch.randn((n, n, n), dtype=torch.float64, device="cuda", generator=g)
                  for _ in range(3))
    f = T.VelocityField.from_arrays(u3, v3, w3, args.nu, 2 * np.pi / n, sz=args.sz)
    del u3, v3, w3
    T.evaluate_transport_rhs(f)
    ev = [torch.cuda.Event(enable_timing=True) for _ in range(2)]
    best = 1e9
    for _ in range(5):
        torch.cuda.synchronize()
        ev[0].record()
        T.evaluate_transport_rhs(f)
        ev[1].record()
        torch.cuda.synchronize()
        best = min(best, ev[0].elapsed_time(ev[1]))
    pts = n ** 3
    print(json.dumps({"workload": f"transport RHS {n}^3, sz={args.sz}, nu={args.nu}",
                      "ms_per_rhs": round(best, 3),
                      "gdof_per_s": round(pts / (best * 1e-3) / 1e9, 2),
                      "logical_gbs": round(BYTES_PER_POINT * pts / (best * 1e-3) / 1e9, 1),
                      "bytes_per_point": BYTES_PER_POINT}))


if __name__ == "__main__":
    main()
