"""512^3 x solve throughput vs the SZ lane width (the reference's default
layout is sz = 8; the benchmark uses 32): k_tma tile widths follow sz.

    python tools/sz_sweep.py [--n 512]
"""
import argparse
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2411_13532_b200 as T  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--n", type=int, default=512)
    ap.add_argument("--iters", type=int, default=30)
    args = ap.parse_args()
    n = args.n
    s, st = T.assemble(T.sixth_order_first_derivative(2 * np.pi / n), n, periodic=True)
    for sz in (32, 16, 8):
        u = torch.randn((n * n // sz, n, sz), dtype=torch.float64, device="cuda")
        out = torch.empty_like(u)
        for _ in range(3):
            T.run_distd2(s, u, stencil=st, out=out)
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        torch.cuda.synchronize()
        a.record()
        for _ in range(args.iters):
            T.run_distd2(s, u, stencil=st, out=out)
        b.record()
        torch.cuda.synchronize()
        ms = a.elapsed_time(b) / args.iters
        print(f"sz={sz}: {ms:.4f} ms/solve {16 * n ** 3 / (ms * 1e-3) / 1e9:.1f} GB/s", flush=True)
        del u, out
        torch.cuda.empty_cache()


if __name__ == "__main__":
    main()
