"""Throughput of the reference-order (bit-identical) kernels: run_distd2
with arithmetic="strict" -- k_thomas at P=1, k_staged_decouple +
k_staged_finish at P>1 -- on an SZ-blocked field of ~2^27 points.

    python tools/strict_bench.py [--n 512] [--p 1 8] [--sz 32]
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
    ap.add_argument("--n", type=int, nargs="*", default=[512, 8192])
    ap.add_argument("--p", type=int, nargs="*", default=[1, 8])
    ap.add_argument("--sz", type=int, default=32)
    ap.add_argument("--iters", type=int, default=10)
    args = ap.parse_args()
    for n in args.n:
        s, st = T.assemble(T.sixth_order_first_derivative(2 * np.pi / n), n)
        groups = max(1, (1 << 27) // (n * args.sz))
        u = torch.randn((groups, n, args.sz), dtype=torch.float64, device="cuda")
        out = torch.empty_like(u)
        for p in args.p:
            part = T.SubdomainPartition.balanced(n, p)
            f = lambda: T.run_distd2(s, u, part=part, stencil=st, out=out, arithmetic="strict")  # noqa
            f()
            torch.cuda.synchronize()
            a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            a.record()
            for _ in range(args.iters):
                f()
            b.record()
            torch.cuda.synchronize()
            ms = a.elapsed_time(b) / args.iters
            print(f"strict n={n} P={p}: {ms:.3f} ms, {16 * u.numel() / ms / 1e6:.1f} GB/s (16 B/pt)",
                  flush=True)


if __name__ == "__main__":
    main()
