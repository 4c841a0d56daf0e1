"""Single-GPU solve throughput vs line length n (P=1 periodic d/dx, sz=32,
~2^27 points per field, x solve repeated), for the A/B knobs given as
KEY=VAL arguments. Prints one line per n: path, chunk rows, ms, GB/s at the
16 B/pt algorithmic traffic.

    python tools/sweep_n.py [n ...] [--iters K] [KEY=VAL ...]
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
    ap.add_argument("n", nargs="*", type=int, default=[256, 512, 1024, 2048, 4096, 8192])
    ap.add_argument("--iters", type=int, default=50)
    ap.add_argument("--points", type=float, default=2 ** 27)
    ap.add_argument("--op", default="d1")
    ap.add_argument("--open", action="store_true")
    kvs = [a for a in sys.argv[1:] if "=" in a and not a.startswith("-")]
    args = ap.parse_args([a for a in sys.argv[1:] if a not in kvs])
    for kv in kvs:
        k, v = kv.split("=", 1)
        os.environ[k] = v
    for n in args.n:
        scheme = (T.sixth_order_first_derivative if args.op == "d1"
                  else T.second_derivative_scheme)(2 * np.pi / n)
        s, st = T.assemble(scheme, n, periodic=not args.open,
                           closure="one-sided" if args.open and args.op == "d2" else None)
        groups = max(1, int(args.points) // (n * 32))
        u = torch.randn((groups, n, 32), dtype=torch.float64, device="cuda")
        out = torch.empty_like(u)
        part = T.SubdomainPartition((n,))
        plan = T.get_plan(s, st, part)
        for _ in range(3):
            T.run_distd2(s, u, part=part, stencil=st, out=out)
        torch.cuda.synchronize()
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record()
        for _ in range(args.iters):
            T.run_distd2(s, u, part=part, stencil=st, out=out)
        b.record()
        torch.cuda.synchronize()
        ms = a.elapsed_time(b) / args.iters
        gbs = 16 * u.numel() / (ms * 1e-3) / 1e9
        print(f"n={n} path={plan.path} M={plan.info.chunk_rows} C={plan.info.chunks} "
              f"{ms:.4f} ms {gbs:.1f} GB/s", flush=True)
        del u, out


if __name__ == "__main__":
    main()
