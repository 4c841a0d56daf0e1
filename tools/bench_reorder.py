"""Bandwidth of the layout kernels (pack / unpack / reorder) on an n^3 fp64
field: 16 B per point moved (one read + one write), CUDA events, best of 10.

    python tools/bench_reorder.py [--n 512] [--sz 32]
"""
import argparse
import json
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2411_13532_b200 as T  # noqa: E402


def timed(fn, reps=10):
    ev = [torch.cuda.Event(enable_timing=True) for _ in range(2)]
    best = 1e9
    fn()
    for _ in range(reps):
        torch.cuda.synchronize()
        ev[0].record()
        fn()
        ev[1].record()
        torch.cuda.synchronize()
        best = min(best, ev[0].elapsed_time(ev[1]))
    return best


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--n", type=int, default=512)
    ap.add_argument("--sz", type=int, default=32)
    args = ap.parse_args()
    n, sz = args.n, args.sz
    cart = torch.randn((n, n, n), dtype=torch.float64, device="cuda")
    gb = 16 * n ** 3 / 1e9
    res = {}
    for d in "xyz":
        lay = T.LayoutDescriptor(n, n, n, sz, d)
        f = T.pack(cart, lay)
        res[f"pack_{d}"] = gb / (timed(lambda: T.pack(cart, lay)) * 1e-3)
        res[f"unpack_{d}"] = gb / (timed(lambda: T.unpack(f)) * 1e-3)
    from paper_2411_13532_b200 import momentum
    fx = T.pack(cart, T.LayoutDescriptor(n, n, n, sz, "x")).data
    fy = torch.empty_like(fx)
    for a, b in (("x", "y"), ("x", "z"), ("y", "x"), ("z", "x")):
        res[f"reorder_{a}{b}"] = gb / (timed(lambda: momentum._reorder_tensor(fx, n, sz, a, b, out=fy)) * 1e-3)
        res[f"reorder_acc_{a}{b}"] = 1.5 * gb / (timed(
            lambda: momentum._reorder_tensor(fx, n, sz, a, b, out=fy, accumulate=True)) * 1e-3)
    copy = torch.empty_like(cart)
    res["torch_copy"] = gb / (timed(lambda: copy.copy_(cart)) * 1e-3)
    print(json.dumps({k: round(v, 1) for k, v in res.items()}))


if __name__ == "__main__":
    main()
