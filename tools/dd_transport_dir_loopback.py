"""Single-GPU loopback harness for the distributed z-direction transport
kernel (k_dd_transport_dir): a rank whose prev and next neighbours are its
own mailbox, so the in-kernel rounds go through local HBM (the values are
not a valid RHS; the timing and the ncu profile are). Compared with the
single-GPU z pass (k_transport_dir, P = 1 plans of the slab's z length) on
the same x-layout slab.

    python tools/dd_transport_dir_loopback.py [--n 1024] [--m 512] [--iters 10]
"""
import argparse
import ctypes
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2411_13532_b200 as T  # noqa: E402
from paper_2411_13532_b200 import _native as N  # noqa: E402
from paper_2411_13532_b200 import momentum  # noqa: E402
from paper_2411_13532_b200.distributed import _stream_handle  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--n", type=int, default=1024)
    ap.add_argument("--m", type=int, default=512)
    ap.add_argument("--iters", type=int, default=10)
    ap.add_argument("--nu", type=float, default=0.01)
    args = ap.parse_args()
    n, m, sz, nu = args.n, args.m, 32, args.nu
    P = n // m
    h = 2 * np.pi / n
    part = T.SubdomainPartition.balanced(n, P)
    s1, st1 = momentum._operator(1, h, n)
    s2, st2 = momentum._operator(2, h, n)
    p1 = T.Plan.create(s1, st1.c, part.local_sizes, 1, N.TDS_FLAG_CHUNK16)
    p2 = T.Plan.create(s2, st2.c, part.local_sizes, 1, N.TDS_FLAG_CHUNK16)
    shape = (n * m // sz, n, sz)                  # x-layout z-slab (nx = ny = n, nz = m)
    u = [torch.randn(shape, dtype=torch.float64, device="cuda") for _ in range(3)]
    acc = [torch.zeros(shape, dtype=torch.float64, device="cuda") for _ in range(3)]
    lib = N.lib()
    words = lib.tds_transport_mailbox_words(n * n // sz, sz)
    mail = torch.full((words,), -1, dtype=torch.int64, device="cuda")
    mp = ctypes.c_void_p(mail.data_ptr())
    N.check(lib.tds_mailbox_init(mp, mail.numel(), _stream_handle()))
    vp = lambda t: ctypes.c_void_p(t.data_ptr())  # noqa: E731

    def fused(e):
        N.check(lib.tds_fused_transport_direction(
            p1.handle, p2.handle, vp(u[0]), vp(u[1]), vp(u[2]), vp(acc[0]), vp(acc[1]),
            vp(acc[2]), nu, n, n, m, sz, mp, mp, mp, e, 0, _stream_handle()))

    plans = momentum._direction_plans(h, nu, m)

    def single(e):
        assert momentum._direction_pass(u, acc, (n, n, m), sz, h, nu, 2)

    ev = [torch.cuda.Event(enable_timing=True) for _ in range(2)]
    pts = n * n * m
    runs = [("k_dd_transport_dir loopback", fused)]
    if plans is not None:
        runs.insert(0, ("k_transport_dir z pass (P=1 plans)", single))
    for name, fn in runs:
        for e in range(1, 4):
            fn(e)
        torch.cuda.synchronize()
        ev[0].record()
        for e in range(4, 4 + args.iters):
            fn(e)
        ev[1].record()
        torch.cuda.synchronize()
        ms = ev[0].elapsed_time(ev[1]) / args.iters
        print(f"{name}: n={n} m={m} {ms:.4f} ms {72 * pts / (ms * 1e-3) / 1e9:.1f} GB/s (72 B/pt)",
              flush=True)
    err = ctypes.c_int(0)
    N.check(lib.tds_transport_mailbox_error(mp, n * n // sz, sz, ctypes.byref(err)))
    print("mailbox error:", err.value)


if __name__ == "__main__":
    main()
