"""Single-GPU loopback harness for the fused per-rank kernel (k_dd).

A rank whose prev and next neighbours are its own mailbox: the in-kernel
halo and boundary messages go through local HBM instead of NVLink. Used to
time and ncu-profile k_dd on one GPU against k_tma (same block, P=1 plan).

    python tools/dd_loopback.py [--m 512] [--iters 50]
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
from paper_2411_13532_b200.distributed import _stream_handle  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--m", type=int, default=512)
    ap.add_argument("--groups", type=int, default=32768)
    ap.add_argument("--iters", type=int, default=50)
    args = ap.parse_args()
    m, G, sz = args.m, args.groups, 32
    n = 1024
    s, st = T.assemble(T.sixth_order_first_derivative(2 * np.pi / n), n)
    loc = T.local_slice(s, T.SubdomainPartition.balanced(n, n // m), 1)
    co = T.preprocess(loc, "interior", True)
    plan = T.Plan.create_local(loc, st.c[:m], True, True, co.s_c[-1], co.s_a[0])
    lib = N.lib()
    u = torch.randn((G, m, sz), dtype=torch.float64, device="cuda")
    out = torch.empty_like(u)
    words = lib.tds_mailbox_words(G, sz)
    mail = torch.full((words,), -1, dtype=torch.int64, device="cuda")   # 0xFF.. sentinel
    mp = ctypes.c_void_p(mail.data_ptr())
    N.check(lib.tds_mailbox_init(mp, mail.numel(), _stream_handle()))
    vp = lambda t: ctypes.c_void_p(t.data_ptr())  # noqa: E731
    ev = [torch.cuda.Event(enable_timing=True) for _ in range(2)]

    grid = lib.tds_fused_grid(plan.handle, G, sz, 0)    # this plan's own kernel variant

    def fused(epoch):
        N.check(lib.tds_fused_solve(plan.handle, vp(u), vp(out), G, sz, mp, mp, mp, epoch,
                                    grid, _stream_handle()))

    p1 = T.get_plan(T.TridiagonalSystem(loc.lower, loc.diag, loc.upper, periodic=True),
                    T.StencilCoeffs(st.c[:m]), T.SubdomainPartition((m,)))

    def single():
        N.check(lib.tds_solve(p1.handle, vp(u), vp(out), G, sz, _stream_handle()))

    for name, fn in (("k_tma (P=1 plan)", lambda e: single()), ("k_dd loopback", fused)):
        for e in range(1, 4):
            fn(e)
        torch.cuda.synchronize()
        ev[0].record()
        for e in range(4, 4 + args.iters):
            fn(e)
        ev[1].record()
        torch.cuda.synchronize()
        ms = ev[0].elapsed_time(ev[1]) / args.iters
        gbs = 16 * G * m * sz / (ms * 1e-3) / 1e9
        print(f"{name}: m={m} {ms:.4f} ms/solve {gbs:.1f} GB/s", flush=True)
    err = ctypes.c_int(0)
    N.check(lib.tds_mailbox_error(mp, G, sz, ctypes.byref(err)))
    print("mailbox error:", err.value)


if __name__ == "__main__":
    main()
