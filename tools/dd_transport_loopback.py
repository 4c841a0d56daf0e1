"""Single-GPU loopback harness for the fused distributed transport kernel
(k_dd_transport): a rank whose prev and next neighbours are its own mailbox,
so the in-kernel rounds go through local HBM. Times it against the
single-GPU fused term (k_transport_tma, P = 1 plans) on the same block.

    python tools/dd_transport_loopback.py [--m 256] [--groups 8192] [--iters 20]
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
    ap.add_argument("--m", type=int, default=256)
    ap.add_argument("--groups", type=int, default=8192)
    ap.add_argument("--iters", type=int, default=20)
    ap.add_argument("--nu", type=float, default=0.01)
    args = ap.parse_args()
    m, G, sz = args.m, args.groups, 32
    n = 4 * m                                   # rank 1 of 4 on a periodic line
    h = 2 * np.pi / n
    part = T.SubdomainPartition.balanced(n, 4)
    s1, st1 = momentum._operator(1, h, n)
    s2, st2 = momentum._operator(2, h, n)
    p1 = T.Plan.create(s1, st1.c, part.local_sizes, 1, N.TDS_FLAG_CHUNK16)
    p2 = T.Plan.create(s2, st2.c, part.local_sizes, 1, N.TDS_FLAG_CHUNK16)
    ui = torch.randn((G, m, sz), dtype=torch.float64, device="cuda")
    uj = torch.randn_like(ui)
    out = torch.empty_like(ui)
    lib = N.lib()
    words = lib.tds_transport_mailbox_words(G, sz)
    mail = torch.full((words,), -1, dtype=torch.int64, device="cuda")
    mp = ctypes.c_void_p(mail.data_ptr())
    N.check(lib.tds_mailbox_init(mp, mail.numel(), _stream_handle()))
    vp = lambda t: ctypes.c_void_p(t.data_ptr())  # noqa: E731

    def fused(e):
        N.check(lib.tds_fused_transport(p1.handle, p2.handle, vp(ui), vp(uj), vp(out), args.nu,
                                        G, sz, mp, mp, mp, e, 0, _stream_handle()))

    def single(e):
        assert momentum._fused_contribution(ui, uj, out, m, h, args.nu, False)

    ev = [torch.cuda.Event(enable_timing=True) for _ in range(2)]
    pts = G * m * sz
    for name, fn in (("k_transport_tma (P=1 plans)", single), ("k_dd_transport loopback", fused)):
        for e in range(1, 4):
            fn(e)
        torch.cuda.synchronize()
        ev[0].record()
        for e in range(4, 4 + args.iters):
            fn(e)
        ev[1].record()
        torch.cuda.synchronize()
        ms = ev[0].elapsed_time(ev[1]) / args.iters
        print(f"{name}: m={m} {ms:.4f} ms/term {24 * pts / (ms * 1e-3) / 1e9:.1f} GB/s (24 B/pt)")
    err = ctypes.c_int(0)
    N.check(lib.tds_transport_mailbox_error(mp, G, sz, ctypes.byref(err)))
    print("mailbox error:", err.value)


if __name__ == "__main__":
    main()
