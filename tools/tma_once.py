"""A few 512^3 DistD2 solves (BASELINE config 2's kernel, k_tma) for ncu:
    ncu --set full -k regex:k_tma -s 3 -c 1 python tools/tma_once.py"""
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2411_13532_b200 as T  # noqa: E402

n = int(os.environ.get("N", "512"))
s, st = T.assemble(T.sixth_order_first_derivative(2 * np.pi / n), n, periodic=True)
g = torch.Generator(device="cuda")
g.manual_seed(1235)
u = torch.randn((n * n // 32, n, 32), dtype=torch.float64, device="cuda", generator=g)
out = torch.empty_like(u)
for _ in range(6):
    T.run_distd2(s, u, stencil=st, out=out)
torch.cuda.synchronize()
