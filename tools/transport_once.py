"""One transport RHS evaluation (after one warm-up) for launch-list profiling:
    ncu --metrics gpu__time_duration.sum --csv python tools/transport_once.py"""
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2411_13532_b200 as T  # noqa: E402

n = int(os.environ.get("N", "512"))
g = torch.Generator(device="cuda")
g.manual_seed(5)
u3, v3, w3 = (torch.randn((n, n, n), dtype=torch.float64, device="cuda", generator=g)
              for _ in range(3))
f = T.VelocityField.from_arrays(u3, v3, w3, 0.01, 2 * np.pi / n, sz=32)
del u3, v3, w3
T.evaluate_transport_rhs(f)
torch.cuda.synchronize()
T.evaluate_transport_rhs(f)
torch.cuda.synchronize()
