"""Debug harness: SlabTransport on P in-process ranks of one GPU vs the
oracle, several rhs() calls per run (mailbox epochs).

    REPS=3 python tools/slab_debug.py
"""
import os, sys, itertools
sys.path.insert(0, "/root/repo")
import numpy as np, torch
import paper_2411_13532_b200 as T
from paper_2411_13532_b200 import transport as TR
from oracle import tds_oracle as O
os.environ["TDS_FUSED_TIMEOUT_MS"] = "2000"
os.environ.setdefault("REPS", "3")
n = 128
h = 2 * np.pi / n
rng = np.random.default_rng(77)
u3, v3, w3 = (rng.standard_normal((n, n, n)) for _ in range(3))
for p, nu, sz, tl in [(2, 0.0, 32, "16"), (2, 0.02, 32, "16"), (2, 0.0, 16, "16"), (2, 0.0, 32, "8"), (4, 0.01, 32, "16")]:
    os.environ["TDS_TRANSPORT_TL"] = tl
    def body(ctx):
        tr = T.SlabTransport(n, sz, nu, h, ctx)
        loc = [tr.local_slab(a) for a in (u3, v3, w3)]
        rhs = tr.rhs(*loc)
        for _ in range(int(os.environ.get("REPS", "1"))):
            rhs2 = tr.rhs(*loc)
        torch.cuda.current_stream().synchronize()
        tr.check()
        carts = [T.unpack(T.GroupedField(tr.lay["x"], c)).cpu().numpy() for c in rhs]
        tr.close()
        return carts
    try:
        res = TR.spawn_ranks(p, True, body, devices=[0] * p)
        full = [np.concatenate([r[i] for r in res], axis=2) for i in range(3)]
        want = O.transport_rhs(u3, v3, w3, nu, h, sz, rank_counts=(1, 1, p))
        print(p, nu, sz, tl, "err", max(O.rel_linf(g, w) for g, w in zip(full, want)), flush=True)
    except Exception as e:
        print(p, nu, sz, tl, "FAIL", repr(e)[:200], flush=True)
