"""Fused per-rank kernels (k_dd, k_dd2) on ONE GPU: a rank whose prev and next
neighbours are its own mailbox. Its block is the whole periodic line and the
DistD2 pair couples its own last and first rows, so the result is the exact
periodic solve up to the dropped coupling (~1e-27 at 512 rows): it must agree
with the oracle's (periodic Thomas) result within 1e-12 relative."""

import ctypes
import os

import numpy as np
import pytest

from oracle import tds_oracle as O

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

import paper_2411_13532_b200 as T  # noqa: E402
from paper_2411_13532_b200 import _native as N  # noqa: E402
from paper_2411_13532_b200.distributed import _stream_handle  # noqa: E402


@pytest.fixture(autouse=True, scope="module")
def _need_gpu():
    if not torch.cuda.is_available():
        pytest.skip("needs a CUDA device")


def _loopback(n, groups, sz, env, seed=0, epochs=3):
    s, st = T.assemble(T.sixth_order_first_derivative(2 * np.pi / n), n)
    # the whole line as one rank of a 1-rank ring: external couplings wrap
    loc = T.TridiagonalSystem(s.lower, s.diag, s.upper, periodic=False)
    co = T.preprocess(loc, "interior", True)
    plan = T.Plan.create_local(loc, st.c, True, True, co.s_c[-1], co.s_a[0])
    lib = N.lib()
    assert lib.tds_fused_eligible(plan.handle, groups, sz) == 1
    u_np = np.random.default_rng(seed).standard_normal((groups, n, sz))
    u = torch.from_numpy(u_np).cuda()
    out = torch.empty_like(u)
    mail = torch.full((lib.tds_mailbox_words(groups, sz),), -1, dtype=torch.int64, device="cuda")
    mp = ctypes.c_void_p(mail.data_ptr())
    N.check(lib.tds_mailbox_init(mp, mail.numel(), _stream_handle()))
    old = {k: os.environ.get(k) for k in env}
    os.environ.update(env)
    try:
        for e in range(1, epochs + 1):
            N.check(lib.tds_fused_solve(plan.handle, ctypes.c_void_p(u.data_ptr()),
                                        ctypes.c_void_p(out.data_ptr()), groups, sz, mp, mp, mp,
                                        e, 0, _stream_handle()))
        torch.cuda.synchronize()
    finally:
        for k, v in old.items():
            if v is None:
                os.environ.pop(k, None)
            else:
                os.environ[k] = v
    err = ctypes.c_int(0)
    N.check(lib.tds_mailbox_error(mp, groups, sz, ctypes.byref(err)))
    assert err.value == 0
    want = O.run_distd2(s.lower, s.diag, s.upper, True, u_np, st.c)
    return O.rel_linf(out.cpu().numpy(), want)


@pytest.mark.parametrize("env", [{"TDS_DEFER": "0"}, {"TDS_DEFER": "1"}, {"TDS_DEFER": "2"},
                                 {"TDS_DEFER": "1", "TDS_TL": "8"}])
@pytest.mark.parametrize("n", [512, 256, 128])
def test_fused_loopback_matches_periodic_solve(n, env):
    assert _loopback(n, 64, 32, env) <= 1e-12


def test_fused_loopback_many_epochs_and_ragged_tail():
    # 33 groups: the persistent grid ends on a partial wave; epochs cycle the
    # mailbox parity halves several times
    assert _loopback(256, 33, 16, {}, seed=3, epochs=6) <= 1e-12
