"""Momentum-transport RHS (BASELINE config 5's consumer of the DistD2 path):
GPU pipeline vs the reference's own evaluate_transport_rhs (golden, 16^3) and
vs the pinned oracle (fused k_transport path, 64^3)."""

import numpy as np
import pytest

from oracle import tds_oracle as O

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

import paper_2411_13532_b200 as T  # noqa: E402

TOL = 1e-12


@pytest.fixture(autouse=True, scope="module")
def _need_gpu():
    if not torch.cuda.is_available():
        pytest.skip("needs a CUDA device")


def _rel(got, want):
    return O.rel_linf(np.asarray(got), want)


@pytest.mark.parametrize("tag,nu", [("nu", 0.1), ("inviscid", 0.0)])
def test_transport_rhs_matches_reference_golden(golden, tag, nu):
    n = 16
    f = T.VelocityField.from_arrays(golden["tr_u"], golden["tr_v"], golden["tr_w"], nu,
                                    2 * np.pi / n, sz=4)
    rhs = T.evaluate_transport_rhs(f)
    want = golden[f"tr_{tag}_rhs"]
    for i in range(3):
        assert _rel(T.unpack(rhs[i]).cpu().numpy(), want[i]) <= TOL


@pytest.mark.parametrize("sz", [32, 8])
def test_fused_transport_kernel_vs_oracle(sz):
    n = 64
    r = np.random.default_rng(sz)
    u3, v3, w3 = (r.standard_normal((n, n, n)) for _ in range(3))
    h, nu = 2 * np.pi / n, 0.05
    f = T.VelocityField.from_arrays(u3, v3, w3, nu, h, sz=sz)
    rhs = T.evaluate_transport_rhs(f)
    want = O.transport_rhs(u3, v3, w3, nu, h, sz)
    for i in range(3):
        assert _rel(T.unpack(rhs[i]).cpu().numpy(), want[i]) <= TOL
    # one directional contribution through the public API as well
    c = T.directional_contribution("v", "x", f)
    lo, di, up, st = O.assemble("d1", n, h, True)
    lo2, di2, up2, st2 = O.assemble("d2", n, h, True)
    pu = O.pack(v3, sz, "x")
    adv = O.pack(u3, sz, "x")
    dc = O.run_distd2(lo, di, up, True, pu, st)
    dp = O.run_distd2(lo, di, up, True, adv * pu, st)
    ref = -0.5 * (adv * dc + dp) + nu * O.run_distd2(lo2, di2, up2, True, pu, st2)
    assert _rel(c.data.cpu().numpy(), ref) <= TOL


def test_transport_emulated_ranks_and_euler_step():
    n = 64
    x = 2 * np.pi * np.arange(n) / n
    X, Y, Z = np.meshgrid(x, x, x, indexing="ij")
    u3 = np.sin(X) * np.cos(Y) + 0.3 * np.cos(Z)
    v3 = np.cos(X) * np.sin(Z) - 0.2 * np.sin(Y)
    w3 = np.sin(Y) * np.cos(Z) + 0.1 * np.cos(X)
    f = T.VelocityField.from_arrays(u3, v3, w3, 0.1, 2 * np.pi / n, sz=32)
    one = T.evaluate_transport_rhs(f)
    two = T.evaluate_transport_rhs(f, rank_count=2)   # DistD2 truncation at 2 ranks
    for a, b in zip(one, two):
        assert _rel(b.data.cpu().numpy(), a.data.cpu().numpy()) <= 1e-10
    step = T.euler_step(f, 1e-3)
    for i in range(3):
        np.testing.assert_allclose(step.component(i).data.cpu().numpy(),
                                   (f.component(i).data + 1e-3 * one[i].data).cpu().numpy(),
                                   rtol=0, atol=1e-15)
    with pytest.raises(ValueError):
        T.directional_contribution("u", "y", f)


@pytest.mark.parametrize("extents,sz", [((64, 48, 16), 16), ((40, 24, 8), 8), ((32, 32, 96), 32)])
def test_reorder3_block_bitwise(extents, sz):
    """One-pass k_reorder on non-cubic blocks (a rank's slab): bitwise equal
    to unpack + pack, and accumulate adds exactly."""
    rng = np.random.default_rng(sum(extents))
    cart = rng.standard_normal(extents)
    for a in "xyz":
        f = T.pack(cart, T.LayoutDescriptor(*extents, sz, a))
        for b in "xyz":
            want = T.pack(cart, T.LayoutDescriptor(*extents, sz, b)).data
            got = T.reorder(f, b)
            np.testing.assert_array_equal(got.data, want)
    fx = torch.from_numpy(T.pack(cart, T.LayoutDescriptor(*extents, sz, "x")).data).cuda()
    lz = T.LayoutDescriptor(*extents, sz, "z")
    acc = torch.from_numpy(T.pack(cart, lz).data).cuda()
    import ctypes
    from paper_2411_13532_b200 import _native as N
    N.check(N.lib().tds_reorder3(ctypes.c_void_p(fx.data_ptr()), ctypes.c_void_p(acc.data_ptr()),
                                 *extents, sz, 0, 2, 1, None))
    np.testing.assert_array_equal(acc.cpu().numpy(), 2 * T.pack(cart, lz).data)


@pytest.mark.parametrize("nu", [0.05, 0.0])
def test_slab_transport_single_rank(nu):
    """SlabTransport with one rank (whole box on this GPU) vs the oracle and
    vs evaluate_transport_rhs."""
    n, sz = 64, 16
    rng = np.random.default_rng(21)
    u3, v3, w3 = (rng.standard_normal((n, n, n)) for _ in range(3))
    tr = T.SlabTransport(n, sz, nu, 2 * np.pi / n)
    rhs = tr.rhs(*(tr.local_slab(a) for a in (u3, v3, w3)))
    want = O.transport_rhs(u3, v3, w3, nu, 2 * np.pi / n, sz)
    f = T.VelocityField.from_arrays(u3, v3, w3, nu, 2 * np.pi / n, sz=sz)
    ev = T.evaluate_transport_rhs(f)
    for i in range(3):
        got = T.unpack(T.GroupedField(tr.lay["x"], rhs[i])).cpu().numpy()
        assert _rel(got, want[i]) <= TOL
        assert torch.equal(rhs[i], ev[i].data)


@pytest.mark.parametrize("n,sz,nu,tl", [(64, 32, 0.05, 16), (64, 8, 0.0, 16), (128, 16, 0.02, 16),
                                        (128, 32, 0.0, 16), (96, 32, 0.01, 16),
                                        (64, 32, 0.02, 8), (128, 32, 0.0, 8)])
def test_in_place_y_z_bitwise_equals_reorder_pipeline(monkeypatch, n, sz, nu, tl):
    """y / z contributions read in place from the x layout and added into the
    accumulators (tds_transport_contribution_in_x; y needs sz = 32) give the
    same bits as the reference-shaped reorder -> contribution ->
    reorder/accumulate pipeline, and match the oracle."""
    monkeypatch.setenv("TDS_TRANSPORT_TL", str(tl))     # 8: the n = 1024 tile width
    rng = np.random.default_rng(n + sz)
    u3, v3, w3 = (rng.standard_normal((n, n, n)) for _ in range(3))
    f = T.VelocityField.from_arrays(u3, v3, w3, nu, 2 * np.pi / n, sz=sz)
    from paper_2411_13532_b200 import momentum
    assert momentum._in_x_plans(f, "z") is not None
    assert (momentum._in_x_plans(f, "y") is not None) == (sz == 32 and n % 32 == 0)
    direct = T.evaluate_transport_rhs(f)
    monkeypatch.setenv("TDS_TRANSPORT_Y", "0")
    monkeypatch.setenv("TDS_TRANSPORT_Z", "0")
    assert momentum._in_x_plans(f, "z") is None and momentum._in_x_plans(f, "y") is None
    staged = T.evaluate_transport_rhs(f)
    for a, b in zip(direct, staged):
        assert torch.equal(a.data, b.data)
    want = O.transport_rhs(u3, v3, w3, nu, 2 * np.pi / n, sz)
    for i in range(3):
        assert _rel(T.unpack(direct[i]).cpu().numpy(), want[i]) <= TOL


@pytest.mark.parametrize("n,sz,groups", [(1024, 8, 3), (1024, 16, 2), (512, 32, 2), (256, 8, 4)])
def test_fused_contribution_kernel_sizes_vs_oracle(n, sz, groups):
    """The fused contribution kernel (16-row chunks, 8/16-line tiles, up to
    64 chunks at n = 1024) on a few groups of lines vs three oracle solves."""
    from paper_2411_13532_b200 import momentum
    rng = np.random.default_rng(n + sz)
    ui = torch.from_numpy(rng.standard_normal((groups, n, sz))).cuda()
    uj = torch.from_numpy(rng.standard_normal((groups, n, sz))).cuda()
    out = torch.empty_like(ui)
    h, nu = 2 * np.pi / n, 0.03
    assert momentum._fused_contribution(ui, uj, out, n, h, nu, False)
    lo, di, up, st = O.assemble("d1", n, h, True)
    lo2, di2, up2, st2 = O.assemble("d2", n, h, True)
    a, b = ui.cpu().numpy(), uj.cpu().numpy()
    ref = (-0.5 * (b * O.run_distd2(lo, di, up, True, a, st)
                   + O.run_distd2(lo, di, up, True, b * a, st))
           + nu * O.run_distd2(lo2, di2, up2, True, a, st2))
    assert _rel(out.cpu().numpy(), ref) <= TOL


@pytest.mark.parametrize("n,sz,tl", [(64, 32, "8"), (64, 32, "16"), (128, 32, "8"),
                                     (64, 16, "8"), (96, 32, "8")])
@pytest.mark.parametrize("nu", [0.0, 0.07])
def test_direction_kernel_vs_oracle_and_per_term(monkeypatch, n, sz, tl, nu):
    """k_transport_dir (all three components of one direction per launch,
    x writes, y / z add in place) against the oracle's reference-shaped RHS
    and against the per-term kernels (TDS_TRANSPORT_DIR=0)."""
    r = np.random.default_rng(n + sz + int(tl))
    u3, v3, w3 = (r.standard_normal((n, n, n)) for _ in range(3))
    h = 2 * np.pi / n
    f = T.VelocityField.from_arrays(u3, v3, w3, nu, h, sz=sz)
    monkeypatch.setenv("TDS_TRANSPORT_DIR_TL", tl)
    from paper_2411_13532_b200 import momentum as MOM
    acc = [torch.empty_like(f.component(i).data) for i in range(3)]
    done = MOM._direction_passes(f, acc, (0, 1, 2))
    assert done == ({0, 1, 2} if sz == 32 else {0})
    rhs = T.evaluate_transport_rhs(f)
    want = O.transport_rhs(u3, v3, w3, nu, h, sz)
    monkeypatch.setenv("TDS_TRANSPORT_DIR", "0")
    per_term = T.evaluate_transport_rhs(f)
    for i in range(3):
        got = T.unpack(rhs[i]).cpu().numpy()
        assert _rel(got, want[i]) <= TOL
        # same solves as the per-term kernels; the circulant band row differs
        # from the per-chunk rows in the last bits
        assert _rel(rhs[i].data.cpu().numpy(), per_term[i].data.cpu().numpy()) <= 1e-14
