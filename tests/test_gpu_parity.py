"""GPU parity: the CUDA path against the reference (golden fixtures produced by
the reference itself) and the pinned oracle.

Bars (north star): relative L-inf <= 1e-12 for the fast path; the strict
path is bit-identical to the reference. rel_linf = max|d| / max|ref|
(reference tests/test_distributed.py:47-48).
"""

import warnings

import numpy as np
import pytest

from conftest import golden_run
from oracle import tds_oracle as O

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

import paper_2411_13532_b200 as T  # noqa: E402

TOL = 1e-12


@pytest.fixture(autouse=True, scope="module")
def _need_gpu():
    if not torch.cuda.is_available():
        pytest.skip("needs a CUDA device")


def _sys(c):
    return T.TridiagonalSystem(c["lower"], c["diag"], c["upper"], periodic=c["periodic"])


def _st(c):
    return None if c["stencil"] is None else T.StencilCoeffs(c["stencil"])


def _run(c, arithmetic, field=None):
    with warnings.catch_warnings():
        warnings.simplefilter("ignore", T.NotDominantWarning)
        return T.run_distd2(_sys(c), c["field"] if field is None else field,
                            part=T.SubdomainPartition(c["sizes"]), stencil=_st(c),
                            arithmetic=arithmetic)


def _tags(golden):
    return [str(t) for t in golden["run_tags"]]


def test_every_golden_case_fast_within_1e12(golden):
    worst = 0.0
    for tag in _tags(golden):
        c = golden_run(golden, tag)
        got = _run(c, "fast")
        err = O.rel_linf(got, c["out"])
        worst = max(worst, err)
        assert err <= TOL, (tag, err)
    print(f"worst fast-path rel L-inf over golden cases: {worst:.3e}")


def test_every_golden_case_strict_bit_identical(golden):
    for tag in _tags(golden):
        c = golden_run(golden, tag)
        np.testing.assert_array_equal(_run(c, "strict"), c["out"], err_msg=tag)


def test_fast_path_is_taken_for_benchmark_shapes(golden):
    c = golden_run(golden, "d1p512_P1")
    plan = T.get_plan(_sys(c), _st(c), T.SubdomainPartition(c["sizes"]))
    assert plan.path == "fast" and plan.info.uniform == 1 and plan.info.chunk_rows == 32
    # open closures only touch the first / last chunk: uniform table + two
    # edge tables (uniform == 2), not the per-row global table
    c = golden_run(golden, "d1o512_P1")
    plan = T.get_plan(_sys(c), _st(c), T.SubdomainPartition(c["sizes"]))
    assert (plan.path, plan.info.uniform) == ("fast", 2)
    # emulated P = 8: the rank truncation lives in the reduced map H, the
    # chunk tables stay those of P = 1
    c = golden_run(golden, "d1o512_P8")
    plan = T.get_plan(_sys(c), _st(c), T.SubdomainPartition(c["sizes"]))
    assert (plan.path, plan.info.uniform) == ("fast", 2)


@pytest.mark.parametrize("sz,groups", [(32, 64), (16, 48), (8, 40)])
def test_open_edge_chunks_tma_sizes(sz, groups):
    """Config 4 (open d/dx, one-sided closures) at sizes that take the
    TMA-staged kernel with edge-special chunk tables, vs the oracle."""
    n = 512
    lo, di, up, st = O.assemble("d1", n, 2 * np.pi / n, False)
    s = T.TridiagonalSystem(lo, di, up, periodic=False)
    fld = np.random.default_rng(sz).standard_normal((groups, n, sz))
    plan = T.get_plan(s, T.StencilCoeffs(st), T.SubdomainPartition([n]))
    assert plan.info.uniform == 2
    want = O.run_distd2(lo, di, up, False, fld, st)
    got = T.run_distd2(s, torch.from_numpy(fld).cuda(), stencil=T.StencilCoeffs(st))
    assert O.rel_linf(got.cpu().numpy(), want) <= TOL


def test_device_tensor_in_device_tensor_out(golden):
    c = golden_run(golden, "d1p1024_P8")
    u = torch.from_numpy(c["field"]).cuda()
    out = T.run_distd2(_sys(c), u, part=T.SubdomainPartition(c["sizes"]), stencil=_st(c))
    assert out.is_cuda and out.shape == u.shape
    assert O.rel_linf(out.cpu().numpy(), c["out"]) <= TOL
    assert torch.equal(u.cpu(), torch.from_numpy(c["field"]))   # input untouched (D1)


def test_config1_64cubed(golden):
    n = 64
    s, st = T.assemble(T.sixth_order_first_derivative(2 * np.pi / n), n)
    u = np.random.default_rng(1234).standard_normal((n, n, n))
    fld = T.pack(u, T.LayoutDescriptor(n, n, n, 8, "x")).data
    np.testing.assert_array_equal(fld[:16], golden["c1_field"])
    out = T.run_distd2(s, fld, stencil=st)
    assert O.rel_linf(out[:16], golden["c1_out"]) <= TOL
    strict = T.run_distd2(s, fld, stencil=st, arithmetic="strict")
    np.testing.assert_array_equal(strict[:16], golden["c1_out"])
    assert float(strict.sum()) == float(golden["c1_full_sum"])


def test_phase_functions_bitwise(golden):
    g = golden
    s = T.TridiagonalSystem(g["dec_lower"], g["dec_diag"], g["dec_upper"])
    with warnings.catch_warnings():
        warnings.simplefilter("ignore", T.NotDominantWarning)
        co = T.preprocess(s, "interior", False)
    d = T.decouple_fused(g["dec_uext"], co, T.StencilCoeffs(g["dec_stencil"]))
    np.testing.assert_array_equal(d, g["dec_d"])
    np.testing.assert_array_equal(T.substitute(d, co, g["sub_us"], g["sub_ue"]), g["sub_out"])
    for row, want in zip(g["pair_in"], g["pair_out"]):
        ul, uf = T.solve_boundary_pair(T.BoundaryPair(np.array([row[0]]), np.array([row[1]]),
                                                      row[2], row[3]))
        assert ul[0] == want[0] and uf[0] == want[1]
    with pytest.raises(T.SingularPair):
        T.solve_boundary_pair(T.BoundaryPair(np.ones(1), np.ones(1), 1.0, 1.0))
    # decouple_unfused on the reference's own build_rhs output (distributed.py:
    # 242-254), bit-equal to the reference and to decouple_fused (D12)
    du = T.decouple_unfused(g["decu_rhs"], co)
    np.testing.assert_array_equal(du, g["decu_d"])
    np.testing.assert_array_equal(du, d)
    dz = T.decouple_unfused(np.zeros((16, 3)), co)
    np.testing.assert_array_equal(dz, np.zeros((16, 3)))


def test_serial_solvers_bitwise(golden):
    g = golden
    so = T.TridiagonalSystem(g["thomas_lower"], g["thomas_diag"], g["thomas_upper"])
    sp = T.TridiagonalSystem(g["pthomas_lower"], g["pthomas_diag"], g["pthomas_upper"],
                             periodic=True)
    rhs = T.RhsBatch(g["thomas_rhs"])
    np.testing.assert_array_equal(T.thomas_solve(so, rhs).values, g["thomas_out"])
    np.testing.assert_array_equal(T.periodic_thomas_solve(sp, rhs).values, g["pthomas_out"])


def test_layout_pack_unpack_reorder_bitwise(golden):
    cart = golden["pack_cart"]
    for d in "xyz":
        f = T.pack(cart, T.LayoutDescriptor(4, 6, 8, 8, d))
        np.testing.assert_array_equal(f.data, golden[f"pack_{d}"])
        np.testing.assert_array_equal(T.unpack(f), cart)
        for d2 in "xyz":
            np.testing.assert_array_equal(T.reorder(f, d2).data, golden[f"pack_{d2}"])
    # ghost lines are zero-filled and stripped again
    lay = T.LayoutDescriptor(4, 6, 6, 8, "x", pad=True)
    c2 = np.random.default_rng(1).standard_normal((4, 6, 6))
    f = T.pack(c2, lay)
    assert f.data.shape == (5, 4, 8)
    np.testing.assert_array_equal(f.data.transpose(0, 2, 1).reshape(40, 4)[36:], 0.0)
    np.testing.assert_array_equal(T.unpack(f), c2)


@pytest.mark.parametrize("direction", "xyz")
def test_512_lines_all_directions_vs_oracle(direction):
    """Config 2 geometry on a subset of lines: a 512 x 8 x 8 box packed for
    each direction has 512-point lines in x only; use a 64^3 cube with sz=32
    for y/z and 512-long x lines for x."""
    rng = np.random.default_rng(5)
    shape = {"x": (512, 8, 8), "y": (8, 512, 8), "z": (8, 8, 512)}[direction]
    cart = rng.standard_normal(shape)
    lay = T.LayoutDescriptor(*shape, 32, direction)
    n = lay.n
    s, st = T.assemble(T.sixth_order_first_derivative(2 * np.pi / n), n)
    fld = T.pack(cart, lay).data
    want = O.run_distd2(s.lower, s.diag, s.upper, True, fld, st.c)
    got = T.run_distd2(s, fld, stencil=st)
    assert O.rel_linf(got, want) <= TOL


@pytest.mark.parametrize("n,p,periodic,kind", [
    (512, 1, False, "d1"), (512, 2, True, "d1"), (1024, 4, True, "d1"), (1024, 8, False, "d1"),
    (2048, 8, True, "d1"), (2048, 1, True, "d1"),
    (256, 1, True, "d2"), (256, 4, True, "d2"), (96, 3, True, "rd"), (48, 1, False, "rd"),
    (80, 5, False, "rd"), (64, 2, True, "rd")])
def test_fast_vs_oracle_sweep(n, p, periodic, kind):
    rng = np.random.default_rng(n * 10 + p)
    if kind == "rd":
        a = 0.3 * (2 * rng.random(n) - 1)
        b = 2 + rng.random(n)
        c = 0.3 * (2 * rng.random(n) - 1)
        st = rng.standard_normal((n, 5))
        lo, di, up = a, b, c
    else:
        lo, di, up, st = O.assemble(kind, n, 2 * np.pi / n, periodic)
    fld = rng.standard_normal((3, n, 16))
    sizes = O.balanced_sizes(n, p)
    want = O.run_distd2(lo, di, up, periodic, fld, st, sizes)
    s = T.TridiagonalSystem(lo, di, up, periodic=periodic)
    with warnings.catch_warnings():
        warnings.simplefilter("ignore", T.NotDominantWarning)
        got = T.run_distd2(s, fld, part=T.SubdomainPartition(sizes), stencil=T.StencilCoeffs(st))
        strict = T.run_distd2(s, fld, part=T.SubdomainPartition(sizes),
                              stencil=T.StencilCoeffs(st), arithmetic="strict")
    assert O.rel_linf(got, want) <= TOL
    np.testing.assert_array_equal(strict, want)


def test_ragged_and_small_shapes():
    """Line counts that do not fill a tile, sz that is not a multiple of 16,
    a single line, and a partition that is not chunk-aligned (staged path)."""
    rng = np.random.default_rng(11)
    for (g, n, sz) in [(1, 64, 1), (3, 64, 5), (7, 128, 8), (2, 48, 3), (1, 20, 8)]:
        lo, di, up, st = O.assemble("d1", n, 0.1, True) if n >= 8 else None
        fld = rng.standard_normal((g, n, sz))
        s = T.TridiagonalSystem(lo, di, up, periodic=True)
        want = O.run_distd2(lo, di, up, True, fld, st)
        got = T.run_distd2(s, fld, stencil=T.StencilCoeffs(st))
        assert O.rel_linf(got, want) <= TOL, (g, n, sz)
    # empty field
    lo, di, up, st = O.assemble("d1", 64, 0.1, True)
    out = T.run_distd2(T.TridiagonalSystem(lo, di, up, True), np.zeros((0, 64, 8)),
                       stencil=T.StencilCoeffs(st))
    assert out.shape == (0, 64, 8)


def test_errors_match_reference():
    s = T.TridiagonalSystem(np.full(16, 0.1), np.ones(16), np.full(16, 0.1), periodic=True)
    with pytest.raises(ValueError):
        T.run_distd2(s, np.zeros((1, 16, 4)), part=T.SubdomainPartition((8, 4)))
    with pytest.raises(ValueError):
        T.run_distd2(s, np.zeros((16, 4)))
    # singular pair across a rank boundary -> RankPanic (transport.py:137-138)
    a = np.zeros(8)
    c = np.zeros(8)
    a[4], c[3] = 1.0, 1.0
    bad = T.TridiagonalSystem(a, np.ones(8), c)
    with warnings.catch_warnings():
        warnings.simplefilter("ignore", T.NotDominantWarning)
        with pytest.raises((T.RankPanic, T.SingularPivot)):
            T.run_distd2(bad, np.ones((1, 8, 1)), rank_count=2)


def test_audit_matches_reference_protocol(golden):
    # reference tests/test_distributed.py:263-286
    for p in (2, 3, 5, 8):
        for cyclic in (False, True):
            n = 16 * p
            r = np.random.default_rng(p)
            s = T.TridiagonalSystem(0.2 * (2 * r.random(n) - 1), 2 + r.random(n),
                                    0.2 * (2 * r.random(n) - 1), periodic=cyclic)
            audit = {}
            T.run_distd2(s, r.standard_normal((1, n, 2)), part=T.SubdomainPartition.balanced(n, p),
                         audit=audit)
            assert audit["rounds_per_rank"] == [2] * p
            edges = 2 * p if cyclic else 2 * (p - 1)
            assert audit["messages_sent"] == 3 * edges


def test_lane_permutation_bitwise_and_sz_independence():
    rng = np.random.default_rng(3)
    n = 512
    s, st = T.assemble(T.sixth_order_first_derivative(2 * np.pi / n), n)
    f = rng.standard_normal((4, n, 32))
    base = T.run_distd2(s, f, stencil=st)
    perm = rng.permutation(32)
    np.testing.assert_array_equal(T.run_distd2(s, f[:, :, perm], stencil=st), base[:, :, perm])
    # same lines in an sz=8 layout give bit-identical results
    f8 = f.transpose(0, 2, 1).reshape(16, 8, n).transpose(0, 2, 1).copy()
    out8 = T.run_distd2(s, f8, stencil=st)
    np.testing.assert_array_equal(out8.transpose(0, 2, 1).reshape(4, 32, n).transpose(0, 2, 1),
                                  base)


def test_operator_accuracy_and_order():
    # reference tests/test_compact.py:150-200
    res = T.order_of_accuracy(T.sixth_order_first_derivative(1.0), T.operator_applier(1),
                              (32, 64, 128, 256))
    assert 5.5 < res.slope < 6.3 and res.error_at(256) < 1e-12
    for n in (128, 256):
        h = 2 * np.pi / n
        s, st = T.assemble(T.sixth_order_first_derivative(h), n)
        u = np.sin(h * np.arange(n))
        d = T.apply_operator(s, st, u, rank_count=2) - T.apply_operator(s, st, u, rank_count=1)
        assert np.max(np.abs(d)) <= 1e-14
    n = 32
    s, st = T.assemble(T.sixth_order_first_derivative(2 * np.pi / n), n)
    assert np.max(np.abs(T.apply_operator(s, st, np.full(n, 7.25)))) < 1e-13
    res2 = T.order_of_accuracy(T.second_derivative_scheme(1.0), T.operator_applier(1),
                               (32, 64, 128, 256))
    assert res2.slope >= 4.0


def test_pinned_host_pipeline_matches_oracle(golden):
    """Pinned CPU tensors take the chunked H2D / kernel / D2H pipeline."""
    from paper_2411_13532_b200 import distributed as D
    c = golden_run(golden, "d1p512_P8")
    s = _sys(c)
    old = D.PIPE_CHUNK_BYTES
    D.PIPE_CHUNK_BYTES = 512 * 32 * 8          # one group per chunk: many chunks
    try:
        rng = np.random.default_rng(8)
        f = rng.standard_normal((9, 512, 32))
        host = torch.from_numpy(f).pin_memory()
        out = torch.empty_like(host).pin_memory()
        for sizes in (c["sizes"], (512,)):
            got = T.run_distd2(s, host, part=T.SubdomainPartition(sizes), stencil=_st(c), out=out)
            assert got.data_ptr() == out.data_ptr()
            want = O.run_distd2(c["lower"], c["diag"], c["upper"], c["periodic"], f,
                                c["stencil"], sizes)
            assert O.rel_linf(got.numpy(), want) <= TOL
    finally:
        D.PIPE_CHUNK_BYTES = old


@pytest.mark.parametrize("sz", [8, 16, 32])
def test_pack_unpack_reorder_ragged_extents(sz):
    """Tiled reorder kernel on extents that are not multiples of its 32x32
    tile, all directions, bitwise against the oracle's pack."""
    cart = np.random.default_rng(sz).standard_normal((48, 40, 72))
    for d in "xyz":
        lay = T.LayoutDescriptor(48, 40, 72, sz, d, pad=True)
        f = T.pack(cart, lay)
        lines = lay.lines
        want = O.pack(cart, 1, d).reshape(lines, lay.n)          # (lines, n), sz-free
        got = f.data.transpose(0, 2, 1).reshape(lay.padded_lines, lay.n)
        np.testing.assert_array_equal(got[:lines], want)
        np.testing.assert_array_equal(got[lines:], 0.0)
        np.testing.assert_array_equal(T.unpack(f), cart)
        for d2 in "xyz":
            np.testing.assert_array_equal(T.unpack(T.reorder(f, d2)), cart)


@pytest.mark.parametrize("n,p,periodic,kind,sz", [
    (2048, 1, True, "d1", 32), (2048, 1, False, "d1", 32), (4096, 1, True, "d1", 32),
    (8192, 1, True, "d1", 32), (8192, 1, False, "d1", 16), (2048, 4, True, "d1", 32),
    (4096, 2, False, "d1", 16), (2048, 1, True, "d2", 32), (2048, 1, True, "rd", 32),
    (4096, 1, False, "rd", 16), (2048, 1, True, "d1", 8), (2048, 2, True, "d1", 4)])
def test_long_lines_cluster_kernel_vs_oracle(n, p, periodic, kind, sz):
    """Lines of 2048..8192 rows (reference bench.py:178-219 sweeps n up to
    8192): the fast 16 B/pt path with each line split over a thread-block
    cluster (k_tmc, reduced rhs exchanged through distributed shared memory).
    sz = 4 has no 8-lane tiles and takes the plan's staged tables instead
    (reference operation order: bit-identical)."""
    rng = np.random.default_rng(n + 7 * p + sz)
    if kind == "rd":
        lo = 0.3 * (2 * rng.random(n) - 1)
        di = 2 + rng.random(n)
        up = 0.3 * (2 * rng.random(n) - 1)
        st = rng.standard_normal((n, 5))
    else:
        lo, di, up, st = O.assemble(kind, n, 2 * np.pi / n, periodic)
    fld = rng.standard_normal((2, n, sz))
    sizes = O.balanced_sizes(n, p)
    want = O.run_distd2(lo, di, up, periodic, fld, st, sizes)
    s = T.TridiagonalSystem(lo, di, up, periodic=periodic)
    part = T.SubdomainPartition(sizes)
    with warnings.catch_warnings():
        warnings.simplefilter("ignore", T.NotDominantWarning)
        plan = T.get_plan(s, T.StencilCoeffs(st), part)
        got = T.run_distd2(s, fld, part=part, stencil=T.StencilCoeffs(st))
    assert plan.path == "fast" and plan.info.chunks > 32
    if sz % 8:
        np.testing.assert_array_equal(got, want)
    else:
        assert O.rel_linf(got, want) <= TOL


@pytest.mark.parametrize("n,periodic", [(512, True), (512, False), (256, True), (2048, True),
                                        (4096, False)])
def test_dynamic_item_schedule_bitwise_and_concurrent(monkeypatch, n, periodic):
    """k_tma hands items past the grid's first out through a per-plan counter
    (TDS_DYN, default): on a field with dozens of items per CTA the result is
    bit-identical to the static round-robin schedule and to the oracle's
    bound, repeated launches reuse the counter slots (last CTA resets them),
    and launches of ONE plan on several streams at once use different slots.
    n >= 2048: the cluster kernel k_tmc (the cluster's CTA 0 claims items)."""
    groups, sz = (2048 if n <= 512 else 256), 32       # >> the persistent grid's items
    lo, di, up, stc = O.assemble("d1", n, 2 * np.pi / n, periodic)
    s = T.TridiagonalSystem(lo, di, up, periodic=periodic)
    st = T.StencilCoeffs(stc)
    u = torch.randn((groups, n, sz), dtype=torch.float64, device="cuda",
                    generator=torch.Generator(device="cuda").manual_seed(n))
    monkeypatch.setenv("TDS_DYN", "0")
    ref = T.run_distd2(s, u, stencil=st)
    torch.cuda.synchronize()
    monkeypatch.setenv("TDS_DYN", "1")
    for _ in range(70):                                # > the 64 counter slots
        got = T.run_distd2(s, u, stencil=st)
    torch.cuda.synchronize()
    assert torch.equal(got, ref)
    streams = [torch.cuda.Stream() for _ in range(4)]
    outs = [torch.empty_like(u) for _ in streams]
    torch.cuda.synchronize()
    for _ in range(3):
        for st_, o in zip(streams, outs):
            with torch.cuda.stream(st_):
                T.run_distd2(s, u, stencil=st, out=o)
    torch.cuda.synchronize()
    for o in outs:
        assert torch.equal(o, ref)
    sub = u[:64].cpu().numpy()
    want = O.run_distd2(lo, di, up, periodic, sub, stc)
    assert O.rel_linf(ref[:64].cpu().numpy(), want) <= 1e-12
