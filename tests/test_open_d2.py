"""Open (non-periodic) second derivative -- BASELINE config 4's "first and
second derivatives, non-periodic" -- a B200-side extension: the reference
raises NotImplementedError (compact.py:79-81), so there is no reference
output to pin it to. It is validated by ORDER OF ACCURACY on smooth
non-periodic fields (the closures are third order at the boundary, the
interior scheme sixth order), and the GPU paths are checked against the
oracle's restatement of the same closures (tds_oracle.assemble_open_d2):
fast paths within 1e-12, the staged / strict kernels bit-identical."""

import warnings

import numpy as np
import pytest

from oracle import tds_oracle as O

import paper_2411_13532_b200 as T

TOL = 1e-12


def _smooth(n):
    h = 1.0 / (n - 1)
    x = h * np.arange(n)
    f = np.sin(2.3 * x + 0.4) * np.exp(0.5 * x)
    d2 = ((0.25 - 2.3 ** 2) * np.sin(2.3 * x + 0.4) + 2.3 * np.cos(2.3 * x + 0.4)) * np.exp(0.5 * x)
    return h, f, d2


def test_default_still_raises_like_the_reference():
    with pytest.raises(NotImplementedError):
        T.assemble(T.second_derivative_scheme(0.1), 32, periodic=False)
    with pytest.raises(ValueError):
        T.assemble(T.second_derivative_scheme(0.1), 32, periodic=False, closure="bogus")


def test_closure_rows_and_shifts_match_oracle():
    n, h = 40, 0.05
    s, st = T.assemble(T.second_derivative_scheme(h), n, periodic=False, closure="one-sided")
    lo, di, up, stc, sh = O.assemble_open_d2(n, h)
    np.testing.assert_array_equal(s.lower, lo)
    np.testing.assert_array_equal(s.diag, di)
    np.testing.assert_array_equal(s.upper, up)
    np.testing.assert_array_equal(st.c, stc)
    np.testing.assert_array_equal(st.shift, sh)
    assert st.shift[0] == 2 and st.shift[-1] == -2 and not np.any(st.shift[1:-1])
    # shifted closure rows reproduce polynomials of degree <= 4 exactly
    x = np.arange(n, dtype=float) * h
    for p in range(5):
        u = x ** p
        ext = np.concatenate([[0, 0], u, [0, 0]])
        rhs = O.build_rhs(ext, stc, sh)
        want = p * (p - 1) * x ** max(p - 2, 0) if p >= 2 else np.zeros(n)
        lhs0 = want[0] + up[0] * want[1]
        assert abs(rhs[0] - lhs0) <= 1e-6 * max(1.0, abs(lhs0))


def test_stencil_shift_validation():
    with pytest.raises(ValueError):
        T.StencilCoeffs(np.zeros((8, 5)), shift=np.zeros(7))
    with pytest.raises(ValueError):
        T.StencilCoeffs(np.zeros((8, 5)), shift=np.full(8, 3))
    assert T.StencilCoeffs(np.zeros((8, 5)), shift=np.zeros(8)).shift is None


def test_oracle_order_of_accuracy():
    errs = []
    ns = (64, 128, 256, 512)
    for n in ns:
        h, f, d2 = _smooth(n)
        lo, di, up, st, sh = O.assemble_open_d2(n, h)
        got = O.run_distd2(lo, di, up, False, f.reshape(1, n, 1), st, shift=sh).reshape(n)
        errs.append(np.max(np.abs(got - d2)))
    slope = -np.polyfit(np.log(ns), np.log(errs), 1)[0]
    assert 2.8 <= slope <= 3.6, (slope, errs)


# ------------------------------------------------------------------ GPU

torch = pytest.importorskip("torch")


@pytest.fixture
def gpu():
    if not torch.cuda.is_available():
        pytest.skip("needs a CUDA device")


def _op(n, h=None):
    h = 2 * np.pi / n if h is None else h
    s, st = T.assemble(T.second_derivative_scheme(h), n, periodic=False, closure="one-sided")
    lo, di, up, stc, sh = O.assemble_open_d2(n, h)
    return s, st, (lo, di, up, stc, sh)


@pytest.mark.gpu
@pytest.mark.parametrize("n,sz,groups", [(512, 32, 40), (512, 8, 24), (64, 16, 6),
                                          (1024, 32, 8), (2048, 16, 4), (96, 8, 3)])
def test_gpu_open_d2_vs_oracle(gpu, n, sz, groups):
    s, st, (lo, di, up, stc, sh) = _op(n)
    fld = np.random.default_rng(n + sz).standard_normal((groups, n, sz))
    want = O.run_distd2(lo, di, up, False, fld, stc, shift=sh)
    with warnings.catch_warnings():
        warnings.simplefilter("ignore", T.NotDominantWarning)
        got = T.run_distd2(s, fld, stencil=st)
        strict = T.run_distd2(s, fld, stencil=st, arithmetic="strict")
    assert O.rel_linf(got, want) <= TOL
    np.testing.assert_array_equal(strict, want)


@pytest.mark.gpu
@pytest.mark.parametrize("p", [2, 4, 8])
def test_gpu_open_d2_ranks_vs_oracle(gpu, p):
    n, sz, groups = 512, 32, 6
    s, st, (lo, di, up, stc, sh) = _op(n)
    sizes = O.balanced_sizes(n, p)
    part = T.SubdomainPartition(sizes)
    fld = np.random.default_rng(p).standard_normal((groups, n, sz))
    want = O.run_distd2(lo, di, up, False, fld, stc, sizes, shift=sh)
    with warnings.catch_warnings():
        warnings.simplefilter("ignore", T.NotDominantWarning)
        emulated = T.run_distd2(s, fld, part=part, stencil=st)
        ranks = T.run_distd2(s, fld, part=part, stencil=st, devices=[0] * p)     # fused k_dd*
        strict = T.run_distd2(s, fld, part=part, stencil=st, arithmetic="strict")
    assert O.rel_linf(emulated, want) <= TOL
    assert O.rel_linf(ranks, want) <= TOL
    np.testing.assert_array_equal(strict, want)


@pytest.mark.gpu
def test_gpu_open_d2_two_pass_ranks_strict_bitwise(gpu, monkeypatch):
    monkeypatch.setenv("TDS_FUSED", "0")
    n, sz, groups = 256, 8, 3
    s, st, (lo, di, up, stc, sh) = _op(n)
    sizes = O.balanced_sizes(n, 4)
    fld = np.random.default_rng(11).standard_normal((groups, n, sz))
    want = O.run_distd2(lo, di, up, False, fld, stc, sizes, shift=sh)
    with warnings.catch_warnings():
        warnings.simplefilter("ignore", T.NotDominantWarning)
        got = T.run_distd2(s, fld, part=T.SubdomainPartition(sizes), stencil=st,
                           arithmetic="strict", devices=[0] * 4)
    np.testing.assert_array_equal(got, want)


@pytest.mark.gpu
def test_gpu_open_d2_order_of_accuracy(gpu):
    errs = []
    ns = (64, 128, 256, 512)
    for n in ns:
        h, f, d2 = _smooth(n)
        s, st, _ = _op(n, h)
        got = T.apply_operator(s, st, f)
        errs.append(np.max(np.abs(got - d2)))
    slope = -np.polyfit(np.log(ns), np.log(errs), 1)[0]
    assert 2.8 <= slope <= 3.6, (slope, errs)


@pytest.mark.gpu
def test_gpu_bad_shift_rejected(gpu):
    n = 64
    s, st, _ = _op(n)
    bad = st.shift.copy()
    bad[5] = 1
    with pytest.raises(ValueError):
        T.run_distd2(s, np.zeros((1, n, 8)), stencil=T.StencilCoeffs(st.c, shift=bad))
    per = T.TridiagonalSystem(s.lower, s.diag, s.upper, periodic=True)
    with pytest.raises(ValueError):
        T.run_distd2(per, np.zeros((1, n, 8)), stencil=st)
