"""CPU-only checks of the native library: it loads, exports every symbol the
C header declares, and its host-side plan code (Alg. 5) is bit-identical to
the reference. No kernel is launched here."""

import os
import re
import warnings

import numpy as np
import pytest

import paper_2411_13532_b200 as T
from paper_2411_13532_b200 import _native as N

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
HEADER = os.path.join(ROOT, "include", "tds_b200.h")


def header_functions():
    text = open(HEADER).read()
    return sorted(set(re.findall(r"^\s*(?:const\s+char\*|int|long\s+long)\s+(tds_\w+)\s*\(",
                                 text, re.M)))


def test_library_exports_every_declared_symbol():
    lib = N.lib()
    declared = header_functions()
    assert len(declared) >= 18
    for name in declared:
        assert hasattr(lib, name), name
        assert name in N.SIGNATURES, f"{name} has no ctypes signature"
    assert set(N.SIGNATURES) == set(declared)
    assert lib.tds_abi_version() == N.ABI_VERSION == 2


def test_library_is_sm100a_build():
    so = N.library_path()
    blob = open(so, "rb").read()
    assert b"sm_100a" in blob


@pytest.mark.parametrize("tag", ["c32", "rd16", "open_r0", "open_r1", "per_r0"])
def test_native_preprocess_bitwise_vs_reference(golden, tag):
    s = T.TridiagonalSystem(golden[f"pre_{tag}_lower"], golden[f"pre_{tag}_diag"],
                            golden[f"pre_{tag}_upper"])
    with warnings.catch_warnings():
        warnings.simplefilter("ignore", T.NotDominantWarning)
        co = T.preprocess(s, "interior", False)
    for k in ("s_a", "s_c", "w", "f", "r"):
        np.testing.assert_array_equal(getattr(co, k), golden[f"pre_{tag}_{k}"], err_msg=k)
    assert [co.dropped_first, co.dropped_last] == list(golden[f"pre_{tag}_dropped"])


def test_preprocess_errors_match_reference():
    # reference tests/test_distributed.py:103-116
    a = np.array([0.0, 1.0, 0.0, 0.0, 0.0])
    c = np.array([1.0, 0.0, 0.0, 0.0, 0.0])
    s = T.TridiagonalSystem(a, np.ones(5), c)
    with warnings.catch_warnings():
        warnings.simplefilter("ignore", T.NotDominantWarning)
        with pytest.raises(T.SingularPivot):
            T.preprocess(s, "interior", cyclic=False)
    third = np.full(3, 1.0 / 3.0)
    with pytest.raises(ValueError):
        T.preprocess(T.TridiagonalSystem(third, np.ones(3), third), "interior", False)


def test_preprocess_warns_when_not_dominant():
    s = T.TridiagonalSystem(np.full(8, 0.6), np.ones(8), np.full(8, 0.6))
    with pytest.warns(T.NotDominantWarning):
        T.preprocess(s, "interior", cyclic=False)
    with warnings.catch_warnings():
        warnings.simplefilter("error")
        T.preprocess(s, "interior", cyclic=False, warn_not_dominant=False)


def test_identity_block_coefficients():
    # reference tests/test_distributed.py:52-59
    co = T.preprocess(T.TridiagonalSystem(np.zeros(8), np.ones(8), np.zeros(8)),
                      "interior", cyclic=False)
    np.testing.assert_array_equal(co.s_a, np.zeros(8))
    np.testing.assert_array_equal(co.s_c, np.zeros(8))
    np.testing.assert_array_equal(co.f, np.ones(8))
    np.testing.assert_array_equal(co.w, np.zeros(8))
    assert co.dropped_first == 0.0 and co.dropped_last == 0.0


def test_coupling_below_1e15_at_64_rows():
    # reference tests/test_distributed.py:89-92
    third = np.full(64, 1.0 / 3.0)
    co = T.preprocess(T.TridiagonalSystem(third, np.ones(64), third), "interior", False)
    assert abs(co.s_a[-2]) < 1e-15 and co.dropped_last < 1e-15


def test_plan_create_without_gpu_reports_cuda_error():
    import torch
    if torch.cuda.is_available():
        pytest.skip("a GPU is present")
    sys_, st = T.assemble(T.sixth_order_first_derivative(0.1), 64)
    with pytest.raises(RuntimeError):
        T.Plan.create(sys_, st.c, (64,))


def test_run_distd2_fails_loudly_without_gpu():
    import torch
    if torch.cuda.is_available():
        pytest.skip("a GPU is present")
    sys_, st = T.assemble(T.sixth_order_first_derivative(0.1), 64)
    with pytest.raises(RuntimeError):
        T.run_distd2(sys_, np.zeros((1, 64, 8)), stencil=st)
