"""Host-side logic that needs no GPU: value types, partitions, operator
assembly, layout descriptors and index maps -- each against the reference's
golden output or its documented behaviour."""

import numpy as np
import pytest

import paper_2411_13532_b200 as T
from oracle import tds_oracle as O


def test_assemble_bitwise_vs_reference(golden):
    cases = (("d1p64", T.sixth_order_first_derivative, 64, True),
             ("d1o64", T.sixth_order_first_derivative, 64, False),
             ("d2p32", T.second_derivative_scheme, 32, True))
    for tag, scheme, n, per in cases:
        s, st = T.assemble(scheme(2 * np.pi / n), n, periodic=per)
        np.testing.assert_array_equal(s.lower, golden[f"asm_{tag}_lower"])
        np.testing.assert_array_equal(s.diag, golden[f"asm_{tag}_diag"])
        np.testing.assert_array_equal(s.upper, golden[f"asm_{tag}_upper"])
        np.testing.assert_array_equal(st.c, golden[f"asm_{tag}_stencil"])


def test_scheme_weights():
    # reference tests/test_compact.py:28-46
    w1 = T.sixth_order_first_derivative(1.0).interior_weights()
    np.testing.assert_allclose(w1, [-1 / 36, -7 / 9, 0, 7 / 9, 1 / 36], rtol=1e-15)
    w2 = T.second_derivative_scheme(1.0).interior_weights()
    np.testing.assert_allclose(w2, [3 / 44, 12 / 11, -51 / 22, 12 / 11, 3 / 44], rtol=1e-15)


def test_open_second_derivative_not_implemented():
    with pytest.raises(NotImplementedError):
        T.assemble(T.second_derivative_scheme(0.1), 32, periodic=False)
    with pytest.raises(ValueError):
        T.assemble(T.sixth_order_first_derivative(0.1), 7)


def test_partition_balanced_and_offsets():
    p = T.SubdomainPartition.balanced(50, 3)
    assert p.local_sizes == O.balanced_sizes(50, 3) == (17, 17, 16)
    assert p.offsets() == (0, 17, 34)
    with pytest.raises(ValueError):
        T.SubdomainPartition((3, 8))
    with pytest.raises(ValueError):
        T.SubdomainPartition.balanced(10, 0)


def test_system_validation():
    with pytest.raises(ValueError):
        T.TridiagonalSystem(np.zeros(4), np.array([1.0, 0.0, 1.0, 1.0]), np.zeros(4))
    with pytest.raises(ValueError):
        T.TridiagonalSystem(np.zeros(2), np.ones(2), np.zeros(2))
    with pytest.raises(ValueError):
        T.TridiagonalSystem(np.zeros(4), np.ones(4), np.array([0, np.nan, 0, 0]))
    s = T.TridiagonalSystem(np.full(5, 0.2), np.ones(5), np.full(5, 0.3), periodic=False)
    assert s.effective_lower()[0] == 0.0 and s.effective_upper()[-1] == 0.0
    assert T.dominance_margin(s) == pytest.approx(0.5)


def test_local_slice_matches_reference_semantics():
    # reference tests/test_distributed.py:342-361
    r = np.random.default_rng(7)
    s = T.TridiagonalSystem(0.3 * r.random(20), 2 + r.random(20), 0.3 * r.random(20),
                            periodic=True)
    part = T.SubdomainPartition((6, 8, 6))
    mids = [T.local_slice(s, part, k) for k in range(3)]
    np.testing.assert_array_equal(np.concatenate([m.diag for m in mids]), s.diag)
    assert mids[0].upper[-1] == s.upper[5]
    assert mids[1].lower[0] == s.lower[6]
    assert mids[0].lower[0] == s.lower[0]
    assert mids[2].upper[-1] == s.upper[-1]
    assert T.rank_position(0, 4) == "first" and T.rank_position(3, 4) == "last"
    assert T.rank_position(2, 4) == "interior"


def test_layout_descriptor_and_index_map():
    lay = T.LayoutDescriptor(4, 6, 8, 8, "y")
    assert (lay.n, lay.lines, lay.n_groups) == (6, 32, 4)
    with pytest.raises(T.DivisibilityError):
        T.LayoutDescriptor(4, 6, 6, 8, "x")
    padded = T.LayoutDescriptor(4, 6, 6, 8, "x", pad=True)
    assert padded.padded_lines == 40 and padded.n_groups == 5
    with pytest.raises(T.OutOfBounds):
        T.cartesian_to_packed(lay, 4, 0, 0)
    # index map agrees with the oracle's pack (which is pinned to the reference)
    cart = np.arange(4 * 6 * 8, dtype=np.float64).reshape(4, 6, 8)
    for d in "xyz":
        lay = T.LayoutDescriptor(4, 6, 8, 8, d)
        flat = O.pack(cart, 8, d).reshape(-1)
        for (i, j, k) in [(0, 0, 0), (3, 5, 7), (1, 2, 3), (2, 4, 6)]:
            assert flat[T.packed_linear_index(lay, i, j, k)] == cart[i, j, k]
