"""Pin the CPU oracle: bit-for-bit against the reference's own outputs.

The fixtures come from running the reference package itself
(tests/golden/make_golden.py). Every oracle function must reproduce them
exactly -- the oracle keeps the reference's association order, so there is
no tolerance here.
"""

import numpy as np
import pytest

from conftest import golden_run
from oracle import tds_oracle as O


def test_assemble_matches_reference(golden):
    for tag, kind, n, per in (("d1p64", "d1", 64, True), ("d1o64", "d1", 64, False),
                              ("d2p32", "d2", 32, True)):
        lo, di, up, st = O.assemble(kind, n, 2 * np.pi / n, per)
        np.testing.assert_array_equal(lo, golden[f"asm_{tag}_lower"])
        np.testing.assert_array_equal(di, golden[f"asm_{tag}_diag"])
        np.testing.assert_array_equal(up, golden[f"asm_{tag}_upper"])
        np.testing.assert_array_equal(st, golden[f"asm_{tag}_stencil"])


@pytest.mark.parametrize("tag", ["c32", "rd16", "open_r0", "open_r1", "per_r0"])
def test_preprocess_bitwise(golden, tag):
    co = O.preprocess(golden[f"pre_{tag}_lower"], golden[f"pre_{tag}_diag"],
                      golden[f"pre_{tag}_upper"])
    for k in ("s_a", "s_c", "w", "f", "r"):
        np.testing.assert_array_equal(co[k], golden[f"pre_{tag}_{k}"], err_msg=k)
    np.testing.assert_array_equal(
        np.abs([co["dropped_first"], co["dropped_last"]]), golden[f"pre_{tag}_dropped"])


def test_decouple_substitute_pair_bitwise(golden):
    g = golden
    co = O.preprocess(g["dec_lower"], g["dec_diag"], g["dec_upper"])
    d = O.decouple_fused(g["dec_uext"], co, g["dec_stencil"])
    np.testing.assert_array_equal(d, g["dec_d"])
    # decouple_unfused on the reference's build_rhs (D12), and build_rhs itself
    np.testing.assert_array_equal(O.build_rhs(g["dec_uext"], g["dec_stencil"]), g["decu_rhs"])
    np.testing.assert_array_equal(O.decouple_unfused(g["decu_rhs"], co), g["decu_d"])
    np.testing.assert_array_equal(O.substitute(d, co, g["sub_us"], g["sub_ue"]),
                                  g["sub_out"])
    for row, want in zip(g["pair_in"], g["pair_out"]):
        got = O.solve_boundary_pair(row[0], row[1], row[2], row[3])
        assert got[0] == want[0] and got[1] == want[1]
    # reference tests/test_distributed.py:171-178 worked example
    ul, uf = O.solve_boundary_pair(1.0, 1.0, 0.1, 0.2)
    assert abs(ul - 0.918367346938775) < 1e-12 and abs(uf - 0.816326530612244) < 1e-12


def test_serial_solvers_bitwise(golden):
    g = golden
    np.testing.assert_array_equal(
        O.thomas_solve(g["thomas_lower"], g["thomas_diag"], g["thomas_upper"],
                       g["thomas_rhs"]), g["thomas_out"])
    np.testing.assert_array_equal(
        O.periodic_thomas_solve(g["pthomas_lower"], g["pthomas_diag"],
                                g["pthomas_upper"], g["thomas_rhs"]), g["pthomas_out"])


def test_run_distd2_bitwise_all_cases(golden):
    tags = [str(t) for t in golden["run_tags"]]
    assert len(tags) == 20
    for tag in tags:
        c = golden_run(golden, tag)
        got = O.run_distd2(c["lower"], c["diag"], c["upper"], c["periodic"],
                           c["field"], c["stencil"], c["sizes"])
        np.testing.assert_array_equal(got, c["out"], err_msg=tag)


def test_threaded_oracle_equals_serial(golden):
    c = golden_run(golden, "d1p512_P8")
    a = O.run_distd2(c["lower"], c["diag"], c["upper"], c["periodic"],
                     c["field"], c["stencil"], c["sizes"])
    b = O.run_distd2_threaded(c["lower"], c["diag"], c["upper"], c["periodic"],
                              c["field"], c["stencil"], c["sizes"], threads=2,
                              groups_per_task=1)
    np.testing.assert_array_equal(a, b)


def test_pack_matches_reference(golden):
    for d in "xyz":
        p = O.pack(golden["pack_cart"], 8, d)
        np.testing.assert_array_equal(p, golden[f"pack_{d}"])
        np.testing.assert_array_equal(O.unpack(p, (4, 6, 8), d), golden["pack_cart"])


def test_config1_64cubed_subsample(golden):
    n = 64
    lo, di, up, st = O.assemble("d1", n, 2 * np.pi / n, True)
    u = np.random.default_rng(1234).standard_normal((n, n, n))
    fld = O.pack(u, 8, "x")
    np.testing.assert_array_equal(fld[:16], golden["c1_field"])
    got = O.run_distd2(lo, di, up, True, fld[:16], st)
    np.testing.assert_array_equal(got, golden["c1_out"])
