"""Generate the golden fixtures by running the REFERENCE package itself.

Run in the build container (the only place /root/reference exists):

    PYTHONDONTWRITEBYTECODE=1 python tests/golden/make_golden.py

It imports `tds` from /root/reference/pkg/src (read-only, pure NumPy) and
writes `tests/golden/golden.npz`: inputs and the reference's outputs for every
function on the DistD2 path. Nothing on the GPU box reads /root/reference;
the tests there read only this committed .npz.
"""

import os
import sys
import warnings

import numpy as np

REF_SRC = "/root/reference/pkg/src"
HERE = os.path.dirname(os.path.abspath(__file__))
OUT = os.path.join(HERE, "golden.npz")


def main():
    sys.dont_write_bytecode = True
    sys.path.insert(0, REF_SRC)
    import tds  # noqa: F401  (the reference)
    from tds.compact import (assemble, second_derivative_scheme,
                             sixth_order_first_derivative)
    from tds.distributed import (BoundaryPair, StencilCoeffs, build_rhs, decouple_fused,
                                 decouple_unfused, local_slice, preprocess, run_distd2,
                                 solve_boundary_pair, substitute)
    from tds.layout import LayoutDescriptor, pack
    from tds.serial import periodic_thomas_solve, thomas_solve
    from tds.system import RhsBatch, SubdomainPartition, TridiagonalSystem

    warnings.simplefilter("ignore")
    out = {"numpy_version": np.array(np.__version__)}

    def random_dominant(n, seed, periodic=False, ratio=0.3):
        # tests/conftest.py:7-13 of the reference
        rng = np.random.default_rng(seed)
        b = 2.0 + rng.random(n)
        a = ratio * (2.0 * rng.random(n) - 1.0)
        c = ratio * (2.0 * rng.random(n) - 1.0)
        return TridiagonalSystem(a, b, c, periodic=periodic)

    # ---- assemble ---------------------------------------------------------
    for tag, scheme, n, per in (("d1p64", sixth_order_first_derivative, 64, True),
                                ("d1o64", sixth_order_first_derivative, 64, False),
                                ("d2p32", second_derivative_scheme, 32, True)):
        sysm, st = assemble(scheme(2 * np.pi / n), n, periodic=per)
        out[f"asm_{tag}_lower"] = sysm.lower
        out[f"asm_{tag}_diag"] = sysm.diag
        out[f"asm_{tag}_upper"] = sysm.upper
        out[f"asm_{tag}_stencil"] = st.c

    # ---- preprocess -------------------------------------------------------
    pre_cases = []
    third = np.full(32, 1.0 / 3.0)
    pre_cases.append(("c32", TridiagonalSystem(third, np.ones(32), third, False)))
    pre_cases.append(("rd16", random_dominant(16, 5)))
    s_open, _ = assemble(sixth_order_first_derivative(0.1), 64, periodic=False)
    part = SubdomainPartition.balanced(64, 2)
    pre_cases.append(("open_r0", local_slice(s_open, part, 0)))
    pre_cases.append(("open_r1", local_slice(s_open, part, 1)))
    s_per = random_dominant(20, 7, periodic=True)
    pre_cases.append(("per_r0", local_slice(s_per, SubdomainPartition((6, 8, 6)), 0)))
    for tag, s in pre_cases:
        co = preprocess(s, "interior", cyclic=False)
        out[f"pre_{tag}_lower"] = s.lower
        out[f"pre_{tag}_diag"] = s.diag
        out[f"pre_{tag}_upper"] = s.upper
        for k in ("s_a", "s_c", "w", "f", "r"):
            out[f"pre_{tag}_{k}"] = getattr(co, k)
        out[f"pre_{tag}_dropped"] = np.array([co.dropped_first, co.dropped_last])

    # ---- decouple_fused / substitute / pair -------------------------------
    rng = np.random.default_rng(20260814)
    s = random_dominant(16, 5)
    co = preprocess(s, "interior", False)
    st = rng.standard_normal((16, 5))
    u_ext = rng.standard_normal((20, 4))
    d = decouple_fused(u_ext, co, StencilCoeffs(st))
    out.update(dec_lower=s.lower, dec_diag=s.diag, dec_upper=s.upper,
               dec_stencil=st, dec_uext=u_ext, dec_d=d)
    # decouple_unfused on the reference's own build_rhs (distributed.py:
    # 227-254; D12: bit-equal to decouple_fused). No new random draws, so
    # every other fixture is unchanged.
    rhs_built = build_rhs(u_ext, StencilCoeffs(st))
    out.update(decu_rhs=rhs_built, decu_d=decouple_unfused(rhs_built, co))
    u_s = rng.standard_normal(4)
    u_e = rng.standard_normal(4)
    out.update(sub_us=u_s, sub_ue=u_e, sub_out=substitute(d, co, u_s, u_e))
    pin = rng.standard_normal((64, 4))
    pin[:, 2:] *= 0.4
    pin[0] = [1.0, 1.0, 0.1, 0.2]          # tests/test_distributed.py:171-178
    res = [solve_boundary_pair(BoundaryPair(np.array([r[0]]), np.array([r[1]]),
                                            r[2], r[3])) for r in pin]
    out.update(pair_in=pin, pair_out=np.array([[a[0], b[0]] for a, b in res]))

    # ---- serial solvers ---------------------------------------------------
    s_open = random_dominant(48, 3)
    s_cyc = random_dominant(48, 4, periodic=True, ratio=0.25)
    rhs = rng.standard_normal((6, 48))
    out.update(thomas_lower=s_open.lower, thomas_diag=s_open.diag,
               thomas_upper=s_open.upper, thomas_rhs=rhs,
               thomas_out=thomas_solve(s_open, RhsBatch(rhs)).values,
               pthomas_lower=s_cyc.lower, pthomas_diag=s_cyc.diag,
               pthomas_upper=s_cyc.upper,
               pthomas_out=periodic_thomas_solve(s_cyc, RhsBatch(rhs)).values)

    # ---- run_distd2 end to end --------------------------------------------
    runs = []

    def add_run(tag, sysm, stencil, field, sizes):
        part = SubdomainPartition(tuple(sizes))
        res = run_distd2(sysm, field, part=part,
                         stencil=None if stencil is None else StencilCoeffs(stencil))
        out[f"run_{tag}_lower"] = sysm.lower
        out[f"run_{tag}_diag"] = sysm.diag
        out[f"run_{tag}_upper"] = sysm.upper
        out[f"run_{tag}_periodic"] = np.array(sysm.periodic)
        out[f"run_{tag}_stencil"] = (np.zeros((0, 5)) if stencil is None else stencil)
        out[f"run_{tag}_field"] = field
        out[f"run_{tag}_sizes"] = np.array(sizes)
        out[f"run_{tag}_out"] = res
        runs.append(tag)

    def compact(kind, n, periodic):
        scheme = sixth_order_first_derivative if kind == 1 else second_derivative_scheme
        sysm, st = assemble(scheme(2 * np.pi / n), n, periodic=periodic)
        return sysm, st.c

    f = rng.standard_normal((4, 64, 8))
    for per in (True, False):
        sysm, st = compact(1, 64, per)
        for p in (1, 2):
            add_run(f"d1{'p' if per else 'o'}64_P{p}", sysm, st, f,
                    SubdomainPartition.balanced(64, p).local_sizes)
    sysm, st = compact(2, 64, True)
    for p in (1, 2):
        add_run(f"d2p64_P{p}", sysm, st, f, SubdomainPartition.balanced(64, p).local_sizes)
    f96 = rng.standard_normal((3, 96, 4))
    s96 = random_dominant(96, 23, periodic=True, ratio=0.25)
    st96 = rng.standard_normal((96, 5))
    for p in (1, 3):
        add_run(f"rd96_P{p}", s96, st96, f96, SubdomainPartition.balanced(96, p).local_sizes)
    f128 = rng.standard_normal((2, 128, 16))
    s128 = random_dominant(128, 29, ratio=0.3)
    for p in (1, 2, 4):
        add_run(f"rd128_P{p}", s128, None, f128,
                SubdomainPartition.balanced(128, p).local_sizes)
    s20 = random_dominant(20, 7, periodic=True)
    add_run("rd20_P3", s20, rng.standard_normal((20, 5)),
            rng.standard_normal((2, 20, 8)), (6, 8, 6))
    s50 = random_dominant(50, 11, periodic=False, ratio=0.2)
    add_run("rd50_P3", s50, None, rng.standard_normal((1, 50, 8)),
            SubdomainPartition.balanced(50, 3).local_sizes)
    f512 = rng.standard_normal((2, 512, 32))
    for per in (True, False):
        sysm, st = compact(1, 512, per)
        for p in (1, 8):
            add_run(f"d1{'p' if per else 'o'}512_P{p}", sysm, st, f512,
                    SubdomainPartition.balanced(512, p).local_sizes)
    f1024 = rng.standard_normal((1, 1024, 32))
    sysm, st = compact(1, 1024, True)
    for p in (1, 2, 8):
        add_run(f"d1p1024_P{p}", sysm, st, f1024,
                SubdomainPartition.balanced(1024, p).local_sizes)
    out["run_tags"] = np.array(runs)

    # ---- layout -----------------------------------------------------------
    cart = rng.standard_normal((4, 6, 8))
    for dname in "xyz":
        lay = LayoutDescriptor(4, 6, 8, 8, dname)
        out[f"pack_{dname}"] = pack(cart, lay).data
    out["pack_cart"] = cart

    # ---- BASELINE config 1: 64^3 periodic d/dx, x, P=1 (subsampled groups) --
    n = 64
    u = np.random.default_rng(1234).standard_normal((n, n, n))
    fld = pack(u, LayoutDescriptor(n, n, n, 8, "x")).data
    sysm, st = compact(1, n, True)
    sub = fld[:16]
    out.update(c1_field=sub, c1_out=run_distd2(sysm, sub, stencil=StencilCoeffs(st)),
               c1_full_sum=np.array(run_distd2(sysm, fld, stencil=StencilCoeffs(st)).sum()))

    # ---- momentum transport RHS (momentum.py:142-169) ----------------------
    from tds.momentum import VelocityField, evaluate_transport_rhs
    from tds.layout import unpack as ref_unpack
    n = 16
    x = 2 * np.pi * np.arange(n) / n
    X, Y, Z = np.meshgrid(x, x, x, indexing="ij")
    u3 = np.sin(X) * np.cos(Y) + 0.3 * np.cos(Z) + 0.01 * rng.standard_normal((n, n, n))
    v3 = np.cos(X) * np.sin(Z) - 0.2 * np.sin(Y)
    w3 = np.sin(Y) * np.cos(Z) + 0.1 * np.cos(X)
    out.update(tr_u=u3, tr_v=v3, tr_w=w3)
    for tag, nu in (("nu", 0.1), ("inviscid", 0.0)):
        f = VelocityField.from_arrays(u3, v3, w3, nu, 2 * np.pi / n, sz=4)
        rhs = evaluate_transport_rhs(f)
        out[f"tr_{tag}_rhs"] = np.stack([ref_unpack(r) for r in rhs])

    np.savez_compressed(OUT, **out)
    print(f"wrote {OUT}: {len(out)} arrays, {len(runs)} run_distd2 cases")


if __name__ == "__main__":
    main()
