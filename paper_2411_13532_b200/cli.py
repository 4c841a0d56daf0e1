"""Benchmark CLI with the reference's CSV schema (reference cli.py:33-62,
bench.py:40-44, 200-296), running the B200 kernels.

    python -m paper_2411_13532_b200.cli bench --solver distd2 --nx 512 --ny 512 --nz 512 \
        --sz 32 --ranks 1 --peak-gbps 6546.6 --out sweep.csv
    python -m paper_2411_13532_b200.cli scaling --nx 1024 --ny 64 --nz 64 --ranks 8
    python -m paper_2411_13532_b200.cli accuracy --ranks 4

Subcommands and columns follow the reference:
  bench     fixed-total-points sweep over n (sweep_sizes, bench.py:200-212)
            CSV: solver,n,sz,P,repeat,runtime_s,points,bytes_per_point,
                 achieved_gbps,pct_peak
  scaling   DistD2 over P = 1, 2, 4, ... emulated ranks at fixed n
            (run_scaling, bench.py:238-281), message rounds audited == 2
  accuracy  order-of-accuracy table (run_accuracy, bench.py:284-316)
Solvers: thomas, periodic_thomas (k_thomas, reference arithmetic) and
distd2 (k_tma fast path). The reference's pdd / modified_thomas
cross-validation solvers are out of scope and the
pde subcommand's movement ledger is not mirrored; both exit with code 2.

Differences, by design: fields live in HBM as (groups, n, sz) SZ-blocked
tensors for every solver; runtimes are wall-clock medians around the
device call with a CUDA synchronize on both sides (no host copies);
bytes_per_point is the reference's logical model (movement.py:54-71,
101-104, write-allocate on) so achieved_gbps is comparable with its
tables. No figure is rendered (matplotlib is out of scope).
Exit codes: 0 ok, 2 configuration error, 3 failed correctness check.
"""

import argparse
import csv
import ctypes
import sys
import time

import numpy as np

SOLVER_NAMES = ("thomas", "periodic_thomas", "pdd", "modified_thomas", "distd2")
CSV_COLUMNS = ("solver", "n", "sz", "P", "repeat", "runtime_s", "points",
               "bytes_per_point", "achieved_gbps", "pct_peak")
ACCURACY_COLUMNS = ("solver", "n", "h", "max_error", "slope", "diff_vs_serial")
EXIT_OK, EXIT_CONFIG, EXIT_CHECK = 0, 2, 3
MIN_REPEATS = 3
# logical field traversals (R + 2W + 2RW with write-allocate) x 8 B;
# reference movement.py:54-71
BYTES_PER_POINT = {"thomas": 40.0, "periodic_thomas": 56.0, "distd2": 56.0}


class ConfigError(ValueError):
    pass


def build_parser():
    parser = argparse.ArgumentParser(prog="tds-b200",
                                     description="B200 batched tridiagonal solver harness")
    sub = parser.add_subparsers(dest="subcommand", required=True)
    for name, descr in (("bench", "throughput sweep at fixed total points"),
                        ("scaling", "emulated-rank strong scaling at fixed global size"),
                        ("accuracy", "derivative order-of-accuracy table"),
                        ("pde", "transport-equation ledger run (not provided)")):
        p = sub.add_parser(name, help=descr)
        p.add_argument("--nx", type=int, default=256)
        p.add_argument("--ny", type=int, default=64)
        p.add_argument("--nz", type=int, default=64)
        p.add_argument("--sz", type=int, default=8)
        p.add_argument("--ranks", type=int, default=2)
        p.add_argument("--solver", choices=SOLVER_NAMES, default="thomas")
        p.add_argument("--repeats", type=int, default=3)
        p.add_argument("--seed", type=int, default=1234)
        p.add_argument("--peak-gbps", type=float, default=0.0)
        p.add_argument("--out", type=str, default="")
        p.add_argument("--cyclic", action="store_true")
        p.add_argument("--pad", action="store_true")
    return parser


def validate(a):
    """bench.py:62-82."""
    if a.repeats < MIN_REPEATS:
        raise ConfigError(f"repeats must be >= {MIN_REPEATS}")
    if min(a.nx, a.ny, a.nz) <= 0:
        raise ConfigError("grid extents must be positive")
    if a.sz <= 0 or a.ranks <= 0:
        raise ConfigError("sz and ranks must be positive")
    if a.solver in ("pdd", "modified_thomas"):
        raise ConfigError(f"solver {a.solver!r} is a cross-validation solver outside the "
                          "DistD2 path; not provided here")
    if a.solver == "thomas" and a.cyclic:
        raise ConfigError("the Thomas kernel handles open systems only")
    if a.solver == "periodic_thomas" and not a.cyclic:
        raise ConfigError("periodic_thomas needs --cyclic")
    if (a.ny * a.nz) % a.sz and not a.pad:
        raise ConfigError(f"sz={a.sz} does not divide {a.ny * a.nz} transverse lines; "
                          "enable --pad or adjust sz")


def make_dominant_system(n, seed, periodic, ratio=0.1):
    """bench.py:116-122 (same seeded construction)."""
    import paper_2411_13532_b200 as T
    rng = np.random.default_rng(seed)
    b = 2.0 + rng.random(n)
    a = ratio * (2.0 * rng.random(n) - 1.0)
    c = ratio * (2.0 * rng.random(n) - 1.0)
    return T.TridiagonalSystem(a, b, c, periodic=periodic)


def sweep_sizes(a):
    """bench.py:200-212."""
    total = a.nx * a.ny * a.nz
    sizes, n = [], 32
    while n <= min(8192, total):
        lanes = total // n
        if total % n == 0 and lanes % a.sz == 0 and n // a.ranks >= 4 and lanes > 0:
            sizes.append(n)
        n *= 2
    if not sizes:
        raise ConfigError("no valid sweep sizes; adjust extents/sz/ranks")
    return sizes


def _device_field(n, lanes, sz, seed):
    import torch
    g = torch.Generator(device="cuda")
    g.manual_seed(seed + 1)
    return torch.randn((lanes // sz, n, sz), dtype=torch.float64, device="cuda", generator=g)


def _solver_fn(a, sys, n):
    """fn(field) -> field on the device (bench.py:125-147)."""
    import torch
    import paper_2411_13532_b200 as T
    from paper_2411_13532_b200 import _native as N
    from paper_2411_13532_b200.distributed import _stream_handle
    if a.solver in ("thomas", "periodic_thomas"):
        lo, di, up = (N.f64(x) for x in (sys.lower, sys.diag, sys.upper))

        def thomas(f):
            out = torch.empty_like(f)
            N.check(N.lib().tds_thomas(N.dptr(lo), N.dptr(di), N.dptr(up), int(sys.periodic),
                                       ctypes.c_void_p(f.data_ptr()),
                                       ctypes.c_void_p(out.data_ptr()), n, f.shape[0],
                                       f.shape[2], T.distributed.PIVOT_FLOOR, _stream_handle()))
            return out
        return thomas
    part = T.SubdomainPartition.balanced(n, a.ranks)
    return lambda f: T.run_distd2(sys, f, part=part)


def _check(a, sys, f, got, n):
    """Cross-check against the serial solve (bench.py:158-182)."""
    import paper_2411_13532_b200 as T
    if a.solver != "distd2" or min(T.SubdomainPartition.balanced(n, a.ranks).local_sizes) < 16:
        return True, ""
    ref = T.run_distd2(sys, f, rank_count=1, arithmetic="strict")
    err = float((got - ref).abs().max() / ref.abs().max())
    if err > 1e-8:
        return False, f"{a.solver} off by {err:.3e} relative at n={n}"
    return True, ""


def _time(fn, f, repeats):
    import torch
    out = []
    for _ in range(repeats):
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        fn(f)
        torch.cuda.synchronize()
        out.append(time.perf_counter() - t0)
    return out


def _rows(a, solver, n, P, lanes, runtimes):
    bpp = BYTES_PER_POINT[solver]
    points = n * lanes
    rows = []
    for r, t in enumerate(runtimes):
        gbps = bpp * points / t / 1e9 if t > 0 else float("nan")
        pct = 100.0 * gbps / a.peak_gbps if a.peak_gbps > 0 else float("nan")
        rows.append([solver, n, a.sz, P, r, f"{t:.9f}", points, f"{bpp:.3f}", f"{gbps:.6f}",
                     f"{pct:.3f}"])
    return rows


def cmd_bench(a):
    validate(a)
    total = a.nx * a.ny * a.nz
    rows = []
    for n in sweep_sizes(a):
        lanes = total // n
        sys_ = make_dominant_system(n, a.seed + n, a.cyclic)
        f = _device_field(n, lanes, a.sz, a.seed + n)
        fn = _solver_fn(a, sys_, n)
        ok, msg = _check(a, sys_, f, fn(f), n)
        if not ok:
            print(msg, file=sys.stderr)
            return EXIT_CHECK
        rt = _time(fn, f, a.repeats)
        rows += _rows(a, a.solver, n, a.ranks, lanes, rt)
        print(f"n={n:6d} median {np.median(rt) * 1e3:9.3f} ms "
              f"({np.median(rt) / (n * lanes) * 1e9:8.4f} ns/point)")
    if a.out:
        _write(a.out, CSV_COLUMNS, rows)
    return EXIT_OK


def cmd_scaling(a):
    """bench.py:238-281: P = 1, 2, 4, ... <= ranks at n = nx."""
    import paper_2411_13532_b200 as T
    a.solver = "distd2"
    validate(a)
    n, lanes = a.nx, a.ny * a.nz
    sys_ = make_dominant_system(n, a.seed, a.cyclic)
    f = _device_field(n, lanes, a.sz, a.seed)
    rows, med, p = [], {}, 1
    while p <= a.ranks and n // p >= 4:
        part = T.SubdomainPartition.balanced(n, p)
        audit = {}
        T.run_distd2(sys_, f, part=part, audit=audit)
        if p > 1 and any(r != 2 for r in audit["rounds_per_rank"]):
            print(f"P={p}: message rounds {audit['rounds_per_rank']}, expected 2",
                  file=sys.stderr)
            return EXIT_CHECK
        rt = _time(lambda x: T.run_distd2(sys_, x, part=part), f, a.repeats)
        rows += _rows(a, "distd2", n, p, lanes, rt)
        med[p] = float(np.median(rt))
        p *= 2
    for p, t in med.items():
        print(f"P={p:3d} median {t * 1e3:9.3f} ms  efficiency {med[1] / t:6.3f}")
    if a.out:
        _write(a.out, CSV_COLUMNS, rows)
    return EXIT_OK


def cmd_accuracy(a):
    """bench.py:284-316: serial and distributed order of accuracy."""
    import paper_2411_13532_b200 as T
    validate(a)
    n_list = (32, 64, 128, 256)
    scheme = T.sixth_order_first_derivative(1.0)
    serial = T.order_of_accuracy(scheme, T.operator_applier(1), n_list)
    dist = T.order_of_accuracy(scheme, T.operator_applier(a.ranks), n_list)
    diffs = {}
    for n in n_list:
        h = 2 * np.pi / n
        s, st = T.assemble(T.sixth_order_first_derivative(h), n, periodic=True)
        fld = np.sin(h * np.arange(n)).reshape(1, n, 1)
        u1 = T.run_distd2(s, fld, stencil=st, rank_count=1)
        up = T.run_distd2(s, fld, stencil=st, part=T.SubdomainPartition.balanced(n, a.ranks))
        diffs[n] = float(np.max(np.abs(u1 - up)))
    rows = [["periodic_thomas", n, f"{2 * np.pi / n:.9e}", f"{e:.6e}", f"{serial.slope:.4f}",
             ""] for n, e in zip(serial.n_list, serial.errors)]
    rows += [["distd2", n, f"{2 * np.pi / n:.9e}", f"{e:.6e}", f"{dist.slope:.4f}",
              f"{diffs[n]:.6e}"] for n, e in zip(dist.n_list, dist.errors)]
    for r in rows:
        print(" ".join(str(x) for x in r))
    if a.out:
        _write(a.out, ACCURACY_COLUMNS, rows)
    return EXIT_OK if abs(serial.slope - 6.0) <= 0.2 else EXIT_CHECK


def _write(path, cols, rows):
    with open(path, "w", newline="") as fh:
        w = csv.writer(fh)
        w.writerow(cols)
        w.writerows(rows)


def main(argv=None):
    a = build_parser().parse_args(argv)
    try:
        if a.subcommand == "pde":
            raise ConfigError("the pde ledger run is not provided (DESIGN.md section 8); use "
                              "tools/bench_transport.py for the transport RHS")
        return {"bench": cmd_bench, "scaling": cmd_scaling, "accuracy": cmd_accuracy}[
            a.subcommand](a)
    except ConfigError as e:
        print(f"configuration error: {e}", file=sys.stderr)
        return EXIT_CONFIG


if __name__ == "__main__":
    sys.exit(main())
