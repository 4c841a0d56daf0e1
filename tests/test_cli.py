"""Bench CLI with the reference's CSV schema (reference cli.py:33-62,
bench.py:40-44): argument validation and exit codes on CPU, a small sweep on
the GPU."""

import csv

import numpy as np
import pytest

from paper_2411_13532_b200 import cli

# reference bench.py:40-44
REF_CSV_COLUMNS = ("solver", "n", "sz", "P", "repeat", "runtime_s", "points",
                   "bytes_per_point", "achieved_gbps", "pct_peak")
REF_ACCURACY_COLUMNS = ("solver", "n", "h", "max_error", "slope", "diff_vs_serial")


def test_schema_matches_reference():
    assert cli.CSV_COLUMNS == REF_CSV_COLUMNS
    assert cli.ACCURACY_COLUMNS == REF_ACCURACY_COLUMNS
    # movement.py:54-71 with write-allocate: (R + 2W + 2RW) x 8 B
    assert cli.BYTES_PER_POINT == {"thomas": 40.0, "periodic_thomas": 56.0, "distd2": 56.0}


@pytest.mark.parametrize("argv", [
    ["bench", "--repeats", "2"],
    ["bench", "--solver", "thomas", "--cyclic"],
    ["bench", "--solver", "periodic_thomas"],
    ["bench", "--solver", "pdd"],
    ["bench", "--sz", "7"],
    ["pde"],
])
def test_config_errors_exit_2(argv):
    assert cli.main(argv) == cli.EXIT_CONFIG


def test_sweep_sizes_follow_reference():
    a = cli.build_parser().parse_args(["bench", "--nx", "256", "--ny", "64", "--nz", "64",
                                       "--ranks", "2"])
    # bench.py:200-212: powers of two from 32 while total % n == 0 and
    # lanes % sz == 0 and n // ranks >= 4
    assert cli.sweep_sizes(a) == [32, 64, 128, 256, 512, 1024, 2048, 4096, 8192]


@pytest.mark.gpu
@pytest.mark.parametrize("solver,extra", [("distd2", ["--ranks", "2"]),
                                          ("thomas", []),
                                          ("periodic_thomas", ["--cyclic"])])
def test_bench_csv_on_gpu(tmp_path, solver, extra):
    torch = pytest.importorskip("torch")
    if not torch.cuda.is_available():
        pytest.skip("needs a CUDA device")
    out = tmp_path / "b.csv"
    rc = cli.main(["bench", "--solver", solver, "--nx", "64", "--ny", "32", "--nz", "32",
                   "--sz", "16", "--peak-gbps", "6546.6", "--out", str(out)] + extra)
    assert rc == cli.EXIT_OK
    rows = list(csv.reader(open(out)))
    assert tuple(rows[0]) == REF_CSV_COLUMNS
    assert len(rows) > 3 and all(float(r[5]) > 0 for r in rows[1:])
    assert {r[0] for r in rows[1:]} == {solver}


@pytest.mark.gpu
def test_scaling_and_accuracy_on_gpu(tmp_path):
    torch = pytest.importorskip("torch")
    if not torch.cuda.is_available():
        pytest.skip("needs a CUDA device")
    assert cli.main(["scaling", "--nx", "256", "--ny", "32", "--nz", "32", "--sz", "16",
                     "--ranks", "8", "--out", str(tmp_path / "s.csv")]) == cli.EXIT_OK
    rows = list(csv.reader(open(tmp_path / "s.csv")))
    assert sorted({int(r[3]) for r in rows[1:]}) == [1, 2, 4, 8]
    assert cli.main(["accuracy", "--ranks", "4", "--out", str(tmp_path / "a.csv")]) == cli.EXIT_OK
    rows = list(csv.reader(open(tmp_path / "a.csv")))
    assert tuple(rows[0]) == REF_ACCURACY_COLUMNS
    slope = float(rows[1][4])
    assert abs(slope - 6.0) <= 0.2 and np.isfinite(slope)
