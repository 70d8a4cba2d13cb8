"""The benchmark CLI on the B200 (paper_2206_07244_b200/bench_cli.py) against the
reference's CLI contract (proj/tests/cli_exit_codes.cmake): stats-only, the CSV record
appended once per invocation under one header, --verify against the CPU check, and the
I/O exit code for a dimension mismatch."""
import os

import pytest

from paper_2206_07244_b200 import bench_cli

pytestmark = pytest.mark.gpu
DATA = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden", "mtx")


def test_stats_only_identity(capsys):
    assert bench_cli.main(["--matrix", os.path.join(DATA, "identity3.mtx"), "--stats-only"]) == 0
    assert capsys.readouterr().out.strip() == "identity3: 3, 3, 3, 3, 1.00"


def test_dimension_mismatch_is_io_error():
    argv = ["--matrix", os.path.join(DATA, "identity3.mtx"), "--b", os.path.join(DATA, "rect2x3.mtx"),
            "--stats-only"]
    assert bench_cli.main(argv) == 2


def test_csv_append_and_verify(tmp_path, capsys):
    csv = str(tmp_path / "cli.csv")
    assert bench_cli.main(["--random", "500,500,0.02", "--seed", "3", "--repeat", "2", "--csv", csv, "--verify"]) == 0
    assert "verify: PASS" in capsys.readouterr().out
    assert bench_cli.main(["--random", "600,600,0.02", "--seed", "4", "--repeat", "2", "--csv", csv]) == 0
    lines = open(csv).read().strip().split("\n")
    assert len(lines) == 3 and lines[0] == bench_cli.CSV_HEADER
    assert lines[1].startswith("random_500x500,500,") and len(lines[2].split(",")) == 14


def test_matrix_times_b(capsys):
    argv = ["--matrix", os.path.join(DATA, "sym3.mtx"), "--b", os.path.join(DATA, "sym3.mtx"), "--repeat", "1",
            "--verify"]
    assert bench_cli.main(argv) == 0
    assert "verify: PASS" in capsys.readouterr().out
