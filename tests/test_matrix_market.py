"""CPU: Matrix Market ingestion (paper_2206_07244_b200/matrix_market.py) against the
reference's contract, case by case after proj/tests/test_matrix_market.cpp (line numbers
cited), plus the benchmark CLI's usage/IO exit codes (proj/tests/cli_exit_codes.cmake) for
the cases decided before the GPU is touched."""
import os

import numpy as np
import pytest

from paper_2206_07244_b200 import bench_cli
from paper_2206_07244_b200.matrix_market import ParseError, parse_matrix_market, read_matrix_market_csr

DATA = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden", "mtx")


def test_real_general_entry():  # :34-43
    coo = parse_matrix_market("%%MatrixMarket matrix coordinate real general\n2 2 1\n1 2 3.5\n")
    assert (coo.rows, coo.cols, len(coo)) == (2, 2, 1)
    assert (coo.row[0], coo.col[0], coo.value[0]) == (0, 1, 3.5)


def test_symmetric_mirror():  # :45-55
    coo = parse_matrix_market("%%MatrixMarket matrix coordinate real symmetric\n2 2 1\n2 1 -4.0\n")
    assert len(coo) == 2
    assert list(coo.row) == [1, 0] and list(coo.col) == [0, 1] and list(coo.value) == [-4.0, -4.0]


def test_symmetric_diagonal_not_duplicated():  # :57-61
    coo = parse_matrix_market("%%MatrixMarket matrix coordinate real symmetric\n2 2 2\n1 1 1.0\n2 1 2.0\n")
    assert len(coo) == 3


def test_pattern_and_integer():  # :63-76
    coo = parse_matrix_market("%%MatrixMarket matrix coordinate pattern general\n3 3 2\n1 3\n2 1\n")
    assert list(coo.value) == [1.0, 1.0]
    coo = parse_matrix_market("%%MatrixMarket matrix coordinate integer general\n1 1 1\n1 1 -7\n")
    assert coo.value[0] == -7.0


def test_comments_blank_lines_scientific():  # :78-89
    coo = parse_matrix_market("%%MatrixMarket matrix coordinate real general\n% a comment\n\n2 2 2\n"
                              "% another\n1 1 1e-3\n2 2 -2.5E+2\n")
    assert len(coo) == 2 and coo.value[0] == pytest.approx(1e-3) and coo.value[1] == pytest.approx(-250.0)


def test_banner_case_insensitive():  # :91-94
    parse_matrix_market("%%MatrixMarket MATRIX Coordinate REAL General\n1 1 1\n1 1 2.0\n")


@pytest.mark.parametrize("text", [
    "",
    "%%NotMatrixMarket x\n1 1 0\n",
    "%%MatrixMarket matrix array real general\n1 1\n1.0\n",
    "%%MatrixMarket matrix coordinate complex general\n1 1 1\n1 1 1 0\n",
    "%%MatrixMarket matrix coordinate real hermitian\n1 1 1\n1 1 1\n",
    "%%MatrixMarket matrix coordinate real general\n2 2 2\n1 1 1.0\n",
    "%%MatrixMarket matrix coordinate real general\n2 2 1\n1 1 1.0\n2 2 1.0\n",
    "%%MatrixMarket matrix coordinate real general\n2 2 1\n3 1 1.0\n",
    "%%MatrixMarket matrix coordinate real general\n2 2 1\n0 1 1.0\n",
    "%%MatrixMarket matrix coordinate real symmetric\n2 2 1\n1 2 1.0\n",
    "%%MatrixMarket matrix coordinate real general\n1 1 1\n1 1 abc\n",
])
def test_malformed_inputs_raise(text):  # :96-125
    with pytest.raises(ParseError):
        parse_matrix_market(text)


def test_error_line_numbers():
    with pytest.raises(ParseError) as e:
        parse_matrix_market("%%MatrixMarket matrix coordinate real general\n% c\n2 2 2\n1 1 1.0\n3 1 1.0\n")
    assert e.value.line == 5


def test_symmetric_expansion_is_structurally_symmetric():  # :127-150
    from paper_2206_07244_b200.synthetic import transpose
    rng = np.random.default_rng(99)
    for _ in range(20):
        n = int(rng.integers(1, 31))
        lines = []
        for _ in range(n):
            i = int(rng.integers(1, n + 1))
            j = int(rng.integers(1, i + 1))
            lines.append(f"{i} {j} {rng.uniform(-1, 1)!r}")
        text = "%%MatrixMarket matrix coordinate real symmetric\n" + f"{n} {n} {n}\n" + "\n".join(lines) + "\n"
        from paper_2206_07244_b200.synthetic import csr_from_coo
        coo = parse_matrix_market(text)
        a = csr_from_coo(coo.rows, coo.cols, coo.row, coo.col, coo.value)
        t = transpose(a)
        assert np.array_equal(a.rpt, t.rpt) and np.array_equal(a.col, t.col)


def test_missing_file():  # :152-154
    with pytest.raises(ParseError):
        read_matrix_market_csr("/nonexistent/file.mtx")


def test_files_to_csr():
    a = read_matrix_market_csr(os.path.join(DATA, "sym3.mtx"))
    assert a.rows == 3 and list(a.rpt) == [0, 2, 4, 6] and list(a.col) == [0, 1, 0, 2, 1, 2]
    assert list(a.val) == [2.0, -1.0, -1.0, 0.5, 0.5, 4.0]


@pytest.mark.parametrize("argv,code", [
    (["--help"], 0),
    (["--no-such-flag"], 1),
    (["--stats-only"], 1),
    (["--matrix", os.path.join(DATA, "identity3.mtx"), "--random", "3,3,0.5", "--stats-only"], 1),
    (["--matrix", os.path.join(DATA, "identity3.mtx"), "--sym-range", "9x"], 1),
    (["--random", "3,3,1.5"], 1),
    (["--matrix", os.path.join(DATA, "does_not_exist.mtx"), "--stats-only"], 2),
    (["--matrix", os.path.join(DATA, "bad_header.mtx"), "--stats-only"], 2),
])
def test_cli_exit_codes_before_the_gpu(argv, code, capsys):  # cli_exit_codes.cmake
    assert bench_cli.main(argv) == code


def test_cli_csv_schema():
    assert bench_cli.CSV_HEADER.split(",") == ["name", "rows", "nnz_a", "nprod", "nnz_c", "cr", "t_setup",
                                               "t_symbin", "t_sym", "t_rpt", "t_numbin", "t_num", "t_total",
                                               "gflops"]
    r = bench_cli.BenchReport(name="m", rows=3, nnz_a=3, nprod=3, nnz_c=3, cr=1.0, mean_total=0.5, gflops=1e-8)
    assert len(bench_cli.csv_row(r).split(",")) == 14


def test_cpu_product_matches_oracle():
    from oracle import oracle as O
    a = bench_cli.random_csr(60, 50, 0.1, 3)
    b = bench_cli.random_csr(50, 40, 0.1, 4)
    c = bench_cli.cpu_product(a, b)
    exp = O.spgemm(a, b)
    assert O.same_pattern(c, exp) and O.max_relative_error(c, exp) <= 1e-12
