"""Shared test inputs (numpy generators; seeds fixed) and comparison helpers."""
from __future__ import annotations

import numpy as np

from paper_2206_07244_b200.api import CsrMatrix
from paper_2206_07244_b200.synthetic import csr_from_coo


def random_csr(rows: int, cols: int, density: float, seed: int) -> CsrMatrix:
    """Uniform random pattern (per-row binomial count of distinct columns), values U[-1,1)."""
    rng = np.random.default_rng(seed)
    rpt = np.zeros(rows + 1, np.int64)
    cols_list, vals_list = [], []
    counts = rng.binomial(cols, density, size=rows) if cols > 0 else np.zeros(rows, np.int64)
    for i in range(rows):
        k = int(counts[i])
        if k:
            c = np.sort(rng.choice(cols, size=k, replace=False))
            cols_list.append(c)
            vals_list.append(rng.uniform(-1.0, 1.0, size=k))
        rpt[i + 1] = rpt[i] + k
    col = np.concatenate(cols_list).astype(np.int32) if cols_list else np.zeros(0, np.int32)
    val = np.concatenate(vals_list) if vals_list else np.zeros(0)
    return CsrMatrix(rows, cols, rpt, col, val)


def random_csr_fixed(rows: int, cols: int, per_row: int, seed: int) -> CsrMatrix:
    """Exactly per_row distinct random columns in every row (vectorised)."""
    rng = np.random.default_rng(seed)
    per_row = min(per_row, cols)
    out = np.empty((rows, per_row), np.int64)
    todo = np.arange(rows)
    while todo.size:
        cand = np.sort(rng.integers(0, cols, size=(todo.size, per_row + 4)), axis=1)
        dup = np.zeros(cand.shape, bool)
        dup[:, 1:] = cand[:, 1:] == cand[:, :-1]
        nuniq = (~dup).sum(1)
        ok = nuniq >= per_row
        good = todo[ok]
        if good.size:
            c = cand[ok]
            d = dup[ok]
            key = np.where(d, np.iinfo(np.int64).max, c)
            key.sort(axis=1)
            out[good] = key[:, :per_row]
        todo = todo[~ok]
    rpt = np.arange(rows + 1, dtype=np.int64) * per_row
    return CsrMatrix(rows, cols, rpt, out.reshape(-1).astype(np.int32), rng.uniform(-1, 1, rows * per_row))


def spill_pair(distinct: int, rows_in_b: int):
    """test_pipeline.cpp:29-43: row 0 of A covers `distinct` columns via `rows_in_b` B rows."""
    per_row = distinct // rows_in_b
    dim = max(distinct, rows_in_b) + 1
    ar = np.zeros(rows_in_b, np.int64)
    ac = np.arange(rows_in_b, dtype=np.int64)
    a = csr_from_coo(dim, dim, ar, ac, np.ones(rows_in_b))
    k = np.repeat(np.arange(rows_in_b, dtype=np.int64), per_row)
    j = np.tile(np.arange(per_row, dtype=np.int64), rows_in_b)
    b = csr_from_coo(dim, dim, k, k * per_row + j, 0.5 + j)
    return a, b


def bitwise_equal(x: CsrMatrix, y) -> bool:
    x = x.to_host()
    return (x.rows == y.rows and x.cols == y.cols and np.array_equal(x.rpt, y.rpt)
            and np.array_equal(x.col, y.col)
            and np.array_equal(np.asarray(x.val).view(np.int64), np.asarray(y.val).view(np.int64)))


def assert_matches_oracle(out_c: CsrMatrix, expected, tol: float = 1e-12, bitwise=True):
    """Structure bit-exact; values within tol and, with the default
    deterministic=True options, bitwise equal to the reference's summation order
    on every row. bitwise=False for deterministic=False runs (heap-tier rows may
    accumulate with fp64 atomics: 1e-12 only)."""
    from oracle import oracle as O
    c = out_c.to_host()
    assert c.rows == expected.rows and c.cols == expected.cols
    assert np.array_equal(c.rpt, expected.rpt), "row pointers differ"
    assert np.array_equal(c.col, expected.col), "column indices differ"
    assert O.max_relative_error(c, expected) <= tol
    if bitwise is False:
        return
    got = np.asarray(c.val).view(np.int64)
    exp = np.asarray(expected.val).view(np.int64)
    assert np.array_equal(got, exp), "values differ bitwise from the reference's summation order"
