"""Symbolic-only sizing (C ABI spgemm_forecast_nnz and
spgemm_forecast_nnz_multi): nnz(C) per row and in total, without computing or
allocating C. Counts must equal the oracle's C structure exactly (bit-exact
integer work), on every tier: thread/group/block symbolic bins, the spilled top
bin (k_big_sym) and rows with no products."""
import numpy as np
import pytest

from helpers import random_csr, spill_pair
from paper_2206_07244_b200 import synthetic as S

pytestmark = pytest.mark.gpu


def _oracle_counts(oracle, a, b):
    c = oracle.spgemm(a, b)
    return np.diff(np.asarray(c.rpt, np.int64)), int(oracle.compute_nprod(a, b)[1])


CASES = {
    "stencil27": lambda: (S.stencil3d_27pt(24),) * 2,
    "laplace2d": lambda: (S.poisson2d_5pt(64),) * 2,
    "random_rect": lambda: (random_csr(300, 500, 0.02, 1), random_csr(500, 200, 0.05, 2)),
    "rmat12": lambda: (S.random_values(S.rmat(12, 16, seed=5), 3),) * 2,
    "spill": lambda: spill_pair(21000, 4),
    "empty_rows": lambda: (random_csr(200, 200, 0.0, 3), random_csr(200, 200, 0.1, 4)),
}


@pytest.mark.parametrize("name", sorted(CASES))
def test_forecast_matches_oracle(sg, oracle, name):
    a, b = CASES[name]()
    want_rows, want_nprod = _oracle_counts(oracle, a, b)
    f = sg.forecast_nnz(a, b)
    assert f.total_nprod == want_nprod
    assert f.total_nnz == int(want_rows.sum())
    np.testing.assert_array_equal(f.row_nnz, want_rows)
    assert f.c_bytes == 8 * (a.rows + 1) + 12 * f.total_nnz
    # totals only, and device-resident operands
    g = sg.forecast_nnz(a.to_device(), b.to_device(), per_row=False)
    assert g.row_nnz is None and (g.total_nnz, g.total_nprod) == (f.total_nnz, f.total_nprod)


def test_forecast_agrees_with_multiply(sg):
    a = S.random_values(S.rmat(13, 16, seed=13), 7)
    out = sg.multiply(a, a)
    f = sg.forecast_nnz(a, a)
    assert f.total_nnz == out.stats.nnz_of_product
    np.testing.assert_array_equal(f.row_nnz, np.diff(out.c.rpt))
    assert f.cr == pytest.approx(out.stats.cr)


def test_forecast_product_larger_than_hbm(sg):
    """An outer product whose C (n^2 = 2.25e10 nonzeros, 270 GB) exceeds a B200's
    HBM: the forecast sizes it from O(n) inputs and O(n) metadata."""
    n = 150_000
    a = sg.CsrMatrix(n, 1, np.arange(n + 1, dtype=np.int64), np.zeros(n, np.int32), np.ones(n))
    b = sg.CsrMatrix(1, n, np.array([0, n], np.int64), np.arange(n, dtype=np.int32), np.ones(n))
    f = sg.forecast_nnz(a, b)
    assert f.total_nprod == n * n and f.total_nnz == n * n
    assert (f.row_nnz == n).all()
    assert f.c_bytes > 180 * 10**9


@pytest.mark.parametrize("parts", [1, 2, 3])
def test_forecast_multi(sg, parts):
    a = S.random_values(S.rmat(12, 16, seed=21), 2)
    f1 = sg.forecast_nnz(a, a)
    fm = sg.forecast_nnz_multi(a, a, devices=[0] * parts)
    assert (fm.total_nnz, fm.total_nprod) == (f1.total_nnz, f1.total_nprod)
    np.testing.assert_array_equal(fm.row_nnz, f1.row_nnz)
    assert fm.row_bounds[0] == 0 and fm.row_bounds[-1] == a.rows and len(fm.row_bounds) == parts + 1
    assert all(x <= y for x, y in zip(fm.row_bounds, fm.row_bounds[1:]))


def test_forecast_shape_mismatch(sg):
    a = random_csr(10, 20, 0.2, 1)
    with pytest.raises(sg.InvalidArgument):
        sg.forecast_nnz(a, a)
