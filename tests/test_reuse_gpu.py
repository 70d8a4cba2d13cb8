"""GPU parity of the structure-reuse route and of the
thread-per-row kernels on the short-row stencils next to it. Reuse: rows whose
structure is their predecessor's shifted by one take its output positions
instead of hashing and sorting -- checked bitwise against the oracle on 3-D
stencils of awkward sizes (chains broken at every grid boundary, runs that end
mid-piece) and with random entries dropped (chains broken at random rows),
asserting that the route ran (per-launch profile names). Short rows (2-D
stencils, tridiagonal, random patterns, values that fold to -0.0) run the
thread-per-row bins; the same bitwise check.
"""
import numpy as np
import pytest

from helpers import assert_matches_oracle, random_csr_fixed
from paper_2206_07244_b200 import synthetic as S
from paper_2206_07244_b200.api import CsrMatrix

pytestmark = pytest.mark.gpu


def _drop(m: CsrMatrix, frac: float, seed: int) -> CsrMatrix:
    """Remove a random fraction of the off-diagonal entries."""
    rng = np.random.default_rng(seed)
    rows = np.repeat(np.arange(m.rows, dtype=np.int64), np.diff(m.rpt))
    col = m.col.astype(np.int64)
    keep = (rows == col) | (rng.random(col.size) >= frac)
    return S.csr_from_coo(m.rows, m.cols, rows[keep], col[keep], m.val[keep])


def _run(sg, oracle, a, b, kernel):
    ctx = sg.get_context()
    ctx.set_profiling(True)
    try:
        ctx.profile_summary()
        out = sg.multiply(a, b)
        names = ctx.profile_summary()
    finally:
        ctx.set_profiling(False)
    assert_matches_oracle(out.c, oracle.spgemm(a, b))
    ran = [k for k in names if k.split("#")[0].split("<")[0] == kernel]
    assert ran, f"{kernel} did not run: {sorted(names)}"
    return out


@pytest.mark.parametrize("n", [2, 3, 31, 33, 64, 100, 257, 700])
def test_short_rows_poisson2d(sg, oracle, n):
    a = S.random_values(S.poisson2d_5pt(n), n)
    _run(sg, oracle, a, a, "k_num_thread")


@pytest.mark.parametrize("n", [5, 1000, 40001])
def test_short_rows_tridiagonal(sg, oracle, n):
    offs = [(0,), (1,), (-1,)]
    a = S.random_values(S._stencil((n,), offs, 2.0, -1.0), 11)
    _run(sg, oracle, a, a, "k_num_thread")


@pytest.mark.parametrize("frac,seed", [(0.001, 1), (0.02, 2), (0.3, 3)])
def test_short_rows_broken_chains(sg, oracle, frac, seed):
    a = S.random_values(_drop(S.poisson2d_5pt(300), frac, seed), seed)
    _run(sg, oracle, a, a, "k_num_thread")


def test_short_rows_all_heads(sg, oracle):
    a = random_csr_fixed(50000, 50000, 3, 9)
    _run(sg, oracle, a, a, "k_num_thread")


def test_short_rows_signed_zeros(sg, oracle):
    # products of +-0.0 and values that cancel exactly: the first product of a
    # position is folded as 0.0 + x (so -0.0 becomes +0.0), as the reference does
    a = S.poisson2d_5pt(80)
    rng = np.random.default_rng(5)
    v = rng.choice(np.array([-0.0, 0.0, 1.0, -1.0, 0.5]), size=a.val.size)
    a = CsrMatrix(a.rows, a.cols, a.rpt, a.col, v)
    _run(sg, oracle, a, a, "k_num_thread")


@pytest.mark.parametrize("n", [5, 9, 17, 40])
def test_wide_route_stencils(sg, oracle, n):
    a = S.random_values(S.stencil3d_27pt(n), n)
    _run(sg, oracle, a, a, "k_num_reuse_multi")


@pytest.mark.parametrize("frac,seed", [(0.001, 4), (0.05, 5)])
def test_wide_route_broken_chains(sg, oracle, frac, seed):
    a = S.random_values(_drop(S.stencil3d_27pt(30), frac, seed), seed)
    _run(sg, oracle, a, a, "k_num_reuse_multi")


def test_wide_route_signed_zeros(sg, oracle):
    a = S.stencil3d_27pt(12)
    rng = np.random.default_rng(6)
    v = rng.choice(np.array([-0.0, 0.0, 1.0, -1.0, 0.5]), size=a.val.size)
    _run(sg, oracle, CsrMatrix(a.rows, a.cols, a.rpt, a.col, v), CsrMatrix(a.rows, a.cols, a.rpt, a.col, v), "k_num_reuse_multi")


def test_routes_off_matches(sg, oracle, monkeypatch):
    # the hashing kernels (SPGEMM_NO_REUSE=1) give the same bits
    a = S.random_values(S.stencil3d_27pt(24), 1)
    with_reuse = sg.multiply(a, a).c.to_host()
    monkeypatch.setenv("SPGEMM_NO_REUSE", "1")
    without = sg.multiply(a, a).c.to_host()
    assert np.array_equal(with_reuse.col, without.col)
    assert np.array_equal(with_reuse.val.view(np.int64), without.val.view(np.int64))


@pytest.mark.parametrize("n", [16, 48])
def test_wide_route_distinct_operands(sg, oracle, n):
    # A and B of one pattern in separate arrays: the row flags compare A's rows
    # themselves instead of reading B's shift flags for them
    a = S.random_values(S.stencil3d_27pt(n), 21)
    b = S.random_values(S.stencil3d_27pt(n), 22)
    b = CsrMatrix(b.rows, b.cols, b.rpt.copy(), b.col.copy(), b.val)
    _run(sg, oracle, a, b, "k_num_reuse_multi")


@pytest.mark.parametrize("frac,seed", [(0.002, 7), (0.05, 8)])
def test_wide_route_other_b_pattern(sg, oracle, frac, seed):
    # B's pattern differs from A's (dropped entries): A's row shifts hold, B's
    # shift flags break the chains wherever a dropped entry is referenced
    a = S.random_values(S.stencil3d_27pt(20), seed)
    b = S.random_values(_drop(S.stencil3d_27pt(20), frac, seed + 100), seed + 1)
    b = CsrMatrix(b.rows, b.cols, b.rpt, b.col, b.val)
    out = sg.multiply(a, b)
    assert_matches_oracle(out.c, oracle.spgemm(a, b))


def test_wide_route_repeatable(sg, oracle):
    a = S.random_values(S.stencil3d_27pt(40), 31)
    first = sg.multiply(a, a).c.to_host()
    again = sg.multiply(a, a).c.to_host()
    assert np.array_equal(first.col, again.col)
    assert np.array_equal(first.val.view(np.int64), again.val.view(np.int64))
