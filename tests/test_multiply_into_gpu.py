"""Host in, host out with overlapped downloads (C ABI spgemm_multiply_into): the row
blocks' C slices land in the caller's buffers with stitched row pointers and must be
bitwise the single-shot product, for any block count; too-small buffers are refused."""
import numpy as np
import pytest

from helpers import random_csr
from paper_2206_07244_b200 import synthetic as S

pytestmark = pytest.mark.gpu


def _bufs(rows, cap):
    return np.full(rows + 1, -7, np.int64), np.zeros(cap, np.int32), np.zeros(cap, np.float64)


CASES = {
    "stencil27": lambda: (S.random_values(S.stencil3d_27pt(20), 3),) * 2,
    "rmat12": lambda: (S.random_values(S.rmat(12, 16, seed=8), 4),) * 2,
    "rect": lambda: (random_csr(400, 300, 0.03, 1), random_csr(300, 500, 0.02, 2)),
    "empty_rows": lambda: (random_csr(300, 300, 0.0, 3), random_csr(300, 300, 0.05, 4)),
}


@pytest.mark.parametrize("parts", [0, 1, 3, 8])
@pytest.mark.parametrize("name", sorted(CASES))
def test_multiply_into_bitwise(sg, name, parts):
    a, b = CASES[name]()
    ref = sg.multiply(a, b)
    c = ref.c
    rpt, col, val = _bufs(a.rows, c.nnz() + 5)
    nnz, out = sg.multiply_into(a, b, rpt, col, val, parts=parts)
    assert nnz == c.nnz() == out.stats.nnz_of_product
    assert out.stats.total_nprod == ref.stats.total_nprod
    np.testing.assert_array_equal(rpt, c.rpt)
    np.testing.assert_array_equal(col[:nnz], c.col)
    assert np.array_equal(val[:nnz].view(np.int64), c.val.view(np.int64))


def test_multiply_into_capacity(sg):
    a = S.random_values(S.stencil3d_27pt(12), 5)
    n = sg.forecast_nnz(a, a, per_row=False).total_nnz
    rpt, col, val = _bufs(a.rows, n - 1)
    with pytest.raises(sg.InvalidArgument):
        sg.multiply_into(a, a, rpt, col, val, parts=2)
    rpt, col, val = _bufs(a.rows, n)
    assert sg.multiply_into(a, a, rpt, col, val)[0] == n


def test_multiply_into_zero_rows(sg):
    a = sg.CsrMatrix(0, 5, np.zeros(1, np.int64), np.zeros(0, np.int32), np.zeros(0))
    b = random_csr(5, 7, 0.5, 1)
    rpt, col, val = _bufs(0, 0)
    assert sg.multiply_into(a, b, rpt, col, val)[0] == 0 and rpt[0] == 0


def test_private_pool_and_trim(sg):
    """The library allocates from its context's own stream-ordered pool:
    Context.trim() returns the cached scratch and pooled HBM, and the context
    keeps working after it."""
    import torch
    from paper_2206_07244_b200 import synthetic as S
    ctx = sg.get_context(0)
    a = S.stencil3d_27pt(40)
    out = sg.multiply(a, a)
    assert out.c.nnz() > 0
    reserved, used = ctx.pool_stats()
    assert reserved > 0
    ctx.trim(0)
    r2, u2 = ctx.pool_stats()
    assert r2 <= reserved and u2 == 0
    # a further multiply works after the trim (the pool regrows)
    assert sg.multiply(a, a).c.nnz() == out.c.nnz()
    torch.cuda.synchronize()
