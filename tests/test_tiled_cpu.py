"""CPU: the host side of the streamed/tiled mode (paper_2206_07244_b200/tiled.py) --
row blocks bounded by an nprod budget, and the checksum of a materialised C."""
import numpy as np
import pytest

from paper_2206_07244_b200 import tiled as T
from paper_2206_07244_b200.api import CsrMatrix


@pytest.mark.parametrize("nprod,budget", [([5, 5, 5, 20, 1, 1, 1], 10), ([1] * 10, 3), ([100], 5), ([3, 3, 3], 100),
                                          ([0, 0, 7, 0, 9, 2, 0], 9)])
def test_row_blocks_cover_and_respect_budget(nprod, budget):
    n = np.asarray(nprod, np.int64)
    b = T.row_blocks(n, budget)
    assert b[0] == 0 and b[-1] == n.size and all(x < y for x, y in zip(b, b[1:]))
    for i in range(len(b) - 1):
        blk = n[b[i]:b[i + 1]]
        assert blk.sum() <= budget or blk.size == 1  # a single oversized row stands alone


def test_row_blocks_random_against_greedy():
    rng = np.random.default_rng(5)
    n = rng.integers(0, 50, 2000)
    b = T.row_blocks(n, 400)
    sums = [int(n[b[i]:b[i + 1]].sum()) for i in range(len(b) - 1)]
    assert sum(sums) == int(n.sum())
    # maximal blocks: adding the next row would exceed the budget
    for i in range(len(b) - 2):
        assert sums[i] + int(n[b[i + 1]]) > 400


def test_checksum_of_definition():
    c = CsrMatrix(2, 5, np.array([0, 2, 3]), np.array([1, 4, 0], np.int32), np.array([1.5, -2.0, 4.0]))
    rep = T.checksum_of(c)
    assert rep.nnz == 3 and rep.val_sum == 3.5
    assert rep.pattern_hash == (1 + 1) * 1 + (4 + 1) * 1 + (0 + 1) * 2
