"""Tiled / streamed SpGEMM (config 5's mode, paper_2206_07244_b200/tiled.py): the
row-block x column-window tiles, each a full device pipeline reduced to checksums,
must add up to the untiled product -- same nprod, nnz and pattern hash, and the
value sum within fp64 tolerance."""
import numpy as np
import pytest

from paper_2206_07244_b200 import synthetic as S
from paper_2206_07244_b200 import tiled as T

pytestmark = pytest.mark.gpu


@pytest.mark.parametrize("window,budget,workers", [(4096, 2_000_000, 1), (1 << 20, 10**12, 1),
                                                   (1000, 500_000, 1), (4096, 2_000_000, 3)])
def test_stream_matches_untiled(sg, window, budget, workers):
    a = S.random_values(S.rmat(13, 16, seed=13), 7)
    full = sg.multiply(a, a).c
    ref = T.checksum_of(full)
    d = a.to_device()
    rep = T.stream_multiply(d, d, budget=budget, window=window, workers=workers)
    assert rep.total_nprod == sg.compute_nprod(a, a)[1]
    assert rep.nnz == ref.nnz
    assert rep.pattern_hash == ref.pattern_hash
    assert abs(rep.val_sum - ref.val_sum) <= 1e-9 * max(1.0, abs(ref.val_sum))
    if window < a.cols:
        assert rep.tiles > 1
    # every tile ran the native kernels (>= K1, scan, one symbolic and numeric launch, checksum)
    assert rep.kernel_launches >= 4 * rep.tiles


def test_split_columns_partition(sg):
    import torch
    a = S.rmat(12, 8, seed=3)
    d = a.to_device()
    wins = T.split_columns(d, 1000)
    assert len(wins) == (a.cols + 999) // 1000
    assert sum(int(w.rpt[-1].item()) for w in wins) == a.nnz()
    # every window's rows stay sorted and within its width
    for w in wins:
        c = w.col.cpu().numpy()
        assert c.size == 0 or (c.min() >= 0 and c.max() < w.cols)
