"""GPU parity on the BASELINE.json config families.

Small instances are checked entry-for-entry (bitwise) against the C oracle;
the full-size stencil configs are checked against the oracle too (they finish
in seconds on the host), and carry the published statistics as known answers.
"""
import numpy as np
import pytest

from helpers import assert_matches_oracle
from paper_2206_07244_b200 import synthetic as S

pytestmark = pytest.mark.gpu


def _check(sg, oracle, a, b, **kw):
    out = sg.multiply(a, b, sg.SpgemmOptions(**kw))
    exp = oracle.spgemm(a, b)
    assert_matches_oracle(out.c, exp)
    return out


@pytest.mark.parametrize("cfg", [1, 2, 3])
def test_small_config_square(sg, oracle, cfg):
    a, b = S.config_matrices(cfg, small=True)
    _check(sg, oracle, a, b)
    _check(sg, oracle, S.random_values(a, 7), S.random_values(b, 7))


def test_small_rap_chain(sg, oracle):
    a, p, r = S.config_matrices(4, small=True)
    ap = _check(sg, oracle, a, p).c
    _check(sg, oracle, r, ap)


@pytest.mark.parametrize("scale", [12, 14])
def test_rmat_mid(sg, oracle, scale):
    a = S.random_values(S.rmat(scale, 16, seed=scale), 3)
    out = _check(sg, oracle, a, a)
    assert out.stats.total_nprod == oracle.compute_nprod(a, a)[1]


def test_config1_full_known_answer(sg, oracle):
    a, _ = S.config_matrices(1)
    out = _check(sg, oracle, a, a)
    assert out.stats.total_nprod == 26_177_544 and out.stats.nnz_of_product == 13_611_012


@pytest.mark.slow
def test_config2_full_known_answer(sg, oracle):
    a, _ = S.config_matrices(2)
    out = _check(sg, oracle, a, a)
    assert out.stats.total_nprod == 1_489_355_288 and out.stats.nnz_of_product == 254_840_104


def test_config4_full_known_answer(sg, oracle):
    a, p, r = S.config_matrices(4)
    ap = _check(sg, oracle, a, p)
    assert ap.stats.total_nprod == 48_556_211 and ap.stats.nnz_of_product == 20_757_689
    rap = _check(sg, oracle, r, ap.c)
    assert rap.stats.total_nprod == 69_839_855 and rap.stats.nnz_of_product == 6_859_000


def test_device_resident_inputs(sg, oracle):
    a, _ = S.config_matrices(2, small=True)
    a = S.random_values(a, 11)
    d = a.to_device()
    dm, rep = sg.multiply_device(d, d)
    c = dm.download()
    dm.free()
    assert_matches_oracle(c, oracle.spgemm(a, a))
    assert rep.stats.total_nprod == oracle.compute_nprod(a, a)[1]


def test_virtual_row_slices_stitch_bitwise(sg, oracle):
    """SURVEY §8(e) on one GPU: G nprod-balanced row blocks multiplied separately and
    stitched equal the single-shot product bitwise."""
    from paper_2206_07244_b200.distributed import nprod_split, slice_rows, stitch
    a = S.random_values(S.stencil3d_27pt(24), 3)
    single = sg.multiply(a, a).c
    nprod, _ = sg.compute_nprod(a, a)
    for parts in (2, 3, 8):
        b = nprod_split(nprod, parts)
        slices = [sg.multiply(slice_rows(a, b[g], b[g + 1]), a).c for g in range(parts)]
        assert stitch(slices, a.cols) == single


def test_download_async_matches_sync(sg, oracle):
    """DeviceMatrix.download_async (copy lane, device buffers released behind the copy)
    delivers the same C as the synchronous download, also when the next product is
    queued before the wait."""
    import torch
    a = S.random_values(S.stencil3d_27pt(20), 4)
    ctx = sg.get_context()
    exp = oracle.spgemm(a, a)
    bufs = []
    for _ in range(2):
        dm, _ = sg.multiply_device(a, a)
        r = torch.empty(a.rows + 1, dtype=torch.int64).pin_memory()
        c = torch.empty(dm.nnz, dtype=torch.int32).pin_memory()
        v = torch.empty(dm.nnz, dtype=torch.float64).pin_memory()
        dm.download_async(r.numpy(), c.numpy(), v.numpy(), release=True)
        dm.free()
        bufs.append((r, c, v))
    ctx.wait_downloads()
    for r, c, v in bufs:
        got = sg.CsrMatrix(a.rows, a.cols, r.numpy(), c.numpy(), v.numpy())
        assert_matches_oracle(got, exp, bitwise=True)


def test_speculative_rows_mixed_with_abandoned(sg, oracle):
    """Regular A (28 entries per row, long B rows) puts every row in a symbolic bin the
    speculative numeric runs on: stencil rows fit its 128-entry scratch and are finished
    there, scattered random rows (~700 distinct columns) overflow it, are abandoned and
    go through the symbolic + numeric kernels. Both kinds in one product, bitwise."""
    from helpers import random_csr_fixed
    from paper_2206_07244_b200.distributed import slice_rows
    sten = S.random_values(S.stencil3d_27pt(14), 2)            # 27 entries/row, CR ~6
    rnd = random_csr_fixed(sten.rows, sten.cols, 28, 8)         # 28 entries/row, CR ~1
    rnd = S.random_values(rnd, 3)
    # interleave: rows alternate between the stencil and the random matrix
    rows = sten.rows
    pick = np.arange(rows) % 2 == 0
    import numpy as _np
    rpt = _np.zeros(rows + 1, _np.int64)
    lens = _np.where(pick, _np.diff(sten.rpt), _np.diff(rnd.rpt))
    _np.cumsum(lens, out=rpt[1:])
    col = _np.concatenate([(sten if pick[i] else rnd).row_cols(i) for i in range(rows)])
    val = _np.concatenate([(sten if pick[i] else rnd).row_vals(i) for i in range(rows)])
    a = sg.CsrMatrix(rows, sten.cols, rpt, col.astype(_np.int32), val)
    out = sg.multiply(a, a)
    exp = oracle.spgemm(a, a)
    assert_matches_oracle(out.c, exp, bitwise=True)
    nnz = np.diff(exp.rpt)
    assert (nnz[pick] <= 128).any() and (nnz[~pick] > 128).any()


@pytest.mark.parametrize("parts", [1, 2, 3])
def test_multiply_multi_stitches_bitwise(sg, oracle, parts):
    """spgemm_multiply_multi (SURVEY §8(e) inside one process): nprod-balanced row blocks
    on separate contexts (here all on device 0, each on its own host thread), slices
    stitched on the host -- bitwise the single-context product."""
    from paper_2206_07244_b200.distributed import nprod_split
    for a in (S.random_values(S.stencil3d_27pt(20), 6), S.random_values(S.rmat(12, 16, seed=12), 7)):
        single = sg.multiply(a, a)
        multi = sg.multiply_multi(a, a, devices=[0] * parts)
        assert multi.c == single.c
        assert multi.stats.total_nprod == single.stats.total_nprod
        assert multi.stats.nnz_of_product == single.stats.nnz_of_product
        nprod, _ = sg.compute_nprod(a, a)
        assert multi.row_bounds == nprod_split(nprod, parts)
