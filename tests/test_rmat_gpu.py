"""GPU parity at R-MAT scale (BASELINE.json config 3 family): skewed rows exercise the
symbolic spill path, the global-memory (heap) tiers and the bitmap ranking.

The full product at scale 20 has 9.7e9 nonzeros (116.7 GB) -- it fits one B200 but not
the host, so C is verified on a deterministic row sample (every row with nprod > 1e5
plus random rows) against the oracle, plus global invariants
(row pointers monotone, the nnz total, the spill count)."""
import numpy as np
import pytest

from helpers import assert_matches_oracle
from paper_2206_07244_b200 import synthetic as S
from paper_2206_07244_b200.api import CsrMatrix

pytestmark = pytest.mark.gpu


def _rows_subset(a, rows):
    rows = np.asarray(rows, np.int64)
    lens = a.rpt[rows + 1] - a.rpt[rows]
    rpt = np.concatenate([[0], np.cumsum(lens)])
    idx = np.concatenate([np.arange(a.rpt[r], a.rpt[r + 1]) for r in rows]) if rows.size else np.zeros(0, np.int64)
    return CsrMatrix(rows.size, a.cols, rpt, a.col[idx], a.val[idx])


def _check_sampled(sg, oracle, a, scale_seed, n_random=400):
    import torch
    d = a.to_device()
    dm, out = sg.multiply_device(d, d)
    try:
        nprod, total = oracle.compute_nprod(a, a)
        assert out.stats.total_nprod == total
        rpt = torch.empty(a.rows + 1, dtype=torch.int64)
        ptr = dm.ptrs[0]
        import ctypes
        rpt_dev = torch.as_tensor(_CAI(ptr, a.rows + 1, "<i8"), device="cuda")
        rpt = rpt_dev.cpu().numpy()
        assert rpt[0] == 0 and (np.diff(rpt) >= 0).all() and rpt[-1] == out.stats.nnz_of_product
        rng = np.random.default_rng(scale_seed)
        heavy = np.nonzero(nprod > 100_000)[0]
        sample = np.unique(np.concatenate([heavy[:300], rng.choice(a.rows, n_random, replace=False)]))
        sub = _rows_subset(a, sample)
        exp = oracle.spgemm(sub, a)
        col_dev = torch.as_tensor(_CAI(dm.ptrs[1], dm.nnz, "<i4"), device="cuda")
        val_dev = torch.as_tensor(_CAI(dm.ptrs[2], dm.nnz, "<f8"), device="cuda")
        idx = torch.from_numpy(np.concatenate([np.arange(rpt[r], rpt[r + 1]) for r in sample])).cuda()
        got_col = col_dev[idx].cpu().numpy()
        got_val = val_dev[idx].cpu().numpy()
        got_rpt = np.concatenate([[0], np.cumsum(rpt[sample + 1] - rpt[sample])])
        got = CsrMatrix(sample.size, a.cols, got_rpt, got_col, got_val)
        assert_matches_oracle(got, exp)
        # spill count: rows of symbolic bin 7 whose nnz exceeds 19660 (reference semantics)
        sym = sg.symbolic_preset("sym_1.2x")
        assert out.spilled_rows == oracle.spilled_rows(nprod, np.diff(rpt), sym.upper)
        return out
    finally:
        dm.free()


class _CAI:
    def __init__(self, ptr, n, typestr):
        self.__cuda_array_interface__ = {"shape": (n,), "typestr": typestr, "data": (ptr, False), "version": 3}


def test_rmat16_full_oracle(sg, oracle):
    a = S.random_values(S.rmat(16, 16, seed=16), 1)
    exp = oracle.spgemm(a, a)
    assert (np.diff(exp.rpt) > 4096).any(), "the case must reach the numeric heap tier"
    out = sg.multiply(a, a)  # deterministic (default): bitwise on every row, heap tier included
    assert_matches_oracle(out.c, exp)
    out = sg.multiply(a, a, sg.SpgemmOptions(deterministic=False))  # fp64 atomics in the heap tier
    assert_matches_oracle(out.c, exp, bitwise=False)
    out = sg.multiply(a, a, sg.SpgemmOptions(deterministic=False, ordered_heap=True))
    assert_matches_oracle(out.c, exp)


def _identical(x, y):
    return (np.array_equal(x.c.rpt, y.c.rpt) and np.array_equal(x.c.col, y.c.col)
            and np.array_equal(x.c.val.view(np.int64), y.c.val.view(np.int64)))


def test_rmat16_deterministic_repeat_and_presets(sg, oracle):
    """test_pipeline.cpp:211-224 and :253-268 (acceptance criterion 3) on a skewed
    matrix whose rows reach every numeric tier, the heap tier included: repeated
    runs and all 12 preset combinations give bitwise-identical C, equal to the
    reference's (num_3x moves rows of 2731..4096 nnz into its bin 7)."""
    a = S.random_values(S.rmat(16, 16, seed=16), 3)
    exp = oracle.spgemm(a, a)
    lens = np.diff(exp.rpt)
    assert (lens > 4096).any() and ((lens > 2730) & (lens <= 4096)).any()
    base = sg.multiply(a, a)
    assert_matches_oracle(base.c, exp)
    for _ in range(3):
        assert _identical(sg.multiply(a, a), base)
    for sym in sg.preset_names(sg.SYMBOLIC):
        for num in sg.preset_names(sg.NUMERIC):
            out = sg.multiply(a, a, sg.SpgemmOptions(sym_preset=sym, num_preset=num))
            assert _identical(out, base), (sym, num)


@pytest.mark.slow
def test_rmat18_sampled(sg, oracle):
    a = S.random_values(S.rmat(18, 16, seed=18), 7)
    out = _check_sampled(sg, oracle, a, 18)
    assert out.spilled_rows > 0


@pytest.mark.slow
def test_rmat20_config3_sampled(sg, oracle):
    a = S.rmat(20, 16, seed=20)
    out = _check_sampled(sg, oracle, a, 20, n_random=200)
    assert out.stats.total_nprod > 2e10 and out.spilled_rows > 0


@pytest.mark.slow
def test_rmat24_config5_sampled(sg, oracle):
    """BASELINE config 5 (R-MAT scale 24, nprod 1.0e12, C ~6 TB: never materialised)
    checked at its own size on a deterministic row sample (SURVEY.md §8(d)
    "Verification for large configs"): every row with nprod > 1e8, the heaviest
    rows below that, 256 consecutive rows of the middle of the matrix (the bench's
    cpu_baseline block) and random rows -- C(sample, :) from the device against the
    REFERENCE's own pipeline (oracle/_ref, spgemm::multiply) on the same rows:
    structure bitwise, values bitwise (deterministic mode)."""
    a = S.random_values(S.rmat(24, 16, seed=24), 24)
    import torch
    d = a.to_device()
    nprod, total = sg.compute_nprod(d, d)
    assert total > 1.0e12
    rng = np.random.default_rng(24)
    order = np.argsort(nprod)[::-1]
    heavy = np.nonzero(nprod > 100_000_000)[0]
    mid = a.rows // 2
    sample = np.unique(np.concatenate([heavy, order[:8], np.arange(mid, mid + 256),
                                       rng.choice(a.rows, 256, replace=False)]))
    sub = _rows_subset(a, sample)
    got = sg.multiply(sub.to_device(), d)
    if oracle.ref_available():
        exp, info = oracle.ref_multiply(sub, a)
        assert info["total_nprod"] == int(nprod[sample].sum())
    else:
        exp = oracle.spgemm(sub, a)
    assert_matches_oracle(got.c, exp)
    del d
    torch.cuda.empty_cache()


@pytest.mark.parametrize("num", ["num_1x", "num_1.5x"])
def test_b200_block_tier(sg, oracle, num):
    """Bin 6 of num_1x / num_1.5x (4096..8191 / 3073..5460 nonzeros; a fixed-table
    tier in the reference) runs on chip in the 16384-slot table
    (k_num_block<16384>: sort keys over the table's keys, 192 KB of the B200's
    227 KB per block) when B's rows are long; bitwise the reference."""
    from helpers import random_csr_fixed
    a = S.random_values(random_csr_fixed(300, 20000, 55, 51), 52)
    b = S.random_values(random_csr_fixed(20000, 20000, 100, 53), 54)
    exp = oracle.spgemm(a, b)
    lens = np.diff(exp.rpt)
    assert ((lens > 4096) & (lens <= 5460)).all()
    ctx = sg.get_context()
    ctx.set_profiling(True)
    try:
        ctx.profile_summary()
        out = sg.multiply(a, b, sg.SpgemmOptions(num_preset=num))
        names = ctx.profile_summary()
    finally:
        ctx.set_profiling(False)
    assert_matches_oracle(out.c, exp)
    assert any(k.split("#")[0] == "k_num_block<16384>" for k in names), sorted(names)
    out = sg.multiply(a, b, sg.SpgemmOptions(num_preset=num, deterministic=False))
    assert_matches_oracle(out.c, exp)  # an on-chip tier: ordered either way
