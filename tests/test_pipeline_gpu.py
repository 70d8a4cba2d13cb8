"""GPU parity for the SpgemmPipeline / multiply path, mirroring the reference's
proj/tests/test_pipeline.cpp case by case (line numbers cited per test). The
checker is the C restatement in oracle/ (bitwise the reference's values)."""
import numpy as np
import pytest

from helpers import assert_matches_oracle, bitwise_equal, random_csr, random_csr_fixed, spill_pair
from paper_2206_07244_b200 import synthetic as S

pytestmark = pytest.mark.gpu


def outputs_identical(x, y):
    return (bitwise_equal(x.c, y.c) and x.stats.total_nprod == y.stats.total_nprod
            and x.stats.nnz_of_product == y.stats.nnz_of_product)


def test_setup_writes_nprod(sg):  # test_pipeline.cpp:70-79
    i3 = S.identity_csr(3)
    p = sg.SpgemmPipeline(i3, i3)
    p.setup()
    assert list(p.rpt_region()) == [1, 1, 1]


@pytest.mark.parametrize("overlap", [True, False])
def test_setup_region_matches_compute_nprod(sg, oracle, overlap):  # :81-97
    a = random_csr(300, 300, 0.03, 31)
    expected, _ = oracle.compute_nprod(a, a)
    p = sg.SpgemmPipeline(a, a, sg.SpgemmOptions(overlap=overlap))
    p.setup()
    assert np.array_equal(p.rpt_region(), expected)


def test_compute_nprod_kernel(sg, oracle):
    a = random_csr(500, 400, 0.03, 5)
    b = random_csr(400, 300, 0.04, 6)
    exp, tot = oracle.compute_nprod(a, b)
    got, gt = sg.compute_nprod(a, b)
    assert np.array_equal(got, exp) and gt == tot


def test_build_rpt(sg):  # :99-123
    r = np.array([2, 0, 3, 0], np.int64)
    assert sg.build_rpt(r) == 5
    assert list(r) == [0, 2, 2, 5]
    z = np.zeros(6, np.int64)
    assert sg.build_rpt(z) == 0 and not z.any()
    rng = np.random.default_rng(32)
    counts = rng.integers(0, 7, 10001).astype(np.int64)
    counts[-1] = 0
    expected = np.concatenate([[0], np.cumsum(counts)[:-1]])
    running = int(counts.sum())
    inplace = counts.copy()
    assert sg.build_rpt(inplace) == running
    assert np.array_equal(inplace, expected)
    big = rng.integers(0, 1000, 3_000_001).astype(np.int64)
    exp = np.concatenate([[0], np.cumsum(big)[:-1]])
    tot = int(big.sum())
    assert sg.build_rpt(big) == tot and np.array_equal(big, exp)


def test_identity_squared_bitwise(sg):  # :125-132
    i5 = S.identity_csr(5)
    out = sg.multiply(i5, i5)
    assert out.c == i5
    assert out.stats.total_nprod == 5 and out.stats.nnz_of_product == 5 and out.stats.cr == 1.0


def test_hand_2x2(sg):  # :134-141
    a = S.csr_from_coo(2, 2, [0, 1], [1, 0], [2.0, 3.0])
    out = sg.multiply(a, a)
    assert list(out.c.rpt) == [0, 1, 2] and list(out.c.col) == [0, 1] and list(out.c.val) == [6.0, 6.0]


def test_empty_and_nilpotent(sg):  # :143-157
    empty = sg.CsrMatrix(0, 0)
    out = sg.multiply(empty, empty)
    assert out.c.rows == 0 and out.c.nnz() == 0
    n = S.csr_from_coo(2, 2, [0], [1], [1.0])
    nil = sg.multiply(n, n)
    assert nil.c.nnz() == 0 and list(nil.c.rpt) == [0, 0, 0] and nil.stats.cr == 0.0


def test_rejects_shapes_and_order(sg):  # :159-168
    with pytest.raises(sg.InvalidArgument):
        sg.multiply(S.identity_csr(3), S.identity_csr(4))
    i3 = S.identity_csr(3)
    p = sg.SpgemmPipeline(i3, i3)
    with pytest.raises(sg.LogicError):
        p.run_symbolic()
    p.setup()
    with pytest.raises(sg.LogicError):
        p.setup()
    with pytest.raises(sg.LogicError):
        p.finalize_rpt()


def test_random_products_match_oracle(sg, oracle):  # :170-184
    rng = np.random.default_rng(33)
    for trial in range(15):
        m, k, n = (1 + int(x) for x in rng.integers(0, 400, 3))
        a = random_csr(m, k, 0.05, 1000 + trial)
        b = random_csr(k, n, 0.05, 2000 + trial)
        out = sg.multiply(a, b)
        expected = oracle.spgemm(a, b)
        assert sg.validate_csr(out.c).ok()
        assert_matches_oracle(out.c, expected)
        assert out.stats.nnz_of_product == out.c.nnz()


def test_per_row_symbolic_counts(sg, oracle):  # :186-199
    a = random_csr(200, 200, 0.06, 34)
    expected = oracle.spgemm(a, a)
    p = sg.SpgemmPipeline(a, a)
    p.setup()
    p.symbolic_binning()
    p.run_symbolic()
    assert np.array_equal(p.rpt_region(), np.diff(expected.rpt))


def test_overlap_invariance(sg):  # :201-209
    a = random_csr(500, 500, 0.03, 35)
    assert outputs_identical(sg.multiply(a, a, sg.SpgemmOptions(overlap=True)),
                             sg.multiply(a, a, sg.SpgemmOptions(overlap=False)))


def test_deterministic_repeatable(sg):  # :211-224
    a = random_csr(600, 600, 0.02, 36)
    base = sg.multiply(a, a)
    for workers in (1, 2, 3, 8):
        o = sg.SpgemmOptions(workers=workers)
        x, y = sg.multiply(a, a, o), sg.multiply(a, a, o)
        assert outputs_identical(x, base) and outputs_identical(x, y)


def test_launch_order_invariance(sg):  # :226-239
    a = random_csr(700, 700, 0.05, 37)
    base = sg.multiply(a, a)
    shuffled = sg.SpgemmOptions(sym_launch_order=[0, 1, 2, 3, 4, 5, 6, 7],
                                num_launch_order=[3, 0, 7, 1, 6, 2, 5, 4])
    assert outputs_identical(sg.multiply(a, a, shuffled), base)
    with pytest.raises(sg.InvalidArgument):
        sg.multiply(a, a, sg.SpgemmOptions(sym_launch_order=[0, 0, 2, 3, 4, 5, 6, 7]))


def test_racing_mode_same_matrix(sg):  # :241-251
    a = random_csr(800, 800, 0.04, 41)
    base = sg.multiply(a, a)
    for _ in range(3):
        assert outputs_identical(sg.multiply(a, a, sg.SpgemmOptions(deterministic=False, workers=4)), base)


def test_preset_combinations_bitwise(sg):  # :253-268
    a = random_csr(400, 400, 0.08, 38)
    base = sg.multiply(a, a)
    for sym in sg.preset_names(sg.SYMBOLIC):
        for num in sg.preset_names(sg.NUMERIC):
            out = sg.multiply(a, a, sg.SpgemmOptions(sym_preset=sym, num_preset=num))
            assert outputs_identical(out, base), (sym, num)


def test_alloc_accounting(sg):  # :270-283
    a = random_csr(300, 300, 0.05, 39)
    stats = sg.AllocStats()
    out = sg.multiply(a, a, sg.SpgemmOptions(alloc_stats=stats))
    assert stats.metadata_calls == 2 and stats.output_calls == 2
    rpt_bytes = (a.rows + 1) * 8
    assert stats.metadata_bytes >= rpt_bytes + a.rows * 8 * 2
    assert stats.output_bytes == out.c.nnz() * 12


def test_spill_to_global_tier(sg, oracle):  # :285-296
    a, b = spill_pair(20000, 200)
    out = sg.multiply(a, b, sg.SpgemmOptions(workers=2))
    assert out.spilled_rows == 1
    assert_matches_oracle(out.c, oracle.spgemm(a, b))
    assert out.c.row_nnz(0) == 20000


@pytest.mark.parametrize("pair", [(20000, 200), (6000, 60), (3000, 30)])
@pytest.mark.parametrize("num", ["num_1x", "num_2x", "num_3x"])
def test_heap_tier_deterministic_is_bitwise(sg, oracle, pair, num):
    """deterministic=True (default): heap-tier rows fold in the reference's order
    (bitwise) under every numeric preset; deterministic=False within 1e-12."""
    a, b = spill_pair(*pair)
    a, b = S.random_values(a, 5), S.random_values(b, 6)
    exp = oracle.spgemm(a, b)
    out = sg.multiply(a, b, sg.SpgemmOptions(num_preset=num))
    assert_matches_oracle(out.c, exp)
    again = sg.multiply(a, b, sg.SpgemmOptions(num_preset=num))
    assert bitwise_equal(again.c, out.c.to_host())
    out = sg.multiply(a, b, sg.SpgemmOptions(num_preset=num, deterministic=False))
    assert_matches_oracle(out.c, exp, bitwise=False)


def test_spill_threshold_stays_fixed(sg):  # :298-303
    a, b = spill_pair(19660, 20)
    out = sg.multiply(a, b)
    assert out.spilled_rows == 0 and out.c.row_nnz(0) == 19660


def test_numeric_heap_tier(sg, oracle):  # :305-314
    a, b = spill_pair(6000, 60)
    out = sg.multiply(a, b)
    assert out.spilled_rows == 0 and out.c.row_nnz(0) == 6000
    assert_matches_oracle(out.c, oracle.spgemm(a, b))


def test_timings_cover_steps(sg):  # :316-325
    a = random_csr(200, 200, 0.05, 40)
    t = sg.multiply(a, a).timings
    parts = t.setup + t.sym_binning + t.symbolic + t.rpt_alloc + t.num_binning + t.numeric + t.cleanup
    assert t.total == pytest.approx(parts) and t.total > 0


def test_workers_reported(sg):
    a = random_csr(50, 50, 0.1, 4)
    assert sg.multiply(a, a).workers > 0


def test_empty_b_rows(sg):  # :327-343
    a = S.csr_from_coo(3, 3, [0, 1, 1], [0, 1, 2], [1.0, 2.0, 3.0])
    b = S.csr_from_coo(3, 3, [0], [2], [5.0])
    out = sg.multiply(a, b)
    assert list(out.c.rpt) == [0, 1, 1, 1] and list(out.c.col) == [2] and list(out.c.val) == [5.0]
    empty_b = sg.CsrMatrix(3, 4, np.zeros(4, np.int64))
    z = sg.multiply(a, empty_b)
    assert z.c.nnz() == 0 and z.c.cols == 4


def test_200k_rows_four_per_row(sg, oracle):  # :345-359
    a = random_csr_fixed(200200, 200200, 4, 42)
    assert a.nnz() == 800800
    out = sg.multiply(a, a)
    assert out.stats.total_nprod == 3203200
    assert sg.validate_csr(out.c).ok()
    assert_matches_oracle(out.c, oracle.spgemm(a, a))
