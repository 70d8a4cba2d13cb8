"""Device binning (K2 k_pass1, K3 k_bin_offsets + k_bin_scatter) through the standalone
run_binning entry (binning.cpp:281-313) against the oracle (pinned to the reference's
golden binnings in test_oracle.py): identical bins, sizes, offsets, max/total and fast-path
flag, bit-exact. Covers one and several 1024-row-block tiles of k_bin_offsets
(2048 rows per row block, so > 2^21 rows takes the multi-tile path)."""
import numpy as np
import pytest

pytestmark = pytest.mark.gpu


def _metric(m: int, seed: int, hi: int) -> np.ndarray:
    rng = np.random.default_rng(seed)
    x = rng.integers(0, hi, size=m, dtype=np.int64)
    x[rng.random(m) < 0.01] *= 50  # a sprinkle of heavy rows in the upper bins
    return x


@pytest.mark.parametrize("m,hi", [(0, 1), (1, 5), (2047, 300), (2048, 300), (100_000, 2000),
                                  (1024 * 2048, 700), (1024 * 2048 + 1, 700), (3_000_001, 3000),
                                  (5_000_000, 40)])
@pytest.mark.parametrize("phase", [0, 1])
def test_run_binning_matches_oracle(sg, oracle, m, hi, phase):
    cfg = sg.preset(phase, sg.kDefaultSymPreset if phase == 0 else sg.kDefaultNumPreset)
    metric = _metric(m, m + phase, hi)
    got = sg.run_binning(metric, cfg)
    exp = oracle.run_binning(metric, np.asarray(cfg.upper, np.int64))
    assert got.fast_path == exp["fast_path"]
    assert list(got.bin_size) == list(exp["bin_size"])
    assert list(got.bin_offset) == list(exp["bin_offset"])
    assert got.max_metric == exp["max_metric"] and got.total_metric == exp["total_metric"]
    if not exp["fast_path"]:
        np.testing.assert_array_equal(got.bins, exp["bins"])
