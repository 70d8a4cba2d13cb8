"""CPU: pin the C restatement (oracle/spgemm_oracle.c) against the reference itself.

Goldens in tests/golden/ were produced by the unmodified reference core
(oracle/_ref, see tests/golden/make_golden.py). When oracle/_ref is present
(this container) the restatement is also cross-checked live."""
import json
import os

import numpy as np
import pytest

from helpers import random_csr, spill_pair

GOLDEN = os.path.join(os.path.dirname(__file__), "golden")


def _load_products():
    d = np.load(os.path.join(GOLDEN, "products.npz"))
    meta = json.loads(bytes(d["meta"]).decode())
    from oracle.oracle import csr
    out = []
    for i, m in enumerate(meta):
        mats = []
        for tag in "abc":
            r, c = d[f"{i}_{tag}_shape"]
            mats.append(csr(r, c, d[f"{i}_{tag}_rpt"], d[f"{i}_{tag}_col"], d[f"{i}_{tag}_val"]))
        out.append((mats[0], mats[1], mats[2], d[f"{i}_nprod"], m))
    return out


PRODUCTS = _load_products()


@pytest.mark.parametrize("idx", range(len(PRODUCTS)))
def test_oracle_matches_reference_golden_bitwise(oracle, idx):
    a, b, c_ref, nprod_ref, meta = PRODUCTS[idx]
    c = oracle.spgemm(a, b)
    assert oracle.same_pattern(c, c_ref)
    assert np.array_equal(c.val.view(np.int64), c_ref.val.view(np.int64))
    nprod, total = oracle.compute_nprod(a, b)
    assert np.array_equal(nprod, nprod_ref) and total == meta["total_nprod"]
    assert c.rpt[-1] == meta["nnz"]


def test_oracle_binning_matches_reference_golden(oracle):
    d = np.load(os.path.join(GOLDEN, "binning.npz"))
    keys = sorted({k.rsplit("_", 1)[0] for k in d.files})
    assert len(keys) == 14
    for key in keys:
        name = key.rsplit("_", 1)[0]
        phase = 0 if name.startswith("sym") else 1
        upper, _ = oracle.preset(phase, name)
        r = oracle.run_binning(d[key + "_metric"], upper)
        info = d[key + "_info"]
        assert np.array_equal(r["bins"], d[key + "_bins"]), key
        assert list(r["bin_size"]) == list(info[:8]) and list(r["bin_offset"]) == list(info[8:16])
        assert r["max_metric"] == info[16] and r["total_metric"] == info[17] and r["fast_path"] == bool(info[18])


def test_oracle_presets_are_the_published_tables(oracle):
    # test_binning.cpp:50-76
    up, tab = oracle.preset(0, "sym_1.2x")
    assert list(up) == [26, 426, 853, 1706, 3413, 6826, 10240, 2**63 - 1]
    assert list(tab) == [32, 512, 1024, 2048, 4096, 8192, 12287, 24575]
    assert list(oracle.preset(0, "sym_1.5x")[0][:3]) == [21, 341, 682]
    assert list(oracle.preset(1, "num_3x")[0][:3]) == [10, 85, 170]
    up1, tab1 = oracle.preset(1, "num_1x")
    assert list(up1[:7]) == list(tab1[:7])
    assert list(oracle.preset(1, "num_2x")[0]) == [16, 128, 256, 512, 1024, 2048, 4096, 2**63 - 1]
    with pytest.raises(ValueError):
        oracle.preset(0, "sym_2x")
    with open(os.path.join(GOLDEN, "kat.json")) as f:
        kat = json.load(f)
    for name, t in kat["presets"].items():
        u, s = oracle.preset(0 if name.startswith("sym") else 1, name)
        assert list(u) == t["upper"] and list(s) == t["table_size"]


def test_oracle_classify_boundaries(oracle):
    # test_binning.cpp:99-116
    sym, _ = oracle.preset(0, "sym_1.2x")
    assert [oracle.classify(v, sym) for v in (26, 27, 0, 10241, 10**9)] == [0, 1, 0, 7, 7]
    num, _ = oracle.preset(1, "num_2x")
    assert [oracle.classify(v, num) for v in (16, 17, 4096, 4097)] == [0, 1, 6, 7]


def test_oracle_exclusive_sum(oracle):
    buf, total = oracle.exclusive_sum([2, 0, 3, 0])
    assert list(buf) == [0, 2, 2, 5] and total == 5


def test_oracle_spill_known_answers(oracle):
    with open(os.path.join(GOLDEN, "kat.json")) as f:
        kat = json.load(f)
    sym, _ = oracle.preset(0, "sym_1.2x")
    for key, exp in kat["spill"].items():
        distinct, rows_in_b = (int(x) for x in key.split("_"))
        a, b = spill_pair(distinct, rows_in_b)
        c = oracle.spgemm(a, b)
        nprod, total = oracle.compute_nprod(a, b)
        assert int(c.rpt[1] - c.rpt[0]) == exp["row0_nnz"] and total == exp["total_nprod"]
        assert oracle.spilled_rows(nprod, np.diff(c.rpt), sym) == exp["spilled_rows"]


@pytest.mark.skipif(not os.path.exists(os.path.join(os.path.dirname(os.path.dirname(__file__)), "oracle", "_ref",
                                                    "libspgemm_ref.so")), reason="oracle/_ref not built")
def test_oracle_matches_live_reference(oracle):
    for seed in range(4):
        a = random_csr(150 + 37 * seed, 170, 0.04, seed)
        b = random_csr(170, 90 + 11 * seed, 0.06, seed + 50)
        c_ref, info = oracle.ref_multiply(a, b)
        c = oracle.spgemm(a, b)
        assert oracle.same_pattern(c, c_ref)
        assert np.array_equal(c.val.view(np.int64), c_ref.val.view(np.int64))
        assert np.array_equal(oracle.compute_nprod(a, b)[0], oracle.ref_rpt_region(a, b, 1))
        assert np.array_equal(np.diff(c.rpt), oracle.ref_rpt_region(a, b, 2))
