"""CPU: the C-ABI library loads, exports every symbol include/spgemm_capi.h declares,
and its host-side configuration entry points (presets, classify, execution plans)
match the reference (binning.cpp:33-82, pipeline.cpp:64-87). No device compute."""
import os
import re
import subprocess

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
HEADER = os.path.join(ROOT, "include", "spgemm_capi.h")


def declared_symbols():
    text = open(HEADER).read()
    text = re.sub(r"/\*.*?\*/", "", text, flags=re.S)
    return sorted(set(re.findall(r"\b(spgemm_[a-z_0-9]+)\s*\(", text)))


def test_library_exports_every_declared_symbol():
    from paper_2206_07244_b200 import _capi
    syms = declared_symbols()
    assert len(syms) >= 30
    for s in syms:
        assert hasattr(_capi.lib, s), s
    out = subprocess.run(["nm", "-D", "--defined-only", _capi.LIB_PATH], capture_output=True, text=True).stdout
    exported = set(re.findall(r" T (spgemm_\w+)", out))
    assert set(syms) <= exported
    assert set(_capi.EXPORTED) == set(syms)


def test_library_is_sm100a():
    from paper_2206_07244_b200 import _capi
    out = subprocess.run(["cuobjdump", "--list-elf", _capi.LIB_PATH], capture_output=True, text=True).stdout
    assert "sm_100a" in out


def test_presets_match_reference(sg, oracle):
    for phase in (sg.SYMBOLIC, sg.NUMERIC):
        for name in sg.preset_names(phase):
            c = sg.preset(phase, name)
            up, tab = oracle.preset(phase, name)
            assert c.upper == list(up) and c.table_size == list(tab) and c.preset_name == name
    with pytest.raises(sg.InvalidArgument):
        sg.symbolic_preset("sym_2x")
    with pytest.raises(sg.InvalidArgument):
        sg.numeric_preset("num_1.2x")


def test_classify_boundaries(sg):
    sym = sg.symbolic_preset("sym_1.2x")
    assert [sg.classify(v, sym) for v in (26, 27, 0, 10241, 10**9)] == [0, 1, 0, 7, 7]
    num = sg.numeric_preset("num_2x")
    assert [sg.classify(v, num) for v in (16, 17, 4096, 4097)] == [0, 1, 6, 7]


def test_execution_plans(sg):  # test_pipeline.cpp:47-68
    sym = sg.make_execution_plan(sg.symbolic_preset("sym_1.2x"))
    assert sym.launch_order() == [7, 6, 5, 4, 3, 2, 1, 0]
    for j, s in enumerate(sym.strategies):
        assert s.tier == "fixed"
        assert s.spill_threshold == (19660 if j == 7 else 0)
        if j > 0:
            assert s.metric_lo == sym.strategies[j - 1].metric_hi + 1
    assert sym.strategies[7].table_size == 24575
    num = sg.make_execution_plan(sg.numeric_preset("num_2x"))
    assert all(num.strategies[j].tier == "fixed" for j in range(7))
    assert num.strategies[7].tier == "heap" and num.strategies[7].spill_threshold == 0
    assert num.strategies[7].metric_lo == 4097
    assert sg.kSymbolicSpillThreshold == 19660


def test_every_finite_range_fits_its_table(sg):  # test_binning.cpp:78-92
    for phase in (sg.SYMBOLIC, sg.NUMERIC):
        for name in sg.preset_names(phase):
            c = sg.preset(phase, name)
            for j in range(8):
                if c.upper[j] != sg.kNoUpperBound and c.table_size[j] > 0:
                    assert c.table_size[j] >= c.upper[j]
                if j > 0:
                    assert c.upper[j] > c.upper[j - 1]


def test_no_gpu_fails_loudly_here(sg):
    from conftest import HAS_GPU
    if HAS_GPU:
        pytest.skip("GPU present")
    with pytest.raises(sg.NoDevice):
        sg.get_context()
    a = sg.CsrMatrix(2, 2, [0, 1, 2], [0, 1], [1.0, 1.0])
    with pytest.raises(sg.NoDevice):
        sg.multiply(a, a)


def test_new_entry_points_fail_loudly_without_gpu(sg):
    """forecast_nnz / multiply_into validate their arguments on the host and then refuse
    to run without an sm_100 device (no CPU fallback)."""
    from conftest import HAS_GPU
    if HAS_GPU:
        pytest.skip("GPU present")
    import numpy as np
    a = sg.CsrMatrix(2, 2, [0, 1, 2], [0, 1], [1.0, 1.0])
    b = sg.CsrMatrix(3, 2, [0, 1, 2, 2], [0, 1], [1.0, 1.0])
    with pytest.raises(sg.InvalidArgument):
        sg.forecast_nnz(a, b)  # a.cols != b.rows
    rpt, col, val = np.zeros(3, np.int64), np.zeros(4, np.int32), np.zeros(4)
    with pytest.raises(sg.InvalidArgument):
        sg.multiply_into(a, a, rpt.astype(np.int32), col, val)  # wrong rpt dtype
    with pytest.raises(sg.InvalidArgument):
        sg.multiply_into(a, a, np.zeros(2, np.int64), col, val)  # rpt too short
    with pytest.raises(sg.NoDevice):
        sg.multiply_into(a, a, rpt, col, val)
    with pytest.raises(sg.NoDevice):
        sg.forecast_nnz(a, a)


def test_validate_csr_reports_violations(sg):  # test_csr.cpp validation messages
    good = sg.CsrMatrix(2, 3, [0, 2, 3], [0, 2, 1], [1.0, 2.0, 3.0])
    assert sg.validate_csr(good).ok()
    bad = sg.CsrMatrix(2, 3, [0, 2, 3], [2, 0, 5], [1.0, 2.0, 3.0])
    rep = sg.validate_csr(bad)
    msgs = rep.to_string()
    assert "unsorted columns" in msgs and "out of range" in msgs
    dup = sg.CsrMatrix(1, 3, [0, 2], [1, 1], [1.0, 2.0])
    assert "duplicate column" in sg.validate_csr(dup).to_string()
