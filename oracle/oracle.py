"""ctypes access to the test-only checkers. TEST INFRASTRUCTURE ONLY.

Two libraries, both built by ``oracle/Makefile``:

* ``liboracle.so`` -- the plain-C restatement (``spgemm_oracle.c``) of the
  reference CPU path. Always buildable (gcc only); this is the oracle used on
  the GPU box, where ``/root/reference`` does not exist.
* ``_ref/libspgemm_ref.so`` -- the unmodified reference core compiled in place
  from ``/root/reference/proj/core/src``. Used (when present) to pin the
  restatement and as the CPU baseline (``bench.py --impl reference``).

Only ``tests/``, ``__graft_entry__.smoke()`` and ``bench.py``'s cpu-baseline /
reference leg import this module. Matrices are passed as any object with
``rows, cols, rpt (int64), col (int32), val (float64)`` attributes.
"""
from __future__ import annotations

import ctypes as C
import os
import subprocess
from types import SimpleNamespace

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
ORACLE_SO = os.path.join(HERE, "liboracle.so")
REF_SO = os.path.join(HERE, "_ref", "libspgemm_ref.so")

_i64p = np.ctypeslib.ndpointer(np.int64, flags="C_CONTIGUOUS")
_i32p = np.ctypeslib.ndpointer(np.int32, flags="C_CONTIGUOUS")
_f64p = np.ctypeslib.ndpointer(np.float64, flags="C_CONTIGUOUS")

_oracle = None
_ref = None


def build_oracle() -> None:
    """Compile liboracle.so (and _ref when /root/reference is present)."""
    targets = ["oracle"]
    if os.path.isdir("/root/reference/proj/core/src"):
        targets.append("ref")
    subprocess.run(["make", "-s", "-C", HERE, *targets], check=True)


def oracle_lib():
    global _oracle
    if _oracle is None:
        if not os.path.exists(ORACLE_SO):
            subprocess.run(["make", "-s", "-C", HERE, "oracle"], check=True)
        lib = C.CDLL(ORACLE_SO)
        lib.oracle_compute_nprod.restype = C.c_int64
        lib.oracle_compute_nprod.argtypes = [C.c_int64, _i64p, _i32p, _i64p, _i64p]
        lib.oracle_spgemm_symbolic.restype = C.c_int64
        lib.oracle_spgemm_symbolic.argtypes = [C.c_int64, C.c_int64, _i64p, _i32p, _i64p, _i32p, _i64p]
        lib.oracle_spgemm_numeric.restype = C.c_int
        lib.oracle_spgemm_numeric.argtypes = [C.c_int64, C.c_int64, _i64p, _i32p, _f64p, _i64p, _i32p,
                                              _f64p, _i64p, _i32p, _f64p]
        lib.oracle_preset.restype = C.c_int
        lib.oracle_preset.argtypes = [C.c_int, C.c_char_p, _i64p, _i64p]
        lib.oracle_classify.restype = C.c_int
        lib.oracle_classify.argtypes = [C.c_int64, _i64p]
        lib.oracle_exclusive_sum.restype = C.c_int64
        lib.oracle_exclusive_sum.argtypes = [_i64p, C.c_int64]
        lib.oracle_run_binning.restype = None
        lib.oracle_run_binning.argtypes = [_i64p, C.c_int64, _i64p, _i64p, _i64p]
        lib.oracle_spilled_rows.restype = C.c_int64
        lib.oracle_spilled_rows.argtypes = [_i64p, _i64p, C.c_int64, _i64p]
        lib.oracle_max_relative_error.restype = C.c_double
        lib.oracle_max_relative_error.argtypes = [_f64p, _f64p, C.c_int64]
        _oracle = lib
    return _oracle


def ref_available() -> bool:
    return os.path.exists(REF_SO)


def ref_lib():
    global _ref
    if _ref is None:
        if not ref_available():
            raise RuntimeError(f"{REF_SO} not built (needs /root/reference; run make -C oracle ref)")
        lib = C.CDLL(REF_SO)
        lib.ref_last_error.restype = C.c_char_p
        lib.ref_csr_new.restype = C.c_void_p
        lib.ref_csr_new.argtypes = [C.c_int64, C.c_int64, _i64p, _i32p, _f64p]
        lib.ref_csr_free.argtypes = [C.c_void_p]
        lib.ref_csr_shape.argtypes = [C.c_void_p, C.POINTER(C.c_int64), C.POINTER(C.c_int64),
                                      C.POINTER(C.c_int64)]
        lib.ref_csr_copy.argtypes = [C.c_void_p, _i64p, _i32p, _f64p]
        lib.ref_random_csr.restype = C.c_void_p
        lib.ref_random_csr.argtypes = [C.c_int64, C.c_int64, C.c_double, C.c_uint64]
        lib.ref_random_csr_fixed.restype = C.c_void_p
        lib.ref_random_csr_fixed.argtypes = [C.c_int64, C.c_int64, C.c_int64, C.c_uint64]
        lib.ref_reference_spgemm.restype = C.c_int
        lib.ref_reference_spgemm.argtypes = [C.c_void_p, C.c_void_p, C.POINTER(C.c_void_p)]
        lib.ref_multiply.restype = C.c_int
        lib.ref_multiply.argtypes = [C.c_void_p, C.c_void_p, C.c_char_p, C.c_char_p, C.c_int, C.c_int,
                                     C.c_int, C.POINTER(C.c_void_p), _i64p, C.POINTER(C.c_double), _f64p]
        lib.ref_rpt_region.restype = C.c_int
        lib.ref_rpt_region.argtypes = [C.c_void_p, C.c_void_p, C.c_char_p, C.c_int, _i64p]
        lib.ref_run_binning.restype = C.c_int
        lib.ref_run_binning.argtypes = [_i64p, C.c_int64, C.c_int, C.c_char_p, C.c_int, C.c_int64, _i64p,
                                        _i64p]
        _ref = lib
    return _ref


def _arrays(m):
    return (np.ascontiguousarray(m.rpt, np.int64), np.ascontiguousarray(m.col, np.int32),
            np.ascontiguousarray(m.val, np.float64))


def csr(rows, cols, rpt, col, val):
    """Minimal CSR record used by the checkers."""
    return SimpleNamespace(rows=int(rows), cols=int(cols), rpt=np.ascontiguousarray(rpt, np.int64),
                           col=np.ascontiguousarray(col, np.int32), val=np.ascontiguousarray(val, np.float64))


# ------------------------------------------------------------ C restatement
def compute_nprod(a, b):
    """reference.cpp:37-55. Returns (per-row nprod int64[M], total)."""
    ar, ac, _ = _arrays(a)
    br, _, _ = _arrays(b)
    out = np.empty(a.rows, np.int64)
    total = oracle_lib().oracle_compute_nprod(a.rows, ar, ac, br, out)
    return out, int(total)


def spgemm(a, b):
    """reference.cpp:9-35, bitwise the reference's values. Returns a CSR record."""
    if a.cols != b.rows:
        raise ValueError("reference_spgemm: a.cols != b.rows")
    lib = oracle_lib()
    ar, ac, av = _arrays(a)
    br, bc, bv = _arrays(b)
    rpt = np.empty(a.rows + 1, np.int64)
    nnz = lib.oracle_spgemm_symbolic(a.rows, b.cols, ar, ac, br, bc, rpt)
    if nnz < 0:
        raise MemoryError("oracle scratch allocation failed")
    col = np.empty(nnz, np.int32)
    val = np.empty(nnz, np.float64)
    rc = lib.oracle_spgemm_numeric(a.rows, b.cols, ar, ac, av, br, bc, bv, rpt, col, val)
    if rc != 0:
        raise RuntimeError(f"oracle numeric failed ({rc})")
    return csr(a.rows, b.cols, rpt, col, val)


def preset(phase: int, name: str):
    upper = np.empty(8, np.int64)
    table = np.empty(8, np.int64)
    if oracle_lib().oracle_preset(phase, name.encode(), upper, table) != 0:
        raise ValueError(f"unknown binning preset '{name}'")
    return upper, table


def classify(value: int, upper) -> int:
    return oracle_lib().oracle_classify(int(value), np.ascontiguousarray(upper, np.int64))


def exclusive_sum(counts):
    buf = np.array(counts, dtype=np.int64, copy=True)
    total = oracle_lib().oracle_exclusive_sum(buf, buf.size)
    return buf, int(total)


def run_binning(metric, upper):
    """binning.cpp:281-313 (deterministic). Returns dict like the reference's BinningResult."""
    metric = np.ascontiguousarray(metric, np.int64)
    bins = np.empty(metric.size, np.int64)
    out = np.empty(19, np.int64)
    oracle_lib().oracle_run_binning(metric, metric.size, np.ascontiguousarray(upper, np.int64), bins, out)
    return dict(bins=bins, bin_size=out[0:8].copy(), bin_offset=out[8:16].copy(), max_metric=int(out[16]),
                total_metric=int(out[17]), fast_path=bool(out[18]))


def spilled_rows(nprod, nnz, sym_upper) -> int:
    return int(oracle_lib().oracle_spilled_rows(np.ascontiguousarray(nprod, np.int64),
                                                np.ascontiguousarray(nnz, np.int64), len(nprod),
                                                np.ascontiguousarray(sym_upper, np.int64)))


def same_pattern(x, y) -> bool:
    """csr.hpp:105-107."""
    return (x.rows == y.rows and x.cols == y.cols and np.array_equal(x.rpt, y.rpt)
            and np.array_equal(x.col, y.col))


def max_relative_error(x, y) -> float:
    """csr.cpp:169-181."""
    if not same_pattern(x, y):
        raise ValueError("max_relative_error: patterns differ")
    xv = np.ascontiguousarray(x.val, np.float64)
    yv = np.ascontiguousarray(y.val, np.float64)
    return float(oracle_lib().oracle_max_relative_error(xv, yv, xv.size))


# ------------------------------------------------------- real reference (_ref)
class RefError(RuntimeError):
    def __init__(self, code, msg):
        super().__init__(msg)
        self.code = code


def _ref_check(lib, rc):
    if rc != 0:
        raise RefError(rc, lib.ref_last_error().decode())


def _ref_new(m):
    r, c, v = _arrays(m)
    return ref_lib().ref_csr_new(m.rows, m.cols, r, c, v)


def _ref_take(h):
    lib = ref_lib()
    rows, cols, nnz = C.c_int64(), C.c_int64(), C.c_int64()
    lib.ref_csr_shape(h, C.byref(rows), C.byref(cols), C.byref(nnz))
    rpt = np.empty(rows.value + 1, np.int64)
    col = np.empty(nnz.value, np.int32)
    val = np.empty(nnz.value, np.float64)
    lib.ref_csr_copy(h, rpt, col, val)
    lib.ref_csr_free(h)
    return csr(rows.value, cols.value, rpt, col, val)


def ref_random_csr(rows, cols, density, seed):
    """synthetic.cpp:46-63 with std::mt19937_64(seed) (libstdc++ distributions)."""
    return _ref_take(ref_lib().ref_random_csr(rows, cols, density, seed))


def ref_random_csr_fixed(rows, cols, per_row, seed):
    return _ref_take(ref_lib().ref_random_csr_fixed(rows, cols, per_row, seed))


def ref_reference_spgemm(a, b):
    lib = ref_lib()
    ha, hb = _ref_new(a), _ref_new(b)
    out = C.c_void_p()
    try:
        _ref_check(lib, lib.ref_reference_spgemm(ha, hb, C.byref(out)))
    finally:
        lib.ref_csr_free(ha)
        lib.ref_csr_free(hb)
    return _ref_take(out)


def ref_multiply(a, b, sym_preset="sym_1.2x", num_preset="num_2x", workers=0, overlap=True,
                 deterministic=True):
    """The reference's own pipeline (pipeline.hpp:170-173). Returns (C, info dict)."""
    lib = ref_lib()
    ha = _ref_new(a)
    hb = ha if b is a else _ref_new(b)
    out = C.c_void_p()
    stats = np.zeros(5, np.int64)
    cr = C.c_double()
    times = np.zeros(8, np.float64)
    try:
        _ref_check(lib, lib.ref_multiply(ha, hb, sym_preset.encode(), num_preset.encode(), workers,
                                         int(overlap), int(deterministic), C.byref(out), stats,
                                         C.byref(cr), times))
    finally:
        lib.ref_csr_free(ha)
        if hb != ha:
            lib.ref_csr_free(hb)
    info = dict(total_nprod=int(stats[0]), nnz_of_product=int(stats[1]), spilled_rows=int(stats[2]),
                workers=int(stats[3]), cr=cr.value, timings=times)
    return _ref_take(out), info


def ref_rpt_region(a, b, stage, sym_preset="sym_1.2x"):
    lib = ref_lib()
    ha, hb = _ref_new(a), _ref_new(b)
    out = np.empty(a.rows, np.int64)
    try:
        _ref_check(lib, lib.ref_rpt_region(ha, hb, sym_preset.encode(), stage, out))
    finally:
        lib.ref_csr_free(ha)
        lib.ref_csr_free(hb)
    return out


def ref_run_binning(metric, phase, preset_name, deterministic=True, chunk=4096):
    lib = ref_lib()
    metric = np.ascontiguousarray(metric, np.int64)
    bins = np.empty(metric.size, np.int64)
    out = np.empty(19, np.int64)
    _ref_check(lib, lib.ref_run_binning(metric, metric.size, phase, preset_name.encode(),
                                        int(deterministic), chunk, bins, out))
    return dict(bins=bins, bin_size=out[0:8].copy(), bin_offset=out[8:16].copy(), max_metric=int(out[16]),
                total_metric=int(out[17]), fast_path=bool(out[18]))
