"""ctypes declarations of include/spgemm_capi.h (the C-ABI boundary).

Loads the in-tree ``lib/libspgemm_b200.so``; there is no fallback: if the
library is missing this module raises at import time.
"""
from __future__ import annotations

import ctypes as C
import os

import importlib.util as _ilu

# build.py is loaded by path so that it never depends on the library itself
_spec = _ilu.spec_from_file_location("_spgemm_build", os.path.join(os.path.dirname(__file__), "build.py"))
_build = _ilu.module_from_spec(_spec)
_spec.loader.exec_module(_build)

NUM_BINS = 8
NO_UPPER_BOUND = (1 << 63) - 1

OK, INVALID_ARGUMENT, LOGIC_ERROR, OVERFLOW, OUT_OF_MEMORY, CUDA_ERROR, NCCL_ERROR, NO_DEVICE = range(8)


class CsrView(C.Structure):
    _fields_ = [("rows", C.c_int64), ("cols", C.c_int64), ("rpt", C.c_void_p), ("col", C.c_void_p),
                ("val", C.c_void_p), ("on_device", C.c_int32)]


class Options(C.Structure):
    _fields_ = [("sym_preset", C.c_char * 16), ("num_preset", C.c_char * 16), ("workers", C.c_int32),
                ("overlap", C.c_int32), ("deterministic", C.c_int32), ("chunk_rows", C.c_int64),
                ("hash_scale", C.c_int64), ("has_sym_launch_order", C.c_int32),
                ("sym_launch_order", C.c_int32 * NUM_BINS), ("has_num_launch_order", C.c_int32),
                ("num_launch_order", C.c_int32 * NUM_BINS), ("ordered_heap", C.c_int32)]


class Timings(C.Structure):
    _fields_ = [(n, C.c_double) for n in
                ("setup", "sym_binning", "symbolic", "rpt_alloc", "num_binning", "numeric", "cleanup",
                 "total")]


class Report(C.Structure):
    _fields_ = [("rows", C.c_int64), ("nnz", C.c_int64), ("nnz_per_row_mean", C.c_double),
                ("max_nnz_per_row", C.c_int64), ("total_nprod", C.c_int64), ("nnz_of_product", C.c_int64),
                ("cr", C.c_double), ("timings", Timings), ("spilled_rows", C.c_int64), ("workers", C.c_int32),
                ("metadata_calls", C.c_int64), ("metadata_bytes", C.c_int64), ("output_calls", C.c_int64),
                ("output_bytes", C.c_int64)]


class BinConfig(C.Structure):
    _fields_ = [("phase", C.c_int32), ("upper", C.c_int64 * NUM_BINS), ("table_size", C.c_int64 * NUM_BINS),
                ("preset_name", C.c_char * 16)]


class BinningInfo(C.Structure):
    _fields_ = [("bin_size", C.c_int64 * NUM_BINS), ("bin_offset", C.c_int64 * NUM_BINS),
                ("max_metric", C.c_int64), ("total_metric", C.c_int64), ("fast_path", C.c_int32)]


class BinStrategy(C.Structure):
    _fields_ = [("bin", C.c_int32), ("metric_lo", C.c_int64), ("metric_hi", C.c_int64),
                ("table_size", C.c_int64), ("tier", C.c_int32), ("spill_threshold", C.c_int64),
                ("launch_rank", C.c_int32)]


class KernelTime(C.Structure):
    _fields_ = [("name", C.c_char * 48), ("launches", C.c_int64), ("total_ms", C.c_double)]


class Plan(C.Structure):
    _fields_ = [("phase", C.c_int32), ("config", BinConfig), ("strategies", BinStrategy * NUM_BINS),
                ("launch_order", C.c_int32 * NUM_BINS)]


LIB_PATH = _build.LIB
if not os.path.exists(LIB_PATH):
    raise ImportError(f"{LIB_PATH} is missing: build it with `python paper_2206_07244_b200/build.py` "
                      "(the CUDA library is the only implementation; there is no CPU fallback)")

lib = C.CDLL(LIB_PATH)
_P = C.c_void_p
_st = C.c_int


def _decl(name, res, args):
    f = getattr(lib, name)
    f.restype = res
    f.argtypes = args


_decl("spgemm_last_error", C.c_char_p, [])
_decl("spgemm_ctx_create", _st, [C.c_int32, C.POINTER(_P)])
_decl("spgemm_ctx_destroy", None, [_P])
_decl("spgemm_ctx_device", C.c_int32, [_P])
_decl("spgemm_ctx_num_sms", C.c_int32, [_P])
_decl("spgemm_ctx_kernel_launches", C.c_int64, [_P])
_decl("spgemm_ctx_synchronize", _st, [_P])
_decl("spgemm_ctx_stream", _P, [_P])
_decl("spgemm_ctx_set_profiling", None, [_P, C.c_int32])
_decl("spgemm_ctx_profile_summary", C.c_int32, [_P, C.POINTER(KernelTime), C.c_int32])
_decl("spgemm_ctx_pool_stats", _st, [_P, C.POINTER(C.c_uint64), C.POINTER(C.c_uint64)])
_decl("spgemm_options_default", None, [C.POINTER(Options)])
_decl("spgemm_preset", _st, [C.c_int32, C.c_char_p, C.POINTER(BinConfig)])
_decl("spgemm_classify", C.c_int32, [C.c_int64, C.POINTER(BinConfig)])
_decl("spgemm_make_plan", _st, [C.POINTER(BinConfig), C.POINTER(Plan)])
_decl("spgemm_pipeline_create", _st, [_P, C.POINTER(CsrView), C.POINTER(CsrView), C.POINTER(Options),
                                      C.POINTER(_P)])
_decl("spgemm_pipeline_destroy", None, [_P])
for _n in ("setup", "symbolic_binning", "run_symbolic", "numeric_binning", "run_numeric"):
    _decl(f"spgemm_pipeline_{_n}", _st, [_P])
_decl("spgemm_pipeline_finalize_rpt", _st, [_P, C.POINTER(C.c_int64)])
_decl("spgemm_pipeline_finish", _st, [_P, C.POINTER(Report)])
_decl("spgemm_pipeline_run", _st, [_P, C.POINTER(Report)])
_decl("spgemm_pipeline_rpt_region", _st, [_P, _P])
_decl("spgemm_pipeline_binning", _st, [_P, C.POINTER(BinningInfo), _P])
_decl("spgemm_pipeline_plan", _st, [_P, C.c_int32, C.POINTER(Plan)])
_decl("spgemm_pipeline_take_result", _st, [_P, C.POINTER(_P)])
_decl("spgemm_multiply", _st, [_P, C.POINTER(CsrView), C.POINTER(CsrView), C.POINTER(Options), C.POINTER(_P),
                               C.POINTER(Report)])
_decl("spgemm_matrix_shape", None, [_P, C.POINTER(C.c_int64), C.POINTER(C.c_int64), C.POINTER(C.c_int64)])
_decl("spgemm_matrix_device_ptrs", None, [_P, C.POINTER(_P), C.POINTER(_P), C.POINTER(_P)])
_decl("spgemm_matrix_download", _st, [_P, _P, _P, _P, _P])
_decl("spgemm_matrix_free", None, [_P])
_decl("spgemm_matrix_as_operand", _st, [_P, C.POINTER(CsrView)])
_decl("spgemm_ctx_trim", _st, [_P, C.c_uint64])
_decl("spgemm_csr_from_coo", _st, [_P, C.c_int64, C.c_int64, C.c_int64, _P, _P, _P, C.c_int32, C.POINTER(_P)])
_decl("spgemm_ctx_wait_stream", _st, [_P, _P])
_decl("spgemm_matrix_checksum", _st, [_P, _P, C.c_int64, C.c_int64, _P, _P])
_decl("spgemm_matrix_download_async", _st, [_P, _P, _P, _P, _P, C.c_int32])
_decl("spgemm_ctx_wait_downloads", _st, [_P])
_decl("spgemm_multiply_multi", _st, [_P, C.c_int32, _P, _P, _P, _P, _P, _P])
_decl("spgemm_matrices_download_stitched", _st, [_P, _P, C.c_int32, _P, _P, _P])
_decl("spgemm_compute_nprod", _st, [_P, C.POINTER(CsrView), C.POINTER(CsrView), _P, C.POINTER(C.c_int64)])
_decl("spgemm_multiply_into", _st, [_P, C.POINTER(CsrView), C.POINTER(CsrView), _P, C.c_int32, _P, C.c_int64,
                                    _P, _P, C.POINTER(C.c_int64), C.POINTER(Report)])
_decl("spgemm_forecast_nnz", _st, [_P, C.POINTER(CsrView), C.POINTER(CsrView), _P, _P, C.POINTER(C.c_int64),
                                   C.POINTER(C.c_int64)])
_decl("spgemm_forecast_nnz_multi", _st, [_P, C.c_int32, C.POINTER(CsrView), C.POINTER(CsrView), _P, _P, _P,
                                         C.POINTER(C.c_int64), C.POINTER(C.c_int64)])
_decl("spgemm_build_rpt", _st, [_P, _P, C.c_int64, C.POINTER(C.c_int64)])
_decl("spgemm_run_binning", _st, [_P, _P, C.c_int64, C.POINTER(BinConfig), C.c_int32, _P,
                                  C.POINTER(BinningInfo)])

EXPORTED = [
    "spgemm_ctx_create", "spgemm_ctx_destroy", "spgemm_last_error", "spgemm_ctx_device", "spgemm_ctx_num_sms",
    "spgemm_ctx_kernel_launches", "spgemm_ctx_synchronize", "spgemm_ctx_stream", "spgemm_ctx_set_profiling",
    "spgemm_ctx_profile_summary", "spgemm_ctx_pool_stats", "spgemm_options_default",
    "spgemm_preset", "spgemm_classify", "spgemm_make_plan", "spgemm_pipeline_create", "spgemm_pipeline_destroy",
    "spgemm_pipeline_setup", "spgemm_pipeline_symbolic_binning", "spgemm_pipeline_run_symbolic",
    "spgemm_pipeline_numeric_binning", "spgemm_pipeline_finalize_rpt", "spgemm_pipeline_run_numeric",
    "spgemm_pipeline_finish", "spgemm_pipeline_run", "spgemm_pipeline_rpt_region", "spgemm_pipeline_binning",
    "spgemm_pipeline_plan", "spgemm_pipeline_take_result", "spgemm_multiply", "spgemm_matrix_shape",
    "spgemm_matrix_device_ptrs", "spgemm_matrix_download", "spgemm_matrix_free", "spgemm_matrix_checksum",
    "spgemm_matrix_download_async", "spgemm_ctx_wait_downloads", "spgemm_multiply_multi",
    "spgemm_matrices_download_stitched", "spgemm_compute_nprod", "spgemm_forecast_nnz", "spgemm_forecast_nnz_multi",
    "spgemm_multiply_into", "spgemm_matrix_as_operand", "spgemm_ctx_wait_stream", "spgemm_ctx_trim",
    "spgemm_csr_from_coo",
    "spgemm_build_rpt", "spgemm_run_binning",
]


def last_error() -> str:
    return lib.spgemm_last_error().decode(errors="replace")
