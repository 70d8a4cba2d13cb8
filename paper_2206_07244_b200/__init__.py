"""B200-native OpSparse SpGEMM (arXiv 2206.07244): C = A*B on CSR (int64 rpt, int32 col, fp64 val).

The product is the sm_100a library ``lib/libspgemm_b200.so`` behind the C ABI in
``include/spgemm_capi.h``; :mod:`.api` mirrors the reference's C++ API on top of it.
"""
from .api import (  # noqa: F401
    AllocStats, BinConfig, csr_from_coo_device, BinningResult, BinStrategy, Context, CsrMatrix, CudaError, DeviceMatrix,
    ExecutionPlan, InvalidArgument, LogicError, MatrixStats, NnzForecast, NoDevice, SpgemmOptions, SpgemmOutput,
    SpgemmPipeline, StepTimings, SYMBOLIC, NUMERIC, build_rpt, classify, compute_nprod, forecast_nnz,
    forecast_nnz_multi, get_context,
    kDefaultNumPreset, kDefaultSymPreset, kMaxSymbolicTableSize, kNoUpperBound, kNumBins,
    kSymbolicSpillThreshold, make_execution_plan, max_relative_error, multiply, multiply_device,
    multiply_into, multiply_multi, numeric_preset, preset, preset_names, run_binning, same_pattern, symbolic_preset, validate_csr,
)
