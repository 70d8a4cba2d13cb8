/*
 * spgemm_capi.h -- the drop-in boundary of the B200-native OpSparse SpGEMM.
 *
 * Plain C ABI (no C++ or torch types): pointers, sizes and POD structs. Every
 * entry point replaces one reference interface from
 * /root/reference/proj/core/include/spgemm (cited per function). The C++
 * drop-in headers in include/spgemm/*.hpp and the Python mirror in
 * paper_2206_07244_b200/api.py are thin layers over exactly these symbols;
 * INTEGRATION.md shows the binding a reference maintainer would add.
 *
 * Error convention: the reference throws (pipeline.hpp / binning.hpp); this
 * ABI never throws. Each call returns an spgemm_status whose value names the
 * exception type the reference would have thrown; spgemm_last_error() holds
 * the message (thread-local).
 *
 * Everything computes on the GPU (sm_100a kernels); there is no CPU fallback.
 */
#ifndef SPGEMM_CAPI_H_
#define SPGEMM_CAPI_H_

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define SPGEMM_NUM_BINS 8
#define SPGEMM_NO_UPPER_BOUND INT64_MAX

typedef enum spgemm_status {
  SPGEMM_OK = 0,
  SPGEMM_INVALID_ARGUMENT = 1, /* std::invalid_argument */
  SPGEMM_LOGIC_ERROR = 2,      /* std::logic_error      */
  SPGEMM_OVERFLOW = 3,         /* std::overflow_error   */
  SPGEMM_OUT_OF_MEMORY = 4,    /* std::bad_alloc        */
  SPGEMM_CUDA_ERROR = 5,
  SPGEMM_NCCL_ERROR = 6,
  SPGEMM_NO_DEVICE = 7
} spgemm_status;

typedef struct spgemm_ctx spgemm_ctx;           /* one (host thread, device) context  */
typedef struct spgemm_pipeline spgemm_pipeline; /* SpgemmPipeline (pipeline.hpp:119)  */
typedef struct spgemm_matrix spgemm_matrix;     /* device-resident CSR owned by the lib */

/* CsrMatrix (csr.hpp:45-63) as a borrowed view: rpt int64[rows+1], col
 * int32[rpt[rows]] strictly increasing per row, val fp64[rpt[rows]]. */
typedef struct spgemm_csr_view {
  int64_t rows;
  int64_t cols;
  const int64_t* rpt;
  const int32_t* col;
  const double* val;
  int32_t on_device; /* 1: the three pointers are device pointers on ctx's GPU */
} spgemm_csr_view;

/* SpgemmOptions (pipeline.hpp:78-91). */
typedef struct spgemm_options {
  char sym_preset[16];     /* "sym_1x" | "sym_1.2x" | "sym_1.5x"           */
  char num_preset[16];     /* "num_1x" | "num_1.5x" | "num_2x" | "num_3x"  */
  int32_t workers;         /* CPU pool size in the reference; reported only */
  int32_t overlap;         /* stream-ordered C allocation overlap on/off    */
  int32_t deterministic;   /* 1: C bitwise reproducible and equal to the
                              reference's summation order on every row
                              (SPEC.md:394); 0: heap-tier rows (bin 7) may
                              accumulate with fp64 atomics (within 1e-12)     */
  int64_t chunk_rows;      /* CPU task granularity in the reference; unused */
  int64_t hash_scale;      /* HashParams::hash_scale, positive odd          */
  int32_t has_sym_launch_order;
  int32_t sym_launch_order[SPGEMM_NUM_BINS];
  int32_t has_num_launch_order;
  int32_t num_launch_order[SPGEMM_NUM_BINS];
  int32_t ordered_heap;    /* B200 extension: 1 = heap-tier rows fold in the
                              reference's order even when deterministic = 0  */
} spgemm_options;

/* StepTimings (pipeline.hpp:93-102), seconds, measured with CUDA events. */
typedef struct spgemm_timings {
  double setup, sym_binning, symbolic, rpt_alloc, num_binning, numeric, cleanup, total;
} spgemm_timings;

/* SpgemmOutput minus the matrix (pipeline.hpp:104-110) + MatrixStats
 * (reference.hpp:23-31) + AllocStats counters (pipeline.hpp:45-50). */
typedef struct spgemm_report {
  int64_t rows;
  int64_t nnz;
  double nnz_per_row_mean;
  int64_t max_nnz_per_row;
  int64_t total_nprod;
  int64_t nnz_of_product;
  double cr;
  spgemm_timings timings;
  int64_t spilled_rows;
  int32_t workers;
  int64_t metadata_calls, metadata_bytes, output_calls, output_bytes;
} spgemm_report;

/* BinConfig (binning.hpp:29-34). phase 0 symbolic, 1 numeric. */
typedef struct spgemm_bin_config {
  int32_t phase;
  int64_t upper[SPGEMM_NUM_BINS];
  int64_t table_size[SPGEMM_NUM_BINS];
  char preset_name[16];
} spgemm_bin_config;

/* BinningResult scalars (binning.hpp:90-102). */
typedef struct spgemm_binning_info {
  int64_t bin_size[SPGEMM_NUM_BINS];
  int64_t bin_offset[SPGEMM_NUM_BINS];
  int64_t max_metric;
  int64_t total_metric;
  int32_t fast_path;
} spgemm_binning_info;

/* BinStrategy / ExecutionPlan (pipeline.hpp:21-39). tier 0 fixed, 1 heap. */
typedef struct spgemm_bin_strategy {
  int32_t bin;
  int64_t metric_lo, metric_hi, table_size;
  int32_t tier;
  int64_t spill_threshold;
  int32_t launch_rank;
} spgemm_bin_strategy;

typedef struct spgemm_plan {
  int32_t phase;
  spgemm_bin_config config;
  spgemm_bin_strategy strategies[SPGEMM_NUM_BINS];
  int32_t launch_order[SPGEMM_NUM_BINS];
} spgemm_plan;

/* ------------------------------------------------------------- context */
spgemm_status spgemm_ctx_create(int32_t device, spgemm_ctx** out);
void spgemm_ctx_destroy(spgemm_ctx* ctx);
const char* spgemm_last_error(void);
int32_t spgemm_ctx_device(const spgemm_ctx* ctx);
int32_t spgemm_ctx_num_sms(const spgemm_ctx* ctx);
/* Number of kernels this library launched on ctx since creation. */
int64_t spgemm_ctx_kernel_launches(const spgemm_ctx* ctx);
spgemm_status spgemm_ctx_synchronize(spgemm_ctx* ctx);
/* The stream all pipeline work is ordered on (cudaStream_t as void*). */
void* spgemm_ctx_stream(spgemm_ctx* ctx);

/* Per-kernel device time: when profiling is on, every launch is bracketed by
 * CUDA events on the stream it is launched on, and the per-bin kernels run in
 * order on the context's main stream (not concurrently) so each launch is timed
 * alone. The summary (aggregated by kernel name, then cleared) synchronises the
 * device. */
typedef struct spgemm_kernel_time {
  char name[48];
  int64_t launches;
  double total_ms;
} spgemm_kernel_time;
void spgemm_ctx_set_profiling(spgemm_ctx* ctx, int32_t on);
/* The context's private stream-ordered pool: bytes reserved from the driver / in use. */
spgemm_status spgemm_ctx_pool_stats(spgemm_ctx* ctx, uint64_t* reserved, uint64_t* used);
/* Gives the context's cached scratch (metadata arenas, staged inputs) back to
 * its private stream-ordered pool and trims the pool to keep_bytes of reserved
 * memory (synchronises the context's streams). */
spgemm_status spgemm_ctx_trim(spgemm_ctx* ctx, uint64_t keep_bytes);
int32_t spgemm_ctx_profile_summary(spgemm_ctx* ctx, spgemm_kernel_time* out, int32_t max);

/* ------------------------------------------------------- configuration */
void spgemm_options_default(spgemm_options* opts);
/* preset() (binning.cpp:33-66): INVALID_ARGUMENT for unknown names. */
spgemm_status spgemm_preset(int32_t phase, const char* name, spgemm_bin_config* out);
/* classify() (binning.cpp:75-82). */
int32_t spgemm_classify(int64_t value, const spgemm_bin_config* config);
/* make_execution_plan() (pipeline.cpp:64-87). */
spgemm_status spgemm_make_plan(const spgemm_bin_config* config, spgemm_plan* out);

/* --------------------------------------------------- SpgemmPipeline API */
/* SpgemmPipeline ctor (pipeline.cpp:109-134): validates shapes/options and
 * stages A and B in HBM (host views are copied, device views borrowed). */
spgemm_status spgemm_pipeline_create(spgemm_ctx* ctx, const spgemm_csr_view* a,
                                     const spgemm_csr_view* b, const spgemm_options* opts,
                                     spgemm_pipeline** out);
void spgemm_pipeline_destroy(spgemm_pipeline* p);
spgemm_status spgemm_pipeline_setup(spgemm_pipeline* p);            /* pipeline.cpp:152-220 */
spgemm_status spgemm_pipeline_symbolic_binning(spgemm_pipeline* p); /* pipeline.cpp:222-230 */
spgemm_status spgemm_pipeline_run_symbolic(spgemm_pipeline* p);     /* pipeline.cpp:232-239 */
spgemm_status spgemm_pipeline_numeric_binning(spgemm_pipeline* p);  /* pipeline.cpp:241-265 */
spgemm_status spgemm_pipeline_finalize_rpt(spgemm_pipeline* p, int64_t* total); /* :278-294 */
spgemm_status spgemm_pipeline_run_numeric(spgemm_pipeline* p);      /* pipeline.cpp:296-302 */
spgemm_status spgemm_pipeline_finish(spgemm_pipeline* p, spgemm_report* report); /* :435-462 */
spgemm_status spgemm_pipeline_run(spgemm_pipeline* p, spgemm_report* report);    /* :464-472 */
/* rpt_region() (pipeline.cpp:148-150): copies the M-slot region to host. */
spgemm_status spgemm_pipeline_rpt_region(spgemm_pipeline* p, int64_t* host_out);
/* binning() accessor: scalars, and the bins array (int64, M) when non-NULL. */
spgemm_status spgemm_pipeline_binning(spgemm_pipeline* p, spgemm_binning_info* info,
                                      int64_t* bins_host);
spgemm_status spgemm_pipeline_plan(spgemm_pipeline* p, int32_t phase, spgemm_plan* out);
/* After finish(): hands C (device-resident) to the caller. */
spgemm_status spgemm_pipeline_take_result(spgemm_pipeline* p, spgemm_matrix** c);

/* multiply() (pipeline.hpp:170-173): one-shot C = A*B, C stays on device. */
spgemm_status spgemm_multiply(spgemm_ctx* ctx, const spgemm_csr_view* a, const spgemm_csr_view* b,
                              const spgemm_options* opts, spgemm_matrix** c,
                              spgemm_report* report);

/* ------------------------------------------------------ result matrices */
void spgemm_matrix_shape(const spgemm_matrix* m, int64_t* rows, int64_t* cols, int64_t* nnz);
void spgemm_matrix_device_ptrs(const spgemm_matrix* m, const int64_t** rpt, const int32_t** col,
                               const double** val);
/* D2H of C into caller buffers (rows+1, nnz, nnz entries). */
spgemm_status spgemm_matrix_download(spgemm_ctx* ctx, const spgemm_matrix* m, int64_t* rpt,
                                     int32_t* col, double* val);
void spgemm_matrix_free(spgemm_matrix* m);
/* B200 extension: device-resident chaining (the reference's --b / RAP chain,
 * spgemm_bench_main.cpp:84, 130-135, without the host round trip). Fills a
 * device view (on_device = 1) of C that can be passed straight back as an
 * operand of spgemm_multiply / spgemm_pipeline_create. The view borrows C's
 * buffers: valid until spgemm_matrix_free or a releasing download. */
spgemm_status spgemm_matrix_as_operand(const spgemm_matrix* m, spgemm_csr_view* out);
/* Orders the context's next work after everything queued so far on `stream`
 * (a cudaStream_t; NULL = the legacy default stream), so device operands a
 * producer wrote on its own stream are complete before K1 reads them. */
spgemm_status spgemm_ctx_wait_stream(spgemm_ctx* ctx, void* stream);
/* B200 extension: stream-ordered D2H of C on the context's copy lane. Returns
 * at once; the copy starts when the work already queued on the context's
 * stream (the product) is done, so it overlaps the NEXT product's H2D and
 * kernels. release != 0 frees C's device buffers behind the copy (the handle
 * stays valid for spgemm_matrix_shape/_free). Host buffers should be pinned;
 * they must stay untouched until spgemm_ctx_wait_downloads() returns. */
spgemm_status spgemm_matrix_download_async(spgemm_ctx* ctx, spgemm_matrix* m, int64_t* rpt, int32_t* col,
                                           double* val, int32_t release);
spgemm_status spgemm_ctx_wait_downloads(spgemm_ctx* ctx);
/* B200 extension (streamed products, tiled.py): checksums of C on the device --
 * nnz, the sum of the values, and sum over entries of (col + col_offset + 1) *
 * (row + row_offset + 1) mod 2^64 -- without copying C to the host. */
spgemm_status spgemm_matrix_checksum(spgemm_ctx* ctx, const spgemm_matrix* m, int64_t row_offset,
                                     int64_t col_offset, double* val_sum, uint64_t* pattern_hash);

/* ------------------------------------------------ several GPUs, one process */
/* B200 extension (§8(b)'s spgemm_multiply_multi): C = A*B over
 * n contexts (normally one per device). A's rows are split into contiguous
 * blocks balanced by the prefix sum of per-row products (row_bounds[0..n]);
 * every context multiplies its block by all of B on its own host thread and
 * keeps its slice of C on its device (slices[0..n)). Host-resident operands
 * when n > 1. report: summed counts, the slowest block's timings. */
spgemm_status spgemm_multiply_multi(spgemm_ctx** ctxs, int32_t n, const spgemm_csr_view* a,
                                    const spgemm_csr_view* b, const spgemm_options* opts,
                                    spgemm_matrix** slices, int64_t* row_bounds, spgemm_report* report);
/* Downloads the slices of spgemm_multiply_multi into one host CSR (rows+1,
 * nnz, nnz entries), row pointers stitched with the slices' nnz offsets. */
spgemm_status spgemm_matrices_download_stitched(spgemm_ctx** ctxs, spgemm_matrix* const* slices, int32_t n,
                                                int64_t* rpt, int32_t* col, double* val);

/* ------------------------------------------- host in, host out, overlapped */
/* B200 extension: C = A*B from host operands into caller-provided host buffers
 * (rpt: a->rows + 1 entries; col/val: capacity entries -- size them with
 * spgemm_forecast_nnz or a previous product; pinned memory gives full PCIe
 * bandwidth). A and B are staged once; A's rows are split into `parts` blocks
 * by the nprod prefix sum (parts <= 0: chosen from the product's size), and
 * each block's C is downloaded on the copy lane while the next block is
 * multiplied, so the device->host transfer of C overlaps the kernels instead of
 * following them. Values and structure are those of spgemm_multiply (rows are
 * independent). *nnz receives nnz(C); SPGEMM_INVALID_ARGUMENT when C exceeds
 * the capacity (nothing past it is written). */
spgemm_status spgemm_multiply_into(spgemm_ctx* ctx, const spgemm_csr_view* a, const spgemm_csr_view* b,
                                   const spgemm_options* opts, int32_t parts, int64_t* rpt, int64_t capacity,
                                   int32_t* col, double* val, int64_t* nnz, spgemm_report* report);

/* ------------------------------------------------ symbolic-only sizing */
/* B200 extension: nnz(C) without computing or
 * allocating C -- the reference's step API run as setup + symbolic_binning +
 * run_symbolic and the row_ptr region read back (pipeline.cpp:152-239,
 * pipeline.hpp:190-201), here as one call. row_nnz (host, rows entries, may be
 * NULL) receives nnz(C(i,:)); total_nnz / total_nprod (may be NULL) the sums.
 * Device memory: the pipeline's O(rows) metadata only, so products whose C
 * exceeds HBM (BASELINE config 5) can be sized before they are committed. */
spgemm_status spgemm_forecast_nnz(spgemm_ctx* ctx, const spgemm_csr_view* a, const spgemm_csr_view* b,
                                  const spgemm_options* opts, int64_t* row_nnz, int64_t* total_nnz,
                                  int64_t* total_nprod);
/* The same over n contexts: rows split as in spgemm_multiply_multi (row_bounds
 * may be NULL), one host thread per context, host-resident operands. */
spgemm_status spgemm_forecast_nnz_multi(spgemm_ctx** ctxs, int32_t n, const spgemm_csr_view* a,
                                        const spgemm_csr_view* b, const spgemm_options* opts, int64_t* row_nnz,
                                        int64_t* row_bounds, int64_t* total_nnz, int64_t* total_nprod);

/* ----------------------------------------------- standalone GPU kernels */
/* csr_from_coo() (csr.cpp:12-72) on the device:
 * n triples (row, col, val) in input order -- host arrays, or device arrays
 * when on_device -- to a device CSR with each row's columns sorted and
 * duplicates summed in input order (the first as is, then +=). Errors as the
 * reference: negative shape, column count beyond 32 bits, an entry outside the
 * shape (INVALID_ARGUMENT with the reference's message). */
spgemm_status spgemm_csr_from_coo(spgemm_ctx* ctx, int64_t rows, int64_t cols, int64_t n, const int64_t* row,
                                  const int64_t* col, const double* val, int32_t on_device, spgemm_matrix** out);
/* compute_nprod() (reference.cpp:37-55) on the device: out[M] host or device. */
spgemm_status spgemm_compute_nprod(spgemm_ctx* ctx, const spgemm_csr_view* a,
                                   const spgemm_csr_view* b, int64_t* out_host,
                                   int64_t* total);
/* build_rpt() / exclusive_sum_inplace() (pipeline.cpp:104-107, binning.cpp:117-168):
 * in-place exclusive sum of n int64 host values on the GPU; returns total. */
spgemm_status spgemm_build_rpt(spgemm_ctx* ctx, int64_t* values_host, int64_t n, int64_t* total);
/* run_binning() (binning.cpp:281-313) on the device for a host metric. */
spgemm_status spgemm_run_binning(spgemm_ctx* ctx, const int64_t* metric_host, int64_t m,
                                 const spgemm_bin_config* config, int32_t deterministic,
                                 int64_t* bins_host, spgemm_binning_info* info);

#ifdef __cplusplus
}
#endif
#endif /* SPGEMM_CAPI_H_ */
