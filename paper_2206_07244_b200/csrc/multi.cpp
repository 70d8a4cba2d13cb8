// multi.cpp -- one process, several B200s: row-block data parallelism behind the
// C ABI (the `spgemm_multiply_multi` entry of §8(b)'s ABI
// proposal). Written purely over the public C ABI (no CUDA calls of its own):
//
//   1. per-row products of A (kernel K1 on the first device) and the
//      nprod-prefix row split -- contiguous row blocks, rows never split;
//   2. every device multiplies its row block by all of B on its own host
//      thread (its own context, streams and HBM; B is staged to each device
//      over its own link);
//   3. C stays distributed as one device-resident slice per device; the row
//      pointers are stitched from the slices' nnz totals when C is downloaded
//      (spgemm_matrices_download_stitched) -- no further exchange.
//   4. symbolic-only sizing (spgemm_forecast_nnz_multi):
//      the same split, every device counting its block's nnz(C) without
//      allocating C, so a TB-scale product is sized before it is committed.
//
// The torch.distributed path (paper_2206_07244_b200/distributed.py) is the same
// decomposition with one process per GPU and an NCCL broadcast of B.
#include <algorithm>
#include <cstring>
#include <string>
#include <thread>
#include <vector>

#include "spgemm_capi.h"

extern "C" void spgemm_internal_set_error(const char* msg);  // capi.cu (thread-local message)

namespace {

struct Block {
  int64_t r0 = 0, r1 = 0;
  std::vector<int64_t> rpt;  // rebased row pointers of the block
  spgemm_csr_view view{};
  spgemm_status status = SPGEMM_OK;
  std::string error;
  spgemm_report report{};
};

// nprod (K1 on ctxs[0]) and the balanced contiguous row split into row_bounds[0..n]
spgemm_status split_rows(spgemm_ctx* ctx, int32_t n, const spgemm_csr_view* a, const spgemm_csr_view* b,
                         int64_t* row_bounds) {
  std::vector<int64_t> nprod(static_cast<size_t>(std::max<int64_t>(a->rows, 0)));
  int64_t total = 0;
  spgemm_status st = spgemm_compute_nprod(ctx, a, b, nprod.data(), &total);
  if (st != SPGEMM_OK) return st;
  row_bounds[0] = 0;
  int64_t acc = 0, row = 0;
  for (int32_t g = 1; g < n; ++g) {
    const int64_t target = total > 0 ? static_cast<int64_t>((static_cast<__int128>(total) * g) / n) : 0;
    // first row whose exclusive prefix reaches the target
    while (row < a->rows && acc < target) acc += nprod[static_cast<size_t>(row++)];
    row_bounds[g] = total > 0 ? row : (a->rows * g) / n;
    if (row_bounds[g] < row_bounds[g - 1]) row_bounds[g] = row_bounds[g - 1];
  }
  row_bounds[n] = a->rows;
  return SPGEMM_OK;
}

// rows [r0, r1) of a host CSR view, row pointers rebased into bl.rpt
void make_block(const spgemm_csr_view* a, int64_t r0, int64_t r1, Block& bl) {
  bl.r0 = r0;
  bl.r1 = r1;
  const int64_t p0 = a->rpt[r0];
  bl.rpt.resize(static_cast<size_t>(r1 - r0 + 1));
  for (int64_t r = r0; r <= r1; ++r) bl.rpt[static_cast<size_t>(r - r0)] = a->rpt[r] - p0;
  bl.view = spgemm_csr_view{r1 - r0, a->cols, bl.rpt.data(), a->col ? a->col + p0 : nullptr,
                            a->val ? a->val + p0 : nullptr, 0};
}

// runs work(i) for i in [0, n): i = 0 on the calling thread, the rest on their own
template <typename F>
void run_parallel(int32_t n, F work) {
  std::vector<std::thread> threads;
  for (int32_t i = 1; i < n; ++i) threads.emplace_back(work, i);
  work(0);
  for (auto& t : threads) t.join();
}

spgemm_status invalid(const char* msg) {
  spgemm_internal_set_error(msg);
  return SPGEMM_INVALID_ARGUMENT;
}

}  // namespace

extern "C" {

spgemm_status spgemm_multiply_multi(spgemm_ctx** ctxs, int32_t n, const spgemm_csr_view* a,
                                    const spgemm_csr_view* b, const spgemm_options* opts,
                                    spgemm_matrix** slices, int64_t* row_bounds, spgemm_report* report) {
  if (n < 1 || !ctxs || !a || !b || !slices || !row_bounds)
    return invalid("spgemm_multiply_multi: null argument or no devices");
  for (int32_t i = 0; i < n; ++i) slices[i] = nullptr;
  if (n == 1) {
    row_bounds[0] = 0;
    row_bounds[1] = a->rows;
    return spgemm_multiply(ctxs[0], a, b, opts, &slices[0], report);
  }
  if (n > 1 && (a->on_device || b->on_device)) {
    // blocks are staged from host memory to every device; device-resident
    // operands would need peer copies (use the per-GPU process path instead)
    return invalid("spgemm_multiply_multi: operands must be host-resident when n > 1");
  }
  if (a->cols != b->rows) return invalid("spgemm: a.cols != b.rows");
  // 1. nprod per row (K1) and the balanced split
  spgemm_status st = split_rows(ctxs[0], n, a, b, row_bounds);
  if (st != SPGEMM_OK) return st;
  // 2. one host thread per device
  std::vector<Block> blocks(static_cast<size_t>(n));
  for (int32_t i = 0; i < n; ++i) make_block(a, row_bounds[i], row_bounds[i + 1], blocks[static_cast<size_t>(i)]);
  run_parallel(n, [&](int32_t i) {
    Block& bl = blocks[static_cast<size_t>(i)];
    bl.status = spgemm_multiply(ctxs[i], &bl.view, b, opts, &slices[i], &bl.report);
    if (bl.status != SPGEMM_OK) bl.error = spgemm_last_error();
  });
  for (int32_t i = 0; i < n; ++i) {
    const Block& bl = blocks[static_cast<size_t>(i)];
    if (bl.status != SPGEMM_OK) {
      for (int32_t j = 0; j < n; ++j) {
        spgemm_matrix_free(slices[j]);
        slices[j] = nullptr;
      }
      spgemm_internal_set_error(("device block " + std::to_string(i) + ": " + bl.error).c_str());
      return bl.status;
    }
  }
  // 3. the combined report: sums of the counts, the slowest block's timings
  if (report) {
    spgemm_report r = blocks[0].report;
    r.rows = a->rows;
    r.nnz = a->rpt[a->rows];
    r.nnz_per_row_mean = a->rows > 0 ? static_cast<double>(r.nnz) / static_cast<double>(a->rows) : 0.0;
    r.total_nprod = 0;
    r.nnz_of_product = 0;
    r.spilled_rows = 0;
    for (const Block& bl : blocks) {
      r.total_nprod += bl.report.total_nprod;
      r.nnz_of_product += bl.report.nnz_of_product;
      r.spilled_rows += bl.report.spilled_rows;
      r.max_nnz_per_row = std::max(r.max_nnz_per_row, bl.report.max_nnz_per_row);
      if (bl.report.timings.total > r.timings.total) r.timings = bl.report.timings;
    }
    r.cr = r.nnz_of_product > 0 ? static_cast<double>(r.total_nprod) / static_cast<double>(r.nnz_of_product) : 0.0;
    r.workers = n;
    *report = r;
  }
  return SPGEMM_OK;
}

spgemm_status spgemm_matrices_download_stitched(spgemm_ctx** ctxs, spgemm_matrix* const* slices, int32_t n,
                                                int64_t* rpt, int32_t* col, double* val) {
  if (n < 1 || !ctxs || !slices || !rpt) return invalid("spgemm_matrices_download_stitched: null argument");
  int64_t row = 0, off = 0;
  for (int32_t i = 0; i < n; ++i) {
    int64_t rows = 0, cols = 0, nnz = 0;
    spgemm_matrix_shape(slices[i], &rows, &cols, &nnz);
    // the slice's rpt lands at rpt[row..row+rows]; its first entry (0) is
    // overwritten by the running offset, then the slice is rebased
    const int64_t keep = row > 0 ? rpt[row] : 0;
    spgemm_status st = spgemm_matrix_download(ctxs[i], slices[i], rpt + row, col ? col + off : nullptr,
                                              val ? val + off : nullptr);
    if (st != SPGEMM_OK) return st;
    for (int64_t r = 0; r <= rows; ++r) rpt[row + r] += off;
    if (row > 0 && rpt[row] != keep) {
      spgemm_internal_set_error("spgemm_matrices_download_stitched: slice offsets disagree");
      return SPGEMM_LOGIC_ERROR;
    }
    row += rows;
    off += nnz;
  }
  return SPGEMM_OK;
}

spgemm_status spgemm_forecast_nnz_multi(spgemm_ctx** ctxs, int32_t n, const spgemm_csr_view* a,
                                        const spgemm_csr_view* b, const spgemm_options* opts, int64_t* row_nnz,
                                        int64_t* row_bounds, int64_t* total_nnz, int64_t* total_nprod) {
  if (n < 1 || !ctxs || !a || !b) return invalid("spgemm_forecast_nnz_multi: null argument or no devices");
  if (n == 1) {
    if (row_bounds) {
      row_bounds[0] = 0;
      row_bounds[1] = a->rows;
    }
    return spgemm_forecast_nnz(ctxs[0], a, b, opts, row_nnz, total_nnz, total_nprod);
  }
  if (a->on_device || b->on_device)
    return invalid("spgemm_forecast_nnz_multi: operands must be host-resident when n > 1");
  if (a->cols != b->rows) return invalid("spgemm: a.cols != b.rows");
  std::vector<int64_t> bounds(static_cast<size_t>(n) + 1);
  spgemm_status st = split_rows(ctxs[0], n, a, b, bounds.data());
  if (st != SPGEMM_OK) return st;
  if (row_bounds) std::copy(bounds.begin(), bounds.end(), row_bounds);
  std::vector<Block> blocks(static_cast<size_t>(n));
  std::vector<int64_t> nnz(static_cast<size_t>(n), 0), np(static_cast<size_t>(n), 0);
  for (int32_t i = 0; i < n; ++i) make_block(a, bounds[i], bounds[i + 1], blocks[static_cast<size_t>(i)]);
  run_parallel(n, [&](int32_t i) {
    Block& bl = blocks[static_cast<size_t>(i)];
    if (bl.r1 == bl.r0) return;
    bl.status = spgemm_forecast_nnz(ctxs[i], &bl.view, b, opts, row_nnz ? row_nnz + bl.r0 : nullptr,
                                    &nnz[static_cast<size_t>(i)], &np[static_cast<size_t>(i)]);
    if (bl.status != SPGEMM_OK) bl.error = spgemm_last_error();
  });
  int64_t tn = 0, tp = 0;
  for (int32_t i = 0; i < n; ++i) {
    const Block& bl = blocks[static_cast<size_t>(i)];
    if (bl.status != SPGEMM_OK) {
      spgemm_internal_set_error(("device block " + std::to_string(i) + ": " + bl.error).c_str());
      return bl.status;
    }
    tn += nnz[static_cast<size_t>(i)];
    tp += np[static_cast<size_t>(i)];
  }
  if (total_nnz) *total_nnz = tn;
  if (total_nprod) *total_nprod = tp;
  return SPGEMM_OK;
}

}  // extern "C"
