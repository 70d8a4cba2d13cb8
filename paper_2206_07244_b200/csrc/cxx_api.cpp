// cxx_api.cpp -- the reference's C++ API (include/spgemm/*.hpp) implemented over the
// C ABI of this library, so reference callers (and the reference's own
// test_pipeline.cpp) build unchanged against libspgemm_b200. Host-side container
// utilities (COO->CSR, validation, comparators) are plain C++; every SpGEMM,
// binning and scan step runs on the GPU through spgemm_capi.h.
#include <algorithm>
#include <cmath>
#include <cstdio>
#include <cstring>
#include <limits>
#include <map>
#include <new>
#include <numeric>
#include <sstream>
#include <stdexcept>
#include <string>

#include "spgemm/binning.hpp"
#include "spgemm/csr.hpp"
#include "spgemm/pipeline.hpp"
#include "spgemm/reference.hpp"
#include "spgemm_capi.h"

namespace spgemm {

namespace {

[[noreturn]] void rethrow(spgemm_status s) {
  const std::string m = spgemm_last_error();
  switch (s) {
    case SPGEMM_INVALID_ARGUMENT:
      throw std::invalid_argument(m);
    case SPGEMM_LOGIC_ERROR:
      throw std::logic_error(m);
    case SPGEMM_OVERFLOW:
      throw std::overflow_error(m);
    case SPGEMM_OUT_OF_MEMORY:
      throw std::bad_alloc();
    default:
      throw std::runtime_error(m);
  }
}

void ok(spgemm_status s) {
  if (s != SPGEMM_OK) rethrow(s);
}

// One context per (host thread, device), created on first use.
spgemm_ctx* ctx_for(int device) {
  struct Holder {
    std::map<int, spgemm_ctx*> by_dev;
    ~Holder() {
      for (auto& kv : by_dev) spgemm_ctx_destroy(kv.second);
    }
  };
  thread_local Holder h;
  auto it = h.by_dev.find(device);
  if (it != h.by_dev.end()) return it->second;
  spgemm_ctx* c = nullptr;
  ok(spgemm_ctx_create(device, &c));
  h.by_dev[device] = c;
  return c;
}

spgemm_csr_view view(const CsrMatrix& m) {
  if (m.rpt.size() != static_cast<std::size_t>(m.rows) + 1)
    throw std::invalid_argument("CsrMatrix: rpt length is not rows+1");
  return spgemm_csr_view{m.rows, m.cols, m.rpt.data(), m.col.data(), m.val.data(), 0};
}

spgemm_options to_c_options(const SpgemmOptions& options) {
  spgemm_options o;
  spgemm_options_default(&o);
  std::snprintf(o.sym_preset, sizeof(o.sym_preset), "%s", options.sym_preset.c_str());
  std::snprintf(o.num_preset, sizeof(o.num_preset), "%s", options.num_preset.c_str());
  o.workers = options.workers;
  o.overlap = options.overlap ? 1 : 0;
  o.deterministic = options.deterministic ? 1 : 0;
  o.chunk_rows = options.chunk_rows;
  o.hash_scale = options.hash.hash_scale;
  o.ordered_heap = options.ordered_heap ? 1 : 0;
  if (options.sym_launch_order) {
    o.has_sym_launch_order = 1;
    std::copy(options.sym_launch_order->begin(), options.sym_launch_order->end(), o.sym_launch_order);
  }
  if (options.num_launch_order) {
    o.has_num_launch_order = 1;
    std::copy(options.num_launch_order->begin(), options.num_launch_order->end(), o.num_launch_order);
  }
  return o;
}

spgemm_bin_config to_c(const BinConfig& c) {
  spgemm_bin_config out;
  std::memset(&out, 0, sizeof(out));
  out.phase = c.phase == Phase::kSymbolic ? 0 : 1;
  for (int j = 0; j < kNumBins; ++j) {
    out.upper[j] = c.upper[static_cast<std::size_t>(j)];
    out.table_size[j] = c.table_size[static_cast<std::size_t>(j)];
  }
  std::snprintf(out.preset_name, sizeof(out.preset_name), "%s", c.preset_name.c_str());
  return out;
}

BinConfig from_c(const spgemm_bin_config& c) {
  BinConfig out;
  out.phase = c.phase == 0 ? Phase::kSymbolic : Phase::kNumeric;
  for (int j = 0; j < kNumBins; ++j) {
    out.upper[static_cast<std::size_t>(j)] = c.upper[j];
    out.table_size[static_cast<std::size_t>(j)] = c.table_size[j];
  }
  out.preset_name = c.preset_name;
  return out;
}

ExecutionPlan from_c(const spgemm_plan& p) {
  ExecutionPlan out;
  out.phase = p.phase == 0 ? Phase::kSymbolic : Phase::kNumeric;
  out.config = from_c(p.config);
  for (int j = 0; j < kNumBins; ++j) {
    const spgemm_bin_strategy& s = p.strategies[j];
    BinStrategy& d = out.strategies[static_cast<std::size_t>(j)];
    d.bin = s.bin;
    d.metric_lo = s.metric_lo;
    d.metric_hi = s.metric_hi;
    d.table_size = s.table_size;
    d.tier = s.tier == 0 ? ScratchTier::kFixedArena : ScratchTier::kGrowableHeap;
    d.spill_threshold = s.spill_threshold;
    d.launch_rank = s.launch_rank;
  }
  return out;
}

}  // namespace

// ------------------------------------------------------------------- csr
// Host container utilities (csr.hpp). Semantics follow the reference
// (csr.cpp:12-181): the exception types and messages are part of the
// interface its tests check; the implementations are this library's own.
namespace {

void check_coo_shape(const CooEntries& coo) {
  if (coo.rows < 0 || coo.cols < 0) throw std::out_of_range("csr_from_coo: negative matrix shape");
  if (coo.cols > std::numeric_limits<index_t>::max())
    throw std::out_of_range("csr_from_coo: column count exceeds 32-bit index range");
  const auto outside = std::find_if(coo.entries.begin(), coo.entries.end(), [&](const CooEntry& e) {
    return static_cast<std::uint64_t>(e.row) >= static_cast<std::uint64_t>(coo.rows) ||
           static_cast<std::uint64_t>(e.col) >= static_cast<std::uint64_t>(coo.cols);
  });
  if (outside != coo.entries.end())
    throw std::out_of_range("csr_from_coo: entry (" + std::to_string(outside->row) + ", " +
                            std::to_string(outside->col) + ") outside " + std::to_string(coo.rows) + "x" +
                            std::to_string(coo.cols) + " shape");
}

}  // namespace

// One global stable order of the triples by (row, column): equal positions keep
// their file order, so a duplicate run folds left to right in input order.
CsrMatrix csr_from_coo(const CooEntries& coo) {
  check_coo_shape(coo);
  const auto& t = coo.entries;
  std::vector<std::size_t> order(t.size());
  std::iota(order.begin(), order.end(), std::size_t{0});
  std::stable_sort(order.begin(), order.end(), [&t](std::size_t x, std::size_t y) {
    return t[x].row != t[y].row ? t[x].row < t[y].row : t[x].col < t[y].col;
  });
  CsrMatrix m;
  m.rows = coo.rows;
  m.cols = coo.cols;
  m.rpt.assign(static_cast<std::size_t>(coo.rows) + 1, 0);
  m.col.reserve(t.size());
  m.val.reserve(t.size());
  std::int64_t last_row = -1;
  std::int64_t last_col = -1;
  for (const std::size_t idx : order) {
    const CooEntry& e = t[idx];
    if (e.row == last_row && e.col == last_col) {
      m.val.back() += e.value;
      continue;
    }
    m.col.push_back(static_cast<index_t>(e.col));
    m.val.push_back(e.value);
    ++m.rpt[static_cast<std::size_t>(e.row) + 1];
    last_row = e.row;
    last_col = e.col;
  }
  std::partial_sum(m.rpt.begin(), m.rpt.end(), m.rpt.begin());
  return m;
}

CooEntries to_coo(const CsrMatrix& m) {
  CooEntries coo{m.rows, m.cols, {}};
  coo.entries.resize(static_cast<std::size_t>(m.nnz()));
  std::int64_t row = 0;
  for (std::size_t p = 0; p < coo.entries.size(); ++p) {
    while (static_cast<offset_t>(p) >= m.rpt[static_cast<std::size_t>(row) + 1]) ++row;
    coo.entries[p] = CooEntry{row, m.col[p], m.val[p]};
  }
  return coo;
}

std::string ValidationReport::to_string() const {
  std::string text;
  for (const Violation& v : violations)
    text += (v.row >= 0 ? "row " + std::to_string(v.row) + ": " : std::string()) + v.message + "\n";
  return text;
}

ValidationReport validate_csr(const CsrMatrix& m) {
  ValidationReport report;
  auto& out = report.violations;
  if (m.rows < 0 || m.cols < 0) {
    out.push_back({-1, "negative matrix shape"});
    return report;
  }
  const auto rows = static_cast<std::size_t>(m.rows);
  if (m.rpt.size() != rows + 1) {
    out.push_back({-1, "rpt length is not rows+1"});
    return report;
  }
  // row pointers
  if (m.rpt.front() != 0) out.push_back({-1, "rpt[0] is not 0"});
  for (std::size_t i = 0; i < rows; ++i)
    if (m.rpt[i + 1] < m.rpt[i])
      out.push_back({static_cast<std::int64_t>(i), "non-monotone rpt at row " + std::to_string(i)});
  if (m.rpt.back() != static_cast<offset_t>(m.col.size())) out.push_back({-1, "rpt[rows] does not equal len(col)"});
  if (m.col.size() != m.val.size()) out.push_back({-1, "len(col) does not equal len(val)"});
  // columns of every row whose extent is readable (others were reported above)
  const auto readable = static_cast<offset_t>(std::min(m.col.size(), m.val.size()));
  for (std::size_t i = 0; i < rows; ++i) {
    const offset_t lo = m.rpt[i], hi = m.rpt[i + 1];
    if (lo < 0 || lo > hi || hi > readable) continue;
    const auto row = static_cast<std::int64_t>(i);
    index_t prev = -1;
    for (offset_t p = lo; p < hi; ++p) {
      const index_t c = m.col[static_cast<std::size_t>(p)];
      if (c < 0 || c >= m.cols) out.push_back({row, "column index " + std::to_string(c) + " out of range"});
      if (p == lo) {
        prev = c;
        continue;
      }
      if (c == prev) out.push_back({row, "duplicate column " + std::to_string(c)});
      if (c < prev)
        out.push_back({row, "unsorted columns (" + std::to_string(prev) + " before " + std::to_string(c) + ")"});
      prev = c;
    }
  }
  return report;
}

std::vector<double> to_dense(const CsrMatrix& m, std::int64_t max_cells) {
  const std::int64_t cells = m.rows * m.cols;
  if (cells > max_cells)
    throw std::length_error("to_dense: matrix exceeds the dense-expansion guard of " + std::to_string(max_cells) +
                            " cells");
  std::vector<double> dense(static_cast<std::size_t>(cells), 0.0);
  const CooEntries coo = to_coo(m);
  for (const CooEntry& e : coo.entries) dense[static_cast<std::size_t>(e.row * m.cols + e.col)] += e.value;
  return dense;
}

double max_relative_error(const CsrMatrix& a, const CsrMatrix& b) {
  if (!same_pattern(a, b)) throw std::invalid_argument("max_relative_error: patterns differ");
  // |x - y| / max(|x|, |y|, 1) (csr.cpp:169-181)
  return std::inner_product(a.val.begin(), a.val.end(), b.val.begin(), 0.0,
                            [](double acc, double e) { return std::max(acc, e); },
                            [](double x, double y) {
                              return std::fabs(x - y) / std::max(1.0, std::max(std::fabs(x), std::fabs(y)));
                            });
}

// -------------------------------------------------------------- reference.hpp
// The reference's statistics and oracle entry points (reference.cpp:9-73).
// compute_nprod runs kernel K1 on the device; reference_spgemm is the device
// product with the default (deterministic) options -- C bitwise equal to the
// reference's row-by-row oracle, whose summation order every numeric kernel keeps.
offset_t compute_nprod(const CsrMatrix& a, const CsrMatrix& b, std::span<offset_t> out) {
  if (a.cols != b.rows) throw std::invalid_argument("compute_nprod: a.cols != b.rows");
  if (out.size() != static_cast<std::size_t>(a.rows))
    throw std::invalid_argument("compute_nprod: out length != a.rows");
  const spgemm_csr_view va = view(a), vb = view(b);
  int64_t total = 0;
  ok(spgemm_compute_nprod(ctx_for(0), &va, &vb, out.data(), &total));
  return total;
}

double compression_ratio(offset_t total_nprod, offset_t total_nnz) {
  if (total_nnz <= 0) throw std::domain_error("compression_ratio: zero nnz");
  return static_cast<double>(total_nprod) / static_cast<double>(total_nnz);
}

MatrixStats input_stats(const CsrMatrix& a) {
  MatrixStats s;
  s.rows = a.rows;
  s.nnz = a.nnz();
  s.nnz_per_row_mean = a.rows > 0 ? static_cast<double>(s.nnz) / static_cast<double>(a.rows) : 0.0;
  for (std::size_t i = 1; i < a.rpt.size(); ++i) s.max_nnz_per_row = std::max(s.max_nnz_per_row, a.rpt[i] - a.rpt[i - 1]);
  return s;
}

CsrMatrix reference_spgemm(const CsrMatrix& a, const CsrMatrix& b) { return multiply(a, b).c; }

// --------------------------------------------------------------- binning
BinConfig preset(Phase phase, const std::string& name) {
  spgemm_bin_config c;
  ok(spgemm_preset(phase == Phase::kSymbolic ? 0 : 1, name.c_str(), &c));
  return from_c(c);
}

std::vector<std::string> preset_names(Phase phase) {
  if (phase == Phase::kSymbolic) return {"sym_1x", "sym_1.2x", "sym_1.5x"};
  return {"num_1x", "num_1.5x", "num_2x", "num_3x"};
}

int classify(std::int64_t value, const BinConfig& config) {
  const spgemm_bin_config c = to_c(config);
  return spgemm_classify(value, &c);
}

namespace {
spgemm_binning_info device_binning(std::span<const std::int64_t> metric, const BinConfig& config,
                                   bool deterministic, std::int64_t* bins) {
  const spgemm_bin_config c = to_c(config);
  spgemm_binning_info info;
  std::vector<std::int64_t> scratch;
  if (!bins) {
    scratch.resize(metric.size());
    bins = scratch.data();
  }
  ok(spgemm_run_binning(ctx_for(0), metric.data(), static_cast<std::int64_t>(metric.size()), &c,
                        deterministic ? 1 : 0, bins, &info));
  return info;
}
}  // namespace

Pass1Result binning_pass1(std::span<const std::int64_t> metric, const BinConfig& config, TaskPool*, std::int64_t) {
  Pass1Result r;
  if (metric.empty()) return r;
  const spgemm_binning_info info = device_binning(metric, config, true, nullptr);
  for (int j = 0; j < kNumBins; ++j) r.bin_size[static_cast<std::size_t>(j)] = info.bin_size[j];
  r.max_metric = info.max_metric;
  r.total_metric = info.total_metric;
  return r;
}

std::int64_t exclusive_sum_inplace(std::span<std::int64_t> buf, TaskPool*, std::span<std::int64_t>, std::int64_t) {
  if (buf.empty()) return 0;
  std::int64_t total = 0;
  ok(spgemm_build_rpt(ctx_for(0), buf.data(), static_cast<std::int64_t>(buf.size()), &total));
  return total;
}

std::vector<std::int64_t> exclusive_sum(std::span<const std::int64_t> counts) {
  std::vector<std::int64_t> out(counts.begin(), counts.end());
  exclusive_sum_inplace(out);
  return out;
}

void binning_pass2(std::span<const std::int64_t> metric, const BinConfig& config, std::span<const std::int64_t>,
                   std::span<std::int64_t> bins, TaskPool*, std::int64_t, bool deterministic) {
  if (metric.empty()) return;
  if (bins.size() != metric.size()) throw std::invalid_argument("binning_pass2: bad storage sizes");
  // The device scatter is the stable partition by bin that the reference's
  // deterministic pass 2 produces for offsets = exclusive_sum(bin sizes).
  device_binning(metric, config, deterministic, bins.data());
}

void binning_fast(std::span<std::int64_t> bins, TaskPool*, std::int64_t) {
  if (bins.empty()) return;
  const std::vector<std::int64_t> zeros(bins.size(), 0);
  device_binning(zeros, preset(Phase::kSymbolic, kDefaultSymPreset), true, bins.data());
}

BinningResult run_binning(std::span<const std::int64_t> metric, const BinConfig& config,
                          std::span<std::int64_t> bins, std::span<std::int64_t> bin_size,
                          std::span<std::int64_t> bin_offset, TaskPool*, std::int64_t, bool deterministic,
                          const Pass1Result*) {
  if (bins.size() != metric.size() || bin_size.size() != static_cast<std::size_t>(kNumBins) ||
      bin_offset.size() != static_cast<std::size_t>(kNumBins))
    throw std::invalid_argument("run_binning: bad storage sizes");
  BinningResult r;
  r.bins = bins;
  r.bin_size = bin_size;
  r.bin_offset = bin_offset;
  if (metric.empty()) {
    std::fill(bin_size.begin(), bin_size.end(), 0);
    std::fill(bin_offset.begin(), bin_offset.end(), 0);
    r.fast_path = true;
    return r;
  }
  const spgemm_binning_info info = device_binning(metric, config, deterministic, bins.data());
  for (int j = 0; j < kNumBins; ++j) {
    bin_size[static_cast<std::size_t>(j)] = info.bin_size[j];
    bin_offset[static_cast<std::size_t>(j)] = info.bin_offset[j];
  }
  r.max_metric = info.max_metric;
  r.total_metric = info.total_metric;
  r.fast_path = info.fast_path != 0;
  return r;
}

// -------------------------------------------------------------- pipeline
std::array<int, kNumBins> ExecutionPlan::launch_order() const {
  std::array<int, kNumBins> order{};
  std::iota(order.begin(), order.end(), 0);
  std::stable_sort(order.begin(), order.end(), [this](int x, int y) {
    return strategies[static_cast<std::size_t>(x)].launch_rank < strategies[static_cast<std::size_t>(y)].launch_rank;
  });
  return order;
}

ExecutionPlan make_execution_plan(const BinConfig& config) {
  const spgemm_bin_config c = to_c(config);
  spgemm_plan p;
  ok(spgemm_make_plan(&c, &p));
  return from_c(p);
}

offset_t build_rpt(std::span<offset_t> rpt_region, TaskPool* pool, std::span<std::int64_t> scratch) {
  return exclusive_sum_inplace(rpt_region, pool, scratch);
}

SpgemmPipeline::SpgemmPipeline(const CsrMatrix& a, const CsrMatrix& b, const SpgemmOptions& options)
    : a_(a),
      b_(b),
      options_(options),
      sym_plan_(make_execution_plan(symbolic_preset(options.sym_preset))),
      num_plan_(make_execution_plan(numeric_preset(options.num_preset))) {
  const spgemm_options o = to_c_options(options);
  if (a.cols != b.rows)
    throw std::invalid_argument("spgemm: a.cols (" + std::to_string(a.cols) + ") != b.rows (" +
                                std::to_string(b.rows) + ")");
  const spgemm_csr_view va = view(a), vb = view(b);
  ok(spgemm_pipeline_create(ctx_for(options.device), &va, &vb, &o, &handle_));
  spgemm_plan p;
  ok(spgemm_pipeline_plan(handle_, 0, &p));
  sym_plan_ = from_c(p);
  ok(spgemm_pipeline_plan(handle_, 1, &p));
  num_plan_ = from_c(p);
}

SpgemmPipeline::~SpgemmPipeline() { spgemm_pipeline_destroy(handle_); }

void SpgemmPipeline::setup() { ok(spgemm_pipeline_setup(handle_)); }
void SpgemmPipeline::symbolic_binning() { ok(spgemm_pipeline_symbolic_binning(handle_)); }
void SpgemmPipeline::run_symbolic() { ok(spgemm_pipeline_run_symbolic(handle_)); }
void SpgemmPipeline::numeric_binning() { ok(spgemm_pipeline_numeric_binning(handle_)); }
void SpgemmPipeline::run_numeric() { ok(spgemm_pipeline_run_numeric(handle_)); }

offset_t SpgemmPipeline::finalize_rpt() {
  std::int64_t total = 0;
  ok(spgemm_pipeline_finalize_rpt(handle_, &total));
  return total;
}

SpgemmOutput SpgemmPipeline::collect() {
  spgemm_report r;
  ok(spgemm_pipeline_finish(handle_, &r));
  spgemm_matrix* c = nullptr;
  ok(spgemm_pipeline_take_result(handle_, &c));
  SpgemmOutput out;
  std::int64_t rows = 0, cols = 0, nnz = 0;
  spgemm_matrix_shape(c, &rows, &cols, &nnz);
  out.c.rows = rows;
  out.c.cols = cols;
  out.c.rpt.resize(static_cast<std::size_t>(rows) + 1);
  out.c.col.resize(static_cast<std::size_t>(nnz));
  out.c.val.resize(static_cast<std::size_t>(nnz));
  const spgemm_status st = spgemm_matrix_download(ctx_for(options_.device), c, out.c.rpt.data(),
                                                  out.c.col.data(), out.c.val.data());
  spgemm_matrix_free(c);
  ok(st);
  out.stats = MatrixStats{r.rows, r.nnz, r.nnz_per_row_mean, r.max_nnz_per_row, r.total_nprod, r.nnz_of_product, r.cr};
  out.timings = StepTimings{r.timings.setup,       r.timings.sym_binning, r.timings.symbolic, r.timings.rpt_alloc,
                            r.timings.num_binning, r.timings.numeric,     r.timings.cleanup,  r.timings.total};
  out.spilled_rows = r.spilled_rows;
  out.workers = r.workers;
  if (options_.alloc_stats) {
    options_.alloc_stats->metadata_calls += r.metadata_calls;
    options_.alloc_stats->metadata_bytes += r.metadata_bytes;
    options_.alloc_stats->output_calls += r.output_calls;
    options_.alloc_stats->output_bytes += r.output_bytes;
  }
  return out;
}

SpgemmOutput SpgemmPipeline::finish() { return collect(); }

// ------------------------------------------------------ device-resident chain
DeviceMatrix& DeviceMatrix::operator=(DeviceMatrix&& o) noexcept {
  if (this != &o) {
    if (handle_) spgemm_matrix_free(handle_);
    handle_ = o.handle_;
    device_ = o.device_;
    o.handle_ = nullptr;
  }
  return *this;
}

DeviceMatrix::~DeviceMatrix() {
  if (handle_) spgemm_matrix_free(handle_);
}

namespace {
struct Shape {
  std::int64_t rows = 0, cols = 0, nnz = 0;
};
Shape shape_of(const spgemm_matrix* h) {
  Shape s;
  if (h) spgemm_matrix_shape(h, &s.rows, &s.cols, &s.nnz);
  return s;
}
}  // namespace

std::int64_t DeviceMatrix::rows() const { return shape_of(handle_).rows; }
std::int64_t DeviceMatrix::cols() const { return shape_of(handle_).cols; }
offset_t DeviceMatrix::nnz() const { return shape_of(handle_).nnz; }

CsrMatrix DeviceMatrix::download() const {
  if (!handle_) throw std::logic_error("DeviceMatrix: empty");
  const Shape sh = shape_of(handle_);
  CsrMatrix m;
  m.rows = sh.rows;
  m.cols = sh.cols;
  m.rpt.resize(static_cast<std::size_t>(sh.rows) + 1);
  m.col.resize(static_cast<std::size_t>(sh.nnz));
  m.val.resize(static_cast<std::size_t>(sh.nnz));
  ok(spgemm_matrix_download(ctx_for(device_), handle_, m.rpt.data(), m.col.data(), m.val.data()));
  return m;
}

DeviceMatrix multiply_device(const Operand& a, const Operand& b, const SpgemmOptions& options,
                             SpgemmOutput* stats) {
  auto operand_view = [&](const Operand& x) {
    if (x.host()) return view(*x.host());
    const DeviceMatrix* d = x.device_matrix();
    if (!d || !d->handle()) throw std::invalid_argument("multiply_device: empty device operand");
    if (d->device() != options.device)
      throw std::invalid_argument("multiply_device: operand lives on another device than options.device");
    spgemm_csr_view v;
    ok(spgemm_matrix_as_operand(d->handle(), &v));
    return v;
  };
  const spgemm_csr_view va = operand_view(a), vb = operand_view(b);
  const spgemm_options o = to_c_options(options);
  spgemm_matrix* c = nullptr;
  spgemm_report r;
  ok(spgemm_multiply(ctx_for(options.device), &va, &vb, &o, &c, &r));
  if (stats) {
    stats->stats = MatrixStats{r.rows, r.nnz, r.nnz_per_row_mean, r.max_nnz_per_row, r.total_nprod, r.nnz_of_product,
                               r.cr};
    stats->timings = StepTimings{r.timings.setup,       r.timings.sym_binning, r.timings.symbolic, r.timings.rpt_alloc,
                                 r.timings.num_binning, r.timings.numeric,     r.timings.cleanup,  r.timings.total};
    stats->spilled_rows = r.spilled_rows;
    stats->workers = r.workers;
  }
  return DeviceMatrix(c, options.device);
}

SpgemmOutput SpgemmPipeline::run() {
  setup();
  symbolic_binning();
  run_symbolic();
  numeric_binning();
  finalize_rpt();
  run_numeric();
  return collect();
}

std::span<const offset_t> SpgemmPipeline::rpt_region() const {
  region_.resize(static_cast<std::size_t>(a_.rows));
  ok(spgemm_pipeline_rpt_region(handle_, region_.data()));
  return {region_.data(), region_.size()};
}

const BinningResult& SpgemmPipeline::binning() const {
  spgemm_binning_info info;
  bins_.resize(static_cast<std::size_t>(a_.rows));
  ok(spgemm_pipeline_binning(handle_, &info, bins_.empty() ? nullptr : bins_.data()));
  for (int j = 0; j < kNumBins; ++j) {
    bin_size_[static_cast<std::size_t>(j)] = info.bin_size[j];
    bin_offset_[static_cast<std::size_t>(j)] = info.bin_offset[j];
  }
  binning_.bins = {bins_.data(), bins_.size()};
  binning_.bin_size = {bin_size_.data(), bin_size_.size()};
  binning_.bin_offset = {bin_offset_.data(), bin_offset_.size()};
  binning_.max_metric = info.max_metric;
  binning_.total_metric = info.total_metric;
  binning_.fast_path = info.fast_path != 0;
  return binning_;
}

SpgemmOutput multiply_multi(const CsrMatrix& a, const CsrMatrix& b, const SpgemmOptions& options,
                            const std::vector<int>& devices) {
  if (devices.empty()) throw std::invalid_argument("multiply_multi: no devices");
  if (a.cols != b.rows)
    throw std::invalid_argument("spgemm: a.cols (" + std::to_string(a.cols) + ") != b.rows (" +
                                std::to_string(b.rows) + ")");
  // one fresh context per entry (a context serves one host thread at a time)
  std::vector<spgemm_ctx*> ctxs;
  struct Release {
    std::vector<spgemm_ctx*>& c;
    ~Release() {
      for (spgemm_ctx* x : c) spgemm_ctx_destroy(x);
    }
  } release{ctxs};
  for (int d : devices) {
    spgemm_ctx* c = nullptr;
    ok(spgemm_ctx_create(d, &c));
    ctxs.push_back(c);
  }
  const int n = static_cast<int>(ctxs.size());
  const spgemm_options o = to_c_options(options);
  const spgemm_csr_view va = view(a), vb = view(b);
  std::vector<spgemm_matrix*> slices(static_cast<std::size_t>(n), nullptr);
  std::vector<std::int64_t> bounds(static_cast<std::size_t>(n) + 1, 0);
  spgemm_report r;
  ok(spgemm_multiply_multi(ctxs.data(), n, &va, &vb, &o, slices.data(), bounds.data(), &r));
  SpgemmOutput out;
  out.c.rows = a.rows;
  out.c.cols = b.cols;
  out.c.rpt.resize(static_cast<std::size_t>(a.rows) + 1);
  out.c.col.resize(static_cast<std::size_t>(r.nnz_of_product));
  out.c.val.resize(static_cast<std::size_t>(r.nnz_of_product));
  const spgemm_status st = spgemm_matrices_download_stitched(ctxs.data(), slices.data(), n, out.c.rpt.data(),
                                                             out.c.col.data(), out.c.val.data());
  for (spgemm_matrix* m : slices) spgemm_matrix_free(m);
  ok(st);
  out.stats = MatrixStats{r.rows, r.nnz, r.nnz_per_row_mean, r.max_nnz_per_row, r.total_nprod, r.nnz_of_product, r.cr};
  out.timings = StepTimings{r.timings.setup,       r.timings.sym_binning, r.timings.symbolic, r.timings.rpt_alloc,
                            r.timings.num_binning, r.timings.numeric,     r.timings.cleanup,  r.timings.total};
  out.spilled_rows = r.spilled_rows;
  out.workers = r.workers;
  return out;
}

NnzForecast forecast_nnz(const CsrMatrix& a, const CsrMatrix& b, const SpgemmOptions& options,
                         const std::vector<int>& devices, bool per_row) {
  if (devices.empty()) throw std::invalid_argument("forecast_nnz: no devices");
  if (a.cols != b.rows)
    throw std::invalid_argument("spgemm: a.cols (" + std::to_string(a.cols) + ") != b.rows (" +
                                std::to_string(b.rows) + ")");
  std::vector<spgemm_ctx*> ctxs;
  struct Release {
    std::vector<spgemm_ctx*>& c;
    ~Release() {
      for (spgemm_ctx* x : c) spgemm_ctx_destroy(x);
    }
  } release{ctxs};
  for (int d : devices) {
    spgemm_ctx* c = nullptr;
    ok(spgemm_ctx_create(d, &c));
    ctxs.push_back(c);
  }
  const int n = static_cast<int>(ctxs.size());
  const spgemm_options o = to_c_options(options);
  const spgemm_csr_view va = view(a), vb = view(b);
  NnzForecast f;
  if (per_row) f.row_nnz.resize(static_cast<std::size_t>(a.rows));
  f.row_bounds.resize(static_cast<std::size_t>(n) + 1);
  ok(spgemm_forecast_nnz_multi(ctxs.data(), n, &va, &vb, &o, per_row && a.rows ? f.row_nnz.data() : nullptr,
                               f.row_bounds.data(), &f.total_nnz, &f.total_nprod));
  return f;
}

std::int64_t multiply_into(const CsrMatrix& a, const CsrMatrix& b, offset_t* rpt, index_t* col, double* val,
                           std::int64_t capacity, const SpgemmOptions& options, int parts) {
  spgemm_ctx* ctx = ctx_for(0);
  const spgemm_options o = to_c_options(options);
  const spgemm_csr_view va = view(a), vb = view(b);
  std::int64_t nnz = 0;
  ok(spgemm_multiply_into(ctx, &va, &vb, &o, parts, rpt, capacity, col, val, &nnz, nullptr));
  return nnz;
}

}  // namespace spgemm
