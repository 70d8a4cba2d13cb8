// ref_capi.cpp -- TEST INFRASTRUCTURE ONLY.
//
// extern "C" shim over the UNMODIFIED reference library
// (/root/reference/proj/core/src/*.cpp, compiled in place by oracle/Makefile
// with the reference's own Release flags plus -Dspgemm=spgemm_ref). It lets
// the Python tests and bench.py's reference arm drive the real CPU pipeline:
//   spgemm::multiply            pipeline.hpp:170-173
//   spgemm::reference_spgemm    reference.cpp:9-35
//   spgemm::random_csr          synthetic.cpp:46-63 (golden-vector generation)
//   SpgemmPipeline step API     pipeline.hpp:119-168
// Nothing here is linked into the product.
#include <cstdint>
#include <cstring>
#include <exception>
#include <random>
#include <stdexcept>
#include <string>

#include "spgemm/pipeline.hpp"
#include "spgemm/reference.hpp"
#include "spgemm/synthetic.hpp"

using spgemm_ref::CsrMatrix;

namespace {

thread_local std::string g_error;

CsrMatrix* to_csr(int64_t rows, int64_t cols, const int64_t* rpt, const int32_t* col,
                  const double* val) {
  auto* m = new CsrMatrix();
  m->rows = rows;
  m->cols = cols;
  m->rpt.assign(rpt, rpt + rows + 1);
  const int64_t nnz = rpt[rows];
  m->col.assign(col, col + nnz);
  m->val.assign(val, val + nnz);
  return m;
}

int fail(const std::exception& e, int code) {
  g_error = e.what();
  return code;
}

// 1 invalid_argument, 2 logic_error, 3 overflow_error, 4 other
int classify(const std::exception_ptr& ep) {
  try {
    std::rethrow_exception(ep);
  } catch (const std::invalid_argument& e) {
    return fail(e, 1);
  } catch (const std::overflow_error& e) {
    return fail(e, 3);
  } catch (const std::logic_error& e) {
    return fail(e, 2);
  } catch (const std::exception& e) {
    return fail(e, 4);
  }
}

}  // namespace

extern "C" {

const char* ref_last_error() { return g_error.c_str(); }

void* ref_csr_new(int64_t rows, int64_t cols, const int64_t* rpt, const int32_t* col,
                  const double* val) {
  return to_csr(rows, cols, rpt, col, val);
}

void ref_csr_free(void* h) { delete static_cast<CsrMatrix*>(h); }

void ref_csr_shape(void* h, int64_t* rows, int64_t* cols, int64_t* nnz) {
  auto* m = static_cast<CsrMatrix*>(h);
  *rows = m->rows;
  *cols = m->cols;
  *nnz = m->nnz();
}

void ref_csr_copy(void* h, int64_t* rpt, int32_t* col, double* val) {
  auto* m = static_cast<CsrMatrix*>(h);
  std::memcpy(rpt, m->rpt.data(), m->rpt.size() * sizeof(int64_t));
  std::memcpy(col, m->col.data(), m->col.size() * sizeof(int32_t));
  std::memcpy(val, m->val.data(), m->val.size() * sizeof(double));
}

void* ref_random_csr(int64_t rows, int64_t cols, double density, uint64_t seed) {
  std::mt19937_64 rng(seed);
  return new CsrMatrix(spgemm_ref::random_csr(rows, cols, density, rng));
}

void* ref_random_csr_fixed(int64_t rows, int64_t cols, int64_t per_row, uint64_t seed) {
  std::mt19937_64 rng(seed);
  return new CsrMatrix(spgemm_ref::random_csr_fixed_row_nnz(rows, cols, per_row, rng));
}

int ref_reference_spgemm(void* a, void* b, void** c) {
  try {
    *c = new CsrMatrix(
        spgemm_ref::reference_spgemm(*static_cast<CsrMatrix*>(a), *static_cast<CsrMatrix*>(b)));
    return 0;
  } catch (...) {
    return classify(std::current_exception());
  }
}

// Runs spgemm_ref::multiply. stats_out: [total_nprod, nnz_of_product,
// spilled_rows, workers, cr_bits]; times_out: the eight StepTimings fields.
int ref_multiply(void* a, void* b, const char* sym_preset, const char* num_preset, int workers,
                 int overlap, int deterministic, void** c, int64_t* stats_out, double* cr_out,
                 double* times_out) {
  try {
    spgemm_ref::SpgemmOptions o;
    o.sym_preset = sym_preset;
    o.num_preset = num_preset;
    o.workers = workers;
    o.overlap = overlap != 0;
    o.deterministic = deterministic != 0;
    spgemm_ref::SpgemmOutput out =
        spgemm_ref::multiply(*static_cast<CsrMatrix*>(a), *static_cast<CsrMatrix*>(b), o);
    stats_out[0] = out.stats.total_nprod;
    stats_out[1] = out.stats.nnz_of_product;
    stats_out[2] = out.spilled_rows;
    stats_out[3] = out.workers;
    *cr_out = out.stats.cr;
    const auto& t = out.timings;
    const double tv[8] = {t.setup, t.sym_binning, t.symbolic, t.rpt_alloc,
                          t.num_binning, t.numeric, t.cleanup, t.total};
    std::memcpy(times_out, tv, sizeof(tv));
    *c = new CsrMatrix(std::move(out.c));
    return 0;
  } catch (...) {
    return classify(std::current_exception());
  }
}

// Step API: region after setup() (stage 1) or after run_symbolic() (stage 2).
int ref_rpt_region(void* a, void* b, const char* sym_preset, int stage, int64_t* out) {
  try {
    spgemm_ref::SpgemmOptions o;
    o.sym_preset = sym_preset;
    spgemm_ref::SpgemmPipeline p(*static_cast<CsrMatrix*>(a), *static_cast<CsrMatrix*>(b), o);
    p.setup();
    if (stage >= 2) {
      p.symbolic_binning();
      p.run_symbolic();
    }
    const auto r = p.rpt_region();
    std::memcpy(out, r.data(), r.size() * sizeof(int64_t));
    return 0;
  } catch (...) {
    return classify(std::current_exception());
  }
}

// run_binning over a host metric (binning.cpp:281-313). out as in the C oracle.
int ref_run_binning(const int64_t* metric, int64_t m, int phase, const char* preset_name,
                    int deterministic, int64_t chunk, int64_t* bins, int64_t* out) {
  try {
    const auto cfg = spgemm_ref::preset(phase == 0 ? spgemm_ref::Phase::kSymbolic
                                                   : spgemm_ref::Phase::kNumeric,
                                        preset_name);
    std::vector<int64_t> size(8), offset(8);
    spgemm_ref::TaskPool pool(4);
    auto r = spgemm_ref::run_binning({metric, static_cast<size_t>(m)}, cfg,
                                     {bins, static_cast<size_t>(m)}, size, offset, &pool, chunk,
                                     deterministic != 0);
    for (int j = 0; j < 8; ++j) {
      out[j] = size[j];
      out[8 + j] = offset[j];
    }
    out[16] = r.max_metric;
    out[17] = r.total_metric;
    out[18] = r.fast_path ? 1 : 0;
    return 0;
  } catch (...) {
    return classify(std::current_exception());
  }
}

}  // extern "C"
