// spgemm/reference.hpp -- statistics types of the reference (reference.hpp:1-36).
// reference_spgemm / compute_nprod / compression_ratio / input_stats are the
// reference's CPU oracle functions; this library does not implement them (it
// ships no CPU SpGEMM). Tests link them from the reference sources (oracle role);
// the device nprod kernel is exposed as spgemm_compute_nprod in spgemm_capi.h.
#pragma once

#include <span>

#include "spgemm/csr.hpp"

namespace spgemm {

CsrMatrix reference_spgemm(const CsrMatrix& a, const CsrMatrix& b);
offset_t compute_nprod(const CsrMatrix& a, const CsrMatrix& b, std::span<offset_t> out);
double compression_ratio(offset_t total_nprod, offset_t total_nnz);

struct MatrixStats {
  std::int64_t rows = 0;
  offset_t nnz = 0;
  double nnz_per_row_mean = 0.0;
  offset_t max_nnz_per_row = 0;
  offset_t total_nprod = 0;
  offset_t nnz_of_product = 0;
  double cr = 0.0;
};

MatrixStats input_stats(const CsrMatrix& a);

}  // namespace spgemm
