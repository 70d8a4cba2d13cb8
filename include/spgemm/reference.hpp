// spgemm/reference.hpp -- the reference's statistics and oracle entry points
// (reference.hpp:1-36), defined by libspgemm_b200 (cxx_api.cpp):
//   compute_nprod      kernel K1 on the device (spgemm_compute_nprod)
//   compression_ratio  nprod / nnz; std::domain_error when nnz <= 0
//   input_stats        host scan of the row pointers
//   reference_spgemm   the device product with default (deterministic)
//                      options: bitwise the reference's row-by-row oracle
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
