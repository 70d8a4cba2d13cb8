// test_product_only.cpp -- a reference-API caller that links ONLY
// libspgemm_b200.so (no reference sources, no oracle): every function of the
// reference's headers it calls must be defined by the product. GPU cases run
// when SPGEMM_CPP_GPU=1 (tests/test_cpp_dropin.py sets it on the B200).
#include <cstdlib>
#include <cstring>
#include <vector>

#define DOCTEST_CONFIG_IMPLEMENT_WITH_MAIN
#include "doctest.h"
#include "spgemm/spgemm.hpp"

using namespace spgemm;

namespace {

bool gpu() {
  const char* v = std::getenv("SPGEMM_CPP_GPU");
  return v && std::strcmp(v, "1") == 0;
}

// 3-D 7-point Poisson on an n^3 grid (diag 6, off -1), natural order.
CsrMatrix poisson7(int n) {
  CooEntries coo{static_cast<std::int64_t>(n) * n * n, static_cast<std::int64_t>(n) * n * n, {}};
  auto id = [n](int x, int y, int z) { return (static_cast<std::int64_t>(z) * n + y) * n + x; };
  for (int z = 0; z < n; ++z)
    for (int y = 0; y < n; ++y)
      for (int x = 0; x < n; ++x) {
        const std::int64_t i = id(x, y, z);
        coo.entries.push_back({i, i, 6.0});
        const int d[6][3] = {{1, 0, 0}, {-1, 0, 0}, {0, 1, 0}, {0, -1, 0}, {0, 0, 1}, {0, 0, -1}};
        for (const auto& o : d) {
          const int X = x + o[0], Y = y + o[1], Z = z + o[2];
          if (X >= 0 && X < n && Y >= 0 && Y < n && Z >= 0 && Z < n) coo.entries.push_back({i, id(X, Y, Z), -1.0});
        }
      }
  return csr_from_coo(coo);
}

// 1-D-style aggregation prolongation: fine i -> coarse i/2 (weight 1) and
// (i+1)/2 for odd i (weight 1/2), rectangular.
CsrMatrix prolong(std::int64_t nf) {
  const std::int64_t nc = (nf + 1) / 2;
  CooEntries coo{nf, nc, {}};
  for (std::int64_t i = 0; i < nf; ++i) {
    coo.entries.push_back({i, i / 2, i % 2 == 0 ? 1.0 : 0.5});
    if (i % 2 == 1 && (i + 1) / 2 < nc) coo.entries.push_back({i, (i + 1) / 2, 0.5});
  }
  return csr_from_coo(coo);
}

CsrMatrix transpose(const CsrMatrix& m) {
  CooEntries coo = to_coo(m);
  for (auto& e : coo.entries) std::swap(e.row, e.col);
  std::swap(coo.rows, coo.cols);
  return csr_from_coo(coo);
}

bool bitwise(const CsrMatrix& x, const CsrMatrix& y) {
  return same_pattern(x, y) && std::memcmp(x.val.data(), y.val.data(), x.val.size() * sizeof(double)) == 0;
}

}  // namespace

TEST_CASE("input_stats and compression_ratio (reference.cpp:57-73)") {
  const CsrMatrix a = poisson7(4);
  const MatrixStats s = input_stats(a);
  CHECK(s.rows == 64);
  CHECK(s.nnz == a.nnz());
  CHECK(s.max_nnz_per_row == 7);
  CHECK(s.nnz_per_row_mean == doctest::Approx(static_cast<double>(a.nnz()) / 64.0));
  CHECK(compression_ratio(30, 10) == doctest::Approx(3.0));
  CHECK_THROWS_AS(compression_ratio(5, 0), std::domain_error);
}

TEST_CASE("csr utilities: coo round trip, validation, dense") {
  const CsrMatrix a = poisson7(3);
  CHECK(validate_csr(a).ok());
  CHECK(csr_from_coo(to_coo(a)) == a);
  CooEntries dup{2, 2, {{0, 1, 1.0}, {0, 1, 2.0}, {1, 0, 3.0}, {0, 1, 4.0}}};
  const CsrMatrix d = csr_from_coo(dup);
  CHECK(d.nnz() == 2);
  CHECK(d.val[0] == 7.0);
  CHECK(to_dense(d) == std::vector<double>({0.0, 7.0, 3.0, 0.0}));
}

TEST_CASE("compute_nprod on the device (reference.cpp:37-55)" * doctest::skip(!gpu())) {
  const CsrMatrix a = poisson7(5);
  std::vector<offset_t> out(static_cast<std::size_t>(a.rows));
  const offset_t total = compute_nprod(a, a, out);
  offset_t want = 0;
  for (std::int64_t i = 0; i < a.rows; ++i) {
    offset_t n = 0;
    for (offset_t p = a.rpt[static_cast<std::size_t>(i)]; p < a.rpt[static_cast<std::size_t>(i) + 1]; ++p)
      n += a.row_nnz(a.col[static_cast<std::size_t>(p)]);
    CHECK(out[static_cast<std::size_t>(i)] == n);
    want += n;
  }
  CHECK(total == want);
  std::vector<offset_t> short_out(3);
  CHECK_THROWS_AS(compute_nprod(a, a, short_out), std::invalid_argument);
}

TEST_CASE("reference_spgemm is the deterministic device product" * doctest::skip(!gpu())) {
  const CsrMatrix a = poisson7(6);
  const CsrMatrix c = reference_spgemm(a, a);
  CHECK(validate_csr(c).ok());
  CHECK(bitwise(c, multiply(a, a).c));
}

TEST_CASE("R*(A*P) chained on the device equals the host chain bitwise" * doctest::skip(!gpu())) {
  const CsrMatrix a = poisson7(8);
  const CsrMatrix p = prolong(a.rows);
  const CsrMatrix r = transpose(p);
  SpgemmOutput s1;
  const DeviceMatrix ap = multiply_device(a, p, SpgemmOptions{}, &s1);
  CHECK(ap.rows() == a.rows);
  CHECK(ap.cols() == p.cols);
  const DeviceMatrix rap = multiply_device(r, ap);  // AP never leaves HBM
  const CsrMatrix host_ap = multiply(a, p).c;
  const CsrMatrix host_rap = multiply(r, host_ap).c;
  CHECK(bitwise(ap.download(), host_ap));
  CHECK(bitwise(rap.download(), host_rap));
  CHECK(s1.stats.nnz_of_product == host_ap.nnz());
  const DeviceMatrix sq = multiply_device(ap, transpose(host_ap));  // device x host operands
  CHECK(bitwise(sq.download(), multiply(host_ap, transpose(host_ap)).c));
}
