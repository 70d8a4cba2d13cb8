// spgemm/hash_tables.hpp -- the hashing parameters of the reference
// (hash_tables.hpp:11-27). The accumulator tables themselves live in shared /
// global memory inside the sm_100a kernels; only the public knobs remain.
#pragma once

#include <cstdint>

namespace spgemm {

inline constexpr std::int64_t kMaxSymbolicTableSize = 24575;
inline constexpr std::int64_t kMaxNumericTableSize = 8191;

inline constexpr std::int64_t spill_threshold_for(std::int64_t table_size) {
  return table_size * 4 / 5;
}
inline constexpr std::int64_t kSymbolicSpillThreshold = spill_threshold_for(kMaxSymbolicTableSize);

struct HashParams {
  std::int64_t hash_scale = 107;  // odd multiplier (std::invalid_argument otherwise)
};

inline constexpr std::int64_t kSpillSignal = -1;
inline constexpr std::int64_t kTableFullSignal = -1;

}  // namespace spgemm
