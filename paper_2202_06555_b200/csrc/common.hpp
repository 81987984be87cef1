// Shared host/device helpers: heap-key arithmetic, error plumbing.
//
// Heap-key packing follows /root/reference/proj/include/ddsg/grid_index.hpp:1-44:
// a 1-d node (l, i), l >= 1, i odd in [1, 2^l - 1], is hk = 2^(l-1) + (i-1)/2;
// level_of = bit_width(hk), index_of = 2(hk - 2^(l-1)) + 1, coordinate = i 2^-l.
#pragma once

#include <cmath>
#include <cstdint>
#include <stdexcept>
#include <string>
#include <vector>

#include "../../include/ddsg_b200.h"

namespace ddsg_b200 {

constexpr int kMaxLevel = 30;  // grid_index.hpp:32

inline int level_of(uint32_t hk) { return hk == 0 ? 0 : 32 - __builtin_clz(hk); }
inline uint32_t cell_of(uint32_t hk) {  // (i-1)/2, the cell index within the level
  const int l = level_of(hk);
  return hk - (uint32_t{1} << (l - 1));
}
inline uint32_t index_of(uint32_t hk) { return 2u * cell_of(hk) + 1u; }
inline double coordinate_of(uint32_t hk) {
  const int l = level_of(hk);
  return static_cast<double>(index_of(hk)) * std::ldexp(1.0, -l);
}
inline bool valid_key(uint32_t hk) { return hk >= 1u && level_of(hk) <= kMaxLevel; }

// Error carrying a ddsg_status; converted to a return code at the C-ABI.
struct Error : std::runtime_error {
  ddsg_status status;
  Error(ddsg_status s, const std::string& msg) : std::runtime_error(msg), status(s) {}
};

[[noreturn]] inline void fail(ddsg_status s, const std::string& msg) { throw Error(s, msg); }

// Build failure carrying the offending point (sparse_grid.hpp:40-48).
struct BuildError : Error {
  std::vector<double> point;
  BuildError(const std::string& msg, std::vector<double> p)
      : Error(DDSG_BUILD_ERROR, msg), point(std::move(p)) {}
};

}  // namespace ddsg_b200
