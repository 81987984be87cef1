// Device-side 1-d basis values, bit-identical to the reference.
//
// Reference: basis_kind / basis_value (basis.hpp:27-54) with inv_h = 2^l and
// center = i / inv_h; the weight of a node is the dim-ordered product
// w = ((1 * v_0) * v_1) * ... with an early exit on w == 0
// (sparse_grid.hpp:116-122).
//
// Exactness argument: with t = x * 2^l (exact, power of two),
//   hat:        1 - |x - c| * 2^l   == fl(1 - |fl(t - i)|)
//   left edge:  2 - x * 2^l         == fl(2 - t)
//   right edge: 2 - (1 - x) * 2^l   == fl(2 - fl(2^l - t))
// because scaling by a power of two commutes with round-to-nearest in the
// normal range (x - c is never subnormal: c >= 2^-30).  Every operation is an
// explicit _rn intrinsic so nvcc cannot contract into FMA.
#pragma once

#include <cstdint>

namespace ddsg_b200 {

// Candidate cell at level l: the only node of level l whose support contains
// x is cell k = floor(x 2^(l-1)), clamped at x == 1.
__device__ __forceinline__ uint32_t cell_at(double x, int l) {
  const uint32_t ncell = 1u << (l - 1);
  uint32_t k = static_cast<uint32_t>(__dmul_rn(x, static_cast<double>(ncell)));
  return k < ncell ? k : ncell - 1u;
}

// Value of the level-l basis function of cell k at x.  mode: 0 zero_boundary, 1 modified_linear.
__device__ __forceinline__ double basis_at(int mode, int l, uint32_t k, double x) {
  if (mode == 1 && l == 1) return 1.0;
  const double scale = static_cast<double>(1u << l);
  const double t = __dmul_rn(x, scale);
  double v;
  if (mode == 1 && k == 0u) {
    v = __dadd_rn(2.0, -t);
  } else if (mode == 1 && 2u * k + 1u == (1u << l) - 1u) {
    v = __dadd_rn(2.0, -__dadd_rn(scale, -t));
  } else {
    v = __dadd_rn(1.0, -fabs(__dadd_rn(t, -static_cast<double>(2u * k + 1u))));
  }
  return v > 0.0 ? v : 0.0;
}

}  // namespace ddsg_b200
