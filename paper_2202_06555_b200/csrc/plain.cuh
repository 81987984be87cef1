// Plain-grid kernel program (see plain.cu).
#pragma once

#include <cuda_runtime.h>

#include <cstdint>
#include <vector>

#include "device.cuh"

namespace ddsg_b200 {

namespace plain {
constexpr int kThreads = 128;
constexpr int kMaxDim = 20;
constexpr int kMaxRuns = 15;
// Morton pre-sort of the points (plain.cu): only for d >= 5 (config 1's
// small grid is launch-bound) and batches of >= 4096 points
constexpr int kSortMinDim = 5;
constexpr int64_t kSortMinPoints = 4096;

// Exact 1-d factor of the candidate cell at (runtime) level l:
// xi = floor(x 2^31), so floor(x 2^(l-1)) = xi >> (32 - l); clamped at x = 1.
template <int kMode>
__device__ __forceinline__ void factor(double x, uint32_t xi, int l, uint32_t& kk, double& v) {
  const uint32_t ncell = 1u << (l - 1);
  kk = min(xi >> (32 - l), ncell - 1u);
  if (kMode == 1 && l == 1) {
    v = 1.0;
    return;
  }
  const double t = __dmul_rn(x, __hiloint2double((1023 + l) << 20, 0));  // x 2^l, exact
  uint32_t B = 2u * kk + 1u;
  double A = 1.0;
  if (kMode == 1) {
    const bool left = kk == 0u, right = kk == ncell - 1u;
    B = left ? 0u : (right ? 2u * ncell : B);
    A = (left || right) ? 2.0 : 1.0;
  }
  v = __dadd_rn(A, -fabs(__dadd_rn(t, -static_cast<double>(B))));  // >= 0 at the candidate cell
}

}  // namespace plain

class PlainGrid {
 public:
  PlainGrid() = default;
  PlainGrid(const PlainGrid&) = delete;
  PlainGrid& operator=(const PlainGrid&) = delete;
  ~PlainGrid();

  // Builds the subspace walk tables when the program is a plain grid with
  // d <= 20 and levels <= 15; `dev` supplies the already uploaded slab and
  // run arrays (the surpluses are re-laid out with a zero row).
  bool build(const HostProgram& hp, const EvalParams& dev);
  bool usable() const { return usable_; }
  // Device workspace the launch needs for n points (Morton keys, permutation
  // and sort scratch; 0 when the points are evaluated in input order).
  size_t workspace_bytes(int64_t n) const;
  int64_t launch(int exact, const double* x, int64_t n, int64_t base, double* y, unsigned long long* bad,
                 void* ws, cudaStream_t st) const;
  bool sorts_points() const { return sort_; }

 private:
  bool usable_ = false;
  bool sort_ = false;  // Morton pre-sort of large batches
  int d_ = 0, m_ = 0, ms_ = 0, mc_ = 1, mode_ = 0, runs_ = 1, zero_row_ = 0;
  std::vector<int> run_off_;
  const uint4* rec_ = nullptr;  // [n_sub][2] packed subspace records
  const int32_t* slab_ = nullptr;
  const int16_t* row_run_ = nullptr;
  const double* surplus_ = nullptr;
  std::vector<void*> allocs_;
  template <typename T>
  const T* put(const std::vector<T>& v);
};

}  // namespace ddsg_b200
