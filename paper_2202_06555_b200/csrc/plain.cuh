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
constexpr int kSparseMaxDim = 64;  // sparse walk: coordinates of 128 points x d dims in shared memory
constexpr int64_t kSortMinPoints = 4096;

// Exact 1-d factor of the candidate cell at (runtime) level l:
// xi = floor(x 2^31) clamped to 2^31 - 1, so xi >> (32 - l) is the candidate
// cell floor(x 2^(l-1)), clamped at x = 1.  The value is
// basis.cuh's restatement v = fl(A - |fl(x 2^l - B)|) with
//  * x 2^l formed by adding l to the exponent field of x: exact for normal
//    x; for x = 0 (or subnormal x) the result is a tiny t that rounds away
//    against B >= 1 (hat) or against A = 2 (modified left edge, B = 0),
//    exactly as t = 0 does;
//  * B as a double by the 2^52 trick (one DADD, fixed latency, no I2F).
template <int kMode>
__device__ __forceinline__ void factor(double x, uint32_t xi, int l, uint32_t& kk, double& v) {
  kk = xi >> (32 - l);
  if (kMode == 1 && l == 1) {
    v = 1.0;
    return;
  }
  const double t = __hiloint2double(__double2hiint(x) + (l << 20), __double2loint(x));
  uint32_t B = 2u * kk + 1u;
  double A = 1.0;
  if (kMode == 1) {
    const uint32_t ncm1 = (1u << (l - 1)) - 1u;
    const bool left = kk == 0u, right = kk == ncm1;
    B = left ? 0u : (right ? 2u * ncm1 + 2u : B);
    A = (left || right) ? 2.0 : 1.0;
  }
  const double Bd = __dadd_rn(__hiloint2double(0x43300000, static_cast<int>(B)), -4503599627370496.0);
  v = __dadd_rn(A, -fabs(__dadd_rn(t, -Bd)));  // >= 0 at the candidate cell
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
  bool build_sparse(const HostProgram& hp);
  bool sparse_ = false;  // modified-linear grids: sparse walk over the non-trivial dims
  int smc_ = 12;         // sparse walk: columns per pass
  std::vector<int> srun_off_;
  const uint4* srec_ = nullptr;
  const int* srun_off_dev_ = nullptr;
  int d_ = 0, m_ = 0, ms_ = 0, mc_ = 1, mode_ = 0, runs_ = 1, zero_row_ = 0;
  std::vector<int> run_off_;
  const int* run_off_dev_ = nullptr;
  const uint4* rec_ = nullptr;  // [n_sub][2] packed subspace records
  const int32_t* slab_ = nullptr;  // [runs][slab_len_] per-run slabs (the program's slab when 1 run)
  int64_t slab_len_ = 0;
  const double* surplus_ = nullptr;
  std::vector<void*> allocs_;
  template <typename T>
  const T* put(const std::vector<T>& v);
};

}  // namespace ddsg_b200
