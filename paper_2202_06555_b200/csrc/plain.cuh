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
  int64_t launch(int exact, const double* x, int64_t n, int64_t base, double* y, unsigned long long* bad,
                 cudaStream_t st) const;

 private:
  bool usable_ = false;
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
