// Device-resident program and the evaluation kernels' parameter block.
#pragma once

#include <cuda_runtime.h>

#include <cstdint>
#include <string>
#include <vector>

#include "program.hpp"

namespace ddsg_b200 {
class FastHdmr;
class PlainGrid;
}

namespace ddsg_b200 {

#define DDSG_CUDA(call)                                                                     \
  do {                                                                                      \
    cudaError_t e_ = (call);                                                                \
    if (e_ != cudaSuccess) {                                                                \
      ::ddsg_b200::fail(e_ == cudaErrorMemoryAllocation ? DDSG_OUT_OF_MEMORY : DDSG_CUDA_ERROR, \
                        std::string(#call) + ": " + cudaGetErrorString(e_));                 \
    }                                                                                       \
  } while (0)

constexpr int kMaxDepth = 32;  // pairwise-sum stack (2^31 active slots)
constexpr int kMaxSlotDim = 64;

// Plain-old-data view of a DeviceProgram passed by value to kernels.
struct EvalParams {
  int d, m, n_active, plain, exact, depth;
  const int32_t* slot_k;
  const int32_t* slot_mode;
  const int32_t* slot_dims_off;
  const int32_t* slot_dims;
  const double* slot_b;
  const int32_t* slot_sub_begin;
  const int32_t* slot_sub_end;
  const int32_t* slot_id;
  const uint8_t* merges;
  const int32_t* sub_lv_off;
  const uint8_t* levels;
  const int64_t* sub_slab_off;
  const int32_t* slab;
  const double* surplus;
  const int32_t* row_stored;
  const int16_t* row_run;
  const int32_t* slot_runs;
  const double* f_anchor;
};

class DeviceProgram {
 public:
  DeviceProgram() = default;
  DeviceProgram(const DeviceProgram&) = delete;
  DeviceProgram& operator=(const DeviceProgram&) = delete;
  ~DeviceProgram();

  void upload(const HostProgram& hp);
  EvalParams params(int exact) const;
  bool ready() const { return ready_; }
  const HostProgram& host() const { return hp_; }
  const FastHdmr* fast() const { return fast_; }
  const PlainGrid* plain() const { return plain_; }
  // Small-batch path of an HDMR program (see launch_eval): the reference's
  // pairwise tree as internal nodes grouped by height.
  struct SlotTree {
    int nodes = 0;    // internal nodes (n_active - 1)
    int heights = 0;  // tree height
    const int32_t* left = nullptr;   // [nodes] child ids (< n_active: leaf / slot row)
    const int32_t* right = nullptr;
    const int32_t* height_off = nullptr;  // [heights + 1] node ranges per height
    // fused small-batch kernel: every subspace of every active slot
    int n_subs = 0;                       // subspaces of all active slots (concatenated, slot order)
    const int32_t* sub_slot = nullptr;    // [n_subs] active slot of the subspace
  };
  const SlotTree& slot_tree() const { return tree_; }
  // Unique per uploaded program (never reused): the key of cached CUDA graphs.
  uint64_t uid() const { return uid_; }

 private:
  HostProgram hp_;
  std::vector<void*> allocs_;
  EvalParams p_{};
  bool ready_ = false;
  FastHdmr* fast_ = nullptr;    // slot-staged kernel program, when the program qualifies
  PlainGrid* plain_ = nullptr;  // prefix-walk plain-grid kernel program, when it qualifies
  SlotTree tree_;
  uint64_t uid_ = 0;
  template <typename T>
  const T* put(const std::vector<T>& v);
};

// Per-call statistics (thread-local, see ddsg_last_eval_stats).
struct EvalStats {
  int64_t launches = 0;
  double kernel_ms = 0.0;  // device time of the whole evaluation (device-resident calls)
  double main_ms = 0.0;    // device time of the dominant (slot) kernel launches
};
EvalStats& last_stats();

// Interval timer for the dominant kernel: begin()/end() record CUDA events on
// the launching stream; collect() sums the intervals after a synchronize.
struct KernelTimer {
  void begin(cudaStream_t st);
  void end(cudaStream_t st);
  double collect();  // ms; resets
};
KernelTimer& kernel_timer();

// Raise-only cudaFuncAttributeMaxDynamicSharedMemorySize for `fn` on the
// current device: the attribute belongs to the kernel function, shared by
// every program and host thread, so it is never lowered (a lowered limit
// would break another program's launch, possibly on another host thread).
void ensure_dynamic_smem(const void* fn, size_t bytes);

// Evaluates the program over n points.  x/y may be host or device memory.
// Returns the lowest out-of-domain point index or -1.
int64_t evaluate(const DeviceProgram& prog, int exact, const double* x, int64_t n, double* y,
                 cudaStream_t stream);

// Pinned-staging workspace for ordinary (pageable) host buffers
// (EvalWorkspace, ddsg_eval.hpp:21-24): two pinned host slots, two device
// slots and two streams on the device current at first use; chunk i's host
// copy-in overlaps chunk i-1's transfers and kernels.
class StagedWorkspace {
 public:
  StagedWorkspace();
  ~StagedWorkspace();
  StagedWorkspace(const StagedWorkspace&) = delete;
  StagedWorkspace& operator=(const StagedWorkspace&) = delete;
  struct Impl;
  Impl* impl() { return impl_; }

 private:
  Impl* impl_;
};

// Evaluates n points held in pageable host memory through `ws`.  Returns the
// lowest out-of-domain point index or -1.
// With xrows / yrows non-null, point i is read from xrows[i] and written to
// yrows[i] (row pointers) instead of x / y.
int64_t evaluate_staged(const DeviceProgram& prog, int exact, const double* x, int64_t n, double* y,
                        StagedWorkspace& ws, const double* const* xrows = nullptr, double* const* yrows = nullptr);

// Device memory (cudaMalloc / managed) as opposed to host memory.
bool is_device_pointer(const void* p);
// out[i] = f[i] - interp[i] (the reference's residual, sparse_grid.hpp:272)
// on device buffers, on stream st.
void residual_on_device(const double* f, const double* interp, int64_t count, double* out, cudaStream_t st);

// Support statistics (nnz and order-sensitive hash per point).
int64_t support(const DeviceProgram& prog, const double* x, int64_t n, int64_t* nnz,
                uint64_t* hash, cudaStream_t stream);

}  // namespace ddsg_b200
