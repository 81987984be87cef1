// Internal: the C-ABI handle types (ddsg_grid / ddsg_hdmr), the per-device
// program cache and the exception -> status translation shared by the C-ABI
// units (abi.cu, abi_json.cpp).
#pragma once

#include <cuda_runtime.h>

#include <map>
#include <memory>
#include <mutex>
#include <string>
#include <utility>
#include <vector>

#include "../../include/ddsg_b200.h"
#include "device.cuh"
#include "grid_host.hpp"
#include "program.hpp"

namespace ddsg_b200::abi {

inline thread_local std::string g_last_error;
inline thread_local std::vector<double> g_last_build_point;

inline ddsg_status set_error(ddsg_status s, const std::string& msg) {
  g_last_error = msg;
  return s;
}

template <typename F>
ddsg_status guarded(F&& f) {
  try {
    f();
    return DDSG_OK;
  } catch (const BuildError& e) {
    g_last_build_point = e.point;
    return set_error(e.status, e.what());
  } catch (const Error& e) {
    return set_error(e.status, e.what());
  } catch (const std::bad_alloc&) {
    return set_error(DDSG_OUT_OF_MEMORY, "host allocation failed");
  } catch (const std::exception& e) {
    return set_error(DDSG_INVALID_ARGUMENT, e.what());
  } catch (...) {
    return set_error(DDSG_INVALID_ARGUMENT, "unknown error");
  }
}

inline int current_device() {
  int dev = 0;
  DDSG_CUDA(cudaGetDevice(&dev));
  return dev;
}

// Device copies of a program, one per CUDA device that evaluated it.  Copies
// are handed out as shared_ptr: a call keeps its copy alive for its whole
// duration even if ddsg_grid_append invalidates the cache concurrently (the
// next call then uploads the appended program).
struct DeviceCache {
  std::mutex mu;
  std::map<int, std::shared_ptr<const DeviceProgram>> per_device;
  std::shared_ptr<const DeviceProgram> get(const HostProgram& hp) {
    const int dev = current_device();
    std::lock_guard<std::mutex> lock(mu);
    auto& slot = per_device[dev];
    if (!slot) {
      auto p = std::make_shared<DeviceProgram>();
      p->upload(hp);
      slot = std::move(p);
    }
    return slot;
  }
  void invalidate() {
    std::lock_guard<std::mutex> lock(mu);
    per_device.clear();
  }
};

}  // namespace ddsg_b200::abi

struct ddsg_grid {
  ddsg_b200::HostGrid g;
  int eval_mode = DDSG_EVAL_EXACT;
  std::mutex prog_mu;
  std::shared_ptr<const ddsg_b200::HostProgram> prog;
  ddsg_b200::abi::DeviceCache dev;

  std::shared_ptr<const ddsg_b200::HostProgram> program() {
    std::lock_guard<std::mutex> lock(prog_mu);
    if (!prog) {
      auto hp = std::make_shared<ddsg_b200::HostProgram>();
      hp->d = g.dim;
      hp->m = g.m;
      hp->plain = 1;
      hp->f_anchor.assign(g.m, 0.0);
      std::vector<int32_t> dims(g.dim);
      for (int j = 0; j < g.dim; ++j) dims[j] = j;
      hp->add_grid_slot(0, g, dims, 1.0);
      hp->finish();
      prog = std::move(hp);
    }
    return prog;
  }
  std::shared_ptr<const ddsg_b200::DeviceProgram> device() { return dev.get(*program()); }
  void invalidate() {
    std::lock_guard<std::mutex> lock(prog_mu);
    prog.reset();
    dev.invalidate();
  }
};

struct ddsg_hdmr {
  int d = 0, m = 0;
  std::vector<double> f_anchor;
  struct Slot {
    std::vector<int32_t> dims;
    int32_t b = 0;
    int grid = -1;  // index into grids
  };
  std::vector<Slot> slots;
  std::vector<ddsg_b200::HostGrid> grids;
  ddsg_b200::HostProgram prog;
  int eval_mode = DDSG_EVAL_EXACT;
  ddsg_b200::abi::DeviceCache dev;
  // Document fields (serialize.hpp:80-110) that evaluation does not use,
  // kept so a loaded policy is written back unchanged.
  int k_max = 1;
  std::vector<double> anchor_coords;               // empty: not provided
  std::vector<std::vector<int32_t>> rejected;      // (order, lex) order
  std::vector<double> cut_quads;                   // [slots][m] in slot order; empty: not provided
  // accepted components without a coefficient entry (kept for documents only)
  std::vector<std::pair<std::vector<int32_t>, ddsg_b200::HostGrid>> extra_accepted;
};

namespace ddsg_b200::abi {
// The body of ddsg_hdmr_create (from_parts + VectorizedDdsg::compile
// validation, ddsg_eval.hpp:40-74); `grids[s]` null for the empty index.
std::unique_ptr<ddsg_hdmr> make_hdmr(int d, int m, const double* f_anchor, int n_slots, const int32_t* slot_order,
                                     const int32_t* slot_dims, const int32_t* b, const ddsg_b200::HostGrid* const* grids,
                                     const std::vector<std::vector<int32_t>>& extra_accepted_dims = {});
}  // namespace ddsg_b200::abi



struct ddsg_workspace {
  ddsg_b200::StagedWorkspace ws;
};
