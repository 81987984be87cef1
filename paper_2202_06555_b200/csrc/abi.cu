// C-ABI (include/ddsg_b200.h): handles, validation, error translation.
//
// Every entry point catches all exceptions and returns a ddsg_status; the
// message goes to a thread-local buffer (ddsg_last_error).
#include <cuda_runtime.h>

#include <algorithm>
#include <atomic>
#include <thread>
#include <cstring>
#include <map>
#include <memory>
#include <mutex>
#include <random>
#include <set>
#include <string>
#include <vector>

#include "../../include/ddsg_b200.h"
#include "device.cuh"
#include "grid_host.hpp"
#include "handles.hpp"
#include "irbc.cuh"
#include "program.hpp"

using namespace ddsg_b200;

using namespace ddsg_b200::abi;

std::unique_ptr<ddsg_hdmr> ddsg_b200::abi::make_hdmr(int d, int m, const double* f_anchor, int n_slots,
                                                     const int32_t* slot_order, const int32_t* slot_dims,
                                                     const int32_t* b, const HostGrid* const* grids,
                                                     const std::vector<std::vector<int32_t>>& extra_accepted_dims) {
  {
    if (d < 1 || m < 1) fail(DDSG_INVALID_ARGUMENT, "hdmr_create: d and m must be >= 1");
    if (n_slots < 1 || !slot_order || !b || !f_anchor)
      fail(DDSG_INVALID_ARGUMENT, "vectorized ddsg: inconsistent accepted family");
    auto h = std::make_unique<ddsg_hdmr>();
    h->d = d;
    h->m = m;
    h->f_anchor.assign(f_anchor, f_anchor + m);
    int64_t dim_off = 0;
    std::set<std::vector<int32_t>> accepted;
    for (int s = 0; s < n_slots; ++s) {
      const int k = slot_order[s];
      if (k < 0 || k > d) fail(DDSG_INVALID_ARGUMENT, "hdmr_create: slot order out of range");
      ddsg_hdmr::Slot slot;
      slot.dims.assign(slot_dims ? slot_dims + dim_off : nullptr, slot_dims ? slot_dims + dim_off + k : nullptr);
      if (k > 0 && !slot_dims) fail(DDSG_INVALID_ARGUMENT, "hdmr_create: null slot dims");
      dim_off += k;
      for (int j = 0; j < k; ++j) {
        if (slot.dims[j] < 0 || slot.dims[j] >= d)
          fail(DDSG_INVALID_ARGUMENT, "component index: dimension id out of range");
        if (j > 0 && slot.dims[j] <= slot.dims[j - 1])
          fail(DDSG_INVALID_ARGUMENT, "component index: dims must be strictly increasing");
      }
      slot.b = b[s];
      if (s == 0 && k != 0) fail(DDSG_INVALID_ARGUMENT, "vectorized ddsg: inconsistent accepted family");
      if (s > 0) {
        // (order, lexicographic) ordering, strictly increasing (component_index.hpp:25-28)
        const auto& prev = h->slots.back().dims;
        const bool less = prev.size() != slot.dims.size() ? prev.size() < slot.dims.size() : prev < slot.dims;
        if (!less) fail(DDSG_INVALID_ARGUMENT, "hdmr_create: slots must be sorted by (order, lex) without duplicates");
      }
      if (k > 0) {
        if (!grids || !grids[s])
          fail(DDSG_INVALID_ARGUMENT, "vectorized ddsg: coefficient for a non-accepted index");
        const HostGrid& G = *grids[s];
        if (G.dim != k) fail(DDSG_INVALID_ARGUMENT, "hdmr_create: grid dimension != slot order");
        if (G.m != m) fail(DDSG_INVALID_ARGUMENT, "hdmr_create: grid output length != m");
        slot.grid = static_cast<int>(h->grids.size());
        h->grids.push_back(G);
        accepted.insert(slot.dims);
      }
      h->slots.push_back(std::move(slot));
    }
    for (const auto& u : extra_accepted_dims) accepted.insert(u);
    // closure: every non-empty proper subset of an accepted index is accepted (ddsg_eval.hpp:63-70)
    for (const auto& u : accepted) {
      const size_t k = u.size();
      for (size_t mask = 1; mask + 1 < (size_t{1} << k); ++mask) {
        std::vector<int32_t> sub;
        for (size_t j = 0; j < k; ++j)
          if (mask & (size_t{1} << j)) sub.push_back(u[j]);
        if (!accepted.count(sub)) {
          auto str = [](const std::vector<int32_t>& v) {
            std::string s = "{";
            for (size_t i = 0; i < v.size(); ++i) s += (i ? "," : "") + std::to_string(v[i]);
            return s + "}";
          };
          fail(DDSG_INVALID_ARGUMENT,
               "vectorized ddsg: accepted family misses subset " + str(sub) + " of " + str(u));
        }
      }
    }
    HostProgram& hp = h->prog;
    hp.d = d;
    hp.m = m;
    hp.plain = 0;
    hp.f_anchor = h->f_anchor;
    for (int s = 0; s < n_slots; ++s) {
      const auto& slot = h->slots[s];
      if (slot.b == 0) continue;
      if (slot.dims.empty())
        hp.add_empty_slot(s, static_cast<double>(slot.b));
      else
        hp.add_grid_slot(s, h->grids[slot.grid], slot.dims, static_cast<double>(slot.b));
    }
    hp.finish();
    return h;
  }
}


extern "C" {

const char* ddsg_last_error(void) { return g_last_error.c_str(); }

int ddsg_device_count(void) {
  int n = 0;
  if (cudaGetDeviceCount(&n) != cudaSuccess) {
    cudaGetLastError();
    return 0;
  }
  return n;
}

ddsg_status ddsg_grid_create(int dim, int m, int mode, int max_level, double eps_gamma, int64_t n_nodes,
                             const uint32_t* heap_keys, const double* surplus, ddsg_grid_t** out) {
  return guarded([&] {
    if (!out) fail(DDSG_INVALID_ARGUMENT, "grid_create: null output handle");
    auto h = std::make_unique<ddsg_grid>();
    h->g = HostGrid::from_nodes(dim, m, mode, max_level, eps_gamma, n_nodes, heap_keys, surplus);
    *out = h.release();
  });
}

ddsg_status ddsg_grid_build(int dim, int m, int mode, int max_level, double eps_gamma, int norm,
                            ddsg_batch_evaluator f, void* ctx, ddsg_grid_t** out) {
  g_last_build_point.clear();
  return guarded([&] {
    if (!out) fail(DDSG_INVALID_ARGUMENT, "grid_build: null output handle");
    if (!f) fail(DDSG_INVALID_ARGUMENT, "grid_build: null evaluator");
    if (norm != DDSG_NORM_INF && norm != DDSG_NORM_L2)
      fail(DDSG_INVALID_ARGUMENT, "grid_build: unknown surplus norm");
    auto h = std::make_unique<ddsg_grid>();
    h->g = HostGrid::build(dim, m, mode, max_level, eps_gamma, norm,
                           [&](const double* xs, int64_t count, double* o) {
                             if (f(xs, count, o, ctx) != 0) {
                               throw BuildError("sparse grid: evaluator failed",
                                                std::vector<double>(xs, xs + dim));
                             }
                           });
    *out = h.release();
  });
}

int ddsg_last_build_point(double* out, int capacity) {
  const int n = static_cast<int>(g_last_build_point.size());
  for (int i = 0; i < std::min(n, capacity); ++i) out[i] = g_last_build_point[i];
  return n;
}

ddsg_status ddsg_grid_append(ddsg_grid_t* g, int64_t n_new, const uint32_t* heap_keys, const double* surplus) {
  return guarded([&] {
    if (!g) fail(DDSG_INVALID_ARGUMENT, "grid_append: null grid");
    g->g.append(n_new, heap_keys, surplus);
    g->invalidate();
  });
}

ddsg_status ddsg_hierarchize(const ddsg_grid_t* g, int64_t n_new, const uint32_t* heap_keys,
                             const double* f_values, double* surplus_out) {
  return guarded([&] {
    if (!g) fail(DDSG_INVALID_ARGUMENT, "hierarchize: null grid");
    if (n_new < 0 || (n_new > 0 && (!heap_keys || !f_values || !surplus_out)))
      fail(DDSG_INVALID_ARGUMENT, "hierarchize: null arrays");
    const HostGrid& G = g->g;
    std::vector<double> x(static_cast<size_t>(n_new) * G.dim);
    for (int64_t i = 0; i < n_new * G.dim; ++i) {
      if (!valid_key(heap_keys[i])) fail(DDSG_INVALID_ARGUMENT, "hierarchize: invalid heap key");
      x[i] = coordinate_of(heap_keys[i]);
    }
    auto* self = const_cast<ddsg_grid_t*>(g);
    const auto prog = self->device();
    const bool f_dev = is_device_pointer(f_values), s_dev = is_device_pointer(surplus_out);
    if (f_dev != s_dev) fail(DDSG_INVALID_ARGUMENT, "hierarchize: f_values and surplus_out must both be host or device");
    if (f_dev) {  // device-resident rows (e.g. straight into an all-gather buffer)
      double* di = nullptr;
      DDSG_CUDA(cudaMalloc(&di, static_cast<size_t>(n_new) * G.m * 8 + 8));
      std::unique_ptr<double, decltype(&cudaFree)> hold(di, cudaFree);
      const int64_t bad = evaluate(*prog, 1, x.data(), n_new, di, nullptr);
      if (bad >= 0) fail(DDSG_DOMAIN_ERROR, "hierarchize: node outside the unit cube");
      residual_on_device(f_values, di, n_new * G.m, surplus_out, nullptr);
      DDSG_CUDA(cudaDeviceSynchronize());
      return;
    }
    std::vector<double> interp(static_cast<size_t>(n_new) * G.m);
    const int64_t bad = evaluate(*prog, 1, x.data(), n_new, interp.data(), nullptr);
    if (bad >= 0) fail(DDSG_DOMAIN_ERROR, "hierarchize: node outside the unit cube");
    for (int64_t i = 0; i < n_new * G.m; ++i) surplus_out[i] = f_values[i] - interp[i];
  });
}

ddsg_status ddsg_hierarchize_host(const ddsg_grid_t* g, int64_t n_new, const uint32_t* heap_keys,
                                  const double* f_values, double* surplus_out) {
  return guarded([&] {
    if (!g) fail(DDSG_INVALID_ARGUMENT, "hierarchize: null grid");
    if (n_new < 0 || (n_new > 0 && (!heap_keys || !f_values || !surplus_out)))
      fail(DDSG_INVALID_ARGUMENT, "hierarchize: null arrays");
    const HostGrid& G = g->g;
    std::vector<double> interp(G.m);
    for (int64_t i = 0; i < n_new; ++i) {
      for (int j = 0; j < G.dim; ++j)
        if (!valid_key(heap_keys[i * G.dim + j])) fail(DDSG_INVALID_ARGUMENT, "hierarchize: invalid heap key");
      std::fill(interp.begin(), interp.end(), 0.0);
      G.interpolate_at_node(heap_keys + i * G.dim, G.size(), interp.data());
      for (int c = 0; c < G.m; ++c) surplus_out[i * G.m + c] = f_values[i * G.m + c] - interp[c];
    }
  });
}

ddsg_status ddsg_grid_refine_candidates(const ddsg_grid_t* g, int level_sum, int64_t* n_out, uint32_t* heap_keys) {
  return guarded([&] {
    if (!g || !n_out) fail(DDSG_INVALID_ARGUMENT, "refine_candidates: null argument");
    const auto c = g->g.refine_candidates(level_sum);
    *n_out = static_cast<int64_t>(c.size());
    if (heap_keys)
      for (size_t i = 0; i < c.size(); ++i) std::copy(c[i].begin(), c[i].end(), heap_keys + i * g->g.dim);
  });
}

ddsg_status ddsg_grid_destroy(ddsg_grid_t* g) {
  return guarded([&] { delete g; });
}

ddsg_status ddsg_grid_info(const ddsg_grid_t* g, int* dim, int* m, int* mode, int* max_level,
                           double* eps_gamma, int64_t* n_nodes) {
  return guarded([&] {
    if (!g) fail(DDSG_INVALID_ARGUMENT, "grid_info: null grid");
    if (dim) *dim = g->g.dim;
    if (m) *m = g->g.m;
    if (mode) *mode = g->g.mode;
    if (max_level) *max_level = g->g.max_level;
    if (eps_gamma) *eps_gamma = g->g.eps_gamma;
    if (n_nodes) *n_nodes = g->g.size();
  });
}

ddsg_status ddsg_grid_nodes(const ddsg_grid_t* g, uint32_t* heap_keys, double* surplus) {
  return guarded([&] {
    if (!g) fail(DDSG_INVALID_ARGUMENT, "grid_nodes: null grid");
    if (heap_keys) std::copy(g->g.keys.begin(), g->g.keys.end(), heap_keys);
    if (surplus) std::copy(g->g.surplus.begin(), g->g.surplus.end(), surplus);
  });
}

ddsg_status ddsg_grid_find(const ddsg_grid_t* g, const uint32_t* heap_key, int64_t* index) {
  return guarded([&] {
    if (!g || !heap_key || !index) fail(DDSG_INVALID_ARGUMENT, "grid_find: null argument");
    *index = g->g.find(heap_key);
  });
}

ddsg_status ddsg_grid_quadrature(const ddsg_grid_t* g, double* out) {
  return guarded([&] {
    if (!g || !out) fail(DDSG_INVALID_ARGUMENT, "grid_quadrature: null argument");
    const auto q = g->g.quadrature();
    std::copy(q.begin(), q.end(), out);
  });
}

ddsg_status ddsg_eval_grid(const ddsg_grid_t* g, const double* x, int64_t n, double* y, int64_t* bad_index,
                           void* stream) {
  if (bad_index) *bad_index = -1;
  return guarded([&] {
    if (!g) fail(DDSG_INVALID_ARGUMENT, "eval_grid: null grid");
    if (n < 0) fail(DDSG_INVALID_ARGUMENT, "eval_grid: negative point count");
    if (n > 0 && (!x || !y)) fail(DDSG_INVALID_ARGUMENT, "eval_grid: null buffers");
    auto* self = const_cast<ddsg_grid_t*>(g);
    const auto prog = self->device();
    const int64_t bad = evaluate(*prog, g->eval_mode == DDSG_EVAL_EXACT, x, n, y,
                                 static_cast<cudaStream_t>(stream));
    if (bad >= 0) {
      if (bad_index) *bad_index = bad;
      fail(DDSG_DOMAIN_ERROR, "task " + std::to_string(bad) +
                                  " failed: sparse grid: query outside the unit cube");
    }
  });
}

ddsg_status ddsg_grid_support(const ddsg_grid_t* g, const double* x, int64_t n, int64_t* nnz, uint64_t* hash,
                              void* stream) {
  return guarded([&] {
    if (!g) fail(DDSG_INVALID_ARGUMENT, "grid_support: null grid");
    if (n > 0 && (!x || !nnz || !hash)) fail(DDSG_INVALID_ARGUMENT, "grid_support: null buffers");
    auto* self = const_cast<ddsg_grid_t*>(g);
    const auto prog = self->device();
    const int64_t bad = support(*prog, x, n, nnz, hash, static_cast<cudaStream_t>(stream));
    if (bad >= 0) fail(DDSG_DOMAIN_ERROR, "grid_support: query outside the unit cube");
  });
}

ddsg_status ddsg_grid_set_eval_mode(ddsg_grid_t* g, int eval_mode) {
  return guarded([&] {
    if (!g) fail(DDSG_INVALID_ARGUMENT, "set_eval_mode: null grid");
    if (eval_mode != DDSG_EVAL_EXACT && eval_mode != DDSG_EVAL_FAST)
      fail(DDSG_INVALID_ARGUMENT, "set_eval_mode: unknown mode");
    g->eval_mode = eval_mode;
  });
}

// ------------------------------------------------------------------ HDMR

ddsg_status ddsg_hdmr_create(int d, int m, const double* f_anchor, int n_slots, const int32_t* slot_order,
                             const int32_t* slot_dims, const int32_t* b, const ddsg_grid_t* const* grids,
                             ddsg_hdmr_t** out) {
  return guarded([&] {
    if (!out) fail(DDSG_INVALID_ARGUMENT, "hdmr_create: null output handle");
    std::vector<const HostGrid*> gs(n_slots > 0 ? static_cast<size_t>(n_slots) : 0, nullptr);
    if (grids)
      for (int s = 0; s < n_slots; ++s) gs[s] = grids[s] ? &grids[s]->g : nullptr;
    *out = make_hdmr(d, m, f_anchor, n_slots, slot_order, slot_dims, b, gs.data()).release();
  });
}

ddsg_status ddsg_hdmr_destroy(ddsg_hdmr_t* h) {
  return guarded([&] { delete h; });
}

ddsg_status ddsg_hdmr_info(const ddsg_hdmr_t* h, int* d, int* m, int* n_slots, int* n_active, int64_t* n_nodes) {
  return guarded([&] {
    if (!h) fail(DDSG_INVALID_ARGUMENT, "hdmr_info: null handle");
    if (d) *d = h->d;
    if (m) *m = h->m;
    if (n_slots) *n_slots = static_cast<int>(h->slots.size());
    if (n_active) *n_active = static_cast<int>(h->prog.slot_k.size());
    if (n_nodes) {
      int64_t t = 0;
      for (const auto& g : h->grids) t += g.size();
      *n_nodes = t;
    }
  });
}

ddsg_status ddsg_eval_hdmr(const ddsg_hdmr_t* h, const double* x, int64_t n, double* y, int64_t* bad_index,
                           void* stream) {
  if (bad_index) *bad_index = -1;
  return guarded([&] {
    if (!h) fail(DDSG_INVALID_ARGUMENT, "eval_hdmr: null handle");
    if (n < 0) fail(DDSG_INVALID_ARGUMENT, "eval_hdmr: negative point count");
    if (n > 0 && (!x || !y)) fail(DDSG_INVALID_ARGUMENT, "eval_hdmr: null buffers");
    auto* self = const_cast<ddsg_hdmr_t*>(h);
    const auto prog = self->dev.get(h->prog);
    const int64_t bad = evaluate(*prog, h->eval_mode == DDSG_EVAL_EXACT, x, n, y,
                                 static_cast<cudaStream_t>(stream));
    if (bad >= 0) {
      if (bad_index) *bad_index = bad;
      fail(DDSG_DOMAIN_ERROR, "task " + std::to_string(bad) + " failed: ddsg: query outside unit cube");
    }
  });
}

ddsg_status ddsg_workspace_create(ddsg_workspace_t** out) {
  return guarded([&] {
    if (!out) fail(DDSG_INVALID_ARGUMENT, "workspace_create: null output handle");
    *out = new ddsg_workspace();
  });
}

ddsg_status ddsg_workspace_destroy(ddsg_workspace_t* ws) {
  return guarded([&] { delete ws; });
}

ddsg_status ddsg_eval_hdmr_ws(const ddsg_hdmr_t* h, ddsg_workspace_t* ws, const double* x, int64_t n, double* y,
                              int64_t* bad_index, uint64_t* interp_calls) {
  if (bad_index) *bad_index = -1;
  return guarded([&] {
    if (!h || !ws) fail(DDSG_INVALID_ARGUMENT, "eval_hdmr_ws: null handle");
    if (n < 0) fail(DDSG_INVALID_ARGUMENT, "eval_hdmr_ws: negative point count");
    if (n > 0 && (!x || !y)) fail(DDSG_INVALID_ARGUMENT, "eval_hdmr_ws: null buffers");
    auto* self = const_cast<ddsg_hdmr_t*>(h);
    const auto prog = self->dev.get(h->prog);
    const int64_t bad = evaluate_staged(*prog, h->eval_mode == DDSG_EVAL_EXACT, x, n, y, ws->ws);
    if (bad >= 0) {
      if (bad_index) *bad_index = bad;
      fail(DDSG_DOMAIN_ERROR, "ddsg: query outside unit cube");
    }
    if (interp_calls) {  // ddsg_eval.hpp:103: one count per active non-empty slot and point
      uint64_t per_point = 0;
      for (int32_t k : h->prog.slot_k) per_point += k > 0 ? 1u : 0u;
      *interp_calls += per_point * static_cast<uint64_t>(n);
    }
  });
}

ddsg_status ddsg_eval_hdmr_rows(const ddsg_hdmr_t* h, ddsg_workspace_t* ws, const double* const* xrows, int64_t n,
                                double* const* yrows, int64_t* bad_index) {
  if (bad_index) *bad_index = -1;
  return guarded([&] {
    if (!h || !ws) fail(DDSG_INVALID_ARGUMENT, "eval_hdmr_rows: null handle");
    if (n < 0) fail(DDSG_INVALID_ARGUMENT, "eval_hdmr_rows: negative point count");
    if (n > 0 && (!xrows || !yrows)) fail(DDSG_INVALID_ARGUMENT, "eval_hdmr_rows: null row arrays");
    auto* self = const_cast<ddsg_hdmr_t*>(h);
    const auto prog = self->dev.get(h->prog);
    const int64_t bad =
        evaluate_staged(*prog, h->eval_mode == DDSG_EVAL_EXACT, nullptr, n, nullptr, ws->ws, xrows, yrows);
    if (bad >= 0) {
      if (bad_index) *bad_index = bad;
      fail(DDSG_DOMAIN_ERROR, "task " + std::to_string(bad) + " failed: ddsg: query outside unit cube");
    }
  });
}

ddsg_status ddsg_eval_grid_ws(const ddsg_grid_t* g, ddsg_workspace_t* ws, const double* x, int64_t n, double* y,
                              int64_t* bad_index) {
  if (bad_index) *bad_index = -1;
  return guarded([&] {
    if (!g || !ws) fail(DDSG_INVALID_ARGUMENT, "eval_grid_ws: null handle");
    if (n < 0) fail(DDSG_INVALID_ARGUMENT, "eval_grid_ws: negative point count");
    if (n > 0 && (!x || !y)) fail(DDSG_INVALID_ARGUMENT, "eval_grid_ws: null buffers");
    auto* self = const_cast<ddsg_grid_t*>(g);
    const auto prog = self->device();
    const int64_t bad = evaluate_staged(*prog, g->eval_mode == DDSG_EVAL_EXACT, x, n, y, ws->ws);
    if (bad >= 0) {
      if (bad_index) *bad_index = bad;
      fail(DDSG_DOMAIN_ERROR, "sparse grid: query outside the unit cube");
    }
  });
}

ddsg_status ddsg_hdmr_support(const ddsg_hdmr_t* h, const double* x, int64_t n, int64_t* nnz, uint64_t* hash,
                              void* stream) {
  return guarded([&] {
    if (!h) fail(DDSG_INVALID_ARGUMENT, "hdmr_support: null handle");
    if (n > 0 && (!x || !nnz || !hash)) fail(DDSG_INVALID_ARGUMENT, "hdmr_support: null buffers");
    auto* self = const_cast<ddsg_hdmr_t*>(h);
    const auto prog = self->dev.get(h->prog);
    const int64_t bad = support(*prog, x, n, nnz, hash, static_cast<cudaStream_t>(stream));
    if (bad >= 0) fail(DDSG_DOMAIN_ERROR, "hdmr_support: query outside unit cube");
  });
}

ddsg_status ddsg_hdmr_quadrature(const ddsg_hdmr_t* h, double* out) {
  return guarded([&] {
    if (!h || !out) fail(DDSG_INVALID_ARGUMENT, "hdmr_quadrature: null argument");
    // ddsg_eval.hpp:143-151: sum over slots with b != 0 of b * cut quadrature
    std::vector<double> q(h->m, 0.0);
    for (const auto& s : h->slots) {
      if (s.b == 0) continue;
      const std::vector<double> qc = s.dims.empty() ? h->f_anchor : h->grids[s.grid].quadrature();
      for (int c = 0; c < h->m; ++c) q[c] += s.b * qc[c];
    }
    std::copy(q.begin(), q.end(), out);
  });
}

ddsg_status ddsg_hdmr_set_eval_mode(ddsg_hdmr_t* h, int eval_mode) {
  return guarded([&] {
    if (!h) fail(DDSG_INVALID_ARGUMENT, "set_eval_mode: null handle");
    if (eval_mode != DDSG_EVAL_EXACT && eval_mode != DDSG_EVAL_FAST)
      fail(DDSG_INVALID_ARGUMENT, "set_eval_mode: unknown mode");
    h->eval_mode = eval_mode;
  });
}

ddsg_status ddsg_last_eval_stats(int64_t* launches, double* kernel_ms, double* main_kernel_ms) {
  const EvalStats& s = last_stats();
  if (launches) *launches = s.launches;
  if (kernel_ms) *kernel_ms = s.kernel_ms;
  if (main_kernel_ms) *main_kernel_ms = s.main_ms;
  return DDSG_OK;
}

ddsg_status ddsg_hdmr_kernel_path(const ddsg_hdmr_t* h, int* fast_path) {
  return guarded([&] {
    if (!h || !fast_path) fail(DDSG_INVALID_ARGUMENT, "hdmr_kernel_path: null argument");
    auto* self = const_cast<ddsg_hdmr_t*>(h);
    *fast_path = self->dev.get(h->prog)->fast() != nullptr ? 1 : 0;
  });
}

void ddsg_uniform_points(uint64_t seed, int64_t n, int dim, double* out) {
  // std::uniform_real_distribution<double>(0,1) over std::mt19937_64, as
  // oracles.hpp:45-53 (libstdc++ generate_canonical with one 64-bit draw).
  std::mt19937_64 rng(seed);
  std::uniform_real_distribution<double> unif(0.0, 1.0);
  for (int64_t i = 0; i < n * dim; ++i) out[i] = unif(rng);
}

void ddsg_uniform_point_blocks(uint64_t seed, int64_t block_points, int64_t first, int64_t n, int dim, double* out) {
  if (n <= 0 || dim <= 0 || block_points <= 0 || first < 0 || !out) return;
  const int64_t b0 = first / block_points, b1 = (first + n - 1) / block_points;
  auto work = [&](int64_t b) {
    const int64_t lo = std::max(first, b * block_points), hi = std::min(first + n, (b + 1) * block_points);
    std::mt19937_64 rng(seed + static_cast<uint64_t>(b));
    rng.discard(static_cast<unsigned long long>((lo - b * block_points) * dim));
    std::uniform_real_distribution<double> unif(0.0, 1.0);
    double* o = out + (lo - first) * dim;
    for (int64_t i = 0; i < (hi - lo) * dim; ++i) o[i] = unif(rng);
  };
  const int64_t nb = b1 - b0 + 1;
  const unsigned hw = std::max(1u, std::thread::hardware_concurrency());
  const int64_t nt = std::min<int64_t>(nb, std::min<unsigned>(hw, 32u));
  std::vector<std::thread> pool;
  std::atomic<int64_t> next{b0};
  for (int64_t t = 0; t < nt; ++t)
    pool.emplace_back([&] {
      for (int64_t b = next++; b <= b1; b = next++) work(b);
    });
  for (auto& th : pool) th.join();
}

}  // extern "C"

// ----------------------------------------------------------- IRBC callers

namespace {

// IrbcParameters -> irbc::Params, with the validation of refresh_derived.
irbc::Params irbc_params(const ddsg_irbc_params* p) {
  if (!p) fail(DDSG_INVALID_ARGUMENT, "irbc: null parameters");
  if (p->countries < 1) fail(DDSG_INVALID_ARGUMENT, "irbc: countries must be >= 1");
  if (p->countries > 2048) fail(DDSG_INVALID_ARGUMENT, "irbc: at most 2048 countries on the device path");
  if (p->variant != DDSG_IRBC_SMOOTH && p->variant != DDSG_IRBC_NONSMOOTH)
    fail(DDSG_INVALID_ARGUMENT, "irbc: unknown variant");
  if (!p->gamma || !p->tau) fail(DDSG_INVALID_ARGUMENT, "irbc: null gamma / tau");
  irbc::Params q;
  q.countries = p->countries;
  q.nonsmooth = p->variant == DDSG_IRBC_NONSMOOTH;
  q.beta = p->beta;
  q.alpha = p->alpha;
  q.delta = p->delta;
  q.sigma = p->sigma;
  q.rho_a = p->rho_a;
  q.phi_adj = p->phi_adj;
  q.lna_half_width = p->lna_half_width;
  q.k_lo = p->k_lo;
  q.k_hi = p->k_hi;
  q.A = p->A;
  q.gamma.assign(p->gamma, p->gamma + p->countries);
  q.tau.assign(p->tau, p->tau + p->countries);
  return q;
}

// The policy as a batched device evaluator (compiled_evaluator,
// time_iteration.hpp:86-91): canonical states [2N] -> flat policy [pdim].
irbc::PolicyFn irbc_policy(const ddsg_hdmr_t* h, const ddsg_grid_t* g, const irbc::Params& p) {
  if ((h == nullptr) == (g == nullptr))
    fail(DDSG_INVALID_ARGUMENT, "irbc: exactly one of policy_hdmr / policy_grid must be given");
  int d = 0, m = 0, exact = 1;
  std::shared_ptr<const DeviceProgram> prog;
  if (h) {
    auto* self = const_cast<ddsg_hdmr_t*>(h);
    d = h->d;
    m = h->m;
    exact = h->eval_mode == DDSG_EVAL_EXACT;
    prog = self->dev.get(h->prog);
  } else {
    auto* self = const_cast<ddsg_grid_t*>(g);
    d = g->g.dim;
    m = g->g.m;
    exact = g->eval_mode == DDSG_EVAL_EXACT;
    prog = self->device();
  }
  if (d != p.state_dim() || m != p.pdim())
    fail(DDSG_INVALID_ARGUMENT, "irbc: policy dimensions do not match the model (dim 2N, out_dim pdim)");
  return [prog, exact](const double* dx, int64_t n, double* dy, cudaStream_t st) {
    return evaluate(*prog, exact, dx, n, dy, st);
  };
}

void irbc_domain_fail(int64_t bad, int64_t* bad_index) {
  if (bad_index) *bad_index = bad;
  fail(DDSG_DOMAIN_ERROR, "task " + std::to_string(bad) + " failed: ddsg: query outside unit cube");
}

}  // namespace

extern "C" {

ddsg_status ddsg_irbc_refresh_derived(ddsg_irbc_params* p, int fill_gamma) {
  return guarded([&] {
    // irbc.hpp:59-92, same checks, messages and arithmetic (host libm)
    if (!p) fail(DDSG_INVALID_ARGUMENT, "irbc: null parameters");
    if (p->countries < 1) fail(DDSG_INVALID_ARGUMENT, "irbc: countries must be >= 1");
    if (!(p->beta > 0.0 && p->beta < 1.0)) fail(DDSG_INVALID_ARGUMENT, "irbc: beta in (0,1)");
    if (!(p->delta > 0.0 && p->delta < 1.0)) fail(DDSG_INVALID_ARGUMENT, "irbc: delta in (0,1)");
    if (!(p->alpha > 0.0 && p->alpha < 1.0)) fail(DDSG_INVALID_ARGUMENT, "irbc: alpha in (0,1)");
    if (!(p->sigma >= 0.0)) fail(DDSG_INVALID_ARGUMENT, "irbc: sigma must be >= 0");
    if (!(p->rho_a >= 0.0 && p->rho_a < 1.0)) fail(DDSG_INVALID_ARGUMENT, "irbc: rho_a in [0,1)");
    if (!(p->phi_adj >= 0.0)) fail(DDSG_INVALID_ARGUMENT, "irbc: phi_adj must be >= 0");
    if (!(p->k_lo > 0.0 && p->k_hi > p->k_lo))
      fail(DDSG_INVALID_ARGUMENT, "irbc: capital box must satisfy 0 < k_lo < k_hi");
    if (!(p->lna_half_width > 0.0)) fail(DDSG_INVALID_ARGUMENT, "irbc: lna_half_width must be > 0");
    if (!p->gamma || !p->tau) fail(DDSG_INVALID_ARGUMENT, "irbc: null gamma / tau");
    const int N = p->countries;
    if (fill_gamma)
      for (int j = 0; j < N; ++j)
        p->gamma[j] = N == 1 ? p->gamma_base
                             : p->gamma_base + 0.75 * static_cast<double>(j) / static_cast<double>(N - 1);
    for (int j = 0; j < N; ++j)
      if (!(p->gamma[j] > 0.0)) fail(DDSG_INVALID_ARGUMENT, "irbc: gamma_j must be > 0");
    p->A = (1.0 - p->beta * (1.0 - p->delta)) / (p->alpha * p->beta);
    for (int j = 0; j < N; ++j) p->tau[j] = std::pow(p->A, 1.0 / p->gamma[j]);
  });
}

ddsg_status ddsg_irbc_steady_state_lambda(const ddsg_irbc_params* p, double* lambda) {
  return guarded([&] {
    // irbc.hpp:248-263: geometric bisection, 200 halvings
    if (!p || !lambda || !p->gamma) fail(DDSG_INVALID_ARGUMENT, "irbc: null argument");
    const double target = static_cast<double>(p->countries) * (p->A - p->delta);
    if (!(target > 0.0)) fail(DDSG_DOMAIN_ERROR, "irbc: steady-state consumption would be non-positive");
    double lo = 1e-8, hi = 1e8;
    auto g = [&](double lam) {
      double s = 0.0;
      for (int j = 0; j < p->countries; ++j) s += p->A * std::pow(lam, -p->gamma[j]);
      return s - target;
    };
    for (int it = 0; it < 200; ++it) {
      const double mid = std::sqrt(lo * hi);
      (g(mid) > 0.0 ? lo : hi) = mid;
    }
    *lambda = std::sqrt(lo * hi);
  });
}

ddsg_status ddsg_irbc_foc_residuals(const ddsg_hdmr_t* policy_hdmr, const ddsg_grid_t* policy_grid,
                                    const ddsg_irbc_params* p, int64_t n, const double* a, const double* k,
                                    const double* candidate, double* residuals, int32_t* clamped,
                                    int64_t* bad_index, void* stream) {
  if (bad_index) *bad_index = -1;
  return guarded([&] {
    const irbc::Params q = irbc_params(p);
    const irbc::PolicyFn pol = irbc_policy(policy_hdmr, policy_grid, q);
    if (n < 0) fail(DDSG_INVALID_ARGUMENT, "foc_residuals: negative state count");
    if (n > 0 && (!a || !k || !candidate || !residuals)) fail(DDSG_INVALID_ARGUMENT, "foc_residuals: null buffers");
    const int64_t bad = irbc::foc_residuals(q, pol, n, a, k, candidate, residuals, clamped,
                                            static_cast<cudaStream_t>(stream));
    if (bad >= 0) irbc_domain_fail(bad, bad_index);
  });
}

ddsg_status ddsg_irbc_foc_jacobian(const ddsg_hdmr_t* policy_hdmr, const ddsg_grid_t* policy_grid,
                                   const ddsg_irbc_params* p, int64_t n, const double* a, const double* k,
                                   const double* z, const double* r0, double fd_epsilon, double* jac,
                                   int64_t* bad_index, void* stream) {
  if (bad_index) *bad_index = -1;
  return guarded([&] {
    const irbc::Params q = irbc_params(p);
    const irbc::PolicyFn pol = irbc_policy(policy_hdmr, policy_grid, q);
    if (n < 0) fail(DDSG_INVALID_ARGUMENT, "foc_jacobian: negative state count");
    if (n > 0 && (!a || !k || !z || !r0 || !jac)) fail(DDSG_INVALID_ARGUMENT, "foc_jacobian: null buffers");
    const int64_t bad =
        irbc::foc_jacobian(q, pol, n, a, k, z, r0, fd_epsilon, jac, static_cast<cudaStream_t>(stream));
    if (bad >= 0) irbc_domain_fail(bad, bad_index);
  });
}

ddsg_status ddsg_irbc_euler_errors(const ddsg_hdmr_t* policy_hdmr, const ddsg_grid_t* policy_grid,
                                   const ddsg_irbc_params* p, int64_t n, const double* xs, double* errs,
                                   double* mean, double* worst, uint64_t* clamp_count, int64_t* bad_index,
                                   void* stream) {
  if (bad_index) *bad_index = -1;
  return guarded([&] {
    const irbc::Params q = irbc_params(p);
    const irbc::PolicyFn pol = irbc_policy(policy_hdmr, policy_grid, q);
    // solver.hpp:381
    if (n < 1) fail(DDSG_INVALID_ARGUMENT, "euler_errors: n_samples must be >= 1");
    if (!xs || !errs || !mean || !worst) fail(DDSG_INVALID_ARGUMENT, "euler_errors: null buffers");
    const int64_t bad = irbc::euler_errors(q, pol, n, xs, errs, mean, worst, clamp_count,
                                           static_cast<cudaStream_t>(stream));
    if (bad >= 0) irbc_domain_fail(bad, bad_index);
  });
}

}  // extern "C"
