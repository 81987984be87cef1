// ddsg_b200.hpp — C++20 drop-in for the reference's interpolation API, over
// the C-ABI of include/ddsg_b200.h (header-only; link libddsg_b200.so).
//
// Class and member names, argument meaning and exception types mirror
// /root/reference/proj/include/ddsg/ (cited per member), so a caller of the
// reference switches by replacing `ddsg::` with `ddsg_b200::`.  Evaluation
// runs on the GPU; every batched call is one C-ABI call.
//
//   node keys, basis     grid_index.hpp:24-55, basis.hpp:25-84 (heap_key, basis_1d, ... host inline)
//   SparseGridFunction   sparse_grid.hpp:72-351 (+ refine_candidates / hierarchize / append, refine_step)
//   DdsgFunction         hdmr.hpp:195-356   (from_parts, evaluate_naive)
//   decompose            hdmr.hpp:45-133,364-483 (select_anchor, cut_evaluator, eta / rho, diagnostics)
//   EvalWorkspace        ddsg_eval.hpp:21-24
//   VectorizedDdsg       ddsg_eval.hpp:28-165
//   JSON documents       serialize.hpp:17-160 (JsonDocument stands in for nlohmann::json)
//   build_error          sparse_grid.hpp:40-48
//   task_error           runtime.hpp:71-92
#pragma once

#include <algorithm>
#include <cmath>
#include <cstdint>
#include <exception>
#include <fstream>
#include <sstream>
#include <functional>
#include <atomic>
#include <bit>
#include <limits>
#include <map>
#include <mutex>
#include <random>
#include <memory>
#include <new>
#include <set>
#include <span>
#include <stdexcept>
#include <string>
#include <thread>
#include <utility>
#include <vector>

#include "ddsg_b200.h"

namespace ddsg_b200 {

using HeapKey = std::uint32_t;            // grid_index.hpp:19
using NodeKey = std::vector<HeapKey>;     // grid_index.hpp:22

enum class BoundaryMode { zero_boundary, modified_linear };  // basis.hpp:22
enum class SurplusNorm { inf, l2 };                          // sparse_grid.hpp:53

// ---- 1-d node bookkeeping (grid_index.hpp:24-55): node (l, i), i odd, as the
// heap key 2^(l-1) + (i-1)/2 (root (1,1) = 1, parent = key >> 1).
inline int level_of(HeapKey hk) { return static_cast<int>(std::bit_width(hk)); }
inline std::uint32_t index_of(HeapKey hk) { return ((hk << 1) | 1u) - (std::uint32_t{1} << level_of(hk)); }
inline HeapKey heap_key(int level, std::uint32_t index) {
  if (level < 1 || level > 30) throw std::invalid_argument("heap_key: level out of range [1,30]");
  const std::uint32_t last = (std::uint32_t{1} << level) - 1u;
  if ((index & 1u) == 0u || index > last)
    throw std::invalid_argument("heap_key: index must be odd in [1, 2^l - 1], got l=" + std::to_string(level) +
                                " i=" + std::to_string(index));
  return (index + last) >> 1;  // 2^(l-1) + (i-1)/2
}
inline double coordinate_of(HeapKey hk) { return std::ldexp(static_cast<double>(index_of(hk)), -level_of(hk)); }
inline bool has_parent(HeapKey hk) { return hk > 1u; }
inline HeapKey parent_key(HeapKey hk) { return hk >> 1; }
inline int level_sum(const NodeKey& key) {
  int total = 0;
  for (HeapKey hk : key) total += level_of(hk);
  return total;
}
inline void coordinates_of(const NodeKey& key, std::vector<double>& out) {
  out.resize(key.size());
  std::transform(key.begin(), key.end(), out.begin(), [](HeapKey hk) { return coordinate_of(hk); });
}

// ---- 1-d basis (basis.hpp:25-84): same expressions, so host values carry the
// reference's bits (the device kernels restate them exactly).
enum class BasisKind : std::uint8_t { hat, constant_one, left_edge, right_edge };
inline BasisKind basis_kind(int level, std::uint32_t index, BoundaryMode mode) {
  if (mode == BoundaryMode::zero_boundary) return BasisKind::hat;
  if (level == 1) return BasisKind::constant_one;
  if (index == 1u) return BasisKind::left_edge;
  return index == (1u << level) - 1u ? BasisKind::right_edge : BasisKind::hat;
}
inline double basis_value(BasisKind kind, double center, double inv_h, double x) {  // inv_h = 2^l, center = i 2^-l
  double v = 1.0;
  if (kind == BasisKind::constant_one) return v;
  if (kind == BasisKind::left_edge)
    v = 2.0 - x * inv_h;
  else if (kind == BasisKind::right_edge)
    v = 2.0 - (1.0 - x) * inv_h;
  else
    v = 1.0 - std::abs(x - center) * inv_h;
  return v > 0.0 ? v : 0.0;
}
inline double basis_weight(BasisKind kind, double h) {  // integral over [0,1]
  if (kind == BasisKind::constant_one) return 1.0;
  return (kind == BasisKind::left_edge || kind == BasisKind::right_edge) ? 2.0 * h : h;
}
inline double basis_1d(int level, std::uint32_t index, double x, BoundaryMode mode) {
  (void)heap_key(level, index);  // validates the pair
  if (x < 0.0 || x > 1.0) throw std::domain_error("basis_1d: x outside [0,1]");
  const double inv_h = std::ldexp(1.0, level);
  return basis_value(basis_kind(level, index, mode), static_cast<double>(index) / inv_h, inv_h, x);
}
inline double basis_nd(const NodeKey& key, std::span<const double> x, BoundaryMode mode) {
  if (key.size() != x.size()) throw std::invalid_argument("basis_nd: dimension mismatch between key and point");
  double w = 1.0;
  for (std::size_t j = 0; j < key.size() && w != 0.0; ++j)
    w *= basis_1d(level_of(key[j]), index_of(key[j]), x[j], mode);
  return w;
}

// ---- node counts (hdmr.hpp:134-171): |V_{L,n}| = sum_{j<L} C(n-1+j, j) 2^j
// and 1 + sum_{k<=k_max} C(d,k) |V_{L,k}|; std::overflow_error beyond 64 bits.
namespace detail {
inline std::uint64_t checked_mul(std::uint64_t a, std::uint64_t b, const char* who) {
  std::uint64_t r;
  if (__builtin_mul_overflow(a, b, &r)) throw std::overflow_error(std::string(who) + ": 64-bit overflow");
  return r;
}
inline std::uint64_t checked_add(std::uint64_t a, std::uint64_t b, const char* who) {
  std::uint64_t r;
  if (__builtin_add_overflow(a, b, &r)) throw std::overflow_error(std::string(who) + ": 64-bit overflow");
  return r;
}
}  // namespace detail
inline std::uint64_t sg_node_count(int dim, int max_level) {
  constexpr const char* who = "sg_node_count";
  std::uint64_t total = 0;
  for (int j = 0; j < max_level; ++j) {
    std::uint64_t binom = 1;  // C(dim-1+j, j), built factor by factor (exact at every step)
    for (int i = 1; i <= j; ++i)
      binom = detail::checked_mul(binom, static_cast<std::uint64_t>(dim - 1 + i), who) / static_cast<std::uint64_t>(i);
    if (j >= 64) throw std::overflow_error(std::string(who) + ": 64-bit overflow");
    total = detail::checked_add(total, detail::checked_mul(binom, std::uint64_t{1} << j, who), who);
  }
  return total;
}
inline std::uint64_t ddsg_grid_count(int d, int k_max, int max_level) {
  constexpr const char* who = "ddsg_grid_count";
  if (d < 0 || k_max < 0 || k_max > d || max_level < 1) throw std::invalid_argument("ddsg_grid_count: invalid arguments");
  std::uint64_t total = 1;  // the anchor
  for (int k = 1; k <= k_max; ++k) {
    std::uint64_t binom = 1;  // C(d, k)
    for (int i = 1; i <= k; ++i)
      binom = detail::checked_mul(binom, static_cast<std::uint64_t>(d - k + i), who) / static_cast<std::uint64_t>(i);
    total = detail::checked_add(total, detail::checked_mul(binom, sg_node_count(k, max_level), who), who);
  }
  return total;
}

class build_error : public std::runtime_error {  // sparse_grid.hpp:40-48
 public:
  build_error(std::string msg, std::vector<double> point)
      : std::runtime_error(std::move(msg)), point_(std::move(point)) {}
  const std::vector<double>& point() const { return point_; }

 private:
  std::vector<double> point_;
};

class task_error : public std::runtime_error {  // runtime.hpp:71-92
 public:
  task_error(std::size_t task_id, std::exception_ptr cause, const std::string& what)
      : std::runtime_error(what), task_id_(task_id), cause_(std::move(cause)) {}
  std::size_t task_id() const { return task_id_; }
  [[noreturn]] void rethrow_cause() const { std::rethrow_exception(cause_); }

 private:
  std::size_t task_id_;
  std::exception_ptr cause_;
};

namespace detail {

// Status -> the reference's exception types.  `batch` selects the
// evaluate_batch convention (domain errors wrapped in task_error with the
// lowest offending point, runtime.hpp:133-136).
[[noreturn]] inline void raise(ddsg_status s, bool batch = false, int64_t bad = -1) {
  const std::string msg = ddsg_last_error();
  switch (s) {
    case DDSG_INVALID_ARGUMENT:
      throw std::invalid_argument(msg);
    case DDSG_DOMAIN_ERROR:
      if (batch && bad >= 0)
        throw task_error(static_cast<std::size_t>(bad), std::make_exception_ptr(std::domain_error(msg)), msg);
      throw std::domain_error(msg);
    case DDSG_BUILD_ERROR: {
      std::vector<double> p(64);
      const int n = ddsg_last_build_point(p.data(), 64);
      p.resize(static_cast<std::size_t>(n < 64 ? n : 64));
      throw build_error(msg, std::move(p));
    }
    case DDSG_OUT_OF_RANGE:
      throw std::out_of_range(msg);
    case DDSG_OUT_OF_MEMORY:
      throw std::bad_alloc();
    default:
      throw std::runtime_error("ddsg_b200: " + msg);
  }
}

inline void check(ddsg_status s) {
  if (s != DDSG_OK) raise(s);
}

}  // namespace detail

struct GridNode {  // sparse_grid.hpp:55-59
  NodeKey key;
  std::vector<double> surplus;
  bool refined = false;
};

struct SgBuildOptions {  // sparse_grid.hpp:61-67
  int max_level = 1;
  double eps_gamma = 0.0;
  BoundaryMode mode = BoundaryMode::zero_boundary;
  SurplusNorm norm = SurplusNorm::inf;
  unsigned workers = 1;  // accepted for source compatibility; evaluation runs on the GPU
};

using GridEvaluator = std::function<void(std::span<const double>, std::span<double>)>;  // sparse_grid.hpp:70

class SparseGridFunction {
 public:
  SparseGridFunction() = default;

  int dim() const { return dim_; }
  int out_dim() const { return out_dim_; }
  int max_level() const { return max_level_; }
  double eps_gamma() const { return eps_gamma_; }
  BoundaryMode boundary_mode() const { return mode_; }
  std::size_t size() const {
    int64_t n = 0;
    detail::check(ddsg_grid_info(h_.get(), nullptr, nullptr, nullptr, nullptr, nullptr, &n));
    return static_cast<std::size_t>(n);
  }

  // sparse_grid.hpp:84-108
  static SparseGridFunction build(const GridEvaluator& f, int dim, int out_dim, const SgBuildOptions& opt) {
    struct Ctx {
      const GridEvaluator* f;
      int dim, m;
      std::exception_ptr err;
    } ctx{&f, dim, out_dim, nullptr};
    auto tramp = [](const double* xs, int64_t count, double* out, void* c) -> int {
      auto* cx = static_cast<Ctx*>(c);
      try {
        for (int64_t i = 0; i < count; ++i)
          (*cx->f)(std::span<const double>(xs + i * cx->dim, static_cast<std::size_t>(cx->dim)),
                   std::span<double>(out + i * cx->m, static_cast<std::size_t>(cx->m)));
        return 0;
      } catch (...) {
        cx->err = std::current_exception();
        return 1;
      }
    };
    ddsg_grid_t* g = nullptr;
    const ddsg_status s =
        ddsg_grid_build(dim, out_dim, static_cast<int>(opt.mode), opt.max_level, opt.eps_gamma,
                        static_cast<int>(opt.norm), tramp, &ctx, &g);
    if (ctx.err) std::rethrow_exception(ctx.err);  // the evaluator's own error type (sparse_grid.hpp:259-262)
    detail::check(s);
    return SparseGridFunction(g);
  }

  // sparse_grid.hpp:160-179
  static SparseGridFunction from_nodes(int dim, int out_dim, int max_level, double eps_gamma, BoundaryMode mode,
                                       const std::vector<GridNode>& nodes) {
    std::vector<uint32_t> keys;
    std::vector<double> sur;
    keys.reserve(nodes.size() * static_cast<std::size_t>(dim > 0 ? dim : 0));
    sur.reserve(nodes.size() * static_cast<std::size_t>(out_dim > 0 ? out_dim : 0));
    for (const auto& n : nodes) {
      if (n.key.size() != static_cast<std::size_t>(dim))
        throw std::invalid_argument("sparse grid: node key dimension mismatch");
      if (n.surplus.size() != static_cast<std::size_t>(out_dim))
        throw std::invalid_argument("sparse grid: node surplus length mismatch");
      keys.insert(keys.end(), n.key.begin(), n.key.end());
      sur.insert(sur.end(), n.surplus.begin(), n.surplus.end());
    }
    ddsg_grid_t* g = nullptr;
    detail::check(ddsg_grid_create(dim, out_dim, static_cast<int>(mode), max_level, eps_gamma,
                                   static_cast<int64_t>(nodes.size()), keys.data(), sur.data(), &g));
    return SparseGridFunction(g);
  }

  // sparse_grid.hpp:81 (stored order).  Read once from the C-ABI and kept
  // (the grid is immutable through the shim), so repeated calls are cheap.
  const std::vector<GridNode>& nodes() const {
    if (!nodes_) {
      const std::size_t n = size();
      std::vector<uint32_t> keys(n * static_cast<std::size_t>(dim_));
      std::vector<double> sur(n * static_cast<std::size_t>(out_dim_));
      detail::check(ddsg_grid_nodes(h_.get(), keys.data(), sur.data()));
      auto out = std::make_shared<std::vector<GridNode>>(n);
      for (std::size_t i = 0; i < n; ++i) {
        (*out)[i].key.assign(keys.begin() + static_cast<std::ptrdiff_t>(i * dim_),
                             keys.begin() + static_cast<std::ptrdiff_t>((i + 1) * dim_));
        (*out)[i].surplus.assign(sur.begin() + static_cast<std::ptrdiff_t>(i * out_dim_),
                                 sur.begin() + static_cast<std::ptrdiff_t>((i + 1) * out_dim_));
      }
      nodes_ = std::move(out);
    }
    return *nodes_;
  }

  // sparse_grid.hpp:111-128 (one point; std::domain_error outside [0,1]^dim)
  void interpolate(std::span<const double> x, std::span<double> out) const {
    if (x.size() != static_cast<std::size_t>(dim_))
      throw std::invalid_argument("sparse grid: query dimension mismatch");
    if (out.size() != static_cast<std::size_t>(out_dim_))
      throw std::invalid_argument("sparse grid: output length mismatch");
    int64_t bad = -1;
    const ddsg_status s = ddsg_eval_grid(h_.get(), x.data(), 1, out.data(), &bad, nullptr);
    if (s != DDSG_OK) detail::raise(s);
  }
  std::vector<double> interpolate(std::span<const double> x) const {  // sparse_grid.hpp:130-134
    std::vector<double> out(static_cast<std::size_t>(out_dim_));
    interpolate(x, out);
    return out;
  }
  // Batched form (x [n][dim], y [n][m]; host or device pointers); failures
  // follow for_each_index: task_error with the lowest failing point.
  void interpolate_batch(const double* x, int64_t n, double* y, void* stream = nullptr) const {
    int64_t bad = -1;
    const ddsg_status s = ddsg_eval_grid(h_.get(), x, n, y, &bad, stream);
    if (s != DDSG_OK) detail::raise(s, true, bad);
  }

  std::vector<double> quadrature() const {  // sparse_grid.hpp:138-149
    std::vector<double> q(static_cast<std::size_t>(out_dim_));
    detail::check(ddsg_grid_quadrature(h_.get(), q.data()));
    return q;
  }

  // sparse_grid.hpp:151-157: hash lookup of a node key
  bool contains(const NodeKey& key) const {
    if (key.size() != static_cast<std::size_t>(dim_)) return false;
    int64_t idx = -1;
    detail::check(ddsg_grid_find(h_.get(), key.data(), &idx));
    return idx >= 0;
  }
  const GridNode& node_at(const NodeKey& key) const {
    int64_t idx = -1;
    if (key.size() == static_cast<std::size_t>(dim_)) detail::check(ddsg_grid_find(h_.get(), key.data(), &idx));
    if (idx < 0) throw std::out_of_range("sparse grid: node not present");
    return nodes()[static_cast<std::size_t>(idx)];
  }

  // ---- refinement (sparse_grid.hpp:215-298; the steps the reference runs
  // inside build, exposed so a host loop -- or several ranks -- can drive them)
  // next_candidates(s): children of the significant nodes at level sum s,
  // closed under missing ancestors, in insertion order.
  std::vector<NodeKey> refine_candidates(int level_sum) const {
    int64_t n = 0;
    detail::check(ddsg_grid_refine_candidates(h_.get(), level_sum, &n, nullptr));
    std::vector<uint32_t> flat(static_cast<std::size_t>(n) * static_cast<std::size_t>(dim_));
    if (n > 0) detail::check(ddsg_grid_refine_candidates(h_.get(), level_sum, &n, flat.data()));
    std::vector<NodeKey> keys(static_cast<std::size_t>(n));
    for (std::size_t i = 0; i < keys.size(); ++i)
      keys[i].assign(flat.begin() + static_cast<std::ptrdiff_t>(i * dim_),
                     flat.begin() + static_cast<std::ptrdiff_t>((i + 1) * dim_));
    return keys;
  }
  // surplus[i] = f_values[i] - interpolate(this grid, x(keys[i])) (sparse_grid.hpp:264-276),
  // on the GPU, or on the host (the reference's own loop) with on_device = false.
  std::vector<std::vector<double>> hierarchize(const std::vector<NodeKey>& keys,
                                               const std::vector<std::vector<double>>& f_values,
                                               bool on_device = true) const {
    if (keys.size() != f_values.size()) throw std::invalid_argument("sparse grid: keys / values count mismatch");
    std::vector<uint32_t> flat;
    std::vector<double> f, sur(keys.size() * static_cast<std::size_t>(out_dim_));
    for (std::size_t i = 0; i < keys.size(); ++i) {
      if (keys[i].size() != static_cast<std::size_t>(dim_))
        throw std::invalid_argument("sparse grid: node key dimension mismatch");
      if (f_values[i].size() != static_cast<std::size_t>(out_dim_))
        throw std::invalid_argument("sparse grid: node surplus length mismatch");
      flat.insert(flat.end(), keys[i].begin(), keys[i].end());
      f.insert(f.end(), f_values[i].begin(), f_values[i].end());
    }
    const int64_t n = static_cast<int64_t>(keys.size());
    detail::check(on_device ? ddsg_hierarchize(h_.get(), n, flat.data(), f.data(), sur.data())
                            : ddsg_hierarchize_host(h_.get(), n, flat.data(), f.data(), sur.data()));
    std::vector<std::vector<double>> out(keys.size());
    for (std::size_t i = 0; i < out.size(); ++i)
      out[i].assign(sur.begin() + static_cast<std::ptrdiff_t>(i * out_dim_),
                    sur.begin() + static_cast<std::ptrdiff_t>((i + 1) * out_dim_));
    return out;
  }
  // insert_batch's append (sparse_grid.hpp:278-298): the only mutation.  Copies
  // of this object share the grid; needs external synchronisation, like the
  // reference's refinement.
  void append(const std::vector<GridNode>& nodes) {
    std::vector<uint32_t> flat;
    std::vector<double> sur;
    for (const auto& n : nodes) {
      if (n.key.size() != static_cast<std::size_t>(dim_))
        throw std::invalid_argument("sparse grid: node key dimension mismatch");
      if (n.surplus.size() != static_cast<std::size_t>(out_dim_))
        throw std::invalid_argument("sparse grid: node surplus length mismatch");
      flat.insert(flat.end(), n.key.begin(), n.key.end());
      sur.insert(sur.end(), n.surplus.begin(), n.surplus.end());
    }
    detail::check(ddsg_grid_append(h_.get(), static_cast<int64_t>(nodes.size()), flat.data(), sur.data()));
    refresh();
  }
  // Re-reads the grid's properties after a mutation through the C-ABI
  // (append, refine_step): drops the nodes() cache, picks up max_level.
  void refresh() {
    nodes_.reset();
    int lvl = max_level_;
    detail::check(ddsg_grid_info(h_.get(), nullptr, nullptr, nullptr, &lvl, nullptr, nullptr));
    max_level_ = lvl;
  }

  const ddsg_grid_t* handle() const { return h_.get(); }
  ddsg_grid_t* mutable_handle() { return h_.get(); }
  // Takes ownership of a C-ABI grid handle (e.g. from ddsg_grid_from_json).
  static SparseGridFunction adopt(ddsg_grid_t* g) { return SparseGridFunction(g); }

 private:
  struct Del {
    void operator()(ddsg_grid_t* g) const { ddsg_grid_destroy(g); }
  };
  std::shared_ptr<ddsg_grid_t> h_;
  mutable std::shared_ptr<const std::vector<GridNode>> nodes_;  // nodes() cache
  int dim_ = 0, out_dim_ = 0, max_level_ = 0;
  double eps_gamma_ = 0.0;
  BoundaryMode mode_ = BoundaryMode::zero_boundary;

  explicit SparseGridFunction(ddsg_grid_t* g) : h_(g, Del{}) {
    int dim = 0, m = 0, mode = 0, lvl = 0;
    double eps = 0.0;
    int64_t n = 0;
    detail::check(ddsg_grid_info(g, &dim, &m, &mode, &lvl, &eps, &n));
    dim_ = dim;
    out_dim_ = m;
    max_level_ = lvl;
    eps_gamma_ = eps;
    mode_ = mode == DDSG_MODIFIED_LINEAR ? BoundaryMode::modified_linear : BoundaryMode::zero_boundary;
  }
};

// One adaptive refinement step of replicated grids across `world` ranks
// (C-ABI ddsg_refine_step / ddsg_refine_step_nccl): grid g's
// next build batch from level sum level_sums[g] is split over the ranks, each
// rank evaluates `f(g, x, out)` at its share and hierarchizes it on its GPU,
// the surplus rows are all-gathered (ncclAllGather over `nccl_comm`, an
// ncclComm_t, on `stream`) and appended on every rank in batch order, so the
// grids stay bit-identical everywhere and equal to the reference's build at
// the next level.  world == 1: no communicator needed; on_device = false
// hierarchizes on the host (no GPU).
struct RefineStats {
  std::int64_t new_nodes = 0, rounds = 0, gathered_bytes = 0;
  double target_s = 0.0, hierarchize_s = 0.0, allgather_s = 0.0;
};
using NodeEvaluator = std::function<void(int grid, std::span<const double> x, std::span<double> out)>;
inline RefineStats refine_step(const std::vector<SparseGridFunction*>& grids, const std::vector<int>& level_sums,
                               const NodeEvaluator& f, void* nccl_comm = nullptr, int rank = 0, int world = 1,
                               void* stream = nullptr, bool on_device = true) {
  if (grids.size() != level_sums.size()) throw std::invalid_argument("refine_step: one level sum per grid");
  struct Ctx {
    const NodeEvaluator* f;
    const std::vector<SparseGridFunction*>* grids;
    std::exception_ptr err;
  } ctx{&f, &grids, nullptr};
  auto tramp = [](int g, const double* xs, int64_t count, double* out, void* c) -> int {
    auto* cx = static_cast<Ctx*>(c);
    const std::size_t d = static_cast<std::size_t>((*cx->grids)[static_cast<std::size_t>(g)]->dim());
    const std::size_t m = static_cast<std::size_t>((*cx->grids)[static_cast<std::size_t>(g)]->out_dim());
    try {
      for (int64_t i = 0; i < count; ++i)
        (*cx->f)(g, std::span<const double>(xs + i * d, d), std::span<double>(out + i * m, m));
      return 0;
    } catch (...) {
      cx->err = std::current_exception();
      return 1;
    }
  };
  std::vector<ddsg_grid_t*> handles;
  for (SparseGridFunction* g : grids) handles.push_back(g->mutable_handle());
  ddsg_refine_stats st{};
  ddsg_status s;
  if (world > 1 || nccl_comm != nullptr)
    s = ddsg_refine_step_nccl(handles.data(), static_cast<int>(handles.size()), level_sums.data(), tramp, &ctx,
                              nccl_comm, rank, world, stream, &st);
  else
    s = ddsg_refine_step(handles.data(), static_cast<int>(handles.size()), level_sums.data(), tramp, &ctx, 0, 1,
                         nullptr, nullptr, on_device ? 1 : 0, &st);
  for (SparseGridFunction* g : grids) g->refresh();
  if (ctx.err) std::rethrow_exception(ctx.err);
  detail::check(s);
  RefineStats out;
  out.new_nodes = st.new_nodes;
  out.rounds = st.rounds;
  out.gathered_bytes = st.gathered_bytes;
  out.target_s = st.target_s;
  out.hierarchize_s = st.hierarchize_s;
  out.allgather_s = st.allgather_s;
  return out;
}

struct ComponentIndex {  // component_index.hpp:16-54
  std::vector<int> dims;
  std::size_t order() const { return dims.size(); }
  bool empty() const { return dims.empty(); }
  bool operator==(const ComponentIndex& o) const { return dims == o.dims; }
  bool operator<(const ComponentIndex& o) const {
    if (dims.size() != o.dims.size()) return dims.size() < o.dims.size();
    return dims < o.dims;
  }
  bool contains(int d) const { return std::binary_search(dims.begin(), dims.end(), d); }
  bool is_superset_of(const ComponentIndex& sub) const {
    return std::includes(dims.begin(), dims.end(), sub.dims.begin(), sub.dims.end());
  }
  std::string to_string() const {
    if (dims.empty()) return "{}";
    std::string s = "{";
    for (std::size_t i = 0; i < dims.size(); ++i) s += (i ? "," : "") + std::to_string(dims[i]);
    return s + "}";
  }
  static ComponentIndex make(std::vector<int> dims, int d) {
    ComponentIndex u{std::move(dims)};
    std::sort(u.dims.begin(), u.dims.end());
    if (std::adjacent_find(u.dims.begin(), u.dims.end()) != u.dims.end())
      throw std::invalid_argument("component index: duplicate dimension");
    if (!u.dims.empty() && (u.dims.front() < 0 || u.dims.back() >= d))
      throw std::invalid_argument("component index: dimension id out of range");
    return u;
  }
};

struct AnchorPoint {  // hdmr.hpp:27-30
  std::vector<double> coords;
  std::vector<double> f_anchor;
};

struct DdsgOptions {  // hdmr.hpp:166-175 (only the fields evaluation uses matter here)
  int k_max = 1;
  double eps_rho = 0.0, eps_eta = 0.0;
  int max_level = 1;
  double eps_gamma = 0.0;
  BoundaryMode mode = BoundaryMode::modified_linear;
  bool exact_cuts = false;
  unsigned workers = 1;
};

using Evaluator = std::function<void(std::span<const double>, std::span<double>)>;  // hdmr.hpp:40

// component_index.hpp:57-72: the order-k index sets of {0..d-1} in
// lexicographic order -- here as the permutations of a k-of-d selection mask
// (std::prev_permutation walks the masks from 1..10..0 downwards, which lists
// the selected positions lexicographically upwards).
inline std::vector<ComponentIndex> order_k_indices(int d, std::size_t k) {
  std::vector<ComponentIndex> all;
  if (d < 0 || k > static_cast<std::size_t>(d)) return all;
  std::vector<char> pick(static_cast<std::size_t>(d), 0);
  std::fill(pick.begin(), pick.begin() + static_cast<std::ptrdiff_t>(k), 1);
  do {
    ComponentIndex u;
    u.dims.reserve(k);
    for (int j = 0; j < d; ++j)
      if (pick[static_cast<std::size_t>(j)]) u.dims.push_back(j);
    all.push_back(std::move(u));
  } while (std::prev_permutation(pick.begin(), pick.end()));
  return all;
}

// component_index.hpp:75-87: every subset of u in (order, lex) order: each
// dim of u doubles the family built so far (with / without it), then sorted.
inline std::vector<ComponentIndex> all_subsets(const ComponentIndex& u) {
  std::vector<ComponentIndex> family(1);  // the empty index
  family.reserve(std::size_t{1} << u.order());
  for (int dim : u.dims) {
    const std::size_t have = family.size();
    for (std::size_t i = 0; i < have; ++i) {
      ComponentIndex with = family[i];
      with.dims.push_back(dim);  // u.dims ascend, so every member stays sorted
      family.push_back(std::move(with));
    }
  }
  std::sort(family.begin(), family.end());
  return family;
}

struct ExpansionDiagnostics {  // hdmr.hpp:178-186
  struct EtaRecord {
    ComponentIndex index;
    double eta = 0.0;
    bool accepted = true;
  };
  std::vector<double> rho_by_order;                  // rho after orders 1..K (NaN: zero denominator)
  std::vector<std::vector<EtaRecord>> eta_by_order;  // order-k records at [k-1] (order 1: none)
};

class rho_denominator_error : public std::runtime_error {  // hdmr.hpp:100-106
 public:
  rho_denominator_error()
      : std::runtime_error("expansion_rho: order-(k-1) cumulative quadrature is zero; "
                           "treat rho as above-threshold and continue expanding") {}
};

// hdmr.hpp:108-119: ||Q_k - Q_{k-1}||_2 / ||Q_{k-1}||_2 over the outputs (sums in output order).
inline double expansion_rho(const std::vector<double>& cumulative_k, const std::vector<double>& cumulative_km1) {
  double diff2 = 0.0, base2 = 0.0;
  for (std::size_t c = 0; c < cumulative_k.size(); ++c) {
    const double delta = cumulative_k[c] - cumulative_km1[c];
    diff2 += delta * delta;
    base2 += cumulative_km1[c] * cumulative_km1[c];
  }
  if (base2 == 0.0) throw rho_denominator_error();
  return std::sqrt(diff2) / std::sqrt(base2);
}

// hdmr.hpp:124-133: quadrature mass of one component against the lower orders (+inf: accept).
inline double eta_coefficient(const std::vector<double>& component_quadrature,
                              const std::vector<double>& lower_order_sum) {
  double mass2 = 0.0, base2 = 0.0;
  for (std::size_t c = 0; c < component_quadrature.size(); ++c) {
    mass2 += component_quadrature[c] * component_quadrature[c];
    base2 += lower_order_sum[c] * lower_order_sum[c];
  }
  if (base2 == 0.0) return std::numeric_limits<double>::infinity();
  return std::sqrt(mass2) / std::sqrt(base2);
}

// hdmr.hpp:45-77: the sample closest (l1 over the outputs) to the sample mean
// of n_samples uniform draws (std::mt19937_64(seed)); lowest index on ties.
inline AnchorPoint select_anchor(const Evaluator& f, int dim, int out_dim, int n_samples, std::uint64_t seed) {
  if (n_samples < 1) throw std::invalid_argument("select_anchor: n_samples must be >= 1");
  struct Sample {
    std::vector<double> x, fx;
  };
  std::mt19937_64 engine(seed);
  std::uniform_real_distribution<double> unit(0.0, 1.0);
  std::vector<Sample> draws(static_cast<std::size_t>(n_samples));
  std::vector<double> center(static_cast<std::size_t>(out_dim), 0.0);  // sums in sample order, then / n
  for (Sample& s : draws) {
    s.x.resize(static_cast<std::size_t>(dim));
    std::generate(s.x.begin(), s.x.end(), [&] { return unit(engine); });
    s.fx.resize(center.size());
    f(s.x, s.fx);
    for (std::size_t c = 0; c < center.size(); ++c) {
      if (!std::isfinite(s.fx[c])) throw build_error("select_anchor: evaluator returned a non-finite value", s.x);
      center[c] += s.fx[c];
    }
  }
  for (double& c : center) c /= static_cast<double>(n_samples);
  auto l1_to_center = [&](const Sample& s) {
    double dist = 0.0;
    for (std::size_t c = 0; c < center.size(); ++c) dist += std::abs(s.fx[c] - center[c]);
    return dist;
  };
  // the first strict minimum: ties go to the lowest sample index; a sample
  // whose distance is not below +inf (a NaN) can only win as sample 0
  std::size_t best = 0;
  double best_dist = std::numeric_limits<double>::infinity();
  for (std::size_t i = 0; i < draws.size(); ++i)
    if (const double dist = l1_to_center(draws[i]); dist < best_dist) {
      best = i;
      best_dist = dist;
    }
  return AnchorPoint{std::move(draws[best].x), std::move(draws[best].fx)};
}

// hdmr.hpp:81-93: f restricted to the cut through the anchor along the dims of u.
inline Evaluator cut_evaluator(const Evaluator& f, const AnchorPoint& anchor, const ComponentIndex& u) {
  if (u.empty()) throw std::invalid_argument("cut_evaluator: component index must be non-empty");
  return [f, base = anchor.coords, dims = u.dims](std::span<const double> y, std::span<double> out) {
    std::vector<double> x = base;  // per call: safe under concurrent grid builds
    for (std::size_t j = 0; j < dims.size(); ++j) x[static_cast<std::size_t>(dims[j])] = y[j];
    f(x, out);
  };
}

class DdsgFunction;
inline DdsgFunction decompose(const Evaluator& f, int dim, int out_dim, const AnchorPoint& anchor, const DdsgOptions& opt,
                       ExpansionDiagnostics* diag = nullptr);

class DdsgFunction {  // hdmr.hpp:195-356
 public:
  friend DdsgFunction decompose(const Evaluator&, int, int, const AnchorPoint&, const DdsgOptions&,
                                ExpansionDiagnostics*);

  int dim() const { return dim_; }
  int out_dim() const { return out_dim_; }
  int k_max() const { return opt_.k_max; }
  bool exact_cuts() const { return opt_.exact_cuts; }
  const DdsgOptions& options() const { return opt_; }
  const AnchorPoint& anchor() const { return anchor_; }
  const std::map<ComponentIndex, SparseGridFunction>& accepted() const { return accepted_; }
  const std::set<ComponentIndex>& rejected() const { return rejected_; }
  const std::map<ComponentIndex, int>& coeff_b() const { return coeff_b_; }

  // hdmr.hpp:213-218
  const std::vector<double>& cut_quadrature(const ComponentIndex& u) const {
    auto it = cut_quadratures_.find(u);
    if (it == cut_quadratures_.end())
      throw std::out_of_range("ddsg: no quadrature for component index " + u.to_string());
    return it->second;
  }
  const std::map<ComponentIndex, std::vector<double>>& cut_quadratures() const { return cut_quadratures_; }

  // hdmr.hpp:222-231: telescopic combination of cut quadratures (f_u's quadrature)
  std::vector<double> component_quadrature(const ComponentIndex& u) const {
    std::vector<double> q(static_cast<std::size_t>(out_dim_), 0.0);
    const std::size_t k = u.order();
    std::vector<ComponentIndex> subs;  // all_subsets(u) in (order, lex) order (component_index.hpp:75-87)
    for (std::size_t mask = 0; mask < (std::size_t{1} << k); ++mask) {
      ComponentIndex v;
      for (std::size_t j = 0; j < k; ++j)
        if (mask & (std::size_t{1} << j)) v.dims.push_back(u.dims[j]);
      subs.push_back(std::move(v));
    }
    std::sort(subs.begin(), subs.end());
    for (const auto& v : subs) {
      const auto& qc = cut_quadrature(v);
      const double sign = ((u.order() - v.order()) % 2 == 0) ? 1.0 : -1.0;
      for (std::size_t c = 0; c < q.size(); ++c) q[c] += sign * qc[c];
    }
    return q;
  }
  // hdmr.hpp:235-243
  std::vector<double> cumulative_quadrature(std::size_t k) const {
    std::vector<double> q = anchor_.f_anchor;
    for (const auto& [u, grid] : accepted_) {
      if (u.order() > k) continue;
      const auto qu = component_quadrature(u);
      for (std::size_t c = 0; c < q.size(); ++c) q[c] += qu[c];
    }
    return q;
  }

  std::size_t total_grid_points() const {  // hdmr.hpp:245-250
    std::size_t n = 1;
    for (const auto& [u, grid] : accepted_)
      if (!u.empty()) n += grid.size();
    return n;
  }
  std::size_t order_reached() const { return order_reached_; }

  // hdmr.hpp:257-270: the telescopic double sum without deduplication -- for
  // every accepted u, every subset v of u contributes (-1)^(|u|-|v|) times the
  // cut interpolant of v, evaluated anew each time (the vectorized form's
  // oracle; terms are added in (u, v) order).
  void evaluate_naive(std::span<const double> x, std::span<double> out, std::uint64_t* interp_calls = nullptr) const {
    check_point(x);
    std::copy(anchor_.f_anchor.begin(), anchor_.f_anchor.end(), out.begin());  // the u = {} term
    std::vector<double> term(anchor_.f_anchor.size()), restricted;
    for (const auto& entry : accepted_) {
      const ComponentIndex& u = entry.first;
      for (const ComponentIndex& v : all_subsets(u)) {
        evaluate_cut(v, x, restricted, term, interp_calls);
        const bool minus = ((u.order() - v.order()) & 1u) != 0u;
        for (std::size_t c = 0; c < term.size(); ++c) out[c] += minus ? -1.0 * term[c] : 1.0 * term[c];
      }
    }
  }
  std::vector<double> evaluate_naive(std::span<const double> x) const {  // hdmr.hpp:272-276
    std::vector<double> out(static_cast<std::size_t>(out_dim_));
    evaluate_naive(x, out);
    return out;
  }
  // hdmr.hpp:280-297: the cut interpolant of an accepted index at x restricted
  // to its dims (the anchor value for the empty index; counted otherwise).
  void evaluate_cut(const ComponentIndex& v, std::span<const double> x, std::vector<double>& restricted_scratch,
                    std::span<double> out, std::uint64_t* interp_calls = nullptr) const {
    if (v.empty()) {
      std::copy(anchor_.f_anchor.begin(), anchor_.f_anchor.end(), out.begin());
      return;
    }
    restricted_scratch.clear();
    for (int j : v.dims) restricted_scratch.push_back(x[static_cast<std::size_t>(j)]);
    if (interp_calls != nullptr) *interp_calls += 1;
    accepted_.at(v).interpolate(restricted_scratch, out);
  }

  void check_point(std::span<const double> x) const {  // hdmr.hpp:299-304
    if (x.size() != static_cast<std::size_t>(dim_)) throw std::invalid_argument("ddsg: query dimension mismatch");
    for (double v : x)
      if (!(v >= 0.0 && v <= 1.0)) throw std::domain_error("ddsg: query outside unit cube");
  }

  // hdmr.hpp:307-325
  static DdsgFunction from_parts(int dim, int out_dim, DdsgOptions opt, AnchorPoint anchor,
                                 std::map<ComponentIndex, SparseGridFunction> accepted,
                                 std::set<ComponentIndex> rejected, std::map<ComponentIndex, int> coeff_b,
                                 std::map<ComponentIndex, std::vector<double>> cut_quadratures) {
    DdsgFunction f;
    f.dim_ = dim;
    f.out_dim_ = out_dim;
    f.opt_ = opt;
    f.opt_.exact_cuts = false;  // exact-cut closures are not serializable
    f.anchor_ = std::move(anchor);
    f.accepted_ = std::move(accepted);
    f.rejected_ = std::move(rejected);
    f.coeff_b_ = std::move(coeff_b);
    f.cut_quadratures_ = std::move(cut_quadratures);
    for (const auto& [u, grid] : f.accepted_) f.order_reached_ = std::max(f.order_reached_, u.order());
    return f;
  }

 private:
  int dim_ = 0, out_dim_ = 0;
  DdsgOptions opt_;
  AnchorPoint anchor_;
  std::map<ComponentIndex, SparseGridFunction> accepted_;
  std::set<ComponentIndex> rejected_;
  std::map<ComponentIndex, int> coeff_b_;
  std::map<ComponentIndex, std::vector<double>> cut_quadratures_;
  std::size_t order_reached_ = 0;

  // hdmr.hpp:339-355: b_i = sum over accepted u containing i of (-1)^(|u| - |i|).
  void finalize_coefficients() {
    coeff_b_.clear();
    std::vector<const ComponentIndex*> family;
    const ComponentIndex none{};
    family.push_back(&none);
    for (const auto& kv : accepted_) family.push_back(&kv.first);
    for (const ComponentIndex* i : family) {
      int b = 0;
      for (const ComponentIndex* u : family)
        if (u->is_superset_of(*i)) b += ((u->order() - i->order()) % 2 == 0) ? 1 : -1;
      coeff_b_[*i] = b;
    }
  }
};

namespace detail {
// The cut grids of one expansion order, built on `workers` host threads
// (an atomic work queue; a component's result does not depend on the
// schedule).  The lowest failing component reports, as
// "decompose: component {..} failed: <cause>" (hdmr.hpp:425-429).
struct CutBuild {
  SparseGridFunction grid;
  std::vector<double> quadrature;
};
inline std::vector<CutBuild> build_cuts(const Evaluator& f, const AnchorPoint& anchor,
                                        const std::vector<ComponentIndex>& wave, int out_dim,
                                        const DdsgOptions& opt) {
  std::vector<CutBuild> cuts(wave.size());
  std::vector<std::string> failure(wave.size());
  std::vector<char> failed(wave.size(), 0);
  SgBuildOptions grid_opt;
  grid_opt.max_level = opt.max_level;
  grid_opt.eps_gamma = opt.eps_gamma;
  grid_opt.mode = opt.mode;
  std::atomic<std::size_t> queue{0};
  auto drain = [&] {
    for (std::size_t id; (id = queue.fetch_add(1)) < wave.size();) try {
        cuts[id].grid = SparseGridFunction::build(cut_evaluator(f, anchor, wave[id]),
                                                  static_cast<int>(wave[id].order()), out_dim, grid_opt);
        cuts[id].quadrature = cuts[id].grid.quadrature();
      } catch (const std::exception& e) {
        failed[id] = 1;
        failure[id] = e.what();
      } catch (...) {  // nothing may leave a pool thread
        failed[id] = 1;
        failure[id] = "unknown error";
      }
  };
  std::vector<std::thread> pool;
  for (std::size_t t = 1; t < std::min<std::size_t>(std::max(1u, opt.workers), wave.size()); ++t) pool.emplace_back(drain);
  drain();
  for (std::thread& t : pool) t.join();
  for (std::size_t id = 0; id < wave.size(); ++id)
    if (failed[id]) throw std::runtime_error("decompose: component " + wave[id].to_string() + " failed: " + failure[id]);
  return cuts;
}
}  // namespace detail

// hdmr.hpp:364-483: the adaptive decomposition, order by order.  The wave of
// order k is every order-k index without a rejected subset; its cut grids
// are built (detail::build_cuts), eta screens the wave against the
// cumulative quadrature of the lower orders (order 1 is always kept; eps_eta
// = 0 keeps everything), and rho -- the relative change of the cumulative
// quadrature -- ends the expansion.  Grids, quadratures, eta, rho, the
// accepted / rejected sets and b are bit-identical to the reference's
// (tests/cpp/test_ref_dropin.cpp).  exact_cuts is not supported.
inline DdsgFunction decompose(const Evaluator& f, int dim, int out_dim, const AnchorPoint& anchor,
                              const DdsgOptions& opt, ExpansionDiagnostics* diag) {
  if (dim < 1) throw std::invalid_argument("decompose: dim must be >= 1");
  if (opt.k_max < 1 || opt.k_max > dim) throw std::invalid_argument("decompose: k_max must satisfy 1 <= k_max <= dim");
  if (opt.eps_rho < 0.0 || opt.eps_eta < 0.0) throw std::invalid_argument("decompose: thresholds must be >= 0");
  if (anchor.coords.size() != static_cast<std::size_t>(dim)) throw std::invalid_argument("decompose: anchor dimension mismatch");
  if (opt.exact_cuts) throw std::invalid_argument("decompose: exact_cuts is not supported by the B200 drop-in");

  DdsgFunction fn;
  fn.dim_ = dim;
  fn.out_dim_ = out_dim;
  fn.opt_ = opt;
  fn.anchor_ = anchor;
  if (fn.anchor_.f_anchor.empty()) {  // the anchor value, if the caller did not bring it
    fn.anchor_.f_anchor.assign(static_cast<std::size_t>(out_dim), 0.0);
    f(fn.anchor_.coords, fn.anchor_.f_anchor);
  }
  fn.cut_quadratures_.emplace(ComponentIndex{}, fn.anchor_.f_anchor);

  const auto has_rejected_subset = [&fn](const ComponentIndex& u) {
    return std::any_of(fn.rejected_.begin(), fn.rejected_.end(),
                       [&u](const ComponentIndex& z) { return u.is_superset_of(z); });
  };
  for (std::size_t order = 1; order <= static_cast<std::size_t>(opt.k_max); ++order) {
    std::vector<ComponentIndex> wave = order_k_indices(dim, order);
    wave.erase(std::remove_if(wave.begin(), wave.end(), has_rejected_subset), wave.end());
    if (wave.empty()) break;
    std::vector<detail::CutBuild> cuts = detail::build_cuts(f, fn.anchor_, wave, out_dim, opt);

    const std::vector<double> below = fn.cumulative_quadrature(order - 1);  // orders < k, before this wave
    std::vector<ExpansionDiagnostics::EtaRecord> screened;
    for (std::size_t id = 0; id < wave.size(); ++id) {
      const ComponentIndex& u = wave[id];
      fn.cut_quadratures_[u] = std::move(cuts[id].quadrature);  // component_quadrature(u) reads it
      double eta = std::numeric_limits<double>::quiet_NaN();
      bool keep = true;
      if (order >= 2) {
        eta = eta_coefficient(fn.component_quadrature(u), below);
        keep = opt.eps_eta == 0.0 || eta > opt.eps_eta;
        screened.push_back({u, eta, keep});
      }
      if (keep) {
        fn.accepted_[u] = std::move(cuts[id].grid);
      } else {
        fn.cut_quadratures_.erase(u);
        fn.rejected_.insert(u);
      }
    }
    fn.order_reached_ = order;
    if (diag) {
      if (diag->eta_by_order.size() < order) diag->eta_by_order.resize(order);
      auto& slot = diag->eta_by_order[order - 1];
      slot.insert(slot.end(), screened.begin(), screened.end());
    }

    double rho = std::numeric_limits<double>::quiet_NaN();  // stays NaN on a zero denominator: no evidence, go on
    try {
      rho = expansion_rho(fn.cumulative_quadrature(order), below);
    } catch (const rho_denominator_error&) {
    }
    if (diag) diag->rho_by_order.push_back(rho);
    if (rho < opt.eps_rho) break;  // false for NaN
  }
  fn.finalize_coefficients();
  return fn;
}

// Reusable evaluation buffers (ddsg_eval.hpp:21-24): pinned host staging,
// device buffers and a stream, created on first use on the current device.
// Like the reference's, one workspace serves one thread at a time; copies
// start with fresh buffers.
class EvalWorkspace {
 public:
  EvalWorkspace() = default;
  EvalWorkspace(const EvalWorkspace&) {}
  EvalWorkspace& operator=(const EvalWorkspace&) { return *this; }
  EvalWorkspace(EvalWorkspace&& o) noexcept : h_(o.h_) { o.h_ = nullptr; }
  EvalWorkspace& operator=(EvalWorkspace&& o) noexcept {
    std::swap(h_, o.h_);
    return *this;
  }
  ~EvalWorkspace() {
    if (h_) ddsg_workspace_destroy(h_);
  }
  ddsg_workspace_t* handle() {
    if (!h_) detail::check(ddsg_workspace_create(&h_));
    return h_;
  }

 private:
  ddsg_workspace_t* h_ = nullptr;
};

class VectorizedDdsg {  // ddsg_eval.hpp:28-165
 public:
  VectorizedDdsg() = default;

  // ddsg_eval.hpp:40-74 — same validation (null source, non-accepted
  // coefficient, missing subsets) through ddsg_hdmr_create.
  static VectorizedDdsg compile(std::shared_ptr<const DdsgFunction> source) {
    if (!source) throw std::invalid_argument("vectorized ddsg: null source");
    VectorizedDdsg v;
    v.source_ = source;
    v.dim_ = source->dim();
    v.out_dim_ = source->out_dim();
    std::vector<int32_t> order, dims, b;
    std::vector<const ddsg_grid_t*> grids;
    for (const auto& [u, bu] : source->coeff_b()) {
      order.push_back(static_cast<int32_t>(u.order()));
      for (int dd : u.dims) dims.push_back(dd);
      b.push_back(bu);
      if (u.empty()) {
        grids.push_back(nullptr);
      } else {
        auto it = source->accepted().find(u);
        if (it == source->accepted().end())
          throw std::invalid_argument("vectorized ddsg: coefficient for a non-accepted index");
        grids.push_back(it->second.handle());
      }
    }
    if (source->anchor().f_anchor.size() != static_cast<std::size_t>(v.out_dim_))
      throw std::invalid_argument("vectorized ddsg: anchor value length != out_dim");
    ddsg_hdmr_t* h = nullptr;
    detail::check(ddsg_hdmr_create(v.dim_, v.out_dim_, source->anchor().f_anchor.data(),
                                   static_cast<int>(order.size()), order.data(), dims.data(), b.data(),
                                   grids.data(), &h));
    v.h_.reset(h, [](ddsg_hdmr_t* p) { ddsg_hdmr_destroy(p); });
    for (const auto& [u, bu] : source->coeff_b()) {
      Slot sl;
      sl.index = u;
      sl.b = bu;
      if (!u.empty()) sl.grid = &source->accepted().find(u)->second;
      v.slots_.push_back(std::move(sl));
    }
    return v;
  }

  struct Slot {  // ddsg_eval.hpp:30-34
    ComponentIndex index;
    int b = 0;
    const SparseGridFunction* grid = nullptr;  // null for the empty index
  };

  int dim() const { return dim_; }
  int out_dim() const { return out_dim_; }
  const std::vector<Slot>& slots() const { return slots_; }  // ddsg_eval.hpp:77
  const DdsgFunction& source() const { return *source_; }

  // ddsg_eval.hpp:83-113 (one point, the reference's hot-loop entry): the
  // point is staged through `ws`; `interp_calls`, when given, counts cut
  // evaluations (one per active non-empty slot).
  void evaluate(std::span<const double> x, std::span<double> out, EvalWorkspace& ws,
                std::uint64_t* interp_calls = nullptr) const {
    source_->check_point(x);  // dimension, then domain (hdmr.hpp:299-304)
    if (out.size() != static_cast<std::size_t>(out_dim_))
      throw std::invalid_argument("vectorized ddsg: output length mismatch");
    int64_t bad = -1;
    const ddsg_status s = ddsg_eval_hdmr_ws(h_.get(), ws.handle(), x.data(), 1, out.data(), &bad, interp_calls);
    if (s != DDSG_OK) detail::raise(s);
  }
  // ddsg_eval.hpp:115-119
  void evaluate(std::span<const double> x, std::span<double> out, std::uint64_t* interp_calls = nullptr) const {
    thread_local EvalWorkspace ws;
    evaluate(x, out, ws, interp_calls);
  }
  std::vector<double> evaluate(std::span<const double> x) const {
    std::vector<double> out(static_cast<std::size_t>(out_dim_));
    evaluate(x, out);
    return out;
  }

  // ddsg_eval.hpp:130-139: elementwise equal to evaluate, independent of
  // `workers`; a failing point raises task_error with the lowest failing
  // index (a wrong query length or a point outside the unit cube, whichever
  // comes first, like for_each_index).  The rows are staged straight from
  // and into the vectors (ddsg_eval_hdmr_rows, no flattened copy).
  std::vector<std::vector<double>> evaluate_batch(const std::vector<std::vector<double>>& xs,
                                                  unsigned workers = 1) const {
    (void)workers;
    const std::size_t n = xs.size();
    std::size_t first_bad_dim = n;
    for (std::size_t i = 0; i < n && first_bad_dim == n; ++i)
      if (xs[i].size() != static_cast<std::size_t>(dim_)) first_bad_dim = i;
    // the result rows (allocated on several threads for large batches: the
    // reference allocates them inside its workers too, ddsg_eval.hpp:134-136)
    std::vector<std::vector<double>> out(n);
    std::vector<const double*> xr(first_bad_dim);
    std::vector<double*> yr(first_bad_dim);
    auto alloc = [&](std::size_t lo, std::size_t hi) {
      for (std::size_t i = lo; i < hi; ++i) {
        out[i].resize(static_cast<std::size_t>(out_dim_));
        if (i < first_bad_dim) {
          xr[i] = xs[i].data();
          yr[i] = out[i].data();
        }
      }
    };
    const std::size_t nt = n < (std::size_t{1} << 16) ? 1 : std::min<std::size_t>(8, std::max(1u, std::thread::hardware_concurrency()));
    if (nt <= 1) {
      alloc(0, n);
    } else {
      std::vector<std::thread> pool;
      const std::size_t part = (n + nt - 1) / nt;
      for (std::size_t t = 0; t < nt; ++t)
        if (t * part < n) pool.emplace_back(alloc, t * part, std::min(n, (t + 1) * part));
      for (auto& th : pool) th.join();
    }
    thread_local EvalWorkspace ws;
    int64_t bad = -1;
    const ddsg_status s = ddsg_eval_hdmr_rows(h_.get(), ws.handle(), xr.data(), static_cast<int64_t>(first_bad_dim),
                                              yr.data(), &bad);
    if (s != DDSG_OK) detail::raise(s, true, bad);
    if (first_bad_dim < n)
      throw task_error(first_bad_dim,
                       std::make_exception_ptr(std::invalid_argument("ddsg: query dimension mismatch")),
                       "task " + std::to_string(first_bad_dim) + " failed: ddsg: query dimension mismatch");
    return out;
  }
  // Flat form: x [n][dim] -> y [n][m], host or device pointers.
  void evaluate_batch(const double* x, int64_t n, double* y, void* stream = nullptr) const {
    int64_t bad = -1;
    const ddsg_status s = ddsg_eval_hdmr(h_.get(), x, n, y, &bad, stream);
    if (s != DDSG_OK) detail::raise(s, true, bad);
  }

  std::vector<double> quadrature() const {  // ddsg_eval.hpp:143-151
    std::vector<double> q(static_cast<std::size_t>(out_dim_));
    detail::check(ddsg_hdmr_quadrature(h_.get(), q.data()));
    return q;
  }

  const ddsg_hdmr_t* handle() const { return h_.get(); }

 private:
  std::shared_ptr<const DdsgFunction> source_;
  std::shared_ptr<ddsg_hdmr_t> h_;
  std::vector<Slot> slots_;
  int dim_ = 0, out_dim_ = 0;
};

// The time iteration's convergence measure (time_iteration.hpp:213-223): the
// sup-norm change max_x max_c |p_new(x)[c] - p_prev(x)[c]| over a point set,
// as two batched evaluations instead of two per-point calls per sample.
inline double policy_change(const VectorizedDdsg& p_new, const VectorizedDdsg& p_prev,
                            const std::vector<std::vector<double>>& points) {
  if (p_new.dim() != p_prev.dim() || p_new.out_dim() != p_prev.out_dim())
    throw std::invalid_argument("policy_change: the two policies differ in shape");
  const std::size_t n = points.size(), d = static_cast<std::size_t>(p_new.dim()),
                    m = static_cast<std::size_t>(p_new.out_dim());
  std::vector<double> x(n * d), a(n * m), b(n * m);
  for (std::size_t i = 0; i < n; ++i) {
    if (points[i].size() != d) throw std::invalid_argument("ddsg: query dimension mismatch");
    std::copy(points[i].begin(), points[i].end(), x.begin() + static_cast<std::ptrdiff_t>(i * d));
  }
  p_new.evaluate_batch(x.data(), static_cast<int64_t>(n), a.data());
  p_prev.evaluate_batch(x.data(), static_cast<int64_t>(n), b.data());
  double change = 0.0;
  for (std::size_t k = 0; k < a.size(); ++k) change = std::max(change, std::abs(a[k] - b[k]));
  return change;
}

// ------------------------------------------------------------ JSON documents
// serialize.hpp:17-160 with JsonDocument in place of nlohmann::json: the
// text of a schema-version-1 document; load_json / save_json do the file
// I/O and the C-ABI (ddsg_*_from_json / ddsg_*_to_json) parses and writes.
struct JsonDocument {
  std::string text;
  std::string dump(int = 2) const { return text; }
};

inline constexpr int kSchemaVersion = 1;  // serialize.hpp:17

inline std::string to_string(BoundaryMode mode) {  // serialize.hpp:19-21
  return mode == BoundaryMode::zero_boundary ? "zero_boundary" : "modified_linear";
}
inline BoundaryMode boundary_mode_from_string(const std::string& s) {  // serialize.hpp:23-27
  if (s == "zero_boundary") return BoundaryMode::zero_boundary;
  if (s == "modified_linear") return BoundaryMode::modified_linear;
  throw std::invalid_argument("unknown boundary mode: " + s);
}

namespace detail {
template <typename F>
JsonDocument read_text(F&& writer) {
  int64_t len = 0;
  check(writer(nullptr, 0, &len));
  std::string text(static_cast<std::size_t>(len) + 1, '\0');
  check(writer(text.data(), len + 1, &len));
  text.resize(static_cast<std::size_t>(len));
  return JsonDocument{std::move(text)};
}
}  // namespace detail

inline JsonDocument to_json(const SparseGridFunction& g) {  // serialize.hpp:31-52
  return detail::read_text(
      [&](char* b, int64_t cap, int64_t* len) { return ddsg_grid_to_json(g.handle(), b, cap, len); });
}

inline SparseGridFunction sparse_grid_from_json(const JsonDocument& doc) {  // serialize.hpp:54-77
  ddsg_grid_t* g = nullptr;
  detail::check(ddsg_grid_from_json(doc.text.data(), static_cast<int64_t>(doc.text.size()), &g));
  return SparseGridFunction::adopt(g);
}

inline JsonDocument to_json(const DdsgFunction& f) {  // serialize.hpp:84-110
  if (f.exact_cuts()) throw std::invalid_argument("ddsg document: exact-cut decompositions are not serializable");
  std::vector<int32_t> order, dims, b;
  std::vector<const ddsg_grid_t*> grids;
  std::vector<double> quads;
  for (const auto& [u, bu] : f.coeff_b()) {
    order.push_back(static_cast<int32_t>(u.order()));
    for (int dd : u.dims) dims.push_back(dd);
    b.push_back(bu);
    auto it = f.accepted().find(u);
    grids.push_back(u.empty() ? nullptr : (it == f.accepted().end() ? nullptr : it->second.handle()));
    const auto& q = f.cut_quadrature(u);  // std::out_of_range when absent, like the reference
    quads.insert(quads.end(), q.begin(), q.end());
  }
  ddsg_hdmr_t* h = nullptr;
  detail::check(ddsg_hdmr_create(f.dim(), f.out_dim(), f.anchor().f_anchor.data(), static_cast<int>(order.size()),
                                 order.data(), dims.data(), b.data(), grids.data(), &h));
  std::unique_ptr<ddsg_hdmr_t, ddsg_status (*)(ddsg_hdmr_t*)> hold(h, ddsg_hdmr_destroy);
  std::vector<int32_t> rorder, rdims;
  for (const auto& u : f.rejected()) {
    rorder.push_back(static_cast<int32_t>(u.order()));
    for (int dd : u.dims) rdims.push_back(dd);
  }
  if (f.anchor().coords.size() != static_cast<std::size_t>(f.dim()))
    throw std::invalid_argument("ddsg document: anchor coordinates length != dim");
  detail::check(ddsg_hdmr_set_document(h, f.k_max(), f.anchor().coords.data(), static_cast<int>(rorder.size()),
                                       rorder.data(), rdims.data(), quads.data()));
  return detail::read_text([&](char* buf, int64_t cap, int64_t* len) { return ddsg_hdmr_to_json(h, buf, cap, len); });
}

inline DdsgFunction ddsg_from_json(const JsonDocument& doc) {  // serialize.hpp:112-145
  ddsg_hdmr_t* h = nullptr;
  detail::check(ddsg_hdmr_from_json(doc.text.data(), static_cast<int64_t>(doc.text.size()), &h));
  std::unique_ptr<ddsg_hdmr_t, ddsg_status (*)(ddsg_hdmr_t*)> hold(h, ddsg_hdmr_destroy);
  int d = 0, m = 0, n_slots = 0;
  detail::check(ddsg_hdmr_info(h, &d, &m, &n_slots, nullptr, nullptr));
  int k_max = 1, n_rej = 0, has_q = 0;
  int64_t n_rej_dims = 0;
  detail::check(ddsg_hdmr_document(h, &k_max, nullptr, nullptr, &n_rej, &n_rej_dims, nullptr, nullptr, &has_q,
                                   nullptr));
  AnchorPoint anchor;
  anchor.coords.resize(static_cast<std::size_t>(d));
  anchor.f_anchor.resize(static_cast<std::size_t>(m));
  std::vector<int32_t> rorder(static_cast<std::size_t>(n_rej)), rdims(static_cast<std::size_t>(n_rej_dims));
  std::vector<double> quads(has_q ? static_cast<std::size_t>(n_slots) * static_cast<std::size_t>(m) : 0);
  detail::check(ddsg_hdmr_document(h, nullptr, anchor.coords.data(), anchor.f_anchor.data(), nullptr, nullptr,
                                   rorder.data(), rdims.data(), nullptr, has_q ? quads.data() : nullptr));
  DdsgOptions opt;
  opt.k_max = k_max;
  std::map<ComponentIndex, SparseGridFunction> accepted;
  std::map<ComponentIndex, int> coeff_b;
  std::map<ComponentIndex, std::vector<double>> cut_q;
  std::vector<int32_t> sd(static_cast<std::size_t>(d));
  for (int s = 0; s < n_slots; ++s) {
    int order = 0;
    int32_t bu = 0;
    ddsg_grid_t* g = nullptr;
    detail::check(ddsg_hdmr_slot(h, s, &order, sd.data(), &bu, &g));
    ComponentIndex u{std::vector<int>(sd.begin(), sd.begin() + order)};
    coeff_b[u] = bu;
    if (has_q)
      cut_q[u] = std::vector<double>(quads.begin() + static_cast<std::ptrdiff_t>(s) * m,
                                     quads.begin() + static_cast<std::ptrdiff_t>(s + 1) * m);
    if (g) {
      SparseGridFunction grid = SparseGridFunction::adopt(g);
      opt.max_level = grid.max_level();  // serialize.hpp:124-127
      opt.eps_gamma = grid.eps_gamma();
      opt.mode = grid.boundary_mode();
      accepted.emplace(std::move(u), std::move(grid));
    }
  }
  std::set<ComponentIndex> rejected;
  for (std::size_t r = 0, off = 0; r < rorder.size(); off += static_cast<std::size_t>(rorder[r]), ++r)
    rejected.insert(ComponentIndex{std::vector<int>(rdims.begin() + static_cast<std::ptrdiff_t>(off),
                                                    rdims.begin() + static_cast<std::ptrdiff_t>(off + rorder[r]))});
  return DdsgFunction::from_parts(d, m, opt, std::move(anchor), std::move(accepted), std::move(rejected),
                                  std::move(coeff_b), std::move(cut_q));
}

inline void save_json(const JsonDocument& doc, const std::string& path) {  // serialize.hpp:147-152
  std::ofstream out(path);
  if (!out) throw std::runtime_error("cannot open for writing: " + path);
  out << doc.text;  // already dump(2) + "\n"
}

inline JsonDocument load_json(const std::string& path) {  // serialize.hpp:154-160
  std::ifstream in(path);
  if (!in) throw std::runtime_error("cannot open for reading: " + path);
  std::ostringstream ss;
  ss << in.rdbuf();
  return JsonDocument{ss.str()};
}

}  // namespace ddsg_b200

// ---------------------------------------------------------------------------
// Batched IRBC policy callers: irbc.hpp /
// solver.hpp names, with the per-point loops replaced by batches whose
// successor states are evaluated in one device call.
namespace ddsg_b200::irbc {

enum class Variant { smooth, nonsmooth };  // irbc.hpp:25

struct IrbcParameters {  // irbc.hpp:27-53, same defaults
  int countries = 2;
  double beta = 0.99;
  double alpha = 0.36;
  double delta = 0.01;
  double sigma = 0.01;
  double rho_a = 0.95;
  double phi_adj = 0.50;
  double gamma_base = 0.25;
  std::vector<double> gamma;
  Variant variant = Variant::smooth;
  double lna_half_width = 0.4;
  double k_lo = 0.5;
  double k_hi = 1.5;
  double A = 0.0;
  std::vector<double> tau;

  int state_dim() const { return 2 * countries; }
  int policy_dim() const { return variant == Variant::smooth ? countries + 1 : 2 * countries + 1; }
};

namespace detail {
// Flat view of the parameters; gamma/tau buffers live in the caller's object.
inline ddsg_irbc_params flat(IrbcParameters& p) {
  p.gamma.resize(static_cast<std::size_t>(p.countries > 0 ? p.countries : 0));
  p.tau.resize(p.gamma.size());
  ddsg_irbc_params c{};
  c.countries = p.countries;
  c.variant = p.variant == Variant::smooth ? DDSG_IRBC_SMOOTH : DDSG_IRBC_NONSMOOTH;
  c.beta = p.beta;
  c.alpha = p.alpha;
  c.delta = p.delta;
  c.sigma = p.sigma;
  c.rho_a = p.rho_a;
  c.phi_adj = p.phi_adj;
  c.gamma_base = p.gamma_base;
  c.lna_half_width = p.lna_half_width;
  c.k_lo = p.k_lo;
  c.k_hi = p.k_hi;
  c.A = p.A;
  c.gamma = p.gamma.data();
  c.tau = p.tau.data();
  return c;
}
}  // namespace detail

// irbc.hpp:59-92
inline void refresh_derived(IrbcParameters& p) {
  if (!p.gamma.empty() && p.gamma.size() != static_cast<std::size_t>(p.countries))
    throw std::invalid_argument("irbc: gamma length must equal countries");
  const bool fill = p.gamma.empty();
  ddsg_irbc_params c = detail::flat(p);
  ::ddsg_b200::detail::check(ddsg_irbc_refresh_derived(&c, fill ? 1 : 0));
  p.A = c.A;
}

inline IrbcParameters make_parameters(int countries, Variant variant, double gamma_base = 0.25) {
  IrbcParameters p;  // irbc.hpp:94-101
  p.countries = countries;
  p.variant = variant;
  p.gamma_base = gamma_base;
  refresh_derived(p);
  return p;
}

inline double steady_state_lambda(IrbcParameters p) {  // irbc.hpp:248-263
  ddsg_irbc_params c = detail::flat(p);
  double lam = 0.0;
  ::ddsg_b200::detail::check(ddsg_irbc_steady_state_lambda(&c, &lam));
  return lam;
}

// foc_residuals (irbc.hpp:306-361) for n states: a, k [n][N], candidate /
// residuals [n][pdim]; returns the clamped-successor count per state.
// Host or device pointers.
inline std::vector<int32_t> foc_residuals_batch(const VectorizedDdsg& policy_next, IrbcParameters p, int64_t n,
                                                const double* a, const double* k, const double* candidate,
                                                double* residuals, void* stream = nullptr) {
  ddsg_irbc_params c = detail::flat(p);
  std::vector<int32_t> clamped(static_cast<std::size_t>(n));
  int64_t bad = -1;
  const ddsg_status s = ddsg_irbc_foc_residuals(policy_next.handle(), nullptr, &c, n, a, k, candidate, residuals,
                                                clamped.data(), &bad, stream);
  if (s != DDSG_OK) ::ddsg_b200::detail::raise(s, true, bad);
  return clamped;
}

// foc_jacobian (solver.hpp:129-165) for n states: jac [n][pdim][pdim].
inline void foc_jacobian_batch(const VectorizedDdsg& policy_next, IrbcParameters p, int64_t n, const double* a,
                               const double* k, const double* z, const double* r0, double* jac,
                               double fd_epsilon = 1e-7, void* stream = nullptr) {
  ddsg_irbc_params c = detail::flat(p);
  int64_t bad = -1;
  const ddsg_status s =
      ddsg_irbc_foc_jacobian(policy_next.handle(), nullptr, &c, n, a, k, z, r0, fd_epsilon, jac, &bad, stream);
  if (s != DDSG_OK) ::ddsg_b200::detail::raise(s, true, bad);
}

struct EulerErrors {  // solver.hpp:369-373
  double avg_log10 = 0.0;
  double max_log10 = 0.0;
  std::vector<double> samples;
};

// euler_errors (solver.hpp:377-436): the same sample stream
// (std::mt19937_64(seed), uniform (0,1), point-major); `workers` kept for
// signature parity (the result never depends on it).
inline EulerErrors euler_errors(const VectorizedDdsg& policy, IrbcParameters p, int n_samples, uint64_t seed,
                                unsigned workers = 1, uint64_t* clamp_count = nullptr) {
  (void)workers;
  if (n_samples < 1) throw std::invalid_argument("euler_errors: n_samples must be >= 1");
  std::vector<double> xs(static_cast<std::size_t>(n_samples) * static_cast<std::size_t>(p.state_dim()));
  ddsg_uniform_points(seed, n_samples, p.state_dim(), xs.data());
  ddsg_irbc_params c = detail::flat(p);
  EulerErrors out;
  out.samples.resize(static_cast<std::size_t>(n_samples));
  double mean = 0.0, worst = 0.0;
  uint64_t cl = 0;
  int64_t bad = -1;
  const ddsg_status s = ddsg_irbc_euler_errors(policy.handle(), nullptr, &c, n_samples, xs.data(),
                                               out.samples.data(), &mean, &worst, &cl, &bad, nullptr);
  if (s != DDSG_OK) ::ddsg_b200::detail::raise(s);
  out.avg_log10 = std::log10(std::max(mean, 1e-16));
  out.max_log10 = std::log10(std::max(worst, 1e-16));
  if (clamp_count) *clamp_count += cl;
  return out;
}

}  // namespace ddsg_b200::irbc
