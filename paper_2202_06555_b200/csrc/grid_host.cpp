// Host-side sparse grid: from_nodes, adaptive build, quadrature, layout compiler.
// Compiled with -ffp-contract=off: every floating-point expression below must
// round exactly like the reference's Release build (mul then add, no FMA).
#include "grid_host.hpp"

#include <cstring>

#include <algorithm>
#include <cmath>
#include <limits>
#include <map>
#include <numeric>
#include <sstream>
#include <unordered_set>

namespace ddsg_b200 {

double basis_value_host(int mode, int level, uint32_t index, double x) {
  // basis_kind (basis.hpp:27-33) + basis_value (basis.hpp:36-54).
  const double inv_h = std::ldexp(1.0, level);
  const double center = static_cast<double>(index) / inv_h;
  if (mode == DDSG_MODIFIED_LINEAR) {
    if (level == 1) return 1.0;
    if (index == 1u) {
      const double v = 2.0 - x * inv_h;
      return v > 0.0 ? v : 0.0;
    }
    if (index == (1u << level) - 1u) {
      const double v = 2.0 - (1.0 - x) * inv_h;
      return v > 0.0 ? v : 0.0;
    }
  }
  const double v = 1.0 - std::abs(x - center) * inv_h;
  return v > 0.0 ? v : 0.0;
}

static double basis_weight_host(int mode, int level, uint32_t index) {
  // basis_weight (basis.hpp:57-65) with h = 1 / inv_h.
  const double h = 1.0 / std::ldexp(1.0, level);
  if (mode == DDSG_MODIFIED_LINEAR) {
    if (level == 1) return 1.0;
    if (index == 1u || index == (1u << level) - 1u) return 2.0 * h;
  }
  return h;
}

static int level_sum_of(const uint32_t* key, int dim) {
  int s = 0;
  for (int j = 0; j < dim; ++j) s += level_of(key[j]);
  return s;
}

static inline uint64_t key_hash(const uint32_t* k, int dim) {
  uint64_t h = 0xcbf29ce484222325ull;  // FNV-1a (grid_index.hpp:60-69)
  for (int j = 0; j < dim; ++j) {
    h ^= k[j];
    h *= 0x100000001b3ull;
  }
  return h ^ (h >> 29);
}

// Flat open-addressing set of dim-word keys stored in an arena (next_candidates).
namespace {
struct KeySet {
  int dim;
  std::vector<uint32_t> arena;
  std::vector<int64_t> table = std::vector<int64_t>(1024, -1);
  int64_t n = 0;
  explicit KeySet(int d) : dim(d) {}
  bool contains(const uint32_t* k) const {
    const uint64_t mask = table.size() - 1;
    for (uint64_t h = key_hash(k, dim) & mask;; h = (h + 1) & mask) {
      const int64_t id = table[h];
      if (id < 0) return false;
      if (std::memcmp(&arena[id * dim], k, sizeof(uint32_t) * dim) == 0) return true;
    }
  }
  bool insert(const uint32_t* k) {  // false if present
    if ((n + 1) * 2 > static_cast<int64_t>(table.size())) grow();
    const uint64_t mask = table.size() - 1;
    uint64_t h = key_hash(k, dim) & mask;
    for (;; h = (h + 1) & mask) {
      const int64_t id = table[h];
      if (id < 0) break;
      if (std::memcmp(&arena[id * dim], k, sizeof(uint32_t) * dim) == 0) return false;
    }
    arena.insert(arena.end(), k, k + dim);
    table[h] = n++;
    return true;
  }
  void grow() {
    std::vector<int64_t> t(table.size() * 2, -1);
    const uint64_t mask = t.size() - 1;
    for (int64_t id = 0; id < n; ++id) {
      uint64_t h = key_hash(&arena[id * dim], dim) & mask;
      while (t[h] >= 0) h = (h + 1) & mask;
      t[h] = id;
    }
    table.swap(t);
  }
};
}  // namespace

void HostGrid::rebuild_index(int64_t n_nodes) {
  size_t cap = 1024;
  while (cap < static_cast<size_t>(n_nodes) * 2) cap *= 2;
  table_.assign(cap, -1);
  indexed_ = 0;
  for (int64_t i = 0; i < n_nodes; ++i) index_node(i);
}

void HostGrid::index_node(int64_t i) {
  if ((indexed_ + 1) * 2 > static_cast<int64_t>(table_.size())) {
    const int64_t n = indexed_;
    size_t cap = std::max<size_t>(1024, table_.size() * 2);
    table_.assign(cap, -1);
    indexed_ = 0;
    for (int64_t r = 0; r < n; ++r) index_node(r);
  }
  const uint32_t* k = &keys[i * dim];
  const uint64_t mask = table_.size() - 1;
  uint64_t h = key_hash(k, dim) & mask;
  for (;; h = (h + 1) & mask) {
    const int64_t id = table_[h];
    if (id < 0) break;
    if (std::memcmp(&keys[id * dim], k, sizeof(uint32_t) * dim) == 0)
      fail(DDSG_INVALID_ARGUMENT, "sparse grid: duplicate node key");
  }
  table_[h] = i;
  ++indexed_;
}

bool HostGrid::contains(const uint32_t* key) const { return find(key) >= 0; }

int64_t HostGrid::find(const uint32_t* key) const {
  if (table_.empty()) return -1;
  const uint64_t mask = table_.size() - 1;
  for (uint64_t h = key_hash(key, dim) & mask;; h = (h + 1) & mask) {
    const int64_t id = table_[h];
    if (id < 0) return -1;
    if (std::memcmp(&keys[id * dim], key, sizeof(uint32_t) * dim) == 0) return id;
  }
}

static void validate_keys(int dim, int64_t n, const uint32_t* keys) {
  for (int64_t i = 0; i < n * dim; ++i)
    if (!valid_key(keys[i]))
      fail(DDSG_INVALID_ARGUMENT, "sparse grid: invalid heap key " + std::to_string(keys[i]) +
                                      " (level must be in [1,30])");
}

HostGrid HostGrid::from_nodes(int dim, int m, int mode, int max_level, double eps_gamma, int64_t n,
                              const uint32_t* keys, const double* surplus) {
  if (dim < 1) fail(DDSG_INVALID_ARGUMENT, "sparse grid: dim must be >= 1");
  if (m < 1) fail(DDSG_INVALID_ARGUMENT, "sparse grid: out_dim must be >= 1");
  if (mode != DDSG_ZERO_BOUNDARY && mode != DDSG_MODIFIED_LINEAR)
    fail(DDSG_INVALID_ARGUMENT, "sparse grid: unknown boundary mode");
  if (n < 0 || (n > 0 && (!keys || !surplus)))
    fail(DDSG_INVALID_ARGUMENT, "sparse grid: null node arrays");
  validate_keys(dim, n, keys);
  HostGrid g;
  g.dim = dim;
  g.m = m;
  g.mode = mode;
  g.max_level = max_level;
  g.eps_gamma = eps_gamma;
  g.keys.assign(keys, keys + n * dim);
  g.surplus.assign(surplus, surplus + n * m);
  g.rebuild_index(n);
  return g;
}

void HostGrid::append(int64_t n, const uint32_t* k, const double* s) {
  if (n < 0 || (n > 0 && (!k || !s))) fail(DDSG_INVALID_ARGUMENT, "grid append: null arrays");
  validate_keys(dim, n, k);
  const int64_t base = size();
  keys.insert(keys.end(), k, k + n * dim);
  surplus.insert(surplus.end(), s, s + n * m);
  for (int64_t i = 0; i < n; ++i) {
    try {
      index_node(base + i);
    } catch (...) {
      // roll back so the grid stays consistent
      keys.resize(base * dim);
      surplus.resize(base * m);
      rebuild_index(base);
      throw;
    }
  }
  // The reference's build caps the level sum at max_level + dim - 1
  // (sparse_grid.hpp:89-107): a grid refined past that cap is the build of
  // the level that admits its deepest level sum, so max_level follows it.
  for (int64_t i = 0; i < n; ++i) {
    int ls = 0;
    for (int j = 0; j < dim; ++j) ls += level_of(k[i * dim + j]);
    max_level = std::max(max_level, ls - dim + 1);
  }
}

std::vector<double> HostGrid::quadrature() const {
  // sparse_grid.hpp:138-149: fixed (stored) node order, mul then add.
  std::vector<double> q(m, 0.0);
  const int64_t n = size();
  for (int64_t i = 0; i < n; ++i) {
    double w = 1.0;
    for (int j = 0; j < dim; ++j) {
      const uint32_t hk = keys[i * dim + j];
      w *= basis_weight_host(mode, level_of(hk), index_of(hk));
    }
    const double* s = &surplus[i * m];
    for (int c = 0; c < m; ++c) q[c] += w * s[c];
  }
  return q;
}

void HostGrid::interpolate_at_node(const uint32_t* key, int64_t upto, double* out) const {
  // Nonzero terms at a grid node x(key) come only from subspaces l <= level(key)
  // componentwise (deeper levels put x on a cell boundary, where every 1-d
  // factor vanishes).  Collect them, order by stored index, accumulate.
  std::vector<double> x(dim);
  std::vector<int> L(dim);
  for (int j = 0; j < dim; ++j) {
    x[j] = coordinate_of(key[j]);
    L[j] = level_of(key[j]);
  }
  struct Term {
    int64_t idx;
    double w;
  };
  std::vector<Term> terms;
  std::vector<int> l(dim, 1);
  std::vector<uint32_t> cand(dim);
  while (true) {
    double w = 1.0;
    bool zero = false;
    for (int j = 0; j < dim; ++j) {
      const int lj = l[j];
      const uint32_t ncell = 1u << (lj - 1);
      uint32_t k = static_cast<uint32_t>(std::ldexp(x[j], lj - 1));  // floor, x >= 0
      if (k >= ncell) k = ncell - 1;
      cand[j] = ncell + k;
    }
    const int64_t idx = find(cand.data());
    if (idx >= 0 && idx < upto) {
      for (int j = 0; j < dim; ++j) {
        w *= basis_value_host(mode, l[j], index_of(cand[j]), x[j]);
        if (w == 0.0) {
          zero = true;
          break;
        }
      }
      if (!zero && w != 0.0) terms.push_back({idx, w});
    }
    int j = 0;
    while (j < dim) {
      if (++l[j] <= L[j]) break;
      l[j] = 1;
      ++j;
    }
    if (j == dim) break;
  }
  std::sort(terms.begin(), terms.end(), [](const Term& a, const Term& b) { return a.idx < b.idx; });
  for (const Term& t : terms) {
    const double* s = &surplus[t.idx * m];
    for (int c = 0; c < m; ++c) out[c] += t.w * s[c];
  }
}

std::vector<std::vector<uint32_t>> HostGrid::next_candidates(int s, std::vector<char>& refined) {
  // sparse_grid.hpp:215-254.
  KeySet seen(dim);  // the candidates, flat in generation order (arena) and indexed
  std::vector<uint32_t> stack, p(dim), c(dim);  // ancestor walk, dim words per entry
  auto push_missing_ancestors = [&](const uint32_t* key) {
    stack.assign(key, key + dim);
    while (!stack.empty()) {
      const size_t top = stack.size() - dim;
      for (int j = 0; j < dim; ++j) {
        if (stack[top + j] <= 1u) continue;
        std::copy(stack.begin() + top, stack.begin() + top + dim, p.begin());
        p[j] >>= 1;
        if (contains(p.data()) || !seen.insert(p.data())) continue;
        stack.insert(stack.end(), p.begin(), p.end());  // walked after this entry's dims
      }
      // drop the entry just expanded (its pushed parents sit above it)
      stack.erase(stack.begin() + top, stack.begin() + top + dim);
    }
  };
  const int64_t n = size();
  for (int64_t i = 0; i < n; ++i) {
    const uint32_t* key = &keys[i * dim];
    if (level_sum_of(key, dim) != s) continue;
    bool significant = eps_gamma == 0.0;
    if (!significant) {
      double g = 0.0;
      const double* sp = &surplus[i * m];
      if (norm == DDSG_NORM_INF) {
        for (int cc = 0; cc < m; ++cc) g = std::max(g, std::abs(sp[cc]));
      } else {
        for (int cc = 0; cc < m; ++cc) g += sp[cc] * sp[cc];
        g = std::sqrt(g);
      }
      significant = g > eps_gamma;
    }
    if (!significant) continue;
    refined[i] = 1;
    for (int j = 0; j < dim; ++j) {
      for (uint32_t child : {key[j] * 2u, key[j] * 2u + 1u}) {
        std::copy(key, key + dim, c.begin());
        c[j] = child;
        if (contains(c.data()) || !seen.insert(c.data())) continue;
        push_missing_ancestors(c.data());
      }
    }
  }
  // batch order: (level sum, key lexicographic) -- a total order, so the
  // generation order above does not matter
  const int64_t nc = seen.n;
  const uint32_t* ar = seen.arena.data();
  std::vector<int> ls(nc);
  for (int64_t i = 0; i < nc; ++i) ls[i] = level_sum_of(ar + i * dim, dim);
  std::vector<int64_t> ord(nc);
  std::iota(ord.begin(), ord.end(), int64_t{0});
  std::sort(ord.begin(), ord.end(), [&](int64_t a, int64_t b) {
    if (ls[a] != ls[b]) return ls[a] < ls[b];
    return std::lexicographical_compare(ar + a * dim, ar + (a + 1) * dim, ar + b * dim, ar + (b + 1) * dim);
  });
  std::vector<std::vector<uint32_t>> out(nc);
  for (int64_t i = 0; i < nc; ++i) out[i].assign(ar + ord[i] * dim, ar + (ord[i] + 1) * dim);
  return out;
}

std::vector<std::vector<uint32_t>> HostGrid::refine_candidates(int s) const {
  std::vector<char> refined(size(), 0);
  return const_cast<HostGrid*>(this)->next_candidates(s, refined);
}

void HostGrid::insert_batch(const std::vector<std::vector<uint32_t>>& batch, const BatchEval& f) {
  // sparse_grid.hpp:256-298: evaluate the whole batch against the frozen grid,
  // reject non-finite values, then hierarchize one by one in batch order.
  const int64_t nb = static_cast<int64_t>(batch.size());
  std::vector<double> xs(nb * dim), vals(nb * m, 0.0);
  for (int64_t i = 0; i < nb; ++i)
    for (int j = 0; j < dim; ++j) xs[i * dim + j] = coordinate_of(batch[i][j]);
  f(xs.data(), nb, vals.data());
  for (int64_t i = 0; i < nb; ++i) {
    for (int c = 0; c < m; ++c) {
      if (!std::isfinite(vals[i * m + c])) {
        std::ostringstream os;
        os << "sparse grid: evaluator returned a non-finite value at grid point (";
        for (int j = 0; j < dim; ++j) os << (j ? ", " : "") << xs[i * dim + j];
        os << ")";
        throw BuildError(os.str(), std::vector<double>(xs.begin() + i * dim, xs.begin() + (i + 1) * dim));
      }
    }
  }
  std::vector<double> interp(m);
  for (int64_t i = 0; i < nb; ++i) {
    std::fill(interp.begin(), interp.end(), 0.0);
    interpolate_at_node(batch[i].data(), size(), interp.data());
    keys.insert(keys.end(), batch[i].begin(), batch[i].end());
    for (int c = 0; c < m; ++c) surplus.push_back(vals[i * m + c] - interp[c]);
    index_node(size() - 1);
  }
}

HostGrid HostGrid::build(int dim, int m, int mode, int max_level, double eps_gamma, int norm,
                         const BatchEval& f) {
  // sparse_grid.hpp:84-108.
  if (dim < 1) fail(DDSG_INVALID_ARGUMENT, "sparse grid: dim must be >= 1");
  if (m < 1) fail(DDSG_INVALID_ARGUMENT, "sparse grid: out_dim must be >= 1");
  if (max_level < 1) fail(DDSG_INVALID_ARGUMENT, "sparse grid: max_level must be >= 1");
  if (max_level > kMaxLevel) fail(DDSG_INVALID_ARGUMENT, "sparse grid: max_level must be <= 30");
  if (!(eps_gamma >= 0.0)) fail(DDSG_INVALID_ARGUMENT, "sparse grid: eps_gamma must be >= 0");
  if (mode != DDSG_ZERO_BOUNDARY && mode != DDSG_MODIFIED_LINEAR)
    fail(DDSG_INVALID_ARGUMENT, "sparse grid: unknown boundary mode");
  HostGrid g;
  g.dim = dim;
  g.m = m;
  g.mode = mode;
  g.max_level = max_level;
  g.eps_gamma = eps_gamma;
  g.norm = norm;
  const int max_sum = max_level + dim - 1;
  std::vector<std::vector<uint32_t>> batch{std::vector<uint32_t>(dim, 1u)};
  std::vector<char> refined;
  for (int s = dim; s <= max_sum && !batch.empty(); ++s) {
    g.insert_batch(batch, f);
    if (s == max_sum) break;
    refined.assign(g.size(), 0);
    batch = g.next_candidates(s, refined);
  }
  return g;
}

GridLayout HostGrid::compile() const {
  const int64_t n = size();
  // group nodes by level vector
  std::map<std::vector<uint8_t>, std::vector<int64_t>> groups;
  for (int64_t i = 0; i < n; ++i) {
    std::vector<uint8_t> l(dim);
    for (int j = 0; j < dim; ++j) l[j] = static_cast<uint8_t>(level_of(keys[i * dim + j]));
    groups[l].push_back(i);
  }
  GridLayout L;
  for (auto& [lv, nodes] : groups) {
    SubspaceInfo s;
    s.levels = lv;
    s.level_sum = 0;
    int cell_bits = 0;
    for (uint8_t v : lv) {
      s.level_sum += v;
      cell_bits += v - 1;
    }
    if (cell_bits > 40) fail(DDSG_INVALID_ARGUMENT, "sparse grid: subspace too deep for the dense layout");
    s.cells = int64_t{1} << cell_bits;
    s.n_nodes = static_cast<int64_t>(nodes.size());
    L.subspaces.push_back(std::move(s));
  }
  // canonical subspace order: (|l|_1, l lexicographic)
  std::vector<size_t> order(L.subspaces.size());
  std::iota(order.begin(), order.end(), 0);
  std::vector<std::vector<int64_t>*> node_lists;
  for (auto& kv : groups) node_lists.push_back(&kv.second);
  std::sort(order.begin(), order.end(), [&](size_t a, size_t b) {
    const auto& A = L.subspaces[a];
    const auto& B = L.subspaces[b];
    if (A.level_sum != B.level_sum) return A.level_sum < B.level_sum;
    return A.levels < B.levels;
  });
  int64_t total_cells = 0;
  for (size_t o : order) total_cells += L.subspaces[o].cells;
  if (total_cells > std::max<int64_t>(8 * n, n + (int64_t{1} << 22)) || total_cells > (int64_t{1} << 31) - 1)
    fail(DDSG_INVALID_ARGUMENT,
         "sparse grid: adaptive grid too sparse for the dense subspace layout (" +
             std::to_string(total_cells) + " cells for " + std::to_string(n) + " nodes)");
  std::vector<SubspaceInfo> sorted;
  sorted.reserve(order.size());
  L.slab.assign(total_cells, -1);
  L.row_to_stored.resize(n);
  int64_t slab_off = 0, row = 0;
  for (size_t o : order) {
    SubspaceInfo s = L.subspaces[o];
    s.slab_offset = slab_off;
    // cell linear index, dim 0 most significant
    std::vector<std::pair<int64_t, int64_t>> cells;  // (cell, stored index)
    for (int64_t i : *node_lists[o]) {
      int64_t lin = 0;
      for (int j = 0; j < dim; ++j) {
        const uint32_t hk = keys[i * dim + j];
        lin = (lin << (level_of(hk) - 1)) | cell_of(hk);
      }
      cells.emplace_back(lin, i);
    }
    std::sort(cells.begin(), cells.end());
    for (auto& [lin, i] : cells) {
      L.slab[slab_off + lin] = static_cast<int32_t>(row);
      L.row_to_stored[row] = static_cast<int32_t>(i);
      ++row;
    }
    slab_off += s.cells;
    sorted.push_back(std::move(s));
  }
  L.subspaces = std::move(sorted);
  L.rows = row;
  // Stored order = concatenation of maximal runs sorted by (level sum, key):
  // the reference's build appends batches sorted that way
  // (sparse_grid.hpp:248-253), closure ancestors making later batches start
  // below earlier ones.  At any point the nonzero nodes of one run come in
  // canonical subspace order, so evaluating run by run reproduces the stored
  // order exactly.
  std::vector<int16_t> run_of(n, 0);
  int run = 0;
  for (int64_t i = 1; i < n; ++i) {
    const uint32_t* a = &keys[(i - 1) * dim];
    const uint32_t* b = &keys[i * dim];
    const int sa = level_sum_of(a, dim), sb = level_sum_of(b, dim);
    const bool ascending = sa != sb ? sa < sb : std::lexicographical_compare(a, a + dim, b, b + dim);
    if (!ascending) ++run;
    if (run > 32767) fail(DDSG_INVALID_ARGUMENT, "sparse grid: stored order has more than 32767 runs");
    run_of[i] = static_cast<int16_t>(run);
  }
  L.runs = n > 0 ? run + 1 : 1;
  L.row_run.resize(L.rows);
  for (int64_t r = 0; r < L.rows; ++r) L.row_run[r] = run_of[L.row_to_stored[r]];
  return L;
}

}  // namespace ddsg_b200
