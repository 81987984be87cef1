// Host-side sparse-grid object: node storage in the caller's order, the
// adaptive build, quadrature, and the compiler from nodes to the device
// subspace layout.
//
// Reference semantics: /root/reference/proj/include/ddsg/sparse_grid.hpp
// (build :84-108, next_candidates :215-254, insert_batch :256-277,
// interpolate_partial :302-315, quadrature :138-149, from_nodes :160-179).
#pragma once

#include <cmath>
#include <cstdint>
#include <functional>
#include <unordered_map>
#include <vector>

#include "common.hpp"

namespace ddsg_b200 {

// One subspace (level vector l) of a grid in the compiled layout.  Cells are
// row-major over dims (dim 0 most significant), cell k_j in [0, 2^(l_j-1)).
struct SubspaceInfo {
  std::vector<uint8_t> levels;  // l_j, j < dim
  int64_t cells = 0;            // prod 2^(l_j - 1)
  int64_t slab_offset = 0;      // into Layout::slab
  int64_t n_nodes = 0;          // present nodes
  int level_sum = 0;
};

// Compiled, evaluation-ready layout of one grid.  Rows of `surplus_rows` are
// ordered subspace by subspace in canonical subspace order (|l|_1, l lex) and
// cell order within a subspace, so a point's nonzero terms are visited in
// exactly the order the reference's canonical node order produces
// (SURVEY.md §A.3).
struct GridLayout {
  std::vector<SubspaceInfo> subspaces;
  std::vector<int32_t> slab;          // [total cells] -> layout row or -1
  std::vector<int32_t> row_to_stored; // layout row -> stored node index
  std::vector<int16_t> row_run;       // layout row -> run of its stored position
  int runs = 1;                       // maximal canonically sorted runs of the stored order
  int64_t rows = 0;
};

class HostGrid {
 public:
  int dim = 0;
  int m = 0;
  int mode = DDSG_ZERO_BOUNDARY;
  int max_level = 1;
  double eps_gamma = 0.0;
  int norm = DDSG_NORM_INF;
  std::vector<uint32_t> keys;   // [N][dim], stored (insertion) order
  std::vector<double> surplus;  // [N][m]

  int64_t size() const { return dim ? static_cast<int64_t>(keys.size() / dim) : 0; }

  // from_nodes (sparse_grid.hpp:160-179): validates and indexes.
  static HostGrid from_nodes(int dim, int m, int mode, int max_level, double eps_gamma,
                             int64_t n, const uint32_t* keys, const double* surplus);

  using BatchEval = std::function<void(const double* xs, int64_t count, double* out)>;
  // build (sparse_grid.hpp:84-108).
  static HostGrid build(int dim, int m, int mode, int max_level, double eps_gamma, int norm,
                        const BatchEval& f);

  void append(int64_t n, const uint32_t* keys, const double* surplus);
  // Refinement candidates from level sum s: children of significant nodes,
  // closed under missing ancestors, sorted by (level sum, key)
  // (sparse_grid.hpp:215-254).  Does not modify the grid.
  std::vector<std::vector<uint32_t>> refine_candidates(int s) const;
  std::vector<double> quadrature() const;
  bool contains(const uint32_t* key) const;
  int64_t find(const uint32_t* key) const;

  GridLayout compile() const;

  // Host residual interpolation at a grid node coordinate, summing nodes
  // [0, upto) in stored order (sparse_grid.hpp:302-315).  Only subspaces
  // l <= level(node) can be nonzero at a node, so this walks Π l_j candidates.
  void interpolate_at_node(const uint32_t* key, int64_t upto, double* out) const;

 private:
  // Node index: open-addressing table of node ids over the flat `keys`
  // array (FNV-1a over the dim words, as NodeKeyHash, grid_index.hpp:60-69);
  // no allocation per lookup.
  std::vector<int64_t> table_;  // -1 = empty; size a power of two, load <= 1/2
  int64_t indexed_ = 0;
  void index_node(int64_t i);
  void rebuild_index(int64_t n_nodes);
  std::vector<std::vector<uint32_t>> next_candidates(int s, std::vector<char>& refined);
  void insert_batch(const std::vector<std::vector<uint32_t>>& batch, const BatchEval& f);
};

// 1-d basis value (basis.hpp:36-54) with inv_h = 2^l, center = i / inv_h.
double basis_value_host(int mode, int level, uint32_t index, double x);

}  // namespace ddsg_b200
