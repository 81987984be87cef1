// Evaluation program: the flattened slot table of a (plain or HDMR)
// interpolant, compiled on the host and uploaded once.
//
// A plain grid is a program with one slot (all dims, b = 1) and no slot sum.
// An HDMR interpolant is the reference's VectorizedDdsg slot table
// (ddsg_eval.hpp:40-74) restricted to active slots (b != 0), in slot order,
// with the pairwise-sum tree (ddsg_eval.hpp:154-158) precompiled into a
// post-order merge schedule: after leaf a, `merges[a]` additions fold the
// top of the partial-sum stack.
#pragma once

#include <cstdint>
#include <vector>

#include "grid_host.hpp"

namespace ddsg_b200 {

struct HostProgram {
  int d = 0;      // point dimension
  int m = 0;      // outputs
  int plain = 0;  // 1: single grid, y = interpolate(x)
  int depth = 0;  // max partial-sum stack depth

  // active slots, in evaluation order
  std::vector<int32_t> slot_id;        // index in the caller's slot table
  std::vector<int32_t> slot_k;         // |u|; 0 = empty index (b * f_anchor)
  std::vector<int32_t> slot_mode;      // boundary mode of the slot's grid
  std::vector<int32_t> slot_dims_off;  // into slot_dims
  std::vector<int32_t> slot_dims;
  std::vector<double> slot_b;
  std::vector<int32_t> slot_sub_begin, slot_sub_end;  // subspace range
  std::vector<int64_t> slot_row_begin, slot_row_end;  // surplus row range
  std::vector<int32_t> slot_runs;                     // stored-order runs of the slot's grid
  std::vector<uint8_t> merges;

  // subspaces (all slots concatenated)
  std::vector<int32_t> sub_lv_off;  // into levels
  std::vector<uint8_t> levels;
  std::vector<int64_t> sub_slab_off;  // into slab
  std::vector<int32_t> sub_nodes;     // present nodes in the subspace
  std::vector<int32_t> slab;          // -> surplus row, or -1
  std::vector<double> surplus;        // [rows][m]
  std::vector<int32_t> row_stored;    // row -> stored node index within its grid
  std::vector<int16_t> row_run;       // row -> stored-order run
  std::vector<double> f_anchor;       // [m]
  int64_t rows = 0;

  void add_grid_slot(int32_t id, const HostGrid& g, const std::vector<int32_t>& dims, double b);
  void add_empty_slot(int32_t id, double b);
  void finish();  // builds the merge schedule
};

// Post-order merge schedule of pairwise_sum over n leaves
// (ddsg_eval.hpp:154-158): sched(1) = leaf; sched(n) = sched(n/2),
// sched(n - n/2), one add.  Returns per-leaf add counts and the max depth.
std::vector<uint8_t> pairwise_schedule(int64_t n, int* max_depth);

}  // namespace ddsg_b200
