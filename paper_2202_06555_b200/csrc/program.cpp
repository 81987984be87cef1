#include "program.hpp"

#include <algorithm>

namespace ddsg_b200 {

static void sched_rec(int64_t n, std::vector<uint8_t>& merges, int64_t& leaf, int depth_now,
                      int* max_depth) {
  if (n == 1) {
    merges.push_back(0);
    ++leaf;
    return;
  }
  const int64_t half = n / 2;
  sched_rec(half, merges, leaf, depth_now, max_depth);
  sched_rec(n - half, merges, leaf, depth_now + 1, max_depth);
  ++merges.back();
}

std::vector<uint8_t> pairwise_schedule(int64_t n, int* max_depth) {
  std::vector<uint8_t> merges;
  if (n <= 0) {
    if (max_depth) *max_depth = 0;
    return merges;
  }
  merges.reserve(n);
  int64_t leaf = 0;
  sched_rec(n, merges, leaf, 1, max_depth);
  // simulate to get the exact stack high-water mark
  int sp = 0, hw = 0;
  for (uint8_t k : merges) {
    ++sp;
    hw = std::max(hw, sp);
    sp -= k;
  }
  if (max_depth) *max_depth = hw;
  return merges;
}

void HostProgram::add_empty_slot(int32_t id, double b) {
  slot_id.push_back(id);
  slot_k.push_back(0);
  slot_mode.push_back(0);
  slot_dims_off.push_back(static_cast<int32_t>(slot_dims.size()));
  slot_b.push_back(b);
  const int32_t s = static_cast<int32_t>(sub_lv_off.size());
  slot_sub_begin.push_back(s);
  slot_sub_end.push_back(s);
  slot_row_begin.push_back(rows);
  slot_row_end.push_back(rows);
  slot_runs.push_back(1);
}

void HostProgram::add_grid_slot(int32_t id, const HostGrid& g, const std::vector<int32_t>& dims,
                                double b) {
  const GridLayout L = g.compile();
  slot_id.push_back(id);
  slot_k.push_back(g.dim);
  slot_mode.push_back(g.mode);
  slot_dims_off.push_back(static_cast<int32_t>(slot_dims.size()));
  slot_dims.insert(slot_dims.end(), dims.begin(), dims.end());
  slot_b.push_back(b);
  slot_sub_begin.push_back(static_cast<int32_t>(sub_lv_off.size()));
  const int64_t slab_base = static_cast<int64_t>(slab.size());
  const int64_t row_base = rows;
  for (const SubspaceInfo& s : L.subspaces) {
    sub_lv_off.push_back(static_cast<int32_t>(levels.size()));
    levels.insert(levels.end(), s.levels.begin(), s.levels.end());
    sub_slab_off.push_back(slab_base + s.slab_offset);
    sub_nodes.push_back(static_cast<int32_t>(s.n_nodes));
  }
  slot_sub_end.push_back(static_cast<int32_t>(sub_lv_off.size()));
  slab.reserve(slab.size() + L.slab.size());
  for (int32_t r : L.slab) slab.push_back(r < 0 ? -1 : static_cast<int32_t>(row_base + r));
  surplus.reserve(surplus.size() + static_cast<size_t>(L.rows) * m);
  for (int64_t r = 0; r < L.rows; ++r) {
    const int32_t st = L.row_to_stored[r];
    surplus.insert(surplus.end(), g.surplus.begin() + static_cast<int64_t>(st) * m,
                   g.surplus.begin() + static_cast<int64_t>(st + 1) * m);
    row_stored.push_back(st);
    row_run.push_back(L.row_run[r]);
  }
  slot_runs.push_back(L.runs);
  slot_row_begin.push_back(rows);
  rows += L.rows;
  slot_row_end.push_back(rows);
  if (rows > (int64_t{1} << 31) - 1) fail(DDSG_INVALID_ARGUMENT, "program: more than 2^31 rows");
}

void HostProgram::finish() {
  const int64_t na = static_cast<int64_t>(slot_k.size());
  if (plain) {
    merges.assign(na, 0);
    depth = 1;
  } else {
    merges = pairwise_schedule(na, &depth);
  }
}

}  // namespace ddsg_b200
