// Slot-staged HDMR evaluation kernel (see fast_hdmr.cuh for the design).
//
// Reference semantics reproduced bit for bit in EXACT mode:
//   VectorizedDdsg::evaluate (ddsg_eval.hpp:83-113): per active slot in slot
//   order, row = interpolate(grid, x|u) (sparse_grid.hpp:111-128, nodes in
//   canonical order, w = dim-ordered product with early exit, out += w*s as
//   mul then add), row *= b; out[c] = pairwise_sum over rows
//   (ddsg_eval.hpp:154-158).
#include <cuda_runtime.h>

#include <algorithm>
#include <cstdlib>
#include <cmath>
#include <cstring>
#include <map>

#include "basis.cuh"
#include "fast_hdmr.cuh"

#include "fast_hdmr_device.cuh"

namespace ddsg_b200 {
namespace fast {

// x [n][d] row-major -> xt [d][n]; flags the lowest point outside [0,1]^d.
__global__ void transpose_check_kernel(const double* __restrict__ x, int64_t n, int d, int64_t base,
                                       double* __restrict__ xt, unsigned long long* bad) {
  __shared__ double tile[32][33];
  const int64_t p0 = static_cast<int64_t>(blockIdx.x) * 32;
  const int j0 = blockIdx.y * 32;
  const int tx = threadIdx.x, ty = threadIdx.y;  // 32 x 8
  for (int r = ty; r < 32; r += 8) {
    const int64_t p = p0 + r;
    const int j = j0 + tx;
    double v = 0.5;
    if (p < n && j < d) {
      v = __ldcs(x + p * d + j);  // read once
      if (!(v >= 0.0 && v <= 1.0)) atomicMin(bad, static_cast<unsigned long long>(base + p));
    }
    tile[r][tx] = v;
  }
  __syncthreads();
  for (int r = ty; r < 32; r += 8) {
    const int j = j0 + r;
    const int64_t p = p0 + tx;
    if (p < n && j < d) xt[static_cast<int64_t>(j) * n + p] = tile[tx][r];
  }
}

}  // namespace fast

using namespace fast;

// The kernel instance of this program: arithmetic mode x multi-run carry x order-3 slots.
LaunchFn FastHdmr::instance_launch(int exact) const {
  static const LaunchFn tab[8] = {fast_launch_000, fast_launch_001, fast_launch_010, fast_launch_011,
                                  fast_launch_100, fast_launch_101, fast_launch_110, fast_launch_111};
  return tab[(exact ? 4 : 0) + (has_carry_ ? 2 : 0) + (has_order3_ ? 1 : 0)];
}
AttrFn FastHdmr::instance_attr(int exact) const {
  static const AttrFn tab[8] = {fast_attr_000, fast_attr_001, fast_attr_010, fast_attr_011,
                                fast_attr_100, fast_attr_101, fast_attr_110, fast_attr_111};
  return tab[(exact ? 4 : 0) + (has_carry_ ? 2 : 0) + (has_order3_ ? 1 : 0)];
}

FastHdmr::~FastHdmr() {
  if (blocks_) cudaFree(blocks_);
  if (block_off_) cudaFree(block_off_);
  if (block_len_) cudaFree(block_len_);
  if (slot_dims_) cudaFree(slot_dims_);
  for (auto& level : split_)
    for (SubTree& t : level) {
      if (t.off) cudaFree(t.off);
      if (t.len) cudaFree(t.len);
    }
}

// Position of subspace l in the canonical (|l|_1, l lex) order of a k-d grid.
static int canon_index(int k, int l1, int l2, int l3 = 0) {
  if (k == 1) return l1 - 1;
  if (k == 2) {
    const int s = l1 + l2;
    return (s - 2) * (s - 1) / 2 + (l1 - 1);
  }
  int idx = 0;  // order 3: subspaces of lower level sum, then lex within the sum
  const int s = l1 + l2 + l3;
  for (int t = 3; t < s; ++t) idx += (t - 1) * (t - 2) / 2;
  for (int a = 1; a < l1; ++a) idx += s - a - 1;  // (a, b, c) with b + c = s - a, b, c >= 1
  return idx + (l2 - 1);
}

bool FastHdmr::build(const HostProgram& hp) {
  usable_ = false;
  if (const char* e = std::getenv("DDSG_SLOT_KERNEL"); e && std::atoi(e) == 0) {  // A/B switch
    why_ = "disabled by DDSG_SLOT_KERNEL=0";
    return false;
  }
  if (hp.plain) {
    why_ = "plain grid";
    return false;
  }
  const int na = static_cast<int>(hp.slot_k.size());
  if (na == 0) {
    why_ = "no active slot";
    return false;
  }
  int levels = 0;
  while ((int64_t{1} << levels) < na) ++levels;
  if (levels > kMaxLevels) {
    why_ = "too many active slots";
    return false;
  }
  d_ = hp.d;
  m_ = hp.m;
  n_active_ = na;
  has_order3_ = 0;
  levels_ = levels;
  n_cb_ = (hp.m + kCols - 1) / kCols;

  // perfect-tree embedding of pairwise_sum (ddsg_eval.hpp:154-158)
  std::vector<int32_t> tree_t, tree_s;
  {
    struct Rec {
      static void go(int64_t lo, int64_t cnt, int depth, int D, std::vector<int32_t>& t,
                     std::vector<int32_t>& s) {
        if (cnt == 1) {
          t.push_back(static_cast<int32_t>(lo));
          s.push_back(D - depth);
          return;
        }
        const int64_t h = cnt / 2;
        go(lo, h, depth + 1, D, t, s);
        go(lo + (int64_t{1} << (D - depth - 1)), cnt - h, depth + 1, D, t, s);
      }
    };
    Rec::go(0, na, 0, levels, tree_t, tree_s);
  }

  // Staged blocks (column-block independent part): one per active slot, or
  // one per stored-order run of a slot whose grid is stored in several
  // canonically sorted runs.  The blocks of a multi-run slot
  // hold disjoint row sets; the kernel accumulates them in run order
  // (b_kind flags kBCont / kBMore), exactly the reference's stored order.
  struct SlotPlan {
    SlotHeader h;
    std::vector<int64_t> rows;  // program rows staged in this block, in order
    std::vector<int16_t> slab;
    int64_t bytes = 0;
    int slot = 0;
    int stride = kStride;  // doubles per staged row (kRotStride for the rotated layout)
  };
  const bool rot_enabled = [] {
    const char* e = std::getenv("DDSG_SLOT_ROT");
    return !(e && std::atoi(e) == 0);
  }();
  const int rot_min_level = [] {  // shallowest max level that takes the rotated layout
    const char* e = std::getenv("DDSG_SLOT_ROT_MIN");
    return e ? std::max(2, std::atoi(e)) : 6;
  }();
  std::vector<SlotPlan> plans;
  std::vector<int16_t> dims16;
  int64_t max_bytes = 0;
  for (int a = 0; a < na; ++a) {
    const int k = hp.slot_k[a];
    if (k > 3) {
      why_ = "slot order > 3";
      return false;
    }
    const int runs = k == 0 ? 1 : hp.slot_runs[a];
    const int64_t row_begin = k == 0 ? 0 : hp.slot_row_begin[a];
    const int64_t row_count = k == 0 ? 0 : hp.slot_row_end[a] - row_begin;
    std::vector<int32_t> local(static_cast<size_t>(row_count), -1);
    for (int r = 0; r < runs; ++r) {
      plans.emplace_back();
      SlotPlan& P = plans.back();
      P.slot = a;
      std::memset(&P.h, 0, sizeof(SlotHeader));
      SlotHeader& H = P.h;
      H.k = k;
      H.mode = hp.slot_mode[a];
      H.tree_t = tree_t[a];
      H.tree_s = tree_s[a];
      H.table_off = kTableOff;
      const int flags = (r > 0 ? kBCont : 0) | (r + 1 < runs ? kBMore : 0);
      dims16.push_back(0);
      dims16.push_back(0);
      dims16.push_back(-1);
      const size_t di = dims16.size() - kSlotDims;
      if (k == 0) {
        H.b_kind = 1;  // b * f_anchor is folded into the staged row
        P.rows.push_back(-1);
      } else {
        const double b = hp.slot_b[a];
        H.b = b;
        H.b_kind = (b == 1.0 ? 1 : (b == -1.0 ? 2 : 0)) | flags;
        H.d0 = hp.slot_dims[hp.slot_dims_off[a]];
        H.d1 = k >= 2 ? hp.slot_dims[hp.slot_dims_off[a] + 1] : 0;
        H.d2 = k == 3 ? hp.slot_dims[hp.slot_dims_off[a] + 2] : 0;
        if (H.d0 > 32767 || H.d1 > 32767 || H.d2 > 32767) {
          why_ = "point dimension above 32767";
          return false;
        }
        dims16[di] = static_cast<int16_t>(H.d0);
        dims16[di + 1] = static_cast<int16_t>(k >= 2 ? H.d1 : 0);  // unused second dim reads dim 0
        dims16[di + 2] = static_cast<int16_t>(k == 3 ? H.d2 : -1);  // -1: not an order-3 block
        has_order3_ = has_order3_ || k == 3;
        std::fill(local.begin(), local.end(), -1);
        for (int64_t q = 0; q < row_count; ++q)
          if (runs == 1 || hp.row_run[row_begin + q] == r) {
            local[q] = static_cast<int32_t>(P.rows.size());
            P.rows.push_back(row_begin + q);
          }
        if (P.rows.size() > 32766) {
          why_ = "slot has more than 32766 nodes";
          return false;
        }
        int nlev = 0;
        for (int sb = hp.slot_sub_begin[a]; sb < hp.slot_sub_end[a]; ++sb) {
          const uint8_t* lv = &hp.levels[hp.sub_lv_off[sb]];
          const int l1 = lv[0], l2 = k >= 2 ? lv[1] : 0, l3 = k == 3 ? lv[2] : 0;
          // the order-k leaf walks every subspace with level sum <= nlev + k - 1
          const int reach = k == 1 ? l1 : (k == 2 ? l1 + l2 - 1 : l1 + l2 + l3 - 2);
          if ((k == 1 && l1 > kL1) || (k == 2 && reach > kL2) || (k == 3 && reach > kL3)) {
            why_ = "slot level above the kernel's static maximum";
            return false;
          }
          const int idx = canon_index(k, l1, l2, l3);
          const int64_t cells = int64_t{1} << (l1 - 1 + (k >= 2 ? l2 - 1 : 0) + (k == 3 ? l3 - 1 : 0));
          const int32_t* slab = &hp.slab[hp.sub_slab_off[sb]];
          int64_t n_in = 0;
          for (int64_t c = 0; c < cells; ++c) n_in += slab[c] >= 0 && local[slab[c] - row_begin] >= 0;
          if (n_in == 0) continue;  // no node of this run in the subspace
          nlev = std::max(nlev, reach);
          H.present |= 1u << idx;
          if (n_in == cells) {  // complete: its rows are consecutive in canonical order
            H.full |= 1u << idx;
            H.sub_base[idx] = static_cast<int16_t>(local[slab[0] - row_begin]);
          } else {
            if (P.slab.size() + cells > 32767) {
              why_ = "slab too large";
              return false;
            }
            H.sub_base[idx] = static_cast<int16_t>(P.slab.size());
            for (int64_t c = 0; c < cells; ++c)
              P.slab.push_back(slab[c] < 0 ? int16_t{-1} : static_cast<int16_t>(local[slab[c] - row_begin]));
          }
        }
        H.nlev = std::max(nlev, 1);
        {
          // fast_full: the block is the full grid of its max level (every
          // canonical subspace present and complete) with finite surpluses
          const int nsub = k == 1 ? nlev : (k == 2 ? nlev * (nlev + 1) / 2 : nlev * (nlev + 1) * (nlev + 2) / 6);
          const uint32_t all = nsub >= 32 ? 0xffffffffu : ((1u << nsub) - 1u);
          bool finite = true;
          for (size_t q = 0; q < P.rows.size() && finite; ++q)
            for (int c = 0; c < m_; ++c)
              if (!std::isfinite(hp.surplus[P.rows[q] * m_ + c])) {
                finite = false;
                break;
              }
          H.fast_full = (nlev > 0 && H.present == all && H.full == all && finite) ? 1 : 0;
          // An adaptive (partial) block with finite surpluses is padded to the
          // full grid of its level with zero rows: the general path already
          // adds w * 0 for every absent canonical node (term_row's zero row),
          // so the padded block adds the same terms in the same order, but
          // through the static-row path (no slab lookups, loads one term ahead).
          const int64_t full_rows = k == 1 ? base1(nlev + 1) : (k == 2 ? base2(1, nlev + 1) : base3(1, 1, nlev + 1));
          if (!H.fast_full && finite && nlev > 0 && (full_rows + 1) * kStride * 8 <= kMaxPaddedBytes) {
            std::vector<int64_t> padded(static_cast<size_t>(full_rows), -1);
            for (int sb = hp.slot_sub_begin[a]; sb < hp.slot_sub_end[a]; ++sb) {
              const uint8_t* lv = &hp.levels[hp.sub_lv_off[sb]];
              const int l1 = lv[0], l2 = k >= 2 ? lv[1] : 0, l3 = k == 3 ? lv[2] : 0;
              const int64_t base = k == 1 ? base1(l1) : (k == 2 ? base2(l1, l2) : base3(l1, l2, l3));
              const int64_t cells = int64_t{1} << (l1 - 1 + (k >= 2 ? l2 - 1 : 0) + (k == 3 ? l3 - 1 : 0));
              const int32_t* slab = &hp.slab[hp.sub_slab_off[sb]];
              for (int64_t c = 0; c < cells; ++c)
                if (slab[c] >= 0 && local[slab[c] - row_begin] >= 0) padded[base + c] = slab[c];
            }
            P.rows.assign(padded.begin(), padded.end());
            P.slab.clear();
            H.present = all;
            H.full = all;
            H.fast_full = 1;
          }
          // full single-run blocks whose deepest level has >= 32 candidate
          // rows (1-d max level >= 6, 2-d max level 6: level sum 7) use the
          // rotated layout (conflict-free deep levels, see leaf_full1_rot /
          // leaf_full2_rot).  Shallower blocks keep stride 9, conflict-free
          // up to 16 rows and a 1-wavefront broadcast for level 1, which the
          // rotation would turn into 2.  DDSG_SLOT_ROT=0 disables it.
          if (H.fast_full == 1 && k <= 2 && nlev >= rot_min_level && runs == 1 && rot_enabled &&
              static_cast<int64_t>(P.rows.size() + 1) * kRotStride * 8 <= kMaxRotBytes)
            H.fast_full = 2;
        }
        H.zero_row = static_cast<int32_t>(P.rows.size());  // all-zero row appended to the table
        P.rows.push_back(-1);
      }
      P.stride = H.fast_full == 2 ? kRotStride : kStride;
      if (H.tree_t >= (1 << 13) || H.tree_s > 15 || H.nlev > 15) {
        why_ = "slot tree position beyond the packed header";
        return false;
      }
      H.pack_core();
      const int64_t table_bytes = static_cast<int64_t>(P.rows.size()) * P.stride * 8;
      H.slab_off = static_cast<int32_t>(kTableOff + table_bytes);
      P.bytes = (kTableOff + table_bytes + P.slab.size() * 2 + 15) / 16 * 16;
      max_bytes = std::max(max_bytes, P.bytes);
    }
  }
  const int nb = static_cast<int>(plans.size());
  n_blocks_ = nb;
  block_bytes_ = (max_bytes + 127) / 128 * 128;
  {
    int64_t per_cb = 0;
    for (const SlotPlan& P : plans) per_cb += P.bytes;
    int64_t budget = int64_t{64} << 20;  // staged tables kept L2-resident per CTA wave
    if (const char* e = std::getenv("DDSG_CB_BUDGET_MB")) budget = std::max<int64_t>(1, std::atoll(e)) << 20;
    cb_group_ = static_cast<int>(std::max<int64_t>(1, std::min<int64_t>(n_cb_, budget / std::max<int64_t>(per_cb, 1))));
  }
  const int64_t deep_bytes = std::min(std::max(0, levels - kTmemLevels), kSmemLevels) * int64_t{kCols} * kPoints * 8;
  has_carry_ = nb > na ? 1 : 0;
  const int64_t fixed = kHeaderBytes + deep_bytes + has_carry_ * int64_t{kCols} * kPoints * 8 + (2 * kSlotDims * int64_t{nb} + 15) / 16 * 16;
  n_stages_ = static_cast<int>(std::min<int64_t>(kMaxStages, (227 * 1024 - fixed) / block_bytes_));
  const int64_t smem = fixed + int64_t{n_stages_} * block_bytes_;
  if (n_stages_ < 2 || smem > 227 * 1024) {
    why_ = "shared-memory footprint too large";
    return false;
  }

  // column-blocked staged blocks
  std::vector<int64_t> off(static_cast<size_t>(n_cb_) * nb);
  std::vector<int32_t> len(static_cast<size_t>(n_cb_) * nb);
  int64_t total = 0;
  for (int cb = 0; cb < n_cb_; ++cb)
    for (int a = 0; a < nb; ++a) {
      off[static_cast<size_t>(cb) * nb + a] = total;
      len[static_cast<size_t>(cb) * nb + a] = static_cast<int32_t>(plans[a].bytes);
      total += plans[a].bytes;
    }
  std::vector<unsigned char> host(total, 0);
  for (int cb = 0; cb < n_cb_; ++cb)
    for (int a = 0; a < nb; ++a) {
      const SlotPlan& P = plans[a];
      unsigned char* blk = host.data() + off[static_cast<size_t>(cb) * nb + a];
      std::memcpy(blk, &P.h, sizeof(SlotHeader));
      double* table = reinterpret_cast<double*>(blk + kTableOff);
      const bool empty_slot = hp.slot_k[P.slot] == 0;
      for (size_t r = 0; r < P.rows.size(); ++r)
        for (int c = 0; c < kCols; ++c) {
          const int col = cb * kCols + c;
          double v = 0.0;
          if (col < m_) {
            if (empty_slot)
              v = hp.slot_b[P.slot] * hp.f_anchor[col];  // row = b * f_anchor (ddsg_eval.hpp:94-96)
            else if (P.rows[r] >= 0)
              v = hp.surplus[P.rows[r] * m_ + col];  // (the zero row stays 0)
          }
          table[r * P.stride + c] = v;
          if (P.stride == kRotStride && kRotCopies == 2) table[r * P.stride + kCols + c] = v;  // second copy
        }
      if (!P.slab.empty())
        std::memcpy(blk + P.h.slab_off, P.slab.data(), P.slab.size() * 2);
    }
  DDSG_CUDA(cudaMalloc(&blocks_, total));
  DDSG_CUDA(cudaMemcpy(blocks_, host.data(), total, cudaMemcpyHostToDevice));
  DDSG_CUDA(cudaMalloc(&block_off_, off.size() * sizeof(int64_t)));
  DDSG_CUDA(cudaMemcpy(block_off_, off.data(), off.size() * sizeof(int64_t), cudaMemcpyHostToDevice));
  DDSG_CUDA(cudaMalloc(&slot_dims_, dims16.size() * sizeof(int16_t)));
  DDSG_CUDA(cudaMemcpy(slot_dims_, dims16.data(), dims16.size() * sizeof(int16_t), cudaMemcpyHostToDevice));
  DDSG_CUDA(cudaMalloc(&block_len_, len.size() * sizeof(int32_t)));
  DDSG_CUDA(cudaMemcpy(block_len_, len.data(), len.size() * sizeof(int32_t), cudaMemcpyHostToDevice));
  for (int e = 0; e < 2; ++e) DDSG_CUDA(instance_attr(e)(static_cast<int>(smem)));

  // subtree block ranges for split launches (see fast_hdmr.cuh)
  max_split_ = 0;
  for (auto& level : split_) {
    for (SubTree& t : level) {
      if (t.off) cudaFree(t.off);
      if (t.len) cudaFree(t.len);
    }
    level.clear();
  }
  for (int S = 1; S <= kMaxSplit && S < levels; ++S) {
    bool ok = true;
    for (int a = 0; a < na && ok; ++a) ok = tree_s[a] <= levels - S;  // every leaf at depth >= S
    if (!ok) break;
    std::vector<SubTree> subs(size_t{1} << S);
    for (int blk = 0; blk < nb; ++blk) {
      SubTree& t = subs[static_cast<size_t>(tree_t[plans[blk].slot] >> (levels - S))];
      if (t.count == 0) t.first = blk;
      ok = ok && t.first + t.count == blk;  // contiguous block range
      ++t.count;
    }
    for (const SubTree& t : subs) ok = ok && t.count > 0;
    if (!ok) break;
    for (SubTree& t : subs) {
      std::vector<int64_t> so(static_cast<size_t>(n_cb_) * t.count);
      std::vector<int32_t> sl(so.size());
      for (int cb = 0; cb < n_cb_; ++cb)
        for (int i = 0; i < t.count; ++i) {
          so[static_cast<size_t>(cb) * t.count + i] = off[static_cast<size_t>(cb) * nb + t.first + i];
          sl[static_cast<size_t>(cb) * t.count + i] = len[static_cast<size_t>(cb) * nb + t.first + i];
        }
      DDSG_CUDA(cudaMalloc(&t.off, so.size() * sizeof(int64_t)));
      DDSG_CUDA(cudaMemcpy(t.off, so.data(), so.size() * sizeof(int64_t), cudaMemcpyHostToDevice));
      DDSG_CUDA(cudaMalloc(&t.len, sl.size() * sizeof(int32_t)));
      DDSG_CUDA(cudaMemcpy(t.len, sl.data(), sl.size() * sizeof(int32_t), cudaMemcpyHostToDevice));
    }
    split_[S] = std::move(subs);
    max_split_ = S;
  }
  usable_ = true;
  why_.clear();
  return true;
}

// Depth at which a launch over n points is split: the deepest S with
// tiles x column blocks x 2^S CTAs still within one wave of the SMs
// (DDSG_SLOT_SPLIT=0 disables; A/B switch).
int FastHdmr::split_levels(int64_t n) const {
  static const bool enabled = [] {
    const char* e = std::getenv("DDSG_SLOT_SPLIT");
    return !(e && std::atoi(e) == 0);
  }();
  if (!enabled || max_split_ == 0 || n <= 0) return 0;
  static thread_local int sms[64] = {0};
  int dev = 0;
  if (cudaGetDevice(&dev) != cudaSuccess || dev < 0 || dev >= 64) return 0;
  if (sms[dev] == 0 && cudaDeviceGetAttribute(&sms[dev], cudaDevAttrMultiProcessorCount, dev) != cudaSuccess) return 0;
  const int64_t ctas = (n + kPoints - 1) / kPoints * n_cb_;
  if (ctas > 16 * static_cast<int64_t>(sms[dev])) return 0;  // many waves: the tail is already small
  // cheapest depth: waves of CTAs (one CTA per SM) x ~2 us per slot a CTA
  // walks, plus ~5 us per sub-launch (fork, launch, join)
  // (profiles/r2_split_latency.jsonl).  Shorter CTAs also fill the last wave:
  // 4,096 points x 19 column blocks are 152 CTAs, two waves unsplit.
  int best = 0;
  double best_us = 0.0;
  for (int S = 0; S <= max_split_; ++S) {
    if (S > 0 && (static_cast<size_t>(n) * m_ * 8) << S > (size_t{256} << 20)) break;  // partial sums <= 256 MiB
    const int64_t waves = ((ctas << S) + sms[dev] - 1) / sms[dev];
    // (+ the subtree roots written and read back: 16 B per output and subtree at ~3 TB/s)
    const double us = static_cast<double>(waves) * kSlotUs * ((n_blocks_ + (1 << S) - 1) >> S) +
                      (S > 0 ? kSubLaunchUs * (1 << S) + 16.0 * n * m_ * (1 << S) / 3.0e6 : 0.0);
    if (S == 0 || us < best_us) {
      best_us = us;
      best = S;
    }
  }
  return best;
}

// Rough device time of a launch over n points that takes the split path (0
// when it would not): lets the caller choose between this and the
// small-batch path.
double FastHdmr::split_cost_us(int64_t n) const {
  const int S = split_levels(n);
  if (S == 0) return 0.0;
  int dev = 0, sm = 148;
  if (cudaGetDevice(&dev) == cudaSuccess) cudaDeviceGetAttribute(&sm, cudaDevAttrMultiProcessorCount, dev);
  const int64_t ctas = (n + kPoints - 1) / kPoints * n_cb_;
  const int64_t waves = ((ctas << S) + sm - 1) / sm;
  return 40.0 + kSubLaunchUs * (1 << S) + static_cast<double>(waves) * kSlotUs * ((n_blocks_ + (1 << S) - 1) >> S);
}

size_t FastHdmr::scratch_bytes(int64_t n, bool allow_split) const {
  const size_t xt = static_cast<size_t>(n) * d_ * 8;
  const int S = allow_split ? split_levels(n) : 0;
  return S == 0 ? xt : (xt + 255) / 256 * 256 + (size_t{1} << S) * static_cast<size_t>(n) * m_ * 8;
}

namespace {
// Streams and events of a split launch, per host thread and device.
struct SplitStreams {
  cudaStream_t s[1 << FastHdmr::kMaxSplitPublic] = {};
  cudaEvent_t fork = nullptr, join[1 << FastHdmr::kMaxSplitPublic] = {};
  bool ready = false;
  void init() {
    if (ready) return;
    DDSG_CUDA(cudaEventCreateWithFlags(&fork, cudaEventDisableTiming));
    for (auto& st : s) DDSG_CUDA(cudaStreamCreateWithFlags(&st, cudaStreamNonBlocking));
    for (auto& e : join) DDSG_CUDA(cudaEventCreateWithFlags(&e, cudaEventDisableTiming));
    ready = true;
  }
};
SplitStreams& split_streams() {
  static thread_local SplitStreams per_dev[64];
  int dev = 0;
  DDSG_CUDA(cudaGetDevice(&dev));
  if (dev < 0 || dev >= 64) fail(DDSG_CUDA_ERROR, "device ordinal out of range");
  per_dev[dev].init();
  return per_dev[dev];
}

// y[p][c] = the pairwise sum of the 2^S subtree roots part[k][p][c], k in tree order.
template <int kExactUnused>
__global__ void split_combine_kernel(const double* __restrict__ part, int64_t outs, int S, double* __restrict__ y) {
  const int64_t i = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
  if (i >= outs) return;
  double v[1 << FastHdmr::kMaxSplitPublic];
  const int K = 1 << S;
#pragma unroll
  for (int k = 0; k < (1 << FastHdmr::kMaxSplitPublic); ++k) v[k] = k < K ? part[static_cast<int64_t>(k) * outs + i] : 0.0;
#pragma unroll
  for (int w = 1; w < (1 << FastHdmr::kMaxSplitPublic); w <<= 1)
    if (w < K) {
#pragma unroll
      for (int k = 0; k < (1 << FastHdmr::kMaxSplitPublic); k += 2 * w) v[k] = __dadd_rn(v[k], v[k + w]);
    }
  y[i] = v[0];
}
}  // namespace

int64_t FastHdmr::launch(int exact, const double* x, int64_t n, int64_t base, double* y,
                         unsigned long long* bad, double* xt, cudaStream_t st, bool allow_split) const {
  // dim-major copy of the points so each slot's coordinate read is coalesced
  dim3 tgrid(static_cast<unsigned>((n + 31) / 32), static_cast<unsigned>((d_ + 31) / 32));
  transpose_check_kernel<<<tgrid, dim3(32, 8), 0, st>>>(x, n, d_, base, xt, bad);
  DDSG_CUDA(cudaGetLastError());
  if (const int S = allow_split ? split_levels(n) : 0; S > 0) {
    // a few tiles only: the subtrees of depth S as concurrent launches
    const int K = 1 << S;
    const int64_t tiles_s = (n + kPoints - 1) / kPoints;
    double* part = reinterpret_cast<double*>(reinterpret_cast<unsigned char*>(xt) +
                                             (static_cast<size_t>(n) * d_ * 8 + 255) / 256 * 256);
    const int lv = levels_ - S;
    const int64_t deep_b = std::min(std::max(0, levels_ - kTmemLevels), kSmemLevels) * int64_t{kCols} * kPoints * 8;
    const size_t smem_s = kHeaderBytes + n_stages_ * block_bytes_ + deep_b + has_carry_ * size_t{kCols} * kPoints * 8 +
                          (2 * kSlotDims * static_cast<size_t>(n_blocks_) + 15) / 16 * 16;
    SplitStreams& ss = split_streams();
    kernel_timer().begin(st);
    DDSG_CUDA(cudaEventRecord(ss.fork, st));
    DDSG_CUDA(instance_attr(exact)(static_cast<int>(smem_s)));
    for (int k = 0; k < K; ++k) {
      const SubTree& t = split_[S][static_cast<size_t>(k)];
      DDSG_CUDA(cudaStreamWaitEvent(ss.s[k], ss.fork, 0));
      const KernelArgs args{static_cast<const unsigned char*>(blocks_), t.off, t.len, slot_dims_ + kSlotDims * t.first,
                            t.count, n_cb_, n_cb_, lv, xt, n, m_, part + static_cast<int64_t>(k) * n * m_,
                            block_bytes_, n_stages_};
      instance_launch(exact)(dim3(static_cast<unsigned>(tiles_s * n_cb_)), smem_s, ss.s[k], args);
      DDSG_CUDA(cudaEventRecord(ss.join[k], ss.s[k]));
      DDSG_CUDA(cudaStreamWaitEvent(st, ss.join[k], 0));
    }
    const int64_t outs = n * m_;
    split_combine_kernel<0><<<static_cast<unsigned>((outs + 255) / 256), 256, 0, st>>>(part, outs, S, y);
    kernel_timer().end(st);
    DDSG_CUDA(cudaGetLastError());
    return 2 + K;
  }
  const int64_t tiles = (n + kPoints - 1) / kPoints;
  const int64_t deep_bytes = std::min(std::max(0, levels_ - kTmemLevels), kSmemLevels) * int64_t{kCols} * kPoints * 8;
  const size_t smem = kHeaderBytes + n_stages_ * block_bytes_ + deep_bytes + has_carry_ * size_t{kCols} * kPoints * 8 +
                      (2 * kSlotDims * static_cast<size_t>(n_blocks_) + 15) / 16 * 16;
  const dim3 grid(static_cast<unsigned>(tiles * n_cb_));
  kernel_timer().begin(st);
  const KernelArgs args{static_cast<const unsigned char*>(blocks_), block_off_, block_len_, slot_dims_, n_blocks_,
                        n_cb_, cb_group_, levels_, xt, n, m_, y, block_bytes_, n_stages_};
  // The dynamic shared-memory limit is a property of the kernel function,
  // shared by every program: set this program's own size before launching
  // (a program built later with smaller stages would otherwise have lowered it).
  DDSG_CUDA(instance_attr(exact)(static_cast<int>(smem)));
  instance_launch(exact)(grid, smem, st, args);
  kernel_timer().end(st);
  DDSG_CUDA(cudaGetLastError());
  return 2;
}

}  // namespace ddsg_b200
