// Slot-staged HDMR evaluation kernel for low-order cut-HDMR programs
// (every active slot of order <= 2): the B200 hot path for BASELINE configs 4-5.
//
// Design:
//  * One CTA = kWarps x 32 points (lanes = points) x one block of kCols output
//    columns.  Every staged block (an active slot, or one stored-order run of
//    it) for that column block is a contiguous global region
//    [header | row table | slab], moved into a shared-memory ring of up to
//    kMaxStages stages by one TMA bulk copy (cp.async.bulk + mbarrier
//    expect-tx; per-stage "empty" mbarriers let warps run ahead).
//  * Each thread walks the block's subspaces in canonical order (statically
//    unrolled for order-1 levels <= kL1, order-2 level sums <= kL2 + 1 and
//    order-3 level sums <= kL3 + 2),
//    computes the candidate cell and the bit-exact weight, and gathers its
//    row with LDS.64: rows of kStride (9) doubles, or for full 1-d blocks the
//    rotated dual-copy rows of kRotStride doubles that keep every half-warp
//    on distinct banks.  Adaptive blocks are padded to full grids with zero
//    rows (same terms, static row bases).
//  * Leaf (slot) values enter the reference's pairwise tree through a
//    perfect-binary-tree embedding (leaf a at position t_a spanning 2^s_a):
//    pending levels 0..7 live in tensor memory (each thread owns its TMEM
//    lane in the warp's lane quarter, 16 columns per level,
//    tcgen05.st/ld 32x32b.x16 -- off the shared-memory pipe that the gathers
//    saturate), the rarely touched levels >= 8 in shared memory; the root is
//    written to y directly.
//  * EXACT mode: DMUL then DADD per term (bit-identical to the reference);
//    FAST mode: one DFMA per term.
#pragma once

#include <cuda_runtime.h>

#include <cstdint>
#include <vector>

#include "device.cuh"

namespace ddsg_b200 {

namespace fast {

#ifndef DDSG_SLOT_COLS
#define DDSG_SLOT_COLS 8                 // 8: 16 warps x 8 columns per CTA; 16: 8 warps x 16 columns
#endif
constexpr int kCols = DDSG_SLOT_COLS;    // output columns per thread / CTA column block
static_assert(kCols == 8 || kCols == 16, "slot kernel column block");
constexpr int kStride = kCols + 1;       // doubles per staged row: odd, so 16 consecutive rows
                                         // fall on 16 distinct 8-byte bank pairs (LDS.64 conflict-free)
constexpr int kWarps = kCols == 8 ? 16 : 8;  // 128 or 255 registers per thread
constexpr int kPoints = kWarps * 32;     // points per CTA
#ifndef DDSG_SLOT_AHEAD
#define DDSG_SLOT_AHEAD 1                // terms whose rows are in flight ahead of the accumulating term
#endif
constexpr int kAhead = DDSG_SLOT_AHEAD;  // (2 needs the 16-column build's registers)
constexpr int kL1 = 10;                  // max level of order-1 slots
constexpr int kL2 = 6;                   // max level (per dim) of order-2 slots
constexpr int kSub2 = kL2 * (kL2 + 1) / 2;  // canonical subspaces of a full order-2 grid
constexpr int kL3 = 4;                   // max level (per dim) of order-3 slots: level sums <= kL3 + 2
constexpr int kSub3 = kL3 * (kL3 + 1) * (kL3 + 2) / 6;  // 20 canonical subspaces (<= 32: bit masks)
constexpr int kMaxSub = (kSub2 > kL1 ? kSub2 : kL1) > kSub3 ? (kSub2 > kL1 ? kSub2 : kL1) : kSub3;
constexpr int kSlotDims = 3;             // point dims per slot in the dims table (order <= 3)
constexpr int kTmemLevels = 8;           // tree levels 1..8 in tensor memory (128 columns per warp)
constexpr int kSmemLevels = 4;           // levels 9..12 in shared memory (level 0 in registers)
constexpr int kMaxLevels = kTmemLevels + kSmemLevels;  // 2^12 active slots
constexpr int kMaxStages = 4;            // shared-memory ring depth (fewer when slot blocks are large)
constexpr int kHeaderBytes = 128;      // mbarriers + TMEM address slot
constexpr int kTableOff = 256;         // byte offset of the row table in a staged block (128-B aligned rows)
constexpr int kRotStride = 16;         // doubles per 128-byte row of the rotated layout
constexpr int kRotCopies = kRotStride / kCols;  // two copies of 8 columns, or the 16 columns once
constexpr int kTmemCols = 512 / (kWarps / 4);   // TMEM columns per warp (the warps of a lane quarter split 512)
static_assert(kTmemCols >= 2 * kCols * 8, "8 tree levels per warp in tensor memory");
constexpr int kMaxPaddedBytes = 96 * 1024;  // largest row table an adaptive block is padded to
constexpr int kMaxRotBytes = 48 * 1024;     // largest rotated table (1-d levels <= 8: 32 KB; 2-d level 6: 41 KB)
constexpr int kBCont = 4;   // b_kind flag: continue the previous block's accumulation (later run)
constexpr int kBMore = 8;   // b_kind flag: another run of the same slot follows

struct KernelArgs;
using LaunchFn = void (*)(dim3, size_t, cudaStream_t, const KernelArgs&);
using AttrFn = cudaError_t (*)(int);

// Per-slot header at the front of every staged block (16-B aligned, 160 B).
// The first 16 bytes are the core every slot needs, read with ONE broadcast
// LDS.128: `packed` = k (2 bits) | mode << 2 | nlev << 3 (4 bits) |
// fast_full << 7 (2 bits) | b_kind << 9 (4 bits) | tree_s << 13 (4 bits) |
// tree_t << 17 (13 bits); then the row table offset and b.  The rest serves
// the general (partial-grid) path.
struct SlotHeader {
  uint32_t packed;    // core (see above); written by pack_core()
  int32_t table_off;  // core: byte offset of the row table within the block
  double b;           // core
  int32_t k;          // slot order 0..2
  int32_t mode;       // boundary mode
  int32_t nlev;       // order 1: max level; order 2: max level per dim
  int32_t d0, d1;     // point dims of the slot (the third of an order-3 slot: d2 below)
  int32_t tree_t;     // leaf position in the perfect-tree embedding
  int32_t tree_s;     // leaf span exponent
  int32_t b_kind;     // bits 0-1: 0 multiply by b, 1 b == 1, 2 b == -1; | kBCont | kBMore
  uint32_t present;   // bit i: canonical subspace i has nodes
  uint32_t full;      // bit i: canonical subspace i has all its cells
  int32_t slab_off;   // byte offset of the int16 slab within the block
  int32_t zero_row;   // index of the all-zero row (target of skipped terms)
  int32_t fast_full;  // 1: full grid of level nlev with finite surpluses (static row layout); 2: same, rotated rows
  int32_t d2;
  int16_t sub_base[kMaxSub];  // first row (full) or slab index (partial) per subspace
  int16_t pad_[(160 - 72 - 2 * kMaxSub) / 2];
  void pack_core() {
    packed = static_cast<uint32_t>(k) | (static_cast<uint32_t>(mode) << 2) | (static_cast<uint32_t>(nlev) << 3) |
             (static_cast<uint32_t>(fast_full) << 7) | (static_cast<uint32_t>(b_kind) << 9) |
             (static_cast<uint32_t>(tree_s) << 13) | (static_cast<uint32_t>(tree_t) << 17);
  }
};
static_assert(sizeof(SlotHeader) == 160, "header layout");

}  // namespace fast

// Host-built, device-resident program of the fast kernel.
class FastHdmr {
 public:
  FastHdmr() = default;
  FastHdmr(const FastHdmr&) = delete;
  FastHdmr& operator=(const FastHdmr&) = delete;
  ~FastHdmr();

  // Builds the staged blocks when the program qualifies; returns usable().
  bool build(const HostProgram& hp);
  bool usable() const { return usable_; }
  // Launches the evaluation of n device points (x row-major [n][d]); xt is a
  // device scratch of at least n*d doubles (the dim-major copy of x).
  // Returns the number of kernel launches.
  int64_t launch(int exact, const double* x, int64_t n, int64_t base, double* y, unsigned long long* bad,
                 double* xt, cudaStream_t st, bool allow_split = true) const;
  // Bytes of the device scratch `xt` a launch over n points needs: the
  // dim-major points, plus the subtree partial sums of a split launch.
  size_t scratch_bytes(int64_t n, bool allow_split = true) const;
  // Subtree split of a launch over n points (0 = one launch walks every slot).
  int split_levels(int64_t n) const;
  double split_cost_us(int64_t n) const;
  static constexpr double kSubLaunchUs = 5.0, kSlotUs = 2.0;  // split cost model (measured, B200)

  int dim() const { return d_; }
  std::string why_not() const { return why_; }

 private:
  bool usable_ = false;
  std::string why_;
  fast::LaunchFn instance_launch(int exact) const;
  fast::AttrFn instance_attr(int exact) const;
  int d_ = 0, m_ = 0, n_cb_ = 0, cb_group_ = 1, n_active_ = 0, n_blocks_ = 0, has_carry_ = 0, has_order3_ = 0, levels_ = 0,
      n_stages_ = fast::kMaxStages;
  int64_t block_bytes_ = 0;  // stage size (max block), multiple of 128
  void* blocks_ = nullptr;   // [n_cb][n_active] blocks of block_bytes_ each (offsets below)
  int64_t* block_off_ = nullptr;  // device: [n_cb * n_active] byte offsets
  int32_t* block_len_ = nullptr;  // device: [n_cb * n_active] byte lengths
  int16_t* slot_dims_ = nullptr;  // device: [n_blocks][kSlotDims] point dims per block

  // Mid-size batches (a few tiles: fewer CTAs than SMs, every CTA walking all
  // slots one after another): the pairwise tree is cut at depth S and the 2^S
  // subtrees run as concurrent launches over their own block ranges of the
  // SAME staged tables (the kernel ignores tree-position bits >= its level
  // count, so a subtree's root comes out where the full launch writes y);
  // split_combine_kernel adds the subtree roots in tree order.  Bit-identical
  // to the single launch: same leaves, same merges.
  struct SubTree {
    int first = 0, count = 0;       // block range
    int64_t* off = nullptr;         // device: [n_cb][count] byte offsets into blocks_
    int32_t* len = nullptr;         // device: [n_cb][count]
  };
  static constexpr int kMaxSplit = 4;
 public:
  static constexpr int kMaxSplitPublic = kMaxSplit;
 private:
  std::vector<SubTree> split_[kMaxSplit + 1];  // [S]: 2^S subtrees (empty: depth S not splittable)
  int max_split_ = 0;
};

}  // namespace ddsg_b200
