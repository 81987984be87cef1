// Device code of the slot-staged HDMR kernel (see fast_hdmr.cuh / DESIGN.md
// §3.2), shared by the explicit-instantiation units fast_inst_*.cu (compiled
// in parallel) and the host builder in fast_hdmr.cu.
#pragma once

#include <cuda_runtime.h>
#include <algorithm>
#include <cstdlib>
#include <cmath>
#include <cstring>
#include <map>
#include "basis.cuh"
#include "fast_hdmr.cuh"

namespace ddsg_b200 {

namespace fast {

__device__ __forceinline__ uint32_t smem_u32(const void* p) {
  return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}

__device__ __forceinline__ void mbar_init(uint64_t* bar, uint32_t count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count) : "memory");
}

__device__ __forceinline__ void mbar_expect_tx(uint64_t* bar, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)), "r"(bytes)
               : "memory");
}

__device__ __forceinline__ void mbar_wait(uint64_t* bar, uint32_t parity) {
  asm volatile(
      "{\n"
      ".reg .pred p;\n"
      "WAIT_%=:\n"
      "mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n"
      "@!p bra WAIT_%=;\n"
      "}\n" ::"r"(smem_u32(bar)),
      "r"(parity)
      : "memory");
}

__device__ __forceinline__ void mbar_arrive(uint64_t* bar) {
  asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_u32(bar)) : "memory");
}

#ifndef DDSG_SLOT_L2HINT
#define DDSG_SLOT_L2HINT 0  // bit 0: point coordinates evict_last; bit 1: outputs evict_first; bit 2: tables evict_last
#endif
__device__ __forceinline__ uint64_t l2_policy_evict_last() {
  uint64_t p;
  asm volatile("createpolicy.fractional.L2::evict_last.b64 %0, 1.0;" : "=l"(p));
  return p;
}
__device__ __forceinline__ uint64_t l2_policy_evict_first() {
  uint64_t p;
  asm volatile("createpolicy.fractional.L2::evict_first.b64 %0, 1.0;" : "=l"(p));
  return p;
}
__device__ __forceinline__ double ldg_x(const double* p) {
  double v;
  asm volatile("ld.global.nc.L2::cache_hint.f64 %0, [%1], %2;" : "=d"(v) : "l"(p), "l"(l2_policy_evict_last()));
  return v;
}
__device__ __forceinline__ void stg_y(double* p, double v) {
  asm volatile("st.global.L2::cache_hint.f64 [%0], %1, %2;" ::"l"(p), "d"(v), "l"(l2_policy_evict_first()) : "memory");
}

__device__ __forceinline__ void bulk_g2s(void* dst, const void* src, uint32_t bytes, uint64_t* bar) {
  if (DDSG_SLOT_L2HINT & 4) {
    asm volatile(
        "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes.L2::cache_hint [%0], [%1], %2, [%3], %4;" ::"r"(
            smem_u32(dst)),
        "l"(src), "r"(bytes), "r"(smem_u32(bar)), "l"(l2_policy_evict_last())
        : "memory");
    return;
  }
  asm volatile(
      "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
          smem_u32(dst)),
      "l"(src), "r"(bytes), "r"(smem_u32(bar))
      : "memory");
}

__device__ __forceinline__ void fence_proxy_async() {
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
}

__device__ __forceinline__ void fence_mbar_init() {
  asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
}

// ---- tensor memory (per-thread scratch for deep pairwise-tree levels)
__device__ __forceinline__ void tmem_alloc(uint32_t* slot, uint32_t ncols) {
  asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(smem_u32(slot)),
               "r"(ncols)
               : "memory");
  asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;" ::: "memory");
}
__device__ __forceinline__ void tmem_dealloc(uint32_t taddr, uint32_t ncols) {
  asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(taddr), "r"(ncols) : "memory");
}
__device__ __forceinline__ void tmem_fence_before() {
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
}
__device__ __forceinline__ void tmem_fence_after() {
  asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
}
// 8 doubles of a thread <-> 16 consecutive 32-bit TMEM columns of its lane
__device__ __forceinline__ void tmem_store16(uint32_t taddr, const double* v) {
  uint32_t r[16];
#pragma unroll
  for (int c = 0; c < 8; ++c) {
    r[2 * c] = __double2loint(v[c]);
    r[2 * c + 1] = __double2hiint(v[c]);
  }
  asm volatile(
      "tcgen05.st.sync.aligned.32x32b.x16.b32 [%0], {%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,%16};" ::"r"(
          taddr),
      "r"(r[0]), "r"(r[1]), "r"(r[2]), "r"(r[3]), "r"(r[4]), "r"(r[5]), "r"(r[6]), "r"(r[7]), "r"(r[8]),
      "r"(r[9]), "r"(r[10]), "r"(r[11]), "r"(r[12]), "r"(r[13]), "r"(r[14]), "r"(r[15])
      : "memory");
}
__device__ __forceinline__ void tmem_load16(uint32_t taddr, uint32_t (&r)[16]) {
  asm volatile(
      "tcgen05.ld.sync.aligned.32x32b.x16.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15}, [%16];"
      : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]), "=r"(r[7]),
        "=r"(r[8]), "=r"(r[9]), "=r"(r[10]), "=r"(r[11]), "=r"(r[12]), "=r"(r[13]), "=r"(r[14]), "=r"(r[15])
      : "r"(taddr)
      : "memory");
}
// A thread's kCols doubles of one tree level: 2 * kCols TMEM columns.
__device__ __forceinline__ void tmem_store8(uint32_t taddr, const double (&v)[kCols]) {
#pragma unroll
  for (int h = 0; h < kCols / 8; ++h) tmem_store16(taddr + 16u * h, v + 8 * h);
  asm volatile("tcgen05.wait::st.sync.aligned;" ::: "memory");
}
__device__ __forceinline__ void tmem_load8(uint32_t taddr, double (&v)[kCols]) {
  uint32_t r[kCols / 8][16];
#pragma unroll
  for (int h = 0; h < kCols / 8; ++h) tmem_load16(taddr + 16u * h, r[h]);
  asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
#pragma unroll
  for (int c = 0; c < kCols; ++c)
    v[c] = __hiloint2double(static_cast<int>(r[c / 8][2 * (c % 8) + 1]), static_cast<int>(r[c / 8][2 * (c % 8)]));
}

template <int kExact>
__device__ __forceinline__ void accum_row(double (&acc)[kCols], double w, const unsigned char* table,
                                          int row) {
  const double* sr = reinterpret_cast<const double*>(table + row * (kStride * 8));
#pragma unroll
  for (int c = 0; c < kCols; ++c) {
    const double v = sr[c];
    acc[c] = kExact ? __dadd_rn(acc[c], __dmul_rn(w, v)) : __fma_rn(w, v, acc[c]);
  }
}

// Branch-free 1-d factor at level l (static): candidate cell and basis value
// (basis_at in basis.cuh, written with selects so the compiler can schedule
// every subspace of a slot as one straight-line block).
template <int l>
__device__ __forceinline__ void factor(int mode, double x, uint32_t& kk, double& v) {
  kk = cell_at(x, l);
  if (l == 1 && mode == 1) {
    v = 1.0;
    return;
  }
  const double scale = static_cast<double>(1u << l);
  const double t = __dmul_rn(x, scale);
  const double hat = __dadd_rn(1.0, -fabs(__dadd_rn(t, -static_cast<double>(2u * kk + 1u))));
  const double left = __dadd_rn(2.0, -t);
  const double right = __dadd_rn(2.0, -__dadd_rn(scale, -t));
  double r = hat;
  if (l >= 2) {
    r = (mode == 1 && kk == 0u) ? left : r;
    r = (mode == 1 && kk == (1u << (l - 1)) - 1u) ? right : r;
  }
  v = r > 0.0 ? r : 0.0;
}

// Row of the candidate node of canonical subspace idx, or the slot's zero row
// when the subspace is absent, the cell is absent, or the weight is 0 (the
// reference skips w == 0 terms; adding w * 0 leaves the accumulator's bits
// unchanged because it is never -0).
__device__ __forceinline__ int term_row(const SlotHeader& H, const unsigned char* blk, int idx, int cell,
                                        double w, bool all_full) {
  const int base = H.sub_base[idx];
  int row;
  if (all_full) {
    row = base + cell;
  } else {
    row = ((H.full >> idx) & 1u) ? base + cell : reinterpret_cast<const int16_t*>(blk + H.slab_off)[base + cell];
  }
  const bool ok = ((H.present >> idx) & 1u) && w != 0.0 && row >= 0;
  return ok ? row : H.zero_row;
}

template <int kExact, int L>
__device__ __forceinline__ void leaf_order1(const SlotHeader& H, const unsigned char* blk, double x,
                                            double (&acc)[kCols], bool all_full) {
  const unsigned char* table = blk + H.table_off;
  const int mode = H.mode;
  double w[L];
  int row[L];
#pragma unroll
  for (int l = 1; l <= L; ++l) {
    uint32_t kk;
    double v;
    switch (l) {  // static level for the factor template
#define DDSG_F(LV) \
  case LV:         \
    factor<LV>(mode, x, kk, v); \
    break;
      DDSG_F(1) DDSG_F(2) DDSG_F(3) DDSG_F(4) DDSG_F(5) DDSG_F(6) DDSG_F(7) DDSG_F(8) DDSG_F(9) DDSG_F(10)
#undef DDSG_F
      default:
        kk = 0;
        v = 0.0;
    }
    row[l - 1] = term_row(H, blk, l - 1, static_cast<int>(kk), v, all_full);
    w[l - 1] = v;
  }
#pragma unroll
  for (int l = 0; l < L; ++l) accum_row<kExact>(acc, w[l], table, row[l]);
}

template <int kExact, int L>
__device__ __forceinline__ void leaf_order2(const SlotHeader& H, const unsigned char* blk, double x0,
                                            double x1, double (&acc)[kCols], bool all_full) {
  const unsigned char* table = blk + H.table_off;
  const int mode = H.mode;
  double v0[L], v1[L];
  uint32_t k0[L], k1[L];
#pragma unroll
  for (int l = 1; l <= L; ++l) {
    switch (l) {
#define DDSG_F(LV)                          \
  case LV:                                  \
    factor<LV>(mode, x0, k0[l - 1], v0[l - 1]); \
    factor<LV>(mode, x1, k1[l - 1], v1[l - 1]); \
    break;
      DDSG_F(1) DDSG_F(2) DDSG_F(3) DDSG_F(4) DDSG_F(5) DDSG_F(6)
#undef DDSG_F
      default:
        break;
    }
  }
  constexpr int kN = L * (L + 1) / 2;
  double w[kN];
  int row[kN];
  int idx = 0;
#pragma unroll
  for (int s = 2; s <= L + 1; ++s) {
#pragma unroll
    for (int l1 = 1; l1 < s; ++l1) {
      const int l2 = s - l1;
      // reference: w = 1 * v0; if (w == 0) break; w *= v1  -> fl(v0 * v1) (0 if v0 == 0)
      const double ww = __dmul_rn(v0[l1 - 1], v1[l2 - 1]);
      const int cell = static_cast<int>((k0[l1 - 1] << (l2 - 1)) | k1[l2 - 1]);
      row[idx] = term_row(H, blk, idx, cell, ww, all_full);
      w[idx] = ww;
      ++idx;
    }
  }
#pragma unroll
  for (int i = 0; i < kN; ++i) accum_row<kExact>(acc, w[i], table, row[i]);
}

// General-path order-3 slot (partial grids with non-finite surpluses: rare):
// a rolled loop over the canonical subspaces with runtime-level factors
// (basis.cuh), compact code instead of the unrolled static leaves.
template <int kExact>
__device__ __forceinline__ void leaf_order3(const SlotHeader& H, const unsigned char* blk, double x0, double x1,
                                            double x2, double (&acc)[kCols], bool all_full) {
  const unsigned char* table = blk + H.table_off;
  const int mode = H.mode;
  const int L = H.nlev;
  int idx = 0;
#pragma unroll 1
  for (int s = 3; s <= L + 2; ++s) {
#pragma unroll 1
    for (int l1 = 1; l1 < s - 1; ++l1) {
#pragma unroll 1
      for (int l2 = 1; l1 + l2 < s; ++l2, ++idx) {
        const int l3 = s - l1 - l2;
        const uint32_t k0 = cell_at(x0, l1), k1 = cell_at(x1, l2), k2 = cell_at(x2, l3);
        // reference: w = 1 * v0, * v1, * v2 in dim order (0 stays 0)
        const double w = __dmul_rn(__dmul_rn(basis_at(mode, l1, k0, x0), basis_at(mode, l2, k1, x1)),
                                   basis_at(mode, l3, k2, x2));
        const int cell = static_cast<int>((k0 << (l2 + l3 - 2)) | (k1 << (l3 - 1)) | k2);
        accum_row<kExact>(acc, w, table, term_row(H, blk, idx, cell, w, all_full));
      }
    }
  }
}

// ------------------------------------------------------------------ full grids
// A full order-1 grid of max level L stores level l's 2^(l-1) cells from row
// 2^(l-1) - 1; a full order-2 grid stores canonical subspace (l1, l2) from
// row base2(l1, l2) (rows of all earlier subspaces in (|l|_1, l lex) order).
__host__ __device__ constexpr int base1(int l) { return (1 << (l - 1)) - 1; }
__host__ __device__ constexpr int base2(int l1, int l2) {
  int b = 0;
  for (int t = 2; t < l1 + l2; ++t) b += (t - 1) << (t - 2);
  return b + ((l1 - 1) << (l1 + l2 - 2));
}
// A full order-3 grid stores canonical subspace (l1, l2, l3) from row
// base3(l1, l2, l3): every subspace of level sum s holds 2^(s-3) cells.
__host__ __device__ constexpr int base3(int l1, int l2, int l3) {
  int b = 0;
  const int s = l1 + l2 + l3;
  for (int t = 3; t < s; ++t) b += ((t - 1) * (t - 2) / 2) << (t - 3);
  for (int a = 1; a < l1; ++a) b += (s - a - 1) << (s - 3);
  return b + ((l2 - 1) << (s - 3));
}

// Exact 1-d factor of the candidate node at static level l (basis.hpp:36-54):
// with t = x 2^l, every kind is v = fl(A - |fl(t - B)|):
//   hat (A, B) = (1, 2k+1); left edge (2, 0); right edge (2, 2^l);
//   modified level 1 is the constant 1.  v >= 0 for the candidate cell, so the
//   reference's max(v, 0) is the identity here.
template <int l, int kMode>
__device__ __forceinline__ void factor_full(double x, uint32_t& kk, double& v) {
  constexpr uint32_t ncell = 1u << (l - 1);
  const uint32_t k = static_cast<uint32_t>(__dmul_rn(x, static_cast<double>(ncell)));
  kk = k < ncell ? k : ncell - 1u;
  if (kMode == 1 && l == 1) {
    v = 1.0;
    return;
  }
  const double t = __dmul_rn(x, static_cast<double>(2u * ncell));
  uint32_t B = 2u * kk + 1u;
  double A = 1.0;
  if (kMode == 1) {
    const bool left = kk == 0u, right = kk == ncell - 1u;
    B = left ? 0u : (right ? 2u * ncell : B);
    A = (left || right) ? 2.0 : 1.0;
  }
  v = __dadd_rn(A, -fabs(__dadd_rn(t, -static_cast<double>(B))));
}

template <int kExact>
__device__ __forceinline__ void fma_row(double (&acc)[kCols], double w, const double (&s)[kCols]) {
#pragma unroll
  for (int c = 0; c < kCols; ++c) {
    if (kExact)
      acc[c] = __dadd_rn(acc[c], __dmul_rn(w, s[c]));
    else
      acc[c] = __fma_rn(w, s[c], acc[c]);
  }
}

// LDS.64 gathers: lanes (points) read the same column of their rows.
__device__ __forceinline__ void load_row(const unsigned char* table, int row, double (&s)[kCols]) {
  const double* sr = reinterpret_cast<const double*>(table + row * (kStride * 8));
#pragma unroll
  for (int c = 0; c < kCols; ++c) s[c] = sr[c];
}

// Full order-1 slot: levels 1..L, one term per level, loads one term ahead.
// Terms with w == 0 are accumulated too: the surpluses are finite (checked on
// the host), so w * s = +-0 and the accumulator (never -0) keeps its bits.
template <int kExact, int kMode, int L>
__device__ __forceinline__ void leaf_full1(const unsigned char* table, double x, double (&acc)[kCols]) {
  double w[L];
  int row[L];
#pragma unroll
  for (int l = 1; l <= L; ++l) {
    uint32_t kk;
    switch (l) {
#define DDSG_F(LV)                               \
  case LV:                                       \
    factor_full<LV, kMode>(x, kk, w[l - 1]);     \
    break;
      DDSG_F(1) DDSG_F(2) DDSG_F(3) DDSG_F(4) DDSG_F(5) DDSG_F(6) DDSG_F(7) DDSG_F(8) DDSG_F(9) DDSG_F(10)
#undef DDSG_F
      default:
        kk = 0;
        w[l - 1] = 0.0;
    }
    row[l - 1] = base1(l) + static_cast<int>(kk);
  }
  double buf[kAhead + 1][kCols];  // static ring: terms i+1..i+kAhead load while term i accumulates
#pragma unroll
  for (int i = 0; i < kAhead && i < L; ++i) load_row(table, row[i], buf[i]);
#pragma unroll
  for (int i = 0; i < L; ++i) {
    if (i + kAhead < L) load_row(table, row[i + kAhead], buf[(i + kAhead) % (kAhead + 1)]);
    fma_row<kExact>(acc, w[i], buf[i % (kAhead + 1)]);
  }
}

__device__ __forceinline__ void lds_f64x2(uint32_t addr, double& a, double& b) {
  asm volatile("ld.shared.v2.f64 {%0, %1}, [%2];" : "=d"(a), "=d"(b) : "r"(addr));
}

__device__ __forceinline__ double lds_f64(uint32_t addr) {
  double v;
  asm volatile("ld.shared.f64 %0, [%1];" : "=d"(v) : "r"(addr));
  return v;
}

// One rotated row (address | lane bits): slot pair j <- column pair (lane rotation) ^ j.
__device__ __forceinline__ void load_row_rot(uint32_t addr, double (&s)[kCols]) {
#pragma unroll
  for (int j = 0; j < kCols / 2; ++j) lds_f64x2(addr ^ static_cast<uint32_t>(j << 4), s[2 * j], s[2 * j + 1]);
}

// Rotated layout: un-rotate an accumulator (see leaf_full1_rot).
__device__ __forceinline__ void unrotate(uint32_t q0, double (&acc)[kCols]) {
  // slot pair j holds column pair p0 ^ j (p0 = this lane's rotation, bits 4-5 of q0)
  const uint32_t p0 = (q0 >> 4) & static_cast<uint32_t>(kCols / 2 - 1);
#pragma unroll
  for (int b = 1; b < kCols / 2; b <<= 1) {
    const bool flip = (p0 & static_cast<uint32_t>(b)) != 0u;
#pragma unroll
    for (int j = 0; j < kCols / 2; ++j)
      if (!(j & b)) {
#pragma unroll
        for (int h = 0; h < 2; ++h) {
          const double lo = acc[2 * j + h], hi = acc[2 * (j | b) + h];
          acc[2 * j + h] = flip ? hi : lo;
          acc[2 * (j | b) + h] = flip ? lo : hi;
        }
      }
  }
}

// Full order-1 slot in the rotated layout (fast_full == 2): rows of 16
// doubles holding the 8 columns twice (two 64-byte copies).  Lane l reads
// copy (l >> 2) & 1 and, at step j, column pair (l & 3) ^ j into slot pair j
// with one LDS.128, so the 8 lanes of a quarter-warp hit the row's 8
// distinct 16-byte units whatever their rows: the deep levels' 32-128
// candidate rows cost 2 wavefronts per column instead of 3.9-5.5
// (profiles/r1_lds_rotate.json).  The slot starts from a zero accumulator
// (rotation-free) and un-rotates it once at the end.  q0 = shared address of
// row 0 | lane bits.
template <int kExact, int kMode, int L>
__device__ __forceinline__ void leaf_full1_rot(uint32_t q0, double x, double (&acc)[kCols]) {
  double w[L];
  uint32_t row[L];
#pragma unroll
  for (int l = 1; l <= L; ++l) {
    uint32_t kk;
    switch (l) {
#define DDSG_F(LV)                               \
  case LV:                                       \
    factor_full<LV, kMode>(x, kk, w[l - 1]);     \
    break;
      DDSG_F(1) DDSG_F(2) DDSG_F(3) DDSG_F(4) DDSG_F(5) DDSG_F(6) DDSG_F(7) DDSG_F(8) DDSG_F(9) DDSG_F(10)
#undef DDSG_F
      default:
        kk = 0;
        w[l - 1] = 0.0;
    }
    row[l - 1] = q0 + ((static_cast<uint32_t>(base1(l)) + kk) << 7);
  }
  double buf[kAhead + 1][kCols];  // static ring: terms i+1..i+kAhead load while term i accumulates
#pragma unroll
  for (int i = 0; i < kAhead && i < L; ++i) load_row_rot(row[i], buf[i]);
#pragma unroll
  for (int i = 0; i < L; ++i) {
    if (i + kAhead < L) load_row_rot(row[i + kAhead], buf[(i + kAhead) % (kAhead + 1)]);
    fma_row<kExact>(acc, w[i], buf[i % (kAhead + 1)]);
  }
  unrotate(q0, acc);
}

// Full order-2 slot with max level L per dim (level sum <= L + 1), canonical
// order; w = fl(v0 * v1) (exact 1 * v when a factor is the modified level-1 constant).
template <int kExact, int kMode, int L>
__device__ __forceinline__ void leaf_full2(const unsigned char* table, double x0, double x1, double (&acc)[kCols]) {
  double v0[L], v1[L];
  uint32_t k0[L], k1[L];
#pragma unroll
  for (int l = 1; l <= L; ++l) {
    switch (l) {
#define DDSG_F(LV)                                  \
  case LV:                                          \
    factor_full<LV, kMode>(x0, k0[l - 1], v0[l - 1]); \
    factor_full<LV, kMode>(x1, k1[l - 1], v1[l - 1]); \
    break;
      DDSG_F(1) DDSG_F(2) DDSG_F(3) DDSG_F(4) DDSG_F(5) DDSG_F(6)
#undef DDSG_F
      default:
        break;
    }
  }
  constexpr int kN = L * (L + 1) / 2;
  // term i of the canonical sequence: (l1, l2) with l1 + l2 = s
  auto term = [&](int i, double& w, int& row) {
    int idx = 0;
#pragma unroll
    for (int s = 2; s <= L + 1; ++s)
#pragma unroll
      for (int l1 = 1; l1 < s; ++l1) {
        const int l2 = s - l1;
        if (idx == i) {
          if (kMode == 1 && l1 == 1)
            w = v1[l2 - 1];
          else if (kMode == 1 && l2 == 1)
            w = v0[l1 - 1];
          else
            w = __dmul_rn(v0[l1 - 1], v1[l2 - 1]);
          row = base2(l1, l2) + static_cast<int>((k0[l1 - 1] << (l2 - 1)) | k1[l2 - 1]);
        }
        ++idx;
      }
  };
  constexpr int kR = kAhead + 1;
  double wb[kR];
  int rb[kR];
  double buf[kR][kCols];  // static ring
#pragma unroll
  for (int i = 0; i < kAhead && i < kN; ++i) {
    term(i, wb[i], rb[i]);
    load_row(table, rb[i], buf[i]);
  }
#pragma unroll
  for (int i = 0; i < kN; ++i) {
    if (i + kAhead < kN) {
      term(i + kAhead, wb[(i + kAhead) % kR], rb[(i + kAhead) % kR]);
      load_row(table, rb[(i + kAhead) % kR], buf[(i + kAhead) % kR]);
    }
    fma_row<kExact>(acc, wb[i % kR], buf[i % kR]);
  }
}

// Canonical order-3 subspace i: (l1, l2, l3) with level sums ascending, lex.
struct Sub3 {
  int l1, l2, l3;
};
__host__ __device__ constexpr Sub3 sub3(int i) {
  int idx = 0;
  for (int s = 3; s < 32; ++s)
    for (int l1 = 1; l1 < s - 1; ++l1)
      for (int l2 = 1; l1 + l2 < s; ++l2) {
        if (idx == i) return Sub3{l1, l2, s - l1 - l2};
        ++idx;
      }
  return Sub3{1, 1, 1};
}

// Term I of a full order-3 leaf: weight and row from compile-time levels.
template <int kMode, int L, int I>
__device__ __forceinline__ void term3(const double (&v0)[L], const double (&v1)[L], const double (&v2)[L],
                                      const uint32_t (&k0)[L], const uint32_t (&k1)[L], const uint32_t (&k2)[L],
                                      double& w, int& row) {
  constexpr Sub3 t = sub3(I);
  w = __dmul_rn(__dmul_rn(v0[t.l1 - 1], v1[t.l2 - 1]), v2[t.l3 - 1]);
  row = base3(t.l1, t.l2, t.l3) + static_cast<int>((k0[t.l1 - 1] << (t.l2 + t.l3 - 2)) |
                                                   (k1[t.l2 - 1] << (t.l3 - 1)) | k2[t.l3 - 1]);
}

// Terms I.. of a full order-3 leaf, one term ahead (static ping-pong).
template <int kExact, int kMode, int L, int I>
__device__ __forceinline__ void walk3(const unsigned char* table, const double (&v0)[L], const double (&v1)[L],
                                      const double (&v2)[L], const uint32_t (&k0)[L], const uint32_t (&k1)[L],
                                      const uint32_t (&k2)[L], double (&acc)[kCols], double w, double (&cur)[kCols]) {
  constexpr int kN = L * (L + 1) * (L + 2) / 6;
  if constexpr (I + 1 < kN) {
    double wn;
    int rn;
    term3<kMode, L, I + 1>(v0, v1, v2, k0, k1, k2, wn, rn);
    double nxt[kCols];
    load_row(table, rn, nxt);
    fma_row<kExact>(acc, w, cur);
    walk3<kExact, kMode, L, I + 1>(table, v0, v1, v2, k0, k1, k2, acc, wn, nxt);
  } else {
    fma_row<kExact>(acc, w, cur);
  }
}

// Full order-3 slot with max level L per dim (level sums <= L + 2),
// canonical order, stride-9 rows; w = ((v0 v1) v2) in dim order (the
// modified level-1 factor 1 makes its products exact).
template <int kExact, int kMode, int L>
__device__ __forceinline__ void leaf_full3(const unsigned char* table, double x0, double x1, double x2,
                                           double (&acc)[kCols]) {
  double v0[L], v1[L], v2[L];
  uint32_t k0[L], k1[L], k2[L];
#pragma unroll
  for (int l = 1; l <= L; ++l) {
    switch (l) {
#define DDSG_F(LV)                                    \
  case LV:                                            \
    factor_full<LV, kMode>(x0, k0[l - 1], v0[l - 1]); \
    factor_full<LV, kMode>(x1, k1[l - 1], v1[l - 1]); \
    factor_full<LV, kMode>(x2, k2[l - 1], v2[l - 1]); \
    break;
      DDSG_F(1) DDSG_F(2) DDSG_F(3) DDSG_F(4)
#undef DDSG_F
      default:
        break;
    }
  }
  double w;
  int row;
  term3<kMode, L, 0>(v0, v1, v2, k0, k1, k2, w, row);
  double cur[kCols];
  load_row(table, row, cur);
  walk3<kExact, kMode, L, 0>(table, v0, v1, v2, k0, k1, k2, acc, w, cur);
}

// Full order-2 slot in the rotated layout (fast_full == 2; max level L >= 6,
// whose level-sum-7 subspaces have 32 candidate rows and conflict in the
// stride-9 layout): leaf_full2's terms and order, leaf_full1_rot's loads.
template <int kExact, int kMode, int L>
__device__ __forceinline__ void leaf_full2_rot(uint32_t q0, double x0, double x1, double (&acc)[kCols]) {
  double v0[L], v1[L];
  uint32_t k0[L], k1[L];
#pragma unroll
  for (int l = 1; l <= L; ++l) {
    switch (l) {
#define DDSG_F(LV)                                  \
  case LV:                                          \
    factor_full<LV, kMode>(x0, k0[l - 1], v0[l - 1]); \
    factor_full<LV, kMode>(x1, k1[l - 1], v1[l - 1]); \
    break;
      DDSG_F(1) DDSG_F(2) DDSG_F(3) DDSG_F(4) DDSG_F(5) DDSG_F(6)
#undef DDSG_F
      default:
        break;
    }
  }
  constexpr int kN = L * (L + 1) / 2;
  auto term = [&](int i, double& w, uint32_t& addr) {
    int idx = 0;
#pragma unroll
    for (int s = 2; s <= L + 1; ++s)
#pragma unroll
      for (int l1 = 1; l1 < s; ++l1) {
        const int l2 = s - l1;
        if (idx == i) {
          if (kMode == 1 && l1 == 1)
            w = v1[l2 - 1];
          else if (kMode == 1 && l2 == 1)
            w = v0[l1 - 1];
          else
            w = __dmul_rn(v0[l1 - 1], v1[l2 - 1]);
          addr = q0 + ((static_cast<uint32_t>(base2(l1, l2)) + ((k0[l1 - 1] << (l2 - 1)) | k1[l2 - 1])) << 7);
        }
        ++idx;
      }
  };
  constexpr int kR = kAhead + 1;
  double wb[kR];
  uint32_t ab[kR];
  double buf[kR][kCols];  // static ring
#pragma unroll
  for (int i = 0; i < kAhead && i < kN; ++i) {
    term(i, wb[i], ab[i]);
    load_row_rot(ab[i], buf[i]);
  }
#pragma unroll
  for (int i = 0; i < kN; ++i) {
    if (i + kAhead < kN) {
      term(i + kAhead, wb[(i + kAhead) % kR], ab[(i + kAhead) % kR]);
      load_row_rot(ab[(i + kAhead) % kR], buf[(i + kAhead) % kR]);
    }
    fma_row<kExact>(acc, wb[i % kR], buf[i % kR]);
  }
  unrotate(q0, acc);
}

// The header fields every slot needs: one broadcast 16-byte load, decoded.
struct HeaderCore {
  int k, mode, nlev, fast_full, b_kind, tree_s, tree_t, table_off;
  double b;
};
__device__ __forceinline__ HeaderCore load_core(const unsigned char* blk) {
  const uint4 raw = *reinterpret_cast<const uint4*>(blk);
  HeaderCore h;
  const uint32_t p = raw.x;
  h.k = static_cast<int>(p & 3u);
  h.mode = static_cast<int>((p >> 2) & 1u);
  h.nlev = static_cast<int>((p >> 3) & 15u);
  h.fast_full = static_cast<int>((p >> 7) & 3u);
  h.b_kind = static_cast<int>((p >> 9) & 15u);
  h.tree_s = static_cast<int>((p >> 13) & 15u);
  h.tree_t = static_cast<int>(p >> 17);
  h.table_off = static_cast<int>(raw.y);
  h.b = __hiloint2double(static_cast<int>(raw.w), static_cast<int>(raw.z));
  return h;
}

template <int kExact, int kOrder3>
__device__ __forceinline__ void leaf_dispatch(const HeaderCore& Hc, const SlotHeader& H, const unsigned char* blk,
                                              double x0, double x1, double x2, double (&acc)[kCols],
                                              uint32_t lanebits) {
  const unsigned char* table = blk + Hc.table_off;
  if (Hc.fast_full == 2) {
    const uint32_t q0 = smem_u32(table) | lanebits;
    if (Hc.k == 2) {
      switch (Hc.mode * 16 + Hc.nlev) {
#define DDSG_R2(MD, LV) \
  case MD * 16 + LV: \
    leaf_full2_rot<kExact, MD, LV>(q0, x0, x1, acc); \
    return;
        DDSG_R2(0, 2) DDSG_R2(0, 3) DDSG_R2(0, 4) DDSG_R2(0, 5) DDSG_R2(0, 6)
        DDSG_R2(1, 2) DDSG_R2(1, 3) DDSG_R2(1, 4) DDSG_R2(1, 5) DDSG_R2(1, 6)
#undef DDSG_R2
        default:
          return;
      }
    }
    switch (Hc.mode * 16 + Hc.nlev) {
#define DDSG_R1(MD, LV) \
  case MD * 16 + LV: \
    leaf_full1_rot<kExact, MD, LV>(q0, x0, acc); \
    return;
      DDSG_R1(0, 1) DDSG_R1(0, 2) DDSG_R1(0, 3) DDSG_R1(0, 4) DDSG_R1(0, 5) DDSG_R1(0, 6) DDSG_R1(0, 7)
      DDSG_R1(0, 8) DDSG_R1(0, 9) DDSG_R1(0, 10)
      DDSG_R1(1, 1) DDSG_R1(1, 2) DDSG_R1(1, 3) DDSG_R1(1, 4) DDSG_R1(1, 5) DDSG_R1(1, 6) DDSG_R1(1, 7)
      DDSG_R1(1, 8) DDSG_R1(1, 9) DDSG_R1(1, 10)
#undef DDSG_R1
      default:
        return;
    }
  }
  if (Hc.fast_full) {
    switch (Hc.mode * 64 + Hc.k * 16 + Hc.nlev) {
#define DDSG_P1(MD, LV) \
  case MD * 64 + 16 + LV: \
    leaf_full1<kExact, MD, LV>(table, x0, acc); \
    return;
#define DDSG_P2(MD, LV) \
  case MD * 64 + 32 + LV: \
    leaf_full2<kExact, MD, LV>(table, x0, x1, acc); \
    return;
      DDSG_P1(0, 1) DDSG_P1(0, 2) DDSG_P1(0, 3) DDSG_P1(0, 4) DDSG_P1(0, 5) DDSG_P1(0, 6) DDSG_P1(0, 7)
      DDSG_P1(0, 8) DDSG_P1(0, 9) DDSG_P1(0, 10)
      DDSG_P1(1, 1) DDSG_P1(1, 2) DDSG_P1(1, 3) DDSG_P1(1, 4) DDSG_P1(1, 5) DDSG_P1(1, 6) DDSG_P1(1, 7)
      DDSG_P1(1, 8) DDSG_P1(1, 9) DDSG_P1(1, 10)
      DDSG_P2(0, 1) DDSG_P2(0, 2) DDSG_P2(0, 3) DDSG_P2(0, 4) DDSG_P2(0, 5) DDSG_P2(0, 6)
      DDSG_P2(1, 1) DDSG_P2(1, 2) DDSG_P2(1, 3) DDSG_P2(1, 4) DDSG_P2(1, 5) DDSG_P2(1, 6)
#define DDSG_P3(MD, LV) \
  case MD * 64 + 48 + LV: \
    if constexpr (kOrder3 != 0) leaf_full3<kExact, MD, LV>(table, x0, x1, x2, acc); \
    return;
      DDSG_P3(0, 1) DDSG_P3(0, 2) DDSG_P3(0, 3) DDSG_P3(0, 4)
      DDSG_P3(1, 1) DDSG_P3(1, 2) DDSG_P3(1, 3) DDSG_P3(1, 4)
#undef DDSG_P1
#undef DDSG_P2
#undef DDSG_P3
      default:
        break;
    }
  }
  // general path: adaptive / partial grids or non-finite surpluses
  const bool all_full = H.full == H.present;
  switch (H.k * 16 + H.nlev) {
#define DDSG_L1(LV) \
  case 16 + LV:     \
    leaf_order1<kExact, LV>(H, blk, x0, acc, all_full); \
    break;
#define DDSG_L2(LV) \
  case 32 + LV:     \
    leaf_order2<kExact, LV>(H, blk, x0, x1, acc, all_full); \
    break;
#define DDSG_L3(LV) \
  case 48 + LV:     \
    if constexpr (kOrder3 != 0) leaf_order3<kExact>(H, blk, x0, x1, x2, acc, all_full); \
    break;
    DDSG_L1(1) DDSG_L1(2) DDSG_L1(3) DDSG_L1(4) DDSG_L1(5) DDSG_L1(6) DDSG_L1(7) DDSG_L1(8) DDSG_L1(9) DDSG_L1(10)
    DDSG_L2(1) DDSG_L2(2) DDSG_L2(3) DDSG_L2(4) DDSG_L2(5) DDSG_L2(6)
    DDSG_L3(1) DDSG_L3(2) DDSG_L3(3) DDSG_L3(4)
#undef DDSG_L1
#undef DDSG_L2
#undef DDSG_L3
    default:
      break;
  }
}

// Pending level i (>= 1) of the pairwise tree for this thread.
struct TreeStore {
  double2* smem;   // [kSmemLevels][kCols/2][kPoints] (levels > kTmemLevels)
  uint32_t tbase;  // TMEM address of this warp's lane quarter / column block
  int tid;
  __device__ __forceinline__ void load(int i, double (&v)[kCols]) const {
    if (i < kTmemLevels) {
      tmem_load8(tbase + static_cast<uint32_t>(2 * kCols * i), v);
    } else {
      const double2* L = smem + (static_cast<int64_t>(i - kTmemLevels) * (kCols / 2)) * kPoints + tid;
#pragma unroll
      for (int q = 0; q < kCols / 2; ++q) {
        const double2 x = L[q * kPoints];
        v[2 * q] = x.x;
        v[2 * q + 1] = x.y;
      }
    }
  }
  __device__ __forceinline__ void store(int i, const double (&v)[kCols]) const {
    if (i < kTmemLevels) {
      tmem_store8(tbase + static_cast<uint32_t>(2 * kCols * i), v);
    } else {
      double2* L = smem + (static_cast<int64_t>(i - kTmemLevels) * (kCols / 2)) * kPoints + tid;
#pragma unroll
      for (int q = 0; q < kCols / 2; ++q) L[q * kPoints] = make_double2(v[2 * q], v[2 * q + 1]);
    }
  }
};

template <int kExact, int kCarry, int kOrder3>
__global__ void __launch_bounds__(kPoints, 1)
    fast_hdmr_kernel(const unsigned char* __restrict__ blocks, const int64_t* __restrict__ block_off,
                     const int32_t* __restrict__ block_len, const int16_t* __restrict__ slot_dims,
                     int n_active, int n_cb, int cb_group, int levels, const double* __restrict__ xt, int64_t n,
                     int m,
                     double* __restrict__ y, int64_t stage_bytes, int n_stages) {
  extern __shared__ __align__(128) unsigned char smem[];
  uint64_t* bars = reinterpret_cast<uint64_t*>(smem);  // [kMaxStages] full, [kMaxStages] empty
  uint64_t* empty = bars + kMaxStages;
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(smem + 16 * kMaxStages);
  unsigned char* stages = smem + kHeaderBytes;
  double2* deep = reinterpret_cast<double2*>(stages + n_stages * stage_bytes);
  const int smem_levels = min(max(levels - kTmemLevels, 0), kSmemLevels);
  // partial sums of multi-run slots between their blocks ([kCols/2][kPoints], only when present)
  double2* carry = deep + static_cast<int64_t>(smem_levels) * (kCols / 2) * kPoints;
  int16_t* sdims = reinterpret_cast<int16_t*>(carry + (kCarry ? (kCols / 2) * kPoints : 0));
  const bool use_tmem = levels > 0;

  // CTA order: column blocks in groups of cb_group; within a group, the
  // group's column blocks of one point tile are adjacent.  Concurrent CTAs
  // then share a few column blocks' slot tables (L2-resident) while each
  // tile's points are re-read only n_cb / cb_group times.
  const int64_t tiles = (n + kPoints - 1) / kPoints;
  const int64_t per_group = tiles * cb_group;
  const int grp = static_cast<int>(blockIdx.x / per_group);
  const int64_t rem = blockIdx.x - grp * per_group;
  const int gsize = min(cb_group, n_cb - grp * cb_group);
  const int64_t tile = rem / gsize;
  const int cb = grp * cb_group + static_cast<int>(rem - tile * gsize);
  const int tid = threadIdx.x;
  const int warp = tid >> 5;
  // rotated-layout lane bits: copy (bit 6) = (lane >> 2) & 1, column-pair
  // rotation (bits 4-5) = lane & 3 -- the 8 lanes of a quarter-warp hit the 8
  // distinct 16-byte units of a 128-byte row in every LDS.128
  // (16 columns: one copy, rotation (bits 4-6) = lane & 7)
  const uint32_t lanebits = kRotCopies == 2 ? static_cast<uint32_t>((((tid >> 2) & 1) << 6) | ((tid & 3) << 4))
                                            : static_cast<uint32_t>((tid & 7) << 4);
  const int64_t p = static_cast<int64_t>(tile) * kPoints + tid;
  const bool valid = p < n;
#ifdef DDSG_SLOT_DEBUG_SAMEX
  // measurement only (wrong results): every tile reads tile 0's coordinates,
  // so the kernel's DRAM reads are its staged tables alone
  const int64_t pc = tid < n ? tid : n - 1;
#else
  const int64_t pc = valid ? p : n - 1;
#endif
  const int64_t* offs = block_off + static_cast<int64_t>(cb) * n_active;
  const int32_t* lens = block_len + static_cast<int64_t>(cb) * n_active;

  if (tid == 0) {
    for (int s = 0; s < n_stages; ++s) {
      mbar_init(&bars[s], 1);
      mbar_init(&empty[s], kWarps);
    }
    fence_mbar_init();
    for (int s = 0; s < n_stages && s < n_active; ++s) {
      mbar_expect_tx(&bars[s], static_cast<uint32_t>(lens[s]));
      bulk_g2s(stages + s * stage_bytes, blocks + offs[s], static_cast<uint32_t>(lens[s]), &bars[s]);
    }
  }
  if (use_tmem && warp == 0) tmem_alloc(tmem_slot, 512);
  for (int i = tid; i < kSlotDims * n_active; i += kPoints) sdims[i] = slot_dims[i];
  tmem_fence_before();
  __syncthreads();
  tmem_fence_after();
  TreeStore store{deep, 0u, tid};
  if (use_tmem)
    store.tbase = *tmem_slot + (static_cast<uint32_t>(32 * (warp & 3)) << 16) + static_cast<uint32_t>(kTmemCols * (warp >> 2));

  // coordinates of the slot's dims (dims table [block][3]: an absent second
  // dim reads dim 0, unused; the third is -1 unless the block is order 3)
  auto coord = [&](int a, int j) {
    if (DDSG_SLOT_L2HINT & 1) return ldg_x(xt + static_cast<int64_t>(sdims[kSlotDims * a + j]) * n + pc);
    return xt[static_cast<int64_t>(sdims[kSlotDims * a + j]) * n + pc];
  };
  double xc0 = coord(0, 0), xc1 = coord(0, 1), xc2 = 0.5;
  if (kOrder3 && sdims[2] >= 0) xc2 = coord(0, 2);
  const int c0 = cb * kCols;

  // ring position of block a (st) with its phase parity, advanced
  // incrementally (no runtime division per block)
  int st = 0, pst = n_stages - 1;
  uint32_t ph = 0, pph = 1;
  for (int a = 0; a < n_active; ++a) {
    if (tid == 0 && a >= 1 && a - 1 + n_stages < n_active) {
      // refill the stage released by block a-1 (all warps arrived on its empty barrier)
      const int nxt = a - 1 + n_stages;
      mbar_wait(&empty[pst], pph);
      fence_proxy_async();
      mbar_expect_tx(&bars[pst], static_cast<uint32_t>(lens[nxt]));
      bulk_g2s(stages + pst * stage_bytes, blocks + offs[nxt], static_cast<uint32_t>(lens[nxt]), &bars[pst]);
    }
    mbar_wait(&bars[st], ph);
    const unsigned char* blk = stages + st * stage_bytes;
    const SlotHeader& H = *reinterpret_cast<const SlotHeader*>(blk);
    const HeaderCore Hc = load_core(blk);
    double acc[kCols];
    if (kCarry && (Hc.b_kind & kBCont)) {  // a later stored-order run of the same slot: resume its sum
      const double2* cs = carry + tid;
#pragma unroll
      for (int q = 0; q < kCols / 2; ++q) {
        const double2 v = cs[q * kPoints];
        acc[2 * q] = v.x;
        acc[2 * q + 1] = v.y;
      }
    } else {
#pragma unroll
      for (int c = 0; c < kCols; ++c) acc[c] = 0.0;
    }
    const int k = Hc.k;
    const double x0 = xc0, x1 = xc1, x2 = xc2;
    if (a + 1 < n_active) {  // prefetch the next block's coordinates
      xc0 = coord(a + 1, 0);
      xc1 = coord(a + 1, 1);
      if (kOrder3 && sdims[kSlotDims * (a + 1) + 2] >= 0) xc2 = coord(a + 1, 2);  // order-3 blocks (warp-uniform)
    }
    bool leaf_done = true;
    if (k == 0) {
      const double* r0 = reinterpret_cast<const double*>(blk + Hc.table_off);
#pragma unroll
      for (int c = 0; c < kCols; ++c) acc[c] = r0[c];
    } else {
      leaf_dispatch<kExact, kOrder3>(Hc, H, blk, x0, x1, x2, acc, lanebits);
      if (kCarry && (Hc.b_kind & kBMore)) {  // more runs of this slot follow: park the partial sum
        double2* cs = carry + tid;
#pragma unroll
        for (int q = 0; q < kCols / 2; ++q) cs[q * kPoints] = make_double2(acc[2 * q], acc[2 * q + 1]);
        leaf_done = false;
      } else if ((Hc.b_kind & 3) == 0) {
        const double b = Hc.b;
#pragma unroll
        for (int c = 0; c < kCols; ++c) acc[c] = __dmul_rn(acc[c], b);
      } else if ((Hc.b_kind & 3) == 2) {
#pragma unroll
        for (int c = 0; c < kCols; ++c) acc[c] = -acc[c];
      }
    }
    // pairwise tree (perfect-tree embedding): merge with the pending left
    // siblings at levels s.. while the position bit is set, then park.
    const int t = Hc.tree_t;
    int i = Hc.tree_s;
    if (!kCarry || leaf_done) {
      while (i < levels && ((t >> i) & 1)) {
        double v[kCols];
        store.load(i, v);
#pragma unroll
        for (int c = 0; c < kCols; ++c) acc[c] = __dadd_rn(v[c], acc[c]);
        ++i;
      }
      if (i < levels) {
        store.store(i, acc);
      } else if (valid) {  // the root: written out directly (keeps no registers live)
        double* yp = y + p * m + c0;
#pragma unroll
        for (int c = 0; c < kCols; ++c)
          if (c0 + c < m) {
            if (DDSG_SLOT_L2HINT & 2)
              stg_y(yp + c, acc[c]);
            else
              yp[c] = acc[c];
          }
      }
    }
    __syncwarp();  // every lane of this warp is done reading stage st
    if ((tid & 31) == 0) mbar_arrive(&empty[st]);  // this warp is done with stage st
    pst = st;
    pph = ph;
    if (++st == n_stages) {
      st = 0;
      ph ^= 1u;
    }
  }
  if (use_tmem) {
    tmem_fence_before();
    __syncthreads();
    tmem_fence_after();
    if (warp == 0) tmem_dealloc(*tmem_slot, 512);
  }
}


struct KernelArgs {
  const unsigned char* blocks;
  const int64_t* block_off;
  const int32_t* block_len;
  const int16_t* slot_dims;
  int n_blocks, n_cb, cb_group, levels;
  const double* xt;
  int64_t n;
  int m;
  double* y;
  int64_t stage_bytes;
  int n_stages;
};

#define DDSG_FAST_INSTANCE(E, C, O)                                                                       \
  void fast_launch_##E##C##O(dim3 grid, size_t smem, cudaStream_t st, const KernelArgs& a) {             \
    fast_hdmr_kernel<E, C, O><<<grid, kPoints, smem, st>>>(a.blocks, a.block_off, a.block_len, a.slot_dims, \
                                                           a.n_blocks, a.n_cb, a.cb_group, a.levels, a.xt,   \
                                                           a.n, a.m, a.y, a.stage_bytes, a.n_stages);        \
  }                                                                                                       \
  cudaError_t fast_attr_##E##C##O(int smem) {                                                             \
    ensure_dynamic_smem(reinterpret_cast<const void*>(fast_hdmr_kernel<E, C, O>), static_cast<size_t>(smem)); \
    return cudaSuccess;                                                                                   \
  }

// Instances: EXACT / FAST x with / without the multi-run carry x with /
// without order-3 slots (programs without them keep the leaner code).
#define DDSG_FAST_DECL(E, C, O) \
  void fast_launch_##E##C##O(dim3, size_t, cudaStream_t, const KernelArgs&); \
  cudaError_t fast_attr_##E##C##O(int);
DDSG_FAST_DECL(0, 0, 0) DDSG_FAST_DECL(0, 0, 1) DDSG_FAST_DECL(0, 1, 0) DDSG_FAST_DECL(0, 1, 1)
DDSG_FAST_DECL(1, 0, 0) DDSG_FAST_DECL(1, 0, 1) DDSG_FAST_DECL(1, 1, 0) DDSG_FAST_DECL(1, 1, 1)
#undef DDSG_FAST_DECL

}  // namespace fast
}  // namespace ddsg_b200
