// Plain-grid evaluation kernel (BASELINE configs 1-3): one thread per point
// and up to kMC output columns, walking the grid's subspaces in canonical
// order (per stored-order run) with incremental prefix products.
//
// Point order: for d >= 5 and batches of >= 4096 points the points are first
// put in Morton order (key_kernel + a CUB radix sort of (key, index) pairs)
// and thread p evaluates point perm[p] (reads its x row, writes its y row).
// The 32 points of a warp then lie in a small box, so at every level they
// share cells and the surplus-row gathers hit fewer L1 sectors (config 2
// 23.4 -> 19.8 ms, config 3 72 -> 61 ms at 2^20 / 2^18 points).  Every point
// is still evaluated by the same per-point code: results are bit-identical.
//
// The reference's node weight is the dim-ordered product
// w = ((1 * v_0) * v_1) * ... (sparse_grid.hpp:116-122): its partial products
// are exactly prefix products, so for consecutive subspaces l, l' whose level
// vectors first differ at dim q only the suffix q..d-1 is recomputed (3.7
// factors per subspace on average for config 2, 6.0 for config 3), entered
// by a warp-uniform jump at q.  The 1-d factors are recomputed in registers:
// the candidate cell from a 31-bit fixed-point copy of x (one shift), the
// value as v = fl(A - |fl(x 2^l - B)|) (basis.cuh's exact restatement, the
// boundary mode a template parameter).  The next term's cell, weight and row
// are computed while the current term's surplus row is in flight (address
// software pipelining); surplus rows are gathered through L1 (95-98 % hits
// on config 2) with 16-byte loads.  Terms the reference skips (w == 0, an
// absent node, a node of another stored-order run) read an all-zero row
// instead: the accumulator is never -0, so adding w * 0 leaves its bits
// unchanged, and non-finite surpluses are never multiplied by 0.  Rounding is
// bit-identical to the reference (EXACT: separate mul and add per term).
#include <cuda_runtime.h>

#include <algorithm>
#include <climits>
#include <cstdlib>
#include <cub/device/device_radix_sort.cuh>

#include "basis.cuh"
#include "plain.cuh"

namespace ddsg_b200 {

namespace plain {

// One 32-byte record per subspace, read with two warp-uniform 16-byte loads:
//   w[0] = first row (full subspace) or slab offset (partial)
//   w[1] = q (first dim to recompute) | full << 8
//   w[2..7] = levels as 4-bit nibbles, dim j in word 2 + j/8, bits 4*(j%8)

struct Params {
  int d, m, runs;
  const int* run_off;  // device array: run r walks records [run_off[r], run_off[r+1])
  const uint4* rec;        // [records][2]: per run, the subspaces holding nodes of that run
  const uint32_t* perm;    // thread p evaluates point perm[p] (Morton order), or p when null
  const int32_t* slab;     // [runs][slab_len]: cell -> row of that stored-order run, or -1
  int64_t slab_len;
  const double* surplus;   // [rows + 1][ms] (ms = m rounded up to even: 16-byte rows); row `zero_row` = 0
  int ms;
  int zero_row;
};

// Opaque to the compiler: the record words stay in ordinary registers up to
// this point (see the walk loops).
__device__ __forceinline__ void pin_record(uint4& r) {
  asm volatile("" : "+r"(r.x), "+r"(r.y), "+r"(r.z), "+r"(r.w));
}

template <int kDMax, int kMC, int kExact, int kMode, int kMultiRun>
__global__ void __launch_bounds__(kThreads, (kMC <= 12 && kDMax <= 10) ? 4 : 1) plain_kernel(Params P, const double* __restrict__ x, int64_t n,
                                                         int64_t base, double* __restrict__ y,
                                                         unsigned long long* bad) {
  const int tid = threadIdx.x;
  const int64_t t = static_cast<int64_t>(blockIdx.x) * kThreads + tid;
  const bool valid = t < n;
  const int64_t p = valid && P.perm ? static_cast<int64_t>(P.perm[t]) : t;  // the point this thread evaluates
  const int d = P.d;
  // dims d..kDMax-1 are padding: x = 1/2 at level 1 gives the factor 1 and
  // cell 0 in both modes, so the prefix product and cell index pass through
  double xr[kDMax];
  uint32_t xi[kDMax];
  bool ok = valid;
#pragma unroll
  for (int j = 0; j < kDMax; ++j) {
    xr[j] = 0.5;
    xi[j] = 0x40000000u;
    if (j < d) {
      const double xv = valid ? x[p * d + j] : 0.5;
      ok &= (xv >= 0.0 && xv <= 1.0);
      xr[j] = xv;
      xi[j] = ok ? min(static_cast<uint32_t>(__dmul_rn(xv, 2147483648.0)), 0x7fffffffu) : 0u;  // factor(): clamped
    }
  }
  if (valid && !ok) atomicMin(bad, static_cast<unsigned long long>(base + p));
  if (!valid || !ok) return;

  for (int c0 = 0; c0 < P.m; c0 += kMC) {
    double acc[kMC];
#pragma unroll
    for (int c = 0; c < kMC; ++c) acc[c] = 0.0;
    for (int run = 0; run < (kMultiRun ? P.runs : 1); ++run) {
      const int32_t* slab_run = P.slab + (kMultiRun ? run * P.slab_len : 0);
      // sparse_grid.hpp:123: w == 0 terms and absent nodes add nothing (zero row)
      auto resolve_row = [&](double w, int r) { return (w != 0.0 && r >= 0) ? r : P.zero_row; };
      double pw[kDMax];
      uint32_t pc[kDMax];
#pragma unroll
      for (int j = 0; j < kDMax; ++j) {
        pw[j] = 0.0;
        pc[j] = 0u;
      }
      // weight and surplus row of the subspace with record (r0, r1); the
      // zero row for skipped terms
      auto term = [&](const uint4& r0, const uint4& r1, double& w, int& row) {
        const uint32_t lw[6] = {r0.z, r0.w, r1.x, r1.y, r1.z, r1.w};
        // recompute the suffix q..kDMax-1: jump in at q (warp-uniform), fall through
        switch (static_cast<int>(r0.y & 0xffu)) {
#define DDSG_DIM(J)                                                                            \
  case J:                                                                                      \
    if ((J) < kDMax) {                                                                         \
      constexpr int jj = (J) < kDMax ? (J) : 0;                                                \
      constexpr int jp = (J) > 0 && (J) <= kDMax ? (J) - 1 : 0;                                \
      const int l = static_cast<int>((lw[jj / 8] >> (4 * (jj % 8))) & 15u);                   \
      uint32_t kk;                                                                             \
      double v;                                                                                \
      factor<kMode>(xr[jj], xi[jj], l, kk, v);                                                 \
      if ((J) == 0) {                                                                          \
        pw[0] = v; /* fl(1 * v_0) */                                                           \
        pc[0] = kk;                                                                            \
      } else {                                                                                 \
        pw[jj] = __dmul_rn(pw[jp], v);                                                         \
        pc[jj] = (pc[jp] << (l - 1)) | kk;                                                     \
      }                                                                                        \
    }                                                                                          \
    [[fallthrough]];
          DDSG_DIM(0) DDSG_DIM(1) DDSG_DIM(2) DDSG_DIM(3) DDSG_DIM(4) DDSG_DIM(5) DDSG_DIM(6) DDSG_DIM(7)
          DDSG_DIM(8) DDSG_DIM(9) DDSG_DIM(10) DDSG_DIM(11) DDSG_DIM(12) DDSG_DIM(13) DDSG_DIM(14)
          DDSG_DIM(15) DDSG_DIM(16) DDSG_DIM(17) DDSG_DIM(18) DDSG_DIM(19)
#undef DDSG_DIM
          default:
            break;
        }
        w = pw[kDMax - 1];
        // full subspace: its row; otherwise this run's slab entry (-1: no
        // node of the run), resolved by resolve_row() after the current
        // term's multiply-adds so the lookup's latency is covered
        row = static_cast<int>(r0.x) + static_cast<int>(pc[kDMax - 1]);
        if (!((r0.y >> 8) & 1u)) row = __ldg(slab_run + row);
      };
      const uint4 zero4 = make_uint4(0u, 0u, 0u, 0u);
      const int off0 = __ldg(P.run_off + run), off1 = __ldg(P.run_off + run + 1);
      const uint4* rec = P.rec + 2 * off0;
      const int n_sub = off1 - off0;
      if (n_sub == 0) continue;

      // subspace records are prefetched one iteration ahead of their use
      uint4 ra = __ldg(rec), rb = kDMax > 16 ? __ldg(rec + 1) : zero4;
      double w_cur;
      int row_cur;
      term(ra, rb, w_cur, row_cur);
      row_cur = resolve_row(w_cur, row_cur);
      if (n_sub > 1) {
        ra = __ldg(rec + 2);
        rb = kDMax > 16 ? __ldg(rec + 3) : zero4;
      }
      for (int s = 0; s < n_sub; ++s) {
        // issue this term's row loads, compute the next term while they fly
        double sv[kMC];
        const double* sr = P.surplus + static_cast<int64_t>(row_cur) * P.ms + c0;
        if (kMC == 1) {
          sv[0] = __ldg(sr);
        } else {
          // rows are padded to whole chunks and 32-byte aligned: one 256-bit
          // load (LDG.E.256) per 4 columns, a whole L1 sector per request
#pragma unroll
          for (int c = 0; c < kMC; c += 4)
            asm("ld.global.nc.v4.f64 {%0,%1,%2,%3}, [%4];"
                : "=d"(sv[c]), "=d"(sv[c + 1]), "=d"(sv[c + 2]), "=d"(sv[c + 3])
                : "l"(sr + c));
        }
        // the record loaded one iteration ago: the empty asm keeps it in
        // ordinary registers until here (otherwise the compiler moves it to
        // uniform registers right after its load and the warp waits out the
        // load latency there -- 18 % of all stall samples on config 2)
        pin_record(ra);
        if (kDMax > 16) pin_record(rb);
        const uint4 ua = ra, ub = rb;
        {  // unconditional (clamped) prefetch: a conditional one is merged through uniform registers
          const int nx = min(s + 2, n_sub - 1);
          ra = __ldg(rec + 2 * nx);
          if (kDMax > 16) rb = __ldg(rec + 2 * nx + 1);
        }
        double w_nxt = 0.0;
        int row_nxt = P.zero_row;
        if (s + 1 < n_sub) term(ua, ub, w_nxt, row_nxt);
#pragma unroll
        for (int c = 0; c < kMC; ++c)
          acc[c] = kExact ? __dadd_rn(acc[c], __dmul_rn(w_cur, sv[c])) : __fma_rn(w_cur, sv[c], acc[c]);
        row_cur = resolve_row(w_nxt, row_nxt);  // after the multiply-adds: the slab lookup's latency is covered
        w_cur = w_nxt;
      }
    }
    const int nc = min(kMC, P.m - c0);
    double* yp = y + p * P.m + c0;
#pragma unroll
    for (int c = 0; c < kMC; ++c)
      if (c < nc) yp[c] = acc[c];
  }
}


// ---------------------------------------------------------------------------
// Term-parallel form for small single-output grids (config 1: d = 4, 70
// subspaces, m = 1).  plain_kernel walks a point's subspaces serially, so a
// batch that fills less than a few waves is bound by that chain's latency
// (65,536 points: 33 us for 9 MFLOP).  Here a CTA of kWarps warps takes 32
// points (lane = point; 16 warps up to 8,192 points, where the kernel is one
// latency-bound wave, 8 beyond) and warp w computes the products
// fl(w_s * s_row) of the subspaces s = w, w + kWarps, ... from scratch (the full dim-ordered weight
// product, same factor() and the same zero row for skipped terms) into shared
// memory; warp 0 then adds them in canonical order, acc = fl(acc + prod_s):
// the reference's operation sequence per point (sparse_grid.hpp:116-126), so
// the result is bit-identical to plain_kernel's EXACT mode (FAST keeps w_s
// and s_row apart and chains one DFMA per term, as plain_kernel's FAST mode
// does).  More instructions per term (no prefix reuse), so it only serves
// batches up to kTermsMaxPoints.
constexpr int kTermsMaxSub = 192;              // 48 KB of products per CTA (FAST keeps weight and surplus: half as many)
constexpr int64_t kTermsMaxPoints = 1 << 16;   // beyond: plain_kernel's prefix reuse wins (crossover just below 2^17 on config 1)

template <int kDMax, int kMode, int kWarps, int kExact>
__global__ void __launch_bounds__(kWarps * 32) plain_terms_kernel(Params P, const double* __restrict__ x,
                                                                       int64_t n, int64_t base,
                                                                       double* __restrict__ y,
                                                                       unsigned long long* bad, int n_sub) {
  extern __shared__ double prod[];  // EXACT: products [n_sub][32]; FAST: weights, then surpluses [2][n_sub][32]
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int64_t p = static_cast<int64_t>(blockIdx.x) * 32 + lane;
  const bool valid = p < n;
  const int d = P.d;
  double xr[kDMax];
  uint32_t xi[kDMax];
  bool ok = valid;
#pragma unroll
  for (int j = 0; j < kDMax; ++j) {
    xr[j] = 0.5;  // padding dims: level 1 at x = 1/2, factor 1 and cell 0
    if (j < d && valid) {
      const double xv = x[p * d + j];
      ok &= (xv >= 0.0 && xv <= 1.0);
      xr[j] = xv;
    }
  }
#pragma unroll
  for (int j = 0; j < kDMax; ++j) {
    if (!ok) xr[j] = 0.5;  // keeps every index in range; nothing of this point is written
    xi[j] = min(static_cast<uint32_t>(__dmul_rn(xr[j], 2147483648.0)), 0x7fffffffu);
  }
  if (warp == 0 && valid && !ok) atomicMin(bad, static_cast<unsigned long long>(base + p));
  const uint4* rec = P.rec + 2 * __ldg(P.run_off);
#pragma unroll 2
  for (int s = warp; s < n_sub; s += kWarps) {
    const uint4 r0 = __ldg(rec + 2 * s);
    const uint32_t lw[2] = {r0.z, r0.w};
    double w = 0.0;
    uint32_t pc = 0u;
#pragma unroll
    for (int j = 0; j < kDMax; ++j) {
      const int l = static_cast<int>((lw[j / 8] >> (4 * (j % 8))) & 15u);
      uint32_t kk;
      double v;
      factor<kMode>(xr[j], xi[j], l, kk, v);
      w = j == 0 ? v : __dmul_rn(w, v);  // ((1 * v_0) * v_1) * ...
      pc = j == 0 ? kk : ((pc << (l - 1)) | kk);
    }
    int row = static_cast<int>(r0.x) + static_cast<int>(pc);
    if (!((r0.y >> 8) & 1u)) row = __ldg(P.slab + row);
    row = (w != 0.0 && row >= 0) ? row : P.zero_row;  // sparse_grid.hpp:123
    const double sv = __ldg(P.surplus + static_cast<int64_t>(row) * P.ms);
    if (kExact) {
      prod[s * 32 + lane] = __dmul_rn(w, sv);
    } else {
      prod[s * 32 + lane] = w;
      prod[(n_sub + s) * 32 + lane] = sv;
    }
  }
  __syncthreads();
  if (warp == 0 && valid && ok) {
    double acc = 0.0;
#pragma unroll 8
    for (int s = 0; s < n_sub; ++s)
      acc = kExact ? __dadd_rn(acc, prod[s * 32 + lane])
                   : __fma_rn(prod[s * 32 + lane], prod[(n_sub + s) * 32 + lane], acc);  // FAST: one DFMA per term
    y[p * P.m] = acc;
  }
}

template <int kDMax, int kWarps, int kExact>
static void launch_terms_w(int mode, const Params& P, const double* x, int64_t n, int64_t base, double* y,
                           unsigned long long* bad, int n_sub, cudaStream_t st) {
  const unsigned grid = static_cast<unsigned>((n + 31) / 32);
  const size_t smem = static_cast<size_t>(n_sub) * 32 * sizeof(double) * (kExact ? 1 : 2);
  if (mode == 1)
    plain_terms_kernel<kDMax, 1, kWarps, kExact><<<grid, kWarps * 32, smem, st>>>(P, x, n, base, y, bad, n_sub);
  else
    plain_terms_kernel<kDMax, 0, kWarps, kExact><<<grid, kWarps * 32, smem, st>>>(P, x, n, base, y, bad, n_sub);
}

template <int kDMax>
static void launch_terms(int mode, int exact, const Params& P, const double* x, int64_t n, int64_t base, double* y,
                         unsigned long long* bad, int n_sub, cudaStream_t st) {
  if (n <= 8192)
    exact ? launch_terms_w<kDMax, 16, 1>(mode, P, x, n, base, y, bad, n_sub, st)
          : launch_terms_w<kDMax, 16, 0>(mode, P, x, n, base, y, bad, n_sub, st);
  else
    exact ? launch_terms_w<kDMax, 8, 1>(mode, P, x, n, base, y, bad, n_sub, st)
          : launch_terms_w<kDMax, 8, 0>(mode, P, x, n, base, y, bad, n_sub, st);
}

// ---------------------------------------------------------------------------
// Sparse walk for modified-linear grids (config 3).  There the level-1 factor
// is exactly 1 (basis.hpp:40), so the reference's dim-ordered product
// w = ((1 * v_0) * v_1) * ... equals the product over the dims with l_j > 1
// only, in dim order (multiplying by 1.0 is exact), and level-1 dims add no
// bits to the cell index.  A subspace record then lists its <= kSparseNT
// non-trivial (dim, level) pairs; the prefix caches hold kSparseNT entries
// instead of d, and the coordinates live in shared memory (dim-major: a warp
// reading one dim hits 32 consecutive words), which frees the registers that
// held d-wide arrays: config 3 (d = 20, at most 4 non-trivial dims) runs at
// a multiple of the occupancy of plain_kernel.
constexpr int kSparseNT = 8;
constexpr int kSparseThreads = 128;

// record: x = first row (full) or slab offset; y = qs | nt << 4 | full << 8
// (qs: pairs reused from the previous record of the run, < nt unless nt = 0);
// z, w, [1].x, [1].y: pair k in 16 bits of word k / 2 (dim | level << 8)
struct SparseParams {
  int d, m, runs, ms, zero_row;
  const int* run_off;  // device array (a dynamic index into a parameter array would copy it to local memory)
  const uint4* rec;
  const uint32_t* perm;
  const int32_t* slab;  // [runs][slab_len], as in Params
  int64_t slab_len;
  const double* surplus;
};

template <int kMC, int kExact, int kMultiRun>
__global__ void __launch_bounds__(kSparseThreads, kMC % 8 == 0 ? 4 : 1) sparse_kernel(SparseParams P, const double* __restrict__ x,
                                                                int64_t n, int64_t base, double* __restrict__ y,
                                                                unsigned long long* bad) {
  extern __shared__ double xs[];  // [d][kSparseThreads] coordinates, then [d][kSparseThreads] fixed point
  const int tid = threadIdx.x;
  const int d = P.d;
  uint32_t* xis = reinterpret_cast<uint32_t*>(xs + d * kSparseThreads);
  const int64_t t = static_cast<int64_t>(blockIdx.x) * kSparseThreads + tid;
  const bool valid = t < n;
  const int64_t p = valid && P.perm ? static_cast<int64_t>(P.perm[t]) : t;
  bool ok = valid;
  for (int j = 0; j < d; ++j) {
    const double xv = valid ? x[p * d + j] : 0.5;
    ok &= (xv >= 0.0 && xv <= 1.0);
    xs[j * kSparseThreads + tid] = xv;
    xis[j * kSparseThreads + tid] = ok ? min(static_cast<uint32_t>(__dmul_rn(xv, 2147483648.0)), 0x7fffffffu) : 0u;
  }
  if (valid && !ok) atomicMin(bad, static_cast<unsigned long long>(base + p));
  if (!valid || !ok) return;  // each thread reads only its own coordinates: no barrier

  for (int c0 = 0; c0 < P.m; c0 += kMC) {
    double acc[kMC];
#pragma unroll
    for (int c = 0; c < kMC; ++c) acc[c] = 0.0;
    for (int run = 0; run < (kMultiRun ? P.runs : 1); ++run) {
      const int32_t* slab_run = P.slab + (kMultiRun ? run * P.slab_len : 0);
      // sparse_grid.hpp:123: w == 0 terms and absent nodes add nothing (zero row)
      auto resolve_row = [&](double w, int r) { return (w != 0.0 && r >= 0) ? r : P.zero_row; };
      double pw[kSparseNT];
      uint32_t pc[kSparseNT];
#pragma unroll
      for (int k = 0; k < kSparseNT; ++k) {
        pw[k] = 1.0;
        pc[k] = 0u;
      }
      auto term = [&](const uint4& r0, const uint4& r1, double& w, int& row) {
        const uint32_t pairw[4] = {r0.z, r0.w, r1.x, r1.y};  // pair k: 16 bits of word k / 2
        const int nt = static_cast<int>((r0.y >> 4) & 15u);
        w = 1.0;
        uint32_t cell = 0u;
        switch (static_cast<int>(r0.y & 15u)) {
#define DDSG_SDIM(K)                                                                           \
  case K: {                                                                                    \
    if ((K) >= nt) break;                                                                      \
    const uint32_t pr = (pairw[(K) / 2] >> (16 * ((K) & 1))) & 0xffffu;                       \
    const int dim = static_cast<int>(pr & 0xffu), l = static_cast<int>(pr >> 8);              \
    uint32_t kk;                                                                               \
    double v;                                                                                  \
    factor<1>(xs[dim * kSparseThreads + tid], xis[dim * kSparseThreads + tid], l, kk, v);      \
    if ((K) == 0) {                                                                            \
      pw[0] = v;                                                                               \
      pc[0] = kk;                                                                              \
    } else {                                                                                   \
      constexpr int kp = (K) > 0 ? (K) - 1 : 0;                                                \
      pw[K] = __dmul_rn(pw[kp], v);                                                            \
      pc[K] = (pc[kp] << (l - 1)) | kk;                                                        \
    }                                                                                          \
    if ((K) == nt - 1) {                                                                       \
      w = pw[K];                                                                               \
      cell = pc[K];                                                                            \
    }                                                                                          \
  }                                                                                            \
    [[fallthrough]];
          DDSG_SDIM(0) DDSG_SDIM(1) DDSG_SDIM(2) DDSG_SDIM(3) DDSG_SDIM(4) DDSG_SDIM(5) DDSG_SDIM(6) DDSG_SDIM(7)
#undef DDSG_SDIM
          default:
            break;
        }
        row = static_cast<int>(r0.x) + static_cast<int>(cell);  // see plain_kernel
        if (!((r0.y >> 8) & 1u)) row = __ldg(slab_run + row);
      };
      const int off0 = __ldg(P.run_off + run), off1 = __ldg(P.run_off + run + 1);
      const uint4* rec = P.rec + 2 * off0;
      const int n_sub = off1 - off0;
      if (n_sub == 0) continue;

      uint4 ra = __ldg(rec), rb = __ldg(rec + 1);
      double w_cur;
      int row_cur;
      term(ra, rb, w_cur, row_cur);
      row_cur = resolve_row(w_cur, row_cur);
      if (n_sub > 1) {
        ra = __ldg(rec + 2);
        rb = __ldg(rec + 3);
      }
      // The row is loaded in two halves: the first flies while the next
      // term's weight is formed, the second after the first half is
      // accumulated, so only half a row of registers is in flight (config 3:
      // 24 columns, 128 registers, 16 warps per SM instead of 12).
      constexpr int kH = kMC % 8 == 0 ? kMC / 2 : kMC;  // halves of whole 32-byte loads, else no split
      auto load_half = [&](const double* sr, double (&sv)[kH]) {
#pragma unroll
        for (int c = 0; c < kH; c += 4)
          asm("ld.global.nc.v4.f64 {%0,%1,%2,%3}, [%4];"
              : "=d"(sv[c]), "=d"(sv[c + 1]), "=d"(sv[c + 2]), "=d"(sv[c + 3])
              : "l"(sr + c));
      };
      for (int s = 0; s < n_sub; ++s) {
        double sv[kH];
        const double* sr = P.surplus + static_cast<int64_t>(row_cur) * P.ms + c0;
        load_half(sr, sv);
        pin_record(ra);  // see plain_kernel
        pin_record(rb);
        const uint4 ua = ra, ub = rb;
        {  // unconditional (clamped) prefetch, see plain_kernel
          const int nx = min(s + 2, n_sub - 1);
          ra = __ldg(rec + 2 * nx);
          rb = __ldg(rec + 2 * nx + 1);
        }
        double w_nxt = 0.0;
        int row_nxt = P.zero_row;
        if (s + 1 < n_sub) term(ua, ub, w_nxt, row_nxt);
#pragma unroll
        for (int c = 0; c < kH; ++c)
          acc[c] = kExact ? __dadd_rn(acc[c], __dmul_rn(w_cur, sv[c])) : __fma_rn(w_cur, sv[c], acc[c]);
        if (kH < kMC) load_half(sr + (kH < kMC ? kH : 0), sv);
        row_cur = resolve_row(w_nxt, row_nxt);  // after the multiply-adds: the slab lookup's latency is covered
        if (kH < kMC) {
#pragma unroll
          for (int c = 0; c < kH; ++c) {
            constexpr int kOff = kH < kMC ? kH : 0;
            acc[kOff + c] =
                kExact ? __dadd_rn(acc[kOff + c], __dmul_rn(w_cur, sv[c])) : __fma_rn(w_cur, sv[c], acc[kOff + c]);
          }
        }
        w_cur = w_nxt;
      }
    }
    const int nc = min(kMC, P.m - c0);
    double* yp = y + p * P.m + c0;
#pragma unroll
    for (int c = 0; c < kMC; ++c)
      if (c < nc) yp[c] = acc[c];
  }
}

}  // namespace plain

using namespace plain;

PlainGrid::~PlainGrid() {
  for (void* p : allocs_) cudaFree(p);
}

template <typename T>
const T* PlainGrid::put(const std::vector<T>& v) {
  if (v.empty()) return nullptr;
  void* p = nullptr;
  DDSG_CUDA(cudaMalloc(&p, v.size() * sizeof(T)));
  allocs_.push_back(p);
  DDSG_CUDA(cudaMemcpy(p, v.data(), v.size() * sizeof(T), cudaMemcpyHostToDevice));
  return static_cast<const T*>(p);
}

// Output columns per thread (one chunk when possible: every further chunk
// repeats the whole subspace walk; config 3 measured 0.19 / 0.25 / 0.44
// TFLOP/s for chunks of 8 / 12 / 24).
static int chunk_width(int d, int m) {
  if (m <= 1) return 1;
  if (d <= 4) return m <= 12 ? 12 : 24;
  if (d <= 10) return 12;
  return 24;
}

bool PlainGrid::build(const HostProgram& hp, const EvalParams& dev) {
  usable_ = false;
  if (!hp.plain || hp.slot_k.size() != 1) return false;
  const int d = hp.d;
  // the dense walk takes d <= 20; modified-linear grids up to kSparseMaxDim
  // dims can still take the sparse walk (build_sparse decides)
  const bool dense_ok = d <= kMaxDim;
  if (!dense_ok && !(hp.slot_mode[0] == 1 && d <= kSparseMaxDim && hp.m > 1)) return false;
  const int s0 = hp.slot_sub_begin[0], s1 = hp.slot_sub_end[0];
  const int n_sub = s1 - s0;
  if (n_sub == 0) return false;
  int lmax = 1;
  int64_t max_bits = 0;  // bits of the concatenated cell index (a uint32 in the kernels)
  for (int s = s0; s < s1; ++s) {
    int64_t bits = 0;
    for (int j = 0; j < d; ++j) {
      lmax = std::max<int>(lmax, hp.levels[hp.sub_lv_off[s] + j]);
      bits += hp.levels[hp.sub_lv_off[s] + j] - 1;
    }
    max_bits = std::max(max_bits, bits);
  }
  if (lmax > 15 || max_bits > 31) return false;  // 4-bit level nibbles, 32-bit cell index
  // Per stored-order run, the subspaces that hold at least one node of the
  // run, in canonical order (a run's walk skips the others: config 3's two
  // runs touch 1,771 and 9,995 of its 10,626 subspaces).
  const int runs = hp.slot_runs[0];
  if (runs > kMaxRuns) return false;
  std::vector<uint32_t> rec;
  run_off_.assign(1, 0);
  for (int run = 0; run < (dense_ok ? runs : 0); ++run) {
    const uint8_t* prev = nullptr;
    for (int s = s0; s < s1; ++s) {
      const uint8_t* lv = &hp.levels[hp.sub_lv_off[s]];
      int64_t cells = 1;
      for (int j = 0; j < d; ++j) cells <<= (lv[j] - 1);
      const int64_t slab_off = hp.sub_slab_off[s];
      if (runs > 1) {
        bool has = false;
        for (int64_t c = 0; c < cells && !has; ++c) {
          const int32_t row = hp.slab[slab_off + c];
          has = row >= 0 && hp.row_run[row] == run;
        }
        if (!has) continue;
      }
      int qq = 0;
      if (prev)
        while (qq < d && prev[qq] == lv[qq]) ++qq;
      prev = lv;
      // several stored-order runs: every term goes through the run's slab
      // (a complete subspace may hold nodes of several runs)
      const bool is_full = hp.sub_nodes[s] == cells && runs == 1;
      uint32_t r[8] = {0u, 0u, 0u, 0u, 0u, 0u, 0u, 0u};
      r[0] = static_cast<uint32_t>(is_full ? hp.slab[slab_off] : slab_off);
      r[1] = static_cast<uint32_t>(qq) | (is_full ? 0x100u : 0u);
      for (int j = 0; j < kMaxDim; ++j)  // padding dims: level 1
        r[2 + j / 8] |= static_cast<uint32_t>(j < d ? lv[j] : 1) << (4 * (j % 8));
      rec.insert(rec.end(), r, r + 8);
    }
    run_off_.push_back(static_cast<int>(rec.size() / 8));
  }
  run_off_dev_ = put(run_off_);
  d_ = d;
  m_ = hp.m;
  mode_ = hp.slot_mode[0];
  runs_ = runs;
  rec_ = reinterpret_cast<const uint4*>(put(rec));
  // row-padded copy of the surpluses (rows padded to whole column chunks, so
  // every chunk is read with unguarded 16-byte loads) plus one all-zero row
  // for skipped terms
  mc_ = chunk_width(d, hp.m);
  ms_ = (hp.m + mc_ - 1) / mc_ * mc_;
  zero_row_ = static_cast<int>(hp.rows);
  std::vector<double> pad(static_cast<size_t>(hp.rows + 1) * ms_, 0.0);
  for (int64_t r = 0; r < hp.rows; ++r)
    std::copy(hp.surplus.begin() + r * hp.m, hp.surplus.begin() + (r + 1) * hp.m, pad.begin() + r * ms_);
  surplus_ = put(pad);
  // per-run slabs: run r's copy keeps only the rows of run r (-1 elsewhere),
  // so a term needs one lookup, not a slab and a row_run lookup
  slab_len_ = static_cast<int64_t>(hp.slab.size());
  if (runs == 1) {
    slab_ = dev.slab;
  } else {
    std::vector<int32_t> sr(static_cast<size_t>(slab_len_) * runs);
    for (int run = 0; run < runs; ++run)
      for (int64_t c = 0; c < slab_len_; ++c) {
        const int32_t row = hp.slab[c];
        sr[run * slab_len_ + c] = (row >= 0 && hp.row_run[row] == run) ? row : -1;
      }
    slab_ = put(sr);
  }
  usable_ = true;
  build_sparse(hp);
  if (!dense_ok && !sparse_) {
    usable_ = false;  // the generic kernel takes it
    return false;
  }
  sort_ = d >= kSortMinDim;
  if (const char* e = std::getenv("DDSG_PLAIN_SORT"))
    if (std::atoi(e) == 0) sort_ = false;
  return true;
}

// Sparse-walk records (modified-linear grids, d >= 5, <= kSparseNT dims above
// level 1 per subspace, d <= kSparseMaxDim): same subspaces and order as the
// dense records.
bool PlainGrid::build_sparse(const HostProgram& hp) {
  sparse_ = false;
  const int d = hp.d;
  if (hp.slot_mode[0] != 1 || d < kSortMinDim || d > kSparseMaxDim || hp.m <= 1) return false;
  if (const char* e = std::getenv("DDSG_PLAIN_SPARSE"))
    if (std::atoi(e) == 0) return false;
  const int s0 = hp.slot_sub_begin[0], s1 = hp.slot_sub_end[0];
  const int runs = hp.slot_runs[0];
  std::vector<uint32_t> rec;
  srun_off_.assign(1, 0);
  for (int run = 0; run < runs; ++run) {
    const uint8_t* prev = nullptr;
    for (int s = s0; s < s1; ++s) {
      const uint8_t* lv = &hp.levels[hp.sub_lv_off[s]];
      int64_t cells = 1;
      int nt = 0;
      for (int j = 0; j < d; ++j) {
        cells <<= (lv[j] - 1);
        nt += lv[j] > 1;
      }
      if (nt > kSparseNT) return false;
      const int64_t slab_off = hp.sub_slab_off[s];
      if (runs > 1) {  // the dense walk's run filter
        bool has = false;
        for (int64_t c = 0; c < cells && !has; ++c) {
          const int32_t row = hp.slab[slab_off + c];
          has = row >= 0 && hp.row_run[row] == run;
        }
        if (!has) continue;
      }
      int qq = 0;  // first dim differing from the previous record of the run
      if (prev)
        while (qq < d && prev[qq] == lv[qq]) ++qq;
      prev = lv;
      int qs = 0;  // non-trivial pairs below qq are unchanged
      for (int j = 0; j < qq; ++j) qs += lv[j] > 1;
      if (nt > 0) qs = std::min(qs, nt - 1);  // recompute >= 1 pair: the last one yields w
      const bool is_full = hp.sub_nodes[s] == cells && runs == 1;  // see build()
      uint32_t r[8] = {0u, 0u, 0u, 0u, 0u, 0u, 0u, 0u};
      r[0] = static_cast<uint32_t>(is_full ? hp.slab[slab_off] : slab_off);
      r[1] = static_cast<uint32_t>(qs) | (static_cast<uint32_t>(nt) << 4) | (is_full ? 0x100u : 0u);
      int k = 0;
      for (int j = 0; j < d; ++j)
        if (lv[j] > 1) {
          r[2 + k / 2] |= (static_cast<uint32_t>(j) | (static_cast<uint32_t>(lv[j]) << 8)) << (16 * (k & 1));
          ++k;
        }
      rec.insert(rec.end(), r, r + 8);
    }
    srun_off_.push_back(static_cast<int>(rec.size() / 8));
  }
  srec_ = reinterpret_cast<const uint4*>(put(rec));
  srun_off_dev_ = put(srun_off_);
  smc_ = hp.m <= 12 ? 12 : 24;
  if (const char* e = std::getenv("DDSG_SPARSE_COLS")) smc_ = std::atoi(e) == 24 ? 24 : 12;
  sparse_ = (ms_ % smc_) == 0;
  return sparse_;
}

// Morton key of each point: `bits` bits per dim from the top of floor(x 2^31)
// (clamped to [0, 2^31)), dim 0 most significant within a bit plane.  Points
// outside the domain get some key; plain_kernel reports them.
__global__ void morton_key_kernel(const double* __restrict__ x, int64_t n, int d, int bits,
                                  unsigned long long* __restrict__ key, uint32_t* __restrict__ idx) {
  const int64_t p = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
  if (p >= n) return;
  unsigned long long k = 0ull;
  for (int j = 0; j < d; ++j) {
    const double v = x[p * d + j];
    const uint32_t xi = (v >= 0.0 && v <= 1.0) ? min(static_cast<uint32_t>(__dmul_rn(v, 2147483648.0)), 0x7fffffffu) : 0u;
    for (int b = 0; b < bits; ++b)
      k |= static_cast<unsigned long long>((xi >> (30 - b)) & 1u) << ((bits - 1 - b) * d + (d - 1 - j));
  }
  key[p] = k;
  idx[p] = static_cast<uint32_t>(p);
}

static int morton_bits(int d) { return std::max(1, std::min(16, 40 / d)); }

template <int kMC, int kExact, int kMulti>
static void launch_sparse_t(const SparseParams& S, unsigned grid, size_t smem, const double* x, int64_t n,
                            int64_t base, double* y, unsigned long long* bad, cudaStream_t st) {
  auto k = sparse_kernel<kMC, kExact, kMulti>;
  if (smem > 48 * 1024) ensure_dynamic_smem(reinterpret_cast<const void*>(k), smem);
  k<<<grid, kSparseThreads, smem, st>>>(S, x, n, base, y, bad);
}

static void launch_sparse(int mc, int exact, bool multi, const SparseParams& S, unsigned grid, size_t smem,
                          const double* x, int64_t n, int64_t base, double* y, unsigned long long* bad,
                          cudaStream_t st) {
  if (mc == 24) {
    if (exact)
      multi ? launch_sparse_t<24, 1, 1>(S, grid, smem, x, n, base, y, bad, st)
            : launch_sparse_t<24, 1, 0>(S, grid, smem, x, n, base, y, bad, st);
    else
      multi ? launch_sparse_t<24, 0, 1>(S, grid, smem, x, n, base, y, bad, st)
            : launch_sparse_t<24, 0, 0>(S, grid, smem, x, n, base, y, bad, st);
  } else {
    if (exact)
      multi ? launch_sparse_t<12, 1, 1>(S, grid, smem, x, n, base, y, bad, st)
            : launch_sparse_t<12, 1, 0>(S, grid, smem, x, n, base, y, bad, st);
    else
      multi ? launch_sparse_t<12, 0, 1>(S, grid, smem, x, n, base, y, bad, st)
            : launch_sparse_t<12, 0, 0>(S, grid, smem, x, n, base, y, bad, st);
  }
}

template <int kDMax, int kMC, int kMode, int kMulti>
static void launch_plain(const Params& P, int exact, const double* x, int64_t n, int64_t base, double* y,
                         unsigned long long* bad, cudaStream_t st) {
  const unsigned grid = static_cast<unsigned>((n + kThreads - 1) / kThreads);
  if (exact)
    plain_kernel<kDMax, kMC, 1, kMode, kMulti><<<grid, kThreads, 0, st>>>(P, x, n, base, y, bad);
  else
    plain_kernel<kDMax, kMC, 0, kMode, kMulti><<<grid, kThreads, 0, st>>>(P, x, n, base, y, bad);
}

template <int kDMax, int kMC>
static void launch_mode(int mode, const Params& P, int exact, const double* x, int64_t n, int64_t base, double* y,
                        unsigned long long* bad, cudaStream_t st) {
  const bool multi = P.runs > 1;
  if (mode == 1)
    multi ? launch_plain<kDMax, kMC, 1, 1>(P, exact, x, n, base, y, bad, st)
          : launch_plain<kDMax, kMC, 1, 0>(P, exact, x, n, base, y, bad, st);
  else
    multi ? launch_plain<kDMax, kMC, 0, 1>(P, exact, x, n, base, y, bad, st)
          : launch_plain<kDMax, kMC, 0, 0>(P, exact, x, n, base, y, bad, st);
}

size_t PlainGrid::workspace_bytes(int64_t n) const {
  if (!sort_ || n < kSortMinPoints || n > INT32_MAX) return 0;
  size_t temp = 0;
  cub::DoubleBuffer<unsigned long long> kb(nullptr, nullptr);
  cub::DoubleBuffer<uint32_t> vb(nullptr, nullptr);
  cub::DeviceRadixSort::SortPairs(nullptr, temp, kb, vb, static_cast<int>(n), 0, morton_bits(d_) * d_);
  return (static_cast<size_t>(n) * 24 + temp + 1024 + 255) / 256 * 256;
}

int64_t PlainGrid::launch(int exact, const double* x, int64_t n, int64_t base, double* y,
                          unsigned long long* bad, void* ws, cudaStream_t st) const {
  int64_t launches = 1;
  const uint32_t* perm = nullptr;
  // small single-output grids, batches of a few waves: term-parallel form
  static const bool terms_on = [] {
    const char* e = std::getenv("DDSG_PLAIN_TERMS");
    return !(e && std::atoi(e) == 0);
  }();
  const int n_sub0 = run_off_.size() > 1 ? run_off_[1] - run_off_[0] : 0;
  if (terms_on && !sparse_ && m_ == 1 && runs_ == 1 && d_ <= 10 && n_sub0 > 0 &&
      n_sub0 <= plain::kTermsMaxSub / (exact ? 1 : 2) &&
      n <= plain::kTermsMaxPoints && !(sort_ && n >= kSortMinPoints)) {  // Morton-sorted batches keep the serial walk
    Params P{};
    P.d = d_;
    P.m = m_;
    P.runs = runs_;
    P.run_off = run_off_dev_;
    P.rec = rec_;
    P.slab = slab_;
    P.slab_len = slab_len_;
    P.surplus = surplus_;
    P.ms = ms_;
    P.zero_row = zero_row_;
    kernel_timer().begin(st);
    if (d_ <= 4)
      plain::launch_terms<4>(mode_, exact, P, x, n, base, y, bad, n_sub0, st);
    else
      plain::launch_terms<10>(mode_, exact, P, x, n, base, y, bad, n_sub0, st);
    kernel_timer().end(st);
    DDSG_CUDA(cudaGetLastError());
    return launches;
  }
  if (ws && workspace_bytes(n) > 0) {
    auto* k0 = static_cast<unsigned long long*>(ws);
    auto* k1 = k0 + n;
    auto* v0 = reinterpret_cast<uint32_t*>(k1 + n);
    auto* v1 = v0 + n;
    void* temp = reinterpret_cast<void*>((reinterpret_cast<uintptr_t>(v1 + n) + 255) / 256 * 256);
    const int bits = morton_bits(d_);
    morton_key_kernel<<<static_cast<unsigned>((n + 255) / 256), 256, 0, st>>>(x, n, d_, bits, k0, v0);
    DDSG_CUDA(cudaGetLastError());
    cub::DoubleBuffer<unsigned long long> kb(k0, k1);
    cub::DoubleBuffer<uint32_t> vb(v0, v1);
    size_t temp_bytes = 0;
    cub::DeviceRadixSort::SortPairs(nullptr, temp_bytes, kb, vb, static_cast<int>(n), 0, bits * d_, st);
    DDSG_CUDA(cub::DeviceRadixSort::SortPairs(temp, temp_bytes, kb, vb, static_cast<int>(n), 0, bits * d_, st));
    perm = vb.Current();
    launches = 2;  // key kernel + evaluation kernel (the sort's kernels are CUB's)
  }
  if (sparse_) {
    SparseParams S{};
    S.d = d_;
    S.m = m_;
    S.runs = runs_;
    S.ms = ms_;
    S.zero_row = zero_row_;
    S.run_off = srun_off_dev_;
    S.rec = srec_;
    S.perm = perm;
    S.slab = slab_;
    S.slab_len = slab_len_;
    S.surplus = surplus_;
    const unsigned grid = static_cast<unsigned>((n + kSparseThreads - 1) / kSparseThreads);
    const size_t smem = static_cast<size_t>(d_) * kSparseThreads * 12;
    kernel_timer().begin(st);
    launch_sparse(smc_, exact, runs_ > 1, S, grid, smem, x, n, base, y, bad, st);
    kernel_timer().end(st);
    DDSG_CUDA(cudaGetLastError());
    return launches;
  }
  Params P{};
  P.perm = perm;
  P.d = d_;
  P.m = m_;
  P.runs = runs_;
  P.run_off = run_off_dev_;
  P.rec = rec_;
  P.slab = slab_;
  P.slab_len = slab_len_;
  P.surplus = surplus_;
  P.ms = ms_;
  P.zero_row = zero_row_;
  kernel_timer().begin(st);
  switch (d_ <= 4 ? 400 + mc_ : (d_ <= 10 ? 1000 + mc_ : 2000 + mc_)) {
    case 401: launch_mode<4, 1>(mode_, P, exact, x, n, base, y, bad, st); break;
    case 412: launch_mode<4, 12>(mode_, P, exact, x, n, base, y, bad, st); break;
    case 424: launch_mode<4, 24>(mode_, P, exact, x, n, base, y, bad, st); break;
    case 1001: launch_mode<10, 1>(mode_, P, exact, x, n, base, y, bad, st); break;
    case 1012: launch_mode<10, 12>(mode_, P, exact, x, n, base, y, bad, st); break;
    case 2001: launch_mode<20, 1>(mode_, P, exact, x, n, base, y, bad, st); break;
    default: launch_mode<20, 24>(mode_, P, exact, x, n, base, y, bad, st); break;
  }
  kernel_timer().end(st);
  DDSG_CUDA(cudaGetLastError());
  return launches;
}

}  // namespace ddsg_b200
