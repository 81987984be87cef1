// Plain-grid evaluation kernel (BASELINE configs 1-3): one thread per point
// and up to kMC output columns, walking the grid's subspaces in canonical
// order (per stored-order run) with incremental prefix products.
//
// The reference's node weight is the dim-ordered product
// w = ((1 * v_0) * v_1) * ... (sparse_grid.hpp:116-122): its partial products
// are exactly prefix products, so for consecutive subspaces l, l' whose level
// vectors first differ at dim q only the suffix q..d-1 is recomputed (3.7
// factors per subspace on average for config 2, 6.0 for config 3).  The 1-d
// factors v(x_j, l) are recomputed from the coordinates held in registers
// (measured 2x faster than a per-thread shared-memory factor table, whose
// footprint capped occupancy at 12 warps/SM on this latency-bound gather;
// the table variant is kept behind kTable).  Surplus rows are gathered
// through L1 (97% hit rate on config 2).  Rounding is bit-identical to the
// reference (EXACT: separate mul and add per term; a zero prefix stays zero,
// which is the reference's early exit).
#include <cuda_runtime.h>

#include <algorithm>

#include "basis.cuh"
#include "plain.cuh"

namespace ddsg_b200 {

namespace plain {

// One 32-byte record per subspace, read with two warp-uniform 16-byte loads:
//   w[0] = first row (full subspace) or slab offset (partial)
//   w[1] = q (first dim to recompute) | full << 8
//   w[2..7] = levels as 4-bit nibbles, dim j in word 2 + j/8, bits 4*(j%8)
struct Params {
  int d, m, n_sub, runs, lmax, mode;
  const uint4* rec;        // [n_sub][2]
  const int32_t* slab;     // partial subspaces: cell -> row or -1
  const int16_t* row_run;  // [rows]
  const double* surplus;   // [rows][ms] (ms = m rounded up to even: 16-byte rows)
  int ms;
};

// kTable: 1 = 1-d factors from a per-thread shared-memory table, 0 =
// recomputed from the coordinates held in registers (no shared memory, so
// more warps per SM hide the gather latency).
template <int kDMax, int kMC, int kExact, int kTable>
__global__ void __launch_bounds__(kThreads) plain_kernel(Params P, const double* __restrict__ x, int64_t n,
                                                         int64_t base, double* __restrict__ y,
                                                         unsigned long long* bad) {
  extern __shared__ __align__(16) unsigned char smem[];
  const int tid = threadIdx.x;
  const int64_t p = static_cast<int64_t>(blockIdx.x) * kThreads + tid;
  const bool valid = p < n;
  const int d = P.d, L = P.lmax;
  double* fv = reinterpret_cast<double*>(smem);                              // [d*L][kThreads]
  uint16_t* fk = reinterpret_cast<uint16_t*>(fv + static_cast<int64_t>(d) * L * kThreads);  // [d*L][kThreads]
  double xr[kDMax];
  bool ok = valid;
#pragma unroll
  for (int j = 0; j < kDMax; ++j) {
    xr[j] = 0.5;
    if (j < d) {
      const double xv = valid ? x[p * d + j] : 0.5;
      xr[j] = xv;
      ok &= (xv >= 0.0 && xv <= 1.0);
      if (kTable) {
        for (int l = 1; l <= L; ++l) {
          const uint32_t kk = cell_at(xv, l);
          fv[(j * L + l - 1) * kThreads + tid] = basis_at(P.mode, l, kk, xv);
          fk[(j * L + l - 1) * kThreads + tid] = static_cast<uint16_t>(kk);
        }
      }
    }
  }
  if (valid && !ok) atomicMin(bad, static_cast<unsigned long long>(base + p));
  if (!valid || !ok) return;  // no block-wide barrier below: each thread owns its table column

  for (int c0 = 0; c0 < P.m; c0 += kMC) {
    const int nc = min(kMC, P.m - c0);
    double acc[kMC];
#pragma unroll
    for (int c = 0; c < kMC; ++c) acc[c] = 0.0;
    for (int run = 0; run < P.runs; ++run) {
      double pw[kDMax];
      uint32_t pc[kDMax];
#pragma unroll
      for (int j = 0; j < kDMax; ++j) {
        pw[j] = 0.0;
        pc[j] = 0u;
      }
      for (int s = 0; s < P.n_sub; ++s) {
        const uint4 r0 = __ldg(P.rec + 2 * s);
        uint4 r1 = make_uint4(0u, 0u, 0u, 0u);
        if (kDMax > 16) r1 = __ldg(P.rec + 2 * s + 1);
        const int q = static_cast<int>(r0.y & 0xffu);
        const uint32_t lw[6] = {r0.z, r0.w, r1.x, r1.y, r1.z, r1.w};
        // recompute the suffix q..kDMax-1 only: jump into the unrolled dim
        // chain at q (warp-uniform) and fall through
        switch (q) {
#define DDSG_DIM(J)                                                                 \
  case J:                                                                           \
    if (J < kDMax) {                                                                \
      if (J < d) {                                                                  \
        const int l = static_cast<int>((lw[(J) / 8] >> (4 * ((J) % 8))) & 15u);     \
        double v;                                                                   \
        uint32_t kk;                                                                \
        if (kTable) {                                                               \
          const int t = ((J) * L + l - 1) * kThreads + tid;                         \
          v = fv[t];                                                                \
          kk = fk[t];                                                               \
        } else {                                                                    \
          kk = cell_at(xr[(J) < kDMax ? (J) : 0], l);                               \
          v = basis_at(P.mode, l, kk, xr[(J) < kDMax ? (J) : 0]);                   \
        }                                                                           \
        if ((J) == 0) {                                                             \
          pw[0] = v; /* fl(1 * v_0) */                                              \
          pc[0] = kk;                                                               \
        } else {                                                                    \
          pw[(J) < kDMax ? (J) : 0] = __dmul_rn(pw[(J) > 0 && (J) <= kDMax ? (J) - 1 : 0], v); \
          pc[(J) < kDMax ? (J) : 0] = (pc[(J) > 0 && (J) <= kDMax ? (J) - 1 : 0] << (l - 1)) | kk; \
        }                                                                           \
      } else if ((J) > 0) {                                                         \
        pw[(J) < kDMax ? (J) : 0] = pw[(J) > 0 && (J) <= kDMax ? (J) - 1 : 0];      \
        pc[(J) < kDMax ? (J) : 0] = pc[(J) > 0 && (J) <= kDMax ? (J) - 1 : 0];      \
      }                                                                             \
    }                                                                               \
    [[fallthrough]];
          DDSG_DIM(0) DDSG_DIM(1) DDSG_DIM(2) DDSG_DIM(3) DDSG_DIM(4) DDSG_DIM(5) DDSG_DIM(6) DDSG_DIM(7)
          DDSG_DIM(8) DDSG_DIM(9) DDSG_DIM(10) DDSG_DIM(11) DDSG_DIM(12) DDSG_DIM(13) DDSG_DIM(14)
          DDSG_DIM(15) DDSG_DIM(16) DDSG_DIM(17) DDSG_DIM(18) DDSG_DIM(19)
#undef DDSG_DIM
          default:
            break;
        }
        const double w = pw[kDMax - 1];
        if (w == 0.0) continue;  // support test (sparse_grid.hpp:123)
        int row = static_cast<int>(r0.x);
        if ((r0.y >> 8) & 1u)
          row += static_cast<int>(pc[kDMax - 1]);
        else
          row = P.slab[row + static_cast<int>(pc[kDMax - 1])];
        if (row < 0) continue;
        if (P.runs > 1 && P.row_run[row] != run) continue;
        const double* sr = P.surplus + static_cast<int64_t>(row) * P.ms + c0;
        if (kMC == 1) {
          const double sv = __ldg(sr);
          acc[0] = kExact ? __dadd_rn(acc[0], __dmul_rn(w, sv)) : __fma_rn(w, sv, acc[0]);
        } else {
          // 16-byte loads: one L1 sector request per lane per two columns
#pragma unroll
          for (int c = 0; c < kMC; c += 2) {
            if (c < nc) {
              const double2 sv = __ldg(reinterpret_cast<const double2*>(sr + c));
              acc[c] = kExact ? __dadd_rn(acc[c], __dmul_rn(w, sv.x)) : __fma_rn(w, sv.x, acc[c]);
              if (kMC > 1)
                acc[c + 1] = kExact ? __dadd_rn(acc[c + 1], __dmul_rn(w, sv.y)) : __fma_rn(w, sv.y, acc[c + 1]);
            }
          }
        }
      }
    }
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

bool PlainGrid::build(const HostProgram& hp, const EvalParams& dev) {
  usable_ = false;
  if (!hp.plain || hp.slot_k.size() != 1) return false;
  const int d = hp.d;
  if (d > kMaxDim) return false;
  const int s0 = hp.slot_sub_begin[0], s1 = hp.slot_sub_end[0];
  const int n_sub = s1 - s0;
  int lmax = 1;
  for (int s = s0; s < s1; ++s)
    for (int j = 0; j < d; ++j) lmax = std::max<int>(lmax, hp.levels[hp.sub_lv_off[s] + j]);
  if (lmax > 16) return false;
  const size_t smem = static_cast<size_t>(d) * lmax * kThreads * (sizeof(double) + sizeof(uint16_t));
  if (smem > 200 * 1024) return false;
  if (lmax > 15) return false;  // 4-bit level nibbles
  std::vector<uint32_t> rec(static_cast<size_t>(n_sub) * 8, 0u);
  for (int s = 0; s < n_sub; ++s) {
    const uint8_t* lv = &hp.levels[hp.sub_lv_off[s0 + s]];
    int qq = 0;
    if (s > 0) {
      const uint8_t* prev = &hp.levels[hp.sub_lv_off[s0 + s - 1]];
      while (qq < d && prev[qq] == lv[qq]) ++qq;
    }
    int64_t cells = 1;
    for (int j = 0; j < d; ++j) cells <<= (lv[j] - 1);
    const int64_t slab_off = hp.sub_slab_off[s0 + s];
    const bool is_full = hp.sub_nodes[s0 + s] == cells;
    uint32_t* r = &rec[static_cast<size_t>(s) * 8];
    r[0] = static_cast<uint32_t>(is_full ? hp.slab[slab_off] : slab_off);
    r[1] = static_cast<uint32_t>(qq) | (is_full ? 0x100u : 0u);
    for (int j = 0; j < d; ++j) r[2 + j / 8] |= static_cast<uint32_t>(lv[j]) << (4 * (j % 8));
  }
  d_ = d;
  m_ = hp.m;
  n_sub_ = n_sub;
  lmax_ = lmax;
  mode_ = hp.slot_mode[0];
  runs_ = hp.slot_runs[0];
  smem_ = smem;
  rec_ = reinterpret_cast<const uint4*>(put(rec));
  // row-padded copy of the surpluses (even stride -> 16-byte aligned rows)
  ms_ = hp.m == 1 ? 1 : (hp.m + 1) / 2 * 2;
  if (ms_ != hp.m) {
    std::vector<double> pad(static_cast<size_t>(hp.rows) * ms_, 0.0);
    for (int64_t r = 0; r < hp.rows; ++r)
      std::copy(hp.surplus.begin() + r * hp.m, hp.surplus.begin() + (r + 1) * hp.m, pad.begin() + r * ms_);
    surplus_ = put(pad);
  } else {
    surplus_ = dev.surplus;
  }
  slab_ = dev.slab;
  row_run_ = dev.row_run;
  usable_ = true;
  return true;
}

template <int kDMax, int kMC>
static void launch_plain(const Params& P, int exact, const double* x, int64_t n, int64_t base, double* y,
                         unsigned long long* bad, cudaStream_t st, size_t smem) {
  const unsigned grid = static_cast<unsigned>((n + kThreads - 1) / kThreads);
  // factor table only pays off when the recompute is long (many dims changed per subspace)
  constexpr int kTab = 0;
  smem = kTab ? smem : 0;
  if (exact) {
    DDSG_CUDA(cudaFuncSetAttribute(plain_kernel<kDMax, kMC, 1, kTab>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                   static_cast<int>(smem)));
    plain_kernel<kDMax, kMC, 1, kTab><<<grid, kThreads, smem, st>>>(P, x, n, base, y, bad);
  } else {
    DDSG_CUDA(cudaFuncSetAttribute(plain_kernel<kDMax, kMC, 0, kTab>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                   static_cast<int>(smem)));
    plain_kernel<kDMax, kMC, 0, kTab><<<grid, kThreads, smem, st>>>(P, x, n, base, y, bad);
  }
}

int64_t PlainGrid::launch(int exact, const double* x, int64_t n, int64_t base, double* y,
                          unsigned long long* bad, cudaStream_t st) const {
  Params P{d_, m_, n_sub_, runs_, lmax_, mode_, rec_, slab_, row_run_, surplus_, ms_};
  kernel_timer().begin(st);
  // column chunk: all outputs per thread when m is small
  const int mc = m_ <= 1 ? 1 : (m_ <= 12 ? 12 : 24);
  if (d_ <= 4) {
    if (mc == 1) launch_plain<4, 1>(P, exact, x, n, base, y, bad, st, smem_);
    else if (mc == 12) launch_plain<4, 12>(P, exact, x, n, base, y, bad, st, smem_);
    else launch_plain<4, 24>(P, exact, x, n, base, y, bad, st, smem_);
  } else if (d_ <= 10) {
    if (mc == 1) launch_plain<10, 1>(P, exact, x, n, base, y, bad, st, smem_);
    else if (mc == 12) launch_plain<10, 12>(P, exact, x, n, base, y, bad, st, smem_);
    else launch_plain<10, 24>(P, exact, x, n, base, y, bad, st, smem_);
  } else {
    if (mc == 1) launch_plain<20, 1>(P, exact, x, n, base, y, bad, st, smem_);
    else if (mc == 12) launch_plain<20, 12>(P, exact, x, n, base, y, bad, st, smem_);
    else launch_plain<20, 24>(P, exact, x, n, base, y, bad, st, smem_);
  }
  kernel_timer().end(st);
  DDSG_CUDA(cudaGetLastError());
  return 1;
}

}  // namespace ddsg_b200
