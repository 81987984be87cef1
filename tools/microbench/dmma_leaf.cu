// DMMA (mma.sync.m8n8k4.f64) vs shared-memory gather for the shallow
// subspaces of a config-5 pair cut (2-d modified-linear grid, max level 5,
// level sum <= 6: 15 canonical subspaces, 129 rows, one nonzero node per
// subspace per point) -- VERDICT r1 next #3(ii) / coverage row N1.
//
// One warp = 32 points (lanes) x 8 output columns, 16 warps per CTA, the
// slot's row table staged in shared memory with the slot kernel's stride-9
// rows (csrc/fast_hdmr_device.cuh).  Per slot and point:
//   V0  gather, FAST:  15 terms, acc = fma(w, s[row][c], acc)   (the slot kernel's leaf)
//   V1  gather, EXACT: 15 terms, acc = acc + w*s (DMUL + DADD)   (the bench mode)
//   V2  DMMA + gather, FAST: the 6 terms of level sums 2-4 (rows 0..16,
//       17 rows = 5 k-chunks of 4) as a dense weight x surplus product on
//       the FP64 tensor path -- the point's 6 nonzero weights scattered into
//       a per-warp dense [32 points][21] weight block in shared memory, A
//       fragments read from it, B fragments (4 rows x 8 columns) read from
//       the table once per chunk and reused by the warp's 4 point groups,
//       C transposed back to lanes = points through shared memory -- then
//       the 9 deep terms (level sums 5, 6) gathered as in V0.
// Output: one JSON object (ns per slot-warp, implied TFLOP/s at 2 m nnz,
// V2's max relative deviation from V0).
//
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -lineinfo -o dmma_leaf dmma_leaf.cu
#include <cstdio>
#include <cstdlib>
#include <cmath>
#include <vector>
#include <cuda_runtime.h>

#define CK(x) do { cudaError_t e_ = (x); if (e_ != cudaSuccess) { \
  fprintf(stderr, "CUDA %s at %s:%d\n", cudaGetErrorString(e_), __FILE__, __LINE__); exit(1);} } while (0)

constexpr int kCols = 8, kStride = 9, kL = 5, kRows = 129, kWarps = 16, kPts = kWarps * 32;
constexpr int kShallowRows = 17, kChunks = 5, kWStride = 21;

__host__ __device__ constexpr int base2(int l1, int l2) {
  int b = 0;
  for (int t = 2; t < l1 + l2; ++t) b += (t - 1) << (t - 2);
  return b + ((l1 - 1) << (l1 + l2 - 2));
}

// modified-linear 1-d factor at static level l (basis.hpp:36-54)
template <int l>
__device__ __forceinline__ void factor(double x, unsigned& kk, double& v) {
  constexpr unsigned ncell = 1u << (l - 1);
  const unsigned k = static_cast<unsigned>(__dmul_rn(x, static_cast<double>(ncell)));
  kk = k < ncell ? k : ncell - 1u;
  if (l == 1) {
    v = 1.0;
    return;
  }
  const double t = __dmul_rn(x, static_cast<double>(2u * ncell));
  const bool left = kk == 0u, right = kk == ncell - 1u;
  const unsigned B = left ? 0u : (right ? 2u * ncell : 2u * kk + 1u);
  const double A = (left || right) ? 2.0 : 1.0;
  v = __dadd_rn(A, -fabs(__dadd_rn(t, -static_cast<double>(B))));
}

template <int V>
__global__ void __launch_bounds__(kPts, 1)
    leaf_kernel(const double* __restrict__ xs, int slots, long long P, const double* __restrict__ tab_g,
                double* __restrict__ out) {
  extern __shared__ double sm[];
  double* tab = sm;                                  // [kRows + 1][kStride]
  double* wsc = tab + (kRows + 1) * kStride;          // [kWarps][32][kWStride]   (V2)
  double* csc = wsc + kWarps * 32 * kWStride;         // [kWarps][32][kStride]    (V2)
  for (int i = threadIdx.x; i < (kRows + 1) * kStride; i += blockDim.x) tab[i] = tab_g[i];
  __syncthreads();
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const long long p = static_cast<long long>(blockIdx.x) * kPts + threadIdx.x;
  double* W = wsc + warp * 32 * kWStride;
  double* Cs = csc + warp * 32 * kStride;
  double total[kCols];
#pragma unroll
  for (int c = 0; c < kCols; ++c) total[c] = 0.0;
  for (int s = 0; s < slots; ++s) {
    const double x0 = xs[(2LL * s) * P + p], x1 = xs[(2LL * s + 1) * P + p];
    double v0[kL], v1[kL];
    unsigned k0[kL], k1[kL];
#define F(LV) factor<LV>(x0, k0[LV - 1], v0[LV - 1]); factor<LV>(x1, k1[LV - 1], v1[LV - 1]);
    F(1) F(2) F(3) F(4) F(5)
#undef F
    double acc[kCols];
#pragma unroll
    for (int c = 0; c < kCols; ++c) acc[c] = 0.0;
    int t = 0;
#pragma unroll
    for (int ls = 2; ls <= kL + 1; ++ls) {
#pragma unroll
      for (int l1 = 1; l1 < ls; ++l1) {
        const int l2 = ls - l1;
        const double w = l1 == 1 ? v1[l2 - 1] : (l2 == 1 ? v0[l1 - 1] : __dmul_rn(v0[l1 - 1], v1[l2 - 1]));
        const int row = base2(l1, l2) + static_cast<int>((k0[l1 - 1] << (l2 - 1)) | k1[l2 - 1]);
        if (V == 2 && ls <= 4) {
          // scatter the shallow weight into the warp's dense block (zeroed below)
          if (t == 0) {
#pragma unroll
            for (int r = 0; r < kWStride; ++r) W[lane * kWStride + r] = 0.0;
            __syncwarp();
          }
          W[lane * kWStride + row] = w;
          ++t;
          continue;
        }
        if (V == 2 && ls == 5 && l1 == 1) {
          // shallow block complete: dense product on the tensor path
          __syncwarp();
          double cg[4][2];
#pragma unroll
          for (int g = 0; g < 4; ++g) cg[g][0] = cg[g][1] = 0.0;
#pragma unroll
          for (int ch = 0; ch < kChunks; ++ch) {
            const int r = 4 * ch + (lane & 3);
            const double b = tab[(r < kShallowRows ? r : kRows) * kStride + (lane >> 2)];
#pragma unroll
            for (int g = 0; g < 4; ++g) {
              const double a = W[(8 * g + (lane >> 2)) * kWStride + r];
              asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
                           : "+d"(cg[g][0]), "+d"(cg[g][1]) : "d"(a), "d"(b));
            }
          }
          // C (lane 4r+j: point 8g+r, columns 2j, 2j+1) -> lanes = points
#pragma unroll
          for (int g = 0; g < 4; ++g)
#pragma unroll
            for (int e = 0; e < 2; ++e) Cs[(8 * g + (lane >> 2)) * kStride + 2 * (lane & 3) + e] = cg[g][e];
          __syncwarp();
#pragma unroll
          for (int c = 0; c < kCols; ++c) acc[c] = Cs[lane * kStride + c];
          __syncwarp();
        }
        const double* sr = tab + row * kStride;
#pragma unroll
        for (int c = 0; c < kCols; ++c)
          acc[c] = V == 1 ? __dadd_rn(acc[c], __dmul_rn(w, sr[c])) : __fma_rn(w, sr[c], acc[c]);
      }
    }
#pragma unroll
    for (int c = 0; c < kCols; ++c) total[c] += acc[c];
  }
#pragma unroll
  for (int c = 0; c < kCols; ++c) out[p * kCols + c] = total[c];
}

template <int V>
static float run(const double* xs, int slots, long long P, const double* tab, double* out, int blocks) {
  const size_t smem = ((kRows + 1) * kStride + kWarps * 32 * kWStride + kWarps * 32 * kStride) * sizeof(double);
  CK(cudaFuncSetAttribute(leaf_kernel<V>, cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(smem)));
  leaf_kernel<V><<<blocks, kPts, smem>>>(xs, 4, P, tab, out);  // warm
  CK(cudaDeviceSynchronize());
  cudaEvent_t a, b;
  CK(cudaEventCreate(&a));
  CK(cudaEventCreate(&b));
  float best = 1e30f;
  for (int r = 0; r < 5; ++r) {
    CK(cudaEventRecord(a));
    leaf_kernel<V><<<blocks, kPts, smem>>>(xs, slots, P, tab, out);
    CK(cudaEventRecord(b));
    CK(cudaEventSynchronize(b));
    float ms;
    CK(cudaEventElapsedTime(&ms, a, b));
    best = ms < best ? ms : best;
  }
  return best;
}

int main() {
  cudaDeviceProp prop;
  CK(cudaGetDeviceProperties(&prop, 0));
  const int blocks = prop.multiProcessorCount * 4;
  const long long P = static_cast<long long>(blocks) * kPts;
  const int slots = 128;
  std::vector<double> hx(2LL * slots * P), ht((kRows + 1) * kStride, 0.0);
  unsigned long long st = 88172645463325252ull;
  auto rnd = [&] {
    st ^= st << 13;
    st ^= st >> 7;
    st ^= st << 17;
    return static_cast<double>(st >> 11) * 0x1.0p-53;
  };
  for (auto& v : hx) v = rnd();
  for (int r = 0; r < kRows; ++r)
    for (int c = 0; c < kCols; ++c) ht[r * kStride + c] = rnd() * 2.0 - 1.0;  // zero row kRows stays 0
  double *xs, *tab, *o0, *o1, *o2;
  CK(cudaMalloc(&xs, hx.size() * 8));
  CK(cudaMalloc(&tab, ht.size() * 8));
  CK(cudaMalloc(&o0, P * kCols * 8));
  CK(cudaMalloc(&o1, P * kCols * 8));
  CK(cudaMalloc(&o2, P * kCols * 8));
  CK(cudaMemcpy(xs, hx.data(), hx.size() * 8, cudaMemcpyHostToDevice));
  CK(cudaMemcpy(tab, ht.data(), ht.size() * 8, cudaMemcpyHostToDevice));
  const float t0 = run<0>(xs, slots, P, tab, o0, blocks);
  const float t1 = run<1>(xs, slots, P, tab, o1, blocks);
  const float t2 = run<2>(xs, slots, P, tab, o2, blocks);
  std::vector<double> r0(P * kCols), r2(P * kCols);
  CK(cudaMemcpy(r0.data(), o0, r0.size() * 8, cudaMemcpyDeviceToHost));
  CK(cudaMemcpy(r2.data(), o2, r2.size() * 8, cudaMemcpyDeviceToHost));
  double dev = 0.0;
  for (size_t i = 0; i < r0.size(); ++i) dev = std::fmax(dev, std::fabs(r0[i] - r2[i]) / (std::fabs(r0[i]) + 1e-300));
  const double flops = 2.0 * kCols * 15.0 * static_cast<double>(slots) * static_cast<double>(P);
  auto line = [&](const char* name, float ms, bool last) {
    printf("  \"%s\": {\"ms\": %.3f, \"ns_per_slot_warp\": %.2f, \"tflops_2m_nnz\": %.3f}%s\n", name, ms,
           ms * 1e6 / (static_cast<double>(slots) * P / 32.0) * prop.multiProcessorCount, flops / (ms * 1e-3) / 1e12,
           last ? "," : ",");
  };
  printf("{\"gpu\": \"%s\", \"what\": \"config-5 pair-cut leaf (2-d, level 5, 15 terms, 8 columns), %d slots x %lld points\",\n",
         prop.name, slots, P);
  line("v0_gather_fast", t0, false);
  line("v1_gather_exact", t1, false);
  line("v2_dmma_shallow_fast", t2, false);
  printf("  \"v2_max_rel_dev_from_v0\": %.3e\n}\n", dev);
  return 0;
}
