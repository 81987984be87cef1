// FP64 / shared-memory microbenchmarks for the B200 roofline denominators.
//
// MEASURED_PEAKS.json (driver-written) carries HBM and bf16 only; the DDSG
// evaluation path is FP64-bound, so this program measures on the box:
//   * DFMA throughput (the FP64 FMA peak used as the roofline denominator),
//   * DMUL+DADD throughput (the exact-rounding accumulation pattern),
//   * DMMA (mma.sync f64) throughput,
//   * shared-memory LDS.64 / LDS.128 delivery for the gather patterns the
//     evaluation kernel issues (distinct rows, broadcast, 2/4/8 distinct rows).
// Output: one JSON object on stdout.
//
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o fp64_peaks fp64_peaks.cu
#include <cstdio>
#include <cstdlib>
#include <cuda_runtime.h>

#define CK(x) do { cudaError_t e_ = (x); if (e_ != cudaSuccess) { \
  fprintf(stderr, "CUDA %s at %s:%d\n", cudaGetErrorString(e_), __FILE__, __LINE__); exit(1);} } while (0)

constexpr int kChains = 8;

__global__ void k_dfma(double* out, int iters, double a, double b) {
  double acc[kChains];
#pragma unroll
  for (int i = 0; i < kChains; ++i) acc[i] = threadIdx.x * 1e-3 + i;
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int r = 0; r < 8; ++r)
#pragma unroll
      for (int i = 0; i < kChains; ++i) acc[i] = fma(acc[i], a, b);
  }
  double s = 0;
#pragma unroll
  for (int i = 0; i < kChains; ++i) s += acc[i];
  if (s == 12345.678) out[threadIdx.x] = s;
}

__global__ void k_dmul_dadd(double* out, int iters, double a, double b) {
  double acc[kChains];
#pragma unroll
  for (int i = 0; i < kChains; ++i) acc[i] = threadIdx.x * 1e-3 + i;
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int r = 0; r < 4; ++r)
#pragma unroll
      for (int i = 0; i < kChains; ++i) acc[i] = __dadd_rn(__dmul_rn(acc[i], a), b);
  }
  double s = 0;
#pragma unroll
  for (int i = 0; i < kChains; ++i) s += acc[i];
  if (s == 12345.678) out[threadIdx.x] = s;
}

// mma.sync m8n8k4 f64: 8*8*4 = 256 FMA per warp-instruction.
__global__ void k_dmma884(double* out, int iters) {
  double a = threadIdx.x * 1e-3, b = 1.0 - threadIdx.x * 1e-4;
  double c[4][2];
#pragma unroll
  for (int i = 0; i < 4; ++i) { c[i][0] = 0; c[i][1] = 0; }
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int r = 0; r < 8; ++r)
#pragma unroll
      for (int i = 0; i < 4; ++i)
        asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
                     : "+d"(c[i][0]), "+d"(c[i][1]) : "d"(a), "d"(b));
  }
  double s = 0;
#pragma unroll
  for (int i = 0; i < 4; ++i) s += c[i][0] + c[i][1];
  if (s == 12345.678) out[threadIdx.x] = s;
}

// m16n8k16 f64 (sm_90+ shape): 16*8*16 = 2048 FMA per warp-instruction.
__global__ void k_dmma16816(double* out, int iters) {
  double a[8], b[4];
#pragma unroll
  for (int i = 0; i < 8; ++i) a[i] = threadIdx.x * 1e-3 + i;
#pragma unroll
  for (int i = 0; i < 4; ++i) b[i] = 1.0 - threadIdx.x * 1e-4 * i;
  double c[2][4];
#pragma unroll
  for (int i = 0; i < 2; ++i)
#pragma unroll
    for (int j = 0; j < 4; ++j) c[i][j] = 0;
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int r = 0; r < 4; ++r)
#pragma unroll
      for (int i = 0; i < 2; ++i)
        asm volatile(
            "mma.sync.aligned.m16n8k16.row.col.f64.f64.f64.f64 {%0,%1,%2,%3}, "
            "{%4,%5,%6,%7,%8,%9,%10,%11}, {%12,%13,%14,%15}, {%0,%1,%2,%3};\n"
            : "+d"(c[i][0]), "+d"(c[i][1]), "+d"(c[i][2]), "+d"(c[i][3])
            : "d"(a[0]), "d"(a[1]), "d"(a[2]), "d"(a[3]), "d"(a[4]), "d"(a[5]), "d"(a[6]), "d"(a[7]),
              "d"(b[0]), "d"(b[1]), "d"(b[2]), "d"(b[3]));
  }
  double s = 0;
#pragma unroll
  for (int i = 0; i < 2; ++i)
#pragma unroll
    for (int j = 0; j < 4; ++j) s += c[i][j];
  if (s == 12345.678) out[threadIdx.x] = s;
}

// Shared-memory gather: every lane loads 8 B (or 16 B) from row rowsel(lane),
// column `c`, rows 16 doubles (+pad) apart.  `groups` = number of distinct
// rows touched by one warp instruction (1 = broadcast, 32 = all distinct).
template <int kVec>
__global__ void k_lds(double* out, int iters, int groups, int pad) {
  extern __shared__ double sm[];
  const int stride = 64 + pad;
  for (int i = threadIdx.x; i < 64 * stride; i += blockDim.x) sm[i] = i * 1e-3;
  __syncthreads();
  const int lane = threadIdx.x & 31;
  // groups > 0: lanes form `groups` broadcast groups, each group reads one
  // address in a different row (same column) -> the s[n(p)][c] gather with
  // `groups` distinct nodes.  groups == 0: every lane reads its own
  // consecutive element (conflict-free contiguous row segment).
  int row, col;
  if (groups == 0) { row = 0; col = lane * kVec; }
  else { row = (lane * groups) / 32; col = 0; }
  unsigned long long acc0 = 0, acc1 = 0;
  const double* base = sm + row * stride + col;
  const unsigned addr = (unsigned)__cvta_generic_to_shared(base);
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int r = 0; r < 16; ++r) {
      const unsigned a = addr + (r & 3) * 256;  // same bank pattern, different words
      if (kVec == 1) {
        unsigned long long v;
        asm volatile("ld.volatile.shared.b64 %0, [%1];" : "=l"(v) : "r"(a));
        acc0 += v;
      } else {
        unsigned long long v0, v1;
        asm volatile("ld.volatile.shared.v2.b64 {%0,%1}, [%2];" : "=l"(v0), "=l"(v1) : "r"(a));
        acc0 += v0;
        acc1 += v1;
      }
    }
  }
  if ((acc0 ^ acc1) == 0x12345ull) out[threadIdx.x] = (double)acc0;
}

static int g_sms = 0;

template <typename F>
static float time_kernel(F launch) {
  cudaEvent_t a, b;
  CK(cudaEventCreate(&a));
  CK(cudaEventCreate(&b));
  launch();  // warm
  CK(cudaDeviceSynchronize());
  float best = 1e30f;
  for (int rep = 0; rep < 5; ++rep) {
    CK(cudaEventRecord(a));
    launch();
    CK(cudaEventRecord(b));
    CK(cudaEventSynchronize(b));
    float ms;
    CK(cudaEventElapsedTime(&ms, a, b));
    if (ms < best) best = ms;
  }
  CK(cudaGetLastError());
  return best;
}

int main() {
  cudaDeviceProp prop;
  CK(cudaGetDeviceProperties(&prop, 0));
  g_sms = prop.multiProcessorCount;
  int clk_khz = 0;
  CK(cudaDeviceGetAttribute(&clk_khz, cudaDevAttrClockRate, 0));
  double* out;
  CK(cudaMalloc(&out, 1 << 20));
  const int threads = 512, blocks = g_sms * 4;
  printf("{\"gpu\": \"%s\", \"sms\": %d, \"clock_rate_khz\": %d", prop.name, g_sms, clk_khz);

  {
    const int iters = 4000;
    float ms = time_kernel([&] { k_dfma<<<blocks, threads>>>(out, iters, 0.999, 1e-3); });
    double flops = 2.0 * kChains * 8.0 * iters * threads * (double)blocks;
    printf(", \"dfma_tflops\": %.3f", flops / ms / 1e9);
  }
  {
    const int iters = 4000;
    float ms = time_kernel([&] { k_dmul_dadd<<<blocks, threads>>>(out, iters, 0.999, 1e-3); });
    double flops = 2.0 * kChains * 4.0 * iters * threads * (double)blocks;  // mul+add = 2 flops
    printf(", \"dmul_dadd_tflops\": %.3f", flops / ms / 1e9);
  }
  {
    const int iters = 2000;
    float ms = time_kernel([&] { k_dmma884<<<blocks, threads>>>(out, iters); });
    double flops = 2.0 * 256.0 * 4 * 8 * iters * (threads / 32) * (double)blocks;
    printf(", \"dmma_m8n8k4_tflops\": %.3f", flops / ms / 1e9);
  }
  {
    const int iters = 500;
    float ms = time_kernel([&] { k_dmma16816<<<blocks, threads>>>(out, iters); });
    double flops = 2.0 * 2048.0 * 2 * 4 * iters * (threads / 32) * (double)blocks;
    printf(", \"dmma_m16n8k16_tflops\": %.3f", flops / ms / 1e9);
  }
  // LDS: report delivered bytes per SM per clock (at the nominal clock) and
  // warp-instructions per SM per clock.
  const int lds_threads = 512, lds_blocks = g_sms * 2;
  for (int vec : {1, 2}) {
    for (int pad : {0, 2}) {
      for (int groups : {0, 1, 2, 4, 8, 16, 32}) {
        const int iters = 2000;
        size_t smem = 64 * (64 + pad) * sizeof(double);
        float ms;
        if (vec == 1)
          ms = time_kernel([&] { k_lds<1><<<lds_blocks, lds_threads, smem>>>(out, iters, groups, pad); });
        else
          ms = time_kernel([&] { k_lds<2><<<lds_blocks, lds_threads, smem>>>(out, iters, groups, pad); });
        double warp_instr = 16.0 * iters * (lds_threads / 32) * (double)lds_blocks;
        double cycles = ms * 1e-3 * clk_khz * 1e3;  // nominal-clock cycles
        double per_sm_clk = warp_instr / g_sms / cycles;
        printf(", \"lds_v%d_pad%d_rows%d_warpinstr_per_sm_clk\": %.3f", vec, pad, groups, per_sm_clk);
      }
    }
  }
  printf("}\n");
  return 0;
}
