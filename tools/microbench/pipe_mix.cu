// Pipe-concurrency microbenchmark: are DMMA (mma.sync f64), DFMA and the
// shared-memory gather (LDS.64, lane-varying rows) separate pipes on B200?
//
// Each kernel runs one instruction mix per loop iteration:
//   D DFMA warp-instructions (8 independent chains),
//   M DMMA m8n8k4 warp-instructions (4 independent accumulators),
//   L LDS.64 warp-instructions, every lane reading its own row of a
//     stride-9 table (conflict-free, 2 wavefronts each -- the slot kernel's
//     gather pattern).
// If two pipes are independent, a mix runs in max(t_a, t_b); if they share a
// pipe, in t_a + t_b.  Output: one JSON object (SM clocks per iteration per
// warp-slot, and the implied per-SM rates).
//
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o pipe_mix pipe_mix.cu
#include <cstdio>
#include <cstdlib>
#include <cuda_runtime.h>

#define CK(x) do { cudaError_t e_ = (x); if (e_ != cudaSuccess) { \
  fprintf(stderr, "CUDA %s at %s:%d\n", cudaGetErrorString(e_), __FILE__, __LINE__); exit(1);} } while (0)

template <int D, int M, int L>
__global__ void __launch_bounds__(512, 1) k_mix(double* out, int iters, double a, double b) {
  __shared__ double tab[128 * 9];
  for (int i = threadIdx.x; i < 128 * 9; i += blockDim.x) tab[i] = i * 1e-3;
  __syncthreads();
  const int lane = threadIdx.x & 31;
  // lane-varying rows: row = (lane * 37 + warp) & 127, stride 9 -> distinct banks
  const unsigned row = static_cast<unsigned>((lane * 37 + (threadIdx.x >> 5)) & 127);
  const unsigned base = static_cast<unsigned>(__cvta_generic_to_shared(tab)) + row * 72u;
  double f[8];
#pragma unroll
  for (int i = 0; i < 8; ++i) f[i] = threadIdx.x * 1e-3 + i;
  double c[4][2];
#pragma unroll
  for (int i = 0; i < 4; ++i) c[i][0] = c[i][1] = 0.0;
  double am = threadIdx.x * 1e-3, bm = 1.0 - threadIdx.x * 1e-4;
  unsigned long long acc = 0;
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int i = 0; i < D; ++i) f[i & 7] = fma(f[i & 7], a, b);
#pragma unroll
    for (int i = 0; i < M; ++i)
      asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
                   : "+d"(c[i & 3][0]), "+d"(c[i & 3][1]) : "d"(am), "d"(bm));
#pragma unroll
    for (int i = 0; i < L; ++i) {
      unsigned long long v;
      asm volatile("ld.volatile.shared.b64 %0, [%1];" : "=l"(v) : "r"(base + static_cast<unsigned>((i & 7) * 8)));
      acc ^= v;  // integer consumer: keeps the FP64 pipe out of the LDS-only mix
    }
  }
  double s = static_cast<double>(acc & 0xff);
#pragma unroll
  for (int i = 0; i < 8; ++i) s += f[i];
#pragma unroll
  for (int i = 0; i < 4; ++i) s += c[i][0] + c[i][1];
  if (s == 12345.678) out[threadIdx.x] = s;
}

static int g_sms = 0, g_clk_khz = 0;

template <int D, int M, int L>
static void run(const char* name, bool last) {
  double* out;
  CK(cudaMalloc(&out, 512 * sizeof(double)));
  const int iters = 4096;
  cudaEvent_t e0, e1;
  CK(cudaEventCreate(&e0));
  CK(cudaEventCreate(&e1));
  k_mix<D, M, L><<<g_sms, 512>>>(out, 64, 1.0000001, 1e-9);
  CK(cudaDeviceSynchronize());
  float best = 1e30f;
  for (int r = 0; r < 5; ++r) {
    CK(cudaEventRecord(e0));
    k_mix<D, M, L><<<g_sms, 512>>>(out, iters, 1.0000001, 1e-9);
    CK(cudaEventRecord(e1));
    CK(cudaEventSynchronize(e1));
    float ms;
    CK(cudaEventElapsedTime(&ms, e0, e1));
    if (ms < best) best = ms;
  }
  // SM clocks per iteration for the whole SM (16 warps resident)
  const double clk = best * 1e-3 * g_clk_khz * 1e3 / iters;
  printf("  \"%s\": {\"D\": %d, \"M\": %d, \"L\": %d, \"sm_clk_per_iter_16warps\": %.2f, "
         "\"dfma_per_clk_sm\": %.2f, \"dmma_per_clk_sm\": %.3f, \"lds_warpinstr_per_clk_sm\": %.3f}%s\n",
         name, D, M, L, clk, D * 16 * 32 / clk, M * 16 / clk, L * 16 / clk, last ? "" : ",");
  CK(cudaFree(out));
}

int main() {
  cudaDeviceProp p;
  CK(cudaGetDeviceProperties(&p, 0));
  g_sms = p.multiProcessorCount;
  int clk = 0;
  CK(cudaDeviceGetAttribute(&clk, cudaDevAttrClockRate, 0));
  g_clk_khz = clk;
  printf("{\"gpu\": \"%s\", \"sms\": %d, \"clock_rate_khz\": %d, \"note\": \"rates at the nominal clock; "
         "compare mixes against their parts\",\n", p.name, g_sms, g_clk_khz);
  run<32, 0, 0>("dfma32", false);
  run<0, 8, 0>("dmma8", false);
  run<0, 0, 16>("lds16", false);
  run<32, 8, 0>("dfma32_dmma8", false);
  run<0, 8, 16>("dmma8_lds16", false);
  run<32, 0, 16>("dfma32_lds16", false);
  run<16, 8, 16>("dfma16_dmma8_lds16", false);
  run<0, 16, 16>("dmma16_lds16", true);
  printf("}\n");
  return 0;
}
