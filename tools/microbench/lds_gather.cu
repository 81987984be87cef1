// Shared-memory gather microbenchmark for the DDSG slot kernel's access
// pattern: 32 lanes (points) each read column c of a row chosen at random
// among K consecutive rows (one subspace of K cells), row stride S doubles.
// Reports warp-instructions per SM per clock for LDS.64 and LDS.128.
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o lds_gather lds_gather.cu
#include <cstdio>
#include <cstdlib>
#include <cuda_runtime.h>

#define CK(x) do { cudaError_t e_ = (x); if (e_ != cudaSuccess) { \
  fprintf(stderr, "CUDA %s at %s:%d\n", cudaGetErrorString(e_), __FILE__, __LINE__); exit(1);} } while (0)

template <int kVec>
__global__ void k_gather(unsigned long long* out, int iters, int K, int stride, unsigned seed) {
  extern __shared__ double sm[];
  for (int i = threadIdx.x; i < 256 * stride; i += blockDim.x) sm[i] = i;
  __syncthreads();
  const int lane = threadIdx.x & 31;
  // 16 random row choices per lane (hash), fixed for the run
  unsigned rows[16];
  unsigned h = seed ^ (threadIdx.x * 2654435761u) ^ (blockIdx.x * 97u);
#pragma unroll
  for (int r = 0; r < 16; ++r) {
    h = h * 1664525u + 1013904223u;
    rows[r] = (h >> 8) % K;
  }
  unsigned long long acc0 = 0, acc1 = 0;
  const unsigned base = (unsigned)__cvta_generic_to_shared(sm);
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int r = 0; r < 16; ++r) {
      const unsigned a = base + (rows[r] * stride + (r & 7) * kVec) * 8;
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
  if ((acc0 ^ acc1) == 0x12345ull) out[threadIdx.x] = acc0;
  (void)lane;
}

int main() {
  cudaDeviceProp prop;
  CK(cudaGetDeviceProperties(&prop, 0));
  int clk_khz = 0;
  CK(cudaDeviceGetAttribute(&clk_khz, cudaDevAttrClockRate, 0));
  unsigned long long* out;
  CK(cudaMalloc(&out, 1 << 20));
  const int threads = 512, blocks = prop.multiProcessorCount * 2, iters = 2000;
  cudaEvent_t a, b;
  CK(cudaEventCreate(&a));
  CK(cudaEventCreate(&b));
  printf("{\"sms\": %d", prop.multiProcessorCount);
  for (int vec : {1, 2})
    for (int stride : {8, 9, 10, 17})
      for (int K : {1, 2, 4, 8, 16, 32, 64, 128}) {
        if (vec == 2 && (stride & 1)) continue;
        size_t smem = 256 * stride * 8;
        auto launch = [&] {
          if (vec == 1)
            k_gather<1><<<blocks, threads, smem>>>(out, iters, K, stride, 12345u);
          else
            k_gather<2><<<blocks, threads, smem>>>(out, iters, K, stride, 12345u);
        };
        launch();
        CK(cudaDeviceSynchronize());
        CK(cudaEventRecord(a));
        launch();
        CK(cudaEventRecord(b));
        CK(cudaEventSynchronize(b));
        float ms;
        CK(cudaEventElapsedTime(&ms, a, b));
        double instr = 16.0 * iters * (threads / 32) * (double)blocks / prop.multiProcessorCount;
        double cyc = ms * 1e-3 * clk_khz * 1e3;
        printf(", \"v%d_s%d_K%d\": %.3f", vec, stride, K, instr / cyc);
      }
  printf("}\n");
  return 0;
}
