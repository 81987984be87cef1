// Shared-memory gather layouts for the slot kernel's 1-d deep levels: each
// lane (point) reads the 8 columns of its own random row among K rows.
//   s9     : row stride 9 doubles, every lane reads column j at step j (current)
//   r16_b3 : stride 16, two copies of each row (bank pairs 0-7 / 8-15), lane
//            bit 3 picks the copy, lane reads column (lane + j) & 7
//   r16_b4 : same, lane bit 4 picks the copy
//   r16_p  : same as r16_b3, rotation by lane pair ((lane >> 1) + j) & 7
//   r8     : stride 8, single copy, column (lane + j) & 7
// Prints warp LDS.64 instructions per SM per clock.
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o lds_rotate lds_rotate.cu
#include <cstdio>
#include <cstdlib>
#include <cuda_runtime.h>

#define CK(x) do { cudaError_t e_ = (x); if (e_ != cudaSuccess) { \
  fprintf(stderr, "CUDA %s at %s:%d\n", cudaGetErrorString(e_), __FILE__, __LINE__); exit(1);} } while (0)

template <int kScheme>
__global__ void k_rot(unsigned long long* out, int iters, int K, unsigned seed) {
  extern __shared__ double sm[];
  for (int i = threadIdx.x; i < 256 * 16; i += blockDim.x) sm[i] = i;
  __syncthreads();
  const int lane = threadIdx.x & 31;
  unsigned h = seed ^ (threadIdx.x * 2654435761u) ^ (blockIdx.x * 97u);
  unsigned addr[8];
  const unsigned base = (unsigned)__cvta_generic_to_shared(sm);
#pragma unroll
  for (int j = 0; j < 8; ++j) {
    h = h * 1664525u + 1013904223u;
    const unsigned r = (h >> 8) % K;
    unsigned a;
    if (kScheme == 0) a = r * 9 + j;
    else if (kScheme == 1) a = r * 16 + 8 * ((lane >> 3) & 1) + ((lane + j) & 7);
    else if (kScheme == 2) a = r * 16 + 8 * ((lane >> 4) & 1) + ((lane + j) & 7);
    else if (kScheme == 3) a = r * 16 + 8 * ((lane >> 3) & 1) + (((lane >> 1) + j) & 7);
    else a = r * 8 + ((lane + j) & 7);
    addr[j] = base + a * 8;
  }
  unsigned long long acc = 0;
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int r = 0; r < 16; ++r) {
      unsigned long long v;
      asm volatile("ld.volatile.shared.b64 %0, [%1];" : "=l"(v) : "r"(addr[r & 7]));
      acc += v;
    }
  }
  if (acc == 0x12345ull) out[threadIdx.x] = acc;
}

template <int S>
double run(int K, int blocks, int threads, int iters, int clk_khz, int sms, unsigned long long* out) {
  cudaEvent_t a, b;
  CK(cudaEventCreate(&a));
  CK(cudaEventCreate(&b));
  const size_t smem = 256 * 16 * 8;
  k_rot<S><<<blocks, threads, smem>>>(out, iters, K, 12345u);
  CK(cudaDeviceSynchronize());
  CK(cudaEventRecord(a));
  k_rot<S><<<blocks, threads, smem>>>(out, iters, K, 12345u);
  CK(cudaEventRecord(b));
  CK(cudaEventSynchronize(b));
  float ms;
  CK(cudaEventElapsedTime(&ms, a, b));
  const double instr = 16.0 * iters * (threads / 32) * (double)blocks / sms;
  return instr / (ms * 1e-3 * clk_khz * 1e3);
}

int main() {
  cudaDeviceProp prop;
  CK(cudaGetDeviceProperties(&prop, 0));
  int clk_khz = 0;
  CK(cudaDeviceGetAttribute(&clk_khz, cudaDevAttrClockRate, 0));
  unsigned long long* out;
  CK(cudaMalloc(&out, 1 << 20));
  const int threads = 512, blocks = prop.multiProcessorCount * 2, iters = 2000, sms = prop.multiProcessorCount;
  const char* names[5] = {"s9", "r16_b3", "r16_b4", "r16_p", "r8"};
  printf("{");
  bool first = true;
  for (int K : {1, 2, 4, 8, 16, 32, 64, 128, 256}) {
    double v[5];
    v[0] = run<0>(K, blocks, threads, iters, clk_khz, sms, out);
    v[1] = run<1>(K, blocks, threads, iters, clk_khz, sms, out);
    v[2] = run<2>(K, blocks, threads, iters, clk_khz, sms, out);
    v[3] = run<3>(K, blocks, threads, iters, clk_khz, sms, out);
    v[4] = run<4>(K, blocks, threads, iters, clk_khz, sms, out);
    for (int s = 0; s < 5; ++s) {
      printf("%s\"%s_K%d\": %.3f", first ? "" : ", ", names[s], K, v[s]);
      first = false;
    }
  }
  printf("}\n");
  return 0;
}
