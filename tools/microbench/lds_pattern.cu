// Which lane -> row mappings does a warp LDS.64 serve in one shared-memory
// cycle?  Each pattern gives row(lane) explicitly; all lanes read column c
// of their row (row stride 9 doubles).  Prints warp-instructions/SM/clk.
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o lds_pattern lds_pattern.cu
#include <cstdio>
#include <cstdlib>
#include <cuda_runtime.h>

#define CK(x) do { cudaError_t e_ = (x); if (e_ != cudaSuccess) { \
  fprintf(stderr, "CUDA %s at %s:%d\n", cudaGetErrorString(e_), __FILE__, __LINE__); exit(1);} } while (0)

__global__ void k_pat(unsigned long long* out, int iters, const int* rows_of_lane, const int* cols_of_lane, int stride) {
  extern __shared__ double sm[];
  for (int i = threadIdx.x; i < 256 * stride; i += blockDim.x) sm[i] = i;
  __syncthreads();
  const int lane = threadIdx.x & 31;
  const unsigned base = (unsigned)__cvta_generic_to_shared(sm);
  const unsigned a0 = base + (rows_of_lane[lane] * stride + cols_of_lane[lane]) * 8;
  unsigned long long acc = 0;
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int r = 0; r < 16; ++r) {
      unsigned long long v;
      asm volatile("ld.volatile.shared.b64 %0, [%1];" : "=l"(v) : "r"(a0 + (r & 3) * 16));
      acc += v;
    }
  }
  if (acc == 0x12345ull) out[threadIdx.x] = acc;
}

int main() {
  cudaDeviceProp prop;
  CK(cudaGetDeviceProperties(&prop, 0));
  int clk_khz = 0;
  CK(cudaDeviceGetAttribute(&clk_khz, cudaDevAttrClockRate, 0));
  unsigned long long* out;
  int* d_rows;
  int* d_cols;
  CK(cudaMalloc(&out, 1 << 20));
  CK(cudaMalloc(&d_rows, 32 * sizeof(int)));
  CK(cudaMalloc(&d_cols, 32 * sizeof(int)));
  struct Pat { const char* name; int rows[32]; int cols[32]; int stride; };
  Pat pats[32];
  int np = 0;
  auto add = [&](const char* name, auto f, auto g, int stride) {
    pats[np].name = name;
    for (int l = 0; l < 32; ++l) { pats[np].rows[l] = f(l); pats[np].cols[l] = g(l); }
    pats[np].stride = stride;
    ++np;
  };
  auto zero = [](int) { return 0; };
  auto pair = [](int l) { return l & 1; };
  static const int R16[16] = {3, 11, 7, 0, 14, 5, 9, 1, 12, 6, 15, 2, 10, 4, 13, 8};
  static const int R8[16] = {3, 1, 7, 0, 4, 5, 6, 1, 2, 6, 3, 2, 0, 4, 5, 7};
  add("all_same", [](int) { return 0; }, zero, 9);
  add("halves_2rows", [](int l) { return l / 16; }, zero, 9);
  add("alternate_2rows", [](int l) { return l & 1; }, zero, 9);
  add("quarters_ABAB", [](int l) { return (l / 8) & 1; }, zero, 9);
  add("mod16", [](int l) { return l % 16; }, zero, 9);
  add("div2_16rows", [](int l) { return l / 2; }, zero, 9);
  add("div4_8rows", [](int l) { return l / 4; }, zero, 9);
  add("mod8", [](int l) { return l % 8; }, zero, 9);
  add("div8_4rows", [](int l) { return l / 8; }, zero, 9);
  add("halfsame_then_distinct", [](int l) { return l < 16 ? 0 : l - 15; }, zero, 9);
  add("distinct32", [](int l) { return l; }, zero, 9);
  add("sorted_rand16", [](int l) { static const int r[32] = {0,0,1,1,1,2,3,3,4,5,5,5,6,7,7,8,8,9,9,10,10,10,11,12,12,13,13,14,14,15,15,15}; return r[l]; }, zero, 9);
  add("sorted_rand8", [](int l) { static const int r[32] = {0,0,0,0,1,1,1,2,2,2,2,2,3,3,3,3,4,4,4,4,4,5,5,5,6,6,6,6,7,7,7,7}; return r[l]; }, zero, 9);
  add("morton_like_2x2", [](int l) { return ((l >> 0) & 1) + 2 * ((l >> 4) & 1); }, zero, 9);
  add("pairs_rand16_adjcols_s10", [](int l) { return R16[l >> 1]; }, pair, 10);
  add("pairs_rand16_adjcols_s9", [](int l) { return R16[l >> 1]; }, pair, 9);
  add("pairs_rand8_adjcols_s10", [](int l) { return R8[l >> 1]; }, pair, 10);
  add("pairs_rand16_samecol_s9", [](int l) { return R16[l >> 1]; }, zero, 9);
  add("quads_rand8_4cols_s10", [](int l) { return R16[l >> 2] & 7; }, [](int l) { return l & 3; }, 10);
  const int threads = 512, blocks = prop.multiProcessorCount * 2, iters = 2000;
  cudaEvent_t a, b;
  CK(cudaEventCreate(&a));
  CK(cudaEventCreate(&b));
  printf("{");
  for (int p = 0; p < np; ++p) {
    CK(cudaMemcpy(d_rows, pats[p].rows, sizeof(pats[p].rows), cudaMemcpyHostToDevice));
    CK(cudaMemcpy(d_cols, pats[p].cols, sizeof(pats[p].cols), cudaMemcpyHostToDevice));
    size_t smem = 256 * 10 * 8;
    k_pat<<<blocks, threads, smem>>>(out, iters, d_rows, d_cols, pats[p].stride);
    CK(cudaDeviceSynchronize());
    CK(cudaEventRecord(a));
    k_pat<<<blocks, threads, smem>>>(out, iters, d_rows, d_cols, pats[p].stride);
    CK(cudaEventRecord(b));
    CK(cudaEventSynchronize(b));
    float ms;
    CK(cudaEventElapsedTime(&ms, a, b));
    double instr = 16.0 * iters * (threads / 32) * (double)blocks / prop.multiProcessorCount;
    double cyc = ms * 1e-3 * clk_khz * 1e3;
    printf("%s\"%s\": %.3f", p ? ", " : "", pats[p].name, instr / cyc);
  }
  printf("}\n");
  return 0;
}
