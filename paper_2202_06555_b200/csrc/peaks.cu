// Live FP64 peak probe (roofline denominator).  MEASURED_PEAKS.json carries
// HBM and bf16 only; the DDSG path is FP64-bound, so bench.py measures the
// DFMA and DMMA (mma.sync f64) issue-rate peaks on the box it runs on.
#include <cuda_runtime.h>

#include "../../include/ddsg_b200.h"
#include "device.cuh"

namespace ddsg_b200 {
namespace {

constexpr int kChains = 8;

__global__ void peak_dfma_kernel(double* out, int iters, double a, double b) {
  double acc[kChains];
#pragma unroll
  for (int i = 0; i < kChains; ++i) acc[i] = threadIdx.x * 1e-3 + i;
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int r = 0; r < 8; ++r)
#pragma unroll
      for (int i = 0; i < kChains; ++i) acc[i] = __fma_rn(acc[i], a, b);
  }
  double s = 0;
#pragma unroll
  for (int i = 0; i < kChains; ++i) s += acc[i];
  if (s == 12345.678) out[threadIdx.x] = s;
}

__global__ void peak_dmma_kernel(double* out, int iters) {
  double a = threadIdx.x * 1e-3, b = 1.0 - threadIdx.x * 1e-4;
  double c[4][2];
#pragma unroll
  for (int i = 0; i < 4; ++i) c[i][0] = c[i][1] = 0;
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int r = 0; r < 8; ++r)
#pragma unroll
      for (int i = 0; i < 4; ++i)
        asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
                     : "+d"(c[i][0]), "+d"(c[i][1])
                     : "d"(a), "d"(b));
  }
  double s = 0;
#pragma unroll
  for (int i = 0; i < 4; ++i) s += c[i][0] + c[i][1];
  if (s == 12345.678) out[threadIdx.x] = s;
}

template <typename F>
float best_ms(F launch) {
  cudaEvent_t a, b;
  DDSG_CUDA(cudaEventCreate(&a));
  DDSG_CUDA(cudaEventCreate(&b));
  launch();
  DDSG_CUDA(cudaDeviceSynchronize());
  float best = 1e30f;
  for (int rep = 0; rep < 5; ++rep) {
    DDSG_CUDA(cudaEventRecord(a));
    launch();
    DDSG_CUDA(cudaEventRecord(b));
    DDSG_CUDA(cudaEventSynchronize(b));
    float ms = 0.f;
    DDSG_CUDA(cudaEventElapsedTime(&ms, a, b));
    best = ms < best ? ms : best;
  }
  DDSG_CUDA(cudaGetLastError());
  cudaEventDestroy(a);
  cudaEventDestroy(b);
  return best;
}

}  // namespace
}  // namespace ddsg_b200

extern "C" ddsg_status ddsg_measure_fp64_peak(double* dfma_tflops, double* dmma_tflops) {
  using namespace ddsg_b200;
  try {
    int dev = 0, sms = 0;
    DDSG_CUDA(cudaGetDevice(&dev));
    DDSG_CUDA(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev));
    double* out = nullptr;
    DDSG_CUDA(cudaMalloc(&out, 1 << 16));
    const int threads = 512, blocks = sms * 4;
    const int it1 = 4000, it2 = 2000;
    const float ms1 = best_ms([&] { peak_dfma_kernel<<<blocks, threads>>>(out, it1, 0.999, 1e-3); });
    const float ms2 = best_ms([&] { peak_dmma_kernel<<<blocks, threads>>>(out, it2); });
    cudaFree(out);
    if (dfma_tflops) *dfma_tflops = 2.0 * kChains * 8.0 * it1 * threads * static_cast<double>(blocks) / ms1 / 1e9;
    if (dmma_tflops)
      *dmma_tflops = 2.0 * 256.0 * 4 * 8 * it2 * (threads / 32) * static_cast<double>(blocks) / ms2 / 1e9;
    return DDSG_OK;
  } catch (const Error& e) {
    return e.status;
  }
}
