// FP64 roofline denominator: a DFMA-throughput microbenchmark (SURVEY.md F7:
// MEASURED_PEAKS.json carries no FP64 figure, so the box's own DFMA peak is
// measured and used for roofline.peak).  16 independent FMA chains per thread
// keep the DFMA pipe saturated; each FMA counts 2 flops.
#include <cuda_runtime.h>

#include "ctx.cuh"

namespace {

__global__ void __launch_bounds__(256) dfma_chains(double* out, int iters, double a, double b) {
  double x[16];
#pragma unroll
  for (int i = 0; i < 16; ++i) x[i] = threadIdx.x * 1e-3 + i;
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int i = 0; i < 16; ++i) x[i] = fma(x[i], a, b);
  }
  double s = 0;
#pragma unroll
  for (int i = 0; i < 16; ++i) s += x[i];
  if (s == 12345.678) out[0] = s;   // keep the chains alive
}

}  // namespace

// Back-to-back DFMA launches for ~seconds: the clock the FP64 pipe holds
// under a sustained load (power cap) -- the denominator for long kernels.
extern "C" int ps_dfma_sustained(int device, double seconds, double* tflops) {
  if (cudaSetDevice(device) != cudaSuccess) return PS_ERR_CUDA;
  int sms = 0;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, device);
  double* d = nullptr;
  if (cudaMalloc(&d, sizeof(double)) != cudaSuccess) return PS_ERR_CUDA;
  const int blocks = sms * 8, threads = 256, iters = 1 << 14;
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  dfma_chains<<<blocks, threads>>>(d, iters, 0.9999999, 1e-7);
  cudaEventRecord(e0);
  cudaEventRecord(e1);
  cudaEventSynchronize(e1);
  float one = 0;
  {
    cudaEventRecord(e0);
    dfma_chains<<<blocks, threads>>>(d, iters, 0.9999999, 1e-7);
    cudaEventRecord(e1);
    cudaEventSynchronize(e1);
    cudaEventElapsedTime(&one, e0, e1);
  }
  int reps = (int)(seconds * 1e3 / (one > 0 ? one : 1.0f));
  if (reps < 1) reps = 1;
  cudaEventRecord(e0);
  for (int r = 0; r < reps; ++r) dfma_chains<<<blocks, threads>>>(d, iters, 0.9999999, 1e-7);
  cudaEventRecord(e1);
  cudaEventSynchronize(e1);
  float t = 0;
  cudaEventElapsedTime(&t, e0, e1);
  cudaEventDestroy(e0);
  cudaEventDestroy(e1);
  cudaFree(d);
  if (cudaGetLastError() != cudaSuccess) return PS_ERR_CUDA;
  const double flops = 2.0 * 16.0 * (double)iters * blocks * threads * reps;
  *tflops = flops / (t * 1e-3) / 1e12;
  return PS_OK;
}

extern "C" int ps_dfma_peak(int device, double* tflops, double* ms) {
  if (cudaSetDevice(device) != cudaSuccess) return PS_ERR_CUDA;
  int sms = 0;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, device);
  double* d = nullptr;
  if (cudaMalloc(&d, sizeof(double)) != cudaSuccess) return PS_ERR_CUDA;
  const int blocks = sms * 8, threads = 256, iters = 1 << 14;
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  dfma_chains<<<blocks, threads>>>(d, iters / 16, 0.9999999, 1e-7);   // warm-up
  float best = 1e30f;
  for (int rep = 0; rep < 5; ++rep) {
    cudaEventRecord(e0);
    dfma_chains<<<blocks, threads>>>(d, iters, 0.9999999, 1e-7);
    cudaEventRecord(e1);
    cudaEventSynchronize(e1);
    float t = 0;
    cudaEventElapsedTime(&t, e0, e1);
    if (t < best) best = t;
  }
  cudaEventDestroy(e0);
  cudaEventDestroy(e1);
  cudaFree(d);
  if (cudaGetLastError() != cudaSuccess) return PS_ERR_CUDA;
  const double flops = 2.0 * 16.0 * (double)iters * blocks * threads;
  *ms = best;
  *tflops = flops / (best * 1e-3) / 1e12;
  return PS_OK;
}
