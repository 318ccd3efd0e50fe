// FP64 roofline denominator: a DFMA-throughput microbenchmark (SURVEY.md F7:
// MEASURED_PEAKS.json carries no FP64 figure, so the box's own DFMA peak is
// measured and used for roofline.peak).  Independent FMA chains keep the
// DFMA pipe saturated; each FMA counts 2 flops.  ps_dmma_peak measures the
// FP64 tensor path (mma.sync f64) for comparison.
#include <cuda_runtime.h>

#include "ctx.cuh"

namespace {

// 8 independent chains per thread at 8 CTAs of 256 threads per SM (64 warps,
// full residency): 36.5 TF/s on the B200, 98% of the nominal 148 x 64 x 2 x
// 1.965 GHz = 37.2 TF/s (tools/fp64_pipes.cu; the 16-CTA launch of round 1
// oversubscribed residency and read 34.2).
constexpr int kChains = 8;
constexpr int kCtasPerSm = 8;
// The multiplier and addend are literals (constant-bank operands), so every
// DFMA reads ONE vector register: with both as kernel arguments the second
// one occupies a register operand and the chain reads 34.2 TF/s -- the DFMA
// rate is bounded by register-file operand bandwidth (tools/fp64_pipes.cu,
// tools/k1s_consumer_bench.cu), not only by the pipe.
__global__ void __launch_bounds__(256) dfma_chains(double* out, int iters, double, double) {
  double x[kChains];
#pragma unroll
  for (int i = 0; i < kChains; ++i) x[i] = threadIdx.x * 1e-3 + i;
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int i = 0; i < kChains; ++i) x[i] = fma(x[i], 0.9999999, 1e-7);
  }
  double s = 0;
#pragma unroll
  for (int i = 0; i < kChains; ++i) s += x[i];
  if (s == 12345.678) out[0] = s;   // keep the chains alive
}

// FP64 tensor path: chains of mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64
// (256 FMA per warp-instruction), 8 independent accumulators per warp.
__global__ void __launch_bounds__(256) dmma_chains(double* out, int iters) {
  double a = 1.0 + threadIdx.x * 1e-9, b = 0.999999;
  double c[8][2];
#pragma unroll
  for (int i = 0; i < 8; ++i) c[i][0] = c[i][1] = i * 1e-3;
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int i = 0; i < 8; ++i)
      asm volatile(
          "mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0, %1}, {%2}, {%3}, {%0, %1};"
          : "+d"(c[i][0]), "+d"(c[i][1])
          : "d"(a), "d"(b));
  }
  double s = 0;
#pragma unroll
  for (int i = 0; i < 8; ++i) s += c[i][0] + c[i][1];
  if (s == 12345.678) out[0] = s;
}

}  // namespace

extern "C" int ps_dmma_peak(int device, double* tflops) {
  if (cudaSetDevice(device) != cudaSuccess) return PS_ERR_CUDA;
  int sms = 0;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, device);
  double* d = nullptr;
  if (cudaMalloc(&d, sizeof(double)) != cudaSuccess) return PS_ERR_CUDA;
  const int blocks = sms * 8, threads = 256, iters = 1 << 12;
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  dmma_chains<<<blocks, threads>>>(d, iters / 16);
  float best = 1e30f;
  for (int rep = 0; rep < 5; ++rep) {
    cudaEventRecord(e0);
    dmma_chains<<<blocks, threads>>>(d, iters);
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
  // per warp-instruction: 8 x 8 x 4 = 256 FMA = 512 flops
  const double flops = 512.0 * 8.0 * (double)iters * blocks * (threads / 32);
  *tflops = flops / (best * 1e-3) / 1e12;
  return PS_OK;
}

// Back-to-back DFMA launches for ~seconds: the clock the FP64 pipe holds
// under a sustained load (power cap) -- the denominator for long kernels.
extern "C" int ps_dfma_sustained(int device, double seconds, double* tflops) {
  if (cudaSetDevice(device) != cudaSuccess) return PS_ERR_CUDA;
  int sms = 0;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, device);
  double* d = nullptr;
  if (cudaMalloc(&d, sizeof(double)) != cudaSuccess) return PS_ERR_CUDA;
  const int blocks = sms * kCtasPerSm, threads = 256, iters = 1 << 14;
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
  const double flops = 2.0 * kChains * (double)iters * blocks * threads * reps;
  *tflops = flops / (t * 1e-3) / 1e12;
  return PS_OK;
}

extern "C" int ps_dfma_peak(int device, double* tflops, double* ms) {
  if (cudaSetDevice(device) != cudaSuccess) return PS_ERR_CUDA;
  int sms = 0;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, device);
  double* d = nullptr;
  if (cudaMalloc(&d, sizeof(double)) != cudaSuccess) return PS_ERR_CUDA;
  const int blocks = sms * kCtasPerSm, threads = 256, iters = 1 << 14;
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
  const double flops = 2.0 * kChains * (double)iters * blocks * threads;
  *ms = best;
  *tflops = flops / (best * 1e-3) / 1e12;
  return PS_OK;
}
