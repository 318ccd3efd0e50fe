// FP64 pipe microbenchmark (B200): DFMA chains, DMMA (mma.sync m8n8k4 f64)
// chains, and both at once in one kernel (some warps DMMA, the others DFMA)
// -- do the FP64 vector pipe and the FP64 tensor sub-pipe overlap?
//
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o tools/fp64_pipes tools/fp64_pipes.cu
#include <cstdio>
#include <cuda_runtime.h>

template <int CH>
__device__ __forceinline__ void dfma_body(int iters, double& sink) {
  double x[CH];
#pragma unroll
  for (int i = 0; i < CH; ++i) x[i] = threadIdx.x * 1e-3 + i;
  const double a = 0.9999999, b = 1e-7;
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int i = 0; i < CH; ++i) x[i] = fma(x[i], a, b);
  }
  double s = 0;
#pragma unroll
  for (int i = 0; i < CH; ++i) s += x[i];
  sink = s;
}

template <int CH>
__device__ __forceinline__ void dmma_body(int iters, double& sink) {
  double a = 1.0 + threadIdx.x * 1e-9, b = 0.999999;
  double c[CH][2];
#pragma unroll
  for (int i = 0; i < CH; ++i) c[i][0] = c[i][1] = i * 1e-3;
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int i = 0; i < CH; ++i)
      asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0, %1}, {%2}, {%3}, {%0, %1};"
                   : "+d"(c[i][0]), "+d"(c[i][1])
                   : "d"(a), "d"(b));
  }
  double s = 0;
#pragma unroll
  for (int i = 0; i < CH; ++i) s += c[i][0] + c[i][1];
  sink = s;
}

// mode 0: all DFMA; 1: all DMMA; 2: warps with (warp % 2 == 0) DMMA, odd DFMA
template <int CHF, int CHM>
__global__ void mixed(double* out, int fiters, int miters, int mode) {
  double s = 0;
  const int warp = threadIdx.x >> 5;
  const bool mma = mode == 1 || (mode == 2 && (warp & 1) == 0);
  if (mma)
    dmma_body<CHM>(miters, s);
  else
    dfma_body<CHF>(fiters, s);
  if (s == 12345.678) out[0] = s;
}

int main() {
  int sms = 0;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  double* d;
  cudaMalloc(&d, 8);
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  auto run = [&](auto kern, int blocks, int threads, int fi, int mi, int mode, const char* name) {
    kern<<<blocks, threads>>>(d, fi / 16, mi / 16, mode);
    float best = 1e30f;
    for (int r = 0; r < 5; ++r) {
      cudaEventRecord(e0);
      kern<<<blocks, threads>>>(d, fi, mi, mode);
      cudaEventRecord(e1);
      cudaEventSynchronize(e1);
      float t;
      cudaEventElapsedTime(&t, e0, e1);
      if (t < best) best = t;
    }
    printf("%-40s blocks %5d threads %4d  %.3f ms\n", name, blocks, threads, best);
    return best;
  };
  const int fit = 1 << 14, mit = 1 << 12;
  // DFMA-only rates at a few ILP / occupancy points
  {
    float t = run(mixed<8, 8>, sms * 8, 256, fit, mit, 0, "dfma ch8 8x256");
    printf("  DFMA TF/s %.2f\n", 2.0 * 8 * fit * (double)sms * 8 * 256 / (t * 1e-3) / 1e12);
    t = run(mixed<16, 8>, sms * 4, 256, fit, mit, 0, "dfma ch16 4x256");
    printf("  DFMA TF/s %.2f\n", 2.0 * 16 * fit * (double)sms * 4 * 256 / (t * 1e-3) / 1e12);
    t = run(mixed<4, 8>, sms * 8, 256, fit, mit, 0, "dfma ch4 8x256");
    printf("  DFMA TF/s %.2f\n", 2.0 * 4 * fit * (double)sms * 8 * 256 / (t * 1e-3) / 1e12);
    t = run(mixed<8, 8>, sms * 1, 384, fit, mit, 0, "dfma ch8 1x384 (12 warps/SM)");
    printf("  DFMA TF/s %.2f\n", 2.0 * 8 * fit * (double)sms * 1 * 384 / (t * 1e-3) / 1e12);
    t = run(mixed<8, 8>, sms * 1, 256, fit, mit, 0, "dfma ch8 1x256 (2 warps/SMSP)");
    printf("  DFMA TF/s %.2f\n", 2.0 * 8 * fit * (double)sms * 1 * 256 / (t * 1e-3) / 1e12);
    t = run(mixed<16, 8>, sms * 1, 256, fit, mit, 0, "dfma ch16 1x256 (2 warps/SMSP)");
    printf("  DFMA TF/s %.2f\n", 2.0 * 16 * fit * (double)sms * 1 * 256 / (t * 1e-3) / 1e12);
    t = run(mixed<40, 8>, sms * 1, 256, fit / 4, mit, 0, "dfma ch40 1x256 (2 warps/SMSP)");
    printf("  DFMA TF/s %.2f\n", 2.0 * 40 * (fit / 4) * (double)sms * 1 * 256 / (t * 1e-3) / 1e12);
    t = run(mixed<40, 8>, sms * 1, 128, fit / 4, mit, 0, "dfma ch40 1x128 (1 warp/SMSP)");
    printf("  DFMA TF/s %.2f\n", 2.0 * 40 * (fit / 4) * (double)sms * 1 * 128 / (t * 1e-3) / 1e12);
    t = run(mixed<16, 8>, sms * 1, 128, fit, mit, 0, "dfma ch16 1x128 (1 warp/SMSP)");
    printf("  DFMA TF/s %.2f\n", 2.0 * 16 * fit * (double)sms * 1 * 128 / (t * 1e-3) / 1e12);
  }
  {
    float t = run(mixed<8, 8>, sms * 8, 256, fit, mit, 1, "dmma ch8 8x256");
    printf("  DMMA TF/s %.2f\n", 512.0 * 8 * mit * (double)sms * 8 * 8 / (t * 1e-3) / 1e12);
  }
  // mixed: half the warps DMMA, half DFMA; iteration counts chosen so each
  // half alone takes about the same time
  for (int scale : {1, 2}) {
    const int mi = mit, fi = fit * scale / 2;
    float t = run(mixed<8, 8>, sms * 8, 256, fi, mi, 2, "mixed half/half");
    const double fl_mma = 512.0 * 8 * mi * (double)sms * 8 * 4;   // 4 of 8 warps
    const double fl_fma = 2.0 * 8 * fi * (double)sms * 8 * 128;    // 128 threads
    printf("  combined TF/s %.2f (dmma part %.2f, dfma part %.2f over the whole time)\n",
           (fl_mma + fl_fma) / (t * 1e-3) / 1e12, fl_mma / (t * 1e-3) / 1e12,
           fl_fma / (t * 1e-3) / 1e12);
  }
  return 0;
}
