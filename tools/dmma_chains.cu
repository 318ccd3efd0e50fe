// DMMA (mma.sync m8n8k4 f64) throughput on B200 against the number of
// independent accumulator chains per warp and warps per SM sub-partition,
// with and without a DADD feeding one operand per step (the K1h Karatsuba
// B-sum pattern) -- what K1h needs to keep the FP64 tensor pipe busy.
//
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o tools/dmma_chains tools/dmma_chains.cu
#include <cstdio>
#include <cuda_runtime.h>

template <int CH, int DADD>
__global__ void k(double* out, int iters) {
  double a = 1.0 + threadIdx.x * 1e-9, b = 0.999999, e = 1e-12;
  double c[CH][2];
#pragma unroll
  for (int i = 0; i < CH; ++i) c[i][0] = c[i][1] = i * 1e-3;
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int i = 0; i < CH; ++i) {
      double bb = b;
      if (DADD && (i % 3 == 2)) {
        asm volatile("add.f64 %0, %1, %2;" : "=d"(bb) : "d"(b), "d"(e));
      }
      asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0, %1}, {%2}, {%3}, {%0, %1};"
                   : "+d"(c[i][0]), "+d"(c[i][1])
                   : "d"(a), "d"(bb));
    }
  }
  double s = 0;
#pragma unroll
  for (int i = 0; i < CH; ++i) s += c[i][0] + c[i][1];
  if (s == 12345.678) out[0] = s;
}

template <int CH, int DADD>
void run(int warps_per_sm, int sms) {
  double* d;
  cudaMalloc(&d, 8);
  const int iters = 4000;
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  k<CH, DADD><<<sms, warps_per_sm * 32>>>(d, 10);
  cudaEventRecord(e0);
  k<CH, DADD><<<sms, warps_per_sm * 32>>>(d, iters);
  cudaEventRecord(e1);
  cudaEventSynchronize(e1);
  float ms;
  cudaEventElapsedTime(&ms, e0, e1);
  const double fl = 512.0 * CH * iters * warps_per_sm * (double)sms;
  printf("chains/warp %2d  warps/SM %2d  dadd %d : %6.2f TF/s\n", CH, warps_per_sm, DADD,
         fl / (ms * 1e-3) / 1e12);
  cudaFree(d);
}

int main() {
  int sms = 0;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  for (int w : {4, 8, 12, 16}) {
    run<1, 0>(w, sms);
    run<2, 0>(w, sms);
    run<3, 0>(w, sms);
    run<3, 1>(w, sms);
    run<6, 0>(w, sms);
    run<6, 1>(w, sms);
    run<12, 0>(w, sms);
  }
  return 0;
}
