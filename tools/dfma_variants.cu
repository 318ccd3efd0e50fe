#include <cstdio>
#include <cuda_runtime.h>
template <int NC>
__global__ void chains(double* out, int iters, double a, double b) {
  double x[NC];
#pragma unroll
  for (int i = 0; i < NC; ++i) x[i] = threadIdx.x * 1e-3 + i;
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int i = 0; i < NC; ++i) x[i] = fma(x[i], a, b);
  }
  double s = 0;
#pragma unroll
  for (int i = 0; i < NC; ++i) s += x[i];
  if (s == 12345.678) out[0] = s;
}
// two distinct source operands per FMA (like the Toeplitz loop: acc += w[i]*b)
template <int NC>
__global__ void chains2(double* out, int iters, double b) {
  double x[NC], w[NC];
#pragma unroll
  for (int i = 0; i < NC; ++i) { x[i] = threadIdx.x * 1e-3 + i; w[i] = 0.999 + i * 1e-6; }
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int i = 0; i < NC; ++i) x[i] = fma(w[i], b, x[i]);
  }
  double s = 0;
#pragma unroll
  for (int i = 0; i < NC; ++i) s += x[i];
  if (s == 12345.678) out[0] = s;
}
template <typename K>
void run(const char* name, K k, int blocks, int threads, double fl_per_iter_thread, int iters) {
  double* d; cudaMalloc(&d, 8);
  cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
  k(d, iters / 8, blocks, threads);
  float best = 1e30f;
  for (int r = 0; r < 5; ++r) {
    cudaEventRecord(e0); k(d, iters, blocks, threads); cudaEventRecord(e1); cudaEventSynchronize(e1);
    float t; cudaEventElapsedTime(&t, e0, e1); if (t < best) best = t;
  }
  double fl = fl_per_iter_thread * iters * (double)blocks * threads;
  printf("%-28s blocks=%4d thr=%4d  %.2f TFLOP/s\n", name, blocks, threads, fl / (best * 1e-3) / 1e12);
  cudaFree(d);
}
int main() {
  int sms; cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  int it = 1 << 14;
  for (int occ : {2, 4, 8, 16}) {
    run("chains<16>", [](double* d, int i, int b, int t) { chains<16><<<b, t>>>(d, i, 0.9999999, 1e-7); }, sms * occ, 256, 32.0, it);
    run("chains<8>", [](double* d, int i, int b, int t) { chains<8><<<b, t>>>(d, i, 0.9999999, 1e-7); }, sms * occ, 256, 16.0, it);
    run("chains2<16>", [](double* d, int i, int b, int t) { chains2<16><<<b, t>>>(d, i, 1e-7); }, sms * occ, 256, 32.0, it);
    run("chains<32>", [](double* d, int i, int b, int t) { chains<32><<<b, t>>>(d, i, 0.9999999, 1e-7); }, sms * occ, 128, 64.0, it);
  }
  return 0;
}
