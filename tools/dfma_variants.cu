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

// mixed: warps with (warp & 1) == 0 run DFMA chains, odd warps run DMMA
// chains (mma.sync m8n8k4 f64): do the two FP64 paths share one pipe?
// mode 0: all DFMA, 1: all DMMA, 2: half/half
__global__ void mixed(double* out, int iters, int mode) {
  const int w = threadIdx.x >> 5;
  const bool use_mma = mode == 1 || (mode == 2 && (w & 1));
  double s = 0;
  if (use_mma) {
    double a = 1.0 + threadIdx.x * 1e-9, b = 0.999999;
    double c[8][2];
#pragma unroll
    for (int i = 0; i < 8; ++i) c[i][0] = c[i][1] = i * 1e-3;
    for (int it = 0; it < iters / 8; ++it) {
#pragma unroll
      for (int i = 0; i < 8; ++i)
        asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0, %1}, {%2}, {%3}, {%0, %1};"
                     : "+d"(c[i][0]), "+d"(c[i][1]) : "d"(a), "d"(b));
    }
#pragma unroll
    for (int i = 0; i < 8; ++i) s += c[i][0] + c[i][1];
  } else {
    double x[16], wv[16];
#pragma unroll
    for (int i = 0; i < 16; ++i) { x[i] = threadIdx.x * 1e-3 + i; wv[i] = 0.999 + i * 1e-6; }
    for (int it = 0; it < iters; ++it) {
#pragma unroll
      for (int i = 0; i < 16; ++i) x[i] = fma(wv[i], 1e-7, x[i]);
    }
#pragma unroll
    for (int i = 0; i < 16; ++i) s += x[i];
  }
  if (s == 12345.678) out[0] = s;
}

// half-active warps: do DFMA instructions with 16 of 32 lanes predicated
// off cost half the FP64 pipe time?  mode 0: all lanes, 1: lanes 0-15 only,
// 2: even lanes only
__global__ void halfwarp(double* out, int iters, int mode) {
  const int lane = threadIdx.x & 31;
  const bool on = mode == 0 || (mode == 1 && lane < 16) || (mode == 2 && !(lane & 1));
  double x[16], wv[16];
#pragma unroll
  for (int i = 0; i < 16; ++i) { x[i] = threadIdx.x * 1e-3 + i; wv[i] = 0.999 + i * 1e-6; }
  if (on) {
    for (int it = 0; it < iters; ++it) {
#pragma unroll
      for (int i = 0; i < 16; ++i) x[i] = fma(wv[i], 1e-7, x[i]);
    }
  }
  double s = 0;
#pragma unroll
  for (int i = 0; i < 16; ++i) s += x[i];
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
int main(int argc, char** argv) {
  int sms; cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  int it = 1 << 14;
  if (argc > 1 && argv[1][0] == 'h') {
    for (int mode = 0; mode < 3; ++mode) {
      double* d; cudaMalloc(&d, 8);
      cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
      halfwarp<<<sms * 4, 256>>>(d, 1024, mode);
      float best = 1e30f;
      for (int r = 0; r < 3; ++r) {
        cudaEventRecord(e0); halfwarp<<<sms * 4, 256>>>(d, it, mode); cudaEventRecord(e1); cudaEventSynchronize(e1);
        float t; cudaEventElapsedTime(&t, e0, e1); if (t < best) best = t;
      }
      printf("halfwarp mode=%d  %.3f ms (same warp-instruction count in every mode)\n", mode, best);
      cudaFree(d);
    }
    return 0;
  }
  if (argc > 1 && argv[1][0] == 'm') {
    // per-warp flops per iteration: DFMA warp 32 thr x 16 fma x 2; DMMA warp 8/8 iters x 8 mma x 512
    for (int thr : {256, 512, 1024}) {
      for (int mode = 0; mode < 3; ++mode) {
        double* d; cudaMalloc(&d, 8);
        cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
        mixed<<<sms, thr>>>(d, 1024, mode);
        float best = 1e30f;
        for (int r = 0; r < 3; ++r) {
          cudaEventRecord(e0); mixed<<<sms, thr>>>(d, it, mode); cudaEventRecord(e1); cudaEventSynchronize(e1);
          float t; cudaEventElapsedTime(&t, e0, e1); if (t < best) best = t;
        }
        const int warps = thr / 32;
        const int wm = mode == 0 ? 0 : mode == 1 ? warps : warps / 2;
        const double fl = (double)sms * ((warps - wm) * 32.0 * 16 * 2 * it + wm * (it / 8) * 8.0 * 512);
        printf("mixed mode=%d thr=%4d  %.2f TFLOP/s\n", mode, thr, fl / (best * 1e-3) / 1e12);
        cudaFree(d);
      }
    }
    return 0;
  }
  if (argc > 1) {   // warps-per-SMSP sweep at one CTA per SM (the K1s shape)
    for (int thr : {128, 256, 384, 512}) {
      run("chains2<26>", [](double* d, int i, int b, int t) { chains2<26><<<b, t>>>(d, i, 1e-7); }, sms, thr, 52.0, it);
      run("chains2<52>", [](double* d, int i, int b, int t) { chains2<52><<<b, t>>>(d, i, 1e-7); }, sms, thr, 104.0, it / 2);
    }
    return 0;
  }
  for (int occ : {2, 4, 8, 16}) {
    run("chains<16>", [](double* d, int i, int b, int t) { chains<16><<<b, t>>>(d, i, 0.9999999, 1e-7); }, sms * occ, 256, 32.0, it);
    run("chains<8>", [](double* d, int i, int b, int t) { chains<8><<<b, t>>>(d, i, 0.9999999, 1e-7); }, sms * occ, 256, 16.0, it);
    run("chains2<16>", [](double* d, int i, int b, int t) { chains2<16><<<b, t>>>(d, i, 1e-7); }, sms * occ, 256, 32.0, it);
    run("chains<32>", [](double* d, int i, int b, int t) { chains<32><<<b, t>>>(d, i, 0.9999999, 1e-7); }, sms * occ, 128, 64.0, it);
  }
  return 0;
}
