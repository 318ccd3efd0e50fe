// Per-SM streaming bandwidth on B200: how fast can a FEW SMs read a large
// array while the rest of the GPU is busy?  (The SM-partitioned Schur step
// streams ~0.93 GB of dense coupling blocks on 2 SMs beside K1s.)
//   (a) LDG.128 with deep unrolling, 1 CTA of 1024 threads per SM;
//   (b) cp.async.bulk (TMA, 1-D bulk) global -> shared, 1 producer thread,
//       NST stages of 32 KB in flight, mbarrier completion.
//
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o tools/sm_stream_bw tools/sm_stream_bw.cu
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>

__global__ void __launch_bounds__(1024) ldg_stream(const double2* __restrict__ a, size_t n,
                                                   double* out) {
  double sx = 0, sy = 0;
  const size_t stride = (size_t)gridDim.x * blockDim.x;
  size_t i = (size_t)blockIdx.x * blockDim.x + threadIdx.x;
  for (; i + 7 * stride < n; i += 8 * stride) {
    double2 v[8];
#pragma unroll
    for (int u = 0; u < 8; ++u) v[u] = __ldcs(a + i + u * stride);
#pragma unroll
    for (int u = 0; u < 8; ++u) {
      sx += v[u].x;
      sy += v[u].y;
    }
  }
  for (; i < n; i += stride) {
    sx += a[i].x;
    sy += a[i].y;
  }
  if (sx + sy == 1234.5) out[0] = sx;
}

constexpr int kStage = 32768;   // bytes per bulk copy
template <int NST>
__global__ void __launch_bounds__(128) tma_stream(const char* __restrict__ a, size_t bytes,
                                                  double* out) {
  extern __shared__ __align__(128) char buf[];
  __shared__ __align__(8) uint64_t bar[NST];
  const size_t chunks = bytes / kStage;
  const size_t per = (chunks + gridDim.x - 1) / gridDim.x;
  const size_t c0 = blockIdx.x * per, c1 = min(chunks, c0 + per);
  if (threadIdx.x == 0)
    for (int s = 0; s < NST; ++s)
      asm volatile("mbarrier.init.shared.b64 [%0], 1;" ::"r"((unsigned)__cvta_generic_to_shared(&bar[s])));
  __syncthreads();
  double acc = 0;
  auto issue = [&](size_t c, int s) {
    const unsigned b = (unsigned)__cvta_generic_to_shared(&bar[s]);
    const unsigned d = (unsigned)__cvta_generic_to_shared(buf + (size_t)s * kStage);
    asm volatile("mbarrier.arrive.expect_tx.shared.b64 _, [%0], %1;" ::"r"(b), "r"(kStage));
    asm volatile(
        "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(d),
        "l"(a + c * kStage), "r"(kStage), "r"(b)
        : "memory");
  };
  if (threadIdx.x == 0)
    for (int s = 0; s < NST && c0 + s < c1; ++s) issue(c0 + s, s);
  unsigned phase[NST];
  for (int s = 0; s < NST; ++s) phase[s] = 0;
  for (size_t c = c0; c < c1; ++c) {
    const int s = (int)((c - c0) % NST);
    const unsigned b = (unsigned)__cvta_generic_to_shared(&bar[s]);
    asm volatile(
        "{ .reg .pred p; W: mbarrier.try_wait.parity.shared.b64 p, [%0], %1; @!p bra W; }" ::"r"(b),
        "r"(phase[s]));
    phase[s] ^= 1;
    acc += reinterpret_cast<const double*>(buf + (size_t)s * kStage)[threadIdx.x];
    __syncthreads();
    if (threadIdx.x == 0 && c + NST < c1) issue(c + NST, s);
  }
  if (acc == 1234.5) out[0] = acc;
}

int main() {
  const size_t bytes = 512ull << 20;
  char* a;
  double* out;
  cudaMalloc(&a, bytes);
  cudaMalloc(&out, 8);
  cudaMemset(a, 0, bytes);
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  auto timeit = [&](auto launch) {
    launch();
    float best = 1e30f;
    for (int r = 0; r < 3; ++r) {
      cudaEventRecord(e0);
      launch();
      cudaEventRecord(e1);
      cudaEventSynchronize(e1);
      float t;
      cudaEventElapsedTime(&t, e0, e1);
      if (t < best) best = t;
    }
    return best;
  };
  for (int sms : {1, 2, 4, 148}) {
    const size_t nb = sms == 148 ? bytes : (64ull << 20) * sms;
    float t = timeit([&] { ldg_stream<<<sms, 1024>>>((const double2*)a, nb / 16, out); });
    printf("LDG  %3d SMs: %7.1f GB/s total, %6.1f GB/s per SM\n", sms, nb / (t * 1e-3) / 1e9,
           nb / (t * 1e-3) / 1e9 / sms);
  }
  constexpr int NST = 6;
  const size_t smem = (size_t)NST * kStage;
  cudaFuncSetAttribute(tma_stream<NST>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  for (int sms : {1, 2, 4, 148}) {
    const size_t nb = sms == 148 ? bytes : (64ull << 20) * sms;
    float t = timeit([&] { tma_stream<NST><<<sms, 128, smem>>>(a, nb, out); });
    printf("TMA  %3d SMs: %7.1f GB/s total, %6.1f GB/s per SM  (%s)\n", sms, nb / (t * 1e-3) / 1e9,
           nb / (t * 1e-3) / 1e9 / sms, cudaGetErrorString(cudaGetLastError()));
  }
  return 0;
}
