// K1s consumer loop in isolation (no producers, symbols resident in shared
// memory, coefficients by __ldg as in K1s): 8 consumer warps with 4 row
// blocks per target (K1s, BO = 13 at p = 25, 2 warps per SMSP) against 16
// warps with 8 row blocks (BO = 7, 4 warps per SMSP, <= 128 registers) --
// does more warps per sub-partition lift the DFMA rate the register-operand
// bound caps at ~77% of the chain peak?
//
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -Xptxas -v \
//        -o tools/k1s_warps_bench tools/k1s_warps_bench.cu
#include <cstdio>
#include <cuda_runtime.h>

template <int V>
struct IC {
  static constexpr int value = V;
};
template <int N, typename F, int I = 0>
__device__ __forceinline__ void static_for(F&& f) {
  if constexpr (I < N) {
    f(IC<I>{});
    static_for<N, F, I + 1>(static_cast<F&&>(f));
  }
}
constexpr int kTT = 8;
template <int P, int NB>
struct Sh {
  static constexpr int L = 2 * P + 1, NS = 4 * P + 1, BO = (L + NB - 1) / NB, ROWS = BO * NB;
  static constexpr int FP = ROWS - L, NSP = FP + NS + 1, SJ = kTT * NSP + 1, SYM = kTT * SJ;
};

template <int P, int NB>
__device__ __forceinline__ void consume(const double2* __restrict__ sp, const double2* __restrict__ bsrc,
                                        const double* __restrict__ ssrc, double (&acc)[3][Sh<P, NB>::BO]) {
  using S = Sh<P, NB>;
  constexpr int BO = S::BO, R0 = S::FP + 2 * P, MODB = 64 * BO;
  double wx[BO], wy[BO], ws[BO];
  static_for<BO>([&](auto i_c) {
    constexpr int i = decltype(i_c)::value;
    const double2 t = sp[-i * kTT];
    constexpr int q = (R0 - i + MODB) % BO;
    wx[q] = t.x;
    wy[q] = t.y;
    ws[q] = t.x + t.y;
  });
  static_for<S::L>([&](auto n_c) {
    constexpr int n = decltype(n_c)::value;
    constexpr int u = n % BO;
    const double2 nxt = sp[(n + 1) * kTT];
    const double2 bb = __ldg(bsrc + n);
    const double bs = __ldg(ssrc + n);
#pragma unroll
    for (int i = 0; i < BO; ++i) acc[0][i] = fma(bb.x, wx[(R0 + u - i + MODB) % BO], acc[0][i]);
#pragma unroll
    for (int i = 0; i < BO; ++i) acc[1][i] = fma(bb.y, wy[(R0 + u - i + MODB) % BO], acc[1][i]);
#pragma unroll
    for (int i = 0; i < BO; ++i) acc[2][i] = fma(bs, ws[(R0 + u - i + MODB) % BO], acc[2][i]);
    constexpr int q = (R0 + u + 1 + MODB) % BO;
    wx[q] = nxt.x;
    wy[q] = nxt.y;
    ws[q] = nxt.x + nxt.y;
  });
}

// NB = 4: 8 warps, lane (h, b 2 bits, s 2 bits), warp = target; NB = 8: 16
// warps, lane (b 3 bits, s 2 bits), warp = (direction, target).  2 passes of
// 4 source slots per batch, __syncthreads per batch as in K1s.
template <int P, int NB, int NT>
__global__ void __launch_bounds__(NT, 1) bench(const double2* __restrict__ bw, const double* __restrict__ bws,
                                               int nbat, int nsrc, double* out) {
  using S = Sh<P, NB>;
  extern __shared__ double2 smem[];
  for (int i = threadIdx.x; i < 2 * S::SYM; i += NT) smem[i] = make_double2(1e-3 * (i % 97), 1e-3 * (i % 89));
  __syncthreads();
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  int h, b, sl, w;
  if constexpr (NB == 4) {
    h = lane >> 4; b = (lane >> 2) & 3; sl = lane & 3; w = warp;
  } else {
    h = warp >> 3; w = warp & 7; b = lane >> 2; sl = lane & 3;
  }
  double acc[3][S::BO];
#pragma unroll
  for (int c = 0; c < 3; ++c)
#pragma unroll
    for (int i = 0; i < S::BO; ++i) acc[c][i] = 0.0;
  constexpr int R0 = S::FP + 2 * P;
  for (int it = 0; it < nbat; ++it) {
    const double2* symc = (it & 1) ? smem + S::SYM : smem;
#pragma unroll
    for (int pass = 0; pass < 2; ++pass) {
      const int s = sl + 4 * pass;
      const int jj = h ? w : s, mm = h ? s : w;
      const int src = (blockIdx.x * 7 + it * 3 + s + 8 * h) % nsrc;
      const double2* rowp = symc + (size_t)jj * S::SJ + (size_t)(R0 - b * S::BO) * kTT + mm;
      consume<P, NB>(rowp, bw + (size_t)src * S::L, bws + (size_t)src * S::L, acc);
    }
    __syncthreads();
  }
  double t = 0;
#pragma unroll
  for (int c = 0; c < 3; ++c)
#pragma unroll
    for (int i = 0; i < S::BO; ++i) t += acc[c][i];
  if (t == 1234.5) out[0] = t;
}

template <int P, int NB, int NT>
void run(const char* name, double2* bw, double* bws, int nsrc, int sms, double* out) {
  using S = Sh<P, NB>;
  const size_t smem = 2 * S::SYM * sizeof(double2);
  cudaFuncSetAttribute(bench<P, NB, NT>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  const int nbat = 400;
  bench<P, NB, NT><<<sms, NT, smem>>>(bw, bws, 10, nsrc, out);
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  float best = 1e30f;
  for (int r = 0; r < 5; ++r) {
    cudaEventRecord(e0);
    bench<P, NB, NT><<<sms, NT, smem>>>(bw, bws, nbat, nsrc, out);
    cudaEventRecord(e1);
    cudaEventSynchronize(e1);
    float t;
    cudaEventElapsedTime(&t, e0, e1);
    if (t < best) best = t;
  }
  // executed DFMA per lane per batch: 2 passes x L steps x 3 BO
  const double dfma = 3.0 * S::BO * S::L * 2 * nbat * (double)NT * sms;
  const double useful = 3.0 * S::L * S::L * 2 * nbat * 256.0 * sms;   // 8 targets x 2 dirs x 4 srcs x 2 passes
  printf("%-28s p=%d BO=%d warps=%2d  %.3f ms  executed DFMA %.2f TF/s  useful %.2f TF/s  %s\n", name, P,
         S::BO, NT / 32, best, 2.0 * dfma / (best * 1e-3) / 1e12, 2.0 * useful / (best * 1e-3) / 1e12,
         cudaGetErrorString(cudaGetLastError()));
}

int main() {
  int sms = 0;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  const int nsrc = 3000;
  double2* bw;
  double* bws;
  double* out;
  cudaMalloc(&bw, nsrc * 51 * sizeof(double2));
  cudaMalloc(&bws, nsrc * 51 * sizeof(double));
  cudaMalloc(&out, 8);
  cudaMemset(bw, 0, nsrc * 51 * sizeof(double2));
  cudaMemset(bws, 0, nsrc * 51 * sizeof(double));
  run<25, 4, 256>("K1s layout (NB 4)", bw, bws, nsrc, sms, out);
  run<25, 8, 512>("NB 8, 16 warps", bw, bws, nsrc, sms, out);
  run<20, 4, 256>("K1s layout (NB 4)", bw, bws, nsrc, sms, out);
  run<20, 8, 512>("NB 8, 16 warps", bw, bws, nsrc, sms, out);
  return 0;
}
