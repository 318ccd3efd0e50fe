// Isolated K1s consumer loop (m2l_sym.cu consume_s) on B200: 8 consumer warps
// per CTA (2 per SMSP), one CTA per SM, symbol rows in shared memory, the
// Bloch-weighted coefficients from global memory -- no producers.  Reports the
// executed-DFMA rate of variants against the ~36.5 TF/s DFMA-chain peak, to
// locate what costs the K1s consumers their pipe time.
//
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -Xptxas -v \
//        -o tools/k1s_consumer_bench tools/k1s_consumer_bench.cu
#include <cstdio>
#include <cstdlib>
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
template <int P, int kNB = 4>
struct Sh {
  static constexpr int L = 2 * P + 1, NS = 4 * P + 1, BO = (L + kNB - 1) / kNB, ROWS = BO * kNB;
  static constexpr int FP = ROWS - L, NSP = FP + NS + 1, SJ = kTT * NSP + 1, SYM = kTT * SJ;
};

// VB: 0 coefficients via __ldg per step (as K1s), 1 from shared memory,
//     2 fixed coefficients in registers (no loads), 3 = 2 and a fixed window
template <int P, int VB, int ORD = 0, int PF = 0, int NB = 4, int SWAP = 0>
__device__ __forceinline__ void consume(const double2* __restrict__ spe, const double2* __restrict__ spo,
                                        const double2* __restrict__ bsrc, const double* __restrict__ ssrc,
                                        double (&acc)[3][Sh<P, NB>::BO]) {
  using S = Sh<P, NB>;
  constexpr int BO = S::BO, R0 = S::FP + 2 * P, MODB = 64 * BO;
  auto ld = [&](auto t_c) -> double2 {
    constexpr int t = decltype(t_c)::value;
    constexpr bool odd = ((R0 + t) / BO) & 1;
    return (odd ? spo : spe)[t * kTT];
  };
  double wx[BO], wy[BO], ws[BO];
  static_for<BO>([&](auto i_c) {
    constexpr int i = decltype(i_c)::value;
    const double2 t = ld(IC<-i>{});
    constexpr int q = (R0 - i + MODB) % BO;
    wx[q] = t.x;
    wy[q] = t.y;
    ws[q] = t.x + t.y;
  });
  // PF > 0: explicit coefficient prefetch ring of depth PF (bs by DADD)
  double2 ring[PF > 0 ? PF : 1];
  if constexpr (PF > 0) {
    static_for<PF>([&](auto k_c) {
      constexpr int k = decltype(k_c)::value;
      ring[k] = __ldg(bsrc + k);
    });
  }
  auto step = [&](auto n_c) {
    constexpr int n = decltype(n_c)::value;
    constexpr int u = n % BO;
    const double2 nxt = ld(IC<n + 1>{});
    double2 bb;
    double bs;
    if constexpr (PF > 0) {
      bb = ring[n % PF];
      bs = bb.x + bb.y;
      if constexpr (n + PF < S::L) ring[n % PF] = __ldg(bsrc + n + PF);
    } else if constexpr (VB == 0) {
      bb = __ldg(bsrc + n);
      bs = __ldg(ssrc + n);
    } else if constexpr (VB == 1) {
      bb = bsrc[n];
      bs = ssrc[n];
    } else if constexpr (VB == 5) {
      bb = __ldg(bsrc + n * kTT);
      bs = __ldg(ssrc + n * kTT);
    } else {
      bb = make_double2(1.0 + 1e-9 * n, 1.0 - 1e-9 * n);
      bs = 1.0 + 2e-9 * n;
    }
    if constexpr (SWAP) {
#pragma unroll
      for (int i = 0; i < BO; ++i) acc[0][i] = fma(wx[(R0 + u - i + MODB) % BO], bb.x, acc[0][i]);
#pragma unroll
      for (int i = 0; i < BO; ++i) acc[1][i] = fma(wy[(R0 + u - i + MODB) % BO], bb.y, acc[1][i]);
#pragma unroll
      for (int i = 0; i < BO; ++i) acc[2][i] = fma(ws[(R0 + u - i + MODB) % BO], bs, acc[2][i]);
    } else if constexpr (ORD == 3) {   // descending rows: the newest symbol (i = 0) is used last in each run
#pragma unroll
      for (int i = BO - 1; i >= 0; --i) acc[0][i] = fma(bb.x, wx[(R0 + u - i + MODB) % BO], acc[0][i]);
#pragma unroll
      for (int i = BO - 1; i >= 0; --i) acc[1][i] = fma(bb.y, wy[(R0 + u - i + MODB) % BO], acc[1][i]);
#pragma unroll
      for (int i = BO - 1; i >= 0; --i) acc[2][i] = fma(bs, ws[(R0 + u - i + MODB) % BO], acc[2][i]);
    } else if constexpr (ORD == 0) {
#pragma unroll
      for (int i = 0; i < BO; ++i) acc[0][i] = fma(bb.x, wx[(R0 + u - i + MODB) % BO], acc[0][i]);
#pragma unroll
      for (int i = 0; i < BO; ++i) acc[1][i] = fma(bb.y, wy[(R0 + u - i + MODB) % BO], acc[1][i]);
#pragma unroll
      for (int i = 0; i < BO; ++i) acc[2][i] = fma(bs, ws[(R0 + u - i + MODB) % BO], acc[2][i]);
    } else {
#pragma unroll
      for (int i = 0; i < BO; ++i) {
        acc[0][i] = fma(bb.x, wx[(R0 + u - i + MODB) % BO], acc[0][i]);
        acc[1][i] = fma(bb.y, wy[(R0 + u - i + MODB) % BO], acc[1][i]);
        acc[2][i] = fma(bs, ws[(R0 + u - i + MODB) % BO], acc[2][i]);
      }
    }
    if constexpr (VB != 3) {
      constexpr int q = (R0 + u + 1 + MODB) % BO;
      wx[q] = nxt.x;
      wy[q] = nxt.y;
      ws[q] = nxt.x + nxt.y;
    }
  };
  if constexpr (VB == 6) {
    // runtime loop over chunks of BO steps (u = step within the chunk is
    // static), then the static tail
    constexpr int NC = S::L / BO, TL = S::L % BO;
    const double2* bsrc0 = bsrc;
    const double* ssrc0 = ssrc;
#pragma unroll 1
    for (int ch = 0; ch < NC; ++ch) {
      static_for<BO>([&](auto u_c) {
        constexpr int u = decltype(u_c)::value;
        const int n = ch * BO + u;
        const double2 nxt = (((R0 + 1 + u) / BO) & 1 ? spo : spe)[(n + 1) * kTT];
        const double2 bb = __ldg(bsrc0 + n);
        const double bs = __ldg(ssrc0 + n);
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
    static_for<TL>([&](auto u_c) { step(IC<NC * BO + decltype(u_c)::value>{}); });
  } else {
    static_for<S::L>(step);
  }
}

template <int P, int VB, int SYNC, int ORD = 0, int PF = 0, int NB = 4, int SWAP = 0>
__global__ void __launch_bounds__(256, 1) bench(const double2* __restrict__ bw, const double* __restrict__ bws,
                                                int nbat, int nsrc, double* out, int sstride) {
  using S = Sh<P, NB>;
  extern __shared__ double2 smem[];
  double2* sym = smem;
  double2* bsm = smem + 2 * S::SYM;                         // VB 1: 16 sources x L coefficients
  double* ssm = reinterpret_cast<double*>(bsm + 16 * S::L);
  for (int i = threadIdx.x; i < 2 * S::SYM; i += blockDim.x)
    sym[i] = make_double2(1e-3 * (i % 97), 1e-3 * (i % 89));
  if (VB == 1)
    for (int i = threadIdx.x; i < 16 * S::L; i += blockDim.x) {
      bsm[i] = bw[i];
      ssm[i] = bws[i];
    }
  __syncthreads();
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  // NB = 4: lane (h, b 2 bits, sl 2 bits), two passes of 4 sources;
  // NB = 2: lane (h, b 1 bit, sl 3 bits), one pass of 8 sources
  constexpr int SB = NB == 4 ? 2 : 3;
  const int h = lane >> 4, b = (lane >> SB) & (NB - 1), sl = lane & ((1 << SB) - 1);
  double acc[3][S::BO];
#pragma unroll
  for (int c = 0; c < 3; ++c)
#pragma unroll
    for (int i = 0; i < S::BO; ++i) acc[c][i] = 0.0;
  constexpr int R0 = S::FP + 2 * P;
  const int sw_e = 4 * (b & 1), sw_o = 4 * ((b & 1) ^ 1);
  for (int it = 0; it < nbat; ++it) {
    const double2* symc = (it & 1) ? sym + S::SYM : sym;
#pragma unroll
    for (int pass = 0; pass < (NB == 4 ? 2 : 1); ++pass) {
      const int s = sl + 4 * pass;
      const int jj = h ? warp : s, mm = h ? s : warp;
      const int src = (blockIdx.x * 7 + it * sstride + s + 8 * h) % nsrc;
      const double2* rowp = symc + (size_t)jj * S::SJ + (size_t)(R0 - b * S::BO) * kTT;
      if (VB == 5) {
        const int tsrc = ((blockIdx.x * 7 + it * 3 + h) % (nsrc / kTT));
        const size_t o = (size_t)tsrc * S::L * kTT + s;
        consume<P, VB, ORD, PF, NB, SWAP>(rowp + (mm ^ sw_e), rowp + (mm ^ sw_o), bw + o, bws + o, acc);
      } else if (VB == 0 || VB >= 2)
        consume<P, VB, ORD, PF, NB, SWAP>(rowp + (mm ^ sw_e), rowp + (mm ^ sw_o), bw + (size_t)src * S::L,
                       bws + (size_t)src * S::L, acc);
      else
        consume<P, 1, ORD, PF, NB, SWAP>(rowp + (mm ^ sw_e), rowp + (mm ^ sw_o), bsm + (size_t)(s + 8 * h) * S::L,
                      ssm + (size_t)(s + 8 * h) * S::L, acc);
    }
    if (SYNC) __syncthreads();
  }
  double t = 0;
#pragma unroll
  for (int c = 0; c < 3; ++c)
#pragma unroll
    for (int i = 0; i < S::BO; ++i) t += acc[c][i];
  if (t == 1234.5) out[0] = t;
}

static int g_stride = 3;   // sources advance per batch: 3 = neighbouring batches share rows (L1 hits), 16 = fresh rows every batch (K1s)
template <int P, int VB, int SYNC, int ORD = 0, int PF = 0, int NB = 4, int SWAP = 0>
void run(const char* name, double2* bw, double* bws, int nsrc, int sms, double* out, int threads = 256) {
  using S = Sh<P, NB>;
  const size_t smem = (2 * S::SYM + 16 * S::L) * sizeof(double2) + 16 * S::L * sizeof(double);
  cudaFuncSetAttribute(bench<P, VB, SYNC, ORD, PF, NB, SWAP>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  const int nbat = 400;
  bench<P, VB, SYNC, ORD, PF, NB, SWAP><<<sms, threads, smem>>>(bw, bws, 10, nsrc, out, g_stride);
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  float best = 1e30f;
  for (int r = 0; r < 5; ++r) {
    cudaEventRecord(e0);
    bench<P, VB, SYNC, ORD, PF, NB, SWAP><<<sms, threads, smem>>>(bw, bws, nbat, nsrc, out, g_stride);
    cudaEventRecord(e1);
    cudaEventSynchronize(e1);
    float t;
    cudaEventElapsedTime(&t, e0, e1);
    if (t < best) best = t;
  }
  const double dfma = 3.0 * S::BO * S::L * (NB == 4 ? 2 : 1) * nbat * (double)threads * sms;
  printf("%-34s p=%d smem %6zu  %.3f ms  executed DFMA %.2f TF/s  %s\n", name, P, smem, best,
         2.0 * dfma / (best * 1e-3) / 1e12, cudaGetErrorString(cudaGetLastError()));
}

int main(int argc, char** argv) {
  if (argc > 1) g_stride = atoi(argv[1]);
  printf("source stride per batch %d\n", g_stride);
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
  run<25, 0, 1>("ldg coef + sync (K1s)", bw, bws, nsrc, sms, out);
  run<25, 0, 1, 3>("descending rows", bw, bws, nsrc, sms, out);
  run<25, 0, 1>("same, 1 warp per SMSP", bw, bws, nsrc, sms, out, 128);
  run<25, 0, 0>("same, no sync", bw, bws, nsrc, sms, out);
  run<25, 0, 0>("same, no sync, 1 warp per SMSP", bw, bws, nsrc, sms, out, 128);
  run<25, 2, 0>("fixed coef regs, no sync", bw, bws, nsrc, sms, out);
  run<25, 2, 0>("fixed coef regs, no sync, 1 warp", bw, bws, nsrc, sms, out, 128);
  run<25, 6, 1>("ldg, chunked runtime loop", bw, bws, nsrc, sms, out);
  run<20, 0, 1>("ldg coef + sync (K1s)", bw, bws, nsrc, sms, out);
  run<20, 6, 1>("ldg, chunked runtime loop", bw, bws, nsrc, sms, out);
  return 0;
}
