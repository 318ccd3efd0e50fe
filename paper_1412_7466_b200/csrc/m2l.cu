// K1: all-pairs Graf M2L translation (multiscat.apply_T, SPEC.md:504-512,
// PAPER.md:690-692 + 758-763; pinned formula SURVEY.md A.1):
//
//   a_m[m'] = sum_{l=-P..P} sum_{j, (l,j) != (0,m)} bloch^l
//             sum_n beta_j[n] H_{n-m'}(k2 rho) e^{i(n-m') phi},
//   (rho, phi) = polar(x_m - x_j - l d e_x).
//
// Work decomposition (one CTA per SM, persistent over a contiguous range of
// the (target tile x source batch) work list):
//   * a target tile is kTT = 8 targets, a source batch kS = 8 source images;
//   * 4 producer warps build the 64 symbol rows t_{-2p..2p} of the next batch
//     into shared memory (one pair per lane, bessel.cuh/symbols.cuh) and stage
//     the batch's bloch-weighted beta vectors;
//   * 8 consumer warps (one per source image of the current batch) apply the
//     Toeplitz sums: lane (b, t) owns rows [b*BO, b*BO+BO) of target t and
//     streams the L columns with a BO-deep sliding window of symbols held in
//     registers; complex MACs use the Karatsuba form, so every column step is
//     3 LDS (beta broadcast, its re+im, one symbol) against 3*BO DFMA;
//   * setmaxnreg splits the register file 216 (consumers) / 72 (producers);
//   * the two roles are double-buffered around one __syncthreads per batch;
//   * at a tile boundary the 8 consumer warps reduce their accumulators
//     through shared memory and write one partial per (CTA, tile segment);
//     m2l_reduce sums the partials in CTA order (deterministic) and applies
//     the Schur epilogue y = v - S (a - b).
#include <cuda_runtime.h>

#include "ctx.cuh"
#include "m2l.cuh"
#include "symbols.cuh"

namespace ps {

namespace {

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

constexpr int kTT = 8;                 // targets per tile
constexpr int kNB = 4;                 // row blocks (lanes) per target
constexpr int kS = 8;                  // source images per batch = consumer warps
#ifndef PS_K1_PW
#define PS_K1_PW 4
#endif
constexpr int kPW = PS_K1_PW;          // producer warps (one per SM sub-partition at 4)
constexpr int kThreads = (kS + kPW) * 32;
constexpr int kPairs = kTT * kS;       // symbol rows per batch
constexpr int kPairsPerWarp = kPairs / kPW;
static_assert(kTT * kNB == 32, "one consumer warp covers a full target tile");
static_assert(kPairs % kPW == 0 && 2 * kPairsPerWarp == 32,
              "two producer lanes per symbol row (t_+nu / t_-nu halves)");
static_assert(kPW == 4, "one producer warp per sub-partition (setmaxnreg split)");
constexpr int kConsumerRegs = 216;
constexpr int kProducerRegs = 504 - 2 * kConsumerRegs;   // 3 warps x 168 per sub-partition

template <int P>
struct Shape {
  static constexpr int L = 2 * P + 1;
  static constexpr int NS = 4 * P + 1;
  static constexpr int BO = (L + kNB - 1) / kNB;
  static constexpr int ROWS = BO * kNB;
  static constexpr int FP = ROWS - L;          // zero pad in front of t_{-2p}
  static constexpr int NSP = FP + NS + 1;      // + one tail slot for the prefetch
  static constexpr int SYM = kS * NSP * kTT;   // double2 per symbol buffer
  static constexpr int BET = kS * L;           // double2 per beta buffer
  static constexpr size_t SMEM =
      2 * (size_t)(SYM + BET) * sizeof(double2) + 2 * (size_t)BET * sizeof(double);
};

struct Args {
  const double* centers;   // [M][2]
  const double2* beta;     // [M][L]
  const double2* bpow;     // [2*copies+1]
  double2* partial;        // [G][maxseg][kTT][L]
  int M, t_begin, nt, copies, ncp, nimg, nbatch, maxseg;
  long long W;
  double period, k2;
};

__device__ __forceinline__ long long work_begin(long long W, int G, int c) {
  return (W * (long long)c) / G;
}

__device__ __forceinline__ void consumer_bar() {
  asm volatile("bar.sync 1, %0;" ::"r"(kS * 32) : "memory");
}

template <int P>
__device__ __forceinline__ void produce(const Args& a, long long w, double2* sym, double2* bet,
                                        double* bets, int pi) {
  using S = Shape<P>;
  const int tile = (int)(w / a.nbatch);
  const int sb = (int)(w % a.nbatch) * kS;
  const int pw = pi >> 5, lane = pi & 31;
  {
    // lanes 2q, 2q+1 build row q: t_{0..2p} and t_{-1..-2p}
    const int pair = pw * kPairsPerWarp + (lane >> 1);
    const bool mirror = lane & 1;
    const int s = pair / kTT, t = pair % kTT;
    const int mloc = tile * kTT + t;
    const int g = sb + s;
    double2* col = sym + (size_t)s * S::NSP * kTT + t;   // slot stride kTT
    bool live = (mloc < a.nt) && (g < a.nimg);
    double dx = 1.0, dy = 0.0;
    if (live) {
      const int m = a.t_begin + mloc;
      const int j = g / a.ncp;
      const int l = g % a.ncp - a.copies;
      const double2 cm = reinterpret_cast<const double2*>(a.centers)[m];
      const double2 cj = reinterpret_cast<const double2*>(a.centers)[j];
      dx = cm.x - cj.x - (double)l * a.period;
      dy = cm.y - cj.y;
      live = !(l == 0 && j == m);
    }
    const double rho = live ? hypot(dx, dy) : 1.0;
    const double z = a.k2 * rho;
    // warp-uniform Miller start: no divergence, uniform constant-bank index
    int N = live ? miller_start_j01(z) : 2;
    N = __reduce_max_sync(0xffffffffu, N);
    const double inv = live ? 1.0 / rho : 0.0;  // dead pairs (self term, padding): c = s = 0
    double2* base = col + (S::FP + 2 * P) * kTT;
    hankel_symbols_half<2 * P>(z, dx * inv, dy * inv, N, mirror,
                               [&](int nu, double re, double im) {
                                 if (nu == 0 && !live) re = im = 0.0;
                                 base[nu * kTT] = make_double2(re, im);
                               });
  }
  // bloch-weighted beta of the batch's source images
  for (int idx = pi; idx < kS * S::L; idx += kPW * 32) {
    const int s2 = idx / S::L, n = idx % S::L;
    const int g2 = sb + s2;
    double2 v = make_double2(0.0, 0.0);
    if (g2 < a.nimg) {
      const int j2 = g2 / a.ncp;
      const double2 b = a.beta[(size_t)j2 * S::L + n];
      const double2 wgt = a.bpow[g2 % a.ncp];
      v.x = fma(b.x, wgt.x, -b.y * wgt.y);
      v.y = fma(b.x, wgt.y, b.y * wgt.x);
    }
    bet[idx] = v;
    bets[idx] = v.x + v.y;
  }
}

// Karatsuba Toeplitz sweep (3 DFMA per complex MAC): for b = beta[n] and
// t = t_{n-r},  S1 += b.x t.x,  S2 += b.y t.y,  S3 += (b.x + b.y)(t.x + t.y);
// Re = S1 - S2, Im = S3 - S1 - S2 at the tile flush.  t.x + t.y is formed as
// the symbol enters the register window; b.x + b.y comes from the producer.
template <int P>
__device__ __forceinline__ void consume(const double2* __restrict__ sym,
                                        const double2* __restrict__ bet,
                                        const double* __restrict__ bets,
                                        double (&acc)[3][Shape<P>::BO], int b, int t) {
  using S = Shape<P>;
  constexpr int BO = S::BO;
  constexpr int R0 = S::FP + 2 * P;              // slot of nu = 0 - 0 at step 0
  constexpr int MODB = 64 * BO;                  // keeps ring indices non-negative
  const double2* sp = sym + (size_t)(R0 - b * BO) * kTT + t;
  double wx[BO], wy[BO], ws[BO];
#pragma unroll
  for (int i = 0; i < BO; ++i) {
    const double2 v = sp[-i * kTT];
    const int q = (R0 - i + MODB) % BO;
    wx[q] = v.x;
    wy[q] = v.y;
    ws[q] = v.x + v.y;
  }
  // one column step; u = n mod BO is compile-time so the ring indices are static
  auto step = [&](auto n_c) {
    constexpr int n = decltype(n_c)::value;
    constexpr int u = n % BO;
    const double2 nxt = sp[(n + 1) * kTT];
    const double2 bb = bet[n];
    const double bs = bets[n];
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
  };
  static_for<S::L>(step);
}

template <int P>
__global__ void __launch_bounds__(kThreads, 1) m2l_kernel(Args a) {
  using S = Shape<P>;
  constexpr int BO = S::BO;
  extern __shared__ double2 smem[];
  double2* sym0 = smem;
  double2* sym1 = smem + S::SYM;
  double2* bet0 = smem + 2 * S::SYM;
  double2* bet1 = bet0 + S::BET;
  double* bets0 = reinterpret_cast<double*>(bet1 + S::BET);
  double* bets1 = bets0 + S::BET;

  const int G = gridDim.x;
  const long long w0 = work_begin(a.W, G, blockIdx.x);
  const long long w1 = work_begin(a.W, G, blockIdx.x + 1);
  if (w0 >= w1) return;

  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const bool producer = warp >= kS;
  const int pi = threadIdx.x - kS * 32;

  // zero the pad slots of both symbol buffers once (only padded rows read them)
  for (int idx = threadIdx.x; idx < 2 * kS * kTT * (S::FP + 1); idx += kThreads) {
    const int buf = idx / (kS * kTT * (S::FP + 1));
    const int r = idx % (kS * kTT * (S::FP + 1));
    const int s = r / (kTT * (S::FP + 1));
    const int r2 = r % (kTT * (S::FP + 1));
    const int q = r2 / kTT, t = r2 % kTT;
    const int slot = q < S::FP ? q : S::FP + S::NS;
    (buf ? sym1 : sym0)[((size_t)s * S::NSP + slot) * kTT + t] = make_double2(0.0, 0.0);
  }
  __syncthreads();

  if (producer) {
    asm volatile("setmaxnreg.dec.sync.aligned.u32 %0;" ::"n"(kProducerRegs));
    produce<P>(a, w0, sym0, bet0, bets0, pi);
    __syncthreads();
    for (long long w = w0; w < w1; ++w) {
      const int cur = (int)((w - w0) & 1);
      if (w + 1 < w1)
        produce<P>(a, w + 1, cur ? sym0 : sym1, cur ? bet0 : bet1, cur ? bets0 : bets1, pi);
      __syncthreads();
    }
    return;
  }
  asm volatile("setmaxnreg.inc.sync.aligned.u32 %0;" ::"n"(kConsumerRegs));
  __syncthreads();

  double acc[3][BO];
#pragma unroll
  for (int c = 0; c < 3; ++c)
#pragma unroll
    for (int i = 0; i < BO; ++i) acc[c][i] = 0.0;
  const int b = lane / kTT, t = lane % kTT;
  int seg = 0;

  for (long long w = w0; w < w1; ++w) {
    const int cur = (int)((w - w0) & 1);
    double2* symc = cur ? sym1 : sym0;
    const double2* betc = cur ? bet1 : bet0;
    const double* betsc = cur ? bets1 : bets0;
    consume<P>(symc + (size_t)warp * S::NSP * kTT, betc + warp * S::L, betsc + warp * S::L, acc,
               b, t);
    const bool flush = (w + 1 == w1) || ((w + 1) % a.nbatch == 0);
    if (flush) {
      // cross-warp reduction through the (now idle) current symbol buffer
      consumer_bar();
      double2* red = symc;   // [kS][kTT][ROWS]
#pragma unroll
      for (int i = 0; i < BO; ++i)
        red[((size_t)warp * kTT + t) * S::ROWS + b * BO + i] =
            make_double2(acc[0][i] - acc[1][i], acc[2][i] - acc[0][i] - acc[1][i]);
      consumer_bar();
      double2* dst = a.partial + ((size_t)blockIdx.x * a.maxseg + seg) * kTT * S::L;
      for (int idx = threadIdx.x; idx < kTT * S::L; idx += kS * 32) {
        const int tt = idx / S::L, r = idx % S::L;
        double2 sum = make_double2(0.0, 0.0);
#pragma unroll
        for (int ww = 0; ww < kS; ++ww) {
          const double2 v = red[((size_t)ww * kTT + tt) * S::ROWS + r];
          sum.x += v.x;
          sum.y += v.y;
        }
        dst[idx] = sum;
      }
      ++seg;
#pragma unroll
      for (int c = 0; c < 3; ++c)
#pragma unroll
        for (int i = 0; i < BO; ++i) acc[c][i] = 0.0;
    }
    __syncthreads();
  }
}

// Sum the per-(CTA, tile-segment) partials of every owned target in CTA order
// and apply the epilogue:
//   mode 0: out = a
//   mode 1: out = v_own - s .* (a - bsub)        (diagonal S)
//   mode 2: out = a - bsub                       (dense S applied afterwards)
__global__ void m2l_reduce(const double2* __restrict__ partial, int G, long long W, int nbatch,
                           int maxseg, int nt, int L, int mode, const double2* __restrict__ v_own,
                           const double2* __restrict__ sdiag, const double2* __restrict__ bsub,
                           double2* __restrict__ out) {
  const int idx = blockIdx.x * blockDim.x + threadIdx.x;
  if (idx >= nt * L) return;
  const int mloc = idx / L, r = idx % L;
  const int tile = mloc / kTT, t = mloc % kTT;
  const long long wa = (long long)tile * nbatch, wb = wa + nbatch;
  int c = (int)((wa * G) / W);
  if (c >= G) c = G - 1;
  while (c > 0 && work_begin(W, G, c) > wa) --c;
  while (c < G - 1 && work_begin(W, G, c + 1) <= wa) ++c;
  double2 sum = make_double2(0.0, 0.0);
  for (; c < G; ++c) {
    const long long c0 = work_begin(W, G, c), c1 = work_begin(W, G, c + 1);
    if (c0 >= wb) break;
    if (c1 <= c0 || c1 <= wa) continue;
    const int seg = tile - (int)(c0 / nbatch);
    const double2 v = partial[(((size_t)c * maxseg + seg) * kTT + t) * L + r];
    sum.x += v.x;
    sum.y += v.y;
  }
  if (mode == 0) {
    out[idx] = sum;
    return;
  }
  if (bsub) {
    sum.x -= bsub[idx].x;
    sum.y -= bsub[idx].y;
  }
  if (mode == 2) {
    out[idx] = sum;
    return;
  }
  const double2 s = sdiag[r];
  const double2 vv = v_own[idx];
  out[idx] = make_double2(vv.x - fma(s.x, sum.x, -s.y * sum.y), vv.y - fma(s.x, sum.y, s.y * sum.x));
}

template <int P>
int launch_p(Ctx* ctx, const double2* beta, const double2* bpow, double2* out, int mode,
             const double2* v_own, const double2* bsub, cudaStream_t st) {
  using S = Shape<P>;
  Args a;
  a.centers = ctx->d_centers;
  a.beta = beta;
  a.bpow = bpow;
  a.M = ctx->M;
  a.t_begin = ctx->t_begin;
  a.nt = ctx->t_end - ctx->t_begin;
  a.copies = ctx->copies;
  a.ncp = 2 * ctx->copies + 1;
  a.nimg = ctx->M * a.ncp;
  a.nbatch = (a.nimg + kS - 1) / kS;
  const int ntiles = (a.nt + kTT - 1) / kTT;
  a.W = (long long)ntiles * a.nbatch;
  a.period = ctx->period;
  a.k2 = ctx->k2;
  if (a.nt <= 0) return PS_OK;
  int G = ctx->sm_count - ctx->k1_reserve_sms;
  if ((long long)G > a.W) G = (int)a.W;
  a.maxseg = (int)((a.W / G + 1) / a.nbatch) + 2;
  const size_t need = (size_t)G * a.maxseg * kTT * S::L;
  if (ctx->partial_elems < need) {
    if (ctx->d_partial) ps::dev_free(ctx->d_partial);
    ctx->d_partial = nullptr;
    ctx->partial_elems = 0;
    PS_CUDA_TRY(ctx, ps::dev_malloc(&ctx->d_partial, need * sizeof(double2)));
    ctx->partial_elems = need;
  }
  a.partial = ctx->d_partial;
  static unsigned long long attr_mask = 0;
  if (first_on_device(&attr_mask, ctx->device)) {
    PS_CUDA_TRY(ctx, cudaFuncSetAttribute(m2l_kernel<P>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                          (int)S::SMEM));
  }
  cudaEvent_t e0 = nullptr, e1 = nullptr;
  if (ctx->profile) {
    PS_CUDA_TRY(ctx, cudaEventCreate(&e0));
    PS_CUDA_TRY(ctx, cudaEventCreate(&e1));
    PS_CUDA_TRY(ctx, cudaEventRecord(e0, st));
  }
  m2l_kernel<P><<<G, kThreads, S::SMEM, st>>>(a);
  PS_CUDA_TRY(ctx, cudaGetLastError());
  if (ctx->profile) {
    PS_CUDA_TRY(ctx, cudaEventRecord(e1, st));
    ctx->k1_events.push_back({e0, e1});
  }
  ctx->launches += 2;
  const int n = a.nt * S::L;
  m2l_reduce<<<(n + 255) / 256, 256, 0, st>>>(ctx->d_partial, G, a.W, a.nbatch, a.maxseg, a.nt,
                                              S::L, mode, v_own, ctx->d_S, bsub, out);
  PS_CUDA_TRY(ctx, cudaGetLastError());
  return PS_OK;
}

}  // namespace

int m2l_max_order() { return PS_M2L_MAX_P; }

bool m2l_sym_selected(const Ctx* ctx) {
  const bool full = ctx->t_begin == 0 && ctx->t_end == ctx->M;
  // crossover measured with tools/probe_variant.py (Karatsuba K1 / K1s): the
  // symmetric kernel wins from M ~ 500 (4% at M = 1000), the tiled one below
  const bool sym = ctx->k1_variant >= 2 || (ctx->k1_variant == 0 && full && ctx->M >= 512);
  return sym && full;
}

int m2l_apply_1(Ctx* ctx, const double2* beta, const double2* bpow, double2* out, int mode,
                const double2* v_own, const double2* bsub, cudaStream_t st) {
  if (m2l_sym_selected(ctx)) return m2l_apply_sym(ctx, beta, bpow, out, mode, v_own, bsub, st);
  return m2l_apply(ctx, beta, bpow, out, mode, v_own, bsub, st);
}

int m2l_apply(Ctx* ctx, const double2* beta, const double2* bpow, double2* out, int mode,
              const double2* v_own, const double2* bsub, cudaStream_t st) {
  switch (ctx->p) {
#define PS_CASE(P) \
  case P:          \
    return launch_p<P>(ctx, beta, bpow, out, mode, v_own, bsub, st);
    PS_M2L_ORDERS(PS_CASE)
#undef PS_CASE
    default:
      ctx->err = "apply_T: multipole order p=" + std::to_string(ctx->p) + " not compiled";
      return PS_ERR_UNSUPPORTED;
  }
}

}  // namespace ps
