// K1m: all-pairs M2L for a batch of right-hand sides sharing one geometry
// (BASELINE cfg5: 16 incidence angles, one k2).  Same operator as m2l.cu
// (multiscat.apply_T), restructured because the symbols
// t_nu(x_m - x_j - l d) do not depend on the RHS:
//
//   * a CTA owns a tile of kTT = 8 targets and a group of up to 16 RHS;
//   * one producer warp builds the 32 symbol rows of a batch of kSB = 4
//     source images (one pair per lane) into shared memory;
//   * 8 consumer warps each own an RHS PAIR for all 8 targets: lane (b, t)
//     keeps BO rows x 2 RHS of complex accumulators and streams the L columns
//     of each source image with the BO-deep symbol window in registers; the
//     bloch-weighted coefficients beta_r,l = bloch_r^l beta_r,j are read as
//     warp-broadcast loads from a pre-weighted copy (bloch_weight kernel);
//   * per column step: 2 broadcast loads + 1 LDS.128 against 8*BO DFMA, and
//     no cross-warp reduction (a warp owns its RHS outright);
//   * the symbol work is amortised over up to 16 RHS (~1% of the FP64 work).
#include <cuda_runtime.h>

#include <algorithm>
#include <string>

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

constexpr int kTT = 8;                  // targets per tile
constexpr int kNB = 4;                  // row blocks per target
constexpr int kSB = 8;                  // source images per batch
constexpr int kRB = 2;                  // RHS per consumer warp
constexpr int kCW = 8;                  // consumer warps (warpgroups 0, 1)
constexpr int kPW = 4;                  // producer warps (warpgroup 2, one per SM sub-partition)
constexpr int kRG = kRB * kCW;          // RHS per CTA group
constexpr int kThreads = (kCW + kPW) * 32;
constexpr int kPairsPerWarp = kTT * kSB / kPW;
static_assert(kPairsPerWarp <= 32, "at most one symbol pair per producer lane");
// register budget per thread after setmaxnreg (launch: 65536 / 384 -> 168)
constexpr int kConsumerRegs = 224;
constexpr int kProducerRegs = 56;
static_assert(2 * kConsumerRegs + kProducerRegs <= 3 * 168, "register file per sub-partition");

template <int P>
struct ShapeM {
  static constexpr int L = 2 * P + 1;
  static constexpr int NS = 4 * P + 1;
  static constexpr int BO = (L + kNB - 1) / kNB;
  static constexpr int ROWS = BO * kNB;
  static constexpr int FP = ROWS - L;
  static constexpr int NSP = FP + NS + 1;
  static constexpr int SYM = kSB * NSP * kTT;
  static constexpr size_t SMEM = 2 * (size_t)SYM * sizeof(double2);
};

struct ArgsM {
  const double* centers;   // [M][2]
  const double2* bw;       // [nrhs][nimg][L]  bloch-weighted beta per source image
  double2* partial;        // [G][maxseg][kRG][kTT][L]
  int nrhs, rg0, M, t_begin, nt, copies, ncp, nimg, nbatch, maxseg;
  long long W;
  long long q;             // work-range quantum (divides nbatch)
  double period, k2;
};

// CTA c's work range starts at a multiple of q = nbatch / kPhases: all CTAs
// sweep the source list in at most kPhases phase groups, so the beta rows a
// batch needs are fetched from DRAM once per group instead of once per CTA
// (the cfg5 weighted-beta copy is 315 MB > 126 MB L2).
constexpr int kPhases = 8;

__host__ __device__ __forceinline__ long long work_begin(long long W, int G, int c, long long q) {
  const long long raw = (W * (long long)c) / G;
  return ((raw + q / 2) / q) * q;
}

template <int P>
__device__ __forceinline__ void produce_m(const ArgsM& a, long long w, double2* sym, int pw,
                                          int lane) {
  using S = ShapeM<P>;
  if (lane >= kPairsPerWarp) return;
  const int tile = (int)(w / a.nbatch);
  const int sb = (int)(w % a.nbatch) * kSB;
  const int pair = pw * kPairsPerWarp + lane;
  const int s = pair / kTT, t = pair % kTT;
  const int mloc = tile * kTT + t;
  const int g = sb + s;
  double2* col = sym + (size_t)s * S::NSP * kTT + t;
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
  int N = live ? miller_start_j01(z) : 2;
  constexpr unsigned kMask = kPairsPerWarp == 32 ? 0xffffffffu : ((1u << kPairsPerWarp) - 1u);
  N = __reduce_max_sync(kMask, N);
  const double inv = live ? 1.0 / rho : 0.0;
  double2* base = col + (S::FP + 2 * P) * kTT;
  hankel_symbols<2 * P>(z, dx * inv, dy * inv, N, [&](int nu, double re, double im) {
    if (nu == 0 && !live) re = im = 0.0;
    base[nu * kTT] = make_double2(re, im);
  });
}

// Pull the bloch-weighted beta rows of batch w into L2 ahead of the consumers
// (the cfg5 copy is 315 MB, beyond the 126 MB L2).  All 128 producer lanes
// take one (rhs, image) row each.
template <int P>
__device__ __forceinline__ void prefetch_bw(const ArgsM& a, long long w, int pl) {
  using S = ShapeM<P>;
  const int sb = (int)(w % a.nbatch) * kSB;
  const int nr = min(kRG, a.nrhs - a.rg0);
  for (int row = pl; row < nr * kSB; row += kPW * 32) {
    const int r = a.rg0 + row / kSB;
    const int g = sb + row % kSB;
    if (g >= a.nimg) continue;
    const char* p = reinterpret_cast<const char*>(a.bw + ((size_t)r * a.nimg + g) * S::L);
    for (int off = 0; off < S::L * 16; off += 128)
      asm volatile("prefetch.global.L2 [%0];" ::"l"(p + off));
  }
}

template <int P>
__device__ __forceinline__ void consume_m(const double2* __restrict__ sym,
                                          const double2* __restrict__ b0,
                                          const double2* __restrict__ b1,
                                          double2 (&acc0)[ShapeM<P>::BO],
                                          double2 (&acc1)[ShapeM<P>::BO], int b, int t) {
  using S = ShapeM<P>;
  constexpr int BO = S::BO;
  constexpr int R0 = S::FP + 2 * P;
  constexpr int MODB = 64 * BO;
  const double2* sp = sym + (size_t)(R0 - b * BO) * kTT + t;
  double2 w[BO];
#pragma unroll
  for (int i = 0; i < BO; ++i) w[(R0 - i + MODB) % BO] = sp[-i * kTT];
  // one column step; u = n mod BO is compile-time so the ring indices are
  // static.  The column loop is unrolled by BO only (a runtime loop over
  // BO-blocks): at cfg5 size this beats the full unroll (80.3% vs 78.2% of
  // DFMA peak, smaller instruction footprint for 8 warps at different PCs).
  auto step = [&](int n, auto u_c) {
    constexpr int u = decltype(u_c)::value;
    const double2 nxt = sp[(n + 1) * kTT];
    const double2 x0 = __ldg(b0 + n);
    const double2 x1 = __ldg(b1 + n);
#pragma unroll
    for (int i = 0; i < BO; ++i) {
      const double2 tt = w[(R0 + u - i + MODB) % BO];
      acc0[i].x = fma(x0.x, tt.x, acc0[i].x);
      acc1[i].x = fma(x1.x, tt.x, acc1[i].x);
      acc0[i].y = fma(x0.x, tt.y, acc0[i].y);
      acc1[i].y = fma(x1.x, tt.y, acc1[i].y);
    }
#pragma unroll
    for (int i = 0; i < BO; ++i) {
      const double2 tt = w[(R0 + u - i + MODB) % BO];
      acc0[i].x = fma(-x0.y, tt.y, acc0[i].x);
      acc1[i].x = fma(-x1.y, tt.y, acc1[i].x);
      acc0[i].y = fma(x0.y, tt.x, acc0[i].y);
      acc1[i].y = fma(x1.y, tt.x, acc1[i].y);
    }
    w[(R0 + u + 1 + MODB) % BO] = nxt;
  };
#ifdef PS_K1M_FULL_UNROLL
  static_for<S::L>([&](auto u) { step(decltype(u)::value, IC<decltype(u)::value % BO>{}); });
#else
  constexpr int NFULL = (S::L / BO) * BO;
#pragma unroll 1
  for (int n0 = 0; n0 < NFULL; n0 += BO)
    static_for<BO>([&](auto u) { step(n0 + decltype(u)::value, u); });
  static_for<S::L - NFULL>([&](auto u) { step(NFULL + decltype(u)::value, u); });
#endif
}

template <int P>
__global__ void __launch_bounds__(kThreads, 1) m2l_mrhs_kernel(ArgsM a) {
  using S = ShapeM<P>;
  constexpr int BO = S::BO, L = S::L;
  extern __shared__ double2 smem[];
  double2* sym0 = smem;
  double2* sym1 = smem + S::SYM;
  const int G = gridDim.x;
  const long long w0 = work_begin(a.W, G, blockIdx.x, a.q);
  const long long w1 = work_begin(a.W, G, blockIdx.x + 1, a.q);
  if (w0 >= w1) return;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const bool producer = warp >= kCW;

  for (int idx = threadIdx.x; idx < 2 * kSB * kTT * (S::FP + 1); idx += kThreads) {
    const int buf = idx / (kSB * kTT * (S::FP + 1));
    const int r = idx % (kSB * kTT * (S::FP + 1));
    const int s = r / (kTT * (S::FP + 1));
    const int r2 = r % (kTT * (S::FP + 1));
    const int q = r2 / kTT, t = r2 % kTT;
    const int slot = q < S::FP ? q : S::FP + S::NS;
    (buf ? sym1 : sym0)[((size_t)s * S::NSP + slot) * kTT + t] = make_double2(0.0, 0.0);
  }
  __syncthreads();
  // warp-specialised register split: the producer warpgroup gives registers
  // to the two consumer warpgroups (accumulators for BO rows x 2 RHS).  The
  // two roles run separate loops with the same __syncthreads schedule so
  // ptxas can allocate each under its own budget.
  if (producer) {
    asm volatile("setmaxnreg.dec.sync.aligned.u32 %0;" ::"n"(kProducerRegs));
    const int pw = warp - kCW;
    prefetch_bw<P>(a, w0, pw * 32 + lane);
    produce_m<P>(a, w0, sym0, pw, lane);
    __syncthreads();
    const int pl = pw * 32 + lane;
    if (w0 + 1 < w1) prefetch_bw<P>(a, w0 + 1, pl);
    for (long long w = w0; w < w1; ++w) {
      const int cur = (int)((w - w0) & 1);
      if (w + 2 < w1) prefetch_bw<P>(a, w + 2, pl);
      if (w + 1 < w1) produce_m<P>(a, w + 1, cur ? sym0 : sym1, pw, lane);
      __syncthreads();
    }
    return;
  }
  asm volatile("setmaxnreg.inc.sync.aligned.u32 %0;" ::"n"(kConsumerRegs));
  __syncthreads();

  // this warp's RHS pair (absolute indices); a missing second RHS reads RHS r0
  const int r0 = a.rg0 + kRB * warp;
  const bool active = r0 < a.nrhs;
  const int r1 = (r0 + 1 < a.nrhs) ? r0 + 1 : r0;
  const int b = lane / kTT, t = lane % kTT;
  double2 acc0[BO], acc1[BO];
#pragma unroll
  for (int i = 0; i < BO; ++i) acc0[i] = acc1[i] = make_double2(0.0, 0.0);
  int seg = 0;

  for (long long w = w0; w < w1; ++w) {
    const int cur = (int)((w - w0) & 1);
    double2* symc = cur ? sym1 : sym0;
    if (active) {
      const int sb = (int)(w % a.nbatch) * kSB;
#pragma unroll 1
      for (int s = 0; s < kSB; ++s) {
        const int g = sb + s < a.nimg ? sb + s : a.nimg - 1;   // dead images have zero symbols
        consume_m<P>(symc + (size_t)s * S::NSP * kTT,
                     a.bw + ((size_t)r0 * a.nimg + g) * L, a.bw + ((size_t)r1 * a.nimg + g) * L,
                     acc0, acc1, b, t);
      }
      if ((w + 1 == w1) || ((w + 1) % a.nbatch == 0)) {
        double2* dst = a.partial + ((size_t)blockIdx.x * a.maxseg + seg) * kRG * kTT * L;
        const int rl = r0 - a.rg0;
#pragma unroll
        for (int i = 0; i < BO; ++i) {
          const int row = b * BO + i;
          if (row < L) {
            dst[((size_t)rl * kTT + t) * L + row] = acc0[i];
            dst[((size_t)(rl + 1) * kTT + t) * L + row] = acc1[i];
          }
          acc0[i] = acc1[i] = make_double2(0.0, 0.0);
        }
        ++seg;
      }
    }
    __syncthreads();
  }
}

// bw[r][g][n] = bloch_r^{l(g)} beta_r[j(g)][n]
__global__ void bloch_weight(const double2* __restrict__ beta, const double2* __restrict__ bpow,
                             int np, int M, int L, int ncp, long long total,
                             double2* __restrict__ bw) {
  for (long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x; i < total;
       i += (long long)gridDim.x * blockDim.x) {
    const int n = (int)(i % L);
    const long long rg = i / L;
    const int g = (int)(rg % ((long long)M * ncp));
    const int r = (int)(rg / ((long long)M * ncp));
    const int j = g / ncp, li = g % ncp;
    const double2 b = beta[((long long)r * M + j) * L + n];
    const double2 wv = bpow[(long long)r * np + 1 + li];
    bw[i] = make_double2(fma(b.x, wv.x, -b.y * wv.y), fma(b.x, wv.y, b.y * wv.x));
  }
}

// Sum partials in CTA order; epilogue as m2l_reduce, per RHS.
__global__ void m2l_mrhs_reduce(const double2* __restrict__ partial, int G, long long W,
                                long long q, int nbatch, int maxseg, int nt, int L, int rg0, int nr, int mode,
                                const double2* __restrict__ v, long long v_stride, int v_off,
                                const double2* __restrict__ sdiag,
                                const double2* __restrict__ bsub, long long b_stride,
                                double2* __restrict__ out, long long out_stride) {
  const long long idx = (long long)blockIdx.x * blockDim.x + threadIdx.x;
  if (idx >= (long long)nr * nt * L) return;
  const int rl = (int)(idx / ((long long)nt * L));
  const int rem = (int)(idx % ((long long)nt * L));
  const int mloc = rem / L, row = rem % L;
  const int tile = mloc / kTT, t = mloc % kTT;
  const long long wa = (long long)tile * nbatch, wb = wa + nbatch;
  int c = (int)((wa * G) / W);
  if (c >= G) c = G - 1;
  while (c > 0 && work_begin(W, G, c, q) > wa) --c;
  while (c < G - 1 && work_begin(W, G, c + 1, q) <= wa) ++c;
  double2 sum = make_double2(0.0, 0.0);
  for (; c < G; ++c) {
    const long long c0 = work_begin(W, G, c, q), c1 = work_begin(W, G, c + 1, q);
    if (c0 >= wb) break;
    if (c1 <= c0 || c1 <= wa) continue;
    const int seg = tile - (int)(c0 / nbatch);
    const double2 pv = partial[((((size_t)c * maxseg + seg) * kRG + rl) * kTT + t) * L + row];
    sum.x += pv.x;
    sum.y += pv.y;
  }
  const int r = rg0 + rl;
  double2* o = out + r * out_stride + rem;
  if (mode == 0) {
    *o = sum;
    return;
  }
  if (bsub) {
    const double2 bb = bsub[r * b_stride + rem];
    sum.x -= bb.x;
    sum.y -= bb.y;
  }
  if (mode == 2) {
    *o = sum;
    return;
  }
  const double2 s = sdiag[row];
  const double2 vv = v[r * v_stride + (long long)v_off * L + rem];
  *o = make_double2(vv.x - fma(s.x, sum.x, -s.y * sum.y), vv.y - fma(s.x, sum.y, s.y * sum.x));
}

template <int P>
int launch_m(Ctx* ctx, const double2* beta, double2* out, int mode, const double2* bsub,
             long long b_stride, cudaStream_t st) {
  using S = ShapeM<P>;
  const int nt = ctx->t_end - ctx->t_begin;
  if (nt <= 0) return PS_OK;
  ArgsM a;
  a.centers = ctx->d_centers;
  a.nrhs = ctx->nrhs;
  a.M = ctx->M;
  a.t_begin = ctx->t_begin;
  a.nt = nt;
  a.copies = ctx->copies;
  a.ncp = 2 * ctx->copies + 1;
  a.nimg = ctx->M * a.ncp;
  a.nbatch = (a.nimg + kSB - 1) / kSB;
  const int ntiles = (nt + kTT - 1) / kTT;
  a.W = (long long)ntiles * a.nbatch;
  a.period = ctx->period;
  a.k2 = ctx->k2;
  int G = ctx->sm_count;
  if ((long long)G > a.W) G = (int)a.W;
  // quantum: a divisor of nbatch near nbatch / kPhases, small enough that
  // every CTA still gets work
  long long q = a.nbatch / kPhases;
  if (q < 1) q = 1;
  while (a.nbatch % q) --q;
  if (q * G > a.W) q = 1;
  a.q = q;
  a.maxseg = (int)((a.W / G + q + 1) / a.nbatch) + 3;
  // bloch-weighted copy of beta (all RHS, all images)
  const long long total = (long long)ctx->nrhs * a.nimg * S::L;
  const size_t need_p = (size_t)G * a.maxseg * kRG * kTT * S::L;
  const size_t need = need_p + (size_t)total;
  if (ctx->partial_elems < need) {
    if (ctx->d_partial) ps::dev_free(ctx->d_partial);
    ctx->d_partial = nullptr;
    ctx->partial_elems = 0;
    PS_CUDA_TRY(ctx, ps::dev_malloc(&ctx->d_partial, need * sizeof(double2)));
    ctx->partial_elems = need;
  }
  a.partial = ctx->d_partial;
  double2* bw = ctx->d_partial + need_p;
  a.bw = bw;
  const int np = 2 * ctx->copies + 3;
  bloch_weight<<<4 * ctx->sm_count, 256, 0, st>>>(beta, ctx->d_blochpow, np, ctx->M, S::L, a.ncp,
                                                  total, bw);
  PS_CUDA_TRY(ctx, cudaGetLastError());
  ctx->launches += 1;
  static unsigned long long attr_mask = 0;
  if (first_on_device(&attr_mask, ctx->device)) {
    PS_CUDA_TRY(ctx, cudaFuncSetAttribute(m2l_mrhs_kernel<P>,
                                          cudaFuncAttributeMaxDynamicSharedMemorySize, (int)S::SMEM));
  }
  const long long in_stride = (long long)ctx->M * S::L, out_stride = (long long)nt * S::L;
  for (a.rg0 = 0; a.rg0 < ctx->nrhs; a.rg0 += kRG) {
    cudaEvent_t e0 = nullptr, e1 = nullptr;
    if (ctx->profile) {
      PS_CUDA_TRY(ctx, cudaEventCreate(&e0));
      PS_CUDA_TRY(ctx, cudaEventCreate(&e1));
      PS_CUDA_TRY(ctx, cudaEventRecord(e0, st));
    }
    m2l_mrhs_kernel<P><<<G, kThreads, S::SMEM, st>>>(a);
    PS_CUDA_TRY(ctx, cudaGetLastError());
    if (ctx->profile) {
      PS_CUDA_TRY(ctx, cudaEventRecord(e1, st));
      ctx->k1_events.push_back({e0, e1});
    }
    const int nr = std::min(kRG, ctx->nrhs - a.rg0);
    const long long n = (long long)nr * nt * S::L;
    m2l_mrhs_reduce<<<(int)((n + 255) / 256), 256, 0, st>>>(
        ctx->d_partial, G, a.W, a.q, a.nbatch, a.maxseg, nt, S::L, a.rg0, nr, mode, beta, in_stride,
        ctx->t_begin, ctx->d_S, bsub, b_stride, out, out_stride);
    PS_CUDA_TRY(ctx, cudaGetLastError());
    ctx->launches += 2;
  }
  return PS_OK;
}

}  // namespace

int m2l_apply_mrhs(Ctx* ctx, const double2* beta, double2* out, int mode, const double2* bsub,
                   long long b_stride, cudaStream_t st) {
  // K1d and K1m process RHS in groups of 16: below 12 RHS most of their
  // MMA columns / consumer warps would idle, and the single-RHS kernels (K1s /
  // K1 at ~80% of the DFMA peak, one launch per RHS) are faster
  if (ctx->mrhs_variant == 2 || (ctx->mrhs_variant == 0 && ctx->nrhs >= 12))
    return m2l_apply_mma(ctx, beta, out, mode, bsub, b_stride, st);
  if (ctx->mrhs_variant == 1) return m2l_apply_mrhs_dfma(ctx, beta, out, mode, bsub, b_stride, st);
  const size_t in_stride = (size_t)ctx->M * ctx->L;
  const size_t out_stride = (size_t)(ctx->t_end - ctx->t_begin) * ctx->L;
  const int np = 2 * ctx->copies + 3;
  for (int r = 0; r < ctx->nrhs; ++r) {
    const double2* br = beta + r * in_stride;
    if (int rc = m2l_apply_1(ctx, br, ctx->d_blochpow + (size_t)r * np + 1, out + r * out_stride,
                             mode, br + (size_t)ctx->t_begin * ctx->L,
                             bsub ? bsub + r * b_stride : nullptr, st))
      return rc;
  }
  return PS_OK;
}

int m2l_apply_mrhs_dfma(Ctx* ctx, const double2* beta, double2* out, int mode,
                        const double2* bsub, long long b_stride, cudaStream_t st) {
  switch (ctx->p) {
#define PS_CASE(P) \
  case P:          \
    return launch_m<P>(ctx, beta, out, mode, bsub, b_stride, st);
    PS_M2L_ORDERS(PS_CASE)
#undef PS_CASE
    default:
      ctx->err = "apply_T (multi-RHS): multipole order p=" + std::to_string(ctx->p) +
                 " not compiled";
      return PS_ERR_UNSUPPORTED;
  }
}

}  // namespace ps
