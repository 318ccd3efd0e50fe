// K1d: all-pairs M2L for >= 12 right-hand sides on the FP64 tensor cores
// (multiscat.apply_T; BASELINE cfg5: 16 incidence angles).
//
// For a source image g and the 8 targets of a tile the batched translation is
// a dense complex contraction
//     C (8L x R)  +=  A_g (8L x L) . B_g (L x R)
//     A_g = [T_{m1,g}; ...; T_{m8,g}],  T_{m,g}[m'][n] = t_{n-m'}(x_m - x_g)
//     B_g[n][r]   = bloch_r^l beta_r,j[n]
// (the Toeplitz blocks of the 8 targets stacked vertically: 8L rows are
// exactly L row tiles of 8, so only the K = L dimension is padded).  It runs
// as mma.sync.m8n8k4.f64 (DMMA, 256 FMA per warp instruction; measured
// 37.1 TF/s on B200 against 34.2 TF/s for DFMA), three real MMAs per complex
// tile (Karatsuba: Ar Br, Ai Bi, (Ar + Ai)(Br + Bi)); the producer stores
// Ar + Ai beside each symbol so the consumers add nothing on the A side.  The symbol rows come from the same producer warpgroup as K1/K1m.
//
// Warps: 12 consumer warps own (row tile, RHS tile) accumulator units
// (2L units per CTA group, <= 7 per warp); 4 producer warps (setmaxnreg).
#include <cuda_runtime.h>

#include <algorithm>
#include <string>

#include "ctx.cuh"
#include "m2l.cuh"
#include "symbols.cuh"

namespace ps {

namespace {

constexpr int kTT = 8;                 // targets per tile (stacked)
constexpr int kSBMax = 8;              // source images per batch (at most; see ShapeD::SB)
constexpr int kCW = 12;                // consumer warps
constexpr int kPW = 4;                 // producer warps
constexpr int kThreads = (kCW + kPW) * 32;
constexpr int kRG = 16;                // RHS per group (2 MMA column tiles)
constexpr int kNT = kRG / 8;
constexpr int kPhases = 8;
static_assert(kTT * kSBMax * 2 == kPW * 32, "up to 64 rows, two producer lanes each");
// per sub-partition: 3 consumer + 1 producer warp; 3*Rc + Rp <= 512
constexpr int kConsumerRegs = 152;
constexpr int kProducerRegs = 56;

template <int P>
struct ShapeD {
  static constexpr int L = 2 * P + 1;
  static constexpr int KT = (L + 3) / 4;          // K tiles
  static constexpr int UNITS = L * kNT;           // (row tile, RHS tile) units per group
  static constexpr int UPW = (UNITS + kCW - 1) / kCW;
  static constexpr int OFF = L - 1;               // slot of nu = 0
  static constexpr int NSPR = 4 * KT + L - 1;     // nu in [-(L-1), 4 KT - 1]
  static constexpr int NSP = NSPR | 1;            // odd row stride
  // Each buffer also holds re + im of every symbol (double, the Karatsuba A
  // operand) so the consumers issue no DADD per A fragment, with as many
  // source images per batch as fit two such buffers in 227 KB (7 at p = 20,
  // 5 at p = 25).  Measured (tools/probe_k1d_p25.py) faster than the
  // in-register DADD with 8 images per batch at every p from 10 to 25.
  static constexpr int SBFIT = 232448 / (2 * kTT * NSP * 24);
  static constexpr int SB = SBFIT < kSBMax ? SBFIT : kSBMax;
  static_assert(SB >= 1, "symbol buffers exceed shared memory");
  static constexpr int SYM = kTT * SB * NSP;      // symbols (double2) or sums (double) per buffer
  static constexpr size_t SMEM = 2 * (size_t)SYM * (sizeof(double2) + sizeof(double));
};

struct ArgsD {
  const double* centers;
  const double2* bw;       // [nrhs][nimg][L]
  double2* partial;        // [G][maxseg][kRG][kTT][L]
  int nrhs, rg0, M, t_begin, nt, copies, ncp, nimg, nbatch, maxseg;
  long long W, q;
  double period, k2;
};

__host__ __device__ __forceinline__ long long work_begin(long long W, int G, int c, long long q) {
  const long long raw = (W * (long long)c) / G;
  return ((raw + q / 2) / q) * q;
}

__device__ __forceinline__ void dmma(double (&d)[2], double a, double b) {
  asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0, %1}, {%2}, {%3}, {%0, %1};"
               : "+d"(d[0]), "+d"(d[1])
               : "d"(a), "d"(b));
}

// rows (s, t) at (s * kTT + t) * NSP; slot = nu + OFF
template <int P>
__device__ __forceinline__ void produce_d(const ArgsD& a, long long w, double2* sym, double* sum,
                                          int pw, int lane) {
  using S = ShapeD<P>;
  const int tile = (int)(w / a.nbatch);
  const int sb = (int)(w % a.nbatch) * S::SB;
  const int row = pw * 16 + (lane & 15);         // quarter-warps write consecutive rows
  const bool rok = row < kTT * S::SB;
  const bool mirror = lane >> 4;
  const int s = row / kTT, t = row % kTT;
  const int mloc = tile * kTT + t;
  const int g = sb + s;
  bool live = rok && (mloc < a.nt) && (g < a.nimg);
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
  N = __reduce_max_sync(0xffffffffu, N);
  const double inv = live ? 1.0 / rho : 0.0;
  double2* base = sym + (size_t)row * S::NSP + S::OFF;
  double* sbase = sum + (size_t)row * S::NSP + S::OFF;
  hankel_symbols_half<2 * P>(z, dx * inv, dy * inv, N, mirror, [&](int nu, double re, double im) {
    if (!rok) return;
    if (nu == 0 && !live) re = im = 0.0;
    base[nu] = make_double2(re, im);
    sbase[nu] = re + im;
  });
}

// L2 prefetch of the weighted-beta rows of batch w (all producer lanes)
template <int P>
__device__ __forceinline__ void prefetch_bw_d(const ArgsD& a, long long w, int pl) {
  using S = ShapeD<P>;
  const int sb = (int)(w % a.nbatch) * S::SB;
  const int nr = min(kRG, a.nrhs - a.rg0);
  for (int row = pl; row < nr * S::SB; row += kPW * 32) {
    const int r = a.rg0 + row / S::SB;
    const int g = sb + row % S::SB;
    if (g >= a.nimg) continue;
    const char* p = reinterpret_cast<const char*>(a.bw + ((size_t)r * a.nimg + g) * S::L);
    for (int off = 0; off < S::L * 16; off += 128)
      asm volatile("prefetch.global.L2 [%0];" ::"l"(p + off));
  }
}

template <int P>
__global__ void __launch_bounds__(kThreads, 1) m2l_mma_kernel(ArgsD a) {
  using S = ShapeD<P>;
  constexpr int L = S::L, UPW = S::UPW;
  extern __shared__ double2 smem[];
  double2* sym0 = smem;
  double2* sym1 = smem + S::SYM;
  double* sum0 = reinterpret_cast<double*>(smem + 2 * S::SYM);
  double* sum1 = sum0 + S::SYM;
  const int G = gridDim.x;
  const long long w0 = work_begin(a.W, G, blockIdx.x, a.q);
  const long long w1 = work_begin(a.W, G, blockIdx.x + 1, a.q);
  if (w0 >= w1) return;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const bool producer = warp >= kCW;

  // zero both buffers once: slots outside |nu| <= 2P are read (padding K
  // columns whose B is zero) and must be finite
  for (int i = threadIdx.x; i < 3 * S::SYM; i += kThreads) smem[i] = make_double2(0.0, 0.0);
  __syncthreads();

  if (producer) {
    asm volatile("setmaxnreg.dec.sync.aligned.u32 %0;" ::"n"(kProducerRegs));
    const int pw = warp - kCW;
    const int pl = pw * 32 + lane;
    prefetch_bw_d<P>(a, w0, pl);
    if (w0 + 1 < w1) prefetch_bw_d<P>(a, w0 + 1, pl);
    produce_d<P>(a, w0, sym0, sum0, pw, lane);
    __syncthreads();
    for (long long w = w0; w < w1; ++w) {
      const int cur = (int)((w - w0) & 1);
      if (w + 2 < w1) prefetch_bw_d<P>(a, w + 2, pl);
      if (w + 1 < w1) produce_d<P>(a, w + 1, cur ? sym0 : sym1, cur ? sum0 : sum1, pw, lane);
      __syncthreads();
    }
    return;
  }
  asm volatile("setmaxnreg.inc.sync.aligned.u32 %0;" ::"n"(kConsumerRegs));
  __syncthreads();

  // fragment coordinates (PTX m8n8k4 f64): A[r][c], B[c][r'], C[r][2c'+i]
  const int fr = lane >> 2, fc = lane & 3;
  // this warp's units u = warp + kCW * k: row tile u / kNT, RHS tile u % kNT
  // = warp % kNT for every k (kCW is a multiple of kNT); only the row offset
  // of the lane's A element is kept per unit (register pressure at p >= 24)
  static_assert(kCW % kNT == 0, "uniform RHS tile per warp");
  const int ntw = warp % kNT;
  const int nk = (S::UNITS - warp + kCW - 1) / kCW;   // valid units of this warp
  int offA[UPW];
#pragma unroll
  for (int k = 0; k < UPW; ++k) {
    const int srow = ((warp + kCW * k) / kNT) * 8 + fr;   // stacked row of the A element
    offA[k] = (srow / L) * S::NSP - (srow % L);           // target slot * NSP - row m'
  }
  // Karatsuba: P1 = Ar Br, P2 = Ai Bi, P3 = (Ar + Ai)(Br + Bi);
  // Re C = P1 - P2, Im C = P3 - P1 - P2 -> three real MMAs per complex tile
  double p1[UPW][2], p2[UPW][2], p3[UPW][2];
#pragma unroll
  for (int k = 0; k < UPW; ++k) p1[k][0] = p1[k][1] = p2[k][0] = p2[k][1] = p3[k][0] = p3[k][1] = 0.0;
  int seg = 0;
  const int rb = a.rg0 + fr;                     // B column (RHS) for tile 0; +8 for tile 1

  for (long long w = w0; w < w1; ++w) {
    const int cur = (int)((w - w0) & 1);
    const double2* symc = cur ? sym1 : sym0;
    const double* sumc = cur ? sum1 : sum0;
    const int sb = (int)(w % a.nbatch) * S::SB;
#pragma unroll 1
    for (int s = 0; s < S::SB; ++s) {
      const int g = min(sb + s, a.nimg - 1);      // dead images have zero symbols
      const double2* bw0 = a.bw + ((size_t)min(rb, a.nrhs - 1) * a.nimg + g) * L;
      const double2* bw1 = a.bw + ((size_t)min(rb + 8, a.nrhs - 1) * a.nimg + g) * L;
      const bool ok0 = rb < a.nrhs, ok1 = rb + 8 < a.nrhs;
      const double2* rowb = symc + (size_t)s * kTT * S::NSP + S::OFF;
      const double* rows = sumc + (size_t)s * kTT * S::NSP + S::OFF;
#pragma unroll
      for (int kt = 0; kt < S::KT; ++kt) {
        const int n = kt * 4 + fc;
        double2 b0 = make_double2(0.0, 0.0), b1 = b0;
        if (n < L) {
          if (ok0) b0 = __ldg(bw0 + n);
          if (ok1) b1 = __ldg(bw1 + n);
        }
        const double bs0 = b0.x + b0.y, bs1 = b1.x + b1.y;
#pragma unroll
        for (int k = 0; k < UPW; ++k) {
          if (k >= nk) continue;
          const int ia = offA[k] + n;
          const double2 av = rowb[ia];
          const double as = rows[ia];
          const double2 bb = ntw ? b1 : b0;
          const double bs = ntw ? bs1 : bs0;
          dmma(p1[k], av.x, bb.x);
          dmma(p2[k], av.y, bb.y);
          dmma(p3[k], as, bs);
        }
      }
    }
    if ((w + 1 == w1) || ((w + 1) % a.nbatch == 0)) {
      double2* dst = a.partial + ((size_t)blockIdx.x * a.maxseg + seg) * kRG * kTT * L;
#pragma unroll
      for (int k = 0; k < UPW; ++k) {
        if (k < nk) {
          const int srow = ((warp + kCW * k) / kNT) * 8 + fr;
          const int t = srow / L, mp = srow % L;
#pragma unroll
          for (int i = 0; i < 2; ++i) {
            const int rl = ntw * 8 + 2 * fc + i;           // RHS within the group
            dst[((size_t)rl * kTT + t) * L + mp] =
                make_double2(p1[k][i] - p2[k][i], p3[k][i] - p1[k][i] - p2[k][i]);
          }
        }
        p1[k][0] = p1[k][1] = p2[k][0] = p2[k][1] = p3[k][0] = p3[k][1] = 0.0;
      }
      ++seg;
    }
    __syncthreads();
  }
}

__global__ void bloch_weight_d(const double2* __restrict__ beta, const double2* __restrict__ bpow,
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

__global__ void m2l_mma_reduce(const double2* __restrict__ partial, int G, long long W,
                               long long q, int nbatch, int maxseg, int nt, int L, int rg0, int nr,
                               int mode, const double2* __restrict__ v, long long v_stride,
                               int v_off, const double2* __restrict__ sdiag,
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
int launch_d(Ctx* ctx, const double2* beta, double2* out, int mode, const double2* bsub,
             long long b_stride, cudaStream_t st) {
  using S = ShapeD<P>;
  const int nt = ctx->t_end - ctx->t_begin;
  if (nt <= 0) return PS_OK;
  ArgsD a;
  a.centers = ctx->d_centers;
  a.nrhs = ctx->nrhs;
  a.M = ctx->M;
  a.t_begin = ctx->t_begin;
  a.nt = nt;
  a.copies = ctx->copies;
  a.ncp = 2 * ctx->copies + 1;
  a.nimg = ctx->M * a.ncp;
  a.nbatch = (a.nimg + S::SB - 1) / S::SB;
  const int ntiles = (nt + kTT - 1) / kTT;
  a.W = (long long)ntiles * a.nbatch;
  a.period = ctx->period;
  a.k2 = ctx->k2;
  int G = ctx->sm_count;
  if ((long long)G > a.W) G = (int)a.W;
  long long q = a.nbatch / kPhases;
  if (q < 1) q = 1;
  while (a.nbatch % q) --q;
  if (q * G > a.W) q = 1;
  a.q = q;
  a.maxseg = (int)((a.W / G + q + 1) / a.nbatch) + 3;
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
  bloch_weight_d<<<4 * ctx->sm_count, 256, 0, st>>>(beta, ctx->d_blochpow, np, ctx->M, S::L,
                                                    a.ncp, total, bw);
  PS_CUDA_TRY(ctx, cudaGetLastError());
  ctx->launches += 1;
  static unsigned long long attr_mask = 0;
  if (first_on_device(&attr_mask, ctx->device)) {
    PS_CUDA_TRY(ctx, cudaFuncSetAttribute(m2l_mma_kernel<P>,
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
    m2l_mma_kernel<P><<<G, kThreads, S::SMEM, st>>>(a);
    PS_CUDA_TRY(ctx, cudaGetLastError());
    if (ctx->profile) {
      PS_CUDA_TRY(ctx, cudaEventRecord(e1, st));
      ctx->k1_events.push_back({e0, e1});
    }
    const int nr = std::min(kRG, ctx->nrhs - a.rg0);
    const long long n = (long long)nr * nt * S::L;
    m2l_mma_reduce<<<(int)((n + 255) / 256), 256, 0, st>>>(
        ctx->d_partial, G, a.W, a.q, a.nbatch, a.maxseg, nt, S::L, a.rg0, nr, mode, beta,
        in_stride, ctx->t_begin, ctx->d_S, bsub, b_stride, out, out_stride);
    PS_CUDA_TRY(ctx, cudaGetLastError());
    ctx->launches += 2;
  }
  return PS_OK;
}

}  // namespace

int m2l_apply_mma(Ctx* ctx, const double2* beta, double2* out, int mode, const double2* bsub,
                  long long b_stride, cudaStream_t st) {
  switch (ctx->p) {
#define PS_CASE(P) \
  case P:          \
    return launch_d<P>(ctx, beta, out, mode, bsub, b_stride, st);
    PS_M2L_ORDERS(PS_CASE)
#undef PS_CASE
    default:
      ctx->err = "apply_T (DMMA): multipole order p=" + std::to_string(ctx->p) + " not compiled";
      return PS_ERR_UNSUPPORTED;
  }
}

}  // namespace ps
