// K1s: symmetric all-pairs M2L for one RHS when the rank owns every target
// (multiscat.apply_T).  The symbol row of the pair
// (m, j, l), t_nu = H_nu(k rho) e^{i nu phi} of x_m - x_j - l d e_x, also
// serves the reverse pair (j, m, -l): its displacement is the negative, so
// t'_nu = (-1)^nu t_nu.  With
//   a_j[m'] += sum_n beta'[n] t'_{n-m'} = (-1)^m' sum_n ((-1)^n beta'[n]) t_{n-m'}
// the reverse apply is the forward Toeplitz sweep over the SAME shared-memory
// row with sign-flipped coefficients and a sign on the output row.  Each
// symbol row therefore feeds two L x L applies and the producer FP64 work per
// translation halves (the single-RHS K1 spends ~14% of the pipe on symbols).
//
// Work: unordered target-tile pairs (A <= B) of 8 inclusions, row-major
// (A, A), (A, A+1), ...; a block is 2c+1 batches (one per image l) of the 64
// rows (m in A, j in B).  Consumer warp w owns target A*8+w (forward) and
// B*8+w (reverse); its lane (b, s) covers row block b against source slot s
// of the batch, so per batch each warp sweeps 8 sources forward and, for
// A < B, 8 sources in reverse, and the source sums are 3-level shuffle trees
// (no shared-memory reduction, no consumer barrier).  Complex MACs use the
// Karatsuba 3-multiplication form (consume_s); one accumulator set is live
// per sweep and is reduced over the source lanes into two persistent rows
// per lane (forward: whole block row, reverse: one block).  Diagonal
// blocks (A = B) run forward only.  k1s_reduce sums the parts in a fixed
// order (deterministic) and applies the Schur epilogue.
#include <cuda_runtime.h>

#include <algorithm>
#include <string>

#include "ctx.cuh"
#include "m2l.cuh"
#include "m2l_sym.cuh"
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

constexpr int kTT = 8;                 // inclusions per tile
constexpr int kNB = 4;                 // row blocks per target
constexpr int kCW = 8;                 // consumer warps (= tile width)
constexpr int kPW = 4;                 // producer warps
constexpr int kThreads = (kCW + kPW) * 32;
#ifndef PS_K1S_CREGS
#define PS_K1S_CREGS 216
#endif
constexpr int kConsumerRegs = PS_K1S_CREGS;
constexpr int kProducerRegs = 504 - 2 * PS_K1S_CREGS;   // the CTA holds 168 x 384 registers (launch bound): 2 C + Pr <= 3 x 168
static_assert(kProducerRegs >= 24 && kProducerRegs % 8 == 0, "setmaxnreg range");
static_assert(2 * kTT * kTT == kPW * 32, "64 rows: two producer lanes per row");

template <int P>
struct ShapeS {
  static constexpr int L = 2 * P + 1;
  static constexpr int NS = 4 * P + 1;
  static constexpr int BO = (L + kNB - 1) / kNB;
  static constexpr int ROWS = BO * kNB;
  static constexpr int FP = ROWS - L;
  static constexpr int NSP = FP + NS + 1;
  static constexpr int SJ = kTT * NSP + 1;        // odd: both access patterns conflict-free
  static constexpr int SYM = kTT * SJ;            // double2 per buffer
  static constexpr size_t SMEM = 2 * (size_t)SYM * sizeof(double2);
};

// Shared-memory layout of a batch: element (row (m, j), slot) at
//   j * SJ + slot * kTT + (m ^ sw(slot)),   sw(slot) = 4 * ((slot / BO) & 1).
// The xor swizzle makes the two row blocks b, b+1 read by one quarter-warp
// land in opposite bank halves, so both consumer access patterns (forward
// rows (w, s), reverse rows (s, w)) are conflict-free with odd SJ.
template <int BO>
__host__ __device__ __forceinline__ int sw_of(int slot) {
  return 4 * ((slot / BO) & 1);
}

template <int P>
__device__ __forceinline__ void produce_s(const ArgsS& a, int A, int B, int li, double2* sym,
                                          int pw, int lane) {
  using S = ShapeS<P>;
  const int row = pw * 16 + (lane >> 1);       // 64 rows over 4 warps x 16 lane pairs
  const bool mirror = lane & 1;
  const int mt = row & 7, jt = row >> 3;       // target slot in A, source slot in B
  const int m = A * kTT + mt, j = B * kTT + jt;
  const int l = li - a.copies;
  bool live = (m < a.M) && (j < a.M) && !(l == 0 && m == j);
  double dx = 1.0, dy = 0.0;
  if (live) {
    const double2 cm = reinterpret_cast<const double2*>(a.centers)[m];
    const double2 cj = reinterpret_cast<const double2*>(a.centers)[j];
    dx = cm.x - cj.x - (double)l * a.period;
    dy = cm.y - cj.y;
  }
  const double rho = live ? hypot(dx, dy) : 1.0;
  const double z = a.k2 * rho;
  int N = live ? miller_start_j01(z) : 2;
  N = __reduce_max_sync(0xffffffffu, N);
  const double inv = live ? 1.0 / rho : 0.0;
  double2* base = sym + (size_t)jt * S::SJ;
  hankel_symbols_half<2 * P>(z, dx * inv, dy * inv, N, mirror, [&](int nu, double re, double im) {
    if (nu == 0 && !live) re = im = 0.0;
    const int slot = S::FP + 2 * P + nu;
    base[slot * kTT + (mt ^ sw_of<S::BO>(slot))] = make_double2(re, im);
  });
}

// One Toeplitz sweep with Karatsuba (3-multiplication) complex products.
// spe / spo: the lane's symbol row at slot R0 - b*BO for the two swizzle
// phases (the phase of slot R0 - b*BO + t is the parity of (R0+t)/BO - b, so
// it is fixed at compile time per step t once b's parity is folded into
// spe / spo).  For c = coef[n] and t = t_{n-r}:
//   S1 += c.x t.x,  S2 += c.y t.y,  S3 += (c.x + c.y)(t.x + t.y)
//   Re = S1 - S2,   Im = S3 - S1 - S2
// so a complex MAC costs 3 DFMA instead of 4; t.x + t.y is formed once per
// symbol as it enters the register window (1 DADD per step, shared by the
// BO rows) and c.x + c.y is precomputed per source (bws / bwsr).
template <int P, bool SMEMCOEF = false>
__device__ __forceinline__ void consume_s(const double2* __restrict__ spe,
                                          const double2* __restrict__ spo,
                                          const double2* __restrict__ bsrc,
                                          const double* __restrict__ ssrc,
                                          double (&acc)[3][ShapeS<P>::BO]) {
  using S = ShapeS<P>;
  constexpr int BO = S::BO;
  constexpr int R0 = S::FP + 2 * P;
  constexpr int MODB = 64 * BO;
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
  auto step = [&](auto n_c) {
    constexpr int n = decltype(n_c)::value;
    constexpr int u = n % BO;
    const double2 nxt = ld(IC<n + 1>{});
    double2 bb;
    double bs;
    if constexpr (SMEMCOEF) {        // rows staged in shared memory (m2l_sym_stage_kernel)
      bb = bsrc[n];
      bs = ssrc[n];
    } else {
      bb = __ldg(bsrc + n);
      bs = __ldg(ssrc + n);
    }
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

// Flush one persistent accumulator set: reduce the Karatsuba sums over the 4
// source lanes s' of a row block (lane bits 0-1; xor 2 then xor 1, each
// level ships half the values -> fixed order, deterministic), then lane s'
// writes rows r0..r0+3 of block b, r0 = 8*bit1 + 4*bit0, as complex values
// (sign_rows: times (-1)^{m'}, reverse parts).  mask: the half-warp whose
// lanes flush together.  The accumulators are cleared.
template <int P>
__device__ __forceinline__ void flush_s(double (&acc)[3][ShapeS<P>::BO], double2* dst, int b,
                                        int sl, bool sign_rows, unsigned mask) {
  using S = ShapeS<P>;
  constexpr int BO = S::BO;
  static_assert(BO <= 16, "four rows per lane");
  auto V = [&](int idx) -> double {           // idx = 3*row + component (row < 16)
    const int r = idx / 3, c = idx % 3;
    return r < BO ? acc[c][r] : 0.0;
  };
  const bool h2 = sl & 2, h1 = sl & 1;
  double v1[24];
#pragma unroll
  for (int k = 0; k < 24; ++k) {
    const double lo = V(k), hi = V(24 + k);
    const double send = h2 ? lo : hi;
    v1[k] = (h2 ? hi : lo) + __shfl_xor_sync(mask, send, 2);
  }
  double v2[12];
#pragma unroll
  for (int k = 0; k < 12; ++k) {
    const double send = h1 ? v1[k] : v1[12 + k];
    v2[k] = (h1 ? v1[12 + k] : v1[k]) + __shfl_xor_sync(mask, send, 1);
  }
  const int r0 = 8 * (h2 ? 1 : 0) + 4 * (h1 ? 1 : 0);
#pragma unroll
  for (int k = 0; k < 4; ++k) {
    const int i = r0 + k, r = b * BO + i;
    if (i < BO && r < S::L) {
      const double s1 = v2[3 * k], s2 = v2[3 * k + 1], s3 = v2[3 * k + 2];
      double2 v = make_double2(s1 - s2, s3 - s1 - s2);
      if (sign_rows && ((r - P) & 1)) v = make_double2(-v.x, -v.y);
      dst[r] = v;
    }
  }
#pragma unroll
  for (int c = 0; c < 3; ++c)
#pragma unroll
    for (int i = 0; i < BO; ++i) acc[c][i] = 0.0;
}

template <int P>
__global__ void __launch_bounds__(kThreads, 1) m2l_sym_kernel(ArgsS a) {
  using S = ShapeS<P>;
  constexpr int BO = S::BO, L = S::L;
  extern __shared__ double2 smem[];
  double2* sym0 = smem;
  double2* sym1 = smem + S::SYM;
  const long long k0 = a.kb0 + (a.nb * blockIdx.x) / gridDim.x;
  const long long k1 = a.kb0 + (a.nb * (blockIdx.x + 1)) / gridDim.x;
  if (k0 >= k1) return;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const bool producer = warp >= kCW;
  const int nbat = (int)(k1 - k0) * a.ncp;      // batches of this CTA

  // zero the pad slots (front FP slots, tail slot) of both buffers once
  // (stored batches carry their own zero pads)
  for (int idx = threadIdx.x; !a.symstore && idx < 2 * kTT * kTT * (S::FP + 1); idx += kThreads) {
    const int buf = idx / (kTT * kTT * (S::FP + 1));
    const int r = idx % (kTT * kTT * (S::FP + 1));
    const int jt = r / (kTT * (S::FP + 1));
    const int r2 = r % (kTT * (S::FP + 1));
    const int q = r2 / kTT, mt = r2 % kTT;
    const int slot = q < S::FP ? q : S::FP + S::NS;
    (buf ? sym1 : sym0)[(size_t)jt * S::SJ + (size_t)slot * kTT + (mt ^ sw_of<S::BO>(slot))] =
        make_double2(0.0, 0.0);
  }
  __syncthreads();

  if (producer) {
    asm volatile("setmaxnreg.dec.sync.aligned.u32 %0;" ::"n"(kProducerRegs));
    const int pw = warp - kCW;
    if (a.symstore) {
      // stored symbols: one lane bulk-copies each batch (TMA, evict-first in
      // L2) into the free buffer and waits for it before the batch barrier
      __shared__ __align__(8) unsigned long long sbar[2];
      const bool lead = pw == 0 && lane == 0;
      const size_t g0 = (size_t)(k0 - a.kb0) * a.ncp;
      unsigned long long pol = 0;
      if (lead) {
        for (int q = 0; q < 2; ++q)
          asm volatile("mbarrier.init.shared.b64 [%0], 1;" ::"r"(
              (unsigned)__cvta_generic_to_shared(&sbar[q])));
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
        asm volatile("createpolicy.fractional.L2::evict_first.b64 %0, 1.0;" : "=l"(pol));
      }
      auto fetch = [&](size_t g, double2* dst, int q) {
        const unsigned bar = (unsigned)__cvta_generic_to_shared(&sbar[q]);
        constexpr unsigned kBytes = (unsigned)(S::SYM * sizeof(double2));
        constexpr unsigned kChunk = 32768;
        asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
        asm volatile("mbarrier.arrive.expect_tx.shared.b64 _, [%0], %1;" ::"r"(bar), "r"(kBytes)
                     : "memory");
        const char* src = reinterpret_cast<const char*>(a.symstore + g * S::SYM);
        const unsigned d0 = (unsigned)__cvta_generic_to_shared(dst);
        for (unsigned off = 0; off < kBytes; off += kChunk) {
          const unsigned n = kBytes - off < kChunk ? kBytes - off : kChunk;
          asm volatile(
              "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes.L2::cache_hint"
              " [%0], [%1], %2, [%3], %4;" ::"r"(d0 + off),
              "l"(src + off), "r"(n), "r"(bar), "l"(pol)
              : "memory");
        }
      };
      auto wait = [&](int q, unsigned parity) {
        const unsigned bar = (unsigned)__cvta_generic_to_shared(&sbar[q]);
        asm volatile(
            "{ .reg .pred p; W: mbarrier.try_wait.parity.shared.b64 p, [%0], %1; @!p bra W; }" ::"r"(
                bar),
            "r"(parity)
            : "memory");
      };
      if (lead) {
        fetch(g0, sym0, 0);
        wait(0, 0);
      }
      __syncthreads();
      for (int it = 0; it < nbat; ++it) {
        if (lead && it + 1 < nbat) {
          const int q = (it + 1) & 1;
          fetch(g0 + it + 1, q ? sym1 : sym0, q);
          wait(q, ((it + 1) >> 1) & 1);
        }
        __syncthreads();
      }
      return;
    }
    int A, B;
    block_ab(k0, a.T, A, B);
    int li = 0;
    produce_s<P>(a, A, B, li, sym0, pw, lane);
    __syncthreads();
    for (int it = 0; it < nbat; ++it) {
      // advance to the batch it + 1
      if (++li == a.ncp) {
        li = 0;
        if (++B == a.T) {
          ++A;
          B = A;
        }
      }
#ifndef PS_K1S_NOPROD   // experiment: consumers alone (wrong results)
      if (it + 1 < nbat) produce_s<P>(a, A, B, li, (it & 1) ? sym0 : sym1, pw, lane);
#endif
      __syncthreads();
    }
    return;
  }
  asm volatile("setmaxnreg.inc.sync.aligned.u32 %0;" ::"n"(kConsumerRegs));
  __syncthreads();

  // Half-warp roles: lanes 0-15 apply the forward rows of target A*8+w,
  // lanes 16-31 the reverse rows of target B*8+w; lane (b, s') covers row
  // block b against source slots s' and s'+4 (two passes per batch).  Each
  // lane keeps ONE persistent accumulator set (forward: whole block row,
  // reverse: one block), so nothing is reduced per sweep.
  const int h = lane >> 4, b = (lane >> 2) & 3, sl = lane & 3;
  const unsigned hmask = h ? 0xffff0000u : 0x0000ffffu;
  double acc[3][BO];
#pragma unroll
  for (int c = 0; c < 3; ++c)
#pragma unroll
    for (int i = 0; i < BO; ++i) acc[c][i] = 0.0;
  const double2* cw = h ? a.bwr : a.bw;
  const double* cs = h ? a.bwsr : a.bws;
  constexpr int R0 = S::FP + 2 * P;
  const int sw_e = 4 * (b & 1), sw_o = 4 * ((b & 1) ^ 1);
  int A, B;
  block_ab(k0, a.T, A, B);
  const int A0 = A;
  long long blk = k0;
  int li = 0;
  for (int it = 0; it < nbat; ++it) {
    const double2* symc = (it & 1) ? sym1 : sym0;
    if (h == 0 || A != B) {
      // forward: row (m = w, j = s), source j = B*8+s image li
      // reverse: row (m = s, j = w), source m = A*8+s image 2c - li
      const int img = h ? 2 * a.copies - li : li;
#pragma unroll
      for (int pass = 0; pass < 2; ++pass) {
        const int s = sl + 4 * pass;
        const int jj = h ? warp : s, mm = h ? s : warp;
        const int src = min((h ? A : B) * kTT + s, a.M - 1);   // dead rows are zero
        const double2* rowp = symc + (size_t)jj * S::SJ + (size_t)(R0 - b * BO) * kTT;
        const size_t g = ((size_t)src * a.ncp + img) * L;
        consume_s<P>(rowp + (mm ^ sw_e), rowp + (mm ^ sw_o), cw + g, cs + g, acc);
      }
    }
    if (li == a.ncp - 1) {                     // block complete
      const bool cross = A != B;
      const long long bdone = blk;
      ++blk;
      li = 0;
      const int Aold = A;
      if (++B == a.T) {
        ++A;
        B = A;
      }
      if (h) {
        if (cross) flush_s<P>(acc, a.bpart + ((size_t)bdone * kTT + warp) * L, b, sl, true, hmask);
      } else if (A != Aold || it + 1 == nbat) {   // block row finished (or CTA done)
        flush_s<P>(acc, a.apart + (((size_t)blockIdx.x * a.maxseg + (Aold - A0)) * kTT + warp) * L,
                   b, sl, false, hmask);
      }
    } else {
      ++li;
    }
    __syncthreads();
  }
}

// K1s fed by the symbol store, with the batch's coefficient rows staged in
// shared memory as well.  The consumers of m2l_sym_kernel read their
// Bloch-weighted coefficient rows with __ldg; every batch touches 16 fresh
// rows, the 28 KB of L1 left beside 211 KB of shared memory do not hold them
// across batches, and the first loads after the batch barrier wait on L2 with
// nothing to hide behind (ncu: long-scoreboard 8.6% of the consumers' time).
// Here the lead producer lane bulk-copies (TMA) the 8 rows of each sweep --
// forward rows of sources B*8 + s, reverse rows of sources A*8 + s, s = 4 pass
// .. 4 pass + 3 -- one sweep ahead:
//   X (first sweep of batch t+1) is refilled once every consumer has left the
//     first sweep of batch t (named barrier 1: consumers arrive, lead waits),
//   Y (second sweep of batch t) right after the batch barrier that ends batch
//     t-1; the consumers wait on its mbarrier before their second sweep.
// Row strides in shared memory (816 B coefficients, 432 B sums) make the
// 8-row LDS.128 / LDS.64 of a warp bank-conflict-free.  The arithmetic and
// its order are those of m2l_sym_kernel: results are bitwise the same.
template <int P>
struct StageS {
  static constexpr int L = 2 * P + 1;
  // global row stride (doubles) of bws / bwsr: a 16-byte multiple for TMA; the
  // sums share a region of 2 L doubles per row, so L + 1 always fits
  static constexpr int LSG = L + 1;
  // shared row stride (doubles) of the sums: = 2 (mod 4), so the 8 rows of a
  // warp's LDS.64 fall in 8 distinct bank pairs (the coefficient rows' 4 L
  // words are = 4 (mod 8) for every odd L: LDS.128 conflict-free as they are)
  static constexpr int LSS = (L + 1) % 4 == 2 ? L + 1 : L + 3;
  static constexpr size_t COEF = 2 * 8 * (size_t)L * sizeof(double2);      // X, Y: [8][L]
  static constexpr size_t SUMS = 2 * 8 * (size_t)LSS * sizeof(double);     // X, Y: [8][LSS]
  static constexpr size_t SMEM = ShapeS<P>::SMEM + COEF + SUMS;
  static constexpr unsigned ROWB = (unsigned)(L * sizeof(double2));        // bytes per coefficient row
  static constexpr unsigned SUMB = (unsigned)(LSG * sizeof(double));       // L sums + 1 pad
};

template <int P>
__global__ void __launch_bounds__(kThreads, 1) m2l_sym_stage_kernel(ArgsS a) {
  using S = ShapeS<P>;
  using G = StageS<P>;
  constexpr int BO = S::BO, L = S::L;
  extern __shared__ double2 smem[];
  double2* sym0 = smem;
  double2* sym1 = smem + S::SYM;
  double2* cbx = smem + 2 * S::SYM;                 // X rows, then Y rows
  double* csx = reinterpret_cast<double*>(cbx + 16 * L);
  __shared__ __align__(8) unsigned long long sbar[2];   // symbol buffers
  __shared__ __align__(8) unsigned long long cbar[2];   // X, Y coefficient rows
  const long long k0 = a.kb0 + (a.nb * blockIdx.x) / gridDim.x;
  const long long k1 = a.kb0 + (a.nb * (blockIdx.x + 1)) / gridDim.x;
  if (k0 >= k1) return;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const bool producer = warp >= kCW;
  const int nbat = (int)(k1 - k0) * a.ncp;
  if (threadIdx.x == 0) {
    for (int q = 0; q < 2; ++q) {
      asm volatile("mbarrier.init.shared.b64 [%0], 1;" ::"r"(
          (unsigned)__cvta_generic_to_shared(&sbar[q])));
      asm volatile("mbarrier.init.shared.b64 [%0], 1;" ::"r"(
          (unsigned)__cvta_generic_to_shared(&cbar[q])));
    }
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __syncthreads();
  auto wait = [&](unsigned long long* b, unsigned parity) {
    const unsigned bar = (unsigned)__cvta_generic_to_shared(b);
    asm volatile(
        "{ .reg .pred p; W: mbarrier.try_wait.parity.shared.b64 p, [%0], %1; @!p bra W; }" ::"r"(bar),
        "r"(parity)
        : "memory");
  };

  if (producer) {
    asm volatile("setmaxnreg.dec.sync.aligned.u32 %0;" ::"n"(kProducerRegs));
    const int pw = warp - kCW;
    if (pw != 0) {                                   // the other producer warps only keep the barrier count
      for (int it = 0; it <= nbat; ++it) __syncthreads();
      return;
    }
    const bool lead = lane == 0;
    const size_t g0 = (size_t)(k0 - a.kb0) * a.ncp;
    unsigned long long pol = 0;
    if (lead) asm volatile("createpolicy.fractional.L2::evict_first.b64 %0, 1.0;" : "=l"(pol));
    auto fetch_sym = [&](size_t g, double2* dst, int q) {
      const unsigned bar = (unsigned)__cvta_generic_to_shared(&sbar[q]);
      constexpr unsigned kBytes = (unsigned)(S::SYM * sizeof(double2));
      constexpr unsigned kChunk = 32768;
      asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
      asm volatile("mbarrier.arrive.expect_tx.shared.b64 _, [%0], %1;" ::"r"(bar), "r"(kBytes)
                   : "memory");
      const char* src = reinterpret_cast<const char*>(a.symstore + g * S::SYM);
      const unsigned d0 = (unsigned)__cvta_generic_to_shared(dst);
      for (unsigned off = 0; off < kBytes; off += kChunk) {
        const unsigned n = kBytes - off < kChunk ? kBytes - off : kChunk;
        asm volatile(
            "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes.L2::cache_hint"
            " [%0], [%1], %2, [%3], %4;" ::"r"(d0 + off),
            "l"(src + off), "r"(n), "r"(bar), "l"(pol)
            : "memory");
      }
    };
    // the 8 coefficient rows (+ sums) of sweep q of batch (A_, B_, li_) into X (q = 0) or Y (q = 1)
    auto fetch_rows = [&](int q, int A_, int B_, int li_) {
      const unsigned bar = (unsigned)__cvta_generic_to_shared(&cbar[q]);
      asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
      asm volatile("mbarrier.arrive.expect_tx.shared.b64 _, [%0], %1;" ::"r"(bar),
                   "r"(8u * (G::ROWB + G::SUMB))
                   : "memory");
      for (int r = 0; r < 8; ++r) {
        const int hh = r >> 2, s = (r & 3) + 4 * q;
        const int src = min((hh ? A_ : B_) * kTT + s, a.M - 1);
        const int img = hh ? 2 * a.copies - li_ : li_;
        const size_t row = (size_t)src * a.ncp + img;
        const double2* gb = (hh ? a.bwr : a.bw) + row * L;
        const double* gs = (hh ? a.bwsr : a.bws) + row * G::LSG;
        const unsigned db = (unsigned)__cvta_generic_to_shared(cbx + (q * 8 + r) * L);
        const unsigned ds = (unsigned)__cvta_generic_to_shared(csx + (q * 8 + r) * G::LSS);
        asm volatile(
            "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::
                "r"(db), "l"(gb), "r"(G::ROWB), "r"(bar)
            : "memory");
        asm volatile(
            "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::
                "r"(ds), "l"(gs), "r"(G::SUMB), "r"(bar)
            : "memory");
      }
    };
    int A, B;
    block_ab(k0, a.T, A, B);
    int li = 0;
    if (lead) {
      fetch_sym(g0, sym0, 0);
      fetch_rows(0, A, B, li);
      fetch_rows(1, A, B, li);
      wait(&sbar[0], 0);
      wait(&cbar[0], 0);
    }
    __syncwarp();
    __syncthreads();
    for (int it = 0; it < nbat; ++it) {
      int An = A, Bn = B, lin = li + 1;               // batch it + 1
      if (lin == a.ncp) {
        lin = 0;
        if (++Bn == a.T) Bn = ++An;
      }
      if (lead) {
        if (it > 0) fetch_rows(1, A, B, li);           // Y(it): batch it - 1 is behind the barrier
        if (it + 1 < nbat) fetch_sym(g0 + it + 1, ((it + 1) & 1) ? sym1 : sym0, (it + 1) & 1);
      }
      __syncwarp();
      asm volatile("bar.sync 1, %0;" ::"n"((kCW + 1) * 32) : "memory");   // consumers left sweep 0
      if (lead && it + 1 < nbat) {
        fetch_rows(0, An, Bn, lin);                    // X(it + 1)
        wait(&sbar[(it + 1) & 1], ((it + 1) >> 1) & 1);
        wait(&cbar[0], (it + 1) & 1);
      }
      __syncwarp();
      __syncthreads();
      A = An;
      B = Bn;
      li = lin;
    }
    return;
  }
  asm volatile("setmaxnreg.inc.sync.aligned.u32 %0;" ::"n"(kConsumerRegs));
  __syncthreads();

  const int h = lane >> 4, b = (lane >> 2) & 3, sl = lane & 3;
  const unsigned hmask = h ? 0xffff0000u : 0x0000ffffu;
  double acc[3][BO];
#pragma unroll
  for (int c = 0; c < 3; ++c)
#pragma unroll
    for (int i = 0; i < BO; ++i) acc[c][i] = 0.0;
  constexpr int R0 = S::FP + 2 * P;
  const int sw_e = 4 * (b & 1), sw_o = 4 * ((b & 1) ^ 1);
  const int crow = h * 4 + sl;                       // this lane's staged row in X / Y
  const double2* cb0 = cbx + crow * L;
  const double2* cb1 = cbx + (8 + crow) * L;
  const double* cs0 = csx + crow * G::LSS;
  const double* cs1 = csx + (8 + crow) * G::LSS;
  int A, B;
  block_ab(k0, a.T, A, B);
  const int A0 = A;
  long long blk = k0;
  int li = 0;
  for (int it = 0; it < nbat; ++it) {
    const double2* symc = (it & 1) ? sym1 : sym0;
    const bool act = h == 0 || A != B;               // diagonal blocks run forward only
    if (act) {
      const int jj = h ? warp : sl, mm = h ? sl : warp;
      const double2* rowp = symc + (size_t)jj * S::SJ + (size_t)(R0 - b * BO) * kTT;
      consume_s<P, true>(rowp + (mm ^ sw_e), rowp + (mm ^ sw_o), cb0, cs0, acc);
    }
    __syncwarp();
    asm volatile("bar.arrive 1, %0;" ::"n"((kCW + 1) * 32) : "memory");   // X may be refilled
    wait(&cbar[1], it & 1);                                            // Y(it) has landed
    if (act) {
      const int s = sl + 4;
      const int jj = h ? warp : s, mm = h ? s : warp;
      const double2* rowp = symc + (size_t)jj * S::SJ + (size_t)(R0 - b * BO) * kTT;
      consume_s<P, true>(rowp + (mm ^ sw_e), rowp + (mm ^ sw_o), cb1, cs1, acc);
    }
    if (li == a.ncp - 1) {                     // block complete
      const bool cross = A != B;
      const long long bdone = blk;
      ++blk;
      li = 0;
      const int Aold = A;
      if (++B == a.T) {
        ++A;
        B = A;
      }
      if (h) {
        if (cross) flush_s<P>(acc, a.bpart + ((size_t)bdone * kTT + warp) * L, b, sl, true, hmask);
      } else if (A != Aold || it + 1 == nbat) {   // block row finished (or CTA done)
        flush_s<P>(acc, a.apart + (((size_t)blockIdx.x * a.maxseg + (Aold - A0)) * kTT + warp) * L,
                   b, sl, false, hmask);
      }
    } else {
      ++li;
    }
    __syncthreads();
  }
}

// bw[g][n] = bloch^{l(g)} beta[j(g)][n]
__global__ void bloch_weight_1(const double2* __restrict__ beta, const double2* __restrict__ bpow,
                               int M, int L, int ncp, int lds, double2* __restrict__ bw,
                               double* __restrict__ bws, double2* __restrict__ bwr,
                               double* __restrict__ bwsr) {
  const long long total = (long long)M * ncp * L;
  for (long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x; i < total;
       i += (long long)gridDim.x * blockDim.x) {
    const int n = (int)(i % L);
    const long long g = i / L;
    const int j = (int)(g / ncp), li = (int)(g % ncp);
    const double2 bv = beta[(long long)j * L + n];
    const double2 wv = bpow[1 + li];
    const double2 v = make_double2(fma(bv.x, wv.x, -bv.y * wv.y), fma(bv.x, wv.y, bv.y * wv.x));
    bw[i] = v;
    const long long is = g * lds + n;                        // sums: row stride lds >= L
    bws[is] = v.x + v.y;
    const bool odd = (n - (L - 1) / 2) & 1;                  // (-1)^{order n}
    bwr[i] = odd ? make_double2(-v.x, -v.y) : v;
    bwsr[is] = odd ? -(v.x + v.y) : v.x + v.y;
  }
}

// The symbol store: batch g of the range [kb0, kb0 + nb) -- block
// kb0 + g / ncp, image g % ncp -- in the K1s shared-memory layout (pad slots
// zero), written by the kernel's own producer code.  One CTA of the 4
// producer warps per batch.
template <int P>
__global__ void __launch_bounds__(kPW * 32) sym_store_kernel(ArgsS a, double2* __restrict__ out) {
  using S = ShapeS<P>;
  const long long g = blockIdx.x;
  const long long k = a.kb0 + g / a.ncp;
  const int li = (int)(g % a.ncp);
  int A, B;
  block_ab(k, a.T, A, B);
  double2* sym = out + (size_t)g * S::SYM;
  for (int idx = threadIdx.x; idx < kTT * kTT * (S::FP + 1); idx += blockDim.x) {
    const int jt = idx / (kTT * (S::FP + 1));
    const int r2 = idx % (kTT * (S::FP + 1));
    const int q = r2 / kTT, mt = r2 % kTT;
    const int slot = q < S::FP ? q : S::FP + S::NS;
    sym[(size_t)jt * S::SJ + (size_t)slot * kTT + (mt ^ sw_of<S::BO>(slot))] = make_double2(0.0, 0.0);
  }
  produce_s<P>(a, A, B, li, sym, threadIdx.x >> 5, threadIdx.x & 31);
}

// out[m][r] for tile X = m / 8, fixed order: reverse parts of the cross
// blocks (A, X), A < X, then the forward parts of the CTAs covering block row
// X -- restricted to the launch's block range [kb0, kb0 + nb) (a multi-GPU
// part; the other parts' contributions arrive through the reduce-scatter).
// The reverse run (up to T - 1 partial rows per output) is split over kRS
// threads in fixed contiguous chunks, combined in chunk order through shared
// memory: deterministic, and the last tiles' long runs no longer serialise
// one thread's L2 loads (a thread per output took ~45 us at cfg3).
constexpr int kRO = 32;   // outputs per CTA
constexpr int kRS = 8;    // chunks of the reverse run per output
__global__ void __launch_bounds__(kRO * kRS) k1s_reduce(
    const double2* __restrict__ apart, const double2* __restrict__ bpart, int T, long long kb0,
    long long nb, int G, int maxseg, int M, int L, int mode, const double2* __restrict__ v_own,
    const double2* __restrict__ sdiag, const double2* __restrict__ bsub, double2* __restrict__ out) {
  __shared__ double2 red[kRS][kRO];
  const int o = threadIdx.x % kRO, q = threadIdx.x / kRO;
  const int idx = blockIdx.x * kRO + o;
  const bool live = idx < M * L;
  const int m = live ? idx / L : 0, r = live ? idx % L : 0;
  const int X = m / kTT, w = m % kTT;
  const long long kb1 = kb0 + nb;
  auto off = [&](int a) -> long long { return (long long)a * T - (long long)a * (a - 1) / 2; };
  auto kbeg = [&](int c) -> long long { return kb0 + (nb * c) / G; };
  double2 sum = make_double2(0.0, 0.0);
  if (live) {
    // the blocks (A, X), A < X, have increasing indices off(A) + X - A: the
    // in-range ones are a contiguous run of A
    int A0 = 0, A1 = X;
    if (kb0 > 0 || kb1 < off(T)) {
      while (A0 < X && off(A0) + (X - A0) < kb0) ++A0;
      A1 = A0;
      while (A1 < X && off(A1) + (X - A1) < kb1) ++A1;
    }
    const int n = A1 - A0;
    const int c0 = A0 + (n * q) / kRS, c1 = A0 + (n * (q + 1)) / kRS;
    double2 s2 = make_double2(0.0, 0.0);
#pragma unroll 4
    for (int A = c0; A < c1; ++A) {
      const long long k = off(A) + (X - A);
      const double2 v = bpart[((size_t)k * kTT + w) * L + r];
      s2.x += v.x;
      s2.y += v.y;
    }
    sum = s2;
  }
  red[q][o] = sum;
  __syncthreads();
  if (q != 0 || !live) return;
  sum = red[0][o];
#pragma unroll
  for (int c = 1; c < kRS; ++c) {
    sum.x += red[c][o].x;
    sum.y += red[c][o].y;
  }
  const long long ra = off(X) > kb0 ? off(X) : kb0;                 // in-range blocks of row X
  const long long rb = off(X + 1) < kb1 ? off(X + 1) : kb1;
  if (ra < rb) {
    int c = (int)(((ra - kb0) * G) / nb);
    if (c >= G) c = G - 1;
    while (c > 0 && kbeg(c) > ra) --c;
    while (c < G - 1 && kbeg(c + 1) <= ra) ++c;
    for (; c < G; ++c) {
      const long long c0 = kbeg(c), c1 = kbeg(c + 1);
      if (c0 >= rb) break;
      if (c1 <= c0 || c1 <= ra) continue;
      // first block row of CTA c
      int a0 = (int)(((2.0 * T + 1.0) - sqrt((2.0 * T + 1.0) * (2.0 * T + 1.0) - 8.0 * (double)c0)) *
                     0.5);
      if (a0 < 0) a0 = 0;
      if (a0 > T - 1) a0 = T - 1;
      while (a0 > 0 && off(a0) > c0) --a0;
      while (a0 < T - 1 && off(a0 + 1) <= c0) ++a0;
      const double2 v = apart[(((size_t)c * maxseg + (X - a0)) * kTT + w) * L + r];
      sum.x += v.x;
      sum.y += v.y;
    }
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
  const double2 sd = sdiag[r];
  const double2 vv = v_own[idx];
  out[idx] = make_double2(vv.x - fma(sd.x, sum.x, -sd.y * sum.y), vv.y - fma(sd.x, sum.y, sd.y * sum.x));
}

// number of block rows a CTA's range touches (host, exact)
int max_rows_per_cta(int T, long long kb0, long long nb, int G) {
  auto off = [&](long long a) { return a * T - a * (a - 1) / 2; };
  auto row_of = [&](long long k) {
    long long a = 0;
    while (a < T - 1 && off(a + 1) <= k) ++a;
    return a;
  };
  int mx = 1;
  for (int c = 0; c < G; ++c) {
    const long long k0 = kb0 + (nb * c) / G, k1 = kb0 + (nb * (c + 1)) / G;
    if (k1 <= k0) continue;
    mx = std::max(mx, (int)(row_of(k1 - 1) - row_of(k0) + 1));
  }
  return mx;
}

// Build (or keep) the symbol store of a's block range when it fits the
// budget and half the free memory; otherwise leave it empty (on-the-fly).
template <int P>
int symbol_store(Ctx* ctx, const ArgsS& a, cudaStream_t st) {
  using S = ShapeS<P>;
  const size_t bytes = (size_t)a.nb * a.ncp * S::SYM * sizeof(double2);
  if (ctx->d_symstore && ctx->sst_kb0 == a.kb0 && ctx->sst_nb == a.nb &&
      ctx->sst_geom == ctx->geom_gen && ctx->sst_p == P)
    return PS_OK;
  if (ctx->d_symstore) ps::dev_free(ctx->d_symstore);
  ctx->d_symstore = nullptr;
  ctx->symstore_bytes = 0;
  ctx->sst_kb0 = ctx->sst_nb = -1;
  if (!(ctx->symstore_max_gb > 0) || (double)bytes > ctx->symstore_max_gb * 1e9 || a.nb <= 0)
    return PS_OK;
  size_t fr = 0, tot = 0;
  PS_CUDA_TRY(ctx, cudaMemGetInfo(&fr, &tot));
  if (bytes > fr / 2) return PS_OK;
  if (ps::dev_malloc(&ctx->d_symstore, bytes) != cudaSuccess) {
    // out of memory (fragmentation despite the free-memory check): no store,
    // the symbols are generated in the kernel as without a budget
    cudaGetLastError();
    ctx->d_symstore = nullptr;
    return PS_OK;
  }
  sym_store_kernel<P><<<(unsigned)(a.nb * a.ncp), kPW * 32, 0, st>>>(a, ctx->d_symstore);
  PS_CUDA_TRY(ctx, cudaGetLastError());
  ctx->launches += 1;
  ctx->symstore_bytes = bytes;
  ctx->sst_kb0 = a.kb0;
  ctx->sst_nb = a.nb;
  ctx->sst_geom = ctx->geom_gen;
  ctx->sst_p = P;
  return PS_OK;
}

template <int P>
int launch_s(Ctx* ctx, const double2* beta, const double2* bpow, double2* out, int mode,
             const double2* v_own, const double2* bsub, cudaStream_t st, const SymOverlap* ov) {
  cudaStream_t ks = ov ? ov->k1_stream : st;
  using S = ShapeS<P>;
  ArgsS a;
  a.centers = ctx->d_centers;
  a.M = ctx->M;
  a.T = (ctx->M + kTT - 1) / kTT;
  a.NB = a.T * (a.T + 1) / 2;
  a.copies = ctx->copies;
  a.ncp = 2 * ctx->copies + 1;
  a.period = ctx->period;
  a.k2 = ctx->k2;
  // multi-GPU part: this launch covers blocks [NB part / nparts, NB (part+1) / nparts)
  a.kb0 = ((long long)a.NB * ctx->sym_part) / ctx->sym_nparts;
  a.nb = ((long long)a.NB * (ctx->sym_part + 1)) / ctx->sym_nparts - a.kb0;
  a.symstore = nullptr;
  int G = ov ? ov->grid : ctx->sm_count - ctx->k1_reserve_sms;
  if (G > a.nb) G = (int)a.nb;
  if (G < 1) G = 1;
  a.maxseg = max_rows_per_cta(a.T, a.kb0, a.nb, G);
  const size_t na = (size_t)G * a.maxseg * kTT * S::L;
  const size_t nbp = (size_t)a.NB * kTT * S::L;
  const size_t npart = na + nbp;
  const bool hmma = ctx->k1_variant == 3;      // K1h (m2l_symh.cu): its own padded weights
  const size_t nbw = (size_t)ctx->M * a.ncp * S::L;
  const size_t nwts = hmma ? symh_weight_elems(P, ctx->M, a.ncp) : 4 * nbw;
  if (ctx->partial_elems < npart + nwts) {
    if (ctx->d_partial) ps::dev_free(ctx->d_partial);
    ctx->d_partial = nullptr;
    ctx->partial_elems = 0;
    PS_CUDA_TRY(ctx, ps::dev_malloc(&ctx->d_partial, (npart + nwts) * sizeof(double2)));
    ctx->partial_elems = npart + nwts;
  }
  a.apart = ctx->d_partial;
  a.bpart = ctx->d_partial + na;
  double2* bw = ctx->d_partial + npart;
  if (hmma) {
    PS_CUDA_TRY(ctx, (cudaError_t)symh_weights(P, &a, beta, bpow - 1, bw, ctx->sm_count, ks));
  } else {
    a.bw = bw;
    double* bws = reinterpret_cast<double*>(bw + nbw);
    double2* bwr = bw + 2 * nbw;
    double* bwsr = reinterpret_cast<double*>(bw + 3 * nbw);
    a.bws = bws;
    a.bwr = bwr;
    a.bwsr = bwsr;
  }
  if (!hmma) {
    if (int rc = symbol_store<P>(ctx, a, ks)) return rc;
    a.symstore = ctx->d_symstore;
  }
  // with the symbol store the coefficient rows are staged in shared memory
  // too (m2l_sym_stage_kernel): their sums then sit at a 16-byte-multiple stride
  const bool stage = !hmma && a.symstore != nullptr && ctx->k1s_stage;
  if (!hmma) {
    bloch_weight_1<<<2 * ctx->sm_count, 256, 0, ks>>>(beta, bpow - 1, ctx->M, S::L, a.ncp,
                                                      stage ? StageS<P>::LSG : S::L, bw,
                                                      const_cast<double*>(a.bws), const_cast<double2*>(a.bwr),
                                                      const_cast<double*>(a.bwsr));
    PS_CUDA_TRY(ctx, cudaGetLastError());
  }
  if (ov) PS_CUDA_TRY(ctx, cudaEventRecord(ov->bw_done, ks));
  static unsigned long long attr_mask = 0;
  if (first_on_device(&attr_mask, ctx->device)) {
    PS_CUDA_TRY(ctx, cudaFuncSetAttribute(m2l_sym_kernel<P>,
                                          cudaFuncAttributeMaxDynamicSharedMemorySize, (int)S::SMEM));
    PS_CUDA_TRY(ctx, cudaFuncSetAttribute(m2l_sym_stage_kernel<P>,
                                          cudaFuncAttributeMaxDynamicSharedMemorySize,
                                          (int)StageS<P>::SMEM));
  }
  cudaEvent_t e0 = nullptr, e1 = nullptr;
  if (ctx->profile) {
    PS_CUDA_TRY(ctx, cudaEventCreate(&e0));
    PS_CUDA_TRY(ctx, cudaEventCreate(&e1));
    PS_CUDA_TRY(ctx, cudaEventRecord(e0, ks));
  }
  if (ctx->k1_variant == 3) {                   // K1h: DMMA consumers (m2l_symh.cu)
    PS_CUDA_TRY(ctx, (cudaError_t)symh_kernel(P, a, G, ks, ctx->device));
  } else if (stage) {
    m2l_sym_stage_kernel<P><<<G, kThreads, StageS<P>::SMEM, ks>>>(a);
    PS_CUDA_TRY(ctx, cudaGetLastError());
  } else {
    m2l_sym_kernel<P><<<G, kThreads, S::SMEM, ks>>>(a);
    PS_CUDA_TRY(ctx, cudaGetLastError());
  }
  if (ctx->profile) {
    PS_CUDA_TRY(ctx, cudaEventRecord(e1, ks));
    ctx->k1_events.push_back({e0, e1});
  }
  const int n = ctx->M * S::L;
  if (ov) {
    if (ctx->tl_k1) PS_CUDA_TRY(ctx, cudaEventRecord(ctx->tl_k1, ks));
    PS_CUDA_TRY(ctx, cudaEventRecord(ov->k1_done, ks));
    if (ov->chain)
      if (int rc = ov->chain(ov->chain_arg)) return rc;
    PS_CUDA_TRY(ctx, cudaStreamWaitEvent(st, ov->k1_done, 0));
    PS_CUDA_TRY(ctx, cudaStreamWaitEvent(st, ov->cpl_done, 0));
  }
  k1s_reduce<<<(n + kRO - 1) / kRO, kRO * kRS, 0, st>>>(a.apart, a.bpart, a.T, a.kb0, a.nb, G,
                                                        a.maxseg, ctx->M, S::L, mode, v_own,
                                                        ctx->d_S, bsub, out);
  PS_CUDA_TRY(ctx, cudaGetLastError());
  ctx->launches += 3;
  return PS_OK;
}

}  // namespace

int m2l_apply_sym(Ctx* ctx, const double2* beta, const double2* bpow, double2* out, int mode,
                  const double2* v_own, const double2* bsub, cudaStream_t st,
                  const SymOverlap* ov) {
  switch (ctx->p) {
#define PS_CASE(P) \
  case P:          \
    return launch_s<P>(ctx, beta, bpow, out, mode, v_own, bsub, st, ov);
    PS_M2L_ORDERS(PS_CASE)
#undef PS_CASE
    default:
      ctx->err = "apply_T (symmetric): multipole order p=" + std::to_string(ctx->p) +
                 " not compiled";
      return PS_ERR_UNSUPPORTED;
  }
}

}  // namespace ps
