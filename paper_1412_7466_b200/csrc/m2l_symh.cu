// K1h: the symmetric all-pairs M2L of K1s (m2l_sym.cu; multiscat.apply_T,
// SPEC.md:504-512) with the Toeplitz applies on the FP64 tensor cores.
//
// The single-RHS apply of a source j to the 8 targets m of a tile,
//   a_m[m'] += sum_n bw_j[n] t^{mj}_{n-m'} = sum_nu bw_j[m' + nu] t^{mj}_nu,
// is a real GEMM once the coefficients are read as a Hankel matrix:
//   C[m'][m] += sum_kappa H_j[m'][kappa] T[kappa][m],
//   H_j[m'][kappa] = bw_j[m' + kappa - 2P - SH],  T[kappa][m] = t^{mj}_{kappa-2P-SH}
// (M = rows m', N = the 8 targets, K = the 4P+1 symbol orders, shifted by SH
// so that every 8-row tile's band starts on a k-tile boundary).  H is banded:
// row tile I only meets the k-tiles K = D - 2I, D in a window of NK values
// that is the SAME for every I, so one source costs NI * NK complex 8x8x4
// tiles -- 0.97 of the algorithmic 8 L^2 flops per translation at p = 25 once
// each tile is three real DMMAs (Karatsuba, as K1d).  The reverse pair
// (j, m, -l) reads the SAME symbol tile with the columns taken along j
// (t' = (-1)^nu t: sign-flipped coefficient copies and a (-1)^{m'} output
// sign, as K1s), so the producer work per translation stays halved.
//
// Warps: one consumer warp per (direction, row tile) -- forward: targets of
// tile A, sources of tile B; reverse: targets of B, sources of A -- all
// running the same code: the row tile only shifts the symbol base by -8I
// (zero-padded kappa range) and the coefficient fragment of D sits at a fixed
// offset of a zero-padded coefficient row.  Each warp keeps its own 8x8 tile
// (three Karatsuba accumulators) over the 8 sources of a batch and flushes it
// straight to the K1s partial layout, so k1s_reduce is shared.  4 producer
// warps build the 64 symbol rows of the next batch; they sit on the
// sub-partitions with the fewest consumer warps (2 NI consumers = 14 at
// p = 25: 4/4/3/3 per SMSP, producers on the two 3s).
#include <cuda_runtime.h>

#include <algorithm>

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

constexpr int kTT = 8;       // inclusions per tile
constexpr int kPW = 4;       // producer warps
constexpr int kWarps = 20;   // launched; roles by role_of (some exit at once)
constexpr int kThreads = kWarps * 32;
static_assert(2 * kTT * kTT == kPW * 32, "64 rows: two producer lanes per row");

template <int P>
struct ShapeH {
  static constexpr int L = 2 * P + 1;
  static constexpr int NI = (L + 7) / 8;                  // row tiles (8 rows each)
  static constexpr int SH = ((7 - 2 * P) % 4 + 4) % 4;    // kappa = nu + 2P + SH
  static constexpr int K00 = (2 * P + SH - 7) / 4;        // first D (exact division)
  static constexpr int NK = (L + 10) / 4;                 // k-tiles per row tile
  static constexpr int NKT = (4 * P + SH) / 4 + 1;        // k-tiles holding symbols
  // per-pair kappa range read by any row tile: K = D - 2I
  static constexpr int KLO = (K00 - 2 * (NI - 1)) < 0 ? (K00 - 2 * (NI - 1)) : 0;
  static constexpr int KHI = (K00 + NK) > NKT ? (K00 + NK) : NKT;
  static constexpr int LEN = 4 * (KHI - KLO);
  // plane layout: symbol (m, j, kappa) at m*SMM + j*SJ + (kappa - 4 KLO), SJ
  // and SMM = 4 mod 8 doubles' quads, so the B-fragment loads (4 columns x 4
  // kappas per half-warp) are conflict-free along m (forward) and j (reverse)
  static constexpr int SJ = ((LEN / 4) & 1) ? LEN : LEN + 4;
  static constexpr int SMM = kTT * SJ + 4;
  static constexpr int PLANE = kTT * SMM;                 // doubles
  static constexpr int BUF = 2 * PLANE;
  static constexpr size_t SMEM = 2 * (size_t)BUF * sizeof(double);
  // zero-padded coefficient rows: element n at F + n, n in [-7, 4 NK - 1]
  static constexpr int F = 8;
  static constexpr int LP = F + 4 * NK;
  static constexpr int NCONS = 2 * NI;
  static_assert(NCONS + kPW <= kWarps, "warp budget");
};

// Warp roles (SMSP = warp % 4, kWarps / 4 slots each): the NCONS consumers
// are spread as evenly as possible over the sub-partitions and the 4
// producers go to the ones with fewer consumers; inside a sub-partition the
// producers take the LOWEST warp ids (the schedulers favour older warps, and
// the producers' latency-bound recurrences sit on the critical path of every
// batch), then the consumers, then idle slots that exit at once.
// Returns 0 consumer, 1 producer, 2 idle; *idx = consumer / producer index.
template <int P>
__host__ __device__ constexpr int role_of(int w, int* idx) {
  constexpr int NC = ShapeH<P>::NCONS;
  int cons[4] = {NC / 4, NC / 4, NC / 4, NC / 4};
  for (int s = 0; s < NC % 4; ++s) ++cons[s];
  int prod[4] = {0, 0, 0, 0};
  for (int n = 0; n < kPW; ++n) {            // fewest warps first, lowest SMSP on ties
    int best = 0;
    for (int s = 1; s < 4; ++s)
      if (cons[s] + prod[s] < cons[best] + prod[best]) best = s;
    ++prod[best];
  }
  for (int s = 0; s < 4; ++s)
    if (cons[s] + prod[s] > kWarps / 4) return -1;   // caught by the static_assert below
  auto role = [&](int u) {                   // role of warp u
    const int s = u % 4, k = u / 4;
    return k < prod[s] ? 1 : (k < prod[s] + cons[s] ? 0 : 2);
  };
  const int r = role(w);
  int n = 0;
  for (int u = 0; u < w; ++u) n += role(u) == r ? 1 : 0;
  *idx = n;
  return r;
}

template <int P>
constexpr bool roles_fit() {
  int i = 0;
  for (int w = 0; w < kWarps; ++w)
    if (role_of<P>(w, &i) < 0) return false;
  return true;
}

__device__ __forceinline__ void dmma(double (&d)[2], double a, double b) {
  asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0, %1}, {%2}, {%3}, {%0, %1};"
               : "+d"(d[0]), "+d"(d[1])
               : "d"(a), "d"(b));
}

template <int P>
__device__ __forceinline__ void produce_h(const ArgsS& a, int A, int B, int li, double* buf, int pw,
                                          int lane) {
  using S = ShapeH<P>;
  const int row = pw * 16 + (lane >> 1);
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
  double* px = buf + mt * S::SMM + jt * S::SJ + (2 * P + S::SH - 4 * S::KLO);
  double* py = px + S::PLANE;
  hankel_symbols_ilp<2 * P>(z, dx * inv, dy * inv, N, mirror, [&](int nu, double re, double im) {
    if (nu == 0 && !live) re = im = 0.0;
    px[nu] = re;
    py[nu] = im;
  });
}

// One source against the warp's row tile.  tx / ty: the lane's B-fragment
// column in the two symbol planes at kappa = -8I + (lane & 3) (so k-tile D
// of the band is at 4D); bsrc / ssrc: the source image's padded coefficient
// row and its re + im at n = rk - 2P - SH (so D is at 4D).
template <int P>
__device__ __forceinline__ void consume_h(const double* __restrict__ tx, const double* __restrict__ ty,
                                          const double2* __restrict__ bsrc,
                                          const double* __restrict__ ssrc, double (&c)[3][2]) {
  using S = ShapeH<P>;
  static_for<S::NK>([&](auto t_c) {
    constexpr int D = S::K00 + decltype(t_c)::value;
    const double bx = tx[4 * D], by = ty[4 * D];
    const double2 av = __ldg(bsrc + 4 * D);
    const double as = __ldg(ssrc + 4 * D);
    dmma(c[0], av.x, bx);
    dmma(c[1], av.y, by);
    dmma(c[2], as, bx + by);
  });
}

template <int P>
__global__ void __launch_bounds__(kThreads, 1) m2l_symh_kernel(ArgsS a) {
  using S = ShapeH<P>;
  static_assert(roles_fit<P>(), "warp roles exceed the sub-partition slots");
  constexpr int L = S::L;
  extern __shared__ double smem_h[];
  double* buf0 = smem_h;
  double* buf1 = smem_h + S::BUF;
  const long long k0 = a.kb0 + (a.nb * blockIdx.x) / gridDim.x;
  const long long k1 = a.kb0 + (a.nb * (blockIdx.x + 1)) / gridDim.x;
  if (k0 >= k1) return;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  int widx = 0;
  const int role = role_of<P>(warp, &widx);
  const int nbat = (int)(k1 - k0) * a.ncp;

  // zero both buffers once: kappa slots outside [SH, 4P + SH] stay zero
  for (int i = threadIdx.x; i < 2 * S::BUF; i += kThreads) smem_h[i] = 0.0;
  __syncthreads();
  if (role == 2) return;                         // idle warp slot (leaves the barriers)

  if (role == 1) {
    int A, B;
    block_ab(k0, a.T, A, B);
    int li = 0;
    produce_h<P>(a, A, B, li, buf0, widx, lane);
    asm volatile("bar.sync 2, %0;" ::"n"((S::NCONS + kPW) * 32));
    for (int it = 0; it < nbat; ++it) {
      if (++li == a.ncp) {
        li = 0;
        if (++B == a.T) {
          ++A;
          B = A;
        }
      }
#ifndef PS_K1H_NOPROD   // experiment: consumers alone (wrong results)
      if (it + 1 < nbat) produce_h<P>(a, A, B, li, (it & 1) ? buf0 : buf1, widx, lane);
#endif
      asm volatile("bar.sync 2, %0;" ::"n"((S::NCONS + kPW) * 32));
    }
    return;
  }
  asm volatile("bar.sync 2, %0;" ::"n"((S::NCONS + kPW) * 32));

  const int dir = widx / S::NI, I = widx % S::NI;   // 0 forward, 1 reverse
  const int fr = lane >> 2, fc = lane & 3;
  // B-fragment column = lane's pair: forward (m = fr, j = s), reverse (m = s, j = fr)
  const int sm_n = dir ? S::SJ : S::SMM;
  const int sm_s = dir ? S::SMM : S::SJ;
  const double2* cw = dir ? a.bwr : a.bw;
  const double* cs = dir ? a.bwsr : a.bws;
  const int boff = fr * sm_n + fc - 8 * I - 4 * S::KLO;   // + 4D: k-tile D - 2I of the band
  const int aoff = S::F + fr + fc - 2 * P - S::SH;        // + 4D: the lane's Hankel element
  double c[3][2] = {{0.0, 0.0}, {0.0, 0.0}, {0.0, 0.0}};
  const int row = 8 * I + fr;

  int A, B;
  block_ab(k0, a.T, A, B);
  const int A0 = A;
  long long blk = k0;
  int li = 0;
  for (int it = 0; it < nbat; ++it) {
    const double* cur = (it & 1) ? buf1 : buf0;
#ifdef PS_K1H_NOCONS    // experiment: producers alone (wrong results)
    if (false) {
#else
    if (dir == 0 || A != B) {
#endif
      const double* px = cur + boff;
      const int img = dir ? 2 * a.copies - li : li;
      const int src0 = (dir ? A : B) * kTT;
#pragma unroll 2
      for (int s0 = 0; s0 < kTT; ++s0) {
        // staggered source order per row tile: the warps of a sub-partition
        // reach their source boundaries (fresh coefficient rows, L1 misses)
        // at different times, so one warp's load bubble is another's issue slot
        const int s = (s0 + I) & (kTT - 1);
        const double* tx = px + sm_s * s;
        const int src = min(src0 + s, a.M - 1);   // dead rows have zero symbols
        const size_t g = ((size_t)src * a.ncp + img) * S::LP + aoff;
        consume_h<P>(tx, tx + S::PLANE, cw + g, cs + g, c);
      }
    }
    if (li == a.ncp - 1) {                       // block complete
      const bool cross = A != B;
      const long long bdone = blk;
      ++blk;
      li = 0;
      const int Aold = A;
      if (++B == a.T) {
        ++A;
        B = A;
      }
      const bool flush = dir == 0 ? ((A != Aold) || (it + 1 == nbat)) : cross;
      if (flush) {
        if (row < L) {
          double2* dst = dir == 0
                             ? a.apart + ((size_t)blockIdx.x * a.maxseg + (Aold - A0)) * kTT * L
                             : a.bpart + (size_t)bdone * kTT * L;
          const bool neg = dir == 1 && ((row - P) & 1);
#pragma unroll
          for (int u = 0; u < 2; ++u) {
            double2 v = make_double2(c[0][u] - c[1][u], c[2][u] - c[0][u] - c[1][u]);
            if (neg) v = make_double2(-v.x, -v.y);
            dst[(2 * fc + u) * L + row] = v;
          }
        }
        c[0][0] = c[0][1] = c[1][0] = c[1][1] = c[2][0] = c[2][1] = 0.0;
      }
    } else {
      ++li;
    }
    asm volatile("bar.sync 2, %0;" ::"n"((S::NCONS + kPW) * 32));
  }
}

// padded Bloch-weighted coefficient rows (K1h A operand):
//   bw[g][F + n] = bloch^{l(g)} beta[j(g)][n], zero outside 0 <= n < L,
// plus re + im and the (-1)^{n-P} reverse copies
template <int P>
__global__ void bloch_weight_h(const double2* __restrict__ beta, const double2* __restrict__ bpow,
                               int M, int ncp, double2* __restrict__ bw, double* __restrict__ bws,
                               double2* __restrict__ bwr, double* __restrict__ bwsr) {
  using S = ShapeH<P>;
  const long long total = (long long)M * ncp * S::LP;
  for (long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x; i < total;
       i += (long long)gridDim.x * blockDim.x) {
    const int n = (int)(i % S::LP) - S::F;
    const long long g = i / S::LP;
    double2 v = make_double2(0.0, 0.0);
    if (n >= 0 && n < S::L) {
      const int j = (int)(g / ncp), li = (int)(g % ncp);
      const double2 bv = beta[(long long)j * S::L + n];
      const double2 wv = bpow[1 + li];
      v = make_double2(fma(bv.x, wv.x, -bv.y * wv.y), fma(bv.x, wv.y, bv.y * wv.x));
    }
    bw[i] = v;
    bws[i] = v.x + v.y;
    const bool odd = (n - P) & 1;
    bwr[i] = odd ? make_double2(-v.x, -v.y) : v;
    bwsr[i] = odd ? -(v.x + v.y) : v.x + v.y;
  }
}

template <int P>
int weights_h(ArgsS* a, const double2* beta, const double2* bpow, double2* wts, int nsm,
              cudaStream_t st) {
  using S = ShapeH<P>;
  const size_t nw = (size_t)a->M * a->ncp * S::LP;
  a->bw = wts;
  a->bws = reinterpret_cast<const double*>(wts + nw);
  a->bwr = wts + 2 * nw;
  a->bwsr = reinterpret_cast<const double*>(wts + 3 * nw);
  bloch_weight_h<P><<<2 * nsm, 256, 0, st>>>(beta, bpow, a->M, a->ncp, wts,
                                             reinterpret_cast<double*>(wts + nw), wts + 2 * nw,
                                             reinterpret_cast<double*>(wts + 3 * nw));
  return (int)cudaGetLastError();
}

template <int P>
int kernel_h(const ArgsS& a, int grid, cudaStream_t st, int device) {
  using S = ShapeH<P>;
  static unsigned long long attr_mask = 0;
  if (!(attr_mask & (1ull << device))) {
    cudaError_t e = cudaFuncSetAttribute(m2l_symh_kernel<P>,
                                         cudaFuncAttributeMaxDynamicSharedMemorySize, (int)S::SMEM);
    if (e != cudaSuccess) return (int)e;
    attr_mask |= 1ull << device;
  }
  m2l_symh_kernel<P><<<grid, kThreads, S::SMEM, st>>>(a);
  return (int)cudaGetLastError();
}

}  // namespace

size_t symh_weight_elems(int p, int M, int ncp) {
  switch (p) {
#define PS_CASE(P) \
  case P:          \
    return 4 * (size_t)M * ncp * ShapeH<P>::LP;
    PS_M2L_ORDERS(PS_CASE)
#undef PS_CASE
    default:
      return 0;
  }
}

int symh_weights(int p, ArgsS* a, const double2* beta, const double2* bpow, double2* wts, int nsm,
                 cudaStream_t st) {
  switch (p) {
#define PS_CASE(P) \
  case P:          \
    return weights_h<P>(a, beta, bpow, wts, nsm, st);
    PS_M2L_ORDERS(PS_CASE)
#undef PS_CASE
    default:
      return (int)cudaErrorInvalidValue;
  }
}

int symh_kernel(int p, const ArgsS& a, int grid, cudaStream_t st, int device) {
  switch (p) {
#define PS_CASE(P) \
  case P:          \
    return kernel_h<P>(a, grid, st, device);
    PS_M2L_ORDERS(PS_CASE)
#undef PS_CASE
    default:
      return (int)cudaErrorInvalidValue;
  }
}

}  // namespace ps
