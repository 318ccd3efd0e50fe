// Schur-complement correction of the preconditioned operator
//   K v = v - S (T v - B_phys A^+ C v)          (B = -B_phys)
// (solver.apply_schur_operator).
//
//   K3 c_kernel   : g = C beta -- particle field values / normal derivatives on
//                   Gamma1 (negated), Gamma2 and the telescoped L2 wall rows
//                   (multiscat.multipole_to_targets_block, SPEC.md:494-502;
//                   wall telescoping as layerpot.wall_discrepancy_blocks,
//                   layerpot.py:211-237).
//   K4 pinv_*     : A^+ g = col_scale .* V (Sigma^+ (U^* g)) restricted to the
//                   rows C touches and the columns B reads
//                   (empty_grating.apply_pinv, empty_grating.py:264-273).
//   K5 b_kernel   : local coefficients at every owned inclusion of the layer-2
//                   field: phased single/double layers on Gamma1, Gamma2 at k2
//                   plus the L2L of the a2 J-expansion
//                   (multiscat.source_to_local_block).
//
// All three reuse the translation-symbol generator of K1: with
// w_n = H_n(k r) e^{i n theta},
//   (d/dx + i d/dy) w_n = -k w_{n+1},  (d/dx - i d/dy) w_n = k w_{n-1},
// so a field gradient and a double-layer (dipole) source are both two extra
// symbol orders of the same row.
#include <cuda_runtime.h>

#include <algorithm>
#include <string>

#include "coupling.cuh"
#include "m2l.cuh"
#include "symbols.cuh"

namespace ps {

namespace {

constexpr int kCT = 128;   // threads per CTA for K3 / K5

__device__ __forceinline__ double2 cmul(double2 a, double2 b) {
  return make_double2(fma(a.x, b.x, -a.y * b.y), fma(a.x, b.y, a.y * b.x));
}
__device__ __forceinline__ double2 cfma(double2 a, double2 b, double2 c) {
  return make_double2(fma(a.x, b.x, fma(-a.y, b.y, c.x)), fma(a.x, b.y, fma(a.y, b.x, c.y)));
}

// ---------------------------------------------------------------- K3: C beta
// grid (target node, source split).  With w_nu = H_nu(k r) e^{i nu theta} about a
// source image evaluated at the node:
//   u     = sum_n beta_n w_n
//   du/dn = (k/2)[(nx + i ny) sum_nu beta_{nu+1} w_nu + (-nx + i ny) sum_nu beta_{nu-1} w_nu]
// so each pair accumulates three sums (val, S+, S-) and the node normal is
// applied once per CTA.
struct CArgs {
  const double* centers;   // [M][2]
  const double2* beta;     // [M][L]
  const double2* bpow;     // bloch^l, l = -(P+1)..P+1 (index l + P + 1)
  const double* g1;        // [n1][5]
  const double* g2;        // [n2][5]
  const double* w2;        // [nw][2]
  double2* gpart;          // [nsplit][nrow_c]
  int n1, n2, nw, copies, s_begin, s_end, nrow_c;
  double period, k2;
};

// One (node, source image) pair of K3: symbols t_{+-nu}, nu = 0..P+1, built
// by the reference recurrence (symbols.cuh) and folded straight into
//   pv += sum_n b_n w_n,  pp += sum_nu b_{nu+1} w_nu,  pm += sum_nu b_{nu-1} w_nu
// with every beta index a compile-time offset (fully unrolled) so the loads
// are hoisted out of the recurrence.
template <int P>
__device__ __forceinline__ void c_pair(double z, double c, double s, int N,
                                       const double2* __restrict__ bj, double2& pv, double2& pp,
                                       double2& pm) {
  auto B = [&](int n) -> double2 {
    return (n >= -P && n <= P) ? __ldg(bj + n + P) : make_double2(0.0, 0.0);
  };
  double j0, j1, y0, y1;
  bessel_jy01(z, N, &j0, &j1, &y0, &y1);
  {
    const double2 w = make_double2(j0, y0);
    pv = cfma(B(0), w, pv);
    pp = cfma(B(1), w, pp);
    pm = cfma(B(-1), w, pm);
  }
  double hmr = j0, hmi = y0, hr = j1, hi = y1, pr = c, pi = s;
  const double tz = 2.0 / z;
#pragma unroll
  for (int nu = 1; nu <= P + 1; ++nu) {
    const double2 tp = make_double2(fma(hr, pr, -hi * pi), fma(hr, pi, hi * pr));
    const double sg = (nu & 1) ? -1.0 : 1.0;
    const double2 tm = make_double2(sg * fma(hr, pr, hi * pi), sg * fma(hi, pr, -hr * pi));
    if (nu <= P) {
      pv = cfma(B(nu), tp, pv);
      pv = cfma(B(-nu), tm, pv);
    }
    pp = cfma(B(nu + 1), tp, pp);
    pp = cfma(B(1 - nu), tm, pp);
    pm = cfma(B(nu - 1), tp, pm);
    pm = cfma(B(-nu - 1), tm, pm);
    const double cf = (double)nu * tz;
    const double nr = fma(cf, hr, -hmr), ni = fma(cf, hi, -hmi);
    hmr = hr;
    hmi = hi;
    hr = nr;
    hi = ni;
    const double qr = fma(pr, c, -pi * s), qi = fma(pr, s, pi * c);
    pr = qr;
    pi = qi;
  }
}

template <int P>
__global__ void __launch_bounds__(kCT) c_kernel(CArgs a) {
  constexpr int L = 2 * P + 1;
  __shared__ double2 red[3 * kCT];
  const int row = blockIdx.x;              // target node index over g1, g2, wall
  double tx, ty, nx, ny, sgn;
  int kind;                                // 0 interface, 1 wall
  int rv, rd;
  if (row < a.n1) {
    const double* q = a.g1 + 5 * row;
    tx = q[0]; ty = q[1]; nx = q[2]; ny = q[3]; sgn = -1.0; kind = 0;
    rv = row; rd = a.n1 + row;
  } else if (row < a.n1 + a.n2) {
    const int i = row - a.n1;
    const double* q = a.g2 + 5 * i;
    tx = q[0]; ty = q[1]; nx = q[2]; ny = q[3]; sgn = 1.0; kind = 0;
    rv = 2 * a.n1 + i; rd = 2 * a.n1 + a.n2 + i;
  } else {
    const int i = row - a.n1 - a.n2;
    tx = a.w2[2 * i]; ty = a.w2[2 * i + 1]; nx = 1.0; ny = 0.0; sgn = 1.0; kind = 1;
    rv = 2 * a.n1 + 2 * a.n2 + i; rd = rv + a.nw;
  }
  const int P_ = a.copies;
  // interface rows: l = -P..P, weight bloch^l; wall rows: the telescoped
  // extremes +bloch^{P+1} at shift +P d and -bloch^{-P} at shift -(P+1) d
  const int nl = kind == 0 ? 2 * P_ + 1 : 2;
  const int npair = (a.s_end - a.s_begin) * nl;
  const int per = (npair + gridDim.y - 1) / gridDim.y;
  const int p0 = blockIdx.y * per;
  const int p1 = min(npair, p0 + per);
  double2 val = make_double2(0, 0), sp = make_double2(0, 0), sm = make_double2(0, 0);
  for (int it = p0 + threadIdx.x; it < p1; it += kCT) {
    const int j = a.s_begin + it / nl;
    const int li = it % nl;
    int l;
    double2 wgt;
    if (kind == 0) {
      l = li - P_;
      wgt = a.bpow[l + P_ + 1];
    } else if (li == 0) {
      l = P_;
      wgt = a.bpow[2 * P_ + 2];
    } else {
      l = -(P_ + 1);
      const double2 b = a.bpow[1];
      wgt = make_double2(-b.x, -b.y);
    }
    const double dx = tx - a.centers[2 * j] - (double)l * a.period;
    const double dy = ty - a.centers[2 * j + 1];
    const double rho = hypot(dx, dy);
    const double inv = 1.0 / rho;
    const double2* bj = a.beta + (size_t)j * L;
    double2 pv = make_double2(0, 0), pp = make_double2(0, 0), pm = make_double2(0, 0);
    const double zz = a.k2 * rho;
    c_pair<P>(zz, dx * inv, dy * inv, miller_start_j01(zz), bj, pv, pp, pm);
    val = cfma(wgt, pv, val);
    sp = cfma(wgt, pp, sp);
    sm = cfma(wgt, pm, sm);
  }
  // deterministic block reduction of (val, S+, S-)
  red[threadIdx.x] = val;
  red[kCT + threadIdx.x] = sp;
  red[2 * kCT + threadIdx.x] = sm;
  __syncthreads();
  for (int st = kCT / 2; st > 0; st >>= 1) {
    if (threadIdx.x < st) {
#pragma unroll
      for (int q = 0; q < 3; ++q) {
        red[q * kCT + threadIdx.x].x += red[q * kCT + threadIdx.x + st].x;
        red[q * kCT + threadIdx.x].y += red[q * kCT + threadIdx.x + st].y;
      }
    }
    __syncthreads();
  }
  if (threadIdx.x == 0) {
    const double hk = 0.5 * a.k2;
    const double2 cp = make_double2(hk * nx, hk * ny);    // (k/2)(nx + i ny)
    const double2 cm = make_double2(-hk * nx, hk * ny);   // (k/2)(-nx + i ny)
    const double2 v = red[0];
    const double2 d = cfma(cm, red[2 * kCT], cmul(cp, red[kCT]));
    double2* gp = a.gpart + (size_t)blockIdx.y * a.nrow_c;
    gp[rv] = make_double2(sgn * v.x, sgn * v.y);
    gp[rd] = make_double2(sgn * d.x, sgn * d.y);
  }
}

// g[i] = sum_s gpart[s][i]  (fixed split order)
__global__ void sum_splits(const double2* __restrict__ part, int nsplit, int n,
                           double2* __restrict__ g) {
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n) return;
  double2 s = make_double2(0, 0);
  for (int q = 0; q < nsplit; ++q) {
    const double2 v = part[(size_t)q * n + i];
    s.x += v.x;
    s.y += v.y;
  }
  g[i] = s;
}

// ---------------------------------------------------------------- K4: A^+ g
// y[r] = scale[r] * sum_k A[r][k] x[k]: kRowT threads per row (kRows rows per
// CTA), each thread's strided elements loaded before any FMA (independent
// loads in flight), warp shuffles then the row's warps summed in warp order
// through shared memory (deterministic).  781 / 635 rows of 576 / 781 complex
// entries: ~400 CTAs instead of ~100 warp-per-row blocks.
constexpr int kRowT = 128, kRows = 2;
__global__ void __launch_bounds__(kRowT * kRows) pinv_gemv(const double2* __restrict__ A,
                                                           const double* __restrict__ scale,
                                                           const double2* __restrict__ x, int nrow,
                                                           int ncol, double2* __restrict__ y) {
  __shared__ double2 red[kRows][kRowT / 32];
  const int rl = threadIdx.x / kRowT, t = threadIdx.x % kRowT;
  const int r = blockIdx.x * kRows + rl;
  double2 s = make_double2(0, 0);
  if (r < nrow) {
    // every element of the thread's stride in flight at once (ncol <= 8 kRowT
    // here: 576 / 781), then the FMAs in order
    const double2* a = A + (size_t)r * ncol;
    constexpr int U = 8;
    double2 av[U], xv[U];
#pragma unroll
    for (int u = 0; u < U; ++u) {
      const int k = t + u * kRowT;
      av[u] = k < ncol ? __ldcs(a + k) : make_double2(0, 0);
      xv[u] = k < ncol ? __ldg(x + k) : make_double2(0, 0);
    }
#pragma unroll
    for (int u = 0; u < U; ++u) s = cfma(av[u], xv[u], s);
    for (int k = t + U * kRowT; k < ncol; k += kRowT) s = cfma(__ldcs(a + k), __ldg(x + k), s);
  }
  for (int o = 16; o > 0; o >>= 1) {
    s.x += __shfl_xor_sync(0xffffffffu, s.x, o);
    s.y += __shfl_xor_sync(0xffffffffu, s.y, o);
  }
  if ((t & 31) == 0) red[rl][t / 32] = s;
  __syncthreads();
  if (t == 0 && r < nrow) {
    double2 v = red[rl][0];
#pragma unroll
    for (int w = 1; w < kRowT / 32; ++w) {
      v.x += red[rl][w].x;
      v.y += red[rl][w].y;
    }
    y[r] = make_double2(v.x * scale[r], v.y * scale[r]);
  }
}

// g_out = f - g_in  (recovery right-hand side)
__global__ void f_minus(const double2* __restrict__ f, const double2* __restrict__ g, int n,
                        double2* __restrict__ out) {
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i < n) out[i] = make_double2(f[i].x - g[i].x, f[i].y - g[i].y);
}

// ---------------------------------------------------------------- K5: B_phys x
// grid (owned inclusion m, source chunk).  A source is an interface node y of
// Gamma1/Gamma2 in copy l: single layer = monopole (i/4) bloch^l w sigma,
// double layer = dipole with outgoing coefficients
//   beta_1 = (k/2)(nx - i ny) c_d,  beta_-1 = -(k/2)(nx + i ny) c_d,
// (c_d = (i/4) bloch^l w mu), translated to x_m with the M2L symbols
// t_nu of (x_m - y_l):  a[n'] += c_s t_{-n'} + beta_1 t_{1-n'} + beta_-1 t_{-1-n'}.
// Chunk c = 0 additionally adds the L2L of the a2 J-expansion (B_pm).
constexpr int kBT = 128;   // threads for K5: two lanes per source (t_+nu / t_-nu halves)
constexpr int kBS = 64;    // sources per chunk

struct BArgs {
  const double* centers;   // [M][2]
  const double2* x;        // [ncol_b] physical empty-grating unknowns
  const double2* bpow;     // bloch^l (index l + P + 1)
  const double* g1;
  const double* g2;
  double2* bpart;          // [nchunk][nt][L]
  int n1, n2, copies, t_begin, nt, Q, nchunk;
  double period, k2, x2x, x2y;
};

template <int P>
struct BShape {
  static constexpr int NU = P + 1;
  static constexpr int NSP = 2 * NU + 1;           // odd: conflict-free row stride
  static constexpr int L = 2 * P + 1;
  static constexpr int NQMAX = 36 + P;             // sized for Q <= 36 (ProblemConfig default)
  static constexpr size_t SMEM_SYM = (size_t)kBS * NSP * sizeof(double2);
  static constexpr size_t SMEM_JL = (size_t)(2 * NQMAX + 1) * sizeof(double2);
  static constexpr size_t SMEM = (SMEM_SYM > SMEM_JL ? SMEM_SYM : SMEM_JL) + 3 * kBS * sizeof(double2);
};

template <int P>
__global__ void __launch_bounds__(kBT) b_kernel(BArgs a) {
  using S = BShape<P>;
  constexpr int NU = S::NU, NSP = S::NSP, L = S::L;
  static_assert(L <= kBT / 2, "one output order per thread of each half-CTA");
  extern __shared__ double2 bsm[];
  double2* sym = bsm;                                   // [kBS][NSP]
  double2* coef = bsm + (S::SMEM_SYM > S::SMEM_JL ? kBS * NSP : 2 * S::NQMAX + 1);   // [kBS][3]
  const int mloc = blockIdx.x;
  const int m = a.t_begin + mloc;
  const int chunk = blockIdx.y;
  const double xm = a.centers[2 * m], ym = a.centers[2 * m + 1];
  const int nl = 2 * a.copies + 1;
  const int nsrc = (a.n1 + a.n2) * nl;
  const double hk = 0.5 * a.k2;
  const int src = threadIdx.x >> 1;          // lanes 2q, 2q+1 share source q
  const bool mirror = threadIdx.x & 1;
  const int it = chunk * kBS + src;
  const int nlive = min(kBS, nsrc - chunk * kBS);
  {
    double2* row = sym + (size_t)src * NSP;
    if (it < nsrc) {
      const int node = it / nl;
      const int l = it % nl - a.copies;
      const bool on1 = node < a.n1;
      const double* q = on1 ? a.g1 + 5 * node : a.g2 + 5 * (node - a.n1);
      const int mu_col = on1 ? node : 2 * a.n1 + (node - a.n1);
      const int sg_col = on1 ? a.n1 + node : 2 * a.n1 + a.n2 + (node - a.n1);
      const double2 wl = a.bpow[l + a.copies + 1];
      const double w = q[4];
      const double2 iw = make_double2(-0.25 * w * wl.y, 0.25 * w * wl.x);   // (i/4) bloch^l w
      const double2 cd = cmul(iw, a.x[mu_col]);
      const double nx = q[2], ny = q[3];
      if (!mirror) {
        coef[3 * src + 0] = cmul(iw, a.x[sg_col]);
        coef[3 * src + 1] = cmul(cd, make_double2(hk * nx, -hk * ny));
        coef[3 * src + 2] = cmul(cd, make_double2(-hk * nx, -hk * ny));
      }
      const double dx = xm - q[0] - (double)l * a.period;
      const double dy = ym - q[1];
      const double rho = hypot(dx, dy);
      const double inv = 1.0 / rho;
      double2* r0 = row + NU;
      const double zz = a.k2 * rho;
      hankel_symbols_half<NU>(zz, dx * inv, dy * inv, miller_start_j01(zz), mirror,
                              [&](int nu, double re, double im) { r0[nu] = make_double2(re, im); });
    }
  }
  __syncthreads();
  // accumulation: half h of the CTA sums sources [h*kBS/2, (h+1)*kBS/2) for
  // output order n' = (threadIdx.x % (kBT/2)) - P, then the halves combine
  double2 out = make_double2(0, 0);
  const int half = threadIdx.x / (kBT / 2), op = threadIdx.x % (kBT / 2);
  if (op < L) {
    const int nprime = op - P;
    // six independent chains: (monopole, dipole+, dipole-) x (even, odd source)
    double2 c0 = make_double2(0, 0), c1 = c0, c2 = c0, c3 = c0, c4 = c0, c5 = c0;
    const int y0 = half * (kBS / 2);
    const int y1 = min(nlive, y0 + kBS / 2);
    int y = y0;
    for (; y + 1 < y1; y += 2) {
      const double2* r = sym + (size_t)y * NSP + NU;
      const double2* r2 = r + NSP;
      c0 = cfma(coef[3 * y + 0], r[-nprime], c0);
      c1 = cfma(coef[3 * y + 1], r[1 - nprime], c1);
      c2 = cfma(coef[3 * y + 2], r[-1 - nprime], c2);
      c3 = cfma(coef[3 * y + 3], r2[-nprime], c3);
      c4 = cfma(coef[3 * y + 4], r2[1 - nprime], c4);
      c5 = cfma(coef[3 * y + 5], r2[-1 - nprime], c5);
    }
    if (y < y1) {
      const double2* r = sym + (size_t)y * NSP + NU;
      c0 = cfma(coef[3 * y + 0], r[-nprime], c0);
      c1 = cfma(coef[3 * y + 1], r[1 - nprime], c1);
      c2 = cfma(coef[3 * y + 2], r[-1 - nprime], c2);
    }
    out = make_double2(((c0.x + c3.x) + (c1.x + c4.x)) + (c2.x + c5.x),
                       ((c0.y + c3.y) + (c1.y + c4.y)) + (c2.y + c5.y));
  }
  __syncthreads();                       // symbol rows no longer needed
  double2* comb = sym;                   // [kBT/2] partials of half 1
  if (half == 1 && op < L) comb[op] = out;
  __syncthreads();
  if (half == 0 && op < L) {
    out.x += comb[op].x;
    out.y += comb[op].y;
  }
  if (chunk == 0) {
    // B_pm: L2L of the a2 expansion about x2:
    //   a[n'] += sum_q a2_q J_{q-n'}(k2 rho) e^{i(q-n') phi},  (rho, phi) = polar(x_m - x2)
    __syncthreads();
    const int NQ = a.Q + P;
    double2* jl = sym;                         // [2*NQ+1] signed orders, reuse
    if (threadIdx.x == 0) {
      const double dx = xm - a.x2x, dy = ym - a.x2y;
      const double rho = hypot(dx, dy);
      double2* j0 = jl + NQ;
      if (rho == 0.0) {
        for (int nu = -NQ; nu <= NQ; ++nu) j0[nu] = make_double2(nu == 0 ? 1.0 : 0.0, 0.0);
      } else {
        const double z = a.k2 * rho;
        double inv_norm, y0, y1;
        bessel_jy_sweep(z, NQ, [&](int nu, double v) { j0[nu].x = v; }, &inv_norm, &y0, &y1);
        const double c = dx / rho, s = dy / rho;
        double pr = 1.0, pi = 0.0;
        j0[0] = make_double2(j0[0].x * inv_norm, 0.0);
        for (int nu = 1; nu <= NQ; ++nu) {
          const double npr = fma(pr, c, -pi * s);
          const double npi = fma(pr, s, pi * c);
          pr = npr;
          pi = npi;
          const double J = j0[nu].x * inv_norm;
          const double sg = (nu & 1) ? -1.0 : 1.0;
          j0[nu] = make_double2(J * pr, J * pi);
          j0[-nu] = make_double2(sg * J * pr, -sg * J * pi);
        }
      }
    }
    __syncthreads();
    if (threadIdx.x < L) {
      const int nprime = threadIdx.x - P;
      const double2* a2 = a.x + 2 * a.n1 + 2 * a.n2;   // a2 column block
      for (int qq = -a.Q; qq <= a.Q; ++qq) out = cfma(a2[qq + a.Q], jl[NQ + qq - nprime], out);
    }
  }
  if (threadIdx.x < L)
    a.bpart[((size_t)chunk * a.nt + mloc) * L + threadIdx.x] = out;
}

// y[m][r] = v[m][r] + sgn sum_n e^{i rot_m (r-n)} s[r][n] u[m][n]  (dense S)
__global__ void dense_s_epilogue(const double2* __restrict__ S, const double* __restrict__ rot,
                                 const double2* __restrict__ v_own, const double2* __restrict__ u,
                                 int t_begin, int L, double sgn, double2* __restrict__ y) {
  extern __shared__ double2 us[];
  const int mloc = blockIdx.x;
  for (int n = threadIdx.x; n < L; n += blockDim.x) us[n] = u[(size_t)mloc * L + n];
  __syncthreads();
  const double phi = rot ? rot[t_begin + mloc] : 0.0;
  for (int r = threadIdx.x; r < L; r += blockDim.x) {
    double2 s = make_double2(0, 0);
    for (int n = 0; n < L; ++n) {
      double2 e = S[(size_t)r * L + n];
      if (rot) {
        double sn, cn;
        sincos(phi * (double)(r - n), &sn, &cn);
        e = cmul(e, make_double2(cn, sn));
      }
      s = cfma(e, us[n], s);
    }
    const double2 vv = v_own ? v_own[(size_t)mloc * L + r] : make_double2(0, 0);
    y[(size_t)mloc * L + r] = make_double2(fma(sgn, s.x, vv.x), fma(sgn, s.y, vv.y));
  }
}

int c_splits(const Ctx* c, int s0, int s1) {
  // one full wave at 8 CTAs/SM, but at least ~2 pairs per thread and at most
  // ~64 pairs per thread
  const int rows = c->n1 + c->n2 + c->nw;
  const long long npair = (long long)(s1 - s0) * (2 * c->copies + 1);
  long long ns = (8LL * c->sm_count + rows - 1) / rows;
  const long long lo = (npair + 64LL * kCT - 1) / (64LL * kCT);
  const long long hi = (npair + 2LL * kCT - 1) / (2LL * kCT);
  if (ns < lo) ns = lo;
  if (ns > hi) ns = hi;
  if (ns < 1) ns = 1;
  if (ns > 512) ns = 512;
  return (int)ns;
}

int b_chunks(const Ctx* c) {
  const int nsrc = (c->n1 + c->n2) * (2 * c->copies + 1);
  return (nsrc + kBS - 1) / kBS;
}

template <int P>
int launch_c(Ctx* c, const double2* beta, const double2* bpow, double2* gpart, double2* g, int s0,
             int s1, cudaStream_t st) {
  CArgs a;
  a.centers = c->d_centers;
  a.beta = beta;
  a.bpow = bpow;
  a.g1 = c->d_g1;
  a.g2 = c->d_g2;
  a.w2 = c->d_w2;
  a.gpart = gpart;
  a.n1 = c->n1;
  a.n2 = c->n2;
  a.nw = c->nw;
  a.copies = c->copies;
  a.s_begin = s0;
  a.s_end = s1;
  a.nrow_c = c->nrow_c;
  a.period = c->period;
  a.k2 = c->k2;
  const int ns = c_splits(c, s0, s1);
  c_kernel<P><<<dim3(c->n1 + c->n2 + c->nw, ns), kCT, 0, st>>>(a);
  PS_CUDA_TRY(c, cudaGetLastError());
  sum_splits<<<(c->nrow_c + 255) / 256, 256, 0, st>>>(gpart, ns, c->nrow_c, g);
  PS_CUDA_TRY(c, cudaGetLastError());
  c->launches += 2;
  return PS_OK;
}

template <int P>
int launch_b(Ctx* c, const double2* x, const double2* bpow, double2* bpart, double2* out,
             cudaStream_t st) {
  using S = BShape<P>;
  if (c->Q > 36) {
    c->err = "apply_B: J-expansion order Q > 36 not supported";
    return PS_ERR_UNSUPPORTED;
  }
  BArgs a;
  a.centers = c->d_centers;
  a.x = x;
  a.bpow = bpow;
  a.g1 = c->d_g1;
  a.g2 = c->d_g2;
  a.bpart = bpart;
  a.n1 = c->n1;
  a.n2 = c->n2;
  a.copies = c->copies;
  a.t_begin = c->t_begin;
  a.nt = c->t_end - c->t_begin;
  a.Q = c->Q;
  a.nchunk = b_chunks(c);
  a.period = c->period;
  a.k2 = c->k2;
  a.x2x = c->x2[0];
  a.x2y = c->x2[1];
  if (a.nt <= 0) return PS_OK;
  static unsigned long long attr_mask = 0;
  if (S::SMEM > 48 * 1024 && first_on_device(&attr_mask, c->device)) {
    PS_CUDA_TRY(c, cudaFuncSetAttribute(b_kernel<P>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                        (int)S::SMEM));
  }
  b_kernel<P><<<dim3(a.nt, a.nchunk), kBT, S::SMEM, st>>>(a);
  PS_CUDA_TRY(c, cudaGetLastError());
  const int n = a.nt * S::L;
  sum_splits<<<(n + 255) / 256, 256, 0, st>>>(bpart, a.nchunk, n, out);
  PS_CUDA_TRY(c, cudaGetLastError());
  c->launches += 2;
  return PS_OK;
}

int dispatch_c(Ctx* c, const double2* beta, const double2* bpow, double2* gpart, double2* g,
               int s0, int s1, cudaStream_t st) {
  switch (c->p) {
#define PS_CASE(P) \
  case P:          \
    return launch_c<P>(c, beta, bpow, gpart, g, s0, s1, st);
    PS_M2L_ORDERS(PS_CASE)
#undef PS_CASE
    default:
      c->err = "apply_C: order not compiled";
      return PS_ERR_UNSUPPORTED;
  }
}

int dispatch_b(Ctx* c, const double2* x, const double2* bpow, double2* bpart, double2* out,
               cudaStream_t st) {
  switch (c->p) {
#define PS_CASE(P) \
  case P:          \
    return launch_b<P>(c, x, bpow, bpart, out, st);
    PS_M2L_ORDERS(PS_CASE)
#undef PS_CASE
    default:
      c->err = "apply_B: order not compiled";
      return PS_ERR_UNSUPPORTED;
  }
}

// workspace layout per RHS:
//   g [nrc] | h [nsv] | x [nout] | bsub [Mt*L] | u [Mt*L] | gpart [gpart_elems] | bpart [nchunk*Mt*L]
struct Work {
  double2 *g, *h, *x, *bsub, *u, *gpart, *bpart;
};

// gpart holds the split partial sums of C beta: at most 512 splits in the
// matrix-free K3 (c_splits) and at most 4*sm_count+1 ct_gemv blocks in the
// dense path (dense_apply_C); size for whichever is larger.
size_t gpart_elems(const Ctx* c) {
  return std::max((size_t)512 * c->nrow_c, dense_gpart_elems(c));
}

size_t work_stride(const Ctx* c) {
  const size_t nrc = c->nrow_c, nsv = c->nsv > 0 ? c->nsv : 1;
  const size_t nout = c->ncol_b + 2 * c->nrb + c->nfield;
  const size_t mtl = (size_t)(c->t_end - c->t_begin) * c->L;
  const size_t nch = c->have_layers ? (size_t)b_chunks(c) : 0;
  return nrc + nsv + nout + 2 * mtl + gpart_elems(c) + nch * mtl + 8;
}

int work(Ctx* c, int r, Work* w) {
  const size_t nrc = c->nrow_c, nsv = c->nsv > 0 ? c->nsv : 1;
  const size_t nout = c->ncol_b + 2 * c->nrb + c->nfield;
  const size_t mtl = (size_t)(c->t_end - c->t_begin) * c->L;
  const size_t per = work_stride(c);
  const size_t need = per * c->nrhs;
  if (c->work_elems < need) {
    if (c->d_work) ps::dev_free(c->d_work);
    c->d_work = nullptr;
    c->work_elems = 0;
    PS_CUDA_TRY(c, ps::dev_malloc(&c->d_work, need * sizeof(double2)));
    c->work_elems = need;
  }
  double2* b = c->d_work + per * r;
  w->g = b;
  w->h = w->g + nrc;
  w->x = w->h + nsv;
  w->bsub = w->x + nout;
  w->u = w->bsub + mtl;
  w->gpart = w->u + mtl;
  w->bpart = w->gpart + gpart_elems(c);
  return PS_OK;
}

int pinv(Ctx* c, int r, const double2* g, double2* x, int nout, cudaStream_t st) {
  const RhsData& R = c->rhs[r];
  Work w;
  if (int rc = work(c, r, &w)) return rc;
  // h = sinv * (U^* g) over the C rows, then x = cscale * (V h) over the read columns
  pinv_gemv<<<(c->nsv + kRows - 1) / kRows, kRowT * kRows, 0, st>>>(R.d_Uh, R.d_sinv, g, c->nsv,
                                                                      c->nrow_c, w.h);
  PS_CUDA_TRY(c, cudaGetLastError());
  pinv_gemv<<<(nout + kRows - 1) / kRows, kRowT * kRows, 0, st>>>(R.d_Vb, R.d_cscale, w.h, nout,
                                                                  c->nsv, x);
  PS_CUDA_TRY(c, cudaGetLastError());
  c->launches += 2;
  return PS_OK;
}

const double2* bpow_of(Ctx* c, int r) { return c->d_blochpow + (size_t)r * (2 * c->copies + 3); }

}  // namespace

int apply_C(Ctx* c, const double2* beta, double2* g, int s0, int s1, cudaStream_t st) {
  const size_t in_stride = (size_t)c->M * c->L;
  for (int r = 0; r < c->nrhs; ++r) {
    Work w;
    if (int rc = work(c, r, &w)) return rc;
    if (c->dense && s0 == c->dcs0 && s1 == c->dcs1) {
      if (int rc = dense_apply_C(c, r, beta + r * in_stride, w.gpart, g + (size_t)r * c->nrow_c, st))
        return rc;
      continue;
    }
    if (int rc = dispatch_c(c, beta + r * in_stride, bpow_of(c, r), w.gpart,
                            g + (size_t)r * c->nrow_c, s0, s1, st))
      return rc;
  }
  return PS_OK;
}

// B_phys A^+ g for RHS r into w.bsub
static int b_pinv(Ctx* c, int r, const double2* g, Work* w, cudaStream_t st) {
  if (int rc = pinv(c, r, g, w->x, c->ncol_b, st)) return rc;
  if (c->dense) return dense_apply_B(c, r, w->x, w->bsub, st);
  return dispatch_b(c, w->x, bpow_of(c, r), w->bpart, w->bsub, st);
}

static int s_apply(Ctx* c, const double2* v_own, const double2* u, double2* y, cudaStream_t st,
                   double sgn = -1.0) {
  // dense-S epilogue: y = v_own + sgn S u
  const int nt = c->t_end - c->t_begin;
  if (nt <= 0) return PS_OK;
  dense_s_epilogue<<<nt, 64, c->L * sizeof(double2), st>>>(c->d_S, c->d_rot, v_own, u,
                                                          c->t_begin, c->L, sgn, y);
  PS_CUDA_TRY(c, cudaGetLastError());
  c->launches += 1;
  return PS_OK;
}

// multi-RHS: coupling per RHS into the workspace slots, then ONE K1m launch
static int schur_mrhs(Ctx* c, const double2* v, double2* y, bool coupled, cudaStream_t st) {
  const size_t in_stride = (size_t)c->M * c->L;
  const size_t out_stride = (size_t)(c->t_end - c->t_begin) * c->L;
  Work w0;
  if (int rc = work(c, 0, &w0)) return rc;
  const long long bstride = (long long)work_stride(c);
  const int mode = c->s_diag ? 1 : 2;
  if (int rc = m2l_apply_mrhs(c, v, y, mode, coupled ? w0.bsub : nullptr, bstride, st)) return rc;
  if (!c->s_diag) {
    for (int r = 0; r < c->nrhs; ++r) {
      const double2* v_own = v + r * in_stride + (size_t)c->t_begin * c->L;
      if (int rc = s_apply(c, v_own, y + r * out_stride, y + r * out_stride, st)) return rc;
    }
  }
  return PS_OK;
}

int apply_schur_g(Ctx* c, const double2* v, const double2* g, double2* y, cudaStream_t st) {
  const size_t in_stride = (size_t)c->M * c->L;
  const size_t out_stride = (size_t)(c->t_end - c->t_begin) * c->L;
  const bool coupled = ps::factors_ready(c) && g;
  if (c->nrhs > 1) {
    if (coupled)
      for (int r = 0; r < c->nrhs; ++r) {
        Work w;
        if (int rc = work(c, r, &w)) return rc;
        if (int rc = b_pinv(c, r, g + (size_t)r * c->nrow_c, &w, st)) return rc;
      }
    return schur_mrhs(c, v, y, coupled, st);
  }
  for (int r = 0; r < c->nrhs; ++r) {
    Work w;
    if (int rc = work(c, r, &w)) return rc;
    const double2* bsub = nullptr;
    if (coupled) {
      if (int rc = b_pinv(c, r, g + (size_t)r * c->nrow_c, &w, st)) return rc;
      bsub = w.bsub;
    }
    const double2* vr = v + r * in_stride;
    const double2* v_own = vr + (size_t)c->t_begin * c->L;
    if (c->s_diag) {
      if (int rc = m2l_apply_1(c, vr, bpow_of(c, r) + 1, y + r * out_stride, 1, v_own, bsub, st))
        return rc;
    } else {
      if (int rc = m2l_apply_1(c, vr, bpow_of(c, r) + 1, w.u, 2, v_own, bsub, st)) return rc;
      if (int rc = s_apply(c, v_own, w.u, y + r * out_stride, st)) return rc;
    }
  }
  return PS_OK;
}

__global__ void finish_diag(const double2* __restrict__ v, const double2* __restrict__ a,
                            const double2* __restrict__ bsub, const double2* __restrict__ sd,
                            int n, int L, double2* __restrict__ y) {
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n) return;
  double2 u = a[i];
  if (bsub) {
    u.x -= bsub[i].x;
    u.y -= bsub[i].y;
  }
  const double2 s = sd[i % L], vv = v[i];
  y[i] = make_double2(vv.x - fma(s.x, u.x, -s.y * u.y), vv.y - fma(s.x, u.y, s.y * u.x));
}

__global__ void sub_rows(const double2* __restrict__ a, const double2* __restrict__ b, int n,
                         double2* __restrict__ u) {
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n) return;
  u[i] = b ? make_double2(a[i].x - b[i].x, a[i].y - b[i].y) : a[i];
}

// Epilogue of a Schur matvec whose M2L sums a_own arrived from elsewhere (the
// multi-GPU symmetric split: partial K1s over a block range on every rank,
// reduce-scattered): y = v_own - S (a_own - B A^+ g), one RHS.
int schur_finish(Ctx* c, const double2* v_own, const double2* a_own, const double2* g,
                 double2* y, cudaStream_t st) {
  const bool coupled = ps::factors_ready(c) && g;
  Work w;
  if (int rc = work(c, 0, &w)) return rc;
  const double2* bsub = nullptr;
  if (coupled) {
    if (int rc = b_pinv(c, 0, g, &w, st)) return rc;
    bsub = w.bsub;
  }
  const int n = (c->t_end - c->t_begin) * c->L;
  if (n <= 0) return PS_OK;
  if (c->s_diag) {
    finish_diag<<<(n + 255) / 256, 256, 0, st>>>(v_own, a_own, bsub, c->d_S, n, c->L, y);
    PS_CUDA_TRY(c, cudaGetLastError());
    c->launches += 1;
    return PS_OK;
  }
  sub_rows<<<(n + 255) / 256, 256, 0, st>>>(a_own, bsub, n, w.u);
  PS_CUDA_TRY(c, cudaGetLastError());
  c->launches += 1;
  return s_apply(c, v_own, w.u, y, st);
}

// One RHS, K1s, dense coupling blocks covering every source, diagonal S:
// K1s on sm_count - overlap_sms CTAs (high-priority stream) runs concurrently
// with the HBM-bound chain C -> A^+ -> B (low-priority stream, which gets
// the SMs K1s leaves free); the deterministic K1s reduce joins both.
// Queued at the fork (default), the 587-CTA C^T GEMV takes every SM for its
// ~0.1 ms at full HBM bandwidth before K1s' CTAs get in, and B streams on the
// free SMs during K1s.  overlap_k1_first queues the chain after K1s behind
// the Bloch weights, so K1s' high-priority CTAs are dispatched first and the
// whole chain streams on the free SMs -- measured slower at cfg3 (2.35 vs
// 2.31 ms): a few SMs pull only ~116 GB/s each with plain loads
// (tools/probe_timeline.py, tools/sm_stream_bw.cu).  TMA bulk copies reach
// ~216 GB/s per SM in isolation, but staged GEMVs built on them ran at
// 64-98 GB/s per SM (per-stage synchronisation), so the chain stays here.
struct ChainArgs {
  Ctx* c;
  const double2* v;
  Work* w;
  cudaEvent_t bw_done;
  cudaEvent_t chain_tl;   // profile timeline event (or null)
};

static int overlapped_chain(void* p) {
  ChainArgs* a = static_cast<ChainArgs*>(p);
  Ctx* c = a->c;
  if (a->bw_done) PS_CUDA_TRY(c, cudaStreamWaitEvent(c->s_lo, a->bw_done, 0));
  if (int rc = dense_apply_C(c, 0, a->v, a->w->gpart, a->w->g, c->s_lo)) return rc;
  if (int rc = b_pinv(c, 0, a->w->g, a->w, c->s_lo)) return rc;
  PS_CUDA_TRY(c, cudaEventRecord(c->ev_cpl, c->s_lo));
  if (a->chain_tl) PS_CUDA_TRY(c, cudaEventRecord(a->chain_tl, c->s_lo));
  return PS_OK;
}

static int schur_overlapped(Ctx* c, const double2* v, double2* y, cudaStream_t st) {
  if (!c->s_hi) {
    int lo = 0, hi = 0;
    PS_CUDA_TRY(c, cudaDeviceGetStreamPriorityRange(&lo, &hi));
    PS_CUDA_TRY(c, cudaStreamCreateWithPriority(&c->s_hi, cudaStreamNonBlocking, hi));
    PS_CUDA_TRY(c, cudaStreamCreateWithPriority(&c->s_lo, cudaStreamNonBlocking, lo));
    PS_CUDA_TRY(c, cudaEventCreateWithFlags(&c->ev_fork, cudaEventDisableTiming));
    PS_CUDA_TRY(c, cudaEventCreateWithFlags(&c->ev_k1, cudaEventDisableTiming));
    PS_CUDA_TRY(c, cudaEventCreateWithFlags(&c->ev_cpl, cudaEventDisableTiming));
    PS_CUDA_TRY(c, cudaEventCreateWithFlags(&c->ev_bw, cudaEventDisableTiming));
  }
  Work w;
  if (int rc = work(c, 0, &w)) return rc;
  PS_CUDA_TRY(c, cudaEventRecord(c->ev_fork, st));
  PS_CUDA_TRY(c, cudaStreamWaitEvent(c->s_hi, c->ev_fork, 0));
  PS_CUDA_TRY(c, cudaStreamWaitEvent(c->s_lo, c->ev_fork, 0));
  Ctx::Timeline tl{};
  if (c->profile) {
    for (cudaEvent_t* e : {&tl.fork, &tl.k1, &tl.chain, &tl.end})
      PS_CUDA_TRY(c, cudaEventCreate(e));
    PS_CUDA_TRY(c, cudaEventRecord(tl.fork, st));
    c->tl_k1 = tl.k1;
  }
  ChainArgs ca{c, v, &w, nullptr, c->profile ? tl.chain : nullptr};
  SymOverlap ov{c->s_hi, c->sm_count - c->overlap_sms, c->ev_k1, c->ev_cpl, c->ev_bw,
                nullptr, nullptr};
  if (c->overlap_k1_first) {
    ca.bw_done = c->ev_bw;
    ov.chain = overlapped_chain;
    ov.chain_arg = &ca;
  } else if (int rc = overlapped_chain(&ca)) {
    return rc;
  }
  const int rc = m2l_apply_sym(c, v, bpow_of(c, 0) + 1, y, 1, v, w.bsub, st, &ov);
  if (c->profile) {
    c->tl_k1 = nullptr;
    PS_CUDA_TRY(c, cudaEventRecord(tl.end, st));
    c->timelines.push_back(tl);
  }
  return rc;
}

int apply_schur(Ctx* c, const double2* v, double2* y, cudaStream_t st) {
  const bool coupled = ps::factors_ready(c);
  if (!coupled) return apply_schur_g(c, v, nullptr, y, st);
  if (c->overlap_sms >= 0 && c->overlap_sms < c->sm_count && c->nrhs == 1 && c->s_diag &&
      c->dense && c->dcs0 == 0 && c->dcs1 == c->M && m2l_sym_selected(c))
    return schur_overlapped(c, v, y, st);
  const size_t in_stride = (size_t)c->M * c->L;
  const size_t out_stride = (size_t)(c->t_end - c->t_begin) * c->L;
  const int nrhs = c->nrhs;
  for (int r = 0; r < nrhs; ++r) {
    Work w;
    if (int rc = work(c, r, &w)) return rc;
    if (c->dense && c->dcs0 == 0 && c->dcs1 == c->M) {
      if (int rc = dense_apply_C(c, r, v + r * in_stride, w.gpart, w.g, st)) return rc;
    } else if (int rc = dispatch_c(c, v + r * in_stride, bpow_of(c, r), w.gpart, w.g, 0, c->M,
                                   st)) {
      return rc;
    }
  }
  if (nrhs > 1) {
    for (int r = 0; r < nrhs; ++r) {
      Work w;
      if (int rc = work(c, r, &w)) return rc;
      if (int rc = b_pinv(c, r, w.g, &w, st)) return rc;
    }
    return schur_mrhs(c, v, y, true, st);
  }
  for (int r = 0; r < nrhs; ++r) {
    Work w;
    if (int rc = work(c, r, &w)) return rc;
    if (int rc = b_pinv(c, r, w.g, &w, st)) return rc;
    const double2* vr = v + r * in_stride;
    const double2* v_own = vr + (size_t)c->t_begin * c->L;
    if (c->s_diag) {
      if (int rc = m2l_apply_1(c, vr, bpow_of(c, r) + 1, y + r * out_stride, 1, v_own, w.bsub, st))
        return rc;
    } else {
      if (int rc = m2l_apply_1(c, vr, bpow_of(c, r) + 1, w.u, 2, v_own, w.bsub, st)) return rc;
      if (int rc = s_apply(c, v_own, w.u, y + r * out_stride, st)) return rc;
    }
  }
  return PS_OK;
}

__global__ void diag_s_apply(const double2* __restrict__ s, const double2* __restrict__ u, int n,
                             int L, double2* __restrict__ y) {
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i < n) y[i] = cmul(s[i % L], u[i]);
}

int schur_rhs(Ctx* c, double2* rhs, cudaStream_t st) {
  const int nt = c->t_end - c->t_begin;
  const size_t out_stride = (size_t)nt * c->L;
  for (int r = 0; r < c->nrhs; ++r) {
    Work w;
    if (int rc = work(c, r, &w)) return rc;
    if (int rc = b_pinv(c, r, c->rhs[r].d_f, &w, st)) return rc;
    const int n = nt * c->L;
    if (n == 0) continue;
    if (c->s_diag) {
      diag_s_apply<<<(n + 255) / 256, 256, 0, st>>>(c->d_S, w.bsub, n, c->L, rhs + r * out_stride);
      PS_CUDA_TRY(c, cudaGetLastError());
      c->launches += 1;
    } else {
      if (int rc = s_apply(c, nullptr, w.bsub, rhs + r * out_stride, st, 1.0)) return rc;
    }
  }
  return PS_OK;
}

// restricted output row o -> column of the empty-grating unknown vector
// (eg:154-156): B columns (mu1..a2) as is, then c, d, then the field rows a1, a3
__global__ void scatter_full(const double2* __restrict__ xr, int ncol_b, int nrb, int nj,
                             int nout, int nfield, double2* __restrict__ x) {
  const int o = blockIdx.x * blockDim.x + threadIdx.x;
  if (o >= nout + nfield) return;
  int col;
  if (o < ncol_b) col = o;
  else if (o < ncol_b + nrb) col = ncol_b + 2 * nj + (o - ncol_b);                // c
  else if (o < nout) col = ncol_b + 2 * nj + nrb + (o - ncol_b - nrb);             // d
  else col = ncol_b + (o - nout);                                                  // a1, a3
  x[col] = xr[o];
}

int recover_full(Ctx* c, const double2* g, double2* x, cudaStream_t st) {
  const int nout = c->ncol_b + 2 * c->nrb;
  const int nj = 2 * c->Q + 1;
  if (c->nfield != 2 * nj) {
    c->err = "recover_full: factors without the a1 / a3 field rows";
    return PS_ERR_STATE;
  }
  const int ncol = nout + c->nfield;
  for (int r = 0; r < c->nrhs; ++r) {
    Work w;
    if (int rc = work(c, r, &w)) return rc;
    f_minus<<<(c->nrow_c + 255) / 256, 256, 0, st>>>(c->rhs[r].d_f, g + (size_t)r * c->nrow_c,
                                                     c->nrow_c, w.g);
    PS_CUDA_TRY(c, cudaGetLastError());
    if (int rc = pinv(c, r, w.g, w.x, ncol, st)) return rc;
    scatter_full<<<(ncol + 255) / 256, 256, 0, st>>>(w.x, c->ncol_b, c->nrb, nj, nout, c->nfield,
                                                      x + (size_t)r * ncol);
    PS_CUDA_TRY(c, cudaGetLastError());
    c->launches += 2;
  }
  return PS_OK;
}

int recover(Ctx* c, const double2* g, double2* x, cudaStream_t st) {
  const int nout = c->ncol_b + 2 * c->nrb;
  for (int r = 0; r < c->nrhs; ++r) {
    Work w;
    if (int rc = work(c, r, &w)) return rc;
    f_minus<<<(c->nrow_c + 255) / 256, 256, 0, st>>>(c->rhs[r].d_f, g + (size_t)r * c->nrow_c,
                                                     c->nrow_c, w.g);
    PS_CUDA_TRY(c, cudaGetLastError());
    c->launches += 1;
    if (int rc = pinv(c, r, w.g, x + (size_t)r * nout, nout, st)) return rc;
  }
  return PS_OK;
}

}  // namespace ps
