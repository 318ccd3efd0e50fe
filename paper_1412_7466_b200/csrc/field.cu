// Particle field at arbitrary points (M2P): the inclusions' phased multipole
// sums of the layer-2 representation (Eq. repre3_mod;
// SPEC.md:619-627 eval_total_field_grid "particle phased multipole sums"):
//
//   u_r(x) = sum_{l=-P..P} bloch_r^l sum_j sum_{n=-p..p} beta_r,j[n] H_n(k2 rho) e^{i n phi},
//   (rho, phi) = polar(x - x_j - l d e_x).
//
// One lane per point, one warp per 32 points; the warps of a CTA and the
// CTAs along grid.y split the source images, and a second kernel sums the
// splits in a fixed order (deterministic).  Per (point, source image) the
// lane builds t_n = H_n e^{i n phi} with the same symbol code as the M2L
// (symbols.cuh: warp-uniform Miller start) and folds it into RC right-hand
// sides at once (the symbols do not depend on the RHS).
#include <cuda_runtime.h>

#include <string>

#include "ctx.cuh"
#include "field.cuh"
#include "m2l.cuh"
#include "symbols.cuh"

namespace ps {

namespace {

constexpr int kWarps = 4;

template <int P, int RC>
__global__ void __launch_bounds__(kWarps * 32) particle_field_kernel(
    const double* __restrict__ centers, const double2* __restrict__ beta,
    const double2* __restrict__ bpow, int np_stride, const double* __restrict__ pts, int npts,
    int M, int copies, double period, double k2, int r0, int nrhs, int nsplit,
    double2* __restrict__ part) {
  constexpr int L = 2 * P + 1;
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int pt = blockIdx.x * 32 + lane;
  const bool live_pt = pt < npts;
  const double px = live_pt ? pts[2 * pt] : 0.0, py = live_pt ? pts[2 * pt + 1] : 0.0;
  const int ncp = 2 * copies + 1;
  const long long nimg = (long long)M * ncp;
  const int split = blockIdx.y * kWarps + warp, nspl = nsplit * kWarps;
  const long long g0 = nimg * split / nspl, g1 = nimg * (split + 1) / nspl;
  double2 acc[RC];
#pragma unroll
  for (int r = 0; r < RC; ++r) acc[r] = make_double2(0.0, 0.0);
  for (long long g = g0; g < g1; ++g) {
    const int j = (int)(g / ncp), li = (int)(g % ncp);
    const int l = li - copies;
    const double2 cj = reinterpret_cast<const double2*>(centers)[j];
    const double dx = px - cj.x - (double)l * period, dy = py - cj.y;
    const double rho = hypot(dx, dy);
    // points on a centre (masked interiors) contribute nothing
    const bool live = live_pt && rho > 0.0;
    const double rr = live ? rho : 1.0;
    const double z = k2 * rr;
    int N = live ? miller_start_j01(z) : 2;
    N = __reduce_max_sync(0xffffffffu, N);
    const double inv = live ? 1.0 / rr : 0.0;
    double2 w[RC];                       // bloch_r^l beta_r,j
    const double2* bj = beta + (size_t)j * L;
#pragma unroll
    for (int r = 0; r < RC; ++r) {
      const double2 b = bpow[(size_t)min(r0 + r, nrhs - 1) * np_stride + 1 + li];
      w[r] = b;
    }
    hankel_symbols<P>(z, dx * inv, dy * inv, N, [&](int nu, double re, double im) {
      if (nu < -P || nu > P) return;
      if (!live) return;
#pragma unroll
      for (int r = 0; r < RC; ++r) {
        if (r0 + r >= nrhs) break;
        const double2 bv = __ldg(bj + (size_t)(r0 + r) * M * L + (nu + P));
        // (bloch^l beta) t
        const double br = fma(w[r].x, bv.x, -w[r].y * bv.y), bi = fma(w[r].x, bv.y, w[r].y * bv.x);
        acc[r].x = fma(br, re, fma(-bi, im, acc[r].x));
        acc[r].y = fma(br, im, fma(bi, re, acc[r].y));
      }
    });
  }
  if (!live_pt) return;
#pragma unroll
  for (int r = 0; r < RC; ++r)
    if (r0 + r < nrhs) part[((size_t)split * nrhs + r0 + r) * npts + pt] = acc[r];
}

__global__ void sum_splits_field(const double2* __restrict__ part, int nspl, int nrhs, int npts,
                                 double2* __restrict__ out) {
  const long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= (long long)nrhs * npts) return;
  double2 s = make_double2(0.0, 0.0);
  for (int k = 0; k < nspl; ++k) {
    const double2 v = part[(size_t)k * nrhs * npts + i];
    s.x += v.x;
    s.y += v.y;
  }
  out[i] = s;
}

template <int P, int RC>
int launch_f(Ctx* c, const double2* beta, const double* pts, int npts, double2* out,
             cudaStream_t st) {
  const int bx = (npts + 31) / 32;
  // fill about two waves of 4-warp CTAs with source splits
  int ny = (2 * c->sm_count * 4 + bx - 1) / bx;
  const long long nimg = (long long)c->M * (2 * c->copies + 1);
  if (ny > nimg / kWarps) ny = (int)(nimg / kWarps);
  if (ny < 1) ny = 1;
  const int nspl = ny * kWarps;
  const size_t need = (size_t)nspl * c->nrhs * npts;
  double2* part = nullptr;
  PS_CUDA_TRY(c, ps::dev_malloc(&part, need * sizeof(double2)));
  const int np_stride = 2 * c->copies + 3;
  for (int r0 = 0; r0 < c->nrhs; r0 += RC) {
    particle_field_kernel<P, RC><<<dim3(bx, ny), kWarps * 32, 0, st>>>(
        c->d_centers, beta, c->d_blochpow, np_stride, pts, npts, c->M, c->copies, c->period,
        c->k2, r0, c->nrhs, ny, part);
    PS_CUDA_TRY(c, cudaGetLastError());
    c->launches += 1;
  }
  const long long n = (long long)c->nrhs * npts;
  sum_splits_field<<<(unsigned)((n + 255) / 256), 256, 0, st>>>(part, nspl, c->nrhs, npts, out);
  PS_CUDA_TRY(c, cudaGetLastError());
  c->launches += 1;
  PS_CUDA_TRY(c, cudaStreamSynchronize(st));
  ps::dev_free(part);
  return PS_OK;
}

template <int P>
int launch_rc(Ctx* c, const double2* beta, const double* pts, int npts, double2* out,
              cudaStream_t st) {
  if (c->nrhs >= 4) return launch_f<P, 4>(c, beta, pts, npts, out, st);
  if (c->nrhs >= 2) return launch_f<P, 2>(c, beta, pts, npts, out, st);
  return launch_f<P, 1>(c, beta, pts, npts, out, st);
}

}  // namespace

int particle_field(Ctx* c, const double2* beta, const double* pts, int npts, double2* out,
                   cudaStream_t st) {
  if (npts <= 0) return PS_OK;
  switch (c->p) {
#define PS_CASE(P) \
  case P:          \
    return launch_rc<P>(c, beta, pts, npts, out, st);
    PS_M2L_ORDERS(PS_CASE)
#undef PS_CASE
    default:
      c->err = "particle_field: multipole order p=" + std::to_string(c->p) + " not compiled";
      return PS_ERR_UNSUPPORTED;
  }
}


// ---------------------------------------------------------------------------
// Empty-grating layer fields at points (empty_grating.eval_empty_field,
// empty_grating.py:352-393, total=True): per point, the representation of the
// layer it lies in -- the phased single + double layers of the bounding
// interfaces (phased_layer_field, eg:319-338, smooth quadrature as
// layerpot.eval_layer_potentials, lp:240-263), the layer's regular expansion
// (specialfn.regular_wave_block, sf:86-125) and, in layer 1, the incident
// wave (incident_field, eg:32-42) -- from the full unknown vector
// x = A^+ (f - C beta) (ps_recover_full).  Thread per (point, RHS).
namespace {

__device__ __forceinline__ double2 fcmul(double2 a, double2 b) {
  return make_double2(a.x * b.x - a.y * b.y, a.x * b.y + a.y * b.x);
}

struct LayerArgs {
  const double2* x;        // [nrhs][ncol]
  const double* pts;       // [npts][2]
  const int* layer;        // [npts]: 1, 2, 3 (anything else -> 0)
  const double* g1;        // [n1][5] x y nx ny aw
  const double* g2;        // [n2][5]
  const double2* bpow;     // [nrhs][2P+3]
  const double* inc;       // [nrhs][2]
  double2* out;            // [nrhs][npts]
  int npts, ncol, n1, n2, Q, copies, np;
  int c_mu1, c_s1, c_mu2, c_s2, c_a2, c_a1, c_a3;
  double k1, k2, k3, period;
  double c1x, c1y, c2x, c2y, c3x, c3y;
};

// sum_l alpha^l sum_j aw_j [S_k(x, y_j + l d) sigma_j + D_k(x, y_j + l d) mu_j]
__device__ double2 layer_potential(const LayerArgs& a, const double* cv, int n, const double2* mu,
                                   const double2* sg, double k, const double2* bp, double px,
                                   double py) {
  double2 tot = make_double2(0.0, 0.0);
  for (int l = -a.copies; l <= a.copies; ++l) {
    double2 acc = make_double2(0.0, 0.0);
    for (int j = 0; j < n; ++j) {
      const double* y = cv + (size_t)j * 5;
      const double u0 = px - (y[0] + l * a.period), u1 = py - y[1];
      const double r = hypot(u0, u1);
      double j0, j1, y0, y1;
      bessel_jy01(k * r, miller_start_j01(k * r), &j0, &j1, &y0, &y1);
      const double udn = (u0 * y[2] + u1 * y[3]) / r;
      // S = (i/4) H0, D = (i/4) k H1 (u . n_y) / r  (layerpot.py:69-91)
      const double2 sv = make_double2(-0.25 * y0, 0.25 * j0);
      const double2 dv = make_double2(-0.25 * k * udn * y1, 0.25 * k * udn * j1);
      const double2 s = sg[j], m = mu[j];
      const double aw = y[4];
      acc.x += aw * (sv.x * s.x - sv.y * s.y + dv.x * m.x - dv.y * m.y);
      acc.y += aw * (sv.x * s.y + sv.y * s.x + dv.x * m.y + dv.y * m.x);
    }
    const double2 w = bp[l + a.copies + 1];
    const double2 t = fcmul(w, acc);
    tot.x += t.x;
    tot.y += t.y;
  }
  return tot;
}

// sum_{n=-Q}^{Q} a_n J_n(k r) e^{i n theta} about (cx, cy)
__device__ double2 regular_sum(const double2* an, int Q, double k, double cx, double cy, double px,
                               double py) {
  const double dx = px - cx, dy = py - cy;
  const double r = hypot(dx, dy);
  if (r == 0.0) return an[Q];
  double J[80];
  double inv, y0, y1;
  bessel_jy_sweep(k * r, Q, [&](int nu, double v) { J[nu] = v; }, &inv, &y0, &y1);
  const double c = dx / r, s = dy / r;
  double2 acc = make_double2(an[Q].x * J[0] * inv, an[Q].y * J[0] * inv);
  double pr = 1.0, pi = 0.0;   // e^{i n theta}
  for (int n = 1; n <= Q; ++n) {
    const double qr = pr * c - pi * s, qi = pr * s + pi * c;
    pr = qr;
    pi = qi;
    const double jn = J[n] * inv;
    const double jm = (n & 1) ? -jn : jn;               // J_{-n} = (-1)^n J_n
    const double2 ap = an[Q + n], am = an[Q - n];
    // a_n J_n e^{in th} + a_{-n} J_{-n} e^{-in th}
    acc.x += jn * (ap.x * pr - ap.y * pi) + jm * (am.x * pr + am.y * pi);
    acc.y += jn * (ap.x * pi + ap.y * pr) + jm * (am.y * pr - am.x * pi);
  }
  return acc;
}

__global__ void __launch_bounds__(128) layer_field_kernel(LayerArgs a) {
  const int pt = blockIdx.x * blockDim.x + threadIdx.x;
  const int r = blockIdx.y;
  if (pt >= a.npts) return;
  const int ly = a.layer[pt];
  double2 u = make_double2(0.0, 0.0);
  const double px = a.pts[2 * pt], py = a.pts[2 * pt + 1];
  const double2* x = a.x + (size_t)r * a.ncol;
  const double2* bp = a.bpow + (size_t)r * a.np;
  if (ly == 1) {
    u = layer_potential(a, a.g1, a.n1, x + a.c_mu1, x + a.c_s1, a.k1, bp, px, py);
    const double2 e = regular_sum(x + a.c_a1, a.Q, a.k1, a.c1x, a.c1y, px, py);
    double sn, cs;
    sincos(px * a.inc[2 * r] + py * a.inc[2 * r + 1], &sn, &cs);
    u = make_double2(u.x + e.x + cs, u.y + e.y + sn);
  } else if (ly == 2) {
    const double2 u1 = layer_potential(a, a.g1, a.n1, x + a.c_mu1, x + a.c_s1, a.k2, bp, px, py);
    const double2 u2 = layer_potential(a, a.g2, a.n2, x + a.c_mu2, x + a.c_s2, a.k2, bp, px, py);
    const double2 e = regular_sum(x + a.c_a2, a.Q, a.k2, a.c2x, a.c2y, px, py);
    u = make_double2(u1.x + u2.x + e.x, u1.y + u2.y + e.y);
  } else if (ly == 3) {
    u = layer_potential(a, a.g2, a.n2, x + a.c_mu2, x + a.c_s2, a.k3, bp, px, py);
    const double2 e = regular_sum(x + a.c_a3, a.Q, a.k3, a.c3x, a.c3y, px, py);
    u = make_double2(u.x + e.x, u.y + e.y);
  }
  a.out[(size_t)r * a.npts + pt] = u;
}

}  // namespace

int layer_field(Ctx* c, const double2* x, const double* pts, const int* layer, int npts,
                double2* out, cudaStream_t st) {
  if (!c->have_layers || !c->have_field || c->nfield == 0) {
    c->err = "ps_layer_field: no empty-grating setup with field data (ps_setup_empty, or "
             "ps_set_pinv + ps_set_field_params)";
    return PS_ERR_STATE;
  }
  if (c->Q + 1 > 79) {
    c->err = "ps_layer_field: j_expansion_order > 78 unsupported";
    return PS_ERR_UNSUPPORTED;
  }
  if (npts == 0) return PS_OK;
  const int nj = 2 * c->Q + 1;
  LayerArgs a;
  a.x = x;
  a.pts = pts;
  a.layer = layer;
  a.g1 = c->d_g1;
  a.g2 = c->d_g2;
  a.bpow = c->d_blochpow;
  a.inc = c->d_inc;
  a.out = out;
  a.npts = npts;
  a.ncol = c->ncol_b + 2 * nj + 2 * c->nrb;
  a.n1 = c->n1;
  a.n2 = c->n2;
  a.Q = c->Q;
  a.copies = c->copies;
  a.np = 2 * c->copies + 3;
  a.c_mu1 = 0;
  a.c_s1 = c->n1;
  a.c_mu2 = 2 * c->n1;
  a.c_s2 = 2 * c->n1 + c->n2;
  a.c_a2 = 2 * c->n1 + 2 * c->n2;
  a.c_a1 = a.c_a2 + nj;
  a.c_a3 = a.c_a1 + nj;
  a.k1 = c->f_k1;
  a.k2 = c->k2;
  a.k3 = c->f_k3;
  a.period = c->period;
  a.c1x = c->f_c1[0];
  a.c1y = c->f_c1[1];
  a.c2x = c->x2[0];
  a.c2y = c->x2[1];
  a.c3x = c->f_c3[0];
  a.c3y = c->f_c3[1];
  layer_field_kernel<<<dim3((npts + 127) / 128, c->nrhs), 128, 0, st>>>(a);
  PS_CUDA_TRY(c, cudaGetLastError());
  c->launches += 1;
  return PS_OK;
}

}  // namespace ps
