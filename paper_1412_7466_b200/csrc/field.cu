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

// GRAD: also the derivative along the unit vector nrm[pt] of the point,
//   d_n (H_n e^{i n phi}) = (k/2) [(nx + i ny) t_{n-1} - (nx - i ny) t_{n+1}]
// ((d_x +- i d_y) identities of the outgoing waves, sf:128-154 restated), so
// per point A = sum_n beta_n t_{n-1} and B = sum_n beta_n t_{n+1} are
// accumulated over the source images and combined once at the end.
template <int P, int RC, bool GRAD>
__global__ void __launch_bounds__(kWarps * 32) particle_field_kernel(
    const double* __restrict__ centers, const double2* __restrict__ beta,
    const double2* __restrict__ bpow, int np_stride, const double* __restrict__ pts,
    const double* __restrict__ nrm, int npts, int M, int copies, double period, double k2,
    int r0, int nrhs, int nsplit, double2* __restrict__ part, double2* __restrict__ part_dn) {
  constexpr int L = 2 * P + 1;
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int pt = blockIdx.x * 32 + lane;
  const bool live_pt = pt < npts;
  const double px = live_pt ? pts[2 * pt] : 0.0, py = live_pt ? pts[2 * pt + 1] : 0.0;
  const int ncp = 2 * copies + 1;
  const long long nimg = (long long)M * ncp;
  const int split = blockIdx.y * kWarps + warp, nspl = nsplit * kWarps;
  const long long g0 = nimg * split / nspl, g1 = nimg * (split + 1) / nspl;
  double2 acc[RC], accA[GRAD ? RC : 1], accB[GRAD ? RC : 1];
#pragma unroll
  for (int r = 0; r < RC; ++r) acc[r] = make_double2(0.0, 0.0);
#pragma unroll
  for (int r = 0; r < (GRAD ? RC : 1); ++r) accA[r] = accB[r] = make_double2(0.0, 0.0);
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
    // (bloch^l beta_r[n]) t into a
    auto fold = [&](int r, int n, double re, double im, double2& a) {
      const double2 bv = __ldg(bj + (size_t)(r0 + r) * M * L + (n + P));
      const double br = fma(w[r].x, bv.x, -w[r].y * bv.y), bi = fma(w[r].x, bv.y, w[r].y * bv.x);
      a.x = fma(br, re, fma(-bi, im, a.x));
      a.y = fma(br, im, fma(bi, re, a.y));
    };
    hankel_symbols<GRAD ? P + 1 : P>(z, dx * inv, dy * inv, N, [&](int nu, double re, double im) {
      if (!live) return;
#pragma unroll
      for (int r = 0; r < RC; ++r) {
        if (r0 + r >= nrhs) break;
        if (nu >= -P && nu <= P) fold(r, nu, re, im, acc[r]);
        if (GRAD) {
          if (nu + 1 >= -P && nu + 1 <= P) fold(r, nu + 1, re, im, accA[GRAD ? r : 0]);  // t_{n-1}
          if (nu - 1 >= -P && nu - 1 <= P) fold(r, nu - 1, re, im, accB[GRAD ? r : 0]);  // t_{n+1}
        }
      }
    });
  }
  if (!live_pt) return;
#pragma unroll
  for (int r = 0; r < RC; ++r)
    if (r0 + r < nrhs) part[((size_t)split * nrhs + r0 + r) * npts + pt] = acc[r];
  if (GRAD) {
    const double nx = nrm[2 * pt], ny = nrm[2 * pt + 1], hk = 0.5 * k2;
#pragma unroll
    for (int r = 0; r < RC; ++r) {
      if (r0 + r >= nrhs) break;
      const double2 A = accA[GRAD ? r : 0], B = accB[GRAD ? r : 0];
      // (k/2) [(nx + i ny) A - (nx - i ny) B]
      const double2 d = make_double2(hk * (nx * (A.x - B.x) - ny * (A.y + B.y)),
                                     hk * (nx * (A.y - B.y) + ny * (A.x + B.x)));
      part_dn[((size_t)split * nrhs + r0 + r) * npts + pt] = d;
    }
  }
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

template <int P, int RC, bool GRAD>
int launch_f(Ctx* c, const double2* beta, const double* pts, const double* nrm, int npts,
             double2* out, double2* out_dn, cudaStream_t st) {
  const int bx = (npts + 31) / 32;
  // fill about two waves of 4-warp CTAs with source splits
  int ny = (2 * c->sm_count * 4 + bx - 1) / bx;
  const long long nimg = (long long)c->M * (2 * c->copies + 1);
  if (ny > nimg / kWarps) ny = (int)(nimg / kWarps);
  if (ny < 1) ny = 1;
  const int nspl = ny * kWarps;
  const size_t need = (size_t)nspl * c->nrhs * npts;
  double2* part = nullptr;
  PS_CUDA_TRY(c, ps::dev_malloc(&part, (GRAD ? 2 : 1) * need * sizeof(double2)));
  double2* part_dn = GRAD ? part + need : nullptr;
  const int np_stride = 2 * c->copies + 3;
  for (int r0 = 0; r0 < c->nrhs; r0 += RC) {
    particle_field_kernel<P, RC, GRAD><<<dim3(bx, ny), kWarps * 32, 0, st>>>(
        c->d_centers, beta, c->d_blochpow, np_stride, pts, nrm, npts, c->M, c->copies, c->period,
        c->k2, r0, c->nrhs, ny, part, part_dn);
    PS_CUDA_TRY(c, cudaGetLastError());
    c->launches += 1;
  }
  const long long n = (long long)c->nrhs * npts;
  sum_splits_field<<<(unsigned)((n + 255) / 256), 256, 0, st>>>(part, nspl, c->nrhs, npts, out);
  PS_CUDA_TRY(c, cudaGetLastError());
  c->launches += 1;
  if (GRAD) {
    sum_splits_field<<<(unsigned)((n + 255) / 256), 256, 0, st>>>(part_dn, nspl, c->nrhs, npts,
                                                                  out_dn);
    PS_CUDA_TRY(c, cudaGetLastError());
    c->launches += 1;
  }
  PS_CUDA_TRY(c, cudaStreamSynchronize(st));
  ps::dev_free(part);
  return PS_OK;
}

template <int P, bool GRAD>
int launch_rc(Ctx* c, const double2* beta, const double* pts, const double* nrm, int npts,
              double2* out, double2* out_dn, cudaStream_t st) {
  if (c->nrhs >= 4) return launch_f<P, 4, GRAD>(c, beta, pts, nrm, npts, out, out_dn, st);
  if (c->nrhs >= 2) return launch_f<P, 2, GRAD>(c, beta, pts, nrm, npts, out, out_dn, st);
  return launch_f<P, 1, GRAD>(c, beta, pts, nrm, npts, out, out_dn, st);
}

}  // namespace

int particle_field(Ctx* c, const double2* beta, const double* pts, const double* nrm, int npts,
                   double2* out, double2* out_dn, cudaStream_t st) {
  if (npts <= 0) return PS_OK;
  const bool grad = nrm && out_dn;
  switch (c->p) {
#define PS_CASE(P)                                                              \
  case P:                                                                       \
    return grad ? launch_rc<P, true>(c, beta, pts, nrm, npts, out, out_dn, st) \
                : launch_rc<P, false>(c, beta, pts, nullptr, npts, out, nullptr, st);
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
  const double* nrm;       // [npts][2] derivative directions (GRAD)
  const double* g1;        // [n1][5] x y nx ny aw
  const double* g2;        // [n2][5]
  const double2* bpow;     // [nrhs][2P+3]
  const double* inc;       // [nrhs][2]
  double2* out;            // [nrhs][npts]
  double2* out_dn;         // [nrhs][npts] (GRAD)
  int npts, ncol, n1, n2, Q, copies, np, incident;
  int c_mu1, c_s1, c_mu2, c_s2, c_a2, c_a1, c_a3;
  double k1, k2, k3, period;
  double c1x, c1y, c2x, c2y, c3x, c3y;
};

// sum_l alpha^l sum_j aw_j [S_k(x, y_j + l d) sigma_j + D_k(x, y_j + l d) mu_j]
// and (GRAD) its derivative along e at x (layerpot.py:67-91: the N / T
// kernels of the single / double layer with the target normal e):
//   d_e S = -(i/4) k H1 (u.e)/r,
//   d_e D = (i/4) k [k H0 P - 2 H1 P / r + H1 (e.n_y) / r],  P = (u.e)(u.n_y)/r^2
template <bool GRAD>
__device__ void layer_potential(const LayerArgs& a, const double* cv, int n, const double2* mu,
                                const double2* sg, double k, const double2* bp, double px,
                                double py, double ex, double ey, double2* val, double2* dn) {
  double2 tot = make_double2(0.0, 0.0), totd = make_double2(0.0, 0.0);
  for (int l = -a.copies; l <= a.copies; ++l) {
    double2 acc = make_double2(0.0, 0.0), accd = make_double2(0.0, 0.0);
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
      if (GRAD) {
        const double ude = (u0 * ex + u1 * ey) / r;          // (u.e)/r
        const double en = ex * y[2] + ey * y[3];
        const double pp = ude * udn;
        // N: -(i/4) k H1 (u.e)/r
        const double2 nv = make_double2(0.25 * k * ude * y1, -0.25 * k * ude * j1);
        // T: (i/4) k [k H0 P + H1 (e.n - 2P) / r]
        const double cr = k * pp, ch = (en - 2.0 * pp) / r;
        const double hr = cr * j0 + ch * j1, hi = cr * y0 + ch * y1;   // k H0 P + H1 (..)/r
        const double2 tv = make_double2(-0.25 * k * hi, 0.25 * k * hr);
        accd.x += aw * (nv.x * s.x - nv.y * s.y + tv.x * m.x - tv.y * m.y);
        accd.y += aw * (nv.x * s.y + nv.y * s.x + tv.x * m.y + tv.y * m.x);
      }
    }
    const double2 w = bp[l + a.copies + 1];
    const double2 t = fcmul(w, acc);
    tot.x += t.x;
    tot.y += t.y;
    if (GRAD) {
      const double2 td = fcmul(w, accd);
      totd.x += td.x;
      totd.y += td.y;
    }
  }
  val->x += tot.x;
  val->y += tot.y;
  if (GRAD) {
    dn->x += totd.x;
    dn->y += totd.y;
  }
}

// sum_{n=-Q}^{Q} a_n W_n, W_n = J_n(k r) e^{i n theta} about (cx, cy), and
// (GRAD) d_e of it: d_e W_n = (k/2) [(ex + i ey) W_{n-1} - (ex - i ey) W_{n+1}]
// (the regular_wave_block gradients, sf:86-125, restated)
template <bool GRAD>
__device__ void regular_sum(const double2* an, int Q, double k, double cx, double cy, double px,
                            double py, double ex, double ey, double2* val, double2* dn) {
  const double dx = px - cx, dy = py - cy;
  const double r = hypot(dx, dy);
  double J[81];
  double inv = 1.0, y0, y1;
  const int nmax = GRAD ? Q + 1 : Q;
  if (r == 0.0) {
    J[0] = 1.0;
    for (int n = 1; n <= nmax; ++n) J[n] = 0.0;
  } else {
    bessel_jy_sweep(k * r, nmax, [&](int nu, double v) { J[nu] = v; }, &inv, &y0, &y1);
  }
  const double c = r > 0.0 ? dx / r : 1.0, s = r > 0.0 ? dy / r : 0.0;
  // W_n and W_{-n} for n = 0..nmax, folded on the fly
  double2 acc = make_double2(an[Q].x * J[0] * inv, an[Q].y * J[0] * inv);
  double2 A = make_double2(0.0, 0.0), B = make_double2(0.0, 0.0);  // sum a_n W_{n-1}, sum a_n W_{n+1}
  auto coef = [&](int n) { return (n >= -Q && n <= Q) ? an[Q + n] : make_double2(0.0, 0.0); };
  auto add = [&](double2& t, double2 a, double wr, double wi) {
    t.x += a.x * wr - a.y * wi;
    t.y += a.x * wi + a.y * wr;
  };
  if (GRAD) {
    const double w0 = J[0] * inv;
    add(A, coef(1), w0, 0.0);     // n = 1: W_0
    add(B, coef(-1), w0, 0.0);    // n = -1: W_0
  }
  double pr = 1.0, pi = 0.0;   // e^{i n theta}
  for (int n = 1; n <= nmax; ++n) {
    const double qr = pr * c - pi * s, qi = pr * s + pi * c;
    pr = qr;
    pi = qi;
    const double jn = J[n] * inv;
    const double jm = (n & 1) ? -jn : jn;               // J_{-n} = (-1)^n J_n
    const double wpr = jn * pr, wpi = jn * pi;          // W_n
    const double wmr = jm * pr, wmi = -jm * pi;         // W_{-n}
    if (n <= Q) {
      add(acc, an[Q + n], wpr, wpi);
      add(acc, an[Q - n], wmr, wmi);
    }
    if (GRAD) {
      add(A, coef(n + 1), wpr, wpi);       // a_{n+1} W_n
      add(A, coef(-n + 1), wmr, wmi);      // a_{1-n} W_{-n}
      add(B, coef(n - 1), wpr, wpi);       // a_{n-1} W_n
      add(B, coef(-n - 1), wmr, wmi);      // a_{-n-1} W_{-n}
    }
  }
  val->x += acc.x;
  val->y += acc.y;
  if (GRAD) {
    const double hk = 0.5 * k;
    dn->x += hk * (ex * (A.x - B.x) - ey * (A.y + B.y));
    dn->y += hk * (ex * (A.y - B.y) + ey * (A.x + B.x));
  }
}

template <bool GRAD>
__global__ void __launch_bounds__(128) layer_field_kernel(LayerArgs a) {
  const int pt = blockIdx.x * blockDim.x + threadIdx.x;
  const int r = blockIdx.y;
  if (pt >= a.npts) return;
  const int ly = a.layer[pt];
  double2 u = make_double2(0.0, 0.0), ud = make_double2(0.0, 0.0);
  const double px = a.pts[2 * pt], py = a.pts[2 * pt + 1];
  const double ex = GRAD ? a.nrm[2 * pt] : 0.0, ey = GRAD ? a.nrm[2 * pt + 1] : 0.0;
  const double2* x = a.x + (size_t)r * a.ncol;
  const double2* bp = a.bpow + (size_t)r * a.np;
  if (ly == 1) {
    layer_potential<GRAD>(a, a.g1, a.n1, x + a.c_mu1, x + a.c_s1, a.k1, bp, px, py, ex, ey, &u, &ud);
    regular_sum<GRAD>(x + a.c_a1, a.Q, a.k1, a.c1x, a.c1y, px, py, ex, ey, &u, &ud);
    if (a.incident) {
      const double kx = a.inc[2 * r], ky = a.inc[2 * r + 1];
      double sn, cs;
      sincos(px * kx + py * ky, &sn, &cs);
      u.x += cs;
      u.y += sn;
      if (GRAD) {                       // i (k . e) e^{i k.x}
        const double ke = kx * ex + ky * ey;
        ud.x -= ke * sn;
        ud.y += ke * cs;
      }
    }
  } else if (ly == 2) {
    layer_potential<GRAD>(a, a.g1, a.n1, x + a.c_mu1, x + a.c_s1, a.k2, bp, px, py, ex, ey, &u, &ud);
    layer_potential<GRAD>(a, a.g2, a.n2, x + a.c_mu2, x + a.c_s2, a.k2, bp, px, py, ex, ey, &u, &ud);
    regular_sum<GRAD>(x + a.c_a2, a.Q, a.k2, a.c2x, a.c2y, px, py, ex, ey, &u, &ud);
  } else if (ly == 3) {
    layer_potential<GRAD>(a, a.g2, a.n2, x + a.c_mu2, x + a.c_s2, a.k3, bp, px, py, ex, ey, &u, &ud);
    regular_sum<GRAD>(x + a.c_a3, a.Q, a.k3, a.c3x, a.c3y, px, py, ex, ey, &u, &ud);
  }
  a.out[(size_t)r * a.npts + pt] = u;
  if (GRAD) a.out_dn[(size_t)r * a.npts + pt] = ud;
}

}  // namespace

int layer_field(Ctx* c, const double2* x, const double* pts, const int* layer,
                const double* nrm, int npts, int incident, double2* out, double2* out_dn,
                cudaStream_t st) {
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
  a.nrm = nrm;
  a.out_dn = out_dn;
  a.incident = incident;
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
  if (nrm && out_dn)
    layer_field_kernel<true><<<dim3((npts + 127) / 128, c->nrhs), 128, 0, st>>>(a);
  else
    layer_field_kernel<false><<<dim3((npts + 127) / 128, c->nrhs), 128, 0, st>>>(a);
  PS_CUDA_TRY(c, cudaGetLastError());
  c->launches += 1;
  return PS_OK;
}

}  // namespace ps
