// Helmholtz Nystrom building blocks shared by the device empty-grating
// assembly (empty.cu) and the particle scattering matrix (scatmat.cu):
// complex helpers, H0/H1 from the Miller/Neumann sweep of bessel.cuh, the four
// layer-potential kernels (layerpot._kernel_values_diff, layerpot.py:69-91),
// the two-wavenumber T difference (layerpot._t_difference, layerpot.py:106-141),
// regular waves with gradients (specialfn.regular_wave_block,
// specialfn.py:86-125), and the host-side Alpert stencil tables
// (quadrature._lagrange_weights, quadrature.py:91-101).
#pragma once
#include <cuda_runtime.h>

#include <cmath>

#include "bessel.cuh"

namespace ps {
namespace nys {
namespace {   // internal linkage in each translation unit

constexpr int kCS = 8;          // doubles per curve node: x y nx ny speed weight t aw
constexpr int kMaxRule = 16;
constexpr int kPsiTerms = 14;   // layerpot._y1_series_coeffs (layerpot.py:94-103)

// ---------------------------------------------------------------- complex helpers
__device__ __forceinline__ double2 c2(double a, double b) { return make_double2(a, b); }
__device__ __forceinline__ double2 cadd(double2 a, double2 b) { return c2(a.x + b.x, a.y + b.y); }
__device__ __forceinline__ double2 csub(double2 a, double2 b) { return c2(a.x - b.x, a.y - b.y); }
__device__ __forceinline__ double2 cmul(double2 a, double2 b) {
  return c2(a.x * b.x - a.y * b.y, a.x * b.y + a.y * b.x);
}
__device__ __forceinline__ double2 cscale(double2 a, double s) { return c2(a.x * s, a.y * s); }
__device__ __forceinline__ double2 cmuli(double2 a) { return c2(-a.y, a.x); }   // i a
__device__ __forceinline__ double2 cexpi(double t) {
  double s, c;
  sincos(t, &s, &c);
  return c2(c, s);
}
__device__ __forceinline__ double2 cexp(double2 z) {
  const double e = exp(z.x);
  double s, c;
  sincos(z.y, &s, &c);
  return c2(e * c, e * s);
}
// principal complex sqrt of a real number (numpy sqrt of x + 0j)
__device__ __forceinline__ double2 csqrt_real(double x) {
  return x >= 0.0 ? c2(sqrt(x), 0.0) : c2(0.0, sqrt(-x));
}

// alpha^l for small integer l (|alpha| = 1 for real kappa; the inverse is the
// complex quotient 1 / alpha^|l|, as Python's complex power does)
__device__ __forceinline__ double2 cpow_int(double2 a, int l) {
  double2 r = c2(1.0, 0.0);
  const int n = l < 0 ? -l : l;
  for (int i = 0; i < n; ++i) r = cmul(r, a);
  if (l < 0) {
    const double d = r.x * r.x + r.y * r.y;
    r = c2(r.x / d, -r.y / d);
  }
  return r;
}

__device__ __forceinline__ void hankel01(double z, double2* h0, double2* h1) {
  double j0, j1, y0, y1;
  bessel_jy01(z, miller_start_j01(z), &j0, &j1, &y0, &y1);
  *h0 = c2(j0, y0);
  *h1 = c2(j1, y1);
}

// The four Helmholtz kernels at one (target, source) pair, target-minus-source
// vector (u0, u1): layerpot._kernel_values_diff (layerpot.py:69-91).
struct K4 {
  double2 S, D, N, T;
};
__device__ __forceinline__ K4 kernel4(double k, double u0, double u1, double tnx, double tny,
                                      double snx, double sny) {
  const double r = hypot(u0, u1);
  double2 h0, h1;
  hankel01(k * r, &h0, &h1);
  const double udy = (u0 * snx + u1 * sny) / r;
  const double udx = (u0 * tnx + u1 * tny) / r;
  const double nxny = tnx * snx + tny * sny;
  K4 o;
  o.S = cmuli(cscale(h0, 0.25));
  o.D = cmuli(cscale(h1, 0.25 * k * udy));
  o.N = cmuli(cscale(h1, -0.25 * k * udx));
  const double2 h1p = csub(h0, cscale(h1, 1.0 / (k * r)));
  const double2 t = cadd(cscale(h1p, k * udx * udy), cscale(h1, (nxny - udx * udy) / r));
  o.T = cmuli(cscale(t, 0.25 * k));
  return o;
}

// T^{ka} - T^{kb} with the 1/r^2 singularity removed (layerpot.py:106-141).
__device__ double2 t_difference(const double* psi, double ka, double kb, double u0, double u1,
                                double tnx, double tny, double snx, double sny) {
  const double r = hypot(u0, u1);
  const double p = ((u0 * tnx + u1 * tny) * (u0 * snx + u1 * sny)) / (r * r);
  const double nxny = tnx * snx + tny * sny;
  double ja0, ja1, ya0, ya1, jb0, jb1, yb0, yb1;
  bessel_jy01(ka * r, miller_start_j01(ka * r), &ja0, &ja1, &ya0, &ya1);
  bessel_jy01(kb * r, miller_start_j01(kb * r), &jb0, &jb1, &yb0, &yb1);
  const double2 h0t = csub(cscale(c2(ja0, ya0), ka * ka), cscale(c2(jb0, yb0), kb * kb));
  const double wj = (ka * ja1 - kb * jb1) / r;
  double wy;
  if (fmax(ka, kb) * r < 1.0) {
    auto smooth = [&](double k, double j1) {
      const double z = k * r;
      const double q = -0.25 * z * z;
      double series = 0.0, qm = 1.0;
      for (int m = 0; m < kPsiTerms; ++m) {
        series += psi[m] * qm;
        qm *= q;
      }
      return (2.0 / kPi) * k * k * log(0.5 * z) * (j1 / z) - k * k / (2.0 * kPi) * series;
    };
    wy = smooth(ka, ja1) - smooth(kb, jb1);
  } else {
    wy = (ka * ya1 - kb * yb1) / r;
  }
  const double2 w = c2(wj, wy);
  return cmuli(cscale(cadd(cscale(h0t, p), cscale(w, nxny - 2.0 * p)), 0.25));
}

__device__ __forceinline__ int floordiv(int a, int b) {
  const int q = a / b;
  return (a % b != 0 && ((a < 0) != (b < 0))) ? q - 1 : q;
}

// regular wave J_n(k r) e^{i n theta} about (cx, cy): value and Cartesian
// gradient (specialfn.regular_wave_block, specialfn.py:86-125)
__device__ void regular_wave(double k, double cx, double cy, int n, int nmax, double x, double y,
                             double2* val, double2* gx, double2* gy) {
  const double dx = x - cx, dy = y - cy;
  const double r = hypot(dx, dy);
  if (r == 0.0) {
    *val = c2(n == 0 ? 1.0 : 0.0, 0.0);
    if (n == 1) {
      *gx = c2(0.5 * k, 0.0);
      *gy = c2(0.0, 0.5 * k);
    } else if (n == -1) {
      *gx = c2(-0.5 * k, 0.0);
      *gy = c2(0.0, 0.5 * k);
    } else {
      *gx = c2(0.0, 0.0);
      *gy = c2(0.0, 0.0);
    }
    return;
  }
  const double theta = atan2(dy, dx);
  const int a0 = n < 0 ? -n : n;
  const int a1 = (n + 1) < 0 ? -(n + 1) : (n + 1);
  double ja = 0.0, jb = 0.0, inv, y0, y1;
  bessel_jy_sweep(k * r, nmax + 1, [&](int nu, double v) {
    if (nu == a0) ja = v;
    if (nu == a1) jb = v;
  }, &inv, &y0, &y1);
  double jn = ja * inv, jn1 = jb * inv;
  if (n < 0 && (a0 & 1)) jn = -jn;
  if (n + 1 < 0 && (a1 & 1)) jn1 = -jn1;
  const double2 ph = cexpi(n * theta);
  *val = cscale(ph, jn);
  const double2 dr = cscale(ph, k * (n * jn / (k * r) - jn1));
  const double2 dth = cmuli(cscale(ph, n * jn / r));
  const double ct = cos(theta), st = sin(theta);
  *gx = csub(cscale(dr, ct), cscale(dth, st));
  *gy = cadd(cscale(dr, st), cscale(dth, ct));
}

// quadrature._lagrange_weights (quadrature.py:91-101)
void lagrange(double frac, int interp, int* start, double* w) {
  const int st = (int)std::floor(frac) - (interp / 2 - 1);
  *start = st;
  for (int r = 0; r < interp; ++r) {
    double v = 1.0;
    for (int q = 0; q < interp; ++q)
      if (q != r) v *= (frac - (double)(st + q)) / (double)((st + r) - (st + q));
    w[r] = v;
  }
}

// (psi(m+1) + psi(m+2)) / (m! (m+1)!), m < kPsiTerms, with psi(n) = -gamma +
// H_{n-1} (layerpot._y1_series_coeffs)
inline void psi_series(double* out) {
  long double harm = 0.0L, fact = 1.0L;   // H_m, m!
  const long double g = 0.577215664901532860606512090082402431L;
  for (int mm = 0; mm < kPsiTerms; ++mm) {
    if (mm > 0) {
      harm += 1.0L / mm;
      fact *= mm;
    }
    const long double psi1 = -g + harm, psi2 = -g + harm + 1.0L / (mm + 1);
    out[mm] = (double)((psi1 + psi2) / (fact * fact * (mm + 1)));
  }
}

}  // namespace
}  // namespace nys
}  // namespace ps
