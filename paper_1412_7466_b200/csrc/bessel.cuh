// Integer-order Bessel / Hankel generation in FP64 for the M2L symbols.
//
// Replaces the reference's scipy-seeded upward recurrence
// (specialfn.hankel1_orders, /root/reference/pkg/src/periscat/specialfn.py:54-67)
// with a self-contained, branch-light device routine:
//
//   * J_0..J_N by Miller's backward recurrence normalised with
//     J_0 + 2 sum_k J_2k = 1 (accurate for every order, including nu > z
//     where the reference's upward recurrence loses the J part);
//   * Y_0, Y_1 from the Neumann series
//       Y_0 = (2/pi)(ln(z/2)+gamma) J_0 - (4/pi) sum_k (-1)^k J_2k / k
//       Y_1 = (2/pi)(ln(z/2)+gamma) J_1 - (2/pi) J_0 / z
//             + (2/pi) sum_k (-1)^k (J_{2k-1} - J_{2k+1}) / k
//     accumulated inside the same backward sweep;
//   * Y_nu, nu >= 2, by the (stable) upward recurrence.
//
// Compiled both for the device and (tests/test_bessel_host.py) for the host,
// where it is checked against scipy.special to <= 1e-14 relative in |H_nu|.
#pragma once

#ifdef __CUDACC__
#define PS_HD __host__ __device__ __forceinline__
#else
#include <cmath>
#define PS_HD inline
#endif

namespace ps {

constexpr double kPi = 3.14159265358979323846;
constexpr double kEulerGamma = 0.57721566490153286061;

// 1/k for the Neumann sums without a per-step division (k < 128 covers
// z <= ~150 at the orders used here).
#define PS_I4(k) 1.0 / (k), 1.0 / ((k) + 1), 1.0 / ((k) + 2), 1.0 / ((k) + 3)
#define PS_I16(k) PS_I4(k), PS_I4((k) + 4), PS_I4((k) + 8), PS_I4((k) + 12)
#ifdef __CUDACC__
static __constant__ double c_inv_int[128] = {
    0.0, 1.0, 0.5, 1.0 / 3.0, PS_I4(4), PS_I4(8), PS_I4(12), PS_I16(16),
    PS_I16(32), PS_I16(48), PS_I16(64), PS_I16(80), PS_I16(96), PS_I16(112)};
#endif
// (-1)^k / k
#define PS_S4(k) (((k) & 1) ? -1.0 : 1.0) / (k), (((k) + 1) & 1 ? -1.0 : 1.0) / ((k) + 1), \
                 (((k) + 2) & 1 ? -1.0 : 1.0) / ((k) + 2), (((k) + 3) & 1 ? -1.0 : 1.0) / ((k) + 3)
#define PS_S16(k) PS_S4(k), PS_S4((k) + 4), PS_S4((k) + 8), PS_S4((k) + 12)
#ifdef __CUDACC__
static __constant__ double c_sinv_int[128] = {
    0.0, -1.0, 0.5, -1.0 / 3.0, PS_S4(4), PS_S4(8), PS_S4(12), PS_S16(16),
    PS_S16(32), PS_S16(48), PS_S16(64), PS_S16(80), PS_S16(96), PS_S16(112)};
#endif
PS_HD double sinv_int(int k) {
#if defined(__CUDA_ARCH__)
  return k < 128 ? c_sinv_int[k] : ((k & 1) ? -1.0 : 1.0) / (double)k;
#else
  return ((k & 1) ? -1.0 : 1.0) / (double)k;
#endif
}

PS_HD double inv_int(int k) {
#if defined(__CUDA_ARCH__)
  return k < 128 ? c_inv_int[k] : 1.0 / (double)k;
#else
  return 1.0 / (double)k;
#endif
}

// Start index of the Miller sweep: even, and far enough above both the
// requested order and the turning point nu ~ z that the truncation error is
// below double rounding (checked over z in [1e-3, 80], nmax <= 64).
PS_HD int miller_start(double z, int nmax) {
  double a = z > (double)nmax ? z : (double)nmax;
  double zc = z > 1.0 ? z : 1.0;
  int n = (int)(a + 16.0 + 6.0 * cbrt(zc));
  return (n + 1) & ~1;
}

// Writes J_nu(z) * scale for nu = 0..nmax into J[] (unnormalised), and returns
// 1/scale in *inv_norm together with Y0, Y1 (already normalised).
// Callers multiply J[nu] by *inv_norm.  z > 0, nmax >= 1.
template <typename Store>
PS_HD void bessel_jy_sweep(double z, int nmax, Store store, double* inv_norm,
                           double* y0, double* y1) {
  const int N = miller_start(z, nmax);
  const double tz = 2.0 / z;
  // j_{N+1} = 0, j_N = tiny; go down two orders per step so the parity of
  // the normalisation / Neumann sums is static.
  double jp1 = 0.0;           // j_{nu+1}
  double j = 1e-280;          // j_nu, nu = N (even)
  double sum_even = 0.0;      // sum_{k>=1} j_{2k}
  double s0 = 0.0;            // sum_{k>=1} (-1)^k j_{2k} / k
  double s1 = 0.0;            // sum_{k>=1} (-1)^k (j_{2k-1} - j_{2k+1}) / k
  double j_odd_above = 0.0;   // j_{2k+1} for the current even nu = 2k
  if (N <= nmax) store(N, j);
  for (int nu = N; nu >= 2; nu -= 2) {
    // nu even = 2k here; j = j_nu, jp1 = j_{nu+1}
    const int k = nu >> 1;
    const double sgn = (k & 1) ? -1.0 : 1.0;
    const double inv_k = inv_int(k);
    sum_even += j;
    s0 = fma(sgn * inv_k, j, s0);
    j_odd_above = jp1;
    // j_{nu-1}
    const double jm1 = fma((double)nu * tz, j, -jp1);
    // j_{nu-2}
    const double jm2 = fma((double)(nu - 1) * tz, jm1, -j);
    // (j_{2k-1} - j_{2k+1}) / k term
    s1 = fma(sgn * inv_k, jm1 - j_odd_above, s1);
    if (nu - 1 <= nmax) store(nu - 1, jm1);
    if (nu - 2 <= nmax) store(nu - 2, jm2);
    jp1 = jm1;
    j = jm2;
  }
  // j = j_0, jp1 = j_1
  const double norm = j + 2.0 * sum_even;
  const double inv = 1.0 / norm;
  const double J0 = j * inv, J1 = jp1 * inv;
  const double lg = log(0.5 * z) + kEulerGamma;
  const double c = 2.0 / kPi;
  *y0 = c * (lg * J0) - 2.0 * c * (s0 * inv);
  *y1 = c * (lg * J1) - c * J0 / z + c * (s1 * inv);
  *inv_norm = inv;
}

// Even Miller start index sufficient for J_0, J_1 (and the Neumann sums) to
// double accuracy; callers may pass any larger even value (e.g. a warp max).
PS_HD int miller_start_j01(double z) {
  double zc = z > 1.0 ? z : 1.0;
  int n = (int)(z + 18.0 + 6.0 * cbrt(zc));
  return (n + 1) & ~1;
}

// J0, J1, Y0, Y1 of z > 0 from a Miller sweep started at even N (no stores).
PS_HD void bessel_jy01(double z, int N, double* j0, double* j1, double* y0, double* y1) {
  const double tz = 2.0 / z;
  double jp1 = 0.0, j = 1e-280;
  double sum_even = 0.0, s0 = 0.0, s1 = 0.0;
  double dnu = (double)N;        // exact small integers: no drift in nu * 2/z
  for (int nu = N; nu >= 2; nu -= 2) {
    const double sk = sinv_int(nu >> 1);   // (-1)^k / k, k = nu/2
    sum_even += j;
    s0 = fma(sk, j, s0);
    const double jm1 = fma(dnu * tz, j, -jp1);
    const double jm2 = fma((dnu - 1.0) * tz, jm1, -j);
    s1 = fma(sk, jm1 - jp1, s1);
    jp1 = jm1;
    j = jm2;
    dnu -= 2.0;
  }
  const double inv = 1.0 / (j + 2.0 * sum_even);
  const double J0 = j * inv, J1 = jp1 * inv;
  const double lg = log(0.5 * z) + kEulerGamma;
  const double c = 2.0 / kPi;
  *j0 = J0;
  *j1 = J1;
  *y0 = c * (lg * J0) - 2.0 * c * (s0 * inv);
  *y1 = c * (lg * J1) - c * J0 / z + c * (s1 * inv);
}

}  // namespace ps
