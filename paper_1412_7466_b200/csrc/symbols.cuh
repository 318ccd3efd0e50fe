// Translation symbols t_nu = H^(1)_nu(z) e^{i nu phi}, nu in [-NU, NU].
//
// One thread generates the full symbol row of one (target, source) pair:
// Miller sweep for J (bessel.cuh), Neumann seeds + upward recurrence for Y,
// phase powers by complex recurrence, negative orders by
// H_{-nu} = (-1)^nu H_nu (reference: specialfn._signed_order, sf:79-83).
// The reference path builds the same numbers with scipy H0/H1 + upward
// recurrence (sf:54-67) and np.exp(1j*nu*phi).
#pragma once
#include "bessel.cuh"

namespace ps {

// jst(nu, v): store unnormalised J_nu (nu <= NU); jld(nu): load it back;
// out(nu, re, im): final symbol for signed order nu.
template <int NU, typename JStore, typename JLoad, typename Out>
PS_HD void hankel_symbols(double z, double c, double s, JStore jst, JLoad jld, Out out) {
  double inv, y0, y1;
  bessel_jy_sweep(z, NU > 1 ? NU : 1, jst, &inv, &y0, &y1);
  // nu = 0
  double ym1 = y0, yc = y1;          // Y_{nu-1}, Y_nu  (after the nu=0 step)
  double pr = 1.0, pi = 0.0;         // e^{i nu phi}
  {
    const double J = jld(0) * inv;
    out(0, J, y0);
  }
  const double tz = 2.0 / z;
  double dnu = 1.0;
#pragma unroll 4
  for (int nu = 1; nu <= NU; ++nu) {
    // phase e^{i nu phi}
    const double npr = fma(pr, c, -pi * s);
    const double npi = fma(pr, s, pi * c);
    pr = npr;
    pi = npi;
    const double J = jld(nu) * inv;
    const double Y = yc;
    // H_nu e^{i nu phi}
    const double ar = fma(J, pr, -Y * pi);
    const double ai = fma(J, pi, Y * pr);
    // H_nu e^{-i nu phi} * (-1)^nu
    const double sg = (nu & 1) ? -1.0 : 1.0;
    const double br = sg * fma(J, pr, Y * pi);
    const double bi = sg * fma(Y, pr, -J * pi);
    out(nu, ar, ai);
    out(-nu, br, bi);
    // Y_{nu+1} = (2 nu / z) Y_nu - Y_{nu-1}
    const double yn = fma(dnu * tz, yc, -ym1);
    ym1 = yc;
    yc = yn;
    dnu += 1.0;
  }
}

}  // namespace ps
