// Translation symbols t_nu = H^(1)_nu(z) e^{i nu phi}, nu in [-NU, NU].
//
// Same algorithm as the reference (specialfn.hankel1_orders,
// /root/reference/pkg/src/periscat/specialfn.py:54-67): H_0, H_1 seed an
// upward recurrence H_{nu+1} = (2 nu / z) H_nu - H_{nu-1}; negative orders by
// H_{-nu} = (-1)^nu H_nu (_signed_order, sf:79-83).  The seeds come from a
// Miller sweep for J_0, J_1 with Neumann series for Y_0, Y_1 (bessel.cuh)
// instead of scipy/AMOS; the phases e^{i nu phi} by complex recurrence from
// e^{i phi} = (dx + i dy) / rho (no sincos).
#pragma once
#include "bessel.cuh"

namespace ps {

// out(nu, re, im) is called for nu = 0, then (nu, -nu) pairs, nu = 1..NU.
// N: even Miller start >= miller_start_j01(z).  With c = s = 0 every order
// but nu = 0 comes out exactly zero (used for dead pairs).
template <int NU, typename Out>
PS_HD void hankel_symbols(double z, double c, double s, int N, Out out) {
  double j0, j1, y0, y1;
  bessel_jy01(z, N, &j0, &j1, &y0, &y1);
  out(0, j0, y0);
  double hmr = j0, hmi = y0;     // H_{nu-1}
  double hr = j1, hi = y1;       // H_nu
  double pr = c, pi = s;         // e^{i nu phi}
  const double tz = 2.0 / z;
  double dnu = 1.0;
  int nu = 1;
  // one order: emit t_nu, t_-nu (sign (-1)^nu folded into the static flag)
  auto step = [&](bool odd) {
    const double ar = fma(hr, pr, -hi * pi);
    const double ai = fma(hr, pi, hi * pr);
    const double br = fma(hr, pr, hi * pi);
    const double bi = fma(hi, pr, -hr * pi);
    out(nu, ar, ai);
    if (odd)
      out(-nu, -br, -bi);
    else
      out(-nu, br, bi);
    const double cf = dnu * tz;
    const double nr = fma(cf, hr, -hmr);
    const double ni = fma(cf, hi, -hmi);
    hmr = hr;
    hmi = hi;
    hr = nr;
    hi = ni;
    dnu += 1.0;
    const double qr = fma(pr, c, -pi * s);
    const double qi = fma(pr, s, pi * c);
    pr = qr;
    pi = qi;
    ++nu;
  };
  for (int it = 0; it < NU / 2; ++it) {
    step(true);
    step(false);
  }
  if (NU & 1) step(true);
}

// Half of a symbol row for two cooperating lanes.  mirror = false emits
// t_nu (nu = 0..NU); mirror = true emits t_{-nu} (nu = 1..NU) from
// G_nu = (-1)^nu H_nu with the conjugate phase:
//   G_0 = H_0, G_1 = -H_1, G_{nu+1} = -(2 nu / z) G_nu - G_{nu-1},
//   t_{-nu} = G_nu e^{-i nu phi}.
// The recurrence runs directly on the phased symbols T_nu = G_nu w^nu
// (w = e^{+-i phi}):  T_{nu+1} = nu (a T_nu) - b T_{nu-1},  a = q (2/z) w,
// b = w^2 -- the reference's H recurrence rotated by w each step, so no
// separate phase recurrence or product (10 FP64 ops per order instead of 11).
// Both lanes of a pair run the same instruction stream.
template <int NU, typename Out>
PS_HD void hankel_symbols_half(double z, double c, double s, int N, bool mirror, Out out) {
  double j0, j1, y0, y1;
  bessel_jy01(z, N, &j0, &j1, &y0, &y1);
  const double q = mirror ? -1.0 : 1.0;
  if (!mirror) out(0, j0, y0);
  const double wr = c, wi = q * s;              // w = e^{i q phi}
  const double tz = q * (2.0 / z);
  const double ar = tz * wr, ai = tz * wi;      // a = q (2/z) w
  const double br = fma(wr, wr, -wi * wi), bi = 2.0 * wr * wi;   // b = w^2
  double tmr = j0, tmi = y0;                    // T_0 = H_0
  const double g1r = q * j1, g1i = q * y1;      // G_1
  double tr = fma(g1r, wr, -g1i * wi), ti = fma(g1r, wi, g1i * wr);   // T_1 = G_1 w
#pragma unroll
  for (int nu = 1; nu <= NU; ++nu) {
    out(mirror ? -nu : nu, tr, ti);
    const double ur = fma(ar, tr, -ai * ti), ui = fma(ar, ti, ai * tr);          // a T_nu
    const double vr = fma(br, tmr, -bi * tmi), vi = fma(br, tmi, bi * tmr);      // b T_{nu-1}
    const double dnu = (double)nu;
    tmr = tr;
    tmi = ti;
    tr = fma(dnu, ur, -vr);
    ti = fma(dnu, ui, -vi);
  }
}


// Same output as hankel_symbols_half, arranged for a short dependency chain
// (producers that share the FP64 pipe with tensor-core or DFMA consumers are
// latency-bound): the reference's own upward recurrence on the unphased
// H_nu = J_nu + i Y_nu (sf:54-67; one FMA per order on each real chain, the
// factor nu * 2/z off the chain), times phases w^nu kept as two power chains
// (even / odd nu, stepping by w^2).  The mirror lane uses w = -e^{-i phi}, so
// (-1)^nu H_nu e^{-i nu phi} = H_nu w^nu needs no sign handling.
template <int NU, typename Out>
PS_HD void hankel_symbols_ilp(double z, double c, double s, int N, bool mirror, Out out) {
  double j0, j1, y0, y1;
  bessel_jy01(z, N, &j0, &j1, &y0, &y1);
  if (!mirror) out(0, j0, y0);
  const double wr = mirror ? -c : c, wi = s;   // mirror: -e^{-i phi} = (-c, s)
  const double w2r = fma(wr, wr, -wi * wi), w2i = 2.0 * wr * wi;
  const double tz = 2.0 / z;
  double hmr = j0, hmi = y0;      // H_{nu-1}
  double hr = j1, hi = y1;        // H_nu
  double per = 1.0, pei = 0.0;    // w^nu for the even chain (nu = 0 here)
  double por = wr, poi = wi;      // w^nu for the odd chain (nu = 1 here)
#pragma unroll
  for (int nu = 1; nu <= NU; ++nu) {
    const bool odd = nu & 1;
    if (!odd) {                   // even chain: w^{nu} = w^{nu-2} w^2
      const double r = fma(per, w2r, -pei * w2i), i = fma(per, w2i, pei * w2r);
      per = r;
      pei = i;
    } else if (nu > 1) {
      const double r = fma(por, w2r, -poi * w2i), i = fma(por, w2i, poi * w2r);
      por = r;
      poi = i;
    }
    const double pr = odd ? por : per, pi = odd ? poi : pei;
    out(mirror ? -nu : nu, fma(hr, pr, -hi * pi), fma(hr, pi, hi * pr));
    const double cf = (double)nu * tz;
    const double nr = fma(cf, hr, -hmr), ni = fma(cf, hi, -hmi);
    hmr = hr;
    hmi = hi;
    hr = nr;
    hi = ni;
  }
}

}  // namespace ps
