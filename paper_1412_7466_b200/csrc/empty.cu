// Empty-grating setup on the device: assembly of the
// column-scaled block matrix A and right-hand side f of the inclusion-free
// three-layer grating, its SVD, and the restricted A^+ factors the Schur
// correction streams every GMRES iteration.
//
// Replaces, per right-hand side (incidence angle):
//   empty_grating.assemble_empty_system   (empty_grating.py:139-256)
//     + layerpot.boundary_operator_matrices (layerpot.py:171-208)
//     + quadrature.nystrom_selfmatrix       (quadrature.py:106-186; Alpert
//       log-corrections with the quasi-periodic stencil wrap)
//     + layerpot._t_difference              (layerpot.py:106-141)
//     + layerpot.wall_discrepancy_blocks    (layerpot.py:211-237)
//     + specialfn.regular_wave_block        (specialfn.py:86-125)
//     + empty_grating.rb_basis / incident_field (empty_grating.py:32-61)
//   empty_grating.factorize                 (empty_grating.py:259-261; cuSOLVER
//                                             zgesvd in place of LAPACK gesdd)
//   and the restriction ps_set_pinv performs on host factors (capi.cu).
//
// Work decomposition: every matrix entry is owned by exactly one work item of
// one task (a (row block, column block) pair of eg:164-238); one launch covers
// all tasks of all right-hand sides (grid.y = RHS).  Interface/lid/wall items
// are (target node, source node) pairs that evaluate H0/H1 once per phased
// copy and write the 2x2 [[D, S], [T, N]] entries; regular-expansion items are
// (node, order) pairs with a Miller sweep per item.  The Alpert corrections of
// the two self blocks are gathered, not scattered: a first kernel evaluates the
// kernel at the 2 x rule_n off-grid nodes of every row, and each entry (i, j)
// sums the (at most one per off-grid node) Lagrange stencil weight landing on
// column j -- the same terms np.add.at accumulates (quadrature.py:166-186).
#include <cuda_runtime.h>
#include <cusolverDn.h>

#include <algorithm>
#include <cmath>
#include <complex>
#include <mutex>
#include <string>
#include <thread>
#include <vector>

#include "bessel.cuh"
#include "coupling.cuh"
#include "ctx.cuh"
#include "empty.cuh"
#include "nystrom.cuh"

namespace ps {

namespace {

using namespace nys;
constexpr int kMaxTasks = 24;
constexpr int kMaxCoef = 8;     // trig coefficients per interface

enum Kind { K_SELF = 0, K_CROSS, K_WALL, K_REG, K_WALLREG, K_RB, K_INC };
enum CurveId { C_G1 = 0, C_G2, C_L1, C_L2, C_L3, C_GU, C_GD, C_NCURVE };

struct Task {
  int kind, src, tgt;
  int row_v, row_d, col_a, col_b;
  int nt, ns;              // items = nt * ns
  int spec;                // interface spec (SELF)
  int up;                  // RB direction
  double k, ksub, sign;
  double cx, cy;           // expansion centre (REG / WALLREG)
  long long item0;
};

struct Spec {
  double mean;
  int nsin, ncos;
  double sc[kMaxCoef], cc[kMaxCoef];
};

struct Tables {
  Task task[kMaxTasks];
  int ntask;
  long long nitems;
  const double* curve[C_NCURVE];
  int ncurve[C_NCURVE];
  Spec spec[2];
  int m, ncol, copies, Q, nrb;
  double period, y0, k1, k3;
  int rule_n, skip, interp;
  double rule_x[kMaxRule], rule_w[kMaxRule];
  int lag_start[2][kMaxRule];
  double lag_w[2][kMaxRule][kMaxRule];
  double psi[kPsiTerms];
};

struct RhsPar {   // per incidence angle
  double ar, ai;        // bloch alpha
  double kappa;         // k1 cos(theta)
  double kix, kiy;      // k1 (cos theta, sin theta)
  double pad;
};

// Interface graph y(x) = mean + sum a_j sin(2 pi j x/d) + b_j cos(2 pi j x/d)
// at parameter tau (geometry.py:198-207): point, tangent speed, unit normal.
__device__ void spec_eval(const Spec& s, double d, double tau, double* px, double* py,
                          double* speed, double* nx, double* ny) {
  const double x = d * (tau - 0.5);
  double y = s.mean, dy = 0.0;
  for (int j = 0; j < s.nsin; ++j) {
    const double w = 2.0 * kPi * (j + 1) / d;
    y += s.sc[j] * sin(2.0 * kPi * (j + 1) * x / d);
    dy += s.sc[j] * w * cos(2.0 * kPi * (j + 1) * x / d);
  }
  for (int j = 0; j < s.ncos; ++j) {
    const double w = 2.0 * kPi * (j + 1) / d;
    y += s.cc[j] * cos(2.0 * kPi * (j + 1) * x / d);
    dy -= s.cc[j] * w * sin(2.0 * kPi * (j + 1) * x / d);
  }
  *px = x;
  *py = y;
  *speed = hypot(d, d * dy);
  const double nn = hypot(-dy, 1.0);
  *nx = -dy / nn;
  *ny = 1.0 / nn;
}

// x(s) - x(tau) without cancellation (geometry.py:209-217)
__device__ void spec_diff(const Spec& sp, double d, double s, double tau, double* u0, double* u1) {
  double dy = 0.0;
  for (int j = 0; j < sp.nsin; ++j)
    dy += 2.0 * sp.sc[j] * cos(kPi * (j + 1) * (s + tau - 1.0)) * sin(kPi * (j + 1) * (s - tau));
  for (int j = 0; j < sp.ncos; ++j)
    dy -= 2.0 * sp.cc[j] * sin(kPi * (j + 1) * (s + tau - 1.0)) * sin(kPi * (j + 1) * (s - tau));
  *u0 = d * (s - tau);
  *u1 = dy;
}

// ---------------------------------------------------------------- kernels
// Alpert off-grid kernel values of the two self blocks:
// kv[slot][i][side*rule_n + m] = {D, S, T, N} * speed(tau) * w_m h
// (quadrature.py:166-178, with the stable parameter difference).
__global__ void alpert_kv_kernel(Tables tb, double2* kv) {
  const int n = tb.rule_n;
  const int per_slot_rows[2] = {tb.ncurve[C_G1], tb.ncurve[C_G2]};
  const int total0 = per_slot_rows[0] * 2 * n;
  const int total = total0 + per_slot_rows[1] * 2 * n;
  for (int id = blockIdx.x * blockDim.x + threadIdx.x; id < total; id += gridDim.x * blockDim.x) {
    const int slot = id < total0 ? 0 : 1;
    const int rem = id - (slot ? total0 : 0);
    const int i = rem / (2 * n);
    const int sm = rem % (2 * n);
    const int side = sm / n, m = sm % n;
    const Task& t = tb.task[slot == 0 ? 0 : 2];    // SELF tasks sit at 0 (g1) and 2 (g2)
    const double* cv = tb.curve[t.src];
    const int nn = tb.ncurve[t.src];
    const double h = 1.0 / nn;                      // curve.dt, parameter period 1
    const double sgn = side == 0 ? 1.0 : -1.0;
    const double ti = cv[i * kCS + 6];
    const double tau = ti + sgn * tb.rule_x[m] * h;
    double px, py, sp, nx, ny;
    spec_eval(tb.spec[t.spec], tb.period, tau, &px, &py, &sp, &nx, &ny);
    double u0, u1;
    spec_diff(tb.spec[t.spec], tb.period, ti, tau, &u0, &u1);
    const double tnx = cv[i * kCS + 2], tny = cv[i * kCS + 3];
    const K4 a = kernel4(t.k, u0, u1, tnx, tny, nx, ny);
    const K4 b = kernel4(t.ksub, u0, u1, tnx, tny, nx, ny);
    const double2 T = t_difference(tb.psi, t.k, t.ksub, u0, u1, tnx, tny, nx, ny);
    const double w = sp * (tb.rule_w[m] * h);
    double2* o = kv + (size_t)id * 4;
    o[0] = cscale(csub(a.D, b.D), w);
    o[1] = cscale(csub(a.S, b.S), w);
    o[2] = cscale(T, w);
    o[3] = cscale(csub(a.N, b.N), w);
  }
}

__device__ __forceinline__ void put(double2* A, int m, int row, int col, double2 v) {
  A[(size_t)col * m + row] = v;
}

__global__ void assemble_kernel(Tables tb, const RhsPar* __restrict__ rp,
                                const double2* __restrict__ kv, double2* __restrict__ Aall,
                                double2* __restrict__ fall) {
  const int r = blockIdx.y;
  const RhsPar P = rp[r];
  const double2 alpha = c2(P.ar, P.ai);
  const int m = tb.m;
  double2* A = Aall + (size_t)r * m * tb.ncol;
  double2* f = fall + (size_t)r * m;
  const int cp = tb.copies;
  for (long long id = (long long)blockIdx.x * blockDim.x + threadIdx.x; id < tb.nitems;
       id += (long long)gridDim.x * blockDim.x) {
    int ti = 0;
    while (ti + 1 < tb.ntask && tb.task[ti + 1].item0 <= id) ++ti;
    const Task& t = tb.task[ti];
    const int loc = (int)(id - t.item0);
    const int i = loc / t.ns, j = loc % t.ns;
    const double* tc = tb.curve[t.tgt];
    const double tx = tc[i * kCS], ty = tc[i * kCS + 1];
    const double tnx = tc[i * kCS + 2], tny = tc[i * kCS + 3];
    switch (t.kind) {
      case K_SELF: {
        // quadrature.nystrom_selfmatrix, open_periodic window of 2P+1 copies
        const double* sc = tb.curve[t.src];
        const int n = t.ns;
        const double h = 1.0 / n;
        const double sx0 = sc[j * kCS], sy = sc[j * kCS + 1];
        const double snx = sc[j * kCS + 2], sny = sc[j * kCS + 3];
        const double sw = sc[j * kCS + 4] * h;
        double2 D = c2(0, 0), S = D, T = D, N = D;
        for (int l = -cp; l <= cp; ++l) {
          const int off = l * n + j - i;
          bool band;
          if (cp == 0) {
            const int om = ((off % n) + n) % n;
            band = min(om, n - om) <= tb.skip - 1;
          } else {
            band = (off < 0 ? -off : off) <= tb.skip - 1;
          }
          if (band) continue;
          const double u0 = tx - (sx0 + l * tb.period), u1 = ty - sy;
          const K4 a = kernel4(t.k, u0, u1, tnx, tny, snx, sny);
          const K4 b = kernel4(t.ksub, u0, u1, tnx, tny, snx, sny);
          const double2 Td = t_difference(tb.psi, t.k, t.ksub, u0, u1, tnx, tny, snx, sny);
          const double2 w = cscale(cpow_int(alpha, l), sw);
          D = cadd(D, cmul(csub(a.D, b.D), w));
          S = cadd(S, cmul(csub(a.S, b.S), w));
          T = cadd(T, cmul(Td, w));
          N = cadd(N, cmul(csub(a.N, b.N), w));
        }
        // gathered Alpert corrections (quadrature.py:166-186)
        const int slot = ti == 0 ? 0 : 1;
        const int rn = tb.rule_n;
        const double2* kr = kv + ((size_t)(slot ? tb.ncurve[C_G1] * 2 * rn : 0) +
                                  (size_t)i * 2 * rn) * 4;
        for (int side = 0; side < 2; ++side)
          for (int mm = 0; mm < rn; ++mm) {
            const int st = tb.lag_start[side][mm];
            int rr = (j - i - st) % n;
            if (rr < 0) rr += n;
            if (rr >= tb.interp) continue;
            const int qr = i + st + rr;
            const double2 cw = cscale(cpow_int(alpha, floordiv(qr, n)), tb.lag_w[side][mm][rr]);
            const double2* q = kr + (size_t)(side * rn + mm) * 4;
            D = cadd(D, cmul(q[0], cw));
            S = cadd(S, cmul(q[1], cw));
            T = cadd(T, cmul(q[2], cw));
            N = cadd(N, cmul(q[3], cw));
          }
        if (i == j) {
          D.x += 1.0;
          N.x -= 1.0;
        }
        put(A, m, t.row_v + i, t.col_a + j, D);
        put(A, m, t.row_v + i, t.col_b + j, S);
        put(A, m, t.row_d + i, t.col_a + j, T);
        put(A, m, t.row_d + i, t.col_b + j, N);
        break;
      }
      case K_CROSS: {
        // layerpot.boundary_operator_matrices, disjoint curves (layerpot.py:194-208)
        const double* sc = tb.curve[t.src];
        const double sx0 = sc[j * kCS], sy = sc[j * kCS + 1];
        const double snx = sc[j * kCS + 2], sny = sc[j * kCS + 3];
        const double aw = sc[j * kCS + 7];
        double2 D = c2(0, 0), S = D, T = D, N = D;
        for (int l = -cp; l <= cp; ++l) {
          const K4 a = kernel4(t.k, tx - (sx0 + l * tb.period), ty - sy, tnx, tny, snx, sny);
          const double2 w = cpow_int(alpha, l);
          D = cadd(D, cmul(w, a.D));
          S = cadd(S, cmul(w, a.S));
          T = cadd(T, cmul(w, a.T));
          N = cadd(N, cmul(w, a.N));
        }
        const double s = t.sign * aw;
        put(A, m, t.row_v + i, t.col_a + j, cscale(D, s));
        put(A, m, t.row_v + i, t.col_b + j, cscale(S, s));
        put(A, m, t.row_d + i, t.col_a + j, cscale(T, s));
        put(A, m, t.row_d + i, t.col_b + j, cscale(N, s));
        break;
      }
      case K_WALL: {
        // telescoped wall discrepancy (layerpot.wall_discrepancy_blocks, lp:211-237)
        const double* sc = tb.curve[t.src];
        const double sx0 = sc[j * kCS], sy = sc[j * kCS + 1];
        const double snx = sc[j * kCS + 2], sny = sc[j * kCS + 3];
        const double aw = sc[j * kCS + 7];
        double2 D = c2(0, 0), S = D, T = D, N = D;
        for (int e = 0; e < 2; ++e) {
          const int l = e == 0 ? cp : -(cp + 1);
          const double2 coef = cscale(cpow_int(alpha, e == 0 ? cp + 1 : -cp), e == 0 ? 1.0 : -1.0);
          const K4 a = kernel4(t.k, tx - (sx0 + l * tb.period), ty - sy, tnx, tny, snx, sny);
          D = cadd(D, cmul(coef, a.D));
          S = cadd(S, cmul(coef, a.S));
          T = cadd(T, cmul(coef, a.T));
          N = cadd(N, cmul(coef, a.N));
        }
        put(A, m, t.row_v + i, t.col_a + j, cscale(D, aw));
        put(A, m, t.row_v + i, t.col_b + j, cscale(S, aw));
        put(A, m, t.row_d + i, t.col_a + j, cscale(T, aw));
        put(A, m, t.row_d + i, t.col_b + j, cscale(N, aw));
        break;
      }
      case K_REG: {
        // regular-expansion traces (empty_grating._regular_block, eg:121-124)
        const int n = j - tb.Q;
        double2 v, gx, gy;
        regular_wave(t.k, t.cx, t.cy, n, tb.Q, tx, ty, &v, &gx, &gy);
        const double2 der = cadd(cscale(gx, tnx), cscale(gy, tny));
        put(A, m, t.row_v + i, t.col_a + j, cscale(v, t.sign));
        put(A, m, t.row_d + i, t.col_a + j, cscale(der, t.sign));
        break;
      }
      case K_WALLREG: {
        // alpha * u(L) - u(R) for the layer's regular expansion (eg:215-218)
        const int n = j - tb.Q;
        double2 vl, gl, gyl, vr, gr, gyr;
        regular_wave(t.k, t.cx, t.cy, n, tb.Q, tx, ty, &vl, &gl, &gyl);
        regular_wave(t.k, t.cx, t.cy, n, tb.Q, tx + tb.period, ty, &vr, &gr, &gyr);
        put(A, m, t.row_v + i, t.col_a + j, csub(cmul(alpha, vl), vr));
        put(A, m, t.row_d + i, t.col_a + j, csub(cmul(alpha, gl), gr));
        break;
      }
      case K_RB: {
        // Rayleigh-Bloch modes on the artificial boundary (empty_grating.rb_basis, eg:44-61)
        const int half = tb.nrb / 2;
        const double kapn = P.kappa + 2.0 * kPi * (double)(j - half) / tb.period;
        const double k = t.up ? tb.k1 : tb.k3;
        // k^2 - kappa_n^2 rounded exactly as numpy does (no FMA contraction):
        // at a Wood anomaly it is a near-cancellation and kyn ~ 1e-7
        const double2 kyn = csqrt_real(__dsub_rn(__dmul_rn(k, k), __dmul_rn(kapn, kapn)));
        const double2 ph = cexpi(tx * kapn);
        const double yy = t.up ? (ty - tb.y0) : (-ty - tb.y0);
        const double2 vert = cexp(cmuli(cscale(kyn, yy)));
        double2 dvert = cmul(cmuli(kyn), vert);
        if (!t.up) dvert = cscale(dvert, -1.0);
        put(A, m, t.row_v + i, t.col_a + j, cscale(cmul(ph, vert), -1.0));
        put(A, m, t.row_d + i, t.col_a + j, cscale(cmul(ph, dvert), -1.0));
        break;
      }
      case K_INC: {
        // f = -(incident trace) on Gamma1 (empty_grating.incident_field, eg:32-42, 241-245)
        const double2 v = cexpi(tx * P.kix + ty * P.kiy);
        const double2 dv = cmul(c2(0.0, tnx * P.kix + tny * P.kiy), v);
        f[t.row_v + i] = cscale(v, -1.0);
        f[t.row_d + i] = cscale(dv, -1.0);
        break;
      }
    }
  }
}

// Column scaling of the expansion and Rayleigh-Bloch columns to unit max
// magnitude (eg:247-254).  grid (ncol - col0, nrhs); cs [nrhs][ncol].
__global__ void colscale_kernel(double2* __restrict__ Aall, double* __restrict__ csall, int m,
                                int ncol, int col0) {
  const int r = blockIdx.y;
  const int col = blockIdx.x;
  double2* a = Aall + (size_t)r * m * ncol + (size_t)col * m;
  double* cs = csall + (size_t)r * ncol;
  __shared__ double red[32];
  if (col < col0) {
    if (threadIdx.x == 0) cs[col] = 1.0;
    return;
  }
  double mx = 0.0;
  for (int i = threadIdx.x; i < m; i += blockDim.x) mx = fmax(mx, hypot(a[i].x, a[i].y));
  for (int o = 16; o; o >>= 1) mx = fmax(mx, __shfl_xor_sync(0xffffffffu, mx, o));
  if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = mx;
  __syncthreads();
  if (threadIdx.x < 32) {
    mx = threadIdx.x < (blockDim.x >> 5) ? red[threadIdx.x] : 0.0;
    for (int o = 16; o; o >>= 1) mx = fmax(mx, __shfl_xor_sync(0xffffffffu, mx, o));
    if (threadIdx.x == 0) red[0] = mx;
  }
  __syncthreads();
  mx = red[0];
  if (mx == 0.0) mx = 1.0;
  for (int i = threadIdx.x; i < m; i += blockDim.x) a[i] = c2(a[i].x / mx, a[i].y / mx);
  if (threadIdx.x == 0) cs[col] = 1.0 / mx;
}

// Restricted A^+ factors from the device SVD (what ps_set_pinv builds on the
// host): Uh[k][i] = conj(U[i][k]) for the C rows, sinv, Vb[o][k] =
// conj(Vh[k][col(o)]), the column scales of the output columns and f on the C
// rows.  U column-major [ncol][m], VT column-major [ncol][ncol] (= Vh).
__global__ void pinv_extract_kernel(const double2* __restrict__ U, const double* __restrict__ s,
                                    const double2* __restrict__ VT,
                                    const double* __restrict__ cs_full,
                                    const double2* __restrict__ f_full, int m, int ncol, int nrc,
                                    int ncol_b, int nrb, int col_c, int col_d, int nfield,
                                    double eps, double2* Uh, double* sinv, double2* Vb, double* cs,
                                    double2* f) {
  const int nout0 = ncol_b + 2 * nrb;
  const int nout = nout0 + nfield;   // + the a1 / a3 field rows
  const long long nu = (long long)ncol * nrc, nv = (long long)nout * ncol;
  const long long tot = nu + nv + ncol + nout + nrc;
  for (long long id = (long long)blockIdx.x * blockDim.x + threadIdx.x; id < tot;
       id += (long long)gridDim.x * blockDim.x) {
    if (id < nu) {
      const int k = (int)(id / nrc), i = (int)(id % nrc);
      const double2 u = U[(size_t)k * m + i];
      Uh[id] = c2(u.x, -u.y);
    } else if (id < nu + nv) {
      const long long q = id - nu;
      const int o = (int)(q / ncol), k = (int)(q % ncol);
      const int col = o < ncol_b ? o : (o < ncol_b + nrb ? col_c + o - ncol_b
                                       : (o < nout0 ? col_d + o - ncol_b - nrb : ncol_b + o - nout0));
      const double2 v = VT[(size_t)col * ncol + k];
      Vb[q] = c2(v.x, -v.y);
    } else if (id < nu + nv + ncol) {
      const int k = (int)(id - nu - nv);
      sinv[k] = fmin(1.0 / s[k], 1.0 / eps);
    } else if (id < nu + nv + ncol + nout) {
      const int o = (int)(id - nu - nv - ncol);
      const int col = o < ncol_b ? o : (o < ncol_b + nrb ? col_c + o - ncol_b
                                       : (o < nout0 ? col_d + o - ncol_b - nrb : ncol_b + o - nout0));
      cs[o] = cs_full[col];
    } else {
      const int i = (int)(id - nu - nv - ncol - nout);
      f[i] = f_full[i];
    }
  }
}

// one cuSOLVER handle + workspace per (device, worker); created lazily and
// kept for the process (cusolverDnCreate costs tens of ms)
struct SvdWorker {
  cusolverDnHandle_t h = nullptr;
  cudaStream_t st = nullptr;
  void* work = nullptr;
  size_t work_bytes = 0;
  double2 *A = nullptr, *U = nullptr, *VT = nullptr;
  double* rwork = nullptr;
  int* info = nullptr;
  int m = 0, n = 0;
};
std::mutex g_svd_mu;
std::mutex g_dev_mu[64];   // one SVD phase per device at a time
std::vector<SvdWorker> g_svd[64];

std::string svd_err(const char* what, int code) {
  return std::string(what) + " failed (status " + std::to_string(code) + ")";
}

// A (m x n column-major, m >= n, on the device) -> U, s, VT (zgesvd:
// Householder bidiagonalisation + implicit QR, the decomposition LAPACK gesdd
// returns) in the worker's buffers; blocks the calling thread until done.
int svd_run(SvdWorker& w, const double2* A, int m, int n, double* s, std::string* err) {
  if (!w.h) {
    if (cudaStreamCreateWithFlags(&w.st, cudaStreamNonBlocking) != cudaSuccess) {
      *err = "svd: stream create";
      return PS_ERR_CUDA;
    }
    cusolverStatus_t cs = cusolverDnCreate(&w.h);
    if (cs != CUSOLVER_STATUS_SUCCESS) {
      *err = svd_err("cusolverDnCreate", cs);
      return PS_ERR_CUDA;
    }
    cusolverDnSetStream(w.h, w.st);
  }
  if (w.m != m || w.n != n) {
    void* bufs[] = {w.work, w.A, w.U, w.VT, w.rwork, w.info};
    for (void* p : bufs)
      if (p) dev_free(p);
    w.work = nullptr;
    int lwork = 0;
    cusolverStatus_t cs = cusolverDnZgesvd_bufferSize(w.h, m, n, &lwork);
    if (cs != CUSOLVER_STATUS_SUCCESS) {
      *err = svd_err("cusolverDnZgesvd_bufferSize", cs);
      return PS_ERR_CUDA;
    }
    const size_t dev_bytes = (size_t)lwork * sizeof(double2);
    w.work_bytes = dev_bytes;
    if (dev_malloc(&w.work, w.work_bytes + 16) != cudaSuccess ||
        dev_malloc(&w.A, (size_t)m * n * sizeof(double2)) != cudaSuccess ||
        dev_malloc(&w.U, (size_t)m * n * sizeof(double2)) != cudaSuccess ||
        dev_malloc(&w.VT, (size_t)n * n * sizeof(double2)) != cudaSuccess ||
        dev_malloc(&w.rwork, (size_t)n * sizeof(double)) != cudaSuccess ||
        dev_malloc(&w.info, sizeof(int)) != cudaSuccess) {
      *err = "svd: workspace allocation";
      return PS_ERR_CUDA;
    }
    w.m = m;
    w.n = n;
  }
  if (cudaMemcpyAsync(w.A, A, (size_t)m * n * sizeof(double2), cudaMemcpyDeviceToDevice, w.st) !=
      cudaSuccess) {
    *err = "svd: copy";
    return PS_ERR_CUDA;
  }
  const int lwork = (int)(w.work_bytes / sizeof(double2));
  cusolverStatus_t cs = cusolverDnZgesvd(
      w.h, 'S', 'S', m, n, reinterpret_cast<cuDoubleComplex*>(w.A), m, s,
      reinterpret_cast<cuDoubleComplex*>(w.U), m, reinterpret_cast<cuDoubleComplex*>(w.VT), n,
      reinterpret_cast<cuDoubleComplex*>(w.work), lwork, w.rwork, w.info);
  if (cs != CUSOLVER_STATUS_SUCCESS) {
    *err = svd_err("cusolverDnZgesvd", cs);
    return PS_ERR_CUDA;
  }
  int info = 0;
  cudaMemcpyAsync(&info, w.info, sizeof(int), cudaMemcpyDeviceToHost, w.st);
  if (cudaStreamSynchronize(w.st) != cudaSuccess) {
    *err = "svd: synchronize";
    return PS_ERR_CUDA;
  }
  if (info != 0) {
    *err = "zgesvd: info = " + std::to_string(info) + " (bidiagonal QR did not converge)";
    return PS_ERR_NUMERICAL;
  }
  return PS_OK;
}

}  // namespace

// per-context storage of the device-assembled systems
struct EmptyState {
  int m = 0, ncol = 0, nrhs = 0;
  double* d_curves = nullptr;        // all curves, kCS doubles per node
  double2* d_kv = nullptr;           // Alpert off-grid kernel values
  RhsPar* d_rp = nullptr;
  double2* d_A = nullptr;            // [nrhs][ncol][m] column-scaled, column-major
  double2* d_f = nullptr;            // [nrhs][m]
  double* d_cs = nullptr;            // [nrhs][ncol]
  double* d_s = nullptr;             // [nrhs][ncol] singular values
  double t_assemble_ms = 0, t_svd_ms = 0;
};

// Residual of the empty-grating rows of the coupled system (Eq.
// finalsys rows [A C][x; beta] = f; solve_empty's residual, eg:289-290):
// r_i = sum_j A_s[i][j] x_j / cs_j + g_i - f_i, g = C beta on its nrow_c
// rows (zero elsewhere).  Thread per row (A_s column-major: coalesced).
__global__ void empty_residual_kernel(const double2* __restrict__ A, const double2* __restrict__ f,
                                      const double* __restrict__ cs, const double2* __restrict__ x,
                                      const double2* __restrict__ g, int m, int ncol, int nrow_c,
                                      double2* __restrict__ res) {
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  const int r = blockIdx.y;
  if (i >= m) return;
  const double2* Ar = A + (size_t)r * m * ncol;
  const double2* xr = x + (size_t)r * ncol;
  const double* cr = cs + (size_t)r * ncol;
  double sx = 0.0, sy = 0.0;
  for (int j = 0; j < ncol; ++j) {
    const double2 a = Ar[(size_t)j * m + i];
    const double2 v = xr[j];
    const double ic = 1.0 / cr[j];
    sx = fma(a.x, v.x * ic, fma(-a.y, v.y * ic, sx));
    sy = fma(a.x, v.y * ic, fma(a.y, v.x * ic, sy));
  }
  const double2 fi = f[(size_t)r * m + i];
  if (g && i < nrow_c) {
    sx += g[(size_t)r * nrow_c + i].x;
    sy += g[(size_t)r * nrow_c + i].y;
  }
  res[(size_t)r * m + i] = make_double2(sx - fi.x, sy - fi.y);
}

// out[r] = (||res_r||^2, ||f_r||^2), one block per RHS, fixed order
__global__ void residual_norms(const double2* __restrict__ res, const double2* __restrict__ f,
                               int m, double* __restrict__ out) {
  __shared__ double sh[2][256];
  const int r = blockIdx.x;
  double a = 0.0, b = 0.0;
  for (int i = threadIdx.x; i < m; i += blockDim.x) {
    const double2 v = res[(size_t)r * m + i], w = f[(size_t)r * m + i];
    a = fma(v.x, v.x, fma(v.y, v.y, a));
    b = fma(w.x, w.x, fma(w.y, w.y, b));
  }
  sh[0][threadIdx.x] = a;
  sh[1][threadIdx.x] = b;
  __syncthreads();
  for (int o = blockDim.x / 2; o > 0; o >>= 1) {
    if ((int)threadIdx.x < o) {
      sh[0][threadIdx.x] += sh[0][threadIdx.x + o];
      sh[1][threadIdx.x] += sh[1][threadIdx.x + o];
    }
    __syncthreads();
  }
  if (threadIdx.x == 0) {
    out[2 * r] = sh[0][0];
    out[2 * r + 1] = sh[1][0];
  }
}

void empty_release(Ctx* c) {
  if (!c->empty) return;
  EmptyState* e = c->empty;
  void* ptrs[] = {e->d_curves, e->d_kv, e->d_rp, e->d_A, e->d_f, e->d_cs, e->d_s};
  for (void* p : ptrs)
    if (p) dev_free(p);
  delete e;
  c->empty = nullptr;
}

}  // namespace ps

using ps::Ctx;

namespace {

int fail(Ctx* c, int code, const std::string& msg) {
  c->err = msg;
  return code;
}

#define PS_TRY_CUDA(call)                                                           \
  do {                                                                              \
    cudaError_t e_ = (call);                                                        \
    if (e_ != cudaSuccess)                                                          \
      return fail(c, PS_ERR_CUDA, std::string(#call) + ": " + cudaGetErrorString(e_)); \
  } while (0)

template <typename T>
int upload(Ctx* c, T** dst, const T* src, size_t n) {
  if (*dst) ps::dev_free(*dst);
  *dst = nullptr;
  if (n == 0) return PS_OK;
  PS_TRY_CUDA(ps::dev_malloc(reinterpret_cast<void**>(dst), n * sizeof(T)));
  if (src) PS_TRY_CUDA(cudaMemcpy(*dst, src, n * sizeof(T), cudaMemcpyHostToDevice));
  return PS_OK;
}

}  // namespace

extern "C" {

int ps_setup_empty_range(ps_ctx* h, const ps_empty_desc* ds, const double* theta, int rb,
                         int re) {
  using namespace ps;
  if (!h) return PS_ERR_ARG;
  Ctx* c = ps::C(h);
  release_dense_coupling(c);
  if (!ds || !theta) return fail(c, PS_ERR_ARG, "ps_setup_empty: null argument");
  const ps_curve_desc* cvs[C_NCURVE] = {&ds->g1, &ds->g2, &ds->wall[0], &ds->wall[1],
                                        &ds->wall[2], &ds->lid_up, &ds->lid_down};
  for (auto* cv : cvs)
    if (cv->n <= 0 || !cv->data) return fail(c, PS_ERR_ARG, "ps_setup_empty: empty curve");
  if (!(ds->period > 0) || !(ds->k1 > 0) || !(ds->k2 > 0) || !(ds->k3 > 0) || ds->copies < 0 ||
      ds->Q < 0 || ds->nrb <= 0 || (ds->nrb % 2) == 0 || !(ds->eps > 0))
    return fail(c, PS_ERR_ARG, "ps_setup_empty: bad scalar parameter");
  if (ds->rule_n <= 0 || ds->rule_n > kMaxRule || ds->rule_interp <= 0 ||
      ds->rule_interp > kMaxRule || ds->rule_skip <= 0 || !ds->rule_x || !ds->rule_w)
    return fail(c, PS_ERR_ARG, "ps_setup_empty: bad correction rule");
  if (ds->g1.n < 4 * ds->rule_skip || ds->g2.n < 4 * ds->rule_skip)
    return fail(c, PS_ERR_ARG, "ps_setup_empty: need at least 4*skip interface nodes "
                               "(quadrature.py:127-128)");
  const ps_interface_desc* sp[2] = {&ds->top, &ds->bottom};
  for (auto* s : sp)
    if (s->nsin < 0 || s->ncos < 0 || s->nsin > kMaxCoef || s->ncos > kMaxCoef ||
        (s->nsin && !s->sin_coeffs) || (s->ncos && !s->cos_coeffs))
      return fail(c, PS_ERR_UNSUPPORTED, "ps_setup_empty: at most 8 sin/cos coefficients per interface");
  if (c->nrhs < 1 || (int)c->rhs.size() < c->nrhs)
    return fail(c, PS_ERR_STATE, "ps_setup_empty: call ps_set_rhs_bloch first");
  if (cudaSetDevice(c->device) != cudaSuccess) return fail(c, PS_ERR_CUDA, "cudaSetDevice");

  const int n1 = ds->g1.n, n2 = ds->g2.n;
  const int nw1 = ds->wall[0].n, nw2 = ds->wall[1].n, nw3 = ds->wall[2].n;
  const int nu = ds->lid_up.n, nd = ds->lid_down.n;
  const int nj = 2 * ds->Q + 1, nrb = ds->nrb;
  // column layout eg:154-156 and row layout eg:157-160
  const int c_mu1 = 0, c_s1 = n1, c_mu2 = 2 * n1, c_s2 = 2 * n1 + n2, c_a2 = 2 * n1 + 2 * n2;
  const int c_a1 = c_a2 + nj, c_a3 = c_a1 + nj, c_c = c_a3 + nj, c_d = c_c + nrb;
  const int ncol = c_d + nrb;
  const int r_g1 = 0, r_g2 = 2 * n1, r_w2 = 2 * n1 + 2 * n2, r_w1 = r_w2 + 2 * nw2;
  const int r_w3 = r_w1 + 2 * nw1, r_gu = r_w3 + 2 * nw3, r_gd = r_gu + 2 * nu;
  const int m = r_gd + 2 * nd;
  if (m < ncol) return fail(c, PS_ERR_ARG, "ps_setup_empty: fewer rows than unknowns");

  Tables tb{};
  tb.m = m;
  tb.ncol = ncol;
  tb.copies = ds->copies;
  tb.Q = ds->Q;
  tb.nrb = nrb;
  tb.period = ds->period;
  tb.y0 = ds->y0;
  tb.k1 = ds->k1;
  tb.k3 = ds->k3;
  tb.rule_n = ds->rule_n;
  tb.skip = ds->rule_skip;
  tb.interp = ds->rule_interp;
  for (int i = 0; i < ds->rule_n; ++i) {
    tb.rule_x[i] = ds->rule_x[i];
    tb.rule_w[i] = ds->rule_w[i];
    for (int side = 0; side < 2; ++side)
      lagrange((side == 0 ? 1.0 : -1.0) * ds->rule_x[i], ds->rule_interp, &tb.lag_start[side][i],
               tb.lag_w[side][i]);
  }
  psi_series(tb.psi);
  for (int s = 0; s < 2; ++s) {
    tb.spec[s].mean = sp[s]->mean;
    tb.spec[s].nsin = sp[s]->nsin;
    tb.spec[s].ncos = sp[s]->ncos;
    for (int j = 0; j < sp[s]->nsin; ++j) tb.spec[s].sc[j] = sp[s]->sin_coeffs[j];
    for (int j = 0; j < sp[s]->ncos; ++j) tb.spec[s].cc[j] = sp[s]->cos_coeffs[j];
  }
  // curves -> one device buffer
  if (!c->empty) c->empty = new EmptyState();
  EmptyState* e = c->empty;
  size_t tot = 0;
  for (auto* cv : cvs) tot += (size_t)cv->n * kCS;
  std::vector<double> hc(tot);
  {
    size_t o = 0;
    for (auto* cv : cvs) {
      std::copy(cv->data, cv->data + (size_t)cv->n * kCS, hc.begin() + o);
      o += (size_t)cv->n * kCS;
    }
  }
  if (int rc = upload(c, &e->d_curves, hc.data(), tot)) return rc;
  {
    size_t o = 0;
    for (int i = 0; i < C_NCURVE; ++i) {
      tb.curve[i] = e->d_curves + o;
      tb.ncurve[i] = cvs[i]->n;
      o += (size_t)cvs[i]->n * kCS;
    }
  }
  const double* ctr = ds->centers;   // centres 1, 2, 3
  auto add = [&](Task t) { tb.task[tb.ntask++] = t; };
  auto pair = [&](int kind, int src, int tgt, int rv, int rd, int ca, int cb, double k,
                  double ksub, double sign, int spec) {
    Task t{};
    t.kind = kind; t.src = src; t.tgt = tgt; t.row_v = rv; t.row_d = rd; t.col_a = ca;
    t.col_b = cb; t.nt = cvs[tgt]->n; t.ns = cvs[src]->n; t.k = k; t.ksub = ksub;
    t.sign = sign; t.spec = spec;
    add(t);
  };
  auto reg = [&](int kind, int tgt, int rv, int rd, int ca, double k, int cid, double sign) {
    Task t{};
    t.kind = kind; t.src = tgt; t.tgt = tgt; t.row_v = rv; t.row_d = rd; t.col_a = ca;
    t.nt = cvs[tgt]->n; t.ns = nj; t.k = k; t.sign = sign;
    t.cx = ctr[2 * (cid - 1)]; t.cy = ctr[2 * (cid - 1) + 1];
    add(t);
  };
  const double k1 = ds->k1, k2 = ds->k2, k3 = ds->k3;
  // interface continuity rows (eg:166-192); SELF tasks must stay at 0 and 2
  pair(K_SELF, C_G1, C_G1, r_g1, r_g1 + n1, c_mu1, c_s1, k1, k2, 1.0, 0);
  pair(K_CROSS, C_G2, C_G1, r_g1, r_g1 + n1, c_mu2, c_s2, k2, 0, -1.0, 0);
  pair(K_SELF, C_G2, C_G2, r_g2, r_g2 + n2, c_mu2, c_s2, k2, k3, 1.0, 1);
  pair(K_CROSS, C_G1, C_G2, r_g2, r_g2 + n2, c_mu1, c_s1, k2, 0, 1.0, 0);
  // regular-expansion traces (eg:194-202)
  reg(K_REG, C_G1, r_g1, r_g1 + n1, c_a2, k2, 2, -1.0);
  reg(K_REG, C_G1, r_g1, r_g1 + n1, c_a1, k1, 1, 1.0);
  reg(K_REG, C_G2, r_g2, r_g2 + n2, c_a2, k2, 2, 1.0);
  reg(K_REG, C_G2, r_g2, r_g2 + n2, c_a3, k3, 3, -1.0);
  // wall discrepancy rows (eg:204-224)
  pair(K_WALL, C_G1, C_L2, r_w2, r_w2 + nw2, c_mu1, c_s1, k2, 0, 1.0, 0);
  pair(K_WALL, C_G2, C_L2, r_w2, r_w2 + nw2, c_mu2, c_s2, k2, 0, 1.0, 0);
  reg(K_WALLREG, C_L2, r_w2, r_w2 + nw2, c_a2, k2, 2, 1.0);
  pair(K_WALL, C_G1, C_L1, r_w1, r_w1 + nw1, c_mu1, c_s1, k1, 0, 1.0, 0);
  reg(K_WALLREG, C_L1, r_w1, r_w1 + nw1, c_a1, k1, 1, 1.0);
  pair(K_WALL, C_G2, C_L3, r_w3, r_w3 + nw3, c_mu2, c_s2, k3, 0, 1.0, 0);
  reg(K_WALLREG, C_L3, r_w3, r_w3 + nw3, c_a3, k3, 3, 1.0);
  // artificial-boundary rows (eg:226-239)
  pair(K_CROSS, C_G1, C_GU, r_gu, r_gu + nu, c_mu1, c_s1, k1, 0, 1.0, 0);
  reg(K_REG, C_GU, r_gu, r_gu + nu, c_a1, k1, 1, 1.0);
  {
    Task t{};
    t.kind = K_RB; t.src = t.tgt = C_GU; t.row_v = r_gu; t.row_d = r_gu + nu; t.col_a = c_c;
    t.nt = nu; t.ns = nrb; t.up = 1;
    add(t);
  }
  pair(K_CROSS, C_G2, C_GD, r_gd, r_gd + nd, c_mu2, c_s2, k3, 0, 1.0, 0);
  reg(K_REG, C_GD, r_gd, r_gd + nd, c_a3, k3, 3, 1.0);
  {
    Task t{};
    t.kind = K_RB; t.src = t.tgt = C_GD; t.row_v = r_gd; t.row_d = r_gd + nd; t.col_a = c_d;
    t.nt = nd; t.ns = nrb; t.up = 0;
    add(t);
  }
  {
    Task t{};
    t.kind = K_INC; t.src = t.tgt = C_G1; t.row_v = r_g1; t.row_d = r_g1 + n1; t.nt = n1; t.ns = 1;
    add(t);
  }
  long long items = 0;
  for (int i = 0; i < tb.ntask; ++i) {
    tb.task[i].item0 = items;
    items += (long long)tb.task[i].nt * tb.task[i].ns;
  }
  tb.nitems = items;

  const int R = c->nrhs;
  std::vector<RhsPar> hp(R);
  for (int r = 0; r < R; ++r) {
    hp[r].ar = c->rhs[r].bloch.x;
    hp[r].ai = c->rhs[r].bloch.y;
    hp[r].kappa = ds->k1 * std::cos(theta[r]);
    hp[r].kix = ds->k1 * std::cos(theta[r]);
    hp[r].kiy = ds->k1 * std::sin(theta[r]);
  }
  if (int rc = upload(c, &e->d_rp, hp.data(), (size_t)R)) return rc;
  const size_t kv_n = (size_t)(n1 + n2) * 2 * ds->rule_n * 4;
  if (int rc = upload<double2>(c, &e->d_kv, nullptr, kv_n)) return rc;
  if (e->m != m || e->ncol != ncol || e->nrhs != R || !e->d_A) {
    if (int rc = upload<double2>(c, &e->d_A, nullptr, (size_t)R * m * ncol)) return rc;
    if (int rc = upload<double2>(c, &e->d_f, nullptr, (size_t)R * m)) return rc;
    if (int rc = upload<double>(c, &e->d_cs, nullptr, (size_t)R * ncol)) return rc;
    if (int rc = upload<double>(c, &e->d_s, nullptr, (size_t)R * ncol)) return rc;
    e->m = m;
    e->ncol = ncol;
    e->nrhs = R;
  }

  cudaEvent_t e0, e1, e2;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  cudaEventCreate(&e2);
  cudaStream_t st = 0;
  cudaEventRecord(e0, st);
  PS_TRY_CUDA(cudaMemsetAsync(e->d_A, 0, (size_t)R * m * ncol * sizeof(double2), st));
  PS_TRY_CUDA(cudaMemsetAsync(e->d_f, 0, (size_t)R * m * sizeof(double2), st));
  {
    const int tot_kv = (n1 + n2) * 2 * ds->rule_n;
    alpert_kv_kernel<<<(tot_kv + 127) / 128, 128, 0, st>>>(tb, e->d_kv);
    const int blocks = (int)std::min<long long>((items + 127) / 128, (long long)c->sm_count * 8);
    assemble_kernel<<<dim3(blocks, R), 128, 0, st>>>(tb, e->d_rp, e->d_kv, e->d_A, e->d_f);
    colscale_kernel<<<dim3(ncol, R), 256, 0, st>>>(e->d_A, e->d_cs, m, ncol, c_a2);
    c->launches += 3;
  }
  PS_TRY_CUDA(cudaGetLastError());
  cudaEventRecord(e1, st);
  PS_TRY_CUDA(cudaStreamSynchronize(st));

  // restricted factor layout of ps_set_pinv
  c->n1 = n1;
  c->n2 = n2;
  c->nw = nw2;
  c->Q = ds->Q;
  c->nrb = nrb;
  c->x2[0] = ctr[2];
  c->x2[1] = ctr[3];
  c->nrow_c = 2 * n1 + 2 * n2 + 2 * nw2;
  c->ncol_b = 2 * n1 + 2 * n2 + nj;
  {
    // coupling node records [n][5] (x, y, nx, ny, arc weight) and L2 wall nodes
    std::vector<double> g1(5 * (size_t)n1), g2(5 * (size_t)n2), w2(2 * (size_t)nw2);
    for (int i = 0; i < n1; ++i) {
      const double* q = ds->g1.data + (size_t)i * kCS;
      double v[5] = {q[0], q[1], q[2], q[3], q[7]};
      std::copy(v, v + 5, g1.begin() + 5 * (size_t)i);
    }
    for (int i = 0; i < n2; ++i) {
      const double* q = ds->g2.data + (size_t)i * kCS;
      double v[5] = {q[0], q[1], q[2], q[3], q[7]};
      std::copy(v, v + 5, g2.begin() + 5 * (size_t)i);
    }
    for (int i = 0; i < nw2; ++i) {
      w2[2 * i] = ds->wall[1].data[(size_t)i * kCS];
      w2[2 * i + 1] = ds->wall[1].data[(size_t)i * kCS + 1];
    }
    if (int rc = upload(c, &c->d_g1, g1.data(), g1.size())) return rc;
    if (int rc = upload(c, &c->d_g2, g2.data(), g2.size())) return rc;
    if (int rc = upload(c, &c->d_w2, w2.data(), w2.size())) return rc;
    c->have_layers = 1;
  }
  const int nsv = ncol, nrc = c->nrow_c;
  c->nsv = nsv;
  c->nfield = 2 * nj;                    // keep the a1 / a3 rows for field evaluation
  const int nout = c->ncol_b + 2 * nrb + c->nfield;
  // layer-field parameters (ps_layer_field)
  {
    std::vector<double> inc(2 * (size_t)R);
    for (int r = 0; r < R; ++r) {
      inc[2 * r] = ds->k1 * std::cos(theta[r]);
      inc[2 * r + 1] = ds->k1 * std::sin(theta[r]);
    }
    if (int rc = upload(c, &c->d_inc, inc.data(), inc.size())) return rc;
    c->f_k1 = ds->k1;
    c->f_k3 = ds->k3;
    c->f_c1[0] = ctr[0];
    c->f_c1[1] = ctr[1];
    c->f_c3[0] = ctr[4];
    c->f_c3[1] = ctr[5];
    c->have_field = 1;
  }
  for (int r = 0; r < R; ++r) {
    auto& Rd = c->rhs[r];
    if (int rc = upload<double2>(c, &Rd.d_Uh, nullptr, (size_t)nsv * nrc)) return rc;
    if (int rc = upload<double>(c, &Rd.d_sinv, nullptr, (size_t)nsv)) return rc;
    if (int rc = upload<double2>(c, &Rd.d_Vb, nullptr, (size_t)nout * nsv)) return rc;
    if (int rc = upload<double>(c, &Rd.d_cscale, nullptr, (size_t)nout)) return rc;
    if (int rc = upload<double2>(c, &Rd.d_f, nullptr, (size_t)nrc)) return rc;
  }

  // SVD per right-hand side, up to c->svd_workers concurrent cuSOLVER streams
  const int dev = c->device;
  if (rb < 0 || re > R || rb > re) return fail(c, PS_ERR_ARG, "ps_setup_empty: bad RHS range");
  const int nown = re - rb;
  const int nwk = std::max(1, std::min(std::max(nown, 1), c->svd_workers));
  std::vector<int> rcs(nwk, PS_OK);
  std::vector<std::string> errs(nwk);
  std::lock_guard<std::mutex> dev_lock(g_dev_mu[dev & 63]);
  {
    std::lock_guard<std::mutex> lk(g_svd_mu);
    if ((int)g_svd[dev].size() < nwk) g_svd[dev].resize(nwk);
  }
  auto work = [&](int wid) {
    cudaSetDevice(dev);
    SvdWorker& w = g_svd[dev][wid];
    for (int r = rb + wid; r < re; r += nwk) {
      int rc = svd_run(w, e->d_A + (size_t)r * m * ncol, m, ncol, e->d_s + (size_t)r * ncol,
                       &errs[wid]);
      if (rc) {
        rcs[wid] = rc;
        return;
      }
      auto& Rd = c->rhs[r];
      const long long totx = (long long)nsv * nrc + (long long)nout * nsv + nsv + nout + nrc;
      pinv_extract_kernel<<<(int)std::min<long long>((totx + 255) / 256, 4096), 256, 0, w.st>>>(
          w.U, e->d_s + (size_t)r * ncol, w.VT, e->d_cs + (size_t)r * ncol,
          e->d_f + (size_t)r * m, m, ncol, nrc, c->ncol_b, nrb, c_c, c_d, c->nfield, ds->eps, Rd.d_Uh,
          Rd.d_sinv, Rd.d_Vb, Rd.d_cscale, Rd.d_f);
      if (cudaStreamSynchronize(w.st) != cudaSuccess || cudaGetLastError() != cudaSuccess) {
        rcs[wid] = PS_ERR_CUDA;
        errs[wid] = "pinv_extract_kernel failed";
        return;
      }
    }
  };
  if (nwk == 1) {
    work(0);
  } else {
    std::vector<std::thread> th;
    for (int w = 0; w < nwk; ++w) th.emplace_back(work, w);
    for (auto& t : th) t.join();
  }
  c->launches += nown;
  cudaEventRecord(e2, st);
  cudaEventSynchronize(e2);
  float ms_a = 0, ms_s = 0;
  cudaEventElapsedTime(&ms_a, e0, e1);
  cudaEventElapsedTime(&ms_s, e1, e2);
  e->t_assemble_ms = ms_a;
  e->t_svd_ms = ms_s;
  cudaEventDestroy(e0);
  cudaEventDestroy(e1);
  cudaEventDestroy(e2);
  for (int w = 0; w < nwk; ++w)
    if (rcs[w]) return fail(c, rcs[w], "ps_setup_empty: " + errs[w]);
  return PS_OK;
}

int ps_setup_empty(ps_ctx* h, const ps_empty_desc* ds, const double* theta) {
  if (!h) return PS_ERR_ARG;
  return ps_setup_empty_range(h, ds, theta, 0, ps::C(h)->nrhs);
}

// packed restricted factors of one RHS: Uh | sinv | Vb | cscale | f
static size_t pinv_bytes(const Ctx* c) {
  const size_t nsv = c->nsv, nrc = c->nrow_c, nout = c->ncol_b + 2 * c->nrb + c->nfield;
  return nsv * nrc * 16 + nsv * 8 + nout * nsv * 16 + nout * 8 + nrc * 16;
}

long long ps_pinv_bytes(const ps_ctx* h) {
  if (!h) return -1;
  const Ctx* c = reinterpret_cast<const Ctx*>(h);
  return c->have_layers && c->nsv > 0 ? (long long)pinv_bytes(c) : -1;
}

static int pinv_copy(ps_ctx* h, int irhs, void* dev, void* stream, bool out) {
  if (!h) return PS_ERR_ARG;
  Ctx* c = ps::C(h);
  if (!dev || irhs < 0 || irhs >= c->nrhs) return fail(c, PS_ERR_ARG, "ps_*_pinv: bad argument");
  auto& R = c->rhs[irhs];
  if (!c->have_layers || c->nsv <= 0 || !R.d_Uh)
    return fail(c, PS_ERR_STATE, "ps_*_pinv: no factors allocated (call ps_setup_empty first)");
  if (cudaSetDevice(c->device) != cudaSuccess) return fail(c, PS_ERR_CUDA, "cudaSetDevice");
  const size_t nsv = c->nsv, nrc = c->nrow_c, nout = c->ncol_b + 2 * c->nrb + c->nfield;
  void* parts[5] = {R.d_Uh, R.d_sinv, R.d_Vb, R.d_cscale, R.d_f};
  const size_t sz[5] = {nsv * nrc * 16, nsv * 8, nout * nsv * 16, nout * 8, nrc * 16};
  auto st = reinterpret_cast<cudaStream_t>(stream);
  char* p = reinterpret_cast<char*>(dev);
  for (int i = 0; i < 5; ++i) {
    const cudaError_t e = out ? cudaMemcpyAsync(p, parts[i], sz[i], cudaMemcpyDeviceToDevice, st)
                              : cudaMemcpyAsync(parts[i], p, sz[i], cudaMemcpyDeviceToDevice, st);
    if (e != cudaSuccess) return fail(c, PS_ERR_CUDA, "ps_*_pinv: copy");
    p += sz[i];
  }
  return PS_OK;
}

int ps_export_pinv(ps_ctx* h, int irhs, void* dst_dev, void* stream) {
  return pinv_copy(h, irhs, dst_dev, stream, true);
}

int ps_import_pinv(ps_ctx* h, int irhs, const void* src_dev, void* stream) {
  return pinv_copy(h, irhs, const_cast<void*>(src_dev), stream, false);
}

int ps_empty_shape(const ps_ctx* h, int* nrow, int* ncol) {
  if (!h || !nrow || !ncol) return PS_ERR_ARG;
  const Ctx* c = reinterpret_cast<const Ctx*>(h);
  if (!c->empty) return PS_ERR_STATE;
  *nrow = c->empty->m;
  *ncol = c->empty->ncol;
  return PS_OK;
}

int ps_get_empty(ps_ctx* h, int irhs, double* A, double* f, double* col_scale, double* s) {
  if (!h) return PS_ERR_ARG;
  Ctx* c = ps::C(h);
  ps::EmptyState* e = c->empty;
  if (!e) return fail(c, PS_ERR_STATE, "ps_get_empty: call ps_setup_empty first");
  if (irhs < 0 || irhs >= e->nrhs) return fail(c, PS_ERR_ARG, "ps_get_empty: bad rhs index");
  if (cudaSetDevice(c->device) != cudaSuccess) return fail(c, PS_ERR_CUDA, "cudaSetDevice");
  const int m = e->m, n = e->ncol;
  if (A) {
    std::vector<double2> cm((size_t)m * n);
    PS_TRY_CUDA(cudaMemcpy(cm.data(), e->d_A + (size_t)irhs * m * n, cm.size() * sizeof(double2),
                           cudaMemcpyDeviceToHost));
    for (int j = 0; j < n; ++j)
      for (int i = 0; i < m; ++i) {
        A[2 * ((size_t)i * n + j)] = cm[(size_t)j * m + i].x;
        A[2 * ((size_t)i * n + j) + 1] = cm[(size_t)j * m + i].y;
      }
  }
  if (f)
    PS_TRY_CUDA(cudaMemcpy(f, e->d_f + (size_t)irhs * m, (size_t)m * sizeof(double2),
                           cudaMemcpyDeviceToHost));
  if (col_scale)
    PS_TRY_CUDA(cudaMemcpy(col_scale, e->d_cs + (size_t)irhs * n, (size_t)n * sizeof(double),
                           cudaMemcpyDeviceToHost));
  if (s)
    PS_TRY_CUDA(cudaMemcpy(s, e->d_s + (size_t)irhs * n, (size_t)n * sizeof(double),
                           cudaMemcpyDeviceToHost));
  return PS_OK;
}

int ps_set_empty_system(ps_ctx* h, int irhs, int m, int ncol, const double* A, const double* f,
                        const double* col_scale) {
  if (!h) return PS_ERR_ARG;
  Ctx* c = ps::C(h);
  if (irhs < 0 || irhs >= c->nrhs || m <= 0 || ncol <= 0 || !A || !f || !col_scale)
    return fail(c, PS_ERR_ARG, "ps_set_empty_system: bad argument");
  if (cudaSetDevice(c->device) != cudaSuccess) return fail(c, PS_ERR_CUDA, "cudaSetDevice");
  ps::EmptyState* e = c->empty;
  if (e && (e->m != m || e->ncol != ncol || e->nrhs != c->nrhs)) {
    ps::empty_release(c);
    e = nullptr;
  }
  if (!e) {
    e = c->empty = new ps::EmptyState();
    e->m = m;
    e->ncol = ncol;
    e->nrhs = c->nrhs;
    const size_t R = (size_t)c->nrhs;
    PS_TRY_CUDA(ps::dev_malloc(&e->d_A, R * m * ncol * sizeof(double2)));
    PS_TRY_CUDA(ps::dev_malloc(&e->d_f, R * m * sizeof(double2)));
    PS_TRY_CUDA(ps::dev_malloc(&e->d_cs, R * ncol * sizeof(double)));
    PS_TRY_CUDA(ps::dev_malloc(&e->d_s, R * ncol * sizeof(double)));
    PS_TRY_CUDA(cudaMemset(e->d_s, 0, R * ncol * sizeof(double)));
  }
  std::vector<double2> cm((size_t)m * ncol);       // row-major host -> column-major device
  for (int i = 0; i < m; ++i)
    for (int j = 0; j < ncol; ++j)
      cm[(size_t)j * m + i] = make_double2(A[2 * ((size_t)i * ncol + j)],
                                           A[2 * ((size_t)i * ncol + j) + 1]);
  PS_TRY_CUDA(cudaMemcpy(e->d_A + (size_t)irhs * m * ncol, cm.data(), cm.size() * sizeof(double2),
                         cudaMemcpyHostToDevice));
  PS_TRY_CUDA(cudaMemcpy(e->d_f + (size_t)irhs * m, f, (size_t)m * sizeof(double2),
                         cudaMemcpyHostToDevice));
  PS_TRY_CUDA(cudaMemcpy(e->d_cs + (size_t)irhs * ncol, col_scale, (size_t)ncol * sizeof(double),
                         cudaMemcpyHostToDevice));
  return PS_OK;
}

int ps_empty_residual(ps_ctx* h, const void* x, const void* g, double* out, void* stream) {
  if (!h) return PS_ERR_ARG;
  Ctx* c = ps::C(h);
  ps::EmptyState* e = c->empty;
  if (!e || !e->d_A) return fail(c, PS_ERR_STATE, "ps_empty_residual: no empty-grating matrix "
                                                   "(ps_setup_empty or ps_set_empty_system)");
  if (!x || !out) return fail(c, PS_ERR_ARG, "ps_empty_residual: null pointer");
  if (cudaSetDevice(c->device) != cudaSuccess) return fail(c, PS_ERR_CUDA, "cudaSetDevice");
  cudaStream_t st = reinterpret_cast<cudaStream_t>(stream);
  double2* res = nullptr;
  PS_TRY_CUDA(ps::dev_malloc(&res, (size_t)e->nrhs * e->m * sizeof(double2)));
  ps::empty_residual_kernel<<<dim3((e->m + 127) / 128, e->nrhs), 128, 0, st>>>(
      e->d_A, e->d_f, e->d_cs, reinterpret_cast<const double2*>(x),
      reinterpret_cast<const double2*>(g), e->m, e->ncol, c->nrow_c, res);
  ps::residual_norms<<<e->nrhs, 256, 0, st>>>(res, e->d_f, e->m, out);
  c->launches += 2;
  const cudaError_t err = cudaGetLastError();
  cudaStreamSynchronize(st);
  ps::dev_free(res);
  if (err != cudaSuccess) return fail(c, PS_ERR_CUDA, std::string("ps_empty_residual: ") +
                                                        cudaGetErrorString(err));
  return PS_OK;
}

int ps_set_svd_workers(ps_ctx* h, int workers) {
  if (!h) return PS_ERR_ARG;
  Ctx* c = ps::C(h);
  if (workers < 1 || workers > 32) return fail(c, PS_ERR_ARG, "ps_set_svd_workers: 1..32");
  c->svd_workers = workers;
  return PS_OK;
}

int ps_setup_timings(const ps_ctx* h, double* assemble_ms, double* svd_ms) {
  if (!h || !assemble_ms || !svd_ms) return PS_ERR_ARG;
  const Ctx* c = reinterpret_cast<const Ctx*>(h);
  if (!c->empty) return PS_ERR_STATE;
  *assemble_ms = c->empty->t_assemble_ms;
  *svd_ms = c->empty->t_svd_ms;
  return PS_OK;
}

}  // extern "C"
