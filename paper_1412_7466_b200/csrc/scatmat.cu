// Single-inclusion scattering matrix of a star-shaped particle from the
// Mueller boundary integral equations, on the device.
//
// Replaces scatmat.solve_muller_particle + scatmat.scattering_matrix
// (Eqs. intg1-intg2 and the s_ln
// projection), built from the reference's own Nystrom machinery restated in
// nystrom.cuh: the closed-curve self matrices of the two-wavenumber
// difference kernels with Alpert corrections (quadrature.nystrom_selfmatrix,
// quadrature.py:106-186, closure "closed", no copies) and the particle
// parametrisation of geometry.sample_particle (geometry.py:224-256).
//
//   [ I + D^{k2}-D^{kp}     S^{k2}-S^{kp}     ] [mu   ]     [ J_n e^{in th}        ]
//   [ T^{k2}-T^{kp}        -I + N^{k2}-N^{kp} ] [sigma] = - [ d/dn (J_n e^{in th}) ]
//
// for the 2p+1 incident regular waves n = -p..p (one LU, 2p+1 right-hand
// sides, Gauss-Jordan with partial pivoting on the device), then
//   s_ln = (i/4) sum_y w_y [ J_l(k2|y|) e^{-il th_y} sigma_n(y)
//                            + n_y . grad(J_l(k2|y|) e^{-il th_y}) mu_n(y) ]
// (Graf's theorem on S^{k2} sigma + D^{k2} mu; the i/4 is the Green's
// function prefactor, which the analytic disk fixes -- SPEC.md:441's open
// question).
#include <cuda_runtime.h>

#include <algorithm>
#include <cmath>
#include <mutex>
#include <string>
#include <vector>

#include "ctx.cuh"
#include "nystrom.cuh"

namespace ps {
namespace {

using namespace nys;

struct Star {   // r(t) = a1 + a2 cos(a3 t), centre 0, rotation 0
  double a1, a2, a3;
};

struct SmParams {
  const double* curve;   // [n][kCS]
  int n, L, p;
  double k2, kp, h;
  Star sh;
  int rule_n, skip, interp;
  double rule_x[kMaxRule], rule_w[kMaxRule];
  int lag_start[2][kMaxRule];
  double lag_w[2][kMaxRule][kMaxRule];
  double psi[kPsiTerms];
};

// geometry.sample_particle evaluate(tau) (geometry.py:233-241)
__device__ void star_eval(const Star& s, double tau, double* speed, double* nx, double* ny) {
  const double rho = s.a1 + s.a2 * cos(s.a3 * tau);
  const double drho = -s.a2 * s.a3 * sin(s.a3 * tau);
  const double ct = cos(tau), st = sin(tau);
  const double tx = drho * ct - rho * st, ty = drho * st + rho * ct;
  const double sp = hypot(tx, ty);
  *speed = sp;
  *nx = ty / sp;
  *ny = -tx / sp;
}

// x(s) - x(tau) without cancellation (geometry.py:243-252)
__device__ void star_diff(const Star& sh, double s, double tau, double* u0, double* u1) {
  const double rho_s = sh.a1 + sh.a2 * cos(sh.a3 * s);
  const double drho = -2.0 * sh.a2 * sin(0.5 * sh.a3 * (s + tau)) * sin(0.5 * sh.a3 * (s - tau));
  const double hs = 0.5 * (s + tau), hd = 0.5 * (s - tau);
  const double dcos = -2.0 * sin(hs) * sin(hd);
  const double dsin = 2.0 * cos(hs) * sin(hd);
  *u0 = rho_s * dcos + drho * cos(tau);
  *u1 = rho_s * dsin + drho * sin(tau);
}

// kernel differences at the Alpert off-grid nodes of every row:
// kv[i][side * rule_n + m] = {D, S, T, N}(k2) - (kp) * speed(tau) w_m h
__global__ void sm_kv_kernel(SmParams P, double2* kv) {
  const int tot = P.n * 2 * P.rule_n;
  for (int id = blockIdx.x * blockDim.x + threadIdx.x; id < tot; id += gridDim.x * blockDim.x) {
    const int i = id / (2 * P.rule_n), sm = id % (2 * P.rule_n);
    const int side = sm / P.rule_n, m = sm % P.rule_n;
    const double ti = P.curve[i * kCS + 6];
    const double tau = ti + (side == 0 ? 1.0 : -1.0) * P.rule_x[m] * P.h;
    double sp, nx, ny, u0, u1;
    star_eval(P.sh, tau, &sp, &nx, &ny);
    star_diff(P.sh, ti, tau, &u0, &u1);
    const double tnx = P.curve[i * kCS + 2], tny = P.curve[i * kCS + 3];
    const K4 a = kernel4(P.k2, u0, u1, tnx, tny, nx, ny);
    const K4 b = kernel4(P.kp, u0, u1, tnx, tny, nx, ny);
    const double2 T = t_difference(P.psi, P.k2, P.kp, u0, u1, tnx, tny, nx, ny);
    const double w = sp * (P.rule_w[m] * P.h);
    double2* o = kv + (size_t)id * 4;
    o[0] = cscale(csub(a.D, b.D), w);
    o[1] = cscale(csub(a.S, b.S), w);
    o[2] = cscale(T, w);
    o[3] = cscale(csub(a.N, b.N), w);
  }
}

// Mueller system (2n x 2n, column-major) -- one (i, j) node pair per item
__global__ void sm_system_kernel(SmParams P, const double2* __restrict__ kv, double2* A) {
  const int n = P.n, m2 = 2 * n;
  for (int id = blockIdx.x * blockDim.x + threadIdx.x; id < n * n; id += gridDim.x * blockDim.x) {
    const int i = id % n, j = id / n;
    const double* ti = P.curve + (size_t)i * kCS;
    const double* sj = P.curve + (size_t)j * kCS;
    double2 D = c2(0, 0), S = D, T = D, N = D;
    int om = j - i;
    if (om < 0) om += n;
    if (min(om, n - om) > P.skip - 1) {   // toroidal band of the closed curve
      const double u0 = ti[0] - sj[0], u1 = ti[1] - sj[1];
      const K4 a = kernel4(P.k2, u0, u1, ti[2], ti[3], sj[2], sj[3]);
      const K4 b = kernel4(P.kp, u0, u1, ti[2], ti[3], sj[2], sj[3]);
      const double2 Td = t_difference(P.psi, P.k2, P.kp, u0, u1, ti[2], ti[3], sj[2], sj[3]);
      const double w = sj[4] * P.h;
      D = cscale(csub(a.D, b.D), w);
      S = cscale(csub(a.S, b.S), w);
      T = cscale(Td, w);
      N = cscale(csub(a.N, b.N), w);
    }
    const double2* kr = kv + (size_t)i * 2 * P.rule_n * 4;
    for (int side = 0; side < 2; ++side)
      for (int mm = 0; mm < P.rule_n; ++mm) {
        int rr = (j - i - P.lag_start[side][mm]) % n;
        if (rr < 0) rr += n;
        if (rr >= P.interp) continue;
        const double lw = P.lag_w[side][mm][rr];
        const double2* q = kr + (size_t)(side * P.rule_n + mm) * 4;
        D = cadd(D, cscale(q[0], lw));
        S = cadd(S, cscale(q[1], lw));
        T = cadd(T, cscale(q[2], lw));
        N = cadd(N, cscale(q[3], lw));
      }
    if (i == j) {
      D.x += 1.0;
      N.x -= 1.0;
    }
    A[(size_t)j * m2 + i] = D;
    A[(size_t)(n + j) * m2 + i] = S;
    A[(size_t)j * m2 + n + i] = T;
    A[(size_t)(n + j) * m2 + n + i] = N;
  }
}

// incident regular waves (right-hand sides, column-major [L][2n]) and the
// projection rows Pr[l][2n] = (i/4) w conj(d/dn wave_l | wave_l)
__global__ void sm_waves_kernel(SmParams P, double2* B, double2* Pr) {
  const int n = P.n, m2 = 2 * n;
  for (int id = blockIdx.x * blockDim.x + threadIdx.x; id < n * P.L;
       id += gridDim.x * blockDim.x) {
    const int i = id % n, o = id / n;
    const double* y = P.curve + (size_t)i * kCS;
    double2 v, gx, gy;
    regular_wave(P.k2, 0.0, 0.0, o - P.p, P.p, y[0], y[1], &v, &gx, &gy);
    const double2 dn = cadd(cscale(gx, y[2]), cscale(gy, y[3]));
    B[(size_t)o * m2 + i] = cscale(v, -1.0);
    B[(size_t)o * m2 + n + i] = cscale(dn, -1.0);
    const double w = 0.25 * y[7];
    Pr[(size_t)o * m2 + i] = cmuli(cscale(c2(dn.x, -dn.y), w));       // mu column
    Pr[(size_t)o * m2 + n + i] = cmuli(cscale(c2(v.x, -v.y), w));     // sigma column
  }
}

// S[l][k] = sum_r Pr[l][r] X[r][k]  (X column-major [L][2n]); and the
// residual rows R = A0 X - B  (A0: the unfactored system)
__global__ void sm_project_kernel(const double2* __restrict__ Pr, const double2* __restrict__ X,
                                  int m2, int L, double2* S) {
  for (int id = blockIdx.x * blockDim.x + threadIdx.x; id < L * L; id += gridDim.x * blockDim.x) {
    const int l = id / L, k = id % L;
    double2 acc = c2(0, 0);
    for (int r = 0; r < m2; ++r) acc = cadd(acc, cmul(Pr[(size_t)l * m2 + r], X[(size_t)k * m2 + r]));
    S[id] = acc;
  }
}

__global__ void sm_residual_kernel(const double2* __restrict__ A0, const double2* __restrict__ X,
                                   const double2* __restrict__ B, int m2, int L, double* out) {
  // out[0] += |A0 X - B|^2, out[1] += |B|^2 (one thread per (row, rhs); atomics
  // only feed a diagnostic)
  for (int id = blockIdx.x * blockDim.x + threadIdx.x; id < m2 * L; id += gridDim.x * blockDim.x) {
    const int row = id % m2, k = id / m2;
    double2 acc = c2(0, 0);
    for (int j = 0; j < m2; ++j) acc = cadd(acc, cmul(A0[(size_t)j * m2 + row], X[(size_t)k * m2 + j]));
    const double2 b = B[(size_t)k * m2 + row];
    const double2 r = csub(acc, b);
    atomicAdd(out, r.x * r.x + r.y * r.y);
    atomicAdd(out + 1, b.x * b.x + b.y * b.y);
  }
}

// Gauss-Jordan elimination with partial pivoting on [A | X] (column-major,
// m2 rows, m2 + L columns; X starts as B), pivots recorded by row instead of
// swapping.  The Mueller system is a second-kind equation (condition ~1e2), so
// GJ is as accurate as LU here; it keeps this setup free of cuBLAS-backed
// solvers.  Step k: pick the unused row r with max |A[r][k]| (one CTA), then
// every other row i: A[i][j] -= (A[i][k] / A[r][k]) A[r][j] for j > k and
// all X columns (column k itself is never read again).
__global__ void gj_pivot_kernel(const double2* __restrict__ A, int m2, int k, int* used,
                                int* prow) {
  __shared__ double bv[1024];
  __shared__ int bi[1024];
  double best = -1.0;
  int arg = -1;
  for (int i = threadIdx.x; i < m2; i += blockDim.x) {
    if (used[i]) continue;
    const double2 a = A[(size_t)k * m2 + i];
    const double v = a.x * a.x + a.y * a.y;
    if (v > best) {
      best = v;
      arg = i;
    }
  }
  bv[threadIdx.x] = best;
  bi[threadIdx.x] = arg;
  __syncthreads();
  for (int s = blockDim.x / 2; s > 0; s >>= 1) {
    if (threadIdx.x < s) {
      const double o = bv[threadIdx.x + s];
      const int oi = bi[threadIdx.x + s];
      if (o > bv[threadIdx.x] || (o == bv[threadIdx.x] && oi >= 0 && oi < bi[threadIdx.x])) {
        bv[threadIdx.x] = o;
        bi[threadIdx.x] = oi;
      }
    }
    __syncthreads();
  }
  if (threadIdx.x == 0) {
    prow[k] = bi[0];
    used[bi[0]] = 1;
  }
}

__global__ void gj_eliminate_kernel(double2* __restrict__ A, double2* __restrict__ X, int m2,
                                    int L, int k, const int* __restrict__ prow) {
  const int r = prow[k];
  const int ncols = (m2 - k - 1) + L;
  const double2 piv = A[(size_t)k * m2 + r];
  const double d = piv.x * piv.x + piv.y * piv.y;
  const double2 pinv = c2(piv.x / d, -piv.y / d);
  for (long long id = (long long)blockIdx.x * blockDim.x + threadIdx.x; id < (long long)m2 * ncols;
       id += (long long)gridDim.x * blockDim.x) {
    const int i = (int)(id % m2), jc = (int)(id / m2);
    if (i == r) continue;
    const double2 f = cmul(A[(size_t)k * m2 + i], pinv);
    double2* col = jc < m2 - k - 1 ? A + (size_t)(k + 1 + jc) * m2 : X + (size_t)(jc - (m2 - k - 1)) * m2;
    col[i] = csub(col[i], cmul(f, col[r]));
  }
}

// x_k = X[r_k] / A[r_k][k] into Y (column-major [L][m2])
__global__ void gj_finish_kernel(const double2* __restrict__ A, const double2* __restrict__ X,
                                 int m2, int L, const int* __restrict__ prow, double2* Y) {
  for (int id = blockIdx.x * blockDim.x + threadIdx.x; id < m2 * L; id += gridDim.x * blockDim.x) {
    const int k = id % m2, c = id / m2;
    const int r = prow[k];
    const double2 piv = A[(size_t)k * m2 + r];
    const double d = piv.x * piv.x + piv.y * piv.y;
    Y[(size_t)c * m2 + k] = cmul(X[(size_t)c * m2 + r], c2(piv.x / d, -piv.y / d));
  }
}


}  // namespace
}  // namespace ps

using ps::Ctx;

extern "C" int ps_scattering_matrix(ps_ctx* h, const ps_particle_desc* ds, int p, double* S_host,
                                    double* residual) {
  using namespace ps;
  using namespace ps::nys;
  if (!h) return PS_ERR_ARG;
  Ctx* c = ps::C(h);
  auto fail = [&](int code, const std::string& m) {
    c->err = "ps_scattering_matrix: " + m;
    return code;
  };
  if (!ds || !S_host || !ds->curve) return fail(PS_ERR_ARG, "null argument");
  if (p < 0 || ds->n < 64 || !(ds->k2 > 0) || !(ds->kp > 0) || ds->lobes < 0 ||
      !(ds->base_radius > 0) || ds->bump_amplitude < 0 || ds->bump_amplitude >= ds->base_radius)
    return fail(PS_ERR_ARG, "bad shape / order (geometry.py:99-113, n >= 64)");
  if (ds->rule_n <= 0 || ds->rule_n > kMaxRule || ds->rule_interp <= 0 ||
      ds->rule_interp > kMaxRule || ds->rule_skip <= 0 || !ds->rule_x || !ds->rule_w ||
      ds->n < 4 * ds->rule_skip)
    return fail(PS_ERR_ARG, "bad correction rule");
  if (cudaSetDevice(c->device) != cudaSuccess) return fail(PS_ERR_CUDA, "cudaSetDevice");
  const int n = ds->n, m2 = 2 * n, L = 2 * p + 1;
  SmParams P{};
  P.n = n;
  P.L = L;
  P.p = p;
  P.k2 = ds->k2;
  P.kp = ds->kp;
  P.h = 2.0 * kPi / n;
  P.sh = Star{ds->base_radius, ds->bump_amplitude, (double)ds->lobes};
  P.rule_n = ds->rule_n;
  P.skip = ds->rule_skip;
  P.interp = ds->rule_interp;
  for (int i = 0; i < ds->rule_n; ++i) {
    P.rule_x[i] = ds->rule_x[i];
    P.rule_w[i] = ds->rule_w[i];
    for (int side = 0; side < 2; ++side)
      lagrange((side == 0 ? 1.0 : -1.0) * ds->rule_x[i], ds->rule_interp, &P.lag_start[side][i],
               P.lag_w[side][i]);
  }
  psi_series(P.psi);

  // one allocation: curve | kv | A | A0 | B | X | Y | Pr | S | sums | pivots
  const size_t nc = (size_t)n * kCS, nkv = (size_t)n * 2 * ds->rule_n * 4;
  const size_t nA = (size_t)m2 * m2, nB = (size_t)m2 * L;
  const size_t bytes = nc * 8 + (nkv + 2 * nA + 4 * nB + (size_t)L * L) * 16 + 16 +
                       (size_t)2 * m2 * sizeof(int);
  char* buf = nullptr;
  if (dev_malloc(&buf, bytes) != cudaSuccess) return fail(PS_ERR_CUDA, "allocation");
  double* d_curve = reinterpret_cast<double*>(buf);
  double2* d_kv = reinterpret_cast<double2*>(buf + nc * 8);
  double2* d_A = d_kv + nkv;
  double2* d_A0 = d_A + nA;
  double2* d_B = d_A0 + nA;
  double2* d_X = d_B + nB;
  double2* d_Y = d_X + nB;
  double2* d_Pr = d_Y + nB;   // [L][2n]
  double2* d_S = d_Pr + nB;
  double* d_sums = reinterpret_cast<double*>(d_S + (size_t)L * L);
  int* d_used = reinterpret_cast<int*>(d_sums + 2);
  int* d_prow = d_used + m2;
  int rc = PS_OK;
  std::vector<double2> hS((size_t)L * L);
  double sums[2] = {0, 0};
  do {
    if (cudaMemcpy(d_curve, ds->curve, nc * 8, cudaMemcpyHostToDevice) != cudaSuccess) {
      rc = fail(PS_ERR_CUDA, "upload");
      break;
    }
    P.curve = d_curve;
    const int tot_kv = n * 2 * ds->rule_n;
    sm_kv_kernel<<<(tot_kv + 127) / 128, 128>>>(P, d_kv);
    sm_system_kernel<<<(n * n + 127) / 128, 128>>>(P, d_kv, d_A);
    sm_waves_kernel<<<(n * L + 127) / 128, 128>>>(P, d_B, d_Pr);
    c->launches += 3;
    cudaMemcpyAsync(d_A0, d_A, nA * 16, cudaMemcpyDeviceToDevice, 0);
    cudaMemcpyAsync(d_X, d_B, nB * 16, cudaMemcpyDeviceToDevice, 0);
    if (cudaGetLastError() != cudaSuccess) {
      rc = fail(PS_ERR_CUDA, "assembly launch");
      break;
    }
    cudaMemsetAsync(d_used, 0, (size_t)m2 * sizeof(int), 0);
    for (int k = 0; k < m2; ++k) {
      gj_pivot_kernel<<<1, 1024>>>(d_A, m2, k, d_used, d_prow);
      const long long work = (long long)m2 * ((m2 - k - 1) + L);
      const int blocks = (int)std::min<long long>((work + 255) / 256, (long long)c->sm_count * 8);
      gj_eliminate_kernel<<<blocks, 256>>>(d_A, d_X, m2, L, k, d_prow);
    }
    gj_finish_kernel<<<(m2 * L + 255) / 256, 256>>>(d_A, d_X, m2, L, d_prow, d_Y);
    c->launches += 2 * m2 + 1;
    if (cudaGetLastError() != cudaSuccess) {
      rc = fail(PS_ERR_CUDA, "Gauss-Jordan launch");
      break;
    }
    sm_project_kernel<<<(L * L + 127) / 128, 128>>>(d_Pr, d_Y, m2, L, d_S);
    cudaMemsetAsync(d_sums, 0, 16, 0);
    sm_residual_kernel<<<(m2 * L + 255) / 256, 256>>>(d_A0, d_Y, d_B, m2, L, d_sums);
    c->launches += 2;
    if (cudaMemcpy(hS.data(), d_S, hS.size() * 16, cudaMemcpyDeviceToHost) != cudaSuccess ||
        cudaMemcpy(sums, d_sums, 16, cudaMemcpyDeviceToHost) != cudaSuccess) {
      rc = fail(PS_ERR_CUDA, "download");
      break;
    }
  } while (0);
  dev_free(buf);
  if (rc) return rc;
  for (size_t i = 0; i < hS.size(); ++i) {
    if (!std::isfinite(hS[i].x) || !std::isfinite(hS[i].y))
      return fail(PS_ERR_NUMERICAL, "non-finite scattering matrix entry");
    S_host[2 * i] = hS[i].x;
    S_host[2 * i + 1] = hS[i].y;
  }
  if (residual) *residual = sums[1] > 0 ? std::sqrt(sums[0] / sums[1]) : 0.0;
  return PS_OK;
}
