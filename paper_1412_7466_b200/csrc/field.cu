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

}  // namespace ps
