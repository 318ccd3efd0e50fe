// Pre-assembled coupling blocks: multiscat.multipole_to_targets_block C and
// source_to_local_block B_phys (SPEC.md:484-502 return them as MATRICES).
//
// Both are geometry + Bloch-phase only, so for a GMRES solve they are built
// once on the device (same symbol generator as K1/K3/K5) and every Schur
// matvec then streams them from HBM:
//   C^T  [ (cs1-cs0) L ][ nrow_c ]   rows = source (inclusion, order), cols = A-row
//   B    [ Mt L ][ ncol_b ]          rows = owned (inclusion, order), cols = x_empty
// K3d: g = C v   (split-k over the source rows, deterministic partial sums)
// K5d: b = B x   (warp per output row, x staged in shared memory)
// Per-RHS matrices (the Bloch weights are folded in); used when they fit the
// memory budget given to ps_precompute_coupling, matrix-free K3/K5 otherwise.
#include <cuda_runtime.h>

#include <string>

#include "coupling.cuh"
#include "m2l.cuh"
#include "symbols.cuh"

namespace ps {

namespace {

__device__ __forceinline__ double2 cmul(double2 a, double2 b) {
  return make_double2(fma(a.x, b.x, -a.y * b.y), fma(a.x, b.y, a.y * b.x));
}
__device__ __forceinline__ double2 cfma(double2 a, double2 b, double2 c) {
  return make_double2(fma(a.x, b.x, fma(-a.y, b.y, c.x)), fma(a.x, b.y, fma(a.y, b.x, c.y)));
}

constexpr int kBuildT = 32;   // static smem: 32 x 53 x 16 B at p = 25

// ---------------------------------------------------------------- C^T builder
// thread = target node (val row rv, derivative row rd), blockIdx.y = source j
template <int P>
__global__ void __launch_bounds__(kBuildT) cbuild_kernel(
    const double* __restrict__ centers, const double2* __restrict__ bpow, const double* g1,
    const double* g2, const double* w2, int n1, int n2, int nw, int copies, int cs0, int nrow_c,
    double period, double k2, double2* __restrict__ CT) {
  constexpr int NU = P + 1, L = 2 * P + 1, NSP = 2 * NU + 1;
  __shared__ double2 rowbuf[kBuildT * NSP];
  const int node = blockIdx.x * kBuildT + threadIdx.x;
  const int j = cs0 + blockIdx.y;
  if (node >= n1 + n2 + nw) return;
  double tx, ty, nx, ny, sgn;
  int kind, rv, rd;
  if (node < n1) {
    const double* q = g1 + 5 * node;
    tx = q[0]; ty = q[1]; nx = q[2]; ny = q[3]; sgn = -1.0; kind = 0;
    rv = node; rd = n1 + node;
  } else if (node < n1 + n2) {
    const int i = node - n1;
    const double* q = g2 + 5 * i;
    tx = q[0]; ty = q[1]; nx = q[2]; ny = q[3]; sgn = 1.0; kind = 0;
    rv = 2 * n1 + i; rd = 2 * n1 + n2 + i;
  } else {
    const int i = node - n1 - n2;
    tx = w2[2 * i]; ty = w2[2 * i + 1]; nx = 1.0; ny = 0.0; sgn = 1.0; kind = 1;
    rv = 2 * n1 + 2 * n2 + i; rd = rv + nw;
  }
  const int nl = kind == 0 ? 2 * copies + 1 : 2;
  double2* row = rowbuf + (size_t)threadIdx.x * NSP + NU;   // t_nu at row[nu]
  const double hk = 0.5 * k2;
  const double2 cp = make_double2(hk * nx, hk * ny);    // (k/2)(nx + i ny)
  const double2 cm = make_double2(-hk * nx, hk * ny);   // (k/2)(-nx + i ny)
  double2* out = CT + (size_t)(j - cs0) * L * nrow_c;
  for (int li = 0; li < nl; ++li) {
    int l;
    double2 wgt;
    if (kind == 0) {
      l = li - copies;
      wgt = bpow[l + copies + 1];
    } else if (li == 0) {
      l = copies;
      wgt = bpow[2 * copies + 2];
    } else {
      l = -(copies + 1);
      wgt = make_double2(-bpow[1].x, -bpow[1].y);
    }
    wgt = make_double2(sgn * wgt.x, sgn * wgt.y);
    const double dx = tx - centers[2 * j] - (double)l * period;
    const double dy = ty - centers[2 * j + 1];
    const double rho = hypot(dx, dy);
    const double inv = 1.0 / rho;
    const double z = k2 * rho;
    hankel_symbols<NU>(z, dx * inv, dy * inv, miller_start_j01(z),
                       [&](int nu, double re, double im) { row[nu] = make_double2(re, im); });
    // value:      coefficient of beta_n is w_n
    // derivative: coefficient of beta_n is (k/2)[(nx+iny) w_{n-1} + (-nx+iny) w_{n+1}]
    for (int n = -P; n <= P; ++n) {
      const double2 v = cmul(wgt, row[n]);
      const double2 d = cmul(wgt, cfma(cm, row[n + 1], cmul(cp, row[n - 1])));
      double2* e = out + (size_t)(n + P) * nrow_c;
      if (li == 0) {
        e[rv] = v;
        e[rd] = d;
      } else {
        e[rv].x += v.x;
        e[rv].y += v.y;
        e[rd].x += d.x;
        e[rd].y += d.y;
      }
    }
  }
}

// ---------------------------------------------------------------- B builder
// thread = interface node (columns mu, sigma), blockIdx.y = owned inclusion
template <int P>
__global__ void __launch_bounds__(kBuildT) bbuild_kernel(
    const double* __restrict__ centers, const double2* __restrict__ bpow, const double* g1,
    const double* g2, int n1, int n2, int copies, int t0, int ncol_b, double period, double k2,
    double2* __restrict__ B) {
  constexpr int NU = P + 1, L = 2 * P + 1, NSP = 2 * NU + 1;
  __shared__ double2 rowbuf[kBuildT * NSP];
  const int node = blockIdx.x * kBuildT + threadIdx.x;
  const int m = t0 + blockIdx.y;
  if (node >= n1 + n2) return;
  const bool on1 = node < n1;
  const double* q = on1 ? g1 + 5 * node : g2 + 5 * (node - n1);
  const int mu_col = on1 ? node : 2 * n1 + (node - n1);
  const int sg_col = on1 ? n1 + node : 2 * n1 + n2 + (node - n1);
  const double nx = q[2], ny = q[3], w = q[4];
  const double hk = 0.5 * k2;
  const double2 dpl = make_double2(hk * nx, -hk * ny);    //  (k/2)(nx - i ny)
  const double2 dmi = make_double2(-hk * nx, -hk * ny);   // -(k/2)(nx + i ny)
  double2* row = rowbuf + (size_t)threadIdx.x * NSP + NU;
  double2* out = B + (size_t)(m - t0) * L * ncol_b;
  const double xm = centers[2 * m], ym = centers[2 * m + 1];
  for (int li = 0; li < 2 * copies + 1; ++li) {
    const int l = li - copies;
    const double2 wl = bpow[l + copies + 1];
    const double2 iw = make_double2(-0.25 * w * wl.y, 0.25 * w * wl.x);   // (i/4) bloch^l w
    const double dx = xm - q[0] - (double)l * period;
    const double dy = ym - q[1];
    const double rho = hypot(dx, dy);
    const double inv = 1.0 / rho;
    const double z = k2 * rho;
    hankel_symbols<NU>(z, dx * inv, dy * inv, miller_start_j01(z),
                       [&](int nu, double re, double im) { row[nu] = make_double2(re, im); });
    for (int np = -P; np <= P; ++np) {
      const double2 s = cmul(iw, row[-np]);
      const double2 d = cmul(iw, cfma(dmi, row[-1 - np], cmul(dpl, row[1 - np])));
      double2* e = out + (size_t)(np + P) * ncol_b;
      if (li == 0) {
        e[sg_col] = s;
        e[mu_col] = d;
      } else {
        e[sg_col].x += s.x;
        e[sg_col].y += s.y;
        e[mu_col].x += d.x;
        e[mu_col].y += d.y;
      }
    }
  }
}

// B_pm columns: J_{q-n'}(k2 rho) e^{i(q-n') phi}, (rho, phi) = polar(x_m - x2)
template <int P>
__global__ void bpm_build_kernel(const double* __restrict__ centers, int t0, int Q, int a2col,
                                 int ncol_b, double k2, double x2x, double x2y,
                                 double2* __restrict__ B) {
  constexpr int L = 2 * P + 1;
  extern __shared__ double2 jl[];
  const int m = t0 + blockIdx.x;
  const int NQ = Q + P;
  if (threadIdx.x == 0) {
    const double dx = centers[2 * m] - x2x, dy = centers[2 * m + 1] - x2y;
    const double rho = hypot(dx, dy);
    double2* j0 = jl + NQ;
    if (rho == 0.0) {
      for (int nu = -NQ; nu <= NQ; ++nu) j0[nu] = make_double2(nu == 0 ? 1.0 : 0.0, 0.0);
    } else {
      double inv_norm, y0, y1;
      bessel_jy_sweep(k2 * rho, NQ, [&](int nu, double v) { j0[nu].x = v; }, &inv_norm, &y0, &y1);
      const double c = dx / rho, s = dy / rho;
      double pr = 1.0, pi = 0.0;
      j0[0] = make_double2(j0[0].x * inv_norm, 0.0);
      for (int nu = 1; nu <= NQ; ++nu) {
        const double npr = fma(pr, c, -pi * s), npi = fma(pr, s, pi * c);
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
  double2* out = B + (size_t)(m - t0) * L * ncol_b;
  for (int idx = threadIdx.x; idx < L * (2 * Q + 1); idx += blockDim.x) {
    const int np = idx / (2 * Q + 1) - P, qq = idx % (2 * Q + 1) - Q;
    out[(size_t)(np + P) * ncol_b + a2col + qq + Q] = jl[NQ + qq - np];
  }
}

// ---------------------------------------------------------------- apply
// gpart[chunk][row] = sum_{k in chunk} CT[k][row] * v[k]
// 192 threads x 3 rows cover nrow_c = 576 exactly at the BASELINE geometry;
// k is unrolled by 4 with independent accumulators to keep loads in flight.
constexpr int kCtT = 192;
constexpr int kCtR = 3;
__global__ void __launch_bounds__(kCtT) ct_gemv(const double2* __restrict__ CT,
                                                const double2* __restrict__ v, int K, int nrow,
                                                int kper, double2* __restrict__ gpart) {
  const int k0 = blockIdx.x * kper;
  const int k1 = min(K, k0 + kper);
  for (int rb = 0; rb < nrow; rb += kCtT * kCtR) {
    double2 acc[kCtR][4];
#pragma unroll
    for (int q = 0; q < kCtR; ++q)
#pragma unroll
      for (int u = 0; u < 4; ++u) acc[q][u] = make_double2(0, 0);
    int k = k0;
    for (; k + 3 < k1; k += 4) {
      double2 vv[4];
#pragma unroll
      for (int u = 0; u < 4; ++u) vv[u] = __ldg(v + k + u);
#pragma unroll
      for (int q = 0; q < kCtR; ++q) {
        const int row = rb + q * kCtT + threadIdx.x;
        if (row < nrow) {
#pragma unroll
          for (int u = 0; u < 4; ++u)
            acc[q][u] = cfma(__ldcs(CT + (size_t)(k + u) * nrow + row), vv[u], acc[q][u]);
        }
      }
    }
    for (; k < k1; ++k) {
      const double2 vv = __ldg(v + k);
#pragma unroll
      for (int q = 0; q < kCtR; ++q) {
        const int row = rb + q * kCtT + threadIdx.x;
        if (row < nrow) acc[q][0] = cfma(__ldcs(CT + (size_t)k * nrow + row), vv, acc[q][0]);
      }
    }
#pragma unroll
    for (int q = 0; q < kCtR; ++q) {
      const int row = rb + q * kCtT + threadIdx.x;
      if (row < nrow)
        gpart[(size_t)blockIdx.x * nrow + row] =
            make_double2((acc[q][0].x + acc[q][1].x) + (acc[q][2].x + acc[q][3].x),
                         (acc[q][0].y + acc[q][1].y) + (acc[q][2].y + acc[q][3].y));
    }
  }
}

// g[i] = sum_q part[q][i]: one warp per output, fixed shuffle tree
__global__ void sum_parts(const double2* __restrict__ part, int np, int n, double2* __restrict__ g) {
  const int i = blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5);
  const int lane = threadIdx.x & 31;
  if (i >= n) return;
  double2 s = make_double2(0, 0);
  for (int q = lane; q < np; q += 32) {
    const double2 v = part[(size_t)q * n + i];
    s.x += v.x;
    s.y += v.y;
  }
  for (int o = 16; o > 0; o >>= 1) {
    s.x += __shfl_xor_sync(0xffffffffu, s.x, o);
    s.y += __shfl_xor_sync(0xffffffffu, s.y, o);
  }
  if (lane == 0) g[i] = s;
}

// b[row] = sum_c B[row][c] x[c]: one warp per row, x in shared memory
__global__ void b_gemv(const double2* __restrict__ B, const double2* __restrict__ x, int nrows,
                       int ncol, double2* __restrict__ b) {
  extern __shared__ double2 xs[];
  for (int c = threadIdx.x; c < ncol; c += blockDim.x) xs[c] = x[c];
  __syncthreads();
  const int lane = threadIdx.x & 31;
  const int row = blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5);
  if (row >= nrows) return;
  const double2* br = B + (size_t)row * ncol;
  double2 acc = make_double2(0, 0);
  // streamed once per matvec: evict-first, so the 0.45 GB pass does not push
  // the K1s partial sums (L2-resident, read by k1s_reduce) out to DRAM
  for (int c = lane; c < ncol; c += 32) acc = cfma(__ldcs(br + c), xs[c], acc);
  for (int o = 16; o > 0; o >>= 1) {
    acc.x += __shfl_xor_sync(0xffffffffu, acc.x, o);
    acc.y += __shfl_xor_sync(0xffffffffu, acc.y, o);
  }
  if (lane == 0) b[row] = acc;
}

template <int P>
int build_p(Ctx* c, int r) {
  auto& R = c->rhs[r];
  const double2* bp = c->d_blochpow + (size_t)r * (2 * c->copies + 3);
  const int nodes = c->n1 + c->n2 + c->nw;
  dim3 gc((nodes + kBuildT - 1) / kBuildT, c->dcs1 - c->dcs0);
  if (c->dcs1 > c->dcs0) {
    cbuild_kernel<P><<<gc, kBuildT>>>(c->d_centers, bp, c->d_g1, c->d_g2, c->d_w2, c->n1, c->n2,
                                      c->nw, c->copies, c->dcs0, c->nrow_c, c->period, c->k2,
                                      R.d_CT);
    PS_CUDA_TRY(c, cudaGetLastError());
  }
  const int nt = c->t_end - c->t_begin;
  if (nt > 0) {
    dim3 gb((c->n1 + c->n2 + kBuildT - 1) / kBuildT, nt);
    bbuild_kernel<P><<<gb, kBuildT>>>(c->d_centers, bp, c->d_g1, c->d_g2, c->n1, c->n2, c->copies,
                                      c->t_begin, c->ncol_b, c->period, c->k2, R.d_B);
    PS_CUDA_TRY(c, cudaGetLastError());
    const int NQ = c->Q + P;
    bpm_build_kernel<P><<<nt, 128, (2 * NQ + 1) * sizeof(double2)>>>(
        c->d_centers, c->t_begin, c->Q, 2 * c->n1 + 2 * c->n2, c->ncol_b, c->k2, c->x2[0],
        c->x2[1], R.d_B);
    PS_CUDA_TRY(c, cudaGetLastError());
  }
  PS_CUDA_TRY(c, cudaDeviceSynchronize());
  return PS_OK;
}

}  // namespace

int precompute_coupling(Ctx* c, double max_bytes) {
  const int nt = c->t_end - c->t_begin;
  const size_t ct = (size_t)(c->t_end - c->t_begin) * c->L * c->nrow_c;
  const size_t bb = (size_t)nt * c->L * c->ncol_b;
  const double need = (double)c->nrhs * (double)(ct + bb) * sizeof(double2);
  release_dense_coupling(c);
  if (need > max_bytes) {
    c->dense = 0;
    return PS_OK;                       // stays matrix-free
  }
  c->dcs0 = c->t_begin;                 // C^T for the owned SOURCE range (== targets)
  c->dcs1 = c->t_end;
  for (int r = 0; r < c->nrhs; ++r) {
    auto& R = c->rhs[r];
    PS_CUDA_TRY(c, ps::dev_malloc(&R.d_CT, ct * sizeof(double2) + 16));
    PS_CUDA_TRY(c, ps::dev_malloc(&R.d_B, bb * sizeof(double2) + 16));
    int rc = PS_OK;
    switch (c->p) {
#define PS_CASE(P) \
  case P:          \
    rc = build_p<P>(c, r); \
    break;
      PS_M2L_ORDERS(PS_CASE)
#undef PS_CASE
      default:
        c->err = "precompute_coupling: order not compiled";
        return PS_ERR_UNSUPPORTED;
    }
    if (rc) return rc;
  }
  c->dense = 1;
  c->launches += 3 * c->nrhs;
  return PS_OK;
}

void release_dense_coupling(Ctx* c) {
  for (auto& R : c->rhs) {
    if (R.d_CT) ps::dev_free(R.d_CT);
    if (R.d_B) ps::dev_free(R.d_B);
    R.d_CT = nullptr;
    R.d_B = nullptr;
  }
  c->dense = 0;
}

// g_r = C_r v_r over sources [s0, s1) (must equal the stored range)
int dense_apply_C(Ctx* c, int r, const double2* v_r, double2* gpart, double2* g_r, cudaStream_t st) {
  const auto& R = c->rhs[r];
  const int K = (c->dcs1 - c->dcs0) * c->L;
  const int nblk = 4 * c->sm_count;
  const int kper = (K + nblk - 1) / nblk;
  const int nb = kper > 0 ? (K + kper - 1) / kper : 0;
  if (nb == 0) {
    PS_CUDA_TRY(c, cudaMemsetAsync(g_r, 0, c->nrow_c * sizeof(double2), st));
    return PS_OK;
  }
  ct_gemv<<<nb, kCtT, 0, st>>>(R.d_CT, v_r + (size_t)c->dcs0 * c->L, K, c->nrow_c, kper, gpart);
  PS_CUDA_TRY(c, cudaGetLastError());
  sum_parts<<<(c->nrow_c + 7) / 8, 256, 0, st>>>(gpart, nb, c->nrow_c, g_r);
  PS_CUDA_TRY(c, cudaGetLastError());
  c->launches += 2;
  return PS_OK;
}

// b_r = B_r x_r for the owned targets
int dense_apply_B(Ctx* c, int r, const double2* x_r, double2* b_r, cudaStream_t st) {
  const int rows = (c->t_end - c->t_begin) * c->L;
  if (rows <= 0) return PS_OK;
  b_gemv<<<(rows + 7) / 8, 256, c->ncol_b * sizeof(double2), st>>>(c->rhs[r].d_B, x_r, rows,
                                                                    c->ncol_b, b_r);
  PS_CUDA_TRY(c, cudaGetLastError());
  c->launches += 1;
  return PS_OK;
}

size_t dense_gpart_elems(const Ctx* c) { return (size_t)(4 * c->sm_count + 1) * c->nrow_c; }

}  // namespace ps
