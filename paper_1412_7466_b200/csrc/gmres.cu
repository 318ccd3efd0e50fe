// K6: unrestarted GMRES on the device (solver.gmres; design
// notes SPEC.md:574-577): zero initial guess, dense Krylov basis, classical
// Gram-Schmidt with one re-orthogonalisation (CGS2), Givens rotations and the
// Hessenberg least-squares solve on the device.  Right-hand sides are batched
// (one Arnoldi process per RHS, sharing each operator application); a RHS
// that reaches tol is frozen.  Per iteration only nrhs residual norms
// (8 bytes each) cross to the host for the stopping test.
//
// Krylov basis layout: V[k][rhs][n] (k-major, so V_k is a contiguous
// [nrhs][n] block the Schur operator consumes directly).
#include <cuda_runtime.h>

#include <algorithm>
#include <cmath>
#include <string>
#include <vector>

#include "coupling.cuh"
#include "gmres.cuh"

namespace ps {

namespace {

constexpr int kDotThreads = 256;
constexpr int kChunk = 2048;    // elements per partial-sum CTA (25 CTAs per Krylov vector at cfg3)

__device__ __forceinline__ double2 cfma_conj(double2 a, double2 b, double2 c) {
  // c + conj(a) * b
  return make_double2(fma(a.x, b.x, fma(a.y, b.y, c.x)), fma(a.x, b.y, fma(-a.y, b.x, c.y)));
}

__device__ double2 block_reduce(double2 v, double2* sh) {
  for (int o = 16; o > 0; o >>= 1) {
    v.x += __shfl_xor_sync(0xffffffffu, v.x, o);
    v.y += __shfl_xor_sync(0xffffffffu, v.y, o);
  }
  const int w = threadIdx.x >> 5, lane = threadIdx.x & 31;
  if (lane == 0) sh[w] = v;
  __syncthreads();
  if (w == 0) {
    v = lane < (int)(blockDim.x >> 5) ? sh[lane] : make_double2(0, 0);
    for (int o = 16; o > 0; o >>= 1) {
      v.x += __shfl_xor_sync(0xffffffffu, v.x, o);
      v.y += __shfl_xor_sync(0xffffffffu, v.y, o);
    }
  }
  return v;
}

// part[r][i][c] = sum_{j in chunk c} conj(V_i^r[j]) w^r[j]
__global__ void dot_partial(const double2* __restrict__ V, const double2* __restrict__ w, int nrhs,
                            long long n, int k, int nchunk, const int* __restrict__ active,
                            double2* __restrict__ part) {
  __shared__ double2 sh[32];
  const int c = blockIdx.x, i = blockIdx.y, r = blockIdx.z;
  double2 s = make_double2(0, 0);
  if (!active || active[r]) {
    const double2* vi = V + ((long long)i * nrhs + r) * n;
    const double2* wr = w + (long long)r * n;
    const long long j0 = (long long)c * kChunk;
    const long long j1 = j0 + kChunk < n ? j0 + kChunk : n;
    for (long long j = j0 + threadIdx.x; j < j1; j += blockDim.x) s = cfma_conj(vi[j], wr[j], s);
  }
  s = block_reduce(s, sh);
  if (threadIdx.x == 0) part[((long long)r * k + i) * nchunk + c] = s;
}

// h[r][i] = sum_c part[r][i][c]   (fixed order: deterministic)
__global__ void dot_final(const double2* __restrict__ part, int nrhs, int k, int nchunk,
                          double2* __restrict__ h, int ldh, int accumulate) {
  const int idx = blockIdx.x * blockDim.x + threadIdx.x;
  if (idx >= nrhs * k) return;
  const int r = idx / k, i = idx % k;
  double2 s = make_double2(0, 0);
  for (int c = 0; c < nchunk; ++c) {
    const double2 v = part[(long long)idx * nchunk + c];
    s.x += v.x;
    s.y += v.y;
  }
  double2* dst = h + (long long)r * ldh + i;
  if (accumulate) {
    dst->x += s.x;
    dst->y += s.y;
  } else {
    *dst = s;
  }
}

// w^r += sgn * sum_i h[r][i] V_i^r
__global__ void axpy_block(const double2* __restrict__ V, const double2* __restrict__ h, int ldh,
                           int nrhs, long long n, int k, double sgn,
                           const int* __restrict__ active, double2* __restrict__ w) {
  const int r = blockIdx.y;
  if (active && !active[r]) return;
  extern __shared__ double2 hs[];
  for (int i = threadIdx.x; i < k; i += blockDim.x) hs[i] = h[(long long)r * ldh + i];
  __syncthreads();
  for (long long j = (long long)blockIdx.x * blockDim.x + threadIdx.x; j < n;
       j += (long long)gridDim.x * blockDim.x) {
    double2 acc = w[(long long)r * n + j];
    for (int i = 0; i < k; ++i) {
      const double2 v = V[((long long)i * nrhs + r) * n + j];
      const double2 c = hs[i];
      acc.x = fma(sgn * c.x, v.x, fma(-sgn * c.y, v.y, acc.x));
      acc.y = fma(sgn * c.x, v.y, fma(sgn * c.y, v.x, acc.y));
    }
    w[(long long)r * n + j] = acc;
  }
}

__global__ void norm2_partial(const double2* __restrict__ w, long long n, int nchunk,
                              double2* __restrict__ part) {
  __shared__ double2 sh[32];
  const int c = blockIdx.x, r = blockIdx.y;
  const double2* wr = w + (long long)r * n;
  const long long j0 = (long long)c * kChunk;
  const long long j1 = j0 + kChunk < n ? j0 + kChunk : n;
  double2 s = make_double2(0, 0);
  for (long long j = j0 + threadIdx.x; j < j1; j += blockDim.x)
    s.x = fma(wr[j].x, wr[j].x, fma(wr[j].y, wr[j].y, s.x));
  s = block_reduce(s, sh);
  if (threadIdx.x == 0) part[(long long)r * nchunk + c] = s;
}

__global__ void norm2_final(const double2* __restrict__ part, int nrhs, int nchunk,
                            double* __restrict__ out) {
  const int r = blockIdx.x * blockDim.x + threadIdx.x;
  if (r >= nrhs) return;
  double s = 0.0;
  for (int c = 0; c < nchunk; ++c) s += part[(long long)r * nchunk + c].x;
  out[r] = s;
}

// V_{k+1}^r = w^r / nrm ; x = b / ||b|| for k = -1 (initialisation)
__global__ void scale_into(const double2* __restrict__ w, const double* __restrict__ nrm2,
                           long long n, const int* __restrict__ active, double2* __restrict__ dst) {
  const int r = blockIdx.y;
  const double nr = sqrt(nrm2[r]);
  const bool live = (!active || active[r]) && nr > 0.0;
  const double inv = live ? 1.0 / nr : 0.0;
  for (long long j = (long long)blockIdx.x * blockDim.x + threadIdx.x; j < n;
       j += (long long)gridDim.x * blockDim.x) {
    const double2 v = w[(long long)r * n + j];
    dst[(long long)r * n + j] = make_double2(v.x * inv, v.y * inv);
  }
}

struct GState {
  double2* H;      // [nrhs][maxit+1][maxit] column-major per rhs: H[r][col*(maxit+1)+row]
  double2* cs;     // [nrhs][maxit]
  double2* sn;     // [nrhs][maxit]
  double2* g;      // [nrhs][maxit+1]
  double* bnorm;   // [nrhs]
  double* res;     // [nrhs] current relative residual
  int* active;     // [nrhs]
  int* nonfinite;  // [1]
};

// Apply previous rotations to column k, build the new rotation, update g and
// the relative residual.  One thread per RHS.  hcol holds the CGS2
// coefficients h[0..k] and nrm2 the squared norm of the orthogonalised w.
__global__ void givens_step(GState s, int nrhs, int k, int maxit, const double2* __restrict__ hcol,
                            int ldh, const double* __restrict__ nrm2) {
  const int r = blockIdx.x * blockDim.x + threadIdx.x;
  if (r >= nrhs) return;
  if (!s.active[r]) return;
  const int ldH = maxit + 1;
  double2* col = s.H + ((long long)r * maxit + k) * ldH;
  for (int i = 0; i <= k; ++i) col[i] = hcol[(long long)r * ldh + i];
  col[k + 1] = make_double2(sqrt(nrm2[r]), 0.0);
  double2* cs = s.cs + (long long)r * maxit;
  double2* sn = s.sn + (long long)r * maxit;
  for (int i = 0; i < k; ++i) {
    const double2 a = col[i], b = col[i + 1];
    // t = conj(cs) a + conj(sn) b ; b' = -sn a + cs b
    const double2 c = cs[i], sv = sn[i];
    const double2 t = make_double2(c.x * a.x + c.y * a.y + sv.x * b.x + sv.y * b.y,
                                   c.x * a.y - c.y * a.x + sv.x * b.y - sv.y * b.x);
    const double2 nb = make_double2(-(sv.x * a.x - sv.y * a.y) + (c.x * b.x - c.y * b.y),
                                    -(sv.x * a.y + sv.y * a.x) + (c.x * b.y + c.y * b.x));
    col[i] = t;
    col[i + 1] = nb;
  }
  const double2 a = col[k], b = col[k + 1];
  const double ra = hypot(a.x, a.y), rb = hypot(b.x, b.y);
  const double rr = hypot(ra, rb);
  double2 c, sv;
  if (rr > 0.0) {
    c = make_double2(a.x / rr, a.y / rr);
    sv = make_double2(b.x / rr, b.y / rr);
  } else {
    c = make_double2(1.0, 0.0);
    sv = make_double2(0.0, 0.0);
  }
  cs[k] = c;
  sn[k] = sv;
  col[k] = make_double2(rr, 0.0);
  col[k + 1] = make_double2(0.0, 0.0);
  double2* g = s.g + (long long)r * (maxit + 1);
  const double2 gk = g[k];
  g[k + 1] = make_double2(-(sv.x * gk.x - sv.y * gk.y), -(sv.x * gk.y + sv.y * gk.x));
  g[k] = make_double2(c.x * gk.x + c.y * gk.y, c.x * gk.y - c.y * gk.x);
  const double res = hypot(g[k + 1].x, g[k + 1].y) / s.bnorm[r];
  s.res[r] = res;
  if (!isfinite(res) || !isfinite(rr)) atomicExch(s.nonfinite, 1);
}

// back substitution R y = g for each RHS (y written over g[0..kk))
__global__ void back_solve(GState s, int nrhs, const int* __restrict__ kk_arr, int maxit,
                           double2* __restrict__ y, int ldy) {
  const int r = blockIdx.x * blockDim.x + threadIdx.x;
  if (r >= nrhs) return;
  const int kk = kk_arr[r];
  const int ldH = maxit + 1;
  const double2* H = s.H + (long long)r * maxit * ldH;
  const double2* g = s.g + (long long)r * (maxit + 1);
  double2* yr = y + (long long)r * ldy;
  for (int i = 0; i < ldy; ++i) yr[i] = make_double2(0, 0);
  for (int i = kk - 1; i >= 0; --i) {
    double2 acc = g[i];
    for (int j = i + 1; j < kk; ++j) {
      const double2 h = H[(long long)j * ldH + i];
      const double2 v = yr[j];
      acc.x -= h.x * v.x - h.y * v.y;
      acc.y -= h.x * v.y + h.y * v.x;
    }
    const double2 d = H[(long long)i * ldH + i];
    const double den = d.x * d.x + d.y * d.y;
    yr[i] = make_double2((acc.x * d.x + acc.y * d.y) / den, (acc.y * d.x - acc.x * d.y) / den);
  }
}

__global__ void init_state(GState s, int nrhs, int maxit, const double* __restrict__ b2) {
  const int r = blockIdx.x * blockDim.x + threadIdx.x;
  if (r >= nrhs) return;
  const double bn = sqrt(b2[r]);
  s.bnorm[r] = bn;
  double2* g = s.g + (long long)r * (maxit + 1);
  for (int i = 0; i <= maxit; ++i) g[i] = make_double2(0, 0);
  g[0] = make_double2(bn, 0.0);
  s.res[r] = bn > 0.0 ? 1.0 : 0.0;
  s.active[r] = bn > 0.0 ? 1 : 0;
  if (!isfinite(bn)) {
    s.active[r] = 0;
    s.nonfinite[1 + r] = 1;      // per-RHS flag, checked by the host after init
  }
}

__global__ void set_flags(int* active, const int* flags, int nrhs) {
  const int r = blockIdx.x * blockDim.x + threadIdx.x;
  if (r < nrhs) active[r] = flags[r];
}

// a[r][i] += b[r][i], i < k, row stride ld
__global__ void cadd_rows(double2* __restrict__ a, const double2* __restrict__ b, int nrhs, int k,
                          int ld) {
  const int idx = blockIdx.x * blockDim.x + threadIdx.x;
  if (idx >= nrhs * k) return;
  const int r = idx / k, i = idx % k;
  a[(long long)r * ld + i].x += b[(long long)r * ld + i].x;
  a[(long long)r * ld + i].y += b[(long long)r * ld + i].y;
}

int nchunks(long long n) { return (int)((n + kChunk - 1) / kChunk); }

// hcol[r][i] = h1[r][i] + h2[r][i]  (i <= k; h1/h2 packed [nrhs][k+1], hcol ld)
__global__ void combine_cols(const double2* __restrict__ h1, const double2* __restrict__ h2,
                             int nrhs, int kp1, double2* __restrict__ hcol, int ld) {
  const int idx = blockIdx.x * blockDim.x + threadIdx.x;
  if (idx >= nrhs * kp1) return;
  const int r = idx / kp1, i = idx % kp1;
  const double2 a = h1[idx], b = h2[idx];
  hcol[(long long)r * ld + i] = make_double2(a.x + b.x, a.y + b.y);
}

// status[r] = relative residual of RHS r, status[nrhs] = non-finite flag
__global__ void write_status(const double* __restrict__ res, const int* __restrict__ nonfinite,
                             int nrhs, double* __restrict__ status) {
  const int r = blockIdx.x * blockDim.x + threadIdx.x;
  if (r < nrhs) status[r] = res[r];
  if (r == nrhs) status[r] = nonfinite[0] ? 1.0 : 0.0;
}

}  // namespace

// Device state of one Arnoldi process batch (per context): the Hessenberg
// columns, Givens rotations and residual vector of every RHS, the CGS2
// coefficient scratch and the chunked dot-product partials.  Owned by the
// context (no process-global state), grown on demand, freed by gmres_release.
struct Krylov {
  void* base = nullptr;
  size_t bytes = 0;
  int nrhs = 0, maxit = 0;
  long long n = 0;
  GState s{};
  double2* hcol = nullptr;   // [nrhs][maxit+1]
  double2* y = nullptr;      // [nrhs][maxit+1]
  double2* part = nullptr;   // [nrhs][maxit+1][nchunks]
  double* nrm2 = nullptr;    // [nrhs]
  int* kk = nullptr;         // [nrhs]
  int* flags = nullptr;      // [nrhs]
};

namespace {

// Sizes the Krylov state for (nrhs, n, maxit) plus `extra` bytes of caller
// scratch at the front (the single-rank driver's basis V and w); reuses the
// previous allocation when it is large enough.
int krylov_state(Ctx* c, int nrhs, long long n, int maxit, size_t extra, Krylov** out,
                 void** extra_out) {
  if (!c->krylov) c->krylov = new Krylov();
  Krylov* K = c->krylov;
  const int nc = nchunks(n);
  const size_t szH = (size_t)nrhs * maxit * (maxit + 1);
  const size_t szCS = (size_t)nrhs * maxit;
  const size_t szG = (size_t)nrhs * (maxit + 1);
  const size_t szPart = (size_t)nrhs * (maxit + 1) * nc;
  const size_t pre = (extra + 255) / 256 * 256;
  const size_t elems = szH + 2 * szCS + 3 * szG + szPart;
  const size_t need = pre + elems * sizeof(double2) + (4 * (size_t)nrhs + 8) * sizeof(double) +
                      (5 * (size_t)nrhs + 8) * sizeof(int) + 256;
  if (K->bytes < need) {
    if (K->base) ps::dev_free(K->base);
    K->base = nullptr;
    K->bytes = 0;
    PS_CUDA_TRY(c, ps::dev_malloc(&K->base, need));
    K->bytes = need;
  }
  K->nrhs = nrhs;
  K->n = n;
  K->maxit = maxit;
  char* b = (char*)K->base;
  if (extra_out) *extra_out = b;
  double2* p = (double2*)(b + pre);
  K->s.H = p; p += szH;
  K->s.cs = p; p += szCS;
  K->s.sn = p; p += szCS;
  K->s.g = p; p += szG;
  K->hcol = p; p += szG;
  K->y = p; p += szG;
  K->part = p; p += szPart;
  double* d = (double*)p;
  K->s.bnorm = d; d += nrhs;
  K->s.res = d; d += nrhs;
  K->nrm2 = d; d += 2 * nrhs;
  int* q = (int*)d;
  K->s.active = q; q += nrhs;
  K->kk = q; q += nrhs;
  K->flags = q; q += nrhs;
  K->s.nonfinite = q;                   // [1 + nrhs]
  *out = K;
  return PS_OK;
}

int dot_impl(Ctx* c, int nrhs, long long n, int k, const double2* V, const double2* w,
             double2* h, int ldh, const int* active, double2* part, cudaStream_t st) {
  if (k == 0) return PS_OK;
  const int nc = nchunks(n);
  dim3 grid(nc, k, nrhs);
  c->launches += 2;
  dot_partial<<<grid, kDotThreads, 0, st>>>(V, w, nrhs, n, k, nc, active, part);
  PS_CUDA_TRY(c, cudaGetLastError());
  dot_final<<<(nrhs * k + 127) / 128, 128, 0, st>>>(part, nrhs, k, nc, h, ldh, 0);
  PS_CUDA_TRY(c, cudaGetLastError());
  return PS_OK;
}

int axpy_impl(Ctx* c, int nrhs, long long n, int k, const double2* V, const double2* h, int ldh,
              double sgn, const int* active, double2* w, cudaStream_t st) {
  if (k == 0) return PS_OK;
  int bx = (int)((n + 255) / 256);
  if (bx > 4 * c->sm_count) bx = 4 * c->sm_count;
  dim3 grid(bx, nrhs);
  c->launches += 1;
  axpy_block<<<grid, 256, k * sizeof(double2), st>>>(V, h, ldh, nrhs, n, k, sgn, active, w);
  PS_CUDA_TRY(c, cudaGetLastError());
  return PS_OK;
}

int norm_impl(Ctx* c, int nrhs, long long n, const double2* w, double* out, double2* part,
              cudaStream_t st) {
  const int nc = nchunks(n);
  c->launches += 2;
  norm2_partial<<<dim3(nc, nrhs), kDotThreads, 0, st>>>(w, n, nc, part);
  PS_CUDA_TRY(c, cudaGetLastError());
  norm2_final<<<(nrhs + 127) / 128, 128, 0, st>>>(part, nrhs, nc, out);
  PS_CUDA_TRY(c, cudaGetLastError());
  return PS_OK;
}

int grid_x(const Ctx* c, long long n) {
  return (int)std::min<long long>(std::max<long long>((n + 255) / 256, 1), 4LL * c->sm_count);
}

// state init from the (global) squared RHS norms, V_0 = b / ||b||
int begin_impl(Ctx* c, Krylov* K, const double2* b, const double* b2, double2* V, cudaStream_t st) {
  const int nrhs = K->nrhs;
  PS_CUDA_TRY(c, cudaMemsetAsync(K->s.nonfinite, 0, (1 + nrhs) * sizeof(int), st));
  c->launches += 2;
  init_state<<<(nrhs + 127) / 128, 128, 0, st>>>(K->s, nrhs, K->maxit, b2);
  PS_CUDA_TRY(c, cudaGetLastError());
  scale_into<<<dim3(grid_x(c, K->n), nrhs), 256, 0, st>>>(b, b2, K->n, nullptr, V);
  PS_CUDA_TRY(c, cudaGetLastError());
  return PS_OK;
}

// Givens update of column k from the CGS2 coefficients (hcol, ld maxit+1) and
// the squared norm of the orthogonalised w; V_{k+1} = w / ||w||
int step_impl(Ctx* c, Krylov* K, int k, const double* wn2, const double2* w, double2* V,
              cudaStream_t st) {
  const int nrhs = K->nrhs;
  c->launches += 2;
  givens_step<<<(nrhs + 127) / 128, 128, 0, st>>>(K->s, nrhs, k, K->maxit, K->hcol, K->maxit + 1,
                                                  wn2);
  PS_CUDA_TRY(c, cudaGetLastError());
  scale_into<<<dim3(grid_x(c, K->n), nrhs), 256, 0, st>>>(
      w, wn2, K->n, K->s.active, V + (size_t)(k + 1) * nrhs * K->n);
  PS_CUDA_TRY(c, cudaGetLastError());
  return PS_OK;
}

int freeze_impl(Ctx* c, Krylov* K, const int* active_host, cudaStream_t st) {
  PS_CUDA_TRY(c, cudaMemcpyAsync(K->flags, active_host, K->nrhs * sizeof(int),
                                 cudaMemcpyHostToDevice, st));
  c->launches += 1;
  set_flags<<<(K->nrhs + 127) / 128, 128, 0, st>>>(K->s.active, K->flags, K->nrhs);
  PS_CUDA_TRY(c, cudaGetLastError());
  return PS_OK;
}

// x = sum_i y_i V_i with R y = g per RHS (kk_host[r] columns)
int solve_impl(Ctx* c, Krylov* K, const int* kk_host, const double2* V, double2* x,
               cudaStream_t st) {
  const int nrhs = K->nrhs;
  PS_CUDA_TRY(c, cudaMemcpyAsync(K->kk, kk_host, nrhs * sizeof(int), cudaMemcpyHostToDevice, st));
  c->launches += 1;
  back_solve<<<(nrhs + 127) / 128, 128, 0, st>>>(K->s, nrhs, K->kk, K->maxit, K->y, K->maxit + 1);
  PS_CUDA_TRY(c, cudaGetLastError());
  PS_CUDA_TRY(c, cudaMemsetAsync(x, 0, (size_t)nrhs * K->n * sizeof(double2), st));
  int kmax = 0;
  for (int r = 0; r < nrhs; ++r) kmax = std::max(kmax, kk_host[r]);
  return axpy_impl(c, nrhs, K->n, kmax, V, K->y, K->maxit + 1, 1.0, nullptr, x, st);
}

int need_state(Ctx* c, const char* fn) {
  if (!c->krylov || !c->krylov->base || c->krylov->nrhs < 1) {
    c->err = std::string(fn) + ": call ps_krylov_begin first";
    return PS_ERR_STATE;
  }
  return PS_OK;
}

}  // namespace

void gmres_release(Ctx* c) {
  if (!c->krylov) return;
  if (c->krylov->base) ps::dev_free(c->krylov->base);
  delete c->krylov;
  c->krylov = nullptr;
}

// ---------------------------------------------------------------- building
// blocks for drivers that apply the operator (and reduce over ranks)
// themselves: krylov.gmres_device (any device operator) and the multi-rank
// parallel.gmres_dist.  h tensors are packed [nrhs][k].
int krylov_begin(Ctx* c, int nrhs, long long n, int maxit, const double2* b, const double* b2,
                 double2* V, cudaStream_t st) {
  Krylov* K;
  if (int rc = krylov_state(c, nrhs, n, maxit, 0, &K, nullptr)) return rc;
  if (int rc = begin_impl(c, K, b, b2, V, st)) return rc;
  std::vector<int> bad(nrhs + 1, 0);
  PS_CUDA_TRY(c, cudaMemcpyAsync(bad.data(), K->s.nonfinite, (nrhs + 1) * sizeof(int),
                                 cudaMemcpyDeviceToHost, st));
  PS_CUDA_TRY(c, cudaStreamSynchronize(st));
  for (int r = 0; r < nrhs; ++r)
    if (bad[1 + r]) {
      c->err = "ps_krylov_begin: NaN/Inf in the right-hand side " + std::to_string(r) +
               " (SPEC.md:553)";
      return PS_ERR_NUMERICAL;
    }
  return PS_OK;
}

int krylov_dot(Ctx* c, int k, const double2* V, const double2* w, double2* h, cudaStream_t st) {
  if (int rc = need_state(c, "ps_krylov_dot")) return rc;
  Krylov* K = c->krylov;
  if (k < 1 || k > K->maxit + 1) {
    c->err = "ps_krylov_dot: k out of range";
    return PS_ERR_ARG;
  }
  return dot_impl(c, K->nrhs, K->n, k, V, w, h, k, K->s.active, K->part, st);
}

int krylov_axpy(Ctx* c, int k, const double2* V, const double2* h, double2* w, cudaStream_t st) {
  if (int rc = need_state(c, "ps_krylov_axpy")) return rc;
  Krylov* K = c->krylov;
  if (k < 1 || k > K->maxit + 1) {
    c->err = "ps_krylov_axpy: k out of range";
    return PS_ERR_ARG;
  }
  return axpy_impl(c, K->nrhs, K->n, k, V, h, k, -1.0, K->s.active, w, st);
}

int krylov_norm2(Ctx* c, int nrhs, long long n, const double2* w, double* out, cudaStream_t st) {
  // usable before ps_krylov_begin (the RHS norm): own partial scratch
  Krylov* K;
  const bool have = c->krylov && c->krylov->base && c->krylov->nrhs == nrhs && c->krylov->n == n;
  if (have) {
    K = c->krylov;
  } else if (int rc = krylov_state(c, nrhs, n, 1, 0, &K, nullptr)) {
    return rc;
  }
  return norm_impl(c, nrhs, n, w, out, K->part, st);
}

int krylov_step(Ctx* c, int k, const double2* h1, const double2* h2, const double* wn2,
                const double2* w, double2* V, double* status, cudaStream_t st) {
  if (int rc = need_state(c, "ps_krylov_step")) return rc;
  Krylov* K = c->krylov;
  if (k < 0 || k >= K->maxit) {
    c->err = "ps_krylov_step: k out of range";
    return PS_ERR_ARG;
  }
  const int nrhs = K->nrhs;
  c->launches += 2;
  combine_cols<<<(nrhs * (k + 1) + 127) / 128, 128, 0, st>>>(h1, h2, nrhs, k + 1, K->hcol,
                                                             K->maxit + 1);
  PS_CUDA_TRY(c, cudaGetLastError());
  if (int rc = step_impl(c, K, k, wn2, w, V, st)) return rc;
  write_status<<<(nrhs + 1 + 127) / 128, 128, 0, st>>>(K->s.res, K->s.nonfinite, nrhs, status);
  PS_CUDA_TRY(c, cudaGetLastError());
  return PS_OK;
}

int krylov_freeze(Ctx* c, const int* active_host, cudaStream_t st) {
  if (int rc = need_state(c, "ps_krylov_freeze")) return rc;
  return freeze_impl(c, c->krylov, active_host, st);
}

int krylov_solve(Ctx* c, const int* iters_host, const double2* V, double2* x, cudaStream_t st) {
  if (int rc = need_state(c, "ps_krylov_solve")) return rc;
  Krylov* K = c->krylov;
  for (int r = 0; r < K->nrhs; ++r)
    if (iters_host[r] < 0 || iters_host[r] > K->maxit) {
      c->err = "ps_krylov_solve: iteration count out of range";
      return PS_ERR_ARG;
    }
  return solve_impl(c, K, iters_host, V, x, st);
}

// ---------------------------------------------------------------- whole
// single-rank GMRES with the Schur operator of the context
int gmres(Ctx* c, const double2* rhs, double2* x, double tol, int maxit, int* iters,
          double* hist, cudaStream_t st) {
  if (c->t_begin != 0 || c->t_end != c->M) {
    c->err = "ps_gmres: single-rank driver needs the full target range";
    return PS_ERR_STATE;
  }
  const int nrhs = c->nrhs;
  const long long n = (long long)c->M * c->L;
  const size_t szV = (size_t)(maxit + 1) * nrhs * n;
  const size_t n2 = (size_t)nrhs * n;
  Krylov* K;
  void* front;
  if (int rc = krylov_state(c, nrhs, n, maxit, (szV + n2) * sizeof(double2), &K, &front)) return rc;
  double2* V = (double2*)front;
  double2* w = V + szV;
  double* nrm2 = K->nrm2;

  if (int rc = norm_impl(c, nrhs, n, rhs, nrm2, K->part, st)) return rc;
  if (int rc = begin_impl(c, K, rhs, nrm2, V, st)) return rc;

  std::vector<double> res(nrhs), bn(nrhs);
  std::vector<int> active(nrhs), kk(nrhs, 0), badrhs(nrhs + 1, 0);
  PS_CUDA_TRY(c, cudaMemcpyAsync(bn.data(), K->s.bnorm, nrhs * sizeof(double),
                                 cudaMemcpyDeviceToHost, st));
  PS_CUDA_TRY(c, cudaMemcpyAsync(badrhs.data(), K->s.nonfinite, (nrhs + 1) * sizeof(int),
                                 cudaMemcpyDeviceToHost, st));
  PS_CUDA_TRY(c, cudaStreamSynchronize(st));
  for (int r = 0; r < nrhs; ++r)
    if (badrhs[1 + r]) {
      c->err = "ps_gmres: NaN/Inf in the right-hand side " + std::to_string(r) + " (SPEC.md:553)";
      return PS_ERR_NUMERICAL;
    }
  for (int r = 0; r < nrhs; ++r) {
    active[r] = bn[r] > 0.0;
    iters[r] = 0;
    if (hist) {
      for (int i = 0; i <= maxit; ++i) hist[(size_t)r * (maxit + 1) + i] = NAN;
      hist[(size_t)r * (maxit + 1)] = bn[r] > 0.0 ? 1.0 : 0.0;
    }
  }
  int nactive = 0;
  for (int r = 0; r < nrhs; ++r) nactive += active[r];
  const int ld = maxit + 1;
  for (int k = 0; k < maxit && nactive > 0; ++k) {
    double2* Vk = V + (size_t)k * nrhs * n;
    // w = K V_k
    if (int rc = apply_schur(c, Vk, w, st)) return rc;
    // CGS2: hcol = first-pass coefficients, y = second-pass ones
    if (int rc = dot_impl(c, nrhs, n, k + 1, V, w, K->hcol, ld, K->s.active, K->part, st)) return rc;
    if (int rc = axpy_impl(c, nrhs, n, k + 1, V, K->hcol, ld, -1.0, K->s.active, w, st)) return rc;
    if (int rc = dot_impl(c, nrhs, n, k + 1, V, w, K->y, ld, K->s.active, K->part, st)) return rc;
    if (int rc = axpy_impl(c, nrhs, n, k + 1, V, K->y, ld, -1.0, K->s.active, w, st)) return rc;
    c->launches += 1;
    cadd_rows<<<(nrhs * (k + 1) + 127) / 128, 128, 0, st>>>(K->hcol, K->y, nrhs, k + 1, ld);
    PS_CUDA_TRY(c, cudaGetLastError());
    if (int rc = norm_impl(c, nrhs, n, w, nrm2, K->part, st)) return rc;
    if (int rc = step_impl(c, K, k, nrm2, w, V, st)) return rc;
    int nonfinite = 0;
    PS_CUDA_TRY(c, cudaMemcpyAsync(res.data(), K->s.res, nrhs * sizeof(double),
                                   cudaMemcpyDeviceToHost, st));
    PS_CUDA_TRY(c, cudaMemcpyAsync(&nonfinite, K->s.nonfinite, sizeof(int), cudaMemcpyDeviceToHost,
                                   st));
    PS_CUDA_TRY(c, cudaStreamSynchronize(st));
    if (nonfinite) {
      c->err = "ps_gmres: NaN/Inf in Krylov vector (SPEC.md:553)";
      return PS_ERR_NUMERICAL;
    }
    bool changed = false;
    for (int r = 0; r < nrhs; ++r) {
      if (!active[r]) continue;
      iters[r] = k + 1;
      kk[r] = k + 1;
      if (hist) hist[(size_t)r * (maxit + 1) + k + 1] = res[r];
      if (res[r] <= tol) {
        active[r] = 0;
        --nactive;
        changed = true;
      }
    }
    if (changed)
      if (int rc = freeze_impl(c, K, active.data(), st)) return rc;
  }
  if (int rc = solve_impl(c, K, kk.data(), V, x, st)) return rc;
  PS_CUDA_TRY(c, cudaStreamSynchronize(st));
  return PS_OK;
}

}  // namespace ps
