// extern "C" entry points of include/periscat_b200.h.
#include <cuda_runtime.h>

#include <cstdlib>

#include <cmath>
#include <complex>
#include <cstring>
#include <string>
#include <vector>

#include "coupling.cuh"
#include "field.cuh"
#include "ctx.cuh"
#include "empty.cuh"
#include "gmres.cuh"
#include "m2l.cuh"

using ps::C;
using ps::Ctx;

namespace {

template <typename T>
int dev_upload(Ctx* c, T** dst, const T* src, size_t n) {
  if (*dst) {
    ps::dev_free(*dst);
    *dst = nullptr;
  }
  if (n == 0) return PS_OK;
  PS_CUDA_TRY(c, ps::dev_malloc(reinterpret_cast<void**>(dst), n * sizeof(T)));
  if (src) PS_CUDA_TRY(c, cudaMemcpy(*dst, src, n * sizeof(T), cudaMemcpyHostToDevice));
  return PS_OK;
}

int set_device(Ctx* c) {
  PS_CUDA_TRY(c, cudaSetDevice(c->device));
  return PS_OK;
}

// bloch^l for l = -(copies+1) .. copies+1 per RHS (the telescoped wall rows
// of C need the two extreme powers, lp:211-237).
int upload_blochpow(Ctx* c) {
  const int np = 2 * c->copies + 3;
  std::vector<double2> h((size_t)c->nrhs * np);
  for (int r = 0; r < c->nrhs; ++r) {
    const std::complex<double> b(c->rhs[r].bloch.x, c->rhs[r].bloch.y);
    for (int i = 0; i < np; ++i) {
      const int l = i - (c->copies + 1);
      const std::complex<double> v = std::pow(b, (double)l);
      h[(size_t)r * np + i] = make_double2(v.real(), v.imag());
    }
  }
  return dev_upload(c, &c->d_blochpow, h.data(), h.size());
}

// Closest pair of centres over the phased copies l = -lmax..lmax (j >= i;
// the self term j == i, l == 0 excluded): thread per i, per-thread result;
// the host reduces the M records (deterministic: smallest distance, then
// smallest i).  Replaces an O(M^2) host scan (1.5e8 pairs at M = 1e4).
__global__ void pair_min_dist(const double2* __restrict__ c, int M, int lmax, double period,
                              double* __restrict__ best, int* __restrict__ bj,
                              int* __restrict__ bl) {
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= M) return;
  const double2 ci = c[i];
  double m = INFINITY;
  int mj = -1, ml = 0;
  for (int j = i; j < M; ++j) {
    const double2 cj = c[j];
    for (int l = -lmax; l <= lmax; ++l) {
      if (j == i && l == 0) continue;
      const double d = hypot(ci.x - cj.x - l * period, ci.y - cj.y);
      if (d < m) {
        m = d;
        mj = j;
        ml = l;
      }
    }
  }
  best[i] = m;
  bj[i] = mj;
  bl[i] = ml;
}

struct Closest {
  double dist = INFINITY;
  int i = -1, j = -1, l = 0;
};

int closest_pair(Ctx* c, int lmax, Closest* out) {
  *out = Closest{};
  const int M = c->M;
  if (M < 1) return PS_OK;
  double* d = nullptr;
  PS_CUDA_TRY(c, ps::dev_malloc(&d, (size_t)M * (sizeof(double) + 2 * sizeof(int))));
  int* dj = reinterpret_cast<int*>(d + M);
  int* dl = dj + M;
  pair_min_dist<<<(M + 127) / 128, 128>>>(reinterpret_cast<const double2*>(c->d_centers), M, lmax,
                                          c->period, d, dj, dl);
  c->launches += 1;
  std::vector<double> hd(M);
  std::vector<int> hj(M), hl(M);
  cudaError_t e = cudaGetLastError();
  if (e == cudaSuccess) e = cudaMemcpy(hd.data(), d, M * sizeof(double), cudaMemcpyDeviceToHost);
  if (e == cudaSuccess) e = cudaMemcpy(hj.data(), dj, M * sizeof(int), cudaMemcpyDeviceToHost);
  if (e == cudaSuccess) e = cudaMemcpy(hl.data(), dl, M * sizeof(int), cudaMemcpyDeviceToHost);
  ps::dev_free(d);
  PS_CUDA_TRY(c, e);
  for (int i = 0; i < M; ++i)
    if (hj[i] >= 0 && hd[i] < out->dist) *out = Closest{hd[i], i, hj[i], hl[i]};
  return PS_OK;
}

}  // namespace

extern "C" {

int ps_version(void) { return 1; }

#ifdef PS_CANARY
}  // extern "C"
namespace {
__global__ void canary_overrun(unsigned char* p, int n) {
  if (threadIdx.x == 0) p[n + 3] = 0x5A;      // deliberately 4 bytes past the end
}
}  // namespace
extern "C" {
#endif

/* Self-test of the guard bands: a deliberate 1-byte overrun must be counted. */
long long ps_canary_selftest(void) {
#ifdef PS_CANARY
  unsigned char* p = nullptr;
  if (ps::dev_malloc(&p, 1024) != cudaSuccess) return -2;
  canary_overrun<<<1, 32>>>(p, 1024);
  cudaDeviceSynchronize();
  long long before;
  {
    std::lock_guard<std::mutex> g(ps::canary_reg().mu);
    before = ps::canary_reg().violations;
  }
  ps::dev_free(p);
  std::lock_guard<std::mutex> g(ps::canary_reg().mu);
  const long long found = ps::canary_reg().violations - before;
  ps::canary_reg().violations = before;        // not a product-kernel violation
  return found;
#else
  return -1;
#endif
}

long long ps_canary_check(void) {
#ifdef PS_CANARY
  std::lock_guard<std::mutex> g(ps::canary_reg().mu);
  for (auto& kv : ps::canary_reg().live) {
    const long long bad = ps::canary_bad_bytes(kv.first, kv.second);
    if (bad) ps::canary_reg().violations += bad;
  }
  return ps::canary_reg().violations;
#else
  return -1;
#endif
}

int ps_max_order(void) { return ps::m2l_max_order(); }

int ps_create(ps_ctx** out, int device) {
  if (!out) return PS_ERR_ARG;
  Ctx* c = new Ctx();
  c->device = device;
  *out = reinterpret_cast<ps_ctx*>(c);
  if (int rc = set_device(c)) return rc;
  int sms = 0;
  PS_CUDA_TRY(c, cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, device));
  c->sm_count = sms;
  if (const char* e = getenv("PS_K1S_STAGE")) c->k1s_stage = e[0] != '0';   // experiment switch
  c->rhs.resize(1);
  return upload_blochpow(c);
}

void ps_destroy(ps_ctx* h) {
  if (!h) return;
  Ctx* c = C(h);
  cudaSetDevice(c->device);
  void* ptrs[] = {c->d_centers, c->d_S, c->d_rot, c->d_g1, c->d_g2, c->d_w2, c->d_blochpow,
                  c->d_partial, c->d_work, c->d_inc, c->d_symstore};
  for (void* p : ptrs)
    if (p) ps::dev_free(p);
  for (auto& r : c->rhs) {
    void* rp[] = {r.d_Uh, r.d_sinv, r.d_Vb, r.d_cscale, r.d_f};
    for (void* p : rp)
      if (p) ps::dev_free(p);
  }
  ps::release_dense_coupling(c);
  ps::gmres_release(c);
  ps::empty_release(c);
  if (c->s_hi) cudaStreamDestroy(c->s_hi);
  if (c->s_lo) cudaStreamDestroy(c->s_lo);
  cudaEvent_t evs[] = {c->ev_fork, c->ev_k1, c->ev_cpl, c->ev_bw};
  for (cudaEvent_t e : evs)
    if (e) cudaEventDestroy(e);
  delete c;
}

const char* ps_last_error(const ps_ctx* h) {
  return h ? reinterpret_cast<const Ctx*>(h)->err.c_str() : "null context";
}

int ps_set_geometry(ps_ctx* h, int M, int p, int copies, double period, double k2,
                    const double* centers) {
  if (!h) return PS_ERR_ARG;
  Ctx* c = C(h);
  ps::release_dense_coupling(c);   // geometry / phases changed
  if (M < 0 || p < 0 || copies < 0 || !(period > 0) || !(k2 > 0) || (M > 0 && !centers)) {
    c->err = "ps_set_geometry: bad argument";
    return PS_ERR_ARG;
  }
  if (p > ps::m2l_max_order()) {
    c->err = "ps_set_geometry: p=" + std::to_string(p) + " exceeds compiled maximum " +
             std::to_string(ps::m2l_max_order());
    return PS_ERR_UNSUPPORTED;
  }
  if (int rc = set_device(c)) return rc;
  ++c->geom_gen;                   // invalidates the K1s symbol store
  if (c->d_symstore) {
    ps::dev_free(c->d_symstore);
    c->d_symstore = nullptr;
    c->symstore_bytes = 0;
  }
  c->M = M;
  c->p = p;
  c->L = 2 * p + 1;
  c->copies = copies;
  c->period = period;
  c->k2 = k2;
  c->t_begin = 0;
  c->t_end = M;
  c->h_centers.assign(centers, centers + 2 * (size_t)M);
  if (int rc = dev_upload(c, &c->d_centers, centers, 2 * (size_t)M)) return rc;
  // coincident centres (incl. phased copies) make the translation singular
  // (SPEC.md:458, 506); disk overlap needs the radius (ps_check_overlap)
  Closest cp;
  if (int rc = closest_pair(c, copies, &cp)) return rc;
  if (cp.i >= 0 && cp.dist == 0.0) {
    c->err = "ps_set_geometry: coincident centres " + std::to_string(cp.i) + ", " +
             std::to_string(cp.j) + " (copy " + std::to_string(cp.l) + ")";
    c->M = 0;
    return PS_ERR_DOMAIN;
  }
  return upload_blochpow(c);
}

int ps_check_overlap(ps_ctx* h, double radius, double* min_gap) {
  if (!h) return PS_ERR_ARG;
  Ctx* c = C(h);
  if (!(radius >= 0.0)) {
    c->err = "ps_check_overlap: bad radius";
    return PS_ERR_ARG;
  }
  if (c->p < 0) {
    c->err = "ps_check_overlap: geometry not set";
    return PS_ERR_STATE;
  }
  if (int rc = set_device(c)) return rc;
  // ParticleSet.min_gap (geometry.py:131-144): all pairs and their +-d
  // copies; fewer than two inclusions -> +inf
  double gap = INFINITY;
  Closest cp;
  if (c->M >= 2) {
    if (int rc = closest_pair(c, 1, &cp)) return rc;
    gap = cp.dist - 2.0 * radius;
  }
  if (min_gap) *min_gap = gap;
  if (gap < 0.0) {
    c->err = "overlapping inclusions " + std::to_string(cp.i) + ", " + std::to_string(cp.j) +
             " (copy " + std::to_string(cp.l) + "): centre distance " + std::to_string(cp.dist) +
             " < 2R = " + std::to_string(2.0 * radius) + " (SPEC.md:458, 506)";
    return PS_ERR_DOMAIN;
  }
  return PS_OK;
}

int ps_set_target_range(ps_ctx* h, int t_begin, int t_end) {
  if (!h) return PS_ERR_ARG;
  Ctx* c = C(h);
  ps::release_dense_coupling(c);   // geometry / phases changed
  if (t_begin < 0 || t_end < t_begin || t_end > c->M) {
    c->err = "ps_set_target_range: bad range";
    return PS_ERR_ARG;
  }
  c->t_begin = t_begin;
  c->t_end = t_end;
  return PS_OK;
}

int ps_set_rhs_bloch(ps_ctx* h, int nrhs, const double* bloch) {
  if (!h) return PS_ERR_ARG;
  Ctx* c = C(h);
  ps::release_dense_coupling(c);   // geometry / phases changed
  if (nrhs < 1 || !bloch) {
    c->err = "ps_set_rhs_bloch: bad argument";
    return PS_ERR_ARG;
  }
  if (int rc = set_device(c)) return rc;
  if ((int)c->rhs.size() != nrhs) {
    // a different RHS count invalidates every per-RHS factor set (and the
    // per-RHS layer-field data): the coupled entry points then report
    // PS_ERR_STATE until the factors are installed again (ps_set_pinv /
    // ps_setup_empty), instead of reading null factors of the new RHS
    for (auto& d : c->rhs) {
      void* rp[] = {d.d_Uh, d.d_sinv, d.d_Vb, d.d_cscale, d.d_f};
      for (void* q : rp)
        if (q) ps::dev_free(q);
      d = ps::RhsData{};
    }
    c->nsv = 0;
    c->nfield = 0;
    if (c->d_inc) ps::dev_free(c->d_inc);
    c->d_inc = nullptr;
    c->have_field = 0;
  }
  c->rhs.resize(nrhs);
  c->nrhs = nrhs;
  for (int r = 0; r < nrhs; ++r) c->rhs[r].bloch = make_double2(bloch[2 * r], bloch[2 * r + 1]);
  return upload_blochpow(c);
}

int ps_set_smatrix(ps_ctx* h, const double* S, int diagonal, const double* rot) {
  if (!h) return PS_ERR_ARG;
  Ctx* c = C(h);
  if (c->p < 0 || !S) {
    c->err = "ps_set_smatrix: set geometry first / null S";
    return c->p < 0 ? PS_ERR_STATE : PS_ERR_ARG;
  }
  if (int rc = set_device(c)) return rc;
  c->s_diag = diagonal ? 1 : 0;
  const size_t n = diagonal ? (size_t)c->L : (size_t)c->L * c->L;
  if (int rc = dev_upload(c, &c->d_S, reinterpret_cast<const double2*>(S), n)) return rc;
  if (!diagonal && rot) return dev_upload(c, &c->d_rot, rot, (size_t)c->M);
  if (c->d_rot) {
    ps::dev_free(c->d_rot);
    c->d_rot = nullptr;
  }
  return PS_OK;
}

int ps_set_layers(ps_ctx* h, int n1, const double* g1, int n2, const double* g2, int nw,
                  const double* w2, const double* x2, int Q, int nrb) {
  if (!h) return PS_ERR_ARG;
  Ctx* c = C(h);
  ps::release_dense_coupling(c);   // geometry / phases changed
  if (n1 <= 0 || n2 <= 0 || nw <= 0 || Q < 0 || nrb <= 0 || !g1 || !g2 || !w2 || !x2) {
    c->err = "ps_set_layers: bad argument";
    return PS_ERR_ARG;
  }
  if (int rc = set_device(c)) return rc;
  c->n1 = n1;
  c->n2 = n2;
  c->nw = nw;
  c->Q = Q;
  c->nrb = nrb;
  c->x2[0] = x2[0];
  c->x2[1] = x2[1];
  c->nrow_c = 2 * n1 + 2 * n2 + 2 * nw;
  c->ncol_b = 2 * n1 + 2 * n2 + 2 * Q + 1;
  if (int rc = dev_upload(c, &c->d_g1, g1, 5 * (size_t)n1)) return rc;
  if (int rc = dev_upload(c, &c->d_g2, g2, 5 * (size_t)n2)) return rc;
  if (int rc = dev_upload(c, &c->d_w2, w2, 2 * (size_t)nw)) return rc;
  c->have_layers = 1;
  return PS_OK;
}

int ps_set_pinv(ps_ctx* h, int irhs, int nrow, int ncol, const double* U, const double* s,
                const double* Vh, const double* col_scale, double eps, const double* f, int col_c,
                int col_d) {
  if (!h) return PS_ERR_ARG;
  Ctx* c = C(h);
  if (!c->have_layers) {
    c->err = "ps_set_pinv: call ps_set_layers first";
    return PS_ERR_STATE;
  }
  if (irhs < 0 || irhs >= c->nrhs || nrow < c->nrow_c || ncol < c->ncol_b || !U || !s || !Vh ||
      !col_scale || !f || !(eps > 0) || col_c < 0 || col_d < 0 || col_c + c->nrb > ncol ||
      col_d + c->nrb > ncol) {
    c->err = "ps_set_pinv: bad argument";
    return PS_ERR_ARG;
  }
  if (int rc = set_device(c)) return rc;
  auto& R = c->rhs[irhs];
  const int nsv = ncol;   // reduced SVD of an nrow x ncol matrix, nrow >= ncol
  c->nsv = nsv;
  const int nrc = c->nrow_c;
  const int nj = 2 * c->Q + 1;
  const int nout0 = c->ncol_b + 2 * c->nrb;
  // field rows: the a1 / a3 columns (eg:154-156: right after a2) when present
  c->nfield = (c->ncol_b + 2 * nj <= ncol) ? 2 * nj : 0;
  const int nout = nout0 + c->nfield;
  // Uh[k][i] = conj(U[i][k]) for the C rows i < nrow_c
  std::vector<double2> uh((size_t)nsv * nrc);
  for (int k = 0; k < nsv; ++k)
    for (int i = 0; i < nrc; ++i) {
      const double* u = U + 2 * ((size_t)i * ncol + k);
      uh[(size_t)k * nrc + i] = make_double2(u[0], -u[1]);
    }
  std::vector<double> sinv(nsv);
  for (int k = 0; k < nsv; ++k) sinv[k] = std::fmin(1.0 / s[k], 1.0 / eps);
  // Vb[o][k] = conj(Vh[k][col(o)]) for the output columns (B cols, c, d, then a1, a3)
  std::vector<int> outcol(nout);
  for (int o = 0; o < c->ncol_b; ++o) outcol[o] = o;
  for (int o = 0; o < c->nrb; ++o) {
    outcol[c->ncol_b + o] = col_c + o;
    outcol[c->ncol_b + c->nrb + o] = col_d + o;
  }
  for (int o = 0; o < c->nfield; ++o) outcol[nout0 + o] = c->ncol_b + o;
  std::vector<double2> vb((size_t)nout * nsv);
  std::vector<double> cs(nout);
  for (int o = 0; o < nout; ++o) {
    cs[o] = col_scale[outcol[o]];
    for (int k = 0; k < nsv; ++k) {
      const double* v = Vh + 2 * ((size_t)k * ncol + outcol[o]);
      vb[(size_t)o * nsv + k] = make_double2(v[0], -v[1]);
    }
  }
  std::vector<double2> fr(nrc);
  for (int i = 0; i < nrc; ++i) fr[i] = make_double2(f[2 * i], f[2 * i + 1]);
  if (int rc = dev_upload(c, &R.d_Uh, uh.data(), uh.size())) return rc;
  if (int rc = dev_upload(c, &R.d_sinv, sinv.data(), sinv.size())) return rc;
  if (int rc = dev_upload(c, &R.d_Vb, vb.data(), vb.size())) return rc;
  if (int rc = dev_upload(c, &R.d_cscale, cs.data(), cs.size())) return rc;
  if (int rc = dev_upload(c, &R.d_f, fr.data(), fr.size())) return rc;
  return PS_OK;
}

int ps_apply_T(ps_ctx* h, const void* beta, void* out, void* stream) {
  if (!h) return PS_ERR_ARG;
  Ctx* c = C(h);
  if (c->p < 0) {
    c->err = "ps_apply_T: geometry not set";
    return PS_ERR_STATE;
  }
  if (!beta || !out) {
    c->err = "ps_apply_T: null pointer";
    return PS_ERR_ARG;
  }
  if (int rc = set_device(c)) return rc;
  auto st = reinterpret_cast<cudaStream_t>(stream);
  const int np = 2 * c->copies + 3;
  if (c->nrhs > 1)
    return ps::m2l_apply_mrhs(c, reinterpret_cast<const double2*>(beta),
                              reinterpret_cast<double2*>(out), 0, nullptr, 0, st);
  const size_t in_stride = (size_t)c->M * c->L, out_stride = (size_t)(c->t_end - c->t_begin) * c->L;
  for (int r = 0; r < c->nrhs; ++r) {
    int rc = ps::m2l_apply_1(c, reinterpret_cast<const double2*>(beta) + r * in_stride,
                           c->d_blochpow + (size_t)r * np + 1,
                           reinterpret_cast<double2*>(out) + r * out_stride, 0, nullptr, nullptr,
                           st);
    if (rc) return rc;
  }
  return PS_OK;
}

int ps_particle_field(ps_ctx* h, const void* beta, int npts, const double* pts, void* out,
                      void* stream) {
  if (!h) return PS_ERR_ARG;
  Ctx* c = C(h);
  if (c->p < 0) {
    c->err = "ps_particle_field: geometry not set";
    return PS_ERR_STATE;
  }
  if (npts < 0 || (npts > 0 && (!beta || !pts || !out))) {
    c->err = "ps_particle_field: bad argument";
    return PS_ERR_ARG;
  }
  if (int rc = set_device(c)) return rc;
  return ps::particle_field(c, reinterpret_cast<const double2*>(beta), pts, nullptr, npts,
                            reinterpret_cast<double2*>(out), nullptr,
                            reinterpret_cast<cudaStream_t>(stream));
}

int ps_particle_field_grad(ps_ctx* h, const void* beta, int npts, const double* pts,
                           const double* dirs, void* out, void* out_dn, void* stream) {
  if (!h) return PS_ERR_ARG;
  Ctx* c = C(h);
  if (c->p < 0) {
    c->err = "ps_particle_field_grad: geometry not set";
    return PS_ERR_STATE;
  }
  if (npts < 0 || (npts > 0 && (!beta || !pts || !dirs || !out || !out_dn))) {
    c->err = "ps_particle_field_grad: bad argument";
    return PS_ERR_ARG;
  }
  if (int rc = set_device(c)) return rc;
  return ps::particle_field(c, reinterpret_cast<const double2*>(beta), pts, dirs, npts,
                            reinterpret_cast<double2*>(out), reinterpret_cast<double2*>(out_dn),
                            reinterpret_cast<cudaStream_t>(stream));
}

int ps_set_field_params(ps_ctx* h, double k1, double k3, const double* c1, const double* c3,
                        const double* inc) {
  if (!h) return PS_ERR_ARG;
  Ctx* c = C(h);
  if (!c1 || !c3 || !inc || !(k1 > 0) || !(k3 > 0)) {
    c->err = "ps_set_field_params: bad argument";
    return PS_ERR_ARG;
  }
  if (int rc = set_device(c)) return rc;
  if (int rc = dev_upload(c, &c->d_inc, inc, 2 * (size_t)c->nrhs)) return rc;
  c->f_k1 = k1;
  c->f_k3 = k3;
  c->f_c1[0] = c1[0];
  c->f_c1[1] = c1[1];
  c->f_c3[0] = c3[0];
  c->f_c3[1] = c3[1];
  c->have_field = 1;
  return PS_OK;
}

int ps_full_columns(const ps_ctx* h) {
  if (!h) return -1;
  const Ctx* c = reinterpret_cast<const Ctx*>(h);
  if (!c->have_layers || c->nfield == 0) return -1;
  return c->ncol_b + 2 * c->nrb + c->nfield;
}

int ps_recover_full(ps_ctx* h, const void* g, void* x, void* stream) {
  if (!h) return PS_ERR_ARG;
  Ctx* c = C(h);
  if (!g || !x) {
    c->err = "ps_recover_full: null pointer";
    return PS_ERR_ARG;
  }
  if (!c->have_layers || c->nsv <= 0) {
    c->err = "ps_recover_full: no empty-grating factors";
    return PS_ERR_STATE;
  }
  if (int rc = set_device(c)) return rc;
  return ps::recover_full(c, reinterpret_cast<const double2*>(g), reinterpret_cast<double2*>(x),
                          reinterpret_cast<cudaStream_t>(stream));
}

int ps_layer_field(ps_ctx* h, const void* x, int npts, const double* pts, const int* layer,
                   void* out, void* stream) {
  if (!h) return PS_ERR_ARG;
  Ctx* c = C(h);
  if (npts < 0 || (npts > 0 && (!x || !pts || !layer || !out))) {
    c->err = "ps_layer_field: bad argument";
    return PS_ERR_ARG;
  }
  if (int rc = set_device(c)) return rc;
  return ps::layer_field(c, reinterpret_cast<const double2*>(x), pts, layer, nullptr, npts, 1,
                         reinterpret_cast<double2*>(out), nullptr,
                         reinterpret_cast<cudaStream_t>(stream));
}

int ps_layer_field_grad(ps_ctx* h, const void* x, int npts, const double* pts, const int* layer,
                        const double* dirs, int incident, void* out, void* out_dn, void* stream) {
  if (!h) return PS_ERR_ARG;
  Ctx* c = C(h);
  if (npts < 0 || (npts > 0 && (!x || !pts || !layer || !dirs || !out || !out_dn))) {
    c->err = "ps_layer_field_grad: bad argument";
    return PS_ERR_ARG;
  }
  if (int rc = set_device(c)) return rc;
  return ps::layer_field(c, reinterpret_cast<const double2*>(x), pts, layer, dirs, npts,
                         incident ? 1 : 0, reinterpret_cast<double2*>(out),
                         reinterpret_cast<double2*>(out_dn), reinterpret_cast<cudaStream_t>(stream));
}

int ps_apply_T_blocks(ps_ctx* h, int part, int nparts, const void* beta, void* out, void* stream) {
  if (!h) return PS_ERR_ARG;
  Ctx* c = C(h);
  if (c->p < 0) {
    c->err = "ps_apply_T_blocks: geometry not set";
    return PS_ERR_STATE;
  }
  if (!beta || !out || nparts < 1 || part < 0 || part >= nparts) {
    c->err = "ps_apply_T_blocks: bad argument";
    return PS_ERR_ARG;
  }
  if (c->nrhs != 1) {
    c->err = "ps_apply_T_blocks: one right-hand side only";
    return PS_ERR_UNSUPPORTED;
  }
  if (int rc = set_device(c)) return rc;
  auto st = reinterpret_cast<cudaStream_t>(stream);
  c->sym_part = part;
  c->sym_nparts = nparts;
  const int rc = ps::m2l_apply_sym(c, reinterpret_cast<const double2*>(beta),
                                   c->d_blochpow + 1, reinterpret_cast<double2*>(out), 0, nullptr,
                                   nullptr, st);
  c->sym_part = 0;
  c->sym_nparts = 1;
  return rc;
}

int ps_schur_finish(ps_ctx* h, const void* v_own, const void* a_own, const void* g, void* y,
                    void* stream) {
  if (!h) return PS_ERR_ARG;
  Ctx* c = C(h);
  if (c->p < 0 || c->rhs.empty()) {
    c->err = "ps_schur_finish: operator not set up";
    return PS_ERR_STATE;
  }
  if (!v_own || !a_own || !y) {
    c->err = "ps_schur_finish: null pointer";
    return PS_ERR_ARG;
  }
  if (c->nrhs != 1) {
    c->err = "ps_schur_finish: one right-hand side only";
    return PS_ERR_UNSUPPORTED;
  }
  if (int rc = set_device(c)) return rc;
  return ps::schur_finish(c, reinterpret_cast<const double2*>(v_own),
                          reinterpret_cast<const double2*>(a_own),
                          reinterpret_cast<const double2*>(g), reinterpret_cast<double2*>(y),
                          reinterpret_cast<cudaStream_t>(stream));
}

int ps_apply_C(ps_ctx* h, const void* beta, void* g, int s_begin, int s_end, void* stream) {
  if (!h) return PS_ERR_ARG;
  Ctx* c = C(h);
  if (c->p < 0 || !c->have_layers) {
    c->err = "ps_apply_C: geometry/layers not set";
    return PS_ERR_STATE;
  }
  if (!beta || !g || s_begin < 0 || s_end > c->M || s_end < s_begin) {
    c->err = "ps_apply_C: bad argument";
    return PS_ERR_ARG;
  }
  if (int rc = set_device(c)) return rc;
  return ps::apply_C(c, reinterpret_cast<const double2*>(beta), reinterpret_cast<double2*>(g),
                     s_begin, s_end, reinterpret_cast<cudaStream_t>(stream));
}

int ps_apply_schur_g(ps_ctx* h, const void* v, const void* g, void* y, void* stream) {
  if (!h) return PS_ERR_ARG;
  Ctx* c = C(h);
  if (c->p < 0 || !c->d_S) {
    c->err = "ps_apply_schur_g: geometry / scattering matrix not set";
    return PS_ERR_STATE;
  }
  if (!v || !y) {
    c->err = "ps_apply_schur_g: null pointer";
    return PS_ERR_ARG;
  }
  if (int rc = set_device(c)) return rc;
  return ps::apply_schur_g(c, reinterpret_cast<const double2*>(v),
                           reinterpret_cast<const double2*>(g), reinterpret_cast<double2*>(y),
                           reinterpret_cast<cudaStream_t>(stream));
}

int ps_apply_schur(ps_ctx* h, const void* v, void* y, void* stream) {
  if (!h) return PS_ERR_ARG;
  Ctx* c = C(h);
  if (c->p < 0 || !c->d_S) {
    c->err = "ps_apply_schur: geometry / scattering matrix not set";
    return PS_ERR_STATE;
  }
  if (!v || !y) {
    c->err = "ps_apply_schur: null pointer";
    return PS_ERR_ARG;
  }
  if (int rc = set_device(c)) return rc;
  return ps::apply_schur(c, reinterpret_cast<const double2*>(v), reinterpret_cast<double2*>(y),
                         reinterpret_cast<cudaStream_t>(stream));
}

int ps_schur_rhs(ps_ctx* h, void* rhs, void* stream) {
  if (!h) return PS_ERR_ARG;
  Ctx* c = C(h);
  if (c->p < 0 || !c->d_S || !ps::factors_ready(c)) {
    c->err = "ps_schur_rhs: geometry / S / layers / pinv not set";
    return PS_ERR_STATE;
  }
  if (!rhs) {
    c->err = "ps_schur_rhs: null pointer";
    return PS_ERR_ARG;
  }
  if (int rc = set_device(c)) return rc;
  return ps::schur_rhs(c, reinterpret_cast<double2*>(rhs), reinterpret_cast<cudaStream_t>(stream));
}

int ps_recover(ps_ctx* h, const void* g, void* x, void* stream) {
  if (!h) return PS_ERR_ARG;
  Ctx* c = C(h);
  if (!ps::factors_ready(c)) {
    c->err = "ps_recover: layers / pinv not set";
    return PS_ERR_STATE;
  }
  if (!g || !x) {
    c->err = "ps_recover: null pointer";
    return PS_ERR_ARG;
  }
  if (int rc = set_device(c)) return rc;
  return ps::recover(c, reinterpret_cast<const double2*>(g), reinterpret_cast<double2*>(x),
                     reinterpret_cast<cudaStream_t>(stream));
}

int ps_krylov_begin(ps_ctx* h, int nrhs, long long n, int maxit, const void* b,
                    const double* bnorm2, void* V, void* stream) {
  if (!h) return PS_ERR_ARG;
  Ctx* c = C(h);
  if (nrhs < 1 || n < 1 || maxit < 1 || !b || !bnorm2 || !V) {
    c->err = "ps_krylov_begin: bad argument";
    return PS_ERR_ARG;
  }
  if (int rc = set_device(c)) return rc;
  return ps::krylov_begin(c, nrhs, n, maxit, reinterpret_cast<const double2*>(b), bnorm2,
                          reinterpret_cast<double2*>(V), reinterpret_cast<cudaStream_t>(stream));
}

int ps_krylov_dot(ps_ctx* h, int k, const void* V, const void* w, void* hout, void* stream) {
  if (!h) return PS_ERR_ARG;
  Ctx* c = C(h);
  if (!V || !w || !hout) {
    c->err = "ps_krylov_dot: null pointer";
    return PS_ERR_ARG;
  }
  if (int rc = set_device(c)) return rc;
  return ps::krylov_dot(c, k, reinterpret_cast<const double2*>(V),
                        reinterpret_cast<const double2*>(w), reinterpret_cast<double2*>(hout),
                        reinterpret_cast<cudaStream_t>(stream));
}

int ps_krylov_axpy(ps_ctx* h, int k, const void* V, const void* hin, void* w, void* stream) {
  if (!h) return PS_ERR_ARG;
  Ctx* c = C(h);
  if (!V || !w || !hin) {
    c->err = "ps_krylov_axpy: null pointer";
    return PS_ERR_ARG;
  }
  if (int rc = set_device(c)) return rc;
  return ps::krylov_axpy(c, k, reinterpret_cast<const double2*>(V),
                         reinterpret_cast<const double2*>(hin), reinterpret_cast<double2*>(w),
                         reinterpret_cast<cudaStream_t>(stream));
}

int ps_krylov_norm2(ps_ctx* h, int nrhs, long long n, const void* w, double* nrm2, void* stream) {
  if (!h) return PS_ERR_ARG;
  Ctx* c = C(h);
  if (nrhs < 1 || n < 1 || !w || !nrm2) {
    c->err = "ps_krylov_norm2: bad argument";
    return PS_ERR_ARG;
  }
  if (int rc = set_device(c)) return rc;
  return ps::krylov_norm2(c, nrhs, n, reinterpret_cast<const double2*>(w), nrm2,
                          reinterpret_cast<cudaStream_t>(stream));
}

int ps_krylov_step(ps_ctx* h, int k, const void* h1, const void* h2, const double* wnorm2,
                   const void* w, void* V, double* status, void* stream) {
  if (!h) return PS_ERR_ARG;
  Ctx* c = C(h);
  if (!h1 || !h2 || !wnorm2 || !w || !V || !status) {
    c->err = "ps_krylov_step: null pointer";
    return PS_ERR_ARG;
  }
  if (int rc = set_device(c)) return rc;
  return ps::krylov_step(c, k, reinterpret_cast<const double2*>(h1),
                         reinterpret_cast<const double2*>(h2), wnorm2,
                         reinterpret_cast<const double2*>(w), reinterpret_cast<double2*>(V), status,
                         reinterpret_cast<cudaStream_t>(stream));
}

int ps_krylov_freeze(ps_ctx* h, const int* active_host, void* stream) {
  if (!h) return PS_ERR_ARG;
  Ctx* c = C(h);
  if (!active_host) {
    c->err = "ps_krylov_freeze: null pointer";
    return PS_ERR_ARG;
  }
  if (int rc = set_device(c)) return rc;
  return ps::krylov_freeze(c, active_host, reinterpret_cast<cudaStream_t>(stream));
}

int ps_krylov_solve(ps_ctx* h, const int* iters_host, const void* V, void* x, void* stream) {
  if (!h) return PS_ERR_ARG;
  Ctx* c = C(h);
  if (!iters_host || !V || !x) {
    c->err = "ps_krylov_solve: null pointer";
    return PS_ERR_ARG;
  }
  if (int rc = set_device(c)) return rc;
  return ps::krylov_solve(c, iters_host, reinterpret_cast<const double2*>(V),
                          reinterpret_cast<double2*>(x), reinterpret_cast<cudaStream_t>(stream));
}

int ps_precompute_coupling(ps_ctx* h, double max_gb) {
  if (!h) return PS_ERR_ARG;
  Ctx* c = C(h);
  if (c->p < 0 || !ps::factors_ready(c)) {
    c->err = "ps_precompute_coupling: geometry / layers / pinv not set";
    return PS_ERR_STATE;
  }
  if (int rc = set_device(c)) return rc;
  return ps::precompute_coupling(c, max_gb * 1e9);
}

int ps_set_symbol_store(ps_ctx* h, double max_gb, size_t* bytes) {
  if (!h) return PS_ERR_ARG;
  Ctx* c = C(h);
  if (bytes) *bytes = c->symstore_bytes;
  if (max_gb < 0) return PS_OK;   // query only
  if (int rc = set_device(c)) return rc;
  c->symstore_max_gb = max_gb;
  if (c->d_symstore && (double)c->symstore_bytes > max_gb * 1e9) {
    ps::dev_free(c->d_symstore);
    c->d_symstore = nullptr;
    c->symstore_bytes = 0;
    c->sst_kb0 = c->sst_nb = -1;
  }
  return PS_OK;
}

int ps_set_k1_variant(ps_ctx* h, int variant) {
  if (!h) return PS_ERR_ARG;
  Ctx* c = C(h);
  if (variant < 0 || variant > 3) {
    c->err = "ps_set_k1_variant: 0 auto, 1 tiled, 2 symmetric (DFMA), 3 symmetric (DMMA)";
    return PS_ERR_ARG;
  }
  c->k1_variant = variant;
  return PS_OK;
}

int ps_set_mrhs_variant(ps_ctx* h, int variant) {
  if (!h) return PS_ERR_ARG;
  Ctx* c = C(h);
  if (variant < 0 || variant > 2) {
    c->err = "ps_set_mrhs_variant: 0 auto, 1 DFMA, 2 DMMA";
    return PS_ERR_ARG;
  }
  c->mrhs_variant = variant;
  return PS_OK;
}

int ps_set_k1_reserve(ps_ctx* h, int sms) {
  if (!h) return PS_ERR_ARG;
  Ctx* c = C(h);
  if (sms < 0 || sms >= c->sm_count) {
    c->err = "ps_set_k1_reserve: need 0 <= sms < SM count";
    return PS_ERR_ARG;
  }
  c->k1_reserve_sms = sms;
  return PS_OK;
}

int ps_set_overlap(ps_ctx* h, int sms) {
  if (!h) return PS_ERR_ARG;
  C(h)->overlap_sms = sms < 0 ? -1 : sms;
  return PS_OK;
}

int ps_set_overlap_order(ps_ctx* h, int k1_first) {
  if (!h) return PS_ERR_ARG;
  C(h)->overlap_k1_first = k1_first ? 1 : 0;
  return PS_OK;
}

int ps_coupling_mode(const ps_ctx* h) { return h ? reinterpret_cast<const Ctx*>(h)->dense : -1; }

int ps_profile(ps_ctx* h, int enable) {
  if (!h) return PS_ERR_ARG;
  Ctx* c = C(h);
  c->profile = enable ? 1 : 0;
  return PS_OK;
}

int ps_stats(ps_ctx* h, long long* launches, double* k1_ms, long long* k1_count) {
  if (!h) return PS_ERR_ARG;
  Ctx* c = C(h);
  // fold completed K1 event pairs into the running total
  for (auto& e : c->k1_events) {
    PS_CUDA_TRY(c, cudaEventSynchronize(e.second));
    float ms = 0.f;
    PS_CUDA_TRY(c, cudaEventElapsedTime(&ms, e.first, e.second));
    c->k1_ms += ms;
    c->k1_count += 1;
    cudaEventDestroy(e.first);
    cudaEventDestroy(e.second);
  }
  c->k1_events.clear();
  if (launches) *launches = c->launches;
  if (k1_ms) *k1_ms = c->k1_ms;
  if (k1_count) *k1_count = c->k1_count;
  return PS_OK;
}

int ps_timeline(ps_ctx* h, double* out3, long long* count) {
  if (!h) return PS_ERR_ARG;
  Ctx* c = C(h);
  for (auto& t : c->timelines) {
    PS_CUDA_TRY(c, cudaEventSynchronize(t.end));
    float a = 0.f, b = 0.f, e = 0.f;
    PS_CUDA_TRY(c, cudaEventElapsedTime(&a, t.fork, t.k1));
    PS_CUDA_TRY(c, cudaEventElapsedTime(&b, t.fork, t.chain));
    PS_CUDA_TRY(c, cudaEventElapsedTime(&e, t.fork, t.end));
    c->tl_sum[0] += a;
    c->tl_sum[1] += b;
    c->tl_sum[2] += e;
    c->tl_count += 1;
    for (cudaEvent_t ev : {t.fork, t.k1, t.chain, t.end}) cudaEventDestroy(ev);
  }
  c->timelines.clear();
  if (out3)
    for (int i = 0; i < 3; ++i) out3[i] = c->tl_count ? c->tl_sum[i] / c->tl_count : 0.0;
  if (count) *count = c->tl_count;
  return PS_OK;
}

int ps_stats_reset(ps_ctx* h) {
  if (!h) return PS_ERR_ARG;
  Ctx* c = C(h);
  long long l;
  double m;
  long long k;
  if (int rc = ps_stats(h, &l, &m, &k)) return rc;
  c->launches = 0;
  c->k1_ms = 0.0;
  c->k1_count = 0;
  if (int rc = ps_timeline(h, nullptr, nullptr)) return rc;
  c->tl_sum[0] = c->tl_sum[1] = c->tl_sum[2] = 0.0;
  c->tl_count = 0;
  return PS_OK;
}

int ps_gmres(ps_ctx* h, const void* rhs, void* x, double tol, int maxit, int* iters,
             double* hist, void* stream) {
  if (!h) return PS_ERR_ARG;
  Ctx* c = C(h);
  if (c->p < 0 || !c->d_S) {
    c->err = "ps_gmres: geometry / scattering matrix not set";
    return PS_ERR_STATE;
  }
  if (!rhs || !x || !iters || maxit < 1 || !(tol > 0)) {
    c->err = "ps_gmres: bad argument";
    return PS_ERR_ARG;
  }
  if (int rc = set_device(c)) return rc;
  return ps::gmres(c, reinterpret_cast<const double2*>(rhs), reinterpret_cast<double2*>(x), tol,
                   maxit, iters, hist, reinterpret_cast<cudaStream_t>(stream));
}

}  // extern "C"
