// Internal state behind the opaque ps_ctx handle of include/periscat_b200.h.
#pragma once
#include <cuda_runtime.h>

#include <cstdint>
#include <string>
#include <vector>
#ifdef PS_CANARY
#include <mutex>
#include <unordered_map>
#endif

#include "../../include/periscat_b200.h"

namespace ps {

struct Dev2 {  // tiny RAII-free device buffer record (freed in ps_destroy)
  void* ptr = nullptr;
  size_t bytes = 0;
};

struct EmptyState;   // device empty-grating setup (empty.cu)
struct Krylov;       // device Arnoldi / Givens state (gmres.cu)

struct RhsData {          // per right-hand side (incidence angle)
  double2 bloch{1.0, 0.0};
  // A^+ factors restricted to what the Schur correction touches
  double2* d_Uh = nullptr;    // [nsv][nrow_c]  = conj(U)^T restricted to C rows
  double* d_sinv = nullptr;   // [nsv]  min(1/s, 1/eps)
  double2* d_Vb = nullptr;    // [ncol_b + 2*nrb][nsv] = conj(Vh)^T rows (B cols, c, d)
  double* d_cscale = nullptr; // [ncol_b + 2*nrb]
  double2* d_f = nullptr;     // [nrow_c] rhs f restricted to C rows
  // pre-assembled coupling blocks (coupling_dense.cu), Bloch weights folded in
  double2* d_CT = nullptr;    // [(dcs1-dcs0) L][nrow_c]
  double2* d_B = nullptr;     // [Mt L][ncol_b]
};

struct Ctx {
  int device = 0;
  int sm_count = 148;
  std::string err;

  // geometry (all M inclusions; sources)
  int M = 0, p = -1, L = 0, copies = 1;
  double period = 1.0, k2 = 1.0;
  double* d_centers = nullptr;  // [M][2]
  std::vector<double> h_centers;
  int t_begin = 0, t_end = 0;   // owned targets [t_begin, t_end)

  // scattering matrix
  int s_diag = 1;
  double2* d_S = nullptr;       // [L] or [L][L]
  double* d_rot = nullptr;      // [M] rotations (dense only), may be null

  // layer coupling (shared by all RHS)
  int have_layers = 0;
  int n1 = 0, n2 = 0, nw = 0, Q = 0;
  double x2[2] = {0, 0};
  double* d_g1 = nullptr;   // [n1][5]: x, y, nx, ny, w
  double* d_g2 = nullptr;   // [n2][5]
  double* d_w2 = nullptr;   // [nw][2] left-wall L2 nodes
  int nrow_c = 0;           // 2*n1 + 2*n2 + 2*nw
  int ncol_b = 0;           // 2*n1 + 2*n2 + (2Q+1)
  int nrb = 0;              // Rayleigh-Bloch orders per direction (c, d)
  int nsv = 0;              // number of singular values
  int nfield = 0;           // extra restricted-V rows kept for field evaluation (a1, a3 columns)
  // layer-field evaluation (ps_layer_field): k1, k3, expansion centres 1 / 3,
  // incident wave vector per RHS k1 (cos theta, sin theta)
  int have_field = 0;
  double f_k1 = 0, f_k3 = 0, f_c1[2] = {0, 0}, f_c3[2] = {0, 0};
  double* d_inc = nullptr;  // [nrhs][2]
  int k1_variant = 0;       // 0 auto (K1s when all targets owned), 1 tiled K1, 2 symmetric K1s
  int mrhs_variant = 0;     // 0 auto (K1d DMMA for >= 12 RHS), 1 DFMA K1m, 2 DMMA K1d
  int dense = 0;            // 1: apply C and B from the pre-assembled matrices
  int dcs0 = 0, dcs1 = 0;   // source range the stored C^T covers
  // SM partitioning (1 RHS, K1s + dense coupling): K1s runs on sm_count -
  // overlap_sms CTAs in a high-priority stream while the HBM-bound coupling
  // chain streams on the remaining SMs in a low-priority stream
  int sym_part = 0, sym_nparts = 1;   // K1s block range (ps_apply_T_blocks)
  int k1_reserve_sms = 0;   // single-RHS M2L grids leave this many SMs free (multi-GPU overlap)
  int overlap_sms = 4;      // < 0: serial (swept with tools/probe_timeline.py at cfg3: 2 was best with the 1.92 ms K1s, 4 with the 1.74 ms staged one)
  int overlap_k1_first = 0; // 1: queue the coupling chain behind K1s (see schur_overlapped)
  cudaStream_t s_hi = nullptr, s_lo = nullptr;
  cudaEvent_t ev_fork = nullptr, ev_k1 = nullptr, ev_cpl = nullptr, ev_bw = nullptr;

  // right-hand sides
  int nrhs = 1;
  std::vector<RhsData> rhs;
  double2* d_blochpow = nullptr;  // [nrhs][2*copies+3]: bloch^l, l=-(copies+1)..copies+1

  // K1s symbol store: every batch of translation symbols of the launch's
  // block range, in the kernel's shared-memory layout, built once per
  // geometry (symbols depend on the centres, k2, period and copies only)
  double2* d_symstore = nullptr;
  size_t symstore_bytes = 0;
  long long sst_kb0 = -1, sst_nb = -1;
  int sst_geom = -1, sst_p = -1;
  int geom_gen = 0;                 // bumped by ps_set_geometry
  double symstore_max_gb = 32.0;    // 0: regenerate the symbols in every launch
  bool k1s_stage = true;            // store-fed K1s stages its coefficient rows in shared memory (env PS_K1S_STAGE=0: off)

  // workspaces
  double2* d_partial = nullptr;
  size_t partial_elems = 0;
  double2* d_work = nullptr;       // misc per-call workspace
  size_t work_elems = 0;

  // device empty-grating assembly + SVD (ps_setup_empty, empty.cu)
  EmptyState* empty = nullptr;
  Krylov* krylov = nullptr;        // GMRES state + scratch (gmres.cu)
  int svd_workers = 4;             // concurrent cuSOLVER streams for multi-RHS setup

  std::vector<void*> owned;        // everything cudaMalloc'ed

  // instrumentation (ps_stats): kernel launches issued by this context and,
  // when enabled, CUDA-event time of every K1 (m2l_kernel) launch
  long long launches = 0;
  int profile = 0;
  double k1_ms = 0.0;
  long long k1_count = 0;
  std::vector<std::pair<cudaEvent_t, cudaEvent_t>> k1_events;
  // overlapped-step timeline (profile mode): events at the fork, K1s end,
  // coupling-chain end and step end; folded by ps_timeline
  struct Timeline {
    cudaEvent_t fork, k1, chain, end;
  };
  std::vector<Timeline> timelines;
  cudaEvent_t tl_k1 = nullptr;     // set by launch_s for the current overlapped step
  double tl_sum[3] = {0, 0, 0};
  long long tl_count = 0;
};

inline Ctx* C(ps_ctx* h) { return reinterpret_cast<Ctx*>(h); }

// the coupled (layer) entry points need the A^+ factors of EVERY right-hand
// side; ps_set_rhs_bloch drops them all when the RHS count changes
inline bool factors_ready(const Ctx* c) {
  if (!c->have_layers || c->nsv <= 0 || c->rhs.empty()) return false;
  for (const auto& r : c->rhs)
    if (!r.d_Uh || !r.d_sinv || !r.d_Vb || !r.d_cscale || !r.d_f) return false;
  return true;
}

// cudaFuncSetAttribute is per device: a launcher keeps one bit per device it
// has configured (a repeated call from racing threads is harmless)
inline bool first_on_device(unsigned long long* mask, int device) {
  const unsigned long long bit = 1ull << (device & 63);
  if (*mask & bit) return false;
  *mask |= bit;
  return true;
}

// Device memory of every context comes from the device's stream-ordered
// default pool with a 32 GiB release threshold: freed blocks stay cached, so a
// new context (e.g. each solve_full) reuses the previous one's coupling
// blocks, symbol store and Krylov basis instead of paying cudaMalloc/cudaFree
// of ~3.5 GB per solve at cfg3.
// Allocation and free are rare (setup, growth, destroy) and fully
// synchronise, so the non-blocking worker streams never race them.
#ifdef PS_CANARY
// Guard-band build (tools/canary_run.sh; compute-sanitizer is not available on
// the GPU pool): every context allocation gets kCanaryBytes of 0xA5 after its
// end, verified when it is freed and by ps_canary_check() -- any kernel
// writing past a workspace it owns is counted.
constexpr size_t kCanaryBytes = 1 << 16;
struct CanaryReg {
  std::mutex mu;
  std::unordered_map<void*, size_t> live;
  long long violations = 0;
};
inline CanaryReg& canary_reg() {
  static CanaryReg r;
  return r;
}
inline long long canary_bad_bytes(void* p, size_t bytes) {
  std::vector<unsigned char> h(kCanaryBytes);
  cudaDeviceSynchronize();
  if (cudaMemcpy(h.data(), static_cast<char*>(p) + bytes, kCanaryBytes, cudaMemcpyDeviceToHost) !=
      cudaSuccess)
    return -1;
  long long bad = 0;
  for (unsigned char b : h) bad += (b != 0xA5);
  return bad;
}
#endif

inline cudaError_t dev_malloc_raw(void** p, size_t bytes) {
  static int pool_ready[64] = {0};
  int dev = 0;
  cudaError_t e = cudaGetDevice(&dev);
  if (e != cudaSuccess) return e;
  if (dev >= 0 && dev < 64 && !pool_ready[dev]) {
    cudaMemPool_t pool;
    if ((e = cudaDeviceGetDefaultMemPool(&pool, dev)) != cudaSuccess) return e;
    uint64_t thr = 32ull << 30;
    if ((e = cudaMemPoolSetAttribute(pool, cudaMemPoolAttrReleaseThreshold, &thr)) != cudaSuccess)
      return e;
    pool_ready[dev] = 1;
  }
#ifdef PS_CANARY
  if ((e = cudaMallocAsync(p, bytes + kCanaryBytes, 0)) != cudaSuccess) return e;
  if ((e = cudaMemsetAsync(static_cast<char*>(*p) + bytes, 0xA5, kCanaryBytes, 0)) != cudaSuccess)
    return e;
  {
    std::lock_guard<std::mutex> g(canary_reg().mu);
    canary_reg().live[*p] = bytes;
  }
#else
  if ((e = cudaMallocAsync(p, bytes, 0)) != cudaSuccess) return e;
#endif
  return cudaStreamSynchronize(0);
}
template <class T>
inline cudaError_t dev_malloc(T** p, size_t bytes) {
  return dev_malloc_raw(reinterpret_cast<void**>(p), bytes);
}
inline void dev_free(void* p) {
  if (!p) return;
  cudaDeviceSynchronize();
#ifdef PS_CANARY
  {
    std::lock_guard<std::mutex> g(canary_reg().mu);
    auto it = canary_reg().live.find(p);
    if (it != canary_reg().live.end()) {
      const long long bad = canary_bad_bytes(p, it->second);
      if (bad) canary_reg().violations += bad;
      canary_reg().live.erase(it);
    }
  }
#endif
  cudaFreeAsync(p, 0);
  cudaStreamSynchronize(0);
}

}  // namespace ps

#define PS_CUDA_TRY(ctx, call)                                                 \
  do {                                                                         \
    cudaError_t e_ = (call);                                                   \
    if (e_ != cudaSuccess) {                                                   \
      (ctx)->err = std::string(#call) + ": " + cudaGetErrorString(e_);         \
      return PS_ERR_CUDA;                                                      \
    }                                                                          \
  } while (0)
