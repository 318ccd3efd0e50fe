#pragma once
#include <cuda_runtime.h>

#include "ctx.cuh"

// Multipole orders p the M2L kernel is instantiated for.
#define PS_M2L_MAX_P 25
#define PS_M2L_ORDERS(X)                                                                 \
  X(0) X(1) X(2) X(3) X(4) X(5) X(6) X(7) X(8) X(9) X(10) X(11) X(12) X(13) X(14) X(15) \
  X(16) X(17) X(18) X(19) X(20) X(21) X(22) X(23) X(24) X(25)

namespace ps {
// K1s launched on its own stream with a reduced grid; the deterministic
// reduce waits for both the M2L and the coupling chain (SM partitioning).
struct SymOverlap {
  cudaStream_t k1_stream;   // bloch weights + K1s
  int grid;                 // CTAs for K1s
  cudaEvent_t k1_done;      // recorded on k1_stream after K1s
  cudaEvent_t cpl_done;     // coupling chain finished (recorded by the chain callback)
  cudaEvent_t bw_done;      // recorded on k1_stream after the Bloch weights
  // enqueues the coupling chain (its stream waits on bw_done first): called
  // after K1s is queued, so K1s and the chain become ready together and the
  // high-priority K1s CTAs are dispatched first; records cpl_done
  int (*chain)(void*);
  void* chain_arg;
};
int m2l_max_order();
// out: [nt][L] for the owned targets; see m2l.cu for the epilogue modes.
int m2l_apply(Ctx* ctx, const double2* beta, const double2* bpow, double2* out, int mode,
              const double2* v_own, const double2* bsub, cudaStream_t st);
// All ctx->nrhs right-hand sides at once (m2l_mrhs.cu).  beta [nrhs][M][L],
// out [nrhs][nt][L]; bsub (mode 1/2) for RHS r at bsub + r * b_stride.
// One RHS, full target range: symmetric variant (m2l_sym.cu), same contract
// as m2l_apply.
int m2l_apply_sym(Ctx* ctx, const double2* beta, const double2* bpow, double2* out, int mode,
                  const double2* v_own, const double2* bsub, cudaStream_t st,
                  const SymOverlap* ov = nullptr);
bool m2l_sym_selected(const Ctx* ctx);
// dispatch: K1s when ctx owns every target and k1_variant allows it, else K1
int m2l_apply_1(Ctx* ctx, const double2* beta, const double2* bpow, double2* out, int mode,
                const double2* v_own, const double2* bsub, cudaStream_t st);
// >= 12 RHS on the FP64 tensor cores (m2l_mma.cu), same contract as m2l_apply_mrhs.
int m2l_apply_mma(Ctx* ctx, const double2* beta, double2* out, int mode, const double2* bsub,
                  long long b_stride, cudaStream_t st);
int m2l_apply_mrhs_dfma(Ctx* ctx, const double2* beta, double2* out, int mode,
                        const double2* bsub, long long b_stride, cudaStream_t st);
// dispatch for nrhs > 1: K1d (DMMA) when nrhs >= 12 (or forced), else K1m (DFMA)
int m2l_apply_mrhs(Ctx* ctx, const double2* beta, double2* out, int mode, const double2* bsub,
                   long long b_stride, cudaStream_t st);
}  // namespace ps
