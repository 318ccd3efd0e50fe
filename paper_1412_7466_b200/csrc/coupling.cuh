#pragma once
#include <cuda_runtime.h>

#include "ctx.cuh"

namespace ps {
int apply_C(Ctx* c, const double2* beta, double2* g, int s0, int s1, cudaStream_t st);
int apply_schur_g(Ctx* c, const double2* v, const double2* g, double2* y, cudaStream_t st);
int apply_schur(Ctx* c, const double2* v, double2* y, cudaStream_t st);
int schur_finish(Ctx* c, const double2* v_own, const double2* a_own, const double2* g,
                 double2* y, cudaStream_t st);
int schur_rhs(Ctx* c, double2* rhs, cudaStream_t st);
int recover(Ctx* c, const double2* g, double2* x, cudaStream_t st);
// all empty-grating unknowns x [nrhs][ncol] in the reference column order
int recover_full(Ctx* c, const double2* g, double2* x, cudaStream_t st);
// coupling_dense.cu
int precompute_coupling(Ctx* c, double max_bytes);
void release_dense_coupling(Ctx* c);
int dense_apply_C(Ctx* c, int r, const double2* v_r, double2* gpart, double2* g_r, cudaStream_t st);
int dense_apply_B(Ctx* c, int r, const double2* x_r, double2* b_r, cudaStream_t st);
size_t dense_gpart_elems(const Ctx* c);

}  // namespace ps
