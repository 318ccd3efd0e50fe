#pragma once
#include <cuda_runtime.h>

#include "ctx.cuh"

namespace ps {
int apply_C(Ctx* c, const double2* beta, double2* g, int s0, int s1, cudaStream_t st);
int apply_schur_g(Ctx* c, const double2* v, const double2* g, double2* y, cudaStream_t st);
int apply_schur(Ctx* c, const double2* v, double2* y, cudaStream_t st);
int schur_rhs(Ctx* c, double2* rhs, cudaStream_t st);
int recover(Ctx* c, const double2* g, double2* x, cudaStream_t st);
}  // namespace ps
