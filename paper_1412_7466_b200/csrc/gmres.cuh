#pragma once
#include <cuda_runtime.h>

#include "ctx.cuh"

namespace ps {
int krylov_begin(Ctx* c, int nrhs, long long n, int maxit, const double2* b, const double* b2,
                 double2* V, cudaStream_t st);
int krylov_dot(Ctx* c, int k, const double2* V, const double2* w, double2* h, cudaStream_t st);
int krylov_axpy(Ctx* c, int k, const double2* V, const double2* h, double2* w, cudaStream_t st);
int krylov_norm2(Ctx* c, int nrhs, long long n, const double2* w, double* out, cudaStream_t st);
int krylov_step(Ctx* c, int k, const double2* h1, const double2* h2, const double* wn2,
                const double2* w, double2* V, double* status, cudaStream_t st);
int krylov_freeze(Ctx* c, const int* active_host, cudaStream_t st);
int krylov_solve(Ctx* c, const int* iters_host, const double2* V, double2* x, cudaStream_t st);
int gmres(Ctx* c, const double2* rhs, double2* x, double tol, int maxit, int* iters, double* hist,
          cudaStream_t st);
void gmres_release(Ctx* c);
}  // namespace ps
