#pragma once
#include <cuda_runtime.h>

#include "ctx.cuh"

namespace ps {
int block_dot(Ctx* c, int nrhs, int n, int k, int kmax, const double2* V, const double2* w,
              double2* h, cudaStream_t st);
int block_axpy(Ctx* c, int nrhs, int n, int k, int kmax, const double2* V, const double2* h,
               double2* w, cudaStream_t st);
int norm2(Ctx* c, int nrhs, int n, const double2* w, double* out, cudaStream_t st);
int gmres(Ctx* c, const double2* rhs, double2* x, double tol, int maxit, int* iters, double* hist,
          cudaStream_t st);
void gmres_release(Ctx* c);
}  // namespace ps
