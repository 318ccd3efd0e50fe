#pragma once
#include <cuda_runtime.h>

#include "ctx.cuh"

namespace ps {
// out[r][pt] = particle (multipole) field of RHS r at pts[pt] (field.cu)
int particle_field(Ctx* c, const double2* beta, const double* pts, int npts, double2* out,
                   cudaStream_t st);
// out[r][pt] = empty-grating layer field of RHS r (eval_empty_field, total=True)
// at pts[pt] in layer layer[pt] (1/2/3; other values -> 0) from x [nrhs][ncol]
int layer_field(Ctx* c, const double2* x, const double* pts, const int* layer, int npts,
                double2* out, cudaStream_t st);
}  // namespace ps
