#pragma once
#include <cuda_runtime.h>

#include "ctx.cuh"

namespace ps {
// out[r][pt] = particle (multipole) field of RHS r at pts[pt] (field.cu)
int particle_field(Ctx* c, const double2* beta, const double* pts, int npts, double2* out,
                   cudaStream_t st);
}  // namespace ps
