#pragma once
#include <cuda_runtime.h>

#include "ctx.cuh"

namespace ps {
// out[r][pt] = particle (multipole) field of RHS r at pts[pt] (field.cu)
// and, with nrm [npts][2] and out_dn, the derivative along nrm[pt]
int particle_field(Ctx* c, const double2* beta, const double* pts, const double* nrm, int npts,
                   double2* out, double2* out_dn, cudaStream_t st);
// out[r][pt] = empty-grating layer field of RHS r (eval_empty_field; the
// incident wave in layer 1 when incident != 0) at pts[pt] in layer layer[pt]
// (1/2/3; other values -> 0) from x [nrhs][ncol]; with nrm and out_dn also
// the derivative along nrm[pt]
int layer_field(Ctx* c, const double2* x, const double* pts, const int* layer, const double* nrm,
                int npts, int incident, double2* out, double2* out_dn, cudaStream_t st);
}  // namespace ps
