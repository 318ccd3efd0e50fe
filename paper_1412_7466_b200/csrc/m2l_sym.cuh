// Shared between K1s (m2l_sym.cu, DFMA consumers) and K1h (m2l_symh.cu,
// DMMA consumers): the launch arguments and the partial-sum layout that the
// deterministic k1s_reduce consumes.
#pragma once
#include <cuda_runtime.h>

#include <cstddef>

namespace ps {

struct ArgsS {
  const double* centers;   // [M][2]
  const double2* bw;       // [M * ncp][L] bloch-weighted beta per source image
  const double* bws;       // [M * ncp][L] re + im of bw (Karatsuba operand)
  const double2* bwr;      // (-1)^(n-P) bw: coefficients of the reverse apply
  const double* bwsr;      // (-1)^(n-P) bws
  double2* apart;          // [G][maxseg][kTT][L]  forward parts, one per (CTA, block row)
  double2* bpart;          // [NB][kTT][L]         reverse parts, one per cross block
  int M, T, NB, copies, ncp, maxseg;
  long long kb0, nb;       // block range [kb0, kb0 + nb) of this launch (multi-GPU part)
  double period, k2;
  // K1s only: precomputed symbol batches of [kb0, kb0 + nb) (batch g = (block
  // - kb0) * ncp + image at g * SYM double2), or null to generate them
  const double2* symstore;
};

// unordered tile pairs (A <= B), row-major: block k -> (A, B)
__device__ inline long long tri_off(int a, int T) {   // blocks with first tile < a
  return (long long)a * T - (long long)a * (a - 1) / 2;
}

__device__ inline void block_ab(long long k, int T, int& A, int& B) {
  int a = 0;
  // small T: linear scan from a floating estimate
  double disc = (2.0 * T + 1.0) * (2.0 * T + 1.0) - 8.0 * (double)k;
  a = (int)(((2.0 * T + 1.0) - sqrt(disc > 0 ? disc : 0)) * 0.5);
  if (a < 0) a = 0;
  if (a > T - 1) a = T - 1;
  while (a > 0 && tri_off(a, T) > k) --a;
  while (a < T - 1 && tri_off(a + 1, T) <= k) ++a;
  A = a;
  B = a + (int)(k - tri_off(a, T));
}

// K1h: the same symmetric tile-pair schedule with the Toeplitz applies on
// the FP64 tensor cores (m2l_symh.cu).  symh_weights writes K1h's padded
// Bloch-weighted coefficient rows into wts (symh_weight_elems double2) and
// points a's coefficient arrays at them; symh_kernel launches the kernel with
// a's partial-sum pointers.  Both return 0 or a cudaError_t.
size_t symh_weight_elems(int p, int M, int ncp);
int symh_weights(int p, ArgsS* a, const double2* beta, const double2* bpow, double2* wts, int nsm,
                 cudaStream_t st);
int symh_kernel(int p, const ArgsS& a, int grid, cudaStream_t st, int device);

}  // namespace ps
