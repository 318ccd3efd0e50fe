// Standalone (no torch in the process) timing of cuSOLVER SVD drivers on the
// 856 x 781 empty-grating matrix: zgesvd, Xgesvdp, zgesvdj, plus zgetrf/zgetrs.
//   python tools/svd_probe_prep.py A.bin && ./svd_probe A.bin
#include <cuda_runtime.h>
#include <cusolverDn.h>
#include <chrono>
#include <cstdio>
#include <vector>
#include <cmath>

#define CK(x) do { auto e_ = (x); if ((int)e_ != 0) { printf("%s -> %d (line %d)\n", #x, (int)e_, __LINE__); } } while (0)

int main(int argc, char** argv) {
  FILE* f = fopen(argv[1], "rb");
  int m, n;
  fread(&m, 4, 1, f); fread(&n, 4, 1, f);
  std::vector<cuDoubleComplex> hA((size_t)m * n);   // column-major
  fread(hA.data(), 16, hA.size(), f);
  fclose(f);
  cusolverDnHandle_t h; CK(cusolverDnCreate(&h));
  cuDoubleComplex *A, *A0, *U, *V; double* S; int* info;
  cudaMalloc(&A, 16 * (size_t)m * n); cudaMalloc(&A0, 16 * (size_t)m * n);
  cudaMalloc(&U, 16 * (size_t)m * n); cudaMalloc(&V, 16 * (size_t)n * n);
  cudaMalloc(&S, 8 * n); cudaMalloc(&info, 8);
  cudaMemcpy(A0, hA.data(), 16 * (size_t)m * n, cudaMemcpyHostToDevice);
  std::vector<double> s_ref(n), s(n);
  auto now = [] { cudaDeviceSynchronize(); return std::chrono::steady_clock::now(); };
  auto ms = [](auto a, auto b) { return std::chrono::duration<double, std::milli>(b - a).count(); };
  // zgesvd
  int lwork = 0; CK(cusolverDnZgesvd_bufferSize(h, m, n, &lwork));
  cuDoubleComplex* work; cudaMalloc(&work, 16 * (size_t)lwork); double* rwork; cudaMalloc(&rwork, 8 * n);
  for (int it = 0; it < 3; ++it) {
    cudaMemcpy(A, A0, 16 * (size_t)m * n, cudaMemcpyDeviceToDevice);
    auto t0 = now();
    CK(cusolverDnZgesvd(h, 'S', 'S', m, n, A, m, S, U, m, V, n, work, lwork, rwork, info));
    auto t1 = now();
    printf("zgesvd %.2f ms\n", ms(t0, t1));
  }
  cudaMemcpy(s_ref.data(), S, 8 * n, cudaMemcpyDeviceToHost);
  // gesvdp
  cusolverDnParams_t prm; CK(cusolverDnCreateParams(&prm));
  size_t dB = 0, hB = 0;
  CK(cusolverDnXgesvdp_bufferSize(h, prm, CUSOLVER_EIG_MODE_VECTOR, 1, m, n, CUDA_C_64F, A, m, CUDA_R_64F, S, CUDA_C_64F, U, m, CUDA_C_64F, V, n, CUDA_C_64F, &dB, &hB));
  void* dW; cudaMalloc(&dW, dB + 16); std::vector<char> hW(hB + 16);
  for (int it = 0; it < 3; ++it) {
    cudaMemcpy(A, A0, 16 * (size_t)m * n, cudaMemcpyDeviceToDevice);
    double err = 0;
    auto t0 = now();
    CK(cusolverDnXgesvdp(h, prm, CUSOLVER_EIG_MODE_VECTOR, 1, m, n, CUDA_C_64F, A, m, CUDA_R_64F, S, CUDA_C_64F, U, m, CUDA_C_64F, V, n, CUDA_C_64F, dW, dB, hW.data(), hB, info, &err));
    auto t1 = now();
    cudaMemcpy(s.data(), S, 8 * n, cudaMemcpyDeviceToHost);
    double mx = 0; for (int i = 0; i < n; ++i) mx = fmax(mx, fabs(s[i] - s_ref[i]));
    printf("gesvdp %.2f ms  err_sigma %.3e  max|ds|/s0 %.3e\n", ms(t0, t1), err, mx / s_ref[0]);
  }
  // gesvdj
  gesvdjInfo_t jp; CK(cusolverDnCreateGesvdjInfo(&jp));
  CK(cusolverDnXgesvdjSetTolerance(jp, 1e-15)); CK(cusolverDnXgesvdjSetMaxSweeps(jp, 30));
  int lj = 0; CK(cusolverDnZgesvdj_bufferSize(h, CUSOLVER_EIG_MODE_VECTOR, 1, m, n, A, m, S, U, m, V, n, &lj, jp));
  cuDoubleComplex* wj; cudaMalloc(&wj, 16 * (size_t)lj);
  for (int it = 0; it < 2; ++it) {
    cudaMemcpy(A, A0, 16 * (size_t)m * n, cudaMemcpyDeviceToDevice);
    auto t0 = now();
    CK(cusolverDnZgesvdj(h, CUSOLVER_EIG_MODE_VECTOR, 1, m, n, A, m, S, U, m, V, n, wj, lj, info, jp));
    auto t1 = now();
    cudaMemcpy(s.data(), S, 8 * n, cudaMemcpyDeviceToHost);
    double mx = 0; for (int i = 0; i < n; ++i) mx = fmax(mx, fabs(s[i] - s_ref[i]));
    int sw = 0; double res = 0; cusolverDnXgesvdjGetSweeps(h, jp, &sw); cusolverDnXgesvdjGetResidual(h, jp, &res);
    printf("gesvdj %.2f ms sweeps %d residual %.3e max|ds|/s0 %.3e\n", ms(t0, t1), sw, res, mx / s_ref[0]);
  }
  // getrf/getrs on the leading n x n block
  int lw2 = 0; CK(cusolverDnZgetrf_bufferSize(h, n, n, A, m, &lw2));
  cuDoubleComplex* w2; cudaMalloc(&w2, 16 * (size_t)lw2); int* ipiv; cudaMalloc(&ipiv, 4 * n);
  cudaMemcpy(A, A0, 16 * (size_t)m * n, cudaMemcpyDeviceToDevice);
  auto t0 = now();
  CK(cusolverDnZgetrf(h, n, n, A, m, w2, ipiv, info));
  CK(cusolverDnZgetrs(h, CUBLAS_OP_N, n, 41, A, m, ipiv, U, m, info));
  auto t1 = now();
  printf("getrf+getrs %.2f ms (%s)\n", ms(t0, t1), cudaGetErrorString(cudaGetLastError()));
  return 0;
}
