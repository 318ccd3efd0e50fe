// Standalone timing of cuSOLVER zgebrd + zungbr (Q and P^H) on the 856 x 781
// empty-grating matrix: the device half of a bidiagonal-SVD setup.
#include <cuda_runtime.h>
#include <cusolverDn.h>
#include <chrono>
#include <cstdio>
#include <vector>
#define CK(x) do { auto e_ = (x); if ((int)e_ != 0) printf("%s -> %d (line %d)\n", #x, (int)e_, __LINE__); } while (0)
int main(int argc, char** argv) {
  FILE* f = fopen(argv[1], "rb");
  int m, n;
  if (fread(&m, 4, 1, f) != 1 || fread(&n, 4, 1, f) != 1) return 1;
  std::vector<cuDoubleComplex> hA((size_t)m * n);
  if (fread(hA.data(), 16, hA.size(), f) != hA.size()) return 1;
  fclose(f);
  cusolverDnHandle_t h; CK(cusolverDnCreate(&h));
  cuDoubleComplex *A, *A0, *Q, *P, *tq, *tp, *work; double *d, *e; int* info;
  cudaMalloc(&A, 16 * (size_t)m * n); cudaMalloc(&A0, 16 * (size_t)m * n);
  cudaMalloc(&Q, 16 * (size_t)m * n); cudaMalloc(&P, 16 * (size_t)n * n);
  cudaMalloc(&tq, 16 * n); cudaMalloc(&tp, 16 * n); cudaMalloc(&d, 8 * n); cudaMalloc(&e, 8 * n);
  cudaMalloc(&info, 4);
  cudaMemcpy(A0, hA.data(), 16 * (size_t)m * n, cudaMemcpyHostToDevice);
  int lw1 = 0, lw2 = 0, lw3 = 0;
  CK(cusolverDnZgebrd_bufferSize(h, m, n, &lw1));
  CK(cusolverDnZungbr_bufferSize(h, CUBLAS_SIDE_LEFT, m, n, n, Q, m, tq, &lw2));
  CK(cusolverDnZungbr_bufferSize(h, CUBLAS_SIDE_RIGHT, n, n, n, P, n, tp, &lw3));
  int lw = std::max(lw1, std::max(lw2, lw3));
  cudaMalloc(&work, 16 * (size_t)lw);
  auto now = [] { cudaDeviceSynchronize(); return std::chrono::steady_clock::now(); };
  for (int it = 0; it < 3; ++it) {
    cudaMemcpy(A, A0, 16 * (size_t)m * n, cudaMemcpyDeviceToDevice);
    auto t0 = now();
    CK(cusolverDnZgebrd(h, m, n, A, m, d, e, tq, tp, work, lw, info));
    auto t1 = now();
    cudaMemcpy(Q, A, 16 * (size_t)m * n, cudaMemcpyDeviceToDevice);
    cudaMemcpy2D(P, 16 * n, A, 16 * m, 16 * n, n, cudaMemcpyDeviceToDevice);
    CK(cusolverDnZungbr(h, CUBLAS_SIDE_LEFT, m, n, n, Q, m, tq, work, lw, info));
    CK(cusolverDnZungbr(h, CUBLAS_SIDE_RIGHT, n, n, n, P, n, tp, work, lw, info));
    auto t2 = now();
    printf("gebrd %.2f ms, ungbr Q+P %.2f ms\n",
           std::chrono::duration<double, std::milli>(t1 - t0).count(),
           std::chrono::duration<double, std::milli>(t2 - t1).count());
  }
  std::vector<double> hd(n), he(n);
  cudaMemcpy(hd.data(), d, 8 * n, cudaMemcpyDeviceToHost);
  cudaMemcpy(he.data(), e, 8 * (n - 1), cudaMemcpyDeviceToHost);
  FILE* o = fopen(argv[2], "wb");
  fwrite(hd.data(), 8, n, o); fwrite(he.data(), 8, n - 1, o); fclose(o);
  return 0;
}
