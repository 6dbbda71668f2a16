// clock64 phase marks of the Jacobi eigensolver (CTA 0, first outer rounds)
#define DNGD_JACOBI_TRACE
#include "../../paper_2505_21404_b200/csrc/eig_cg.cu"
#include <cstdio>
#include <vector>
#include <random>
int main(int argc, char** argv) {
  int n = argc > 1 ? atoi(argv[1]) : 64;
  dngd_ctx* ctx = nullptr;
  if (dngd_ctx_create(0, &ctx)) { printf("ctx failed\n"); return 1; }
  std::vector<double> A(n * n);
  std::mt19937_64 g(1); std::normal_distribution<double> nd;
  std::vector<double> B(n * n); for (auto& x : B) x = nd(g);
  for (int i = 0; i < n; ++i) for (int j = 0; j < n; ++j) { double s = 0; for (int k = 0; k < n; ++k) s += B[i*n+k]*B[j*n+k]; A[i*n+j] = s; }
  double *dA, *w, *V; int* sw; void* ws; size_t wb;
  dngd_syev_workspace(ctx, n, &wb);
  cudaMalloc(&dA, n*n*8); cudaMalloc(&w, n*8); cudaMalloc(&V, n*n*8); cudaMalloc(&sw, 4); cudaMalloc(&ws, wb);
  cudaMemcpy(dA, A.data(), n*n*8, cudaMemcpyHostToDevice);
  int rc = dngd_syev_jacobi(ctx, 0, dA, n, n, w, V, n, sw, ws, wb);
  rc |= dngd_syev_jacobi(ctx, 0, dA, n, n, w, V, n, sw, ws, wb);
  cudaDeviceSynchronize();
  long long tr[256]; cudaMemcpy(tr, dngd_jacobi_trace_ptr, sizeof tr, cudaMemcpyDeviceToHost);
  int sweeps; cudaMemcpy(&sweeps, sw, 4, cudaMemcpyDeviceToHost);
  printf("rc %d sweeps %d\n", rc, sweeps);
  for (int i = 1; i < 80; ++i) if (tr[i]) printf("%d:%lld ", i, tr[i] - tr[i-1]);
  printf("\n");
}
