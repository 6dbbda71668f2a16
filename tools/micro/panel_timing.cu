// Phase timing of k_potrf_panel (clock64 marks), standalone.
#define DNGD_PANEL_TIMING
#include "../../paper_2505_21404_b200/csrc/chol.cu"
#include <vector>
#include <cstdio>
int main() {
  const int m = 2800; const long long ld = 2800;
  std::vector<double> h((size_t)m * ld, 0.0);
  for (int i = 0; i < m; ++i) for (int j = 0; j <= i; ++j) h[(size_t)i * ld + j] = (i == j) ? m : 1.0 / (1 + i + j);
  double* L; int* info; cudaMalloc(&L, h.size() * 8); cudaMalloc(&info, 4);
  cudaMemcpy(L, h.data(), h.size() * 8, cudaMemcpyHostToDevice); cudaMemset(info, 0, 4);
  cudaFuncSetAttribute(dngd::k_potrf_panel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)dngd::kDynSmem);
  for (int rep = 0; rep < 3; ++rep) {
    cudaEvent_t a, b; cudaEventCreate(&a); cudaEventCreate(&b);
    cudaEventRecord(a);
    dngd::k_potrf_panel<<<44, 128, dngd::kDynSmem>>>(L, m, ld, 0, info);
    cudaEventRecord(b); cudaEventSynchronize(b);
    float ms; cudaEventElapsedTime(&ms, a, b);
    printf("err %s  kernel %.1f us\n", cudaGetErrorString(cudaGetLastError()), ms * 1e3);
  }
  long long c[4][16]; cudaMemcpyFromSymbol(c, dngd::g_panel_clk, sizeof c);
  for (int b = 0; b < 2; ++b) {
    printf("cta %d:", b);
    for (int k = 1; k < 14; ++k) printf(" %lld", c[b][k] - c[b][k - 1]);
    printf("  total %lld cycles\n", c[b][13] - c[b][0]);
  }
}
