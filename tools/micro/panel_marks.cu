// clock64 phase marks of the potrf panel kernel (last panel with >= 2 CTAs).
#define DNGD_PANEL_TIMING
#include "../../paper_2505_21404_b200/csrc/chol.cu"
#include <cstdio>
#include <vector>
int main(int argc, char** argv) {
  const int m = argc > 1 ? atoi(argv[1]) : 2800;
  const long long ld = m + (m & 1);
  std::vector<double> h((size_t)m * ld, 0.0);
  for (int i = 0; i < m; ++i)
    for (int j = 0; j <= i; ++j) h[(size_t)i * ld + j] = (i == j) ? m : 1.0 / (1 + i + j);
  double *L, *ws; int* info;
  cudaMalloc(&L, h.size() * 8); cudaMalloc(&info, 4);
  size_t wsb; dngd_ctx ctx;
  cudaDriverEntryPointQueryResult q;
  cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", reinterpret_cast<void**>(&ctx.encode), cudaEnableDefault, &q);
  dngd_potrf_workspace(&ctx, m, &wsb);
  cudaMalloc(&ws, wsb);
  for (int rep = 0; rep < 3; ++rep) {
    cudaMemcpy(L, h.data(), h.size() * 8, cudaMemcpyHostToDevice);
    cudaEvent_t a, b; cudaEventCreate(&a); cudaEventCreate(&b);
    cudaEventRecord(a);
    int rc = dngd_potrf(&ctx, nullptr, L, m, ld, ws, info);
    cudaEventRecord(b); cudaEventSynchronize(b);
    float ms; cudaEventElapsedTime(&ms, a, b);
    printf("rc %d err %s  potrf %.1f us\n", rc, cudaGetErrorString(cudaGetLastError()), ms * 1e3);
  }
  long long c[4][16]; cudaMemcpyFromSymbol(c, dngd::g_panel_clk, sizeof c);
  for (int b = 0; b < 2; ++b) {
    printf("cta %d: load+fused %lld |", b, c[b][1] - c[b][0]);
    for (int t = 0; t < 4; ++t)
      printf(" f %lld t %lld u %lld |", c[b][2 + 3 * t] - c[b][1 + 3 * t], c[b][3 + 3 * t] - c[b][2 + 3 * t], c[b][4 + 3 * t] - c[b][3 + 3 * t]);
    printf(" total %lld\n", c[b][13] - c[b][0]);
  }
  long long pre[4][4][16]; cudaMemcpyFromSymbol(pre, dngd::g_panel_pre, sizeof pre);
  for (int b = 0; b < 2; ++b)
    for (int w = 0; w < 4; ++w) {
      printf("cta %d warp %d arrive (rel. to phase start):", b, w);
      for (int k = 1; k < 14; ++k) printf(" %lld", pre[b][w][k] - c[b][k - 1]);
      printf("\n");
    }
}
