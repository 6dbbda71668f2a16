// Timeline of the dataflow potrf units (globaltimer marks), standalone.
#define DNGD_DF_TRACE
#include "../../paper_2505_21404_b200/csrc/chol.cu"
#include <cstdio>
#include <vector>
#include <dlfcn.h>
int main(int argc, char** argv) {
  const int m = argc > 1 ? atoi(argv[1]) : 2800;
  const long long ld = m + (m & 1);
  std::vector<double> h((size_t)m * ld, 0.0);
  for (int i = 0; i < m; ++i)
    for (int j = 0; j <= i; ++j) h[(size_t)i * ld + j] = (i == j) ? m : 1.0 / (1 + i + j);
  double *L, *ws; int* info;
  const long long nblk = (m + 63) / 64;
  cudaMalloc(&L, h.size() * 8); cudaMalloc(&info, 4);
  size_t wsb; dngd_ctx ctx;
  ctx.encode = nullptr;
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
  static unsigned long long tr[8192][4];
  cudaMemcpyFromSymbol(tr, dngd::g_df_trace, sizeof tr);
  const int nunits = nblk * (nblk - 1) / 2 + 1;
  unsigned long long t0 = ~0ull;
  for (int u = 0; u < nunits; ++u) if (tr[u][0] < t0) t0 = tr[u][0];
  // per column: pair unit (start, acc, end) and the first single (start, acc, Ljj, end)
  int u = 0;
  for (int j = 0; j < nblk; ++j) {
    const int nu = j < nblk - 1 ? nblk - j - 1 : 1;
    auto us = [&](unsigned long long v) { return v ? (double)(v - t0) * 1e-3 : -1.0; };
    printf("col %3d pair: start %8.1f acc %8.1f end %8.1f", j, us(tr[u][0]), us(tr[u][1]), us(tr[u][3]));
    if (nu > 1) printf(" | single(j+2): start %8.1f acc %8.1f Ljj %8.1f end %8.1f", us(tr[u + 1][0]), us(tr[u + 1][1]), us(tr[u + 1][2]), us(tr[u + 1][3]));
    printf("\n");
    u += nu;
  }
}
