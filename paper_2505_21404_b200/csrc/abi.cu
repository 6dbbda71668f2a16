// Context management, error mapping and the dense-path entry points of the
// C ABI declared in include/dngd_b200.h.

#include <cstdio>
#include <string>

#include "common.cuh"
#include "internal.h"

namespace dngd {

int set_error(dngd_ctx* ctx, int code, const std::string& msg) {
  if (ctx) ctx->last_error = msg;
  return code;
}

int cuda_status(dngd_ctx* ctx, cudaError_t e, const char* where) {
  if (e == cudaSuccess) return DNGD_OK;
  return set_error(ctx, DNGD_ERR_CUDA, std::string(where) + ": " + cudaGetErrorString(e));
}

}  // namespace dngd

using namespace dngd;

extern "C" int dngd_version(void) { return 1; }

extern "C" int dngd_ctx_create(int device, dngd_ctx** out) {
  if (out == nullptr) return DNGD_ERR_DIMENSION;
  *out = nullptr;
  dngd_ctx* ctx = new dngd_ctx();
  ctx->device = device;
  cudaError_t e = cudaSetDevice(device);
  if (e != cudaSuccess) {
    delete ctx;
    return DNGD_ERR_CUDA;
  }
  int sms = 0;
  e = cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, device);
  if (e != cudaSuccess) {
    delete ctx;
    return DNGD_ERR_CUDA;
  }
  ctx->num_sms = sms;
  int major = 0;
  cudaDeviceGetAttribute(&major, cudaDevAttrComputeCapabilityMajor, device);
  if (major != 10) {
    delete ctx;
    return DNGD_ERR_UNSUPPORTED;  // this build is sm_100a only
  }
  void* fn = nullptr;
  cudaDriverEntryPointQueryResult q;
  e = cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &fn, cudaEnableDefault, &q);
  if (e != cudaSuccess || fn == nullptr || q != cudaDriverEntryPointSuccess) {
    delete ctx;
    return DNGD_ERR_CUDA;
  }
  ctx->encode = reinterpret_cast<PFN_cuTensorMapEncodeTiled_v12000>(fn);
  // stream-ordered setup on the context's own non-blocking stream: nothing here may
  // touch the legacy stream or synchronise the device, because another thread may
  // be capturing a CUDA graph at this moment (reentrancy)
  e = cudaStreamCreateWithFlags(&ctx->own, cudaStreamNonBlocking);
  if (e == cudaSuccess) {
    e = cudaMallocAsync(reinterpret_cast<void**>(&ctx->dot_part),
                        (dngd::kDotBlocks + 3) * sizeof(double), ctx->own);
  }
  if (e == cudaSuccess) {
    ctx->dot_counter = reinterpret_cast<unsigned*>(ctx->dot_part + dngd::kDotBlocks);
    ctx->nf_word = reinterpret_cast<unsigned long long*>(ctx->dot_part + dngd::kDotBlocks + 2);
    e = cudaMemsetAsync(ctx->dot_counter, 0, 2 * sizeof(double), ctx->own);
  }
  if (e == cudaSuccess) e = cudaStreamSynchronize(ctx->own);
  if (e != cudaSuccess) {
    if (ctx->dot_part) cudaFreeAsync(ctx->dot_part, ctx->own);
    if (ctx->own) {
      cudaStreamSynchronize(ctx->own);
      cudaStreamDestroy(ctx->own);
    }
    delete ctx;
    return DNGD_ERR_CUDA;
  }
  *out = ctx;
  return DNGD_OK;
}

extern "C" int dngd_ctx_destroy(dngd_ctx* ctx) {
  if (ctx) {
    if (ctx->ev_panel) cudaEventDestroy(ctx->ev_panel);
    if (ctx->ev_update) cudaEventDestroy(ctx->ev_update);
    if (ctx->ev_update2) cudaEventDestroy(ctx->ev_update2);
    if (ctx->ev_fork) cudaEventDestroy(ctx->ev_fork);
    if (ctx->aux) cudaStreamDestroy(ctx->aux);
    if (ctx->aux2) cudaStreamDestroy(ctx->aux2);
    for (int q = 0; q < 3; ++q) {
      if (ctx->ev_u1[q]) cudaEventDestroy(ctx->ev_u1[q]);
      if (ctx->ev_u2[q]) cudaEventDestroy(ctx->ev_u2[q]);
    }
    if (ctx->ev_join2) cudaEventDestroy(ctx->ev_join2);
    if (ctx->hi) cudaStreamDestroy(ctx->hi);
    if (ctx->ev_join) cudaEventDestroy(ctx->ev_join);
    // stream-ordered free (no device-wide synchronisation: see dngd_ctx_create);
    // the caller guarantees its streams no longer run work of this context
    if (ctx->dot_part) cudaFreeAsync(ctx->dot_part, ctx->own);
    if (ctx->own) {
      cudaStreamSynchronize(ctx->own);
      cudaStreamDestroy(ctx->own);
    }
  }
  delete ctx;
  return DNGD_OK;
}

extern "C" const char* dngd_ctx_last_error(const dngd_ctx* ctx) {
  return ctx ? ctx->last_error.c_str() : "null context";
}

extern "C" int dngd_syrk_workspace(dngd_ctx* ctx, int64_t m, int64_t ncols, size_t* bytes) {
  int S;
  long long nt;
  return syrk_plan(ctx, m, ncols, &S, &nt, bytes);
}

extern "C" int dngd_syrk(dngd_ctx* ctx, void* stream, const double* J, int64_t m, int64_t ncols,
                         int64_t ldJ, double* K, int64_t ldK, int accumulate, void* work,
                         size_t work_bytes) {
  return syrk(ctx, static_cast<cudaStream_t>(stream), J, m, ncols, ldJ, K, ldK, accumulate, work,
              work_bytes);
}

extern "C" int dngd_gemm_nt(dngd_ctx* ctx, void* stream, int64_t M, int64_t N, int64_t K,
                            const double* A, int64_t lda, int64_t sA, const double* B,
                            int64_t ldb, int64_t sB, double* C, int64_t ldc, int64_t sC,
                            int batch, double alpha, double beta, int lower) {
  GemmCall g;
  g.M = M;
  g.N = N;
  g.K = K;
  g.A = A;
  g.lda = lda;
  g.sA = sA;
  g.B = B;
  g.ldb = ldb;
  g.sB = sB;
  g.C = C;
  g.ldc = ldc;
  g.sC = sC;
  g.batch = batch;
  g.alpha = alpha;
  g.beta = beta;
  g.lower = lower;
  if (lower && M != N) return set_error(ctx, DNGD_ERR_DIMENSION, "gemm_nt lower needs M == N");
  return gemm_nt(ctx, static_cast<cudaStream_t>(stream), g);
}
