// Host-side internals shared by the .cu translation units.
#pragma once

#include <cuda.h>
#include <cuda_runtime.h>
#include <cudaTypedefs.h>

#include <atomic>
#include <string>

#include "../../include/dngd_b200.h"

struct dngd_ctx {
  int device = 0;
  int num_sms = 148;
  PFN_cuTensorMapEncodeTiled_v12000 encode = nullptr;
  std::string last_error;
  // look-ahead Cholesky: auxiliary stream + fork/join events (created lazily)
  cudaStream_t aux = nullptr;
  cudaStream_t hi = nullptr;  // high-priority stream for the potrf panels
  cudaEvent_t ev_join = nullptr;
  CUtensorMap potrf_mapS, potrf_mapP;  // panel-load boxes over L (encoded per dngd_potrf call)
  cudaEvent_t ev_panel = nullptr, ev_update = nullptr, ev_update2 = nullptr, ev_fork = nullptr;
  // split trailing updates: U1 (next-but-one block column) on aux, U2 (the rest) on aux2
  cudaStream_t aux2 = nullptr;
  cudaEvent_t ev_u1[3] = {nullptr, nullptr, nullptr}, ev_u2[3] = {nullptr, nullptr, nullptr};
  cudaEvent_t ev_join2 = nullptr;
  // multi-CTA dot products: per-CTA partials + arrival counter (calls on one context
  // are stream-ordered; the counter is reset by the last CTA)
  double* dot_part = nullptr;
  unsigned* dot_counter = nullptr;
  cudaStream_t own = nullptr;  // the context's private stream (setup / teardown only)
  unsigned long long* nf_word = nullptr;  // dngd_nonfinite_report: first non-finite index
};

namespace dngd {

constexpr int kDotBlocks = 256;  // fixed CTA count: the summation order is device independent

int set_error(dngd_ctx* ctx, int code, const std::string& msg);
int cuda_status(dngd_ctx* ctx, cudaError_t e, const char* where);

// FP64 tensor-core GEMM engine (gemm.cu).  partial != nullptr selects the
// split-K partial-tile output used by the SYRK (see syrk()).
struct GemmCall {
  long long M = 0, N = 0, K = 0;
  const double* A = nullptr;
  long long lda = 0, sA = 0;
  const double* B = nullptr;
  long long ldb = 0, sB = 0;
  double* C = nullptr;
  long long ldc = 0, sC = 0;
  int batch = 1;
  double alpha = 1.0, beta = 0.0;
  int lower = 0;
  int splits = 1;          // >1 only with partial
  double* partial = nullptr;
};
int gemm_nt(dngd_ctx* ctx, cudaStream_t s, const GemmCall& g);
size_t gemm_splitk_bytes(long long M, long long N, int splits);
int gemm_splitk_choose(dngd_ctx* ctx, long long M, long long N, long long K);
int gemm_nt_splitk(dngd_ctx* ctx, cudaStream_t s, const GemmCall& g, int splits, double* partial,
                   size_t partial_bytes);
int syrk_plan(dngd_ctx* ctx, long long m, long long ncols, int* splits, long long* ntiles,
              size_t* work_bytes);
int syrk(dngd_ctx* ctx, cudaStream_t s, const double* J, long long m, long long ncols,
         long long ldJ, double* K, long long ldK, int accumulate, void* work, size_t wb);

// Ozaki slicing (ozaki.cu): rows x K doubles (pitch ld) -> int8 digits Q[slices][rows][kpad]
// (kpad = K rounded up to 32, zero digits past K) and per-row power-of-two scales;
// a row with a non-finite entry gets scale NaN.
int oz_slice_into(dngd_ctx* ctx, cudaStream_t s, const double* X, long long rows, long long K,
                  long long ld, long long kpad, size_t plane, int slices, int8_t* Q, double* scale);
size_t oz_splitk_bytes(long long M, long long N, long long K, int slices, int splits);
int oz_splitk_choose(dngd_ctx* ctx, long long M, long long N, long long K);
struct OzSplitK {  // oz_gemm_splitk's workspace: planes, scales, partials
  long long kl, kp;
  int8_t *qa, *qb;
  double *sa, *sb, *part;
};
OzSplitK oz_splitk_layout(void* work, long long M, long long N, long long K, int slices, int splits);
int oz_splitk_finish(dngd_ctx* ctx, cudaStream_t s, const OzSplitK& L, long long M, long long N,
                     int slices, int splits, double alpha, double* C, long long ldc);
int oz_gemm_splitk(dngd_ctx* ctx, cudaStream_t s, const double* A, long long lda, const double* B,
                   long long ldb, long long M, long long N, long long K, double alpha, double* C,
                   long long ldc, int slices, int splits, void* work, size_t work_bytes);
int oz_slice(dngd_ctx* ctx, cudaStream_t s, const double* X, long long rows, long long K,
             long long ld, int slices, int8_t* Q, double* scale);
// 3-D TMA map over Q: box {box_bytes (32 or 64), box_rows, slices}, swizzle of the
// same width; rows past the end (and K past kpad) read as zero digits.  64-byte
// rows feed twice the bytes per TMA row request (tools/micro/tma_rate.cu)
int oz_encode(dngd_ctx* ctx, CUtensorMap* map, const int8_t* Q, long long rows, long long kpad,
              int slices, int box_rows, int box_bytes = 32);
// C_z = A_z B_z^T (z < batch) over sliced operands: A_z rows z a_brows .. + M of the
// a_rows-row digit planes QA (scales scA), likewise B; C_z = C + z sC (pitch ldc)
int oz_gemm_batched(dngd_ctx* ctx, cudaStream_t s, const int8_t* QA, const double* scA,
                    long long a_rows, long long a_brows, const int8_t* QB, const double* scB,
                    long long b_rows, long long b_brows, long long kpad, int slices, long long M,
                    long long N, int batch, double* C, long long ldc, long long sC);

}  // namespace dngd
