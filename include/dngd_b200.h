/*
 * dngd_b200.h -- C ABI of the B200-native D-NGD step library (libdngd_b200.so).
 *
 * Drop-in boundary for the hot path of the reference package `dngd`
 * (arXiv 2505.21404 reference, /root/reference/pkg/src/dngd).  Every entry
 * point below replaces one numeric call site of the reference; the cited
 * file:line is the reference interface it stands in for.  The Python layer
 * (paper_2505_21404_b200/) keeps the reference's function names and calls
 * these symbols through ctypes.
 *
 * Conventions
 *  - All buffers are DEVICE pointers owned by the caller (PyTorch tensors);
 *    the library never allocates or frees caller-visible memory.  Scratch is
 *    passed explicitly as (work, work_bytes); *_workspace() reports the size.
 *  - Matrices are row-major FP64 with an explicit leading dimension (in
 *    elements).  Leading dimensions of matrices that the tensor-core kernels
 *    stage through TMA must be even (16-byte row pitch) and base pointers
 *    16-byte aligned.
 *  - Every call is asynchronous on the caller's stream (`stream` is a
 *    cudaStream_t passed as void*); nothing synchronises the device except
 *    where stated.  Calls are reentrant: state lives in the dngd_ctx, one
 *    context per calling thread (reference service.py:125-128 fans seeds
 *    over threads).  The calls of one context are stream-ordered: issue them
 *    on one stream at a time (the multi-CTA reductions keep their partials in
 *    the context).  Context creation and destruction never touch the legacy
 *    stream nor synchronise the device, so they are safe while another thread
 *    captures a CUDA graph; destroy a context only after its work has drained.
 *  - Status codes map 1:1 onto the reference's errors.py classes.
 */
#ifndef DNGD_B200_H
#define DNGD_B200_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

/* ---- status codes (reference errors.py:6-36) ---------------------------- */
enum {
  DNGD_OK = 0,
  DNGD_ERR_DIMENSION = 1,   /* DimensionError   errors.py:10 */
  DNGD_ERR_DOMAIN = 2,      /* DomainError      errors.py:23 */
  DNGD_ERR_NOT_PD = 3,      /* -> host retry ladder, then FactorizationError errors.py:27 */
  DNGD_ERR_NONFINITE = 4,   /* NonFiniteError   errors.py:14-20 */
  DNGD_ERR_CUDA = 5,        /* DngdError        errors.py:6 */
  DNGD_ERR_UNSUPPORTED = 6  /* DngdError (shape/config outside this build) */
};

typedef struct dngd_ctx dngd_ctx;

int dngd_version(void);
int dngd_ctx_create(int device, dngd_ctx** out);
int dngd_ctx_destroy(dngd_ctx* ctx);
const char* dngd_ctx_last_error(const dngd_ctx* ctx);

/* ---- dense Gram (replaces solver.py:142-155 `K = J @ J.T; 0.5(K+K^T)`) ----
 * K = J J^T over the first m rows / ncols columns of J (ldJ >= ncols, even).
 * FP64 DMMA tensor-core SYRK, lower tiles only, deterministic split-K; the
 * full symmetric K is written (both triangles).  accumulate != 0 adds to K
 * (column-panel streaming and per-rank partial Grams). */
int dngd_syrk_workspace(dngd_ctx* ctx, int64_t m, int64_t ncols, size_t* bytes);
int dngd_syrk(dngd_ctx* ctx, void* stream, const double* J, int64_t m, int64_t ncols,
              int64_t ldJ, double* K, int64_t ldK, int accumulate, void* work,
              size_t work_bytes);

/* ---- Cholesky with damping (replaces solver.py:161-173 cho_factor) --------
 * L = lower(K) + lam*I copied into L (ldL), then factored in place (lower).
 * info_dev (device int) receives 0 or the 1-based column of the first
 * non-positive / non-finite pivot (LAPACK convention); the host retry ladder
 * (lam *= 10, at most 5 retries) reads it.  dinv receives the inverses of
 * the 64x64 diagonal blocks used by dngd_potrs, followed by the
 * factorisation's scratch (tile flags); size: dngd_potrf_workspace.
 * One persistent dataflow launch + one launch for the block inverses. */
int dngd_potrf_workspace(dngd_ctx* ctx, int64_t m, size_t* dinv_bytes);
int dngd_shift_copy(dngd_ctx* ctx, void* stream, const double* K, int64_t m, int64_t ldK,
                    double lam, double* L, int64_t ldL);
/* Same with the damping read on the device: lam = mult * *lam_dev (the loop's
 * lm_damping(loss) * 10^rejections without a host round trip for the loss). */
int dngd_shift_copy_dev(dngd_ctx* ctx, void* stream, const double* K, int64_t m, int64_t ldK,
                        const double* lam_dev, double mult, double* L, int64_t ldL);
int dngd_potrf(dngd_ctx* ctx, void* stream, double* L, int64_t m, int64_t ldL, double* dinv,
               int* info_dev);

/* ---- triangular solves (replaces solver.py:199,209 cho_solve) -------------
 * b <- (L L^T)^{-1} b in place.  scratch: dngd_potrs_workspace(m) bytes of
 * device memory (the hand-off copies of the block solutions). */
int dngd_potrs_workspace(dngd_ctx* ctx, int64_t m, size_t* bytes);
int dngd_potrs(dngd_ctx* ctx, void* stream, const double* L, int64_t m, int64_t ldL,
               const double* dinv, double* b, double* scratch);

/* ---- streaming matvecs over J (replaces residuals.py:220-227 vjp and
 *      residuals.py:282-292 jvp on the materialised J) ------------------------
 * gemv_t: out = scale * (J^T y + g)   (g may be NULL)      -- solver.py:200,210
 * gemv_n: out = alpha * A x + beta * add  (add may be NULL) -- solver.py:198,208 */
int dngd_gemv_t_workspace(dngd_ctx* ctx, int64_t m, int64_t ncols, size_t* bytes);
int dngd_gemv_t(dngd_ctx* ctx, void* stream, const double* J, int64_t m, int64_t ncols,
                int64_t ldJ, const double* y, const double* g, double scale, double* out,
                void* work, size_t work_bytes);
int dngd_gemv_n(dngd_ctx* ctx, void* stream, const double* A, int64_t m, int64_t ncols,
                int64_t ldA, const double* x, double alpha, const double* add, double beta,
                double* out);

/* ---- generic FP64 tensor-core GEMM  C = alpha * A B^T + beta * C ----------
 * A (M x K, lda), B (N x K, ldb) row-major (K contiguous); batch > 1 uses
 * strides sA, sB, sC (elements).  lower != 0 computes only C[i][j], j <= i. */
int dngd_gemm_nt(dngd_ctx* ctx, void* stream, int64_t M, int64_t N, int64_t K,
                 const double* A, int64_t lda, int64_t sA, const double* B, int64_t ldb,
                 int64_t sB, double* C, int64_t ldc, int64_t sC, int batch, double alpha,
                 double beta, int lower);

/* ---- emulated-FP64 GEMM on the int8 tensor cores (Ozaki scheme) ------------
 * C = A B^T with A (M x K, lda), B (N x K, ldb) row-major doubles, C (M x N, ldc).
 * Every row is split into `slices` (6 or 7) balanced base-256 int8 digits below a per-row
 * power-of-two scale; the S(S+1)/2 digit products that reach FP64 accuracy run
 * as exact int32 tcgen05 MMAs (kind::i8).  Same contract as the FP64 products
 * of solver.py:153 / model.py:88-97 it can replace; K <= 16384.  A row with a
 * non-finite entry yields NaN in its C row/column. */
int dngd_oz_gemm_workspace(dngd_ctx* ctx, int64_t M, int64_t N, int64_t K, int slices,
                           size_t* bytes);
int dngd_oz_gemm_nt(dngd_ctx* ctx, void* stream, int64_t M, int64_t N, int64_t K,
                    const double* A, int64_t lda, const double* B, int64_t ldb, double* C,
                    int64_t ldc, int slices, void* work, size_t work_bytes);

/* ---- vector kernels for the device-resident PCG (solver.py:334-356) ------- */
int dngd_dot(dngd_ctx* ctx, void* stream, int64_t n, const double* x, const double* y,
             double* out_dev);
int dngd_axpby(dngd_ctx* ctx, void* stream, int64_t n, double a, const double* x, double b,
               const double* y, double* out);

/* ---- device-side loop decisions (optimizer.py:148-166 line_search selection and
 *      optimizer.py:226-247 accept / reject bookkeeping), so that consecutive loop
 *      iterations can be queued without a host round trip ---------------------
 * dngd_ls_select: from the ncand line-search losses along etas (descending), the
 * current residual sum of squares rr (loss = rr / 2), the Cholesky info (as a
 * double, 0 = success) and
 * anyd (delta has a nonzero entry, as a double 0/1) writes
 *   sel[0] = eta, sel[1] = loss after the step, sel[2] = status, sel[3] = index
 * with status 0 = accepted, 1 = rejected (no finite candidate, or worse than the
 * current loss when reject_if_worse), 2 = factorisation failed, 3 = non-finite
 * current loss.  Ties pick the larger eta (first minimum, like numpy argmin);
 * anyd = 0 accepts eta = 1 with the current loss.  mult (the damping multiplier
 * 10^rejections) becomes 1 on acceptance, 10 * mult on rejection, and is left
 * alone for status 2 / 3 (the host handles those). */
int dngd_ls_select(dngd_ctx* ctx, void* stream, const double* losses, int ncand,
                   const double* etas, const double* rr, const double* info, const double* anyd,
                   int reject_if_worse, double* mult, double* sel);
/* GA combination (solver.py:211-213) with the gate evaluated on the device:
 * scal[2] = |v|^2, scal[3] = |a|^2 (a may be NULL: no GA); take = |v| > 1e-12 and
 * 2|a| <= 0.5 |v|; out = take ? v + a/2 : v; *anyd = 1.0 if out has a nonzero
 * entry (it must hold 0.0 on entry).  out may alias v. */
int dngd_ga_combine(dngd_ctx* ctx, void* stream, int64_t n, const double* v, const double* a,
                    const double* scal, double* out, double* anyd);
/* out = theta + sel[0] * delta if sel[2] == 0 (accepted), else theta -- the
 * parameter update of optimizer.py:250 (eta = 2^-j, so eta*delta is exact and
 * the fma equals the reference's theta + eta*delta bit for bit) without reading
 * eta back (out may not alias delta; it may alias theta). */
int dngd_theta_update(dngd_ctx* ctx, void* stream, int64_t n, const double* theta,
                      const double* delta, const double* sel, double* out);

/* ---- PINN residual map on device (replaces residuals.py:139-323 for
 *      PinnResidualMap with tanh MLPs; model.py:88-97, jets.py:285-294) ----- */
#define DNGD_MAX_LAYERS 8
#define DNGD_MAX_CLASSES 4
#define DNGD_MAX_GRAD 12

typedef struct {
  int nlayers;                         /* number of affine layers L */
  int widths[DNGD_MAX_LAYERS + 1];     /* widths[0] = input dim, widths[L] = 1 */
} dngd_mlp_desc;

/* r_i = weight * (cu*u + c3*u^3 + sum_g cg[g] d_{grad_dims[g]} u
 *                + cl * sum_{j in lap} d_jj u - f_i)
 * grad channels are numbered 1..ngrad; lap_grad[] lists the grad-channel
 * indices (0-based into grad_dims) summed into the Laplacian channel.
 * inputs (optional): the network-input channels of an input embedding
 * (model.py:148-175), N x nch x widths[0] row-major -- value phi(x), d phi per
 * grad dim, sum of d_jj phi over the Laplacian dims -- replacing points. */
typedef struct {
  int64_t count;                      /* points N */
  int ngrad;
  int nlap;
  int grad_dims[DNGD_MAX_GRAD];
  int lap_grad[DNGD_MAX_GRAD];
  double cg[DNGD_MAX_GRAD];
  double cu, cl, weight;
  const double* points;               /* device, N x widths[0] row-major (identity embedding) */
  const double* f;                    /* device, N data values */
  double c3;                          /* cubic coefficient (Allen-Cahn reaction), 0 if linear */
  const double* inputs;               /* device, N x nch x widths[0], or NULL */
  /* per-point operator (STDE, problems.py:331-402): derivative dims of the grad
   * channels (N x ngrad int32) and channel coefficients (N x nch, replacing
   * cu, cg[], cl; the class weight still applies); NULL = class-wide */
  const int* grad_idx;
  const double* coefs;
} dngd_class_desc;

/* scratch for one assembly / f_vv / loss_many(ncand) evaluation */
int dngd_pinn_workspace(dngd_ctx* ctx, const dngd_mlp_desc* mlp, const dngd_class_desc* classes,
                        int nclass, int ncand, size_t* bytes);

/* r (m) and J[:, col_begin:col_end) (m x (col_end-col_begin), ldJ) in one
 * forward-Laplacian + per-point adjoint pass (residuals.py:241-256).  J may
 * be NULL (residuals only). */
int dngd_assemble(dngd_ctx* ctx, void* stream, const dngd_mlp_desc* mlp, const double* theta,
                  const dngd_class_desc* classes, int nclass, int64_t col_begin,
                  int64_t col_end, double* r, double* J, int64_t ldJ, void* work,
                  size_t work_bytes);

/* r and the full Gram K = J J^T WITHOUT materialising J (replaces
 * residuals.py:241-256 + solver.py:153-154): per layer k and channel pair,
 * K += (Hext_k Hext_k'^T) o (Zbar_k Zbar_k'^T) on the FP64 tensor cores.  K
 * (m x m, ldK) receives both triangles. */
int dngd_gram_factored(dngd_ctx* ctx, void* stream, const dngd_mlp_desc* mlp,
                       const double* theta, const dngd_class_desc* classes, int nclass,
                       double* r, double* K, int64_t ldK, void* work, size_t work_bytes);
/* Tile-sharded variant (multi-GPU): writes only the entries of K
 * covered by part `part` of `nparts` equal tile ranges; the caller zeroes K and
 * sums the parts over the ranks (NCCL all-reduce).  part 0 of 1 == the above. */
int dngd_gram_factored_part(dngd_ctx* ctx, void* stream, const dngd_mlp_desc* mlp,
                            const double* theta, const dngd_class_desc* classes, int nclass,
                            double* r, double* K, int64_t ldK, int part, int nparts, void* work,
                            size_t work_bytes);

/* K (or part `part` of `nparts` of its tiles) from the activations left in
 * act_work by dngd_activations at the same theta: the Gram kernel alone, so the
 * activation pass and the tensor-core Gram can be timed (and scheduled)
 * separately.  Same K as dngd_gram_factored_part, bit for bit. */
int dngd_gram_factored_act(dngd_ctx* ctx, void* stream, const dngd_mlp_desc* mlp,
                           const dngd_class_desc* classes, int nclass, double* K, int64_t ldK,
                           int part, int nparts, void* act_work, size_t act_bytes);

/* ---- factored dual Gram with emulated-FP64 products (solver.py:142-155) -----
 * Same result and tile sharding as dngd_gram_factored_act (K = J J^T from the
 * activations left in act_work by dngd_activations), with every G-space GEMM
 * computed from `slices` (6 or 7) balanced base-256 int8 Ozaki digits per activation row on the
 * tcgen05 tensor cores.  oz_work: dngd_gram_oz_workspace bytes (digit planes). */
int dngd_gram_oz_workspace(dngd_ctx* ctx, const dngd_mlp_desc* mlp,
                           const dngd_class_desc* classes, int nclass, int slices,
                           size_t* bytes);
int dngd_gram_oz_act(dngd_ctx* ctx, void* stream, const dngd_mlp_desc* mlp,
                     const dngd_class_desc* classes, int nclass, double* K, int64_t ldK,
                     int part, int nparts, int slices, void* act_work, size_t act_bytes,
                     void* oz_work, size_t oz_bytes);


/* r plus the forward channels and per-point adjoints (no J) left in work for
 * dngd_jt_factored (the tape sweep of residuals.py:241-256 without the rows) */
int dngd_activations(dngd_ctx* ctx, void* stream, const dngd_mlp_desc* mlp, const double* theta,
                     const dngd_class_desc* classes, int nclass, double* r, void* work,
                     size_t work_bytes);

/* out = scale * J^T w WITHOUT J (replaces residuals.py:220-227 vjp): uses the
 * activations left in act_work by the last dngd_gram_factored / dngd_assemble
 * call for the same theta; scratch sized by dngd_jt_workspace. */
int dngd_jt_workspace(dngd_ctx* ctx, const dngd_mlp_desc* mlp, const dngd_class_desc* classes,
                      int nclass, size_t* bytes);
int dngd_jt_factored(dngd_ctx* ctx, void* stream, const dngd_mlp_desc* mlp,
                     const dngd_class_desc* classes, int nclass, const double* w, double scale,
                     double* out, void* act_work, size_t act_bytes, void* scratch,
                     size_t scratch_bytes);

/* Column slice of the same product: out[j - col_begin] = scale (J^T w)[j] for
 * j in [col_begin, col_end) -- rank p's J_p^T w of the column-sharded step
 * (solver.py:200,210).  Boundaries inside a hidden layer block
 * must fall on one of its rows (a multiple of w_{k+1} from the block start);
 * only the owned rows' tensor-core GEMMs run. */
int dngd_jt_factored_range(dngd_ctx* ctx, void* stream, const dngd_mlp_desc* mlp,
                           const dngd_class_desc* classes, int nclass, const double* w,
                           double scale, double* out, int64_t col_begin, int64_t col_end,
                           void* act_work, size_t act_bytes, void* scratch,
                           size_t scratch_bytes);

/* f_vv = d^2/dt^2 r(theta + t v) at t = 0 (residuals.py:304-317) */
int dngd_fvv(dngd_ctx* ctx, void* stream, const dngd_mlp_desc* mlp, const double* theta,
             const double* v, const dngd_class_desc* classes, int nclass, double* fvv,
             void* work, size_t work_bytes);
/* dngd_fvv / dngd_loss_many reusing x W0(theta) from an activation workspace that
 * holds the last assembly / activation pass AT THE SAME theta (caller's contract;
 * residuals.py:304-317 / 188-201 semantics unchanged).  Only the large-din input
 * layer (din >= 64) uses it: there x W0 is a split-K GEMM over din. */
int dngd_fvv_act(dngd_ctx* ctx, void* stream, const dngd_mlp_desc* mlp, const double* theta,
                 const double* v, const dngd_class_desc* classes, int nclass, double* fvv,
                 void* work, size_t work_bytes, void* act_work, size_t act_bytes);

/* K[:, I] WITHOUT J (replaces the Nystrom sketch J J_I^T of solver.py:259-261):
 * the activations of the sorted landmark rows `landmarks` (host int64, ell of
 * them) are gathered into `scratch` (dngd_gram_cols_workspace bytes) and the
 * factored Gram kernel fills Kc (m x ell, ldKc).  Needs the activations of the
 * same theta in act_work (dngd_activations); linear residual operators only. */
int dngd_gram_cols_workspace(dngd_ctx* ctx, const dngd_mlp_desc* mlp,
                             const dngd_class_desc* classes, int nclass, int ell, size_t* bytes);
int dngd_gram_factored_cols(dngd_ctx* ctx, void* stream, const dngd_mlp_desc* mlp,
                            const dngd_class_desc* classes, int nclass, const int64_t* landmarks,
                            int ell, double* Kc, int64_t ldKc, void* act_work, size_t act_bytes,
                            void* scratch, size_t scratch_bytes);

/* out = J v WITHOUT J (replaces residuals.py:282-292 jvp): the first-order
 * forward t-jets of the f_vv pass (same workspace as dngd_fvv) */
int dngd_jvp_factored(dngd_ctx* ctx, void* stream, const dngd_mlp_desc* mlp,
                      const double* theta, const double* v, const dngd_class_desc* classes,
                      int nclass, double* out, void* work, size_t work_bytes);

/* losses[c] = 0.5 |r(theta + etas[c] * delta)|^2 for c < ncand
 * (residuals.py:188-201 via optimizer.py:148-166); etas is a device array.
 * delta == NULL: theta is an explicit (ncand x n) candidate stack. */
int dngd_loss_many(dngd_ctx* ctx, void* stream, const dngd_mlp_desc* mlp, const double* theta,
                   const double* delta, const double* etas, int ncand,
                   const dngd_class_desc* classes, int nclass, double* losses, void* work,
                   size_t work_bytes);
int dngd_loss_many_act(dngd_ctx* ctx, void* stream, const dngd_mlp_desc* mlp,
                       const double* theta, const double* delta, const double* etas, int ncand,
                       const dngd_class_desc* classes, int nclass, double* losses, void* work,
                       size_t work_bytes, void* act_work, size_t act_bytes);

/* The first non-finite entry of x (n values, rows in class order; class_ends[c]
 * = end row of class c): returns DNGD_ERR_NONFINITE with *class_out (class
 * index) and *point_out (point within the class) when one exists, DNGD_OK
 * otherwise (residuals.py:125-136, errors.py:14-20).  Synchronises `stream`. */
int dngd_nonfinite_report(dngd_ctx* ctx, void* stream, const double* x, int64_t n,
                          const int64_t* class_ends, int nclass, int* class_out,
                          int64_t* point_out);

/* ---- Nystrom-PCG numerics (reference solver.py:237-366) --------------------- */

/* Symmetric eigendecomposition A = V diag(w) V^T of an n x n matrix (the landmark
 * block K_II, solver.py:264 scipy eigh): parallel cyclic two-sided Jacobi in one
 * cooperative launch, threshold rotations until a sweep rotates nothing.
 * Eigenpairs unsorted; *sweeps (device int) receives the sweep count. */
int dngd_syev_workspace(dngd_ctx* ctx, int64_t n, size_t* bytes);
int dngd_syev_jacobi(dngd_ctx* ctx, void* stream, const double* A, int64_t n, int64_t lda,
                     double* w, double* V, int64_t ldv, int* sweeps, void* work,
                     size_t work_bytes);
/* Wt[j, :] = V[:, j] / sqrt(lam_j), Qst[j, :] = V[:, j] sqrt(lam_j) for the kept
 * eigenpairs (lam_j > floor_rel * max lam, solver.py:265-266), zero rows otherwise;
 * *rank = the kept count (device int, may be NULL). */
int dngd_nystrom_scale(dngd_ctx* ctx, void* stream, const double* V, int64_t ldv,
                       const double* lam, int l, double floor_rel, double* Wt, int64_t ldw,
                       double* Qst, int64_t ldq, int* rank);
/* K (l x l PSD) ~ L L^T by diagonally pivoted Cholesky, stopped once every
 * remaining diagonal entry is <= tol * max diag (or at kmax columns): Lt (k x l,
 * row j = column j of L), *k_out = k (device int).  work: 12 l + 64 bytes. */
int dngd_pivoted_cholesky(dngd_ctx* ctx, void* stream, const double* K, int64_t l, int64_t ldk,
                          double tol, int kmax, double* Lt, int64_t ldl, void* work,
                          size_t work_bytes, int* k_out);
/* From the k x k eigenpairs (lam, W) of L^T L: Qst[j, :] = (L W)[:, j] and
 * Wt[j, :] = Qst[j, :] / lam_j for the kept j (lam_j > floor_rel max lam), zero
 * rows otherwise; *rank = kept count. */
int dngd_nystrom_from_chol(dngd_ctx* ctx, void* stream, const double* W, int64_t ldw,
                           const double* lam, int k, const double* Lt, int64_t ldl, int l,
                           double floor_rel, double* Wt, int64_t ldwt, double* Qst,
                           int64_t ldq, int* rank);
/* Mt[r, landmarks[i]] = Qst[r, i] for r < rows (U~[I] = Q, solver.py:272). */
int dngd_nystrom_scatter(dngd_ctx* ctx, void* stream, const double* Qst, int64_t ldq, int rows,
                         int l, const int64_t* landmarks_dev, double* Mt, int64_t ldm);

/* Device-resident CG control flow (solver.py:321-366) over a state block of 13
 * doubles [rho, p.Ap, r.r, r.z, alpha, best |r|, tol |b|, floor, |b|, iteration,
 * stop, warning (1 curvature, 2 collapse), max_iters] and an int arrival flag
 * (zeroed once).  dngd_cg_update_p sets the WHILE condition `cond` of a loop
 * graph (dngd_loop_graph_*): 1 = run another iteration. */
int dngd_cg_init(dngd_ctx* ctx, void* stream, double* state, double tol, int max_iters);
int dngd_cg_after_pap(dngd_ctx* ctx, void* stream, double* state, int64_t m, double* y,
                      double* r, const double* p, const double* Ap);
int dngd_cg_after_r(dngd_ctx* ctx, void* stream, double* state, int64_t m, const double* y,
                    double* ybest, int* flag);
int dngd_cg_update_p(dngd_ctx* ctx, void* stream, double* state, int64_t m, double* p,
                     const double* z, int* flag, uint64_t cond);
int dngd_cg_finish(dngd_ctx* ctx, void* stream, const double* state, int64_t m, double* y,
                   const double* ybest, const double* radd);
int dngd_axmy(dngd_ctx* ctx, void* stream, int64_t m, double c, const double* v,
              const double* u, double* z);

/* A CUDA graph whose only node is a WHILE conditional; its body is captured from
 * the launches issued on `stream` between _begin and _end (thread-local capture
 * mode).  The condition handle is returned for dngd_cg_update_p. */
int dngd_loop_graph_create(dngd_ctx* ctx, void** graph, uint64_t* handle);
int dngd_loop_graph_begin(dngd_ctx* ctx, void* graph, void* stream);
int dngd_loop_graph_end(dngd_ctx* ctx, void* graph, void* stream);
int dngd_loop_graph_launch(dngd_ctx* ctx, void* graph, void* stream);
int dngd_loop_graph_destroy(dngd_ctx* ctx, void* graph);

#ifdef __cplusplus
}
#endif
#endif /* DNGD_B200_H */
