/* brsvd.h -- C ABI of the B200-native block randomized SVD (BRSVD) hot path.
 *
 * Drop-in boundary for the reference package `blocksvd`
 * (/root/reference/pkg/src/blocksvd).  The reference is pure Python/numpy, so
 * it has no FFI of its own; each entry point below replaces one Python
 * function on the hot path and is bound from Python with ctypes by
 * paper_1706_07191_b200/_lib.py (see INTEGRATION.md for the binding a
 * maintainer would add to the reference):
 *
 *   brsvd_rsvd        <- rsvd_incore(a, cfg)              rsvd.py:126-141
 *   brsvd_rsvd_stream <- brsvd_run / rsvd_naive_ooc       rsvd.py:188-284
 *                        (row panels streamed from host memory)
 *   brsvd_tsqr        <- tsqr_factor(y)                   kernels.py:139-164
 *   brsvd_small_svd   <- small_svd(b)                     kernels.py:173-188
 *   brsvd_gaussian    <- gaussian_matrix(...)             kernels.py:98-118
 *   brsvd_rpca_*      <- _ialm_rpca_incore update step     rpca.py:188-211
 *
 * Conventions
 *   - dtype codes are the .oocm element codes (store.py:14-15):
 *     1 = binary64, 2 = binary32.
 *   - Tall-skinny matrices (Omega, U, V) are column-major with leading
 *     dimension = rows; Vt (l x n, row-major) is the same memory as V (n x l,
 *     column-major).  A may be row- or column-major (`layout`).
 *   - `where` flags say whether a pointer is host (pageable or pinned) or
 *     device memory.  Host inputs are copied in, host outputs copied out;
 *     calls are synchronous with respect to the host.
 *   - Return value is a status code; brsvd_last_error() gives the message of
 *     the last failing call on the calling thread.
 *   - A context is not re-entrant: use one per thread (and per GPU).
 */
#ifndef BRSVD_H
#define BRSVD_H

#include <stdint.h>

#if defined(__GNUC__)
#define BRSVD_API __attribute__((visibility("default")))
#else
#define BRSVD_API
#endif

#ifdef __cplusplus
extern "C" {
#endif

enum brsvd_status {
  BRSVD_OK = 0,
  BRSVD_ERR_CONFIG = 1,   /* ConfigError   rsvd.py:43-44      */
  BRSVD_ERR_SHAPE = 2,    /* ShapeError    kernels.py:27-28   */
  BRSVD_ERR_BUDGET = 3,   /* BudgetError   store.py:42-47     */
  BRSVD_ERR_OVERFLOW = 4, /* FloatingPointError rsvd.py:84-91 */
  BRSVD_ERR_CUDA = 5,
  BRSVD_ERR_NCCL = 6,
  BRSVD_ERR_ARG = 7
};

enum brsvd_dtype { BRSVD_F64 = 1, BRSVD_F32 = 2 };
enum brsvd_layout { BRSVD_COL_MAJOR = 0, BRSVD_ROW_MAJOR = 1 };
enum brsvd_where { BRSVD_DEVICE = 0, BRSVD_HOST = 1 };

typedef struct brsvd_ctx brsvd_ctx;

/* Mirrors PassStats (store.py:50-79) plus the diagnostics the reference
 * raises as warnings/exceptions. */
typedef struct brsvd_stats {
  int64_t words_read;       /* elements of A read across the boundary   */
  int64_t block_reads;      /* panel / block reads                       */
  int64_t passes_num;       /* full passes = passes_num / passes_den     */
  int64_t passes_den;
  int64_t flop_estimate;    /* reference flop model rsvd.py:175-213       */
  int32_t detected_rank;    /* numerical rank of the sample matrix Y      */
  int32_t core_rank;        /* numerical rank of B^T inside small_svd     */
  double max_abs_y0;        /* max |A Omega|                              */
  double log10_peak_est;    /* log10 max|(A A^T)^q A Omega| (unnormalised) */
  int32_t overflow;         /* 1 when the overflow guard fired            */
  int32_t reserved;
  double seconds_sketch;    /* stage timings (device events)             */
  double seconds_orthonormalize;
  double seconds_form_core;
  double seconds_svd;
} brsvd_stats;

/* Device-side profile of the calls made between begin and end on this
 * context: the big A-streaming products (CUDA events on the context stream)
 * and the number of kernels launched by this thread. */
typedef struct brsvd_profile {
  int64_t big_launches;     /* launches of the A-streaming products        */
  double big_ms;            /* summed event time of those launches          */
  double big_flops;         /* algorithmic flops 2*m*n*l per launch, summed */
  double big_bytes;         /* algorithmic A bytes m*n*elsize, summed       */
  int64_t gpu_launches;     /* every kernel this library launched           */
} brsvd_profile;

BRSVD_API int brsvd_version(void);
BRSVD_API const char* brsvd_last_error(void);

/* Create a context on `device`.  `stream` is a cudaStream_t (NULL: the
 * context creates its own non-blocking stream). */
BRSVD_API int brsvd_ctx_create(int device, void* stream, brsvd_ctx** out);
BRSVD_API int brsvd_ctx_set_stream(brsvd_ctx* ctx, void* stream);
BRSVD_API int brsvd_ctx_destroy(brsvd_ctx* ctx);

/* NCCL communicator of a context, for the row-sharded decomposition
 * (BASELINE config 4): rank 0 draws a unique id
 * (brsvd_nccl_unique_id, 128 bytes), every rank attaches with it; the
 * collectives below then run on the context's stream, in order with its
 * kernels.  libnccl.so.2 is opened at run time (BRSVD_NCCL_LIB overrides);
 * failures return BRSVD_ERR_NCCL.  dtype: 1 f64, 2 f32, 3 int64; op: 0 sum,
 * 2 max.  Buffers are device memory. */
BRSVD_API int brsvd_nccl_unique_id(char* unique_id_128);
BRSVD_API int brsvd_ctx_attach_nccl(brsvd_ctx* ctx, const char* unique_id_128, int nranks,
                                    int rank);
BRSVD_API int brsvd_allreduce(brsvd_ctx* ctx, void* buf, int64_t count, int dtype, int op);
BRSVD_API int brsvd_allgather(brsvd_ctx* ctx, const void* send, void* recv, int64_t count,
                              int dtype);

BRSVD_API int brsvd_profile_begin(brsvd_ctx* ctx);
BRSVD_API int brsvd_profile_end(brsvd_ctx* ctx, brsvd_profile* out);

/* In-core randomized SVD, global power iteration (rsvd_incore, rsvd.py:126).
 *   A      m x n, leading dimension lda, `layout`, in `a_where` memory
 *   k, p, q target rank, oversampling, power exponent (l = k + p)
 *   omega  optional n x l column-major sketch (NULL: generated on device
 *          from `seed`, stream 0, like rsvd.py:135-136)
 *   U      m x l column-major,  sigma  l,  Vt  l x n row-major   (out_where)
 * Returns BRSVD_ERR_OVERFLOW (after filling stats) when the unnormalised
 * reference iteration would trip the guard of rsvd.py:84-91. */
BRSVD_API int brsvd_rsvd(brsvd_ctx* ctx, const void* A, int64_t m, int64_t n, int64_t lda,
               int dtype, int layout, int a_where, int k, int p, int q,
               const void* omega, int omega_where, uint64_t seed, void* U,
               void* sigma, void* Vt, int out_where, brsvd_stats* stats);

/* Paper-literal block randomized SVD (block_range_finder + brsvd_run,
 * rsvd.py:150-215; Alg. 2): the sample is the sum over the column
 * blocks [col_bounds[b], col_bounds[b+1]) of (A_J A_J^T)^q A_J Omega_J, each
 * block's power iteration unnormalised and complete before the next block.
 * nblocks + 1 bounds, col_bounds[0] = 0, col_bounds[nblocks] = n.  With
 * nblocks <= 1 or q = 0 this is brsvd_rsvd.  Other arguments as brsvd_rsvd. */
BRSVD_API int brsvd_rsvd_blocked(brsvd_ctx* ctx, const void* A, int64_t m, int64_t n,
                                 int64_t lda, int dtype, int layout, int a_where, int k,
                                 int p, int q, const void* omega, int omega_where,
                                 uint64_t seed, const int64_t* col_bounds, int nblocks,
                                 void* U, void* sigma, void* Vt, int out_where,
                                 brsvd_stats* stats);

/* Range finder (block_range_finder, rsvd.py:150-185): the sample of
 * brsvd_rsvd_blocked (global power iteration when nblocks <= 1, else the
 * per-block iteration over the column blocks) and its orthonormal basis,
 * with no core projection.  Q is m x l column-major (out_where); it spans the
 * range of the sample like the reference's tsqr Q (a different orthonormal
 * basis of the same span).  stats: words_read / block_reads of the sample
 * pass(es), detected_rank, the exact overflow peak.  Other arguments as
 * brsvd_rsvd_blocked. */
BRSVD_API int brsvd_range_finder(brsvd_ctx* ctx, const void* A, int64_t m, int64_t n,
                                 int64_t lda, int dtype, int layout, int a_where, int k,
                                 int p, int q, const void* omega, int omega_where,
                                 uint64_t seed, const int64_t* col_bounds, int nblocks,
                                 void* Q, int out_where, brsvd_stats* stats);

/* One pass over A -- the A-streaming product of the power iteration and of
 * the core projection (a @ omega, a.T @ y: rsvd.py:94-102, :140):
 *   trans = 0:  C (m x l) = A X,    X (n x l)
 *   trans = 1:  C (n x l) = A^T X,  X (m x l)
 * Device pointers; X and C column-major (ldx, ldc).  fp32 runs on the
 * tcgen05 3xTF32 kernel, fp64 on the fp64 SIMT kernel. */
BRSVD_API int brsvd_sketch_product(brsvd_ctx* ctx, const void* A, int64_t m, int64_t n,
                                   int64_t lda, int dtype, int layout, int trans,
                                   const void* X, int64_t ldx, int64_t l, void* C,
                                   int64_t ldc);

/* brsvd_sketch_product with the per-row (trans = 0) or per-column (trans = 1)
 * maxima |A| of brsvd_absmax (float, device; NULL: computed per call), which
 * set the power-of-two scales of the fp16-split tensor-core product.  A caller
 * issuing several products on the same A computes them once. */
BRSVD_API int brsvd_sketch_product_scaled(brsvd_ctx* ctx, const void* A, int64_t m,
                                          int64_t n, int64_t lda, int dtype, int layout,
                                          int trans, const void* X, int64_t ldx, int64_t l,
                                          void* C, int64_t ldc, const float* amax);

/* Row maxima (m) and column maxima (n) of |A| (fp32 A, device outputs; either
 * may be NULL). */
BRSVD_API int brsvd_absmax(brsvd_ctx* ctx, const void* A, int64_t m, int64_t n, int64_t lda,
                           int dtype, int layout, float* row_max, float* col_max);

/* Fused residual of a rank-l factorisation, one pass over A
 * (relative_frobenius_error, rsvd.py:396-432):
 *   out[0] = ||A - U diag(sigma) Vt||_F^2,   out[1] = ||A||_F^2   (fp64, host)
 * A (m x n, lda, layout), U (m x l column-major, ldu), sigma (l), Vt (l x n
 * row-major, ldv): device pointers of `dtype`.  A column block of a larger
 * matrix is handled by passing Vt + j0 with the full ldv. */
BRSVD_API int brsvd_residual(brsvd_ctx* ctx, const void* A, int64_t m, int64_t n, int64_t lda,
                             int dtype, int layout, const void* U, int64_t ldu,
                             const void* sigma, const void* Vt, int64_t ldv, int64_t l,
                             double* out);

/* Out-of-core randomized SVD of a host-resident A (brsvd_run /
 * rsvd_naive_ooc, rsvd.py:188-284, global power iteration): A is streamed
 * over PCIe in panels of `panel` rows (row-major A) or columns (column-major
 * A) through `nbuf` device buffers, the copy of the next panel overlapping
 * the products on the current one (pinned host memory for true overlap).
 * Costs q + 2 passes over A; stats->words_read / passes report them.
 * Other arguments as brsvd_rsvd. */
BRSVD_API int brsvd_rsvd_stream(brsvd_ctx* ctx, const void* A, int64_t m, int64_t n,
                                int64_t lda, int dtype, int layout, int k, int p, int q,
                                const void* omega, int omega_where, uint64_t seed, void* U,
                                void* sigma, void* Vt, int out_where, int64_t panel, int nbuf,
                                brsvd_stats* stats);

/* brsvd_rsvd_stream with block_power = 1: the paper's two-pass BRSVD
 * (brsvd_run with s > 1 and q >= 1, rsvd.py:150-215): each streamed column
 * panel runs its whole power iteration while resident and the panel samples
 * are summed, then one pass forms B; column-major A only. */
BRSVD_API int brsvd_rsvd_stream_blocked(brsvd_ctx* ctx, const void* A, int64_t m, int64_t n,
                                        int64_t lda, int dtype, int layout, int k, int p,
                                        int q, const void* omega, int omega_where,
                                        uint64_t seed, void* U, void* sigma, void* Vt,
                                        int out_where, int64_t panel, int nbuf,
                                        int block_power, brsvd_stats* stats);

/* Orthonormal basis of range(Y) (tsqr_factor, kernels.py:139-164).
 *   Y m x l column-major (ldy); Q m x l column-major; R (optional) l x l
 *   column-major with Y = Q R.  *detected_rank receives the numerical rank. */
BRSVD_API int brsvd_tsqr(brsvd_ctx* ctx, const void* Y, int64_t m, int64_t l, int64_t ldy,
               int dtype, int where, void* Q, void* R, int32_t* detected_rank);

/* SVD of a short-fat l x n matrix B (small_svd, kernels.py:173-188).
 *   B is given as its transpose Bt (n x l column-major, ldb), which is the
 *   memory of a row-major l x n array.  Outputs W (l x l col-major), sigma
 *   (l), Vt (l x n row-major). */
BRSVD_API int brsvd_small_svd(brsvd_ctx* ctx, const void* Bt, int64_t n, int64_t l,
                    int64_t ldb, int dtype, int where, void* W, void* sigma,
                    void* Vt, int32_t* core_rank);

/* Seeded i.i.d. N(0,1) matrix (gaussian_matrix, kernels.py:98-118):
 * entry (i, j) is a pure function of (seed, stream, row_offset + i, j).
 * out: rows x cols column-major (ld), device memory. */
BRSVD_API int brsvd_gaussian(brsvd_ctx* ctx, void* out, int64_t rows, int64_t cols,
                   int64_t ld, int dtype, uint64_t seed, uint64_t stream,
                   int64_t row_offset);

/* Largest singular value by power iteration on M^T M
 * (spectral_norm_estimate, rpca.py:72-100): stops when the estimate changes
 * by at most tol relative or after max_iterations; *out = 0 for a zero
 * matrix.  M is m x n, dense, `layout`, in `where` memory. */
BRSVD_API int brsvd_spectral_norm(brsvd_ctx* ctx, const void* M, int64_t m, int64_t n,
                                  int64_t ldm, int dtype, int layout, int where,
                                  uint64_t seed, double tol, int max_iterations,
                                  double* out, int32_t* iterations);

/* brsvd_spectral_norm from an injected start vector (host, n doubles; the
 * reference's gaussian_matrix(n, 1, seed, stream_index=7) for parity, NULL:
 * this library's stream-7 sketch column). */
BRSVD_API int brsvd_spectral_norm_start(brsvd_ctx* ctx, const void* M, int64_t m, int64_t n,
                                        int64_t ldm, int dtype, int layout, int where,
                                        uint64_t seed, const double* start, double tol,
                                        int max_iterations, double* out, int32_t* iterations);

/* Inexact-ALM robust PCA with the randomized SVD inside
 * (ialm_rpca / _ialm_rpca_incore, rpca.py:153-213).  lam / mu0 = NaN select
 * the defaults 1/sqrt(max(m, n)) and 1.25/||M||_2.  L and S (m x n, same
 * layout as M) are written to out_where memory; residuals, mus,
 * svd_seconds, iter_seconds (host arrays of max_iterations entries) receive
 * the history.  Non-convergence is not an error (*converged = 0).  `omega`
 * (optional, n x (k+p) column-major, `where` memory) injects the sketch the
 * inner SVD uses every iteration (rpca.py:180-192: same seed each time). */
BRSVD_API int brsvd_ialm(brsvd_ctx* ctx, const void* M, int64_t m, int64_t n,
                         int64_t ldm, int dtype, int layout, int where, int k, int p,
                         int q, uint64_t seed, const void* omega, double lam,
                         double mu0, double rho,
                         double tol, int max_iterations, void* L, void* S,
                         int out_where, int32_t* iterations, int32_t* converged,
                         double* residuals, double* mus, double* svd_seconds,
                         double* iter_seconds);

/* brsvd_ialm whose inner SVDs use the per-block power iteration over the
 * column blocks [col_bounds[b], col_bounds[b+1]) -- the reference's
 * out-of-core branch, which calls brsvd_run with the budget's plan
 * (rpca.py:216-304, :274).  nblocks = 0: brsvd_ialm. */
BRSVD_API int brsvd_ialm_blocked(brsvd_ctx* ctx, const void* M, int64_t m, int64_t n,
                                 int64_t ldm, int dtype, int layout, int where, int k, int p,
                                 int q, uint64_t seed, const void* omega, double lam,
                                 double mu0, double rho, double tol, int max_iterations,
                                 const int64_t* col_bounds, int nblocks, void* L, void* S,
                                 int out_where, int32_t* iterations, int32_t* converged,
                                 double* residuals, double* mus, double* svd_seconds,
                                 double* iter_seconds);

/* Host-streamed IALM (the reference's out-of-core branch, _ialm_rpca_ooc,
 * rpca.py:216-304): M (host, column-major m x n, ld ldm -- e.g. a store's
 * payload), the sparse part S and the dual workspace Y (host, m x n, ld ldm,
 * caller-allocated; pinned memory overlaps the copies) never reside on the
 * device; every pass streams their column blocks col_bounds[0..nblocks]
 * (the memory budget's plan, which is also the inner SVD's block partition:
 * brsvd_run's per-block power iteration, rpca.py:274) through `nslots`
 * device slots, H2D and D2H on separate streams.  L (host, m x n) receives
 * the low-rank part.  History arrays as brsvd_ialm. */
BRSVD_API int brsvd_ialm_stream(brsvd_ctx* ctx, const void* M, int64_t m, int64_t n,
                                int64_t ldm, int dtype, int k, int p, int q, uint64_t seed,
                                const void* omega, double lam, double mu0, double rho,
                                double tol, int max_iterations, const int64_t* col_bounds,
                                int nblocks, void* L, void* S, void* Y, int nslots,
                                int32_t* iterations, int32_t* converged, double* residuals,
                                double* mus, double* svd_seconds, double* iter_seconds);

/* ---- stage entry points for the row-sharded driver ---------------------
 * (paper_1706_07191_b200/distributed.py).  Device pointers only; the small
 * matrices are fp64 column-major.  Each replaces one step of the reference
 * pipeline when the rows of A are spread over ranks and only the small
 * products are all-reduced. */

/* G (k1 x k2, fp64) = X^T W (fp64 accumulation); W == NULL means W = X. */
BRSVD_API int brsvd_gram(brsvd_ctx* ctx, const void* X, int64_t r, int64_t k1, int64_t ldx,
                         int dtype, const void* W, int64_t k2, int64_t ldw, double* G);

/* Rank-revealing Cholesky basis of an (all-reduced) Gram G (l x l fp64,
 * overwritten): with s_j = 1/sqrt(G_jj), factor S G S + shift I = L L^T in
 * column order, dropping columns whose pivot ratio is below drop_ratio
 * (0: none) and columns with G_jj <= col_drop^2 max G_ii.  T (l x l) receives
 * S L^-T with the kept columns first; *kept their number; *rank_ref the
 * |diag R| > rank_tol ||X||_F count (tsqr_factor, kernels.py:155-157). */
BRSVD_API int brsvd_chol_basis(brsvd_ctx* ctx, double* G, int64_t l, double shift,
                               double col_drop, double rank_tol, double drop_ratio,
                               double* T, int32_t* kept, int32_t* rank_ref);

/* out (r x kt) = alpha X T + beta out, X (r x k, dtype), T (k x kt, fp64),
 * out in out_dtype (fp64 accumulation). */
BRSVD_API int brsvd_apply(brsvd_ctx* ctx, const void* X, int64_t r, int64_t k, int64_t ldx,
                          int dtype, const double* T, int64_t kt, void* out, int64_t ldo,
                          int out_dtype, double alpha, double beta);

/* Power-iteration basis change of a replicated Z (n x l): Zout spans range(Z)
 * with restored conditioning (shifted Cholesky QR). */
BRSVD_API int brsvd_normalize(brsvd_ctx* ctx, const void* Z, int64_t n, int64_t l,
                              int64_t ldz, int dtype, void* Zout, int64_t ldo);

/* Per column of U (r x l): the largest |u_ij| and the global index
 * row_offset + i of its first occurrence (vals, idx: host arrays of l). */
BRSVD_API int brsvd_colmax(brsvd_ctx* ctx, const void* U, int64_t r, int64_t l, int64_t ldu,
                           int dtype, int64_t row_offset, double* vals, int64_t* idx);

/* brsvd_colmax plus the signed entry at each argmax, in one host array of
 * 3*l doubles: [max |u_ij| (l) | global row index (l) | u at that index (l)]
 * -- the per-rank candidates of _fix_signs (rsvd.py:105-115) for one
 * all-gather, with no per-column device reads. */
BRSVD_API int brsvd_colmax_entries(brsvd_ctx* ctx, const void* U, int64_t r, int64_t l,
                                   int64_t ldu, int dtype, int64_t row_offset, double* out);

/* One streamed pass over a host-resident row shard A (m x n, `layout`,
 * pinned host memory for overlapped DMA), the per-rank unit of the sharded
 * out-of-core decomposition (rsvd_naive_ooc's passes, rsvd.py:218-284, rows
 * split over ranks).  Row panels of `panel` rows go through `nbuf` device
 * buffers on a copy stream; per panel A_i:
 *   X != NULL (device n x l):  Y_i = A_i X    -> Y rows (device m x l)
 *   Z != NULL (device n x l, fp64):  Z = sum_i A_i^T Y_i  (Y as formed, or
 *                                    as given when X == NULL: B^T = A^T Q)
 * pass_ms (optional): device time of the pass. */
BRSVD_API int brsvd_stream_rows_pass(brsvd_ctx* ctx, const void* A, int64_t m, int64_t n,
                                     int64_t lda, int dtype, int layout, const void* X,
                                     int64_t ldx, int64_t l, void* Y, int64_t ldy, double* Z,
                                     int64_t ldz, int64_t panel, int nbuf, double* pass_ms);

/* brsvd_normalize of an fp64 Z (the all-reduced sum of brsvd_stream_rows_pass)
 * into a basis in `dtype` (fp32: taken to unit order by a power of two first). */
BRSVD_API int brsvd_normalize_f64(brsvd_ctx* ctx, const double* Z, int64_t n, int64_t l,
                                  int64_t ldz, int dtype, void* Zout, int64_t ldo, double* T,
                                  double* scale);

/* brsvd_normalize returning the applied transform: Zout = Z T (T: device
 * l x l fp64, upper triangular on the Cholesky route; for fp32 data its
 * fp32-rounded entries); brsvd_normalize_f64's T / scale (optional) give
 * Zout = (scale Z) T.  The sharded driver keeps them for its exact overflow
 * guard. */
BRSVD_API int brsvd_normalize_t(brsvd_ctx* ctx, const void* Z, int64_t n, int64_t l,
                                int64_t ldz, int dtype, void* Zout, int64_t ldo, double* T);

/* Exact overflow guard of the global power iteration (rsvd.py:84-91): the
 * peak of the reference's unnormalised sample (A A^T)^q A Omega, formed in
 * fp64 from this rank's rows Yq (m x l, column-major, ld m) of the
 * normalised sample and the q applied transforms Ts (device, q x l x l,
 * each upper triangular) with their scales zfac (host, q): max |Yq (prod
 * zfac_i T_i)^-1|. */
BRSVD_API int brsvd_unnormalised_peak(brsvd_ctx* ctx, const void* Yq, int64_t m, int64_t l,
                                      int dtype, int q, const double* Ts, const double* zfac,
                                      double* peak);

/* X[:, j] *= scale[j] (scale: host array of l doubles). */
BRSVD_API int brsvd_scale_cols(brsvd_ctx* ctx, void* X, int64_t r, int64_t l, int64_t ldx,
                               int dtype, const double* scale);

#ifdef __cplusplus
}
#endif
#endif /* BRSVD_H */
