// C++ runtime for the BRSVD hot path: device context, stream-ordered scratch
// buffers, kernel launchers, rank-revealing orthonormalisation and the
// in-core randomized SVD pipeline.
//
// Algorithm map (reference: /root/reference/pkg/src/blocksvd):
//   rsvd_device      <- rsvd_incore        rsvd.py:126-141 (global power iter.)
//   orth_full        <- tsqr / tsqr_factor kernels.py:139-170
//   small_svd_device <- small_svd          kernels.py:173-188
//   fix_signs        <- _fix_signs         rsvd.py:105-115
//   overflow guard   <- _check_overflow    rsvd.py:84-91
#pragma once
#include <algorithm>
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <vector>

#include "common.cuh"
#include "gemm_simt.cuh"
#include "chol.cuh"
#include "jacobi.cuh"
#include "jacobi_cluster.cuh"
#include "small_kernels.cuh"

namespace brsvd {

struct Ctx {
  int device = 0;
  cudaStream_t stream = nullptr;
  bool own_stream = false;
  unsigned long long* h_pinned = nullptr;  // small pinned readback area
  int num_sms = kNumSMs;
  int cc_major = 0, cc_minor = 0;
  size_t max_smem_optin = 0;
  // profiling of the big A-streaming products (brsvd_profile_begin/end)
  bool prof = false;
  std::vector<cudaEvent_t> prof_ev;  // start/stop pairs
  double prof_flops = 0.0, prof_bytes = 0.0;
  long long prof_launch0 = 0;
};

// Brackets one big-product launch with events when profiling is on.
struct ProfScope {
  Ctx& c;
  bool on;
  ProfScope(Ctx& c_, double flops, double bytes) : c(c_), on(c_.prof) {
    if (!on) return;
    cudaEvent_t e;
    BRSVD_CUDA(cudaEventCreate(&e));
    BRSVD_CUDA(cudaEventRecord(e, c.stream));
    c.prof_ev.push_back(e);
    c.prof_flops += flops;
    c.prof_bytes += bytes;
  }
  ~ProfScope() {
    if (!on) return;
    cudaEvent_t e;
    if (cudaEventCreate(&e) == cudaSuccess) {
      cudaEventRecord(e, c.stream);
      c.prof_ev.push_back(e);
    }
  }
};

// Stream-ordered device buffer (cudaMallocAsync from the device default pool).
template <typename T>
struct DBuf {
  T* p = nullptr;
  size_t n = 0;
  cudaStream_t s = nullptr;
  DBuf() = default;
  DBuf(Ctx& c, size_t count) { alloc(c, count); }
  void alloc(Ctx& c, size_t count) {
    release();
    s = c.stream;
    n = count;
    if (count) BRSVD_CUDA(cudaMallocAsync((void**)&p, count * sizeof(T), s));
  }
  void release() {
    if (p) cudaFreeAsync(p, s);
    p = nullptr;
    n = 0;
  }
  ~DBuf() { release(); }
  DBuf(const DBuf&) = delete;
  DBuf& operator=(const DBuf&) = delete;
  operator T*() const { return p; }
};

inline int grid_for(int64_t total, int threads = 256, int max_blocks = 148 * 16) {
  int64_t b = ceil_div(std::max<int64_t>(total, 1), threads);
  return (int)std::min<int64_t>(b, max_blocks);
}

// ---------------------------------------------------------------------------
// Strided GEMM launcher (deterministic split-K).
template <typename TA, typename TB, typename TAcc, typename TC>
void gemm(Ctx& c, int64_t M, int64_t N, int64_t K, const TA* A, int64_t sam,
          int64_t sak, const TB* B, int64_t sbk, int64_t sbn, TC* C,
          int64_t scm, int64_t scn, TAcc alpha = TAcc(1), TAcc beta = TAcc(0),
          const TC* C0 = nullptr, int64_t sc0m = 0, int64_t sc0n = 0) {
  if (M <= 0 || N <= 0) return;
  constexpr bool dbl = sizeof(TAcc) == 8;
  constexpr int BM = 64, BK = dbl ? 8 : 16, TM = 4;
  const bool narrow = N <= 32;
  const int BN = narrow ? 32 : 64;
  const int64_t tiles = ceil_div(M, BM) * ceil_div(N, BN);
  const int64_t target = 4 * c.num_sms;
  const int64_t max_split = std::max<int64_t>(1, K / (BK * 4));
  int64_t splits = std::min<int64_t>(std::max<int64_t>(1, ceil_div(target, tiles)),
                                     std::min<int64_t>(max_split, 256));
  int64_t kchunk = ceil_div(std::max<int64_t>(K, 1), splits);
  kchunk = ceil_div(kchunk, BK) * BK;
  splits = std::max<int64_t>(1, ceil_div(K, kchunk));
  DBuf<TAcc> part;
  if (splits > 1) part.alloc(c, (size_t)(splits * M * N));
  dim3 grid((unsigned)ceil_div(M, BM), (unsigned)ceil_div(N, BN), (unsigned)splits);
  if (narrow) {
    gemm_strided_kernel<TA, TB, TAcc, TC, BM, 32, BK, TM, 2>
        <<<grid, 256, 0, c.stream>>>(M, N, K, A, sam, sak, B, sbk, sbn, C, scm,
                                      scn, alpha, beta, C0, sc0m, sc0n, kchunk,
                                      part.p);
  } else {
    gemm_strided_kernel<TA, TB, TAcc, TC, BM, 64, BK, TM, 4>
        <<<grid, 256, 0, c.stream>>>(M, N, K, A, sam, sak, B, sbk, sbn, C, scm,
                                      scn, alpha, beta, C0, sc0m, sc0n, kchunk,
                                      part.p);
  }
  BRSVD_CHECK_LAUNCH();
  if (splits > 1) {
    splitk_reduce_kernel<TAcc, TC><<<grid_for(M * N), 256, 0, c.stream>>>(
        M, N, (int)splits, part.p, C, scm, scn, alpha, beta, C0, sc0m, sc0n);
    BRSVD_CHECK_LAUNCH();
  }
}

// Column-major helpers: C = op(X)... written out for readability.
//   XtY:  C (a x b) = X(r x a)^T Y(r x b)
template <typename TX, typename TY, typename TC>
void gemm_tn_cm(Ctx& c, int64_t a, int64_t b, int64_t r, const TX* X, int64_t ldx,
                const TY* Y, int64_t ldy, TC* C, int64_t ldc) {
  gemm<TX, TY, double, TC>(c, a, b, r, X, ldx, 1, Y, 1, ldy, C, 1, ldc);
}
//   XT:  C (r x b) = alpha X(r x a) T(a x b) + beta C0
template <typename TX, typename TT, typename TC>
void gemm_nn_cm(Ctx& c, int64_t r, int64_t b, int64_t a, const TX* X, int64_t ldx,
                const TT* T, int64_t ldt, TC* C, int64_t ldc, double alpha = 1.0,
                double beta = 0.0, const TC* C0 = nullptr, int64_t ldc0 = 0) {
  gemm<TX, TT, double, TC>(c, r, b, a, X, 1, ldx, T, 1, ldt, C, 1, ldc, alpha,
                           beta, C0, 1, ldc0);
}

// Readback of a few device scalars (one synchronisation).
inline void readback(Ctx& c, const void* d, void* h, size_t bytes) {
  BRSVD_CUDA(cudaMemcpyAsync(c.h_pinned, d, bytes, cudaMemcpyDeviceToHost, c.stream));
  BRSVD_CUDA(cudaStreamSynchronize(c.stream));
  std::memcpy(h, c.h_pinned, bytes);
}

inline int read_int(Ctx& c, const int* d) {
  int v;
  readback(c, d, &v, sizeof(int));
  return v;
}

// ---------------------------------------------------------------------------
// Jacobi SVD launcher: G (nrow x ncol, ldg) <- G V, V (ncol x ncol) accumulated.
// tol: rotate a column pair while |x.y| > tol * ||x|| ||y||.  The dot products
// carry ~sqrt(nrow) eps of rounding, so tol_tight() is the accuracy floor; the
// Gram-based basis changes only need tol ~ 1e-8 (a Newton-Schulz step absorbs
// the rest) and the power-iteration normalisation ~ 1e-4.
inline double jacobi_tol_tight(int nrow) {
  return 8.0 * std::sqrt((double)nrow) * 2.220446049250313e-16;
}
constexpr double kJacobiTolOrth = 1e-8;
constexpr double kJacobiTolNormalize = 1e-4;

// Cluster-resident Jacobi (jacobi_cluster.cuh) for square problems that are
// too big for one CTA but fit the shared memory of an 8- or 16-CTA cluster.
// Returns false (nothing launched) when the shape or the device does not fit.
template <typename R, int NP2>
bool jacobi_cluster_launch(Ctx& c, const JacobiClusterArgs<R>& args, int csize,
                           size_t smem, int threads) {
  auto kern = jacobi_cluster_kernel<R, NP2>;
  BRSVD_CUDA(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                  (int)smem));
  if (csize > 8)
    BRSVD_CUDA(cudaFuncSetAttribute(kern, cudaFuncAttributeNonPortableClusterSizeAllowed, 1));
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3(csize);
  cfg.blockDim = dim3(threads);
  cfg.dynamicSmemBytes = smem;
  cfg.stream = c.stream;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeClusterDimension;
  attr[0].val.clusterDim.x = csize;
  attr[0].val.clusterDim.y = 1;
  attr[0].val.clusterDim.z = 1;
  cfg.attrs = attr;
  cfg.numAttrs = 1;
  int nclusters = 0;
  if (cudaOccupancyMaxActiveClusters(&nclusters, kern, &cfg) != cudaSuccess ||
      nclusters < 1) {
    cudaGetLastError();
    return false;
  }
  BRSVD_CUDA(cudaLaunchKernelEx(&cfg, kern, args));
  BRSVD_CHECK_LAUNCH();
  return true;
}

template <typename R>
bool jacobi_cluster(Ctx& c, R* G, int l, int64_t ldg, R* V, int64_t ldv, double tol,
                    double floor_rel, int max_sweeps, int* sweeps_done) {
  if (l > 512 || l < 64 || std::getenv("BRSVD_NO_CLUSTER_JACOBI")) return false;
  const size_t lim = c.max_smem_optin > 4096 ? c.max_smem_optin - 4096 : 0;
  for (int csize : {16, 8}) {
    const int bw = (int)ceil_div(l, 2 * csize);
    const size_t smem = jacobi_cluster_smem<R>(l, bw);
    if (smem > lim) continue;
    JacobiClusterArgs<R> a;
    a.G = G;
    a.ldg = ldg;
    a.V = V;
    a.ldv = ldv;
    a.l = l;
    a.bw = bw;
    a.max_sweeps = max_sweeps;
    a.tol = tol;
    a.floor_rel = floor_rel;
    a.sweeps_done = sweeps_done;
    const int threads = std::min(1024, std::max(256, 32 * bw));
    const int np2 = (int)ceil_div((l + 3) & ~3, 64);  // row pairs per lane
    bool ok;
    if (np2 <= 2) ok = jacobi_cluster_launch<R, 2>(c, a, csize, smem, threads);
    else if (np2 <= 3) ok = jacobi_cluster_launch<R, 3>(c, a, csize, smem, threads);
    else if (np2 <= 4) ok = jacobi_cluster_launch<R, 4>(c, a, csize, smem, threads);
    else if (np2 <= 5) ok = jacobi_cluster_launch<R, 5>(c, a, csize, smem, threads);
    else if (np2 <= 6) ok = jacobi_cluster_launch<R, 6>(c, a, csize, smem, threads);
    else ok = jacobi_cluster_launch<R, 8>(c, a, csize, smem, threads);
    if (ok) return true;
  }
  return false;
}

// floor_rel < 0: the default null-column floor 16 nrow eps(R).  The fp32 phase
// of the two-phase small SVD passes a lower one so that small but resolvable
// columns (noise-level singular values of fp32 data) converge already in fp32.
template <typename R = double>
inline int jacobi(Ctx& c, R* G, int nrow, int ncol, int64_t ldg, R* V, int64_t ldv,
                  double tol, int max_sweeps = 40, double floor_rel = -1.0) {
  BRSVD_REQUIRE(ncol >= 1 && ncol <= 1024 && nrow >= 1, kErrShape,
                "jacobi: unsupported small-problem shape");
  const double eps_r0 = sizeof(R) == 8 ? 2.220446049250313e-16 : 1.1920928955078125e-07;
  const double tol_eff = std::max(tol, 8.0 * std::sqrt((double)nrow) * eps_r0);
  const double floor_eff = floor_rel >= 0.0 ? floor_rel : 16.0 * nrow * eps_r0;
  if (nrow == ncol) {
    DBuf<int> sw(c, 1);
    if (jacobi_cluster<R>(c, G, nrow, ldg, V, ldv, tol_eff, floor_eff, max_sweeps, sw.p)) {
      if (std::getenv("BRSVD_DEBUG")) {
        const int nsw = read_int(c, sw.p);
        std::fprintf(stderr, "[brsvd] jacobi(cluster) %dx%d tol %.1e: %d sweeps\n", nrow,
                     ncol, tol_eff, nsw);
      }
      return 0;
    }
  }
  const size_t budget = std::min<size_t>(c.max_smem_optin, 200 * 1024);
  const size_t per_col = (size_t)(nrow + ncol) * sizeof(R) + sizeof(int);
  int bw_fit = (int)(budget / (2 * per_col));
  BRSVD_REQUIRE(bw_fit >= 1, kErrShape, "jacobi: column too long for shared memory");
  int bw = (ncol + 1) / 2;
  bool single = true;
  if (bw > bw_fit) {
    bw = std::min(bw_fit, 32);
    single = false;
  }
  int nb = (int)ceil_div(ncol, bw);
  if (nb < 2) nb = 2;
  if (nb & 1) ++nb;
  if (nb == 2) single = true;
  const int threads = std::min(1024, std::max(64, bw * 32));
  const size_t smem = (size_t)2 * bw * per_col;
  static bool attr_set = false;
  if (!attr_set) {
    BRSVD_CUDA(cudaFuncSetAttribute(jacobi_block_kernel<R>,
                                    cudaFuncAttributeMaxDynamicSharedMemorySize,
                                    (int)budget));
    attr_set = true;
  }
  DBuf<int> counters(c, (size_t)max_sweeps + 1);
  BRSVD_CUDA(cudaMemsetAsync(counters.p, 0, sizeof(int) * (max_sweeps + 1), c.stream));
  JacobiArgs<R> args;
  args.G = G;
  args.ldg = ldg;
  args.nrow = nrow;
  args.ncol = ncol;
  args.V = V;
  args.ldv = ldv;
  args.bw = bw;
  args.nb = nb;
  args.max_sweeps = max_sweeps;
  args.tol = tol_eff;
  args.floor_rel = floor_eff;
  args.rot_count = counters.p;
  args.sweeps_done = counters.p + max_sweeps;
  if (single) {
    jacobi_block_kernel<R><<<1, threads, smem, c.stream>>>(args);
    BRSVD_CHECK_LAUNCH();
  } else {
    int grid = nb / 2;
    int per_sm = 0;
    BRSVD_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(
        &per_sm, jacobi_block_kernel<R>, threads, smem));
    grid = std::min(grid, std::max(1, per_sm) * c.num_sms);
    void* kargs[] = {&args};
    BRSVD_CUDA(cudaLaunchCooperativeKernel((void*)jacobi_block_kernel<R>, dim3(grid),
                                           dim3(threads), kargs, smem, c.stream));
    ++g_brsvd_launches;
  }
  if (std::getenv("BRSVD_DEBUG")) {
    int sw = 0;
    readback(c, counters.p + max_sweeps, &sw, sizeof(int));
    std::fprintf(stderr, "[brsvd] jacobi %dx%d tol %.1e: %d sweeps (nb %d, bw %d)\n", nrow,
                 ncol, args.tol, sw, nb, bw);
  }
  return nb;
}

inline void jacobi_finish(Ctx& c, const double* G, int nrow, int ncol, int64_t ldg,
                          const double* V, int64_t ldv, double* sv, double* Uout,
                          int64_t ldu, double* Vout, int64_t ldvo) {
  const size_t smem = (size_t)ncol * (sizeof(double) + sizeof(int));
  jacobi_finish_kernel<<<1, 1024, smem, c.stream>>>(G, ldg, nrow, ncol, V, ldv, sv,
                                                    Uout, ldu, Vout, ldvo);
  BRSVD_CHECK_LAUNCH();
}

// ---------------------------------------------------------------------------
// Eigen-decomposition of the (optionally column-scaled) Gram of X (r x l):
//   s_j = 1/||x_j|| (or 1),  (S X^T X S) = E diag(lam) E^T  (lam sorted desc)
// trace (device, optional) receives ||X||_F^2.
template <typename T>
void gram_eig(Ctx& c, const T* X, int64_t r, int l, int64_t ldx, double* E,
              double* lam, double* s, double tol, bool scale = true,
              double* trace = nullptr, double drop = 0.0) {
  DBuf<double> G(c, (size_t)l * l), V(c, (size_t)l * l);
  gemm_tn_cm<T, T, double>(c, l, l, r, X, ldx, X, ldx, G.p, l);
  gram_prep_kernel<<<1, 1024, 0, c.stream>>>(G.p, l, s, V.p, scale ? 1 : 0, trace,
                                             drop);
  BRSVD_CHECK_LAUNCH();
  jacobi(c, G.p, l, l, l, V.p, l, tol);
  jacobi_finish(c, G.p, l, l, l, V.p, l, lam, nullptr, 0, E, l);
}

inline double orth_tau(int64_t r, int l) {
  return 8.0 * (double)std::max<int64_t>(r, l) * 2.220446049250313e-16;
}

constexpr int kCholMaxL = 384;  // chol_kernel shared-memory limit (~197 KB)

// Cholesky basis change of X (r x l): with s_j = 1/||x_j|| and the scaled Gram
// G~ = S X^T X S, factor G~ + shift I = L L^T and return T = S L^-T in Tm
// (l x l, column-major).  Returns min pivot / diagonal (1 = orthogonal
// columns, ~1/cond^2 otherwise, <= 0 on breakdown) when `ratio` is requested.
struct CholInfo {
  double min_ratio = 0.0;  // min pivot / diagonal over the kept columns
  int rank_ref = 0;        // reference-style |diag R| rank (kernels.py:155-157)
  int kept = 0;            // columns kept by the rank-revealing pass
};

// Cholesky basis change of X (r x l): with s_j = 1/||x_j|| and the scaled Gram
// G~ = S X^T X S, factor G~ + shift I = L L^T and return T = S L^-T in Tm
// (l x l, column-major).  drop_ratio > 0 drops (in column order) the columns
// whose pivot falls below it; `keep` (device, l ints) then lists the kept
// columns.  Host-visible diagnostics only when `sync` is set.
template <typename T>
CholInfo chol_basis(Ctx& c, const T* X, int64_t r, int l, int64_t ldx, double shift,
                    double* Tm, bool sync, double col_drop = 0.0, double rank_tol = 0.0,
                    double drop_ratio = 0.0, int* keep = nullptr,
                    double* info_dev = nullptr) {
  DBuf<double> G(c, (size_t)l * l), W(c, (size_t)l * l), infob;
  double* info = info_dev;
  if (!info) {
    infob.alloc(c, 3);
    info = infob.p;
  }
  gemm_tn_cm<T, T, double>(c, l, l, r, X, ldx, X, ldx, G.p, l);
  cholinv_launch(c.stream, c.max_smem_optin, G.p, l, l, 1, col_drop, shift, drop_ratio,
                 rank_tol, W.p, Tm, nullptr, info, keep);
  BRSVD_CHECK_LAUNCH();
  CholInfo ci;
  if (sync) {
    double h[3];
    readback(c, info, h, sizeof(h));
    ci.min_ratio = h[0];
    ci.rank_ref = (int)h[1];
    ci.kept = (int)h[2];
  }
  return ci;
}

inline void set_chol_attrs(Ctx& c) {
  static bool done = false;
  if (done) return;
  const int lim = (int)c.max_smem_optin - 2048;  // leave room for static smem
  BRSVD_CUDA(cudaFuncSetAttribute(chol_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, lim));
  BRSVD_CUDA(cudaFuncSetAttribute(trinv_t_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                  lim));
  done = true;
}

// Basis change for the power iteration: Xout spans range(X) with restored
// conditioning.  Shifted Cholesky QR (shift ~ l*eps of the unit diagonal,
// never breaks down) when l fits the Cholesky kernel, else the regularised
// Gram-eigen basis X S E Lam^-1/2 (eigenvalues floored at tau*lam_0).  No
// host synchronisation either way.
template <typename T>
void normalize_sketch(Ctx& c, const T* X, int64_t r, int l, int64_t ldx, T* Xout,
                      int64_t ldo) {
  DBuf<double> Tm(c, (size_t)l * l);
  if (l <= kCholMaxL) {
    set_chol_attrs(c);
    chol_basis<T>(c, X, r, l, ldx, 16.0 * l * 2.220446049250313e-16, Tm.p, false);
  } else {
    DBuf<double> E(c, (size_t)l * l), lam(c, l), s(c, l);
    gram_eig<T>(c, X, r, l, ldx, E.p, lam.p, s.p, kJacobiTolNormalize);
    build_basis_kernel<<<1, 1024, 0, c.stream>>>(E.p, lam.p, s.p, l, orth_tau(r, l), 0,
                                                 Tm.p, nullptr);
    BRSVD_CHECK_LAUNCH();
  }
  gemm_nn_cm<T, double, T>(c, r, l, l, X, ldx, Tm.p, l, Xout, ldo);
}

// Block projection X <- X - Qb (Qb^T X), applied twice ("twice is enough").
inline void project_out(Ctx& c, const double* Qb, int64_t r, int kq, double* X,
                        int cols) {
  if (kq <= 0 || cols <= 0) return;
  DBuf<double> Cm(c, (size_t)kq * cols);
  for (int pass = 0; pass < 2; ++pass) {
    gemm_tn_cm<double, double, double>(c, kq, cols, r, Qb, r, X, r, Cm.p, kq);
    gemm_nn_cm<double, double, double>(c, r, cols, kq, Qb, r, Cm.p, kq, X, r, -1.0,
                                       1.0, X, r);
  }
}

// Newton-Schulz polar refinement of the r x k block Q: Q <- Q (1.5 I - 0.5 Q^T Q).
inline void ns_refine(Ctx& c, double* Q, int64_t r, int k, int iters) {
  if (k <= 0 || iters <= 0) return;
  DBuf<double> G2(c, (size_t)k * k), T2(c, (size_t)k * k), Qt(c, (size_t)r * k);
  for (int it = 0; it < iters; ++it) {
    gemm_tn_cm<double, double, double>(c, k, k, r, Q, r, Q, r, G2.p, k);
    ns_matrix_kernel<<<grid_for((int64_t)k * k), 256, 0, c.stream>>>(G2.p, k, T2.p);
    BRSVD_CHECK_LAUNCH();
    gemm_nn_cm<double, double, double>(c, r, k, k, Q, r, T2.p, k, Qt.p, r);
    BRSVD_CUDA(cudaMemcpyAsync(Q, Qt.p, sizeof(double) * r * k,
                               cudaMemcpyDeviceToDevice, c.stream));
  }
}

// Deflation levels: the part of X that level 1 left unresolved,
// R = (I - Q Q^T) X, is re-factored with an unscaled Gram (eigen route, so the
// threshold is relative to R's own scale) while ||R||_F^2 > stop2.  A Gram
// resolves directions down to ~sqrt(tau) of its largest, Householder QR (the
// reference's tsqr, kernels.py:121-164) down to eps; each level buys another
// factor sqrt(tau).  Appends columns to Q and to the reported rank.
template <typename T>
void deflate_levels(Ctx& c, const T* X, int64_t r, int l, int64_t ldx, double* Q,
                    int& total, int& rank, double stop2, double tau, int ns_iters) {
  if (total >= l || !(stop2 > 0.0)) return;
  DBuf<double> E(c, (size_t)l * l), lam(c, l), s(c, l), Tm(c, (size_t)l * l);
  DBuf<double> scal(c, 4);
  DBuf<int> drank(c, 1);
  DBuf<double> R(c, (size_t)r * l);
  copy2d_kernel<T, double><<<grid_for(r * l), 256, 0, c.stream>>>(X, r, l, ldx, R.p, r);
  BRSVD_CHECK_LAUNCH();
  DBuf<double> G(c, (size_t)l * l), V(c, (size_t)l * l);
  for (int level = 0; level < 4 && total < l; ++level) {
    project_out(c, Q, r, total, R.p, l);
    // ||R||_F^2 first: most calls stop here without an eigen-solve
    gemm_tn_cm<double, double, double>(c, l, l, r, R.p, r, R.p, r, G.p, l);
    gram_prep_kernel<<<1, 1024, 0, c.stream>>>(G.p, l, s.p, V.p, 0, scal.p, 0.0);
    BRSVD_CHECK_LAUNCH();
    double nr2;
    readback(c, scal.p, &nr2, sizeof(double));
    if (!(nr2 > stop2)) break;
    jacobi(c, G.p, l, l, l, V.p, l, kJacobiTolOrth);
    jacobi_finish(c, G.p, l, l, l, V.p, l, lam.p, nullptr, 0, E.p, l);
    build_basis_kernel<<<1, 1024, 0, c.stream>>>(E.p, lam.p, s.p, l, tau, 1, Tm.p,
                                                 drank.p);
    BRSVD_CHECK_LAUNCH();
    int rk2 = read_int(c, drank.p);
    if (rk2 <= 0) break;
    rk2 = std::min(rk2, l - total);
    double* Qn = Q + (int64_t)total * r;
    gemm_nn_cm<double, double, double>(c, r, rk2, l, R.p, r, Tm.p, l, Qn, r);
    project_out(c, Q, r, total, Qn, rk2);
    ns_refine(c, Qn, r, rk2, std::max(ns_iters, 1));
    total += rk2;
    rank += rk2;
  }
}

template <typename T>
int orth_full(Ctx& c, const T* X, int64_t r, int l, int64_t ldx, double* Q,
              uint64_t seed, int ns_iters);

// Numerically null directions: Gaussian columns projected out twice and
// orthonormalised (kernels.py:142-144, "columns of Q remain orthonormal").
inline void complete_basis(Ctx& c, double* Q, int64_t r, int l, int total, uint64_t seed,
                           int ns_iters) {
  if (total >= l) return;
  const int cnt = l - total;
  double* W = Q + (int64_t)total * r;
  gaussian_kernel<double><<<grid_for(r * ((cnt + 1) / 2)), 256, 0, c.stream>>>(
      W, r, cnt, r, seed, 0x636f6d706c657465ull, 0);
  BRSVD_CHECK_LAUNCH();
  project_out(c, Q, r, total, W, cnt);
  DBuf<double> Wq(c, (size_t)r * cnt);
  orth_full<double>(c, W, r, cnt, r, Wq.p, seed * 0x9E3779B97F4A7C15ull + 1,
                    std::max(ns_iters, 1));
  BRSVD_CUDA(cudaMemcpyAsync(W, Wq.p, sizeof(double) * r * cnt, cudaMemcpyDeviceToDevice,
                             c.stream));
  project_out(c, Q, r, total, W, cnt);
  ns_refine(c, W, r, cnt, 1);
}

// Rank-revealing orthonormal basis of range(X), X (r x l), r >= l
// (tsqr / tsqr_factor, kernels.py:139-170).  Returns the detected numerical
// rank; Q is r x l, fp64, ld r, always with l orthonormal columns.
//
// Level 1 (l <= kCholMaxL): rank-revealing Cholesky QR in column order.
// Columns whose pivot falls below 1e-12 of their norm lie numerically in the
// span of the earlier ones and are set aside; the kept ones get a second
// CholQR pass (orthonormal to rounding).  The reported rank is the
// reference's |diag R| > l eps ||X||_F cut, since the Cholesky factor of the
// Gram is the R of an unpivoted QR (kernels.py:155-157).
// Level 1 (larger l): Gram eigenpairs by Jacobi, keep lam > tau lam_0.
// Then deflation levels for what is still resolvable in the data's precision
// and a Gaussian completion of the null directions.
template <typename T>
int orth_full(Ctx& c, const T* X, int64_t r, int l, int64_t ldx, double* Q,
              uint64_t seed, int ns_iters) {
  const double eps_data = sizeof(T) == 8 ? 2.220446049250313e-16 : 1.1920928955078125e-07;
  const double tau = orth_tau(r, l);
  const double drop = 4.0 * l * eps_data;  // the reference's rank cut, kernels.py:155-157
  int total = 0, rank = 0;
  double normx2 = 0.0;
  if (l <= kCholMaxL) {
    set_chol_attrs(c);
    DBuf<int> keep(c, l);
    DBuf<double> info(c, 3), Tm(c, (size_t)l * l), Tc(c, (size_t)l * l);
    const CholInfo ci = chol_basis<T>(c, X, r, l, ldx, 0.0, Tm.p, true, drop, l * eps_data,
                                      1e-12, keep.p, info.p);
    const int k1 = ci.kept;
    if (sizeof(T) == 4 && k1 < l) {
      // fp32 data: the dropped directions are below the data's resolution.
      // Complete in the same second CholQR pass: [Q1 | Gaussian columns] is
      // well conditioned, so one pass returns l orthonormal columns whose
      // first k1 span the kept part of range(X) (kernels.py:142-144, "columns
      // of Q remain orthonormal").
      DBuf<double> Q1(c, (size_t)r * l);
      if (k1 > 0) {
        compact_cols_kernel<<<grid_for((int64_t)l * k1), 256, 0, c.stream>>>(
            Tm.p, l, keep.p, info.p, Tc.p);
        BRSVD_CHECK_LAUNCH();
        gemm_nn_cm<T, double, double>(c, r, k1, l, X, ldx, Tc.p, l, Q1.p, r);
      }
      const int cnt = l - k1;
      gaussian_kernel<double><<<grid_for(r * ((cnt + 1) / 2)), 256, 0, c.stream>>>(
          Q1.p + (int64_t)k1 * r, r, cnt, r, seed, 0x636f6d706c657465ull, 0);
      BRSVD_CHECK_LAUNCH();
      chol_basis<double>(c, Q1.p, r, l, r, 0.0, Tm.p, false);
      gemm_nn_cm<double, double, double>(c, r, l, l, Q1.p, r, Tm.p, l, Q, r);
      return std::min(ci.rank_ref, k1);
    }
    if (k1 > 0) {
      const double* Tk = Tm.p;
      if (k1 < l) {
        compact_cols_kernel<<<grid_for((int64_t)l * k1), 256, 0, c.stream>>>(
            Tm.p, l, keep.p, info.p, Tc.p);
        BRSVD_CHECK_LAUNCH();
        Tk = Tc.p;
      }
      DBuf<double> Q1(c, (size_t)r * k1);
      gemm_nn_cm<T, double, double>(c, r, k1, l, X, ldx, Tk, l, Q1.p, r);
      chol_basis<double>(c, Q1.p, r, k1, r, 0.0, Tm.p, false);
      gemm_nn_cm<double, double, double>(c, r, k1, k1, Q1.p, r, Tm.p, k1, Q, r);
      if (ns_iters > 1) ns_refine(c, Q, r, k1, 1);
    }
    total = k1;
    rank = std::min(ci.rank_ref, k1);
    if (total == l) return rank;
    if (sizeof(T) == 4) {
      complete_basis(c, Q, r, l, total, seed, ns_iters);
      return rank;
    }
    // ||X||_F^2 for the deflation stop rule
    DBuf<double> nf(c, 1);
    DBuf<double> G(c, (size_t)l * l), Wd(c, (size_t)l * l), sd(c, l);
    gemm_tn_cm<T, T, double>(c, l, l, r, X, ldx, X, ldx, G.p, l);
    gram_prep_kernel<<<1, 1024, 0, c.stream>>>(G.p, l, sd.p, Wd.p, 0, nf.p, 0.0);
    BRSVD_CHECK_LAUNCH();
    readback(c, nf.p, &normx2, sizeof(double));
  } else {
    DBuf<double> E(c, (size_t)l * l), lam(c, l), s(c, l), Tm(c, (size_t)l * l);
    DBuf<double> scal(c, 4);
    DBuf<int> drank(c, 1);
    gram_eig<T>(c, X, r, l, ldx, E.p, lam.p, s.p, kJacobiTolOrth, true, scal.p, drop);
    build_basis_kernel<<<1, 1024, 0, c.stream>>>(E.p, lam.p, s.p, l, tau, 1, Tm.p, drank.p);
    BRSVD_CHECK_LAUNCH();
    BRSVD_CUDA(cudaMemcpyAsync(scal.p + 1, drank.p, sizeof(int), cudaMemcpyDeviceToDevice,
                               c.stream));
    double hs[2];
    readback(c, scal.p, hs, sizeof(hs));
    normx2 = hs[0];
    std::memcpy(&total, &hs[1], sizeof(int));
    rank = total;
    if (total > 0) {
      gemm_nn_cm<T, double, double>(c, r, total, l, X, ldx, Tm.p, l, Q, r);
      ns_refine(c, Q, r, total, ns_iters);
    }
  }
  // fp64 data only: for fp32 data the level-1 cut (1e-6 of a column's norm)
  // is already below the reference's own rank cut (l eps32 ||X||_F).
  if (sizeof(T) == 8 && total < l && normx2 > 0.0)
    deflate_levels<T>(c, X, r, l, ldx, Q, total, rank, drop * drop * normx2, tau, ns_iters);
  complete_basis(c, Q, r, l, total, seed, ns_iters);
  return rank;
}

// ---------------------------------------------------------------------------
// small_svd (kernels.py:173-188): B^T (n x l, given as Bt) = Qb R,
// R^T = W diag(sigma) Zj^T  (one-sided Jacobi),  V = Qb Zj.
// Outputs: W (l x l fp64, ld l), sigma (fp64), Vout (n x l, T, ld ldv).
template <typename T>
int small_svd_device(Ctx& c, const T* Bt, int64_t n, int l, int64_t ldb, double* W,
                     double* sigma, T* Vout, int64_t ldv, int ns_iters) {
  DBuf<double> Qb(c, (size_t)n * l), M(c, (size_t)l * l), Vj(c, (size_t)l * l),
      Zj(c, (size_t)l * l);
  const int rank = orth_full<T>(c, Bt, n, l, ldb, Qb.p, 0x5eedb5ull, ns_iters);
  // M = Bt^T Qb = R^T
  gemm_tn_cm<T, double, double>(c, l, l, n, Bt, ldb, Qb.p, n, M.p, l);
  if (l > 64) {
    // Two-phase Jacobi: sweeps in fp32 (native rsqrt/rcp, half the shuffles
    // and shared memory) down to ~1e-5 orthogonality, then the fp64 sweeps
    // start from M V0 with V0 polished to an fp64-orthogonal matrix; the
    // quadratic convergence leaves only ~2 fp64 sweeps.
    DBuf<float> M32(c, (size_t)l * l), V32(c, (size_t)l * l);
    copy2d_kernel<double, float><<<grid_for((int64_t)l * l), 256, 0, c.stream>>>(M.p, l, l, l,
                                                                                M32.p, l);
    eye_kernel<float><<<grid_for((int64_t)l * l), 256, 0, c.stream>>>(V32.p, l);
    BRSVD_CHECK_LAUNCH();
    jacobi<float>(c, M32.p, l, l, l, V32.p, l, 1e-5, 40, 16.0 * l * 2.220446049250313e-16);
    copy2d_kernel<float, double><<<grid_for((int64_t)l * l), 256, 0, c.stream>>>(V32.p, l, l, l,
                                                                                Vj.p, l);
    BRSVD_CHECK_LAUNCH();
    ns_refine(c, Vj.p, l, l, 2);
    DBuf<double> M1(c, (size_t)l * l);
    gemm_nn_cm<double, double, double>(c, l, l, l, M.p, l, Vj.p, l, M1.p, l);
    BRSVD_CUDA(cudaMemcpyAsync(M.p, M1.p, sizeof(double) * l * l, cudaMemcpyDeviceToDevice,
                               c.stream));
  } else {
    eye_kernel<double><<<grid_for((int64_t)l * l), 256, 0, c.stream>>>(Vj.p, l);
    BRSVD_CHECK_LAUNCH();
  }
  // fp32 data: singular vectors orthogonal to 1e-7 (the output precision) and
  // singular values to ~1e-14 relative; fp64 data: tight.
  const double tol = sizeof(T) == 8 ? jacobi_tol_tight(l) : 1e-7;
  jacobi(c, M.p, l, l, l, Vj.p, l, tol);
  jacobi_finish(c, M.p, l, l, l, Vj.p, l, sigma, W, l, Zj.p, l);
  complete_null_columns_kernel<<<1, 1024, (size_t)l * sizeof(double), c.stream>>>(
      W, l, l, l, sigma, 16.0 * l * 2.220446049250313e-16);
  BRSVD_CHECK_LAUNCH();
  gemm_nn_cm<double, double, T>(c, n, l, l, Qb.p, n, Zj.p, l, Vout, ldv);
  return rank;
}

template <typename T>
void fix_signs(Ctx& c, T* U, int64_t m, int l, int64_t ldu, T* V, int64_t n,
               int64_t ldv) {
  DBuf<T> sign(c, l);
  colsign_kernel<T><<<l, 256, 0, c.stream>>>(U, m, ldu, sign.p);
  BRSVD_CHECK_LAUNCH();
  scale_cols_kernel<T><<<grid_for(m * l), 256, 0, c.stream>>>(U, m, l, ldu, sign.p);
  BRSVD_CHECK_LAUNCH();
  scale_cols_kernel<T><<<grid_for(n * l), 256, 0, c.stream>>>(V, n, l, ldv, sign.p);
  BRSVD_CHECK_LAUNCH();
}

struct MaxAbs {
  double peak;
  bool nonfinite;
};

template <typename T>
MaxAbs maxabs(Ctx& c, const T* X, int64_t rows, int64_t cols, int64_t ld) {
  DBuf<unsigned long long> out(c, 2);
  BRSVD_CUDA(cudaMemsetAsync(out.p, 0, 2 * sizeof(unsigned long long), c.stream));
  maxabs_kernel<T><<<grid_for(rows * cols), 256, 0, c.stream>>>(X, rows, cols, ld,
                                                                 out.p);
  BRSVD_CHECK_LAUNCH();
  BRSVD_CUDA(cudaMemcpyAsync(c.h_pinned, out.p, 2 * sizeof(unsigned long long),
                             cudaMemcpyDeviceToHost, c.stream));
  BRSVD_CUDA(cudaStreamSynchronize(c.stream));
  MaxAbs r;
  long long bits = (long long)c.h_pinned[0];
  std::memcpy(&r.peak, &bits, sizeof(double));
  r.nonfinite = c.h_pinned[1] != 0;
  return r;
}

}  // namespace brsvd
