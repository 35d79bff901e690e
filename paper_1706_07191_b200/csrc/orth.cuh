// Orthonormalisation and the small SVD on the GPU.
//   chol_basis / normalize_sketch  <- basis changes of the power iteration
//   orth_full        <- tsqr / tsqr_factor kernels.py:139-170
//   small_svd_device <- small_svd          kernels.py:173-188
// fp32 data keeps its tall-skinny operands in fp32: Grams accumulate in fp64
// (SIMT), the l x l factorisations run in fp64, and the tall-skinny basis
// changes X T are tcgen05 3xTF32 products (apply_basis).
#pragma once
#include "big_gemm.cuh"

namespace brsvd {

// Basis change Out (r x lo) = X (r x li) Tm (li x lo, fp64, ld ldt).  fp32
// data: tcgen05 3xTF32 product with Tm rounded to fp32 (the rounding selects
// a different, equally conditioned basis of the same span; the product error
// is that of the fp32 data itself); fp64 data: SIMT fp64.
template <typename T>
void apply_basis(Ctx& c, const T* X, int64_t r, int li, int64_t ldx, const double* Tm,
                 int64_t ldt, int lo, T* Out, int64_t ldo) {
  if (sizeof(T) == 4 && tc_gemm_supported<T>(c, X, ldx, r, li, lo)) {
    DBuf<float> T32(c, (size_t)li * lo);
    copy2d_kernel<double, float><<<grid_for((int64_t)li * lo), 256, 0, c.stream>>>(
        Tm, li, lo, ldt, T32.p, li);
    BRSVD_CHECK_LAUNCH();
    tc_product(c, reinterpret_cast<const float*>(X), r, li, ldx, false, false, T32.p, li, lo,
               reinterpret_cast<float*>(Out), ldo);
    return;
  }
  gemm_nn_cm<T, double, T>(c, r, lo, li, X, ldx, Tm, ldt, Out, ldo);
}

// fp64 data near the ends of the exponent range: Cholesky QR and the Jacobi
// sweeps square magnitudes, which the reference's Householder QR and gesdd
// never do (LAPACK's norms are scale-safe), so such operands are brought to
// unit order by a power of two first (exact; Q and the rank cut are
// scale-invariant).  Returns e with X * 2^-e of unit order, or 0 when X is
// within 2^+-400 already (fp32 data: Grams are fp64, always 0).
template <typename T>
int unit_exponent(Ctx& c, const T* X, int64_t rows, int cols, int64_t ld) {
  if (sizeof(T) != 8 || rows * cols == 0) return 0;
  const MaxAbs pk = maxabs<T>(c, X, rows, cols, ld);
  if (pk.nonfinite || !(pk.peak > 0.0)) return 0;
  int e;
  std::frexp(pk.peak, &e);
  return (e > 400 || e < -400) ? e : 0;
}

constexpr int kCholMaxL = 320;  // cholinv_kernel shared-memory limit (~196 KB at 320)

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
// tc_gram: the Gram of an already well-conditioned fp32 basis (second CholQR
// pass) may use the tcgen05 product (fp32-level accuracy suffices there).
template <typename T>
CholInfo chol_basis(Ctx& c, const T* X, int64_t r, int l, int64_t ldx, double shift,
                    double* Tm, bool sync, double col_drop = 0.0, double rank_tol = 0.0,
                    double drop_ratio = 0.0, int* keep = nullptr,
                    double* info_dev = nullptr, bool tc_gram_ok = false) {
  DBuf<double> G(c, (size_t)l * l), W(c, (size_t)l * l), infob;
  double* info = info_dev;
  if (!info) {
    infob.alloc(c, 3);
    info = infob.p;
  }
  if (!(sizeof(T) == 4 && tc_gram_ok &&
        tc_gram(c, reinterpret_cast<const float*>(X), r, l, ldx,
                reinterpret_cast<const float*>(X), ldx, l, G.p, l)))
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


// Basis change for the power iteration: Xout spans range(X) with restored
// conditioning.  Shifted Cholesky QR (shift ~ l*eps of the unit diagonal,
// never breaks down) when l fits the Cholesky kernel, else the regularised
// Gram-eigen basis X S E Lam^-1/2 (eigenvalues floored at tau*lam_0).  No
// host synchronisation either way.
// Tout (optional, l x l fp64): the transform actually applied, Xout = X Tout
// (for fp32 data its fp32-rounded entries), for the exact overflow guard.
template <typename T>
void normalize_sketch(Ctx& c, const T* X, int64_t r, int l, int64_t ldx, T* Xout,
                      int64_t ldo, double* Tout = nullptr, bool scale_check = false) {
  DBuf<double> Tm(c, (size_t)l * l);
  // fp64 X near the exponent limits (its Gram would overflow / underflow):
  // factor 2^-e X and fold 2^-e into the basis change, X (2^-e T) = (2^-e X) T
  const int e = scale_check ? unit_exponent<T>(c, X, r, l, ldx) : 0;
  DBuf<T> Xs;
  const T* Xf = X;
  int64_t ldf = ldx;
  if (e != 0) {
    Xs.alloc(c, (size_t)r * l);
    scale_copy_kernel<T><<<grid_for(r * l), 256, 0, c.stream>>>(X, r, l, ldx, Xs.p, r,
                                                                std::ldexp(1.0, -e));
    BRSVD_CHECK_LAUNCH();
    Xf = Xs.p;
    ldf = r;
  }
  if (l <= kCholMaxL) {
    chol_basis<T>(c, Xf, r, l, ldf, 16.0 * l * 2.220446049250313e-16, Tm.p, false);
  } else {
    DBuf<double> E(c, (size_t)l * l), lam(c, l), s(c, l);
    gram_eig<T>(c, Xf, r, l, ldf, E.p, lam.p, s.p, kJacobiTolNormalize);
    build_basis_kernel<<<1, 1024, 0, c.stream>>>(E.p, lam.p, s.p, l, orth_tau(r, l), 0,
                                                 Tm.p, nullptr);
    BRSVD_CHECK_LAUNCH();
  }
  if (e != 0) {
    scale_copy_kernel<double><<<grid_for((int64_t)l * l), 256, 0, c.stream>>>(
        Tm.p, l, l, l, Tm.p, l, std::ldexp(1.0, -e));
    BRSVD_CHECK_LAUNCH();
  }
  apply_basis<T>(c, X, r, l, ldx, Tm.p, l, l, Xout, ldo);
  if (Tout) {
    if (sizeof(T) == 4 && tc_gemm_supported<T>(c, X, ldx, r, l, l)) {
      DBuf<float> T32(c, (size_t)l * l);
      copy2d_kernel<double, float><<<grid_for((int64_t)l * l), 256, 0, c.stream>>>(
          Tm.p, l, l, l, T32.p, l);
      copy2d_kernel<float, double><<<grid_for((int64_t)l * l), 256, 0, c.stream>>>(
          T32.p, l, l, l, Tout, l);
      BRSVD_CHECK_LAUNCH();
    } else {
      BRSVD_CUDA(cudaMemcpyAsync(Tout, Tm.p, sizeof(double) * l * l,
                                 cudaMemcpyDeviceToDevice, c.stream));
    }
  }
}

// Inverse of an upper-triangular l x l matrix (column-major, fp64), one
// column per thread by back substitution.  Serves the exact overflow guard
// only (rare path), so it is written for clarity, not speed.
__global__ void triu_inverse_kernel(const double* __restrict__ T, int l,
                                    double* __restrict__ X) {
  for (int j = threadIdx.x; j < l; j += blockDim.x) {
    double* x = X + (int64_t)j * l;
    for (int i = l - 1; i > j; --i) x[i] = 0.0;
    for (int i = j; i >= 0; --i) {
      double v = i == j ? 1.0 : 0.0;
      for (int k = i + 1; k <= j; ++k) v -= T[(int64_t)k * l + i] * x[k];
      const double d = T[(int64_t)i * l + i];
      x[i] = d != 0.0 ? v / d : 0.0;
    }
  }
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
int orth_full_f64(Ctx& c, const T* X, int64_t r, int l, int64_t ldx, double* Q,
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
  orth_full_f64<double>(c, W, r, cnt, r, Wq.p, seed * 0x9E3779B97F4A7C15ull + 1,
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
int orth_full_f64(Ctx& c, const T* X, int64_t r, int l, int64_t ldx, double* Q,
                  uint64_t seed, int ns_iters) {
  const double eps_data = sizeof(T) == 8 ? 2.220446049250313e-16 : 1.1920928955078125e-07;
  const double tau = orth_tau(r, l);
  const double drop = 4.0 * l * eps_data;  // the reference's rank cut, kernels.py:155-157
  int total = 0, rank = 0;
  double normx2 = 0.0;
  if (l <= kCholMaxL) {
    DBuf<int> keep(c, l);
    DBuf<double> info(c, 3), Tm(c, (size_t)l * l), Tc(c, (size_t)l * l);
    const CholInfo ci = chol_basis<T>(c, X, r, l, ldx, 0.0, Tm.p, true, drop, l * eps_data,
                                      1e-12, keep.p, info.p);
    const int k1 = ci.kept;
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


// fp32 data (l <= kCholMaxL): rank-revealing Cholesky QR whose dropped
// directions (below the data's resolution) are completed in the same second
// pass: [X Tk | Gaussian columns] is well conditioned, so one more CholQR
// returns l orthonormal columns whose first k1 span the kept part of range(X)
// (kernels.py:142-144, "columns of Q remain orthonormal").  Q is fp32; the
// Grams and factors are fp64, the basis changes tcgen05 products.
// rank_dev: the rank is written to the device (read by the caller's final
// synchronisation) and -1 returned -- no host read in the middle of the
// pipeline: the kept columns are applied as l columns with the dropped ones
// zeroed and the Gaussian completion starts at the device-side kept count.
inline int orth_full_f32(Ctx& c, const float* X, int64_t r, int l, int64_t ldx, float* Q,
                         uint64_t seed, int* rank_dev = nullptr) {
  const double eps_data = 1.1920928955078125e-07;
  const double drop = 4.0 * l * eps_data;  // the reference's rank cut, kernels.py:155-157
  DBuf<int> keep(c, l);
  DBuf<double> info(c, 3), Tm(c, (size_t)l * l), Tc(c, (size_t)l * l);
  const CholInfo ci = chol_basis<float>(c, X, r, l, ldx, 0.0, Tm.p, rank_dev == nullptr, drop,
                                        l * eps_data, 1e-12, keep.p, info.p);
  if (rank_dev) {
    DBuf<float> Q1(c, (size_t)r * l);
    compact_cols_kernel<<<grid_for((int64_t)l * l), 256, 0, c.stream>>>(Tm.p, l, keep.p,
                                                                        info.p, Tc.p, 1);
    BRSVD_CHECK_LAUNCH();
    apply_basis<float>(c, X, r, l, ldx, Tc.p, l, l, Q1.p, r);
    gaussian_tail_kernel<float><<<grid_for(r * ((l + 1) / 2)), 256, 0, c.stream>>>(
        Q1.p, r, l, r, info.p, seed, 0x636f6d706c657465ull);
    BRSVD_CHECK_LAUNCH();
    chol_basis<float>(c, Q1.p, r, l, r, 0.0, Tm.p, false, 0.0, 0.0, 0.0, nullptr, nullptr,
                      /*tc_gram_ok=*/true);
    apply_basis<float>(c, Q1.p, r, l, r, Tm.p, l, l, Q, r);
    chol_rank_kernel<<<1, 1, 0, c.stream>>>(info.p, rank_dev);
    BRSVD_CHECK_LAUNCH();
    return -1;
  }
  const int k1 = ci.kept;
  DBuf<float> Q1(c, (size_t)r * l);
  if (k1 > 0) {
    const double* Tk = Tm.p;
    if (k1 < l) {
      compact_cols_kernel<<<grid_for((int64_t)l * k1), 256, 0, c.stream>>>(Tm.p, l, keep.p,
                                                                           info.p, Tc.p);
      BRSVD_CHECK_LAUNCH();
      Tk = Tc.p;
    }
    apply_basis<float>(c, X, r, l, ldx, Tk, l, k1, Q1.p, r);
  }
  if (k1 < l) {
    const int cnt = l - k1;
    gaussian_kernel<float><<<grid_for(r * ((cnt + 1) / 2)), 256, 0, c.stream>>>(
        Q1.p + (int64_t)k1 * r, r, cnt, r, seed, 0x636f6d706c657465ull, 0);
    BRSVD_CHECK_LAUNCH();
  }
  chol_basis<float>(c, Q1.p, r, l, r, 0.0, Tm.p, false, 0.0, 0.0, 0.0, nullptr, nullptr,
                    /*tc_gram_ok=*/true);
  apply_basis<float>(c, Q1.p, r, l, r, Tm.p, l, l, Q, r);
  return std::min(ci.rank_ref, k1);
}


template <typename T>
int orth_full(Ctx& c, const T* X, int64_t r, int l, int64_t ldx, T* Q, uint64_t seed,
              int ns_iters, bool scale_check = true, int* rank_dev = nullptr) {
  if (sizeof(T) == 8) {
    const int e = scale_check ? unit_exponent<T>(c, X, r, l, ldx) : 0;
    if (e != 0) {
      DBuf<T> Xs(c, (size_t)r * l);
      scale_copy_kernel<T><<<grid_for(r * l), 256, 0, c.stream>>>(X, r, l, ldx, Xs.p, r,
                                                                  std::ldexp(1.0, -e));
      BRSVD_CHECK_LAUNCH();
      return orth_full_f64<T>(c, Xs.p, r, l, r, reinterpret_cast<double*>(Q), seed,
                              ns_iters);
    }
    return orth_full_f64<T>(c, X, r, l, ldx, reinterpret_cast<double*>(Q), seed, ns_iters);
  }
  if (l <= kCholMaxL)
    return orth_full_f32(c, reinterpret_cast<const float*>(X), r, l, ldx,
                         reinterpret_cast<float*>(Q), seed, rank_dev);
  DBuf<double> Qw(c, (size_t)r * l);
  const int rank = orth_full_f64<T>(c, X, r, l, ldx, Qw.p, seed, ns_iters);
  copy2d_kernel<double, T><<<grid_for(r * l), 256, 0, c.stream>>>(Qw.p, r, l, r, Q, r);
  BRSVD_CHECK_LAUNCH();
  return rank;
}

// ---------------------------------------------------------------------------
// small_svd (kernels.py:173-188): B^T (n x l, given as Bt) = Qb R,
// R^T = W diag(sigma) Zj^T  (one-sided Jacobi),  V = Qb Zj.
// Outputs: W (l x l fp64, ld l), sigma (fp64), Vout (n x l, T, ld ldv).
template <typename T>
int small_svd_device(Ctx& c, const T* Bt, int64_t n, int l, int64_t ldb, double* W,
                     double* sigma, T* Vout, int64_t ldv, int ns_iters,
                     int* rank_dev = nullptr) {
  // fp64 B near the range limits: factor 2^-e B, scale sigma back at the end
  const int e = unit_exponent<T>(c, Bt, n, l, ldb);
  DBuf<T> Bs;
  if (e != 0) {
    Bs.alloc(c, (size_t)n * l);
    scale_copy_kernel<T><<<grid_for(n * l), 256, 0, c.stream>>>(Bt, n, l, ldb, Bs.p, n,
                                                                std::ldexp(1.0, -e));
    BRSVD_CHECK_LAUNCH();
    Bt = Bs.p;
    ldb = n;
  }
  DBuf<T> Qb(c, (size_t)n * l);
  DBuf<double> M(c, (size_t)l * l), Vj(c, (size_t)l * l), Zj(c, (size_t)l * l);
  // rank_dev: rank deferred to the caller's final read (-1 returned)
  const int rank = orth_full<T>(c, Bt, n, l, ldb, Qb.p, 0x5eedb5ull, ns_iters, false, rank_dev);
  // M = Bt^T Qb = R^T
  gemm_tn_cm<T, T, double>(c, l, l, n, Bt, ldb, Qb.p, n, M.p, l);
  if (l > 64) {
    // Two-phase Jacobi: sweeps in fp32 (native rsqrt/rcp, half the shuffles
    // and shared memory) down to ~1e-5 orthogonality, then the fp64 sweeps
    // start from M V0 with V0 polished to an fp64-orthogonal matrix; the
    // quadratic convergence leaves only ~2 fp64 sweeps.
    DBuf<float> M32(c, (size_t)l * l), V32;
    copy2d_kernel<double, float><<<grid_for((int64_t)l * l), 256, 0, c.stream>>>(M.p, l, l, l,
                                                                                M32.p, l);
    BRSVD_CHECK_LAUNCH();
    // predicted stop at sqrt(tol): this phase only preconditions the fp64 one
    const double tol32 = std::max(1e-5, 8.0 * std::sqrt((double)l) * 1.1920928955078125e-07);
    const double floor32 = 16.0 * l * 2.220446049250313e-16, stop32 = std::sqrt(1.6e-5);
    eye_kernel<double><<<grid_for((int64_t)l * l), 256, 0, c.stream>>>(Vj.p, l);
    BRSVD_CHECK_LAUNCH();
    // cluster tournament: its rotations are replayed on an fp64 V0, each
    // renormalised in fp64, so V0 is orthogonal to fp64 rounding and needs
    // no polish; otherwise fp32 V0, then two Newton-Schulz steps in fp64
    if (!jacobi_cluster<float, double>(c, M32.p, l, l, Vj.p, l, tol32, floor32, 40, nullptr,
                                       stop32)) {
      V32.alloc(c, (size_t)l * l);
      eye_kernel<float><<<grid_for((int64_t)l * l), 256, 0, c.stream>>>(V32.p, l);
      BRSVD_CHECK_LAUNCH();
      jacobi<float>(c, M32.p, l, l, l, V32.p, l, 1e-5, 40, floor32, stop32);
      copy2d_kernel<float, double><<<grid_for((int64_t)l * l), 256, 0, c.stream>>>(
          V32.p, l, l, l, Vj.p, l);
      BRSVD_CHECK_LAUNCH();
      ns_refine(c, Vj.p, l, l, 2);
    }
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
  // fp32 data: the polish stops after a sweep whose largest rotated |cos|
  // stayed below 3.4e-5: the sweep after it would find at most K c^2 with
  // the measured quadratic-convergence constant K ~ 100 (config 2: sweep
  // maxima 1.1e-4 -> 1.2e-6 -> nothing above tol), i.e. ~1e-7, the fp32
  // output resolution -- so the empty confirmation sweep after the 1.2e-6
  // sweep is not run (3 -> 2 fp64 sweeps).  fp64 data always confirms.
  const double tol = sizeof(T) == 8 ? jacobi_tol_tight(l) : 1e-7;
  jacobi(c, M.p, l, l, l, Vj.p, l, tol, 40, -1.0, sizeof(T) == 8 ? 0.0 : 3.4e-5);
  jacobi_finish(c, M.p, l, l, l, Vj.p, l, sigma, W, l, Zj.p, l);
  complete_null_columns_kernel<<<1, 1024, (size_t)l * sizeof(double), c.stream>>>(
      W, l, l, l, sigma, 16.0 * l * 2.220446049250313e-16);
  BRSVD_CHECK_LAUNCH();
  apply_basis<T>(c, Qb.p, n, l, n, Zj.p, l, l, Vout, ldv);
  if (e != 0) {
    scale_copy_kernel<double><<<1, 256, 0, c.stream>>>(sigma, l, 1, l, sigma, l,
                                                       std::ldexp(1.0, e));
    BRSVD_CHECK_LAUNCH();
  }
  return rank;
}

}  // namespace brsvd
