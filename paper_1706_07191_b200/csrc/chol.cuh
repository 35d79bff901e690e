// Small dense Cholesky factorisation and triangular inverse (fp64, one CTA).
//
// These turn a Gram matrix G = X^T X into the basis change T = L^-T that
// makes X T orthonormal (Cholesky QR).  They replace, on the fast path, the
// Householder QR of tsqr (kernels.py:121-164) and the Gram eigen-solves of the
// Jacobi route, whose sequential depth is O(sweeps * l) against O(l / NB) here.
#pragma once
#include "common.cuh"

namespace brsvd {

constexpr int kCholNB = 32;

// In-place lower Cholesky of (A + shift I) (n x n, column-major, ld), blocked
// left-looking with NB-column panels staged in shared memory.  On exit the
// lower triangle holds L and the strict upper triangle is zero.
// info[0] = min_j pivot_j / (A_jj + shift) (1 for a perfectly orthogonal
// problem, <= 0 when the factorisation broke down); non-positive pivots are
// replaced by a tiny positive value so the output stays finite.
//
// With colnorm (||x_j||, the inverse column scaling) and rank_tol > 0,
// info[1] = #{j : L_jj ||x_j|| > rank_tol ||X||_F} -- the |diag R| criterion of
// the reference's tsqr_factor (kernels.py:155-157), since the Cholesky factor
// of the Gram is the R of an unpivoted QR of X.
//
// drop_ratio > 0 turns the factorisation rank-revealing in column order: a
// column whose pivot falls below drop_ratio of its diagonal lies numerically in
// the span of the earlier ones; its L column is zeroed (unit diagonal, so L
// stays invertible) and it is left out of `keep` (kept column indices, in
// order).  info[2] = number of kept columns, info[0] = min ratio over kept.
__global__ void chol_kernel(double* __restrict__ A, int n, int64_t ld, double shift,
                            double* __restrict__ info,
                            const double* __restrict__ colnorm_inv = nullptr,
                            double rank_tol = 0.0, double drop_ratio = 0.0,
                            int* __restrict__ keep = nullptr) {
  extern __shared__ double csm[];
  double* P = csm;                          // panel, rows x NB  (P[c * n + i])
  double* Lp = csm + (size_t)n * kCholNB;   // panel rows of L: Lp[k * NB + c], k < p0
  double* diag0 = Lp + (size_t)n * kCholNB; // original diagonal (+ shift)
  int* dropped = reinterpret_cast<int*>(diag0 + n);
  __shared__ double s_minr;
  const int tid = threadIdx.x, nt = blockDim.x;
  for (int j = tid; j < n; j += nt) diag0[j] = A[j * ld + j] + shift;
  if (tid == 0) s_minr = 1.0;
  __syncthreads();
  for (int p0 = 0; p0 < n; p0 += kCholNB) {
    const int nb = min(kCholNB, n - p0), rows = n - p0;
    for (int e = tid; e < rows * nb; e += nt) {
      const int i = e % rows, c = e / rows;
      double v = (i >= c) ? A[(int64_t)(p0 + c) * ld + (p0 + i)] : 0.0;
      if (i == c) v += shift;
      P[c * n + i] = v;
    }
    for (int e = tid; e < p0 * nb; e += nt) {
      const int c = e % nb, k = e / nb;
      Lp[k * kCholNB + c] = A[(int64_t)k * ld + (p0 + c)];
    }
    __syncthreads();
    // P -= L[p0:, :p0] Lp^T   (only the lower part i >= c matters)
    if (p0 > 0) {
      for (int e = tid; e < rows * nb; e += nt) {
        const int i = e % rows, c = e / rows;
        if (i < c) continue;
        double acc = 0.0;
        const double* lrow = A + (p0 + i);
#pragma unroll 8
        for (int k = 0; k < p0; ++k) acc = fma(lrow[(int64_t)k * ld], Lp[k * kCholNB + c], acc);
        P[c * n + i] -= acc;
      }
      __syncthreads();
    }
    // unblocked right-looking factorisation of the panel
    for (int c = 0; c < nb; ++c) {
      __shared__ double s_d;
      if (tid == 0) {
        double piv = P[c * n + c];
        const double dg = diag0[p0 + c];
        // a zero (dropped) column or a NaN pivot counts as a breakdown
        const double ratio = (dg > 0.0 && piv == piv) ? piv / dg : -1.0;
        // dropped (rank-revealing mode) or broken down (non-positive pivot):
        // zero column below a unit diagonal, so L stays finite and invertible
        if ((drop_ratio > 0.0 && !(ratio > drop_ratio)) || !(piv > 0.0)) {
          if (ratio < s_minr) s_minr = ratio;
          s_d = 0.0;
          P[c * n + c] = 1.0;
          dropped[p0 + c] = 1;
        } else {
          if (ratio < s_minr) s_minr = ratio;
          s_d = sqrt(piv);
          P[c * n + c] = s_d;
          dropped[p0 + c] = 0;
        }
      }
      __syncthreads();
      const double d = s_d;
      if (d == 0.0) {
        for (int i = c + 1 + tid; i < rows; i += nt) P[c * n + i] = 0.0;
      } else {
        for (int i = c + 1 + tid; i < rows; i += nt) P[c * n + i] /= d;
      }
      __syncthreads();
      for (int e = tid; e < rows * (nb - c - 1); e += nt) {
        const int i = e % rows, c2 = c + 1 + e / rows;
        if (i < c2) continue;
        P[c2 * n + i] = fma(-P[c * n + i], P[c * n + c2], P[c2 * n + i]);
      }
      __syncthreads();
    }
    for (int e = tid; e < rows * nb; e += nt) {
      const int i = e % rows, c = e / rows;
      if (i >= c) A[(int64_t)(p0 + c) * ld + (p0 + i)] = P[c * n + i];
    }
    __syncthreads();
  }
  for (int e = tid; e < n * n; e += nt) {
    const int i = e % n, j = e / n;
    if (i < j) A[(int64_t)j * ld + i] = 0.0;
  }
  __syncthreads();
  if (tid == 0 && info) {
    info[0] = s_minr;
    int kept = 0;
    for (int j = 0; j < n; ++j)
      if (!dropped[j]) {
        if (keep) keep[kept] = j;
        ++kept;
      }
    info[2] = (double)kept;
    if (colnorm_inv != nullptr) {
      double fro2 = 0.0;
      for (int j = 0; j < n; ++j)
        if (colnorm_inv[j] > 0.0) fro2 += 1.0 / (colnorm_inv[j] * colnorm_inv[j]);
      const double cut = rank_tol * sqrt(fro2);
      int rk = 0;
      for (int j = 0; j < n; ++j)
        if (!dropped[j] && colnorm_inv[j] > 0.0 && A[(int64_t)j * ld + j] / colnorm_inv[j] > cut)
          ++rk;
      info[1] = (double)rk;
    }
  }
}

// Tc[:, c] = T[:, keep[c]] for the kept columns (count from info[2]).
__global__ void compact_cols_kernel(const double* __restrict__ T, int l,
                                    const int* __restrict__ keep,
                                    const double* __restrict__ info, double* __restrict__ Tc) {
  const int k = (int)info[2];
  for (int e = blockIdx.x * blockDim.x + threadIdx.x; e < l * k; e += gridDim.x * blockDim.x) {
    const int i = e % l, c = e / l;
    Tc[(int64_t)c * l + i] = T[(int64_t)keep[c] * l + i];
  }
}

// X = L^-1 for lower-triangular L (n x n, column-major), by block rows:
// X_i = L_ii^-1 (E_i - sum_{k<i} L_ik X_k).  Writes T = s .* X^T, i.e.
// T[k, j] = s_k X[j, k], the basis change with the column scaling folded in
// (s may be NULL for no scaling).  One CTA.
__global__ void trinv_t_kernel(const double* __restrict__ L, int n, int64_t ld,
                               const double* __restrict__ s, double* __restrict__ X,
                               double* __restrict__ T) {
  extern __shared__ double tsm[];
  double* Lr = tsm;                               // block row of L: Lr[k * NB + r], k < i0
  double* Li = tsm + (size_t)n * kCholNB;         // L_ii inverse, NB x NB: Li[c * NB + r]
  double* R = Li + kCholNB * kCholNB;             // rhs block: R[c * NB + r], c < n
  const int tid = threadIdx.x, nt = blockDim.x;
  for (int e = tid; e < n * n; e += nt) X[e] = 0.0;
  __syncthreads();
  for (int i0 = 0; i0 < n; i0 += kCholNB) {
    const int nb = min(kCholNB, n - i0);
    const int ncols = i0 + nb;  // columns 0..ncols-1 have nonzeros in this row block
    for (int e = tid; e < i0 * nb; e += nt) {
      const int r = e % nb, k = e / nb;
      Lr[k * kCholNB + r] = L[(int64_t)k * ld + (i0 + r)];
    }
    // diagonal block staged in shared memory (R doubles as scratch here)
    for (int e = tid; e < nb * nb; e += nt) {
      const int r = e % nb, k = e / nb;
      R[k * kCholNB + r] = L[(int64_t)(i0 + k) * ld + (i0 + r)];
    }
    __syncthreads();
    // inverse of the diagonal block by forward substitution, one thread per column
    if (tid < nb) {
      const int c = tid;
      for (int r = 0; r < nb; ++r) {
        double v = (r == c) ? 1.0 : 0.0;
        for (int k = c; k < r; ++k) v = fma(-R[k * kCholNB + r], Li[c * kCholNB + k], v);
        Li[c * kCholNB + r] = (r >= c) ? v / R[r * kCholNB + r] : 0.0;
      }
    }
    __syncthreads();
    // R = E_i - L[i-block, :i0] X[:i0, :ncols]
    for (int e = tid; e < nb * ncols; e += nt) {
      const int r = e % nb, c = e / nb;
      double acc = (i0 + r == c) ? 1.0 : 0.0;
      for (int k = c; k < i0; ++k) acc = fma(-Lr[k * kCholNB + r], X[(int64_t)c * n + k], acc);
      R[c * kCholNB + r] = acc;
    }
    __syncthreads();
    // X[i-block, :ncols] = Li R
    for (int e = tid; e < nb * ncols; e += nt) {
      const int r = e % nb, c = e / nb;
      double acc = 0.0;
      for (int k = 0; k <= r; ++k) acc = fma(Li[k * kCholNB + r], R[c * kCholNB + k], acc);
      X[(int64_t)c * n + (i0 + r)] = acc;
    }
    __syncthreads();
  }
  for (int e = tid; e < n * n; e += nt) {
    const int k = e % n, j = e / n;
    const double sk = s ? s[k] : 1.0;
    T[(int64_t)j * n + k] = sk * X[(int64_t)k * n + j];
  }
}

inline size_t chol_smem(int n) {
  return ((size_t)n * kCholNB * 2 + (size_t)n) * sizeof(double) + (size_t)n * sizeof(int);
}
inline size_t trinv_smem(int n) {
  return ((size_t)n * kCholNB + kCholNB * kCholNB + (size_t)n * kCholNB) * sizeof(double);
}

}  // namespace brsvd
