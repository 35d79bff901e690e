// Small helper kernels: Gram preparation, basis construction, Newton-Schulz
// correction, overflow probe, sign canonicalisation, Gaussian sketch.
#pragma once
#include "common.cuh"

namespace brsvd {

// --- Gram preparation --------------------------------------------------------
// s_j = 1/sqrt(G_jj) (0 for a zero column; 1 everywhere when !scale),
// G <- S G S (symmetrised), V <- I, trace[0] = sum_j G_jj (before scaling).
__global__ void gram_prep_kernel(double* __restrict__ G, int l,
                                 double* __restrict__ s,
                                 double* __restrict__ V, int scale,
                                 double* __restrict__ trace, double drop) {
  __shared__ double red[32], redm[32];
  double tr = 0.0, dmax = 0.0;
  for (int j = threadIdx.x; j < l; j += blockDim.x) {
    const double d = G[j * (int64_t)l + j];
    tr += d;
    dmax = fmax(dmax, d);
  }
  tr = warp_sum(tr);
  dmax = warp_max(dmax);
  if ((threadIdx.x & 31) == 0) {
    red[threadIdx.x >> 5] = tr;
    redm[threadIdx.x >> 5] = dmax;
  }
  __syncthreads();
  if (threadIdx.x == 0) {
    double t = 0.0, mx = 0.0;
    for (int w = 0; w < (int)(blockDim.x >> 5); ++w) {
      t += red[w];
      mx = fmax(mx, redm[w]);
    }
    red[0] = t;
    redm[0] = mx;
    if (trace != nullptr) *trace = t;
  }
  __syncthreads();
  // Columns negligible against the largest (||x_j|| <= drop * max ||x_i||)
  // are left out of the scaled problem: their content is below the data's
  // resolution, and the deflation level / completion of orth_full handles it.
  const double floor2 = drop * drop * redm[0];
  for (int j = threadIdx.x; j < l; j += blockDim.x) {
    const double d = G[j * (int64_t)l + j];
    s[j] = scale ? (d > floor2 && d > 0.0 ? 1.0 / sqrt(d) : 0.0) : 1.0;
  }
  __syncthreads();
  for (int idx = threadIdx.x; idx < l * l; idx += blockDim.x) {
    const int i = idx % l, j = idx / l;
    if (i > j) continue;
    const double g = 0.5 * (G[j * (int64_t)l + i] + G[i * (int64_t)l + j]);
    const double v = s[i] * g * s[j];
    G[j * (int64_t)l + i] = v;
    G[i * (int64_t)l + j] = v;
  }
  for (int idx = threadIdx.x; idx < l * l; idx += blockDim.x) {
    const int i = idx % l, j = idx / l;
    V[idx] = (i == j) ? 1.0 : 0.0;
  }
}

// --- basis construction from the eigenpairs of the scaled Gram ---------------
// mode 0 (regularised, for the power-iteration normalisation):
//     T[:, j] = s .* E[:, j] / sqrt(max(lam_j, tau * lam_0))
// mode 1 (rank-revealing, for orthonormal bases):
//     rank = #{j : lam_j > tau * lam_0};  T[:, j] = s .* E[:, j] / sqrt(lam_j)
//     for j < rank, zero otherwise.
// lam (= sv from jacobi_finish on the symmetric PSD Gram) is sorted desc.
__global__ void build_basis_kernel(const double* __restrict__ E,
                                   const double* __restrict__ lam,
                                   const double* __restrict__ s, int l,
                                   double tau, int mode,
                                   double* __restrict__ T,
                                   int* __restrict__ rank_out) {
  const double lam0 = lam[0];
  const double floor_ = tau * lam0;
  __shared__ int s_rank;
  if (threadIdx.x == 0) {
    int r = 0;
    if (lam0 > 0.0)
      for (int j = 0; j < l; ++j) r += lam[j] > floor_;
    s_rank = r;
    if (rank_out != nullptr) *rank_out = r;
  }
  __syncthreads();
  const int rank = s_rank;
  for (int idx = threadIdx.x; idx < l * l; idx += blockDim.x) {
    const int i = idx % l, j = idx / l;
    double w;
    if (mode == 0) {
      const double d = fmax(lam[j], floor_);
      w = d > 0.0 ? 1.0 / sqrt(d) : 0.0;
    } else {
      w = j < rank ? 1.0 / sqrt(lam[j]) : 0.0;
    }
    T[idx] = s[i] * E[idx] * w;
  }
}

// T2 = 1.5 I - 0.5 G2   (one Newton-Schulz step toward the polar factor).
__global__ void ns_matrix_kernel(const double* __restrict__ G2, int r,
                                 double* __restrict__ T2) {
  for (int idx = blockIdx.x * blockDim.x + threadIdx.x; idx < r * r;
       idx += gridDim.x * blockDim.x) {
    const int i = idx % r, j = idx / r;
    const double g = 0.5 * (G2[idx] + G2[i * r + j]);
    T2[idx] = (i == j ? 1.5 : 0.0) - 0.5 * g;
  }
}

__global__ void transpose_square_kernel(const double* __restrict__ A, int l,
                                        double* __restrict__ At) {
  for (int idx = blockIdx.x * blockDim.x + threadIdx.x; idx < l * l;
       idx += gridDim.x * blockDim.x) {
    const int i = idx % l, j = idx / l;
    At[i * (int64_t)l + j] = A[idx];
  }
}

template <typename R = double>
__global__ void eye_kernel(R* __restrict__ V, int l) {
  for (int idx = blockIdx.x * blockDim.x + threadIdx.x; idx < l * l;
       idx += gridDim.x * blockDim.x)
    V[idx] = (idx % l == idx / l) ? R(1) : R(0);
}

// --- max |x| and finiteness (the overflow guard of rsvd.py:84-91) -------------
// out[0] receives the bit pattern of max|x| (non-negative doubles order like
// their bit patterns), out[1] a non-finite flag.
template <typename T>
__global__ void maxabs_kernel(const T* __restrict__ x, int64_t rows,
                              int64_t cols, int64_t ld,
                              unsigned long long* __restrict__ out) {
  double m = 0.0;
  int bad = 0;
  const int64_t total = rows * cols;
  if (ld == rows) {  // contiguous: a flat scan (no 64-bit index division)
    for (int64_t idx = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; idx < total;
         idx += (int64_t)gridDim.x * blockDim.x) {
      const double v = (double)x[idx];
      if (!isfinite(v)) bad = 1;
      else m = fmax(m, fabs(v));
    }
  } else {
    for (int64_t idx = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
         idx < total; idx += (int64_t)gridDim.x * blockDim.x) {
      const int64_t i = idx % rows, j = idx / rows;
      const double v = (double)x[i + j * ld];
      if (!isfinite(v)) bad = 1;
      else m = fmax(m, fabs(v));
    }
  }
  m = warp_max(m);
  bad = __reduce_or_sync(0xffffffffu, bad);
  if ((threadIdx.x & 31) == 0) {
    atomicMax(out, (unsigned long long)__double_as_longlong(m));
    if (bad) atomicOr(out + 1, 1ull);
  }
}

// --- _fix_signs (rsvd.py:105-115) ---------------------------------------------
// Per column of U (rows x l, col-major): index of the first largest |u_ij|,
// sign of that entry (0 -> +1).
template <typename T>
__global__ void colsign_kernel(const T* __restrict__ U, int64_t rows,
                               int64_t ldu, T* __restrict__ sign) {
  const int j = blockIdx.x;
  double best = -1.0;
  int64_t bidx = 0;
  for (int64_t i = threadIdx.x; i < rows; i += blockDim.x) {
    const double v = fabs((double)U[i + j * ldu]);
    if (v > best) { best = v; bidx = i; }
  }
  // warp argmax with lowest-index tie break
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) {
    const double ob = __shfl_xor_sync(0xffffffffu, best, o);
    const int64_t oi = __shfl_xor_sync(0xffffffffu, bidx, o);
    if (ob > best || (ob == best && oi < bidx)) { best = ob; bidx = oi; }
  }
  __shared__ double sb[32];
  __shared__ int64_t si[32];
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  if (lane == 0) { sb[warp] = best; si[warp] = bidx; }
  __syncthreads();
  if (threadIdx.x == 0) {
    const int nw = blockDim.x >> 5;
    for (int w = 1; w < nw; ++w)
      if (sb[w] > best || (sb[w] == best && si[w] < bidx)) { best = sb[w]; bidx = si[w]; }
    const T u = U[bidx + j * ldu];
    sign[j] = u < T(0) ? T(-1) : T(1);
  }
}

// Per column: max |U[i, j]| and the first row index attaining it (global
// index = row_offset + i).  One block per column.
template <typename T>
__global__ void colmax_kernel(const T* __restrict__ U, int64_t rows, int64_t ldu,
                              int64_t row_offset, double* __restrict__ vals,
                              int64_t* __restrict__ idx, double* __restrict__ entry = nullptr) {
  const int j = blockIdx.x;
  double best = -1.0;
  int64_t bidx = 0;
  for (int64_t i = threadIdx.x; i < rows; i += blockDim.x) {
    double v = fabs((double)U[i + j * ldu]);
    if (v != v) v = INFINITY;   // NaN propagates as non-finite (overflow guard)
    if (v > best) { best = v; bidx = i; }
  }
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) {
    const double ob = __shfl_xor_sync(0xffffffffu, best, o);
    const int64_t oi = __shfl_xor_sync(0xffffffffu, bidx, o);
    if (ob > best || (ob == best && oi < bidx)) { best = ob; bidx = oi; }
  }
  __shared__ double sb[32];
  __shared__ int64_t si[32];
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  if (lane == 0) { sb[warp] = best; si[warp] = bidx; }
  __syncthreads();
  if (threadIdx.x == 0) {
    for (int w = 1; w < (int)(blockDim.x >> 5); ++w)
      if (sb[w] > best || (sb[w] == best && si[w] < bidx)) { best = sb[w]; bidx = si[w]; }
    vals[j] = best;
    idx[j] = row_offset + bidx;
    if (entry) entry[j] = rows > 0 ? (double)U[bidx + j * ldu] : 0.0;
  }
}

// max |R| and max |strictly-lower R| of an l x l column-major matrix, as the
// bit patterns of non-negative doubles (atomicMax on the unsigned image).
template <typename T>
__global__ void tri_check_kernel(const T* __restrict__ R, int l,
                                 unsigned long long* __restrict__ out) {
  for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < (int64_t)l * l;
       e += (int64_t)gridDim.x * blockDim.x) {
    const int i = (int)(e % l), j = (int)(e / l);
    const double v = fabs((double)R[e]);
    const unsigned long long b = __double_as_longlong(v);
    atomicMax(out, b);
    if (i > j) atomicMax(out + 1, b);
  }
}
template <typename T>
__global__ void zero_strict_lower_kernel(T* __restrict__ R, int l) {
  for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < (int64_t)l * l;
       e += (int64_t)gridDim.x * blockDim.x)
    if ((int)(e % l) > (int)(e / l)) R[e] = T(0);
}

// In-place int64 -> double of a small index vector (exact below 2^53).
__global__ void idx_to_double_kernel(int64_t* idx, int64_t l) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < l;
       i += (int64_t)gridDim.x * blockDim.x) {
    const double d = (double)idx[i];
    reinterpret_cast<double*>(idx)[i] = d;
  }
}

template <typename T, typename S>
__global__ void scale_cols_by_kernel(T* __restrict__ X, int64_t rows, int64_t cols,
                                     int64_t ld, const S* __restrict__ scale) {
  const int64_t total = rows * cols;
  for (int64_t id = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; id < total;
       id += (int64_t)gridDim.x * blockDim.x) {
    const int64_t i = id % rows, j = id / rows;
    X[i + j * ld] = (T)((S)X[i + j * ld] * scale[j]);
  }
}

template <typename T>
__global__ void scale_cols_kernel(T* __restrict__ X, int64_t rows, int64_t cols,
                                  int64_t ld, const T* __restrict__ sign) {
  const int64_t total = rows * cols;
  if (total < (1ll << 31)) {  // 32-bit index arithmetic (cheaper division)
    const uint32_t r32 = (uint32_t)rows;
    for (uint32_t idx = blockIdx.x * blockDim.x + threadIdx.x; idx < (uint32_t)total;
         idx += gridDim.x * blockDim.x) {
      const uint32_t i = idx % r32, j = idx / r32;
      X[i + (int64_t)j * ld] *= sign[j];
    }
    return;
  }
  for (int64_t idx = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
       idx < total; idx += (int64_t)gridDim.x * blockDim.x) {
    const int64_t i = idx % rows, j = idx / rows;
    X[i + j * ld] *= sign[j];
  }
}

template <typename TS, typename TD>
__global__ void copy2d_kernel(const TS* __restrict__ src, int64_t rows,
                              int64_t cols, int64_t lds, TD* __restrict__ dst,
                              int64_t ldd) {
  const int64_t total = rows * cols;
  if (total < (1ll << 31)) {  // 32-bit index arithmetic (cheaper division)
    const uint32_t r32 = (uint32_t)rows;
    for (uint32_t idx = blockIdx.x * blockDim.x + threadIdx.x; idx < (uint32_t)total;
         idx += gridDim.x * blockDim.x) {
      const uint32_t i = idx % r32, j = idx / r32;
      dst[i + (int64_t)j * ldd] = (TD)src[i + (int64_t)j * lds];
    }
    return;
  }
  for (int64_t idx = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
       idx < total; idx += (int64_t)gridDim.x * blockDim.x) {
    const int64_t i = idx % rows, j = idx / rows;
    dst[i + j * ldd] = (TD)src[i + j * lds];
  }
}

// dst = src * s (s a power of two: exact), any leading dimensions.
template <typename T>
__global__ void scale_copy_kernel(const T* __restrict__ src, int64_t rows, int64_t cols,
                                  int64_t lds, T* __restrict__ dst, int64_t ldd, double s) {
  const int64_t total = rows * cols;
  for (int64_t idx = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; idx < total;
       idx += (int64_t)gridDim.x * blockDim.x) {
    const int64_t i = idx % rows, j = idx / rows;
    dst[i + j * ldd] = (T)((double)src[i + j * lds] * s);
  }
}

// dst = (TD)(src * s), s a power of two, any leading dimensions.
template <typename TS, typename TD>
__global__ void scale_cast_kernel(const TS* __restrict__ src, int64_t rows, int64_t cols,
                                  int64_t lds, TD* __restrict__ dst, int64_t ldd, double s) {
  const int64_t total = rows * cols;
  for (int64_t idx = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; idx < total;
       idx += (int64_t)gridDim.x * blockDim.x) {
    const int64_t i = idx % rows, j = idx / rows;
    dst[i + j * ldd] = (TD)((double)src[i + j * lds] * s);
  }
}

// --- Gaussian sketch ------------------------------------------------------------
// Counter-based Philox4x32-10: entry (row, col) is a pure function of
// (seed, stream, row, col), so a block generated with a row offset equals the
// matching slice of the full matrix -- the property gaussian_matrix
// (kernels.py:98-118) guarantees and tests/test_kernels.py:78-81 checks.
__device__ __forceinline__ uint4 philox4x32_10(uint4 c, uint2 k) {
#pragma unroll
  for (int r = 0; r < 10; ++r) {
    const uint32_t hi0 = __umulhi(0xD2511F53u, c.x), lo0 = 0xD2511F53u * c.x;
    const uint32_t hi1 = __umulhi(0xCD9E8D57u, c.z), lo1 = 0xCD9E8D57u * c.z;
    c = make_uint4(hi1 ^ c.y ^ k.x, lo1, hi0 ^ c.w ^ k.y, lo0);
    k.x += 0x9E3779B9u;
    k.y += 0xBB67AE85u;
  }
  return c;
}

// Two normals of the sketch stream for (global row, column pair pj): Philox
// counter (pj, row, stream), Box-Muller on two 53-bit uniforms.
__device__ __forceinline__ void gaussian_pair(uint64_t seed, uint64_t stream, uint64_t grow,
                                              int64_t pj, double& v0, double& v1) {
  const uint2 key = make_uint2((uint32_t)seed, (uint32_t)(seed >> 32));
  const uint4 ctr = make_uint4((uint32_t)pj, (uint32_t)grow, (uint32_t)(grow >> 32),
                               (uint32_t)stream ^ ((uint32_t)(stream >> 32) * 0x85EBCA6Bu));
  const uint4 x = philox4x32_10(ctr, key);
  // two 53-bit uniforms in (0, 1]
  const uint64_t a = ((uint64_t)x.x << 32) | x.y;
  const uint64_t b = ((uint64_t)x.z << 32) | x.w;
  const double u1 = ((a >> 11) + 1) * (1.0 / 9007199254740992.0);
  const double u2 = (b >> 11) * (1.0 / 9007199254740992.0);
  const double rad = sqrt(-2.0 * log(u1));
  double sn, cs;
  sincospi(2.0 * u2, &sn, &cs);
  v0 = rad * cs;
  v1 = rad * sn;
}

template <typename T>
__global__ void gaussian_kernel(T* __restrict__ out, int64_t rows, int64_t cols,
                                int64_t ld, uint64_t seed, uint64_t stream,
                                int64_t row_offset) {
  const int64_t half = (cols + 1) / 2;
  const int64_t total = rows * half;
  for (int64_t idx = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
       idx < total; idx += (int64_t)gridDim.x * blockDim.x) {
    const int64_t r = idx % rows, pj = idx / rows;
    double v0, v1;
    gaussian_pair(seed, stream, (uint64_t)(row_offset + r), pj, v0, v1);
    const int64_t c0 = 2 * pj;
    out[r + c0 * ld] = (T)v0;
    if (c0 + 1 < cols) out[r + (c0 + 1) * ld] = (T)v1;
  }
}

// The same stream as gaussian_kernel(out + k0 * ld, rows, l - k0, ...) with
// k0 = (int)info[2] read on the device (the kept count of a rank-revealing
// Cholesky pass): the completion columns k0 .. l-1, without a host read.
template <typename T>
__global__ void gaussian_tail_kernel(T* __restrict__ out, int64_t rows, int l, int64_t ld,
                                     const double* __restrict__ info, uint64_t seed,
                                     uint64_t stream) {
  const int k0 = (int)info[2];
  const int64_t cols = l - k0;
  const int64_t total = rows * ((cols + 1) / 2);
  for (int64_t idx = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
       idx < total; idx += (int64_t)gridDim.x * blockDim.x) {
    const int64_t r = idx % rows, pj = idx / rows;
    double v0, v1;
    gaussian_pair(seed, stream, (uint64_t)r, pj, v0, v1);
    const int64_t c0 = k0 + 2 * pj;
    out[r + c0 * ld] = (T)v0;
    if (2 * pj + 1 < cols) out[r + (c0 + 1) * ld] = (T)v1;
  }
}

}  // namespace brsvd
