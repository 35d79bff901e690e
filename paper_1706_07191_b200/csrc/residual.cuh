// Fused residual of a rank-l factorisation (relative_frobenius_error,
// rsvd.py:396-432): one streaming pass over A computing
//   num = ||A - U diag(sigma) Vt||_F^2,   den = ||A||_F^2
// without materialising the m x n reconstruction.  Each CTA forms a 128 x 128
// tile of U diag(sigma) Vt in registers (K = l in 16-deep shared slabs,
// 8 x 8 outputs per thread), subtracts it from the A tile as it is read, and
// reduces both sums of squares in fp64.  Per-CTA partials are summed in a
// fixed order (deterministic).
#pragma once
#include "runtime.cuh"

namespace brsvd {
namespace res {

constexpr int BT = 128, BK = 16, NT = 256;

template <typename T>
__global__ void __launch_bounds__(NT)
    residual_kernel(int64_t m, int64_t n, const T* __restrict__ A, int64_t lda, int row_major,
                    const T* __restrict__ U, int64_t ldu, const T* __restrict__ sig,
                    const T* __restrict__ Vt, int64_t ldv, int l, int tiles_n,
                    double* __restrict__ part) {
  __shared__ __align__(16) T Us[BK][BT];
  __shared__ __align__(16) T Vs[BK][BT];
  __shared__ double red[2][NT / 32];
  const int tid = threadIdx.x, tx = tid & 15, ty = tid >> 4;
  const int64_t i0 = (int64_t)(blockIdx.x / tiles_n) * BT;
  const int64_t j0 = (int64_t)(blockIdx.x % tiles_n) * BT;
  T acc[8][8];
#pragma unroll
  for (int u = 0; u < 8; ++u)
#pragma unroll
    for (int v = 0; v < 8; ++v) acc[u][v] = T(0);
  for (int k0 = 0; k0 < l; k0 += BK) {
    // U diag(sigma) slab (k-major) and Vt slab; 2048 elements each
#pragma unroll
    for (int q = 0; q < BT * BK / NT; ++q) {
      const int e = tid + q * NT;
      const int c = e % BT, k = e / BT;
      const int kk = k0 + k;
      const int64_t gi = i0 + c, gj = j0 + c;
      Us[k][c] = (kk < l && gi < m) ? U[gi + (int64_t)kk * ldu] * sig[kk] : T(0);
      Vs[k][c] = (kk < l && gj < n) ? Vt[(int64_t)kk * ldv + gj] : T(0);
    }
    __syncthreads();
#pragma unroll
    for (int k = 0; k < BK; ++k) {
      T av[8], bv[8];
#pragma unroll
      for (int q = 0; q < 4; ++q) {
        av[q] = Us[k][ty * 4 + q];
        av[4 + q] = Us[k][64 + ty * 4 + q];
        bv[q] = Vs[k][tx * 4 + q];
        bv[4 + q] = Vs[k][64 + tx * 4 + q];
      }
#pragma unroll
      for (int u = 0; u < 8; ++u)
#pragma unroll
        for (int v = 0; v < 8; ++v) acc[u][v] = fma(av[u], bv[v], acc[u][v]);
    }
    __syncthreads();
  }
  double num = 0.0, den = 0.0;
#pragma unroll
  for (int u = 0; u < 8; ++u) {
    const int64_t i = i0 + (u < 4 ? ty * 4 + u : 64 + ty * 4 + u - 4);
    if (i >= m) continue;
#pragma unroll
    for (int v = 0; v < 8; ++v) {
      const int64_t j = j0 + (v < 4 ? tx * 4 + v : 64 + tx * 4 + v - 4);
      if (j >= n) continue;
      const double a = (double)A[row_major ? i * lda + j : i + j * lda];
      const double d = a - (double)acc[u][v];
      num = fma(d, d, num);
      den = fma(a, a, den);
    }
  }
  num = warp_sum(num);
  den = warp_sum(den);
  if ((tid & 31) == 0) {
    red[0][tid >> 5] = num;
    red[1][tid >> 5] = den;
  }
  __syncthreads();
  if (tid == 0) {
    double s0 = 0.0, s1 = 0.0;
    for (int w = 0; w < NT / 32; ++w) {
      s0 += red[0][w];
      s1 += red[1][w];
    }
    part[2 * (int64_t)blockIdx.x] = s0;
    part[2 * (int64_t)blockIdx.x + 1] = s1;
  }
}

// Fixed-order sum of the per-CTA partials: out[0] += num, out[1] += den.
__global__ void residual_sum_kernel(const double* __restrict__ part, int64_t count,
                                    double* __restrict__ out) {
  __shared__ double red[2][32];
  double s0 = 0.0, s1 = 0.0;
  for (int64_t i = threadIdx.x; i < count; i += blockDim.x) {
    s0 += part[2 * i];
    s1 += part[2 * i + 1];
  }
  s0 = warp_sum(s0);
  s1 = warp_sum(s1);
  if ((threadIdx.x & 31) == 0) {
    red[0][threadIdx.x >> 5] = s0;
    red[1][threadIdx.x >> 5] = s1;
  }
  __syncthreads();
  if (threadIdx.x == 0) {
    double t0 = 0.0, t1 = 0.0;
    for (int w = 0; w < (int)(blockDim.x >> 5); ++w) {
      t0 += red[0][w];
      t1 += red[1][w];
    }
    out[0] += t0;
    out[1] += t1;
  }
}

}  // namespace res

template <typename T>
void residual_device(Ctx& c, const T* A, int64_t m, int64_t n, int64_t lda, bool row_major,
                     const T* U, int64_t ldu, const T* sig, const T* Vt, int64_t ldv, int l,
                     double* out_host) {
  using namespace res;
  const int tiles_n = (int)ceil_div(n, BT);
  const int64_t tiles = ceil_div(m, BT) * tiles_n;
  DBuf<double> part(c, (size_t)(2 * tiles)), sums(c, 2);
  BRSVD_CUDA(cudaMemsetAsync(sums.p, 0, 2 * sizeof(double), c.stream));
  if (tiles > 0) {
    residual_kernel<T><<<(unsigned)tiles, NT, 0, c.stream>>>(m, n, A, lda, row_major ? 1 : 0,
                                                              U, ldu, sig, Vt, ldv, l, tiles_n,
                                                              part.p);
    BRSVD_CHECK_LAUNCH();
    residual_sum_kernel<<<1, 1024, 0, c.stream>>>(part.p, tiles, sums.p);
    BRSVD_CHECK_LAUNCH();
  }
  readback(c, sums.p, out_host, 2 * sizeof(double));
}

}  // namespace brsvd
