// Strided SIMT GEMM for the small/skinny products of the pipeline (Gram
// matrices, l-by-l basis changes, projections) and the generic fallback for
// the big tall-skinny passes.  Deterministic split-K: partial tiles go to a
// workspace and are summed in a fixed order, so results are bit-identical run
// to run (tests/test_gpu_parity.py::test_deterministic mirrors the reference's
// tests/test_rsvd.py:79-82).
//
//   C(M x N) = alpha * opA(M x K) * opB(K x N) + beta * C0
//   opA(i, k) = A[i * sam + k * sak],  opB(k, j) = B[k * sbk + j * sbn]
#pragma once
#include "common.cuh"

namespace brsvd {

template <typename TA, typename TB, typename TAcc, typename TC, int BM, int BN,
          int BK, int TM, int TN>
__global__ void __launch_bounds__((BM / TM) * (BN / TN))
    gemm_strided_kernel(int64_t M, int64_t N, int64_t K,
                        const TA* __restrict__ A, int64_t sam, int64_t sak,
                        const TB* __restrict__ B, int64_t sbk, int64_t sbn,
                        TC* C, int64_t scm, int64_t scn, TAcc alpha, TAcc beta,
                        const TC* C0, int64_t sc0m, int64_t sc0n,
                        int64_t kchunk, TAcc* __restrict__ part) {
  constexpr int NTX = BN / TN, NTY = BM / TM, NT = NTX * NTY;
  __shared__ TAcc As[BK][BM + 1];
  __shared__ TAcc Bs[BK][BN + 1];
  const int tid = threadIdx.x;
  const int tx = tid % NTX, ty = tid / NTX;
  const int64_t m0 = (int64_t)blockIdx.x * BM, n0 = (int64_t)blockIdx.y * BN;
  const int64_t kbeg = (int64_t)blockIdx.z * kchunk;
  const int64_t kend = min(K, kbeg + kchunk);
  TAcc acc[TM][TN];
#pragma unroll
  for (int r = 0; r < TM; ++r)
#pragma unroll
    for (int c = 0; c < TN; ++c) acc[r][c] = TAcc(0);
  const bool a_kfast = (sak == 1);
  const bool b_kfast = (sbk == 1);
  for (int64_t k0 = kbeg; k0 < kend; k0 += BK) {
    for (int e = tid; e < BM * BK; e += NT) {
      int i, k;
      if (a_kfast) { k = e % BK; i = e / BK; } else { i = e % BM; k = e / BM; }
      const int64_t gi = m0 + i, gk = k0 + k;
      TAcc v = TAcc(0);
      if (gi < M && gk < kend) v = (TAcc)A[gi * sam + gk * sak];
      As[k][i] = v;
    }
    for (int e = tid; e < BN * BK; e += NT) {
      int j, k;
      if (b_kfast) { k = e % BK; j = e / BK; } else { j = e % BN; k = e / BN; }
      const int64_t gj = n0 + j, gk = k0 + k;
      TAcc v = TAcc(0);
      if (gj < N && gk < kend) v = (TAcc)B[gk * sbk + gj * sbn];
      Bs[k][j] = v;
    }
    __syncthreads();
#pragma unroll
    for (int kk = 0; kk < BK; ++kk) {
      TAcc a[TM], b[TN];
#pragma unroll
      for (int r = 0; r < TM; ++r) a[r] = As[kk][ty + r * NTY];
#pragma unroll
      for (int c = 0; c < TN; ++c) b[c] = Bs[kk][tx + c * NTX];
#pragma unroll
      for (int r = 0; r < TM; ++r)
#pragma unroll
        for (int c = 0; c < TN; ++c) acc[r][c] = fma(a[r], b[c], acc[r][c]);
    }
    __syncthreads();
  }
  const bool split = gridDim.z > 1;
#pragma unroll
  for (int r = 0; r < TM; ++r) {
    const int64_t i = m0 + ty + r * NTY;
    if (i >= M) continue;
#pragma unroll
    for (int c = 0; c < TN; ++c) {
      const int64_t j = n0 + tx + c * NTX;
      if (j >= N) continue;
      if (split) {
        part[(int64_t)blockIdx.z * M * N + i + j * M] = acc[r][c];
      } else {
        TAcc v = alpha * acc[r][c];
        if (C0 != nullptr) v += beta * (TAcc)C0[i * sc0m + j * sc0n];
        C[i * scm + j * scn] = (TC)v;
      }
    }
  }
}

template <typename TAcc, typename TC>
__global__ void splitk_reduce_kernel(int64_t M, int64_t N, int splits,
                                     const TAcc* __restrict__ part, TC* C,
                                     int64_t scm, int64_t scn, TAcc alpha,
                                     TAcc beta, const TC* C0, int64_t sc0m,
                                     int64_t sc0n) {
  const int64_t total = M * N;
  for (int64_t idx = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
       idx < total; idx += (int64_t)gridDim.x * blockDim.x) {
    const int64_t i = idx % M, j = idx / M;
    TAcc s = TAcc(0);
    for (int z = 0; z < splits; ++z) s += part[(int64_t)z * total + idx];
    TAcc v = alpha * s;
    if (C0 != nullptr) v += beta * (TAcc)C0[i * sc0m + j * sc0n];
    C[i * scm + j * scn] = (TC)v;
  }
}

// Same sum for small outputs with many splits: one warp per output, lanes
// take a fixed strided subset of the splits, then a fixed butterfly --
// deterministic, and ~splits/32 dependent adds instead of splits.
template <typename TAcc, typename TC>
__global__ void splitk_reduce_warp_kernel(int64_t M, int64_t N, int splits,
                                          const TAcc* __restrict__ part, TC* C, int64_t scm,
                                          int64_t scn, TAcc alpha, TAcc beta, const TC* C0,
                                          int64_t sc0m, int64_t sc0n) {
  const int64_t total = M * N;
  const int lane = threadIdx.x & 31;
  for (int64_t idx = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) >> 5; idx < total;
       idx += ((int64_t)gridDim.x * blockDim.x) >> 5) {
    TAcc s = TAcc(0);
    for (int z = lane; z < splits; z += 32) s += part[(int64_t)z * total + idx];
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) s += __shfl_xor_sync(0xffffffffu, s, o);
    if (lane == 0) {
      const int64_t i = idx % M, j = idx / M;
      TAcc v = alpha * s;
      if (C0 != nullptr) v += beta * (TAcc)C0[i * sc0m + j * sc0n];
      C[i * scm + j * scn] = (TC)v;
    }
  }
}

}  // namespace brsvd
