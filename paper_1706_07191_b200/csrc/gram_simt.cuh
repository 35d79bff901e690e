// Tall-skinny Gram products in fp64: C (a x b) = X^T Y for column-major
// X (r x a), Y (r x b) of fp32 or fp64 data, r >> a, b.
//
// These are the fp64 Grams of the Cholesky QR passes (the Cholesky factor of
// X^T X is the R of tsqr, kernels.py:121-164) and the core M = B Q_b of
// small_svd (kernels.py:173-188).  fp32 inputs are exact in fp64 and every
// product is exact, so the only rounding is the fp64 accumulation.
//
// 96 x 96 or 128 x 128 output tiles (the one that pads l least; symmetric
// case: lower-triangle tiles only), 8 x 4 register tiles per thread fed by 16-byte shared loads of k-major
// slabs, register-prefetched double buffering, and a deterministic split-K:
// every split writes its partial tile, a second kernel sums the partials in a
// fixed order (bitwise reproducible, tests/test_gpu_parity.py::test_deterministic).
#pragma once
#include "common.cuh"

namespace brsvd {
namespace gram {

constexpr int BK = 32;  // k slab
// NCG column groups of stride CS = BT / NCG: each thread owns 8 rows (two
// halves) x 2 NCG columns (2 per group); NCG = 3 at BT = 96 gives 8 x 6
// register tiles (48 FMAs per 7 16-byte shared loads)
template <int BT, int NCG = 2> struct Cfg {
  static constexpr int LDS = BT + 4;                       // padded k-major row (doubles)
  static constexpr int CS = BT / NCG;                      // column-group stride
  static constexpr int TY = BT / 8, TX = CS / 2;           // 8 x (2 NCG) outputs per thread
  static constexpr int NT = TX * TY;
  static_assert(TX % 8 == 0 && TY % 4 == 0, "warp patches of 8 x 4 threads");
  static constexpr int PER = (BT * BK + NT - 1) / NT;      // loader elements per thread
  static constexpr size_t SMEM = (size_t)2 * 2 * BK * LDS * sizeof(double);
};

template <typename TX, typename TY, int BT, int NCG>
__global__ void __launch_bounds__(Cfg<BT, NCG>::NT,
                                  (Cfg<BT, NCG>::NT <= 288 && sizeof(TX) == 4) ? 2 : 1)
    gram_tile_kernel(int64_t r, int a, int b, const TX* __restrict__ X, int64_t ldx,
                     const TY* __restrict__ Y, int64_t ldy, int sym, int ntj, int64_t kchunk,
                     double* __restrict__ part) {
  using C = Cfg<BT, NCG>;
  constexpr int LDS = C::LDS, NTX = C::TX, NT = C::NT, PER = C::PER, H = BT / 2;
  constexpr int CS = C::CS, NV = 2 * NCG;
  extern __shared__ __align__(16) double gsm[];
  double(*As)[BK][LDS] = reinterpret_cast<double(*)[BK][LDS]>(gsm);
  double(*Bs)[BK][LDS] = reinterpret_cast<double(*)[BK][LDS]>(gsm + 2 * BK * LDS);
  const int tid = threadIdx.x;
  // each warp covers an 8 (tx) x 4 (ty) patch of threads, so its 16-byte
  // shared loads touch 8 (B) / 4 (A) contiguous addresses: one wavefront each
  const int lane = tid & 31, wid = tid >> 5;
  const int tx = (wid % (NTX / 8)) * 8 + (lane & 7);
  const int ty = (wid / (NTX / 8)) * 4 + (lane >> 3);
  // tile index -> (ti, tj)
  int ti, tj;
  const int t = blockIdx.x;
  if (sym) {
    ti = (int)((sqrt(8.0 * t + 1.0) - 1.0) * 0.5);
    while ((ti + 1) * (ti + 2) / 2 <= t) ++ti;
    while (ti * (ti + 1) / 2 > t) --ti;
    tj = t - ti * (ti + 1) / 2;
  } else {
    ti = t / ntj;
    tj = t % ntj;
  }
  const int i0 = ti * BT, j0 = tj * BT;
  const int64_t kb = (int64_t)blockIdx.y * kchunk;
  const int64_t ke = min(r, kb + kchunk);

  // loader: element e -> column e / BK, k e % BK (consecutive threads read
  // consecutive rows of one column: coalesced)
  // raw (unconverted) prefetch registers: the fp64 conversion happens at the
  // shared store, after the compute of the current slab, so the global load
  // latency stays hidden
  TX ra[PER];
  TY rb[PER];
  auto load = [&](int64_t k0) {
#pragma unroll
    for (int q = 0; q < PER; ++q) {
      const int e = tid + q * NT;
      const int lc = e / BK, lk = e % BK;
      const int64_t k = k0 + lk;
      const bool ok = e < BT * BK && k < ke;
      ra[q] = (ok && i0 + lc < a) ? X[k + (int64_t)(i0 + lc) * ldx] : TX(0);
      rb[q] = (ok && j0 + lc < b) ? Y[k + (int64_t)(j0 + lc) * ldy] : TY(0);
    }
  };
  auto store = [&](int buf) {
#pragma unroll
    for (int q = 0; q < PER; ++q) {
      const int e = tid + q * NT;
      if (e < BT * BK) {
        As[buf][e % BK][e / BK] = (double)ra[q];
        Bs[buf][e % BK][e / BK] = (double)rb[q];
      }
    }
  };
  double acc[8][NV];
#pragma unroll
  for (int u = 0; u < 8; ++u)
#pragma unroll
    for (int v = 0; v < NV; ++v) acc[u][v] = 0.0;

  int buf = 0;
  if (kb < ke) {
    load(kb);
    store(0);
  }
  __syncthreads();
  for (int64_t k0 = kb; k0 < ke; k0 += BK) {
    const bool more = k0 + BK < ke;
    if (more) load(k0 + BK);
#pragma unroll 4
    for (int kk = 0; kk < BK; ++kk) {
      // rows ty*4 .. +3 and BT/2 + ty*4 .. +3 (about two distinct row groups
      // per warp: broadcasts); columns tx*2, +1 and BT/2 + tx*2, +1 (each
      // 16-byte load spans contiguous bytes across the warp)
      const double2* pa = reinterpret_cast<const double2*>(&As[buf][kk][ty * 4]);
      const double2* pb = reinterpret_cast<const double2*>(&Bs[buf][kk][tx * 2]);
      const double2 a01 = pa[0], a23 = pa[1], a45 = pa[H / 2], a67 = pa[H / 2 + 1];
      const double av[8] = {a01.x, a01.y, a23.x, a23.y, a45.x, a45.y, a67.x, a67.y};
      double bv[NV];
#pragma unroll
      for (int q = 0; q < NCG; ++q) {
        const double2 bq = pb[q * (CS / 2)];
        bv[2 * q] = bq.x;
        bv[2 * q + 1] = bq.y;
      }
#pragma unroll
      for (int u = 0; u < 8; ++u)
#pragma unroll
        for (int v = 0; v < NV; ++v) acc[u][v] = fma(av[u], bv[v], acc[u][v]);
    }
    if (more) {
      store(buf ^ 1);
      __syncthreads();
      buf ^= 1;
    }
  }
  // partial tile -> part[split][a x b] (column-major, ld a)
  double* P = part + (int64_t)blockIdx.y * a * b;
#pragma unroll
  for (int u = 0; u < 8; ++u) {
    const int i = i0 + (u < 4 ? ty * 4 + u : H + ty * 4 + u - 4);
    if (i >= a) continue;
#pragma unroll
    for (int v = 0; v < NV; ++v) {
      const int j = j0 + (v >> 1) * CS + tx * 2 + (v & 1);
      if (j < b) P[i + (int64_t)j * a] = acc[u][v];
    }
  }
}

// ---------------------------------------------------------------------------
// FP64 tensor-core (DMMA, mma.sync m8n8k4 f64) variant of the same tiled,
// split-K Gram: BT x BT output tiles, one 32 x 32 warp tile each (4 x 4 DMMA
// blocks, 32 fp64 accumulators per thread); X, Y slabs staged i-major
// (k contiguous, padded) so the loader's coalesced k-runs store without
// bank conflicts and each fragment load is two wavefronts.  Products of
// fp32 data are exact in fp64; fp64 accumulation as the SIMT kernel (the
// summation order differs, the partials are summed in the same fixed order).
constexpr int DBK = 16;   // k slab of the DMMA kernel
template <int BT> struct DCfg {
  static constexpr int LDK = DBK + 4;                       // padded k run (doubles)
  static constexpr int WT = BT / 32;                        // warp tiles per side
  static constexpr int NT = WT * WT * 32;
  static constexpr int PER = (BT * DBK + NT - 1) / NT;
  static constexpr size_t SMEM = (size_t)2 * 2 * BT * LDK * sizeof(double);
};

__device__ __forceinline__ void dmma_8x8x4(double& c0, double& c1, double a, double b) {
  asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0, %1}, {%2}, {%3}, "
               "{%0, %1};"
               : "+d"(c0), "+d"(c1)
               : "d"(a), "d"(b));
}

template <typename TX, typename TY, int BT>
__global__ void __launch_bounds__(DCfg<BT>::NT,
                                  (DCfg<BT>::NT <= 288 && sizeof(TX) == 4) ? 2 : 1)
    gram_dmma_kernel(int64_t r, int a, int b, const TX* __restrict__ X, int64_t ldx,
                     const TY* __restrict__ Y, int64_t ldy, int sym, int ntj, int64_t kchunk,
                     double* __restrict__ part) {
  using C = DCfg<BT>;
  constexpr int LDK = C::LDK, NT = C::NT, PER = C::PER, WT = C::WT;
  extern __shared__ __align__(16) double gsm[];
  double(*As)[BT][LDK] = reinterpret_cast<double(*)[BT][LDK]>(gsm);
  double(*Bs)[BT][LDK] = reinterpret_cast<double(*)[BT][LDK]>(gsm + 2 * BT * LDK);
  const int tid = threadIdx.x, lane = tid & 31, wid = tid >> 5;
  const int wi = wid / WT, wj = wid % WT;
  int ti, tj;
  const int t = blockIdx.x;
  if (sym) {
    ti = (int)((sqrt(8.0 * t + 1.0) - 1.0) * 0.5);
    while ((ti + 1) * (ti + 2) / 2 <= t) ++ti;
    while (ti * (ti + 1) / 2 > t) --ti;
    tj = t - ti * (ti + 1) / 2;
  } else {
    ti = t / ntj;
    tj = t % ntj;
  }
  const int i0 = ti * BT, j0 = tj * BT;
  const int64_t kb = (int64_t)blockIdx.y * kchunk;
  const int64_t ke = min(r, kb + kchunk);
  TX ra[PER];
  TY rb[PER];
  auto load = [&](int64_t k0) {
#pragma unroll
    for (int q = 0; q < PER; ++q) {
      const int e = tid + q * NT;
      const int lc = e / DBK, lk = e % DBK;
      const int64_t k = k0 + lk;
      const bool ok = e < BT * DBK && k < ke;
      ra[q] = (ok && i0 + lc < a) ? X[k + (int64_t)(i0 + lc) * ldx] : TX(0);
      rb[q] = (ok && j0 + lc < b) ? Y[k + (int64_t)(j0 + lc) * ldy] : TY(0);
    }
  };
  auto store = [&](int buf) {
#pragma unroll
    for (int q = 0; q < PER; ++q) {
      const int e = tid + q * NT;
      if (e < BT * DBK) {
        As[buf][e / DBK][e % DBK] = (double)ra[q];
        Bs[buf][e / DBK][e % DBK] = (double)rb[q];
      }
    }
  };
  double acc[4][4][2];
#pragma unroll
  for (int u = 0; u < 4; ++u)
#pragma unroll
    for (int v = 0; v < 4; ++v) acc[u][v][0] = acc[u][v][1] = 0.0;
  const int fr = lane >> 2, fk = lane & 3;   // fragment row / k of this lane
  int buf = 0;
  if (kb < ke) {
    load(kb);
    store(0);
  }
  __syncthreads();
  for (int64_t k0 = kb; k0 < ke; k0 += DBK) {
    const bool more = k0 + DBK < ke;
    if (more) load(k0 + DBK);
#pragma unroll
    for (int kk = 0; kk < DBK; kk += 4) {
      double av[4], bv[4];
#pragma unroll
      for (int u = 0; u < 4; ++u) av[u] = As[buf][wi * 32 + u * 8 + fr][kk + fk];
#pragma unroll
      for (int v = 0; v < 4; ++v) bv[v] = Bs[buf][wj * 32 + v * 8 + fr][kk + fk];
#pragma unroll
      for (int u = 0; u < 4; ++u)
#pragma unroll
        for (int v = 0; v < 4; ++v) dmma_8x8x4(acc[u][v][0], acc[u][v][1], av[u], bv[v]);
    }
    if (more) {
      store(buf ^ 1);
      __syncthreads();
      buf ^= 1;
    }
  }
  double* P = part + (int64_t)blockIdx.y * a * b;
#pragma unroll
  for (int u = 0; u < 4; ++u) {
    const int i = i0 + wi * 32 + u * 8 + fr;
    if (i >= a) continue;
#pragma unroll
    for (int v = 0; v < 4; ++v)
#pragma unroll
      for (int e = 0; e < 2; ++e) {
        const int j = j0 + wj * 32 + v * 8 + 2 * fk + e;
        if (j < b) P[i + (int64_t)j * a] = acc[u][v][e];
      }
  }
}

// C = sum over splits (fixed order); sym: mirror the lower-triangle tiles.
__global__ void gram_reduce_kernel(const double* __restrict__ part, int a, int b, int splits,
                                   int sym, int BT, double* __restrict__ C, int64_t ldc) {
  const int64_t total = (int64_t)a * b;
  for (int64_t idx = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; idx < total;
       idx += (int64_t)gridDim.x * blockDim.x) {
    int i = (int)(idx % a), j = (int)(idx / a);
    int si = i, sj = j;
    if (sym && (i / BT) < (j / BT)) {  // upper tile: read the mirrored lower entry
      si = j;
      sj = i;
    }
    const int64_t src = si + (int64_t)sj * a;
    double s = 0.0;
    for (int z = 0; z < splits; ++z) s += part[(int64_t)z * total + src];
    C[i + (int64_t)j * ldc] = s;
  }
}

}  // namespace gram
}  // namespace brsvd
