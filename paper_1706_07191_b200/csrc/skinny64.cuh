// fp64 A-streaming products for skinny right-hand sides (l <= 64): the fp64
// path of big_nn / big_tn (Y = A X, Z = A^T Y).  HBM-bound by design: A is
// read exactly once, in 128-row x 32-k tiles moved by cp.async (16-byte,
// L2-only) through a 4-stage shared-memory ring, so ~100 KB per SM are in
// flight while the previous tiles are consumed.  Each thread owns R rows of
// op(A) (2 for l <= 24, else 1) for one k group of the tile (8 warps per
// block split the tile's k range) and their R x l fp64 accumulators, so every
// B value read from shared memory feeds 2R FMAs; the 32 x l slice of B (copied
// once per call into row-major k x LB order) is read as shared-memory
// broadcasts.  The two storage orders of op(A) differ only in the tile
// layout:
//   KC  op(A)(i, k) = A[i*lda + k]  (row-major A x, column-major A^T y):
//       tile As[row][k], rows padded to 34 doubles (conflict-free 16-byte
//       reads of k pairs);
//   MC  op(A)(i, k) = A[i + k*lda]  (row-major A^T y, column-major A x):
//       tile As[k][row].
// Long K is split over grid.y so the units fill up to 16 waves while the
// partials stay within ~1/8 of the A bytes (fp64 partials, summed in a fixed
// order by splitk_reduce_kernel): deterministic.
#pragma once
#include "runtime.cuh"

namespace brsvd {
namespace sk {

constexpr int kRows = 128;   // rows per tile
constexpr int kKT = 32;      // k per tile
constexpr int kStages = 4;
constexpr int kKcPitch = kKT + 2;
constexpr int kThreads = 256;

__device__ __forceinline__ void cp_async16(uint32_t dst, const void* src, int bytes) {
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16, %2;" ::"r"(dst), "l"(src),
               "r"(bytes)
               : "memory");
}
__device__ __forceinline__ void cp_async_commit() {
  asm volatile("cp.async.commit_group;" ::: "memory");
}
template <int N>
__device__ __forceinline__ void cp_async_wait() {
  asm volatile("cp.async.wait_group %0;" ::"n"(N) : "memory");
}

// Thread t: k group g = t / (kRows / R) takes k [g*GK, (g+1)*GK) of every
// tile for rows ri + (kRows / R) * r, ri = t % (kRows / R); the G groups'
// accumulators are summed (fixed order) at the end.
template <bool KC, int LB>
struct Layout {
  static constexpr int R = LB <= 24 ? 2 : 1;  // rows per thread
  static constexpr int RT = kRows / R;        // threads per k group
  static constexpr int G = kThreads / RT;     // k groups
  static constexpr int GK = kKT / G;          // k per group per tile
  static constexpr int a_elems = KC ? kRows * kKcPitch : kKT * kRows;
  static constexpr int b_elems = kKT * LB;
  static constexpr int stage_elems = a_elems + b_elems;
  static constexpr size_t smem = sizeof(double) * (size_t)stage_elems * kStages;
  static_assert((G - 1) * RT * R * LB <= stage_elems * kStages, "reduction scratch");
};

// Bt (K x LB, row-major, zero beyond l) <- B (K x l, column-major)
template <int LB>
__global__ void pack_b_kernel(const double* __restrict__ B, int64_t ldb, int64_t K, int l,
                              double* __restrict__ Bt) {
  for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < K * LB;
       e += (int64_t)gridDim.x * blockDim.x) {
    const int c = (int)(e % LB);
    const int64_t k = e / LB;
    Bt[e] = c < l ? B[k + (int64_t)c * ldb] : 0.0;
  }
}

template <bool KC, int LB>
__global__ void __launch_bounds__(kThreads)
    skinny_kernel(const double* __restrict__ A, int64_t M, int64_t K, int64_t lda,
                  const double* __restrict__ Bt, int l, int64_t kchunk,
                  double* __restrict__ C, int64_t ldc, double* __restrict__ part) {
  using L = Layout<KC, LB>;
  constexpr int R = L::R, RT = L::RT, GK = L::GK;
  extern __shared__ __align__(16) double sm[];
  const int tid = threadIdx.x;
  const int g = tid / RT, ri = tid % RT;
  const int64_t i0 = (int64_t)blockIdx.x * kRows;
  const int64_t kb = (int64_t)blockIdx.y * kchunk;
  const int64_t ke = min(K, kb + kchunk);
  const int nt = (int)((ke - kb + kKT - 1) / kKT);
  const uint32_t sbase = (uint32_t)__cvta_generic_to_shared(sm);

  // A-tile copy plan: every thread moves APT 16-byte pieces per tile, all in
  // one column of pieces, so the addresses are a per-thread base plus a
  // constant stride (computed once).
  constexpr int APT = kRows * kKT / 2 / kThreads;
  constexpr int PPR = KC ? kKT / 2 : kRows / 2;  // pieces per tile row (KC) / k row (MC)
  constexpr int LPJ = kThreads / PPR;            // tile rows (KC) / k rows (MC) per j
  const int pc = tid % PPR, pl = tid / PPR;
  const double* abase;
  int64_t astride;
  uint32_t adst0, rowmask = 0;
  int mc_bytes = 0;
  if (KC) {
    abase = A + (i0 + pl) * lda + 2 * pc;
    astride = (int64_t)LPJ * lda;
    adst0 = (uint32_t)(pl * kKcPitch + 2 * pc) * 8u;
#pragma unroll
    for (int j = 0; j < APT; ++j)
      if (i0 + pl + LPJ * j < M) rowmask |= 1u << j;
  } else {
    const int64_t row = i0 + 2 * pc;
    mc_bytes = row < M ? (row + 1 < M ? 16 : 8) : 0;
    abase = A + row + (int64_t)pl * lda;
    astride = (int64_t)LPJ * lda;
    adst0 = (uint32_t)(pl * kRows + 2 * pc) * 8u;
  }

  auto issue = [&](int t) {
    const int slot = t % kStages;
    const int64_t k0 = kb + (int64_t)t * kKT;
    const uint32_t sa = sbase + (uint32_t)(slot * L::stage_elems) * 8u;
    if (KC) {
      const int64_t kp = k0 + 2 * pc;
      const int kbytes = kp < ke ? (kp + 1 < ke ? 16 : 8) : 0;
      const double* src = abase + k0;
#pragma unroll
      for (int j = 0; j < APT; ++j) {
        const int bytes = ((rowmask >> j) & 1u) ? kbytes : 0;
        cp_async16(sa + adst0 + (uint32_t)(j * LPJ * kKcPitch) * 8u,
                   bytes ? src + j * astride : A, bytes);
      }
    } else {
      const double* src = abase + k0 * lda;
#pragma unroll
      for (int j = 0; j < APT; ++j) {
        const int bytes = (k0 + pl + LPJ * j < ke) ? mc_bytes : 0;
        cp_async16(sa + adst0 + (uint32_t)(j * LPJ * kRows) * 8u,
                   bytes ? src + j * astride : A, bytes);
      }
    }
    // B slice: kKT rows of LB doubles
    const uint32_t sb = sa + (uint32_t)L::a_elems * 8u;
    for (int p = tid; p < kKT * LB / 2; p += kThreads) {
      const int kk = p / (LB / 2), piece = p % (LB / 2);
      const int64_t k = k0 + kk;
      const int bytes = k < ke ? 16 : 0;
      cp_async16(sb + (uint32_t)(kk * LB + 2 * piece) * 8u,
                 bytes ? Bt + k * LB + 2 * piece : Bt, bytes);
    }
  };

  double acc[R][LB];
#pragma unroll
  for (int r = 0; r < R; ++r)
#pragma unroll
    for (int c = 0; c < LB; ++c) acc[r][c] = 0.0;
#pragma unroll
  for (int s = 0; s < kStages - 1; ++s) {
    if (s < nt) issue(s);
    cp_async_commit();
  }
  for (int t = 0; t < nt; ++t) {
    cp_async_wait<kStages - 2>();
    __syncthreads();  // tile t landed for all; slot (t-1) % kStages is free
    if (t + kStages - 1 < nt) issue(t + kStages - 1);
    cp_async_commit();
    const double* st = sm + (t % kStages) * L::stage_elems;
    const double* bs = st + L::a_elems;
#pragma unroll
    for (int k2 = 0; k2 < GK; k2 += 2) {
      const int kk = g * GK + k2;
      double a0[R], a1[R];
#pragma unroll
      for (int r = 0; r < R; ++r) {
        const int row = ri + RT * r;
        if (KC) {
          const double2 av = *reinterpret_cast<const double2*>(st + row * kKcPitch + kk);
          a0[r] = av.x;
          a1[r] = av.y;
        } else {
          a0[r] = st[kk * kRows + row];
          a1[r] = st[(kk + 1) * kRows + row];
        }
      }
      const double2* b0 = reinterpret_cast<const double2*>(bs + kk * LB);
      const double2* b1 = reinterpret_cast<const double2*>(bs + (kk + 1) * LB);
      // k then k + 1 over all columns: an accumulator's two updates are
      // R * LB FMAs apart (no back-to-back dependent DFMAs)
#pragma unroll
      for (int c2 = 0; c2 < LB / 2; ++c2) {
        const double2 x0 = b0[c2];
#pragma unroll
        for (int r = 0; r < R; ++r) {
          acc[r][2 * c2] = fma(a0[r], x0.x, acc[r][2 * c2]);
          acc[r][2 * c2 + 1] = fma(a0[r], x0.y, acc[r][2 * c2 + 1]);
        }
      }
#pragma unroll
      for (int c2 = 0; c2 < LB / 2; ++c2) {
        const double2 x1 = b1[c2];
#pragma unroll
        for (int r = 0; r < R; ++r) {
          acc[r][2 * c2] = fma(a1[r], x1.x, acc[r][2 * c2]);
          acc[r][2 * c2 + 1] = fma(a1[r], x1.y, acc[r][2 * c2 + 1]);
        }
      }
    }
  }
  cp_async_wait<0>();
  __syncthreads();
  // groups 1.. park their sums in the (now idle) ring; group 0 adds them in order
  double* red = sm;
  if (g > 0) {
#pragma unroll
    for (int r = 0; r < R; ++r)
#pragma unroll
      for (int c = 0; c < LB; ++c)
        red[(((g - 1) * R + r) * LB + c) * RT + ri] = acc[r][c];
  }
  __syncthreads();
  if (g > 0) return;
#pragma unroll 1
  for (int gg = 1; gg < L::G; ++gg)
#pragma unroll
    for (int r = 0; r < R; ++r)
#pragma unroll
      for (int c = 0; c < LB; ++c) acc[r][c] += red[(((gg - 1) * R + r) * LB + c) * RT + ri];
  double* out = part ? part + (int64_t)blockIdx.y * M * l : C;
  const int64_t ld = part ? M : ldc;
#pragma unroll
  for (int r = 0; r < R; ++r) {
    const int64_t i = i0 + ri + RT * r;
    if (i >= M) continue;
#pragma unroll
    for (int c = 0; c < LB; ++c)
      if (c < l) out[i + (int64_t)c * ld] = acc[r][c];
  }
}

// ---------------------------------------------------------------------------
// DMMA variant (fp64 tensor core, mma.sync m8n8k4): same 128-row x 32-k A
// tiles through the same 4-stage cp.async ring, but each of the 8 warps owns
// 16 rows of op(A) (two m8 blocks) and every column block (LB8 / 8 n8 blocks)
// over the whole k range of the tile, so there is no k-group reduction; the
// fp64 tensor pipe issues one instruction per 256 FMAs (the SIMT kernel needs
// eight), which is what keeps it fed at 8 warps per SM (scripts/micro:
// 36.6 TF/s DMMA vs 33 TF/s DFMA at 8 warps).  Shared-memory pitches are
// padded so each fragment load is two wavefronts: KC rows 36 doubles, MC
// k-rows 132, the B slice LB8 + 4.
template <bool KC, int LB8>
struct DLayout {
  // 128 rows x 32 k tiles (32 KB of A): KC rows are 256-byte DRAM runs, MC
  // k-rows 1 KB runs.  (64 x 64 KC tiles -- 512-byte runs -- measured no
  // faster at config 5, and 12 % slower for the transposed column-major case.)
  static constexpr bool WIDE = false;
  static constexpr int ROWS = WIDE ? 64 : 128;
  static constexpr int KT = WIDE ? 64 : 32;
  static constexpr int MB = ROWS / 64;               // m8 blocks per warp
  static constexpr int NB = LB8 / 8;                 // n8 blocks
  static constexpr int LBP = LB8 + 4;                // B slice pitch (doubles)
  static constexpr int APITCH = KC ? KT + 4 : ROWS + 4;   // row (KC) / k-row (MC) pitch
  static constexpr int a_elems = KC ? ROWS * APITCH : KT * APITCH;
  static constexpr int b_elems = KT * LBP;
  static constexpr int stage_elems = a_elems + b_elems;
  static constexpr size_t smem = sizeof(double) * (size_t)stage_elems * kStages;
  static_assert(smem <= 227 * 1024, "shared-memory ring exceeds the opt-in limit");
};

// Bt (K x LBP, row-major, zero beyond l) <- B (K x l, column-major)
template <int LBP>
__global__ void pack_bp_kernel(const double* __restrict__ B, int64_t ldb, int64_t K, int l,
                               double* __restrict__ Bt) {
  for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < K * LBP;
       e += (int64_t)gridDim.x * blockDim.x) {
    const int c = (int)(e % LBP);
    const int64_t k = e / LBP;
    Bt[e] = c < l ? B[k + (int64_t)c * ldb] : 0.0;
  }
}

__device__ __forceinline__ void dmma884(double& c0, double& c1, double a, double b) {
  asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0, %1}, {%2}, {%3}, "
               "{%0, %1};"
               : "+d"(c0), "+d"(c1)
               : "d"(a), "d"(b));
}

template <bool KC, int LB8>
__global__ void __launch_bounds__(kThreads)
    skinny_dmma_kernel(const double* __restrict__ A, int64_t M, int64_t K, int64_t lda,
                       const double* __restrict__ Bt, int l, int64_t kchunk,
                       double* __restrict__ C, int64_t ldc, double* __restrict__ part) {
  using L = DLayout<KC, LB8>;
  constexpr int NB = L::NB, MB = L::MB, LBP = L::LBP, AP = L::APITCH;
  constexpr int ROWS = L::ROWS, KT = L::KT;
  extern __shared__ __align__(16) double sm[];
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int64_t i0 = (int64_t)blockIdx.x * ROWS;
  const int64_t kb = (int64_t)blockIdx.y * kchunk;
  const int64_t ke = min(K, kb + kchunk);
  const int nt = (int)((ke - kb + KT - 1) / KT);
  const uint32_t sbase = (uint32_t)__cvta_generic_to_shared(sm);

  // A-tile copy plan (16-byte pieces): every thread moves APT pieces of one
  // column of pieces, addresses a per-thread base plus a constant stride
  constexpr int APT = ROWS * KT / 2 / kThreads;
  constexpr int PPR = KC ? KT / 2 : ROWS / 2;    // pieces per tile row (KC) / k row (MC)
  constexpr int LPJ = kThreads / PPR;            // tile rows (KC) / k rows (MC) per j
  const int pc = tid % PPR, pl = tid / PPR;
  const double* abase;
  int64_t astride;
  uint32_t adst0, rowmask = 0;
  int mc_bytes = 0;
  if (KC) {
    abase = A + (i0 + pl) * lda + 2 * pc;
    astride = (int64_t)LPJ * lda;
    adst0 = (uint32_t)(pl * AP + 2 * pc) * 8u;
#pragma unroll
    for (int j = 0; j < APT; ++j)
      if (i0 + pl + LPJ * j < M) rowmask |= 1u << j;
  } else {
    const int64_t row = i0 + 2 * pc;
    mc_bytes = row < M ? (row + 1 < M ? 16 : 8) : 0;
    abase = A + row + (int64_t)pl * lda;
    astride = (int64_t)LPJ * lda;
    adst0 = (uint32_t)(pl * AP + 2 * pc) * 8u;
  }
  auto issue = [&](int t) {
    const int slot = t % kStages;
    const int64_t k0 = kb + (int64_t)t * KT;
    const uint32_t sa = sbase + (uint32_t)(slot * L::stage_elems) * 8u;
    if (KC) {
      const int64_t kp = k0 + 2 * pc;
      const int kbytes = kp < ke ? (kp + 1 < ke ? 16 : 8) : 0;
      const double* src = abase + k0;
#pragma unroll
      for (int j = 0; j < APT; ++j) {
        const int bytes = ((rowmask >> j) & 1u) ? kbytes : 0;
        cp_async16(sa + adst0 + (uint32_t)(j * LPJ * AP) * 8u, bytes ? src + j * astride : A,
                   bytes);
      }
    } else {
      const double* src = abase + k0 * lda;
#pragma unroll
      for (int j = 0; j < APT; ++j) {
        const int bytes = (k0 + pl + LPJ * j < ke) ? mc_bytes : 0;
        cp_async16(sa + adst0 + (uint32_t)(j * LPJ * AP) * 8u, bytes ? src + j * astride : A,
                   bytes);
      }
    }
    const uint32_t sb = sa + (uint32_t)L::a_elems * 8u;
    for (int p = tid; p < KT * LBP / 2; p += kThreads) {
      const int64_t k = k0 + p / (LBP / 2);
      const int bytes = k < ke ? 16 : 0;
      cp_async16(sb + (uint32_t)(2 * p) * 8u, bytes ? Bt + k0 * LBP + 2 * p : Bt, bytes);
    }
  };

  double acc[MB][NB][2];
#pragma unroll
  for (int u = 0; u < MB; ++u)
#pragma unroll
    for (int v = 0; v < NB; ++v) acc[u][v][0] = acc[u][v][1] = 0.0;
#pragma unroll
  for (int s = 0; s < kStages - 1; ++s) {
    if (s < nt) issue(s);
    cp_async_commit();
  }
  const int fr = lane >> 2, fk = lane & 3;
  const int rbase = warp * (8 * MB) + fr;
  for (int t = 0; t < nt; ++t) {
    cp_async_wait<kStages - 2>();
    __syncthreads();
    if (t + kStages - 1 < nt) issue(t + kStages - 1);
    cp_async_commit();
    const double* st = sm + (t % kStages) * L::stage_elems;
    const double* bs = st + L::a_elems;
#pragma unroll 4
    for (int k4 = 0; k4 < KT; k4 += 4) {
      const int kk = k4 + fk;
      double a[MB], b[NB];
#pragma unroll
      for (int u = 0; u < MB; ++u)
        a[u] = KC ? st[(rbase + 8 * u) * AP + kk] : st[kk * AP + rbase + 8 * u];
#pragma unroll
      for (int v = 0; v < NB; ++v) b[v] = bs[kk * LBP + 8 * v + fr];
#pragma unroll
      for (int u = 0; u < MB; ++u)
#pragma unroll
        for (int v = 0; v < NB; ++v) dmma884(acc[u][v][0], acc[u][v][1], a[u], b[v]);
    }
  }
  cp_async_wait<0>();
  double* out = part ? part + (int64_t)blockIdx.y * M * l : C;
  const int64_t ld = part ? M : ldc;
#pragma unroll
  for (int u = 0; u < MB; ++u) {
    const int64_t i = i0 + warp * (8 * MB) + 8 * u + fr;
    if (i >= M) continue;
#pragma unroll
    for (int v = 0; v < NB; ++v)
#pragma unroll
      for (int e = 0; e < 2; ++e) {
        const int cc = 8 * v + 2 * fk + e;
        if (cc < l) out[i + (int64_t)cc * ld] = acc[u][v][e];
      }
  }
}

template <bool KC, int LB8>
void launch_dmma(Ctx& c, const double* A, int64_t M, int64_t K, int64_t lda, const double* B,
                 int64_t ldb, int l, double* C, int64_t ldc) {
  using L = DLayout<KC, LB8>;
  DBuf<double> Bt(c, (size_t)(K * L::LBP));
  pack_bp_kernel<L::LBP><<<grid_for(K * L::LBP), 256, 0, c.stream>>>(B, ldb, K, l, Bt.p);
  BRSVD_CHECK_LAUNCH();
  const int64_t blocks = ceil_div(M, (int64_t)L::ROWS);
  int64_t splits = std::max<int64_t>(1, ceil_div(16 * (int64_t)c.num_sms, blocks));
  splits = std::min<int64_t>(splits, std::max<int64_t>(1, K / 256));
  splits = std::min<int64_t>(splits, std::max<int64_t>(1, K / (8 * (int64_t)l)));
  int64_t kchunk = ceil_div(ceil_div(K, splits), (int64_t)L::KT) * L::KT;
  splits = std::max<int64_t>(1, ceil_div(K, kchunk));
  DBuf<double> part;
  if (splits > 1) part.alloc(c, (size_t)(splits * M * l));
  const size_t smem = L::smem;
  BRSVD_CUDA(cudaFuncSetAttribute(skinny_dmma_kernel<KC, LB8>,
                                  cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
  skinny_dmma_kernel<KC, LB8><<<dim3((unsigned)blocks, (unsigned)splits), kThreads, smem,
                                c.stream>>>(A, M, K, lda, Bt.p, l, kchunk, C, ldc, part.p);
  BRSVD_CHECK_LAUNCH();
  if (splits > 1) {
    splitk_reduce_kernel<double, double><<<grid_for(M * l), 256, 0, c.stream>>>(
        M, l, (int)splits, part.p, C, 1, ldc, 1.0, 0.0, nullptr, 0, 0);
    BRSVD_CHECK_LAUNCH();
  }
}

inline bool skinny_simt_forced() {
  const char* e = std::getenv("BRSVD_SKINNY_SIMT");
  return e && e[0] == '1';
}

template <bool KC, int LB>
void launch(Ctx& c, const double* A, int64_t M, int64_t K, int64_t lda, const double* B,
            int64_t ldb, int l, double* C, int64_t ldc) {
  if (LB >= 8 && !skinny_simt_forced()) {   // l > 4: the DMMA kernel
    constexpr int LB8 = LB < 8 ? 8 : ((LB + 7) / 8) * 8;
    launch_dmma<KC, LB8>(c, A, M, K, lda, B, ldb, l, C, ldc);
    return;
  }
  DBuf<double> Bt(c, (size_t)(K * LB));
  pack_b_kernel<LB><<<grid_for(K * LB), 256, 0, c.stream>>>(B, ldb, K, l, Bt.p);
  BRSVD_CHECK_LAUNCH();
  const int64_t blocks = ceil_div(M, (int64_t)kRows);
  // >= 16 waves of (row tile, k split) units, k splits of >= 256
  int64_t splits = std::max<int64_t>(1, ceil_div(16 * (int64_t)c.num_sms, blocks));
  splits = std::min<int64_t>(splits, std::max<int64_t>(1, K / 256));
  // the fp64 partials (splits * M * l) stay within ~1/8 of the A stream
  splits = std::min<int64_t>(splits, std::max<int64_t>(1, K / (8 * (int64_t)l)));
  int64_t kchunk = ceil_div(ceil_div(K, splits), (int64_t)kKT) * kKT;
  splits = std::max<int64_t>(1, ceil_div(K, kchunk));
  DBuf<double> part;
  if (splits > 1) part.alloc(c, (size_t)(splits * M * l));
  const size_t smem = Layout<KC, LB>::smem;
  BRSVD_CUDA(cudaFuncSetAttribute(skinny_kernel<KC, LB>,
                                  cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
  skinny_kernel<KC, LB><<<dim3((unsigned)blocks, (unsigned)splits), kThreads, smem,
                          c.stream>>>(A, M, K, lda, Bt.p, l, kchunk, C, ldc, part.p);
  BRSVD_CHECK_LAUNCH();
  if (splits > 1) {
    splitk_reduce_kernel<double, double><<<grid_for(M * l), 256, 0, c.stream>>>(
        M, l, (int)splits, part.p, C, 1, ldc, 1.0, 0.0, nullptr, 0, 0);
    BRSVD_CHECK_LAUNCH();
  }
}

template <int LB>
void launch_lb(Ctx& c, bool kcontig, const double* A, int64_t M, int64_t K, int64_t lda,
               const double* B, int64_t ldb, int l, double* C, int64_t ldc) {
  if (kcontig) launch<true, LB>(c, A, M, K, lda, B, ldb, l, C, ldc);
  else launch<false, LB>(c, A, M, K, lda, B, ldb, l, C, ldc);
}

}  // namespace sk

// C (M x l, column-major, ldc) = op(A) (M x K) B (K x l, column-major, ldb);
// op(A)(i, k) = A[i*lda + k] when kcontig, else A[i + k*lda].  Returns false
// (nothing launched) outside its range: l > 64, or A / lda not 16-byte
// aligned (the caller's generic tiled kernel takes those).
inline bool skinny_f64(Ctx& c, bool kcontig, const double* A, int64_t M, int64_t K,
                       int64_t lda, const double* B, int64_t ldb, int l, double* C,
                       int64_t ldc) {
  if (l < 1 || l > 64 || M < 1 || K < 1) return false;
  if ((reinterpret_cast<uintptr_t>(A) & 15) != 0 || (lda & 1) != 0) return false;
  if (l <= 2) sk::launch_lb<2>(c, kcontig, A, M, K, lda, B, ldb, l, C, ldc);
  else if (l <= 4) sk::launch_lb<4>(c, kcontig, A, M, K, lda, B, ldb, l, C, ldc);
  else if (l <= 8) sk::launch_lb<8>(c, kcontig, A, M, K, lda, B, ldb, l, C, ldc);
  else if (l <= 16) sk::launch_lb<16>(c, kcontig, A, M, K, lda, B, ldb, l, C, ldc);
  else if (l <= 20) sk::launch_lb<20>(c, kcontig, A, M, K, lda, B, ldb, l, C, ldc);
  else if (l <= 24) sk::launch_lb<24>(c, kcontig, A, M, K, lda, B, ldb, l, C, ldc);
  else if (l <= 32) sk::launch_lb<32>(c, kcontig, A, M, K, lda, B, ldb, l, C, ldc);
  else if (l <= 48) sk::launch_lb<48>(c, kcontig, A, M, K, lda, B, ldb, l, C, ldc);
  else sk::launch_lb<64>(c, kcontig, A, M, K, lda, B, ldb, l, C, ldc);
  return true;
}

}  // namespace brsvd
