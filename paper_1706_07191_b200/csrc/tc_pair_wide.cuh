// Single-chunk CTA-pair product for 160 < l <= 288: all l columns of a
// 256-row tile in one pair, so A is streamed and converted ONCE per product
// (tc3p_gemm_kernel splits l = 288 into two 144-column chunks, and its
// l-sweep shows the second chunk re-streaming and re-converting A costs most
// of the difference to the one-chunk case).
//
// TMEM per CTA: two accumulator regions R0 = columns [0, nc), R1 = [nc, 2nc)
// (nc = 96 or 144, the pair MMA N; each CTA's B half holds nc/2 rows of each
// region) and the three 64-column A staging slots -- 2 nc + 192 <= 512, so
// the regions are NOT double-buffered.  Their 128-k accumulation chunks are
// staggered by one 64-k stage (R0 chunks start at even stages, R1 chunks at
// odd ones), and in every stage the MMA issuer runs first the region that is
// in mid-chunk, then the one that starts a new chunk: the new chunk's region
// was drained while two stages' worth of the other region's MMAs kept the
// tensor pipe busy (its flush loads queue behind them), so the wait on its
// accfree barrier finds it free or nearly so.
//
// Warps (1024 threads, 64 registers): 0 A/B TMA producer, 1 MMA issuer (pair
// leader), 2 TMEM allocator, 3 idle, 4-7 converters (one per TMEM lane
// quadrant, the whole 64-k stage: fp32 A -> scaled fp16 hi / lo ->
// tcgen05.st), 8-31 flush warps (lane quadrant x sixth of the 2 nc columns:
// nc/3 fp32 running sums each, round-to-nearest accumulation of every 128-k
// chunk, then the epilogue).  Precision and scales exactly as tc3 / tc3p.
#pragma once
#include "tc_pair.cuh"

namespace brsvd {
namespace tcw {

using namespace tc;
using tcp::arrive_remote;
using tcp::cluster_sync;
using tcp::commit2;
using tcp::cta_rank;
using tcp::leader_addr;
using tcp::mma2_f16;

constexpr int kStages = 3;                  // = TMEM A slots
constexpr uint32_t kASlotW = 512 - kStages * 64;
constexpr uint32_t ASB = A_STAGE_BYTES_H16;
constexpr int kConvW = 4;
constexpr int kFlushW = 24;
constexpr int kThreadsW = 32 * (4 + kConvW + kFlushW);

__host__ __device__ constexpr uint32_t b_quarter_bytes(int nc) {
  return (uint32_t)(nc / 2) * 128u;   // one region's half, one of hi / lo
}
__host__ __device__ constexpr size_t smem_bytes(int nc) {
  return (size_t)kStages * (ASB + 4u * b_quarter_bytes(nc)) + 1024 + 1024;
}

// Region chunking: R0 chunks {0,1},{2,3},..; R1 chunks {0},{1,2},{3,4},..
__device__ __forceinline__ int chunk_of(int r, int kb) { return r == 0 ? kb >> 1 : (kb + 1) >> 1; }
__device__ __forceinline__ bool chunk_start(int r, int kb) {
  return r == 0 ? (kb & 1) == 0 : ((kb & 1) == 1 || kb == 0);
}
__device__ __forceinline__ bool chunk_end(int r, int kb, int nk) {
  return kb == nk - 1 || (r == 0 ? (kb & 1) == 1 : (kb & 1) == 0);
}
__device__ __forceinline__ int nchunks_of(int r, int nk) {
  return nk <= 0 ? 0 : (r == 0 ? ((nk - 1) >> 1) + 1 : (nk >> 1) + 1);
}

template <bool A_KMAJOR, int NC>
__global__ void __launch_bounds__(kThreadsW, 1)
    tc3w_gemm_kernel(const __grid_constant__ CUtensorMap mapA,
                     const __grid_constant__ CUtensorMap mapBhi,
                     const __grid_constant__ CUtensorMap mapBlo, const Params p) {
  constexpr int NF = NC / 3;                      // columns per flush warp
  constexpr uint32_t BQ = b_quarter_bytes(NC);
  constexpr uint32_t STAGE = ASB + 4 * BQ;
  static_assert(NF % 8 == 0, "flush warps drain 8-column groups");
  extern __shared__ uint8_t smem_dyn[];
  uint8_t* smem = (uint8_t*)(((uintptr_t)smem_dyn + 1023) & ~(uintptr_t)1023);
  uint64_t* full = reinterpret_cast<uint64_t*>(smem + kStages * STAGE);
  uint64_t* freeb = full + kStages;
  uint64_t* tfull = freeb + kStages;
  uint64_t* accready = tfull + kStages;        // [2], per region
  uint64_t* accfree = accready + 2;            // [2], per region
  uint32_t* tmem_holder = reinterpret_cast<uint32_t*>(accfree + 2);

  if (p.run_flag != nullptr && *p.run_flag == 0) return;   // uniform: the whole grid
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const uint32_t crank = cta_rank();
  const bool leader = crank == 0;
  const int unit = blockIdx.x >> 1;
  const int ks = unit % p.ksplit;
  const int tile = unit / p.ksplit;
  const int64_t m0 = (int64_t)tile * (2 * BM) + (int64_t)crank * BM;
  const int nk_all = (int)((p.K + BK_H16 - 1) / BK_H16);
  const int per = (nk_all + p.ksplit - 1) / p.ksplit;
  const int kb_begin = ks * per;
  const int nk = max(0, min(nk_all, kb_begin + per) - kb_begin);

  if (warp == 0 && lane == 0) {
    for (int s = 0; s < kStages; ++s) {
      mbar_init(&full[s], 1);
      mbar_init(&freeb[s], 1);
      mbar_init(&tfull[s], 2 * kConvW);
    }
    for (int r = 0; r < 2; ++r) {
      mbar_init(&accready[r], 1);
      mbar_init(&accfree[r], 2 * (kFlushW / 2));
    }
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    asm volatile("prefetch.tensormap [%0];" ::"l"(&mapA) : "memory");
    asm volatile("prefetch.tensormap [%0];" ::"l"(&mapBhi) : "memory");
    asm volatile("prefetch.tensormap [%0];" ::"l"(&mapBlo) : "memory");
  }
  if (warp == 2) {
    asm volatile("tcgen05.alloc.cta_group::2.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(
                     smem_u32(tmem_holder)),
                 "r"(kTmemCols)
                 : "memory");
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::2.sync.aligned;" ::: "memory");
  }
  tc_before_sync();
  cluster_sync();
  tc_after_sync();
  const uint32_t tmem = *tmem_holder;

  if (warp == 0) {
    if (lane == 0) {  // ---------------- TMA producer (both CTAs)
      const int br = (int)crank * (NC / 2);   // this CTA's half of each region's B rows
      for (int kb = 0; kb < nk; ++kb) {
        const int s = kb % kStages;
        const uint32_t ph = (kb / kStages) & 1;
        mbar_wait(&freeb[s], ph ^ 1);
        uint8_t* st = smem + (size_t)s * STAGE;
        const int k0 = (kb_begin + kb) * BK_H16;
        mbar_expect_tx(&full[s], STAGE);
        if (A_KMAJOR) {
          tma_load_2d(st, &mapA, &full[s], k0, (int)m0);
          tma_load_2d(st + BM * 128, &mapA, &full[s], k0 + 32, (int)m0);
        } else {
#pragma unroll
          for (int b = 0; b < 4; ++b)
            tma_load_2d(st + b * (32 * BK_H16 * 4), &mapA, &full[s], (int)m0 + 32 * b, k0);
        }
        // [hi R0][hi R1][lo R0][lo R1], each NC/2 rows of 128 B
        tma_load_2d(st + ASB, &mapBhi, &full[s], k0, br);
        tma_load_2d(st + ASB + BQ, &mapBhi, &full[s], k0, NC + br);
        tma_load_2d(st + ASB + 2 * BQ, &mapBlo, &full[s], k0, br);
        tma_load_2d(st + ASB + 3 * BQ, &mapBlo, &full[s], k0, NC + br);
      }
    }
  } else if (warp == 1) {
    if (lane == 0 && leader) {  // ---------------- MMA issuer (pair leader)
      const uint32_t idesc =
          (1u << 4) | ((uint32_t)(NC >> 3) << 17) | ((uint32_t)((2 * BM) >> 4) << 24);
      for (int kb = 0; kb < nk; ++kb) {
        const int s = kb % kStages;
        const uint32_t ph = (kb / kStages) & 1;
        mbar_wait(&tfull[s], ph);
        mbar_wait(&full[s], ph);
        tc_after_sync();
        const uint32_t sb = smem_u32(smem + (size_t)s * STAGE + ASB);
        const uint32_t a_hi = tmem + kASlotW + s * 64, a_lo = a_hi + 32;
        // the region in mid-chunk first, then the one starting a chunk
        const int r_first = (kb & 1) ? 0 : 1;
#pragma unroll
        for (int rr = 0; rr < 2; ++rr) {
          const int r = rr == 0 ? r_first : 1 - r_first;
          const bool start = chunk_start(r, kb);
          const int ci = chunk_of(r, kb);
          if (start && ci >= 1) {
            mbar_wait(&accfree[r], (ci - 1) & 1);
            tc_after_sync();
          }
          const uint32_t d = tmem + (uint32_t)(r * NC);
          const uint32_t bh = sb + r * BQ, bl = sb + (2 + r) * BQ;
#pragma unroll
          for (int kk = 0; kk < 4; ++kk) {
            const uint64_t dh = desc_kmajor_sw128(bh + kk * 32);
            const uint64_t dl = desc_kmajor_sw128(bl + kk * 32);
            const uint32_t acc = (start && kk == 0) ? 0u : 1u;
            mma2_f16(d, a_lo + kk * 8, dh, idesc, acc);
            mma2_f16(d, a_hi + kk * 8, dl, idesc, 1u);
            mma2_f16(d, a_hi + kk * 8, dh, idesc, 1u);
          }
          if (chunk_end(r, kb, nk)) commit2(&accready[r]);
        }
        commit2(&freeb[s]);
      }
    }
  } else if (warp >= 4 && warp < 4 + kConvW) {  // ---------------- converters
    const int wq = warp & 3;
    const int r = wq * 32 + lane;
    const uint32_t lane_base = (uint32_t)(wq * 32) << 16;
    const uint32_t tfull_l = leader_addr(tfull);
    const uint32_t smem_base = smem_u32(smem);
    const int64_t grow = m0 + r;
    const float rscale =
        (p.row_max != nullptr && grow < p.M) ? h16_scale(p.row_max[grow]) : 1.f;
    const bool want_max = p.amax_out != nullptr;
    float amax = 0.f;
    for (int kb = 0; kb < nk; ++kb) {
      const int s = kb % kStages;
      const uint32_t ph = (kb / kStages) & 1;
      mbar_wait(&full[s], ph);
      const uint32_t sa = smem_base + (uint32_t)s * STAGE;
#pragma unroll
      for (int qtr = 0; qtr < 4; ++qtr) {   // 16 k values per step (64 registers)
        float v[16];
        if (A_KMAJOR) {
          const uint32_t row = sa + (qtr >> 1) * (BM * 128) + r * 128;
#pragma unroll
          for (int jj = 0; jj < 4; ++jj) {
            const int j = 4 * (qtr & 1) + jj;
            const float4 x = lds128(row + ((j ^ (r & 7)) << 4));
            v[4 * jj + 0] = x.x;
            v[4 * jj + 1] = x.y;
            v[4 * jj + 2] = x.z;
            v[4 * jj + 3] = x.w;
          }
        } else {
          const uint32_t box = sa + wq * (32 * BK_H16 * 4) + lane * 4;
#pragma unroll
          for (int k = 0; k < 16; ++k) v[k] = lds32(box + (16 * qtr + k) * 128);
        }
        if (want_max) {
#pragma unroll
          for (int k = 0; k < 16; ++k) amax = fmaxf(amax, fabsf(v[k]));
        }
        uint32_t hi[8], lo[8];
#pragma unroll
        for (int i2 = 0; i2 < 8; ++i2) {
          const float x0 = v[2 * i2] * rscale, x1 = v[2 * i2 + 1] * rscale;
          hi[i2] = pack_h2(x0, x1);
          const float2 hf = unpack_h2(hi[i2]);
          lo[i2] = pack_h2(x0 - hf.x, x1 - hf.y);
        }
        tmem_st8(tmem + lane_base + kASlotW + s * 64 + 8 * qtr, hi);
        tmem_st8(tmem + lane_base + kASlotW + s * 64 + 32 + 8 * qtr, lo);
      }
      asm volatile("tcgen05.wait::st.sync.aligned;" ::: "memory");
      tc_before_sync();
      __syncwarp();
      if (lane == 0) arrive_remote(tfull_l + 8u * s);
    }
    if (want_max && grow < p.M) atomicMax(p.amax_out + grow, __float_as_uint(amax));
  } else if (warp >= 4 + kConvW) {  // ---------------- flushes + epilogue
    const int idx = warp - 4 - kConvW;          // 0..23
    const int wq = warp & 3;
    const int part = idx >> 2;                  // 0..5
    const int reg = part / 3;                   // accumulator region
    const int c0 = reg * NC + (part % 3) * NF;  // first output column
    const int r = wq * 32 + lane;
    const uint32_t lane_base = (uint32_t)(wq * 32) << 16;
    const uint32_t accfree_l = leader_addr(accfree);
    float run[NF];
#pragma unroll
    for (int j = 0; j < NF; ++j) run[j] = 0.f;
    const int nch = nchunks_of(reg, nk);
    for (int ci = 0; ci < nch; ++ci) {
      mbar_wait(&accready[reg], ci & 1);
      tc_after_sync();
#pragma unroll
      for (int j0 = 0; j0 < NF; j0 += 4) {   // 4-column loads: 64-register budget
        uint32_t acc[4];
        asm volatile("tcgen05.ld.sync.aligned.32x32b.x4.b32 {%0,%1,%2,%3}, [%4];"
                     : "=r"(acc[0]), "=r"(acc[1]), "=r"(acc[2]), "=r"(acc[3])
                     : "r"(tmem + lane_base + (uint32_t)(c0 + j0))
                     : "memory");
        asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
#pragma unroll
        for (int i2 = 0; i2 < 4; ++i2) run[j0 + i2] += __uint_as_float(acc[i2]);
      }
      tc_before_sync();
      __syncwarp();
      if (lane == 0) arrive_remote(accfree_l + 8u * reg);
    }
    const int64_t row = m0 + r;
    const float rscale =
        (p.row_max != nullptr && row < p.M) ? h16_scale(p.row_max[row]) : 1.f;
    const float rinv = 1.f / rscale;
    if (row < p.M) {
#pragma unroll
      for (int j = 0; j < NF; ++j) {
        const int col = c0 + j;
        if (col < p.n_out) {
          const float v = (float)((double)run[j] *
                                  ((double)rinv * (double)p.col_inv[col] * p.out_scale));
          if (p.part != nullptr) {   // > 2 K-splits: partials, summed in a fixed order
            p.part[(int64_t)ks * p.M * p.n_out + row + (int64_t)col * p.M] = v;
          } else {
            float* dst = p.C + row + (int64_t)col * p.ldc;
            if (p.ksplit > 1) atomicAdd(dst, v);   // two partial sums: order-free
            else *dst = v;
          }
        }
      }
    }
  }
  tc_before_sync();
  __syncthreads();
  cluster_sync();
  if (warp == 2) {
    tc_after_sync();
    asm volatile("tcgen05.dealloc.cta_group::2.sync.aligned.b32 %0, %1;" ::"r"(tmem),
                 "r"(kTmemCols)
                 : "memory");
  }
}

// C = sum of the K-split partials in split order (deterministic), fp32
__global__ void splitk_sum_f32_kernel(const float* __restrict__ part, int64_t M, int n,
                                      int splits, float* __restrict__ C, int64_t ldc,
                                      const int* __restrict__ run_flag) {
  if (run_flag != nullptr && *run_flag == 0) return;
  const int64_t total = M * n;
  if ((M & 3) == 0 && (ldc & 3) == 0 && ((reinterpret_cast<uintptr_t>(C) & 15) == 0)) {
    // float4 along the columns (M % 4 == 0: a quad never straddles two)
    const int64_t mq = M >> 2;
    const float4* p4 = reinterpret_cast<const float4*>(part);
    for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < (total >> 2);
         e += (int64_t)gridDim.x * blockDim.x) {
      float4 v = p4[e];
      for (int z = 1; z < splits; ++z) {
        const float4 w = p4[(int64_t)z * (total >> 2) + e];
        v.x += w.x;
        v.y += w.y;
        v.z += w.z;
        v.w += w.w;
      }
      const int64_t col = e / mq, r4 = e - col * mq;
      *reinterpret_cast<float4*>(C + col * ldc + 4 * r4) = v;
    }
    return;
  }
  for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < total;
       e += (int64_t)gridDim.x * blockDim.x) {
    float v = 0.f;
    for (int z = 0; z < splits; ++z) v += part[(int64_t)z * total + e];
    C[(e % M) + (e / M) * ldc] = v;
  }
}

// C (M x n) = 0 unless run_flag reads 0 (the two-split accumulator of a
// launch that may be skipped)
__global__ void zero_if_kernel(float* __restrict__ C, int64_t M, int n, int64_t ldc,
                               const int* __restrict__ run_flag) {
  if (run_flag != nullptr && *run_flag == 0) return;
  for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < M * n;
       e += (int64_t)gridDim.x * blockDim.x)
    C[(e % M) + (e / M) * ldc] = 0.f;
}

// The single-chunk pair kernel for 160 < l <= 288 unless BRSVD_TCW=0.
inline bool enabled() {
  const char* e = std::getenv("BRSVD_TCW");
  return !(e && e[0] == '0');
}
inline int nc_for(int l) { return l <= 192 ? 96 : 144; }
inline bool fits(int l) { return l > 160 && l <= 288; }

}  // namespace tcw

inline void tcw_gemm_launch(Ctx& c, const float* A, int64_t m, int64_t n, int64_t lda,
                            bool row_major, bool trans, const float* X, int64_t ldx, int l,
                            float* C, int64_t ldc, const float* opa_max, double out_scale,
                            unsigned* amax_out = nullptr, const int* run_flag = nullptr) {
  using namespace tc;
  const int64_t M = trans ? n : m, K = trans ? m : n;
  const bool kmajor = row_major != trans;
  const int nc = tcw::nc_for(l);
  const int npad = 2 * nc;
  const uint64_t inner = row_major ? (uint64_t)n : (uint64_t)m;
  const uint64_t outer = row_major ? (uint64_t)m : (uint64_t)n;
  const CUtensorMap mapA =
      kmajor ? make_map(A, inner, outer, (uint64_t)lda * 4, 32u, BM, CU_TENSOR_MAP_SWIZZLE_128B)
             : make_map(A, inner, outer, (uint64_t)lda * 4, 32, BK_H16,
                        CU_TENSOR_MAP_SWIZZLE_NONE);
  Params p;
  p.M = M;
  p.K = K;
  p.npad = npad;
  p.nchunks = 1;
  p.rows_c = nc;
  p.n_out = l;
  p.C = C;
  p.ldc = ldc;
  p.part = nullptr;
  p.keep_scaled = 0;
  p.out_scale = out_scale;
  p.b_terms = 3;
  p.amax_out = amax_out;
  p.run_flag = run_flag;
  DBuf<float> hi, lo, opmax, cinv;
  const int64_t kld = ceil_div(K, 8) * 8;
  if (opa_max == nullptr) {
    opmax.alloc(c, (size_t)M);
    if (trans) absmax_rows_cols(c, A, m, n, lda, row_major, nullptr, opmax.p);
    else absmax_rows_cols(c, A, m, n, lda, row_major, opmax.p, nullptr);
    opa_max = opmax.p;
  }
  cinv.alloc(c, (size_t)npad);
  hi.alloc(c, (size_t)npad * kld / 2 + 8);
  lo.alloc(c, (size_t)npad * kld / 2 + 8);
  tc_split16_col_kernel<<<(unsigned)npad, 512, 0, c.stream>>>(
      X, K, l, ldx, kld, reinterpret_cast<uint16_t*>(hi.p), reinterpret_cast<uint16_t*>(lo.p),
      cinv.p, 0, run_flag);
  BRSVD_CHECK_LAUNCH();
  const CUtensorMap mapBhi =
      make_map(hi.p, (uint64_t)kld, (uint64_t)npad, (uint64_t)kld * 2, BK_H16,
               (uint32_t)(nc / 2), CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_DATA_TYPE_FLOAT16);
  const CUtensorMap mapBlo =
      make_map(lo.p, (uint64_t)kld, (uint64_t)npad, (uint64_t)kld * 2, BK_H16,
               (uint32_t)(nc / 2), CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_DATA_TYPE_FLOAT16);
  p.row_max = opa_max;
  p.col_inv = cinv.p;
  // K splits so that the (tile x split) units fill their last wave of pairs
  // well: the fraction of busy pair-slots over the waves, best of 1..4 splits
  // (each split >= 4096 k).  Two partials combine by atomicAdd into a zeroed
  // C (order-free); more go through a workspace summed in a fixed order.
  const int64_t tiles = ceil_div(M, 2 * BM);
  const int slots = std::max(1, c.num_sms / 2);
  int best = 1;
  double best_eff = 0.0;
  for (int ks = 1; ks <= 4; ++ks) {
    if (ks > 1 && K / ks < 4096) break;
    const int64_t units = tiles * ks;
    const double eff = (double)units / (double)(ceil_div(units, (int64_t)slots) * slots);
    if (eff > best_eff + 0.02) {
      best_eff = eff;
      best = ks;
    }
  }
  if (const char* f = std::getenv("BRSVD_TCW_KSPLIT")) best = std::max(1, std::min(8, atoi(f)));
  p.ksplit = best;
  DBuf<float> part;
  if (p.ksplit > 2) {
    part.alloc(c, (size_t)p.ksplit * M * l);
    p.part = part.p;
  } else if (p.ksplit == 2) {
    if (run_flag != nullptr) {
      tcw::zero_if_kernel<<<grid_for(M * l), 256, 0, c.stream>>>(C, M, l, ldc, run_flag);
      BRSVD_CHECK_LAUNCH();
    } else {
      BRSVD_CUDA(cudaMemset2DAsync(C, (size_t)ldc * sizeof(float), 0,
                                   (size_t)M * sizeof(float), (size_t)l, c.stream));
    }
  }
  const size_t smem = tcw::smem_bytes(nc);
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3((unsigned)(2 * tiles * p.ksplit));
  cfg.blockDim = dim3(tcw::kThreadsW);
  cfg.dynamicSmemBytes = smem;
  cfg.stream = c.stream;
  cudaLaunchAttribute at[1];
  at[0].id = cudaLaunchAttributeClusterDimension;
  at[0].val.clusterDim.x = 2;
  at[0].val.clusterDim.y = 1;
  at[0].val.clusterDim.z = 1;
  cfg.attrs = at;
  cfg.numAttrs = 1;
#define BRSVD_TCW_LAUNCH(KM, NCV)                                                          \
  do {                                                                                     \
    auto kern = tcw::tc3w_gemm_kernel<KM, NCV>;                                             \
    BRSVD_CUDA(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize,     \
                                    (int)smem));                                           \
    BRSVD_CUDA(cudaLaunchKernelEx(&cfg, kern, mapA, mapBhi, mapBlo, p));                    \
  } while (0)
  if (kmajor) {
    if (nc == 96) BRSVD_TCW_LAUNCH(true, 96);
    else BRSVD_TCW_LAUNCH(true, 144);
  } else {
    if (nc == 96) BRSVD_TCW_LAUNCH(false, 96);
    else BRSVD_TCW_LAUNCH(false, 144);
  }
#undef BRSVD_TCW_LAUNCH
  ++g_brsvd_launches;
  if (p.part != nullptr) {
    tcw::splitk_sum_f32_kernel<<<grid_for(M * l), 256, 0, c.stream>>>(part.p, M, l, p.ksplit, C,
                                                                  ldc, run_flag);
    BRSVD_CHECK_LAUNCH();
  }
}

}  // namespace brsvd
