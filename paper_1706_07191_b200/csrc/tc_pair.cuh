// CTA-pair variant of the fp16-split A-streaming product (tc3_gemm_kernel,
// tc_gemm.cuh), for the products `a_block @ omega`, `a_block.T @ y`
// (rsvd.py:99-101) and `q.T @ a` (rsvd.py:140).
//
// What bounds tc3 is the bytes delivered from L2 into each SM (~10 TB/s over
// the chip, 18.3 GB per config-2 launch: A twice -- two 144-column chunks --
// and all of the chunk's B_hi / B_lo per 128-row tile).  Here two CTAs of a
// cluster (one TPC) compute a 256-row tile with tcgen05.mma.cta_group::2
// (M = 256): each CTA stages its own 128 rows of A, converted to fp16 (hi,
// lo) in its own TMEM (the .ts operand, as tc3), and loads only HALF of the
// chunk's B columns; the pair MMA reads both halves.  Per 64-k stage a CTA
// takes in 32 KB of A + 18 KB of B instead of 32 + 36 KB (-27 %), and the
// smaller stage lets a 4-deep shared-memory ring fit beside the 3 TMEM A
// slots (a converter reuses slot kb % 3 once the MMAs of stage kb - 3 have
// completed).  Everything else is tc3: power-of-two row / column scales,
// three kind::f16 MMAs per product term, the TMEM accumulator double-buffered
// and flushed every 128 k into round-to-nearest fp32 running sums held by the
// converter warps of each CTA (its own 128 rows).
//
// Barriers: full[s] (own A + own B half landed, TMA tx), freeb[s] and
// accready[b] (arrived on in both CTAs by the leader's multicast commit),
// tfull[s] and accfree[b] (the leader's, 16 + 16 converter warps arriving
// over the cluster).  Only the pair leader (rank 0) issues MMAs.
#pragma once
#include "tc_gemm.cuh"

namespace brsvd {
namespace tcp {

using namespace tc;

constexpr int kStages = 4;     // shared-memory ring (64 k per stage)
constexpr int kSlots = 3;      // TMEM A staging slots (64 columns each)
constexpr uint32_t kASlotP = 512 - kSlots * 64;
constexpr uint32_t ASB = A_STAGE_BYTES_H16;   // 32 KB of fp32 A per stage
constexpr int CHUNK = 128 / BK_H16;           // stages per accumulator flush
constexpr int kConvP = 8;                     // converter warps (quadrant x k half)
constexpr int kFlushP = 16;                   // flush warps (quadrant x column quarter)
constexpr int kThreadsP = 32 * (4 + kConvP + kFlushP);

__host__ __device__ constexpr uint32_t b_half_bytes(int nc) {
  return (uint32_t)(nc / 2) * 128u;   // nc/2 B rows of 64 fp16 (one of hi / lo)
}
__host__ __device__ constexpr size_t smem_bytes(int nc) {
  return (size_t)kStages * (ASB + 2u * b_half_bytes(nc)) + 512 + 1024;
}

__device__ __forceinline__ uint32_t cta_rank() {
  uint32_t r;
  asm volatile("mov.u32 %0, %%cluster_ctarank;" : "=r"(r));
  return r;
}
__device__ __forceinline__ void cluster_sync() {
  asm volatile("barrier.cluster.arrive.release.aligned;\n"
               "barrier.cluster.wait.acquire.aligned;" ::: "memory");
}
// shared::cluster address of this shared variable in the pair leader (rank 0)
__device__ __forceinline__ uint32_t leader_addr(const void* p) {
  uint32_t r;
  asm volatile("mapa.shared::cluster.u32 %0, %1, 0;" : "=r"(r) : "r"(smem_u32(p)));
  return r;
}
// Remote arrive without release semantics: what it orders -- this warp's
// TMEM stores / loads -- is complete already (tcgen05.wait::st / wait::ld and
// the tcgen05 fence precede it); a release.cluster arrive costs ~0.6 us.
__device__ __forceinline__ void arrive_remote(uint32_t cluster_addr) {
  asm volatile("mbarrier.arrive.relaxed.cluster.shared::cluster.b64 _, [%0];" ::"r"(
                   cluster_addr)
               : "memory");
}
__device__ __forceinline__ void mma2_f16(uint32_t d, uint32_t a, uint64_t bdesc,
                                         uint32_t idesc, uint32_t accumulate) {
  asm volatile(
      "{\n.reg .pred p;\nsetp.ne.b32 p, %4, 0;\n"
      "tcgen05.mma.cta_group::2.kind::f16 [%0], [%1], %2, %3, p;\n}" ::"r"(d),
      "r"(a), "l"(bdesc), "r"(idesc), "r"(accumulate)
      : "memory");
}
__device__ __forceinline__ void commit2(uint64_t* bar) {
  asm volatile(
      "tcgen05.commit.cta_group::2.mbarrier::arrive::one.shared::cluster.multicast::cluster.b64"
      " [%0], %1;" ::"r"(smem_u32(bar)),
      "h"((uint16_t)3)
      : "memory");
}

template <bool A_KMAJOR, int NCMAX>
__global__ void __launch_bounds__(kThreadsP, 1)
    tc3p_gemm_kernel(const __grid_constant__ CUtensorMap mapA,
                     const __grid_constant__ CUtensorMap mapBhi,
                     const __grid_constant__ CUtensorMap mapBlo, const Params p) {
  constexpr int NH = NCMAX / 4;
  extern __shared__ uint8_t smem_dyn[];
  uint8_t* smem = (uint8_t*)(((uintptr_t)smem_dyn + 1023) & ~(uintptr_t)1023);
  const int nc = p.rows_c;                     // columns of this pair's chunk
  const uint32_t bhb = b_half_bytes(nc);
  const uint32_t stage_bytes = ASB + 2 * bhb;
  uint64_t* full = reinterpret_cast<uint64_t*>(smem + kStages * stage_bytes);
  uint64_t* freeb = full + kStages;
  uint64_t* tfull = freeb + kStages;
  uint64_t* accready = tfull + kStages;        // [2]
  uint64_t* accfree = accready + 2;            // [2]
  uint32_t* tmem_holder = reinterpret_cast<uint32_t*>(accfree + 2);

  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const uint32_t crank = cta_rank();
  const bool leader = crank == 0;
  const int unit = blockIdx.x >> 1;
  const int ks = unit % p.ksplit;
  const int tile = unit / p.ksplit;
  const int64_t m0 = (int64_t)(tile / p.nchunks) * (2 * BM) + (int64_t)crank * BM;
  const int n0 = (tile % p.nchunks) * nc;
  const int nk_all = (int)((p.K + BK_H16 - 1) / BK_H16);
  const int per = (nk_all + p.ksplit - 1) / p.ksplit;
  const int kb_begin = ks * per;
  const int nk = max(0, min(nk_all, kb_begin + per) - kb_begin);
  const int nchunk = (nk + CHUNK - 1) / CHUNK;
  const bool two = p.b_terms == 2;   // sketch operand rounded to fp16: no B_lo term

  if (warp == 0 && lane == 0) {
    for (int s = 0; s < kStages; ++s) {
      mbar_init(&full[s], 1);
      mbar_init(&freeb[s], 1);
      mbar_init(&tfull[s], 2 * kConvP);    // the converter warps of both CTAs
    }
    for (int b = 0; b < 2; ++b) {
      mbar_init(&accready[b], 1);
      mbar_init(&accfree[b], 2 * kFlushP);
    }
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    asm volatile("prefetch.tensormap [%0];" ::"l"(&mapA) : "memory");
    asm volatile("prefetch.tensormap [%0];" ::"l"(&mapBhi) : "memory");
    asm volatile("prefetch.tensormap [%0];" ::"l"(&mapBlo) : "memory");
  }
  if (warp == 2) {   // the same warp of both CTAs allocates the pair's TMEM
    asm volatile("tcgen05.alloc.cta_group::2.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(
                     smem_u32(tmem_holder)),
                 "r"(kTmemCols)
                 : "memory");
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::2.sync.aligned;" ::: "memory");
  }
  tc_before_sync();
  cluster_sync();   // both CTAs' barriers exist before any remote arrival
  tc_after_sync();
  const uint32_t tmem = *tmem_holder;

  if (warp == 0) {
    if (lane == 0) {  // ---------------- TMA producer (both CTAs)
      const int br = n0 + (int)crank * (nc / 2);   // this CTA's half of the chunk's B rows
      for (int kb = 0; kb < nk; ++kb) {
        const int s = kb % kStages;
        const uint32_t ph = (kb / kStages) & 1;
        mbar_wait(&freeb[s], ph ^ 1);
        uint8_t* st = smem + (size_t)s * stage_bytes;
        const int k0 = (kb_begin + kb) * BK_H16;
        mbar_expect_tx(&full[s], two ? ASB + bhb : stage_bytes);
        if (A_KMAJOR) {
          tma_load_2d(st, &mapA, &full[s], k0, (int)m0);
          tma_load_2d(st + BM * 128, &mapA, &full[s], k0 + 32, (int)m0);
        } else {
#pragma unroll
          for (int b = 0; b < 4; ++b)
            tma_load_2d(st + b * (32 * BK_H16 * 4), &mapA, &full[s], (int)m0 + 32 * b, k0);
        }
        tma_load_2d(st + ASB, &mapBhi, &full[s], k0, br);
        if (!two) tma_load_2d(st + ASB + bhb, &mapBlo, &full[s], k0, br);
      }
    }
  } else if (warp == 1) {
    if (lane == 0 && leader) {  // ---------------- MMA issuer (pair leader)
      // c_format f32, a / b f16, K-major A and B, N = nc, M = 256
      const uint32_t idesc =
          (1u << 4) | ((uint32_t)(nc >> 3) << 17) | ((uint32_t)((2 * BM) >> 4) << 24);
      for (int kb = 0; kb < nk; ++kb) {
        const int s = kb % kStages;
        const uint32_t ph = (kb / kStages) & 1;
        const int slot = kb % kSlots;
        const int chunk = kb / CHUNK;
        const int buf = chunk & 1;
        const bool chunk_start = (kb % CHUNK) == 0;
        if (chunk_start && chunk >= 2) mbar_wait(&accfree[buf], ((chunk >> 1) - 1) & 1);
        mbar_wait(&tfull[s], ph);
        tc_after_sync();
        const uint32_t bh = smem_u32(smem + (size_t)s * stage_bytes + ASB);
        const uint32_t bl = bh + bhb;
        const uint32_t d = tmem + (uint32_t)(buf * nc);
        const uint32_t a_hi = tmem + kASlotP + slot * 64, a_lo = a_hi + 32;
#pragma unroll
        for (int kk = 0; kk < 4; ++kk) {
          const uint64_t dh = desc_kmajor_sw128(bh + kk * 32);
          const uint64_t dl = desc_kmajor_sw128(bl + kk * 32);
          const uint32_t acc = (chunk_start && kk == 0) ? 0u : 1u;
          mma2_f16(d, a_lo + kk * 8, dh, idesc, acc);
          if (!two) mma2_f16(d, a_hi + kk * 8, dl, idesc, 1u);
          mma2_f16(d, a_hi + kk * 8, dh, idesc, 1u);
        }
        commit2(&freeb[s]);
        if ((kb % CHUNK) == CHUNK - 1 || kb == nk - 1) commit2(&accready[buf]);
      }
    }
  } else if (warp >= 4 && warp < 4 + kConvP) {  // ---------------- converters
    // lane quadrant wq (TMEM lanes / this CTA's rows 32 wq ..) x k half of
    // every 64-k stage (two 16-k quarters, one tcgen05.st pair each)
    const int idx = warp - 4;
    const int wq = idx & 3;
    const int half = idx >> 2;
    const int r = wq * 32 + lane;
    const uint32_t lane_base = (uint32_t)(wq * 32) << 16;
    const uint32_t tfull_l = leader_addr(tfull);
    const uint32_t smem_base = smem_u32(smem);
    const int64_t grow = m0 + r;
    const float rscale =
        (p.row_max != nullptr && grow < p.M) ? h16_scale(p.row_max[grow]) : 1.f;
    for (int kb = 0; kb < nk; ++kb) {
      const int s = kb % kStages;
      const uint32_t ph = (kb / kStages) & 1;
      const int slot = kb % kSlots;
      mbar_wait(&full[s], ph);
      if (kb >= kSlots) {   // TMEM slot reuse: the MMAs of stage kb - 3 are done
        const int kp = kb - kSlots;
        mbar_wait(&freeb[kp % kStages], (kp / kStages) & 1);
      }
      const uint32_t sa = smem_base + (uint32_t)s * stage_bytes;
      // both 16-k quarters of this warp's k half: 16 adjacent TMEM columns of
      // hi and of lo, one 16-column store each
      uint32_t hi[16], lo[16];
#pragma unroll
      for (int sub = 0; sub < 2; ++sub) {
        const int qtr = 2 * half + sub;     // k values 16 qtr .. + 15
        float v[16];
        if (A_KMAJOR) {
          // two boxes of 128-byte rows (k 0-31, 32-63); TMA 128B swizzle puts
          // 16B chunk j of row r at j^(r&7)
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
#pragma unroll
        for (int i2 = 0; i2 < 8; ++i2) {
          const float x0 = v[2 * i2] * rscale, x1 = v[2 * i2 + 1] * rscale;
          hi[8 * sub + i2] = pack_h2(x0, x1);
          const float2 hf = unpack_h2(hi[8 * sub + i2]);
          lo[8 * sub + i2] = pack_h2(x0 - hf.x, x1 - hf.y);
        }
      }
      tmem_st16(tmem + lane_base + kASlotP + slot * 64 + 16 * half, hi);
      tmem_st16(tmem + lane_base + kASlotP + slot * 64 + 32 + 16 * half, lo);
      asm volatile("tcgen05.wait::st.sync.aligned;" ::: "memory");
      tc_before_sync();
      __syncwarp();
      if (lane == 0) arrive_remote(tfull_l + 8u * s);
    }
  } else if (warp >= 4 + kConvP) {  // ---------------- accumulator flushes + epilogue
    // dedicated warps: the TMEM loads of a flush queue behind the MMAs in the
    // tensor pipe (~1 us), so they must not sit on the converters' path.
    // Lane quadrant wq x column quarter qtr of the accumulator.
    const int idx = warp - 4 - kConvP;
    const int wq = idx & 3;
    const int qtr = idx >> 2;
    const int r = wq * 32 + lane;
    const uint32_t lane_base = (uint32_t)(wq * 32) << 16;
    const int hc = nc >> 2;
    const int c0 = qtr * hc;
    const uint32_t accfree_l = leader_addr(accfree);
    float run[NH];
#pragma unroll
    for (int j = 0; j < NH; ++j) run[j] = 0.f;
    for (int chunk = 0; chunk < nchunk; ++chunk) {
      const int buf = chunk & 1;
      mbar_wait(&accready[buf], (chunk >> 1) & 1);
      tc_after_sync();
#pragma unroll
      for (int j0 = 0; j0 < NH; j0 += 8) {
        if (j0 < hc) {
          uint32_t acc[8];
          tmem_ld8(tmem + lane_base + (uint32_t)(buf * nc + c0 + j0), acc);
          asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
#pragma unroll
          for (int i2 = 0; i2 < 8; ++i2) run[j0 + i2] += __uint_as_float(acc[i2]);
        }
      }
      tc_before_sync();
      __syncwarp();
      if (lane == 0) arrive_remote(accfree_l + 8u * buf);
    }
    const int64_t row = m0 + r;
    const float rscale =
        (p.row_max != nullptr && row < p.M) ? h16_scale(p.row_max[row]) : 1.f;
    if (!p.keep_scaled) {
      const float rinv = 1.f / rscale;
#pragma unroll
      for (int j = 0; j < NH; ++j) {
        const int col = n0 + c0 + j;
        if (j < hc && col < p.n_out)
          run[j] = (float)((double)run[j] *
                           ((double)rinv * (double)p.col_inv[col] * p.out_scale));
      }
    }
    if (row < p.M) {
#pragma unroll
      for (int j = 0; j < NH; ++j) {
        const int col = n0 + c0 + j;
        if (j < hc && col < p.n_out) {
          if (p.part != nullptr) {
            p.part[(int64_t)ks * p.M * p.n_out + row + (int64_t)col * p.M] = run[j];
          } else {
            float* dst = p.C + row + (int64_t)col * p.ldc;
            if (p.ksplit > 1) atomicAdd(dst, run[j]);   // two partial sums: order-free
            else *dst = run[j];
          }
        }
      }
    }
  }
  tc_before_sync();
  __syncthreads();
  cluster_sync();   // no CTA releases its TMEM while its peer may still signal it
  if (warp == 2) {
    tc_after_sync();
    asm volatile("tcgen05.dealloc.cta_group::2.sync.aligned.b32 %0, %1;" ::"r"(tmem),
                 "r"(kTmemCols)
                 : "memory");
  }
}

// l within the pair kernel's envelope (the same column chunks as tc3, each
// split in two 8-row-aligned halves)
inline bool tcp_fits(int l) {
  const Geometry g = geometry(l);
  return l >= 1 && g.npad <= NPAD_MAX && g.rows_c % 16 == 0 && g.rows_c <= 160;
}

// The pair kernel unless BRSVD_TCP=0.
inline bool enabled() {
  const char* e = std::getenv("BRSVD_TCP");
  return !(e && e[0] == '0');
}

}  // namespace tcp

// C (M x l, column-major, ldc) = opA * X on CTA pairs (fp16 split); the same
// operands, scales and output contract as tc_gemm_launch<float> without
// split-K workspaces or scaled outputs.  opa_max: max |opA| per row (else
// computed here).
inline void tcp_gemm_launch(Ctx& c, const float* A, int64_t m, int64_t n, int64_t lda,
                            bool row_major, bool trans, const float* X, int64_t ldx, int l,
                            float* C, int64_t ldc, const float* opa_max, double out_scale) {
  using namespace tc;
  const int64_t M = trans ? n : m, K = trans ? m : n;
  const bool kmajor = row_major != trans;
  const Geometry g = geometry(l);
  const uint64_t inner = row_major ? (uint64_t)n : (uint64_t)m;
  const uint64_t outer = row_major ? (uint64_t)m : (uint64_t)n;
  const CUtensorMap mapA =
      kmajor ? make_map(A, inner, outer, (uint64_t)lda * 4, 32u, BM, CU_TENSOR_MAP_SWIZZLE_128B)
             : make_map(A, inner, outer, (uint64_t)lda * 4, 32, BK_H16,
                        CU_TENSOR_MAP_SWIZZLE_NONE);
  Params p;
  p.M = M;
  p.K = K;
  p.npad = g.npad;
  p.nchunks = g.nchunks;
  p.rows_c = g.rows_c;
  p.n_out = l;
  p.C = C;
  p.ldc = ldc;
  p.part = nullptr;
  p.keep_scaled = 0;
  p.out_scale = out_scale;
  p.b_terms = c.b_hi_only ? 2 : 3;
  DBuf<float> hi, lo, opmax, cinv;
  const int64_t kld = ceil_div(K, 8) * 8;
  if (opa_max == nullptr) {
    opmax.alloc(c, (size_t)M);
    if (trans) absmax_rows_cols(c, A, m, n, lda, row_major, nullptr, opmax.p);
    else absmax_rows_cols(c, A, m, n, lda, row_major, opmax.p, nullptr);
    opa_max = opmax.p;
  }
  cinv.alloc(c, (size_t)g.npad);
  hi.alloc(c, (size_t)g.npad * kld / 2 + 8);
  lo.alloc(c, (size_t)g.npad * kld / 2 + 8);
  tc_split16_col_kernel<<<(unsigned)g.npad, 512, 0, c.stream>>>(
      X, K, l, ldx, kld, reinterpret_cast<uint16_t*>(hi.p), reinterpret_cast<uint16_t*>(lo.p),
      cinv.p);
  BRSVD_CHECK_LAUNCH();
  // each CTA of a pair loads half of the chunk's B rows
  const CUtensorMap mapBhi =
      make_map(hi.p, (uint64_t)kld, (uint64_t)g.npad, (uint64_t)kld * 2, BK_H16,
               (uint32_t)(g.rows_c / 2), CU_TENSOR_MAP_SWIZZLE_128B,
               CU_TENSOR_MAP_DATA_TYPE_FLOAT16);
  const CUtensorMap mapBlo =
      make_map(lo.p, (uint64_t)kld, (uint64_t)g.npad, (uint64_t)kld * 2, BK_H16,
               (uint32_t)(g.rows_c / 2), CU_TENSOR_MAP_SWIZZLE_128B,
               CU_TENSOR_MAP_DATA_TYPE_FLOAT16);
  p.row_max = opa_max;
  p.col_inv = cinv.p;
  // two K-halves per tile when the pair tiles leave the last wave badly
  // filled (partials combined by atomicAdd into a zeroed C: order-free for two)
  const int64_t tiles = ceil_div(M, 2 * BM) * g.nchunks;
  const double waves = (double)tiles / (c.num_sms / 2);
  p.ksplit = (K >= 8192 && waves > 1.0 && waves < 8.0 && waves - std::floor(waves) > 0.0 &&
              waves - std::floor(waves) < 0.75)
                 ? 2
                 : 1;
  if (p.ksplit > 1)
    BRSVD_CUDA(cudaMemset2DAsync(C, (size_t)ldc * sizeof(float), 0, (size_t)M * sizeof(float),
                                 (size_t)l, c.stream));
  const size_t smem = tcp::smem_bytes(g.rows_c);
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3((unsigned)(2 * tiles * p.ksplit));
  cfg.blockDim = dim3(tcp::kThreadsP);
  cfg.dynamicSmemBytes = smem;
  cfg.stream = c.stream;
  cudaLaunchAttribute at[1];
  at[0].id = cudaLaunchAttributeClusterDimension;
  at[0].val.clusterDim.x = 2;
  at[0].val.clusterDim.y = 1;
  at[0].val.clusterDim.z = 1;
  cfg.attrs = at;
  cfg.numAttrs = 1;
#define BRSVD_TCP_LAUNCH(KM, NCM)                                                          \
  do {                                                                                     \
    auto kern = tcp::tc3p_gemm_kernel<KM, NCM>;                                             \
    BRSVD_CUDA(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize,     \
                                    (int)smem));                                           \
    BRSVD_CUDA(cudaLaunchKernelEx(&cfg, kern, mapA, mapBhi, mapBlo, p));                    \
  } while (0)
#define BRSVD_TCP_NC(KM)                                          \
  do {                                                            \
    if (g.rows_c <= 32) BRSVD_TCP_LAUNCH(KM, 32);                 \
    else if (g.rows_c <= 64) BRSVD_TCP_LAUNCH(KM, 64);            \
    else if (g.rows_c <= 96) BRSVD_TCP_LAUNCH(KM, 96);            \
    else if (g.rows_c <= 128) BRSVD_TCP_LAUNCH(KM, 128);          \
    else BRSVD_TCP_LAUNCH(KM, 160);                               \
  } while (0)
  if (kmajor) BRSVD_TCP_NC(true);
  else BRSVD_TCP_NC(false);
#undef BRSVD_TCP_NC
#undef BRSVD_TCP_LAUNCH
  ++g_brsvd_launches;
}

}  // namespace brsvd
