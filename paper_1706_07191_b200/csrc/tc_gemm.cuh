// 5th-generation tensor-core (tcgen05) path for the A-streaming products of
// the fp32 pipeline (big_nn / big_tn):   C (M x N) = opA (M x K) * B (K x N)
// with opA the big matrix (A or A^T, K-major or MN-major in memory) and B the
// tall-skinny sketch (column-major, N = l <= 320).
//
// Precision: 3xTF32 split.  a = a_hi + a_lo, b = b_hi + b_lo with tf32 hi
// parts (cvt.rna) and fp32 remainders; C += a_lo b_hi + a_hi b_lo + a_hi b_hi
// in the fp32 TMEM accumulator -- fp32-level products, the sgemm the
// reference calls (rsvd.py:99-101, :140) to within accumulation order.
//
// Data flow per CTA (one 128-row tile of C, all N columns):
//   warp 0   TMA producer: A tile (128 x 16 fp32) + B_hi/B_lo tiles
//            (N x 16 each, K-major, 64B swizzle) into a 4-stage smem ring;
//   warps4-7 converters: A tile smem -> registers -> (hi, lo) -> tcgen05.st
//            into a TMEM staging slot (one TMEM lane per row of the tile);
//   warp 1   MMA issuer: tcgen05.mma.kind::tf32 with A from TMEM (.ts form)
//            and B from shared memory, N split in <=256 chunks, accumulator
//            N fp32 columns of TMEM; tcgen05.commit frees the stage;
//   warps4-7 epilogue: tcgen05.ld the accumulator, coalesced column-major
//            stores of C.
// Putting A in TMEM keeps the tensor core's shared-memory reads to the B
// operand only; B_hi/B_lo are split once per product (tc_split_kernel) and
// stay L2-resident across the M tiles.
#pragma once
#include <cuda.h>
#include <cuda_fp16.h>

#include <cstdlib>

#include "runtime.cuh"

namespace brsvd {
namespace tc {

constexpr int BM = 128;
constexpr int BK = 16;              // fp32 K elements per stage (64-byte rows)
constexpr int STAGES_TF32 = 6;   // smem ring depth (TMEM A slots: 6 x 32 columns)
constexpr int STAGES_H16 = 3;    // fp16 split: 3 x 64 TMEM columns (64 k per stage)
constexpr int NPAD_MAX = 320;   // l <= 320: two CTAs of <= 160 columns
constexpr int kThreads = 640;   // 4 role warps + 16 converter warps
constexpr uint32_t kTmemCols = 512;
constexpr uint32_t kASlot = 320;    // TMEM columns [320, 512): six A staging slots
constexpr uint32_t A_STAGE_BYTES = BM * BK * 4;
// fp16 split: 64 k values per stage (two 128-byte-swizzled fp32 A boxes,
// 128-byte fp16 B rows) -- a quarter of the stages, barrier round trips and
// TMA issues per byte of A of the 16-k tf32 ring
constexpr int BK_H16 = 64;
constexpr uint32_t A_STAGE_BYTES_H16 = BM * BK_H16 * 4;

struct Params {
  int64_t M, K;
  int npad, nchunks, rows_c, n_out;
  int ksplit;  // K-splits per tile (part == nullptr: 1 or 2, atomicAdd of two partials)
  float* C;
  int64_t ldc;
  float* part;  // split-K workspace: split s writes its partial to part + s * M * n_out
  // fp16 split (H16 kernels): row_max[M] = max |opA(row, :)| (power-of-two
  // row scale 2^(14 - ceil(log2 max)) applied before the split, undone in the
  // epilogue), col_inv[npad] = inverse power-of-two scales of the B columns
  const float* row_max;
  const float* col_inv;
  int keep_scaled;  // H16: leave the row/column scales in (caller unscales)
  double out_scale;  // H16: output multiplied by this power of two (range control)
  int b_terms;       // pair kernel: 3 (a_lo b_hi + a_hi b_lo + a_hi b_hi) or 2 (no b_lo)
  // single-chunk pair kernel: max |opA(row, :)| of the rows it converts
  // (float bits, atomicMax; the exact maxima behind a run on sampled scales),
  // and a device flag that skips the whole launch while it reads 0
  unsigned* amax_out = nullptr;
  const int* run_flag = nullptr;
};

__device__ __forceinline__ uint32_t smem_u32(const void* p) {
  return (uint32_t)__cvta_generic_to_shared(p);
}
__device__ __forceinline__ void mbar_init(uint64_t* bar, uint32_t count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count));
}
__device__ __forceinline__ void mbar_expect_tx(uint64_t* bar, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)),
               "r"(bytes)
               : "memory");
}
__device__ __forceinline__ void mbar_arrive(uint64_t* bar) {
  asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_u32(bar)) : "memory");
}
__device__ __forceinline__ void mbar_wait(uint64_t* bar, uint32_t parity) {
  asm volatile(
      "{\n"
      ".reg .pred P1;\n"
      "LAB_WAIT:\n"
      "mbarrier.try_wait.parity.shared::cta.b64 P1, [%0], %1;\n"
      "@P1 bra DONE;\n"
      "bra LAB_WAIT;\n"
      "DONE:\n"
      "}\n" ::"r"(smem_u32(bar)),
      "r"(parity)
      : "memory");
}
__device__ __forceinline__ void tma_load_2d(void* dst, const CUtensorMap* map, uint64_t* bar,
                                            int x, int y) {
  asm volatile(
      "cp.async.bulk.tensor.2d.shared::cluster.global.mbarrier::complete_tx::bytes"
      " [%0], [%1, {%3, %4}], [%2];" ::"r"(smem_u32(dst)),
      "l"(map), "r"(smem_u32(bar)), "r"(x), "r"(y)
      : "memory");
}
__device__ __forceinline__ void tc_before_sync() {
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
}
__device__ __forceinline__ void tc_after_sync() {
  asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
}
// K-major operand, 64-byte swizzle: 8-row groups 512 B apart (SBO), version 1.
__device__ __forceinline__ uint64_t desc_kmajor_sw64(uint32_t saddr) {
  uint64_t d = 0;
  d |= (uint64_t)((saddr >> 4) & 0x3FFF);
  d |= (uint64_t)1 << 16;            // LBO (unused for swizzled K-major)
  d |= (uint64_t)(512 >> 4) << 32;   // SBO
  d |= (uint64_t)1 << 46;            // descriptor version (sm100)
  d |= (uint64_t)4 << 61;            // SWIZZLE_64B
  return d;
}
// K-major operand, 32-byte swizzle (16 fp16 per row): 8-row groups 256 B apart.
__device__ __forceinline__ uint64_t desc_kmajor_sw32(uint32_t saddr) {
  uint64_t d = 0;
  d |= (uint64_t)((saddr >> 4) & 0x3FFF);
  d |= (uint64_t)1 << 16;            // LBO (unused for swizzled K-major)
  d |= (uint64_t)(256 >> 4) << 32;   // SBO
  d |= (uint64_t)1 << 46;            // descriptor version (sm100)
  d |= (uint64_t)6 << 61;            // SWIZZLE_32B
  return d;
}
// K-major operand, 128-byte swizzle (64 fp16 per row): 8-row groups 1024 B apart.
__device__ __forceinline__ uint64_t desc_kmajor_sw128(uint32_t saddr) {
  uint64_t d = 0;
  d |= (uint64_t)((saddr >> 4) & 0x3FFF);
  d |= (uint64_t)1 << 16;            // LBO (unused for swizzled K-major)
  d |= (uint64_t)(1024 >> 4) << 32;  // SBO
  d |= (uint64_t)1 << 46;            // descriptor version (sm100)
  d |= (uint64_t)2 << 61;            // SWIZZLE_128B
  return d;
}
__device__ __forceinline__ void mma_f16_ts(uint32_t d, uint32_t a, uint64_t bdesc,
                                           uint32_t idesc, uint32_t accumulate) {
  asm volatile(
      "{\n.reg .pred p;\nsetp.ne.b32 p, %4, 0;\n"
      "tcgen05.mma.cta_group::1.kind::f16 [%0], [%1], %2, %3, p;\n}" ::"r"(d),
      "r"(a), "l"(bdesc), "r"(idesc), "r"(accumulate)
      : "memory");
}
__device__ __forceinline__ void tmem_st4(uint32_t taddr, const uint32_t (&v)[4]) {
  asm volatile("tcgen05.st.sync.aligned.32x32b.x4.b32 [%0], {%1,%2,%3,%4};" ::"r"(taddr),
               "r"(v[0]), "r"(v[1]), "r"(v[2]), "r"(v[3])
               : "memory");
}
// Power-of-two scale mapping max |x| to <= 2^14 (fp16 split without overflow).
__host__ __device__ __forceinline__ float h16_scale(float mx) {
  if (!(mx > 0.f) || !(mx < 3.0e38f)) return 1.f;
  int e;
  frexpf(mx, &e);  // mx = f * 2^e, f in [0.5, 1)
  // capped so the scale and its inverse stay normal floats (rows whose max is
  // below 2^-112 keep fewer than 22 bits, as their inputs already do)
  return ldexpf(1.f, min(14 - e, 126));
}
__device__ __forceinline__ uint32_t pack_h2(float a, float b) {
  // a -> low half (lower k), b -> high half
  uint32_t r;
  asm("cvt.rn.f16x2.f32 %0, %1, %2;" : "=r"(r) : "f"(b), "f"(a));
  return r;
}
__device__ __forceinline__ float2 unpack_h2(uint32_t h) {
  float lo, hi;
  asm("{\n.reg .f16 l, h;\nmov.b32 {l, h}, %2;\ncvt.f32.f16 %0, l;\ncvt.f32.f16 %1, h;\n}"
      : "=f"(lo), "=f"(hi)
      : "r"(h));
  return make_float2(lo, hi);
}

__device__ __forceinline__ void mma_tf32_ts(uint32_t d, uint32_t a, uint64_t bdesc,
                                            uint32_t idesc, uint32_t accumulate) {
  asm volatile(
      "{\n.reg .pred p;\nsetp.ne.b32 p, %4, 0;\n"
      "tcgen05.mma.cta_group::1.kind::tf32 [%0], [%1], %2, %3, p;\n}" ::"r"(d),
      "r"(a), "l"(bdesc), "r"(idesc), "r"(accumulate)
      : "memory");
}
__device__ __forceinline__ void mma_commit(uint64_t* bar) {
  asm volatile(
      "tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(
          smem_u32(bar))
      : "memory");
}
__device__ __forceinline__ void tmem_st16(uint32_t taddr, const uint32_t (&v)[16]) {
  asm volatile(
      "tcgen05.st.sync.aligned.32x32b.x16.b32 [%0], {%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,"
      "%13,%14,%15,%16};" ::"r"(taddr),
      "r"(v[0]), "r"(v[1]), "r"(v[2]), "r"(v[3]), "r"(v[4]), "r"(v[5]), "r"(v[6]), "r"(v[7]),
      "r"(v[8]), "r"(v[9]), "r"(v[10]), "r"(v[11]), "r"(v[12]), "r"(v[13]), "r"(v[14]),
      "r"(v[15])
      : "memory");
}
__device__ __forceinline__ void tmem_ld16(uint32_t taddr, uint32_t (&v)[16]) {
  asm volatile(
      "tcgen05.ld.sync.aligned.32x32b.x16.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,"
      "%14,%15}, [%16];"
      : "=r"(v[0]), "=r"(v[1]), "=r"(v[2]), "=r"(v[3]), "=r"(v[4]), "=r"(v[5]), "=r"(v[6]),
        "=r"(v[7]), "=r"(v[8]), "=r"(v[9]), "=r"(v[10]), "=r"(v[11]), "=r"(v[12]), "=r"(v[13]),
        "=r"(v[14]), "=r"(v[15])
      : "r"(taddr)
      : "memory");
}
__device__ __forceinline__ uint32_t tf32_rna(float x) {
  uint32_t h;
  asm("cvt.rna.tf32.f32 %0, %1;" : "=r"(h) : "f"(x));
  return h;
}

// Tensor-core accumulation truncates (round-toward-zero) on every MMA add
// into TMEM, a bias of ~0.4 ulp per add that grows linearly with K
// (scripts/probe.py bias: -2.3e-6 at K=256, -1.7e-4 at K=16384).  The
// accumulator is therefore double-buffered and flushed every kChunkKB
// k-blocks (128 k values = 48 MMA adds, bias ~1e-6) into round-to-nearest
// fp32 running sums held in the converter warps' registers.
constexpr int kChunkKB = 8;

__device__ __forceinline__ void tmem_st8(uint32_t taddr, const uint32_t (&v)[8]) {
  asm volatile(
      "tcgen05.st.sync.aligned.32x32b.x8.b32 [%0], {%1,%2,%3,%4,%5,%6,%7,%8};" ::"r"(taddr),
      "r"(v[0]), "r"(v[1]), "r"(v[2]), "r"(v[3]), "r"(v[4]), "r"(v[5]), "r"(v[6]), "r"(v[7])
      : "memory");
}
__device__ __forceinline__ void tmem_ld8(uint32_t taddr, uint32_t (&v)[8]) {
  asm volatile("tcgen05.ld.sync.aligned.32x32b.x8.b32 {%0,%1,%2,%3,%4,%5,%6,%7}, [%8];"
               : "=r"(v[0]), "=r"(v[1]), "=r"(v[2]), "=r"(v[3]), "=r"(v[4]), "=r"(v[5]),
                 "=r"(v[6]), "=r"(v[7])
               : "r"(taddr)
               : "memory");
}
__device__ __forceinline__ float4 lds128(uint32_t addr) {
  float4 v;
  asm volatile("ld.shared.v4.f32 {%0,%1,%2,%3}, [%4];"
               : "=f"(v.x), "=f"(v.y), "=f"(v.z), "=f"(v.w)
               : "r"(addr));
  return v;
}
__device__ __forceinline__ float lds32(uint32_t addr) {
  float v;
  asm volatile("ld.shared.f32 %0, [%1];" : "=f"(v) : "r"(addr));
  return v;
}

// Warp roles (384 threads): warp 0 TMA producer, warp 1 MMA issuer, warp 2
// TMEM allocator, warps 4-11 converters/flushers.  Converter warp w owns TMEM
// lane quadrant (w % 4) -- the rows 32(w%4)..+31 of the tile -- and half
// h = (w - 4) / 4 of the work: k values [8h, 8h+8) of each A stage and the
// accumulator columns [h nc/2, (h+1) nc/2) of every flush.
// H16: the split uses fp16 (hi, lo) pairs and kind::f16 MMAs (twice the
// tf32 rate): with a power-of-two scale per row of opA and per column of B,
// hi + lo carries 22 significant bits like the tf32 pair, and the three
// products are exact in the fp32 accumulator.
template <bool A_KMAJOR, int NCMAX, bool H16>
__global__ void __launch_bounds__(kThreads, 1)
    tc3_gemm_kernel(const __grid_constant__ CUtensorMap mapA,
                    const __grid_constant__ CUtensorMap mapBhi,
                    const __grid_constant__ CUtensorMap mapBlo, const Params p) {
  constexpr int NH = NCMAX / 4;                          // running sums per thread
  // deeper ring for the fp16 split: the stage round trip (TMA -> convert ->
  // MMA -> commit) is latency-bound, so throughput scales with stages in flight
  constexpr int STAGES = H16 ? STAGES_H16 : STAGES_TF32;
  constexpr int BKK = H16 ? BK_H16 : BK;                  // k values per stage
  constexpr uint32_t ASB = H16 ? A_STAGE_BYTES_H16 : A_STAGE_BYTES;
  constexpr int CHUNK = 128 / BKK;                        // stages per accumulator chunk
  extern __shared__ uint8_t smem_dyn[];
  uint8_t* smem = (uint8_t*)(((uintptr_t)smem_dyn + 1023) & ~(uintptr_t)1023);
  const int nc = p.rows_c;                               // columns of this CTA
  const uint32_t b_bytes = (uint32_t)nc * BKK * (H16 ? 2 : 4);  // one of hi / lo
  const uint32_t stage_bytes = ASB + 2 * b_bytes;
  uint64_t* full = reinterpret_cast<uint64_t*>(smem + STAGES * stage_bytes);
  uint64_t* freeb = full + STAGES;
  uint64_t* tfull = freeb + STAGES;
  uint64_t* accready = tfull + STAGES;                   // [2]
  uint64_t* accfree = accready + 2;                      // [2]
  uint32_t* tmem_holder = reinterpret_cast<uint32_t*>(accfree + 2);

  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int tiles_n = p.nchunks;
  const int ks = blockIdx.x % p.ksplit;
  const int tile = blockIdx.x / p.ksplit;
  const int64_t m0 = (int64_t)(tile / tiles_n) * BM;
  const int n0 = (tile % tiles_n) * nc;
  const int nk_all = (int)((p.K + BKK - 1) / BKK);
  const int per = (nk_all + p.ksplit - 1) / p.ksplit;
  const int kb_begin = ks * per;
  const int nk = max(0, min(nk_all, kb_begin + per) - kb_begin);
  const int nchunk = (nk + CHUNK - 1) / CHUNK;

  if (warp == 0 && lane == 0) {
    for (int s = 0; s < STAGES; ++s) {
      mbar_init(&full[s], 1);
      mbar_init(&freeb[s], 1);
      mbar_init(&tfull[s], H16 ? 16 : 8);
    }
    for (int b = 0; b < 2; ++b) {
      mbar_init(&accready[b], 1);
      mbar_init(&accfree[b], 16);
    }
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    asm volatile("prefetch.tensormap [%0];" ::"l"(&mapA) : "memory");
    asm volatile("prefetch.tensormap [%0];" ::"l"(&mapBhi) : "memory");
    asm volatile("prefetch.tensormap [%0];" ::"l"(&mapBlo) : "memory");
  }
  if (warp == 2) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(
                     smem_u32(tmem_holder)),
                 "r"(kTmemCols)
                 : "memory");
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;" ::: "memory");
  }
  tc_before_sync();
  __syncthreads();
  tc_after_sync();
  const uint32_t tmem = *tmem_holder;

  if (warp == 0) {
    if (lane == 0) {  // ---------------- TMA producer
      for (int kb = 0; kb < nk; ++kb) {
        const int s = kb % STAGES;
        const uint32_t ph = (kb / STAGES) & 1;
        mbar_wait(&freeb[s], ph ^ 1);
        uint8_t* st = smem + (size_t)s * stage_bytes;
        const int k0 = (kb_begin + kb) * BKK;
        mbar_expect_tx(&full[s], stage_bytes);
        if (A_KMAJOR) {
          if constexpr (H16) {  // two 32-k boxes of 128-byte rows
            tma_load_2d(st, &mapA, &full[s], k0, (int)m0);
            tma_load_2d(st + BM * 128, &mapA, &full[s], k0 + 32, (int)m0);
          } else {
            tma_load_2d(st, &mapA, &full[s], k0, (int)m0);
          }
        } else {
#pragma unroll
          for (int b = 0; b < 4; ++b)
            tma_load_2d(st + b * (32 * BKK * 4), &mapA, &full[s], (int)m0 + 32 * b, k0);
        }
        tma_load_2d(st + ASB, &mapBhi, &full[s], k0, n0);
        tma_load_2d(st + ASB + b_bytes, &mapBlo, &full[s], k0, n0);
      }
    }
  } else if (warp == 1) {
    if (lane == 0) {  // ---------------- MMA issuer
      // c_format f32; a/b format tf32 (2) or f16 (0); K-major A and B
      const uint32_t fmt = H16 ? 0u : 2u;
      const uint32_t idesc = (1u << 4) | (fmt << 7) | (fmt << 10) |
                             ((uint32_t)(nc >> 3) << 17) | ((uint32_t)(BM >> 4) << 24);
      for (int kb = 0; kb < nk; ++kb) {
        const int s = kb % STAGES;
        const uint32_t ph = (kb / STAGES) & 1;
        const int chunk = kb / CHUNK;
        const int buf = chunk & 1;
        const bool chunk_start = (kb % CHUNK) == 0;
        if (chunk_start && chunk >= 2) mbar_wait(&accfree[buf], ((chunk >> 1) - 1) & 1);
        mbar_wait(&tfull[s], ph);
        mbar_wait(&full[s], ph);
        tc_after_sync();
        const uint32_t bh = smem_u32(smem + (size_t)s * stage_bytes + ASB);
        const uint32_t bl = bh + b_bytes;
        const uint32_t d = tmem + (uint32_t)(buf * nc);
        if constexpr (H16) {
          // four K=16 steps; A hi / lo in 32 TMEM columns each (fp16 pairs),
          // B rows of 128 bytes (64 fp16), 128-byte swizzle
          const uint32_t a_hi = tmem + kASlot + s * 64, a_lo = a_hi + 32;
#pragma unroll
          for (int kk = 0; kk < 4; ++kk) {
            const uint64_t dh = desc_kmajor_sw128(bh + kk * 32);
            const uint64_t dl = desc_kmajor_sw128(bl + kk * 32);
            const uint32_t acc = (chunk_start && kk == 0) ? 0u : 1u;
            mma_f16_ts(d, a_lo + kk * 8, dh, idesc, acc);
            mma_f16_ts(d, a_hi + kk * 8, dl, idesc, 1u);
            mma_f16_ts(d, a_hi + kk * 8, dh, idesc, 1u);
          }
        } else {
          const uint32_t a_hi = tmem + kASlot + s * 32, a_lo = a_hi + 16;
#pragma unroll
          for (int kk = 0; kk < BK / 8; ++kk) {
            const uint64_t dh = desc_kmajor_sw64(bh + kk * 32);
            const uint64_t dl = desc_kmajor_sw64(bl + kk * 32);
            const uint32_t acc = (chunk_start && kk == 0) ? 0u : 1u;
            mma_tf32_ts(d, a_lo + kk * 8, dh, idesc, acc);
            mma_tf32_ts(d, a_hi + kk * 8, dl, idesc, 1u);
            mma_tf32_ts(d, a_hi + kk * 8, dh, idesc, 1u);
          }
        }
        mma_commit(&freeb[s]);
        if ((kb % CHUNK) == CHUNK - 1 || kb == nk - 1) mma_commit(&accready[buf]);
      }
    }
  } else if (warp >= 4) {  // ---------------- converters + accumulator flushes
    // 16 warps: lane quadrant wq (TMEM lanes / tile rows 32 wq ..), k half of
    // each stage, stage parity par (even / odd k-blocks, so each warp's
    // split -> tcgen05.st -> wait chain has two stages of MMA time), and a
    // quarter of the accumulator columns for the flushes and the epilogue.
    // (H16: lane quadrant x k quarter of each 64-k stage, every stage.)
    const int idx = warp - 4;
    const int wq = idx & 3;
    const int half = (idx >> 2) & 1;
    const int par = H16 ? 0 : idx >> 3;
    const int qtr = idx >> 2;               // H16: k values 16 qtr .. + 15
    const int kstep = H16 ? 1 : 2;
    const int r = wq * 32 + lane;
    const uint32_t lane_base = (uint32_t)(wq * 32) << 16;
    const int hc = nc >> 2;                 // accumulator columns per warp
    const int c0 = (H16 ? qtr : 2 * par + half) * hc;
    float run[NH];
#pragma unroll
    for (int j = 0; j < NH; ++j) run[j] = 0.f;
    auto flush = [&](int chunk) {
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
          for (int i = 0; i < 8; ++i) run[j0 + i] += __uint_as_float(acc[i]);
        }
      }
      tc_before_sync();
      __syncwarp();
      if (lane == 0) mbar_arrive(&accfree[buf]);
    };
    const uint32_t smem_base = smem_u32(smem);
    float rscale = 1.f;
    if constexpr (H16) {
      const int64_t grow = m0 + r;
      rscale = (p.row_max != nullptr && grow < p.M) ? h16_scale(p.row_max[grow]) : 1.f;
    }
    int flushed = 0;
    for (int kb = par; kb < nk; kb += kstep) {
      const int s = kb % STAGES;
      const uint32_t ph = (kb / STAGES) & 1;
      mbar_wait(&full[s], ph);
      const uint32_t sa = smem_base + (uint32_t)s * stage_bytes;
      if constexpr (H16) {
        // 16 k values of row r: k = 16 qtr .. + 15
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
          // four (32 rows x 64 k) boxes, 32 consecutive rows per k
          const uint32_t box = sa + wq * (32 * BKK * 4) + lane * 4;
#pragma unroll
          for (int k = 0; k < 16; ++k) v[k] = lds32(box + (16 * qtr + k) * 128);
        }
        uint32_t hi[8], lo[8];
#pragma unroll
        for (int i = 0; i < 8; ++i) {
          const float x0 = v[2 * i] * rscale, x1 = v[2 * i + 1] * rscale;
          hi[i] = pack_h2(x0, x1);
          const float2 hf = unpack_h2(hi[i]);
          lo[i] = pack_h2(x0 - hf.x, x1 - hf.y);
        }
        tmem_st8(tmem + lane_base + kASlot + s * 64 + 8 * qtr, hi);
        tmem_st8(tmem + lane_base + kASlot + s * 64 + 32 + 8 * qtr, lo);
      } else {
        float v[8];
        if (A_KMAJOR) {
          // 64-byte rows; TMA 64B swizzle puts 16B chunk j of row r at j^((r>>1)&3)
          const uint32_t row = sa + r * 64;
#pragma unroll
          for (int jj = 0; jj < 2; ++jj) {
            const int j = 2 * half + jj;
            const float4 x = lds128(row + ((j ^ ((r >> 1) & 3)) << 4));
            v[4 * jj + 0] = x.x;
            v[4 * jj + 1] = x.y;
            v[4 * jj + 2] = x.z;
            v[4 * jj + 3] = x.w;
          }
        } else {
          // four (32 rows x 16 k) boxes, 32 consecutive rows per k
          const uint32_t box = sa + wq * (32 * BK * 4) + lane * 4;
#pragma unroll
          for (int k = 0; k < 8; ++k) v[k] = lds32(box + (8 * half + k) * 128);
        }
        uint32_t hi[8], lo[8];
#pragma unroll
        for (int i = 0; i < 8; ++i) {
          const uint32_t h = tf32_rna(v[i]);
          hi[i] = h;
          lo[i] = __float_as_uint(v[i] - __uint_as_float(h));
        }
        tmem_st8(tmem + lane_base + kASlot + s * 32 + 8 * half, hi);
        tmem_st8(tmem + lane_base + kASlot + s * 32 + 16 + 8 * half, lo);
      }
      asm volatile("tcgen05.wait::st.sync.aligned;" ::: "memory");
      tc_before_sync();
      __syncwarp();
      if (lane == 0) mbar_arrive(&tfull[s]);
      // earlier chunks' accumulators are complete once this chunk started
      while (flushed < kb / CHUNK - 1) flush(flushed++);
    }
    while (flushed < nchunk) flush(flushed++);
    const int64_t row = m0 + r;
    if (H16 && !p.keep_scaled) {
      const float rinv = 1.f / rscale;
#pragma unroll
      for (int j = 0; j < NH; ++j) {
        const int col = n0 + c0 + j;
        // power-of-two unscale in fp64: exact, one rounding, no spurious
        // over/underflow of the combined factor
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
  if (warp == 2) {
    tc_after_sync();
    asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem),
                 "r"(kTmemCols)
                 : "memory");
  }
}

// B (K x n_src, column-major, ld ldx) -> hi, lo ([npad][kld] row-major, zero
// padded): the tf32 split of the sketch, done once per product.
__global__ void tc_split_kernel(const float* __restrict__ X, int64_t K, int n_src,
                                int64_t ldx, int npad, int64_t kld,
                                float* __restrict__ hi, float* __restrict__ lo) {
  const int64_t total = (int64_t)npad * kld;
  for (int64_t idx = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; idx < total;
       idx += (int64_t)gridDim.x * blockDim.x) {
    const int64_t k = idx % kld, j = idx / kld;
    const float x = (j < n_src && k < K) ? X[k + j * ldx] : 0.f;
    const uint32_t h = tf32_rna(x);
    hi[idx] = __uint_as_float(h);
    lo[idx] = x - __uint_as_float(h);
  }
}

// One CTA per (padded) column: max |X[:, j]| by a block reduction, then the
// scaled fp16 (hi, lo) split of that column -- one pass, no atomics.
// qw > 0: column j is written to row perm(j) of the planes, the layout of the
// CTA-pair kernel (tc_stream.cuh): thirds of 2 qw columns, each split in two
// qw-column halves, one per CTA; CTA r's halves stacked in rows
// [r npad/2, (r+1) npad/2).
__global__ void __launch_bounds__(512)
    tc_split16_col_kernel(const float* __restrict__ X, int64_t K, int n_src, int64_t ldx,
                          int64_t kld, uint16_t* __restrict__ hi, uint16_t* __restrict__ lo,
                          float* __restrict__ col_inv, int qw = 0,
                          const int* __restrict__ run_flag = nullptr) {
  if (run_flag != nullptr && *run_flag == 0) return;   // the product is skipped too
  __shared__ unsigned red[16];
  const int j = blockIdx.x;
  const float* col = X + (int64_t)j * ldx;
  const bool real = j < n_src;
  // 16-byte loads / 8-byte stores when the column allows it (kld % 8 == 0)
  const bool vec = ((reinterpret_cast<uintptr_t>(col) & 15) == 0) && (K % 4 == 0);
  unsigned m = 0;
  if (real) {
    if (vec) {
      const float4* c4 = reinterpret_cast<const float4*>(col);
      for (int64_t k = threadIdx.x; k < K / 4; k += blockDim.x) {
        const float4 v = c4[k];
        m = max(m, max(max(__float_as_uint(fabsf(v.x)), __float_as_uint(fabsf(v.y))),
                       max(__float_as_uint(fabsf(v.z)), __float_as_uint(fabsf(v.w)))));
      }
    } else {
      for (int64_t k = threadIdx.x; k < K; k += blockDim.x)
        m = max(m, __float_as_uint(fabsf(col[k])));
    }
  }
  m = __reduce_max_sync(0xffffffffu, m);
  if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = m;
  __syncthreads();
  if (threadIdx.x == 0) {
    unsigned t = 0;
    for (int w = 0; w < (int)(blockDim.x >> 5); ++w) t = max(t, red[w]);
    red[0] = t;
  }
  __syncthreads();
  const float sc = real ? h16_scale(__uint_as_float(red[0])) : 1.f;
  if (threadIdx.x == 0) col_inv[j] = 1.f / sc;
  const int prow = qw > 0 ? ((j % (2 * qw)) / qw) * (int)(gridDim.x / 2) + (j / (2 * qw)) * qw +
                               j % qw
                         : j;
  uint16_t* h = hi + (int64_t)prow * kld;
  uint16_t* l = lo + (int64_t)prow * kld;
  if (vec) {
    const float4* c4 = reinterpret_cast<const float4*>(col);
    for (int64_t q = threadIdx.x; q < kld / 4; q += blockDim.x) {
      float4 v = make_float4(0.f, 0.f, 0.f, 0.f);
      if (real && 4 * q < K) v = c4[q];
      const float xs[4] = {v.x * sc, v.y * sc, v.z * sc, v.w * sc};
      uint16_t hh[4], ll[4];
#pragma unroll
      for (int e = 0; e < 4; ++e) {
        const __half hv = __float2half_rn(xs[e]);
        hh[e] = __half_as_ushort(hv);
        ll[e] = __half_as_ushort(__float2half_rn(xs[e] - __half2float(hv)));
      }
      reinterpret_cast<uint2*>(h)[q] =
          make_uint2(hh[0] | ((uint32_t)hh[1] << 16), hh[2] | ((uint32_t)hh[3] << 16));
      reinterpret_cast<uint2*>(l)[q] =
          make_uint2(ll[0] | ((uint32_t)ll[1] << 16), ll[2] | ((uint32_t)ll[3] << 16));
    }
  } else {
    for (int64_t k = threadIdx.x; k < kld; k += blockDim.x) {
      const float x = (real && k < K) ? col[k] * sc : 0.f;
      const __half hh = __float2half_rn(x);
      h[k] = __half_as_ushort(hh);
      l[k] = __half_as_ushort(__float2half_rn(x - __half2float(hh)));
    }
  }
}

// max |S[i, :]| (rmax) and max |S[:, j]| (cmax) of a column-major S (sr x sc,
// ld), accumulated with atomicMax on the 32-bit patterns of |x| (monotone for
// non-negative floats; NaN propagates).  CTA tile: 256 rows (one per thread,
// coalesced) x 128 columns.
__global__ void __launch_bounds__(256)
    absmax_rc_kernel(const float* __restrict__ S, int64_t sr, int64_t sc, int64_t ld,
                     unsigned* __restrict__ rmax, unsigned* __restrict__ cmax) {
  __shared__ unsigned wmax[8][128];
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int64_t row = (int64_t)blockIdx.x * 256 + threadIdx.x;
  const int64_t j0 = (int64_t)blockIdx.y * 128;
  const bool ok = row < sr;
  unsigned rm = 0;
#pragma unroll 8
  for (int jj = 0; jj < 128; ++jj) {
    const int64_t j = j0 + jj;
    const unsigned v = (ok && j < sc) ? __float_as_uint(fabsf(S[row + j * ld])) : 0u;
    rm = max(rm, v);
    const unsigned cm = __reduce_max_sync(0xffffffffu, v);
    if (lane == 0) wmax[warp][jj] = cm;
  }
  if (ok) atomicMax(&rmax[row], rm);
  __syncthreads();
  if (threadIdx.x < 128) {
    const int64_t j = j0 + threadIdx.x;
    unsigned m = 0;
#pragma unroll
    for (int w = 0; w < 8; ++w) m = max(m, wmax[w][threadIdx.x]);
    if (j < sc && m) atomicMax(&cmax[j], m);
  }
}

// Vectorised variant (sr % 4 == 0, ld % 4 == 0, 16-byte aligned S): each
// thread takes 4 consecutive rows as one float4 per column, so a warp covers
// 128 rows per 512-byte load and one warp reduction serves 128 rows.  CTA
// tile: 1024 rows x 64 columns.
__global__ void __launch_bounds__(256)
    absmax_rc4_kernel(const float* __restrict__ S, int64_t sr, int64_t sc, int64_t ld,
                      unsigned* __restrict__ rmax, unsigned* __restrict__ cmax) {
  __shared__ unsigned wmax[8][64];
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int64_t row = ((int64_t)blockIdx.x * 256 + threadIdx.x) * 4;
  const int64_t j0 = (int64_t)blockIdx.y * 64;
  const bool ok = row < sr;
  unsigned r0 = 0, r1 = 0, r2 = 0, r3 = 0;
  for (int jb = 0; jb < 64; jb += 16) {
    float4 v[16];  // all 16 loads in flight before the reductions
    if (ok && j0 + jb + 16 <= sc) {
      const float* p = S + row + (j0 + jb) * ld;
#pragma unroll
      for (int u = 0; u < 16; ++u) v[u] = __ldcs(reinterpret_cast<const float4*>(p + u * ld));
    } else {
#pragma unroll
      for (int u = 0; u < 16; ++u) {
        const int64_t j = j0 + jb + u;
        v[u] = (ok && j < sc) ? __ldcs(reinterpret_cast<const float4*>(S + row + j * ld))
                              : make_float4(0.f, 0.f, 0.f, 0.f);
      }
    }
#pragma unroll
    for (int u = 0; u < 16; ++u) {
      const unsigned a = __float_as_uint(fabsf(v[u].x)), b = __float_as_uint(fabsf(v[u].y)),
                     e = __float_as_uint(fabsf(v[u].z)), d = __float_as_uint(fabsf(v[u].w));
      r0 = max(r0, a);
      r1 = max(r1, b);
      r2 = max(r2, e);
      r3 = max(r3, d);
      const unsigned cm = __reduce_max_sync(0xffffffffu, max(max(a, b), max(e, d)));
      if (lane == 0) wmax[warp][jb + u] = cm;
    }
  }
  if (ok) {
    atomicMax(&rmax[row], r0);
    atomicMax(&rmax[row + 1], r1);
    atomicMax(&rmax[row + 2], r2);
    atomicMax(&rmax[row + 3], r3);
  }
  __syncthreads();
  if (threadIdx.x < 64) {
    const int64_t j = j0 + threadIdx.x;
    unsigned m = 0;
#pragma unroll
    for (int w = 0; w < 8; ++w) m = max(m, wmax[w][threadIdx.x]);
    if (j < sc && m) atomicMax(&cmax[j], m);
  }
}

typedef CUresult (*EncodeTiledFn)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*,
                                  const cuuint64_t*, const cuuint64_t*, const cuuint32_t*,
                                  const cuuint32_t*, CUtensorMapInterleave,
                                  CUtensorMapSwizzle, CUtensorMapL2promotion,
                                  CUtensorMapFloatOOBfill);

inline EncodeTiledFn encode_fn() {
  static EncodeTiledFn fn = nullptr;
  if (!fn) {
    void* ptr = nullptr;
    cudaDriverEntryPointQueryResult q;
    BRSVD_CUDA(cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &ptr, cudaEnableDefault, &q));
    BRSVD_REQUIRE(ptr != nullptr && q == cudaDriverEntryPointSuccess, kErrCuda,
                  "cuTensorMapEncodeTiled unavailable");
    fn = reinterpret_cast<EncodeTiledFn>(ptr);
  }
  return fn;
}

// 2-D fp32 tensor map: inner dimension `inner` (contiguous), `outer` rows of
// `row_bytes` stride; box (box_inner x box_outer).
inline CUtensorMap make_map(const void* base, uint64_t inner, uint64_t outer,
                            uint64_t row_bytes, uint32_t box_inner, uint32_t box_outer,
                            CUtensorMapSwizzle swz,
                            CUtensorMapDataType dt = CU_TENSOR_MAP_DATA_TYPE_FLOAT32) {
  CUtensorMap m;
  const cuuint64_t dims[2] = {inner, outer};
  const cuuint64_t strides[1] = {row_bytes};
  const cuuint32_t box[2] = {box_inner, box_outer};
  const cuuint32_t estr[2] = {1, 1};
  const CUresult r = encode_fn()(&m, dt, 2, const_cast<void*>(base),
                                 dims, strides, box, estr, CU_TENSOR_MAP_INTERLEAVE_NONE, swz,
                                 CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                                 CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  BRSVD_REQUIRE(r == CUDA_SUCCESS, kErrCuda, "cuTensorMapEncodeTiled failed");
  return m;
}

struct Geometry {
  int npad, nchunks, rows_c;
};

// Columns are split over CTAs so that two accumulator buffers (2 x rows_c)
// plus the A staging slots fit the 512 TMEM columns: rows_c <= 192.
inline Geometry geometry(int l) {
  Geometry g;
  g.nchunks = (int)ceil_div(l, 160);
  g.rows_c = (int)ceil_div(ceil_div(l, g.nchunks), 16) * 16;
  g.npad = g.rows_c * g.nchunks;
  return g;
}

inline size_t smem_bytes(int rows_c, bool h16 = false) {
  return h16 ? (size_t)STAGES_H16 * (A_STAGE_BYTES_H16 + 2u * (uint32_t)rows_c * BK_H16 * 2) +
                   512 + 1024
             : (size_t)STAGES_TF32 * (A_STAGE_BYTES + 2u * (uint32_t)rows_c * BK * 4) + 512 +
                   1024;
}

inline bool env_enabled() {
  const char* e = std::getenv("BRSVD_TC");
  return !(e && e[0] == '0');
}

// fp16-split products (2x the tf32 MMA rate) unless BRSVD_TC_H16=0.
inline bool h16_enabled() {
  const char* e = std::getenv("BRSVD_TC_H16");
  return !(e && e[0] == '0');
}

}  // namespace tc

template <typename T>
bool tc_gemm_supported(Ctx& c, const T* A, int64_t lda, int64_t m, int64_t n, int l) {
  if (sizeof(T) != 4 || !tc::env_enabled() || c.cc_major != 10) return false;
  // TMA: 16-byte aligned base and row stride
  if ((reinterpret_cast<uintptr_t>(A) & 15) != 0 || (lda * (int64_t)sizeof(T)) % 16 != 0)
    return false;
  const tc::Geometry g = tc::geometry(l);
  if (g.npad > tc::NPAD_MAX) return false;
  if (tc::smem_bytes(g.rows_c) > c.max_smem_optin) return false;
  return m >= 1 && n >= 1;
}

// Row and column maxima |A| of the big operand (one pass), as floats:
// amax_rows[m], amax_cols[n] (either may be NULL).  Used for the power-of-two
// scales of the fp16-split products; computed once per decomposition.
inline void absmax_rows_cols(Ctx& c, const float* A, int64_t m, int64_t n, int64_t lda,
                             bool row_major, float* amax_rows, float* amax_cols,
                             bool init = true) {
  const int64_t sr = row_major ? n : m, sc = row_major ? m : n;
  DBuf<unsigned> rbuf, cbuf;
  unsigned* S_r = reinterpret_cast<unsigned*>(row_major ? amax_cols : amax_rows);
  unsigned* S_c = reinterpret_cast<unsigned*>(row_major ? amax_rows : amax_cols);
  if (!S_r) {
    rbuf.alloc(c, (size_t)sr);
    S_r = rbuf.p;
    BRSVD_CUDA(cudaMemsetAsync(S_r, 0, sizeof(unsigned) * sr, c.stream));
  } else if (init) {
    BRSVD_CUDA(cudaMemsetAsync(S_r, 0, sizeof(unsigned) * sr, c.stream));
  }
  if (!S_c) {
    cbuf.alloc(c, (size_t)sc);
    S_c = cbuf.p;
    BRSVD_CUDA(cudaMemsetAsync(S_c, 0, sizeof(unsigned) * sc, c.stream));
  } else if (init) {
    BRSVD_CUDA(cudaMemsetAsync(S_c, 0, sizeof(unsigned) * sc, c.stream));
  }
  if (sr < 1 || sc < 1) return;
  if (sr % 4 == 0 && lda % 4 == 0 && (reinterpret_cast<uintptr_t>(A) & 15) == 0) {
    const dim3 grid((unsigned)ceil_div(sr, 1024), (unsigned)ceil_div(sc, 64));
    tc::absmax_rc4_kernel<<<grid, 256, 0, c.stream>>>(A, sr, sc, lda, S_r, S_c);
  } else {
    const dim3 grid((unsigned)ceil_div(sr, 256), (unsigned)ceil_div(sc, 128));
    tc::absmax_rc_kernel<<<grid, 256, 0, c.stream>>>(A, sr, sc, lda, S_r, S_c);
  }
  BRSVD_CHECK_LAUNCH();
}

namespace tc {
// Sampled maxima along the outer index: per outer j, max |S| over chunks of
// 128 contiguous entries every 4096 (1/32 of the line; one warp per line, a
// chunk is one coalesced 512-byte load, all chunks of the line in flight).
__global__ void amax_sample_outer_kernel(const float* __restrict__ S, int64_t sr, int64_t sc,
                                         int64_t ld, float* __restrict__ out) {
  constexpr int kChunks = 8;
  const int lane = threadIdx.x & 31;
  for (int64_t j = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5; j < sc;
       j += ((int64_t)gridDim.x * blockDim.x) >> 5) {
    const float* col = S + j * ld;
    const bool vec = ((reinterpret_cast<uintptr_t>(col) & 15) == 0);
    float mx = 0.f;
    for (int64_t c00 = 0; c00 < sr; c00 += (int64_t)kChunks * 4096) {
      float4 v[kChunks];
#pragma unroll
      for (int it = 0; it < kChunks; ++it) {
        const int64_t c0 = c00 + (int64_t)it * 4096 + 4 * lane;
        if (vec && c0 + 4 <= sr) {
          v[it] = __ldcs(reinterpret_cast<const float4*>(col + c0));
        } else {
          v[it].x = c0 < sr ? col[c0] : 0.f;
          v[it].y = c0 + 1 < sr ? col[c0 + 1] : 0.f;
          v[it].z = c0 + 2 < sr ? col[c0 + 2] : 0.f;
          v[it].w = c0 + 3 < sr ? col[c0 + 3] : 0.f;
        }
      }
#pragma unroll
      for (int it = 0; it < kChunks; ++it)
        mx = fmaxf(mx, fmaxf(fmaxf(fabsf(v[it].x), fabsf(v[it].y)),
                             fmaxf(fabsf(v[it].z), fabsf(v[it].w))));
    }
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) mx = fmaxf(mx, __shfl_xor_sync(0xffffffffu, mx, o));
    if (lane == 0) out[j] = mx;
  }
}
__global__ void scale_by_kernel(float* __restrict__ x, int64_t n, float f) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n;
       i += (int64_t)gridDim.x * blockDim.x)
    x[i] *= f;
}
// flag = 1 if some row's exact maximum, under the scale its sampled maximum
// gave, leaves [2^3, 65504): overflow of the fp16 high part, or fewer than
// the split's 22 bits above the fp16 subnormal floor
__global__ void lazy_scale_check_kernel(const float* __restrict__ guess,
                                        const float* __restrict__ exact, int64_t n,
                                        int* __restrict__ flag) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n;
       i += (int64_t)gridDim.x * blockDim.x) {
    const float x = exact[i];
    if (!(x > 0.f) || !(x < INFINITY)) continue;
    const float y = x * h16_scale(guess[i]);
    if (!(y >= 8.f && y < 65504.f)) *flag = 1;
  }
}
}  // namespace tc

// Sampled row / column maxima of |A| (about 1/16 of A read), times 2^7: the
// scales they give hold the true maxima in [2^3, 65504) unless a line's
// largest entry is over 2^9 x its sampled one (lazy_scale_check_kernel).
inline void amax_sampled(Ctx& c, const float* A, int64_t m, int64_t n, int64_t lda,
                         bool row_major, float* g_rows, float* g_cols) {
  const int64_t sr = row_major ? n : m, sc = row_major ? m : n;
  // contiguous index: every 32nd line read whole
  const int64_t sc32 = ceil_div(sc, 32);
  if (row_major)
    absmax_rows_cols(c, A, sc32, n, 32 * lda, true, nullptr, g_cols);
  else
    absmax_rows_cols(c, A, m, sc32, 32 * lda, false, g_rows, nullptr);
  float* outer = row_major ? g_rows : g_cols;
  tc::amax_sample_outer_kernel<<<(unsigned)std::min<int64_t>(ceil_div(sc, 8), 4096), 256, 0,
                                 c.stream>>>(A, sr, sc, lda, outer);
  BRSVD_CHECK_LAUNCH();
  tc::scale_by_kernel<<<grid_for(m), 256, 0, c.stream>>>(g_rows, m, 128.f);
  tc::scale_by_kernel<<<grid_for(n), 256, 0, c.stream>>>(g_cols, n, 128.f);
  BRSVD_CHECK_LAUNCH();
}

namespace tc {
// out[0..M) = 1 / (row scale of opA), out[M..M+l) = column inverse scales
__global__ void export_scales_kernel(const float* __restrict__ row_max, int64_t M,
                                     const float* __restrict__ col_inv, int l,
                                     float* __restrict__ out) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < M + l;
       i += (int64_t)gridDim.x * blockDim.x)
    out[i] = i < M ? 1.f / h16_scale(row_max[i]) : col_inv[i - M];
}
}  // namespace tc

template <typename T>
void tc_gemm_launch(Ctx& c, const T* A, int64_t m, int64_t n, int64_t lda, bool row_major,
                    bool trans, const T* X, int64_t ldx, int l, T* C, int64_t ldc,
                    int splits = 0, float* part = nullptr, const float* opa_max = nullptr,
                    float* scales_out = nullptr, double out_scale = 1.0);

template <>
inline void tc_gemm_launch<float>(Ctx& c, const float* A, int64_t m, int64_t n, int64_t lda,
                                  bool row_major, bool trans, const float* X, int64_t ldx,
                                  int l, float* C, int64_t ldc, int splits, float* part,
                                  const float* opa_max, float* scales_out,
                                  double out_scale) {
  using namespace tc;
  const int64_t M = trans ? n : m, K = trans ? m : n;
  const bool kmajor = row_major != trans;
  const Geometry g = geometry(l);
  const bool h16 = h16_enabled();
  // A as stored: row-major (m x n) has n contiguous; column-major has m contiguous.
  const uint64_t inner = row_major ? (uint64_t)n : (uint64_t)m;
  const uint64_t outer = row_major ? (uint64_t)m : (uint64_t)n;
  const bool h16m = h16_enabled();
  const uint32_t bka = h16m ? BK_H16 : BK;
  const CUtensorMap mapA =
      kmajor ? make_map(A, inner, outer, (uint64_t)lda * 4, h16m ? 32u : bka, BM,
                        h16m ? CU_TENSOR_MAP_SWIZZLE_128B : CU_TENSOR_MAP_SWIZZLE_64B)
             : make_map(A, inner, outer, (uint64_t)lda * 4, 32, bka, CU_TENSOR_MAP_SWIZZLE_NONE);
  Params p;
  p.M = M;
  p.K = K;
  p.npad = g.npad;
  p.nchunks = g.nchunks;
  p.rows_c = g.rows_c;
  p.n_out = l;
  p.C = C;
  p.ldc = ldc;
  p.part = part;
  p.row_max = nullptr;
  p.col_inv = nullptr;
  p.keep_scaled = 0;
  p.out_scale = out_scale;
  p.b_terms = 3;
  DBuf<float> hi, lo, opmax, cinv;
  CUtensorMap mapBhi, mapBlo;
  if (h16) {
    const int64_t kld = ceil_div(K, 8) * 8;
    if (opa_max == nullptr) {
      opmax.alloc(c, (size_t)M);
      if (trans)
        absmax_rows_cols(c, A, m, n, lda, row_major, nullptr, opmax.p);
      else
        absmax_rows_cols(c, A, m, n, lda, row_major, opmax.p, nullptr);
      opa_max = opmax.p;
    }
    cinv.alloc(c, (size_t)g.npad);
    hi.alloc(c, (size_t)g.npad * kld / 2 + 8);
    lo.alloc(c, (size_t)g.npad * kld / 2 + 8);
    tc_split16_col_kernel<<<(unsigned)g.npad, 512, 0, c.stream>>>(
        X, K, l, ldx, kld, reinterpret_cast<uint16_t*>(hi.p),
        reinterpret_cast<uint16_t*>(lo.p), cinv.p);
    BRSVD_CHECK_LAUNCH();
    mapBhi = make_map(hi.p, (uint64_t)kld, (uint64_t)g.npad, (uint64_t)kld * 2, BK_H16,
                      (uint32_t)g.rows_c, CU_TENSOR_MAP_SWIZZLE_128B,
                      CU_TENSOR_MAP_DATA_TYPE_FLOAT16);
    mapBlo = make_map(lo.p, (uint64_t)kld, (uint64_t)g.npad, (uint64_t)kld * 2, BK_H16,
                      (uint32_t)g.rows_c, CU_TENSOR_MAP_SWIZZLE_128B,
                      CU_TENSOR_MAP_DATA_TYPE_FLOAT16);
    p.row_max = opa_max;
    p.col_inv = cinv.p;
    if (scales_out != nullptr) {  // scaled output: export the inverse scales
      p.keep_scaled = 1;
      export_scales_kernel<<<grid_for(M + l), 256, 0, c.stream>>>(opa_max, M, cinv.p, l,
                                                                   scales_out);
      BRSVD_CHECK_LAUNCH();
    }
  } else {
    const int64_t kld = ceil_div(K, 4) * 4;
    hi.alloc(c, (size_t)g.npad * kld);
    lo.alloc(c, (size_t)g.npad * kld);
    tc_split_kernel<<<grid_for((int64_t)g.npad * kld), 256, 0, c.stream>>>(
        X, K, l, ldx, g.npad, kld, hi.p, lo.p);
    BRSVD_CHECK_LAUNCH();
    mapBhi = make_map(hi.p, (uint64_t)kld, (uint64_t)g.npad, (uint64_t)kld * 4, BK,
                      (uint32_t)g.rows_c, CU_TENSOR_MAP_SWIZZLE_64B);
    mapBlo = make_map(lo.p, (uint64_t)kld, (uint64_t)g.npad, (uint64_t)kld * 4, BK,
                      (uint32_t)g.rows_c, CU_TENSOR_MAP_SWIZZLE_64B);
  }
  // Two K-halves per tile when the tile count leaves the last wave of CTAs
  // (one per SM) badly filled: the two fp32 partial sums are combined with
  // atomicAdd into a zeroed C, which is order-independent for two terms.
  const int64_t tiles = ceil_div(M, BM) * g.nchunks;
  const double waves = (double)tiles / c.num_sms;
  p.ksplit = (K >= 8192 && waves > 1.0 && waves < 8.0 &&
              waves - std::floor(waves) > 0.0 && waves - std::floor(waves) < 0.75)
                 ? 2
                 : 1;
  if (part != nullptr) p.ksplit = splits;
  else if (p.ksplit > 1)
    BRSVD_CUDA(cudaMemset2DAsync(C, (size_t)ldc * sizeof(float), 0, (size_t)M * sizeof(float),
                                 (size_t)l, c.stream));
  const size_t smem = smem_bytes(g.rows_c, h16);
  const dim3 grid((unsigned)(tiles * p.ksplit));
#define BRSVD_TC_LAUNCH(KM, NCM, H)                                                      \
  do {                                                                                   \
    BRSVD_CUDA(cudaFuncSetAttribute(tc3_gemm_kernel<KM, NCM, H>,                         \
                                    cudaFuncAttributeMaxDynamicSharedMemorySize,         \
                                    (int)smem));                                         \
    tc3_gemm_kernel<KM, NCM, H><<<grid, kThreads, smem, c.stream>>>(mapA, mapBhi, mapBlo, \
                                                                    p);                  \
  } while (0)
#define BRSVD_TC_NC(KM, H)                                       \
  do {                                                           \
    if (g.rows_c <= 32) BRSVD_TC_LAUNCH(KM, 32, H);              \
    else if (g.rows_c <= 64) BRSVD_TC_LAUNCH(KM, 64, H);         \
    else if (g.rows_c <= 96) BRSVD_TC_LAUNCH(KM, 96, H);         \
    else if (g.rows_c <= 128) BRSVD_TC_LAUNCH(KM, 128, H);       \
    else BRSVD_TC_LAUNCH(KM, 160, H);                            \
  } while (0)
  if (h16) {
    if (kmajor) BRSVD_TC_NC(true, true);
    else BRSVD_TC_NC(false, true);
  } else {
    if (kmajor) BRSVD_TC_NC(true, false);
    else BRSVD_TC_NC(false, false);
  }
#undef BRSVD_TC_NC
#undef BRSVD_TC_LAUNCH
  BRSVD_CHECK_LAUNCH();
}

template <>
inline void tc_gemm_launch<double>(Ctx&, const double*, int64_t, int64_t, int64_t, bool, bool,
                                   const double*, int64_t, int, double*, int64_t, int, float*,
                                   const float*, float*, double) {
  throw Error(kErrArg, "tcgen05 path is fp32-only");
}

// Fixed-order sum of the split-K partials (deterministic), fp64 output;
// scales (optional) = [row inverse scales (M), column inverse scales (N)] of
// a keep_scaled product, applied in fp64 so Grams of tiny or huge fp32 data
// neither underflow nor overflow.
__global__ void splitk_sum_kernel(const float* __restrict__ part, int64_t M, int64_t N,
                                  int splits, double* __restrict__ C, int64_t ldc,
                                  const float* __restrict__ scales = nullptr) {
  const int64_t total = M * N;
  for (int64_t idx = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; idx < total;
       idx += (int64_t)gridDim.x * blockDim.x) {
    double s = 0.0;
    for (int z = 0; z < splits; ++z) s += (double)part[(int64_t)z * total + idx];
    const int64_t i = idx % M, j = idx / M;
    if (scales) s *= (double)scales[i] * (double)scales[M + j];
    C[i + j * ldc] = s;
  }
}

// C (a x b, fp64) = X^T Y for tall-skinny fp32 X (r x a), Y (r x b): the
// tcgen05 3xTF32 product with the long K = r split over CTAs (fp32 partial
// sums of <= r / splits terms, summed in fp64 in a fixed order).  fp32-level
// accuracy: for Grams of well-conditioned bases only.
inline bool tc_gram(Ctx& c, const float* X, int64_t r, int a, int64_t ldx, const float* Y,
                    int64_t ldy, int b, double* C, int64_t ldc) {
  if (!tc_gemm_supported<float>(c, X, ldx, r, a, b) || r < 1024) return false;
  const tc::Geometry g = tc::geometry(b);
  const int64_t tiles = ceil_div(a, tc::BM) * g.nchunks;
  int splits = (int)std::max<int64_t>(1, ceil_div(2 * c.num_sms, tiles));
  splits = (int)std::min<int64_t>(splits, ceil_div(r, 512));
  DBuf<float> part(c, (size_t)splits * a * b), scales;
  if (tc::h16_enabled()) scales.alloc(c, (size_t)a + b);
  // Z = A^T Y with A = X (r x a, column-major): trans=true; the fp16-split
  // partials stay in scaled units and are unscaled in fp64 by the sum
  tc_gemm_launch<float>(c, X, r, a, ldx, /*row_major=*/false, /*trans=*/true, Y, ldy, b,
                        nullptr, 0, splits, part.p, nullptr, scales.p);
  splitk_sum_kernel<<<grid_for((int64_t)a * b), 256, 0, c.stream>>>(part.p, a, b, splits, C,
                                                                    ldc, scales.p);
  BRSVD_CHECK_LAUNCH();
  return true;
}

}  // namespace brsvd
