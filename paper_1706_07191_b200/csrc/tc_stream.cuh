// Persistent, cluster-paired fp16-split tcgen05 product for the A-streaming
// passes of the fp32 pipeline (big_nn / big_tn):
//     C (M x l) = opA (M x K) * B (K x l)
// opA is the big matrix (A or A^T, K-major or MN-major in memory), B the
// tall-skinny sketch (Omega, Y, Z or Q), l <= 288.  These are the products
// `a_block @ omega`, `a_block.T @ y` (rsvd.py:99-101) and `q.T @ a`
// (rsvd.py:140) of the reference.
//
// Compared with tc3_gemm_kernel (tc_gemm.cuh) this kernel
//   * keeps ALL l columns of a row tile in TMEM (accumulator = npad
//     columns), so A is read from L2 once per product instead of once per
//     column chunk;
//   * runs on CTA pairs (tcgen05.mma.cta_group::2, M = 256): each CTA of a
//     2-CTA cluster converts its own 128 rows of A into its TMEM and loads
//     only HALF of every B stage; the pair MMA reads both halves.  What
//     limits this product is the bytes delivered from L2 into the SMs
//     (measured: the data pipeline alone, without MMAs or conversion, takes
//     ~1.5 ms at config 2 when every SM receives all of B; multicast does
//     not reduce the per-SM ingest), and the pair halves B's share of it;
//   * is persistent (one pair per TPC) with a stream-K split of the
//     (row-tile-pair x 128-k chunk) work over the pairs, so no wave runs
//     partly empty; a tile split between two pairs is combined through a
//     workspace and an arrival ticket (deterministic, no fp32 atomics).
//
// Precision (as tc3): power-of-two scale per row of opA (max -> 2^14) and per
// column of B, fp16 (hi, lo) pairs carrying 22 significant bits, three
// kind::f16 MMAs per product term (a_lo b_hi + a_hi b_lo + a_hi b_hi), TMEM
// accumulator flushed every 128 k into round-to-nearest fp32 running sums in
// the converter warps' registers (the tensor core's accumulation truncates).
// The accumulator is drained a third at a time: the MMAs of a stage run over
// the column thirds T0, T1, T2 (N = npad / 3 each), so draining T0 overlaps
// the T1 / T2 MMAs and so on -- no double buffer is needed, which is what
// lets all l <= 288 columns share TMEM with six A staging slots.
//
// Warp roles (448 threads: 14 warps, which the register file accounts as 16,
// so 128 registers per thread for the running sums): warp 0 TMA producer,
// warp 1 TMEM allocator and (pair leader only) MMA issuer, warps 2-13
// converters (A tile smem -> scaled fp16 hi/lo -> tcgen05.st into a TMEM
// staging slot, the .ts operand of the MMA), drains and epilogue.
#pragma once
#include <map>
#include <mutex>
#include <utility>

#include "tc_gemm.cuh"
#include "tc_pair.cuh"
#include "tc_pair_wide.cuh"

namespace brsvd {
namespace tcs {

using tc::desc_kmajor_sw64;
using tc::h16_scale;
using tc::mbar_arrive;
using tc::mbar_expect_tx;
using tc::mbar_init;
using tc::mbar_wait;
using tc::mma_f16_ts;
using tc::pack_h2;
using tc::smem_u32;
using tc::tc_after_sync;
using tc::tc_before_sync;
using tc::unpack_h2;

constexpr int BM = 128;      // rows of opA per CTA
constexpr int BKS = 32;      // k values per stage
constexpr int CHUNK = 4;     // stages per accumulator flush (128 k)
constexpr int kConv = 12;    // converter warps: three per TMEM lane quadrant
constexpr int kThreads = 64 + 32 * kConv;   // 2 role warps + converters
constexpr uint32_t A_BYTES = BM * BKS * 4;   // fp32 A stage (16 KB)
constexpr int NPAD_MAX = 288;
constexpr int kBarBytes = 512;

__host__ __device__ constexpr uint32_t b_stage_bytes(int npad) {
  return (uint32_t)npad * 64u;   // this CTA's half of B_hi + B_lo: npad/2 rows x 64 B x 2
}
__host__ __device__ constexpr int stages_for(int npad) {
  // as many 32-k stages as ~212 KB of shared memory holds (max 6)
  return (int)((217088u / (A_BYTES + b_stage_bytes(npad))) > 6u
                   ? 6u
                   : (217088u / (A_BYTES + b_stage_bytes(npad))));
}
__host__ __device__ constexpr size_t smem_bytes(int npad) {
  return (size_t)stages_for(npad) * (A_BYTES + b_stage_bytes(npad)) + kBarBytes + 1024;
}

struct Params {
  int64_t M, K;
  int npad, n_out;
  int nkb, nch;        // 32-k stages and 128-k chunks along K
  int ptiles;          // pairs of 128-row tiles
  int nclusters;       // clusters launched
  int nsplit;          // 0: stream-K ranges; 1 / 2: tiles in nsplit fixed parts
  float* C;
  int64_t ldc;
  float* ws;              // split tiles: the two parts' partial sums
  int* cnt;               // split tiles: arrival tickets (zero between launches)
  const float* row_max;   // max |opA(row, :)| (power-of-two row scales)
  const float* col_inv;   // inverse power-of-two scales of the B columns
  int out_exp;            // the output is multiplied by 2^out_exp
  unsigned long long* dbg;   // BRSVD_TCS_DEBUG: event times of cluster 0 (globaltimer)
  int flags;              // experiments (BRSVD_TCS_FLAGS): 1 no multicast, 2 no MMAs,
                          // 4 no conversion
};

struct Item {
  int p, ch0, ch1;
  bool split;
};

// The clusters' shares of the (tile pair x chunk) work, identical in every
// role of both CTAs of a cluster.
struct Sched {
  int u, u1;   // units (tile pair x chunk) < 2^31 (checked by the launcher)
  int h, hend;
  __device__ void init(const Params& P, int cl) {
    if (P.nsplit == 0) {
      const int64_t U = (int64_t)P.ptiles * P.nch;
      u = (int)((int64_t)cl * U / P.nclusters);
      u1 = (int)((int64_t)(cl + 1) * U / P.nclusters);
    } else {
      h = cl;
      hend = P.ptiles * P.nsplit;
    }
  }
  __device__ bool next(const Params& P, Item& it) {
    if (P.nsplit == 0) {
      if (u >= u1) return false;
      it.p = (int)(u / P.nch);
      it.ch0 = (int)(u % P.nch);
      it.ch1 = min(P.nch, it.ch0 + (u1 - u));
      u += it.ch1 - it.ch0;
      it.split = !(it.ch0 == 0 && it.ch1 == P.nch);
      return true;
    }
    if (h >= hend) return false;
    it.p = h / P.nsplit;
    const int part = h % P.nsplit;
    it.ch0 = (int)((int64_t)part * P.nch / P.nsplit);
    it.ch1 = (int)((int64_t)(part + 1) * P.nch / P.nsplit);
    it.split = P.nsplit > 1;
    h += P.nclusters;
    return true;
  }
};

__device__ __forceinline__ uint32_t cluster_rank() {
  uint32_t r;
  asm volatile("mov.u32 %0, %%cluster_ctarank;" : "=r"(r));
  return r;
}
__device__ __forceinline__ uint32_t cluster_id() {
  uint32_t r;
  asm volatile("mov.u32 %0, %%clusterid.x;" : "=r"(r));
  return r;
}
__device__ __forceinline__ void cluster_sync_all() {
  asm volatile("barrier.cluster.arrive.release.aligned;\n"
               "barrier.cluster.wait.acquire.aligned;" ::: "memory");
}
__device__ __forceinline__ void tmem_st4(uint32_t taddr, const uint32_t (&v)[4]) {
  asm volatile("tcgen05.st.sync.aligned.32x32b.x4.b32 [%0], {%1,%2,%3,%4};" ::"r"(taddr),
               "r"(v[0]), "r"(v[1]), "r"(v[2]), "r"(v[3])
               : "memory");
}
// Non-blocking phase test, the lane-0 result broadcast (warp-uniform control).
__device__ __forceinline__ bool mbar_test_warp(uint64_t* bar, uint32_t parity) {
  uint32_t ok;
  asm volatile(
      "{\n.reg .pred p;\nmbarrier.test_wait.parity.shared::cta.b64 p, [%1], %2;\n"
      "selp.u32 %0, 1, 0, p;\n}"
      : "=r"(ok)
      : "r"(smem_u32(bar)), "r"(parity)
      : "memory");
  return __shfl_sync(0xffffffffu, ok, 0) != 0;
}
__device__ __forceinline__ void tma_prefetch_2d(const CUtensorMap* map, int x, int y) {
  asm volatile("cp.async.bulk.prefetch.tensor.2d.L2.global.tile [%0, {%1, %2}];" ::"l"(map),
               "r"(x), "r"(y)
               : "memory");
}
// shared::cluster address of the same shared variable in CTA rank 0
__device__ __forceinline__ uint32_t mapa_rank0(uint32_t addr) {
  uint32_t r;
  asm volatile("mapa.shared::cluster.u32 %0, %1, 0;" : "=r"(r) : "r"(addr));
  return r;
}
// Remote arrive without release semantics: what it orders (TMEM loads / stores
// of this warp) is complete already (tcgen05.wait::ld / wait::st precede it).
__device__ __forceinline__ void mbar_arrive_cluster(uint32_t cluster_addr) {
  asm volatile("mbarrier.arrive.relaxed.cluster.shared::cluster.b64 _, [%0];" ::"r"(
                   cluster_addr)
               : "memory");
}
// 2-CTA TMA load into this CTA's shared memory, completing on a barrier that
// may live in the peer CTA (the pair leader's)
__device__ __forceinline__ void tma_load_2d_pair(void* dst, const CUtensorMap* map,
                                                 uint32_t bar_cluster, int x, int y) {
  asm volatile(
      "cp.async.bulk.tensor.2d.cta_group::2.shared::cluster.global.mbarrier::complete_tx::bytes"
      " [%0], [%1, {%3, %4}], [%2];" ::"r"(smem_u32(dst)),
      "l"(map), "r"(bar_cluster), "r"(x), "r"(y)
      : "memory");
}
__device__ __forceinline__ void mma2_f16_ts(uint32_t d, uint32_t a, uint64_t bdesc,
                                            uint32_t idesc, uint32_t accumulate) {
  asm volatile(
      "{\n.reg .pred p;\nsetp.ne.b32 p, %4, 0;\n"
      "tcgen05.mma.cta_group::2.kind::f16 [%0], [%1], %2, %3, p;\n}" ::"r"(d),
      "r"(a), "l"(bdesc), "r"(idesc), "r"(accumulate)
      : "memory");
}
__device__ __forceinline__ void mma2_commit_mc(uint64_t* bar, uint16_t mask) {
  asm volatile(
      "tcgen05.commit.cta_group::2.mbarrier::arrive::one.shared::cluster.multicast::cluster.b64"
      " [%0], %1;" ::"r"(smem_u32(bar)),
      "h"(mask)
      : "memory");
}
__device__ __forceinline__ void dbg_mark(const Params& P, int cl, int role, uint32_t g) {
  if (P.dbg != nullptr && cl == 0 && g < 256) {
    unsigned long long t;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
    P.dbg[role * 256 + g] = t;
  }
}
__device__ __forceinline__ void tmem_st2(uint32_t taddr, const uint32_t (&v)[2]) {
  asm volatile("tcgen05.st.sync.aligned.32x32b.x2.b32 [%0], {%1,%2};" ::"r"(taddr), "r"(v[0]),
               "r"(v[1])
               : "memory");
}
__device__ __forceinline__ void tmem_ld4(uint32_t taddr, uint32_t (&v)[4]) {
  asm volatile("tcgen05.ld.sync.aligned.32x32b.x4.b32 {%0,%1,%2,%3}, [%4];"
               : "=r"(v[0]), "=r"(v[1]), "=r"(v[2]), "=r"(v[3])
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

// NPAD: padded l (96, 192 or 288); A_KMAJOR: opA rows contiguous in k.
template <bool A_KMAJOR, int NPAD>
__global__ void __launch_bounds__(kThreads, 1)
    tcs_gemm_kernel(const __grid_constant__ CUtensorMap mapA,
                    const __grid_constant__ CUtensorMap mapBhi,
                    const __grid_constant__ CUtensorMap mapBlo, const Params P) {
  constexpr int STAGES = stages_for(NPAD);
  constexpr int NW = NPAD / 3;            // columns per accumulator third (one MMA, N = NW)
  constexpr int QW = NW / 2;              // B columns of a third held by each CTA
  constexpr int G4 = NW / 4;              // 4-column groups per third
  constexpr int CWG = (G4 + 2) / 3;       // groups per converter warp per third (at most)
  constexpr int CW = 4 * CWG;             // running sums per third per thread
  constexpr uint32_t BPL = (uint32_t)NPAD / 2 * 64;    // this CTA's rows of one B plane
  constexpr uint32_t STAGE = A_BYTES + 2 * BPL;
  constexpr uint32_t kASlot = 512 - STAGES * 32;       // TMEM A staging slots
  constexpr int PF = 12;                               // A prefetch distance (stages)
  static_assert(NPAD % 96 == 0 && NPAD <= NPAD_MAX, "npad: thirds of 2 x 16k columns");
  static_assert(kASlot >= (uint32_t)NPAD, "TMEM budget");

  extern __shared__ uint8_t smem_dyn[];
  uint8_t* smem = (uint8_t*)(((uintptr_t)smem_dyn + 1023) & ~(uintptr_t)1023);
  uint64_t* fullA = reinterpret_cast<uint64_t*>(smem + STAGES * STAGE);  // own A landed
  uint64_t* fullB = fullA + STAGES;      // leader: both B halves landed
  uint64_t* freeb = fullB + STAGES;      // stage consumed by the pair MMA
  uint64_t* tfull = freeb + STAGES;      // leader: both CTAs' A converted into TMEM
  uint64_t* accready = tfull + STAGES;   // [3]: accumulator third complete
  uint64_t* accfree = accready + 3;      // [3] leader: both CTAs drained the third
  uint32_t* tmem_holder = reinterpret_cast<uint32_t*>(accfree + 3);
  int* ticket = reinterpret_cast<int*>(tmem_holder + 1);   // split-tile ticket

  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const uint32_t crank = cluster_rank();
  const bool leader = crank == 0;
  const int cl = (int)cluster_id();

  if (warp == 0 && lane == 0) {
    for (int s = 0; s < STAGES; ++s) {
      mbar_init(&fullA[s], 1);
      mbar_init(&fullB[s], 1);
      mbar_init(&freeb[s], 1);
      mbar_init(&tfull[s], 2 * kConv);
    }
    for (int t = 0; t < 3; ++t) {
      mbar_init(&accready[t], 1);
      mbar_init(&accfree[t], 2 * kConv);
    }
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    asm volatile("prefetch.tensormap [%0];" ::"l"(&mapA) : "memory");
    asm volatile("prefetch.tensormap [%0];" ::"l"(&mapBhi) : "memory");
    asm volatile("prefetch.tensormap [%0];" ::"l"(&mapBlo) : "memory");
  }
  if (warp == 1) {   // the same warp of both CTAs allocates the pair's TMEM
    asm volatile("tcgen05.alloc.cta_group::2.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(
                     smem_u32(tmem_holder)),
                 "r"(512)
                 : "memory");
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::2.sync.aligned;" ::: "memory");
  }
  tc_before_sync();
  cluster_sync_all();   // both CTAs' barriers exist before any remote signal
  tc_after_sync();
  const uint32_t tmem = *tmem_holder;
  const int nkb = P.nkb;
  // the leader's barriers, as seen from this CTA (identical offsets)
  const uint32_t fullB0 = mapa_rank0(smem_u32(fullB));
  const uint32_t tfull0 = mapa_rank0(smem_u32(tfull));
  const uint32_t accfree0 = mapa_rank0(smem_u32(accfree));

  if (warp == 0) {
    if (lane == 0) {  // ------------------------------------------ TMA producer
      Sched sc;
      sc.init(P, cl);
      Item it;
      uint32_t g = 0;
      while (sc.next(P, it)) {
        const int row0 = it.p * (2 * BM) + (int)crank * BM;
        const int kb1 = min(nkb, it.ch1 * CHUNK);
        // L2 prefetch of the A tiles PF stages ahead (A is read exactly once)
        for (int kb = it.ch0 * CHUNK; kb < min(kb1, it.ch0 * CHUNK + PF) && !(P.flags & 32);
             ++kb) {
          if (A_KMAJOR) tma_prefetch_2d(&mapA, kb * BKS, row0);
          else tma_prefetch_2d(&mapA, row0, kb * BKS);
        }
        for (int kb = it.ch0 * CHUNK; kb < kb1; ++kb, ++g) {
          if (kb + PF < kb1 && !(P.flags & 32)) {
            if (A_KMAJOR) tma_prefetch_2d(&mapA, (kb + PF) * BKS, row0);
            else tma_prefetch_2d(&mapA, row0, (kb + PF) * BKS);
          }
          const int s = (int)(g % STAGES);
          const uint32_t ph = (g / STAGES) & 1;
          mbar_wait(&freeb[s], ph ^ 1);
          dbg_mark(P, cl, (int)crank, g);
          uint8_t* st = smem + (size_t)s * STAGE;
          const int k0 = kb * BKS;
          mbar_expect_tx(&fullA[s], A_BYTES);
          if (A_KMAJOR) tc::tma_load_2d(st, &mapA, &fullA[s], k0, row0);
          else tc::tma_load_2d(st, &mapA, &fullA[s], row0, k0);
          // this CTA's half of B (rows [crank npad/2, ..) of the permuted
          // planes); both halves complete on the leader's fullB
          const int br = (int)crank * (NPAD / 2);
          if (P.flags & 64) {   // each half on its own CTA's barrier
            mbar_expect_tx(&fullB[s], 2 * BPL);
            tc::tma_load_2d(st + A_BYTES, &mapBhi, &fullB[s], k0, br);
            tc::tma_load_2d(st + A_BYTES + BPL, &mapBlo, &fullB[s], k0, br);
          } else {
            if (leader) mbar_expect_tx(&fullB[s], 4 * BPL);
            tma_load_2d_pair(st + A_BYTES, &mapBhi, fullB0 + 8 * s, k0, br);
            tma_load_2d_pair(st + A_BYTES + BPL, &mapBlo, fullB0 + 8 * s, k0, br);
          }
        }
      }
      // every stage's final release has landed before the pair may retire
      for (uint32_t e = g; e < g + STAGES; ++e)
        if (e >= (uint32_t)STAGES) mbar_wait(&freeb[e % STAGES], ((e / STAGES) & 1) ^ 1);
    }
  } else if (warp == 1) {
    if (lane == 0 && leader) {  // ---------------------- MMA issuer (pair leader)
      // c_format f32 (bit 4); a, b fp16 (0); K-major A and B; N = NW; M = 256
      constexpr uint32_t idesc =
          (1u << 4) | ((uint32_t)(NW >> 3) << 17) | ((uint32_t)((2 * BM) >> 4) << 24);
      Sched sc;
      sc.init(P, cl);
      Item it;
      uint32_t g = 0, gc = 0;
      while (sc.next(P, it)) {
        for (int ch = it.ch0; ch < it.ch1; ++ch, ++gc) {
          const int nst = min(CHUNK, nkb - ch * CHUNK);
          for (int st = 0; st < nst; ++st, ++g) {
            const int s = (int)(g % STAGES);
            const uint32_t ph = (g / STAGES) & 1;
            mbar_wait(&tfull[s], ph);
            dbg_mark(P, cl, 6, g);
            mbar_wait(&fullB[s], ph);
            dbg_mark(P, cl, 7, g);
            tc_after_sync();
            const uint32_t bh = smem_u32(smem + (size_t)s * STAGE + A_BYTES);
            const uint32_t bl = bh + BPL;
            const uint32_t a_hi = tmem + kASlot + (uint32_t)s * 32, a_lo = a_hi + 16;
#pragma unroll
            for (int t = 0; t < 3; ++t) {
              if (st == 0 && gc > 0) {   // the previous chunk's third t is drained
                mbar_wait(&accfree[t], (gc - 1) & 1);
                if (t == 2) dbg_mark(P, cl, 13, gc - 1);
                tc_after_sync();
              }
              const uint32_t d = tmem + (uint32_t)(t * NW);
#pragma unroll
              for (int kk = 0; kk < 2; ++kk) {
                const uint64_t dh = desc_kmajor_sw64(bh + t * QW * 64 + kk * 32);
                const uint64_t dl = desc_kmajor_sw64(bl + t * QW * 64 + kk * 32);
                const uint32_t acc = (st == 0 && kk == 0) ? 0u : 1u;
                if (!(P.flags & 2)) {
                  mma2_f16_ts(d, a_lo + kk * 8, dh, idesc, acc);
                  mma2_f16_ts(d, a_hi + kk * 8, dl, idesc, 1u);
                  mma2_f16_ts(d, a_hi + kk * 8, dh, idesc, 1u);
                }
              }
              if (st == nst - 1) mma2_commit_mc(&accready[t], 0x3);
            }
            mma2_commit_mc(&freeb[s], 0x3);
            dbg_mark(P, cl, 8, g);
          }
        }
      }
    }
  } else {  // ---------------------------------- converters, drains, epilogue
    // a warp reaches the TMEM lanes 32 (warp % 4) .. + 31 only
    const int wq = warp & 3;         // TMEM lane quadrant: rows 32 wq .. 32 wq + 31
    const int jw = (warp - 2) >> 2;  // share within the quadrant: k groups jw, jw+3, jw+6
                                     // (4 k each) of a stage; column groups [g0, g0+ng)
                                     // of each third
    const int g0 = jw * G4 / 3, ng = (jw + 1) * G4 / 3 - g0;
    const int r = wq * 32 + lane;
    const uint32_t lane_base = (uint32_t)(wq * 32) << 16;
    const uint32_t smem_base = smem_u32(smem);
    float run[3 * CW];
#pragma unroll
    for (int j = 0; j < 3 * CW; ++j) run[j] = 0.f;

    // drain cursor: walks the same items / chunks as the MMA issuer
    Sched sd;
    sd.init(P, cl);
    Item itd;
    bool dvalid = sd.next(P, itd);
    int dch = dvalid ? itd.ch0 : 0;
    int dthird = 0;                                    // next third to drain
    uint32_t dgc = 0;                                  // chunk counter
    uint32_t dend = dvalid ? (uint32_t)(min(CHUNK, nkb - dch * CHUNK) - 1) : 0;  // last stage

    auto epilogue = [&](const Item& e) {
      const int64_t row = (int64_t)e.p * (2 * BM) + (int64_t)crank * BM + r;
      // power-of-two unscale in fp64: exact, one rounding, no spurious
      // over/underflow of the combined factor
      const double rf =
          row < P.M ? ldexp(1.0, P.out_exp - (P.row_max != nullptr
                                                  ? ilogbf(h16_scale(P.row_max[row]))
                                                  : 0))
                    : 0.0;
      auto col_of = [&](int t, int j) { return t * NW + g0 * 4 + j; };
      auto val = [&](int t, int j) {
        return (float)((double)run[t * CW + j] * (rf * (double)P.col_inv[col_of(t, j)]));
      };
      if (!e.split) {
        if (row < P.M) {
#pragma unroll
          for (int t = 0; t < 3; ++t)
#pragma unroll
            for (int j = 0; j < CW; ++j)
              if (j < 4 * ng && col_of(t, j) < P.n_out)
                P.C[row + (int64_t)col_of(t, j) * P.ldc] = val(t, j);
        }
      } else {
        // a tile in two parts: both park their unscaled partial in the
        // workspace; the second to arrive (ticket 1) adds the other's and
        // writes C.  a + b is commutative, so the result does not depend on
        // which part finishes first (no atomics: fp32 atomics flush
        // subnormal partials to zero).
        const int part = e.ch0 == 0 ? 0 : 1;
        const int slot =
            P.nsplit == 0
                ? (int)((((int64_t)e.p * P.nch + P.nch) * P.nclusters - 1) /
                        ((int64_t)P.ptiles * P.nch))
                : e.p;
        float* mine = P.ws + (size_t)((slot * 2 + part) * 2 + (int)crank) * NPAD * BM;
        const float* other =
            P.ws + (size_t)((slot * 2 + (part ^ 1)) * 2 + (int)crank) * NPAD * BM;
#pragma unroll
        for (int t = 0; t < 3; ++t)
#pragma unroll
          for (int j = 0; j < CW; ++j)
            if (j < 4 * ng) __stcg(mine + col_of(t, j) * BM + r, val(t, j));
        __threadfence();
        asm volatile("bar.sync 1, %0;" ::"n"(32 * kConv) : "memory");
        if (threadIdx.x == 64) {
          *ticket = atomicAdd(P.cnt + slot * 2 + (int)crank, 1);
          __threadfence();
        }
        asm volatile("bar.sync 1, %0;" ::"n"(32 * kConv) : "memory");
        if (*ticket == 1) {
          if (row < P.M) {
#pragma unroll
            for (int t = 0; t < 3; ++t)
#pragma unroll
              for (int j = 0; j < CW; ++j)
                if (j < 4 * ng && col_of(t, j) < P.n_out)
                  P.C[row + (int64_t)col_of(t, j) * P.ldc] =
                      val(t, j) + __ldcg(other + col_of(t, j) * BM + r);
          }
          if (threadIdx.x == 64) P.cnt[slot * 2 + (int)crank] = 0;   // for the next launch
        }
        asm volatile("bar.sync 1, %0;" ::"n"(32 * kConv) : "memory");
      }
#pragma unroll
      for (int j = 0; j < 3 * CW; ++j) run[j] = 0.f;
    };
    // drain one accumulator third (its MMAs have completed)
    auto drain_third = [&]() {
      const int t = dthird;
      if (warp == 2 && lane == 0 && crank == 0) dbg_mark(P, cl, 9 + 2 * t, dgc);
      tc_after_sync();
      // up to four 4-column loads in flight per wait (a TMEM load round trip
      // costs ~250 cycles while the MMAs run)
#pragma unroll
      for (int j0 = 0; j0 < CWG; j0 += 4) {
        uint32_t v[4][4];
#pragma unroll
        for (int u = 0; u < 4; ++u)
          if (j0 + u < CWG && j0 + u < ng)
            tmem_ld4(tmem + lane_base + (uint32_t)(t * NW + (g0 + j0 + u) * 4), v[u]);
        asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
#pragma unroll
        for (int u = 0; u < 4; ++u)
          if (j0 + u < CWG && j0 + u < ng)
#pragma unroll
            for (int i = 0; i < 4; ++i) {
              const int jj = 4 * (j0 + u) + i;
              if (t == 0) run[jj] += __uint_as_float(v[u][i]);
              else if (t == 1) run[CW + jj] += __uint_as_float(v[u][i]);
              else run[2 * CW + jj] += __uint_as_float(v[u][i]);
            }
      }
      tc_before_sync();
      __syncwarp();
      if (warp == 2 && lane == 0 && crank == 0) dbg_mark(P, cl, 15 + t, dgc);
      if (lane == 0) mbar_arrive_cluster(accfree0 + 8 * t);
      if (warp == 2 && lane == 0 && crank == 0) dbg_mark(P, cl, 10 + 2 * t, dgc);
      if (t < 2) {
        dthird = t + 1;
        return;
      }
      dthird = 0;
      ++dgc;
      ++dch;
      if (dch >= itd.ch1) {   // the item's last chunk: write it out
        epilogue(itd);
        dvalid = sd.next(P, itd);
        if (!dvalid) return;
        dch = itd.ch0;
      }
      dend += (uint32_t)min(CHUNK, nkb - dch * CHUNK);
    };
    // drain whatever accumulator third is complete, without blocking; only a
    // chunk whose last stage this warp has converted (dend < g) can be
    auto poll_drain = [&](uint32_t g) -> bool {
      if (!dvalid || dend >= g) return false;
      if (!mbar_test_warp(&accready[dthird], dgc & 1)) return false;
      drain_third();
      return true;
    };

    Sched sc;
    sc.init(P, cl);
    Item it;
    uint32_t g = 0;
    while (sc.next(P, it)) {
      const int64_t grow = (int64_t)it.p * (2 * BM) + (int64_t)crank * BM + r;
      const float rscale =
          (P.row_max != nullptr && grow < P.M) ? h16_scale(P.row_max[grow]) : 1.f;
      const int kb1 = min(nkb, it.ch1 * CHUNK);
      for (int kb = it.ch0 * CHUNK; kb < kb1; ++kb, ++g) {
        const int s = (int)(g % STAGES);
        const uint32_t ph = (g / STAGES) & 1;
        // wait for this stage's A; drain accumulator thirds as they complete
        for (;;) {
          while (poll_drain(g)) {
          }
          if (mbar_test_warp(&fullA[s], ph)) break;
        }
        if (warp == 2 && lane == 0) dbg_mark(P, cl, 2 + (int)crank, g);
        const uint32_t sa = smem_base + (uint32_t)s * STAGE;
#pragma unroll
        for (int t = 0; t < 3; ++t) {
          const int kg = jw + 3 * t;        // k values 4 kg .. 4 kg + 3
          if (kg < 8 && !(P.flags & 4)) {
            float v[4];
            if (A_KMAJOR) {
              // 128-byte rows (32 fp32 k), TMA 128B swizzle: 16-byte chunk kg of
              // row r sits at kg ^ (r & 7)
              const float4 x = lds128(sa + r * 128 + ((kg ^ (r & 7)) << 4));
              v[0] = x.x;
              v[1] = x.y;
              v[2] = x.z;
              v[3] = x.w;
            } else {
              // one (128 rows x 32 k) box, rows contiguous: 512 bytes per k
#pragma unroll
              for (int i = 0; i < 4; ++i) v[i] = lds32(sa + (4 * kg + i) * 512 + r * 4);
            }
            uint32_t hi[2], lo[2];
#pragma unroll
            for (int i = 0; i < 2; ++i) {
              const float x0 = v[2 * i] * rscale, x1 = v[2 * i + 1] * rscale;
              hi[i] = pack_h2(x0, x1);
              const float2 hf = unpack_h2(hi[i]);
              lo[i] = pack_h2(x0 - hf.x, x1 - hf.y);
            }
            tmem_st2(tmem + lane_base + kASlot + (uint32_t)s * 32 + 2 * kg, hi);
            tmem_st2(tmem + lane_base + kASlot + (uint32_t)s * 32 + 16 + 2 * kg, lo);
          }
        }
        asm volatile("tcgen05.wait::st.sync.aligned;" ::: "memory");
        if ((P.flags & 64) && !leader) mbar_wait(&fullB[s], ph);   // this CTA's B half too
        tc_before_sync();
        __syncwarp();
        if (lane == 0) mbar_arrive_cluster(tfull0 + 8 * s);
        if (warp == 2 && lane == 0) dbg_mark(P, cl, 4 + (int)crank, g);
      }
    }
    while (dvalid) {   // the remaining chunks
      mbar_wait(&accready[dthird], dgc & 1);
      drain_third();
    }
  }
  tc_before_sync();
  __syncthreads();
  cluster_sync_all();   // no CTA retires while its peer may still signal it
  if (warp == 1) {
    tc_after_sync();
    asm volatile("tcgen05.dealloc.cta_group::2.sync.aligned.b32 %0, %1;" ::"r"(tmem), "r"(512)
                 : "memory");
  }
}

// l -> accumulator width: column halves of a multiple of 48 (MMA N multiple of
// 16, drained by three warps per lane quadrant in 4-column groups)
inline int npad_bucket(int l) {
  if (l <= 96) return 96;
  if (l <= 192) return 192;
  return 288;
}

// Opt-in (BRSVD_TCS=1): measured slower than tc3 at config 2 (see DESIGN.md
// section 7), kept with its tests as the base of the next attempt.
inline bool env_enabled() {
  const char* e = std::getenv("BRSVD_TCS");
  return e && e[0] == '1';
}

}  // namespace tcs

// C (M x l, column-major, ldc) = opA * X through the persistent cluster
// kernel; returns false when the shape is outside its envelope (the caller
// falls back to tc3).  opa_max: max |opA| per row (else computed here).
inline bool tcs_gemm_launch(Ctx& c, const float* A, int64_t m, int64_t n, int64_t lda,
                            bool row_major, bool trans, const float* X, int64_t ldx, int l,
                            float* C, int64_t ldc, const float* opa_max, double out_scale) {
  using namespace tcs;
  if (!tcs::env_enabled() || !tc::h16_enabled() || l < 1 || l > NPAD_MAX) return false;
  const int64_t M = trans ? n : m, K = trans ? m : n;
  if (M > (int64_t)INT32_MAX - 2 * BM || K > (int64_t)INT32_MAX - 2 * BKS) return false;
  if (ceil_div(M, 2 * BM) * ceil_div(ceil_div(K, BKS), CHUNK) >= (int64_t)INT32_MAX) return false;
  const bool kmajor = row_major != trans;
  const int npad = npad_bucket(l);
  if (smem_bytes(npad) > c.max_smem_optin) return false;
  const uint64_t inner = row_major ? (uint64_t)n : (uint64_t)m;
  const uint64_t outer = row_major ? (uint64_t)m : (uint64_t)n;
  const CUtensorMap mapA =
      kmajor ? tc::make_map(A, inner, outer, (uint64_t)lda * 4, 32, BM,
                            CU_TENSOR_MAP_SWIZZLE_128B)
             : tc::make_map(A, inner, outer, (uint64_t)lda * 4, BM, BKS,
                            CU_TENSOR_MAP_SWIZZLE_NONE);
  DBuf<float> hi, lo, opmax, cinv, ws;
  DBuf<int> cnt;
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
  tc::tc_split16_col_kernel<<<(unsigned)npad, 512, 0, c.stream>>>(
      X, K, l, ldx, kld, reinterpret_cast<uint16_t*>(hi.p), reinterpret_cast<uint16_t*>(lo.p),
      cinv.p, npad / 6);
  BRSVD_CHECK_LAUNCH();
  const CUtensorMap mapBhi =
      tc::make_map(hi.p, (uint64_t)kld, (uint64_t)npad, (uint64_t)kld * 2, BKS,
                   (uint32_t)(npad / 2), CU_TENSOR_MAP_SWIZZLE_64B,
                   CU_TENSOR_MAP_DATA_TYPE_FLOAT16);
  const CUtensorMap mapBlo =
      tc::make_map(lo.p, (uint64_t)kld, (uint64_t)npad, (uint64_t)kld * 2, BKS,
                   (uint32_t)(npad / 2), CU_TENSOR_MAP_SWIZZLE_64B,
                   CU_TENSOR_MAP_DATA_TYPE_FLOAT16);
  Params p;
  p.M = M;
  p.K = K;
  p.npad = npad;
  p.n_out = l;
  p.nkb = (int)ceil_div(K, BKS);
  p.nch = (int)ceil_div(p.nkb, CHUNK);
  p.ptiles = (int)ceil_div(M, 2 * BM);
  p.C = C;
  p.ldc = ldc;
  p.row_max = opa_max;
  p.col_inv = cinv.p;
  {
    int e = 0;
    const double f = std::frexp(out_scale, &e);   // out_scale = 2^(e-1) (a power of two)
    BRSVD_REQUIRE(f == 0.5, kErrArg, "output scale must be a power of two");
    p.out_exp = e - 1;
  }
  const size_t smem = smem_bytes(npad);
  p.flags = std::getenv("BRSVD_TCS_FLAGS") ? std::atoi(std::getenv("BRSVD_TCS_FLAGS")) : 0;
  DBuf<unsigned long long> dbgbuf;
  p.dbg = nullptr;
  if (std::getenv("BRSVD_TCS_DEBUG")) {
    dbgbuf.alloc(c, 18 * 256);
    BRSVD_CUDA(cudaMemsetAsync(dbgbuf.p, 0, 18 * 256 * 8, c.stream));
    p.dbg = dbgbuf.p;
  }

  auto launch = [&](auto kern) {
    BRSVD_CUDA(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                    (int)smem));
    cudaLaunchConfig_t cfg = {};
    cudaLaunchAttribute attr[1];
    attr[0].id = cudaLaunchAttributeClusterDimension;
    attr[0].val.clusterDim.x = 2;
    attr[0].val.clusterDim.y = 1;
    attr[0].val.clusterDim.z = 1;
    cfg.blockDim = dim3(kThreads);
    cfg.dynamicSmemBytes = smem;
    cfg.stream = c.stream;
    cfg.attrs = attr;
    cfg.numAttrs = 1;
    cfg.gridDim = dim3(2);
    // resident clusters of this kernel (queried once per device and variant)
    static std::mutex mu;
    static std::map<std::pair<const void*, int>, int> cache;
    int maxc = 0;
    {
      std::lock_guard<std::mutex> lk(mu);
      const auto key = std::make_pair(reinterpret_cast<const void*>(kern), c.device);
      auto f = cache.find(key);
      if (f != cache.end()) {
        maxc = f->second;
      } else {
        BRSVD_CUDA(cudaOccupancyMaxActiveClusters(&maxc, kern, &cfg));
        if (maxc < 1) maxc = 1;
        cache[key] = maxc;
      }
    }
    // stream-K over all resident clusters when every cluster gets at least a
    // whole tile pair (then no tile has more than two parts); otherwise the
    // tile pairs in two fixed K halves (or whole)
    if (p.ptiles >= maxc) {
      p.nsplit = 0;
      p.nclusters = maxc;
    } else {
      p.nsplit = p.nch >= 2 ? 2 : 1;
      p.nclusters = std::min(maxc, p.ptiles * p.nsplit);
    }
    // split tiles: one workspace slot per cluster boundary (stream-K) or per
    // tile pair (halves); 2 parts x 2 CTAs x npad x 128 floats each
    const int nslots = p.nsplit == 0 ? p.nclusters : (p.nsplit == 2 ? p.ptiles : 0);
    if (nslots > 0) {
      ws.alloc(c, (size_t)nslots * 4 * npad * BM);
      cnt.alloc(c, (size_t)nslots * 2);
      BRSVD_CUDA(cudaMemsetAsync(cnt.p, 0, sizeof(int) * nslots * 2, c.stream));
    }
    p.ws = ws.p;
    p.cnt = cnt.p;
    cfg.gridDim = dim3((unsigned)(2 * p.nclusters));
    if (std::getenv("BRSVD_DEBUG")) {
      cudaFuncAttributes fa;
      cudaFuncGetAttributes(&fa, kern);
      std::fprintf(stderr,
                   "[brsvd] tcs npad %d kmajor %d M %lld K %lld: regs %d maxthr %d local %zu "
                   "smem %zu clusters %d (max %d) nsplit %d\n",
                   npad, (int)kmajor, (long long)M, (long long)K, fa.numRegs,
                   fa.maxThreadsPerBlock, (size_t)fa.localSizeBytes, smem, p.nclusters, maxc,
                   p.nsplit);
    }
    BRSVD_CUDA(cudaLaunchKernelEx(&cfg, kern, mapA, mapBhi, mapBlo, p));
  };
#define BRSVD_TCS_CASE(NP)                                                        \
  case NP:                                                                        \
    if (kmajor) launch(tcs_gemm_kernel<true, NP>);                                \
    else launch(tcs_gemm_kernel<false, NP>);                                      \
    break;
  switch (npad) {
    BRSVD_TCS_CASE(96)
    BRSVD_TCS_CASE(192)
    BRSVD_TCS_CASE(288)
    default:
      return false;
  }
#undef BRSVD_TCS_CASE
  BRSVD_CHECK_LAUNCH();
  if (p.dbg != nullptr) {   // event table of cluster 0 (ns, relative to the first issue)
    std::vector<unsigned long long> h(18 * 256);
    BRSVD_CUDA(cudaMemcpyAsync(h.data(), p.dbg, h.size() * 8, cudaMemcpyDeviceToHost, c.stream));
    BRSVD_CUDA(cudaStreamSynchronize(c.stream));
    const unsigned long long t0 = h[0];
    std::fprintf(stderr, "[tcs dbg] g: issue0 issue1 fullA0 fullA1 arr0 arr1 tfull fullB commit\n");
    std::fprintf(stderr, "[tcs dbg] chunk: s0 a0 s1 a1 s2 a2 (rank0 warp2: third start, after arrive) mma_accfree ld0 ld1 ld2\n");
    for (int g = 0; g < 16; ++g) {
      std::fprintf(stderr, "[tcs dbg] c%3d:", g);
      for (int r = 9; r < 18; ++r)
        std::fprintf(stderr, " %7lld", h[r * 256 + g] ? (long long)(h[r * 256 + g] - t0) : -1LL);
      std::fprintf(stderr, "\n");
    }
    for (int g = 0; g < 32; ++g) {
      std::fprintf(stderr, "[tcs dbg] %3d:", g);
      for (int r = 0; r < 9; ++r)
        std::fprintf(stderr, " %7lld", h[r * 256 + g] ? (long long)(h[r * 256 + g] - t0) : -1LL);
      std::fprintf(stderr, "\n");
    }
  }
  return true;
}

// The fp32 A-streaming product: the persistent cluster kernel when the shape
// allows, else the per-tile tc3 kernel.
// The product dispatch below picks the single-chunk pair kernel for this l
// (the only one that can run on sampled scales, LazyScales in pipeline.cuh).
inline bool tcw_selected(Ctx& c, int l) {
  return !tcs::env_enabled() && tcw::enabled() && tcp::enabled() && tc::h16_enabled() &&
         tcw::fits(l) && !c.b_hi_only;
}

// amax_out / run_flag: see Params (single-chunk pair kernel only; the caller
// checks tcw_selected first).
inline void tc_product(Ctx& c, const float* A, int64_t m, int64_t n, int64_t lda,
                       bool row_major, bool trans, const float* X, int64_t ldx, int l, float* C,
                       int64_t ldc, const float* opa_max = nullptr, double out_scale = 1.0,
                       unsigned* amax_out = nullptr, const int* run_flag = nullptr) {
  if (amax_out != nullptr || run_flag != nullptr) {
    if (!tcw_selected(c, l))
      throw Error(kErrArg, "tc_product: sampled scales need the single-chunk pair kernel");
    tcw_gemm_launch(c, A, m, n, lda, row_major, trans, X, ldx, l, C, ldc, opa_max, out_scale,
                    amax_out, run_flag);
    return;
  }
  if (tcs_gemm_launch(c, A, m, n, lda, row_major, trans, X, ldx, l, C, ldc, opa_max,
                      out_scale))
    return;
  if (tcw::enabled() && tcp::enabled() && tc::h16_enabled() && tcw::fits(l) &&
      !c.b_hi_only) {
    tcw_gemm_launch(c, A, m, n, lda, row_major, trans, X, ldx, l, C, ldc, opa_max, out_scale);
    return;
  }
  if (tcp::enabled() && tc::h16_enabled() && tcp::tcp_fits(l)) {
    tcp_gemm_launch(c, A, m, n, lda, row_major, trans, X, ldx, l, C, ldc, opa_max, out_scale);
    return;
  }
  tc_gemm_launch<float>(c, A, m, n, lda, row_major, trans, X, ldx, l, C, ldc, 0, nullptr,
                        opa_max, nullptr, out_scale);
}

}  // namespace brsvd
