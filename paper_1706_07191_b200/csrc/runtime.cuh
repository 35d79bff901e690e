// C++ runtime for the BRSVD hot path: device context, stream-ordered scratch
// buffers, kernel launchers, rank-revealing orthonormalisation and the
// in-core randomized SVD pipeline.
//
// Algorithm map (reference: /root/reference/pkg/src/blocksvd):
//   rsvd_device      <- rsvd_incore        rsvd.py:126-141 (global power iter.)
//   orth_full        <- tsqr / tsqr_factor kernels.py:139-170
//   small_svd_device <- small_svd          kernels.py:173-188
//   fix_signs        <- _fix_signs         rsvd.py:105-115
//   overflow guard   <- _check_overflow    rsvd.py:84-91
#pragma once
#include <algorithm>
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <vector>

#include "common.cuh"
#include "gemm_simt.cuh"
#include "gram_simt.cuh"
#include "chol.cuh"
#include "jacobi.cuh"
#include "jacobi_cluster.cuh"
#include "small_kernels.cuh"

namespace brsvd {

struct Ctx {
  int device = 0;
  cudaStream_t stream = nullptr;
  bool own_stream = false;
  unsigned long long* h_pinned = nullptr;  // small pinned readback area
  int num_sms = kNumSMs;
  int cc_major = 0, cc_minor = 0;
  size_t max_smem_optin = 0;
  // profiling of the big A-streaming products (brsvd_profile_begin/end)
  bool prof = false;
  std::vector<cudaEvent_t> prof_ev;  // start/stop pairs
  double prof_flops = 0.0, prof_bytes = 0.0;
  long long prof_launch0 = 0;
  // fp16-split products of the power iteration with the sketch operand
  // rounded to fp16 (two MMAs per term instead of three), see PowerLowp
  bool b_hi_only = false;
};

// Scope in which the fp32 A-streaming products may use the two-term split
// (a_hi b_hi + a_lo b_hi: A keeps its 22 bits, the sketch operand X / Y
// rounded to fp16) -- the power-iteration products only; the core product
// B = Q^T A and every basis change stay three-term.  OFF by default (the
// shipped products carry ~22 bits in both operands, fp32-equivalent);
// BRSVD_POWER_LOWP=1 opts in: measured 19.3 -> 17.7 ms at config 2 with
// every GPU parity test still inside the north-star tolerances, but the
// sketch operand of those products is then below fp32 precision.
struct PowerLowp {
  Ctx& c;
  bool prev;
  explicit PowerLowp(Ctx& c_) : c(c_), prev(c_.b_hi_only) {
    const char* e = std::getenv("BRSVD_POWER_LOWP");
    c.b_hi_only = e && e[0] == '1';
  }
  ~PowerLowp() { c.b_hi_only = prev; }
};

// Brackets one big-product launch with events when profiling is on.
struct ProfScope {
  Ctx& c;
  bool on;
  ProfScope(Ctx& c_, double flops, double bytes, bool counted = true)
      : c(c_), on(c_.prof && counted) {
    if (!on) return;
    cudaEvent_t e;
    BRSVD_CUDA(cudaEventCreate(&e));
    BRSVD_CUDA(cudaEventRecord(e, c.stream));
    c.prof_ev.push_back(e);
    c.prof_flops += flops;
    c.prof_bytes += bytes;
  }
  ~ProfScope() {
    if (!on) return;
    cudaEvent_t e;
    if (cudaEventCreate(&e) == cudaSuccess) {
      cudaEventRecord(e, c.stream);
      c.prof_ev.push_back(e);
    }
  }
};

// Stream-ordered device buffer (cudaMallocAsync from the device default pool).
template <typename T>
struct DBuf {
  T* p = nullptr;
  size_t n = 0;
  cudaStream_t s = nullptr;
  DBuf() = default;
  DBuf(Ctx& c, size_t count) { alloc(c, count); }
  void alloc(Ctx& c, size_t count) {
    release();
    s = c.stream;
    n = count;
    if (count) BRSVD_CUDA(cudaMallocAsync((void**)&p, count * sizeof(T), s));
  }
  void release() {
    if (p) cudaFreeAsync(p, s);
    p = nullptr;
    n = 0;
  }
  ~DBuf() { release(); }
  DBuf(const DBuf&) = delete;
  DBuf& operator=(const DBuf&) = delete;
  operator T*() const { return p; }
};

inline int grid_for(int64_t total, int threads = 256, int max_blocks = 148 * 16) {
  int64_t b = ceil_div(std::max<int64_t>(total, 1), threads);
  return (int)std::min<int64_t>(b, max_blocks);
}

// ---------------------------------------------------------------------------
// Strided GEMM launcher (deterministic split-K).
template <typename TA, typename TB, typename TAcc, typename TC>
void gemm(Ctx& c, int64_t M, int64_t N, int64_t K, const TA* A, int64_t sam,
          int64_t sak, const TB* B, int64_t sbk, int64_t sbn, TC* C,
          int64_t scm, int64_t scn, TAcc alpha = TAcc(1), TAcc beta = TAcc(0),
          const TC* C0 = nullptr, int64_t sc0m = 0, int64_t sc0n = 0) {
  if (M <= 0 || N <= 0) return;
  constexpr bool dbl = sizeof(TAcc) == 8;
  constexpr int BM = 64, BK = dbl ? 8 : 16, TM = 4;
  const bool narrow = N <= 32;
  const int BN = narrow ? 32 : 64;
  const int64_t tiles = ceil_div(M, BM) * ceil_div(N, BN);
  const int64_t target = 4 * c.num_sms;
  const int64_t max_split = std::max<int64_t>(1, K / (BK * 4));
  int64_t splits = std::min<int64_t>(std::max<int64_t>(1, ceil_div(target, tiles)),
                                     std::min<int64_t>(max_split, 256));
  int64_t kchunk = ceil_div(std::max<int64_t>(K, 1), splits);
  kchunk = ceil_div(kchunk, BK) * BK;
  splits = std::max<int64_t>(1, ceil_div(K, kchunk));
  DBuf<TAcc> part;
  if (splits > 1) part.alloc(c, (size_t)(splits * M * N));
  dim3 grid((unsigned)ceil_div(M, BM), (unsigned)ceil_div(N, BN), (unsigned)splits);
  if (narrow) {
    gemm_strided_kernel<TA, TB, TAcc, TC, BM, 32, BK, TM, 2>
        <<<grid, 256, 0, c.stream>>>(M, N, K, A, sam, sak, B, sbk, sbn, C, scm,
                                      scn, alpha, beta, C0, sc0m, sc0n, kchunk,
                                      part.p);
  } else {
    gemm_strided_kernel<TA, TB, TAcc, TC, BM, 64, BK, TM, 4>
        <<<grid, 256, 0, c.stream>>>(M, N, K, A, sam, sak, B, sbk, sbn, C, scm,
                                      scn, alpha, beta, C0, sc0m, sc0n, kchunk,
                                      part.p);
  }
  BRSVD_CHECK_LAUNCH();
  if (splits > 1) {
    if (splits >= 32 && M * N <= 32768)
      splitk_reduce_warp_kernel<TAcc, TC><<<grid_for(M * N * 32), 256, 0, c.stream>>>(
          M, N, (int)splits, part.p, C, scm, scn, alpha, beta, C0, sc0m, sc0n);
    else
      splitk_reduce_kernel<TAcc, TC><<<grid_for(M * N), 256, 0, c.stream>>>(
          M, N, (int)splits, part.p, C, scm, scn, alpha, beta, C0, sc0m, sc0n);
    BRSVD_CHECK_LAUNCH();
  }
}

// Tall-skinny fp64 Gram C (a x b) = X^T Y (gram_simt.cuh), deterministic
// split-K; symmetric when X is Y.
template <typename TX, typename TY, int BT, int NCG = 2>
void gram_fp64_bt(Ctx& c, int64_t a, int64_t b, int64_t r, const TX* X, int64_t ldx,
                  const TY* Y, int64_t ldy, double* C, int64_t ldc, bool sym) {
  using namespace gram;
  const int nti = (int)ceil_div(a, BT), ntj = (int)ceil_div(b, BT);
  const int tiles = sym ? nti * (nti + 1) / 2 : nti * ntj;
  const int per_sm = (Cfg<BT, NCG>::NT <= 288 && sizeof(TX) == 4) ? 2 : 1;
  // one full wave: tiles * splits <= resident CTAs (a ceil here left a
  // second wave of a few CTAs that doubled the kernel time)
  int64_t splits = std::max<int64_t>(1, ((int64_t)per_sm * c.num_sms) / tiles);
  splits = std::min<int64_t>(splits, std::max<int64_t>(1, r / (4 * BK)));
  int64_t kchunk = ceil_div(ceil_div(r, splits), BK) * BK;
  splits = ceil_div(r, kchunk);
  DBuf<double> part(c, (size_t)(splits * a * b));
  // (function attributes are per device: set on every call, ~1 us of host time)
  BRSVD_CUDA(cudaFuncSetAttribute(gram_tile_kernel<TX, TY, BT, NCG>,
                                  cudaFuncAttributeMaxDynamicSharedMemorySize,
                                  (int)Cfg<BT, NCG>::SMEM));
  gram_tile_kernel<TX, TY, BT, NCG><<<dim3(tiles, (unsigned)splits), Cfg<BT, NCG>::NT,
                                      Cfg<BT, NCG>::SMEM, c.stream>>>(r, (int)a, (int)b, X, ldx, Y, ldy, sym ? 1 : 0,
                                             ntj, kchunk, part.p);
  BRSVD_CHECK_LAUNCH();
  gram_reduce_kernel<<<grid_for(a * b), 256, 0, c.stream>>>(part.p, (int)a, (int)b,
                                                            (int)splits, sym ? 1 : 0, BT, C,
                                                            ldc);
  BRSVD_CHECK_LAUNCH();
}

// DMMA (fp64 tensor core) Gram: same tiles, split-K and fixed-order partial
// sum as gram_fp64_bt.
template <typename TX, typename TY, int BT>
void gram_dmma_bt(Ctx& c, int64_t a, int64_t b, int64_t r, const TX* X, int64_t ldx,
                  const TY* Y, int64_t ldy, double* C, int64_t ldc, bool sym) {
  using namespace gram;
  using Cf = DCfg<BT>;
  const int nti = (int)ceil_div(a, BT), ntj = (int)ceil_div(b, BT);
  const int tiles = sym ? nti * (nti + 1) / 2 : nti * ntj;
  const int per_sm = (Cf::NT <= 288 && sizeof(TX) == 4) ? 2 : 1;
  // one full wave: tiles * splits <= resident CTAs (a ceil here left a
  // second wave of a few CTAs that doubled the kernel time)
  int64_t splits = std::max<int64_t>(1, ((int64_t)per_sm * c.num_sms) / tiles);
  splits = std::min<int64_t>(splits, std::max<int64_t>(1, r / (8 * DBK)));
  int64_t kchunk = ceil_div(ceil_div(r, splits), DBK) * DBK;
  splits = ceil_div(r, kchunk);
  DBuf<double> part(c, (size_t)(splits * a * b));
  BRSVD_CUDA(cudaFuncSetAttribute(gram_dmma_kernel<TX, TY, BT>,
                                  cudaFuncAttributeMaxDynamicSharedMemorySize,
                                  (int)Cf::SMEM));
  gram_dmma_kernel<TX, TY, BT><<<dim3(tiles, (unsigned)splits), Cf::NT, Cf::SMEM,
                                 c.stream>>>(r, (int)a, (int)b, X, ldx, Y, ldy, sym ? 1 : 0,
                                             ntj, kchunk, part.p);
  BRSVD_CHECK_LAUNCH();
  gram_reduce_kernel<<<grid_for(a * b), 256, 0, c.stream>>>(part.p, (int)a, (int)b,
                                                            (int)splits, sym ? 1 : 0, BT, C,
                                                            ldc);
  BRSVD_CHECK_LAUNCH();
}

inline bool gram_simt_forced() {
  const char* e = std::getenv("BRSVD_GRAM_SIMT");
  return e && e[0] == '1';
}

// Tall-skinny fp64 Gram C (a x b) = X^T Y (gram_simt.cuh), deterministic
// split-K; symmetric when X is Y.  The tile size pads a, b least.  DMMA
// tensor-core tiles unless BRSVD_GRAM_SIMT=1.
template <typename TX, typename TY>
void gram_fp64(Ctx& c, int64_t a, int64_t b, int64_t r, const TX* X, int64_t ldx,
               const TY* Y, int64_t ldy, double* C, int64_t ldc) {
  const bool sym = (a == b) && ((const void*)X == (const void*)Y) && ldx == ldy;
  const int64_t w96 = ceil_div(a, 96) * ceil_div(b, 96) * 96 * 96;
  const int64_t w128 = ceil_div(a, 128) * ceil_div(b, 128) * 128 * 128;
  if (!gram_simt_forced()) {
    if (w96 < w128) gram_dmma_bt<TX, TY, 96>(c, a, b, r, X, ldx, Y, ldy, C, ldc, sym);
    else gram_dmma_bt<TX, TY, 128>(c, a, b, r, X, ldx, Y, ldy, C, ldc, sym);
    return;
  }
  if (w96 < w128)
    gram_fp64_bt<TX, TY, 96, (sizeof(TX) == 4 && sizeof(TY) == 4) ? 3 : 2>(c, a, b, r, X, ldx,
                                                                           Y, ldy, C, ldc, sym);
  else
    gram_fp64_bt<TX, TY, 128>(c, a, b, r, X, ldx, Y, ldy, C, ldc, sym);
}

// Column-major helpers: C = op(X)... written out for readability.
//   XtY:  C (a x b) = X(r x a)^T Y(r x b)
template <typename TX, typename TY, typename TC>
void gemm_tn_cm(Ctx& c, int64_t a, int64_t b, int64_t r, const TX* X, int64_t ldx,
                const TY* Y, int64_t ldy, TC* C, int64_t ldc) {
  if (sizeof(TC) == 8 && r >= 2048 && a >= 32 && b >= 32) {
    gram_fp64<TX, TY>(c, a, b, r, X, ldx, Y, ldy, reinterpret_cast<double*>(C), ldc);
    return;
  }
  gemm<TX, TY, double, TC>(c, a, b, r, X, ldx, 1, Y, 1, ldy, C, 1, ldc);
}
//   XT:  C (r x b) = alpha X(r x a) T(a x b) + beta C0
template <typename TX, typename TT, typename TC>
void gemm_nn_cm(Ctx& c, int64_t r, int64_t b, int64_t a, const TX* X, int64_t ldx,
                const TT* T, int64_t ldt, TC* C, int64_t ldc, double alpha = 1.0,
                double beta = 0.0, const TC* C0 = nullptr, int64_t ldc0 = 0) {
  gemm<TX, TT, double, TC>(c, r, b, a, X, 1, ldx, T, 1, ldt, C, 1, ldc, alpha,
                           beta, C0, 1, ldc0);
}

// Readback of a few device scalars (one synchronisation).
inline void readback(Ctx& c, const void* d, void* h, size_t bytes) {
  BRSVD_CUDA(cudaMemcpyAsync(c.h_pinned, d, bytes, cudaMemcpyDeviceToHost, c.stream));
  BRSVD_CUDA(cudaStreamSynchronize(c.stream));
  std::memcpy(h, c.h_pinned, bytes);
}

inline int read_int(Ctx& c, const int* d) {
  int v;
  readback(c, d, &v, sizeof(int));
  return v;
}

// ---------------------------------------------------------------------------
// Jacobi SVD launcher: G (nrow x ncol, ldg) <- G V, V (ncol x ncol) accumulated.
// tol: rotate a column pair while |x.y| > tol * ||x|| ||y||.  The dot products
// carry ~sqrt(nrow) eps of rounding, so tol_tight() is the accuracy floor; the
// Gram-based basis changes only need tol ~ 1e-8 (a Newton-Schulz step absorbs
// the rest) and the power-iteration normalisation ~ 1e-4.
inline double jacobi_tol_tight(int nrow) {
  return 8.0 * std::sqrt((double)nrow) * 2.220446049250313e-16;
}
constexpr double kJacobiTolOrth = 1e-8;
constexpr double kJacobiTolNormalize = 1e-4;

// Cluster-resident Jacobi (jacobi_cluster.cuh) for square problems that are
// too big for one CTA but fit the shared memory of an 8- or 16-CTA cluster.
// Returns false (nothing launched) when the shape or the device does not fit.
template <typename R, int NP2>
bool jacobi_cluster_launch(Ctx& c, const JacobiClusterArgs<R>& args, int csize,
                           size_t smem, int threads) {
  auto kern = jacobi_cluster_kernel<R, NP2>;
  BRSVD_CUDA(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                  (int)smem));
  if (csize > 8)
    BRSVD_CUDA(cudaFuncSetAttribute(kern, cudaFuncAttributeNonPortableClusterSizeAllowed, 1));
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3(csize);
  cfg.blockDim = dim3(threads);
  cfg.dynamicSmemBytes = smem;
  cfg.stream = c.stream;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeClusterDimension;
  attr[0].val.clusterDim.x = csize;
  attr[0].val.clusterDim.y = 1;
  attr[0].val.clusterDim.z = 1;
  cfg.attrs = attr;
  cfg.numAttrs = 1;
  int nclusters = 0;
  if (cudaOccupancyMaxActiveClusters(&nclusters, kern, &cfg) != cudaSuccess ||
      nclusters < 1) {
    cudaGetLastError();
    return false;
  }
  BRSVD_CUDA(cudaLaunchKernelEx(&cfg, kern, args));
  BRSVD_CHECK_LAUNCH();
  return true;
}

// RV: V's element type (fp64 V for the fp32 tournament: see jacobi_vreplay_kernel)
template <typename R, typename RV = R>
bool jacobi_cluster(Ctx& c, R* G, int l, int64_t ldg, RV* V, int64_t ldv, double tol,
                    double floor_rel, int max_sweeps, int* sweeps_done, double stop_cos = 0.0) {
  if (l > 512 || l < 64 || std::getenv("BRSVD_NO_CLUSTER_JACOBI")) return false;
  const size_t lim = c.max_smem_optin > 4096 ? c.max_smem_optin - 4096 : 0;
  for (int csize : {16, 8}) {
    const int bw = (int)ceil_div(l, 2 * csize);
    const size_t smem = jacobi_cluster_smem<R>(l, bw);
    if (smem > lim) continue;
    const int P = csize * bw;   // logged rotations per step
    const int64_t steps = (int64_t)max_sweeps * jc_sweep_steps(bw, 2 * csize);
    DBuf<JcRot<R>> log(c, (size_t)steps * P);
    DBuf<int> prog(c, 2);
    BRSVD_CUDA(cudaMemsetAsync(prog.p, 0, 2 * sizeof(int), c.stream));
    JacobiClusterArgs<R> a;
    a.G = G;
    a.ldg = ldg;
    a.log = log.p;
    a.prog = prog.p;
    a.l = l;
    a.bw = bw;
    a.max_sweeps = max_sweeps;
    a.tol = tol;
    a.floor_rel = floor_rel;
    a.sweeps_done = sweeps_done;
    a.stop_cos = stop_cos;
    const int threads = std::min(1024, std::max(256, 32 * bw));
    const int np2 = (int)ceil_div((l + 3) & ~3, 64);  // row pairs per lane
    bool ok;
    if (np2 <= 2) ok = jacobi_cluster_launch<R, 2>(c, a, csize, smem, threads);
    else if (np2 <= 3) ok = jacobi_cluster_launch<R, 3>(c, a, csize, smem, threads);
    else if (np2 <= 4) ok = jacobi_cluster_launch<R, 4>(c, a, csize, smem, threads);
    else if (np2 <= 5) ok = jacobi_cluster_launch<R, 5>(c, a, csize, smem, threads);
    else if (np2 <= 6) ok = jacobi_cluster_launch<R, 6>(c, a, csize, smem, threads);
    else ok = jacobi_cluster_launch<R, 8>(c, a, csize, smem, threads);
    if (ok) {
      // V <- V * the logged rotations, one CTA per row
      // V <- V * the logged rotations: launched programmatically dependent
      // on the tournament, so it streams the log while the tournament runs
      const int rpw = 32 / bw;
      // shared memory sized so a replay CTA never shares an SM with a
      // tournament CTA (the latency-bound tournament would lose issue slots)
      const size_t rs = std::max(jacobi_vreplay_smem(l, bw, csize, sizeof(RV), sizeof(R)),
                                 std::min(lim, (size_t)c.max_smem_optin + 1024 - smem));
      auto rk = jacobi_vreplay_kernel<R, RV>;
      BRSVD_CUDA(cudaFuncSetAttribute(rk, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)rs));
      cudaLaunchConfig_t rc = {};
      rc.gridDim = dim3((unsigned)ceil_div(l, rpw));
      rc.blockDim = dim3(32 * csize);
      rc.dynamicSmemBytes = rs;
      rc.stream = c.stream;
      cudaLaunchAttribute ra[1];
      ra[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
      // BRSVD_NO_PDL=1: plain stream order (the replay after the tournament)
      ra[0].val.programmaticStreamSerializationAllowed = std::getenv("BRSVD_NO_PDL") ? 0 : 1;
      rc.attrs = ra;
      rc.numAttrs = 1;
      const JcRot<R>* lp = log.p;
      const int* pp = prog.p;
      BRSVD_CUDA(cudaLaunchKernelEx(&rc, rk, V, ldv, l, bw, csize, lp, pp));
      BRSVD_CHECK_LAUNCH();
      return true;
    }
  }
  return false;
}

// floor_rel < 0: the default null-column floor 16 nrow eps(R).  The fp32 phase
// of the two-phase small SVD passes a lower one so that small but resolvable
// columns (noise-level singular values of fp32 data) converge already in fp32.
template <typename R = double>
inline int jacobi(Ctx& c, R* G, int nrow, int ncol, int64_t ldg, R* V, int64_t ldv,
                  double tol, int max_sweeps = 40, double floor_rel = -1.0,
                  double stop_cos = 0.0) {
  BRSVD_REQUIRE(ncol >= 1 && ncol <= 1024 && nrow >= 1, kErrShape,
                "jacobi: unsupported small-problem shape");
  const double eps_r0 = sizeof(R) == 8 ? 2.220446049250313e-16 : 1.1920928955078125e-07;
  const double tol_eff = std::max(tol, 8.0 * std::sqrt((double)nrow) * eps_r0);
  const double floor_eff = floor_rel >= 0.0 ? floor_rel : 16.0 * nrow * eps_r0;
  if (nrow == ncol) {
    DBuf<int> sw(c, 1);
    if (jacobi_cluster<R>(c, G, nrow, ldg, V, ldv, tol_eff, floor_eff, max_sweeps, sw.p,
                          stop_cos)) {
      if (std::getenv("BRSVD_DEBUG")) {
        const int nsw = read_int(c, sw.p);
        std::fprintf(stderr, "[brsvd] jacobi(cluster) %dx%d tol %.1e: %d sweeps\n", nrow,
                     ncol, tol_eff, nsw);
        if (std::getenv("BRSVD_JC_TIMING")) {
          long long t[4];
          BRSVD_CUDA(cudaMemcpyFromSymbol(t, g_jc_t, sizeof(t)));
          std::fprintf(stderr,
                       "[brsvd]   cycles: rotations %lld  cluster barriers %lld  pulls %lld"
                       "  (%lld rounds)\n", t[0], t[1], t[2], t[3]);
          float c2[64];
          BRSVD_CUDA(cudaMemcpyFromSymbol(c2, g_jc_c2, sizeof(c2)));
          for (int s = 0; s < nsw && s < 64; ++s)
            std::fprintf(stderr, "[brsvd]   sweep %d: max |cos| %.3e\n", s, std::sqrt((double)c2[s]));
        }
      }
      return 0;
    }
  }
  const size_t budget = std::min<size_t>(c.max_smem_optin, 200 * 1024);
  const size_t per_col = (size_t)(nrow + ncol) * sizeof(R) + sizeof(int);
  int bw_fit = (int)(budget / (2 * per_col));
  BRSVD_REQUIRE(bw_fit >= 1, kErrShape, "jacobi: column too long for shared memory");
  int bw = (ncol + 1) / 2;
  bool single = true;
  if (bw > bw_fit) {
    bw = std::min(bw_fit, 32);
    single = false;
  }
  int nb = (int)ceil_div(ncol, bw);
  if (nb < 2) nb = 2;
  if (nb & 1) ++nb;
  if (nb == 2) single = true;
  const int threads = std::min(1024, std::max(64, bw * 32));
  const size_t smem = (size_t)2 * bw * per_col;
  BRSVD_CUDA(cudaFuncSetAttribute(jacobi_block_kernel<R>,
                                  cudaFuncAttributeMaxDynamicSharedMemorySize, (int)budget));
  DBuf<int> counters(c, (size_t)max_sweeps + 1);
  BRSVD_CUDA(cudaMemsetAsync(counters.p, 0, sizeof(int) * (max_sweeps + 1), c.stream));
  JacobiArgs<R> args;
  args.G = G;
  args.ldg = ldg;
  args.nrow = nrow;
  args.ncol = ncol;
  args.V = V;
  args.ldv = ldv;
  args.bw = bw;
  args.nb = nb;
  args.max_sweeps = max_sweeps;
  args.tol = tol_eff;
  args.floor_rel = floor_eff;
  args.rot_count = counters.p;
  args.sweeps_done = counters.p + max_sweeps;
  if (single) {
    jacobi_block_kernel<R><<<1, threads, smem, c.stream>>>(args);
    BRSVD_CHECK_LAUNCH();
  } else {
    int grid = nb / 2;
    int per_sm = 0;
    BRSVD_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(
        &per_sm, jacobi_block_kernel<R>, threads, smem));
    grid = std::min(grid, std::max(1, per_sm) * c.num_sms);
    void* kargs[] = {&args};
    BRSVD_CUDA(cudaLaunchCooperativeKernel((void*)jacobi_block_kernel<R>, dim3(grid),
                                           dim3(threads), kargs, smem, c.stream));
    ++g_brsvd_launches;
  }
  if (std::getenv("BRSVD_DEBUG")) {
    int sw = 0;
    readback(c, counters.p + max_sweeps, &sw, sizeof(int));
    std::fprintf(stderr, "[brsvd] jacobi %dx%d tol %.1e: %d sweeps (nb %d, bw %d)\n", nrow,
                 ncol, args.tol, sw, nb, bw);
  }
  return nb;
}

inline void jacobi_finish(Ctx& c, const double* G, int nrow, int ncol, int64_t ldg,
                          const double* V, int64_t ldv, double* sv, double* Uout,
                          int64_t ldu, double* Vout, int64_t ldvo) {
  const size_t smem = (size_t)ncol * (sizeof(double) + sizeof(int));
  const int ctas = std::max(1, std::min(c.num_sms / 4, ncol / 32));
  jacobi_finish_kernel<<<ctas, 1024, smem, c.stream>>>(G, ldg, nrow, ncol, V, ldv, sv, Uout,
                                                       ldu, Vout, ldvo);
  BRSVD_CHECK_LAUNCH();
}

// ---------------------------------------------------------------------------
// Eigen-decomposition of the (optionally column-scaled) Gram of X (r x l):
//   s_j = 1/||x_j|| (or 1),  (S X^T X S) = E diag(lam) E^T  (lam sorted desc)
// trace (device, optional) receives ||X||_F^2.
template <typename T>
void gram_eig(Ctx& c, const T* X, int64_t r, int l, int64_t ldx, double* E,
              double* lam, double* s, double tol, bool scale = true,
              double* trace = nullptr, double drop = 0.0) {
  DBuf<double> G(c, (size_t)l * l), V(c, (size_t)l * l);
  gemm_tn_cm<T, T, double>(c, l, l, r, X, ldx, X, ldx, G.p, l);
  gram_prep_kernel<<<1, 1024, 0, c.stream>>>(G.p, l, s, V.p, scale ? 1 : 0, trace,
                                             drop);
  BRSVD_CHECK_LAUNCH();
  jacobi(c, G.p, l, l, l, V.p, l, tol);
  jacobi_finish(c, G.p, l, l, l, V.p, l, lam, nullptr, 0, E, l);
}

inline double orth_tau(int64_t r, int l) {
  return 8.0 * (double)std::max<int64_t>(r, l) * 2.220446049250313e-16;
}

template <typename T>
void fix_signs(Ctx& c, T* U, int64_t m, int l, int64_t ldu, T* V, int64_t n,
               int64_t ldv) {
  DBuf<T> sign(c, l);
  colsign_kernel<T><<<l, 256, 0, c.stream>>>(U, m, ldu, sign.p);
  BRSVD_CHECK_LAUNCH();
  scale_cols_kernel<T><<<grid_for(m * l), 256, 0, c.stream>>>(U, m, l, ldu, sign.p);
  BRSVD_CHECK_LAUNCH();
  scale_cols_kernel<T><<<grid_for(n * l), 256, 0, c.stream>>>(V, n, l, ldv, sign.p);
  BRSVD_CHECK_LAUNCH();
}

struct MaxAbs {
  double peak;
  bool nonfinite;
};

template <typename T>
MaxAbs maxabs(Ctx& c, const T* X, int64_t rows, int64_t cols, int64_t ld) {
  DBuf<unsigned long long> out(c, 2);
  BRSVD_CUDA(cudaMemsetAsync(out.p, 0, 2 * sizeof(unsigned long long), c.stream));
  maxabs_kernel<T><<<grid_for(rows * cols), 256, 0, c.stream>>>(X, rows, cols, ld,
                                                                 out.p);
  BRSVD_CHECK_LAUNCH();
  BRSVD_CUDA(cudaMemcpyAsync(c.h_pinned, out.p, 2 * sizeof(unsigned long long),
                             cudaMemcpyDeviceToHost, c.stream));
  BRSVD_CUDA(cudaStreamSynchronize(c.stream));
  MaxAbs r;
  long long bits = (long long)c.h_pinned[0];
  std::memcpy(&r.peak, &bits, sizeof(double));
  r.nonfinite = c.h_pinned[1] != 0;
  return r;
}

}  // namespace brsvd
