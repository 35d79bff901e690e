// Small dense Cholesky factorisation and triangular inverse (fp64, one CTA).
//
// These turn a Gram matrix G = X^T X into the basis change T = L^-T that
// makes X T orthonormal (Cholesky QR).  They replace, on the fast path, the
// Householder QR of tsqr (kernels.py:121-164) and the Gram eigen-solves of the
// Jacobi route, whose sequential depth is O(sweeps * l) against O(l / NB) here.
#pragma once
#include <algorithm>
#include <cstdio>
#include <cstdlib>
#include <type_traits>
#include <cooperative_groups.h>
#include "common.cuh"

namespace brsvd {

constexpr int kCholNB = 32;

// Tc[:, c] = T[:, keep[c]] for the kept columns (count from info[2]); with
// zero_rest the columns k .. l-1 of Tc are zeroed (device-driven callers that
// apply all l columns without reading k on the host).
__global__ void compact_cols_kernel(const double* __restrict__ T, int l,
                                    const int* __restrict__ keep,
                                    const double* __restrict__ info, double* __restrict__ Tc,
                                    int zero_rest = 0) {
  const int k = (int)info[2];
  const int nc = zero_rest ? l : k;
  for (int e = blockIdx.x * blockDim.x + threadIdx.x; e < l * nc; e += gridDim.x * blockDim.x) {
    const int i = e % l, c = e / l;
    Tc[(int64_t)c * l + i] = c < k ? T[(int64_t)keep[c] * l + i] : 0.0;
  }
}

// rank = min(reference rank cut, kept count) of a Cholesky pass, on the device
__global__ void chol_rank_kernel(const double* __restrict__ info, int* __restrict__ rank) {
  rank[0] = min((int)info[1], (int)info[2]);
}

// ---------------------------------------------------------------------------
// Fused Cholesky basis change on one thread-block cluster: from a Gram matrix
// G = X^T X (n x n, lower triangle read) to T = S L^-T, where
//   s_j = 1/sqrt(G_jj) (column scaling; 0 for columns below col_drop of the
//   largest), S G S + shift I = L L^T.
// One launch (it replaced three single-CTA kernels -- Gram scaling, Cholesky,
// triangular inverse -- whose inner loops were latency-bound):
//   * blocked right-looking factorisation with 32-column panels.  Every CTA of
//     the cluster redundantly factors the 32 x 32 diagonal block (one warp,
//     rows in registers, column values broadcast by shuffles), inverts it (a
//     column per lane) and solves the panel below against that inverse; the
//     trailing SYRK update of the L2-resident matrix is split over the CTAs
//     (4 x 4 register tiles fed by 16-byte shared loads of a k-major panel);
//   * the inverse by block rows, X_IJ = -L_II^-1 sum_K L_IK X_KJ, columns
//     split over the CTAs, with the diagonal-block inverses from the panels;
//   * one cluster barrier per panel / block row orders the global updates.
// Pivot drop: a column whose pivot falls below drop_ratio of its diagonal
// lies numerically in the span of the earlier ones; its L column is e_c (L
// stays invertible) and it is left out of `keep`.  info[0] = min pivot /
// diagonal, info[1] = #{j : |R_jj| > rank_tol ||X||_F} (the reference's rank
// cut, kernels.py:155-157), info[2] = kept count.
constexpr int kCiNB = 32;
constexpr int kCiLd = 33;       // padded row stride of the shared panel
constexpr int kCiThreads = 512;
constexpr int kCiMaxBlk = 10;   // block rows of the largest order (kCholMaxL = 320)
__device__ long long g_ci_t[64];
#define CI_T(k) do { if (me == 0 && tid == 0) g_ci_t[(k)] = clock64(); } while (0)

__host__ __device__ inline int cholinv_ldp(int n) { return (n + 3) & ~3; }
// offset of the k-major L21 copy PT after the n x 33 panel: even, so that its
// 16-byte (double2) reads stay aligned for odd n
__host__ __device__ inline size_t cholinv_pt_off(int n) { return ((size_t)n * kCiLd + 1) & ~size_t(1); }
// Columns of each block column of X = L^-1 owned by one CTA in phase 2 (the
// launch uses an 8-CTA cluster for n > 96, one CTA otherwise).
__host__ __device__ inline int cholinv_cpc(int n) { return n > 96 ? kCiNB / 8 : kCiNB; }
__host__ __device__ inline size_t cholinv_big(int n) {
  const size_t p1 = cholinv_pt_off(n) + (size_t)kCiNB * cholinv_ldp(n);  // phase 1 panels
  const size_t nblk = (size_t)(n + kCiNB - 1) / kCiNB;
  const size_t ldxm = nblk * cholinv_cpc(n);
  const size_t xm = nblk * kCiNB * ldxm;
  // phase 2: Dinv blocks, X columns (also the staging area of the diagonal
  // blocks), one staged L block, the block-row sums
  const size_t p2 = nblk * kCiNB * kCiLd + (xm > nblk * kCiNB * kCiLd ? xm : nblk * kCiNB * kCiLd) +
                    (size_t)kCiNB * kCiNB + kCiNB * ldxm;
  return p1 > p2 ? p1 : p2;
}
inline size_t cholinv_smem(int n) {
  return (cholinv_big(n) + (size_t)kCiNB * kCiLd + 4 * (size_t)n + 130) * sizeof(double) +
         (size_t)n * sizeof(int);
}

__global__ void __launch_bounds__(kCiThreads, 1)
    cholinv_kernel(double* __restrict__ A, int n, int64_t ld, int scale, double col_drop,
                   double shift, double drop_ratio, double rank_tol,
                   double* __restrict__ X, double* __restrict__ T,
                   double* __restrict__ s_out, double* __restrict__ info,
                   int* __restrict__ keep) {
  namespace cg = cooperative_groups;
  cg::cluster_group cluster = cg::this_cluster();
  extern __shared__ __align__(16) double cism[];
  const size_t big = cholinv_big(n);
  const int ldp = cholinv_ldp(n);
  double* Lp = cism;                      // phase 1: panel, row-major rows x 33
  double* PT = cism + cholinv_pt_off(n);  // phase 1: L21 k-major, 32 x ldp
  double* Di = cism + big;                // 32 x 33: inverse of the diagonal block
  double* sc = Di + kCiNB * kCiLd;        // column scaling
  double* d0 = sc + n;                    // scaled diagonal + shift
  double* dL = d0 + n;                    // diagonal of L
  double* Rat = dL + n;                   // pivots (for info[0] = min pivot / diagonal)
  // column broadcast of the diagonal factor (128, 16-byte aligned)
  double* bcst = Rat + n + ((reinterpret_cast<uintptr_t>(Rat + n) & 15) ? 1 : 0);
  int* dropped = reinterpret_cast<int*>(Rat + n + 130);
  __shared__ double s_red[32];
  const int tid = threadIdx.x, nt = blockDim.x;
  const int lane = tid & 31, warp = tid >> 5, nw = nt >> 5;
  const int me = (int)cluster.block_rank(), C = (int)cluster.num_blocks();
  const int gw = me * nw + warp, gnw = C * nw;     // cluster-wide warp index
  const bool leader = (me == 0);

  CI_T(0);
  // ---- phase 0: scaling (redundant per CTA; the matrix write is split) ----
  double dm = 0.0;
  for (int j = tid; j < n; j += nt) dm = fmax(dm, A[(int64_t)j * ld + j]);
  dm = warp_max(dm);
  if (lane == 0) s_red[warp] = dm;
  __syncthreads();
  if (tid == 0) {
    double m = 0.0;
    for (int w = 0; w < nw; ++w) m = fmax(m, s_red[w]);
    s_red[0] = m;
  }
  __syncthreads();
  const double fl2 = col_drop * col_drop * s_red[0];
  for (int j = tid; j < n; j += nt) {
    const double d = A[(int64_t)j * ld + j];
    const double s = scale ? ((d > fl2 && d > 0.0) ? 1.0 / sqrt(d) : 0.0) : 1.0;
    sc[j] = s;
    d0[j] = s * s * d + shift;
    if (s_out && leader) s_out[j] = s;
  }
  cluster.sync();  // every CTA has read the unscaled diagonal
  for (int j = gw; j < n; j += gnw) {
    const double sj = sc[j];
    double* col = A + (int64_t)j * ld;
    for (int i = j + lane; i < n; i += 32) col[i] = (i == j) ? d0[j] : col[i] * sc[i] * sj;
  }
  cluster.sync();

  CI_T(1);
  // ---- phase 1: blocked right-looking factorisation --------------------
  for (int p0 = 0; p0 < n; p0 += kCiNB) {
    const int pi = p0 / kCiNB;
    const int nb = min(kCiNB, n - p0), rows = n - p0;
    {
      // batched loads (8 in flight per thread) before the shared stores
      constexpr int U = 8;
      const int tot = rows * nb;
      for (int e0 = tid; e0 < tot; e0 += U * nt) {
        double v[U];
#pragma unroll
        for (int u = 0; u < U; ++u) {
          const int e = e0 + u * nt;
          const int i = e % rows, c = e / rows;
          v[u] = (e < tot && i >= c) ? A[(int64_t)(p0 + c) * ld + (p0 + i)] : 0.0;
        }
#pragma unroll
        for (int u = 0; u < U; ++u) {
          const int e = e0 + u * nt;
          if (e < tot) Lp[(e % rows) * kCiLd + e / rows] = v[u];
        }
      }
    }
    __syncthreads();
    if (pi == 0) CI_T(2);
    // factor the diagonal block in ONE warp, rows in registers: lane i holds
    // row i of the block, shifted so that the current column is always a[0]
    // (the column loop is not unrolled: straight-line code for 32 columns does
    // not fit the instruction cache).  Per column the pivot comes from lane c
    // by a shuffle, rsqrt (no divisions -- piv/dg is only recorded for
    // info[0]), and the rank-1 update reads the scaled column back from a
    // shared broadcast buffer: lane i stores l_i at slot 32 + i - c - 1 (and a
    // zero 32 slots further, so slots past the block read 0), every lane then
    // loads slots 32..63 with 16-byte broadcast loads -- 16 loads per column
    // instead of 64 fp64 shuffle halves; no block barriers.
    double* rinv = Di + kCiNB * kCiLd - kCiNB;   // 1 / L11[c][c] for the TRSM
    if (warp == 0) {
      const int i = lane;
      double a[kCiNB];
#pragma unroll
      for (int jj = 0; jj < kCiNB; ++jj)
        a[jj] = (i < nb && jj <= i) ? Lp[i * kCiLd + jj] : 0.0;
      const double2* b2 = reinterpret_cast<const double2*>(bcst + 32);
      // one column; J = live row length bound for this column (32 - 8 g in
      // phase g, columns 8 g .. 8 g + 7): entries a[J..] are zero and stay
      // zero, so the rank-1 update and the broadcast loads stop at J
      auto column = [&](auto Jc, int c) {
        constexpr int J = decltype(Jc)::value;
        const double piv = __shfl_sync(0xffffffffu, a[0], c);
        const double dg = d0[p0 + c];
        const bool drop = !(piv > 0.0) ||
                          (drop_ratio > 0.0 && (!(dg > 0.0) || !(piv > drop_ratio * dg)));
        const double inv = drop ? 0.0 : rsqrt(piv);
        const double lc = (i > c && i < nb) ? a[0] * inv : 0.0;
        __syncwarp();   // the previous column's broadcast loads are done
        bcst[32 + i - c - 1] = lc;
        bcst[64 + i - c - 1] = 0.0;
        __syncwarp();
        if (i == c) {
          const double dsq = piv * inv;
          Lp[c * kCiLd + c] = drop ? 1.0 : dsq;
          rinv[c] = drop ? 1.0 : inv;
          dropped[p0 + c] = drop ? 1 : 0;
          dL[p0 + c] = drop ? 0.0 : dsq;
          Rat[p0 + c] = piv;
        } else if (i < nb) {
          Lp[i * kCiLd + c] = lc;   // 0 above the diagonal
        }
        // lanes i <= c hold lc = 0, so a[jj] of lanes i < c + jj only ever
        // gets lc_i * lc_j with one factor zero or is unused
        double2 lj[J / 2];
#pragma unroll
        for (int q = 0; q < J / 2; ++q) lj[q] = b2[q];
#pragma unroll
        for (int q = 0; q < J / 2; ++q) {
          const int jj = 2 * q + 1;
          a[jj - 1] = fma(-lc, lj[q].x, a[jj]);
          if (jj + 1 < J) a[jj] = fma(-lc, lj[q].y, a[jj + 1]);
        }
        a[J - 1] = 0.0;
      };
#pragma unroll 1
      for (int c = 0; c < min(nb, 8); ++c) column(std::integral_constant<int, 32>{}, c);
#pragma unroll 1
      for (int c = 8; c < min(nb, 16); ++c) column(std::integral_constant<int, 24>{}, c);
#pragma unroll 1
      for (int c = 16; c < min(nb, 24); ++c) column(std::integral_constant<int, 16>{}, c);
#pragma unroll 1
      for (int c = 24; c < nb; ++c) column(std::integral_constant<int, 8>{}, c);
    }
    __syncthreads();
    if (pi == 0) CI_T(3);
    // TRSM: L21 = A21 L11^-T (rows nb..rows-1) by forward substitution, one
    // thread per row with the row in registers (L11 rows broadcast from
    // shared memory), into the k-major copy PT (zero-padded to a multiple of 4
    // rows).  Dropped columns are zero (their L11 column is e_c).
    const int rpad = (rows + 3) & ~3;
    {
      for (int i = nb + tid; i < rpad; i += nt) {
        double x[kCiNB];
#pragma unroll
        for (int c = 0; c < kCiNB; ++c) x[c] = (i < rows && c < nb) ? Lp[i * kCiLd + c] : 0.0;
#pragma unroll
        for (int c = 0; c < kCiNB; ++c) {
          if (c < nb) {
            const double* lc = Lp + c * kCiLd;
            double v = x[c];
#pragma unroll
            for (int k = 0; k < c; ++k) v = fma(-x[k], lc[k], v);
            x[c] = dropped[p0 + c] ? 0.0 : v * rinv[c];
          }
        }
#pragma unroll
        for (int c = 0; c < kCiNB; ++c)
          if (c < nb) PT[c * ldp + i] = i < rows ? x[c] : 0.0;
      }
    }
    __syncthreads();
    // write the panel (L) back, its columns split over the cluster (every
    // CTA holds the same panel; the leader alone writing it held up the
    // cluster barrier below)
    for (int c = me; c < nb; c += C) {
      double* dst = A + (int64_t)(p0 + c) * ld + p0;
      for (int i = c + tid; i < rows; i += nt) dst[i] = i < nb ? Lp[i * kCiLd + c] : PT[c * ldp + i];
    }
    if (pi == 0) CI_T(4);
    // trailing update: A22 -= L21 L21^T (lower), 4x4 register tiles, split
    // over the cluster
    const int R2 = rows - nb;
    if (R2 > 0) {
      // one warp per super-tile of 8 (i) x 4 (j) tiles, lane = 4 ty + tx, so
      // the 16-byte PT reads of a warp touch 8 / 4 distinct addresses
      // (2 / 1 wavefronts) instead of 32; super-tiles on or below the
      // diagonal, row si holding min(nsj, 2 si + 2) of them
      const int nti = (R2 + 3) / 4;
      const int nsi = (nti + 7) / 8, nsj = (nti + 3) / 4;
      int nst = 0;
      for (int si = 0; si < nsi; ++si) nst += min(nsj, 2 * si + 2);
      for (int st = gw; st < nst; st += gnw) {
        int si = 0, rem = st;
        while (rem >= min(nsj, 2 * si + 2)) {
          rem -= min(nsj, 2 * si + 2);
          ++si;
        }
        const int ti = si * 8 + (lane >> 2), tj = rem * 4 + (lane & 3);
        if (ti >= nti || tj > ti) continue;
        const int i0 = nb + 4 * ti, j0 = nb + 4 * tj;
        double acc[4][4];
#pragma unroll
        for (int a = 0; a < 4; ++a)
#pragma unroll
          for (int b = 0; b < 4; ++b) acc[a][b] = 0.0;
        double old[4][4];
#pragma unroll
        for (int b = 0; b < 4; ++b)
#pragma unroll
          for (int a = 0; a < 4; ++a) {
            const int gi = i0 + a, gj = j0 + b;
            old[a][b] = (gi < rows && gj < rows && gi >= gj)
                            ? A[(int64_t)(p0 + gj) * ld + (p0 + gi)] : 0.0;
          }
#pragma unroll 4
        for (int k = 0; k < nb; ++k) {
          const double2* pa = reinterpret_cast<const double2*>(PT + k * ldp + i0);
          const double2* pb = reinterpret_cast<const double2*>(PT + k * ldp + j0);
          const double2 a01 = pa[0], a23 = pa[1], b01 = pb[0], b23 = pb[1];
          const double av[4] = {a01.x, a01.y, a23.x, a23.y};
          const double bv[4] = {b01.x, b01.y, b23.x, b23.y};
#pragma unroll
          for (int a = 0; a < 4; ++a)
#pragma unroll
            for (int b = 0; b < 4; ++b) acc[a][b] = fma(av[a], bv[b], acc[a][b]);
        }
#pragma unroll
        for (int b = 0; b < 4; ++b) {
          const int gj = j0 + b;
          if (gj >= rows) continue;
#pragma unroll
          for (int a = 0; a < 4; ++a) {
            const int gi = i0 + a;
            if (gi >= rows || gi < gj) continue;
            A[(int64_t)(p0 + gj) * ld + (p0 + gi)] = old[a][b] - acc[a][b];
          }
        }
      }
    }
    if (pi == 0) CI_T(5);
    cluster.sync();
  }

  CI_T(6);
  // ---- phase 2: T = S L^-T from X = L^-1, columns split over the cluster --
  // Every block column J of X obeys X_JJ = L_JJ^-1 and, for I > J,
  // X_IJ = -L_II^-1 sum_{K=J..I-1} L_IK X_KJ, and the columns of X are
  // independent: CTA me owns columns me*cpc .. me*cpc+cpc-1 of EVERY block
  // column (cpc = 32 / cluster size), so the work is balanced and the chain
  // is one block row per step.  Every CTA inverts the diagonal blocks (one
  // warp each), then walks the block rows I = 1..: the sums over K are
  // accumulated with 2 x 2 register tiles against L_IK staged k-major in
  // shared memory, then multiplied by -L_II^-1.  Rows k of T (k one of this
  // CTA's columns) are written directly: T[k][j] = s_k X[j][k]; no cluster
  // barrier.
  const int nblk = (n + kCiNB - 1) / kCiNB;
  const int cpc = kCiNB / C;                             // == cholinv_cpc(n)
  const int ldxm = nblk * cpc;                           // this CTA's columns
  constexpr int BB = kCiNB * kCiLd;                      // one 32 x 33 block
  double* Dinv = cism;                                   // nblk blocks: L_II^-1
  double* XM = cism + (size_t)nblk * BB;                 // X rows x this CTA's columns
  const size_t xm_sz = (size_t)nblk * kCiNB * ldxm;
  double* Lt = XM + (xm_sz > (size_t)nblk * BB ? xm_sz : (size_t)nblk * BB);  // L_IK, k-major
  double* Rb = Lt + kCiNB * kCiNB;                       // 32 x ldxm block-row sums
  // diagonal blocks of L -> XM (scratch), inverted by one warp each into Dinv
  double* Xs = XM;
  for (int e = tid; e < nblk * kCiNB * kCiNB; e += nt) {
    const int bI = e / (kCiNB * kCiNB), rc = e % (kCiNB * kCiNB);
    const int r = rc % kCiNB, cc = rc / kCiNB, i0 = bI * kCiNB;
    const bool ok = i0 + r < n && i0 + cc < n && r >= cc;
    Xs[(size_t)bI * BB + r * kCiLd + cc] = ok ? A[(int64_t)(i0 + cc) * ld + (i0 + r)] : 0.0;
  }
  __syncthreads();
  // Each diagonal block inverted by one warp, right-looking: lane c owns
  // column c of X = L_II^-1 and the pending sums acc[j] of rows k + j (the
  // array shifts by one row per step, so the loop body is compact);
  // X[k][c] = (delta_kc - acc) / L[k][k] with the reciprocals formed up
  // front by all lanes, then acc[j] += L[k+j][k] X[k][c] (broadcast reads).
  // The dependent chain per row is one multiply and one FMA.
  for (int bI = warp; bI < nblk; bI += nw) {
    const int nbI = min(kCiNB, n - bI * kCiNB);
    const double* Lb = Xs + (size_t)bI * BB;
    double* Dv = Dinv + (size_t)bI * BB;
    const int c = lane;
    const double dgl = Lb[c * kCiLd + c];
    const double rl = (c < nbI && dgl != 0.0) ? 1.0 / dgl : 0.0;
    double acc[kCiNB];
#pragma unroll
    for (int j = 0; j < kCiNB; ++j) acc[j] = 0.0;
#pragma unroll 1
    for (int k = 0; k < kCiNB; ++k) {
      const double rk = __shfl_sync(0xffffffffu, rl, k);
      const double x = ((k == c ? 1.0 : 0.0) - acc[0]) * rk;
      Dv[k * kCiLd + c] = x;
#pragma unroll
      for (int j = 1; j < kCiNB; ++j) {
        const double l = (k + j < kCiNB) ? Lb[(k + j) * kCiLd + k] : 0.0;
        acc[j] = fma(l, x, acc[j]);
      }
#pragma unroll
      for (int j = 0; j < kCiNB - 1; ++j) acc[j] = acc[j + 1];
      acc[kCiNB - 1] = 0.0;
    }
  }
  __syncthreads();
  CI_T(9);
  // block row 0: X_00 restricted to this CTA's columns
  for (int e = tid; e < kCiNB * cpc; e += nt) {
    const int r = e / cpc, u = e % cpc;
    XM[r * ldxm + u] = Dinv[r * kCiLd + me * cpc + u];
  }
  for (int bI = 1; bI < nblk; ++bI) {
    const int i0 = bI * kCiNB, nbI = min(kCiNB, n - i0);
    const int na = bI * cpc;            // active columns: blocks J < I
    // work item: rows 2 rp, 2 rp + 1 and local columns 2 cp, 2 cp + 1 (same J)
    const int rp = tid & 15, cp = tid >> 4;
    const bool act = 2 * cp < na;
    const int jcol = act ? (2 * cp) / cpc : 0;
    double acc[2][2] = {{0.0, 0.0}, {0.0, 0.0}};
    // the whole block row L_I,0..I-1 is loaded into registers up front (one
    // global latency per block row instead of one per block)
    double pre[kCiMaxBlk][2];
#pragma unroll
    for (int bK = 0; bK < kCiMaxBlk; ++bK)
#pragma unroll
      for (int q = 0; q < 2; ++q) {
        const int e = tid + q * nt;
        const int r = e % kCiNB, kk = e / kCiNB;
        pre[bK][q] = (bK < bI && r < nbI) ? A[(int64_t)(bK * kCiNB + kk) * ld + (i0 + r)] : 0.0;
      }
#pragma unroll
    for (int bK = 0; bK < kCiMaxBlk; ++bK) {
      if (bK >= bI) break;
      __syncthreads();   // previous Lt consumed (and XM rows of block bK written)
#pragma unroll
      for (int q = 0; q < 2; ++q) Lt[tid + q * nt] = pre[bK][q];   // Lt[kk][r]
      __syncthreads();
      if (act && jcol <= bK) {
        const double* xr = XM + (size_t)bK * kCiNB * ldxm + 2 * cp;
#pragma unroll 8
        for (int kk = 0; kk < kCiNB; ++kk) {
          const double2 lv = *reinterpret_cast<const double2*>(Lt + kk * kCiNB + 2 * rp);
          const double2 xv = *reinterpret_cast<const double2*>(xr + (size_t)kk * ldxm);
          acc[0][0] = fma(lv.x, xv.x, acc[0][0]);
          acc[0][1] = fma(lv.x, xv.y, acc[0][1]);
          acc[1][0] = fma(lv.y, xv.x, acc[1][0]);
          acc[1][1] = fma(lv.y, xv.y, acc[1][1]);
        }
      }
    }
    if (act) {
      *reinterpret_cast<double2*>(Rb + (2 * rp) * ldxm + 2 * cp) = make_double2(acc[0][0], acc[0][1]);
      *reinterpret_cast<double2*>(Rb + (2 * rp + 1) * ldxm + 2 * cp) =
          make_double2(acc[1][0], acc[1][1]);
    }
    __syncthreads();
    // X_IJ = -L_II^-1 Rb (J < I); X_II = L_II^-1 restricted to our columns
    const double* Dv = Dinv + (size_t)bI * BB;
    double* xo = XM + (size_t)i0 * ldxm;
    for (int e = tid; e < kCiNB * na; e += nt) {
      const int r = e % kCiNB, cc = e / kCiNB;
      double v = 0.0;   // Dv is zero above the diagonal: fixed trip count
#pragma unroll 8
      for (int j = 0; j < kCiNB; ++j) v = fma(Dv[r * kCiLd + j], Rb[j * ldxm + cc], v);
      xo[r * ldxm + cc] = -v;
    }
    for (int e = tid; e < kCiNB * cpc; e += nt) {
      const int r = e / cpc, u = e % cpc;
      xo[r * ldxm + na + u] = Dv[r * kCiLd + me * cpc + u];
    }
  }
  __syncthreads();
  CI_T(10);
  // rows k of T for this CTA's columns k: T[k][j] = s_k X[j][k] for j >= k, 0
  // below the diagonal; zero the strict upper triangle of A (L) in these
  // columns
  for (int e = tid; e < ldxm * n; e += nt) {
    const int lc = e % ldxm, j = e / ldxm;
    const int k = (lc / cpc) * kCiNB + me * cpc + lc % cpc;
    if (k >= n) continue;
    T[(int64_t)j * n + k] = j >= k ? sc[k] * XM[(size_t)j * ldxm + lc] : 0.0;
  }
  for (int e = tid; e < ldxm * n; e += nt) {
    const int lc = e / n, i = e % n;
    const int k = (lc / cpc) * kCiNB + me * cpc + lc % cpc;
    if (k < n && i < k) A[(int64_t)k * ld + i] = 0.0;
  }
  __syncthreads();
  CI_T(7);
  if (leader && info) {
    // info[0] = min pivot / diagonal, info[1] = reference rank, info[2] =
    // kept count (block reductions); keep[] in column order (thread 0)
    __shared__ double r_min[32], r_fro[32];
    __shared__ int r_kept[32];
    double mn = 1.0, fro2 = 0.0;
    int kc = 0;
    for (int j = tid; j < n; j += nt) {
      const double rt = (d0[j] > 0.0 && Rat[j] == Rat[j]) ? Rat[j] / d0[j] : -1.0;
      mn = fmin(mn, rt);
      if (sc[j] > 0.0) fro2 += 1.0 / (sc[j] * sc[j]);
      kc += dropped[j] ? 0 : 1;
    }
    for (int o = 16; o > 0; o >>= 1) {
      mn = fmin(mn, __shfl_xor_sync(0xffffffffu, mn, o));
      fro2 += __shfl_xor_sync(0xffffffffu, fro2, o);
      kc += __shfl_xor_sync(0xffffffffu, kc, o);
    }
    if (lane == 0) {
      r_min[warp] = mn;
      r_fro[warp] = fro2;
      r_kept[warp] = kc;
    }
    __syncthreads();
    if (warp == 0) {
      mn = lane < nw ? r_min[lane] : 1.0;
      fro2 = lane < nw ? r_fro[lane] : 0.0;
      kc = lane < nw ? r_kept[lane] : 0;
      for (int o = 16; o > 0; o >>= 1) {
        mn = fmin(mn, __shfl_xor_sync(0xffffffffu, mn, o));
        fro2 += __shfl_xor_sync(0xffffffffu, fro2, o);
        kc += __shfl_xor_sync(0xffffffffu, kc, o);
      }
      if (lane == 0) {
        r_min[0] = mn;
        r_fro[0] = fro2;
        r_kept[0] = kc;
      }
    }
    __syncthreads();
    const double cut = rank_tol * sqrt(r_fro[0]);
    int rk = 0;
    for (int j = tid; j < n; j += nt)
      rk += (!dropped[j] && sc[j] > 0.0 && dL[j] / sc[j] > cut) ? 1 : 0;
    rk = __reduce_add_sync(0xffffffffu, rk);
    __syncthreads();
    if (lane == 0) r_kept[warp] = rk;
    __syncthreads();
    if (tid == 0) {
      int tot = 0;
      for (int w = 0; w < nw; ++w) tot += r_kept[w];
      info[0] = r_min[0];
      info[2] = (double)kc;
      info[1] = rank_tol > 0.0 ? (double)tot : 0.0;
      if (keep) {
        int kept = 0;
        for (int j = 0; j < n; ++j)
          if (!dropped[j]) keep[kept++] = j;
      }
      CI_T(8);
    }
  }
}


// Launch of cholinv_kernel on one cluster (8 CTAs for n > 96).
inline void cholinv_launch(cudaStream_t st, size_t smem_limit, double* A, int n, int64_t ld,
                           int scale, double col_drop, double shift, double drop_ratio,
                           double rank_tol, double* X, double* T, double* s_out,
                           double* info, int* keep) {
  const size_t smem = cholinv_smem(n);
  {  // function attributes are per device: set on every call
    const cudaError_t e = cudaFuncSetAttribute(
        cholinv_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    if (e != cudaSuccess)
      throw Error(kErrCuda, std::string("cholinv smem attribute: ") + cudaGetErrorString(e));
  }
  (void)smem_limit;
  cudaLaunchConfig_t cfg = {};
  const int csize = n > 96 ? 8 : 1;
  cfg.gridDim = dim3(csize);
  cfg.blockDim = dim3(kCiThreads);
  cfg.dynamicSmemBytes = smem;
  cfg.stream = st;
  cudaLaunchAttribute at[1];
  at[0].id = cudaLaunchAttributeClusterDimension;
  at[0].val.clusterDim.x = csize;
  at[0].val.clusterDim.y = 1;
  at[0].val.clusterDim.z = 1;
  cfg.attrs = at;
  cfg.numAttrs = 1;
  const cudaError_t e = cudaLaunchKernelEx(&cfg, cholinv_kernel, A, n, ld, scale, col_drop,
                                           shift, drop_ratio, rank_tol, X, T, s_out, info,
                                           keep);
  if (e != cudaSuccess)
    throw Error(kErrCuda, std::string("cholinv launch: ") + cudaGetErrorString(e));
  if (std::getenv("BRSVD_CI_TIMING")) {
    long long t[11];
    cudaStreamSynchronize(st);
    cudaMemcpyFromSymbol(t, g_ci_t, sizeof(t));
    std::fprintf(stderr, "[cholinv n=%d] scale %lld | p0: load %lld diag %lld trsm %lld trail %lld | "
                 "panels %lld | inverse %lld (diag blocks %lld, block rows %lld) | out %lld (cycles)\n", n,
                 t[1] - t[0], t[2] - t[1], t[3] - t[2], t[4] - t[3], t[5] - t[4], t[6] - t[1],
                 t[7] - t[6], t[9] - t[6], t[10] - t[9], t[8] - t[7]);
  }
}

}  // namespace brsvd
