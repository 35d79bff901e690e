// One-sided Jacobi SVD of a square l x l matrix held entirely in the
// distributed shared memory of ONE thread-block cluster (8 or 16 CTAs).
//
// Replaces, for the l-by-l core problems of the pipeline (np.linalg.svd(r.T)
// in small_svd, kernels.py:173-188, and the Gram eigen-solves behind tsqr,
// kernels.py:121-164), the cooperative-grid block Jacobi of jacobi.cuh whose
// every tournament round went through global memory and a grid barrier.
//
// Layout: the columns of G (and of the accumulated rotation V) are grouped in
// nb = 2 * cluster_size blocks of bw columns.  CTA c plays positions c and
// nb-1-c of a round-robin ("circle method") tournament over the blocks, so in
// every round each CTA owns one block pair in its shared memory:
//   * the first round of a sweep orthogonalises all 2bw columns of the pair,
//   * later rounds only the bw^2 cross pairs (block a column i against block
//     b column (i + s) mod bw, s = 0..bw-1),
// so every column pair meets exactly once per sweep.  Between rounds every CTA
// PULLS its next two blocks from their current owners over DSMEM into the
// other half of a ping-pong buffer; one cluster barrier per round orders the
// pulls against the previous round's rotations (see the hazard note below).
// A column rotation is one warp: the two columns stay in registers from the
// dot products to the update (NP2 row pairs per lane, 8/16-byte shared-memory
// accesses), the three reductions share one butterfly.
// The accumulated rotation V is NOT carried through the tournament: every
// scheduled pair logs its rotation (c, s, columns) and jacobi_vreplay_kernel
// applies the log to V afterwards, one row of V per CTA (the rows are
// independent under column rotations).  The cluster kernel then moves and
// rotates G columns only -- half the DSMEM pull bytes and no V update on the
// chain of every step.
#pragma once
#include <cooperative_groups.h>
#include "common.cuh"

namespace brsvd {

template <typename R> struct Vec2;
template <> struct Vec2<float> { using type = float2; };
template <> struct Vec2<double> { using type = double2; };

// One logged rotation (c, s): the scheduled pair (x, y) of V columns becomes
// (c x - s y, s x + c y); (1, 0) for a pair that was not rotated (exact
// identity).  The columns follow from the tournament schedule.
template <typename R>
using JcRot = typename Vec2<R>::type;

template <typename R>
struct JacobiClusterArgs {
  R* G;          // l x l, column-major, ld ldg  (overwritten by G V)
  int64_t ldg;
  JcRot<R>* log;     // rotation log: step t, slot (CTA, warp) at t * C * bw + slot;
                     // max_sweeps * jc_sweep_steps steps (the sweep cap bounds it)
  int* prog;         // [0] steps logged so far, [1] 1 when final (read by the replay)
  int l;         // matrix order
  int bw;        // block width
  int max_sweeps;
  double tol;        // rotate while |x.y| > tol ||x|| ||y||
  double floor_rel;  // columns below floor_rel * ||G||_F are numerically null
  int* sweeps_done;  // optional
  // > 0: also stop after a sweep whose largest rotated |cos(x, y)| stayed
  // below stop_cos (quadratic convergence: the next sweep would find nothing
  // above ~stop_cos^2); the fp32 preconditioning phase uses sqrt(tol)
  double stop_cos;
};

__device__ __forceinline__ int tourn_pos(int pos, int r, int n) {
  return pos == 0 ? 0 : ((pos - 1 + r) % (n - 1)) + 1;
}
// Inverse of tourn_pos: the position block b sits at in round r.
__device__ __forceinline__ int tourn_inv(int b, int r, int n) {
  return b == 0 ? 0 : ((b - 1 - r) % (n - 1) + (n - 1)) % (n - 1) + 1;
}

template <typename R>
__device__ __forceinline__ R jc_rsqrt(R x);
template <>
__device__ __forceinline__ float jc_rsqrt<float>(float x) { return rsqrtf(x); }
template <>
__device__ __forceinline__ double jc_rsqrt<double>(double x) { return rsqrt(x); }  // 1 ulp


// Rotate columns (x, y) of G so that they become orthogonal; (c, s) of the
// rotation are returned in cr, sr.  One warp; columns are zero-padded to lp (a multiple of 4) and
// each lane owns row pairs (2 lane + 64 k, +1), k < NP2, kept in registers
// from the dot products to the update.  Returns true if rotated.
template <typename R, int NP2>
__device__ __forceinline__ bool jc_rotate(R* __restrict__ x, R* __restrict__ y, int lp,
                                          R tol2, R floor2, int lane, R& c2max, R& cr,
                                          R& sr) {
  using V2 = typename Vec2<R>::type;
  V2 xr[NP2], yr[NP2];
  R a = 0, b = 0, g = 0;
#pragma unroll
  for (int k = 0; k < NP2; ++k) {
    const int i = 2 * lane + 64 * k;
    if (i < lp) {
      xr[k] = *reinterpret_cast<const V2*>(x + i);
      yr[k] = *reinterpret_cast<const V2*>(y + i);
    } else {
      xr[k].x = xr[k].y = yr[k].x = yr[k].y = R(0);
    }
  }
#pragma unroll
  for (int k = 0; k < NP2; ++k) {
    a = fma(xr[k].x, xr[k].x, a);
    b = fma(yr[k].x, yr[k].x, b);
    g = fma(xr[k].x, yr[k].x, g);
    a = fma(xr[k].y, xr[k].y, a);
    b = fma(yr[k].y, yr[k].y, b);
    g = fma(xr[k].y, yr[k].y, g);
  }
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) {
    a += __shfl_xor_sync(0xffffffffu, a, o);
    b += __shfl_xor_sync(0xffffffffu, b, o);
    g += __shfl_xor_sync(0xffffffffu, g, o);
  }
  if (!(a > floor2 && b > floor2)) return false;
  if (!(g * g > tol2 * a * b)) return false;
  c2max = max(c2max, (R)((g * g) / (a * b)));
  R t;
  if (sizeof(R) == 4) {
    // fp32 phase (a preconditioner for the fp64 sweeps): approximate
    // reciprocal / square root; c and s stay consistent through rsqrt.
    const float zeta = __fdividef((float)(b - a), 2.0f * (float)g);
    const float az = fabsf(zeta);
    if (az > 1e18f) {
      t = (R)__fdividef(0.5f, zeta);
    } else {
      const float w = fmaf(zeta, zeta, 1.0f);
      t = (R)copysignf(__fdividef(1.0f, az + w * rsqrtf(w)), zeta);
    }
  } else {
    const R zeta = (b - a) / (R(2) * g);
    if (fabs(zeta) > R(1e150)) {
      t = R(0.5) / zeta;
    } else {
      t = copysign(R(1), zeta) / (fabs(zeta) + sqrt(fma(zeta, zeta, R(1))));
    }
  }
  if (t == R(0)) return false;
  const R c = jc_rsqrt<R>(fma(t, t, R(1)));
  const R s = c * t;
#pragma unroll
  for (int k = 0; k < NP2; ++k) {
    const int i = 2 * lane + 64 * k;
    if (i < lp) {
      V2 nx, ny;
      nx.x = c * xr[k].x - s * yr[k].x;
      nx.y = c * xr[k].y - s * yr[k].y;
      ny.x = s * xr[k].x + c * yr[k].x;
      ny.y = s * xr[k].y + c * yr[k].y;
      *reinterpret_cast<V2*>(x + i) = nx;
      *reinterpret_cast<V2*>(y + i) = ny;
    }
  }
  cr = c;
  sr = s;
  return true;
}

// Cross-round rotation with the block-a column x held in registers for the
// whole round and the partner y in shared memory: the x loads and stores of
// jc_rotate disappear from every step.  Returns true if rotated.
template <typename R, int NP2>
__device__ __forceinline__ bool jc_rotate_x(typename Vec2<R>::type (&xr)[NP2],
                                            R* __restrict__ y, int lp, R tol2, R floor2,
                                            int lane, R& c2max, R& cr, R& sr) {
  using V2 = typename Vec2<R>::type;
  V2 yr[NP2];
  R g = 0, aa = 0, b = 0;
#pragma unroll
  for (int k = 0; k < NP2; ++k) {
    const int i = 2 * lane + 64 * k;
    if (i < lp) {
      yr[k] = *reinterpret_cast<const V2*>(y + i);
    } else {
      yr[k].x = yr[k].y = R(0);
    }
    g = fma(xr[k].x, yr[k].x, g);
    aa = fma(xr[k].x, xr[k].x, aa);
    b = fma(yr[k].x, yr[k].x, b);
    g = fma(xr[k].y, yr[k].y, g);
    aa = fma(xr[k].y, xr[k].y, aa);
    b = fma(yr[k].y, yr[k].y, b);
  }
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) {
    g += __shfl_xor_sync(0xffffffffu, g, o);
    aa += __shfl_xor_sync(0xffffffffu, aa, o);
    b += __shfl_xor_sync(0xffffffffu, b, o);
  }
  const R a = aa;   // exact norms: cached ones drift and cost a sweep
  if (!(a > floor2 && b > floor2)) return false;
  if (!(g * g > tol2 * a * b)) return false;
  c2max = max(c2max, (R)((g * g) / (a * b)));
  R t;
  if (sizeof(R) == 4) {
    const float zeta = __fdividef((float)(b - a), 2.0f * (float)g);
    const float az = fabsf(zeta);
    if (az > 1e18f) {
      t = (R)__fdividef(0.5f, zeta);
    } else {
      const float w = fmaf(zeta, zeta, 1.0f);
      t = (R)copysignf(__fdividef(1.0f, az + w * rsqrtf(w)), zeta);
    }
  } else {
    const R zeta = (b - a) / (R(2) * g);
    if (fabs(zeta) > R(1e150)) {
      t = R(0.5) / zeta;
    } else {
      t = copysign(R(1), zeta) / (fabs(zeta) + sqrt(fma(zeta, zeta, R(1))));
    }
  }
  if (t == R(0)) return false;
  const R c = jc_rsqrt<R>(fma(t, t, R(1)));
  const R s = c * t;
#pragma unroll
  for (int k = 0; k < NP2; ++k) {
    const int i = 2 * lane + 64 * k;
    const V2 x0 = xr[k];
    xr[k].x = c * x0.x - s * yr[k].x;
    xr[k].y = c * x0.y - s * yr[k].y;
    V2 ny;
    ny.x = s * x0.x + c * yr[k].x;
    ny.y = s * x0.y + c * yr[k].y;
    if (i < lp) *reinterpret_cast<V2*>(y + i) = ny;
  }
  cr = c;
  sr = s;
  return true;
}

// Shared memory: buf[2][2 slots][bw columns][lp] of R (lp = l rounded up to 4).
template <typename R>
__host__ __device__ inline size_t jacobi_cluster_smem(int l, int bw) {
  const int lp = (l + 3) & ~3;
  return (size_t)2 * 2 * bw * lp * sizeof(R);
}

// Logged steps per sweep: the first round orthogonalises the 2 bw columns of
// every block pair (2 bw - 1 steps), the nb - 2 other rounds the cross pairs
// (bw steps).  Step index of round r, step st: jc_step(r, ..) + st.
__host__ __device__ inline int64_t jc_sweep_steps(int bw, int nb) {
  return (int64_t)(2 * bw - 1) + (int64_t)(nb - 2) * bw;
}
__device__ __forceinline__ void jc_st_release(int* p, int v) {
  asm volatile("st.release.gpu.global.b32 [%0], %1;" ::"l"(p), "r"(v) : "memory");
}
__device__ __forceinline__ int jc_ld_acquire(const int* p) {
  int v;
  asm volatile("ld.acquire.gpu.global.b32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
  return v;
}
__device__ __forceinline__ int64_t jc_step(int r, int bw, int nb) {
  const int tr = r % (nb - 1);
  return (int64_t)(r / (nb - 1)) * jc_sweep_steps(bw, nb) +
         (tr == 0 ? 0 : (int64_t)(2 * bw - 1) + (int64_t)(tr - 1) * bw);
}

// Cycle split of the last launch (CTA 0, thread 0): rotations, cluster
// barriers, block pulls, rounds (BRSVD_JC_TIMING=1 prints it).
__device__ long long g_jc_t[4];
__device__ float g_jc_c2[64];   // largest rotated cos^2 of each sweep (last launch)

template <typename R, int NP2>
__global__ void jacobi_cluster_kernel(JacobiClusterArgs<R> a) {
  namespace cg = cooperative_groups;
  cg::cluster_group cluster = cg::this_cluster();
  extern __shared__ __align__(16) unsigned char jc_raw[];
  R* buf = reinterpret_cast<R*>(jc_raw);
  __shared__ int s_cnt[2];     // rotations of the current sweep, by sweep parity
  __shared__ float s_c2[2];    // largest rotated cos^2 of the sweep, by parity
  __shared__ double s_red[32];
  __shared__ int s_stop;

  const int l = a.l, bw = a.bw;
  const int lp = (l + 3) & ~3;
  const int colsz = lp;                        // G columns only
  const size_t slotsz = (size_t)bw * colsz;    // one block
  const size_t bufsz = 2 * slotsz;             // two blocks
  const int C = (int)cluster.num_blocks();
  const int me = (int)cluster.block_rank();
  const int nb = 2 * C;
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int nwarps = blockDim.x >> 5;
  const int tid = threadIdx.x, nt = blockDim.x;
  // the V replay (launched programmatically dependent on this kernel) may
  // start now: this grid is resident, so its spinning cannot block us
  asm volatile("griddepcontrol.launch_dependents;" ::: "memory");

  // ||G||_F^2 is invariant under the rotations: fix the null floor once.
  {
    double f = 0.0;
    for (int c = warp; c < l; c += nwarps)
      for (int i = lane; i < l; i += 32) {
        const double v = (double)a.G[c * a.ldg + i];
        f = fma(v, v, f);
      }
    f = warp_sum(f);
    if (lane == 0) s_red[warp] = f;
    if (tid < 2) {
      s_cnt[tid] = 0;
      s_c2[tid] = 0.f;
    }
    __syncthreads();
    if (tid == 0) {
      double t = 0.0;
      for (int w = 0; w < nwarps; ++w) t += s_red[w];
      s_red[0] = t;
    }
    __syncthreads();
  }
  const R floor2 = (R)(a.floor_rel * a.floor_rel * s_red[0]);
  const R tol2 = (R)(a.tol * a.tol);

  // Initial load of round 0's block pair from global memory into buf[0].
  {
    R* dst = buf;
    for (int e = tid; e < 2 * bw * lp; e += nt) {
      const int cl = e / lp, i = e % lp;         // local column, row
      const int slot = cl / bw, j = cl % bw;
      const int blk = tourn_pos(slot == 0 ? me : nb - 1 - me, 0, nb);
      const int gc = blk * bw + j;
      R* col = dst + slot * slotsz + (size_t)j * colsz;
      const bool ok = gc < l && i < l;
      col[i] = ok ? a.G[(int64_t)gc * a.ldg + i] : R(0);
    }
  }
  cluster.sync();

  int r = 0;  // global round counter; tournament round = r % (nb - 1)
  int sweep = 0;
  int my_rot = 0;
  R my_c2 = 0;
  long long t_rot = 0, t_sync = 0, t_pull = 0, t0 = clock64();
  for (;;) {
    const int tr = r % (nb - 1);
    R* cur = buf + (size_t)(r & 1) * bufsz;
    const int ba = tourn_pos(me, tr, nb), bb = tourn_pos(nb - 1 - me, tr, nb);
    // valid column counts of the two blocks (ragged last block)
    const int va = max(0, min(bw, l - ba * bw)), vb = max(0, min(bw, l - bb * bw));
    JcRot<R>* lg = a.log + jc_step(r, bw, nb) * (C * bw) + me * bw;
    __syncthreads();
    if (tr == 0) {
      // all pairs of the 2bw columns: inner circle tournament over W = 2bw
      const int W = 2 * bw;
      for (int st = 0; st < W - 1; ++st) {
        for (int p = warp; p < bw; p += nwarps) {
          const int ca = tourn_pos(p, st, W), cb = tourn_pos(W - 1 - p, st, W);
          const int ja = ca % bw, jb = cb % bw;
          const bool oka = ca < bw ? ja < va : ja < vb;
          const bool okb = cb < bw ? jb < va : jb < vb;
          JcRot<R> e;
          e.x = R(1);
          e.y = R(0);
          if (oka && okb) {
            R* x = cur + (size_t)(ca / bw) * slotsz + (size_t)ja * colsz;
            R* y = cur + (size_t)(cb / bw) * slotsz + (size_t)jb * colsz;
            if (jc_rotate<R, NP2>(x, y, lp, tol2, floor2, lane, my_c2, e.x, e.y)) ++my_rot;
          }
          if (lane == 0) lg[(int64_t)st * (C * bw) + p] = e;
        }
        __syncthreads();
      }
    } else {
      // cross pairs: warp p keeps column p of block a in registers for the
      // whole round; the block-b columns pass from warp to warp through shared
      // memory (nwarps >= bw)
      using V2 = typename Vec2<R>::type;
      const int p = warp;
      const bool own = p < bw && p < va;
      V2 xr[NP2];
      R* xcol = cur + (size_t)p * colsz;
      if (own) {
#pragma unroll
        for (int k = 0; k < NP2; ++k) {
          const int i = 2 * lane + 64 * k;
          if (i < lp) {
            xr[k] = *reinterpret_cast<const V2*>(xcol + i);
          } else {
            xr[k].x = xr[k].y = R(0);
          }
        }
      }
      for (int st = 0; st < bw; ++st) {
        const int jb = p + st < bw ? p + st : p + st - bw;
        JcRot<R> e;
        e.x = R(1);
        e.y = R(0);
        if (own && jb < vb) {
          R* y = cur + slotsz + (size_t)jb * colsz;
          if (jc_rotate_x<R, NP2>(xr, y, lp, tol2, floor2, lane, my_c2, e.x, e.y)) ++my_rot;
        }
        if (p < bw && lane == 0) lg[(int64_t)st * (C * bw) + p] = e;
        __syncthreads();
      }
      if (own) {
#pragma unroll
        for (int k = 0; k < NP2; ++k) {
          const int i = 2 * lane + 64 * k;
          if (i < lp) *reinterpret_cast<V2*>(xcol + i) = xr[k];
        }
      }
    }
    const bool sweep_end = (tr == nb - 2);
    if (sweep_end && lane == 0 && my_rot) {
      atomicAdd(&s_cnt[sweep & 1], my_rot);
      atomicMax(reinterpret_cast<int*>(&s_c2[sweep & 1]), __float_as_int((float)my_c2));
    }
    if (sweep_end) {
      my_rot = 0;
      my_c2 = 0;
    }
    // Hazards: the pull below reads the peers' buf[r&1] (rotated in this
    // round, before this barrier) and writes our buf[(r+1)&1], which the peers
    // last read while pulling for round r (before this barrier).
    long long t1 = clock64();
    t_rot += t1 - t0;
    cluster.sync();
    t0 = clock64();
    t_sync += t0 - t1;
    // rounds 0..r are logged by every CTA (ordered by the cluster barrier):
    // publish them to the replay
    if (me == 0 && tid == 0) {
      __threadfence();
      jc_st_release(a.prog, (int)jc_step(r + 1, bw, nb));
    }
    if (sweep_end) {
      if (tid == 0) {
        int tot = 0;
        float c2 = 0.f;
        for (int q = 0; q < C; ++q) {
          tot += *cluster.map_shared_rank(&s_cnt[sweep & 1], q);
          c2 = fmaxf(c2, *cluster.map_shared_rank(&s_c2[sweep & 1], q));
        }
        if (me == 0 && sweep < 64) g_jc_c2[sweep] = c2;
        s_stop = (tot == 0) || (sweep + 1 >= a.max_sweeps) ||
                 (a.stop_cos > 0.0 && (double)c2 < a.stop_cos * a.stop_cos);
        s_cnt[(sweep + 1) & 1] = 0;
        s_c2[(sweep + 1) & 1] = 0.f;
      }
      __syncthreads();
      if (s_stop) break;
      ++sweep;
    }
    // pull the blocks of round r+1 into buf[(r+1)&1]
    const int tn = (r + 1) % (nb - 1);
    R* nxt = buf + (size_t)((r + 1) & 1) * bufsz;
    {
      const int4* s4[2];
      for (int slot = 0; slot < 2; ++slot) {
        const int blk = tourn_pos(slot == 0 ? me : nb - 1 - me, tn, nb);
        const int pos = tourn_inv(blk, tr, nb);         // where it sat this round
        const int owner = pos < C ? pos : nb - 1 - pos;
        const int oslot = pos < C ? 0 : 1;
        s4[slot] = reinterpret_cast<const int4*>(
            cluster.map_shared_rank(cur + oslot * slotsz, owner));
      }
      int4* d4 = reinterpret_cast<int4*>(nxt);
      const int n4 = (int)(slotsz * sizeof(R) / 16);  // per slot
      // DSMEM loads have ~200 cycles of latency: keep 8 in flight per thread
      constexpr int U = 8;
      for (int e0 = tid; e0 < 2 * n4; e0 += U * nt) {
        int4 v[U];
#pragma unroll
        for (int u = 0; u < U; ++u) {
          const int e = e0 + u * nt;
          if (e < 2 * n4) v[u] = e < n4 ? s4[0][e] : s4[1][e - n4];
        }
#pragma unroll
        for (int u = 0; u < U; ++u) {
          const int e = e0 + u * nt;
          if (e < 2 * n4) d4[e] = v[u];
        }
      }
    }
    t1 = clock64();
    t_pull += t1 - t0;
    t0 = t1;
    ++r;
  }
  if (me == 0 && tid == 0) {
    g_jc_t[0] = t_rot;
    g_jc_t[1] = t_sync;
    g_jc_t[2] = t_pull;
    g_jc_t[3] = r;
  }
  // converged: our current pair is in buf[r&1]; write it back
  {
    const int tr = r % (nb - 1);
    const R* cur = buf + (size_t)(r & 1) * bufsz;
    for (int e = tid; e < 2 * bw * l; e += nt) {
      const int cl = e / l, i = e % l;
      const int slot = cl / bw, j = cl % bw;
      const int blk = tourn_pos(slot == 0 ? me : nb - 1 - me, tr, nb);
      const int gc = blk * bw + j;
      if (gc >= l) continue;
      const R* col = cur + slot * slotsz + (size_t)j * colsz;
      a.G[(int64_t)gc * a.ldg + i] = col[i];
    }
  }
  if (me == 0 && tid == 0 && a.sweeps_done) *a.sweeps_done = sweep + 1;
  // keep the cluster alive until every peer finished reading our counters
  cluster.sync();
  if (me == 0 && tid == 0) {   // G written back by every CTA: final
    __threadfence();
    jc_st_release(a.prog + 1, 1);
  }
}

// V <- V * (the logged rotations, in order).  The rows of V are independent
// under column rotations and, within a tournament round, so are the block
// pairs: warp j of a CTA replays block pair (slot) j of every round on the
// rows of V held in shared memory, lane = (row, pair index p), one __syncwarp
// per step and one block barrier per round.  rows_per_warp = 32 / bw rows of
// V per CTA.  The replay is launched programmatically dependent on the
// tournament and runs concurrently with it on the idle SMs: it consumes the
// log in chunks of kJrK steps as the tournament publishes whole rounds
// (prog[0], release / acquire), so only the last round's replay is left when
// the tournament ends.  The columns of an entry follow from the schedule;
// same arithmetic per element as an in-place update of V in the tournament.
constexpr int kJrK = 16;
// vsz: bytes of a V element, rsz: of a logged rotation component.
__host__ __device__ inline size_t jacobi_vreplay_smem(int l, int bw, int C, size_t vsz,
                                                      size_t rsz) {
  const int rpw = 32 / bw, LP = (2 * C * bw) | 1;
  return (size_t)rpw * LP * vsz + 16 + (size_t)(2 * bw - 1) * bw * 4 +
         (size_t)kJrK * C * bw * 2 * rsz + 16;
}
// RV: the element type of V.  A wider V than the log (fp64 V of the fp32
// tournament) takes each rotation renormalised in RV, so V stays orthogonal
// to RV's rounding however many fp32 rotations it absorbs.
template <typename R, typename RV>
__global__ void __launch_bounds__(512) jacobi_vreplay_kernel(RV* __restrict__ V, int64_t ldv,
                                                             int l, int bw, int C,
                                                             const JcRot<R>* __restrict__ log,
                                                             const int* __restrict__ prog) {
  extern __shared__ __align__(16) unsigned char jr_raw[];
  // LP odd: the rows of a warp's lanes sit in different banks
  const int nb = 2 * C, S = 2 * bw - 1, P = C * bw, LP = (nb * bw) | 1;
  const int rpw = 32 / bw;                       // rows of V per CTA
  JcRot<R>* ebuf = reinterpret_cast<JcRot<R>*>(jr_raw);            // [warp][kJrK][bw]
  RV* rows = reinterpret_cast<RV*>(ebuf + (size_t)kJrK * P);       // rpw x LP
  short2* tab = reinterpret_cast<short2*>(
      (reinterpret_cast<uintptr_t>(rows + (size_t)rpw * LP) + 15) & ~uintptr_t(15));  // S x bw
  const int i0 = blockIdx.x * rpw;
  const int tid = threadIdx.x, nt = blockDim.x, lane = tid & 31, j = tid >> 5;
  for (int e = tid; e < rpw * LP; e += nt) {
    const int rr = e / LP, col = e % LP;
    rows[e] = (col < l && i0 + rr < l) ? V[(int64_t)col * ldv + i0 + rr] : RV(0);
  }
  for (int e = tid; e < S * bw; e += nt) {
    const int st = e / bw, p = e % bw, W = 2 * bw;
    tab[e] = make_short2((short)tourn_pos(p, st, W), (short)tourn_pos(W - 1 - p, st, W));
  }
  const int rr = lane / bw, p = lane % bw;
  const bool act = rr < rpw && i0 + rr < l;
  const bool loader = lane < bw;                 // lane p fetches slot (j, p)
  RV* row = rows + (size_t)(rr < rpw ? rr : 0) * LP;
  JcRot<R>* ew = ebuf + (size_t)j * kJrK * bw;   // this warp's chunk
  __syncthreads();
  // per-round state: round 0 is a full round (schedule table), the others
  // are cross rounds (block a column p fixed, block b column jb advancing)
  int r = 0, st = 0, steps = S, ti = p, jb = p;
  bool full = true;
  int ba = tourn_pos(j, 0, nb), bb = tourn_pos(nb - 1 - j, 0, nb);
  int gxa = ba * bw + p, gyb = bb * bw;
  for (int c = 0;; ++c) {
    // wait until the chunk is published (or the tournament is over)
    int avail = 0, dn = 0;
    for (long long spin = 0;; ++spin) {
      if (spin > (1ll << 26)) __trap();           // ~20 s: never hang the device
      if (lane == 0) {
        dn = jc_ld_acquire(prog + 1);
        avail = jc_ld_acquire(prog);   // final once dn was seen
      }
      dn = __shfl_sync(0xffffffffu, dn, 0);
      avail = __shfl_sync(0xffffffffu, avail, 0);
      if (dn || avail >= (c + 1) * kJrK) break;
      __nanosleep(256);
    }
    const int n = min(kJrK, avail - c * kJrK);
    if (n <= 0) break;                            // dn: every step replayed
    if (loader) {
      JcRot<R> v[kJrK];
      const JcRot<R>* src = log + (int64_t)c * kJrK * P + (size_t)j * bw + lane;
#pragma unroll
      for (int k = 0; k < kJrK; ++k) {
        v[k].x = R(1);
        v[k].y = R(0);
        if (k < n) v[k] = __ldcg(src + (int64_t)k * P);
      }
#pragma unroll
      for (int k = 0; k < kJrK; ++k) ew[k * bw + lane] = v[k];
    }
    __syncwarp();
    for (int k = 0; k < n; ++k) {
      const JcRot<R> e = ew[k * bw + p];
      int gx, gy;
      if (full) {
        const short2 cc = tab[ti];
        ti += bw;
        gx = cc.x < bw ? ba * bw + cc.x : bb * bw + cc.x - bw;
        gy = cc.y < bw ? ba * bw + cc.y : bb * bw + cc.y - bw;
      } else {
        gx = gxa;
        gy = gyb + jb;
        jb = (jb + 1 == bw) ? 0 : jb + 1;
      }
      if (act) {
        RV cr = (RV)e.x, sr = (RV)e.y;
        if (sizeof(RV) > sizeof(R)) {
          const RV nr = rsqrt(cr * cr + sr * sr);
          cr *= nr;
          sr *= nr;
        }
        const RV x = row[gx], y = row[gy];
        row[gx] = cr * x - sr * y;
        row[gy] = sr * x + cr * y;
      }
      __syncwarp();
      if (++st == steps) {   // end of round (uniform over the CTA)
        ++r;
        const int tr = r % (nb - 1);
        ba = tourn_pos(j, tr, nb);
        bb = tourn_pos(nb - 1 - j, tr, nb);
        full = tr == 0;
        steps = full ? S : bw;
        st = 0;
        ti = p;
        jb = p;
        gxa = ba * bw + p;
        gyb = bb * bw;
        __syncthreads();
      }
    }
    __syncwarp();                                 // the chunk buffer is reused
    if (n < kJrK) break;                          // that was the final chunk
  }
  __syncthreads();
  for (int e = tid; e < rpw * LP; e += nt) {
    const int q = e / LP, col = e % LP;
    if (col < l && i0 + q < l) V[(int64_t)col * ldv + i0 + q] = rows[e];
  }
}

}  // namespace brsvd
