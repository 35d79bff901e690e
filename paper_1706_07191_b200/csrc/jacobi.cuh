// Block one-sided (Hestenes) Jacobi SVD of a small dense matrix (fp32 or fp64).
//
// Replaces the LAPACK calls on the l-by-l problems of the reference:
// np.linalg.svd(r.T) in small_svd (kernels.py:173-188) and, through the Gram
// route, the Householder QR inside tsqr (kernels.py:121-164).
//
// G (nrow x ncol, column-major) is overwritten by G*V where V accumulates the
// plane rotations (V must be the identity on entry).  Columns are grouped in
// blocks of width bw; a round-robin tournament over the blocks pairs them up,
// and each CTA of a cooperative grid orthogonalises the 2*bw columns of its
// block pair in shared memory (one inner sweep per visit).  A single block pair
// (small l: everything fits in one CTA) iterates its inner sweeps to
// convergence, so the l <= ~110 case never touches the grid barrier.
#pragma once
#include <cooperative_groups.h>
#include "common.cuh"

namespace brsvd {
namespace cg = cooperative_groups;

template <typename R>
struct JacobiArgs {
  R* G;
  int64_t ldg;
  int nrow, ncol;
  R* V;
  int64_t ldv;
  int bw, nb;  // block width; number of blocks (even)
  int max_sweeps;
  double tol;
  double floor_rel;  // columns below floor_rel * ||G||_F are numerically null
  int* rot_count;  // [max_sweeps] zero-initialised rotation counters
  int* sweeps_done;
};

// Round-robin ("circle method") tournament: the player sitting at position
// `pos` in round `r` among `n` (even) players.  Position i plays n-1-i.
__device__ __forceinline__ int tourn(int pos, int r, int n) {
  return pos == 0 ? 0 : ((pos - 1 + r) % (n - 1)) + 1;
}

// Rotate columns x, y (length nrow in Gs, length ncol in Vs) so they become
// orthogonal.  Returns true if a rotation was applied.  Executed by one warp;
// the three reductions share one butterfly so their shuffles overlap.
template <typename R>
__device__ __forceinline__ bool jacobi_rotate_pair(R* x, R* y, R* vx, R* vy, int nrow,
                                                   int ncol, R tol2, R floor2, int lane) {
  R a = 0, b = 0, g = 0;
  for (int i = lane; i < nrow; i += 32) {
    const R p = x[i], q = y[i];
    a = fma(p, p, a);
    b = fma(q, q, b);
    g = fma(p, q, g);
  }
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) {
    a += __shfl_xor_sync(0xffffffffu, a, o);
    b += __shfl_xor_sync(0xffffffffu, b, o);
    g += __shfl_xor_sync(0xffffffffu, g, o);
  }
  // a pair involving a numerically null column (rounding noise) never
  // converges in the relative sense and carries no information: skip it
  if (!(a > floor2 && b > floor2)) return false;
  if (!(g * g > tol2 * a * b)) return false;
  const R zeta = (b - a) / (R(2) * g);
  R t;
  if (fabs(zeta) > (sizeof(R) == 8 ? R(1e150) : R(1e18))) {
    t = R(0.5) / zeta;
  } else {
    t = copysign(R(1), zeta) / (fabs(zeta) + sqrt(fma(zeta, zeta, R(1))));
  }
  if (t == R(0)) return false;
  const R c = rsqrt(fma(t, t, R(1)));  // 1 ulp; s = c t keeps c^2 + s^2 = 1 to ~2 ulp
  const R s = c * t;
  if (nrow == ncol) {
    for (int i = lane; i < nrow; i += 32) {
      const R p = x[i], q = y[i], pv = vx[i], qv = vy[i];
      x[i] = c * p - s * q;
      y[i] = s * p + c * q;
      vx[i] = c * pv - s * qv;
      vy[i] = s * pv + c * qv;
    }
  } else {
    for (int i = lane; i < nrow; i += 32) {
      const R p = x[i], q = y[i];
      x[i] = c * p - s * q;
      y[i] = s * p + c * q;
    }
    for (int i = lane; i < ncol; i += 32) {
      const R p = vx[i], q = vy[i];
      vx[i] = c * p - s * q;
      vy[i] = s * p + c * q;
    }
  }
  return true;
}

template <typename R>
__global__ void jacobi_block_kernel(JacobiArgs<R> a) {
  extern __shared__ __align__(16) unsigned char jsm_raw[];
  R* jsm = reinterpret_cast<R*>(jsm_raw);
  const int W = 2 * a.bw;
  const int nrow = a.nrow, ncol = a.ncol;
  R* Gs = jsm;                        // W columns of length nrow
  R* Vs = jsm + (size_t)W * nrow;     // W columns of length ncol
  int* cols = reinterpret_cast<int*>(Vs + (size_t)W * ncol);
  __shared__ int s_rot;
  __shared__ int s_stop;
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int nwarps = blockDim.x >> 5;
  const int npairs = a.nb / 2;
  const bool single = (a.nb == 2);
  cg::grid_group grid = cg::this_grid();
  // ||G||_F^2 is invariant under the rotations: fix the null floor once
  __shared__ double s_fro[32];
  {
    double f = 0.0;
    for (int c = warp; c < ncol; c += nwarps)
      for (int i = lane; i < nrow; i += 32) {
        const double v = (double)a.G[c * a.ldg + i];
        f = fma(v, v, f);
      }
    f = warp_sum(f);
    if (lane == 0) s_fro[warp] = f;
    __syncthreads();
    if (threadIdx.x == 0) {
      double t = 0.0;
      for (int w = 0; w < nwarps; ++w) t += s_fro[w];
      s_fro[0] = t;
    }
    __syncthreads();
  }
  const R floor2 = (R)(a.floor_rel * a.floor_rel * s_fro[0]);

  for (int sweep = 0; sweep < a.max_sweeps; ++sweep) {
    for (int round = 0; round < a.nb - 1; ++round) {
      for (int pair = blockIdx.x; pair < npairs; pair += gridDim.x) {
        const int ba = tourn(pair, round, a.nb);
        const int bb = tourn(a.nb - 1 - pair, round, a.nb);
        for (int c = threadIdx.x; c < W; c += blockDim.x) {
          const int blk = c < a.bw ? ba : bb;
          const int gc = blk * a.bw + (c % a.bw);
          cols[c] = gc < ncol ? gc : -1;
        }
        __syncthreads();
        for (int c = warp; c < W; c += nwarps) {
          const int gc = cols[c];
          for (int i = lane; i < nrow; i += 32)
            Gs[(size_t)c * nrow + i] = gc >= 0 ? a.G[gc * a.ldg + i] : R(0);
          for (int i = lane; i < ncol; i += 32)
            Vs[(size_t)c * ncol + i] = gc >= 0 ? a.V[gc * a.ldv + i] : R(0);
        }
        __syncthreads();
        const int inner = single ? 64 : 1;
        // Round 0 of a sweep orthogonalises all 2bw columns of the pair
        // (within-block and cross pairs); later rounds only need the cross
        // pairs (block a column i against block b column (i + ir) mod bw),
        // which halves the sequential depth of a sweep to ~l + bw rounds.
        const bool full_inner = single || round == 0;
        const int n_inner = full_inner ? W - 1 : a.bw;
        int total = 0;
        for (int is = 0; is < inner; ++is) {
          if (threadIdx.x == 0) s_rot = 0;
          __syncthreads();
          for (int ir = 0; ir < n_inner; ++ir) {
            for (int p = warp; p < W / 2; p += nwarps) {
              int ca, cb;
              if (full_inner) {
                ca = tourn(p, ir, W);
                cb = tourn(W - 1 - p, ir, W);
              } else {
                ca = p;
                cb = a.bw + (p + ir) % a.bw;
              }
              if (cols[ca] < 0 || cols[cb] < 0) continue;
              const bool rot = jacobi_rotate_pair(
                  Gs + (size_t)ca * nrow, Gs + (size_t)cb * nrow,
                  Vs + (size_t)ca * ncol, Vs + (size_t)cb * ncol, nrow, ncol,
                  (R)(a.tol * a.tol), floor2, lane);
              if (rot && lane == 0) atomicAdd(&s_rot, 1);
            }
            __syncthreads();
          }
          const int r = s_rot;
          total += r;
          __syncthreads();
          if (r == 0) break;
        }
        if (threadIdx.x == 0 && total > 0) atomicAdd(&a.rot_count[sweep], total);
        for (int c = warp; c < W; c += nwarps) {
          const int gc = cols[c];
          if (gc < 0) continue;
          for (int i = lane; i < nrow; i += 32)
            a.G[gc * a.ldg + i] = Gs[(size_t)c * nrow + i];
          for (int i = lane; i < ncol; i += 32)
            a.V[gc * a.ldv + i] = Vs[(size_t)c * ncol + i];
        }
        __syncthreads();
      }
      if (!single) grid.sync();
    }
    if (single) __threadfence_block(); else __threadfence();
    if (!single) grid.sync();
    if (threadIdx.x == 0) {
      const int rc = atomicAdd(&a.rot_count[sweep], 0);
      s_stop = (rc == 0);
    }
    __syncthreads();
    if (s_stop) {
      if (blockIdx.x == 0 && threadIdx.x == 0) *a.sweeps_done = sweep + 1;
      return;
    }
  }
  if (blockIdx.x == 0 && threadIdx.x == 0) *a.sweeps_done = a.max_sweeps;
}

// Column norms of G*V, descending rank sort, permuted outputs.
//   sv[j]  = ||(G V)_{:, perm j}||,  Vout[:, j] = V[:, perm j],
//   Uout[:, j] = (G V)[:, perm j] / sv[j]   (zero column if sv == 0).
// Any grid: the columns are split over the CTAs' warps (grid-stride).
__global__ void jacobi_finish_kernel(const double* __restrict__ G, int64_t ldg,
                                     int nrow, int ncol,
                                     const double* __restrict__ V, int64_t ldv,
                                     double* __restrict__ sv,
                                     double* __restrict__ Uout, int64_t ldu,
                                     double* __restrict__ Vout, int64_t ldvo) {
  extern __shared__ double fsm[];
  double* nrm = fsm;                                  // ncol
  int* perm = reinterpret_cast<int*>(fsm + ncol);     // ncol
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int nwarps = blockDim.x >> 5;
  for (int c = warp; c < ncol; c += nwarps) {
    double s = 0.0;
    for (int i = lane; i < nrow; i += 32) {
      const double v = G[c * ldg + i];
      s = fma(v, v, s);
    }
    s = warp_sum(s);
    // NaN (non-finite input) sorts last: the key order must be total so the
    // ranks form a permutation.
    if (lane == 0) nrm[c] = (s == s) ? sqrt(s) : -1.0;
  }
  __syncthreads();
  for (int c = threadIdx.x; c < ncol; c += blockDim.x) {
    const double v = nrm[c];
    int rank = 0;
    for (int o = 0; o < ncol; ++o) {
      const double w = nrm[o];
      rank += (w > v) || (w == v && o < c);
    }
    perm[rank] = c;
  }
  __syncthreads();
  // the permuted copies are split over the CTAs (every CTA ranks redundantly)
  for (int j = blockIdx.x * nwarps + warp; j < ncol; j += gridDim.x * nwarps) {
    const int c = perm[j];
    const double s = nrm[c];
    if (lane == 0 && sv != nullptr) sv[j] = s;
    if (Uout != nullptr) {
      const double inv = s > 0.0 ? 1.0 / s : 0.0;
      for (int i = lane; i < nrow; i += 32) Uout[j * ldu + i] = G[c * ldg + i] * inv;
    }
    if (Vout != nullptr)
      for (int i = lane; i < ncol; i += 32) Vout[j * ldvo + i] = V[c * ldv + i];
  }
}

// Left singular vectors of numerically null singular values (sv_j below
// floor_rel * ||sv||_2; the Jacobi sweep never rotates those columns, so their
// normalised columns are rounding noise) are replaced by an orthonormal
// completion, as LAPACK's SVD returns a full orthonormal U (the reference's
// np.linalg.svd in small_svd, kernels.py:186).  sv is sorted descending, so the
// null columns are a suffix.  One CTA.
__global__ void complete_null_columns_kernel(double* __restrict__ U, int64_t ldu, int nrow,
                                             int ncol, const double* __restrict__ sv,
                                             double floor_rel) {
  extern __shared__ double csm[];
  double* coef = csm;  // ncol
  __shared__ int s_r0;
  __shared__ double s_red[32];
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5, nwarps = blockDim.x >> 5;
  if (threadIdx.x == 0) {
    double f = 0.0;
    for (int j = 0; j < ncol; ++j) f += sv[j] * sv[j];
    const double fl = floor_rel * sqrt(f);
    int r0 = ncol;
    for (int j = 0; j < ncol; ++j)
      if (!(sv[j] > fl)) { r0 = j; break; }
    s_r0 = r0;
  }
  __syncthreads();
  const int r0 = s_r0;
  for (int j = r0; j < ncol; ++j) {
    double* v = U + (int64_t)j * ldu;
    for (int i = threadIdx.x; i < nrow; i += blockDim.x) {
      uint32_t h = (uint32_t)(i * 0x9E3779B1u) ^ (uint32_t)(j * 0x85EBCA77u) ^ 0xC2B2AE3Du;
      h ^= h >> 15; h *= 0x2C1B3C6Du; h ^= h >> 12; h *= 0x297A2D39u; h ^= h >> 15;
      v[i] = (double)h * (1.0 / 4294967296.0) - 0.5;
    }
    __syncthreads();
    for (int pass = 0; pass < 2; ++pass) {
      for (int c = warp; c < j; c += nwarps) {
        const double* u = U + (int64_t)c * ldu;
        double d = 0.0;
        for (int i = lane; i < nrow; i += 32) d = fma(u[i], v[i], d);
        d = warp_sum(d);
        if (lane == 0) coef[c] = d;
      }
      __syncthreads();
      for (int i = threadIdx.x; i < nrow; i += blockDim.x) {
        double acc = v[i];
        for (int c = 0; c < j; ++c) acc = fma(-coef[c], U[(int64_t)c * ldu + i], acc);
        v[i] = acc;
      }
      __syncthreads();
    }
    double nn = 0.0;
    for (int i = threadIdx.x; i < nrow; i += blockDim.x) nn = fma(v[i], v[i], nn);
    nn = warp_sum(nn);
    if (lane == 0) s_red[warp] = nn;
    __syncthreads();
    if (threadIdx.x == 0) {
      double t = 0.0;
      for (int w = 0; w < nwarps; ++w) t += s_red[w];
      s_red[0] = t > 0.0 ? 1.0 / sqrt(t) : 0.0;
    }
    __syncthreads();
    const double inv = s_red[0];
    for (int i = threadIdx.x; i < nrow; i += blockDim.x) v[i] *= inv;
    __syncthreads();
  }
}

}  // namespace brsvd
