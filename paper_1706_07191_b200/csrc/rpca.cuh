// Inexact-ALM robust PCA on the GPU (rpca.py:153-213) and the spectral-norm
// power iteration it starts from (rpca.py:72-100).
//
// Per iteration the m x n iterates are touched by exactly two kinds of
// kernels: the randomized SVD of W (pipeline.cuh; HBM-streaming products of
// rank l) and ONE fused element pass (rpca_step_kernel) that forms
//   L = U shrink(s, 1/mu) V^T            (rank-l, on the fly, never stored)
//   S = shrink(M - L + Y/mu, lam/mu),  Z = M - L - S,  Y += mu Z,
//   ||Z||_F^2 (deterministic block partials),
//   W = M - S + Y/(mu rho)              (the next iteration's SVD input)
// i.e. 2 reads (M, Y) + 3 writes (S, Y, W) per element, where the reference
// materialises ~8 m x n temporaries per iteration (rpca.py:190-199).
#pragma once
#include "pipeline.cuh"

namespace brsvd {

// ---- vector helpers (single CTA; vectors here have length m or n) ----------
__global__ void vec_norm2_kernel(const double* __restrict__ x, int64_t n,
                                 double* __restrict__ out) {
  __shared__ double red[32];
  double s = 0.0;
  for (int64_t i = threadIdx.x; i < n; i += blockDim.x) s = fma(x[i], x[i], s);
  s = warp_sum(s);
  if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = s;
  __syncthreads();
  if (threadIdx.x == 0) {
    double t = 0.0;
    for (int w = 0; w < (int)(blockDim.x >> 5); ++w) t += red[w];
    *out = sqrt(t);
  }
}

__global__ void vec_scale_kernel(double* __restrict__ x, int64_t n,
                                 const double* __restrict__ by, int invert) {
  const double d = *by;
  const double f = invert ? (d != 0.0 ? 1.0 / d : 0.0) : d;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n;
       i += (int64_t)gridDim.x * blockDim.x)
    x[i] *= f;
}

// ---- matrix-vector products -------------------------------------------------
// out[o] = sum_k X(o, k) x[k],  X(o, k) = X[o*so + k*sk]  (fp64 accumulation).
// Contiguous-k form: one warp per output.
template <typename T>
__global__ void matvec_dot_kernel(const T* __restrict__ X, int64_t O, int64_t Kd,
                                  int64_t so, const double* __restrict__ x,
                                  double* __restrict__ out) {
  const int lane = threadIdx.x & 31;
  const int64_t warp = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) >> 5;
  const int64_t nwarps = ((int64_t)gridDim.x * blockDim.x) >> 5;
  for (int64_t o = warp; o < O; o += nwarps) {
    const T* row = X + o * so;
    double s = 0.0;
    for (int64_t k = lane; k < Kd; k += 32) s = fma((double)row[k], x[k], s);
    s = warp_sum(s);
    if (lane == 0) out[o] = s;
  }
}

// Contiguous-o form: one thread per output, k split in chunks (grid.y) with
// partial sums reduced in fixed order by matvec_reduce_kernel.
template <typename T>
__global__ void matvec_sweep_kernel(const T* __restrict__ X, int64_t O, int64_t Kd,
                                    int64_t sk, int64_t kchunk,
                                    const double* __restrict__ x,
                                    double* __restrict__ part) {
  const int64_t o = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (o >= O) return;
  const int64_t k0 = blockIdx.y * kchunk, k1 = min(Kd, k0 + kchunk);
  double s = 0.0;
  for (int64_t k = k0; k < k1; ++k) s = fma((double)X[o + k * sk], x[k], s);
  part[blockIdx.y * O + o] = s;
}

__global__ void matvec_reduce_kernel(const double* __restrict__ part, int64_t O,
                                     int chunks, double* __restrict__ out) {
  for (int64_t o = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; o < O;
       o += (int64_t)gridDim.x * blockDim.x) {
    double s = 0.0;
    for (int c = 0; c < chunks; ++c) s += part[c * O + o];
    out[o] = s;
  }
}

template <typename T>
void matvec(Ctx& c, const T* X, int64_t O, int64_t Kd, int64_t so, int64_t sk,
            const double* x, double* out) {
  if constexpr (sizeof(T) == 8) {  // fp64: the streaming skinny product, l = 1
    if ((sk == 1 || so == 1) &&
        skinny_f64(c, sk == 1, reinterpret_cast<const double*>(X), O, Kd, sk == 1 ? so : sk,
                   x, Kd, 1, out, O))
      return;
  }
  if (sk == 1) {
    matvec_dot_kernel<T><<<grid_for(O * 32, 256, 148 * 32), 256, 0, c.stream>>>(
        X, O, Kd, so, x, out);
    BRSVD_CHECK_LAUNCH();
    return;
  }
  const int64_t oblocks = ceil_div(O, 256);
  int64_t chunks = std::max<int64_t>(1, std::min<int64_t>(ceil_div(148 * 8, oblocks),
                                                         ceil_div(Kd, 64)));
  const int64_t kchunk = ceil_div(Kd, chunks);
  chunks = ceil_div(Kd, kchunk);
  DBuf<double> part(c, (size_t)(chunks * O));
  matvec_sweep_kernel<T><<<dim3((unsigned)oblocks, (unsigned)chunks), 256, 0, c.stream>>>(
      X, O, Kd, sk, kchunk, x, part.p);
  BRSVD_CHECK_LAUNCH();
  matvec_reduce_kernel<<<grid_for(O), 256, 0, c.stream>>>(part.p, O, (int)chunks, out);
  BRSVD_CHECK_LAUNCH();
}

// Largest singular value by power iteration on M^T M, stopping rule of
// rpca.py:72-100 (|s_new - s| <= tol * s_new, at most max_it iterations).
// M (m x n): element (i, j) at M[i*sm + j*sn].  Returns 0 for a zero matrix.
template <typename T>
double spectral_norm(Ctx& c, const T* Mx, int64_t m, int64_t n, int64_t sm, int64_t sn,
                     uint64_t seed, double tol, int max_it, int* iters_out,
                     const double* start = nullptr) {
  DBuf<double> v(c, n), u(c, m), nrm(c, 1);
  if (start != nullptr) {   // injected start vector (host, n doubles)
    BRSVD_CUDA(cudaMemcpyAsync(v.p, start, sizeof(double) * n, cudaMemcpyHostToDevice,
                               c.stream));
  } else {
    gaussian_kernel<double><<<grid_for(n), 256, 0, c.stream>>>(v.p, n, 1, n, seed, 7, 0);
    BRSVD_CHECK_LAUNCH();
  }
  vec_norm2_kernel<<<1, 1024, 0, c.stream>>>(v.p, n, nrm.p);
  BRSVD_CHECK_LAUNCH();
  vec_scale_kernel<<<grid_for(n), 256, 0, c.stream>>>(v.p, n, nrm.p, 1);
  BRSVD_CHECK_LAUNCH();
  double sigma = 0.0;
  int it = 0;
  for (it = 0; it < max_it; ++it) {
    matvec<T>(c, Mx, m, n, sm, sn, v.p, u.p);
    vec_norm2_kernel<<<1, 1024, 0, c.stream>>>(u.p, m, nrm.p);
    BRSVD_CHECK_LAUNCH();
    double nu;
    readback(c, nrm.p, &nu, sizeof(double));
    if (nu == 0.0) {
      if (iters_out) *iters_out = it + 1;
      return 0.0;
    }
    vec_scale_kernel<<<grid_for(m), 256, 0, c.stream>>>(u.p, m, nrm.p, 1);
    BRSVD_CHECK_LAUNCH();
    matvec<T>(c, Mx, n, m, sn, sm, u.p, v.p);
    vec_norm2_kernel<<<1, 1024, 0, c.stream>>>(v.p, n, nrm.p);
    BRSVD_CHECK_LAUNCH();
    double s_new;
    readback(c, nrm.p, &s_new, sizeof(double));
    vec_scale_kernel<<<grid_for(n), 256, 0, c.stream>>>(v.p, n, nrm.p, 1);
    BRSVD_CHECK_LAUNCH();
    if (std::fabs(s_new - sigma) <= tol * s_new) {
      if (iters_out) *iters_out = it + 1;
      return s_new;
    }
    sigma = s_new;
  }
  if (iters_out) *iters_out = it;
  return sigma;
}

// ---- element passes ------------------------------------------------------------
// Frobenius norm^2 and max |x| of a dense m*n array (block partials).
template <typename T>
__global__ void fro_max_kernel(const T* __restrict__ X, int64_t total,
                               double* __restrict__ part_sq,
                               double* __restrict__ part_max) {
  __shared__ double r1[32], r2[32];
  double s = 0.0, mx = 0.0;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < total;
       i += (int64_t)gridDim.x * blockDim.x) {
    const double v = (double)X[i];
    s = fma(v, v, s);
    mx = fmax(mx, fabs(v));
  }
  s = warp_sum(s);
  mx = warp_max(mx);
  if ((threadIdx.x & 31) == 0) {
    r1[threadIdx.x >> 5] = s;
    r2[threadIdx.x >> 5] = mx;
  }
  __syncthreads();
  if (threadIdx.x == 0) {
    double a = 0.0, b = 0.0;
    for (int w = 0; w < (int)(blockDim.x >> 5); ++w) {
      a += r1[w];
      b = fmax(b, r2[w]);
    }
    part_sq[blockIdx.x] = a;
    if (part_max) part_max[blockIdx.x] = b;
  }
}

// Sum (and max) of nb block partials: one CTA of 1024 threads, each thread a
// fixed strided subset, then a fixed-shape tree -- deterministic.
__global__ void __launch_bounds__(1024)
    sum_max_finalize_kernel(const double* __restrict__ part_sq,
                            const double* __restrict__ part_max, int nb,
                            double* __restrict__ out) {
  __shared__ double r1[32], r2[32];
  double a = 0.0, b = 0.0;
  for (int i = threadIdx.x; i < nb; i += blockDim.x) {
    a += part_sq[i];
    if (part_max) b = fmax(b, part_max[i]);
  }
  a = warp_sum(a);
  b = warp_max(b);
  if ((threadIdx.x & 31) == 0) {
    r1[threadIdx.x >> 5] = a;
    r2[threadIdx.x >> 5] = b;
  }
  __syncthreads();
  if (threadIdx.x < 32) {
    const int nw = blockDim.x >> 5;
    a = threadIdx.x < nw ? r1[threadIdx.x] : 0.0;
    b = threadIdx.x < nw ? r2[threadIdx.x] : 0.0;
    a = warp_sum(a);
    b = warp_max(b);
    if (threadIdx.x == 0) {
      out[0] = a;
      out[1] = b;
    }
  }
}

// Y = scale*M, S = 0, W = M + Y/mu.
template <typename T>
__global__ void rpca_init_kernel(const T* __restrict__ Mx, int64_t total, double scale,
                                 double mu, T* __restrict__ Y, T* __restrict__ S,
                                 T* __restrict__ W) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < total;
       i += (int64_t)gridDim.x * blockDim.x) {
    const T mv = Mx[i];
    const T y = (T)(scale * (double)mv);
    Y[i] = y;
    S[i] = T(0);
    W[i] = mv - T(0) + y / (T)mu;
  }
}

// Fused IALM update.  Element (f, s) of every m x n array sits at s*ld + f
// (f = contiguous index).  F (nf x l) and G (ns x l) are the column-major
// factors indexed by f and s: row-major M -> F = V, G = U; column-major M ->
// F = U, G = V.  The singular values are shrunk on the fly.
//   mode 0: full update (S, Y, W written, ||Z||^2 partials)
//   mode 1: L = F diag(shrink(sigma)) G^T only (written to Lout)
constexpr int kStepLMax = 32;
constexpr int kStepTS = 16;
constexpr int kStepGS = 8;  // rows whose loads are batched

template <typename T, int LMAX>
__global__ void __launch_bounds__(256)
    rpca_step_kernel(int mode, int64_t nf, int64_t ns, int64_t ld, int l,
                     const T* __restrict__ F, int64_t ldf, const T* __restrict__ G,
                     int64_t ldg, const T* __restrict__ sigma, double inv_mu,
                     double lam_over_mu, double mu, double inv_mu_next,
                     const T* __restrict__ Mx, T* __restrict__ Y, T* __restrict__ S,
                     T* __restrict__ W, T* __restrict__ Lout,
                     double* __restrict__ part) {
  __shared__ double Gs[kStepTS][LMAX];
  __shared__ double red[8];
  const int64_t f = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  const int64_t s0 = (int64_t)blockIdx.y * kStepTS;
  // slow-factor tile, shrunk singular values folded in
  for (int e = threadIdx.x; e < kStepTS * LMAX; e += blockDim.x) {
    const int si = e / LMAX, r = e % LMAX;
    double v = 0.0;
    if (r < l && s0 + si < ns) {
      const double sg = (double)sigma[r];
      const double sh = sg > inv_mu ? sg - inv_mu : (sg < -inv_mu ? sg + inv_mu : 0.0);
      v = sh * (double)G[(s0 + si) + (int64_t)r * ldg];
    }
    Gs[si][r] = v;
  }
  double fr[LMAX];
#pragma unroll
  for (int r = 0; r < LMAX; ++r)
    fr[r] = (f < nf && r < l) ? (double)F[f + (int64_t)r * ldf] : 0.0;
  __syncthreads();
  double zz = 0.0;
  if (f < nf) {
    // groups of kStepGS rows: all loads of a group issued before any use
    for (int g0 = 0; g0 < kStepTS; g0 += kStepGS) {
      T mvs[kStepGS], yvs[kStepGS];
      if (mode == 0) {
#pragma unroll
        for (int j = 0; j < kStepGS; ++j) {
          const int64_t s = s0 + g0 + j;
          const bool ok = s < ns;
          mvs[j] = ok ? __ldcs(Mx + s * ld + f) : T(0);
          yvs[j] = ok ? __ldcs(Y + s * ld + f) : T(0);
        }
      }
#pragma unroll
      for (int j = 0; j < kStepGS; ++j) {
        const int64_t s = s0 + g0 + j;
        if (s >= ns) break;
        double L = 0.0;
#pragma unroll
        for (int r = 0; r < LMAX; ++r) L = fma(fr[r], Gs[g0 + j][r], L);
        const int64_t idx = s * ld + f;
        if (mode == 1) {
          Lout[idx] = (T)L;
          continue;
        }
        // the reference evaluates these in the array dtype (rpca.py:195-198)
        const T Lt = (T)L;
        const T mv = mvs[j];
        const T yv = yvs[j];
        const T arg = mv - Lt + yv * (T)inv_mu;
        const T th = (T)lam_over_mu;
        const T sv = arg > th ? arg - th : (arg < -th ? arg + th : T(0));
        const T z = mv - Lt - sv;
        const T yn = yv + (T)mu * z;
        __stcs(S + idx, sv);
        __stcs(Y + idx, yn);
        __stcs(W + idx, mv - sv + yn * (T)inv_mu_next);
        zz = fma((double)z, (double)z, zz);
      }
    }
  }
  if (mode == 1) return;
  zz = warp_sum(zz);
  if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = zz;
  __syncthreads();
  if (threadIdx.x == 0) {
    double t = 0.0;
    for (int w = 0; w < (int)(blockDim.x >> 5); ++w) t += red[w];
    part[blockIdx.y * (int64_t)gridDim.x + blockIdx.x] = t;
  }
}

template <typename T>
void rpca_step(Ctx& c, int mode, int64_t nf, int64_t ns, int64_t ld, int l, const T* F,
               int64_t ldf, const T* G, int64_t ldg, const T* sigma, double mu,
               double lam, double rho, const T* Mx, T* Y, T* S, T* W, T* Lout,
               double* part, int64_t* nparts) {
  dim3 grid((unsigned)ceil_div(nf, 256), (unsigned)ceil_div(ns, kStepTS));
  if (nparts) *nparts = (int64_t)grid.x * grid.y;
  const double inv_mu = 1.0 / mu, lm = lam / mu, inv_next = 1.0 / (mu * rho);
#define BRSVD_STEP(LM)                                                              \
  rpca_step_kernel<T, LM><<<grid, 256, 0, c.stream>>>(                              \
      mode, nf, ns, ld, l, F, ldf, G, ldg, sigma, inv_mu, lm, mu, inv_next, Mx, Y, \
      S, W, Lout, part)
  if (l <= 8) BRSVD_STEP(8);
  else if (l <= 16) BRSVD_STEP(16);
  else if (l <= 24) BRSVD_STEP(24);
  else if (l <= 32) BRSVD_STEP(32);
  else if (l <= 64) BRSVD_STEP(64);
  else throw Error(kErrConfig, "ialm_rpca on the GPU supports k + p <= 64");
#undef BRSVD_STEP
  BRSVD_CHECK_LAUNCH();
}

struct IalmOut {
  int iterations = 0;
  bool converged = false;
};

// The IALM loop (rpca.py:168-213).  Mx (device, m x n, row- or column-major,
// dense).  L and S are written (device, same layout).  History arrays (host)
// have max_it entries.
template <typename T>
IalmOut ialm_device(Ctx& c, const T* Mx, int64_t m, int64_t n, bool row_major, int k,
                    int p, int q, uint64_t seed, const T* omega, double lam, double mu0,
                    double rho,
                    double tol, int max_it, T* Lout, T* Sout, double* residuals,
                    double* mus, double* svd_s, double* iter_s,
                    const int64_t* blocks = nullptr, int nblk = 0) {
  const int l = k + p;
  const int64_t total = m * n;
  const int64_t ld = row_major ? n : m;
  const int64_t sm = row_major ? n : 1, sn = row_major ? 1 : m;
  if (std::isnan(lam)) lam = 1.0 / std::sqrt((double)std::max(m, n));
  const double norm2 = spectral_norm<T>(c, Mx, m, n, sm, sn, seed, 1e-10, 100, nullptr);
  BRSVD_REQUIRE(norm2 != 0.0, kErrArg, "RPCA input is the zero matrix");
  double mu = std::isnan(mu0) ? 1.25 / norm2 : mu0;
  // ||M||_F and max |M|
  const int nb = grid_for(total, 256, 148 * 8);
  DBuf<double> psq(c, nb), pmx(c, nb), sc(c, 2);
  fro_max_kernel<T><<<nb, 256, 0, c.stream>>>(Mx, total, psq.p, pmx.p);
  BRSVD_CHECK_LAUNCH();
  sum_max_finalize_kernel<<<1, 1024, 0, c.stream>>>(psq.p, pmx.p, nb, sc.p);
  BRSVD_CHECK_LAUNCH();
  double hs[2];
  readback(c, sc.p, hs, sizeof(hs));
  const double norm_f = std::sqrt(hs[0]);
  const double scale = 1.0 / std::max(norm2, hs[1] / lam);
  DBuf<T> Y(c, (size_t)total), W(c, (size_t)total);
  T* S = Sout;
  rpca_init_kernel<T><<<grid_for(total, 256, 148 * 16), 256, 0, c.stream>>>(
      Mx, total, scale, mu, Y.p, S, W.p);
  BRSVD_CHECK_LAUNCH();
  DBuf<T> Om(c, (size_t)n * l), U(c, (size_t)m * l), V(c, (size_t)n * l), sig(c, l);
  if (omega != nullptr) {
    BRSVD_CUDA(cudaMemcpyAsync(Om.p, omega, sizeof(T) * n * l, cudaMemcpyDeviceToDevice,
                               c.stream));
  } else {
    gaussian_kernel<T><<<grid_for(n * ((l + 1) / 2)), 256, 0, c.stream>>>(Om.p, n, l, n,
                                                                           seed, 0, 0);
    BRSVD_CHECK_LAUNCH();
  }
  const int64_t nf = row_major ? n : m, ns = row_major ? m : n;
  const T* F = row_major ? V.p : U.p;
  const T* G = row_major ? U.p : V.p;
  const int64_t ldf = row_major ? n : m, ldg = row_major ? m : n;
  const int64_t nparts_max = ceil_div(nf, 256) * ceil_div(ns, kStepTS);
  DBuf<double> part(c, (size_t)nparts_max), zsum(c, 2);
  StageEvents ev;
  IalmOut out;
  for (int it = 1; it <= max_it; ++it) {
    const auto t0 = std::chrono::steady_clock::now();
    ev.rec(0, c.stream);
    // blocks: the reference's out-of-core branch runs brsvd_run with the
    // budget's column blocks (per-block power iteration, rpca.py:274)
    rsvd_device<T>(c, W.p, m, n, ld, row_major, k, p, q, Om.p, seed, U.p, sig.p, V.p,
                   nullptr, blocks, nblk);
    ev.rec(1, c.stream);
    int64_t np = 0;
    rpca_step<T>(c, 0, nf, ns, ld, l, F, ldf, G, ldg, sig.p, mu, lam, rho, Mx, Y.p, S,
                 W.p, nullptr, part.p, &np);
    sum_max_finalize_kernel<<<1, 1024, 0, c.stream>>>(part.p, nullptr, (int)np, zsum.p);
    BRSVD_CHECK_LAUNCH();
    double z2[2];
    readback(c, zsum.p, z2, sizeof(z2));
    const double residual = std::sqrt(z2[0]) / norm_f;
    const auto t1 = std::chrono::steady_clock::now();
    residuals[it - 1] = residual;
    mus[it - 1] = mu;
    svd_s[it - 1] = ev.ms(0, 1) * 1e-3;
    iter_s[it - 1] = std::chrono::duration<double>(t1 - t0).count();
    out.iterations = it;
    if (residual < tol) {
      out.converged = true;
      break;
    }
    if (it < max_it) mu *= rho;
  }
  // L from the last factors and the last mu (rpca.py:194-195)
  rpca_step<T>(c, 1, nf, ns, ld, l, F, ldf, G, ldg, sig.p, mu, lam, rho, Mx, nullptr,
               nullptr, nullptr, Lout, nullptr, nullptr);
  return out;
}

}  // namespace brsvd
