// In-core randomized SVD pipeline (global power iteration).
//
// Semantics follow rsvd_incore (rsvd.py:126-141): Y = (A A^T)^q A Omega,
// Q = orth(Y), B = Q^T A, B = W S Vt, U = Q W, canonical signs.  The power
// iteration is evaluated with a basis change of Z = A^T Y between passes
// (normalize_sketch): same column space in exact arithmetic, so the factors
// match the reference's to rounding while the sketch never overflows or loses
// rank to cancellation.
#pragma once
#include "orth.cuh"

namespace brsvd {

struct RsvdInfo {
  int rank_y = 0, rank_b = 0;
  double max_abs_y0 = 0.0;
  double log10_peak = 0.0;
  bool overflow = false;
  int64_t words_read = 0, block_reads = 0;
  float ms_sketch = 0, ms_orth = 0, ms_core = 0, ms_svd = 0;
};

template <typename T>
constexpr double finfo_max() {
  return sizeof(T) == 8 ? 1.7976931348623157e308 : 3.4028234663852886e38;
}

struct StageEvents {
  cudaEvent_t ev[5];
  StageEvents() {
    for (auto& e : ev) BRSVD_CUDA(cudaEventCreate(&e));
  }
  ~StageEvents() {
    for (auto& e : ev) cudaEventDestroy(e);
  }
  void rec(int i, cudaStream_t s) { BRSVD_CUDA(cudaEventRecord(ev[i], s)); }
  float ms(int a, int b) {
    float t = 0;
    cudaEventElapsedTime(&t, ev[a], ev[b]);
    return t;
  }
};

template <typename T>
RsvdInfo rsvd_device(Ctx& c, const T* A, int64_t m, int64_t n, int64_t lda,
                     bool row_major, int k, int p, int q, const T* omega,
                     uint64_t seed, T* U, T* sigma, T* V) {
  const int l = k + p;
  RsvdInfo info;
  StageEvents ev;
  ev.rec(0, c.stream);
  DBuf<T> Xg;
  const T* X = omega;
  if (X == nullptr) {
    Xg.alloc(c, (size_t)n * l);
    gaussian_kernel<T><<<grid_for(n * ((l + 1) / 2)), 256, 0, c.stream>>>(
        Xg.p, n, l, n, seed, 0, 0);
    BRSVD_CHECK_LAUNCH();
    X = Xg.p;
  }
  DBuf<T> Y(c, (size_t)m * l), Z(c, (size_t)n * l), Zn(c, (size_t)n * l);
  big_nn<T>(c, A, m, n, lda, row_major, X, n, l, Y.p, m);
  const MaxAbs p0 = maxabs<T>(c, Y.p, m, l, m);
  info.max_abs_y0 = p0.peak;
  bool nonfinite = p0.nonfinite;
  if (nonfinite) {  // the reference's guard fires on the first sample already
    info.overflow = true;
    info.log10_peak = INFINITY;
    return info;
  }
  for (int it = 0; it < q; ++it) {
    big_tn<T>(c, A, m, n, lda, row_major, Y.p, m, l, Z.p, n);
    normalize_sketch<T>(c, Z.p, n, l, n, Zn.p, n);
    big_nn<T>(c, A, m, n, lda, row_major, Zn.p, n, l, Y.p, m);
  }
  info.words_read += (int64_t)(2 * q + 1) * m * n;
  info.block_reads += 2 * q + 1;
  if (q > 0) {
    const MaxAbs pq = maxabs<T>(c, Y.p, m, l, m);
    if (pq.nonfinite) {
      info.overflow = true;
      info.log10_peak = INFINITY;
      return info;
    }
  }
  ev.rec(1, c.stream);
  Zn.release();
  Z.release();
  const int ns = sizeof(T) == 8 ? 2 : 1;
  DBuf<T> Qw(c, (size_t)m * l);
  info.rank_y = orth_full<T>(c, Y.p, m, l, m, Qw.p, seed ^ 0x7153ull, ns);
  Y.release();
  const T* Qop = Qw.p;
  ev.rec(2, c.stream);
  DBuf<T> Bt(c, (size_t)n * l);
  big_tn<T>(c, A, m, n, lda, row_major, Qop, m, l, Bt.p, n);
  info.words_read += m * n;
  info.block_reads += 1;
  ev.rec(3, c.stream);
  DBuf<double> W(c, (size_t)l * l), sig(c, l);
  info.rank_b = small_svd_device<T>(c, Bt.p, n, l, n, W.p, sig.p, V, n, ns);
  apply_basis<T>(c, Qw.p, m, l, m, W.p, l, l, U, m);
  fix_signs<T>(c, U, m, l, m, V, n, n);
  copy2d_kernel<double, T><<<1, 256, 0, c.stream>>>(sig.p, l, 1, l, sigma, l);
  BRSVD_CHECK_LAUNCH();
  ev.rec(4, c.stream);
  double s0 = 0.0;
  BRSVD_CUDA(cudaMemcpyAsync(c.h_pinned, sig.p, sizeof(double),
                             cudaMemcpyDeviceToHost, c.stream));
  BRSVD_CUDA(cudaStreamSynchronize(c.stream));
  std::memcpy(&s0, c.h_pinned, sizeof(double));
  info.ms_sketch = ev.ms(0, 1);
  info.ms_orth = ev.ms(1, 2);
  info.ms_core = ev.ms(2, 3);
  info.ms_svd = ev.ms(3, 4);
  // Overflow guard of the unnormalised reference iteration: its sample is
  // (A A^T)^q A Omega, whose peak grows like max|A Omega| * sigma_1^(2q).
  const double lim = std::log10(0.01 * finfo_max<T>());
  if (info.max_abs_y0 > 0.0 && s0 > 0.0)
    info.log10_peak = std::log10(info.max_abs_y0) + 2.0 * q * std::log10(s0);
  else
    info.log10_peak = info.max_abs_y0 > 0.0 ? std::log10(info.max_abs_y0) : -400.0;
  info.overflow = nonfinite || !std::isfinite(s0) || info.log10_peak > lim;
  return info;
}

}  // namespace brsvd
