// In-core randomized SVD pipeline (global power iteration).
//
// Semantics follow rsvd_incore (rsvd.py:126-141): Y = (A A^T)^q A Omega,
// Q = orth(Y), B = Q^T A, B = W S Vt, U = Q W, canonical signs.  The power
// iteration is evaluated with a basis change of Z = A^T Y between passes
// (normalize_sketch): same column space in exact arithmetic, so the factors
// match the reference's to rounding while the sketch never overflows or loses
// rank to cancellation.
#pragma once
#include <vector>
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

// Host-resident input: A (device, ld lda, allocated by the caller) is filled
// from host memory by the pipeline itself so that the H2D transfer overlaps
// the sample pass.  Row-major A arrives in row panels on a copy stream and
// Y[rows] = A[rows, :] X is computed per panel as soon as it lands (the
// remaining passes need all of A); column-major A is copied whole first.
struct HostFeed {
  const void* host = nullptr;
  int64_t ldh = 0;   // host leading dimension (elements)
  int panels = 8;
};

template <typename T>
__global__ void sum_slices_kernel(const T* __restrict__ parts, int64_t count, int slices,
                                  T* __restrict__ out) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < count;
       i += (int64_t)gridDim.x * blockDim.x) {
    T s = T(0);
    for (int z = 0; z < slices; ++z) s += parts[(int64_t)z * count + i];
    out[i] = s;
  }
}

// Returns true when Z = A^T Y (n x l) was also formed panel by panel
// (Z += A_i^T Y_i, the fused power step of the north star: each panel is used
// for both products while it is fresh), so the first transpose pass is done
// by the time the transfer completes.
// Row / column maxima of |A| for the fp16-split products (fp32 data only).
template <typename T>
bool want_amax(Ctx& c, const T* A, int64_t lda, int64_t m, int64_t n, int l) {
  return sizeof(T) == 4 && tc::h16_enabled() && tc_gemm_supported<T>(c, A, lda, m, n, l);
}

template <typename T>
bool feed_and_sample(Ctx& c, T* A, int64_t m, int64_t n, int64_t lda, bool row_major,
                     const HostFeed& f, const T* X, int l, T* Y, T* Z, float* arow,
                     float* acol) {
  const int64_t a_rows = row_major ? n : m, a_cols = row_major ? m : n;
  if (!row_major) {
    BRSVD_CUDA(cudaMemcpy2DAsync(A, lda * sizeof(T), f.host, f.ldh * sizeof(T),
                                 a_rows * sizeof(T), a_cols, cudaMemcpyHostToDevice,
                                 c.stream));
    if (arow)
      absmax_rows_cols(c, reinterpret_cast<const float*>(A), m, n, lda, row_major, arow, acol,
                       /*init=*/false);
    big_nn<T>(c, A, m, n, lda, row_major, X, n, l, Y, m, arow);
    return false;
  }
  cudaStream_t cs;
  BRSVD_CUDA(cudaStreamCreateWithFlags(&cs, cudaStreamNonBlocking));
  cudaEvent_t ready;
  BRSVD_CUDA(cudaEventCreateWithFlags(&ready, cudaEventDisableTiming));
  // the copy stream must not overwrite A before earlier work on it finished
  BRSVD_CUDA(cudaEventRecord(ready, c.stream));
  BRSVD_CUDA(cudaStreamWaitEvent(cs, ready, 0));
  const int P = (int)std::max<int64_t>(1, std::min<int64_t>(f.panels, m / 128));
  const int64_t step = ceil_div(ceil_div(m, P), 128) * 128;
  const int npan = (int)ceil_div(m, step);
  DBuf<T> Zp;
  if (Z != nullptr) Zp.alloc(c, (size_t)npan * n * l);
  std::vector<cudaEvent_t> evs;
  int pi = 0;
  for (int64_t r0 = 0; r0 < m; r0 += step, ++pi) {
    const int64_t r1 = std::min(m, r0 + step);
    const T* src = reinterpret_cast<const T*>(f.host) + r0 * f.ldh;
    BRSVD_CUDA(cudaMemcpy2DAsync(A + r0 * lda, lda * sizeof(T), src, f.ldh * sizeof(T),
                                 n * sizeof(T), r1 - r0, cudaMemcpyHostToDevice, cs));
    cudaEvent_t e;
    BRSVD_CUDA(cudaEventCreateWithFlags(&e, cudaEventDisableTiming));
    BRSVD_CUDA(cudaEventRecord(e, cs));
    evs.push_back(e);
    BRSVD_CUDA(cudaStreamWaitEvent(c.stream, e, 0));
    // panel maxima: rows land in arow[r0:r1], columns accumulate over panels
    if (arow)
      absmax_rows_cols(c, reinterpret_cast<const float*>(A + r0 * lda), r1 - r0, n, lda, true,
                       arow + r0, acol, /*init=*/false);
    big_nn<T>(c, A + r0 * lda, r1 - r0, n, lda, true, X, n, l, Y + r0, m,
              arow ? arow + r0 : nullptr);
    if (Z != nullptr)
      big_tn<T>(c, A + r0 * lda, r1 - r0, n, lda, true, Y + r0, m, l,
                Zp.p + (int64_t)pi * n * l, n, acol);
  }
  if (Z != nullptr) {
    sum_slices_kernel<T><<<grid_for(n * l), 256, 0, c.stream>>>(Zp.p, n * l, npan, Z);
    BRSVD_CHECK_LAUNCH();
  }
  for (auto e : evs) cudaEventDestroy(e);
  cudaEventDestroy(ready);
  cudaStreamDestroy(cs);  // returns at once; the stream is released when its work is done
  return Z != nullptr;
}

template <typename T>
__global__ void axpy_kernel(const T* __restrict__ x, int64_t rows, int64_t cols, int64_t ldx,
                            T* __restrict__ y, int64_t ldy) {
  const int64_t total = rows * cols;
  for (int64_t id = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; id < total;
       id += (int64_t)gridDim.x * blockDim.x) {
    const int64_t i = id % rows, j = id / rows;
    y[i + j * ldy] += x[i + j * ldx];
  }
}

template <typename T>
void axpy(Ctx& c, const T* x, int64_t rows, int64_t cols, int64_t ldx, T* y, int64_t ldy) {
  axpy_kernel<T><<<grid_for(rows * cols), 256, 0, c.stream>>>(x, rows, cols, ldx, y, ldy);
  BRSVD_CHECK_LAUNCH();
}

// Paper-literal block sketch (block_range_finder, rsvd.py:150-185; PAPER.md
// Alg. 2): Y = sum_J (A_J A_J^T)^q A_J Omega_J over the column blocks J of the
// plan, each block's power iteration run to completion on the block (no
// normalisation, like the reference), the block samples summed.  For q = 0
// or one block this equals the global sample.
template <typename T>
void paper_sketch(Ctx& c, const T* A, int64_t m, int64_t n, int64_t lda, bool row_major,
                  const T* X, int l, int q, const int64_t* bounds, int nblk, T* Y,
                  const float* arow, const float* acol) {
  int64_t wmax = 0;
  for (int b = 0; b < nblk; ++b) wmax = std::max(wmax, bounds[b + 1] - bounds[b]);
  DBuf<T> YJ(c, (size_t)m * l), ZJ(c, (size_t)std::max<int64_t>(wmax, 1) * l);
  BRSVD_CUDA(cudaMemsetAsync(Y, 0, sizeof(T) * m * l, c.stream));
  for (int b = 0; b < nblk; ++b) {
    const int64_t j0 = bounds[b], w = bounds[b + 1] - bounds[b];
    if (w <= 0) continue;
    const T* AJ = row_major ? A + j0 : A + j0 * lda;
    big_nn<T>(c, AJ, m, w, lda, row_major, X + j0, n, l, YJ.p, m, arow);
    for (int it = 0; it < q; ++it) {
      big_tn<T>(c, AJ, m, w, lda, row_major, YJ.p, m, l, ZJ.p, w, acol ? acol + j0 : nullptr);
      big_nn<T>(c, AJ, m, w, lda, row_major, ZJ.p, w, l, YJ.p, m, arow);
    }
    axpy_kernel<T><<<grid_for(m * l), 256, 0, c.stream>>>(YJ.p, m, l, m, Y, m);
    BRSVD_CHECK_LAUNCH();
  }
}

// Exact overflow guard of the global power iteration (rsvd.py:84-91).  The
// sample the reference tests is Y_ref = (A A^T)^q A Omega; ours is
// Y_q = Y_ref C with C = prod_i (z_i T_i) (z_i the power-of-two scale of
// A^T Y, T_i the upper-triangular Cholesky basis change actually applied),
// so max |Y_ref| = max |Y_q C^-1|, formed in fp64 (its entries may exceed
// the data's range -- that is what the guard detects).  Ts holds the q
// transforms (l x l each); returns the exact peak.
template <typename T>
double unnormalised_peak(Ctx& c, const T* Yq, int64_t m, int l, int q, const double* Ts,
                         const double* zfac) {
  DBuf<double> P(c, (size_t)l * l), Ti(c, (size_t)l * l), Pn(c, (size_t)l * l);
  eye_kernel<double><<<grid_for((int64_t)l * l), 256, 0, c.stream>>>(P.p, l);
  BRSVD_CHECK_LAUNCH();
  double scale = 1.0;
  for (int it = 0; it < q; ++it) {   // P <- T_it^-1 P  (C^-1 = T_q^-1 ... T_1^-1)
    triu_inverse_kernel<<<1, 512, 0, c.stream>>>(Ts + (size_t)it * l * l, l, Ti.p);
    BRSVD_CHECK_LAUNCH();
    gemm_nn_cm<double, double, double>(c, l, l, l, Ti.p, l, P.p, l, Pn.p, l);
    std::swap(P.p, Pn.p);
    scale *= zfac[it];
  }
  DBuf<double> Yr(c, (size_t)m * l);
  gemm_nn_cm<T, double, double>(c, m, l, l, Yq, m, P.p, l, Yr.p, m);
  const MaxAbs pk = maxabs<double>(c, Yr.p, m, l, m);
  return pk.nonfinite ? INFINITY : pk.peak / scale;
}

// fp16-split scales without an up-front pass over A.  The products need
// per-line power-of-two scales of A (rows for Y = A X, columns for A^T Y); a
// full absmax pass costs as much HBM traffic as a sixth of a product.  The
// first product of each orientation instead runs on SAMPLED maxima
// (amax_sampled: 1/16 of A) and, as its converters see every entry, writes
// the exact maxima; a check kernel flags any line whose exact maximum the
// sampled scale does not serve at full precision, and the same product is
// launched again on the exact scales -- a launch that returns at once unless
// flagged.  Later products use the exact maxima.  Only the single-chunk pair
// kernel produces maxima (tcw_selected); otherwise the pass runs as before.
struct LazyScales {
  bool pend_r = false, pend_c = false;
  DBuf<float> gr, gc;   // sampled maxima x 2^7
  DBuf<int> flag;       // [2]: rows, columns
};

template <typename T>
bool lazy_scales_ok(Ctx& c, int l) {
  if (sizeof(T) != 4 || !tcw_selected(c, l)) return false;
  const char* e = std::getenv("BRSVD_LAZY_SCALES");
  return !(e && e[0] == '0');
}

template <typename T>
void nn_product(Ctx& c, LazyScales& lz, const T* A, int64_t m, int64_t n, int64_t lda,
                bool row_major, const T* X, int64_t ldx, int l, T* Y, int64_t ldy,
                float* arow) {
  if (lz.pend_r) {
    lz.pend_r = false;
    if (tcw_selected(c, l)) {
      big_nn<T>(c, A, m, n, lda, row_major, X, ldx, l, Y, ldy, lz.gr.p,
                reinterpret_cast<unsigned*>(arow));
      tc::lazy_scale_check_kernel<<<grid_for(m), 256, 0, c.stream>>>(lz.gr.p, arow, m,
                                                                      lz.flag.p);
      BRSVD_CHECK_LAUNCH();
      big_nn<T>(c, A, m, n, lda, row_major, X, ldx, l, Y, ldy, arow, nullptr, lz.flag.p);
      return;
    }
    absmax_rows_cols(c, reinterpret_cast<const float*>(A), m, n, lda, row_major, arow,
                     nullptr);
  }
  big_nn<T>(c, A, m, n, lda, row_major, X, ldx, l, Y, ldy, arow);
}

template <typename T>
void tn_product(Ctx& c, LazyScales& lz, const T* A, int64_t m, int64_t n, int64_t lda,
                bool row_major, const T* Yin, int64_t ldy, int l, T* Z, int64_t ldz,
                float* acol, double out_scale = 1.0) {
  if (lz.pend_c) {
    lz.pend_c = false;
    if (tcw_selected(c, l)) {
      big_tn<T>(c, A, m, n, lda, row_major, Yin, ldy, l, Z, ldz, lz.gc.p, out_scale,
                reinterpret_cast<unsigned*>(acol));
      tc::lazy_scale_check_kernel<<<grid_for(n), 256, 0, c.stream>>>(lz.gc.p, acol, n,
                                                                      lz.flag.p + 1);
      BRSVD_CHECK_LAUNCH();
      big_tn<T>(c, A, m, n, lda, row_major, Yin, ldy, l, Z, ldz, acol, out_scale, nullptr,
                lz.flag.p + 1);
      return;
    }
    absmax_rows_cols(c, reinterpret_cast<const float*>(A), m, n, lda, row_major, nullptr,
                     acol);
  }
  big_tn<T>(c, A, m, n, lda, row_major, Yin, ldy, l, Z, ldz, acol, out_scale);
}

// range_only: stop after the orthonormal basis of the sample (block_range_finder,
// rsvd.py:150-185); Q (m x l) is written to U.
template <typename T>
RsvdInfo rsvd_device(Ctx& c, const T* A, int64_t m, int64_t n, int64_t lda,
                     bool row_major, int k, int p, int q, const T* omega,
                     uint64_t seed, T* U, T* sigma, T* V, const HostFeed* feed = nullptr,
                     const int64_t* blocks = nullptr, int nblk = 0, bool range_only = false) {
  const bool paper = blocks != nullptr && nblk > 1 && q > 0;
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
  // per-row / per-column maxima of |A| (one pass, reused by every product)
  DBuf<float> arow, acol;
  LazyScales lz;
  if (want_amax<T>(c, A, lda, m, n, l)) {
    arow.alloc(c, (size_t)m);
    acol.alloc(c, (size_t)n);
    if (feed == nullptr && !paper && lazy_scales_ok<T>(c, l)) {
      lz.gr.alloc(c, (size_t)m);
      lz.gc.alloc(c, (size_t)n);
      lz.flag.alloc(c, 2);
      BRSVD_CUDA(cudaMemsetAsync(lz.flag.p, 0, 2 * sizeof(int), c.stream));
      BRSVD_CUDA(cudaMemsetAsync(arow.p, 0, sizeof(float) * m, c.stream));
      BRSVD_CUDA(cudaMemsetAsync(acol.p, 0, sizeof(float) * n, c.stream));
      amax_sampled(c, reinterpret_cast<const float*>(A), m, n, lda, row_major, lz.gr.p,
                   lz.gc.p);
      lz.pend_r = lz.pend_c = true;
    } else if (feed == nullptr) {
      absmax_rows_cols(c, reinterpret_cast<const float*>(A), m, n, lda, row_major, arow.p,
                       acol.p);
    } else {  // the feed accumulates panel by panel
      BRSVD_CUDA(cudaMemsetAsync(arow.p, 0, sizeof(float) * m, c.stream));
      BRSVD_CUDA(cudaMemsetAsync(acol.p, 0, sizeof(float) * n, c.stream));
    }
  }
  bool z_ready = false;
  if (paper) {
    if (feed != nullptr) {  // land A first; the block sketch revisits every block q times
      const int64_t a_rows = row_major ? n : m, a_cols = row_major ? m : n;
      BRSVD_CUDA(cudaMemcpy2DAsync(const_cast<T*>(A), lda * sizeof(T), feed->host,
                                   feed->ldh * sizeof(T), a_rows * sizeof(T), a_cols,
                                   cudaMemcpyHostToDevice, c.stream));
      if (arow.p)
        absmax_rows_cols(c, reinterpret_cast<const float*>(A), m, n, lda, row_major, arow.p,
                         acol.p, false);
    }
    paper_sketch<T>(c, A, m, n, lda, row_major, X, l, q, blocks, nblk, Y.p, arow.p, acol.p);
  } else if (feed != nullptr) {
    z_ready = feed_and_sample<T>(c, const_cast<T*>(A), m, n, lda, row_major, *feed, X, l, Y.p,
                                 q > 0 ? Z.p : nullptr, arow.p, acol.p);
  } else {
    PowerLowp lowp(c);
    nn_product<T>(c, lz, A, m, n, lda, row_major, X, n, l, Y.p, m, arow.p);
  }
  const MaxAbs p0 = maxabs<T>(c, Y.p, m, l, m);
  info.max_abs_y0 = p0.peak;
  bool nonfinite = p0.nonfinite;
  if (nonfinite) {  // the reference's guard fires on the first sample already
    info.overflow = true;
    info.log10_peak = INFINITY;
    return info;
  }
  // A^T Y scaled by 2^-e (e = exponent of max |Y0|): Y and A^T Y of inputs
  // far from unit magnitude stay in fp32 range (Z is renormalised next)
  double zscale = 1.0;
  if (sizeof(T) == 4 && p0.peak > 0.0) {
    int e;
    std::frexp(p0.peak, &e);
    zscale = std::ldexp(1.0, -e);
    // the feed's fused A_i^T Y_i ran unscaled: keep it only when Y0 is of
    // ordinary magnitude, else recompute A^T Y scaled (A is resident now)
    if (e < -40 || e > 40) z_ready = false;
  }
  // fp64 inputs of extreme magnitude: A^T Y would square it in the Gram of the
  // basis change, so that Gram is formed at unit scale (normalize_sketch)
  const bool f64_extreme =
      sizeof(T) == 8 && (p0.peak > 0x1p150 || (p0.peak > 0.0 && p0.peak < 0x1p-150));
  // the applied basis changes, for the exact overflow guard (Cholesky route)
  const bool track = !paper && q > 0 && l <= kCholMaxL;
  DBuf<double> Ts;
  std::vector<double> zfac;
  if (track) Ts.alloc(c, (size_t)q * l * l);
  for (int it = 0; it < (paper ? 0 : q); ++it) {
    const bool fused = it == 0 && z_ready;   // the feed's A^T Y ran unscaled
    PowerLowp lowp(c);
    if (!fused)
      tn_product<T>(c, lz, A, m, n, lda, row_major, Y.p, m, l, Z.p, n, acol.p, zscale);
    zfac.push_back(fused ? 1.0 : zscale);
    {
      const bool keep = c.b_hi_only;   // the basis change stays three-term
      c.b_hi_only = false;
      normalize_sketch<T>(c, Z.p, n, l, n, Zn.p, n, track ? Ts.p + (size_t)it * l * l : nullptr,
                          f64_extreme);
      c.b_hi_only = keep;
    }
    nn_product<T>(c, lz, A, m, n, lda, row_major, Zn.p, n, l, Y.p, m, arow.p);
  }
  info.words_read += (int64_t)(2 * q + 1) * m * n;
  info.block_reads += 2 * q + 1;
  double ypeak = p0.peak;   // max |Y| of the sample being orthonormalised
  // fp32 (the peak only steers fp64 scaling): the non-finite check of the
  // powered sample is read at the final synchronisation instead of here
  DBuf<unsigned long long> yq_chk;
  const bool yq_defer = sizeof(T) == 4 && q > 0 && !range_only && !std::getenv("BRSVD_DEBUG");
  if (yq_defer) {
    yq_chk.alloc(c, 2);
    BRSVD_CUDA(cudaMemsetAsync(yq_chk.p, 0, 2 * sizeof(unsigned long long), c.stream));
    maxabs_kernel<T><<<grid_for(m * l), 256, 0, c.stream>>>(Y.p, m, l, m, yq_chk.p);
    BRSVD_CHECK_LAUNCH();
  } else if (q > 0) {
    const MaxAbs pq = maxabs<T>(c, Y.p, m, l, m);
    ypeak = pq.peak;
    if (std::getenv("BRSVD_DEBUG"))
      std::fprintf(stderr, "[brsvd] sample peak %.3e -> after %d passes %.3e%s\n", p0.peak, q,
                   pq.peak, pq.nonfinite ? " (non-finite)" : "");
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
  const bool y_extreme = ypeak > 0x1p400 || (ypeak > 0.0 && ypeak < 0x1p-400);
  // ranks of the fp32 path are read at the final synchronisation (no host
  // read in the middle of the pipeline); -1 until then
  DBuf<int> ranks(c, 2);
  info.rank_y = orth_full<T>(c, Y.p, m, l, m, Qw.p, seed ^ 0x7153ull, ns, y_extreme,
                             range_only ? nullptr : ranks.p);
  const double lim = 0.01 * finfo_max<T>();
  if (range_only) {
    BRSVD_CUDA(cudaMemcpyAsync(U, Qw.p, sizeof(T) * m * l, cudaMemcpyDeviceToDevice,
                               c.stream));
    ev.rec(2, c.stream);
    double peak = info.max_abs_y0;            // paper mode: the sample is unnormalised
    if (track) peak = unnormalised_peak<T>(c, Y.p, m, l, q, Ts.p, zfac.data());
    info.log10_peak = peak > 0.0 ? std::log10(peak) : -400.0;
    info.overflow = !(peak <= lim);
    info.ms_sketch = ev.ms(0, 1);
    info.ms_orth = ev.ms(1, 2);
    return info;
  }
  const T* Qop = Qw.p;
  ev.rec(2, c.stream);
  DBuf<T> Bt(c, (size_t)n * l);
  tn_product<T>(c, lz, A, m, n, lda, row_major, Qop, m, l, Bt.p, n, acol.p);
  info.words_read += m * n;
  info.block_reads += 1;
  ev.rec(3, c.stream);
  DBuf<double> W(c, (size_t)l * l), sig(c, l);
  info.rank_b = small_svd_device<T>(c, Bt.p, n, l, n, W.p, sig.p, V, n, ns, ranks.p + 1);
  apply_basis<T>(c, Qw.p, m, l, m, W.p, l, l, U, m);
  fix_signs<T>(c, U, m, l, m, V, n, n);
  copy2d_kernel<double, T><<<1, 256, 0, c.stream>>>(sig.p, l, 1, l, sigma, l);
  BRSVD_CHECK_LAUNCH();
  ev.rec(4, c.stream);
  double s0 = 0.0;
  BRSVD_CUDA(cudaMemcpyAsync(c.h_pinned, sig.p, sizeof(double),
                             cudaMemcpyDeviceToHost, c.stream));
  BRSVD_CUDA(cudaMemcpyAsync(c.h_pinned + 1, ranks.p, 2 * sizeof(int), cudaMemcpyDeviceToHost,
                             c.stream));
  c.h_pinned[2] = 0;
  if (yq_defer)
    BRSVD_CUDA(cudaMemcpyAsync(c.h_pinned + 2, yq_chk.p + 1, sizeof(unsigned long long),
                               cudaMemcpyDeviceToHost, c.stream));
  BRSVD_CUDA(cudaStreamSynchronize(c.stream));
  std::memcpy(&s0, c.h_pinned, sizeof(double));
  {
    int rk[2];
    std::memcpy(rk, c.h_pinned + 1, sizeof(rk));
    if (info.rank_y < 0) info.rank_y = rk[0];
    if (info.rank_b < 0) info.rank_b = rk[1];
  }
  if (c.h_pinned[2] != 0) {   // the powered sample was non-finite (deferred check)
    info.overflow = true;
    info.log10_peak = INFINITY;
    return info;
  }
  info.ms_sketch = ev.ms(0, 1);
  info.ms_orth = ev.ms(1, 2);
  info.ms_core = ev.ms(2, 3);
  info.ms_svd = ev.ms(3, 4);
  // Overflow guard of the unnormalised reference iteration (rsvd.py:84-91):
  // its sample (A A^T)^q A Omega peaks below max|A Omega| sqrt(m) s_1^(2q).
  // Far below the threshold that bound settles it; near or above it the
  // peak is formed exactly (unnormalised_peak).  The paper-mode sample is the
  // unnormalised one already, so its max is exact.
  const double loglim = std::log10(lim);
  const int qg = paper ? 0 : q;
  if (info.max_abs_y0 > 0.0 && s0 > 0.0)
    info.log10_peak = std::log10(info.max_abs_y0) + 2.0 * qg * std::log10(s0);
  else
    info.log10_peak = info.max_abs_y0 > 0.0 ? std::log10(info.max_abs_y0) : -400.0;
  bool over = nonfinite || !std::isfinite(s0);
  if (!over && qg > 0) {
    const double bound = info.log10_peak + 0.5 * std::log10((double)m) + 0.05;
    if (bound > loglim) {
      if (track) {
        const double peak = unnormalised_peak<T>(c, Y.p, m, l, q, Ts.p, zfac.data());
        info.log10_peak = peak > 0.0 ? std::log10(peak) : -400.0;
        over = !(peak <= lim);
      } else {
        over = info.log10_peak > loglim;   // l > kCholMaxL: estimate
      }
    }
  } else if (!over) {
    over = info.max_abs_y0 > lim;
  }
  info.overflow = over;
  return info;
}

}  // namespace brsvd
