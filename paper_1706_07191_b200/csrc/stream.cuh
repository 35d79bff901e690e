// Out-of-core randomized SVD: A stays in host memory and is streamed over
// PCIe in panels (brsvd_run / rsvd_naive_ooc, rsvd.py:188-284, with the
// global power iteration of rsvd_incore).
//
// Panels go through a ring of NB device buffers: a dedicated copy stream
// issues cudaMemcpy2DAsync (pinned host memory makes it a true async DMA)
// while the compute stream runs the products on the previous panel; events
// order buffer reuse.  Each panel crosses PCIe once per pass and is read
// twice from HBM when a pass needs both products:
//   row panels (row-major A):   Y_i = A_i X,  Z += A_i^T Y_i
//   column panels (col-major):  Z_J = A_J^T Yn, Y' += A_J Z_J
// so the whole decomposition costs q + 2 passes over A: the
// sketch pass (which also starts the first power step), q - 1 more power
// passes, the pass that forms the final sample, and the B = Q^T A pass.
#pragma once
#include "pipeline.cuh"

namespace brsvd {

// Ring of device panel buffers fed from host memory on a side stream.
template <typename T>
struct PanelStreamer {
  Ctx& c;
  const T* host;
  int64_t m, n, lda;
  bool row_major;
  int64_t panel;  // rows (row-major) or columns (column-major) per panel
  int nb;
  cudaStream_t copy = nullptr;
  std::vector<cudaEvent_t> copied, consumed;
  std::vector<DBuf<T>*> bufs;
  int64_t panels_streamed = 0;

  // rows_of_cm: row panels of a column-major A (a rank's row shard of a
  // column-major matrix): each panel lands column-major with ld = panel
  bool rows_of_cm = false;

  PanelStreamer(Ctx& c_, const T* host_, int64_t m_, int64_t n_, int64_t lda_, bool rm,
                int64_t panel_, int nb_, bool rows_of_cm_ = false)
      : c(c_), host(host_), m(m_), n(n_), lda(lda_), row_major(rm), panel(panel_), nb(nb_),
        rows_of_cm(rows_of_cm_ && !rm) {
    BRSVD_CUDA(cudaStreamCreateWithFlags(&copy, cudaStreamNonBlocking));
    const int64_t inner = rows_of_cm ? n : (row_major ? n : m);
    for (int b = 0; b < nb; ++b) {
      cudaEvent_t e1, e2;
      BRSVD_CUDA(cudaEventCreateWithFlags(&e1, cudaEventDisableTiming));
      BRSVD_CUDA(cudaEventCreateWithFlags(&e2, cudaEventDisableTiming));
      copied.push_back(e1);
      consumed.push_back(e2);
      bufs.push_back(new DBuf<T>(c, (size_t)(panel * inner)));
    }
    // buffers start "consumed"
    for (int b = 0; b < nb; ++b) BRSVD_CUDA(cudaEventRecord(consumed[b], c.stream));
  }
  ~PanelStreamer() {
    cudaStreamSynchronize(copy);
    cudaStreamSynchronize(c.stream);
    for (auto e : copied) cudaEventDestroy(e);
    for (auto e : consumed) cudaEventDestroy(e);
    for (auto b : bufs) delete b;
    if (copy) cudaStreamDestroy(copy);
  }
  int64_t extent() const { return (row_major || rows_of_cm) ? m : n; }
  int64_t count() const { return ceil_div(extent(), panel); }

  // f(device panel pointer, ld, p0, p1) runs on the compute stream.
  template <class F>
  void pass(F&& f) {
    const int64_t np = count();
    const int64_t inner = row_major ? n : m;
    for (int64_t i = 0; i < np; ++i) {
      const int b = (int)(i % nb);
      const int64_t p0 = i * panel, p1 = std::min(extent(), p0 + panel);
      BRSVD_CUDA(cudaStreamWaitEvent(copy, consumed[b], 0));
      int64_t ld = inner;
      if (rows_of_cm) {   // rows p0..p1 of every column: n strided runs
        ld = panel;
        BRSVD_CUDA(cudaMemcpy2DAsync(bufs[b]->p, panel * sizeof(T), host + p0,
                                     lda * sizeof(T), (p1 - p0) * sizeof(T), n,
                                     cudaMemcpyHostToDevice, copy));
      } else {
        BRSVD_CUDA(cudaMemcpy2DAsync(bufs[b]->p, inner * sizeof(T), host + p0 * lda,
                                     lda * sizeof(T), inner * sizeof(T), p1 - p0,
                                     cudaMemcpyHostToDevice, copy));
      }
      BRSVD_CUDA(cudaEventRecord(copied[b], copy));
      BRSVD_CUDA(cudaStreamWaitEvent(c.stream, copied[b], 0));
      f(bufs[b]->p, ld, p0, p1);
      BRSVD_CUDA(cudaEventRecord(consumed[b], c.stream));
      ++panels_streamed;
    }
  }
};

// Z (fp64, ldz) += op(A) X, op(A) = A^T (trans) or A: the product's magnitude
// is carried into the fp64 sum -- for fp32 data the fp16-split product is
// left in its power-of-two row / column scales (tc_gemm_launch scales_out)
// and unscaled in fp64 by the accumulation, so no fp32 over- or underflow
// can occur in the partial product and no host-known scale is needed.
__global__ void accum_unscaled_kernel(const float* __restrict__ P, int64_t rows, int cols,
                                      int64_t ldp, const float* __restrict__ scales,
                                      double* __restrict__ Z, int64_t ldz) {
  const int64_t total = rows * cols;
  for (int64_t idx = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; idx < total;
       idx += (int64_t)gridDim.x * blockDim.x) {
    const int64_t i = idx % rows, j = idx / rows;
    double v = (double)P[i + j * ldp];
    if (scales) v *= (double)scales[i] * (double)scales[rows + j];
    Z[i + j * ldz] += v;
  }
}

template <typename T>
__global__ void accum_f64_kernel(const T* __restrict__ P, int64_t rows, int cols, int64_t ldp,
                                 double* __restrict__ Z, int64_t ldz) {
  const int64_t total = rows * cols;
  for (int64_t idx = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; idx < total;
       idx += (int64_t)gridDim.x * blockDim.x) {
    const int64_t i = idx % rows, j = idx / rows;
    Z[i + j * ldz] += (double)P[i + j * ldp];
  }
}

template <typename T>
void product_accum(Ctx& c, const T* A, int64_t m, int64_t n, int64_t lda, bool row_major,
                   bool trans, const T* X, int64_t ldx, int l, T* tmp, float* scales,
                   double* Z, int64_t ldz) {
  const int64_t rows = trans ? n : m;
  if constexpr (sizeof(T) == 4) {
    if (scales != nullptr && tc_gemm_supported<float>(c, A, lda, m, n, l) &&
        tc::h16_enabled()) {
      tc_gemm_launch<float>(c, A, m, n, lda, row_major, trans, X, ldx, l, tmp, rows, 0,
                            nullptr, nullptr, scales);
      accum_unscaled_kernel<<<grid_for(rows * l), 256, 0, c.stream>>>(tmp, rows, l, rows,
                                                                      scales, Z, ldz);
      BRSVD_CHECK_LAUNCH();
      return;
    }
  }
  if (trans) big_tn<T>(c, A, m, n, lda, row_major, X, ldx, l, tmp, rows);
  else big_nn<T>(c, A, m, n, lda, row_major, X, ldx, l, tmp, rows);
  accum_f64_kernel<T><<<grid_for(rows * l), 256, 0, c.stream>>>(tmp, rows, l, rows, Z, ldz);
  BRSVD_CHECK_LAUNCH();
}

// Z (n x l, fp64) -> a conditioned basis of its span in the data's precision
// (the power iteration's basis change, normalize_sketch): fp32 data first
// takes Z to unit order by a power of two (exact) so any magnitude the fp64
// sum holds fits fp32; fp64 data is unit-scaled inside normalize_sketch.
template <typename T>
void normalize_from_f64(Ctx& c, const double* Z, int64_t n, int l, int64_t ldz, T* Zout,
                        int64_t ldo, double* Tout = nullptr, double* scale_out = nullptr) {
  // Tout / scale_out (optional): Zout = (scale_out Z) Tout, the transform the
  // exact overflow guard of the sharded driver inverts
  if (scale_out) *scale_out = 1.0;
  if constexpr (sizeof(T) == 8) {
    normalize_sketch<double>(c, Z, n, l, ldz, Zout, ldo, Tout, /*scale_check=*/true);
  } else {
    const MaxAbs pk = maxabs<double>(c, Z, n, l, ldz);
    if (pk.nonfinite)
      throw Error(kErrOverflow, "sample matrix is not finite; the overflow guard fires");
    double s = 1.0;
    if (pk.peak > 0.0) {
      int e;
      std::frexp(pk.peak, &e);
      s = std::ldexp(1.0, -e);
    }
    DBuf<float> Zs(c, (size_t)n * l);
    scale_cast_kernel<double, float><<<grid_for(n * l), 256, 0, c.stream>>>(Z, n, l, ldz, Zs.p,
                                                                            n, s);
    BRSVD_CHECK_LAUNCH();
    normalize_sketch<float>(c, Zs.p, n, l, n, reinterpret_cast<float*>(Zout), ldo, Tout);
    if (scale_out) *scale_out = s;
  }
}

// Y (T, m x l) = 2^-e Y64 with 2^e the order of max |Y64| (exact); returns the
// unscaled peak (max |Y64|, +inf when not finite).
template <typename T>
double unit_cast(Ctx& c, const double* Y64, int64_t m, int l, T* Y, int64_t ldy) {
  const MaxAbs pk = maxabs<double>(c, Y64, m, l, m);
  if (pk.nonfinite) return INFINITY;
  double s = 1.0;
  if (pk.peak > 0.0) {
    int e;
    std::frexp(pk.peak, &e);
    s = std::ldexp(1.0, -e);
  }
  scale_cast_kernel<double, T><<<grid_for(m * l), 256, 0, c.stream>>>(Y64, m, l, m, Y, ldy, s);
  BRSVD_CHECK_LAUNCH();
  return pk.peak;
}

// block_power (column panels only): the paper's two-pass scheme -- each panel
// J runs its whole power iteration (A_J A_J^T)^q A_J Omega_J while resident,
// the block samples are summed (block_range_finder, rsvd.py:150-185), then the
// B pass: 2 passes for any q.
template <typename T>
RsvdInfo rsvd_stream(Ctx& c, const T* Ah, int64_t m, int64_t n, int64_t lda, bool row_major,
                     int k, int p, int q, const T* omega, uint64_t seed, T* U, T* sigma, T* V,
                     int64_t panel, int nbuf, bool block_power = false) {
  const int l = k + p;
  RsvdInfo info;
  StageEvents ev;
  PanelStreamer<T> ps(c, Ah, m, n, lda, row_major, panel, nbuf);
  ev.rec(0, c.stream);
  DBuf<T> Xg;
  const T* X = omega;
  if (X == nullptr) {
    Xg.alloc(c, (size_t)n * l);
    gaussian_kernel<T><<<grid_for(n * ((l + 1) / 2)), 256, 0, c.stream>>>(Xg.p, n, l, n, seed,
                                                                           0, 0);
    BRSVD_CHECK_LAUNCH();
    X = Xg.p;
  }
  DBuf<T> Y(c, (size_t)m * l), Z(c, (size_t)n * l), Zn(c, (size_t)n * l);
  const int64_t pmax = panel;
  DBuf<T> tmpZ(c, (size_t)(row_major ? n : pmax) * l);
  DBuf<T> tmpY(c, row_major ? (size_t)1 : (size_t)m * l);
  int passes = 0;
  double peak0 = 0.0;
  // A^T Y (row panels) and A_J (A_J^T Yn) (column panels) are summed in fp64
  // with the partial products' magnitudes carried exactly (product_accum), so
  // inputs of any magnitude stream without under- or overflow and no scale
  // has to be fixed from a first panel; the sums are brought back to unit
  // order before the basis change.
  DBuf<double> acc64(c, (size_t)std::max(m, n) * l);
  DBuf<float> scales(c, (size_t)(std::max(m, n) + l));
  DBuf<T> tmpP(c, (size_t)std::max(m, n) * l);
  if (row_major) {
    // pass 0: Y_i = A_i Omega (+ first power step Z = sum A_i^T Y_i)
    for (int it = 0; it <= q; ++it) {
      const T* Xin = it == 0 ? X : Zn.p;
      const bool more = it < q;
      if (more) BRSVD_CUDA(cudaMemsetAsync(acc64.p, 0, sizeof(double) * n * l, c.stream));
      ps.pass([&](const T* Ap, int64_t ld, int64_t r0, int64_t r1) {
        big_nn<T>(c, Ap, r1 - r0, n, ld, true, Xin, n, l, Y.p + r0, m);
        if (more)
          product_accum<T>(c, Ap, r1 - r0, n, ld, true, /*trans=*/true, Y.p + r0, m, l,
                           tmpP.p, scales.p, acc64.p, n);
      });
      ++passes;
      if (it == 0) {
        const MaxAbs p0 = maxabs<T>(c, Y.p, m, l, m);
        peak0 = p0.peak;
        if (p0.nonfinite) {
          info.overflow = true;
          info.log10_peak = INFINITY;
          return info;
        }
      }
      if (more) normalize_from_f64<T>(c, acc64.p, n, l, n, Zn.p, n);
    }
  } else {
    // column panels: Y = sum_J A_J Omega_J, then Y' = sum_J A_J (A_J^T Yn)
    DBuf<T> Yn(c, (size_t)m * l);
    const int iters = block_power ? 0 : q;
    for (int it = 0; it <= iters; ++it) {
      BRSVD_CUDA(cudaMemsetAsync(acc64.p, 0, sizeof(double) * m * l, c.stream));
      if (it > 0) normalize_sketch<T>(c, Y.p, m, l, m, Yn.p, m);
      ps.pass([&](const T* Ap, int64_t ld, int64_t j0, int64_t j1) {
        const int64_t w = j1 - j0;
        if (it == 0) {
          big_nn<T>(c, Ap, m, w, ld, false, X + j0, n, l, tmpY.p, m);
          for (int pw = 0; block_power && pw < q; ++pw) {
            big_tn<T>(c, Ap, m, w, ld, false, tmpY.p, m, l, tmpZ.p, pmax);
            big_nn<T>(c, Ap, m, w, ld, false, tmpZ.p, pmax, l, tmpY.p, m);
          }
          accum_f64_kernel<T><<<grid_for(m * l), 256, 0, c.stream>>>(tmpY.p, m, l, m,
                                                                     acc64.p, m);
          BRSVD_CHECK_LAUNCH();
        } else {
          big_tn<T>(c, Ap, m, w, ld, false, Yn.p, m, l, tmpZ.p, pmax);   // Yn unit columns
          product_accum<T>(c, Ap, m, w, ld, false, /*trans=*/false, tmpZ.p, pmax, l, tmpP.p,
                           scales.p, acc64.p, m);
        }
      });
      ++passes;
      const double pk = unit_cast<T>(c, acc64.p, m, l, Y.p, m);
      if (it == 0) {
        peak0 = pk;
        // the reference's sample lives in the data's precision (rsvd.py:84-91)
        if (!(pk <= (double)finfo_max<T>())) {
          info.overflow = true;
          info.log10_peak = INFINITY;
          return info;
        }
      }
    }
  }
  ev.rec(1, c.stream);
  const int ns = sizeof(T) == 8 ? 2 : 1;
  DBuf<T> Qw(c, (size_t)m * l);
  info.rank_y = orth_full<T>(c, Y.p, m, l, m, Qw.p, seed ^ 0x7153ull, ns);
  const T* Qop = Qw.p;
  ev.rec(2, c.stream);
  DBuf<T> Bt(c, (size_t)n * l);
  if (row_major) BRSVD_CUDA(cudaMemsetAsync(Bt.p, 0, sizeof(T) * n * l, c.stream));
  ps.pass([&](const T* Ap, int64_t ld, int64_t p0, int64_t p1) {
    if (row_major) {
      big_tn<T>(c, Ap, p1 - p0, n, ld, true, Qop + p0, m, l, tmpZ.p, n);
      axpy<T>(c, tmpZ.p, n, l, n, Bt.p, n);
    } else {
      big_tn<T>(c, Ap, m, p1 - p0, ld, false, Qop, m, l, Bt.p + p0, n);
    }
  });
  ++passes;
  ev.rec(3, c.stream);
  Y.release();
  DBuf<double> W(c, (size_t)l * l), sig(c, l);
  info.rank_b = small_svd_device<T>(c, Bt.p, n, l, n, W.p, sig.p, V, n, ns);
  apply_basis<T>(c, Qw.p, m, l, m, W.p, l, l, U, m);
  fix_signs<T>(c, U, m, l, m, V, n, n);
  copy2d_kernel<double, T><<<1, 256, 0, c.stream>>>(sig.p, l, 1, l, sigma, l);
  BRSVD_CHECK_LAUNCH();
  ev.rec(4, c.stream);
  double s0 = 0.0;
  readback(c, sig.p, &s0, sizeof(double));
  info.max_abs_y0 = peak0;
  info.words_read = (int64_t)passes * m * n;
  info.block_reads = (int64_t)passes * ps.count();
  info.ms_sketch = ev.ms(0, 1);
  info.ms_orth = ev.ms(1, 2);
  info.ms_core = ev.ms(2, 3);
  info.ms_svd = ev.ms(3, 4);
  const double lim = std::log10(0.01 * finfo_max<T>());
  const int qg = (block_power && !row_major) ? 0 : q;  // block sample is already powered
  info.log10_peak = (peak0 > 0.0 && s0 > 0.0)
                        ? std::log10(peak0) + 2.0 * qg * std::log10(s0)
                        : (peak0 > 0.0 ? std::log10(peak0) : -400.0);
  info.overflow = !std::isfinite(s0) || info.log10_peak > lim;
  return info;
}

// ---------------------------------------------------------------------------
// One streamed pass over a host-resident row shard A (m x n; row-major, or
// column-major streamed as row panels) -- the per-rank unit of the sharded
// out-of-core decomposition (BASELINE config 4; rsvd_naive_ooc's passes,
// rsvd.py:218-284, with the rows of A split over ranks as store.py:165-175
// splits its columns).  For each row panel A_i, on the compute stream while
// the next panel is in flight on the copy stream:
//   X != NULL:  Y_i = A_i X                       (sample rows, into Y)
//   Z != NULL:  Z  += A_i^T Y_i   (fp64 accumulator; Y_i as just formed, or
//                                  as given when X == NULL: B^T = A^T Q)
// fp32 data: each A_i^T Y_i is the fp16-split tcgen05 product left in its
// power-of-two row/column scales and unscaled into the fp64 sum, so Z holds
// inputs of any fp32 magnitude without over- or underflow and no host-side
// scale has to be known before the pass.
struct PassInfo {
  int64_t panels = 0;
  double ms = 0.0;     // pass time on the compute stream
};

template <typename T>
PassInfo stream_rows_pass(Ctx& c, const T* Ah, int64_t m, int64_t n, int64_t lda,
                          bool row_major, const T* X, int64_t ldx, int l, T* Y, int64_t ldy,
                          double* Z, int64_t ldz, int64_t panel, int nbuf) {
  PassInfo pi;
  if (m < 1 || n < 1) return pi;
  panel = std::max<int64_t>(1, std::min(panel, m));
  StageEvents ev;
  PanelStreamer<T> ps(c, Ah, m, n, lda, row_major, panel, nbuf, /*rows_of_cm=*/!row_major);
  ev.rec(0, c.stream);
  DBuf<T> tmp;
  DBuf<float> scales;
  if (Z != nullptr) {
    BRSVD_CUDA(cudaMemset2DAsync(Z, (size_t)ldz * sizeof(double), 0, (size_t)n * sizeof(double),
                                 (size_t)l, c.stream));
    tmp.alloc(c, (size_t)n * l);
    if (sizeof(T) == 4) scales.alloc(c, (size_t)n + l);
  }
  ps.pass([&](const T* Ap, int64_t ld, int64_t r0, int64_t r1) {
    const int64_t rows = r1 - r0;
    if (X != nullptr) big_nn<T>(c, Ap, rows, n, ld, row_major, X, ldx, l, Y + r0, ldy);
    if (Z != nullptr)
      product_accum<T>(c, Ap, rows, n, ld, row_major, /*trans=*/true, Y + r0, ldy, l, tmp.p,
                       scales.p, Z, ldz);
  });
  ev.rec(1, c.stream);
  pi.panels = ps.count();
  pi.ms = ev.ms(0, 1);
  return pi;
}

}  // namespace brsvd
