// Host-streamed inexact-ALM robust PCA: the reference's out-of-core branch
// (_ialm_rpca_ooc, rpca.py:216-304) for matrices whose iterates do not fit
// in device memory.  M (the store payload), the dual Y and the sparse part S
// stay in host memory, column-major; every pass streams their column blocks
// (the budget's plan, _BlockLoop / plan_blocks) through a ring of device
// slots with the H2D copies on one stream, the D2H write-backs on another and
// the compute on the context stream, so both PCIe directions overlap the
// block kernels.  Per iteration (rpca.py:262-300):
//   pass A  W_J = M_J - S_J + Y_J / mu  formed on the device; the inner SVD's
//           per-block power iteration (brsvd_run's block_range_finder,
//           rsvd.py:169-175) sums (W_J W_J^T)^q W_J Omega_J into the sample
//   orth    Q = orth(sample)
//   pass B  W_J again; B^T_J = W_J^T Q (rsvd.py:202-208)
//   svd     small SVD of B, U = Q W, canonical signs
//   pass C  the fused update on M_J, Y_J: L_J on the fly, S_J, Y_J written
//           back to the host, ||Z||^2 partials (rpca.py:286-293)
// and after the loop one pass writes L = U shrink(s) V^T to the host.  The
// spectral-norm estimate streams M twice per power step (rpca.py:48-100).
#pragma once
#include "rpca.cuh"

namespace brsvd {

// Column blocks of several host arrays (same m x n geometry, column-major,
// leading dimension ldh) streamed in lockstep through `nslots` device slots.
template <typename T>
struct BlockStreamer {
  Ctx& c;
  int64_t m, ldh;
  std::vector<int64_t> bounds;   // block edges, bounds[0] = 0 .. bounds[nb] = n
  int nslots, nbuf;              // slots; device buffers per slot
  int64_t wmax = 0;
  cudaStream_t h2d = nullptr, d2h = nullptr;
  std::vector<std::vector<DBuf<T>*>> buf;
  std::vector<cudaEvent_t> in_done, comp_done, out_done;

  BlockStreamer(Ctx& c_, int64_t m_, int64_t ldh_, const std::vector<int64_t>& b, int ns,
                int nb)
      : c(c_), m(m_), ldh(ldh_), bounds(b), nslots(ns), nbuf(nb) {
    for (size_t i = 0; i + 1 < bounds.size(); ++i)
      wmax = std::max(wmax, bounds[i + 1] - bounds[i]);
    BRSVD_CUDA(cudaStreamCreateWithFlags(&h2d, cudaStreamNonBlocking));
    BRSVD_CUDA(cudaStreamCreateWithFlags(&d2h, cudaStreamNonBlocking));
    buf.resize(nslots);
    for (int s = 0; s < nslots; ++s) {
      for (int k = 0; k < nbuf; ++k) buf[s].push_back(new DBuf<T>(c, (size_t)(m * wmax)));
      cudaEvent_t e[3];
      for (auto& x : e) BRSVD_CUDA(cudaEventCreateWithFlags(&x, cudaEventDisableTiming));
      in_done.push_back(e[0]);
      comp_done.push_back(e[1]);
      out_done.push_back(e[2]);
      BRSVD_CUDA(cudaEventRecord(comp_done[s], c.stream));
      BRSVD_CUDA(cudaEventRecord(out_done[s], c.stream));
    }
  }
  ~BlockStreamer() {
    cudaStreamSynchronize(h2d);
    cudaStreamSynchronize(d2h);
    cudaStreamSynchronize(c.stream);
    for (auto& v : buf)
      for (auto* b : v) delete b;
    for (auto* ev : {&in_done, &comp_done, &out_done})
      for (auto e : *ev) cudaEventDestroy(e);
    if (h2d) cudaStreamDestroy(h2d);
    if (d2h) cudaStreamDestroy(d2h);
  }
  int nblocks() const { return (int)bounds.size() - 1; }

  // in[k] (host array or nullptr) lands in slot buffer k; f(T** slot buffers,
  // j0, j1) runs on the compute stream; then slot buffer out[i].first is
  // written back to host array out[i].second.
  template <class F>
  void pass(const std::vector<const T*>& in, const std::vector<std::pair<int, T*>>& out,
            F&& f) {
    const size_t es = sizeof(T);
    std::vector<T*> ptrs(nbuf);
    for (int b = 0; b < nblocks(); ++b) {
      const int s = b % nslots;
      const int64_t j0 = bounds[b], j1 = bounds[b + 1], w = j1 - j0;
      if (w <= 0) continue;
      BRSVD_CUDA(cudaStreamWaitEvent(h2d, comp_done[s], 0));
      BRSVD_CUDA(cudaStreamWaitEvent(h2d, out_done[s], 0));
      for (size_t k = 0; k < in.size(); ++k) {
        if (in[k] == nullptr) continue;
        BRSVD_CUDA(cudaMemcpy2DAsync(buf[s][k]->p, m * es, in[k] + j0 * ldh, ldh * es, m * es,
                                     w, cudaMemcpyHostToDevice, h2d));
      }
      BRSVD_CUDA(cudaEventRecord(in_done[s], h2d));
      BRSVD_CUDA(cudaStreamWaitEvent(c.stream, in_done[s], 0));
      for (int k = 0; k < nbuf; ++k) ptrs[k] = buf[s][k]->p;
      f(ptrs.data(), j0, j1);
      BRSVD_CUDA(cudaEventRecord(comp_done[s], c.stream));
      if (!out.empty()) {
        BRSVD_CUDA(cudaStreamWaitEvent(d2h, comp_done[s], 0));
        for (const auto& o : out)
          BRSVD_CUDA(cudaMemcpy2DAsync(o.second + j0 * ldh, ldh * es, buf[s][o.first]->p,
                                       m * es, m * es, w, cudaMemcpyDeviceToHost, d2h));
        BRSVD_CUDA(cudaEventRecord(out_done[s], d2h));
      }
    }
    BRSVD_CUDA(cudaStreamSynchronize(d2h));
    // the compute stream must see the write-backs before host arrays are reused
    BRSVD_CUDA(cudaStreamSynchronize(c.stream));
  }
};

// W = M - S + Y * inv_mu (one block, dense, column-major)
template <typename T>
__global__ void w_form_kernel(const T* __restrict__ Mx, const T* __restrict__ S,
                              const T* __restrict__ Y, int64_t total, double inv_mu,
                              T* __restrict__ W) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < total;
       i += (int64_t)gridDim.x * blockDim.x)
    W[i] = Mx[i] - S[i] + Y[i] * (T)inv_mu;
}

// Y = scale * M (the dual's initial value, rpca.py:252-255)
template <typename T>
__global__ void scale_block_kernel(const T* __restrict__ Mx, int64_t total, double scale,
                                   T* __restrict__ Y) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < total;
       i += (int64_t)gridDim.x * blockDim.x)
    Y[i] = (T)(scale * (double)Mx[i]);
}

__global__ void add_scalar_kernel(const double* __restrict__ src, double* __restrict__ acc,
                                  int n) {
  if (threadIdx.x < n) acc[threadIdx.x] += src[threadIdx.x];
}

template <typename T>
IalmOut ialm_stream(Ctx& c, const T* Mh, int64_t m, int64_t n, int64_t ldm, int k, int p,
                    int q, uint64_t seed, const T* omega, double lam, double mu0, double rho,
                    double tol, int max_it, const std::vector<int64_t>& bounds, T* Lh, T* Sh,
                    T* Yh, int nslots, double* residuals, double* mus, double* svd_s,
                    double* iter_s) {
  const int l = k + p;
  if (std::isnan(lam)) lam = 1.0 / std::sqrt((double)std::max(m, n));
  // three slot buffers: M_J, S_J / scratch, Y_J; a fourth for W_J
  BlockStreamer<T> bs(c, m, ldm, bounds, nslots, 4);
  const int64_t wmax = bs.wmax;
  DBuf<double> v(c, n), u(c, m), nrm(c, 1), red(c, 2), acc(c, 2);
  // ---- spectral norm: power iteration on M^T M, two streamed passes per
  // step (_matvec / _rmatvec, rpca.py:48-70) ----
  gaussian_kernel<double><<<grid_for(n), 256, 0, c.stream>>>(v.p, n, 1, n, seed, 7, 0);
  BRSVD_CHECK_LAUNCH();
  vec_norm2_kernel<<<1, 1024, 0, c.stream>>>(v.p, n, nrm.p);
  vec_scale_kernel<<<grid_for(n), 256, 0, c.stream>>>(v.p, n, nrm.p, 1);
  BRSVD_CHECK_LAUNCH();
  double norm2 = 0.0, sigma = 0.0;
  DBuf<double> ublk(c, (size_t)m);
  for (int it = 0; it < 100; ++it) {
    BRSVD_CUDA(cudaMemsetAsync(u.p, 0, sizeof(double) * m, c.stream));
    bs.pass({Mh}, {}, [&](T** b, int64_t j0, int64_t j1) {
      matvec<T>(c, b[0], m, j1 - j0, 1, m, v.p + j0, ublk.p);
      axpy_kernel<double><<<grid_for(m), 256, 0, c.stream>>>(ublk.p, m, 1, m, u.p, m);
      BRSVD_CHECK_LAUNCH();
    });
    vec_norm2_kernel<<<1, 1024, 0, c.stream>>>(u.p, m, nrm.p);
    BRSVD_CHECK_LAUNCH();
    double nu;
    readback(c, nrm.p, &nu, sizeof(double));
    BRSVD_REQUIRE(nu != 0.0, kErrArg, "RPCA input is the zero matrix");
    vec_scale_kernel<<<grid_for(m), 256, 0, c.stream>>>(u.p, m, nrm.p, 1);
    BRSVD_CHECK_LAUNCH();
    bs.pass({Mh}, {}, [&](T** b, int64_t j0, int64_t j1) {
      matvec<T>(c, b[0], j1 - j0, m, m, 1, u.p, v.p + j0);
    });
    vec_norm2_kernel<<<1, 1024, 0, c.stream>>>(v.p, n, nrm.p);
    BRSVD_CHECK_LAUNCH();
    double s_new;
    readback(c, nrm.p, &s_new, sizeof(double));
    vec_scale_kernel<<<grid_for(n), 256, 0, c.stream>>>(v.p, n, nrm.p, 1);
    BRSVD_CHECK_LAUNCH();
    norm2 = s_new;
    if (std::fabs(s_new - sigma) <= 1e-10 * s_new) break;
    sigma = s_new;
  }
  double mu = std::isnan(mu0) ? 1.25 / norm2 : mu0;
  // ---- ||M||_F, max |M| (rpca.py:245-250) ----
  const int nbp = grid_for(m * wmax, 256, 148 * 8);
  DBuf<double> psq(c, nbp), pmx(c, nbp);
  BRSVD_CUDA(cudaMemsetAsync(acc.p, 0, 2 * sizeof(double), c.stream));
  double norm_f_sq = 0.0, max_abs = 0.0;
  bs.pass({Mh}, {}, [&](T** b, int64_t j0, int64_t j1) {
    fro_max_kernel<T><<<nbp, 256, 0, c.stream>>>(b[0], m * (j1 - j0), psq.p, pmx.p);
    sum_max_finalize_kernel<<<1, 1024, 0, c.stream>>>(psq.p, pmx.p, nbp, red.p);
    BRSVD_CHECK_LAUNCH();
    double h[2];
    readback(c, red.p, h, sizeof(h));
    norm_f_sq += h[0];
    max_abs = std::max(max_abs, h[1]);
  });
  const double norm_f = std::sqrt(norm_f_sq);
  const double y_scale = 1.0 / std::max(norm2, max_abs / lam);
  // Y = y_scale M, S = 0 (host arrays written by the D2H stream)
  bs.pass({Mh}, {{2, Yh}, {1, Sh}}, [&](T** b, int64_t j0, int64_t j1) {
    const int64_t tot = m * (j1 - j0);
    scale_block_kernel<T><<<grid_for(tot), 256, 0, c.stream>>>(b[0], tot, y_scale, b[2]);
    BRSVD_CHECK_LAUNCH();
    BRSVD_CUDA(cudaMemsetAsync(b[1], 0, sizeof(T) * tot, c.stream));
  });
  // ---- the loop ----
  DBuf<T> Om(c, (size_t)n * l), Ys(c, (size_t)m * l), YJ(c, (size_t)m * l),
      ZJ(c, (size_t)wmax * l), Qw(c, (size_t)m * l), U(c, (size_t)m * l), V(c, (size_t)n * l),
      Bt(c, (size_t)n * l), sig(c, l);
  DBuf<double> Wsm(c, (size_t)l * l), sigd(c, l);
  if (omega != nullptr) {
    BRSVD_CUDA(cudaMemcpyAsync(Om.p, omega, sizeof(T) * n * l, cudaMemcpyDeviceToDevice,
                               c.stream));
  } else {
    gaussian_kernel<T><<<grid_for(n * ((l + 1) / 2)), 256, 0, c.stream>>>(Om.p, n, l, n,
                                                                           seed, 0, 0);
    BRSVD_CHECK_LAUNCH();
  }
  const int ns_it = sizeof(T) == 8 ? 2 : 1;
  const int64_t nparts_max = ceil_div(m, 256) * ceil_div(wmax, kStepTS);
  DBuf<double> part(c, (size_t)nparts_max), zsum(c, 2), zacc(c, 1);
  StageEvents ev;
  IalmOut out;
  for (int it = 1; it <= max_it; ++it) {
    const auto t0 = std::chrono::steady_clock::now();
    ev.rec(0, c.stream);
    const double inv_mu = 1.0 / mu;
    // pass A: per-block power iteration of W_J, summed
    BRSVD_CUDA(cudaMemsetAsync(Ys.p, 0, sizeof(T) * m * l, c.stream));
    bs.pass({Mh, Sh, Yh}, {}, [&](T** b, int64_t j0, int64_t j1) {
      const int64_t w = j1 - j0, tot = m * w;
      w_form_kernel<T><<<grid_for(tot), 256, 0, c.stream>>>(b[0], b[1], b[2], tot, inv_mu,
                                                             b[3]);
      BRSVD_CHECK_LAUNCH();
      big_nn<T>(c, b[3], m, w, m, false, Om.p + j0, n, l, YJ.p, m);
      for (int pw = 0; pw < q; ++pw) {
        big_tn<T>(c, b[3], m, w, m, false, YJ.p, m, l, ZJ.p, w);
        big_nn<T>(c, b[3], m, w, m, false, ZJ.p, w, l, YJ.p, m);
      }
      axpy_kernel<T><<<grid_for(m * l), 256, 0, c.stream>>>(YJ.p, m, l, m, Ys.p, m);
      BRSVD_CHECK_LAUNCH();
    });
    const MaxAbs pk = maxabs<T>(c, Ys.p, m, l, m);
    if (pk.nonfinite || pk.peak > 0.01 * finfo_max<T>())
      throw Error(kErrOverflow, "sample matrix magnitude exceeds the overflow guard");
    orth_full<T>(c, Ys.p, m, l, m, Qw.p, seed ^ 0x7153ull, ns_it);
    // pass B: B^T = W^T Q, block by block
    bs.pass({Mh, Sh, Yh}, {}, [&](T** b, int64_t j0, int64_t j1) {
      const int64_t w = j1 - j0, tot = m * w;
      w_form_kernel<T><<<grid_for(tot), 256, 0, c.stream>>>(b[0], b[1], b[2], tot, inv_mu,
                                                             b[3]);
      BRSVD_CHECK_LAUNCH();
      big_tn<T>(c, b[3], m, w, m, false, Qw.p, m, l, Bt.p + j0, n);
    });
    small_svd_device<T>(c, Bt.p, n, l, n, Wsm.p, sigd.p, V.p, n, ns_it);
    apply_basis<T>(c, Qw.p, m, l, m, Wsm.p, l, l, U.p, m);
    fix_signs<T>(c, U.p, m, l, m, V.p, n, n);
    copy2d_kernel<double, T><<<1, 256, 0, c.stream>>>(sigd.p, l, 1, l, sig.p, l);
    BRSVD_CHECK_LAUNCH();
    ev.rec(1, c.stream);
    // pass C: fused update (S_J into slot buffer 1, Y_J in place), written back
    BRSVD_CUDA(cudaMemsetAsync(zacc.p, 0, sizeof(double), c.stream));
    bs.pass({Mh, nullptr, Yh}, {{1, Sh}, {2, Yh}}, [&](T** b, int64_t j0, int64_t j1) {
      int64_t np = 0;
      rpca_step<T>(c, 0, m, j1 - j0, m, l, U.p, m, V.p + j0, n, sig.p, mu, lam, rho, b[0],
                   b[2], b[1], b[3], nullptr, part.p, &np);
      sum_max_finalize_kernel<<<1, 1024, 0, c.stream>>>(part.p, nullptr, (int)np, zsum.p);
      add_scalar_kernel<<<1, 32, 0, c.stream>>>(zsum.p, zacc.p, 1);
      BRSVD_CHECK_LAUNCH();
    });
    double z2;
    readback(c, zacc.p, &z2, sizeof(double));
    const double residual = std::sqrt(z2) / norm_f;
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
  // L = U shrink(s, 1/mu) V^T from the last factors (rpca.py:282-283)
  bs.pass({}, {{3, Lh}}, [&](T** b, int64_t j0, int64_t j1) {
    rpca_step<T>(c, 1, m, j1 - j0, m, l, U.p, m, V.p + j0, n, sig.p, mu, lam, rho, nullptr,
                 nullptr, nullptr, nullptr, b[3], nullptr, nullptr);
  });
  return out;
}

}  // namespace brsvd
