// extern "C" entry points declared in include/brsvd.h.  Each wraps the C++
// runtime, converts exceptions into status codes and keeps the message for
// brsvd_last_error() (per thread).
#include <string>

#include "../../include/brsvd.h"
#include <chrono>

#include "pipeline.cuh"
#include "rpca.cuh"
#include "rpca_stream.cuh"
#include "stream.cuh"
#include "residual.cuh"
#include "nccl_rt.cuh"

using namespace brsvd;

namespace brsvd {
thread_local long long g_brsvd_launches = 0;
}

struct brsvd_ctx {
  Ctx c;
  nccl::ncclComm_t comm = nullptr;   // brsvd_ctx_attach_nccl (sharded path)
  int nranks = 1, rank = 0;
};

namespace {

thread_local std::string g_last_error;

template <typename F>
int guarded(F&& f) {
  try {
    g_last_error.clear();
    return f();
  } catch (const Error& e) {
    g_last_error = e.what();
    return e.code;
  } catch (const std::exception& e) {
    g_last_error = e.what();
    return kErrArg;
  } catch (...) {
    g_last_error = "unknown error";
    return kErrArg;
  }
}

size_t esize(int dtype) {
  if (dtype == BRSVD_F64) return 8;
  if (dtype == BRSVD_F32) return 4;
  throw Error(kErrArg, "dtype must be 1 (binary64) or 2 (binary32)");
}

// Device view of a (rows x cols, ld) column-major operand that may live on the
// host: copies it in when needed.
struct InView {
  const void* dptr = nullptr;
  int64_t ld = 0;
  void* owned = nullptr;
  cudaStream_t s = nullptr;
  InView(Ctx& c, const void* p, int64_t rows, int64_t cols, int64_t ld_, size_t es,
         int where) {
    s = c.stream;
    if (where == BRSVD_DEVICE) {
      dptr = p;
      ld = ld_;
      return;
    }
    BRSVD_CUDA(cudaMallocAsync(&owned, (size_t)rows * cols * es, s));
    BRSVD_CUDA(cudaMemcpy2DAsync(owned, rows * es, p, ld_ * es, rows * es, cols,
                                 cudaMemcpyHostToDevice, s));
    dptr = owned;
    ld = rows;
  }
  ~InView() {
    if (owned) cudaFreeAsync(owned, s);
  }
};

struct OutView {
  void* dptr = nullptr;
  void* host = nullptr;
  size_t bytes = 0;
  cudaStream_t s = nullptr;
  OutView(Ctx& c, void* p, size_t bytes_, int where) {
    s = c.stream;
    bytes = bytes_;
    if (where == BRSVD_DEVICE || p == nullptr) {
      dptr = p;
      return;
    }
    host = p;
    BRSVD_CUDA(cudaMallocAsync(&dptr, bytes, s));
  }
  void flush() {
    if (host) BRSVD_CUDA(cudaMemcpyAsync(host, dptr, bytes, cudaMemcpyDeviceToHost, s));
  }
  ~OutView() {
    if (host && dptr) cudaFreeAsync(dptr, s);
  }
};

void fill_stats(brsvd_stats* stats, const RsvdInfo& info, int64_t m, int64_t n, int l,
                int q) {
  if (stats) {
    std::memset(stats, 0, sizeof(*stats));
    stats->words_read = info.words_read;
    stats->block_reads = info.block_reads;
    stats->passes_num = info.words_read;
    stats->passes_den = m * n;
    stats->flop_estimate = (int64_t)2 * m * n * l * (2 * q + 2) + (int64_t)4 * m * l * l +
                           (int64_t)2 * n * l * l;
    stats->detected_rank = info.rank_y;
    stats->core_rank = info.rank_b;
    stats->max_abs_y0 = info.max_abs_y0;
    stats->log10_peak_est = info.log10_peak;
    stats->overflow = info.overflow ? 1 : 0;
    stats->seconds_sketch = info.ms_sketch * 1e-3;
    stats->seconds_orthonormalize = info.ms_orth * 1e-3;
    stats->seconds_form_core = info.ms_core * 1e-3;
    stats->seconds_svd = info.ms_svd * 1e-3;
  }
  if (info.overflow)
    throw Error(kErrOverflow,
                "sample matrix magnitude exceeds the overflow guard; lower the power exponent "
                "or rescale the input");
}

}  // namespace

extern "C" {

int brsvd_version(void) { return 1; }

const char* brsvd_last_error(void) { return g_last_error.c_str(); }

int brsvd_ctx_create(int device, void* stream, brsvd_ctx** out) {
  return guarded([&] {
    BRSVD_REQUIRE(out != nullptr, kErrArg, "out is NULL");
    BRSVD_CUDA(cudaSetDevice(device));
    auto* h = new brsvd_ctx();
    h->c.device = device;
    if (stream) {
      h->c.stream = (cudaStream_t)stream;
    } else {
      BRSVD_CUDA(cudaStreamCreateWithFlags(&h->c.stream, cudaStreamNonBlocking));
      h->c.own_stream = true;
    }
    BRSVD_CUDA(cudaHostAlloc((void**)&h->c.h_pinned, 64, cudaHostAllocDefault));
    int sms = 0, optin = 0;
    BRSVD_CUDA(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, device));
    BRSVD_CUDA(cudaDeviceGetAttribute(&optin, cudaDevAttrMaxSharedMemoryPerBlockOptin,
                                      device));
    h->c.num_sms = sms;
    BRSVD_CUDA(cudaDeviceGetAttribute(&h->c.cc_major, cudaDevAttrComputeCapabilityMajor, device));
    BRSVD_CUDA(cudaDeviceGetAttribute(&h->c.cc_minor, cudaDevAttrComputeCapabilityMinor, device));
    h->c.max_smem_optin = (size_t)optin;
    cudaMemPool_t pool;
    BRSVD_CUDA(cudaDeviceGetDefaultMemPool(&pool, device));
    uint64_t thr = UINT64_MAX;
    BRSVD_CUDA(cudaMemPoolSetAttribute(pool, cudaMemPoolAttrReleaseThreshold, &thr));
    *out = h;
    return (int)kOk;
  });
}

int brsvd_ctx_set_stream(brsvd_ctx* ctx, void* stream) {
  return guarded([&] {
    BRSVD_REQUIRE(ctx != nullptr, kErrArg, "ctx is NULL");
    if (ctx->c.own_stream) {
      BRSVD_CUDA(cudaStreamSynchronize(ctx->c.stream));
      BRSVD_CUDA(cudaStreamDestroy(ctx->c.stream));
      ctx->c.own_stream = false;
    }
    ctx->c.stream = (cudaStream_t)stream;
    return (int)kOk;
  });
}

int brsvd_ctx_destroy(brsvd_ctx* ctx) {
  return guarded([&] {
    if (!ctx) return (int)kOk;
    cudaStreamSynchronize(ctx->c.stream);
    if (ctx->comm) nccl::api().CommDestroy(ctx->comm);
    if (ctx->c.own_stream) cudaStreamDestroy(ctx->c.stream);
    if (ctx->c.h_pinned) cudaFreeHost(ctx->c.h_pinned);
    delete ctx;
    return (int)kOk;
  });
}

int brsvd_nccl_unique_id(char* out) {
  return guarded([&] {
    BRSVD_REQUIRE(out != nullptr, kErrArg, "out is NULL");
    nccl::ncclUniqueId id;
    nccl::check(nccl::api().GetUniqueId(&id), "ncclGetUniqueId");
    std::memcpy(out, id.internal, nccl::kUniqueIdBytes);
    return (int)kOk;
  });
}

int brsvd_ctx_attach_nccl(brsvd_ctx* ctx, const char* unique_id, int nranks, int rank) {
  return guarded([&] {
    BRSVD_REQUIRE(ctx != nullptr && unique_id != nullptr, kErrArg, "NULL argument");
    BRSVD_REQUIRE(nranks >= 1 && rank >= 0 && rank < nranks, kErrArg, "bad rank / nranks");
    BRSVD_CUDA(cudaSetDevice(ctx->c.device));
    if (ctx->comm) {
      nccl::api().CommDestroy(ctx->comm);
      ctx->comm = nullptr;
    }
    nccl::ncclUniqueId id;
    std::memcpy(id.internal, unique_id, nccl::kUniqueIdBytes);
    nccl::check(nccl::api().CommInitRank(&ctx->comm, nranks, id, rank), "ncclCommInitRank");
    ctx->nranks = nranks;
    ctx->rank = rank;
    return (int)kOk;
  });
}

int brsvd_allreduce(brsvd_ctx* ctx, void* buf, int64_t count, int dtype, int op) {
  return guarded([&] {
    BRSVD_REQUIRE(ctx != nullptr && ctx->comm != nullptr, kErrNccl,
                  "no NCCL communicator attached (brsvd_ctx_attach_nccl)");
    BRSVD_REQUIRE(op == 0 || op == 2, kErrArg, "op must be 0 (sum) or 2 (max)");
    BRSVD_CUDA(cudaSetDevice(ctx->c.device));
    if (count > 0)
      nccl::check(nccl::api().AllReduce(buf, buf, (size_t)count, nccl::dtype_of(dtype), op,
                                        ctx->comm, ctx->c.stream),
                  "ncclAllReduce");
    return (int)kOk;
  });
}

int brsvd_allgather(brsvd_ctx* ctx, const void* send, void* recv, int64_t count, int dtype) {
  return guarded([&] {
    BRSVD_REQUIRE(ctx != nullptr && ctx->comm != nullptr, kErrNccl,
                  "no NCCL communicator attached (brsvd_ctx_attach_nccl)");
    BRSVD_CUDA(cudaSetDevice(ctx->c.device));
    if (count > 0)
      nccl::check(nccl::api().AllGather(send, recv, (size_t)count, nccl::dtype_of(dtype),
                                        ctx->comm, ctx->c.stream),
                  "ncclAllGather");
    return (int)kOk;
  });
}

int brsvd_profile_begin(brsvd_ctx* ctx) {
  return guarded([&] {
    BRSVD_REQUIRE(ctx != nullptr, kErrArg, "ctx is NULL");
    Ctx& c = ctx->c;
    for (auto e : c.prof_ev) cudaEventDestroy(e);
    c.prof_ev.clear();
    c.prof_flops = c.prof_bytes = 0.0;
    c.prof = true;
    c.prof_launch0 = g_brsvd_launches;
    return (int)kOk;
  });
}

int brsvd_profile_end(brsvd_ctx* ctx, brsvd_profile* out) {
  return guarded([&] {
    BRSVD_REQUIRE(ctx != nullptr && out != nullptr, kErrArg, "NULL argument");
    Ctx& c = ctx->c;
    BRSVD_CUDA(cudaStreamSynchronize(c.stream));
    double ms = 0.0;
    for (size_t i = 0; i + 1 < c.prof_ev.size(); i += 2) {
      float t = 0.f;
      BRSVD_CUDA(cudaEventElapsedTime(&t, c.prof_ev[i], c.prof_ev[i + 1]));
      ms += t;
    }
    out->big_launches = (int64_t)(c.prof_ev.size() / 2);
    out->big_ms = ms;
    out->big_flops = c.prof_flops;
    out->big_bytes = c.prof_bytes;
    out->gpu_launches = g_brsvd_launches - c.prof_launch0;
    for (auto e : c.prof_ev) cudaEventDestroy(e);
    c.prof_ev.clear();
    c.prof = false;
    return (int)kOk;
  });
}

int brsvd_rsvd(brsvd_ctx* ctx, const void* A, int64_t m, int64_t n, int64_t lda,
               int dtype, int layout, int a_where, int k, int p, int q,
               const void* omega, int omega_where, uint64_t seed, void* U,
               void* sigma, void* Vt, int out_where, brsvd_stats* stats) {
  return brsvd_rsvd_blocked(ctx, A, m, n, lda, dtype, layout, a_where, k, p, q, omega,
                            omega_where, seed, nullptr, 0, U, sigma, Vt, out_where, stats);
}

namespace {
int rsvd_entry(brsvd_ctx* ctx, const void* A, int64_t m, int64_t n, int64_t lda, int dtype,
               int layout, int a_where, int k, int p, int q, const void* omega,
               int omega_where, uint64_t seed, const int64_t* col_bounds, int nblocks, void* U,
               void* sigma, void* Vt, int out_where, brsvd_stats* stats, bool range_only);
}

int brsvd_rsvd_blocked(brsvd_ctx* ctx, const void* A, int64_t m, int64_t n, int64_t lda,
                       int dtype, int layout, int a_where, int k, int p, int q,
                       const void* omega, int omega_where, uint64_t seed,
                       const int64_t* col_bounds, int nblocks, void* U, void* sigma,
                       void* Vt, int out_where, brsvd_stats* stats) {
  return rsvd_entry(ctx, A, m, n, lda, dtype, layout, a_where, k, p, q, omega, omega_where,
                    seed, col_bounds, nblocks, U, sigma, Vt, out_where, stats, false);
}

int brsvd_range_finder(brsvd_ctx* ctx, const void* A, int64_t m, int64_t n, int64_t lda,
                       int dtype, int layout, int a_where, int k, int p, int q,
                       const void* omega, int omega_where, uint64_t seed,
                       const int64_t* col_bounds, int nblocks, void* Q, int out_where,
                       brsvd_stats* stats) {
  return rsvd_entry(ctx, A, m, n, lda, dtype, layout, a_where, k, p, q, omega, omega_where,
                    seed, col_bounds, nblocks, Q, nullptr, nullptr, out_where, stats, true);
}

}  // extern "C"

namespace {
int rsvd_entry(brsvd_ctx* ctx, const void* A, int64_t m, int64_t n, int64_t lda, int dtype,
               int layout, int a_where, int k, int p, int q, const void* omega,
               int omega_where, uint64_t seed, const int64_t* col_bounds, int nblocks, void* U,
               void* sigma, void* Vt, int out_where, brsvd_stats* stats, bool range_only) {
  return guarded([&] {
    if (nblocks > 0) {
      BRSVD_REQUIRE(col_bounds != nullptr, kErrArg, "col_bounds is NULL");
      BRSVD_REQUIRE(col_bounds[0] == 0 && col_bounds[nblocks] == n, kErrShape,
                    "column blocks must tile [0, n)");
      for (int b = 0; b < nblocks; ++b)
        BRSVD_REQUIRE(col_bounds[b + 1] > col_bounds[b], kErrShape,
                      "column blocks must be non-empty and increasing");
    }
    BRSVD_REQUIRE(ctx != nullptr, kErrArg, "ctx is NULL");
    Ctx& c = ctx->c;
    BRSVD_CUDA(cudaSetDevice(c.device));
    const size_t es = esize(dtype);
    BRSVD_REQUIRE(m >= 1 && n >= 1, kErrShape, "matrix must be non-empty");
    BRSVD_REQUIRE(k >= 1, kErrConfig, "target rank must be positive");
    BRSVD_REQUIRE(p >= 0, kErrConfig, "oversampling must be non-negative");
    BRSVD_REQUIRE(k + p <= std::min(m, n), kErrConfig, "k + p exceeds min(m, n)");
    BRSVD_REQUIRE(q >= 0, kErrConfig, "power exponent must be non-negative");
    BRSVD_REQUIRE(k + p <= 1024, kErrConfig, "k + p above 1024 is not supported");
    const int l = k + p;
    const bool row_major = layout == BRSVD_ROW_MAJOR;
    // A as a column-major (rows x cols) array: row-major A is A^T col-major.
    const int64_t a_rows = row_major ? n : m, a_cols = row_major ? m : n;
    BRSVD_REQUIRE(lda >= a_rows, kErrShape, "lda too small");
    // host input: the pipeline streams A in (H2D overlapped with the sample
    // pass, HostFeed); device input is used in place
    const bool on_host = a_where != BRSVD_DEVICE;
    InView av(c, on_host ? nullptr : A, a_rows, a_cols, lda, es, BRSVD_DEVICE);
    DBuf<unsigned char> adev;
    HostFeed feed;
    const void* aptr = av.dptr;
    int64_t ald = av.ld;
    if (on_host) {
      adev.alloc(c, (size_t)a_rows * a_cols * es);
      aptr = adev.p;
      ald = a_rows;
      feed.host = A;
      feed.ldh = lda;
    }
    InView ov(c, omega, n, l, n, es, omega ? omega_where : BRSVD_DEVICE);
    BRSVD_REQUIRE(U != nullptr && (range_only || (sigma != nullptr && Vt != nullptr)),
                  kErrArg, "output pointer is NULL");
    OutView uo(c, U, (size_t)m * l * es, out_where);
    OutView so(c, sigma, (size_t)l * es, out_where);
    OutView vo(c, Vt, (size_t)n * l * es, out_where);
    RsvdInfo info;
    if (dtype == BRSVD_F64) {
      info = rsvd_device<double>(c, (const double*)aptr, m, n, ald, row_major, k, p, q,
                                 (const double*)ov.dptr, seed, (double*)uo.dptr,
                                 (double*)so.dptr, (double*)vo.dptr,
                                 on_host ? &feed : nullptr, col_bounds, nblocks, range_only);
    } else {
      info = rsvd_device<float>(c, (const float*)aptr, m, n, ald, row_major, k, p, q,
                                (const float*)ov.dptr, seed, (float*)uo.dptr,
                                (float*)so.dptr, (float*)vo.dptr, on_host ? &feed : nullptr,
                                col_bounds, nblocks, range_only);
    }
    uo.flush();
    so.flush();
    vo.flush();
    BRSVD_CUDA(cudaStreamSynchronize(c.stream));
    fill_stats(stats, info, m, n, l, q);
    return (int)kOk;
  });
}
}  // namespace

extern "C" {

int brsvd_rsvd_stream(brsvd_ctx* ctx, const void* A, int64_t m, int64_t n, int64_t lda,
                      int dtype, int layout, int k, int p, int q, const void* omega,
                      int omega_where, uint64_t seed, void* U, void* sigma, void* Vt,
                      int out_where, int64_t panel, int nbuf, brsvd_stats* stats) {
  return brsvd_rsvd_stream_blocked(ctx, A, m, n, lda, dtype, layout, k, p, q, omega,
                                   omega_where, seed, U, sigma, Vt, out_where, panel, nbuf, 0,
                                   stats);
}

int brsvd_rsvd_stream_blocked(brsvd_ctx* ctx, const void* A, int64_t m, int64_t n,
                              int64_t lda, int dtype, int layout, int k, int p, int q,
                              const void* omega, int omega_where, uint64_t seed, void* U,
                              void* sigma, void* Vt, int out_where, int64_t panel, int nbuf,
                              int block_power, brsvd_stats* stats) {
  return guarded([&] {
    BRSVD_REQUIRE(!block_power || layout == BRSVD_COL_MAJOR, kErrArg,
                  "per-block power iteration streams column blocks (column-major A)");
    BRSVD_REQUIRE(ctx != nullptr && A != nullptr, kErrArg, "NULL argument");
    Ctx& c = ctx->c;
    BRSVD_CUDA(cudaSetDevice(c.device));
    const size_t es = esize(dtype);
    BRSVD_REQUIRE(m >= 1 && n >= 1, kErrShape, "matrix must be non-empty");
    BRSVD_REQUIRE(k >= 1 && p >= 0 && k + p <= std::min(m, n), kErrConfig,
                  "k + p exceeds min(m, n)");
    BRSVD_REQUIRE(q >= 0, kErrConfig, "power exponent must be non-negative");
    BRSVD_REQUIRE(panel >= 1 && nbuf >= 1, kErrArg, "panel and nbuf must be positive");
    const int l = k + p;
    const bool row_major = layout == BRSVD_ROW_MAJOR;
    BRSVD_REQUIRE(lda >= (row_major ? n : m), kErrShape, "lda too small");
    InView ov(c, omega, n, l, n, es, omega ? omega_where : BRSVD_DEVICE);
    OutView uo(c, U, (size_t)m * l * es, out_where);
    OutView so(c, sigma, (size_t)l * es, out_where);
    OutView vo(c, Vt, (size_t)n * l * es, out_where);
    RsvdInfo info;
    if (dtype == BRSVD_F64)
      info = rsvd_stream<double>(c, (const double*)A, m, n, lda, row_major, k, p, q,
                                 (const double*)ov.dptr, seed, (double*)uo.dptr,
                                 (double*)so.dptr, (double*)vo.dptr, panel, nbuf,
                                 block_power != 0);
    else
      info = rsvd_stream<float>(c, (const float*)A, m, n, lda, row_major, k, p, q,
                                (const float*)ov.dptr, seed, (float*)uo.dptr,
                                (float*)so.dptr, (float*)vo.dptr, panel, nbuf,
                                block_power != 0);
    uo.flush();
    so.flush();
    vo.flush();
    BRSVD_CUDA(cudaStreamSynchronize(c.stream));
    fill_stats(stats, info, m, n, l, q);
    return (int)kOk;
  });
}

int brsvd_residual(brsvd_ctx* ctx, const void* A, int64_t m, int64_t n, int64_t lda, int dtype,
                   int layout, const void* U, int64_t ldu, const void* sigma, const void* Vt,
                   int64_t ldv, int64_t l, double* out) {
  return guarded([&] {
    BRSVD_REQUIRE(ctx != nullptr && out != nullptr, kErrArg, "NULL argument");
    Ctx& c = ctx->c;
    BRSVD_CUDA(cudaSetDevice(c.device));
    esize(dtype);
    BRSVD_REQUIRE(m >= 0 && n >= 0 && l >= 0, kErrShape, "bad shape");
    const bool row_major = layout == BRSVD_ROW_MAJOR;
    if (dtype == BRSVD_F64)
      residual_device<double>(c, (const double*)A, m, n, lda, row_major, (const double*)U, ldu,
                              (const double*)sigma, (const double*)Vt, ldv, (int)l, out);
    else
      residual_device<float>(c, (const float*)A, m, n, lda, row_major, (const float*)U, ldu,
                             (const float*)sigma, (const float*)Vt, ldv, (int)l, out);
    return (int)kOk;
  });
}

int brsvd_sketch_product(brsvd_ctx* ctx, const void* A, int64_t m, int64_t n, int64_t lda,
                         int dtype, int layout, int trans, const void* X, int64_t ldx,
                         int64_t l, void* C, int64_t ldc) {
  return brsvd_sketch_product_scaled(ctx, A, m, n, lda, dtype, layout, trans, X, ldx, l, C,
                                     ldc, nullptr);
}

int brsvd_sketch_product_scaled(brsvd_ctx* ctx, const void* A, int64_t m, int64_t n,
                                int64_t lda, int dtype, int layout, int trans, const void* X,
                                int64_t ldx, int64_t l, void* C, int64_t ldc,
                                const float* amax) {
  return guarded([&] {
    BRSVD_REQUIRE(ctx != nullptr, kErrArg, "ctx is NULL");
    Ctx& c = ctx->c;
    BRSVD_CUDA(cudaSetDevice(c.device));
    esize(dtype);
    BRSVD_REQUIRE(m >= 1 && n >= 1 && l >= 1 && l <= 1024, kErrShape, "bad shape");
    const bool row_major = layout == BRSVD_ROW_MAJOR;
    if (dtype == BRSVD_F64) {
      if (trans)
        big_tn<double>(c, (const double*)A, m, n, lda, row_major, (const double*)X, ldx,
                       (int)l, (double*)C, ldc);
      else
        big_nn<double>(c, (const double*)A, m, n, lda, row_major, (const double*)X, ldx,
                       (int)l, (double*)C, ldc);
    } else {
      if (trans)
        big_tn<float>(c, (const float*)A, m, n, lda, row_major, (const float*)X, ldx, (int)l,
                      (float*)C, ldc, amax);
      else
        big_nn<float>(c, (const float*)A, m, n, lda, row_major, (const float*)X, ldx, (int)l,
                      (float*)C, ldc, amax);
    }
    return (int)kOk;
  });
}

int brsvd_absmax(brsvd_ctx* ctx, const void* A, int64_t m, int64_t n, int64_t lda, int dtype,
                 int layout, float* row_max, float* col_max) {
  return guarded([&] {
    BRSVD_REQUIRE(ctx != nullptr && A != nullptr, kErrArg, "NULL argument");
    BRSVD_REQUIRE(dtype == BRSVD_F32, kErrArg, "absmax scales serve the fp32 products");
    Ctx& c = ctx->c;
    BRSVD_CUDA(cudaSetDevice(c.device));
    absmax_rows_cols(c, (const float*)A, m, n, lda, layout == BRSVD_ROW_MAJOR, row_max,
                     col_max);
    return (int)kOk;
  });
}

int brsvd_tsqr(brsvd_ctx* ctx, const void* Y, int64_t m, int64_t l, int64_t ldy,
               int dtype, int where, void* Q, void* R, int32_t* detected_rank) {
  return guarded([&] {
    BRSVD_REQUIRE(ctx != nullptr, kErrArg, "ctx is NULL");
    Ctx& c = ctx->c;
    BRSVD_CUDA(cudaSetDevice(c.device));
    const size_t es = esize(dtype);
    BRSVD_REQUIRE(l >= 1 && m >= l, kErrShape, "tsqr requires rows >= cols >= 1");
    BRSVD_REQUIRE(l <= 1024, kErrShape, "tsqr supports at most 1024 columns");
    InView yv(c, Y, m, l, ldy, es, where);
    OutView qo(c, Q, (size_t)m * l * es, where);
    OutView ro(c, R, (size_t)l * l * es, where);
    int rank;
    if (dtype == BRSVD_F64) {
      DBuf<double> Qw(c, (size_t)m * l);
      rank = orth_full<double>(c, (const double*)yv.dptr, m, (int)l, yv.ld, Qw.p,
                               0x75717221ull, 2);
      BRSVD_CUDA(cudaMemcpyAsync(qo.dptr, Qw.p, (size_t)m * l * 8,
                                 cudaMemcpyDeviceToDevice, c.stream));
      if (ro.dptr)
        gemm_tn_cm<double, double, double>(c, l, l, m, Qw.p, m, (const double*)yv.dptr,
                                           yv.ld, (double*)ro.dptr, l);
    } else {
      DBuf<float> Qw(c, (size_t)m * l);
      rank = orth_full<float>(c, (const float*)yv.dptr, m, (int)l, yv.ld, Qw.p,
                              0x75717221ull, 1);
      BRSVD_CUDA(cudaMemcpyAsync(qo.dptr, Qw.p, (size_t)m * l * 4,
                                 cudaMemcpyDeviceToDevice, c.stream));
      if (ro.dptr)
        gemm_tn_cm<float, float, float>(c, l, l, m, Qw.p, m, (const float*)yv.dptr,
                                        yv.ld, (float*)ro.dptr, l);
    }
    if (ro.dptr) {
      // full-rank inputs: Q = Y T with T upper triangular (Cholesky QR in
      // column order), so R = Q^T Y is upper triangular up to rounding --
      // make it exactly so, as Householder QR returns it (kernels.py:139-164).
      // Rank-deficient inputs (completed columns) keep the full Q^T Y.
      DBuf<unsigned long long> tc(c, 2);
      BRSVD_CUDA(cudaMemsetAsync(tc.p, 0, 2 * sizeof(unsigned long long), c.stream));
      if (dtype == BRSVD_F64)
        tri_check_kernel<double><<<grid_for(l * l), 256, 0, c.stream>>>((double*)ro.dptr,
                                                                         (int)l, tc.p);
      else
        tri_check_kernel<float><<<grid_for(l * l), 256, 0, c.stream>>>((float*)ro.dptr,
                                                                        (int)l, tc.p);
      BRSVD_CHECK_LAUNCH();
      unsigned long long hb[2];
      readback(c, tc.p, hb, sizeof(hb));
      double mx, low;
      std::memcpy(&mx, &hb[0], 8);
      std::memcpy(&low, &hb[1], 8);
      const double eps = dtype == BRSVD_F64 ? 2.220446049250313e-16 : 1.1920928955078125e-07;
      if (low <= 64.0 * l * eps * mx) {
        if (dtype == BRSVD_F64)
          zero_strict_lower_kernel<double><<<grid_for(l * l), 256, 0, c.stream>>>(
              (double*)ro.dptr, (int)l);
        else
          zero_strict_lower_kernel<float><<<grid_for(l * l), 256, 0, c.stream>>>(
              (float*)ro.dptr, (int)l);
        BRSVD_CHECK_LAUNCH();
      }
    }
    qo.flush();
    ro.flush();
    BRSVD_CUDA(cudaStreamSynchronize(c.stream));
    if (detected_rank) *detected_rank = rank;
    return (int)kOk;
  });
}

int brsvd_small_svd(brsvd_ctx* ctx, const void* Bt, int64_t n, int64_t l,
                    int64_t ldb, int dtype, int where, void* W, void* sigma,
                    void* Vt, int32_t* core_rank) {
  return guarded([&] {
    BRSVD_REQUIRE(ctx != nullptr, kErrArg, "ctx is NULL");
    Ctx& c = ctx->c;
    BRSVD_CUDA(cudaSetDevice(c.device));
    const size_t es = esize(dtype);
    BRSVD_REQUIRE(l >= 1 && n >= l, kErrShape, "small_svd requires rows <= cols");
    BRSVD_REQUIRE(l <= 1024, kErrShape, "small_svd supports at most 1024 rows");
    InView bv(c, Bt, n, l, ldb, es, where);
    OutView wo(c, W, (size_t)l * l * es, where);
    OutView so(c, sigma, (size_t)l * es, where);
    OutView vo(c, Vt, (size_t)n * l * es, where);
    DBuf<double> Wd(c, (size_t)l * l), sd(c, l);
    int rank;
    if (dtype == BRSVD_F64) {
      rank = small_svd_device<double>(c, (const double*)bv.dptr, n, (int)l, bv.ld, Wd.p,
                                      sd.p, (double*)vo.dptr, n, 2);
    } else {
      rank = small_svd_device<float>(c, (const float*)bv.dptr, n, (int)l, bv.ld, Wd.p,
                                     sd.p, (float*)vo.dptr, n, 1);
    }
    if (dtype == BRSVD_F64) {
      BRSVD_CUDA(cudaMemcpyAsync(wo.dptr, Wd.p, (size_t)l * l * 8,
                                 cudaMemcpyDeviceToDevice, c.stream));
      BRSVD_CUDA(cudaMemcpyAsync(so.dptr, sd.p, (size_t)l * 8, cudaMemcpyDeviceToDevice,
                                 c.stream));
    } else {
      copy2d_kernel<double, float><<<grid_for(l * l), 256, 0, c.stream>>>(
          Wd.p, l, l, l, (float*)wo.dptr, l);
      copy2d_kernel<double, float><<<1, 256, 0, c.stream>>>(sd.p, l, 1, l,
                                                           (float*)so.dptr, l);
      BRSVD_CHECK_LAUNCH();
    }
    wo.flush();
    so.flush();
    vo.flush();
    BRSVD_CUDA(cudaStreamSynchronize(c.stream));
    if (core_rank) *core_rank = rank;
    return (int)kOk;
  });
}

int brsvd_gaussian(brsvd_ctx* ctx, void* out, int64_t rows, int64_t cols, int64_t ld,
                   int dtype, uint64_t seed, uint64_t stream, int64_t row_offset) {
  return guarded([&] {
    BRSVD_REQUIRE(ctx != nullptr, kErrArg, "ctx is NULL");
    Ctx& c = ctx->c;
    BRSVD_CUDA(cudaSetDevice(c.device));
    BRSVD_REQUIRE(rows >= 1 && cols >= 1, kErrShape, "gaussian_matrix needs positive shape");
    BRSVD_REQUIRE(ld >= rows, kErrShape, "ld too small");
    const int g = grid_for(rows * ((cols + 1) / 2));
    if (dtype == BRSVD_F64)
      gaussian_kernel<double><<<g, 256, 0, c.stream>>>((double*)out, rows, cols, ld, seed,
                                                       stream, row_offset);
    else if (dtype == BRSVD_F32)
      gaussian_kernel<float><<<g, 256, 0, c.stream>>>((float*)out, rows, cols, ld, seed,
                                                      stream, row_offset);
    else
      throw Error(kErrArg, "bad dtype");
    BRSVD_CHECK_LAUNCH();
    BRSVD_CUDA(cudaStreamSynchronize(c.stream));
    return (int)kOk;
  });
}

int brsvd_spectral_norm(brsvd_ctx* ctx, const void* M, int64_t m, int64_t n, int64_t ldm,
                        int dtype, int layout, int where, uint64_t seed, double tol,
                        int max_iterations, double* out, int32_t* iterations) {
  return brsvd_spectral_norm_start(ctx, M, m, n, ldm, dtype, layout, where, seed, nullptr, tol,
                                   max_iterations, out, iterations);
}

int brsvd_spectral_norm_start(brsvd_ctx* ctx, const void* M, int64_t m, int64_t n,
                              int64_t ldm, int dtype, int layout, int where, uint64_t seed,
                              const double* start, double tol, int max_iterations,
                              double* out, int32_t* iterations) {
  return guarded([&] {
    BRSVD_REQUIRE(ctx != nullptr && out != nullptr, kErrArg, "NULL argument");
    Ctx& c = ctx->c;
    BRSVD_CUDA(cudaSetDevice(c.device));
    const size_t es = esize(dtype);
    BRSVD_REQUIRE(m >= 1 && n >= 1, kErrShape, "matrix must be non-empty");
    const bool row_major = layout == BRSVD_ROW_MAJOR;
    const int64_t a_rows = row_major ? n : m, a_cols = row_major ? m : n;
    InView mv(c, M, a_rows, a_cols, ldm, es, where);
    const int64_t sm = row_major ? mv.ld : 1, sn = row_major ? 1 : mv.ld;
    int it = 0;
    double v;
    if (dtype == BRSVD_F64)
      v = spectral_norm<double>(c, (const double*)mv.dptr, m, n, sm, sn, seed, tol,
                                max_iterations, &it, start);
    else
      v = spectral_norm<float>(c, (const float*)mv.dptr, m, n, sm, sn, seed, tol,
                               max_iterations, &it, start);
    BRSVD_CUDA(cudaStreamSynchronize(c.stream));
    *out = v;
    if (iterations) *iterations = it;
    return (int)kOk;
  });
}

int brsvd_ialm(brsvd_ctx* ctx, const void* M, int64_t m, int64_t n, int64_t ldm,
               int dtype, int layout, int where, int k, int p, int q, uint64_t seed,
               const void* omega, double lam, double mu0, double rho, double tol,
               int max_iterations,
               void* L, void* S, int out_where, int32_t* iterations,
               int32_t* converged, double* residuals, double* mus, double* svd_seconds,
               double* iter_seconds) {
  return brsvd_ialm_blocked(ctx, M, m, n, ldm, dtype, layout, where, k, p, q, seed, omega,
                            lam, mu0, rho, tol, max_iterations, nullptr, 0, L, S, out_where,
                            iterations, converged, residuals, mus, svd_seconds, iter_seconds);
}

int brsvd_ialm_blocked(brsvd_ctx* ctx, const void* M, int64_t m, int64_t n, int64_t ldm,
                       int dtype, int layout, int where, int k, int p, int q, uint64_t seed,
                       const void* omega, double lam, double mu0, double rho, double tol,
                       int max_iterations, const int64_t* col_bounds, int nblocks, void* L,
                       void* S, int out_where, int32_t* iterations, int32_t* converged,
                       double* residuals, double* mus, double* svd_seconds,
                       double* iter_seconds) {
  return guarded([&] {
    if (nblocks > 0)
      BRSVD_REQUIRE(col_bounds != nullptr && col_bounds[0] == 0 && col_bounds[nblocks] == n,
                    kErrShape, "column blocks must tile [0, n)");
    BRSVD_REQUIRE(ctx != nullptr, kErrArg, "ctx is NULL");
    BRSVD_REQUIRE(residuals && mus && svd_seconds && iter_seconds, kErrArg,
                  "history arrays are required");
    Ctx& c = ctx->c;
    BRSVD_CUDA(cudaSetDevice(c.device));
    const size_t es = esize(dtype);
    BRSVD_REQUIRE(m >= 1 && n >= 1, kErrShape, "matrix must be non-empty");
    BRSVD_REQUIRE(k >= 1 && p >= 0 && k + p <= std::min(m, n), kErrConfig,
                  "k + p exceeds min(m, n)");
    BRSVD_REQUIRE(q >= 0, kErrConfig, "power exponent must be non-negative");
    BRSVD_REQUIRE(rho > 1.0 && tol > 0.0 && max_iterations >= 1, kErrArg,
                  "rho must exceed 1, tol and max_iterations must be positive");
    const bool row_major = layout == BRSVD_ROW_MAJOR;
    const int64_t a_rows = row_major ? n : m, a_cols = row_major ? m : n;
    BRSVD_REQUIRE(ldm == a_rows, kErrShape, "M must be dense");
    InView mv(c, M, a_rows, a_cols, ldm, es, where);
    InView ov(c, omega, n, k + p, n, es, omega ? where : BRSVD_DEVICE);
    OutView lo(c, L, (size_t)m * n * es, out_where);
    OutView so(c, S, (size_t)m * n * es, out_where);
    IalmOut r;
    if (dtype == BRSVD_F64)
      r = ialm_device<double>(c, (const double*)mv.dptr, m, n, row_major, k, p, q, seed,
                              (const double*)ov.dptr, lam, mu0, rho, tol, max_iterations, (double*)lo.dptr,
                              (double*)so.dptr, residuals, mus, svd_seconds,
                              iter_seconds, col_bounds, nblocks);
    else
      r = ialm_device<float>(c, (const float*)mv.dptr, m, n, row_major, k, p, q, seed,
                             (const float*)ov.dptr, lam, mu0, rho, tol, max_iterations, (float*)lo.dptr,
                             (float*)so.dptr, residuals, mus, svd_seconds, iter_seconds,
                             col_bounds, nblocks);
    lo.flush();
    so.flush();
    BRSVD_CUDA(cudaStreamSynchronize(c.stream));
    if (iterations) *iterations = r.iterations;
    if (converged) *converged = r.converged ? 1 : 0;
    return (int)kOk;
  });
}

int brsvd_ialm_stream(brsvd_ctx* ctx, const void* M, int64_t m, int64_t n, int64_t ldm,
                      int dtype, int k, int p, int q, uint64_t seed, const void* omega,
                      double lam, double mu0, double rho, double tol, int max_iterations,
                      const int64_t* col_bounds, int nblocks, void* L, void* S, void* Y,
                      int nslots, int32_t* iterations, int32_t* converged, double* residuals,
                      double* mus, double* svd_seconds, double* iter_seconds) {
  return guarded([&] {
    BRSVD_REQUIRE(ctx != nullptr && M != nullptr && L && S && Y, kErrArg, "NULL argument");
    BRSVD_REQUIRE(residuals && mus && svd_seconds && iter_seconds, kErrArg,
                  "history arrays are required");
    BRSVD_REQUIRE(nblocks >= 1 && col_bounds != nullptr && col_bounds[0] == 0 &&
                      col_bounds[nblocks] == n,
                  kErrShape, "column blocks must tile [0, n)");
    Ctx& c = ctx->c;
    BRSVD_CUDA(cudaSetDevice(c.device));
    const size_t es = esize(dtype);
    BRSVD_REQUIRE(m >= 1 && n >= 1 && ldm >= m, kErrShape, "bad shape");
    BRSVD_REQUIRE(k >= 1 && p >= 0 && k + p <= std::min(m, n), kErrConfig,
                  "k + p exceeds min(m, n)");
    BRSVD_REQUIRE(q >= 0, kErrConfig, "power exponent must be non-negative");
    BRSVD_REQUIRE(rho > 1.0 && tol > 0.0 && max_iterations >= 1, kErrArg,
                  "rho must exceed 1, tol and max_iterations must be positive");
    BRSVD_REQUIRE(nslots >= 1, kErrArg, "nslots must be positive");
    std::vector<int64_t> bounds(col_bounds, col_bounds + nblocks + 1);
    InView ov(c, omega, n, k + p, n, es, omega ? BRSVD_HOST : BRSVD_DEVICE);
    IalmOut r;
    if (dtype == BRSVD_F64)
      r = ialm_stream<double>(c, (const double*)M, m, n, ldm, k, p, q, seed,
                              (const double*)ov.dptr, lam, mu0, rho, tol, max_iterations,
                              bounds, (double*)L, (double*)S, (double*)Y, nslots, residuals,
                              mus, svd_seconds, iter_seconds);
    else
      r = ialm_stream<float>(c, (const float*)M, m, n, ldm, k, p, q, seed,
                             (const float*)ov.dptr, lam, mu0, rho, tol, max_iterations, bounds,
                             (float*)L, (float*)S, (float*)Y, nslots, residuals, mus,
                             svd_seconds, iter_seconds);
    BRSVD_CUDA(cudaStreamSynchronize(c.stream));
    if (iterations) *iterations = r.iterations;
    if (converged) *converged = r.converged ? 1 : 0;
    return (int)kOk;
  });
}

int brsvd_gram(brsvd_ctx* ctx, const void* X, int64_t r, int64_t k1, int64_t ldx, int dtype,
               const void* W, int64_t k2, int64_t ldw, double* G) {
  return guarded([&] {
    BRSVD_REQUIRE(ctx != nullptr && X != nullptr && G != nullptr, kErrArg, "NULL argument");
    Ctx& c = ctx->c;
    BRSVD_CUDA(cudaSetDevice(c.device));
    esize(dtype);
    if (W == nullptr) {
      W = X;
      k2 = k1;
      ldw = ldx;
    }
    if (dtype == BRSVD_F64)
      gemm_tn_cm<double, double, double>(c, k1, k2, r, (const double*)X, ldx,
                                         (const double*)W, ldw, G, k1);
    else
      gemm_tn_cm<float, float, double>(c, k1, k2, r, (const float*)X, ldx, (const float*)W,
                                       ldw, G, k1);
    return (int)kOk;
  });
}

int brsvd_chol_basis(brsvd_ctx* ctx, double* G, int64_t l, double shift, double col_drop,
                     double rank_tol, double drop_ratio, double* T, int32_t* kept,
                     int32_t* rank_ref) {
  return guarded([&] {
    BRSVD_REQUIRE(ctx != nullptr && G != nullptr && T != nullptr, kErrArg, "NULL argument");
    Ctx& c = ctx->c;
    BRSVD_CUDA(cudaSetDevice(c.device));
    BRSVD_REQUIRE(l >= 1 && l <= kCholMaxL, kErrShape, "chol_basis supports 1 <= l <= 320");
    const int li = (int)l;
    DBuf<double> Wd(c, (size_t)l * l), info(c, 3), Tm(c, (size_t)l * l);
    DBuf<int> keep(c, l);
    cholinv_launch(c.stream, c.max_smem_optin, G, li, li, 1, col_drop, shift, drop_ratio,
                   rank_tol, Wd.p, Tm.p, nullptr, info.p, keep.p);
    BRSVD_CHECK_LAUNCH();
    BRSVD_CUDA(cudaMemsetAsync(T, 0, sizeof(double) * l * l, c.stream));
    compact_cols_kernel<<<grid_for((int64_t)l * l), 256, 0, c.stream>>>(Tm.p, li, keep.p,
                                                                        info.p, T);
    BRSVD_CHECK_LAUNCH();
    double h[3];
    readback(c, info.p, h, sizeof(h));
    if (kept) *kept = (int32_t)h[2];
    if (rank_ref) *rank_ref = (int32_t)h[1];
    return (int)kOk;
  });
}

int brsvd_apply(brsvd_ctx* ctx, const void* X, int64_t r, int64_t k, int64_t ldx, int dtype,
                const double* T, int64_t kt, void* out, int64_t ldo, int out_dtype,
                double alpha, double beta) {
  return guarded([&] {
    BRSVD_REQUIRE(ctx != nullptr && X != nullptr && T != nullptr && out != nullptr, kErrArg,
                  "NULL argument");
    Ctx& c = ctx->c;
    BRSVD_CUDA(cudaSetDevice(c.device));
    esize(dtype);
    esize(out_dtype);
#define BRSVD_APPLY(TX, TO)                                                                \
  gemm_nn_cm<TX, double, TO>(c, r, kt, k, (const TX*)X, ldx, T, k, (TO*)out, ldo, alpha, \
                             beta, beta != 0.0 ? (const TO*)out : nullptr, ldo)
    if (dtype == BRSVD_F32 && out_dtype == BRSVD_F32 && alpha == 1.0 && beta == 0.0)
      apply_basis<float>(c, (const float*)X, r, (int)k, ldx, T, k, (int)kt, (float*)out, ldo);
    else if (dtype == BRSVD_F64 && out_dtype == BRSVD_F64) BRSVD_APPLY(double, double);
    else if (dtype == BRSVD_F64) BRSVD_APPLY(double, float);
    else if (out_dtype == BRSVD_F64) BRSVD_APPLY(float, double);
    else BRSVD_APPLY(float, float);
#undef BRSVD_APPLY
    return (int)kOk;
  });
}

int brsvd_normalize(brsvd_ctx* ctx, const void* Z, int64_t n, int64_t l, int64_t ldz,
                    int dtype, void* Zout, int64_t ldo) {
  return guarded([&] {
    BRSVD_REQUIRE(ctx != nullptr && Z != nullptr && Zout != nullptr, kErrArg, "NULL argument");
    Ctx& c = ctx->c;
    BRSVD_CUDA(cudaSetDevice(c.device));
    esize(dtype);
    if (dtype == BRSVD_F64)
      normalize_sketch<double>(c, (const double*)Z, n, (int)l, ldz, (double*)Zout, ldo,
                               nullptr, /*scale_check=*/true);
    else
      normalize_sketch<float>(c, (const float*)Z, n, (int)l, ldz, (float*)Zout, ldo);
    return (int)kOk;
  });
}

int brsvd_colmax(brsvd_ctx* ctx, const void* U, int64_t r, int64_t l, int64_t ldu, int dtype,
                 int64_t row_offset, double* vals, int64_t* idx) {
  return guarded([&] {
    BRSVD_REQUIRE(ctx != nullptr && U != nullptr && vals && idx, kErrArg, "NULL argument");
    Ctx& c = ctx->c;
    BRSVD_CUDA(cudaSetDevice(c.device));
    esize(dtype);
    DBuf<double> dv(c, l);
    DBuf<int64_t> di(c, l);
    if (dtype == BRSVD_F64)
      colmax_kernel<double><<<(unsigned)l, 256, 0, c.stream>>>((const double*)U, r, ldu,
                                                               row_offset, dv.p, di.p);
    else
      colmax_kernel<float><<<(unsigned)l, 256, 0, c.stream>>>((const float*)U, r, ldu,
                                                              row_offset, dv.p, di.p);
    BRSVD_CHECK_LAUNCH();
    BRSVD_CUDA(cudaMemcpyAsync(vals, dv.p, sizeof(double) * l, cudaMemcpyDeviceToHost, c.stream));
    BRSVD_CUDA(cudaMemcpyAsync(idx, di.p, sizeof(int64_t) * l, cudaMemcpyDeviceToHost, c.stream));
    BRSVD_CUDA(cudaStreamSynchronize(c.stream));
    return (int)kOk;
  });
}

int brsvd_colmax_entries(brsvd_ctx* ctx, const void* U, int64_t r, int64_t l, int64_t ldu,
                         int dtype, int64_t row_offset, double* out) {
  return guarded([&] {
    BRSVD_REQUIRE(ctx != nullptr && U != nullptr && out != nullptr, kErrArg, "NULL argument");
    Ctx& c = ctx->c;
    BRSVD_CUDA(cudaSetDevice(c.device));
    esize(dtype);
    DBuf<double> dv(c, (size_t)3 * l);
    double* vals = dv.p;
    int64_t* idx = reinterpret_cast<int64_t*>(dv.p + l);
    double* ent = dv.p + 2 * l;
    if (dtype == BRSVD_F64)
      colmax_kernel<double><<<(unsigned)l, 256, 0, c.stream>>>((const double*)U, r, ldu,
                                                               row_offset, vals, idx, ent);
    else
      colmax_kernel<float><<<(unsigned)l, 256, 0, c.stream>>>((const float*)U, r, ldu,
                                                              row_offset, vals, idx, ent);
    BRSVD_CHECK_LAUNCH();
    // out = [vals (l) | idx as doubles (l) | signed entries (l)], one copy
    idx_to_double_kernel<<<grid_for(l), 256, 0, c.stream>>>(idx, l);
    BRSVD_CHECK_LAUNCH();
    BRSVD_CUDA(cudaMemcpyAsync(out, dv.p, sizeof(double) * 3 * l, cudaMemcpyDeviceToHost,
                               c.stream));
    BRSVD_CUDA(cudaStreamSynchronize(c.stream));
    return (int)kOk;
  });
}

int brsvd_stream_rows_pass(brsvd_ctx* ctx, const void* A, int64_t m, int64_t n, int64_t lda,
                           int dtype, int layout, const void* X, int64_t ldx, int64_t l,
                           void* Y, int64_t ldy, double* Z, int64_t ldz, int64_t panel,
                           int nbuf, double* pass_ms) {
  return guarded([&] {
    BRSVD_REQUIRE(ctx != nullptr && A != nullptr && Y != nullptr, kErrArg, "NULL argument");
    BRSVD_REQUIRE(X != nullptr || Z != nullptr, kErrArg, "nothing to compute");
    Ctx& c = ctx->c;
    BRSVD_CUDA(cudaSetDevice(c.device));
    esize(dtype);
    BRSVD_REQUIRE(m >= 0 && n >= 1 && l >= 1 && l <= 1024, kErrShape, "bad shape");
    BRSVD_REQUIRE(panel >= 1 && nbuf >= 1, kErrArg, "panel and nbuf must be positive");
    const bool row_major = layout == BRSVD_ROW_MAJOR;
    BRSVD_REQUIRE(lda >= (row_major ? n : m), kErrShape, "lda too small");
    PassInfo pi;
    if (dtype == BRSVD_F64)
      pi = stream_rows_pass<double>(c, (const double*)A, m, n, lda, row_major,
                                    (const double*)X, ldx, (int)l, (double*)Y, ldy, Z, ldz,
                                    panel, nbuf);
    else
      pi = stream_rows_pass<float>(c, (const float*)A, m, n, lda, row_major, (const float*)X,
                                   ldx, (int)l, (float*)Y, ldy, Z, ldz, panel, nbuf);
    if (pass_ms) *pass_ms = pi.ms;
    return (int)kOk;
  });
}

int brsvd_normalize_f64(brsvd_ctx* ctx, const double* Z, int64_t n, int64_t l, int64_t ldz,
                        int dtype, void* Zout, int64_t ldo, double* T, double* scale) {
  return guarded([&] {
    BRSVD_REQUIRE(ctx != nullptr && Z != nullptr && Zout != nullptr, kErrArg, "NULL argument");
    Ctx& c = ctx->c;
    BRSVD_CUDA(cudaSetDevice(c.device));
    esize(dtype);
    if (dtype == BRSVD_F64)
      normalize_from_f64<double>(c, Z, n, (int)l, ldz, (double*)Zout, ldo, T, scale);
    else
      normalize_from_f64<float>(c, Z, n, (int)l, ldz, (float*)Zout, ldo, T, scale);
    return (int)kOk;
  });
}

int brsvd_normalize_t(brsvd_ctx* ctx, const void* Z, int64_t n, int64_t l, int64_t ldz,
                      int dtype, void* Zout, int64_t ldo, double* T) {
  return guarded([&] {
    BRSVD_REQUIRE(ctx != nullptr && Z != nullptr && Zout != nullptr, kErrArg, "NULL argument");
    Ctx& c = ctx->c;
    BRSVD_CUDA(cudaSetDevice(c.device));
    esize(dtype);
    if (dtype == BRSVD_F64)   // fp64 near the exponent limits: Gram at unit scale
      normalize_sketch<double>(c, (const double*)Z, n, (int)l, ldz, (double*)Zout, ldo, T,
                               /*scale_check=*/true);
    else
      normalize_sketch<float>(c, (const float*)Z, n, (int)l, ldz, (float*)Zout, ldo, T);
    return (int)kOk;
  });
}

int brsvd_unnormalised_peak(brsvd_ctx* ctx, const void* Yq, int64_t m, int64_t l, int dtype,
                            int q, const double* Ts, const double* zfac, double* peak) {
  return guarded([&] {
    BRSVD_REQUIRE(ctx != nullptr && Yq != nullptr && Ts != nullptr && zfac && peak, kErrArg,
                  "NULL argument");
    BRSVD_REQUIRE(q >= 1 && l >= 1 && m >= 0, kErrArg, "bad shape");
    Ctx& c = ctx->c;
    BRSVD_CUDA(cudaSetDevice(c.device));
    esize(dtype);
    if (m == 0) {
      *peak = 0.0;
      return (int)kOk;
    }
    *peak = dtype == BRSVD_F64
                ? unnormalised_peak<double>(c, (const double*)Yq, m, (int)l, q, Ts, zfac)
                : unnormalised_peak<float>(c, (const float*)Yq, m, (int)l, q, Ts, zfac);
    return (int)kOk;
  });
}

int brsvd_scale_cols(brsvd_ctx* ctx, void* X, int64_t r, int64_t l, int64_t ldx, int dtype,
                     const double* scale) {
  return guarded([&] {
    BRSVD_REQUIRE(ctx != nullptr && X != nullptr && scale != nullptr, kErrArg, "NULL argument");
    Ctx& c = ctx->c;
    BRSVD_CUDA(cudaSetDevice(c.device));
    esize(dtype);
    DBuf<double> ds(c, l);
    BRSVD_CUDA(cudaMemcpyAsync(ds.p, scale, sizeof(double) * l, cudaMemcpyHostToDevice,
                               c.stream));
    if (dtype == BRSVD_F64)
      scale_cols_by_kernel<double, double><<<grid_for(r * l), 256, 0, c.stream>>>(
          (double*)X, r, l, ldx, ds.p);
    else
      scale_cols_by_kernel<float, double><<<grid_for(r * l), 256, 0, c.stream>>>(
          (float*)X, r, l, ldx, ds.p);
    BRSVD_CHECK_LAUNCH();
    return (int)kOk;
  });
}

}  // extern "C"
