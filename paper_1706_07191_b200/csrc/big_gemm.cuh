// The two products that stream the big matrix A once per call:
//   big_nn:  Y (m x l) = A X,    X (n x l)     -- sample pass
//   big_tn:  Z (n x l) = A^T Y,  Y (m x l)     -- transpose pass
// They replace `a_block @ omega` / `a_block.T @ y` of _sketch_block
// (rsvd.py:94-102) and `q_basis.T @ a` (rsvd.py:140).  A may be row- or
// column-major; the tall-skinny operands are column-major.
#pragma once
#include "runtime.cuh"
#include "tc_stream.cuh"
#include "skinny64.cuh"

namespace brsvd {

// amax (optional): max |A| per row (big_nn) / per column (big_tn), float,
// for the fp16-split products (absmax_rows_cols once per decomposition, or
// sampled: amax_out / run_flag, see LazyScales in pipeline.cuh).
// out_scale (big_tn, power of two): the fp16-split product returns
// out_scale * A^T Y, rounded once -- the power iteration uses it to keep
// A^T Y in fp32 range for inputs of extreme magnitude (other paths ignore it;
// the sample is renormalised right after, so the factor never shows).
template <typename T>
void big_nn(Ctx& c, const T* A, int64_t m, int64_t n, int64_t lda, bool row_major,
            const T* X, int64_t ldx, int l, T* Y, int64_t ldy, const float* amax = nullptr,
            unsigned* amax_out = nullptr, const int* run_flag = nullptr) {
  // a re-run on exact scales (run_flag) normally exits at once: not profiled
  ProfScope ps(c, 2.0 * m * n * l, (double)m * n * sizeof(T), run_flag == nullptr);
  if (tc_gemm_supported<T>(c, A, lda, m, n, l)) {
    if constexpr (sizeof(T) == 4) {
      tc_product(c, A, m, n, lda, row_major, /*trans=*/false, X, ldx, l, Y, ldy, amax, 1.0,
                 amax_out, run_flag);
      return;
    }
  }
  BRSVD_REQUIRE(amax_out == nullptr && run_flag == nullptr, kErrArg,
                "big_nn: sampled scales need the fp16-split product");
  if constexpr (sizeof(T) == 8) {
    if (skinny_f64(c, row_major, reinterpret_cast<const double*>(A), m, n, lda,
                   reinterpret_cast<const double*>(X), ldx, l,
                   reinterpret_cast<double*>(Y), ldy))
      return;
  }
  const int64_t sam = row_major ? lda : 1, sak = row_major ? 1 : lda;
  gemm<T, T, T, T>(c, m, l, n, A, sam, sak, X, 1, ldx, Y, 1, ldy);
}

template <typename T>
void big_tn(Ctx& c, const T* A, int64_t m, int64_t n, int64_t lda, bool row_major,
            const T* Yin, int64_t ldy, int l, T* Z, int64_t ldz, const float* amax = nullptr,
            double out_scale = 1.0, unsigned* amax_out = nullptr,
            const int* run_flag = nullptr) {
  ProfScope ps(c, 2.0 * m * n * l, (double)m * n * sizeof(T), run_flag == nullptr);
  if (tc_gemm_supported<T>(c, A, lda, m, n, l)) {
    if constexpr (sizeof(T) == 4) {
      tc_product(c, A, m, n, lda, row_major, /*trans=*/true, Yin, ldy, l, Z, ldz, amax,
                 out_scale, amax_out, run_flag);
      return;
    }
  }
  BRSVD_REQUIRE(amax_out == nullptr && run_flag == nullptr, kErrArg,
                "big_tn: sampled scales need the fp16-split product");
  if constexpr (sizeof(T) == 8) {
    if (skinny_f64(c, !row_major, reinterpret_cast<const double*>(A), n, m, lda,
                   reinterpret_cast<const double*>(Yin), ldy, l,
                   reinterpret_cast<double*>(Z), ldz))
      return;
  }
  const int64_t sam = row_major ? 1 : lda, sak = row_major ? lda : 1;
  gemm<T, T, T, T>(c, n, l, m, A, sam, sak, Yin, 1, ldy, Z, 1, ldz);
}

}  // namespace brsvd
