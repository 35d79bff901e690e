// Shared helpers for the BRSVD sm_100a kernels and the C++ runtime.
#pragma once
#include <cuda_runtime.h>
#include <cstdint>
#include <stdexcept>
#include <string>

namespace brsvd {

// Status codes mirror include/brsvd.h.
enum Status : int {
  kOk = 0,
  kErrConfig = 1,
  kErrShape = 2,
  kErrBudget = 3,
  kErrOverflow = 4,
  kErrCuda = 5,
  kErrNccl = 6,
  kErrArg = 7,
};

struct Error : std::runtime_error {
  int code;
  Error(int c, const std::string& m) : std::runtime_error(m), code(c) {}
};

#define BRSVD_CUDA(x)                                                          \
  do {                                                                         \
    cudaError_t e_ = (x);                                                      \
    if (e_ != cudaSuccess)                                                     \
      throw ::brsvd::Error(::brsvd::kErrCuda, std::string(#x) + ": " +         \
                                                  cudaGetErrorString(e_));     \
  } while (0)

// Every kernel launch site ends with BRSVD_CHECK_LAUNCH(), which also counts
// the launch (brsvd_profile_end reports the count as `gpu_launches`).
extern thread_local long long g_brsvd_launches;
#define BRSVD_CHECK_LAUNCH()           \
  do {                                 \
    ++::brsvd::g_brsvd_launches;       \
    BRSVD_CUDA(cudaGetLastError());    \
  } while (0)

#define BRSVD_REQUIRE(cond, code, msg)                                         \
  do {                                                                         \
    if (!(cond)) throw ::brsvd::Error((code), (msg));                          \
  } while (0)

constexpr int kNumSMs = 148;

inline int64_t ceil_div(int64_t a, int64_t b) { return (a + b - 1) / b; }

template <typename T>
__device__ __forceinline__ T warp_sum(T v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  return v;
}

template <typename T>
__device__ __forceinline__ T warp_max(T v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v = max(v, __shfl_xor_sync(0xffffffffu, v, o));
  return v;
}

template <typename T> struct DTypeCode;
template <> struct DTypeCode<double> { static constexpr int value = 1; };
template <> struct DTypeCode<float> { static constexpr int value = 2; };

}  // namespace brsvd
