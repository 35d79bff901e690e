// tcgen05 (5th-gen tensor core) path for the big tall-skinny products.
// Placeholder until the 3xTF32 kernel lands: the SIMT path handles every case.
#pragma once
#include "runtime.cuh"

namespace brsvd {

template <typename T>
bool tc_gemm_supported(Ctx&, bool, int64_t, int64_t, int, bool) {
  return false;
}

template <typename T>
void tc_gemm_launch(Ctx&, const T*, int64_t, int64_t, int64_t, bool, bool, const T*,
                    int64_t, int, T*, int64_t) {}

}  // namespace brsvd
