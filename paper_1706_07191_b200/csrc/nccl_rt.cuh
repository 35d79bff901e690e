// NCCL for the row-sharded decomposition, resolved at run time.
//
// The sharded path (BASELINE config 4) exchanges per pass the
// n x l partial Z, the l x l Grams and B^T (all-reduce sum), the first
// sample's peak (all-reduce max) and the sign candidates (all-gather).  A
// context can own an NCCL communicator for these (brsvd_ctx_attach_nccl),
// so the collectives run on the library's stream, in stream order with the
// kernels that produce and consume them, and failures surface as
// BRSVD_ERR_NCCL.  libnccl is opened with dlopen rather than linked: the
// process usually has one loaded already (PyTorch's), and a second copy of a
// different version must not be forced into it.
#pragma once
#include <dlfcn.h>

#include <cstring>
#include <mutex>

#include "common.cuh"

namespace brsvd {
namespace nccl {

// The subset of nccl.h this library uses (the ABI has been stable since 2.x).
typedef struct ncclComm* ncclComm_t;
constexpr int kUniqueIdBytes = 128;
typedef struct {
  char internal[kUniqueIdBytes];
} ncclUniqueId;
typedef int ncclResult_t;   // 0 = ncclSuccess
enum DataType { kInt8 = 0, kInt32 = 2, kInt64 = 4, kFloat32 = 7, kFloat64 = 8 };
enum RedOp { kSum = 0, kProd = 1, kMax = 2, kMin = 3 };

struct Api {
  ncclResult_t (*GetUniqueId)(ncclUniqueId*) = nullptr;
  ncclResult_t (*CommInitRank)(ncclComm_t*, int, ncclUniqueId, int) = nullptr;
  ncclResult_t (*CommDestroy)(ncclComm_t) = nullptr;
  ncclResult_t (*AllReduce)(const void*, void*, size_t, int, int, ncclComm_t,
                            cudaStream_t) = nullptr;
  ncclResult_t (*AllGather)(const void*, void*, size_t, int, ncclComm_t,
                            cudaStream_t) = nullptr;
  const char* (*GetErrorString)(ncclResult_t) = nullptr;
  ncclResult_t (*GetVersion)(int*) = nullptr;
};

inline const Api& api() {
  static Api a;
  static std::once_flag once;
  static std::string why;
  std::call_once(once, [] {
    void* h = nullptr;
    const char* override_path = std::getenv("BRSVD_NCCL_LIB");
    for (const char* name : {override_path, "libnccl.so.2", "libnccl.so"}) {
      if (name == nullptr) continue;
      h = dlopen(name, RTLD_NOW | RTLD_GLOBAL);
      if (h) break;
    }
    if (!h) {
      why = "libnccl.so.2 not found (set BRSVD_NCCL_LIB)";
      return;
    }
    auto sym = [&](const char* s) { return dlsym(h, s); };
    a.GetUniqueId = (decltype(a.GetUniqueId))sym("ncclGetUniqueId");
    a.CommInitRank = (decltype(a.CommInitRank))sym("ncclCommInitRank");
    a.CommDestroy = (decltype(a.CommDestroy))sym("ncclCommDestroy");
    a.AllReduce = (decltype(a.AllReduce))sym("ncclAllReduce");
    a.AllGather = (decltype(a.AllGather))sym("ncclAllGather");
    a.GetErrorString = (decltype(a.GetErrorString))sym("ncclGetErrorString");
    a.GetVersion = (decltype(a.GetVersion))sym("ncclGetVersion");
  });
  if (!a.GetUniqueId || !a.CommInitRank || !a.AllReduce || !a.AllGather)
    throw Error(kErrNccl, why.empty() ? "NCCL symbols missing" : why);
  return a;
}

inline void check(ncclResult_t r, const char* what) {
  if (r != 0) {
    const char* s = api().GetErrorString ? api().GetErrorString(r) : "unknown";
    throw Error(kErrNccl, std::string(what) + ": " + s);
  }
}

inline int dtype_of(int code) {   // BRSVD_F64 = 1, BRSVD_F32 = 2, 3 = int64
  if (code == 1) return kFloat64;
  if (code == 2) return kFloat32;
  if (code == 3) return kInt64;
  throw Error(kErrArg, "collective dtype must be 1 (f64), 2 (f32) or 3 (int64)");
}

}  // namespace nccl
}  // namespace brsvd
