// nccl_dyn.h — the few NCCL entry points the subtree-split data plane uses, resolved at run time.
//
// The library does not link libnccl: a process that already loaded NCCL (e.g. PyTorch's bundled
// libnccl.so.2) must hand us communicators of THAT library instance, so the symbols are taken from
// the loaded copy when there is one (dlopen RTLD_NOLOAD), else libnccl.so.2 is loaded. The types
// below are the stable NCCL 2.x ABI (nccl.h: ncclUniqueId is 128 bytes, ncclFloat32 = 7,
// ncclFloat64 = 8, ncclSuccess = 0).
#pragma once

#include <cuda_runtime.h>
#include <dlfcn.h>

#include <cstddef>
#include <mutex>
#include <string>

namespace gofmm {
namespace nccl {

struct Comm;  // opaque ncclComm
using comm_t = Comm*;
struct UniqueId {
  char internal[128];
};
using result_t = int;
enum : int { kSuccess = 0, kFloat32 = 7, kFloat64 = 8 };

struct Api {
  result_t (*GetUniqueId)(UniqueId*) = nullptr;
  result_t (*CommInitRank)(comm_t*, int, UniqueId, int) = nullptr;
  result_t (*CommDestroy)(comm_t) = nullptr;
  result_t (*CommCount)(const comm_t, int*) = nullptr;
  result_t (*CommUserRank)(const comm_t, int*) = nullptr;
  result_t (*AllGather)(const void*, void*, size_t, int, comm_t, cudaStream_t) = nullptr;
  const char* (*GetErrorString)(result_t) = nullptr;
  result_t (*GetVersion)(int*) = nullptr;
  void* handle = nullptr;
  std::string error;
};

// Resolve once per process; returns nullptr (and sets *why) when NCCL is unavailable.
inline const Api* api(std::string* why) {
  static Api a;
  static std::once_flag once;
  std::call_once(once, [] {
    const char* names[] = {"libnccl.so.2", "libnccl.so"};
    for (const char* nm : names) {
      a.handle = dlopen(nm, RTLD_NOW | RTLD_NOLOAD);  // already in the process (torch)
      if (a.handle) break;
    }
    for (const char* nm : names) {
      if (a.handle) break;
      a.handle = dlopen(nm, RTLD_NOW | RTLD_GLOBAL);
    }
    if (!a.handle) {
      const char* e = dlerror();
      a.error = std::string("NCCL not found (libnccl.so.2): ") + (e ? e : "");
      return;
    }
    auto sym = [&](const char* n) { return dlsym(a.handle, n); };
    a.GetUniqueId = reinterpret_cast<decltype(a.GetUniqueId)>(sym("ncclGetUniqueId"));
    a.CommInitRank = reinterpret_cast<decltype(a.CommInitRank)>(sym("ncclCommInitRank"));
    a.CommDestroy = reinterpret_cast<decltype(a.CommDestroy)>(sym("ncclCommDestroy"));
    a.CommCount = reinterpret_cast<decltype(a.CommCount)>(sym("ncclCommCount"));
    a.CommUserRank = reinterpret_cast<decltype(a.CommUserRank)>(sym("ncclCommUserRank"));
    a.AllGather = reinterpret_cast<decltype(a.AllGather)>(sym("ncclAllGather"));
    a.GetErrorString = reinterpret_cast<decltype(a.GetErrorString)>(sym("ncclGetErrorString"));
    a.GetVersion = reinterpret_cast<decltype(a.GetVersion)>(sym("ncclGetVersion"));
    if (!a.GetUniqueId || !a.CommInitRank || !a.CommDestroy || !a.CommCount || !a.CommUserRank || !a.AllGather ||
        !a.GetErrorString) {
      a.error = "libnccl.so.2 lacks an entry point the data plane needs";
      a.handle = nullptr;
    }
  });
  if (!a.handle) {
    if (why) *why = a.error;
    return nullptr;
  }
  return &a;
}

}  // namespace nccl
}  // namespace gofmm
