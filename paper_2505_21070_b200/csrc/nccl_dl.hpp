// NCCL loaded lazily with dlopen, so the library does not pin a libnccl.so.2
// at load time (torch bundles a newer NCCL under the same soname; whichever is
// already loaded in the process, or BP_NCCL_LIB, or the system one is used).
#pragma once

#include <dlfcn.h>
#include <nccl.h>

#include <cstdlib>
#include <mutex>
#include <string>

#include "common.hpp"

namespace bp {

struct NcclApi {
  ncclResult_t (*GetUniqueId)(ncclUniqueId*) = nullptr;
  ncclResult_t (*CommInitRank)(ncclComm_t*, int, ncclUniqueId, int) = nullptr;
  ncclResult_t (*CommDestroy)(ncclComm_t) = nullptr;
  ncclResult_t (*CommAbort)(ncclComm_t) = nullptr;
  ncclResult_t (*Send)(const void*, size_t, ncclDataType_t, int, ncclComm_t, cudaStream_t) = nullptr;
  ncclResult_t (*Recv)(void*, size_t, ncclDataType_t, int, ncclComm_t, cudaStream_t) = nullptr;
  const char* (*GetErrorString)(ncclResult_t) = nullptr;
  // user-buffer API (NCCL >= 2.19); null when the loaded NCCL lacks it
  ncclResult_t (*MemAlloc)(void**, size_t) = nullptr;
  ncclResult_t (*MemFree)(void*) = nullptr;
  ncclResult_t (*CommRegister)(ncclComm_t, void*, size_t, void**) = nullptr;
  ncclResult_t (*CommDeregister)(ncclComm_t, void*) = nullptr;
};

inline const NcclApi& nccl() {
  static NcclApi api;
  static std::once_flag once;
  static std::string err;
  std::call_once(once, [] {
    void* h = dlopen("libnccl.so.2", RTLD_NOW | RTLD_NOLOAD);  // already in the process (e.g. torch's)
    if (!h) {
      const char* env = std::getenv("BP_NCCL_LIB");
      if (env && *env) h = dlopen(env, RTLD_NOW | RTLD_GLOBAL);
    }
    if (!h) h = dlopen("libnccl.so.2", RTLD_NOW | RTLD_GLOBAL);
    if (!h) {
      err = dlerror();
      return;
    }
    api.GetUniqueId = reinterpret_cast<decltype(api.GetUniqueId)>(dlsym(h, "ncclGetUniqueId"));
    api.CommInitRank = reinterpret_cast<decltype(api.CommInitRank)>(dlsym(h, "ncclCommInitRank"));
    api.CommDestroy = reinterpret_cast<decltype(api.CommDestroy)>(dlsym(h, "ncclCommDestroy"));
    api.CommAbort = reinterpret_cast<decltype(api.CommAbort)>(dlsym(h, "ncclCommAbort"));
    api.Send = reinterpret_cast<decltype(api.Send)>(dlsym(h, "ncclSend"));
    api.Recv = reinterpret_cast<decltype(api.Recv)>(dlsym(h, "ncclRecv"));
    api.GetErrorString = reinterpret_cast<decltype(api.GetErrorString)>(dlsym(h, "ncclGetErrorString"));
    api.MemAlloc = reinterpret_cast<decltype(api.MemAlloc)>(dlsym(h, "ncclMemAlloc"));
    api.MemFree = reinterpret_cast<decltype(api.MemFree)>(dlsym(h, "ncclMemFree"));
    api.CommRegister = reinterpret_cast<decltype(api.CommRegister)>(dlsym(h, "ncclCommRegister"));
    api.CommDeregister = reinterpret_cast<decltype(api.CommDeregister)>(dlsym(h, "ncclCommDeregister"));
  });
  if (!api.Send) fail(BP_ERR_NCCL, "NCCL unavailable: " + err);
  return api;
}

}  // namespace bp
