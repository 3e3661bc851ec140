// NCCL, resolved at run time (dlopen): the library links no NCCL, and a
// process that already loaded one (torch.distributed's) shares it — the
// soname lookup returns the loaded copy.  Only the five calls of the
// edge-sharded backend are bound (reduce / broadcast over NVLink).
#pragma once
#include <dlfcn.h>
#include <nccl.h>

#include "pmx_common.cuh"

namespace pmx {

struct NcclApi {
  ncclResult_t (*GetUniqueId)(ncclUniqueId*) = nullptr;
  ncclResult_t (*CommInitRank)(ncclComm_t*, int, ncclUniqueId, int) = nullptr;
  ncclResult_t (*CommDestroy)(ncclComm_t) = nullptr;
  ncclResult_t (*Reduce)(const void*, void*, size_t, ncclDataType_t, ncclRedOp_t, int, ncclComm_t,
                         cudaStream_t) = nullptr;
  ncclResult_t (*Broadcast)(const void*, void*, size_t, ncclDataType_t, int, ncclComm_t, cudaStream_t) = nullptr;
  const char* (*GetErrorString)(ncclResult_t) = nullptr;
};

inline NcclApi& nccl_api() {
  static NcclApi api;
  static bool tried = false;
  if (!tried) {
    tried = true;
    void* h = dlopen("libnccl.so.2", RTLD_NOW | RTLD_NOLOAD | RTLD_GLOBAL);  // already loaded (torch)
    if (!h) h = dlopen("libnccl.so.2", RTLD_NOW | RTLD_GLOBAL);
    if (h) {
      api.GetUniqueId = reinterpret_cast<decltype(api.GetUniqueId)>(dlsym(h, "ncclGetUniqueId"));
      api.CommInitRank = reinterpret_cast<decltype(api.CommInitRank)>(dlsym(h, "ncclCommInitRank"));
      api.CommDestroy = reinterpret_cast<decltype(api.CommDestroy)>(dlsym(h, "ncclCommDestroy"));
      api.Reduce = reinterpret_cast<decltype(api.Reduce)>(dlsym(h, "ncclReduce"));
      api.Broadcast = reinterpret_cast<decltype(api.Broadcast)>(dlsym(h, "ncclBroadcast"));
      api.GetErrorString = reinterpret_cast<decltype(api.GetErrorString)>(dlsym(h, "ncclGetErrorString"));
    }
  }
  if (!api.GetUniqueId || !api.CommInitRank || !api.Reduce || !api.Broadcast)
    throw Error(PMX_ERR_NCCL, "NCCL (libnccl.so.2) not available");
  return api;
}

#define PMX_NCCL(call)                                                                                    \
  do {                                                                                                    \
    ncclResult_t r_ = (call);                                                                             \
    if (r_ != ncclSuccess)                                                                                \
      throw ::pmx::Error(PMX_ERR_NCCL, std::string(#call) + ": " +                                        \
                                           (::pmx::nccl_api().GetErrorString                              \
                                                ? ::pmx::nccl_api().GetErrorString(r_)                    \
                                                : "error"));                                              \
  } while (0)

}  // namespace pmx
