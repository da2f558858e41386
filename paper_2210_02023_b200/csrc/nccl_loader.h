// nccl_loader.h — NCCL resolved at run time, only when a multi-rank context
// is created. The process usually already holds torch's libnccl.so.2 (which
// is newer than the system one); binding to the library already loaded
// avoids two NCCLs with one soname in one process. SP_NCCL_LIBRARY
// overrides the path.
#pragma once

#include <dlfcn.h>
#include <nccl.h>

#include <cstdlib>
#include <mutex>
#include <string>

#include "common.h"

namespace sp {

struct NcclApi {
  ncclResult_t (*GetUniqueId)(ncclUniqueId*) = nullptr;
  ncclResult_t (*CommInitRank)(ncclComm_t*, int, ncclUniqueId, int) = nullptr;
  ncclResult_t (*CommDestroy)(ncclComm_t) = nullptr;
  const char* (*GetErrorString)(ncclResult_t) = nullptr;
  ncclResult_t (*AllReduce)(const void*, void*, size_t, ncclDataType_t, ncclRedOp_t,
                            ncclComm_t, cudaStream_t) = nullptr;
  ncclResult_t (*AllGather)(const void*, void*, size_t, ncclDataType_t, ncclComm_t,
                            cudaStream_t) = nullptr;
  ncclResult_t (*Send)(const void*, size_t, ncclDataType_t, int, ncclComm_t,
                       cudaStream_t) = nullptr;
  ncclResult_t (*Recv)(void*, size_t, ncclDataType_t, int, ncclComm_t,
                       cudaStream_t) = nullptr;
  ncclResult_t (*GroupStart)() = nullptr;
  ncclResult_t (*GroupEnd)() = nullptr;
};

inline const NcclApi& nccl() {
  static NcclApi api;
  static std::once_flag once;
  static std::string err;
  std::call_once(once, [] {
    void* h = nullptr;
    if (const char* p = std::getenv("SP_NCCL_LIBRARY")) h = dlopen(p, RTLD_NOW | RTLD_GLOBAL);
    if (!h) h = dlopen("libnccl.so.2", RTLD_NOW | RTLD_NOLOAD | RTLD_GLOBAL);
    if (!h) h = dlopen("libnccl.so.2", RTLD_NOW | RTLD_GLOBAL);
    if (!h) {
      err = std::string("cannot load libnccl.so.2: ") + dlerror();
      return;
    }
#define SP_SYM(f)                                                         \
  api.f = reinterpret_cast<decltype(api.f)>(dlsym(h, "nccl" #f));         \
  if (!api.f) err += std::string(" missing nccl" #f);
    SP_SYM(GetUniqueId)
    SP_SYM(CommInitRank)
    SP_SYM(CommDestroy)
    SP_SYM(GetErrorString)
    SP_SYM(AllReduce)
    SP_SYM(AllGather)
    SP_SYM(Send)
    SP_SYM(Recv)
    SP_SYM(GroupStart)
    SP_SYM(GroupEnd)
#undef SP_SYM
  });
  if (!err.empty()) raise(SP_ERR_NCCL, err);
  return api;
}

}  // namespace sp

#define SP_NCCL(x)                                                             \
  do {                                                                         \
    ncclResult_t r_ = (x);                                                     \
    if (r_ != ncclSuccess)                                                     \
      ::sp::raise(SP_ERR_NCCL,                                                 \
                  std::string(#x) + ": " + ::sp::nccl().GetErrorString(r_));   \
  } while (0)
