// nccl_dyn.hpp -- NCCL resolved at run time (dlopen), not at link time.
//
// torch ships its own libnccl.so.2 (2.28.x); the system one is 2.27.3.  Linking
// -lnccl would let whichever loads first win the soname and break the other
// (torch needs symbols 2.27 lacks).  So the library binds NCCL lazily, reusing a
// libnccl.so.2 already in the process when there is one.
#pragma once
#include <dlfcn.h>
#include <nccl.h>

#include <mutex>
#include <stdexcept>
#include <string>

namespace lmra_host {

struct NcclApi {
  decltype(&ncclGetUniqueId) GetUniqueId = nullptr;
  decltype(&ncclCommInitRank) CommInitRank = nullptr;
  decltype(&ncclCommDestroy) CommDestroy = nullptr;
  decltype(&ncclCommAbort) CommAbort = nullptr;
  decltype(&ncclCommInitAll) CommInitAll = nullptr;
  decltype(&ncclAllReduce) AllReduce = nullptr;
  decltype(&ncclAllGather) AllGather = nullptr;
  decltype(&ncclBroadcast) Broadcast = nullptr;
  decltype(&ncclGroupStart) GroupStart = nullptr;
  decltype(&ncclGroupEnd) GroupEnd = nullptr;
  decltype(&ncclGetErrorString) GetErrorString = nullptr;
};

inline const NcclApi& nccl() {
  static NcclApi api;
  static std::once_flag once;
  static std::string err;
  std::call_once(once, [] {
    void* h = dlopen("libnccl.so.2", RTLD_NOW | RTLD_NOLOAD);
    if (!h) h = dlopen("libnccl.so.2", RTLD_NOW | RTLD_GLOBAL);
    if (!h) {
      err = std::string("cannot load libnccl.so.2: ") + dlerror();
      return;
    }
#define LMRA_NCCL_SYM(field, name) api.field = reinterpret_cast<decltype(api.field)>(dlsym(h, name))
    LMRA_NCCL_SYM(GetUniqueId, "ncclGetUniqueId");
    LMRA_NCCL_SYM(CommInitRank, "ncclCommInitRank");
    LMRA_NCCL_SYM(CommDestroy, "ncclCommDestroy");
    LMRA_NCCL_SYM(CommAbort, "ncclCommAbort");
    LMRA_NCCL_SYM(CommInitAll, "ncclCommInitAll");
    LMRA_NCCL_SYM(AllReduce, "ncclAllReduce");
    LMRA_NCCL_SYM(AllGather, "ncclAllGather");
    LMRA_NCCL_SYM(Broadcast, "ncclBroadcast");
    LMRA_NCCL_SYM(GroupStart, "ncclGroupStart");
    LMRA_NCCL_SYM(GroupEnd, "ncclGroupEnd");
    LMRA_NCCL_SYM(GetErrorString, "ncclGetErrorString");
#undef LMRA_NCCL_SYM
    if (!api.GetUniqueId || !api.CommInitRank || !api.AllReduce || !api.AllGather)
      err = "libnccl.so.2 lacks required symbols";
  });
  if (!err.empty()) throw std::runtime_error(err);
  return api;
}

}  // namespace lmra_host
