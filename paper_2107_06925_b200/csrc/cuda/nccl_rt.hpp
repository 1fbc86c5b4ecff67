// NCCL resolved at run time (dlopen) instead of at link time.
//
// libchimera.so must coexist with whatever NCCL the host process already uses (e.g.
// torch's bundled libnccl.so.2): a link-time dependency would pin one copy by soname
// and break the other.  The library is only needed by multi-process training, so it
// is looked up lazily at connect(): an already-loaded libnccl.so.2 first, else
// $CK_NCCL_LIB, else the loader's default search.
#pragma once

#include <dlfcn.h>
#include <nccl.h>

#include <cstdlib>
#include <mutex>
#include <string>

#include "capi_util.hpp"

namespace chimera::gpt {

struct Nccl {
  decltype(&ncclGetUniqueId) GetUniqueId = nullptr;
  decltype(&ncclCommInitRank) CommInitRank = nullptr;
  decltype(&ncclCommInitRankConfig) CommInitRankConfig = nullptr;  // optional (CTA caps)
  decltype(&ncclCommSplit) CommSplit = nullptr;
  decltype(&ncclAllReduce) AllReduce = nullptr;
  decltype(&ncclReduceScatter) ReduceScatter = nullptr;
  decltype(&ncclAllGather) AllGather = nullptr;
  decltype(&ncclCommDestroy) CommDestroy = nullptr;
  decltype(&ncclGetErrorString) GetErrorString = nullptr;

  static const Nccl& get() {
    static Nccl n;
    static std::once_flag once;
    std::call_once(once, [] {
      void* h = dlopen("libnccl.so.2", RTLD_NOW | RTLD_NOLOAD);
      if (!h && std::getenv("CK_NCCL_LIB")) h = dlopen(std::getenv("CK_NCCL_LIB"), RTLD_NOW | RTLD_GLOBAL);
      if (!h) h = dlopen("libnccl.so.2", RTLD_NOW | RTLD_GLOBAL);
      if (!h) throw capi::InternalError(std::string("cannot load libnccl.so.2: ") + dlerror());
      auto sym = [&](const char* name) {
        void* p = dlsym(h, name);
        if (!p) throw capi::InternalError(std::string("NCCL symbol missing: ") + name);
        return p;
      };
      n.GetUniqueId = reinterpret_cast<decltype(n.GetUniqueId)>(sym("ncclGetUniqueId"));
      n.CommInitRank = reinterpret_cast<decltype(n.CommInitRank)>(sym("ncclCommInitRank"));
      n.CommInitRankConfig =
          reinterpret_cast<decltype(n.CommInitRankConfig)>(dlsym(h, "ncclCommInitRankConfig"));
      n.CommSplit = reinterpret_cast<decltype(n.CommSplit)>(sym("ncclCommSplit"));
      n.AllReduce = reinterpret_cast<decltype(n.AllReduce)>(sym("ncclAllReduce"));
      n.ReduceScatter = reinterpret_cast<decltype(n.ReduceScatter)>(sym("ncclReduceScatter"));
      n.AllGather = reinterpret_cast<decltype(n.AllGather)>(sym("ncclAllGather"));
      n.CommDestroy = reinterpret_cast<decltype(n.CommDestroy)>(sym("ncclCommDestroy"));
      n.GetErrorString = reinterpret_cast<decltype(n.GetErrorString)>(sym("ncclGetErrorString"));
    });
    return n;
  }
};

}  // namespace chimera::gpt
