#include "nccl_loader.hpp"

#include <dlfcn.h>

#include <mutex>
#include <string>

#include "fpmm_b200.h"
#include "rules.hpp"

namespace fpmm_b200 {

namespace {
template <typename F>
void bind(void* h, F& fn, const char* name) {
  fn = reinterpret_cast<F>(dlsym(h, name));
  if (!fn) throw Failure(FPMM_B200_ENCCL, std::string("libnccl.so.2 lacks ") + name);
}
}  // namespace

const NcclApi& nccl() {
  static NcclApi api{};
  static std::once_flag once;
  static std::string err;
  std::call_once(once, [] {
    void* h = dlopen("libnccl.so.2", RTLD_NOW | RTLD_NOLOAD);
    if (!h) h = dlopen("libnccl.so.2", RTLD_NOW | RTLD_GLOBAL);
    if (!h) h = dlopen("/usr/lib/x86_64-linux-gnu/libnccl.so.2", RTLD_NOW | RTLD_GLOBAL);
    if (!h) {
      err = std::string("cannot load libnccl.so.2: ") + dlerror();
      return;
    }
    try {
      bind(h, api.GetUniqueId, "ncclGetUniqueId");
      bind(h, api.CommInitRank, "ncclCommInitRank");
      bind(h, api.CommInitAll, "ncclCommInitAll");
      bind(h, api.CommDestroy, "ncclCommDestroy");
      bind(h, api.Broadcast, "ncclBroadcast");
      bind(h, api.AllReduce, "ncclAllReduce");
      bind(h, api.Send, "ncclSend");
      bind(h, api.Recv, "ncclRecv");
      bind(h, api.GroupStart, "ncclGroupStart");
      bind(h, api.GroupEnd, "ncclGroupEnd");
      bind(h, api.GetErrorString, "ncclGetErrorString");
    } catch (const Failure& f) {
      err = f.what();
      api = NcclApi{};
    }
  });
  if (!api.GetUniqueId) throw Failure(FPMM_B200_ENCCL, err.empty() ? "NCCL unavailable" : err);
  return api;
}

}  // namespace fpmm_b200
