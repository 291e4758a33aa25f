// nccl_dl.cpp -- see nccl_dl.hpp.
#include "nccl_dl.hpp"

#include <dlfcn.h>

#include <mutex>

namespace fda {

const Nccl& nccl() {
  static Nccl t;
  static std::once_flag once;
  std::call_once(once, [] {
    void* h = dlopen("libnccl.so.2", RTLD_NOW | RTLD_GLOBAL);
    if (!h) h = dlopen("libnccl.so", RTLD_NOW | RTLD_GLOBAL);
    if (!h) return;
    auto sym = [&](auto& f, const char* name) {
      f = reinterpret_cast<std::remove_reference_t<decltype(f)>>(dlsym(h, name));
      return f != nullptr;
    };
    t.ok = sym(t.GetUniqueId, "ncclGetUniqueId") && sym(t.CommInitRank, "ncclCommInitRank") &&
           sym(t.CommDestroy, "ncclCommDestroy") && sym(t.GroupStart, "ncclGroupStart") &&
           sym(t.GroupEnd, "ncclGroupEnd") && sym(t.Send, "ncclSend") && sym(t.Recv, "ncclRecv") &&
           sym(t.Broadcast, "ncclBroadcast");
  });
  return t;
}

}  // namespace fda
