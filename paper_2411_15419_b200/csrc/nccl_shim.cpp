#include "nccl_shim.h"

#include <dlfcn.h>

#include <mutex>

namespace luffy {
namespace nccl {

const Api* api() {
  static Api a;
  static bool ok = false;
  static std::once_flag once;
  std::call_once(once, [] {
    void* h = dlopen("libnccl.so.2", RTLD_NOW | RTLD_NOLOAD | RTLD_GLOBAL);
    if (!h) h = dlopen("libnccl.so.2", RTLD_NOW | RTLD_GLOBAL);
    if (!h) h = dlopen("libnccl.so", RTLD_NOW | RTLD_GLOBAL);
    if (!h) return;
#define LUFFY_SYM(field, name)                                          \
  a.field = reinterpret_cast<decltype(a.field)>(dlsym(h, name));        \
  if (!a.field) return;
    LUFFY_SYM(GetUniqueId, "ncclGetUniqueId");
    LUFFY_SYM(CommInitRank, "ncclCommInitRank");
    LUFFY_SYM(CommDestroy, "ncclCommDestroy");
    LUFFY_SYM(AllGather, "ncclAllGather");
    LUFFY_SYM(Send, "ncclSend");
    LUFFY_SYM(Recv, "ncclRecv");
    LUFFY_SYM(GroupStart, "ncclGroupStart");
    LUFFY_SYM(GroupEnd, "ncclGroupEnd");
    LUFFY_SYM(GetErrorString, "ncclGetErrorString");
#undef LUFFY_SYM
    ok = true;
  });
  return ok ? &a : nullptr;
}

}  // namespace nccl
}  // namespace luffy
