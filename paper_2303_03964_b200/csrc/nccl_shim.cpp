#include "nccl_shim.h"

#include <dlfcn.h>

#include <cstdlib>

#include <mutex>

namespace tfdp {

const NcclApi* nccl_api(const char** err) {
  static NcclApi api;
  static std::once_flag once;
  static const char* load_err = nullptr;
  std::call_once(once, [] {
    // TFDP_NCCL_LIB: another implementation of the NCCL API (the tests' in-process loopback
    // stand-in, tests/nccl_loopback), loaded privately so it cannot shadow torch's NCCL
    const char* alt = getenv("TFDP_NCCL_LIB");
    void* h = nullptr;
    if (alt && alt[0]) {
      h = dlopen(alt, RTLD_NOW | RTLD_LOCAL);
      if (!h) {
        load_err = "TFDP_NCCL_LIB could not be loaded";
        return;
      }
    } else {
      h = dlopen("libnccl.so.2", RTLD_NOW | RTLD_GLOBAL | RTLD_NOLOAD);
      if (!h) h = dlopen("libnccl.so.2", RTLD_NOW | RTLD_GLOBAL);
    }
    if (!h) {
      load_err = "libnccl.so.2 not found (import torch first, or set LD_LIBRARY_PATH)";
      return;
    }
#define TFDP_SYM(field, name)                                          \
  api.field = reinterpret_cast<decltype(api.field)>(dlsym(h, name));   \
  if (!api.field) {                                                    \
    load_err = "libnccl.so.2 lacks symbol " name;                      \
    return;                                                            \
  }
    TFDP_SYM(GetUniqueId, "ncclGetUniqueId");
    TFDP_SYM(CommInitRank, "ncclCommInitRank");
    TFDP_SYM(CommDestroy, "ncclCommDestroy");
    TFDP_SYM(GroupStart, "ncclGroupStart");
    TFDP_SYM(GroupEnd, "ncclGroupEnd");
    TFDP_SYM(Broadcast, "ncclBroadcast");
    TFDP_SYM(AllReduce, "ncclAllReduce");
    TFDP_SYM(Send, "ncclSend");
    TFDP_SYM(Recv, "ncclRecv");
    TFDP_SYM(GetErrorString, "ncclGetErrorString");
#undef TFDP_SYM
    api.loaded = true;
  });
  if (!api.loaded) {
    if (err) *err = load_err;
    return nullptr;
  }
  return &api;
}

}  // namespace tfdp
