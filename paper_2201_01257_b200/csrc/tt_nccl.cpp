// tt_nccl.cpp -- run-time binding of NCCL (see tt_nccl.h).
#include "tt_nccl.h"

#include <dlfcn.h>

#include <cstring>
#include <mutex>
#include <string>

namespace tt {

namespace {
NcclApi g_api;
bool g_tried = false;
std::string g_err;
std::mutex g_mu;

struct UniqueId { char b[128]; };
typedef int (*InitRankFn)(void** comm, int nranks, UniqueId id, int rank);
InitRankFn g_init = nullptr;

void* open_nccl() {
  // Prefer the instance already mapped into the process (torch's), then the torch wheel, then system.
  const char* names[] = {"libnccl.so.2", "libnccl.so"};
  for (const char* n : names) {
    void* h = dlopen(n, RTLD_NOW | RTLD_NOLOAD | RTLD_GLOBAL);
    if (h) return h;
  }
  const char* env = getenv("TT_NCCL_LIB");
  if (env) {
    void* h = dlopen(env, RTLD_NOW | RTLD_GLOBAL);
    if (h) return h;
  }
  for (const char* n : names) {
    void* h = dlopen(n, RTLD_NOW | RTLD_GLOBAL);
    if (h) return h;
  }
  return nullptr;
}
}  // namespace

const NcclApi* nccl_api(const char** err) {
  std::lock_guard<std::mutex> lk(g_mu);
  if (!g_tried) {
    g_tried = true;
    void* h = open_nccl();
    if (!h) {
      g_err = std::string("cannot load libnccl.so.2: ") + (dlerror() ? dlerror() : "not found");
    } else {
      g_api.handle = h;
      bool ok = true;
      auto sym = [&](const char* n) {
        void* p = dlsym(h, n);
        if (!p) { ok = false; g_err = std::string("NCCL symbol missing: ") + n; }
        return p;
      };
      g_api.GetUniqueId = (int (*)(void*))sym("ncclGetUniqueId");
      g_init = (InitRankFn)sym("ncclCommInitRank");
      g_api.CommDestroy = (int (*)(void*))sym("ncclCommDestroy");
      g_api.GroupStart = (int (*)())sym("ncclGroupStart");
      g_api.GroupEnd = (int (*)())sym("ncclGroupEnd");
      g_api.Send = (int (*)(const void*, size_t, int, int, void*, cudaStream_t))sym("ncclSend");
      g_api.Recv = (int (*)(void*, size_t, int, int, void*, cudaStream_t))sym("ncclRecv");
      g_api.AllReduce = (int (*)(const void*, void*, size_t, int, int, void*, cudaStream_t))sym("ncclAllReduce");
      g_api.GetErrorString = (const char* (*)(int))sym("ncclGetErrorString");
      if (!ok) g_api.handle = nullptr;
    }
  }
  if (!g_api.handle) {
    if (err) *err = g_err.c_str();
    return nullptr;
  }
  return &g_api;
}

int nccl_comm_init(const NcclApi* api, void** comm, int nranks, const void* id128, int rank) {
  (void)api;
  UniqueId id;
  std::memcpy(id.b, id128, 128);
  return g_init(comm, nranks, id, rank);
}

}  // namespace tt
