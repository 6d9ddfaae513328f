// nccl_dl.cpp -- see nccl_dl.h.
#include "nccl_dl.h"

#include <dlfcn.h>

#include <cstdio>
#include <cstdlib>
#include <mutex>

namespace evox {

namespace {
NcclApi g_api;
std::once_flag g_once;

template <class F>
bool sym(void* h, const char* name, F& out) {
    out = reinterpret_cast<F>(dlsym(h, name));
    return out != nullptr;
}

void load() {
    void* h = nullptr;
    // 1) the copy already in the process (torch links libnccl.so.2)
    h = dlopen("libnccl.so.2", RTLD_NOW | RTLD_NOLOAD);
    // 2) an explicit override
    if (!h) {
        const char* p = std::getenv("EVOX_NCCL_LIB");
        if (p && *p) h = dlopen(p, RTLD_NOW | RTLD_LOCAL);
    }
    // 3) the default search path
    if (!h) h = dlopen("libnccl.so.2", RTLD_NOW | RTLD_LOCAL);
    if (!h) {
        std::snprintf(g_api.error, sizeof g_api.error, "dlopen(libnccl.so.2) failed: %s",
                      dlerror());
        return;
    }
    bool ok = sym(h, "ncclGetUniqueId", g_api.GetUniqueId) &&
              sym(h, "ncclCommInitRank", g_api.CommInitRank) &&
              sym(h, "ncclCommDestroy", g_api.CommDestroy) &&
              sym(h, "ncclCommAbort", g_api.CommAbort) &&
              sym(h, "ncclCommGetAsyncError", g_api.CommGetAsyncError) &&
              sym(h, "ncclAllGather", g_api.AllGather) &&
              sym(h, "ncclAllReduce", g_api.AllReduce) &&
              sym(h, "ncclGetErrorString", g_api.GetErrorString);
    if (!ok) {
        std::snprintf(g_api.error, sizeof g_api.error, "libnccl.so.2 lacks a required symbol");
        return;
    }
    g_api.ok = true;
}
}  // namespace

const NcclApi* nccl_api(const char** why) {
    std::call_once(g_once, load);
    if (!g_api.ok) {
        if (why) *why = g_api.error;
        return nullptr;
    }
    return &g_api;
}

}  // namespace evox
