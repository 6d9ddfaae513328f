// nccl_dl.h -- NCCL loaded at run time (dlopen), so the library has no link-time
// NCCL dependency and reuses the libnccl.so.2 torch has already loaded.
#pragma once

#include <nccl.h>

namespace evox {

struct NcclApi {
    bool ok = false;
    ncclResult_t (*GetUniqueId)(ncclUniqueId*) = nullptr;
    ncclResult_t (*CommInitRank)(ncclComm_t*, int, ncclUniqueId, int) = nullptr;
    ncclResult_t (*CommDestroy)(ncclComm_t) = nullptr;
    ncclResult_t (*CommAbort)(ncclComm_t) = nullptr;
    ncclResult_t (*CommGetAsyncError)(ncclComm_t, ncclResult_t*) = nullptr;
    ncclResult_t (*AllGather)(const void*, void*, size_t, ncclDataType_t, ncclComm_t,
                              cudaStream_t) = nullptr;
    ncclResult_t (*AllReduce)(const void*, void*, size_t, ncclDataType_t, ncclRedOp_t, ncclComm_t,
                              cudaStream_t) = nullptr;
    const char* (*GetErrorString)(ncclResult_t) = nullptr;
    char error[256] = {0};
};

// Loads once (thread-safe).  Returns nullptr (with a reason in *why) if NCCL
// cannot be loaded.
const NcclApi* nccl_api(const char** why);

}  // namespace evox
