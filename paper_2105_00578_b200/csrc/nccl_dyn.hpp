// nccl_dyn.hpp — NCCL resolved at runtime (dlopen) instead of at link time.
//
// Single-GPU use never loads NCCL, and a multi-GPU process shares whatever
// libnccl.so.2 is already loaded (e.g. the one torch.distributed brought in),
// so the library can be loaded before or after torch without two NCCL builds
// fighting over the same soname.
#pragma once

#include <nccl.h>

namespace spb {

struct NcclApi {
    ncclResult_t (*GetUniqueId)(ncclUniqueId*) = nullptr;
    ncclResult_t (*CommInitRank)(ncclComm_t*, int, ncclUniqueId, int) = nullptr;
    ncclResult_t (*CommDestroy)(ncclComm_t) = nullptr;
    ncclResult_t (*AllGather)(const void*, void*, size_t, ncclDataType_t, ncclComm_t, cudaStream_t) = nullptr;
    ncclResult_t (*Send)(const void*, size_t, ncclDataType_t, int, ncclComm_t, cudaStream_t) = nullptr;
    ncclResult_t (*Recv)(void*, size_t, ncclDataType_t, int, ncclComm_t, cudaStream_t) = nullptr;
    ncclResult_t (*GroupStart)() = nullptr;
    ncclResult_t (*GroupEnd)() = nullptr;
    const char* (*GetErrorString)(ncclResult_t) = nullptr;
};

// Throws SpError(SP_NCCL) if libnccl.so.2 cannot be loaded.
const NcclApi& nccl();

} // namespace spb
