// NCCL is resolved at run time (dlopen) only when a context has world > 1.
// Linking libnccl.so.2 at load time would bind the system NCCL (2.27) into
// the process before torch's bundled one and break `import torch`.
#pragma once

#include <nccl.h>

namespace dgs_b200 {

struct NcclApi {
    ncclResult_t (*GetUniqueId)(ncclUniqueId*);
    ncclResult_t (*CommInitRank)(ncclComm_t*, int, ncclUniqueId, int);
    ncclResult_t (*CommDestroy)(ncclComm_t);
    const char* (*GetErrorString)(ncclResult_t);
    ncclResult_t (*GroupStart)();
    ncclResult_t (*GroupEnd)();
    ncclResult_t (*Send)(const void*, size_t, ncclDataType_t, int, ncclComm_t, cudaStream_t);
    ncclResult_t (*Recv)(void*, size_t, ncclDataType_t, int, ncclComm_t, cudaStream_t);
    ncclResult_t (*AllReduce)(const void*, void*, size_t, ncclDataType_t, ncclRedOp_t, ncclComm_t, cudaStream_t);
};

/// Loads libnccl.so.2 on first use (throws NcclError if unavailable).
const NcclApi& nccl();

}  // namespace dgs_b200
