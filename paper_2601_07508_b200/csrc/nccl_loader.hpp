// nccl_loader.hpp -- NCCL resolved at run time (dlopen), not at link time.
//
// libfpmm_b200.so must coexist with whichever libnccl.so.2 the host process
// already uses (torch bundles a newer one than the system's).  Linking it
// would pin the soname to the first library found and break the other user,
// so the partitioner binds the handful of NCCL entry points it needs on
// first use, preferring an already-loaded libnccl.so.2 (RTLD_NOLOAD).
#pragma once

#include <nccl.h>

namespace fpmm_b200 {

struct NcclApi {
  ncclResult_t (*GetUniqueId)(ncclUniqueId*);
  ncclResult_t (*CommInitRank)(ncclComm_t*, int, ncclUniqueId, int);
  ncclResult_t (*CommInitAll)(ncclComm_t*, int, const int*);
  ncclResult_t (*CommDestroy)(ncclComm_t);
  ncclResult_t (*Broadcast)(const void*, void*, size_t, ncclDataType_t, int, ncclComm_t, cudaStream_t);
  ncclResult_t (*AllReduce)(const void*, void*, size_t, ncclDataType_t, ncclRedOp_t, ncclComm_t, cudaStream_t);
  ncclResult_t (*Send)(const void*, size_t, ncclDataType_t, int, ncclComm_t, cudaStream_t);
  ncclResult_t (*Recv)(void*, size_t, ncclDataType_t, int, ncclComm_t, cudaStream_t);
  ncclResult_t (*GroupStart)();
  ncclResult_t (*GroupEnd)();
  const char* (*GetErrorString)(ncclResult_t);
};

// throws Failure(FPMM_B200_ENCCL) if no libnccl.so.2 can be loaded
const NcclApi& nccl();

}  // namespace fpmm_b200
