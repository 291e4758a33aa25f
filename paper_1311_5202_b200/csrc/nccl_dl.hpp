// nccl_dl.hpp -- NCCL entry points resolved at run time (dlopen "libnccl.so.2").
//
// libfda does not link NCCL: a single-GPU plan never touches it, and in a process that already
// loaded NCCL (torch) dlopen returns that same library (same soname), so the library and the
// caller's process group share one NCCL.  Only the handful of calls of the multi-GPU data plane
// are resolved.
#pragma once
#include <cuda_runtime.h>
#include <nccl.h>

namespace fda {

struct Nccl {
  bool ok = false;
  ncclResult_t (*GetUniqueId)(ncclUniqueId*) = nullptr;
  ncclResult_t (*CommInitRank)(ncclComm_t*, int, ncclUniqueId, int) = nullptr;
  ncclResult_t (*CommDestroy)(ncclComm_t) = nullptr;
  ncclResult_t (*GroupStart)() = nullptr;
  ncclResult_t (*GroupEnd)() = nullptr;
  ncclResult_t (*Send)(const void*, size_t, ncclDataType_t, int, ncclComm_t, cudaStream_t) = nullptr;
  ncclResult_t (*Recv)(void*, size_t, ncclDataType_t, int, ncclComm_t, cudaStream_t) = nullptr;
  ncclResult_t (*Broadcast)(const void*, void*, size_t, ncclDataType_t, int, ncclComm_t, cudaStream_t) = nullptr;
};

// the resolved table (ok == false when libnccl.so.2 or a symbol is missing)
const Nccl& nccl();

}  // namespace fda
