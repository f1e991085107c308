// tt_nccl.h -- NCCL entry points resolved at run time (dlopen of the libnccl.so.2 that torch
// already loaded, so one NCCL instance serves torch.distributed and libtt).
#pragma once

#include <cstddef>
#include <cuda_runtime.h>

namespace tt {

typedef void* ncclComm_t_;
struct NcclApi {
  int (*GetUniqueId)(void* id) = nullptr;
  int (*CommDestroy)(ncclComm_t_ comm) = nullptr;
  int (*GroupStart)() = nullptr;
  int (*GroupEnd)() = nullptr;
  int (*Send)(const void* buf, size_t count, int dtype, int peer, ncclComm_t_ comm, cudaStream_t s) = nullptr;
  int (*Recv)(void* buf, size_t count, int dtype, int peer, ncclComm_t_ comm, cudaStream_t s) = nullptr;
  int (*AllReduce)(const void* sb, void* rb, size_t count, int dtype, int op, ncclComm_t_ comm, cudaStream_t s) = nullptr;
  const char* (*GetErrorString)(int res) = nullptr;
  void* handle = nullptr;
};

// Loads NCCL once; returns nullptr and sets *err on failure.
const NcclApi* nccl_api(const char** err);
// ncclCommInitRank takes ncclUniqueId BY VALUE (128 bytes); wrapped here.
int nccl_comm_init(const NcclApi* api, void** comm, int nranks, const void* id128, int rank);

constexpr int kNcclFloat64 = 8;   // ncclDouble
constexpr int kNcclInt8 = 0;      // ncclInt8
constexpr int kNcclSum = 0;       // ncclSum

}  // namespace tt
