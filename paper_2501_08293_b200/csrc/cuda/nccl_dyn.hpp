// NCCL, bound at run time (dlopen) for the partitioned multi-GPU solve.
//
// libdopf_cuda.so does not link NCCL: a process that already holds an NCCL
// (PyTorch loads its own libnccl.so.2) shares that copy, and a process
// without one loads libnccl.so.2 from the library path (or DOPF_NCCL_SO)
// only when a communicator is created. Single-GPU solves never touch it, and
// a missing NCCL surfaces as DOPF_ERR_NCCL with a message, not a load error.
#pragma once

#include <cuda_runtime.h>
#include <nccl.h>

#include <string>

namespace dopf::cuda::nccl {

struct Api {
  ncclResult_t (*GetVersion)(int*);
  ncclResult_t (*GetUniqueId)(ncclUniqueId*);
  ncclResult_t (*CommInitRank)(ncclComm_t*, int, ncclUniqueId, int);
  ncclResult_t (*CommInitAll)(ncclComm_t*, int, const int*);
  ncclResult_t (*CommDestroy)(ncclComm_t);
  ncclResult_t (*CommAbort)(ncclComm_t);
  ncclResult_t (*CommGetAsyncError)(ncclComm_t, ncclResult_t*);
  ncclResult_t (*AllGather)(const void*, void*, size_t, ncclDataType_t, ncclComm_t, cudaStream_t);
  ncclResult_t (*AllReduce)(const void*, void*, size_t, ncclDataType_t, ncclRedOp_t, ncclComm_t, cudaStream_t);
  const char* (*GetErrorString)(ncclResult_t);
};

/// The bound API, loading NCCL on first use. Throws NcclFailure when no
/// usable libnccl.so.2 is found.
const Api& api();

/// Path (or "already loaded") of the NCCL in use, and its version code.
std::string describe();

struct NcclFailure : std::exception {
  std::string msg;
  explicit NcclFailure(std::string m) : msg(std::move(m)) {}
  const char* what() const noexcept override { return msg.c_str(); }
};

/// Throws NcclFailure naming `what` unless r == ncclSuccess.
void check(ncclResult_t r, const char* what);

}  // namespace dopf::cuda::nccl
