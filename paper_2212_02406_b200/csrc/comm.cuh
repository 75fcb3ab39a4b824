// The NCCL communicator behind nnb_comm_t and the thin wrappers the sharded
// drivers use (NCCL is dlopen'ed by sharded.cu so single-GPU users need no
// libnccl; an already-loaded copy, e.g. torch's, is reused).
#pragma once

#include <nccl.h>

#include <cuda_runtime.h>

struct nnb_comm {
  ncclComm_t comm = nullptr;
  int world = 1, rank = 0, device = 0;
  cudaStream_t cs = nullptr;  // communication stream
};

namespace nnb {
ncclResult_t nccl_send(const void* buf, size_t count_doubles, int peer, nnb_comm* c, cudaStream_t s);
ncclResult_t nccl_recv(void* buf, size_t count_doubles, int peer, nnb_comm* c, cudaStream_t s);
ncclResult_t nccl_group(bool start);
ncclResult_t nccl_allgather(const void* send, void* recv, size_t count_doubles, nnb_comm* c, cudaStream_t s);
const char* nccl_error(ncclResult_t r);
}  // namespace nnb
