// Multi-GPU communicator of a ttn_ctx: NCCL, loaded at run time (dlopen of libnccl.so.2 --
// the copy torch already loaded when present), so the library has no link-time NCCL
// dependency and a process that never calls ttn_ctx_set_comm never touches NCCL.
// All collectives are enqueued on the ctx stream.
#pragma once
#include <cuda_runtime.h>
#include <cstddef>

namespace tcbc {

struct Comm {
  void* comm = nullptr;   // ncclComm_t
  int rank = 0, world = 1;
  // in-place broadcast of `bytes` from `root`
  void bcast(void* buf, size_t bytes, int root, cudaStream_t s);
  // in-place sum of `n` doubles / int32s
  void allreduce_sum(double* buf, size_t n, cudaStream_t s);
  void allreduce_sum(int* buf, size_t n, cudaStream_t s);
  void allreduce_max(int* buf, size_t n, cudaStream_t s);
  void group_start();
  void group_end();
  ~Comm();
};

// 128-byte unique id (ncclGetUniqueId); throws Error(TTN_ERR_NCCL) when NCCL is unavailable.
void comm_unique_id(void* out128);
Comm* comm_create(const void* id128, int rank, int world, int device);

}  // namespace tcbc
