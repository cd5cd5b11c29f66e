// Multi-GPU communicator of a ttn_ctx: NCCL, loaded at run time (dlopen of libnccl.so.2 --
// the copy torch already loaded when present), so the library has no link-time NCCL
// dependency and a process that never calls ttn_ctx_set_comm never touches NCCL.
// All collectives are enqueued on the ctx stream.
#pragma once
#include <cuda_runtime.h>
#include <cstddef>

namespace tcbc {

// The collectives of a partitioned apply, enqueued on the caller's stream.  Every rank issues
// the same sequence (it depends only on the tree).
struct Comm {
  int rank = 0, world = 1;
  // in-place broadcast of `bytes` from `root`
  virtual void bcast(void* buf, size_t bytes, int root, cudaStream_t s) = 0;
  // in-place sum of `n` doubles / int32s, max of int32s
  virtual void allreduce_sum(double* buf, size_t n, cudaStream_t s) = 0;
  virtual void allreduce_sum(int* buf, size_t n, cudaStream_t s) = 0;
  virtual void allreduce_max(int* buf, size_t n, cudaStream_t s) = 0;
  virtual void group_start() {}
  virtual void group_end() {}
  virtual ~Comm() {}
};

// NCCL (one process per GPU): 128-byte unique id (ncclGetUniqueId); throws
// Error(TTN_ERR_NCCL) when NCCL is unavailable.
void comm_unique_id(void* out128);
Comm* comm_create(const void* id128, int rank, int world, int device);

// In-process loopback communicator: `world` ranks = contexts on the SAME device, each driven
// by its own host thread.  A collective is two host barriers between the rank threads plus
// stream-event dependencies (cudaStreamWaitEvent) and device copies / reduction kernels: no
// kernel ever waits on another rank, so the ranks' streams need not run concurrently.  It runs
// the multi-rank schedule (rank-asymmetric broadcasts, split-row all-reduces) on one GPU.
struct LoopGroup;
LoopGroup* loop_group_create(int world);
void loop_group_release(LoopGroup* g);   // reference counted (creator + one per rank)
Comm* loop_comm_create(LoopGroup* g, int rank, int device);

}  // namespace tcbc
