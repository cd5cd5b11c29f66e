// Host runtime of libttncbc: context (device, stream, staging, arenas), TTN handles,
// and the status plumbing behind the C ABI (include/ttn_cbc.h).
#pragma once
#include "../../include/ttn_cbc.h"
#include "comm.h"
#include "kernels.h"

#include <cuda_runtime.h>
#include <cstdint>
#include <cstdlib>
#include <functional>
#include <stdexcept>
#include <string>
#include <vector>

namespace tcbc {

// Error carried to the ABI boundary (converted to a ttn_status there).
struct Error : std::runtime_error {
  ttn_status status;
  Error(ttn_status s, const std::string& m) : std::runtime_error(m), status(s) {}
};

#define TTN_CUDA(x)                                                                          \
  do {                                                                                       \
    cudaError_t e__ = (x);                                                                   \
    if (e__ != cudaSuccess)                                                                  \
      throw ::tcbc::Error(e__ == cudaErrorMemoryAllocation ? TTN_ERR_OOM : TTN_ERR_CUDA,      \
                         std::string(#x) + ": " + cudaGetErrorString(e__));                  \
  } while (0)

// Device memory source of a context: the caller's ttn_allocator, else a stream-ordered pool
// owned by the context (cudaMallocFromPoolAsync on the ctx stream).
struct MemSource {
  virtual void* get(size_t bytes) = 0;
  virtual void put(void* p) = 0;   // stream-ordered free (after the work enqueued so far)
  virtual ~MemSource() {}
};

// Bump allocator over device chunks.  reset() recycles the memory for later work on the
// SAME stream (stream order makes the reuse safe without a host sync).
class Arena {
 public:
  explicit Arena(size_t chunk = 256ull << 20) : chunk_(chunk) {}
  ~Arena();
  void set_source(MemSource* src) { src_ = src; }
  bool frozen = false;   // set during a graph capture: a new chunk would escape the graph
  void* alloc(size_t bytes);
  void reset();
  void release();
  size_t high_water() const { return high_; }

 private:
  struct Chunk { char* p; size_t size; size_t used; };
  std::vector<Chunk> chunks_;
  size_t cur_ = 0, chunk_, high_ = 0, live_ = 0;
  MemSource* src_ = nullptr;
};

// Pinned host ring mirrored in device memory; put() enqueues one H2D copy.
class RingStager : public Stager {
 public:
  RingStager(cudaStream_t s, size_t bytes = 64ull << 20);
  ~RingStager();
  void* put(const void* host, size_t bytes) override;
  void* reserve(size_t bytes) override;
  void* commit(void* host, size_t bytes) override;
  void epoch() override;   // call after a stream synchronisation: the whole ring is free again
  size_t staged = 0;       // bytes staged since the last reset (the size a capture needs)
 private:
  cudaStream_t s_;
  char* h_ = nullptr;
  char* d_ = nullptr;
  size_t size_, off_ = 0;
};

// Stager of a CUDA-graph capture: descriptors are written to a host shadow at the offsets
// they will have in a device buffer owned by the graph (addresses known while capturing);
// the shadow is uploaded once after the capture ends.  Never copies or synchronises.
class CaptureStager : public Stager {
 public:
  CaptureStager(char* dev, size_t cap) : d_(dev), cap_(cap) {}
  void* put(const void* host, size_t bytes) override;
  void* reserve(size_t bytes) override;
  void* commit(void* host, size_t bytes) override;
  std::vector<char> shadow;
 private:
  char* d_;
  size_t cap_;
  std::vector<char> tmp_;
};

}  // namespace tcbc

namespace tcbc { struct GraphCache; }

struct ttn_ctx_s : tcbc::MemSource {
  int device = 0;
  cudaStream_t stream = nullptr;
  std::string last_error;
  // level-synchronous schedule options (ttn_ctx_set_schedule): speculative ranks (no host
  // synchronisation inside an apply) and CUDA-graph replay of speculative applies
  bool speculate = getenv("TTN_NO_SPECULATE") == nullptr;   // (A/B knob; ttn_ctx_set_schedule)
  bool graphs = true;
  bool capturing = false;        // a graph capture is in progress on this ctx (no arena growth)
  tcbc::GraphCache* gr = nullptr;          // graph cache and the shapes whose speculation failed
  char* spec_host = nullptr;     // pinned result block of a speculative apply
  size_t spec_host_size = 0;
  // device memory: the caller's allocator (ttn_ctx_create), else `pool` (owned by the root
  // context; worker contexts share it).  Frees through a caller's allocator are deferred until
  // the ctx stream has passed an event recorded at the free, so the allocator may hand the
  // block to any stream at once.
  ttn_allocator user_alloc{};
  bool has_user_alloc = false;
  cudaMemPool_t pool = nullptr;
  bool owns_pool = false;
  std::vector<std::pair<cudaEvent_t, void*>> pending_free;
  void* get(size_t bytes) override;
  void put(void* p) override;
  void reap(bool all);   // hand completed deferred frees to the caller's allocator
  tcbc::RingStager* ring = nullptr;   // the descriptor ring (owned)
  tcbc::Stager* stager = nullptr;     // current stager: the ring, or a capture's
  tcbc::Arena scratch;      // per-stage temporaries (reset between stages)
  tcbc::Arena env;          // per-apply environment factors (reset per apply)
  // pinned host buffer for small D2H reads (ranks, weights, norms)
  char* hbuf = nullptr;
  size_t hbuf_size = 0;
  char* dbuf = nullptr;    // device mirror of small results
  size_t dbuf_size = 0;
  int host_syncs = 0;
  double sync_wait_s = 0.0;     // host time blocked in sync() (TTN_HOST_PROF diagnostics)
  tcbc::Comm* comm = nullptr;   // multi-GPU apply (ttn_ctx_set_comm)
  std::vector<ttn_ctx_s*> workers;   // concurrent sub-batches (ttn_ctx_set_workers); own streams
  bool owns_stream = false;
  int parts = 1;                // subtree groups of a partitioned apply
  void sync();             // cudaStreamSynchronize + stager epoch
  // partial synchronisation: mark a point in the stream, then wait for it only (the work
  // enqueued after the mark keeps running; the staging ring is not recycled)
  cudaEvent_t rank_ev = nullptr;
  void mark_ranks();
  void wait_ranks();
  void ensure_small(size_t bytes);
};

struct ttn_s {
  ttn_ctx_s* ctx = nullptr;
  int kind = TTN_STATE;
  int n = 0;
  int root = -1;
  std::vector<int> parent, phys;
  std::vector<int64_t> bond;
  std::vector<std::vector<int>> children;
  std::vector<int> depth;
  std::vector<std::vector<int64_t>> shape;
  std::vector<int64_t> offset;   // element offset of node i in data
  int64_t total = 0;
  tcbc::cplx* data = nullptr;     // one device allocation (cudaMallocAsync)
  tcbc::cplx* node(int i) const { return data + offset[i]; }
};

namespace tcbc {

// Topology helpers shared by create / apply / overlap.
void build_topology(ttn_s* t, const int32_t* parent, int n);
void finalize_shapes(ttn_s* t);   // shapes / offsets / total from kind, phys, bond
// data from `alloc` when given (a graph capture's output buffer), else from the ctx
ttn_s* new_ttn_like(ttn_ctx_s* ctx, const ttn_s* tmpl, int kind, const std::vector<int64_t>& bond,
                    const std::function<cplx*(int64_t)>& alloc = std::function<cplx*(int64_t)>());
void free_ttn(ttn_s* t);

// Batched drivers (cbc.cpp)
void cbc_apply_impl(ttn_ctx_s* ctx, int nb, const ttn_s* const* ops, const ttn_s* const* sts,
                    int64_t max_bond, double tol, ttn_s** outs, ttn_cbc_report* reps);
void graphs_release(ttn_ctx_s* ctx);   // before the ctx's arenas / pool go
void overlap_impl(ttn_ctx_s* ctx, int nb, const ttn_s* const* a, const ttn_s* const* b, cplx* out);
// One layer of a <bra| O_1 ... O_m |ket> sweep (per-instance handles).
struct SweepLayer {
  const ttn_s* const* h;
  bool op = false, conj = false, dagger = false;
};
void sweep_impl(ttn_ctx_s* ctx, int nb, const std::vector<SweepLayer>& layers, cplx* out);
// Subtree groups of a parts-way partitioned apply (group -1: replicated top); cuts_out gets
// the subtree roots.  Host-only.
std::vector<int> partition_groups(const ttn_s* ref, int parts, std::vector<int>* cuts_out);

}  // namespace tcbc
