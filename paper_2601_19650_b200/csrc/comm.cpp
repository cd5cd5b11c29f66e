// NCCL binding of the ctx communicator (see comm.h).
#include "comm.h"
#include "runtime.h"

#include <dlfcn.h>
#include <cstring>
#include <algorithm>
#include <atomic>
#include <condition_variable>
#include <mutex>
#include <vector>
#include <string>

namespace tcbc {

namespace {

typedef int nres_t;   // ncclResult_t
typedef void* ncomm_t;
struct NcclId { char internal[128]; };
enum { nccl_int32 = 2, nccl_float64 = 8 };   // ncclDataType_t
enum { nccl_sum = 0, nccl_max = 2 };           // ncclRedOp_t

struct Nccl {
  void* h = nullptr;
  nres_t (*GetUniqueId)(NcclId*) = nullptr;
  nres_t (*CommInitRank)(ncomm_t*, int, NcclId, int) = nullptr;
  nres_t (*CommDestroy)(ncomm_t) = nullptr;
  nres_t (*Broadcast)(const void*, void*, size_t, int, int, ncomm_t, cudaStream_t) = nullptr;
  nres_t (*AllReduce)(const void*, void*, size_t, int, int, ncomm_t, cudaStream_t) = nullptr;
  nres_t (*GroupStart)() = nullptr;
  nres_t (*GroupEnd)() = nullptr;
  const char* (*GetErrorString)(nres_t) = nullptr;
};

Nccl& nccl() {
  static Nccl n;
  static std::once_flag once;
  std::call_once(once, [] {
    const char* names[] = {"libnccl.so.2", "libnccl.so"};
    for (const char* nm : names) {
      n.h = dlopen(nm, RTLD_NOW | RTLD_GLOBAL);
      if (n.h) break;
    }
    if (!n.h) return;
    n.GetUniqueId = reinterpret_cast<decltype(n.GetUniqueId)>(dlsym(n.h, "ncclGetUniqueId"));
    n.CommInitRank = reinterpret_cast<decltype(n.CommInitRank)>(dlsym(n.h, "ncclCommInitRank"));
    n.CommDestroy = reinterpret_cast<decltype(n.CommDestroy)>(dlsym(n.h, "ncclCommDestroy"));
    n.Broadcast = reinterpret_cast<decltype(n.Broadcast)>(dlsym(n.h, "ncclBroadcast"));
    n.AllReduce = reinterpret_cast<decltype(n.AllReduce)>(dlsym(n.h, "ncclAllReduce"));
    n.GroupStart = reinterpret_cast<decltype(n.GroupStart)>(dlsym(n.h, "ncclGroupStart"));
    n.GroupEnd = reinterpret_cast<decltype(n.GroupEnd)>(dlsym(n.h, "ncclGroupEnd"));
    n.GetErrorString = reinterpret_cast<decltype(n.GetErrorString)>(dlsym(n.h, "ncclGetErrorString"));
  });
  if (!n.h || !n.GetUniqueId || !n.CommInitRank || !n.Broadcast || !n.AllReduce || !n.GroupStart || !n.GroupEnd)
    throw Error(TTN_ERR_NCCL, "NCCL (libnccl.so.2) not available");
  return n;
}

void check(nres_t r, const char* what) {
  if (r != 0) {
    const char* m = nccl().GetErrorString ? nccl().GetErrorString(r) : "?";
    throw Error(TTN_ERR_NCCL, std::string(what) + ": " + m);
  }
}

}  // namespace

void comm_unique_id(void* out128) {
  NcclId id;
  check(nccl().GetUniqueId(&id), "ncclGetUniqueId");
  std::memcpy(out128, &id, sizeof(id));
}

namespace {
struct NcclComm : Comm {
  void* comm = nullptr;   // ncclComm_t
  ~NcclComm() override {
    if (comm && nccl().CommDestroy) nccl().CommDestroy(comm);
  }
  void bcast(void* buf, size_t bytes, int root, cudaStream_t s) override {
    if (!comm || bytes == 0) return;
    check(nccl().Broadcast(buf, buf, bytes, /*ncclInt8*/ 0, root, comm, s), "ncclBroadcast");
  }
  void allreduce_sum(double* buf, size_t n, cudaStream_t s) override {
    if (!comm || n == 0) return;
    check(nccl().AllReduce(buf, buf, n, nccl_float64, nccl_sum, comm, s), "ncclAllReduce");
  }
  void allreduce_sum(int* buf, size_t n, cudaStream_t s) override {
    if (!comm || n == 0) return;
    check(nccl().AllReduce(buf, buf, n, nccl_int32, nccl_sum, comm, s), "ncclAllReduce");
  }
  void allreduce_max(int* buf, size_t n, cudaStream_t s) override {
    if (!comm || n == 0) return;
    check(nccl().AllReduce(buf, buf, n, nccl_int32, nccl_max, comm, s), "ncclAllReduce");
  }
  void group_start() override {
    if (comm) check(nccl().GroupStart(), "ncclGroupStart");
  }
  void group_end() override {
    if (comm) check(nccl().GroupEnd(), "ncclGroupEnd");
  }
};
}  // namespace

Comm* comm_create(const void* id128, int rank, int world, int device) {
  if (world < 1 || rank < 0 || rank >= world) throw Error(TTN_ERR_ARG, "bad rank / world");
  NcclId id;
  std::memcpy(&id, id128, sizeof(id));
  TTN_CUDA(cudaSetDevice(device));
  NcclComm* c = new NcclComm();
  c->rank = rank;
  c->world = world;
  check(nccl().CommInitRank(&c->comm, world, id, rank), "ncclCommInitRank");
  return c;
}

// ---------------------------------------------------------------- in-process loopback
struct LoopGroup {
  int world;
  std::mutex mu;
  std::condition_variable cv;
  int arrived = 0;
  long long gen = 0;
  std::vector<void*> ptr;
  std::vector<cudaEvent_t> ev1, ev2;
  std::atomic<int> refs{1};
  explicit LoopGroup(int w) : world(w), ptr(w, nullptr), ev1(w, nullptr), ev2(w, nullptr) {}
  void barrier() {
    std::unique_lock<std::mutex> lk(mu);
    const long long g = gen;
    if (++arrived == world) {
      arrived = 0;
      ++gen;
      cv.notify_all();
    } else {
      cv.wait(lk, [&] { return gen != g; });
    }
  }
};

LoopGroup* loop_group_create(int world) {
  if (world < 1) throw Error(TTN_ERR_ARG, "loopback world must be >= 1");
  return new LoopGroup(world);
}

void loop_group_release(LoopGroup* g) {
  if (g && g->refs.fetch_sub(1) == 1) delete g;
}

namespace {

template <typename T, int OP>   // OP 0: sum, 1: max
__global__ void loop_reduce(T* __restrict__ out, const T* const* __restrict__ in, int world, size_t n) {
  TCBC_PDL_WAIT();
  for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < n; i += (size_t)gridDim.x * blockDim.x) {
    T v = in[0][i];
    for (int r = 1; r < world; ++r) v = OP == 0 ? v + in[r][i] : (in[r][i] > v ? in[r][i] : v);
    out[i] = v;
  }
}

struct LoopComm : Comm {
  LoopGroup* g;
  cudaEvent_t e1 = nullptr, e2 = nullptr;
  void* tmp = nullptr;      // reduction result (device)
  size_t tmp_bytes = 0;
  void** dptrs = nullptr;   // device copy of the peers' buffer addresses
  LoopComm(LoopGroup* grp, int r) : g(grp) {
    rank = r;
    world = grp->world;
    g->refs.fetch_add(1);
    TTN_CUDA(cudaEventCreateWithFlags(&e1, cudaEventDisableTiming));
    TTN_CUDA(cudaEventCreateWithFlags(&e2, cudaEventDisableTiming));
    TTN_CUDA(cudaMalloc(&dptrs, sizeof(void*) * world));
  }
  ~LoopComm() override {
    if (tmp) cudaFree(tmp);
    if (dptrs) cudaFree(dptrs);
    cudaEventDestroy(e1);
    cudaEventDestroy(e2);
    loop_group_release(g);
  }
  // phase 1: publish (buffer, ready event); every rank sees every other's
  void publish(void* buf, cudaStream_t s) {
    TTN_CUDA(cudaEventRecord(e1, s));
    g->ptr[rank] = buf;
    g->ev1[rank] = e1;
    g->barrier();
  }
  // phase 2: after this rank's reads of the peers' buffers, publish "done reading"
  void done(cudaStream_t s) {
    TTN_CUDA(cudaEventRecord(e2, s));
    g->ev2[rank] = e2;
    g->barrier();
  }
  template <typename T, int OP>
  void allreduce(T* buf, size_t n, cudaStream_t s) {
    if (n == 0 || world == 1) return;
    publish(buf, s);
    for (int r = 0; r < world; ++r)
      if (r != rank) TTN_CUDA(cudaStreamWaitEvent(s, g->ev1[r], 0));
    if (tmp_bytes < n * sizeof(T)) {   // grow (synchronous; the stream is drained first)
      TTN_CUDA(cudaStreamSynchronize(s));
      if (tmp) cudaFree(tmp);
      tmp = nullptr;
      TTN_CUDA(cudaMalloc(&tmp, n * sizeof(T)));
      tmp_bytes = n * sizeof(T);
    }
    std::vector<void*> hp(g->ptr.begin(), g->ptr.end());
    TTN_CUDA(cudaMemcpyAsync(dptrs, hp.data(), sizeof(void*) * world, cudaMemcpyHostToDevice, s));
    const int blocks = (int)std::min<size_t>((n + 255) / 256, 1184);
    launch_k(loop_reduce<T, OP>, blocks, 256, 0, s, static_cast<T*>(tmp), reinterpret_cast<const T* const*>(dptrs), world, n);
    TTN_CUDA(cudaGetLastError());
    TTN_CUDA(cudaStreamSynchronize(s));   // hp (pageable) is read by the copy above
    done(s);
    for (int r = 0; r < world; ++r)
      if (r != rank) TTN_CUDA(cudaStreamWaitEvent(s, g->ev2[r], 0));   // everyone has read buf
    TTN_CUDA(cudaMemcpyAsync(buf, tmp, n * sizeof(T), cudaMemcpyDeviceToDevice, s));
  }
  void bcast(void* buf, size_t bytes, int root, cudaStream_t s) override {
    if (bytes == 0 || world == 1) return;
    publish(buf, s);
    if (rank != root) {
      TTN_CUDA(cudaStreamWaitEvent(s, g->ev1[root], 0));
      TTN_CUDA(cudaMemcpyAsync(buf, g->ptr[root], bytes, cudaMemcpyDeviceToDevice, s));
    }
    done(s);
    if (rank == root)   // the root's buffer stays unchanged until every copy has read it
      for (int r = 0; r < world; ++r)
        if (r != rank) TTN_CUDA(cudaStreamWaitEvent(s, g->ev2[r], 0));
  }
  void allreduce_sum(double* buf, size_t n, cudaStream_t s) override { allreduce<double, 0>(buf, n, s); }
  void allreduce_sum(int* buf, size_t n, cudaStream_t s) override { allreduce<int, 0>(buf, n, s); }
  void allreduce_max(int* buf, size_t n, cudaStream_t s) override { allreduce<int, 1>(buf, n, s); }
};

}  // namespace

Comm* loop_comm_create(LoopGroup* g, int rank, int device) {
  if (!g || rank < 0 || rank >= g->world) throw Error(TTN_ERR_ARG, "bad loopback rank");
  TTN_CUDA(cudaSetDevice(device));
  return new LoopComm(g, rank);
}

}  // namespace tcbc
