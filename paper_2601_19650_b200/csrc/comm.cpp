// NCCL binding of the ctx communicator (see comm.h).
#include "comm.h"
#include "runtime.h"

#include <dlfcn.h>
#include <cstring>
#include <mutex>
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

Comm* comm_create(const void* id128, int rank, int world, int device) {
  if (world < 1 || rank < 0 || rank >= world) throw Error(TTN_ERR_ARG, "bad rank / world");
  NcclId id;
  std::memcpy(&id, id128, sizeof(id));
  TTN_CUDA(cudaSetDevice(device));
  Comm* c = new Comm();
  c->rank = rank;
  c->world = world;
  check(nccl().CommInitRank(&c->comm, world, id, rank), "ncclCommInitRank");
  return c;
}

Comm::~Comm() {
  if (comm && nccl().CommDestroy) nccl().CommDestroy(comm);
}

void Comm::bcast(void* buf, size_t bytes, int root, cudaStream_t s) {
  if (!comm || bytes == 0) return;
  check(nccl().Broadcast(buf, buf, bytes, /*ncclInt8*/ 0, root, comm, s), "ncclBroadcast");
}

void Comm::allreduce_sum(double* buf, size_t n, cudaStream_t s) {
  if (!comm || n == 0) return;
  check(nccl().AllReduce(buf, buf, n, nccl_float64, nccl_sum, comm, s), "ncclAllReduce");
}

void Comm::allreduce_sum(int* buf, size_t n, cudaStream_t s) {
  if (!comm || n == 0) return;
  check(nccl().AllReduce(buf, buf, n, nccl_int32, nccl_sum, comm, s), "ncclAllReduce");
}

void Comm::allreduce_max(int* buf, size_t n, cudaStream_t s) {
  if (!comm || n == 0) return;
  check(nccl().AllReduce(buf, buf, n, nccl_int32, nccl_max, comm, s), "ncclAllReduce");
}

void Comm::group_start() {
  if (comm) check(nccl().GroupStart(), "ncclGroupStart");
}
void Comm::group_end() {
  if (comm) check(nccl().GroupEnd(), "ncclGroupEnd");
}

}  // namespace tcbc
