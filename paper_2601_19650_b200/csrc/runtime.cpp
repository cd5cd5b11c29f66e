#include <chrono>
// Host runtime: arenas, staging ring, context helpers, TTN handle construction.
#include "runtime.h"
#include "prof.h"

#include <algorithm>
#include <cstring>

namespace tcbc {

Arena::~Arena() { release(); }

void* Arena::alloc(size_t bytes) {
  bytes = (bytes + 255) & ~size_t(255);
  if (bytes == 0) bytes = 256;
  while (cur_ < chunks_.size()) {
    Chunk& c = chunks_[cur_];
    if (c.used + bytes <= c.size) {
      void* p = c.p + c.used;
      c.used += bytes;
      live_ += bytes;
      high_ = std::max(high_, live_);
      return p;
    }
    ++cur_;
  }
  size_t sz = std::max(bytes, chunk_);
  if (frozen) throw Error(TTN_ERR_UNSUPPORTED, "arena growth during a graph capture");
  char* p = nullptr;
  if (src_) {
    p = static_cast<char*>(src_->get(sz));
  } else {
    cudaError_t e = cudaMalloc(&p, sz);
    if (e != cudaSuccess) {
      cudaGetLastError();
      throw Error(TTN_ERR_OOM, "device allocation of " + std::to_string(sz) + " bytes failed");
    }
  }
  chunks_.push_back(Chunk{p, sz, bytes});
  cur_ = chunks_.size() - 1;
  live_ += bytes;
  high_ = std::max(high_, live_);
  return p;
}

void Arena::reset() {
  for (auto& c : chunks_) c.used = 0;
  cur_ = 0;
  live_ = 0;
}

void Arena::release() {
  for (auto& c : chunks_) {
    if (src_) src_->put(c.p);
    else cudaFree(c.p);
  }
  chunks_.clear();
  cur_ = 0;
  live_ = 0;
}

RingStager::RingStager(cudaStream_t s, size_t bytes) : s_(s), size_(bytes) {
  TTN_CUDA(cudaMallocHost(&h_, size_));
  TTN_CUDA(cudaMalloc(&d_, size_));
}

RingStager::~RingStager() {
  if (h_) cudaFreeHost(h_);
  if (d_) cudaFree(d_);
}

void* RingStager::put(const void* host, size_t bytes) {
  size_t b = (bytes + 255) & ~size_t(255);
  if (b > size_) throw Error(TTN_ERR_UNSUPPORTED, "descriptor array larger than the staging ring");
  if (off_ + b > size_) {  // wrap: earlier copies must have completed before reuse
    TTN_CUDA(cudaStreamSynchronize(s_));
    off_ = 0;
  }
  std::memcpy(h_ + off_, host, bytes);
  TTN_CUDA(cudaMemcpyAsync(d_ + off_, h_ + off_, bytes, cudaMemcpyHostToDevice, s_));
  void* d = d_ + off_;
  off_ += b;
  staged += b;
  return d;
}

void* RingStager::reserve(size_t bytes) {
  size_t b = (bytes + 255) & ~size_t(255);
  if (b > size_) throw Error(TTN_ERR_UNSUPPORTED, "descriptor array larger than the staging ring");
  if (off_ + b > size_) {  // wrap: earlier copies must have completed before reuse
    TTN_CUDA(cudaStreamSynchronize(s_));
    off_ = 0;
  }
  return h_ + off_;
}

void* RingStager::commit(void* host, size_t bytes) {
  char* h = static_cast<char*>(host);
  if (h != h_ + off_) return put(host, bytes);   // not the reserved slot
  TTN_CUDA(cudaMemcpyAsync(d_ + off_, h, bytes, cudaMemcpyHostToDevice, s_));
  void* d = d_ + off_;
  off_ += (bytes + 255) & ~size_t(255);
  staged += (bytes + 255) & ~size_t(255);
  return d;
}

void* CaptureStager::put(const void* host, size_t bytes) {
  const size_t off = shadow.size(), b = (bytes + 255) & ~size_t(255);
  if (off + b > cap_) throw Error(TTN_ERR_UNSUPPORTED, "graph descriptor buffer too small");
  shadow.resize(off + b);
  std::memcpy(shadow.data() + off, host, bytes);
  return d_ + off;
}

void* CaptureStager::reserve(size_t bytes) {
  tmp_.resize(bytes);
  return tmp_.data();
}

void* CaptureStager::commit(void* host, size_t bytes) { return put(host, bytes); }

void RingStager::epoch() { off_ = 0; }

void build_topology(ttn_s* t, const int32_t* parent, int n) {
  if (n < 1) throw Error(TTN_ERR_ARG, "n_nodes must be >= 1");
  t->n = n;
  t->parent.assign(parent, parent + n);
  t->root = -1;
  for (int i = 0; i < n; ++i) {
    int p = parent[i];
    if (p == -1) {
      if (t->root >= 0) throw Error(TTN_ERR_TOPOLOGY, "more than one root");
      t->root = i;
    } else if (p < 0 || p >= n || p == i) {
      throw Error(TTN_ERR_TOPOLOGY, "parent index out of range");
    }
  }
  if (t->root < 0) throw Error(TTN_ERR_TOPOLOGY, "no root");
  t->children.assign(n, {});
  for (int i = 0; i < n; ++i)
    if (parent[i] >= 0) t->children[parent[i]].push_back(i);
  t->depth.assign(n, -1);
  for (int i = 0; i < n; ++i) {
    int d = 0, j = i;
    while (parent[j] != -1) {
      j = parent[j];
      if (++d > n) throw Error(TTN_ERR_TOPOLOGY, "cycle in parent array");
    }
    t->depth[i] = d;
  }
}

void finalize_shapes(ttn_s* t) {
  t->shape.assign(t->n, {});
  t->offset.assign(t->n, 0);
  int64_t off = 0;
  for (int i = 0; i < t->n; ++i) {
    std::vector<int64_t> s;
    s.push_back(t->phys[i]);
    if (t->kind == TTN_OPERATOR) s.push_back(t->phys[i]);
    s.push_back(i == t->root ? 1 : t->bond[i]);
    for (int c : t->children[i]) s.push_back(t->bond[c]);
    int64_t e = 1;
    for (auto x : s) e *= x;
    t->shape[i] = s;
    t->offset[i] = off;
    off += e;
  }
  t->total = off;
}

ttn_s* new_ttn_like(ttn_ctx_s* ctx, const ttn_s* tmpl, int kind, const std::vector<int64_t>& bond,
                    const std::function<cplx*(int64_t)>& alloc) {
  ttn_s* t = new ttn_s();
  t->ctx = ctx;
  t->kind = kind;
  t->n = tmpl->n;
  t->root = tmpl->root;
  t->parent = tmpl->parent;
  t->phys = tmpl->phys;
  t->children = tmpl->children;
  t->depth = tmpl->depth;
  t->bond = bond;
  t->bond[t->root] = 1;
  finalize_shapes(t);
  try {
    t->data = alloc ? alloc(t->total) : static_cast<cplx*>(ctx->get(sizeof(cplx) * std::max<int64_t>(t->total, 1)));
  } catch (...) {
    delete t;
    throw;
  }
  return t;
}

void free_ttn(ttn_s* t) {
  if (!t) return;
  if (t->data && t->ctx) t->ctx->put(t->data);
  delete t;
}

}  // namespace tcbc

void ttn_ctx_s::sync() {
  const auto t0 = std::chrono::steady_clock::now();
  TTN_CUDA(cudaStreamSynchronize(stream));
  const double w = std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count();
  sync_wait_s += w;
  tcbc::host_prof_wait(w);
  tcbc::prof_mark_sync(stream);
  if (stager) stager->epoch();
  ++host_syncs;
}

void ttn_ctx_s::mark_ranks() {
  if (!rank_ev) TTN_CUDA(cudaEventCreateWithFlags(&rank_ev, cudaEventDisableTiming));
  TTN_CUDA(cudaEventRecord(rank_ev, stream));
}

void ttn_ctx_s::wait_ranks() {
  const auto t0 = std::chrono::steady_clock::now();
  TTN_CUDA(cudaEventSynchronize(rank_ev));
  const double w = std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count();
  sync_wait_s += w;
  tcbc::host_prof_wait(w);
  ++host_syncs;
}

void ttn_ctx_s::ensure_small(size_t bytes) {
  if (bytes <= hbuf_size) return;
  if (hbuf) cudaFreeHost(hbuf);
  hbuf = nullptr;
  size_t sz = std::max<size_t>(bytes, 1 << 20);
  TTN_CUDA(cudaMallocHost(&hbuf, sz));
  hbuf_size = sz;
}

void* ttn_ctx_s::get(size_t bytes) {
  if (!pending_free.empty()) reap(false);
  void* p = nullptr;
  if (has_user_alloc) {
    p = user_alloc.alloc(user_alloc.state, bytes, stream);
    if (!p) throw tcbc::Error(TTN_ERR_OOM, "the caller's allocator returned NULL for " + std::to_string(bytes) + " bytes");
    return p;
  }
  cudaError_t e = cudaMallocFromPoolAsync(&p, bytes, pool, stream);
  if (e != cudaSuccess) {
    cudaGetLastError();
    throw tcbc::Error(TTN_ERR_OOM, "device allocation of " + std::to_string(bytes) + " bytes failed");
  }
  return p;
}

void ttn_ctx_s::put(void* p) {
  if (!p) return;
  if (!has_user_alloc) {
    cudaFreeAsync(p, stream);
    return;
  }
  cudaEvent_t ev = nullptr;
  if (cudaEventCreateWithFlags(&ev, cudaEventDisableTiming) != cudaSuccess || cudaEventRecord(ev, stream) != cudaSuccess) {
    cudaGetLastError();
    if (ev) cudaEventDestroy(ev);
    cudaStreamSynchronize(stream);
    user_alloc.free(user_alloc.state, p, stream);
    return;
  }
  pending_free.emplace_back(ev, p);
}

void ttn_ctx_s::reap(bool all) {
  size_t keep = 0;
  for (size_t i = 0; i < pending_free.size(); ++i) {
    auto& pf = pending_free[i];
    const bool done = all ? (cudaEventSynchronize(pf.first), true) : cudaEventQuery(pf.first) == cudaSuccess;
    if (done) {
      user_alloc.free(user_alloc.state, pf.second, stream);
      cudaEventDestroy(pf.first);
    } else {
      pending_free[keep++] = pf;
    }
  }
  pending_free.resize(keep);
}
