// extern "C" entry points of libttncbc (include/ttn_cbc.h).  Every call converts
// exceptions to a ttn_status and records the message on the context.
#include "prof.h"
#include "runtime.h"
#include "heev2s.h"

#include <cmath>
#include <cstring>
#include <exception>
#include <new>
#include <thread>
#include <vector>

using namespace tcbc;

namespace {

template <typename F>
ttn_status guard(ttn_ctx ctx, F&& f) {
  try {
    f();
    return TTN_OK;
  } catch (const Error& e) {
    if (ctx) ctx->last_error = e.what();
    return e.status;
  } catch (const std::bad_alloc&) {
    if (ctx) ctx->last_error = "host allocation failed";
    return TTN_ERR_OOM;
  } catch (const std::exception& e) {
    if (ctx) ctx->last_error = e.what();
    return TTN_ERR_CUDA;
  }
}

struct DeviceGuard {
  int prev = -1;
  explicit DeviceGuard(int dev) {
    cudaGetDevice(&prev);
    if (prev != dev) cudaSetDevice(dev);
  }
  ~DeviceGuard() {
    int cur = -1;
    cudaGetDevice(&cur);
    if (prev >= 0 && cur != prev) cudaSetDevice(prev);
  }
};

}  // namespace

extern "C" {

const char* ttn_version(void) { return "ttncbc 0.1 sm_100a (DMMA complex-FP64)"; }

namespace {
// common part of ttn_ctx_create and the worker contexts of ttn_ctx_set_workers: a worker
// shares its parent's memory source (pool or caller allocator), so results handed to the
// parent are freed from the source they came from
ttn_status ctx_create_impl(int device, void* cuda_stream, const ttn_allocator* alloc, const ttn_ctx_s* parent,
                           ttn_ctx* out) {
  if (!out) return TTN_ERR_ARG;
  *out = nullptr;
  if (alloc && (!alloc->alloc || !alloc->free)) return TTN_ERR_ARG;
  ttn_ctx_s* c = new (std::nothrow) ttn_ctx_s();
  if (!c) return TTN_ERR_OOM;
  ttn_status s = guard(nullptr, [&] {
    int n = 0;
    TTN_CUDA(cudaGetDeviceCount(&n));
    if (device < 0 || device >= n) throw Error(TTN_ERR_ARG, "bad device id");
    TTN_CUDA(cudaSetDevice(device));
    c->device = device;
    c->stream = static_cast<cudaStream_t>(cuda_stream);
    if (parent) {
      c->speculate = parent->speculate;
      c->graphs = parent->graphs;
      c->has_user_alloc = parent->has_user_alloc;
      c->user_alloc = parent->user_alloc;
      c->pool = parent->pool;
    } else if (alloc) {
      c->has_user_alloc = true;
      c->user_alloc = *alloc;
    } else {
      // a pool of this context (the device's default pool is left as other libraries set it);
      // freed blocks stay cached in the pool across applies, and go back to the device at
      // ttn_ctx_destroy
      cudaMemPoolProps props{};
      props.allocType = cudaMemAllocationTypePinned;
      props.handleTypes = cudaMemHandleTypeNone;
      props.location.type = cudaMemLocationTypeDevice;
      props.location.id = device;
      TTN_CUDA(cudaMemPoolCreate(&c->pool, &props));
      c->owns_pool = true;
      uint64_t thr = UINT64_MAX;
      TTN_CUDA(cudaMemPoolSetAttribute(c->pool, cudaMemPoolAttrReleaseThreshold, &thr));
    }
    c->scratch.set_source(c);
    c->env.set_source(c);
    c->ring = new RingStager(c->stream);
    c->stager = c->ring;
    c->ensure_small(1 << 20);
  });
  if (s != TTN_OK) {
    delete c->ring;
    if (c->owns_pool) cudaMemPoolDestroy(c->pool);
    delete c;
    return s;
  }
  *out = c;
  return TTN_OK;
}
}  // namespace

ttn_status ttn_ctx_create(int device, void* cuda_stream, const ttn_allocator* alloc, ttn_ctx* out) {
  return ctx_create_impl(device, cuda_stream, alloc, nullptr, out);
}

ttn_status ttn_ctx_destroy(ttn_ctx ctx) {
  if (!ctx) return TTN_ERR_ARG;
  DeviceGuard g(ctx->device);
  cudaStreamSynchronize(ctx->stream);
  for (auto* w : ctx->workers) ttn_ctx_destroy(w);
  ctx->workers.clear();
  graphs_release(ctx);
  ctx->scratch.release();
  ctx->env.release();
  cudaStreamSynchronize(ctx->stream);
  ctx->reap(true);
  delete ctx->ring;
  delete ctx->comm;
  if (ctx->hbuf) cudaFreeHost(ctx->hbuf);
  if (ctx->spec_host) cudaFreeHost(ctx->spec_host);
  if (ctx->rank_ev) cudaEventDestroy(ctx->rank_ev);
  // outstanding TTN handles keep their blocks: the pool is released once they are freed
  if (ctx->owns_pool) cudaMemPoolDestroy(ctx->pool);
  if (ctx->owns_stream) cudaStreamDestroy(ctx->stream);
  delete ctx;
  return TTN_OK;
}

const char* ttn_last_error(ttn_ctx ctx) { return ctx ? ctx->last_error.c_str() : "NULL context"; }

ttn_status ttn_create(ttn_ctx ctx, ttn_kind kind, int32_t n_nodes, const int32_t* parent, const int32_t* phys_dim,
                      const int64_t* bond, const ttn_c128* const* data, int data_on_device, ttn* out) {
  if (!ctx || !out) return TTN_ERR_ARG;
  *out = nullptr;
  DeviceGuard g(ctx->device);
  ttn_s* t = nullptr;
  ttn_status s = guard(ctx, [&] {
    if (!parent || !phys_dim || !bond || !data) throw Error(TTN_ERR_ARG, "NULL argument");
    if (kind != TTN_STATE && kind != TTN_OPERATOR) throw Error(TTN_ERR_ARG, "bad kind");
    t = new ttn_s();
    t->ctx = ctx;
    t->kind = kind;
    build_topology(t, parent, n_nodes);
    t->phys.assign(phys_dim, phys_dim + n_nodes);
    t->bond.assign(bond, bond + n_nodes);
    for (int i = 0; i < n_nodes; ++i) {
      if (t->phys[i] < 1) throw Error(TTN_ERR_ARG, "phys_dim must be >= 1");
      if (i != t->root && t->bond[i] < 1) throw Error(TTN_ERR_ARG, "bond must be >= 1");
      if (!data[i]) throw Error(TTN_ERR_ARG, "NULL tensor pointer");
    }
    t->bond[t->root] = 1;
    finalize_shapes(t);
    t->data = static_cast<cplx*>(ctx->get(sizeof(cplx) * std::max<int64_t>(t->total, 1)));
    // runs of nodes whose source tensors are adjacent in memory (a packed TTN buffer) move
    // with one copy each
    const cudaMemcpyKind kind_cp = data_on_device ? cudaMemcpyDeviceToDevice : cudaMemcpyHostToDevice;
    bool pinned = !data_on_device;
    for (int i = 0; i < n_nodes;) {
      int j = i + 1;
      int64_t run = 0;
      for (auto x : t->shape[i]) run = (run ? run : 1) * x;
      while (j < n_nodes && data[j] == data[i] + run) {
        int64_t e = 1;
        for (auto x : t->shape[j]) e *= x;
        run += e;
        ++j;
      }
      if (pinned) {
        cudaPointerAttributes at;
        pinned = cudaPointerGetAttributes(&at, data[i]) == cudaSuccess && at.type == cudaMemoryTypeHost;
        cudaGetLastError();
      }
      TTN_CUDA(cudaMemcpyAsync(t->node(i), data[i], sizeof(cplx) * run, kind_cp, ctx->stream));
      i = j;
    }
    // pageable host buffers: finish before returning; pinned ones stay stream-ordered (the
    // caller keeps them unchanged until the ctx stream has passed the copy)
    if (!data_on_device && !pinned) ctx->sync();
  });
  if (s != TTN_OK) {
    if (t) {
      if (t->data) ctx->put(t->data);
      delete t;
    }
    return s;
  }
  *out = t;
  return TTN_OK;
}

ttn_status ttn_destroy(ttn t) {
  if (!t) return TTN_ERR_ARG;
  DeviceGuard g(t->ctx->device);
  free_ttn(t);
  return TTN_OK;
}

ttn_status ttn_n_nodes(ttn t, int32_t* out) {
  if (!t || !out) return TTN_ERR_ARG;
  *out = t->n;
  return TTN_OK;
}

ttn_status ttn_node_shape(ttn t, int32_t node, int32_t* ndim, int64_t* dims) {
  if (!t || !ndim || !dims || node < 0 || node >= t->n) return TTN_ERR_ARG;
  const auto& s = t->shape[node];
  if (s.size() > 16) return TTN_ERR_UNSUPPORTED;
  *ndim = (int32_t)s.size();
  for (size_t i = 0; i < s.size(); ++i) dims[i] = s[i];
  return TTN_OK;
}

ttn_status ttn_get_tensor(ttn_ctx ctx, ttn t, int32_t node, ttn_c128* host_out, size_t capacity_elems) {
  if (!ctx || !t || !host_out) return TTN_ERR_ARG;
  DeviceGuard g(ctx->device);
  return guard(ctx, [&] {
    if (node < 0 || node >= t->n) throw Error(TTN_ERR_ARG, "bad node id");
    int64_t e = 1;
    for (auto x : t->shape[node]) e *= x;
    if ((size_t)e > capacity_elems) throw Error(TTN_ERR_ARG, "output buffer too small");
    TTN_CUDA(cudaMemcpyAsync(host_out, t->node(node), sizeof(cplx) * e, cudaMemcpyDeviceToHost, ctx->stream));
    ctx->sync();
  });
}

ttn_status ttn_get_data(ttn_ctx ctx, ttn t, ttn_c128* host_out, size_t capacity_elems) {
  if (!ctx || !t || !host_out) return TTN_ERR_ARG;
  DeviceGuard g(ctx->device);
  return guard(ctx, [&] {
    if ((size_t)t->total > capacity_elems) throw Error(TTN_ERR_ARG, "output buffer too small");
    TTN_CUDA(cudaMemcpyAsync(host_out, t->data, sizeof(cplx) * t->total, cudaMemcpyDeviceToHost, ctx->stream));
    ctx->sync();
  });
}

ttn_status ttn_get_data_batch(ttn_ctx ctx, int32_t n, const ttn* t, ttn_c128* const* host_out,
                              const size_t* capacity_elems) {
  if (!ctx || n < 0 || (n > 0 && (!t || !host_out || !capacity_elems))) return TTN_ERR_ARG;
  DeviceGuard g(ctx->device);
  return guard(ctx, [&] {
    for (int i = 0; i < n; ++i) {
      if (!t[i] || !host_out[i]) throw Error(TTN_ERR_ARG, "NULL handle or buffer");
      if ((size_t)t[i]->total > capacity_elems[i]) throw Error(TTN_ERR_ARG, "output buffer too small");
    }
    for (int i = 0; i < n; ++i)
      TTN_CUDA(cudaMemcpyAsync(host_out[i], t[i]->data, sizeof(cplx) * t[i]->total, cudaMemcpyDeviceToHost,
                               ctx->stream));
    ctx->sync();
  });
}

ttn_status cbc_apply(ttn_ctx ctx, ttn op, ttn state, int64_t max_bond, double tol, ttn* out, ttn_cbc_report* rep) {
  if (!ctx || !out) return TTN_ERR_ARG;
  return cbc_apply_batch(ctx, 1, &op, &state, max_bond, tol, out, rep);
}

ttn_status cbc_apply_batch(ttn_ctx ctx, int32_t n, const ttn* ops, const ttn* states, int64_t max_bond, double tol,
                           ttn* outs, ttn_cbc_report* reps) {
  if (!ctx || !ops || !states || !outs || n < 1) return TTN_ERR_ARG;
  for (int i = 0; i < n; ++i) outs[i] = nullptr;
  DeviceGuard g(ctx->device);
  std::vector<ttn_s*> res(n, nullptr);
  ttn_status s = guard(ctx, [&] {
    std::vector<const ttn_s*> o(ops, ops + n), st(states, states + n);
    const int W = (int)ctx->workers.size();
    if (W < 2 || ctx->comm || n < 2 * W) {
      cbc_apply_impl(ctx, n, o.data(), st.data(), max_bond, tol, res.data(), reps);
      return;
    }
    // W concurrent sub-batches, each on a worker context (own stream, staging ring, arenas)
    // driven by its own host thread: one sub-batch's host-side planning and rank syncs
    // overlap the others' kernels.  Streams are joined with events both ways.
    cudaEvent_t start;
    TTN_CUDA(cudaEventCreateWithFlags(&start, cudaEventDisableTiming));
    TTN_CUDA(cudaEventRecord(start, ctx->stream));
    std::vector<std::exception_ptr> err(W);
    std::vector<std::thread> th;
    for (int w = 0; w < W; ++w) {
      const int b0 = (int)((long long)n * w / W), b1 = (int)((long long)n * (w + 1) / W);
      th.emplace_back([&, w, b0, b1] {
        try {
          ttn_ctx_s* wc = ctx->workers[w];
          DeviceGuard gw(wc->device);
          TTN_CUDA(cudaStreamWaitEvent(wc->stream, start, 0));
          cbc_apply_impl(wc, b1 - b0, o.data() + b0, st.data() + b0, max_bond, tol, res.data() + b0,
                         reps ? reps + b0 : nullptr);
        } catch (...) {
          err[w] = std::current_exception();
        }
      });
    }
    for (auto& t : th) t.join();
    for (int w = 0; w < W; ++w) {
      cudaEvent_t done;
      TTN_CUDA(cudaEventCreateWithFlags(&done, cudaEventDisableTiming));
      TTN_CUDA(cudaEventRecord(done, ctx->workers[w]->stream));
      TTN_CUDA(cudaStreamWaitEvent(ctx->stream, done, 0));
      cudaEventDestroy(done);
    }
    cudaEventDestroy(start);
    for (auto& r : res)
      if (r) r->ctx = ctx;   // results belong to the caller's context from here on
    for (auto& e : err)
      if (e) std::rethrow_exception(e);
  });
  if (s != TTN_OK) {
    for (auto* r : res) free_ttn(r);
    cudaGetLastError();
    return s;
  }
  for (int i = 0; i < n; ++i) outs[i] = res[i];
  return TTN_OK;
}

ttn_status ttn_overlap_batch(ttn_ctx ctx, int32_t n, const ttn* a, const ttn* b, ttn_c128* out) {
  if (!ctx || !a || !b || !out || n < 1) return TTN_ERR_ARG;
  DeviceGuard g(ctx->device);
  return guard(ctx, [&] {
    std::vector<const ttn_s*> x(a, a + n), y(b, b + n);
    std::vector<cplx> r(n);
    overlap_impl(ctx, n, x.data(), y.data(), r.data());
    for (int i = 0; i < n; ++i) out[i] = ttn_c128{r[i].x, r[i].y};
  });
}

ttn_status ttn_overlap(ttn_ctx ctx, ttn a, ttn b, ttn_c128* out) { return ttn_overlap_batch(ctx, 1, &a, &b, out); }

ttn_status ttn_sandwich(ttn_ctx ctx, ttn bra, ttn op, ttn ket, ttn_c128* out) {
  if (!ctx || !bra || !op || !ket || !out) return TTN_ERR_ARG;
  DeviceGuard g(ctx->device);
  return guard(ctx, [&] {
    const ttn_s* b[1] = {bra};
    const ttn_s* o[1] = {op};
    const ttn_s* k[1] = {ket};
    std::vector<SweepLayer> L(3);
    L[0].h = b; L[0].conj = true;
    L[1].h = o; L[1].op = true;
    L[2].h = k;
    cplx r;
    sweep_impl(ctx, 1, L, &r);
    *out = ttn_c128{r.x, r.y};
  });
}

ttn_status ttn_op_norm2(ttn_ctx ctx, ttn op, ttn ket, double* out) {
  if (!ctx || !op || !ket || !out) return TTN_ERR_ARG;
  DeviceGuard g(ctx->device);
  return guard(ctx, [&] {
    const ttn_s* o[1] = {op};
    const ttn_s* k[1] = {ket};
    std::vector<SweepLayer> L(4);
    L[0].h = k; L[0].conj = true;
    L[1].h = o; L[1].op = true; L[1].conj = true; L[1].dagger = true;
    L[2].h = o; L[2].op = true;
    L[3].h = k;
    cplx r;
    sweep_impl(ctx, 1, L, &r);
    *out = r.x;
  });
}

ttn_status ttn_test_heev(ttn_ctx ctx, int32_t nmat, int32_t n, int32_t kmax, int32_t max_bond, double tol,
                         int32_t route, const ttn_c128* a_host, double* lam_host, ttn_c128* vt_host,
                         int32_t* k_host, double* w_host) {
  if (!ctx || nmat < 1 || n < 1 || kmax < 1 || kmax > n || max_bond < 1 || !(tol >= 0.0 && tol < 1.0) || !a_host ||
      !lam_host || !vt_host || !k_host || !w_host || route < 0 || route > 2)
    return TTN_ERR_ARG;
  DeviceGuard g(ctx->device);
  return guard(ctx, [&] {
    if (n > tcbc::heev_max_n()) throw Error(TTN_ERR_UNSUPPORTED, "ttn_test_heev: order beyond the eigensolver");
    using tcbc::cplx;
    const size_t nn = (size_t)n * n;
    cplx* dA = static_cast<cplx*>(ctx->scratch.alloc(sizeof(cplx) * nn * nmat));
    double* dlam = static_cast<double*>(ctx->scratch.alloc(sizeof(double) * (size_t)kmax * nmat));
    cplx* dVt = static_cast<cplx*>(ctx->scratch.alloc(sizeof(cplx) * (size_t)kmax * n * nmat));
    int* dk = static_cast<int*>(ctx->scratch.alloc(sizeof(int) * nmat));
    double* dw = static_cast<double*>(ctx->scratch.alloc(sizeof(double) * nmat));
    TTN_CUDA(cudaMemcpyAsync(dA, a_host, sizeof(cplx) * nn * nmat, cudaMemcpyHostToDevice, ctx->stream));
    std::vector<tcbc::HeevProblem> hp(nmat);
    for (int i = 0; i < nmat; ++i) {
      tcbc::HeevProblem& h = hp[i];
      h = tcbc::HeevProblem{};
      h.A = dA + nn * i;
      h.n = n;
      h.kmax = kmax;
      h.lam = dlam + (size_t)kmax * i;
      h.Vt = dVt + (size_t)kmax * n * i;
      h.k_out = dk + i;
      h.w_out = dw + i;
      h.work = static_cast<double*>(ctx->scratch.alloc(sizeof(double) * tcbc::heev_work_doubles(n, kmax)));
      h.tau = static_cast<cplx*>(ctx->scratch.alloc(sizeof(cplx) * n));
      h.tol2 = tol * tol;
      h.floor_rel = 1e-13;
      h.max_bond = max_bond;
    }
    tcbc::heev2s_set_route(route);
    try {
      tcbc::launch_heev(hp.data(), nmat, *ctx->stager, ctx->stream);
    } catch (...) {
      tcbc::heev2s_set_route(0);
      throw;
    }
    tcbc::heev2s_set_route(0);
    TTN_CUDA(cudaGetLastError());
    TTN_CUDA(cudaMemcpyAsync(lam_host, dlam, sizeof(double) * (size_t)kmax * nmat, cudaMemcpyDeviceToHost, ctx->stream));
    TTN_CUDA(cudaMemcpyAsync(vt_host, dVt, sizeof(cplx) * (size_t)kmax * n * nmat, cudaMemcpyDeviceToHost, ctx->stream));
    TTN_CUDA(cudaMemcpyAsync(k_host, dk, sizeof(int) * nmat, cudaMemcpyDeviceToHost, ctx->stream));
    TTN_CUDA(cudaMemcpyAsync(w_host, dw, sizeof(double) * nmat, cudaMemcpyDeviceToHost, ctx->stream));
    ctx->sync();
    TTN_CUDA(cudaGetLastError());
    ctx->scratch.reset();
  });
}

ttn_status ttn_ctx_set_workers(ttn_ctx ctx, int n) {
  if (!ctx || n < 1 || n > 64) return TTN_ERR_ARG;
  DeviceGuard g(ctx->device);
  return guard(ctx, [&] {
    cudaStreamSynchronize(ctx->stream);
    for (auto* w : ctx->workers) ttn_ctx_destroy(w);
    ctx->workers.clear();
    if (n == 1) return;
    for (int i = 0; i < n; ++i) {
      cudaStream_t st;
      TTN_CUDA(cudaStreamCreateWithFlags(&st, cudaStreamNonBlocking));
      ttn_ctx w = nullptr;
      ttn_status s = ctx_create_impl(ctx->device, st, nullptr, ctx, &w);
      if (s != TTN_OK) {
        cudaStreamDestroy(st);
        throw Error(s, "worker context creation failed");
      }
      w->owns_stream = true;
      ctx->workers.push_back(w);
    }
  });
}

ttn_status ttn_ctx_set_schedule(ttn_ctx ctx, int speculate, int graphs) {
  if (!ctx) return TTN_ERR_ARG;
  DeviceGuard g(ctx->device);
  return guard(ctx, [&] {
    cudaStreamSynchronize(ctx->stream);
    graphs_release(ctx);   // also forgets the shapes whose speculation failed
    ctx->speculate = speculate != 0;
    ctx->graphs = graphs != 0 && speculate != 0;
    for (auto* w : ctx->workers) {
      graphs_release(w);
      w->speculate = ctx->speculate;
      w->graphs = ctx->graphs;
    }
  });
}

ttn_status ttn_comm_unique_id(void* out128) {
  if (!out128) return TTN_ERR_ARG;
  return guard(nullptr, [&] { comm_unique_id(out128); });
}

ttn_status ttn_ctx_set_comm(ttn_ctx ctx, const void* unique_id128, int rank, int world, int parts) {
  if (!ctx) return TTN_ERR_ARG;
  DeviceGuard g(ctx->device);
  return guard(ctx, [&] {
    cudaStreamSynchronize(ctx->stream);
    delete ctx->comm;
    ctx->comm = nullptr;
    ctx->parts = 1;
    if (!unique_id128) return;
    if (world < 1 || rank < 0 || rank >= world || parts < world) throw Error(TTN_ERR_ARG, "need 0 <= rank < world <= parts");
    ctx->comm = comm_create(unique_id128, rank, world, ctx->device);
    ctx->parts = parts;
  });
}

ttn_status ttn_loopback_create(int world, void** group_out) {
  if (!group_out || world < 1) return TTN_ERR_ARG;
  *group_out = nullptr;
  return guard(nullptr, [&] { *group_out = loop_group_create(world); });
}

ttn_status ttn_loopback_destroy(void* group) {
  if (!group) return TTN_ERR_ARG;
  loop_group_release(static_cast<LoopGroup*>(group));
  return TTN_OK;
}

ttn_status ttn_ctx_set_comm_loopback(ttn_ctx ctx, void* group, int rank, int parts) {
  if (!ctx || !group) return TTN_ERR_ARG;
  DeviceGuard g(ctx->device);
  return guard(ctx, [&] {
    LoopGroup* lg = static_cast<LoopGroup*>(group);
    cudaStreamSynchronize(ctx->stream);
    delete ctx->comm;
    ctx->comm = nullptr;
    ctx->parts = 1;
    Comm* c = loop_comm_create(lg, rank, ctx->device);
    if (parts < c->world) {
      delete c;
      throw Error(TTN_ERR_ARG, "need parts >= world");
    }
    ctx->comm = c;
    ctx->parts = parts;
  });
}

ttn_status ttn_partition_plan(int32_t n_nodes, const int32_t* parent, int parts, int32_t* group_out) {
  if (!parent || !group_out || n_nodes < 1 || parts < 1) return TTN_ERR_ARG;
  return guard(nullptr, [&] {
    ttn_s t;
    build_topology(&t, parent, n_nodes);
    std::vector<int> g = partition_groups(&t, parts, nullptr);
    for (int i = 0; i < n_nodes; ++i) group_out[i] = g[i];
  });
}

ttn_status ttn_profile_enable(int on) {
  prof_enable(on != 0);
  return TTN_OK;
}

ttn_status ttn_profile_read(const char* family, double* ms, double* flops, double* bytes, int64_t* launches) {
  if (!family || !ms || !flops || !bytes || !launches) return TTN_ERR_ARG;
  long long l = 0;
  prof_read(family, ms, flops, bytes, &l);
  *launches = l;
  return TTN_OK;
}

ttn_status ttn_launch_count(int64_t* out) {
  if (!out) return TTN_ERR_ARG;
  *out = launch_count();
  return TTN_OK;
}

ttn_status ttn_norm(ttn_ctx ctx, ttn a, double* out) {
  if (!out) return TTN_ERR_ARG;
  ttn_c128 v;
  ttn_status s = ttn_overlap(ctx, a, a, &v);
  if (s != TTN_OK) return s;
  *out = v.re > 0 ? std::sqrt(v.re) : 0.0;
  return TTN_OK;
}

}  // extern "C"
