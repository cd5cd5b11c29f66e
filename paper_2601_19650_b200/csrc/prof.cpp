#include <cstdlib>
#include <cstdio>
#include <chrono>
#include "prof.h"

#include <map>
#include <mutex>
#include <string>
#include <vector>

namespace tcbc {

namespace {

struct Pending {
  cudaEvent_t a, b;
  std::string family;
  double flops, bytes;
  bool owned = false;   // events belong to a graph (ProfSink): not returned to the pool
};

struct Acc {
  double ms = 0.0, flops = 0.0, bytes = 0.0;
  long long launches = 0;
};

struct Profiler {
  std::mutex mu;
  bool on = false;
  std::vector<cudaEvent_t> pool;
  std::vector<Pending> pending;
  std::map<std::string, Acc> acc;

  cudaEvent_t get() {
    if (!pool.empty()) {
      cudaEvent_t e = pool.back();
      pool.pop_back();
      return e;
    }
    cudaEvent_t e;
    cudaEventCreate(&e);
    return e;
  }
  void harvest() {
    for (auto& p : pending) {
      float ms = 0.f;
      cudaEventSynchronize(p.b);
      cudaEventElapsedTime(&ms, p.a, p.b);
      Acc& a = acc[p.family];
      a.ms += ms;
      a.flops += p.flops;
      a.bytes += p.bytes;
      a.launches += 1;
      if (p.family == "gap_after_sync") {   // idle time, not kernel time
        pool.push_back(p.a);
        pool.push_back(p.b);
        continue;
      }
      Acc& t = acc["all"];
      t.ms += ms;
      t.flops += p.flops;
      t.bytes += p.bytes;
      t.launches += 1;
      if (!p.owned) {
        pool.push_back(p.a);
        pool.push_back(p.b);
      }
    }
    pending.clear();
  }
};

Profiler& P() {
  static Profiler p;
  return p;
}

thread_local cudaEvent_t t_open = nullptr;   // per host thread (worker contexts run concurrently)
thread_local cudaEvent_t t_gap = nullptr;    // recorded right after a host synchronisation
thread_local ProfSink* t_sink = nullptr;     // graph capture in progress on this thread

}  // namespace

ProfSink::~ProfSink() {
  for (auto& r : recs) {
    cudaEventDestroy(r.a);
    cudaEventDestroy(r.b);
  }
}

void prof_set_sink(ProfSink* s) { t_sink = s; }

bool prof_on() { return P().on; }

void prof_replay(const ProfSink& s) {
  Profiler& p = P();
  if (!p.on || s.recs.empty()) return;
  std::lock_guard<std::mutex> g(p.mu);
  for (auto& r : s.recs) p.pending.push_back(Pending{r.a, r.b, r.family, r.flops, r.bytes, true});
  p.harvest();   // the next replay re-records these events: read them now (the caller synchronised)
}

void prof_mark_sync(cudaStream_t s) {
  Profiler& p = P();
  if (!p.on || t_sink) return;
  std::lock_guard<std::mutex> g(p.mu);
  if (t_gap) p.pool.push_back(t_gap);
  t_gap = p.get();
  cudaEventRecord(t_gap, s);
}

void prof_begin(cudaStream_t s) {
  Profiler& p = P();
  if (!p.on) return;
  if (t_sink) {   // capture: a fresh event owned by the graph
    cudaEvent_t e;
    cudaEventCreate(&e);
    cudaEventRecord(e, s);
    t_open = e;
    return;
  }
  std::lock_guard<std::mutex> g(p.mu);
  if (t_gap) {   // device idle from the synchronisation to this launch set: host work in between
    cudaEvent_t e = p.get();
    cudaEventRecord(e, s);
    p.pending.push_back(Pending{t_gap, e, "gap_after_sync", 0.0, 0.0});
    t_gap = nullptr;
  }
  t_open = p.get();
  cudaEventRecord(t_open, s);
}

void prof_end(cudaStream_t s, const char* family, double flops, double bytes) {
  Profiler& p = P();
  if (!p.on) return;
  if (t_sink) {
    if (!t_open) return;
    cudaEvent_t b;
    cudaEventCreate(&b);
    cudaEventRecord(b, s);
    t_sink->recs.push_back(ProfSink::Rec{t_open, b, family, flops, bytes});
    t_open = nullptr;
    return;
  }
  std::lock_guard<std::mutex> g(p.mu);
  if (!t_open) return;
  cudaEvent_t b = p.get();
  cudaEventRecord(b, s);
  p.pending.push_back(Pending{t_open, b, family, flops, bytes});
  t_open = nullptr;
  if (p.pending.size() > 4096) p.harvest();
}

void prof_enable(bool on) {
  Profiler& p = P();
  std::lock_guard<std::mutex> g(p.mu);
  p.harvest();
  p.acc.clear();
  p.on = on;
}

bool prof_read(const char* family, double* ms, double* flops, double* bytes, long long* launches) {
  Profiler& p = P();
  std::lock_guard<std::mutex> g(p.mu);
  p.harvest();
  auto it = p.acc.find(family);
  if (it == p.acc.end()) {
    *ms = *flops = *bytes = 0.0;
    *launches = 0;
    return false;
  }
  *ms = it->second.ms;
  *flops = it->second.flops;
  *bytes = it->second.bytes;
  *launches = it->second.launches;
  return true;
}

}  // namespace tcbc

namespace tcbc {
namespace {
std::mutex g_hmu;
std::map<std::string, double>& hmap() {
  static std::map<std::string, double> m;
  return m;
}
double now_s() {
  return std::chrono::duration<double>(std::chrono::steady_clock::now().time_since_epoch()).count();
}
}  // namespace
thread_local double t_wait = 0.0;
void host_prof_wait(double seconds) { t_wait += seconds; }
bool host_prof_on() {
  static const bool on = getenv("TTN_HOST_PROF") != nullptr;
  return on;
}
void host_prof_add(const char* name, double seconds) {
  std::lock_guard<std::mutex> lk(g_hmu);
  hmap()[name] += seconds;
}
void host_prof_dump() {
  std::lock_guard<std::mutex> lk(g_hmu);
  for (auto& kv : hmap()) fprintf(stderr, "  [host] %-18s %8.3f ms\n", kv.first.c_str(), kv.second * 1e3);
  hmap().clear();
}
HostScope::HostScope(const char* n) : name(n), t0(host_prof_on() ? now_s() : 0.0), w0(t_wait) {}
HostScope::~HostScope() {
  if (host_prof_on()) host_prof_add(name, now_s() - t0 - (t_wait - w0));
}
}  // namespace tcbc
