// Optional per-kernel-family CUDA-event timing (ttn_profile_enable / ttn_profile_read).
// When enabled, every launcher brackets its launch with two events on the launching stream;
// elapsed times are harvested lazily (ttn_profile_read synchronises the device).
#pragma once
#include <cuda_runtime.h>
#include <vector>

namespace tcbc {

void prof_begin(cudaStream_t s);                       // no-op unless enabled
void prof_mark_sync(cudaStream_t s);                   // after a host synchronisation of s
void prof_end(cudaStream_t s, const char* family, double flops, double bytes);
void prof_enable(bool on);
bool prof_on();
// CUDA-graph capture: while a sink is set on this thread, prof_begin / prof_end record events
// owned by the sink (they become event-record nodes of the graph); prof_replay queues the
// sink's records after each launch of that graph, so graph replays are timed per family too.
struct ProfSink {
  struct Rec { cudaEvent_t a, b; const char* family; double flops, bytes; };
  std::vector<Rec> recs;
  ~ProfSink();
};
void prof_set_sink(ProfSink* s);
void prof_replay(const ProfSink& s);
bool prof_read(const char* family, double* ms, double* flops, double* bytes, long long* launches);

// Host wall-time accumulators (TTN_HOST_PROF diagnostics; no-ops otherwise).  Nested scopes
// double count; host_prof_dump prints and clears.
bool host_prof_on();
void host_prof_add(const char* name, double seconds);
void host_prof_dump();
void host_prof_wait(double seconds);   // time blocked in stream synchronisation (excluded)
struct HostScope {
  const char* name;
  double t0, w0;
  explicit HostScope(const char* n);
  ~HostScope();
};

}  // namespace tcbc
