// Optional per-kernel-family CUDA-event timing (ttn_profile_enable / ttn_profile_read).
// When enabled, every launcher brackets its launch with two events on the launching stream;
// elapsed times are harvested lazily (ttn_profile_read synchronises the device).
#pragma once
#include <cuda_runtime.h>

namespace tcbc {

void prof_begin(cudaStream_t s);                       // no-op unless enabled
void prof_end(cudaStream_t s, const char* family, double flops, double bytes);
void prof_enable(bool on);
bool prof_read(const char* family, double* ms, double* flops, double* bytes, long long* launches);

}  // namespace tcbc
