// Two-stage Hermitian tridiagonalisation (K1 of the batched eigensolver for 64 < n <= 256):
// dense -> band (panel QR + compact-WY two-sided update on DMMA) -> real tridiagonal (bulge
// chasing in shared memory), and the matching back-transform.  See heev2s.cu.
#pragma once
#include "kernels.h"

namespace tcbc {

constexpr int H2S_NB = 8;        // band width of stage 1
constexpr int H2S_MIN_N = 65;    // smaller Grams keep the one-stage kernel (whole matrix on chip)
constexpr int H2S_MAX_N = 256;
constexpr int H2S_ROUTE_N = 160;  // default route: two-stage from this order (measured, heev2s_use)
// scalar slots of the eigensolver's work array (must match heev.cu's enum)
constexpr int H2S_S_TRACE = 4;

// per-problem work layout of heev.cu (doubles) before the two-stage area:
// d[n] e[n] scalars[8] Z[n*kmax] LU[5*n*kmax] W[kmax*kmax] clusters[2*kmax] warp scratch[8*6n]
__host__ __device__ inline size_t heev_base_doubles(int n, int kmax) {
  return (size_t)2 * n + 8 + (size_t)n * kmax * 6 + (size_t)kmax * kmax + 2 * (size_t)kmax + (size_t)8 * 6 * n;
}
// stage-2 tasks of sweep s (reflectors acting on rows s+1+t*NB ..)
__host__ __device__ inline int h2s_ntask(int n, int s) { return (n - 1 - s + H2S_NB - 1) / H2S_NB; }
// sum_{u=1}^{x} ceil(u / NB)
__host__ __device__ inline int h2s_F(int x) {
  const int q = x / H2S_NB, r = x % H2S_NB;
  return H2S_NB * q * (q + 1) / 2 + (q + 1) * r;
}
// index of the first reflector of sweep s; h2s_ref_base(n, n - 1) = total
__host__ __device__ inline int h2s_ref_base(int n, int s) { return h2s_F(n - 1) - h2s_F(n - 1 - s); }
__host__ __device__ inline int h2s_panels(int n) {
  int p = 0;
  while (n - (p + 1) * H2S_NB >= 2) ++p;
  return p;
}
// two-stage area (doubles): T factors [panels][NB][NB] complex, then the stage-2 reflectors
// [nref][NB] complex and their tau [nref] complex
__host__ __device__ inline size_t h2s_extra_doubles(int n) {
  if (n < H2S_MIN_N || n > H2S_MAX_N) return 0;
  const size_t nref = (size_t)h2s_ref_base(n, n - 1);
  return 2 * ((size_t)h2s_panels(n) * H2S_NB * H2S_NB + nref * H2S_NB + nref);
}

// Route override for tests (ttn_test_heev): 0 = default, 1 = one-stage only, 2 = two-stage
// wherever the order allows.
void heev2s_set_route(int route);
int heev2s_route();
// whether launch_heev sends a Gram of order n (one of `count` one-CTA Grams) to the two-stage path
bool heev2s_use(int n, int count);

// K1 (stage 1 + stage 2 + the tridiagonal's statistics) for nprob problems of order <= maxn
void launch_heev2s_reduce(const HeevProblem* d, int nprob, int maxn, cudaStream_t s);
// K5 for the same problems: h is the host copy (bstart is filled here), staged by the caller
void heev2s_assign_blocks(HeevProblem* h, int nprob, int& nblocks);
void launch_heev2s_backtr(const HeevProblem* d, int nprob, int nblocks, int maxn, cudaStream_t s);

}  // namespace tcbc
