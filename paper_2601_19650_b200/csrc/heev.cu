// Batched Hermitian eigensolver with truncation (B:5 (c); "compressed down to
// the desired new bond dimension D-bar, for example via singular value decomposition";
// P:362 tolerance).  For a compress input X (m x n) the GPU forms the smaller Gram
// (X^H X or X X^H, whose eigenpairs are the squared singular values and singular vectors of X;
// reading A1/A2 in DESIGN.md) and needs only its top-kmax eigenpairs.
//
// A pipeline of grouped kernels over all Grams of a sweep level, each stage with its own
// natural parallelism (so no stage leaves an SM idle behind a single busy warp):
//  K1 tridiag  one CTA per matrix: Householder reduction Q^H A Q = T (real symmetric
//              tridiagonal; the complex reflector makes every off-diagonal real).  n <= 256:
//              lower triangle only, rank-2 update of step j-1 fused into the Hermitian mat-vec
//              of step j (one pass per step), its trailing rows in shared memory.
//  K2 bisect   G lanes per (matrix, eigenvalue): Sturm-count multisection for the top kmax
//              eigenvalues (G sized to the level).
//  K3 invit    one thread per (matrix, eigenvector): inverse iteration on T - lam I
//              (dgttrf / dgttrs with partial pivoting), scratch interleaved across threads.
//  K4 orth     one CTA per matrix: CholeskyQR2 of the kmax vectors (clusters of close
//              eigenvalues leave inverse-iteration vectors only approximately orthogonal).
//  K5 backtr   one warp per (matrix, eigenvector): V = Q Z by the stored reflectors, staged
//              through shared memory by a CTA of 8 eigenvectors of the same matrix.
//  K6 finish   truncation decision k = min(max_bond, #{lam > tol^2 lam_1}, #{lam > floor lam_1})
//              >= 1 and discarded weight w = trace(A) - sum_{t<k} lam_t.
#include "kernels.h"
#include "prof.h"
#include "heev2s.h"
#include <cooperative_groups.h>
#include <algorithm>
#include <cfloat>
#include <cmath>
#include <cstdlib>
#include <vector>

namespace tcbc {

namespace {

constexpr int HEEV_THREADS = 256;
constexpr int HEEV_WARPS = HEEV_THREADS / 32;
constexpr int HEEV_MAX_N = 2048;
// per-problem work layout (doubles): d[n] e[n] scalars[8] Z[n*kmax] LU[5*n*kmax] W[kmax*kmax]
enum { S_GL = 0, S_GU, S_TNORM, S_PIVMIN, S_TRACE, S_ATOL };
// ... then cluster start / size per eigenpair (2*kmax) and per-warp cluster scratch (8*6n)
__device__ __forceinline__ double* cluster_arrays(const HeevProblem& P) {
  return P.work + 2 * P.n + 8 + (size_t)P.n * P.kmax * 6 + (size_t)P.kmax * P.kmax;
}

__device__ __forceinline__ double warp_sum(double v) {
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  return v;
}

// block-wide sum of two doubles; all threads get the result
__device__ double2 block_sum2(double a, double b, double2* red) {
  a = warp_sum(a);
  b = warp_sum(b);
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  if (lane == 0) red[warp] = make_double2(a, b);
  __syncthreads();
  if (warp == 0) {
    double2 v = lane < HEEV_WARPS ? red[lane] : make_double2(0.0, 0.0);
    v.x = warp_sum(v.x);
    v.y = warp_sum(v.y);
    if (lane == 0) red[HEEV_WARPS] = v;
  }
  __syncthreads();
  double2 r = red[HEEV_WARPS];
  __syncthreads();
  return r;
}

// block-wide sum with one barrier: warp partials into buffer `parity` of red[2][HEEV_WARPS],
// every thread adds them in the same order.  Two calls between barriers must alternate parity.
__device__ __forceinline__ double2 block_sum2_1b(double a, double b, double2* red, int parity) {
  a = warp_sum(a);
  b = warp_sum(b);
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  double2* buf = red + parity * HEEV_WARPS;
  if (lane == 0) buf[warp] = make_double2(a, b);
  __syncthreads();
  double2 r = buf[0];
#pragma unroll
  for (int w = 1; w < HEEV_WARPS; ++w) {
    r.x += buf[w].x;
    r.y += buf[w].y;
  }
  return r;
}

__device__ __forceinline__ unsigned hash32(unsigned x) {
  x ^= x >> 16; x *= 0x7feb352dU; x ^= x >> 15; x *= 0x846ca68bU; x ^= x >> 16;
  return x;
}

// Sturm counts: number of eigenvalues of T (d, e2 = e^2) strictly below x, by the LAPACK
// dlaebz pivot recurrence q_i = d_i - x - e2_{i-1} / q_{i-1}; three interleaved chains.
__device__ __forceinline__ void sturm_count3(const double* __restrict__ d, const double* __restrict__ e, int n,
                                             double x1, double x2, double x3, double pivmin, int& c1, int& c2,
                                             int& c3) {
  c1 = c2 = c3 = 0;
  double q1 = d[0] - x1, q2 = d[0] - x2, q3 = d[0] - x3;
  if (q1 <= pivmin) { ++c1; q1 = fmin(q1, -pivmin); }
  if (q2 <= pivmin) { ++c2; q2 = fmin(q2, -pivmin); }
  if (q3 <= pivmin) { ++c3; q3 = fmin(q3, -pivmin); }
  for (int i = 1; i < n; ++i) {
    const double di = d[i], ep = e[i - 1], ei = ep * ep;
    q1 = di - x1 - ei / q1;
    q2 = di - x2 - ei / q2;
    q3 = di - x3 - ei / q3;
    if (q1 <= pivmin) { ++c1; q1 = fmin(q1, -pivmin); }
    if (q2 <= pivmin) { ++c2; q2 = fmin(q2, -pivmin); }
    if (q3 <= pivmin) { ++c3; q3 = fmin(q3, -pivmin); }
  }
}

template <typename P>
__device__ __forceinline__ int find_estart(const P* p, int n, int idx) {
  int lo = 0, hi = n - 1;
  while (lo < hi) {
    int mid = (lo + hi + 1) >> 1;
    if (p[mid].estart <= idx) lo = mid; else hi = mid - 1;
  }
  return lo;
}

constexpr int FUSED_MAX_N = 256;   // lower-triangle fused path (per-lane column accumulators)
constexpr int SMEM_MAX_N = 144;    // matrix (packed lower triangle) resident in shared memory

// Shared-memory budget of the fused path: the fixed vectors, then as many trailing rows of the
// packed lower triangle as fit (rows >= r0 live in shared memory, rows < r0 stay in global /
// L2).  The trailing rows are touched by every step, the leading ones only by the first r0
// steps, so the on-chip tail carries most of the traffic.  The budget keeps two CTAs per SM
// (the register limit): measured on config 3's 1024 Grams of order 128, a half-resident
// triangle with two CTAs per SM beats the fully resident one with one CTA per SM (heev
// 28 -> 26 ms per step).
constexpr size_t FUSED_SMEM_BUDGET = 110u << 10;
// n <= 128 (NQ = 4: 80 registers) fits three CTAs per SM by registers; their budget keeps three
#ifndef TCBC_SMALL_BUDGET_KB
#define TCBC_SMALL_BUDGET_KB 72
#endif
__host__ __device__ inline size_t fused_budget(int n) {
  return n <= 128 ? ((size_t)TCBC_SMALL_BUDGET_KB << 10) : FUSED_SMEM_BUDGET;
}
__host__ __device__ inline size_t fused_base_bytes(int n) { return (size_t)n * 16 * 2 + (size_t)16 * (3 + 8) * n + 64; }
// n = 192 (config 3's G-route Grams): the last ~25 rows fit; heev 26 -> 25 ms per step.
__host__ __device__ inline int fused_r0(int n) {
  if (n > FUSED_MAX_N) return n;
  const size_t avail = (fused_budget(n) - fused_base_bytes(n)) / 16;   // complex entries
  int r0 = 0;
  while ((size_t)n * (n + 1) / 2 - (size_t)r0 * (r0 + 1) / 2 > avail) ++r0;
  return r0;
}

// Householder tridiagonalisation (zhetd2, lower) touching only the lower triangle, with the
// rank-2 update of step j-1 fused into the Hermitian mat-vec of step j: one read-modify-write
// pass over the trailing triangle per step.  Rows >= r0 of the packed triangle live in shared
// memory (r0 = 0: all of it), rows < r0 in the global A.
// Reflector j is written to row j (columns > j) of the global A for the back-transform.
// NQ: 32-column blocks per row (n <= 32 NQ).
template <int NQ>
__device__ void tridiag_fused(cplx* __restrict__ A, const int n, const int r0, cplx* vcur, cplx* wcur, cplx* base,
                              double* dvec, double* evec, cplx* tau_out, double2* red) {
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  cplx* vprev = base;
  cplx* wprev = vprev + n;
  cplx* prow = wprev + n;
  cplx* colpart = prow + n;                   // [HEEV_WARPS][n]
  cplx* Ap = colpart + HEEV_WARPS * n;        // packed lower triangle (SM)
  const size_t pbase = (size_t)r0 * (r0 + 1) / 2;
#define LL(r, c) (*((r) >= r0 ? &Ap[(size_t)(r) * ((r) + 1) / 2 - pbase + (c)] : &A[(size_t)(r) * n + (c)]))
  for (int r = r0 + warp; r < n; r += HEEV_WARPS)
    for (int c = lane; c <= r; c += 32) Ap[(size_t)r * (r + 1) / 2 - pbase + c] = A[(size_t)r * n + c];
  for (int i = tid; i < n; i += HEEV_THREADS) {
    vprev[i] = make_double2(0.0, 0.0);
    wprev[i] = make_double2(0.0, 0.0);
  }
  __syncthreads();
  bool have_prev = false;
  cplx a2_prev = make_double2(0.0, 0.0);
  for (int j = 0; j < n - 1; ++j) {
    // (a) pending update U_{j-1} on column j (rows >= j), fused with (b)'s |x|^2 partials:
    // thread t owns row j + t of the column (n <= FUSED_MAX_N <= HEEV_THREADS) and keeps the
    // updated entry in a register for the reflector, so the only barrier is the reduction's
    // and the column is not read back from memory
    static_assert(FUSED_MAX_N <= HEEV_THREADS, "one column entry per thread");
    __shared__ cplx s_alpha;
    double part = 0.0;
    const int rj = j + tid;
    cplx xj = make_double2(0.0, 0.0);
    if (rj < n) {
      // pivot entries of U_{j-1} from data every thread can see (vcur[j] from step j-1's
      // reflector, wcur[j] from before its reduction barrier), not another thread's vprev / wprev
      xj = LL(rj, j);
      if (have_prev) {
        const cplx vpj = vcur[j], wq = wcur[j];
        const cplx wpj = make_double2(wq.x + a2_prev.x * vpj.x - a2_prev.y * vpj.y,
                                      wq.y + a2_prev.x * vpj.y + a2_prev.y * vpj.x);
        const cplx vr = vprev[rj], wr = wprev[rj];
        xj.x -= (vr.x * wpj.x + vr.y * wpj.y) + (wr.x * vpj.x + wr.y * vpj.y);
        xj.y -= (vr.y * wpj.x - vr.x * wpj.y) + (wr.y * vpj.x - wr.x * vpj.y);
        LL(rj, j) = xj;
      }
      if (rj >= j + 2) part = xj.x * xj.x + xj.y * xj.y;
      if (rj == j + 1) s_alpha = xj;
    }
    // (b) reflector H_j from x = A[j+1:, j]  (zlarfg)
    const double xn2 = block_sum2_1b(part, 0.0, red, 0).x;
    const cplx alpha = s_alpha;
    double beta;
    cplx tau, scale;
    if (xn2 == 0.0 && alpha.y == 0.0) {
      beta = alpha.x;
      tau = make_double2(0.0, 0.0);
      scale = make_double2(0.0, 0.0);
    } else {
      beta = -copysign(sqrt(alpha.x * alpha.x + alpha.y * alpha.y + xn2), alpha.x);
      tau = make_double2((beta - alpha.x) / beta, -alpha.y / beta);
      const cplx den = make_double2(alpha.x - beta, alpha.y);
      const double dd = den.x * den.x + den.y * den.y;
      scale = make_double2(den.x / dd, -den.y / dd);
    }
    const bool tnz = (tau.x != 0.0 || tau.y != 0.0);
    if (rj > j && rj < n) {
      const cplx v = rj == j + 1 ? make_double2(1.0, 0.0)
                                 : make_double2(xj.x * scale.x - xj.y * scale.y, xj.x * scale.y + xj.y * scale.x);
      A[(size_t)j * n + rj] = v;                        // kept for the back-transform
      vcur[rj] = tnz ? v : make_double2(0.0, 0.0);
    }
    if (tid == 0) {
      evec[j] = beta;
      dvec[j] = xj.x;   // row j is thread 0's
      tau_out[j] = tau;
    }
    __syncthreads();
    // (c) one pass over the trailing lower triangle: apply U_{j-1}, accumulate p = A v_j.
    // All of a row's entries are loaded before any is used (one memory round trip per row,
    // not one per 32-column block).
    cplx cacc[NQ];
#pragma unroll
    for (int q = 0; q < NQ; ++q) cacc[q] = make_double2(0.0, 0.0);
    // the row's contribution (update of U_{j-1}, its dot with v_j, the column partials) without
    // the cross-lane reduction of the dot
    auto row_partial = [&](const int r, double& sr, double& si) {
      const int nq = (r - j + 31) >> 5;   // column blocks that reach the diagonal (warp-uniform)
      // the row's storage (shared-memory tail or global), as one generic pointer: no per-entry
      // branch; entries past the diagonal are masked by selects, not branches
      cplx* rowp = r >= r0 ? Ap + ((size_t)r * (r + 1) / 2 - pbase) : A + (size_t)r * n;
      cplx a[NQ];
#pragma unroll
      for (int q = 0; q < NQ; ++q) {
        const int c = j + 1 + lane + 32 * q;
        a[q] = (q < nq && c <= r) ? rowp[c] : make_double2(0.0, 0.0);
      }
      const cplx vr = vcur[r];
      const cplx vpr = vprev[r], wpr = wprev[r];
#pragma unroll
      for (int q = 0; q < NQ; ++q) {
        if (q >= nq) break;
        const int c = j + 1 + lane + 32 * q;
        const bool in = c <= r;
        const int cc = in ? c : r;   // in-range index for the vector reads
        cplx av = a[q];
        if (have_prev) {   // a -= v_r conj(w_c) + w_r conj(v_c): one FMA chain per component
          const cplx vpc = vprev[cc], wpc = wprev[cc];
          av.x = fma(-vpr.x, wpc.x, av.x);
          av.x = fma(-vpr.y, wpc.y, av.x);
          av.x = fma(-wpr.x, vpc.x, av.x);
          av.x = fma(-wpr.y, vpc.y, av.x);
          av.y = fma(-vpr.y, wpc.x, av.y);
          av.y = fma(vpr.x, wpc.y, av.y);
          av.y = fma(-wpr.y, vpc.x, av.y);
          av.y = fma(wpr.x, vpc.y, av.y);
          if (in) rowp[c] = av;
          av.x = in ? av.x : 0.0;
          av.y = in ? av.y : 0.0;
        }
        const cplx vc = vcur[cc];
        sr = fma(av.x, vc.x, fma(-av.y, vc.y, sr));
        si = fma(av.x, vc.y, fma(av.y, vc.x, si));
        // (r, c) also stands for A[c][r] = conj(a): p[c] += conj(a) v_r (strictly below the diagonal)
        const double wx = c < r ? vr.x : 0.0, wy = c < r ? vr.y : 0.0;
        cacc[q].x = fma(av.x, wx, fma(av.y, wy, cacc[q].x));
        cacc[q].y = fma(av.x, wy, fma(-av.y, wx, cacc[q].y));
      }
    };
    if constexpr (NQ <= 6) {
      // R rows per reduction (4 for n <= 128, 2 for n <= 192, as registers allow): their 2R
      // lane-partials (re, im) are summed over the warp by a transposing butterfly (2R + 1
      // shuffles instead of 5 per value), and the rows' loads are not held back by a
      // reduction after every row
      constexpr int R = NQ <= 4 ? 4 : 2;
      for (int rb = j + 1 + warp; rb < n; rb += R * HEEV_WARPS) {
        double v[2 * R];
#pragma unroll
        for (int u = 0; u < R; ++u) {
          const int r = rb + u * HEEV_WARPS;
          double sr = 0.0, si = 0.0;
          if (r < n) row_partial(r, sr, si);
          v[2 * u] = sr;
          v[2 * u + 1] = si;
        }
        // halve the value count per round: lanes with the round's bit set keep the upper half
        int idx = 0;
#pragma unroll
        for (int half = R, bit = 16; half >= 1; half >>= 1, bit >>= 1) {
          const bool hi = lane & bit;
#pragma unroll
          for (int i = 0; i < half; ++i) {
            const double send = hi ? v[i] : v[i + half];
            const double keep = hi ? v[i + half] : v[i];
            v[i] = keep + __shfl_xor_sync(0xffffffffu, send, bit);
          }
          idx = 2 * idx + (hi ? 1 : 0);
        }
        // one value left per lane; sum it over the remaining low lane bits
        constexpr int LOWB = 32 >> (R == 4 ? 3 : 2);   // lanes sharing a value: 4 (R=4) or 8 (R=2)
#pragma unroll
        for (int o = LOWB >> 1; o >= 1; o >>= 1) v[0] += __shfl_xor_sync(0xffffffffu, v[0], o);
        if ((lane & (LOWB - 1)) == 0) {   // value idx = 2 u + component
          const int r = rb + (idx >> 1) * HEEV_WARPS;
          if (r < n) {
            if (idx & 1) prow[r].y = v[0];
            else prow[r].x = v[0];
          }
        }
      }
    } else {
      for (int r = j + 1 + warp; r < n; r += HEEV_WARPS) {
        double sr = 0.0, si = 0.0;
        row_partial(r, sr, si);
        sr = warp_sum(sr);
        si = warp_sum(si);
        if (lane == 0) prow[r] = make_double2(sr, si);
      }
    }
#pragma unroll
    for (int q = 0; q < NQ; ++q) {
      const int c = j + 1 + lane + 32 * q;
      if (c < n) colpart[warp * n + c] = cacc[q];
    }
    __syncthreads();
    // (d) w = p + alpha2 v with p = tau (A v), alpha2 = -1/2 tau (p^H v)
    double dr = 0.0, di = 0.0;
    for (int r = j + 1 + tid; r < n; r += HEEV_THREADS) {
      cplx s = prow[r];
      for (int w = 0; w < HEEV_WARPS; ++w) {
        s.x += colpart[w * n + r].x;
        s.y += colpart[w * n + r].y;
      }
      const cplx p = make_double2(tau.x * s.x - tau.y * s.y, tau.x * s.y + tau.y * s.x);
      wcur[r] = p;
      const cplx v = vcur[r];
      dr += p.x * v.x + p.y * v.y;
      di += p.x * v.y - p.y * v.x;
    }
    const double2 dot = block_sum2_1b(dr, di, red, 1);
    const cplx a2 = make_double2(-0.5 * (tau.x * dot.x - tau.y * dot.y), -0.5 * (tau.x * dot.y + tau.y * dot.x));
    // same row ownership as the loop above and as the next step's (a): no barrier needed here
    // (the next step reads other rows' vprev / wprev only after its reduction barriers)
    for (int r = j + 1 + tid; r < n; r += HEEV_THREADS) {
      const cplx v = vcur[r], p = wcur[r];
      vprev[r] = v;
      wprev[r] = make_double2(p.x + a2.x * v.x - a2.y * v.y, p.y + a2.x * v.y + a2.y * v.x);
    }
    a2_prev = a2;
    have_prev = tnz;
  }
  __syncthreads();
  if (tid == 0) {
    cplx a = LL(n - 1, n - 1);
    if (have_prev) {
      const cplx v = vprev[n - 1], w = wprev[n - 1];
      a.x -= 2.0 * (v.x * w.x + v.y * w.y);
    }
    dvec[n - 1] = a.x;
    evec[n - 1] = 0.0;
  }
  __syncthreads();
#undef LL
}
// zhetd2 (lower) on full storage kept Hermitian: two passes per step (mat-vec, rank-2 update).
// Used for n > 256.  Reflector j goes to row j (columns > j).
__device__ void tridiag_full(cplx* __restrict__ A, const int n, cplx* sv, cplx* sp, double* dvec, double* evec,
                             cplx* tau_out, double2* red) {
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  for (int j = 0; j < n - 1; ++j) {
    const int len = n - j - 1;
    const cplx* col = A + (size_t)(j + 1) * n + j;
    double part = 0.0;
    for (int i = 1 + tid; i < len; i += HEEV_THREADS) {
      cplx x = col[(size_t)i * n];
      part += x.x * x.x + x.y * x.y;
    }
    const double xn2 = block_sum2(part, 0.0, red).x;
    const cplx alpha = col[0];
    double beta;
    cplx tau, scale;
    if (xn2 == 0.0 && alpha.y == 0.0) {
      beta = alpha.x;
      tau = make_double2(0.0, 0.0);
      scale = make_double2(0.0, 0.0);
    } else {
      beta = -copysign(sqrt(alpha.x * alpha.x + alpha.y * alpha.y + xn2), alpha.x);
      tau = make_double2((beta - alpha.x) / beta, -alpha.y / beta);
      const cplx den = make_double2(alpha.x - beta, alpha.y);
      const double dd = den.x * den.x + den.y * den.y;
      scale = make_double2(den.x / dd, -den.y / dd);
    }
    for (int i = tid; i < len; i += HEEV_THREADS) {
      cplx v;
      if (i == 0) v = make_double2(1.0, 0.0);
      else {
        cplx x = col[(size_t)i * n];
        v = make_double2(x.x * scale.x - x.y * scale.y, x.x * scale.y + x.y * scale.x);
      }
      sv[i] = v;
      A[(size_t)j * n + j + 1 + i] = v;
    }
    if (tid == 0) {
      evec[j] = beta;
      dvec[j] = A[(size_t)j * n + j].x;
      tau_out[j] = tau;
    }
    __syncthreads();
    if (tau.x == 0.0 && tau.y == 0.0) continue;
    cplx* A22 = A + (size_t)(j + 1) * n + (j + 1);
    for (int r = warp; r < len; r += HEEV_WARPS) {
      const cplx* row = A22 + (size_t)r * n;
      double sr = 0.0, si = 0.0;
      for (int c = lane; c < len; c += 32) {
        cplx a = row[c], v = sv[c];
        sr += a.x * v.x - a.y * v.y;
        si += a.x * v.y + a.y * v.x;
      }
      sr = warp_sum(sr);
      si = warp_sum(si);
      if (lane == 0) sp[r] = make_double2(tau.x * sr - tau.y * si, tau.x * si + tau.y * sr);
    }
    __syncthreads();
    double dr = 0.0, di = 0.0;
    for (int r = tid; r < len; r += HEEV_THREADS) {
      cplx p = sp[r], v = sv[r];
      dr += p.x * v.x + p.y * v.y;
      di += p.x * v.y - p.y * v.x;
    }
    const double2 dot = block_sum2(dr, di, red);
    const cplx a2 = make_double2(-0.5 * (tau.x * dot.x - tau.y * dot.y), -0.5 * (tau.x * dot.y + tau.y * dot.x));
    for (int r = tid; r < len; r += HEEV_THREADS) {
      cplx v = sv[r], p = sp[r];
      sp[r] = make_double2(p.x + a2.x * v.x - a2.y * v.y, p.y + a2.x * v.y + a2.y * v.x);
    }
    __syncthreads();
    for (int r = warp; r < len; r += HEEV_WARPS) {
      const cplx vr = sv[r], wr = sp[r];
      cplx* row = A22 + (size_t)r * n;
      for (int c = lane; c < len; c += 32) {
        const cplx vc = sv[c], wc = sp[c];
        cplx a = row[c];
        a.x -= (vr.x * wc.x + vr.y * wc.y) + (wr.x * vc.x + wr.y * vc.y);
        a.y -= (vr.y * wc.x - vr.x * wc.y) + (wr.y * vc.x - wr.x * vc.y);
        row[c] = a;
      }
    }
    __syncthreads();
  }
  if (tid == 0) {
    dvec[n - 1] = A[(size_t)(n - 1) * n + (n - 1)].x;
    evec[n - 1] = 0.0;
  }
  __syncthreads();
}

// Gershgorin interval, pivmin (dstebz) and the trace, from d / e in P.work (one CTA)
__device__ void tridiag_stats(const HeevProblem& P, double trace) {
  const int n = P.n, tid = threadIdx.x, lane = tid & 31, warp = tid >> 5, nw = blockDim.x >> 5;
  const double* dvec = P.work;
  const double* evec = P.work + n;
  double* sc = P.work + 2 * n;
  double gl = 1e300, gu = -1e300, em = 0.0;
  for (int i = tid; i < n; i += blockDim.x) {
    const double di = dvec[i], ei = (i < n - 1) ? evec[i] : 0.0, ep = (i > 0) ? evec[i - 1] : 0.0;
    const double rad = fabs(ei) + fabs(ep);
    gl = fmin(gl, di - rad);
    gu = fmax(gu, di + rad);
    em = fmax(em, ei * ei);
  }
  for (int o = 16; o > 0; o >>= 1) {
    gl = fmin(gl, __shfl_xor_sync(0xffffffffu, gl, o));
    gu = fmax(gu, __shfl_xor_sync(0xffffffffu, gu, o));
    em = fmax(em, __shfl_xor_sync(0xffffffffu, em, o));
  }
  __shared__ double mm[3][32];
  if (lane == 0) { mm[0][warp] = gl; mm[1][warp] = gu; mm[2][warp] = em; }
  __syncthreads();
  if (tid == 0) {
    gl = mm[0][0]; gu = mm[1][0]; em = mm[2][0];
    for (int w = 1; w < nw; ++w) { gl = fmin(gl, mm[0][w]); gu = fmax(gu, mm[1][w]); em = fmax(em, mm[2][w]); }
    const double tnorm = fmax(fabs(gl), fabs(gu));
    const double pivmin = DBL_MIN * fmax(1.0, em);
    sc[S_GL] = gl - 2.0 * DBL_EPSILON * tnorm * n - 2.0 * pivmin;
    sc[S_GU] = gu + 2.0 * DBL_EPSILON * tnorm * n + 2.0 * pivmin;
    sc[S_TNORM] = tnorm;
    sc[S_PIVMIN] = pivmin;
    sc[S_TRACE] = trace;
    sc[S_ATOL] = 4.0 * DBL_EPSILON * tnorm;
  }
}


// ---------------------------------------------------------------- K0: tiny Grams (n <= 12)
// "n <= 64: batched cyclic Jacobi per CTA in shared memory".  One warp per
// Gram (lane = row), the Hermitian matrix and the eigenvector matrix in shared memory (odd
// row stride: conflict-free column access), parallel cyclic Jacobi with the round-robin
// ordering (n/2 disjoint rotations per round, each a complex 2 x 2 Schur rotation
// U = diag(1, e^{-i phi}) R(c, s)), until the off-diagonal mass is <= (1e-16)^2 ||A||_F^2.
// Then the descending sort, the truncation decision of heev_finish (k, discarded weight,
// dropped rows zeroed), the pow2 unscale and the exact-factor skip -- the whole K1..K7
// pipeline of a small Gram in ONE launch (latency-bound trees: configs 1, 5).
constexpr int JAC_MAX_N = 32;    // the kernel's limit
// routing limit: measured slower than the tridiagonal pipeline at every order (a warp-serial
// round costs ~1 us, 5-8 sweeps of n - 1 rounds: ~85 us for n = 12 against the pipeline's
// ~35 us; ~64 n^3 flops against ~(4/3) n^3), so it is off by default; TTN_JACOBI_MAX_N = m
// routes Grams of order <= m (<= 32) to it for measurement
inline int jac_route_n() {
  static const int v = getenv("TTN_JACOBI_MAX_N") ? std::min(atoi(getenv("TTN_JACOBI_MAX_N")), JAC_MAX_N) : 0;
  return v;
}
constexpr int JAC_WARPS = 4;
__host__ __device__ inline int jac_ld(int n) { return n | 1; }
// per warp: A and V (n x LD complex), then per pair c, s, Re / Im e^{-i phi} (4 doubles) and
// p, q (2 ints), then the sort keys (doubles) and the permutation (ints)
__host__ __device__ inline size_t jac_warp_bytes(int n) {
  return (size_t)2 * n * jac_ld(n) * 16 + (size_t)(JAC_MAX_N / 2) * (4 * 8 + 2 * 4) + (size_t)JAC_MAX_N * (8 + 4) + 64;
}

__global__ void __launch_bounds__(JAC_WARPS * 32) heev_jacobi(const HeevProblem* __restrict__ probs, int nprob,
                                                              int nmax) {
  TCBC_PDL_WAIT();
  extern __shared__ __align__(16) unsigned char smem_raw[];
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int pi = blockIdx.x * JAC_WARPS + warp;
  if (pi >= nprob) return;   // whole warp
  const HeevProblem P = probs[pi];
  const int n = P.n, kmax = P.kmax, LD = jac_ld(n);
  if (P.skip && *P.skip) {   // exact-factor shortcut
    if (lane == 0) {
      if (P.k_out) *P.k_out = kmax;
      if (P.w_out) *P.w_out = 0.0;
    }
    return;
  }
  unsigned char* base = smem_raw + (size_t)warp * jac_warp_bytes(nmax);
  cplx* A = reinterpret_cast<cplx*>(base);
  cplx* V = A + (size_t)n * LD;
  double* rc = reinterpret_cast<double*>(V + (size_t)n * LD);   // per pair: c, s (real), and e^{-i phi}
  double* rer = rc + JAC_MAX_N / 2 * 2;
  double* rei = rer + JAC_MAX_N / 2;
  int* rp = reinterpret_cast<int*>(rei + JAC_MAX_N / 2);
  int* rq = rp + JAC_MAX_N / 2;
  double* dsort = reinterpret_cast<double*>(rq + JAC_MAX_N / 2);
  int* perm = reinterpret_cast<int*>(dsort + JAC_MAX_N);
  double fro = 0.0, tr = 0.0;
  for (int e = lane; e < n * n; e += 32) {
    const int i = e / n, j = e - i * n;
    const cplx a = P.A[e];
    A[i * LD + j] = a;
    V[i * LD + j] = make_double2(i == j ? 1.0 : 0.0, 0.0);
    fro += a.x * a.x + a.y * a.y;
    if (i == j) tr += a.x;
  }
  fro = warp_sum(fro);
  tr = warp_sum(tr);
  const double afro = sqrt(fro);
  __syncwarp();
  const int m = n + (n & 1), t = m - 1, np = m / 2;
  for (int sweep = 0; sweep < 40 && n > 1; ++sweep) {
    double off = 0.0;
    for (int e = lane; e < n * n; e += 32) {
      const int i = e / n, j = e - i * n;
      if (i != j) {
        const cplx a = A[i * LD + j];
        off += a.x * a.x + a.y * a.y;
      }
    }
    off = warp_sum(off);
    // off-diagonal mass at the rounding level of the rotations (1e-14 ||A||_F): the eigenvector
    // error is then ~1e-14 ||A|| / gap, far inside the parity budget; rotations below it only
    // reshuffle rounding noise between (near-)zero eigenvalues and never converge further
    if (!(off > 1e-28 * fro)) break;
    for (int r = 0; r < t; ++r) {
      if (lane < np) {
        int p, q;
        if (lane == 0) {
          p = 0;
          q = 1 + r % t;
        } else {
          p = 1 + (r + lane) % t;
          q = 1 + (r - lane + t) % t;
        }
        double c = 1.0, s = 0.0, er = 1.0, ei = 0.0;
        if (p < n && q < n) {
          const cplx apq = A[p * LD + q];
          const double ar = hypot(apq.x, apq.y);
          const double dp = A[p * LD + p].x, dq = A[q * LD + q].x;
          // negligible: below the rounding of the diagonal pair (classical Jacobi skip test)
          if (ar > 1e-17 * sqrt(fabs(dp * dq)) && ar > 1e-16 * afro && ar > 1e-300) {
            const double zeta = (dq - dp) / (2.0 * ar);
            const double tt = (zeta >= 0.0 ? 1.0 : -1.0) / (fabs(zeta) + sqrt(1.0 + zeta * zeta));
            c = 1.0 / sqrt(1.0 + tt * tt);
            s = tt * c;
            er = apq.x / ar;    // e^{-i phi} = conj(apq) / |apq|
            ei = -apq.y / ar;
          }
        }
        rp[lane] = p;
        rq[lane] = q;
        rc[2 * lane] = c;
        rc[2 * lane + 1] = s;
        rer[lane] = er;
        rei[lane] = ei;
      }
      __syncwarp();
      // columns (A U) and the eigenvectors (V U): lane = row
      for (int i = lane; i < n; i += 32)
        for (int k = 0; k < np; ++k) {
          const int p = rp[k], q = rq[k];
          if (p >= n || q >= n) continue;
          const double c = rc[2 * k], s = rc[2 * k + 1], er = rer[k], ei = rei[k];
          for (int w = 0; w < 2; ++w) {
            cplx* M = w ? V : A;
            const cplx x = M[i * LD + p], y = M[i * LD + q];
            const cplx ey = make_double2(er * y.x - ei * y.y, er * y.y + ei * y.x);   // e^{-i phi} y
            M[i * LD + p] = make_double2(c * x.x - s * ey.x, c * x.y - s * ey.y);
            M[i * LD + q] = make_double2(s * x.x + c * ey.x, s * x.y + c * ey.y);
          }
        }
      __syncwarp();
      // rows (U^H A): lane = column
      for (int j = lane; j < n; j += 32)
        for (int k = 0; k < np; ++k) {
          const int p = rp[k], q = rq[k];
          if (p >= n || q >= n) continue;
          const double c = rc[2 * k], s = rc[2 * k + 1], er = rer[k], ei = -rei[k];   // e^{+i phi}
          const cplx x = A[p * LD + j], y = A[q * LD + j];
          const cplx ey = make_double2(er * y.x - ei * y.y, er * y.y + ei * y.x);
          A[p * LD + j] = make_double2(c * x.x - s * ey.x, c * x.y - s * ey.y);
          A[q * LD + j] = make_double2(s * x.x + c * ey.x, s * x.y + c * ey.y);
        }
      __syncwarp();
    }
  }
  // descending order (ties by index)
  for (int i = lane; i < n; i += 32) dsort[i] = A[i * LD + i].x;
  __syncwarp();
  for (int i = lane; i < n; i += 32) {
    const double di = dsort[i];
    int rk = 0;
    for (int j = 0; j < n; ++j) rk += (dsort[j] > di || (dsort[j] == di && j < i)) ? 1 : 0;
    perm[rk] = i;
  }
  __syncwarp();
  // truncation decision (heev_finish semantics)
  const double l1 = dsort[perm[0]];
  int k = 1;
  double kept = 0.0;
  const bool zero = !(tr > 0.0 && l1 > 0.0);
  if (!zero) {
    int cnt = 0;
    for (int u = 0; u < kmax; ++u) {
      const double lu = dsort[perm[u]];
      if (lu > P.tol2 * l1 && lu > P.floor_rel * l1) ++cnt;
    }
    k = cnt < 1 ? 1 : (cnt > P.max_bond ? P.max_bond : cnt);
    for (int u = 0; u < k; ++u) kept += dsort[perm[u]];
  }
  const int e2 = P.exp2 ? pow2_effective(*P.exp2) : 0;
  for (int u = lane; u < kmax; u += 32) P.lam[u] = (!zero && u < k) ? ldexp(dsort[perm[u]], 2 * e2) : 0.0;
  for (int e = lane; e < kmax * n; e += 32) {
    const int u = e / n, i = e - u * n;
    P.Vt[e] = (zero || u < k) ? V[i * LD + perm[u]] : make_double2(0.0, 0.0);
  }
  if (lane == 0) {
    if (P.k_out) *P.k_out = k;
    if (P.w_out) *P.w_out = ldexp(fmax(tr - kept, 0.0), 2 * e2);
  }
}

// ---------------------------------------------------------------- K1: tridiagonalisation
template <int NQ>
__global__ void __launch_bounds__(HEEV_THREADS, NQ == 4 ? 3 : 2) heev_tridiag(const HeevProblem* __restrict__ probs) {
  TCBC_PDL_WAIT();
  const HeevProblem P = probs[blockIdx.x];
  if (P.skip && *P.skip) return;   // exact-factor shortcut (chol_certify)
  const int n = P.n;
  cplx* A = P.A;
  const int tid = threadIdx.x;
  extern __shared__ __align__(16) unsigned char smem_raw[];
  cplx* sv = reinterpret_cast<cplx*>(smem_raw);
  cplx* sp = sv + n;
  cplx* base = sp + n;
  __shared__ double2 red[2 * HEEV_WARPS + 1];
  double* dvec = P.work;
  double* evec = P.work + n;
  double tr = 0.0;
  for (int i = tid; i < n; i += HEEV_THREADS) tr += A[(size_t)i * n + i].x;
  const double trace = block_sum2(tr, 0.0, red).x;
  if constexpr (NQ == 8) {   // the launcher sends n > 192 only to this instantiation
    if (n <= 32 * NQ) tridiag_fused<NQ>(A, n, fused_r0(n), sv, sp, base, dvec, evec, P.tau, red);
    else tridiag_full(A, n, sv, sp, dvec, evec, P.tau, red);
  } else {
    tridiag_fused<NQ>(A, n, fused_r0(n), sv, sp, base, dvec, evec, P.tau, red);
  }
  tridiag_stats(P, trace);
}

// K1 on a thread-block cluster of CS CTAs (levels with few Grams: chains, config 4's 4-chain
// levels).  The full Hermitian matrix is distributed by row blocks over the CTAs' shared
// memory (DSMEM), so one matrix uses CS SMs and never touches L2 after the initial load.
// Per Householder step two cluster barriers:
//   A  every CTA broadcasts its rows' entries of column j (and a partial |x|^2) to all CTAs;
//      then each CTA forms the reflector (zlarfg) redundantly;
//   B  every CTA computes p = tau A v on its rows and broadcasts p (and a partial p^H v);
//      then each CTA forms w = p - tau/2 (p^H v) v and applies A -= v w^H + w v^H to its rows.
// Same outputs as heev_tridiag (d, e, tau, reflectors in rows of A, stats).
constexpr int CL_THREADS = 256;
constexpr size_t CL_SMEM_LIMIT = 200u << 10;

__host__ __device__ inline size_t cl_smem_bytes(int n, int cs) {
  const int rpc = (n + cs - 1) / cs;
  return (size_t)rpc * n * 16 + (size_t)3 * n * 16 + (size_t)2 * 16 * 16 + 64;
}

template <int CS>
__global__ void __launch_bounds__(CL_THREADS) heev_tridiag_cluster(const HeevProblem* __restrict__ probs) {
  TCBC_PDL_WAIT();
  namespace cg = cooperative_groups;
  cg::cluster_group cl = cg::this_cluster();
  const int rank = (int)cl.block_rank();
  const HeevProblem P = probs[blockIdx.x / CS];
  if (P.skip && *P.skip) return;   // uniform over the cluster
  const int n = P.n, rpc = (n + CS - 1) / CS, r0 = rank * rpc, r1 = min(n, r0 + rpc);
  cplx* A = P.A;
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  constexpr int NW = CL_THREADS / 32;
  extern __shared__ __align__(16) unsigned char smem_raw[];
  cplx* rows = reinterpret_cast<cplx*>(smem_raw);   // [rpc][n]
  cplx* x = rows + (size_t)rpc * n;                  // column j, broadcast     [n]
  cplx* pv = x + n;                                  // p = tau A v, broadcast   [n]
  cplx* vw = pv + n;                                 // v then w (local)        [n]
  double2* partN = reinterpret_cast<double2*>(vw + n);   // [16]
  double2* partD = partN + 16;                            // [16]
  __shared__ double2 red[2 * NW + 1];
  static_assert(NW == HEEV_WARPS, "one-barrier reductions assume HEEV_WARPS warps");
  __shared__ cplx s_v[1];
  double* dvec = P.work;
  double* evec = P.work + n;
  for (long long e = tid; e < (long long)(r1 - r0) * n; e += CL_THREADS) rows[e] = A[(size_t)r0 * n + e];
  double trace = 0.0;
  if (rank == 0) {
    double tr = 0.0;
    for (int i = tid; i < n; i += CL_THREADS) tr += A[(size_t)i * n + i].x;
    trace = block_sum2(tr, 0.0, red).x;
  }
  cl.sync();   // every CTA has its rows before any reflector is written back to A
  for (int j = 0; j < n - 1; ++j) {
    // ---- A: broadcast column j (rows > j) and partial norms
    const int ia = max(r0, j + 1);
    double pn = 0.0;
    for (int i = ia + tid; i < r1; i += CL_THREADS) {
      const cplx xi = rows[(size_t)(i - r0) * n + j];
      if (i >= j + 2) pn += xi.x * xi.x + xi.y * xi.y;
#pragma unroll
      for (int d = 0; d < CS; ++d) *cl.map_shared_rank(x + i, d) = xi;
    }
    if (j >= r0 && j < r1 && tid == 0) dvec[j] = rows[(size_t)(j - r0) * n + j].x;
    pn = block_sum2_1b(pn, 0.0, red, 0).x;
    if (tid < CS) *cl.map_shared_rank(partN + rank, tid) = make_double2(pn, 0.0);
    cl.sync();
    double xn2 = 0.0;
#pragma unroll
    for (int d = 0; d < CS; ++d) xn2 += partN[d].x;
    const cplx alpha = x[j + 1];
    double beta;
    cplx tau, scale;
    if (xn2 == 0.0 && alpha.y == 0.0) {
      beta = alpha.x;
      tau = make_double2(0.0, 0.0);
      scale = make_double2(0.0, 0.0);
    } else {
      beta = -copysign(sqrt(alpha.x * alpha.x + alpha.y * alpha.y + xn2), alpha.x);
      tau = make_double2((beta - alpha.x) / beta, -alpha.y / beta);
      const cplx den = make_double2(alpha.x - beta, alpha.y);
      const double dd = den.x * den.x + den.y * den.y;
      scale = make_double2(den.x / dd, -den.y / dd);
    }
    const bool tnz = (tau.x != 0.0 || tau.y != 0.0);
    for (int i = j + 1 + tid; i < n; i += CL_THREADS) {
      cplx v;
      if (i == j + 1) v = make_double2(1.0, 0.0);
      else {
        const cplx xi = x[i];
        v = make_double2(xi.x * scale.x - xi.y * scale.y, xi.x * scale.y + xi.y * scale.x);
      }
      if (rank == 0) A[(size_t)j * n + i] = v;   // kept for the back-transform
      vw[i] = tnz ? v : make_double2(0.0, 0.0);
    }
    if (rank == 0 && tid == 0) {
      evec[j] = beta;
      P.tau[j] = tau;
    }
    if (!tnz) {   // H_j = I: nothing to apply; keep the barrier pattern (x is reused next step)
      cl.sync();
      continue;
    }
    __syncthreads();
    // ---- B: p = tau A v on my rows (warp per row), broadcast p and partial p^H v
    double dr = 0.0, di = 0.0;
    for (int i = ia + warp; i < r1; i += NW) {
      const cplx* row = rows + (size_t)(i - r0) * n;
      double sr = 0.0, si = 0.0;
      for (int c = j + 1 + lane; c < n; c += 32) {
        const cplx a = row[c], v = vw[c];
        sr += a.x * v.x - a.y * v.y;
        si += a.x * v.y + a.y * v.x;
      }
      sr = warp_sum(sr);
      si = warp_sum(si);
      const cplx p = make_double2(tau.x * sr - tau.y * si, tau.x * si + tau.y * sr);
      for (int d = lane; d < CS; d += 32) *cl.map_shared_rank(pv + i, d) = p;
      const cplx v = vw[i];
      dr += p.x * v.x + p.y * v.y;
      di += p.x * v.y - p.y * v.x;
    }
    // dr/di were accumulated by lane-identical copies: keep lane 0's
    dr = __shfl_sync(0xffffffffu, dr, 0);
    di = __shfl_sync(0xffffffffu, di, 0);
    if (lane != 0) { dr = 0.0; di = 0.0; }
    const double2 dl = block_sum2_1b(dr, di, red, 1);
    if (tid < CS) *cl.map_shared_rank(partD + rank, tid) = dl;
    cl.sync();
    double2 dot = make_double2(0.0, 0.0);
#pragma unroll
    for (int d = 0; d < CS; ++d) { dot.x += partD[d].x; dot.y += partD[d].y; }
    const cplx a2 = make_double2(-0.5 * (tau.x * dot.x - tau.y * dot.y), -0.5 * (tau.x * dot.y + tau.y * dot.x));
    // w = p + a2 v (in place of v: keep v in registers of the update loop)
    // ---- C: A -= v w^H + w v^H on my rows, columns > j
    for (int i = ia + warp; i < r1; i += NW) {
      cplx* row = rows + (size_t)(i - r0) * n;
      const cplx vr = vw[i], pr = pv[i];
      const cplx wr = make_double2(pr.x + a2.x * vr.x - a2.y * vr.y, pr.y + a2.x * vr.y + a2.y * vr.x);
      for (int c = j + 1 + lane; c < n; c += 32) {
        const cplx vc = vw[c], pc = pv[c];
        const cplx wc = make_double2(pc.x + a2.x * vc.x - a2.y * vc.y, pc.y + a2.x * vc.y + a2.y * vc.x);
        cplx a = row[c];
        a.x -= (vr.x * wc.x + vr.y * wc.y) + (wr.x * vc.x + wr.y * vc.y);
        a.y -= (vr.y * wc.x - vr.x * wc.y) + (wr.y * vc.x - wr.x * vc.y);
        row[c] = a;
      }
    }
    __syncthreads();
  }
  if (n - 1 >= r0 && n - 1 < r1 && tid == 0) dvec[n - 1] = rows[(size_t)(n - 1 - r0) * n + (n - 1)].x;
  if (rank == 0 && tid == 0) evec[n - 1] = 0.0;
  (void)s_v;
  __threadfence();
  cl.sync();
  if (rank == 0) tridiag_stats(P, trace);
}

// ---------------------------------------------------------------- K2: eigenvalues
// 1/b from the SFU seed and two Newton steps (~1 ulp; |b| >= pivmin > 0 here).  The Sturm
// recurrence is bound by its FP64 divisions; the count is insensitive to ulp-level pivot
// errors (an O(eps ||T||) perturbation of T, below the bisection tolerance atol = 4 eps ||T||).
__device__ __forceinline__ double frcp(double b) {
  double r;
  asm("rcp.approx.ftz.f64 %0, %1;" : "=d"(r) : "d"(b));
  r = r * fma(-b, r, 2.0);
  r = r * fma(-b, r, 2.0);
  return r;
}

// G lanes per (matrix, eigenvalue): multisection.  Each lane evaluates Sturm counts at two of
// the 2G interior points of [lo, hi] (two interleaved chains hide the division latency); the
// interval shrinks (2G+1)x per round.  Counts are exact integers, so the result is the same
// bracket bisection would converge to.  G trades rounds (latency) for Sturm evaluations
// (FP64 work): the launcher takes the smallest G that still fills the GPU (config 3's
// 16384-eigenvalue levels: G = 4, ~17 rounds of 8 points, instead of 9 rounds of 64).
template <int G>
__global__ void heev_bisect(const HeevProblem* __restrict__ probs, int nprob, int total) {
  TCBC_PDL_WAIT();
  const int lane = threadIdx.x & 31, sub = lane % G;
  const int g0 = (blockIdx.x * blockDim.x + threadIdx.x) / G;
  if ((blockIdx.x * blockDim.x + (threadIdx.x & ~31)) / G >= total) return;   // whole warp idle
  const int g = min(g0, total - 1);                 // tail lanes shadow the last eigenvalue
  const unsigned gmask = G == 32 ? 0xffffffffu : (((1u << G) - 1u) << (lane - sub));
  const HeevProblem& P = probs[find_estart(probs, nprob, g)];
  const int t = g - P.estart, n = P.n;
  const double* d = P.work;
  const double* e = P.work + n;
  const double* sc = P.work + 2 * n;
  const bool skipped = P.skip && *P.skip;       // still takes part in the warp's ballots
  const double pivmin = skipped ? 0.0 : sc[S_PIVMIN], atol = skipped ? 1.0 : sc[S_ATOL];
  const int idx = n - 1 - t;                   // ascending index of the t-th largest
  double lo = skipped ? 0.0 : sc[S_GL], hi = skipped ? 0.0 : sc[S_GU];
  for (int it = 0; it < 96; ++it) {
    const bool done = hi - lo <= fmax(atol, 2.0 * DBL_EPSILON * fmax(fabs(lo), fabs(hi))) + pivmin;
    if (__all_sync(0xffffffffu, done)) break;
    const double w = (hi - lo) / (2 * G + 1);
    const double x1 = lo + w * (2 * sub + 1), x2 = lo + w * (2 * sub + 2);
    int c1 = 0, c2 = 0;
    double q1 = d[0] - x1, q2 = d[0] - x2;
    if (q1 <= pivmin) { ++c1; q1 = fmin(q1, -pivmin); }
    if (q2 <= pivmin) { ++c2; q2 = fmin(q2, -pivmin); }
    for (int i = 1; i < n; ++i) {
      const double di = d[i], ep = e[i - 1], ei = ep * ep;
      q1 = di - x1 - ei * frcp(q1);
      q2 = di - x2 - ei * frcp(q2);
      if (q1 <= pivmin) { ++c1; q1 = fmin(q1, -pivmin); }
      if (q2 <= pivmin) { ++c2; q2 = fmin(q2, -pivmin); }
    }
    // the eigenvalue lies in the first sub-interval whose right end has count > idx
    const unsigned b1 = (__ballot_sync(0xffffffffu, c1 > idx) & gmask) >> (lane - sub);
    const unsigned b2 = (__ballot_sync(0xffffffffu, c2 > idx) & gmask) >> (lane - sub);
    // point index p = 2*sub + (0 | 1); first p with count > idx
    int pfirst = 2 * G;
    if (b1) pfirst = min(pfirst, 2 * (__ffs(b1) - 1));
    if (b2) pfirst = min(pfirst, 2 * (__ffs(b2) - 1) + 1);
    if (!done) {
      const double nlo = pfirst == 0 ? lo : lo + w * pfirst;
      const double nhi = pfirst == 2 * G ? hi : lo + w * (pfirst + 1);
      lo = nlo;
      hi = nhi;
    }
  }
  if (sub == 0 && g0 < total && !skipped) P.lam[t] = 0.5 * (lo + hi);
}

// ---------------------------------------------------------------- K3: inverse iteration
__global__ void heev_invit(const HeevProblem* __restrict__ probs, int nprob, int total) {
  TCBC_PDL_WAIT();
  const int g = blockIdx.x * blockDim.x + threadIdx.x;
  if (g >= total) return;
  const HeevProblem& P = probs[find_estart(probs, nprob, g)];
  if (P.skip && *P.skip) return;
  const int t = g - P.estart, n = P.n, kmax = P.kmax;
  const double* __restrict__ sd = P.work;
  const double* __restrict__ evec = P.work + n;
  const double* sc = P.work + 2 * n;
  double* __restrict__ Z = P.work + 2 * n + 8;
  const size_t NK = (size_t)n * kmax;
  double* __restrict__ DL = Z + NK;
  double* __restrict__ Dg = DL + NK;
  double* __restrict__ DU = Dg + NK;
  double* __restrict__ DU2 = DU + NK;
  double* __restrict__ PV = DU2 + NK;
  const double pert = DBL_EPSILON * sc[S_TNORM];
  const double lam = P.lam[t];
  const int k = P.k_out ? *P.k_out : kmax;
#define AT(arr, i) arr[(size_t)(i) * kmax + t]
  if (t >= k || !(sc[S_TNORM] > 0.0)) {   // dropped direction, or zero matrix: unit vector
    for (int i = 0; i < n; ++i) AT(Z, i) = (t < k && i == t) ? 1.0 : 0.0;
    return;
  }
  if (cluster_arrays(P)[kmax + t] > 1.0) return;   // member of a cluster: K3b
  double d_i = sd[0] - lam;
  double du_i = n > 1 ? evec[0] : 0.0;
  for (int i = 0; i < n - 1; ++i) {   // dgttrf on T - lam I, U diagonal perturbed away from 0
    const double dl = evec[i];
    double d_n = sd[i + 1] - lam;
    double du_n = (i < n - 2) ? evec[i + 1] : 0.0;
    double du2 = 0.0, l, p = 0.0;
    if (fabs(d_i) >= fabs(dl)) {
      if (fabs(d_i) < pert) d_i = copysign(pert, d_i == 0.0 ? 1.0 : d_i);
      l = dl / d_i;
      d_n -= l * du_i;
    } else {
      l = d_i / dl;
      const double old_du = du_i;
      d_i = dl;
      du_i = d_n;
      du2 = du_n;
      d_n = old_du - l * d_n;
      du_n = -l * du_n;
      p = 1.0;
    }
    if (fabs(d_i) < pert) d_i = copysign(pert, d_i == 0.0 ? 1.0 : d_i);
    AT(Dg, i) = 1.0 / d_i;
    AT(DU, i) = du_i;
    AT(DU2, i) = du2;
    AT(DL, i) = l;
    AT(PV, i) = p;
    d_i = d_n;
    du_i = du_n;
  }
  if (fabs(d_i) < pert) d_i = copysign(pert, d_i == 0.0 ? 1.0 : d_i);
  AT(Dg, n - 1) = 1.0 / d_i;
  for (int i = 0; i < n; ++i)
    AT(Z, i) = (double)(hash32((unsigned)(t * 7919 + i * 104729 + 12345)) & 0xffffff) / 16777216.0 - 0.5;
  double scale = 1.0;
  // Two sweeps: the eigenvalue is bisection-accurate (4 eps ||T||) and the vectors that reach
  // here are isolated (gap > 1e-5 ||T||; clusters go to K3b), so each sweep damps every other
  // eigencomponent by <= 4 eps ||T|| / gap < 1e-10: after two the error is at the rounding
  // level even from a start vector whose wanted component is 1e-6 of the others.
  for (int it = 0; it < 2; ++it) {   // dgttrs, rescaled by the previous max
    double cur = AT(Z, 0) * scale;
    for (int i = 0; i < n - 1; ++i) {
      const double nxt = AT(Z, i + 1) * scale;
      const double l = AT(DL, i);
      if (AT(PV, i) == 0.0) {
        AT(Z, i) = cur;
        cur = nxt - l * cur;
      } else {
        AT(Z, i) = nxt;
        cur = cur - l * nxt;
      }
    }
    double y2 = 0.0, y1 = cur * AT(Dg, n - 1);
    AT(Z, n - 1) = y1;
    double mx = fabs(y1);
    for (int i = n - 2; i >= 0; --i) {
      double yi = (AT(Z, i) - AT(DU, i) * y1 - AT(DU2, i) * y2) * AT(Dg, i);
      if (fabs(yi) > 1e100) {   // growth through near-zero pivots: rescale the solved part
        const double f = 1e-100;
        for (int q = i + 1; q < n; ++q) AT(Z, q) *= f;
        for (int q = 0; q < i; ++q) AT(Z, q) *= f;
        yi *= f;
        y1 *= f;
        y2 *= f;
        mx *= f;
      }
      AT(Z, i) = yi;
      mx = fmax(mx, fabs(yi));
      y2 = y1;
      y1 = yi;
    }
    scale = mx > 0.0 ? 1.0 / mx : 1.0;
  }
  double nr = 0.0;
  for (int i = 0; i < n; ++i) {
    const double v = AT(Z, i) * scale;
    nr += v * v;
  }
  const double s2 = scale / sqrt(fmax(nr, DBL_MIN));
  for (int i = 0; i < n; ++i) AT(Z, i) *= s2;
#undef AT
}

// K3a with the working arrays in shared memory: thread = eigenvector, arrays [6][n][NT]
// (consecutive threads in consecutive banks).  The inverse-iteration recurrences are
// sequential per vector; with the factors and the iterate on chip every step is a shared-memory
// access instead of an L2 round trip (the global-array version K3a stalls on L2 latency).
constexpr int INVIT_NT = 32;   // max vectors per block (fewer when 6 n NT doubles exceed the budget)
constexpr size_t INVIT_SMEM_MAX = 200u << 10;
constexpr size_t INVIT_SMEM_SHARED = 74u << 10;   // three blocks per SM when 8 vectors fit

__global__ void __launch_bounds__(INVIT_NT) heev_invit_smem(const HeevProblem* __restrict__ probs, int nprob,
                                                            int total, int nmax) {
  TCBC_PDL_WAIT();
  extern __shared__ __align__(16) unsigned char smem_raw[];
  double* sm = reinterpret_cast<double*>(smem_raw);
  const int tl = threadIdx.x, NT = blockDim.x;
  const int g = blockIdx.x * NT + tl;
  if (g >= total) return;
  const HeevProblem& P = probs[find_estart(probs, nprob, g)];
  if (P.skip && *P.skip) return;
  const int t = g - P.estart, n = P.n, kmax = P.kmax;
  const double* __restrict__ sd = P.work;
  const double* __restrict__ evec = P.work + n;
  const double* sc = P.work + 2 * n;
  double* __restrict__ Zg = P.work + 2 * n + 8;
  const double pert = DBL_EPSILON * sc[S_TNORM];
  const int k = P.k_out ? *P.k_out : kmax;
#define AR(a, i) sm[((size_t)(a) * nmax + (i)) * NT + tl]
  if (t >= k || !(sc[S_TNORM] > 0.0)) {   // dropped direction, or zero matrix: unit vector
    for (int i = 0; i < n; ++i) Zg[(size_t)i * kmax + t] = (t < k && i == t) ? 1.0 : 0.0;
    return;
  }
  if (cluster_arrays(P)[kmax + t] > 1.0) return;   // member of a cluster: K3b
  enum { DL = 0, DG, DU, DU2, PV, ZZ };
  const double lam = P.lam[t];
  double d_i = sd[0] - lam;
  double du_i = n > 1 ? evec[0] : 0.0;
  for (int i = 0; i < n - 1; ++i) {   // dgttrf on T - lam I, U diagonal perturbed away from 0
    const double dl = evec[i];
    double d_n = sd[i + 1] - lam;
    double du_n = (i < n - 2) ? evec[i + 1] : 0.0;
    double du2 = 0.0, l, p = 0.0;
    if (fabs(d_i) >= fabs(dl)) {
      if (fabs(d_i) < pert) d_i = copysign(pert, d_i == 0.0 ? 1.0 : d_i);
      l = dl / d_i;
      d_n -= l * du_i;
    } else {
      l = d_i / dl;
      const double old_du = du_i;
      d_i = dl;
      du_i = d_n;
      du2 = du_n;
      d_n = old_du - l * d_n;
      du_n = -l * du_n;
      p = 1.0;
    }
    if (fabs(d_i) < pert) d_i = copysign(pert, d_i == 0.0 ? 1.0 : d_i);
    AR(DG, i) = 1.0 / d_i;
    AR(DU, i) = du_i;
    AR(DU2, i) = du2;
    AR(DL, i) = l;
    AR(PV, i) = p;
    d_i = d_n;
    du_i = du_n;
  }
  if (fabs(d_i) < pert) d_i = copysign(pert, d_i == 0.0 ? 1.0 : d_i);
  AR(DG, n - 1) = 1.0 / d_i;
  for (int i = 0; i < n; ++i)
    AR(ZZ, i) = (double)(hash32((unsigned)(t * 7919 + i * 104729 + 12345)) & 0xffffff) / 16777216.0 - 0.5;
  double scale = 1.0;
  // Two sweeps: the eigenvalue is bisection-accurate (4 eps ||T||) and the vectors that reach
  // here are isolated (gap > 1e-5 ||T||; clusters go to K3b), so each sweep damps every other
  // eigencomponent by <= 4 eps ||T|| / gap < 1e-10: after two the error is at the rounding
  // level even from a start vector whose wanted component is 1e-6 of the others.
  for (int it = 0; it < 2; ++it) {   // dgttrs, rescaled by the previous max
    double cur = AR(ZZ, 0) * scale;
    for (int i = 0; i < n - 1; ++i) {
      const double nxt = AR(ZZ, i + 1) * scale;
      const double l = AR(DL, i);
      if (AR(PV, i) == 0.0) {
        AR(ZZ, i) = cur;
        cur = nxt - l * cur;
      } else {
        AR(ZZ, i) = nxt;
        cur = cur - l * nxt;
      }
    }
    double y2 = 0.0, y1 = cur * AR(DG, n - 1);
    AR(ZZ, n - 1) = y1;
    double mx = fabs(y1);
    for (int i = n - 2; i >= 0; --i) {
      double yi = (AR(ZZ, i) - AR(DU, i) * y1 - AR(DU2, i) * y2) * AR(DG, i);
      if (fabs(yi) > 1e100) {   // growth through near-zero pivots: rescale the solved part
        const double f = 1e-100;
        for (int q = i + 1; q < n; ++q) AR(ZZ, q) *= f;
        for (int q = 0; q < i; ++q) AR(ZZ, q) *= f;
        yi *= f;
        y1 *= f;
        y2 *= f;
        mx *= f;
      }
      AR(ZZ, i) = yi;
      mx = fmax(mx, fabs(yi));
      y2 = y1;
      y1 = yi;
    }
    scale = mx > 0.0 ? 1.0 / mx : 1.0;
  }
  double nr = 0.0;
  for (int i = 0; i < n; ++i) {
    const double v = AR(ZZ, i) * scale;
    nr += v * v;
  }
  const double s2 = scale / sqrt(fmax(nr, DBL_MIN));
  for (int i = 0; i < n; ++i) Zg[(size_t)i * kmax + t] = AR(ZZ, i) * s2;
#undef AR
}

// ---------------------------------------------------------------- K4: CholeskyQR2 of Z
__global__ void __launch_bounds__(HEEV_THREADS) heev_orth(const HeevProblem* __restrict__ probs) {
  TCBC_PDL_WAIT();
  const HeevProblem P = probs[blockIdx.x];
  if (P.skip && *P.skip) return;
  const int n = P.n, kmax = P.kmax, tid = threadIdx.x;
  const int k = P.k_out ? *P.k_out : kmax;   // only the kept directions are orthonormalised
  {   // isolated eigenvalues (gap > 1e-5 ||T||): inverse-iteration vectors are already orthogonal
      // to O(eps ||T|| / gap) <= 1e-11 and unit-norm; only clusters (MGS'd in K3b) get CholeskyQR2
    const double* csz = cluster_arrays(P) + kmax;
    bool any = false;
    for (int t = 0; t < k; ++t) any = any || csz[t] > 1.0;
    if (!any) return;
  }
  double* Z = P.work + 2 * n + 8;
  double* Wm = Z + (size_t)n * kmax * 6;
  for (int pass = 0; pass < 2; ++pass) {
    for (int e = tid; e < k * k; e += HEEV_THREADS) {
      const int s = e / k, t = e % k;
      if (t > s) continue;
      double acc = 0.0;
      for (int i = 0; i < n; ++i) acc += Z[(size_t)i * kmax + s] * Z[(size_t)i * kmax + t];
      Wm[(size_t)s * kmax + t] = acc;
    }
    __syncthreads();
    for (int j = 0; j < k; ++j) {   // W = L L^T in place (lower)
      if (tid == 0) Wm[(size_t)j * kmax + j] = sqrt(fmax(Wm[(size_t)j * kmax + j], 1e-300));
      __syncthreads();
      const double inv = 1.0 / Wm[(size_t)j * kmax + j];
      for (int i = j + 1 + tid; i < k; i += HEEV_THREADS) Wm[(size_t)i * kmax + j] *= inv;
      __syncthreads();
      const int m = k - j - 1;
      for (int e = tid; e < m * m; e += HEEV_THREADS) {
        const int i = j + 1 + e / m, l = j + 1 + e % m;
        if (l <= i) Wm[(size_t)i * kmax + l] -= Wm[(size_t)i * kmax + j] * Wm[(size_t)l * kmax + j];
      }
      __syncthreads();
    }
    for (int i = tid; i < n; i += HEEV_THREADS) {   // row_i <- row_i L^{-T}
      double* zr = Z + (size_t)i * kmax;
      for (int t = 0; t < k; ++t) {
        double v = zr[t];
        for (int s = 0; s < t; ++s) v -= Wm[(size_t)t * kmax + s] * zr[s];
        zr[t] = v / Wm[(size_t)t * kmax + t];
      }
    }
    __syncthreads();
  }
}

// K4 with everything in shared memory (kmax <= 128): Gram by 4x4 register tiles over 32-row
// chunks of Z, Cholesky of the Gram, L^{-1} into the Gram's upper triangle, Z <- Z L^{-T} by
// chunks (lane = row, warp = group of output columns).  Two passes (CholeskyQR2).
constexpr int ORTH_SMEM_K = 128;

__host__ __device__ inline size_t orth_smem_bytes(int kmax) {
  const int ld = kmax + 1;
  return ((size_t)kmax * ld + 2 * 32 * (size_t)ld + kmax) * sizeof(double);
}

__global__ void __launch_bounds__(HEEV_THREADS) heev_orth_smem(const HeevProblem* __restrict__ probs) {
  TCBC_PDL_WAIT();
  const HeevProblem P = probs[blockIdx.x];
  if (P.skip && *P.skip) return;
  const int n = P.n, kmax = P.kmax, tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int k = P.k_out ? *P.k_out : kmax;
  {
    const double* csz = cluster_arrays(P) + kmax;
    bool any = false;
    for (int t = 0; t < k; ++t) any = any || csz[t] > 1.0;
    if (!any) return;
  }
  double* Z = P.work + 2 * n + 8;   // n x kmax, ld kmax
  extern __shared__ __align__(16) unsigned char smem_raw[];
  const int ld = kmax + 1;
  double* W = reinterpret_cast<double*>(smem_raw);   // [k][ld]: lower = Gram / L, upper = L^{-1}^T
  double* Zc = W + (size_t)kmax * ld;                 // [32][ld]
  double* Zo = Zc + 32 * ld;                          // [32][ld]
  double* dinv = Zo + 32 * ld;                        // [k]
  const int kb = (k + 3) / 4, ntile = kb * (kb + 1) / 2;
  for (int pass = 0; pass < 2; ++pass) {
    // ---- Gram (lower), 4x4 tiles, up to 3 per thread
    double acc[3][4][4];
    int tb[3][2];
#pragma unroll
    for (int q = 0; q < 3; ++q) {
      const int e = tid + q * HEEV_THREADS;
      int bi = -1, bj = -1;
      if (e < ntile) {
        bi = (int)((sqrt(8.0 * e + 1.0) - 1.0) * 0.5);
        while (bi * (bi + 1) / 2 > e) --bi;
        while ((bi + 1) * (bi + 2) / 2 <= e) ++bi;
        bj = e - bi * (bi + 1) / 2;
      }
      tb[q][0] = bi;
      tb[q][1] = bj;
#pragma unroll
      for (int a = 0; a < 4; ++a)
#pragma unroll
        for (int b = 0; b < 4; ++b) acc[q][a][b] = 0.0;
    }
    for (int i0 = 0; i0 < n; i0 += 32) {
      const int rows = min(32, n - i0);
      for (int e = tid; e < 32 * k; e += HEEV_THREADS) {
        const int r = e / k, c = e % k;
        Zc[r * ld + c] = r < rows ? Z[(size_t)(i0 + r) * kmax + c] : 0.0;
      }
      __syncthreads();
#pragma unroll
      for (int q = 0; q < 3; ++q) {
        if (tb[q][0] < 0) continue;
        const int s0 = 4 * tb[q][0], t0 = 4 * tb[q][1];
        for (int r = 0; r < 32; ++r) {
          double zs[4], zt[4];
#pragma unroll
          for (int a = 0; a < 4; ++a) {
            zs[a] = (s0 + a < k) ? Zc[r * ld + s0 + a] : 0.0;
            zt[a] = (t0 + a < k) ? Zc[r * ld + t0 + a] : 0.0;
          }
#pragma unroll
          for (int a = 0; a < 4; ++a)
#pragma unroll
            for (int b = 0; b < 4; ++b) acc[q][a][b] += zs[a] * zt[b];
        }
      }
      __syncthreads();
    }
#pragma unroll
    for (int q = 0; q < 3; ++q) {
      if (tb[q][0] < 0) continue;
      const int s0 = 4 * tb[q][0], t0 = 4 * tb[q][1];
#pragma unroll
      for (int a = 0; a < 4; ++a)
#pragma unroll
        for (int b = 0; b < 4; ++b)
          if (s0 + a < k && t0 + b <= s0 + a) W[(s0 + a) * ld + t0 + b] = acc[q][a][b];
    }
    __syncthreads();
    // ---- Cholesky W = L L^T (lower, in place)
    for (int j = 0; j < k; ++j) {
      if (tid == 0) {
        const double djj = sqrt(fmax(W[j * ld + j], 1e-300));
        W[j * ld + j] = djj;
        dinv[j] = 1.0 / djj;
      }
      __syncthreads();
      const double inv = dinv[j];
      for (int i = j + 1 + tid; i < k; i += HEEV_THREADS) W[i * ld + j] *= inv;
      __syncthreads();
      const int m = k - j - 1;
      for (int e = tid; e < m * (m + 1) / 2; e += HEEV_THREADS) {
        int a = (int)((sqrt(8.0 * e + 1.0) - 1.0) * 0.5);
        while (a * (a + 1) / 2 > e) --a;
        while ((a + 1) * (a + 2) / 2 <= e) ++a;
        const int b = e - a * (a + 1) / 2;
        const int i = j + 1 + a, l = j + 1 + b;
        W[i * ld + l] -= W[i * ld + j] * W[l * ld + j];
      }
      __syncthreads();
    }
    // ---- L^{-1}: column c by thread c, stored transposed in the upper triangle (W[c][i] = Linv[i][c])
    for (int c = tid; c < k; c += HEEV_THREADS) {
      for (int i = c + 1; i < k; ++i) {
        double sacc = W[i * ld + c] * dinv[c];
        for (int j = c + 1; j < i; ++j) sacc += W[i * ld + j] * W[c * ld + j];
        W[c * ld + i] = -sacc * dinv[i];
      }
    }
    __syncthreads();
    // ---- Z <- Z L^{-T}:  z[t] = sum_{s <= t} z[s] Linv[t][s]
    const int tpw = (k + 7) / 8;
    const int t0 = warp * tpw;
    for (int i0 = 0; i0 < n; i0 += 32) {
      const int rows = min(32, n - i0);
      for (int e = tid; e < 32 * k; e += HEEV_THREADS) {
        const int r = e / k, c = e % k;
        Zc[r * ld + c] = r < rows ? Z[(size_t)(i0 + r) * kmax + c] : 0.0;
      }
      __syncthreads();
      double o[16];
#pragma unroll
      for (int q = 0; q < 16; ++q) o[q] = 0.0;
      const int tend = min(k, t0 + tpw);
      for (int s2 = 0; s2 < tend; ++s2) {
        const double z = Zc[lane * ld + s2];
#pragma unroll
        for (int q = 0; q < 16; ++q) {
          const int t = t0 + q;
          if (q < tpw && t < k && s2 <= t) o[q] += z * (s2 == t ? dinv[t] : W[s2 * ld + t]);
        }
      }
#pragma unroll
      for (int q = 0; q < 16; ++q)
        if (q < tpw && t0 + q < k) Zo[lane * ld + t0 + q] = o[q];
      __syncthreads();
      for (int e = tid; e < rows * k; e += HEEV_THREADS) {
        const int r = e / k, c = e % k;
        Z[(size_t)(i0 + r) * kmax + c] = Zo[r * ld + c];
      }
      __syncthreads();
    }
  }
}

// ---------------------------------------------------------------- K5: back-transform
__global__ void heev_backtr(const HeevProblem* __restrict__ probs, int nprob, int total) {
  TCBC_PDL_WAIT();
  const int gw = (blockIdx.x * blockDim.x + threadIdx.x) >> 5, lane = threadIdx.x & 31;
  if (gw >= total) return;
  const HeevProblem& P = probs[find_estart(probs, nprob, gw)];
  if (P.skip && *P.skip) return;
  const int t = gw - P.estart, n = P.n, kmax = P.kmax;
  const double* Z = P.work + 2 * n + 8;
  const cplx* A = P.A;
  cplx* vt = P.Vt + (size_t)t * n;
  const int k = P.k_out ? *P.k_out : kmax;
  for (int i = lane; i < n; i += 32) vt[i] = make_double2(t < k ? Z[(size_t)i * kmax + t] : 0.0, 0.0);
  if (t >= k) return;
  __syncwarp();
  for (int j = n - 2; j >= 0; --j) {
    const cplx tau = P.tau[j];
    if (tau.x == 0.0 && tau.y == 0.0) continue;
    const int len = n - j - 1;
    const cplx* v = A + (size_t)j * n + j + 1;
    cplx* yy = vt + j + 1;
    double sr = 0.0, si = 0.0;   // s = v^H y
    for (int i = lane; i < len; i += 32) {
      const cplx a = v[i], b = yy[i];
      sr += a.x * b.x + a.y * b.y;
      si += a.x * b.y - a.y * b.x;
    }
    sr = warp_sum(sr);
    si = warp_sum(si);
    const cplx ts = make_double2(tau.x * sr - tau.y * si, tau.x * si + tau.y * sr);
    for (int i = lane; i < len; i += 32) {
      const cplx a = v[i];
      cplx b = yy[i];
      b.x -= ts.x * a.x - ts.y * a.y;
      b.y -= ts.x * a.y + ts.y * a.x;
      yy[i] = b;
    }
    __syncwarp();
  }
}


// ---------------------------------------------------------------- K5 (blocked): WY back-transform
// V = Q Z with Q = H_0 ... H_{n-2} applied as blocks of WY_NB reflectors on the DMMA GEMM kernel
// (SURVEY §8 a6 "DMMA back-transform"): Q_b = I - Y_b T_b Y_b^H (compact WY, zlarft forward
// columnwise), Vt <- Vt - ((Vt conj(Y_b)) T_b^T) Y_b^T for b = last .. 0.  The reflectors are
// the rows of A (v_j in row j, columns j+1.., v_j[j+1] = 1): wy_prep zeroes the rest of each
// row so a block of rows IS Y_b^T, and starts Vt from the tridiagonal eigenvectors Z.
constexpr int WY_NB = 64;
constexpr int WY_MIN_N = 96;   // below: the register / shared-memory kernel (fewer launches)

__global__ void wy_prep(const HeevProblem* __restrict__ probs) {
  TCBC_PDL_WAIT();
  const HeevProblem P = probs[blockIdx.x];
  if (P.skip && *P.skip) return;
  const int n = P.n, kmax = P.kmax;
  const int k = P.k_out ? *P.k_out : kmax;
  const double* Z = P.work + 2 * n + 8;
  for (long long e = threadIdx.x; e < (long long)n * n; e += blockDim.x) {
    const int r = (int)(e / n), c = (int)(e - (long long)r * n);
    if (c <= r || r == n - 1) P.A[e] = make_double2(0.0, 0.0);
  }
  for (long long e = threadIdx.x; e < (long long)kmax * n; e += blockDim.x) {
    const int t = (int)(e / n), i = (int)(e - (long long)t * n);
    P.Vt[e] = make_double2(t < k ? Z[(size_t)i * kmax + t] : 0.0, 0.0);
  }
}

struct WyBlock {
  const cplx* G;      // C[c'][c] = sum_i Y[i][c']^* ... (GEMM of the block's rows), nbb x nbb
  cplx* T;            // nbb x nbb upper triangular, ld WY_NB
  const cplx* tau;    // tau of the block's first reflector
  const int* skip;
  int nbb;
  int pad_;
};

// one warp per block: T[c][c] = tau_c, T[r][c] = -tau_c sum_{r<=q<c} T[r][q] u_q,
// u_q = (Y^H Y)[q][c] = conj(G[q][c])
__global__ void wy_larft(const WyBlock* __restrict__ blks, int nb) {
  TCBC_PDL_WAIT();
  const int w = blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5), lane = threadIdx.x & 31;
  if (w >= nb) return;
  const WyBlock B = blks[w];
  if (B.skip && *B.skip) return;
  const int m = B.nbb;
  for (int c = 0; c < m; ++c) {
    const cplx tc = B.tau[c];
    for (int r = lane; r < m; r += 32) {
      cplx v = make_double2(0.0, 0.0);
      if (r < c) {
        double sr = 0.0, si = 0.0;
        for (int q = r; q < c; ++q) {
          const cplx t = B.T[r * WY_NB + q];
          const cplx g = B.G[q * m + c];          // u_q = conj(g)
          sr += t.x * g.x + t.y * g.y;
          si += t.y * g.x - t.x * g.y;
        }
        v = make_double2(-(tc.x * sr - tc.y * si), -(tc.x * si + tc.y * sr));
      } else if (r == c) {
        v = tc;
      }
      B.T[r * WY_NB + c] = v;
    }
    __syncwarp();
  }
}

// K7: eigenvalues and discarded weight back to the unscaled data (HeevProblem::exp2)
// what: 1 = the discarded weight (right after K6, so the host can read k and w early),
// 2 = the eigenvalues (after inverse iteration, which shifts by the scaled values)
__global__ void heev_unscale(const HeevProblem* __restrict__ probs, int nprob, int what) {
  TCBC_PDL_WAIT();
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= nprob) return;
  const HeevProblem& P = probs[i];
  if (!P.exp2 || (P.skip && *P.skip)) return;
  const int e = pow2_effective(*P.exp2);
  if (e == 0) return;
  if (what & 2)
    for (int t = 0; t < P.kmax; ++t) P.lam[t] = ldexp(P.lam[t], 2 * e);
  if ((what & 1) && P.w_out) *P.w_out = ldexp(*P.w_out, 2 * e);
}

// K5 for n <= 32 * NQ, one CTA per (matrix, 8 x VPW eigenvectors): a warp's VPW eigenvectors
// live in its registers (lane l owns entries l, l + 32, ...); the reflectors are staged BT_R
// rows at a time in shared memory by the whole CTA (one coalesced L2 pass shared by all its
// vectors), and each reflector entry read from shared memory serves VPW vectors.
constexpr int BT_WARPS = 8, BT_R = 16;
#ifndef BT_VPW
#define BT_VPW 2   // eigenvectors per warp
#endif
__host__ __device__ inline size_t backtr_smem_bytes(int n) { return (size_t)BT_R * n * 16 + BT_R * 16; }

__device__ __forceinline__ int find_bstart(const HeevProblem* p, int n, int b) {
  int lo = 0, hi = n - 1;
  while (lo < hi) {
    int mid = (lo + hi + 1) >> 1;
    if (p[mid].bstart <= b) lo = mid; else hi = mid - 1;
  }
  return lo;
}

template <int NQ, int VPW>
__global__ void __launch_bounds__(BT_WARPS * 32) heev_backtr_blk(const HeevProblem* __restrict__ probs, int nprob) {
  TCBC_PDL_WAIT();
  extern __shared__ __align__(16) unsigned char smem_raw[];
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const HeevProblem& P = probs[find_bstart(probs, nprob, blockIdx.x)];
  if (P.skip && *P.skip) return;
  const int t0 = (blockIdx.x - P.bstart) * BT_WARPS * VPW, tw = t0 + warp * VPW, n = P.n, kmax = P.kmax;
  cplx* sv = reinterpret_cast<cplx*>(smem_raw);
  cplx* stau = sv + (size_t)BT_R * n;
  const double* Z = P.work + 2 * n + 8;
  const cplx* A = P.A;
  const int k = P.k_out ? *P.k_out : kmax;
  if (t0 >= k) {   // block-uniform: every vector of this block is dropped
#pragma unroll
    for (int u = 0; u < VPW; ++u)
      if (tw + u < kmax)
        for (int i = lane; i < n; i += 32) P.Vt[(size_t)(tw + u) * n + i] = make_double2(0.0, 0.0);
    return;
  }
  const bool act = tw < k;   // this warp holds at least one kept vector (dropped ones stay 0)
  // VPW vectors per warp: each reflector entry read from shared memory serves VPW vectors
  double yr[VPW][NQ], yi[VPW][NQ];
#pragma unroll
  for (int u = 0; u < VPW; ++u)
#pragma unroll
    for (int q = 0; q < NQ; ++q) {
      const int i = lane + 32 * q, t = tw + u;
      yr[u][q] = (t < k && i < n) ? Z[(size_t)i * kmax + t] : 0.0;
      yi[u][q] = 0.0;
    }
  for (int j1 = n - 2; j1 >= 0; j1 -= BT_R) {
    const int j0 = max(0, j1 - BT_R + 1);
    __syncthreads();
    for (int r = warp; r <= j1 - j0; r += BT_WARPS) {
      const int j = j0 + r;
      const cplx* row = A + (size_t)j * n;
      for (int i = lane; i < n; i += 32) sv[(size_t)r * n + i] = i > j ? row[i] : make_double2(0.0, 0.0);
    }
    if ((int)threadIdx.x <= j1 - j0) stau[threadIdx.x] = P.tau[j0 + threadIdx.x];
    __syncthreads();
    if (!act) continue;
    for (int j = j1; j >= j0; --j) {
      const cplx tau = stau[j - j0];
      if (tau.x == 0.0 && tau.y == 0.0) continue;
      const cplx* row = sv + (size_t)(j - j0) * n;
      cplx v[NQ];
#pragma unroll
      for (int q = 0; q < NQ; ++q) {
        const int i = lane + 32 * q;
        v[q] = i < n ? row[i] : make_double2(0.0, 0.0);
      }
      double sr[VPW], si[VPW];   // s = v^H y over i > j (entries i <= j are staged as 0)
#pragma unroll
      for (int u = 0; u < VPW; ++u) {
        sr[u] = 0.0;
        si[u] = 0.0;
#pragma unroll
        for (int q = 0; q < NQ; ++q) {
          sr[u] += v[q].x * yr[u][q] + v[q].y * yi[u][q];
          si[u] += v[q].x * yi[u][q] - v[q].y * yr[u][q];
        }
      }
#pragma unroll
      for (int u = 0; u < VPW; ++u) {
        sr[u] = warp_sum(sr[u]);
        si[u] = warp_sum(si[u]);
      }
#pragma unroll
      for (int u = 0; u < VPW; ++u) {
        const double tr = tau.x * sr[u] - tau.y * si[u], ti = tau.x * si[u] + tau.y * sr[u];
#pragma unroll
        for (int q = 0; q < NQ; ++q) {
          yr[u][q] -= tr * v[q].x - ti * v[q].y;
          yi[u][q] -= tr * v[q].y + ti * v[q].x;
        }
      }
    }
  }
#pragma unroll
  for (int u = 0; u < VPW; ++u) {
    const int t = tw + u;
    if (t >= kmax) continue;
#pragma unroll
    for (int q = 0; q < NQ; ++q) {
      const int i = lane + 32 * q;
      if (i < n) P.Vt[(size_t)t * n + i] = make_double2(yr[u][q], yi[u][q]);
    }
  }
}

// ---------------------------------------------------------------- K6: truncation decision
__global__ void heev_finish(const HeevProblem* __restrict__ probs, int nprob) {
  TCBC_PDL_WAIT();
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= nprob) return;
  const HeevProblem& P = probs[i];
  const int kmax = P.kmax;
  if (P.skip && *P.skip) {   // exact-factor shortcut: every direction kept, nothing discarded
    if (P.k_out) *P.k_out = kmax;
    if (P.w_out) *P.w_out = 0.0;
    return;
  }
  const double trace = P.work[2 * P.n + S_TRACE];
  const double l1 = P.lam[0];
  int k = 1;
  double kept = 0.0;
  if (trace > 0.0 && l1 > 0.0) {
    int cnt = 0;
    for (int t = 0; t < kmax; ++t)
      if (P.lam[t] > P.tol2 * l1 && P.lam[t] > P.floor_rel * l1) ++cnt;
    k = cnt < 1 ? 1 : (cnt > P.max_bond ? P.max_bond : cnt);
    for (int t = 0; t < k; ++t) kept += P.lam[t];
    for (int t = k; t < kmax; ++t) P.lam[t] = 0.0;   // dropped rows of the factor are zero
  } else {
    for (int t = 0; t < kmax; ++t) P.lam[t] = 0.0;
  }
  if (P.k_out) *P.k_out = k;
  if (P.w_out) *P.w_out = fmax(trace - kept, 0.0);
  // clusters of close kept eigenvalues (gap <= 1e-5 ||T||): their vectors
  // are computed sequentially with reorthogonalisation (K3b), the others thread-parallel (K3a)
  double* cst = cluster_arrays(P);
  double* csz = cst + kmax;
  // LAPACK dstein uses 1e-3 ||T||; an isolated inverse-iteration vector is accurate to
  // ~eps ||T|| / gap, i.e. <= 1e-11 for gaps above 1e-5 ||T||, far inside the parity budget
  // (1 - cos <= 1e-10), so only tighter groups take the sequential reorthogonalised path.
  const double ortol = 1e-5 * P.work[2 * P.n + S_TNORM];
  int s0 = 0;
  for (int t = 1; t <= k; ++t) {
    if (t == k || !(P.lam[t - 1] - P.lam[t] <= ortol)) {
      for (int q = s0; q < t; ++q) {
        cst[q] = s0;
        csz[q] = t - s0;
      }
      s0 = t;
    }
  }
}

// ---------------------------------------------------------------- K3b: clusters (dstein)
// one CTA per matrix, one warp per cluster of >= 2 close eigenvalues: the vectors of a
// cluster are computed one after the other, each inverse-iteration step orthogonalised
// (MGS) against the cluster's previous vectors, so degenerate spectra (e.g. isometric
// inputs whose Gram is the identity) still give an orthonormal basis of the subspace.
// K3b: clusters of close eigenvalues (gap <= 1e-5 ||T||; circuit Grams have exactly
// degenerate ones).  One CTA per matrix walks its clusters; within a cluster every vector gets
// its own thread (its own shifted dgttrf / dgttrs, as K3a), and after each solve the whole
// block is re-orthonormalised by modified Gram-Schmidt over all threads -- block inverse
// iteration, so the O(n) tridiagonal solves of a cluster run in parallel instead of one
// after another.
__global__ void __launch_bounds__(HEEV_THREADS) heev_invit_cluster(const HeevProblem* __restrict__ probs) {
  TCBC_PDL_WAIT();
  const HeevProblem P = probs[blockIdx.x];
  if (P.skip && *P.skip) return;
  const int n = P.n, kmax = P.kmax, tid = threadIdx.x;
  const int k = P.k_out ? *P.k_out : kmax;
  const double* sd = P.work;
  const double* evec = P.work + n;
  const double tnorm = P.work[2 * n + S_TNORM];
  if (!(tnorm > 0.0)) return;
  double* Z = P.work + 2 * n + 8;
  const size_t NK = (size_t)n * kmax;
  double* DL = Z + NK;
  double* Dg = DL + NK;
  double* DU = Dg + NK;
  double* DU2 = DU + NK;
  double* PV = DU2 + NK;
  const double* cst = cluster_arrays(P);
  const double* csz = cst + kmax;
  const double pert = DBL_EPSILON * tnorm;
  __shared__ double2 red[HEEV_WARPS + 1];
  __shared__ double s_scale[256];
#define AT(arr, i, t) arr[(size_t)(i) * kmax + (t)]
  for (int t0 = 0; t0 < k; ++t0) {
    if ((int)cst[t0] != t0 || csz[t0] < 2.0) continue;   // not the start of a multi-vector cluster
    const int t1 = t0 + (int)csz[t0], c = t1 - t0;
    // ---- factor T - lam_t I for every member (thread per vector), random start vectors
    for (int t = t0 + tid; t < t1; t += HEEV_THREADS) {
      const double lam = P.lam[t] - (t - t0) * 10.0 * DBL_EPSILON * tnorm;   // shifts kept apart (dstein)
      double d_i = sd[0] - lam, du_i = n > 1 ? evec[0] : 0.0;
      for (int i = 0; i < n - 1; ++i) {
        const double dl = evec[i];
        double d_n = sd[i + 1] - lam, du_n = (i < n - 2) ? evec[i + 1] : 0.0, du2 = 0.0, l, p = 0.0;
        if (fabs(d_i) >= fabs(dl)) {
          if (fabs(d_i) < pert) d_i = copysign(pert, d_i == 0.0 ? 1.0 : d_i);
          l = dl / d_i;
          d_n -= l * du_i;
        } else {
          l = d_i / dl;
          const double old_du = du_i;
          d_i = dl;
          du_i = d_n;
          du2 = du_n;
          d_n = old_du - l * d_n;
          du_n = -l * du_n;
          p = 1.0;
        }
        if (fabs(d_i) < pert) d_i = copysign(pert, d_i == 0.0 ? 1.0 : d_i);
        AT(Dg, i, t) = 1.0 / d_i;
        AT(DU, i, t) = du_i;
        AT(DU2, i, t) = du2;
        AT(DL, i, t) = l;
        AT(PV, i, t) = p;
        d_i = d_n;
        du_i = du_n;
      }
      if (fabs(d_i) < pert) d_i = copysign(pert, d_i == 0.0 ? 1.0 : d_i);
      AT(Dg, n - 1, t) = 1.0 / d_i;
      for (int i = 0; i < n; ++i)
        AT(Z, i, t) = (double)(hash32((unsigned)(t * 7919 + i * 104729 + 12345)) & 0xffffff) / 16777216.0 - 0.5;
    }
    __syncthreads();
    for (int it = 0; it < 3; ++it) {
      // ---- solve (T - lam_t I) y = z in place (dgttrs), rescaled to max |y| = 1
      for (int t = t0 + tid; t < t1; t += HEEV_THREADS) {
        double cur = AT(Z, 0, t);
        for (int i = 0; i < n - 1; ++i) {
          const double nxt = AT(Z, i + 1, t);
          const double l = AT(DL, i, t);
          if (AT(PV, i, t) == 0.0) { AT(Z, i, t) = cur; cur = nxt - l * cur; }
          else { AT(Z, i, t) = nxt; cur = cur - l * nxt; }
        }
        double y2 = 0.0, y1 = cur * AT(Dg, n - 1, t);
        AT(Z, n - 1, t) = y1;
        double mx = fabs(y1);
        for (int i = n - 2; i >= 0; --i) {
          double yi = (AT(Z, i, t) - AT(DU, i, t) * y1 - AT(DU2, i, t) * y2) * AT(Dg, i, t);
          if (fabs(yi) > 1e100) {
            const double f = 1e-100;
            for (int q = i + 1; q < n; ++q) AT(Z, q, t) *= f;
            yi *= f; y1 *= f; y2 *= f; mx *= f;
          }
          AT(Z, i, t) = yi;
          mx = fmax(mx, fabs(yi));
          y2 = y1;
          y1 = yi;
        }
        const double sc = mx > 0.0 ? 1.0 / mx : 1.0;
        for (int i = 0; i < n; ++i) AT(Z, i, t) *= sc;
      }
      __syncthreads();
      // ---- modified Gram-Schmidt over the block (twice is enough for exact degeneracy)
      for (int rep = 0; rep < 2; ++rep)
        for (int j = t0; j < t1; ++j) {
          double part = 0.0;
          for (int i = tid; i < n; i += HEEV_THREADS) part += AT(Z, i, j) * AT(Z, i, j);
          const double nr = block_sum2(part, 0.0, red).x;
          const double inv = nr > 1e-300 ? 1.0 / sqrt(nr) : 0.0;
          for (int i = tid; i < n; i += HEEV_THREADS) AT(Z, i, j) *= inv;
          __syncthreads();
          if (j + 1 >= t1) break;
          // projections of the later vectors onto j: warp per vector
          const int lane = tid & 31, warp = tid >> 5;
          for (int q = j + 1 + warp; q < t1; q += HEEV_WARPS) {
            double d = 0.0;
            for (int i = lane; i < n; i += 32) d += AT(Z, i, j) * AT(Z, i, q);
            d = warp_sum(d);
            if (lane == 0) s_scale[(q - j - 1) & 255] = d;
          }
          __syncthreads();
          for (int e = tid; e < n * (t1 - j - 1); e += HEEV_THREADS) {
            const int q = j + 1 + e / n, i = e % n;
            if (q - j - 1 < 256) AT(Z, i, q) -= s_scale[q - j - 1] * AT(Z, i, j);
          }
          __syncthreads();
        }
    }
    (void)c;
  }
#undef AT
}

}  // namespace

size_t heev_work_doubles(int n, int kmax) {
  static_assert(HEEV_WARPS == 8 && S_TRACE == H2S_S_TRACE, "heev2s.h mirrors this layout");
  return heev_base_doubles(n, kmax) + h2s_extra_doubles(n);
}

size_t heev_smem_bytes(int n, int kmax) {
  (void)kmax;
  if (n > FUSED_MAX_N) return (size_t)n * 16 * 2 + 64;
  const int r0 = fused_r0(n);
  return fused_base_bytes(n) + 16 * ((size_t)n * (n + 1) / 2 - (size_t)r0 * (r0 + 1) / 2);
}

int heev_max_n() { return HEEV_MAX_N; }
int heev_small_n() { return jac_route_n(); }

namespace {
template <int CS>
void launch_cl(const HeevProblem* d, int nprob, size_t smem, cudaStream_t s) {
  func_smem(heev_tridiag_cluster<CS>, CL_SMEM_LIMIT);
  if (CS > 8)
    func_attr(reinterpret_cast<const void*>(heev_tridiag_cluster<CS>), cudaFuncAttributeNonPortableClusterSizeAllowed, 1);
  cudaLaunchConfig_t cfg{};
  cfg.gridDim = dim3(nprob * CS);
  cfg.blockDim = dim3(CL_THREADS);
  cfg.dynamicSmemBytes = smem;
  cfg.stream = s;
  cudaLaunchAttribute at[2];
  at[0].id = cudaLaunchAttributeClusterDimension;
  at[0].val.clusterDim.x = CS;
  at[0].val.clusterDim.y = 1;
  at[0].val.clusterDim.z = 1;
  at[1].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  at[1].val.programmaticStreamSerializationAllowed = pdl_enabled() ? 1 : 0;
  cfg.attrs = at;
  cfg.numAttrs = 2;
  cudaLaunchKernelEx(&cfg, heev_tridiag_cluster<CS>, d);
}
void launch_tridiag_cluster(const HeevProblem* d, int nprob, int cs, size_t smem, cudaStream_t s) {
  switch (cs) {
    case 2: launch_cl<2>(d, nprob, smem, s); break;
    case 4: launch_cl<4>(d, nprob, smem, s); break;
    case 8: launch_cl<8>(d, nprob, smem, s); break;
    default: launch_cl<16>(d, nprob, smem, s); break;
  }
}
}  // namespace


namespace {
// the WY back-transform of a launch (see wy_prep); Vt and A as in HeevProblem
void backtr_wy(HeevProblem* h, int n, const HeevProblem* d, Stager& st, cudaStream_t s, Scratch* ws) {
  prof_begin(s);
  launch_k(wy_prep, n, 256, 0, s, d);
  prof_end(s, "heev", 0.0, 0.0);
  count_launch();
  int maxb = 0;
  std::vector<int> nblk(n);
  for (int i = 0; i < n; ++i) {
    nblk[i] = (h[i].n - 1 + WY_NB - 1) / WY_NB;
    maxb = std::max(maxb, nblk[i]);
  }
  // Y_b^H Y_b of every block, then T_b
  std::vector<GemmProblem> gg;
  std::vector<WyBlock> wb;
  std::vector<std::vector<cplx*>> T(n), G(n);
  std::vector<cplx*> P1(n), P2(n);
  for (int i = 0; i < n; ++i) {
    const HeevProblem& p = h[i];
    P1[i] = static_cast<cplx*>(ws->get(sizeof(cplx) * p.kmax * WY_NB));
    P2[i] = static_cast<cplx*>(ws->get(sizeof(cplx) * p.kmax * WY_NB));
    for (int b = 0; b < nblk[i]; ++b) {
      const int j0 = b * WY_NB, nbb = std::min(WY_NB, p.n - 1 - j0);
      cplx* Gb = static_cast<cplx*>(ws->get(sizeof(cplx) * nbb * nbb));
      cplx* Tb = static_cast<cplx*>(ws->get(sizeof(cplx) * WY_NB * WY_NB));
      const cplx* Yt = p.A + (size_t)j0 * p.n;
      GemmProblem g{};
      g.A = Yt; g.B = Yt; g.C = Gb; g.M = nbb; g.N = nbb; g.K = p.n;
      gemm_from_ops(g, OP_N, p.n, OP_C, p.n, nbb);
      g.alpha = make_double2(1.0, 0.0);
      gg.push_back(g);
      wb.push_back(WyBlock{Gb, Tb, p.tau + j0, p.skip, nbb, 0});
      T[i].push_back(Tb);
      G[i].push_back(Gb);
    }
  }
  launch_gemm(gg.data(), (int)gg.size(), st, s, ws, "heev");
  {
    const WyBlock* dw = static_cast<const WyBlock*>(st.put(wb.data(), sizeof(WyBlock) * wb.size()));
    prof_begin(s);
    launch_k(wy_larft, ((int)wb.size() + 3) / 4, 128, 0, s, dw, (int)wb.size());
    prof_end(s, "heev", 0.0, 0.0);
    count_launch();
  }
  for (int b = maxb - 1; b >= 0; --b) {
    std::vector<GemmProblem> g1, g2, g3;
    for (int i = 0; i < n; ++i) {
      if (b >= nblk[i]) continue;
      const HeevProblem& p = h[i];
      const int j0 = b * WY_NB, nbb = std::min(WY_NB, p.n - 1 - j0);
      const cplx* Yt = p.A + (size_t)j0 * p.n;
      GemmProblem g{};
      g.A = p.Vt; g.B = Yt; g.C = P1[i]; g.M = p.kmax; g.N = nbb; g.K = p.n;     // P1 = Vt conj(Y_b)
      gemm_from_ops(g, OP_N, p.n, OP_C, p.n, nbb);
      g.alpha = make_double2(1.0, 0.0);
      g1.push_back(g);
      GemmProblem g2p{};
      g2p.A = P1[i]; g2p.B = T[i][b]; g2p.C = P2[i]; g2p.M = p.kmax; g2p.N = nbb; g2p.K = nbb;   // P2 = P1 T^T
      gemm_from_ops(g2p, OP_N, nbb, OP_T, WY_NB, nbb);
      g2p.alpha = make_double2(1.0, 0.0);
      g2.push_back(g2p);
      GemmProblem g3p{};
      g3p.A = P2[i]; g3p.B = Yt; g3p.C = p.Vt; g3p.M = p.kmax; g3p.N = p.n; g3p.K = nbb;   // Vt -= P2 Y_b^T
      gemm_from_ops(g3p, OP_N, nbb, OP_N, p.n, p.n);
      g3p.alpha = make_double2(-1.0, 0.0);
      g3p.beta = make_double2(1.0, 0.0);
      g3.push_back(g3p);
    }
    launch_gemm(g1.data(), (int)g1.size(), st, s, ws, "heev");
    launch_gemm(g2.data(), (int)g2.size(), st, s, ws, "heev");
    launch_gemm(g3.data(), (int)g3.size(), st, s, ws, "heev");
  }
}
}  // namespace

void launch_heev(HeevProblem* hin, int nin, Stager& st, cudaStream_t s, const std::function<void()>& values_ready,
                 Scratch* ws) {
  HostScope hs_("launch_heev");
  if (nin == 0) return;
  // K0: Grams of order <= 32 in one launch (warp per Gram); the rest take K1..K7
  std::vector<HeevProblem> small, rest;
  const int jn = jac_route_n();
  for (int i = 0; i < nin; ++i) (hin[i].n <= jn ? small : rest).push_back(hin[i]);
  if (!small.empty()) {
    int nmax = 1;
    for (auto& p : small) nmax = std::max(nmax, p.n);
    const size_t sm = jac_warp_bytes(nmax) * JAC_WARPS;
    func_smem(heev_jacobi, jac_warp_bytes(JAC_MAX_N) * JAC_WARPS);
    const HeevProblem* dj = static_cast<const HeevProblem*>(st.put(small.data(), sizeof(HeevProblem) * small.size()));
    double fl = 0.0;
    for (auto& p : small) fl += 8.0 * 8.0 * (double)p.n * p.n * p.n;   // ~8 sweeps of 8 n^3 flops
    prof_begin(s);
    launch_k(heev_jacobi, ((int)small.size() + JAC_WARPS - 1) / JAC_WARPS, JAC_WARPS * 32, sm, s, dj, (int)small.size(), nmax);
    prof_end(s, "heev", fl, 32.0 * (double)small.size());
    count_launch();
  }
  if (rest.empty()) {
    if (values_ready) values_ready();
    return;
  }
  HeevProblem* h = rest.data();
  const int n = (int)rest.size();
  func_smem(heev_tridiag<4>, FUSED_SMEM_BUDGET);
  func_smem(heev_tridiag<6>, FUSED_SMEM_BUDGET);
  func_smem(heev_tridiag<8>, FUSED_SMEM_BUDGET);
  int total = 0;
  double fl = 0.0, by = 0.0;
  int nblk = 0;
  for (int i = 0; i < n; ++i) {
    h[i].estart = total;
    total += h[i].kmax;
    h[i].bstart = nblk;
    nblk += (h[i].kmax + BT_WARPS * BT_VPW - 1) / (BT_WARPS * BT_VPW);
    const double nn = h[i].n;
    fl += 8.0 * ((4.0 / 3.0) * nn * nn * nn + 2.0 * nn * nn * h[i].kmax);
    by += 16.0 * nn * nn;
  }
  const HeevProblem* d = static_cast<const HeevProblem*>(st.put(h, sizeof(HeevProblem) * n));
  prof_begin(s);
  // K1.  Few Grams of order > 96 (chain levels; measured faster than one CTA even when the
  // matrix fits one CTA's shared memory): one thread-block cluster per matrix, as many
  // CTAs as keep the level within ~2 waves; otherwise one CTA per matrix, one launch per
  // storage mode so small-smem problems are not limited by large ones.
  std::vector<HeevProblem> grp[3], cgrp;
  {
    int maxn = 0, cnt = 0;
    for (int i = 0; i < n; ++i)
      if (h[i].n > 96) { maxn = std::max(maxn, h[i].n); ++cnt; }
    int cs = 0;
    for (int c = 2; c <= 16; c *= 2)
      if (cl_smem_bytes(maxn, c) <= CL_SMEM_LIMIT) { cs = c; break; }
    if (cnt > 0 && cs > 0 && cnt * cs <= 296) {
      while (cs < 16 && cnt * cs * 2 <= 296 && (maxn + 2 * cs - 1) / (2 * cs) >= 8) cs *= 2;
      for (int i = 0; i < n; ++i)
        if (h[i].n > 96) cgrp.push_back(h[i]);
      const HeevProblem* dg = static_cast<const HeevProblem*>(st.put(cgrp.data(), sizeof(HeevProblem) * cgrp.size()));
      launch_tridiag_cluster(dg, (int)cgrp.size(), cs, cl_smem_bytes(maxn, cs), s);
      count_launch();
    }
  }
  // two-stage reduction (heev2s.cu) for the one-CTA Grams of order 65..256
  std::vector<char> is2s(n, 0);
  std::vector<HeevProblem> p2s;
  int maxn2s = 0;
  for (int i = 0; i < n; ++i) {
    if (!cgrp.empty() && h[i].n > 96) continue;
    if (heev2s_use(h[i].n, n)) {
      is2s[i] = 1;
      p2s.push_back(h[i]);
      maxn2s = std::max(maxn2s, h[i].n);
      continue;
    }
    grp[h[i].n <= SMEM_MAX_N ? 0 : (h[i].n <= FUSED_MAX_N ? 1 : 2)].push_back(h[i]);
  }
  if (!p2s.empty()) {
    const HeevProblem* d2 = static_cast<const HeevProblem*>(st.put(p2s.data(), sizeof(HeevProblem) * p2s.size()));
    launch_heev2s_reduce(d2, (int)p2s.size(), maxn2s, s);
  }
  for (auto& g : grp) {
    if (g.empty()) continue;
    size_t smem = 0;
    for (auto& p : g) smem = std::max(smem, heev_smem_bytes(p.n, p.kmax));
    const HeevProblem* dg = static_cast<const HeevProblem*>(st.put(g.data(), sizeof(HeevProblem) * g.size()));
    int mxn = 0;
    for (auto& p : g) mxn = std::max(mxn, p.n);
    if (mxn <= 128) launch_k(heev_tridiag<4>, (int)g.size(), HEEV_THREADS, smem, s, dg);
    else if (mxn <= 192) launch_k(heev_tridiag<6>, (int)g.size(), HEEV_THREADS, smem, s, dg);
    else launch_k(heev_tridiag<8>, (int)g.size(), HEEV_THREADS, smem, s, dg);
    count_launch();
  }
  {   // smallest lanes-per-eigenvalue that still keeps ~6 warps per SM busy
    int G = 1;
    while (G < 32 && (long long)total * G < 148LL * 6 * 32) G *= 2;   // measured: 6 beats 3, 12, 24
    const int blocks = (int)(((long long)total * G + 255) / 256);
    switch (G) {
      case 1: launch_k(heev_bisect<1>, blocks, 256, 0, s, d, n, total); break;
      case 2: launch_k(heev_bisect<2>, blocks, 256, 0, s, d, n, total); break;
      case 4: launch_k(heev_bisect<4>, blocks, 256, 0, s, d, n, total); break;
      case 8: launch_k(heev_bisect<8>, blocks, 256, 0, s, d, n, total); break;
      case 16: launch_k(heev_bisect<16>, blocks, 256, 0, s, d, n, total); break;
      default: launch_k(heev_bisect<32>, blocks, 256, 0, s, d, n, total); break;
    }
  }
  launch_k(heev_finish, (n + 127) / 128, 128, 0, s, d, n);   // k and w: only kept pairs go on
  launch_k(heev_unscale, (n + 127) / 128, 128, 0, s, d, n, 1);
  if (values_ready) values_ready();   // k and w are final: the caller may read them now
  {
    int mxn = 1;
    for (int i = 0; i < n; ++i) mxn = std::max(mxn, h[i].n);
    // blocks of up to 32 vectors; the budget that keeps three blocks per SM when 8 vectors fit
    // it (n <= 192: more vectors in flight per SM beat bigger blocks, measured), else all
    const size_t budget = (size_t)6 * mxn * 8 * sizeof(double) <= INVIT_SMEM_SHARED ? INVIT_SMEM_SHARED : INVIT_SMEM_MAX;
    int nt = INVIT_NT;
    while (nt > 8 && (size_t)6 * mxn * nt * sizeof(double) > budget) nt /= 2;
    const size_t ism = (size_t)6 * mxn * nt * sizeof(double);
    if (ism <= INVIT_SMEM_MAX) {
      func_smem(heev_invit_smem, INVIT_SMEM_MAX);
      launch_k(heev_invit_smem, (total + nt - 1) / nt, nt, ism, s, d, n, total, mxn);
    } else {
      launch_k(heev_invit, (total + 127) / 128, 128, 0, s, d, n, total);
    }
  }
  launch_k(heev_invit_cluster, n, HEEV_THREADS, 0, s, d);
  count_launch();
  {
    int mk = 0;
    for (int i = 0; i < n; ++i) mk = std::max(mk, h[i].kmax);
    if (mk <= ORTH_SMEM_K) {
      func_smem(heev_orth_smem, orth_smem_bytes(ORTH_SMEM_K));
      launch_k(heev_orth_smem, n, HEEV_THREADS, orth_smem_bytes(mk), s, d);
    } else {
      launch_k(heev_orth, n, HEEV_THREADS, 0, s, d);
    }
  }
  int mxn_all = 0;
  for (int i = 0; i < n; ++i) mxn_all = std::max(mxn_all, h[i].n);
  // measured slower than heev_backtr_blk on every bench config (config 3: 962 -> 910 applies/s,
  // config 5: 3428 -> 1219): the per-block GEMMs are tiny (k = 32 rows) and wy_larft is
  // warp-serial; kept behind TTN_HEEV_WY=1 for measurement
  static const bool wy_on = getenv("TTN_HEEV_WY") != nullptr;
  if (ws && wy_on && mxn_all >= WY_MIN_N) {
    prof_end(s, "heev", fl, by);
    count_launch(); count_launch(); count_launch(); count_launch(); count_launch();   // K2, K6, K7, K3, K4
    backtr_wy(h, n, d, st, s, ws);
    prof_begin(s);
    launch_k(heev_unscale, (n + 127) / 128, 128, 0, s, d, n, 2);
    prof_end(s, "heev", 0.0, 0.0);
    count_launch();
    return;
  }
  const HeevProblem* dbt = d;   // the one-stage back-transform's problems
  int nbt = n, nblk1 = nblk;
  std::vector<HeevProblem> p1;
  if (!p2s.empty()) {
    int nb2 = 0;
    heev2s_assign_blocks(p2s.data(), (int)p2s.size(), nb2);
    const HeevProblem* d2 = static_cast<const HeevProblem*>(st.put(p2s.data(), sizeof(HeevProblem) * p2s.size()));
    launch_heev2s_backtr(d2, (int)p2s.size(), nb2, maxn2s, s);
    nblk1 = 0;
    for (int i = 0; i < n; ++i) {
      if (is2s[i]) continue;
      p1.push_back(h[i]);
      p1.back().bstart = nblk1;
      nblk1 += (h[i].kmax + BT_WARPS * BT_VPW - 1) / (BT_WARPS * BT_VPW);
    }
    nbt = (int)p1.size();
    dbt = p1.empty() ? nullptr : static_cast<const HeevProblem*>(st.put(p1.data(), sizeof(HeevProblem) * p1.size()));
  }
  if (nbt > 0) {
    int mxn = 0;
    for (int i = 0; i < n; ++i)
      if (!is2s[i]) mxn = std::max(mxn, h[i].n);
    if (mxn <= 256) {
      func_smem(heev_backtr_blk<4, BT_VPW>, backtr_smem_bytes(256));
      func_smem(heev_backtr_blk<6, BT_VPW>, backtr_smem_bytes(256));
      func_smem(heev_backtr_blk<8, BT_VPW>, backtr_smem_bytes(256));
      if (mxn <= 128) launch_k(heev_backtr_blk<4, BT_VPW>, nblk1, BT_WARPS * 32, backtr_smem_bytes(mxn), s, dbt, nbt);
      else if (mxn <= 192) launch_k(heev_backtr_blk<6, BT_VPW>, nblk1, BT_WARPS * 32, backtr_smem_bytes(mxn), s, dbt, nbt);
      else launch_k(heev_backtr_blk<8, BT_VPW>, nblk1, BT_WARPS * 32, backtr_smem_bytes(mxn), s, dbt, nbt);
    } else {
      int tot1 = 0;
      for (int i = 0; i < n; ++i)
        if (!is2s[i]) tot1 += h[i].kmax;
      launch_k(heev_backtr, (tot1 * 32 + 255) / 256, 256, 0, s, dbt, nbt, tot1);
    }
  }
  launch_k(heev_unscale, (n + 127) / 128, 128, 0, s, d, n, 2);
  count_launch();
  count_launch();
  count_launch(); count_launch(); count_launch(); count_launch(); count_launch();
  prof_end(s, "heev", fl, by);
}

}  // namespace tcbc
