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
//              of step j (one pass per step), the packed triangle in shared memory for n <= 144.
//  K2 bisect   one thread per (matrix, eigenvalue): Sturm-count quartersection (3 interleaved
//              chains hide the division latency) for the top kmax eigenvalues.
//  K3 invit    one thread per (matrix, eigenvector): inverse iteration on T - lam I
//              (dgttrf / dgttrs with partial pivoting), scratch interleaved across threads.
//  K4 orth     one CTA per matrix: CholeskyQR2 of the kmax vectors (clusters of close
//              eigenvalues leave inverse-iteration vectors only approximately orthogonal).
//  K5 backtr   one warp per (matrix, eigenvector): V = Q Z by the stored reflectors.
//  K6 finish   truncation decision k = min(max_bond, #{lam > tol^2 lam_1}, #{lam > floor lam_1})
//              >= 1 and discarded weight w = trace(A) - sum_{t<k} lam_t.
#include "kernels.h"
#include "prof.h"
#include <algorithm>
#include <cfloat>
#include <cmath>
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

// Householder tridiagonalisation (zhetd2, lower) touching only the lower triangle, with the
// rank-2 update of step j-1 fused into the Hermitian mat-vec of step j: one read-modify-write
// pass over the trailing triangle per step.  SM: the packed triangle lives in shared memory.
// Reflector j is written to row j (columns > j) of the global A for the back-transform.
template <bool SM>
__device__ void tridiag_fused(cplx* __restrict__ A, const int n, cplx* vcur, cplx* wcur, cplx* base, double* dvec,
                              double* evec, cplx* tau_out, double2* red) {
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  cplx* vprev = base;
  cplx* wprev = vprev + n;
  cplx* prow = wprev + n;
  cplx* colpart = prow + n;                   // [HEEV_WARPS][n]
  cplx* Ap = colpart + HEEV_WARPS * n;        // packed lower triangle (SM)
#define LL(r, c) (SM ? Ap[(size_t)(r) * ((r) + 1) / 2 + (c)] : A[(size_t)(r) * n + (c)])
  if (SM) {
    for (int r = warp; r < n; r += HEEV_WARPS)
      for (int c = lane; c <= r; c += 32) Ap[(size_t)r * (r + 1) / 2 + c] = A[(size_t)r * n + c];
  }
  for (int i = tid; i < n; i += HEEV_THREADS) {
    vprev[i] = make_double2(0.0, 0.0);
    wprev[i] = make_double2(0.0, 0.0);
  }
  __syncthreads();
  bool have_prev = false;
  for (int j = 0; j < n - 1; ++j) {
    // (a) pending update U_{j-1} on column j (rows >= j)
    if (have_prev) {
      const cplx vpj = vprev[j], wpj = wprev[j];
      for (int r = j + tid; r < n; r += HEEV_THREADS) {
        cplx a = LL(r, j);
        const cplx vr = vprev[r], wr = wprev[r];
        a.x -= (vr.x * wpj.x + vr.y * wpj.y) + (wr.x * vpj.x + wr.y * vpj.y);
        a.y -= (vr.y * wpj.x - vr.x * wpj.y) + (wr.y * vpj.x - wr.x * vpj.y);
        LL(r, j) = a;
      }
      __syncthreads();
    }
    // (b) reflector H_j from x = A[j+1:, j]  (zlarfg)
    double part = 0.0;
    for (int r = j + 2 + tid; r < n; r += HEEV_THREADS) {
      const cplx x = LL(r, j);
      part += x.x * x.x + x.y * x.y;
    }
    const double xn2 = block_sum2(part, 0.0, red).x;
    const cplx alpha = LL(j + 1, j);
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
    for (int r = j + 1 + tid; r < n; r += HEEV_THREADS) {
      cplx v;
      if (r == j + 1) v = make_double2(1.0, 0.0);
      else {
        const cplx x = LL(r, j);
        v = make_double2(x.x * scale.x - x.y * scale.y, x.x * scale.y + x.y * scale.x);
      }
      A[(size_t)j * n + r] = v;                        // kept for the back-transform
      vcur[r] = tnz ? v : make_double2(0.0, 0.0);
    }
    if (tid == 0) {
      evec[j] = beta;
      dvec[j] = LL(j, j).x;
      tau_out[j] = tau;
    }
    __syncthreads();
    // (c) one pass over the trailing lower triangle: apply U_{j-1}, accumulate p = A v_j
    cplx cacc[8];
#pragma unroll
    for (int q = 0; q < 8; ++q) cacc[q] = make_double2(0.0, 0.0);
    for (int r = j + 1 + warp; r < n; r += HEEV_WARPS) {
      const cplx vr = vcur[r];
      const cplx vpr = vprev[r], wpr = wprev[r];
      double sr = 0.0, si = 0.0;
#pragma unroll
      for (int q = 0; q < 8; ++q) {
        const int c = j + 1 + lane + 32 * q;
        if (c > r) break;
        cplx a = LL(r, c);
        if (have_prev) {
          const cplx vpc = vprev[c], wpc = wprev[c];
          a.x -= (vpr.x * wpc.x + vpr.y * wpc.y) + (wpr.x * vpc.x + wpr.y * vpc.y);
          a.y -= (vpr.y * wpc.x - vpr.x * wpc.y) + (wpr.y * vpc.x - wpr.x * vpc.y);
          LL(r, c) = a;
        }
        const cplx vc = vcur[c];
        sr += a.x * vc.x - a.y * vc.y;
        si += a.x * vc.y + a.y * vc.x;
        if (c < r) {   // (r, c) also stands for A[c][r] = conj(a): p[c] += conj(a) v_r
          cacc[q].x += a.x * vr.x + a.y * vr.y;
          cacc[q].y += a.x * vr.y - a.y * vr.x;
        }
      }
      sr = warp_sum(sr);
      si = warp_sum(si);
      if (lane == 0) prow[r] = make_double2(sr, si);
    }
#pragma unroll
    for (int q = 0; q < 8; ++q) {
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
    const double2 dot = block_sum2(dr, di, red);
    const cplx a2 = make_double2(-0.5 * (tau.x * dot.x - tau.y * dot.y), -0.5 * (tau.x * dot.y + tau.y * dot.x));
    for (int r = tid; r < n; r += HEEV_THREADS) {
      if (r <= j) {
        vprev[r] = make_double2(0.0, 0.0);
        wprev[r] = make_double2(0.0, 0.0);
      } else {
        const cplx v = vcur[r], p = wcur[r];
        vprev[r] = v;
        wprev[r] = make_double2(p.x + a2.x * v.x - a2.y * v.y, p.y + a2.x * v.y + a2.y * v.x);
      }
    }
    have_prev = tnz;
    __syncthreads();
  }
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

// ---------------------------------------------------------------- K1: tridiagonalisation
__global__ void __launch_bounds__(HEEV_THREADS) heev_tridiag(const HeevProblem* __restrict__ probs) {
  const HeevProblem P = probs[blockIdx.x];
  const int n = P.n;
  cplx* A = P.A;
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  extern __shared__ __align__(16) unsigned char smem_raw[];
  cplx* sv = reinterpret_cast<cplx*>(smem_raw);
  cplx* sp = sv + n;
  cplx* base = sp + n;
  __shared__ double2 red[HEEV_WARPS + 1];
  double* dvec = P.work;
  double* evec = P.work + n;
  double* sc = P.work + 2 * n;
  double tr = 0.0;
  for (int i = tid; i < n; i += HEEV_THREADS) tr += A[(size_t)i * n + i].x;
  const double trace = block_sum2(tr, 0.0, red).x;
  if (n <= SMEM_MAX_N) tridiag_fused<true>(A, n, sv, sp, base, dvec, evec, P.tau, red);
  else if (n <= FUSED_MAX_N) tridiag_fused<false>(A, n, sv, sp, base, dvec, evec, P.tau, red);
  else tridiag_full(A, n, sv, sp, dvec, evec, P.tau, red);
  // Gershgorin interval, pivmin (dstebz)
  double gl = 1e300, gu = -1e300, em = 0.0;
  for (int i = tid; i < n; i += HEEV_THREADS) {
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
  __shared__ double mm[3][HEEV_WARPS];
  if (lane == 0) { mm[0][warp] = gl; mm[1][warp] = gu; mm[2][warp] = em; }
  __syncthreads();
  if (tid == 0) {
    gl = mm[0][0]; gu = mm[1][0]; em = mm[2][0];
    for (int w = 1; w < HEEV_WARPS; ++w) { gl = fmin(gl, mm[0][w]); gu = fmax(gu, mm[1][w]); em = fmax(em, mm[2][w]); }
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

// ---------------------------------------------------------------- K2: eigenvalues
__global__ void heev_bisect(const HeevProblem* __restrict__ probs, int nprob, int total) {
  const int g = blockIdx.x * blockDim.x + threadIdx.x;
  if (g >= total) return;
  const HeevProblem& P = probs[find_estart(probs, nprob, g)];
  const int t = g - P.estart, n = P.n;
  const double* d = P.work;
  const double* e = P.work + n;
  const double* sc = P.work + 2 * n;
  const double pivmin = sc[S_PIVMIN], atol = sc[S_ATOL];
  const int idx = n - 1 - t;                   // ascending index of the t-th largest
  double lo = sc[S_GL], hi = sc[S_GU];
  for (int it = 0; it < 96; ++it) {
    if (hi - lo <= fmax(atol, 2.0 * DBL_EPSILON * fmax(fabs(lo), fabs(hi))) + pivmin) break;
    const double w = 0.25 * (hi - lo);
    const double x1 = lo + w, x2 = lo + 2.0 * w, x3 = lo + 3.0 * w;
    int c1, c2, c3;
    sturm_count3(d, e, n, x1, x2, x3, pivmin, c1, c2, c3);
    if (c1 > idx) hi = x1;
    else if (c2 > idx) { lo = x1; hi = x2; }
    else if (c3 > idx) { lo = x2; hi = x3; }
    else lo = x3;
  }
  P.lam[t] = 0.5 * (lo + hi);
}

// ---------------------------------------------------------------- K3: inverse iteration
__global__ void heev_invit(const HeevProblem* __restrict__ probs, int nprob, int total) {
  const int g = blockIdx.x * blockDim.x + threadIdx.x;
  if (g >= total) return;
  const HeevProblem& P = probs[find_estart(probs, nprob, g)];
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
  for (int it = 0; it < 3; ++it) {   // dgttrs, rescaled by the previous max
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

// ---------------------------------------------------------------- K4: CholeskyQR2 of Z
__global__ void __launch_bounds__(HEEV_THREADS) heev_orth(const HeevProblem* __restrict__ probs) {
  const HeevProblem P = probs[blockIdx.x];
  const int n = P.n, kmax = P.kmax, tid = threadIdx.x;
  const int k = P.k_out ? *P.k_out : kmax;   // only the kept directions are orthonormalised
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

// ---------------------------------------------------------------- K5: back-transform
__global__ void heev_backtr(const HeevProblem* __restrict__ probs, int nprob, int total) {
  const int gw = (blockIdx.x * blockDim.x + threadIdx.x) >> 5, lane = threadIdx.x & 31;
  if (gw >= total) return;
  const HeevProblem& P = probs[find_estart(probs, nprob, gw)];
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

// ---------------------------------------------------------------- K6: truncation decision
__global__ void heev_finish(const HeevProblem* __restrict__ probs, int nprob) {
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= nprob) return;
  const HeevProblem& P = probs[i];
  const int kmax = P.kmax;
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
  // clusters of close kept eigenvalues (gap <= 1e-3 ||T||, as LAPACK dstein): their vectors
  // are computed sequentially with reorthogonalisation (K3b), the others thread-parallel (K3a)
  double* cst = cluster_arrays(P);
  double* csz = cst + kmax;
  const double ortol = 1e-3 * P.work[2 * P.n + S_TNORM];
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
__global__ void __launch_bounds__(HEEV_THREADS) heev_invit_cluster(const HeevProblem* __restrict__ probs) {
  const HeevProblem P = probs[blockIdx.x];
  const int n = P.n, kmax = P.kmax, lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int k = P.k_out ? *P.k_out : kmax;
  const double* sd = P.work;
  const double* evec = P.work + n;
  const double tnorm = P.work[2 * n + S_TNORM];
  if (!(tnorm > 0.0)) return;
  double* Z = P.work + 2 * n + 8;
  const double* cst = cluster_arrays(P);
  const double* csz = cst + kmax;
  double* scr = const_cast<double*>(csz) + kmax + (size_t)warp * 6 * n;
  double* DL = scr;
  double* Dg = scr + n;
  double* DU = scr + 2 * n;
  double* DU2 = scr + 3 * n;
  double* PV = scr + 4 * n;
  double* y = scr + 5 * n;
  const double pert = DBL_EPSILON * tnorm;
  int ci = 0;
  for (int t0 = 0; t0 < k; ++t0) {
    if ((int)cst[t0] != t0 || csz[t0] < 2.0) continue;   // not the start of a multi-vector cluster
    if ((ci++ % HEEV_WARPS) != warp) continue;
    const int t1 = t0 + (int)csz[t0];
    for (int t = t0; t < t1; ++t) {
      double lam = P.lam[t];
      if (t > t0) lam = fmin(lam, P.lam[t - 1] - 10.0 * DBL_EPSILON * tnorm);   // keep shifts apart (dstein)
      if (lane == 0) {   // dgttrf of T - lam I
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
          Dg[i] = 1.0 / d_i;
          DU[i] = du_i;
          DU2[i] = du2;
          DL[i] = l;
          PV[i] = p;
          d_i = d_n;
          du_i = du_n;
        }
        if (fabs(d_i) < pert) d_i = copysign(pert, d_i == 0.0 ? 1.0 : d_i);
        Dg[n - 1] = 1.0 / d_i;
      }
      for (int i = lane; i < n; i += 32)
        y[i] = (double)(hash32((unsigned)(t * 7919 + i * 104729 + 12345)) & 0xffffff) / 16777216.0 - 0.5;
      __syncwarp();
      for (int it = 0; it < 4; ++it) {
        if (lane == 0) {   // dgttrs with overflow rescaling
          double cur = y[0];
          for (int i = 0; i < n - 1; ++i) {
            const double nxt = y[i + 1];
            if (PV[i] == 0.0) { y[i] = cur; cur = nxt - DL[i] * cur; }
            else { y[i] = nxt; cur = cur - DL[i] * nxt; }
          }
          double y2 = 0.0, y1 = cur * Dg[n - 1];
          y[n - 1] = y1;
          for (int i = n - 2; i >= 0; --i) {
            double yi = (y[i] - DU[i] * y1 - DU2[i] * y2) * Dg[i];
            if (fabs(yi) > 1e100) {
              for (int q = 0; q < n; ++q) if (q != i) y[q] *= 1e-100;
              yi *= 1e-100; y1 *= 1e-100; y2 *= 1e-100;
            }
            y[i] = yi;
            y2 = y1;
            y1 = yi;
          }
        }
        __syncwarp();
        double mx = 0.0;
        for (int i = lane; i < n; i += 32) mx = fmax(mx, fabs(y[i]));
        for (int o = 16; o > 0; o >>= 1) mx = fmax(mx, __shfl_xor_sync(0xffffffffu, mx, o));
        const double inv = mx > 0.0 ? 1.0 / mx : 1.0;
        for (int i = lane; i < n; i += 32) y[i] *= inv;
        __syncwarp();
        for (int rep = 0; rep < 2; ++rep)
          for (int q = t0; q < t; ++q) {   // MGS against the cluster's previous vectors
            double dt = 0.0;
            for (int i = lane; i < n; i += 32) dt += y[i] * Z[(size_t)i * kmax + q];
            dt = warp_sum(dt);
            for (int i = lane; i < n; i += 32) y[i] -= dt * Z[(size_t)i * kmax + q];
            __syncwarp();
          }
        double nr = 0.0;
        for (int i = lane; i < n; i += 32) nr += y[i] * y[i];
        nr = warp_sum(nr);
        if (!(nr > 1e-200)) {   // collapsed onto the previous vectors: restart from a new direction
          for (int i = lane; i < n; i += 32)
            y[i] = (double)(hash32((unsigned)(t * 31 + i * 7877 + it * 131071 + 99)) & 0xffffff) / 16777216.0 - 0.5;
          __syncwarp();
          continue;
        }
        const double s = 1.0 / sqrt(nr);
        for (int i = lane; i < n; i += 32) y[i] *= s;
        __syncwarp();
      }
      for (int q = t0; q < t; ++q) {   // final projection + normalisation
        double dt = 0.0;
        for (int i = lane; i < n; i += 32) dt += y[i] * Z[(size_t)i * kmax + q];
        dt = warp_sum(dt);
        for (int i = lane; i < n; i += 32) y[i] -= dt * Z[(size_t)i * kmax + q];
        __syncwarp();
      }
      double nr = 0.0;
      for (int i = lane; i < n; i += 32) nr += y[i] * y[i];
      nr = warp_sum(nr);
      const double s = nr > 0.0 ? 1.0 / sqrt(nr) : 0.0;
      for (int i = lane; i < n; i += 32) Z[(size_t)i * kmax + t] = y[i] * s;
      __syncwarp();
    }
  }
}

}  // namespace

size_t heev_work_doubles(int n, int kmax) {
  return (size_t)2 * n + 8 + (size_t)n * kmax * 6 + (size_t)kmax * kmax + 2 * (size_t)kmax +
         (size_t)HEEV_WARPS * 6 * n;
}

size_t heev_smem_bytes(int n, int kmax) {
  (void)kmax;
  size_t b = (size_t)n * 16 * 2;
  if (n <= FUSED_MAX_N) b += (size_t)16 * (3 + HEEV_WARPS) * n;
  if (n <= SMEM_MAX_N) b += (size_t)16 * n * (n + 1) / 2;
  return b + 64;
}

int heev_max_n() { return HEEV_MAX_N; }

void launch_heev(HeevProblem* h, int n, Stager& st, cudaStream_t s) {
  if (n == 0) return;
  static bool attr = false;
  if (!attr) {
    size_t mx = std::max(heev_smem_bytes(SMEM_MAX_N, 1), heev_smem_bytes(HEEV_MAX_N, 1));
    cudaFuncSetAttribute(heev_tridiag, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)mx);
    attr = true;
  }
  int total = 0;
  double fl = 0.0, by = 0.0;
  for (int i = 0; i < n; ++i) {
    h[i].estart = total;
    total += h[i].kmax;
    const double nn = h[i].n;
    fl += 8.0 * ((4.0 / 3.0) * nn * nn * nn + 2.0 * nn * nn * h[i].kmax);
    by += 16.0 * nn * nn;
  }
  const HeevProblem* d = static_cast<const HeevProblem*>(st.put(h, sizeof(HeevProblem) * n));
  prof_begin(s);
  // K1, one launch per storage mode so small-smem problems are not limited by large ones
  std::vector<HeevProblem> grp[3];
  for (int i = 0; i < n; ++i) grp[h[i].n <= SMEM_MAX_N ? 0 : (h[i].n <= FUSED_MAX_N ? 1 : 2)].push_back(h[i]);
  for (auto& g : grp) {
    if (g.empty()) continue;
    size_t smem = 0;
    for (auto& p : g) smem = std::max(smem, heev_smem_bytes(p.n, p.kmax));
    const HeevProblem* dg = static_cast<const HeevProblem*>(st.put(g.data(), sizeof(HeevProblem) * g.size()));
    heev_tridiag<<<(int)g.size(), HEEV_THREADS, smem, s>>>(dg);
    count_launch();
  }
  heev_bisect<<<(total + 127) / 128, 128, 0, s>>>(d, n, total);
  heev_finish<<<(n + 127) / 128, 128, 0, s>>>(d, n);   // k and w: only kept pairs go on
  heev_invit<<<(total + 127) / 128, 128, 0, s>>>(d, n, total);
  heev_invit_cluster<<<n, HEEV_THREADS, 0, s>>>(d);
  count_launch();
  heev_orth<<<n, HEEV_THREADS, 0, s>>>(d);
  heev_backtr<<<(total * 32 + 255) / 256, 256, 0, s>>>(d, n, total);
  count_launch(); count_launch(); count_launch(); count_launch(); count_launch();
  prof_end(s, "heev", fl, by);
}

}  // namespace tcbc
