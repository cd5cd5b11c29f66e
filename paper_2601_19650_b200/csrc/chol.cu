// Batched Cholesky factorisation and triangular inverse (B:5 (b)).
//
// The paper's central observation is that every positive tensor built by the
// density-matrix method is a product G = M^H M, "a Cholesky decomposition of G".  On the GPU
// the literal Cholesky runs where a Gram is factored:
//   * CholeskyQR2 of S^{[i]} for the QR of Eq. 13:  W = S^H S = L L^H,
//     Q = S L^{-H}, repeated once;
//   * residual / rank checks (a non-positive pivot flags a rank-deficient S).
// One CTA per matrix; right-looking column algorithm with the trailing Hermitian update
// spread over the CTA.
#include "kernels.h"
#include "prof.h"
#include <algorithm>
#include <cmath>
#include <vector>

namespace tcbc {

namespace {

__device__ __forceinline__ cplx cmul(cplx a, cplx b) { return make_double2(a.x * b.x - a.y * b.y, a.x * b.y + a.y * b.x); }
__device__ __forceinline__ cplx cmulc(cplx a, cplx b) {  // a * conj(b)
  return make_double2(a.x * b.x + a.y * b.y, a.y * b.x - a.x * b.y);
}
__device__ __forceinline__ cplx cdiv(cplx a, cplx b) {
  double den = b.x * b.x + b.y * b.y;
  return make_double2((a.x * b.x + a.y * b.y) / den, (a.y * b.x - a.x * b.y) / den);
}

// one DMMA (mma.sync m8n8k4 f64): {c0, c1} += a (8x4 row) * b (4x8 col), one element per lane
__device__ __forceinline__ void dmma8(double& c0, double& c1, double a, double b) {
  asm("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
      : "+d"(c0), "+d"(c1)
      : "d"(a), "d"(b));
}

__device__ double block_max(double v, double* red) {
  for (int o = 16; o > 0; o >>= 1) v = fmax(v, __shfl_xor_sync(0xffffffffu, v, o));
  if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = v;
  __syncthreads();
  if (threadIdx.x < 32) {
    v = (threadIdx.x < (blockDim.x >> 5)) ? red[threadIdx.x] : -1e300;
    for (int o = 16; o > 0; o >>= 1) v = fmax(v, __shfl_xor_sync(0xffffffffu, v, o));
    if (threadIdx.x == 0) red[0] = v;
  }
  __syncthreads();
  double r = red[0];
  __syncthreads();
  return r;
}

constexpr int CH_NB = 16;      // panel / row-block width
constexpr int CH_THREADS = 512;

// Blocked right-looking Cholesky (lower; B:5 (b)): for each 16-column panel, (1) the panel is
// staged in shared memory, (2) its 16 x 16 diagonal block is factored by one warp (lane =
// row), (3) the rows below are solved against L11^H (thread per row), (4) the panel is written
// back and the trailing lower triangle is updated once per panel (A22 -= P P^H) on the FP64
// tensor cores (DMMA), reading the staged panel (one global read-modify-write per element per
// panel instead of per column).  One CTA per matrix.
__global__ void __launch_bounds__(CH_THREADS) potrf_grouped(const PotrfProblem* __restrict__ probs) {
  TCBC_PDL_WAIT();
  const PotrfProblem P = probs[blockIdx.x];
  const int n = P.n;
  const long long ld = P.lda;
  cplx* A = P.A;
  extern __shared__ __align__(16) unsigned char ch_smem[];
  cplx* Pn = reinterpret_cast<cplx*>(ch_smem);   // [n][CH_NB]
  __shared__ double red[32];
  __shared__ int s_fail;
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  double md = -1e300;
  for (int i = tid; i < n; i += CH_THREADS) md = fmax(md, A[i * ld + i].x);
  md = block_max(md, red);
  if (P.shift_rel > 0.0 && md > 0.0) {
    const double sh = P.shift_rel * md;
    for (int i = tid; i < n; i += CH_THREADS) A[i * ld + i].x += sh;
    md += sh;
  }
  const double thresh = P.rel_tol * md;
  if (tid == 0) s_fail = (md > 0.0 && isfinite(md)) ? 0 : 1;
  __syncthreads();
  for (int j0 = 0; j0 < n && !s_fail; j0 += CH_NB) {
    const int jb = min(CH_NB, n - j0), rows = n - j0;
    for (int e = tid; e < rows * jb; e += CH_THREADS) {
      const int r = e / jb, c = e % jb;
      Pn[r * CH_NB + c] = A[(long long)(j0 + r) * ld + j0 + c];
    }
    __syncthreads();
    if (warp == 0) {   // diagonal block, unblocked, lane = row
      for (int c = 0; c < jb; ++c) {
        if (lane == c) {
          const double d = Pn[c * CH_NB + c].x;
          if (!(d > thresh) || !isfinite(d)) s_fail = j0 + c + 1;
          else Pn[c * CH_NB + c] = make_double2(sqrt(d), 0.0);
        }
        __syncwarp();
        if (s_fail) break;
        const double inv = 1.0 / Pn[c * CH_NB + c].x;
        if (lane > c && lane < jb) {
          const cplx v = Pn[lane * CH_NB + c];
          Pn[lane * CH_NB + c] = make_double2(v.x * inv, v.y * inv);
        }
        __syncwarp();
        if (lane > c && lane < jb) {
          const cplx lc = Pn[lane * CH_NB + c];
          for (int l = c + 1; l <= lane; ++l) {
            const cplx u = cmulc(lc, Pn[l * CH_NB + c]);
            Pn[lane * CH_NB + l].x -= u.x;
            Pn[lane * CH_NB + l].y -= u.y;
          }
        }
        __syncwarp();
      }
    }
    __syncthreads();
    if (s_fail) break;
    for (int r = jb + tid; r < rows; r += CH_THREADS) {   // x L11^H = p
      cplx x[CH_NB];
#pragma unroll
      for (int c = 0; c < CH_NB; ++c) {
        if (c >= jb) break;
        cplx v = Pn[r * CH_NB + c];
        for (int l = 0; l < c; ++l) {
          const cplx u = cmulc(x[l], Pn[c * CH_NB + l]);
          v.x -= u.x;
          v.y -= u.y;
        }
        const double inv = 1.0 / Pn[c * CH_NB + c].x;
        x[c] = make_double2(v.x * inv, v.y * inv);
        Pn[r * CH_NB + c] = x[c];
      }
    }
    __syncthreads();
    for (int e = tid; e < rows * jb; e += CH_THREADS) {
      const int r = e / jb, c = e % jb;
      if (c <= r) A[(long long)(j0 + r) * ld + j0 + c] = Pn[r * CH_NB + c];
    }
    // trailing update A22 -= P P^H on the FP64 tensor path: warp per 8x8 tile of the lower
    // triangle, 4 k-steps of DMMA m8n8k4 per complex product (4M rule), both operand
    // fragments read straight from the staged panel (B = conj(P)^T uses the same index map)
    const int t = rows - jb, tb = (t + 7) / 8;
    const int ntiles = tb * (tb + 1) / 2;
    const int fr = lane >> 2, fc = lane & 3;
    for (int e = warp; e < ntiles; e += CH_THREADS / 32) {
      int bi = (int)((sqrt(8.0 * e + 1.0) - 1.0) * 0.5);
      while (bi * (bi + 1) / 2 > e) --bi;
      while ((bi + 1) * (bi + 2) / 2 <= e) ++bi;
      const int bj = e - bi * (bi + 1) / 2;
      const int r0 = jb + 8 * bi, l0 = jb + 8 * bj;
      double cr0 = 0.0, cr1 = 0.0, ci0 = 0.0, ci1 = 0.0;
#pragma unroll
      for (int q = 0; q < CH_NB / 4; ++q) {
        const int k = q * 4 + fc;
        const cplx a = (r0 + fr < rows && k < jb) ? Pn[(r0 + fr) * CH_NB + k] : make_double2(0.0, 0.0);
        const cplx bb = (l0 + fr < rows && k < jb) ? Pn[(l0 + fr) * CH_NB + k] : make_double2(0.0, 0.0);
        const double br = bb.x, bim = -bb.y;   // B = conj(P_l)^T
        dmma8(cr0, cr1, a.x, br);
        dmma8(ci0, ci1, a.x, bim);
        dmma8(cr0, cr1, -a.y, bim);
        dmma8(ci0, ci1, a.y, br);
      }
      const int r = r0 + fr;
#pragma unroll
      for (int h = 0; h < 2; ++h) {
        const int l = l0 + 2 * fc + h;
        if (r < rows && l <= r) {
          cplx* p = A + (long long)(j0 + r) * ld + j0 + l;
          p->x -= h ? cr1 : cr0;
          p->y -= h ? ci1 : ci0;
        }
      }
    }
    __syncthreads();
  }
  __syncthreads();
  if (!s_fail) {
    for (long long e = tid; e < (long long)n * n; e += CH_THREADS) {
      int i = (int)(e / n), l = (int)(e % n);
      if (l > i) A[i * ld + l] = make_double2(0.0, 0.0);
    }
  }
  if (tid == 0 && P.info) *P.info = s_fail;
}

// Small orders (n <= 64, config 2's CholeskyQR Grams of order 64): the whole matrix in shared
// memory, unblocked right-looking Cholesky (two barriers per column) -- a sequential chain of
// 64 short steps instead of four panels of staged blocks.  Same outputs and info as above.
constexpr int CH_SMALL = 64;

__global__ void __launch_bounds__(256) potrf_small(const PotrfProblem* __restrict__ probs) {
  TCBC_PDL_WAIT();
  const PotrfProblem P = probs[blockIdx.x];
  const int n = P.n, ldS = n + 1;
  const long long ld = P.lda;
  cplx* A = P.A;
  extern __shared__ __align__(16) unsigned char ch_smem[];
  cplx* S = reinterpret_cast<cplx*>(ch_smem);   // [n][n + 1], lower triangle used
  __shared__ double red[32];
  __shared__ int s_fail;
  const int tid = threadIdx.x;
  double md = -1e300;
  for (int e = tid; e < n * n; e += 256) {
    const int r = e / n, c = e % n;
    if (c <= r) {
      const cplx v = A[r * ld + c];
      S[r * ldS + c] = v;
      if (c == r) md = fmax(md, v.x);
    }
  }
  md = block_max(md, red);   // (its barriers also publish S)
  if (P.shift_rel > 0.0 && md > 0.0) {
    const double sh = P.shift_rel * md;
    for (int i = tid; i < n; i += 256) S[i * ldS + i].x += sh;
    md += sh;
  }
  const double thresh = P.rel_tol * md;
  if (tid == 0) s_fail = (md > 0.0 && isfinite(md)) ? 0 : 1;
  __syncthreads();
  for (int c = 0; c < n && !s_fail; ++c) {
    const double d = S[c * ldS + c].x;
    if (!(d > thresh) || !isfinite(d)) {   // uniform: every thread reads the same pivot
      if (tid == 0) s_fail = c + 1;
      break;
    }
    const double sd = sqrt(d), inv = 1.0 / sd;
    for (int r = c + 1 + tid; r < n; r += 256) {
      const cplx v = S[r * ldS + c];
      S[r * ldS + c] = make_double2(v.x * inv, v.y * inv);
    }
    __syncthreads();
    if (tid == 0) S[c * ldS + c] = make_double2(sd, 0.0);
    // A22 -= l l^H (lower part): 16 x 16 thread grid over (row, column), no index division
    for (int r = c + 1 + (tid >> 4); r < n; r += 16) {
      const cplx lr = S[r * ldS + c];
      for (int l = c + 1 + (tid & 15); l <= r; l += 16) {
        const cplx u = cmulc(lr, S[l * ldS + c]);
        S[r * ldS + l].x -= u.x;
        S[r * ldS + l].y -= u.y;
      }
    }
    __syncthreads();
  }
  __syncthreads();
  if (!s_fail) {
    for (int e = tid; e < n * n; e += 256) {
      const int r = e / n, c = e % n;
      A[r * ld + c] = c <= r ? S[r * ldS + c] : make_double2(0.0, 0.0);
    }
  }
  if (tid == 0 && P.info) *P.info = s_fail;
}

// Linv = L^{-1} for n <= 64: L in shared memory, four lanes per column of Linv (forward
// substitution down the column, the column's inner products split over the four lanes and
// combined by shuffles; diagonal reciprocals precomputed).
__global__ void __launch_bounds__(4 * CH_SMALL) trtri_small(const TrtriProblem* __restrict__ probs) {
  TCBC_PDL_WAIT();
  const TrtriProblem P = probs[blockIdx.x];
  const int n = P.n, ldS = n + 1;
  const long long ld = P.ld;
  extern __shared__ __align__(16) unsigned char ch_smem[];
  cplx* L = reinterpret_cast<cplx*>(ch_smem);   // [n][n + 1]
  cplx* X = L + (size_t)n * ldS;                // [n][n + 1]: X[a][b] = Linv[a][b]
  cplx* R = X + (size_t)n * ldS;                // [n]: 1 / L[a][a]
  const int tid = threadIdx.x, b = tid >> 2, sub = tid & 3;
  for (int e = tid; e < n * n; e += 4 * CH_SMALL) {
    const int r = e / n, c = e % n;
    if (c <= r) L[r * ldS + c] = P.L[r * ld + c];
  }
  __syncthreads();
  for (int a = tid; a < n; a += 4 * CH_SMALL) R[a] = cdiv(make_double2(1.0, 0.0), L[a * ldS + a]);
  __syncthreads();
  // a warp holds columns b0 .. b0 + 7; all its lanes run the same rows a >= b0 (the shuffles
  // need every lane), a lane contributing only once a >= its own column
  const int b0 = (tid >> 5) * 8;
  if (b0 < n) {
    if (sub == 0 && b < n)
      for (int a = 0; a < b; ++a) X[a * ldS + b] = make_double2(0.0, 0.0);
    __syncwarp();
    for (int a = b0; a < n; ++a) {
      const bool act = b < n && a >= b;
      double sr = 0.0, si = 0.0;
      if (act)
        for (int j = b + sub; j < a; j += 4) {
          const cplx u = cmul(L[a * ldS + j], X[j * ldS + b]);
          sr += u.x;
          si += u.y;
        }
      sr += __shfl_xor_sync(0xffffffffu, sr, 1);
      si += __shfl_xor_sync(0xffffffffu, si, 1);
      sr += __shfl_xor_sync(0xffffffffu, sr, 2);
      si += __shfl_xor_sync(0xffffffffu, si, 2);
      if (act && sub == 0) X[a * ldS + b] = cmul(make_double2((a == b ? 1.0 : 0.0) - sr, -si), R[a]);
      __syncwarp();
    }
  }
  __syncthreads();
  for (int e = tid; e < n * n; e += 4 * CH_SMALL) {
    const int r = e / n, c = e % n;
    P.Linv[r * ld + c] = X[r * ldS + c];
  }
}

// Blocked triangular inverse Linv = L^{-1} (lower), by 16-row blocks top to bottom: the block's
// rows of L are staged in shared memory, one warp inverts the 16 x 16 diagonal block D, and
// every column c < R0 is formed as  Linv[R, c] = -D^{-1} sum_{j in [c, R0)} L[R, j] Linv[j, c]
// (thread per column, Linv rows already written read back coalesced).
__global__ void __launch_bounds__(CH_THREADS) trtri_grouped(const TrtriProblem* __restrict__ probs) {
  TCBC_PDL_WAIT();
  const TrtriProblem P = probs[blockIdx.x];
  const int n = P.n;
  const long long ld = P.ld;
  extern __shared__ __align__(16) unsigned char ch_smem[];
  cplx* Ls = reinterpret_cast<cplx*>(ch_smem);     // [CH_NB][n]
  __shared__ cplx Dinv[CH_NB][CH_NB + 1];
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  for (int R0 = 0; R0 < n; R0 += CH_NB) {
    const int rb = min(CH_NB, n - R0), w = R0 + rb;
    for (int e = tid; e < rb * w; e += CH_THREADS) {
      const int a = e / w, j = e % w;
      Ls[a * n + j] = P.L[(long long)(R0 + a) * ld + j];
    }
    __syncthreads();
    if (warp == 0 && lane < rb) {   // column lane of D^{-1}: forward substitution
      const int b = lane;
      for (int a = 0; a < rb; ++a) {
        cplx s = make_double2(a == b ? 1.0 : 0.0, 0.0);
        if (a < b) { Dinv[a][b] = make_double2(0.0, 0.0); continue; }
        for (int j = b; j < a; ++j) {
          const cplx u = cmul(Ls[a * n + R0 + j], Dinv[j][b]);
          s.x -= u.x;
          s.y -= u.y;
        }
        Dinv[a][b] = cdiv(s, Ls[a * n + R0 + a]);
      }
    }
    __syncthreads();
    for (int c = tid; c < n; c += CH_THREADS) {
      if (c < R0) {
        cplx acc[CH_NB];
#pragma unroll
        for (int a = 0; a < CH_NB; ++a) acc[a] = make_double2(0.0, 0.0);
        for (int j = c; j < R0; ++j) {
          const cplx lv = P.Linv[(long long)j * ld + c];
#pragma unroll
          for (int a = 0; a < CH_NB; ++a) {
            const cplx u = cmul(Ls[a * n + j], lv);   // rows a >= rb are never stored
            acc[a].x += u.x;
            acc[a].y += u.y;
          }
        }
#pragma unroll
        for (int a = 0; a < CH_NB; ++a) {
          if (a >= rb) break;
          cplx v = make_double2(0.0, 0.0);
#pragma unroll
          for (int b = 0; b <= a; ++b) {
            const cplx u = cmul(Dinv[a][b], acc[b]);
            v.x -= u.x;
            v.y -= u.y;
          }
          P.Linv[(long long)(R0 + a) * ld + c] = v;
        }
      } else {
        for (int a = 0; a < rb; ++a)
          P.Linv[(long long)(R0 + a) * ld + c] = (c < w) ? Dinv[a][c - R0] : make_double2(0.0, 0.0);
      }
    }
    __syncthreads();
  }
}

// Householder QR (zgeqr2) of a tall m x k matrix A (row-major, ld k; destroyed) and the
// thin Q = H_0 ... H_{k-1} [I; 0] written to Q (ld k).  Used for the S of Eq. 13 when
// CholeskyQR2 flags a rank-deficient S (circuit layers, zero states): Householder gives an
// isometry Q spanning range(S) for any rank, as the oracle's LAPACK QR does.
__global__ void __launch_bounds__(256) geqr_q_grouped(const GeqrProblem* __restrict__ probs) {
  TCBC_PDL_WAIT();
  const GeqrProblem P = probs[blockIdx.x];
  const int m = P.m, k = P.k;
  cplx* A = P.A;
  cplx* Q = P.Q;
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  __shared__ double red[32];
  __shared__ cplx cred[8][33];
  __shared__ cplx s_w[32];
  for (int j = 0; j < k; ++j) {
    double part = 0.0;
    for (int i = j + 1 + tid; i < m; i += 256) {
      cplx x = A[(size_t)i * k + j];
      part += x.x * x.x + x.y * x.y;
    }
    for (int o = 16; o > 0; o >>= 1) part += __shfl_xor_sync(0xffffffffu, part, o);
    if (lane == 0) red[warp] = part;
    __syncthreads();
    double xn2 = 0.0;
    for (int w = 0; w < 8; ++w) xn2 += red[w];
    const cplx alpha = A[(size_t)j * k + j];
    cplx tau = make_double2(0.0, 0.0), scale = make_double2(0.0, 0.0);
    if (!(xn2 == 0.0 && alpha.y == 0.0)) {
      const double beta = -copysign(sqrt(alpha.x * alpha.x + alpha.y * alpha.y + xn2), alpha.x);
      tau = make_double2((beta - alpha.x) / beta, -alpha.y / beta);
      const cplx den = make_double2(alpha.x - beta, alpha.y);
      const double dd = den.x * den.x + den.y * den.y;
      scale = make_double2(den.x / dd, -den.y / dd);
    }
    __syncthreads();
    if (tid == 0) P.tau[j] = tau;
    for (int i = j + 1 + tid; i < m; i += 256) A[(size_t)i * k + j] = cmul(A[(size_t)i * k + j], scale);
    if (tid == 0) A[(size_t)j * k + j] = make_double2(1.0, 0.0);   // v_j = 1 (R_jj not needed)
    __syncthreads();
    if (tau.x == 0.0 && tau.y == 0.0) continue;
    const cplx ctau = make_double2(tau.x, -tau.y);
    for (int c0 = j + 1; c0 < k; c0 += 32) {   // A[j:, j+1:] -= conj(tau) v (v^H A)
      const int c = c0 + lane;
      cplx s = make_double2(0.0, 0.0);
      if (c < k)
        for (int i = j + warp; i < m; i += 8) {
          cplx v = A[(size_t)i * k + j], a = A[(size_t)i * k + c];
          s.x += v.x * a.x + v.y * a.y;
          s.y += v.x * a.y - v.y * a.x;
        }
      cred[warp][lane] = s;
      __syncthreads();
      if (warp == 0) {
        cplx t = make_double2(0.0, 0.0);
        for (int w = 0; w < 8; ++w) { t.x += cred[w][lane].x; t.y += cred[w][lane].y; }
        s_w[lane] = cmul(ctau, t);
      }
      __syncthreads();
      if (c < k) {
        const cplx w = s_w[lane];
        for (int i = j + warp; i < m; i += 8) {
          cplx v = A[(size_t)i * k + j];
          cplx u = cmul(v, w);
          cplx a = A[(size_t)i * k + c];
          A[(size_t)i * k + c] = make_double2(a.x - u.x, a.y - u.y);
        }
      }
      __syncthreads();
    }
  }
  for (size_t e = tid; e < (size_t)m * k; e += 256) {
    int i = (int)(e / k), c = (int)(e % k);
    Q[e] = make_double2(i == c ? 1.0 : 0.0, 0.0);
  }
  __syncthreads();
  for (int j = k - 1; j >= 0; --j) {   // Q = H_j Q on columns c >= j
    const cplx tau = P.tau[j];
    if (tau.x == 0.0 && tau.y == 0.0) continue;
    for (int c0 = j; c0 < k; c0 += 32) {
      const int c = c0 + lane;
      cplx s = make_double2(0.0, 0.0);
      if (c < k)
        for (int i = j + warp; i < m; i += 8) {
          cplx v = A[(size_t)i * k + j], q = Q[(size_t)i * k + c];
          s.x += v.x * q.x + v.y * q.y;
          s.y += v.x * q.y - v.y * q.x;
        }
      cred[warp][lane] = s;
      __syncthreads();
      if (warp == 0) {
        cplx t = make_double2(0.0, 0.0);
        for (int w = 0; w < 8; ++w) { t.x += cred[w][lane].x; t.y += cred[w][lane].y; }
        s_w[lane] = cmul(tau, t);
      }
      __syncthreads();
      if (c < k) {
        const cplx w = s_w[lane];
        for (int i = j + warp; i < m; i += 8) {
          cplx v = A[(size_t)i * k + j];
          cplx u = cmul(v, w);
          cplx q = Q[(size_t)i * k + c];
          Q[(size_t)i * k + c] = make_double2(q.x - u.x, q.y - u.y);
        }
      }
      __syncthreads();
    }
  }
}


// potrf_small followed by trtri_small in the same CTA (orders <= 64): the factor stays in
// shared memory between the two, one launch instead of two (latency-bound QR / certificate
// levels of the small-tree configs)
__global__ void __launch_bounds__(256) potri_small(const PotriProblem* __restrict__ probs) {
  TCBC_PDL_WAIT();
  const PotriProblem P = probs[blockIdx.x];
  const int n = P.n, ldS = n + 1;
  const long long ld = P.lda;
  cplx* A = P.A;
  extern __shared__ __align__(16) unsigned char ch_smem[];
  cplx* S = reinterpret_cast<cplx*>(ch_smem);   // [n][n + 1], lower triangle: L
  cplx* X = S + (size_t)n * ldS;                // [n][n + 1]: L^{-1}
  cplx* R = X + (size_t)n * ldS;                // [n]: 1 / L[a][a]
  __shared__ double red[32];
  __shared__ int s_fail;
  const int tid = threadIdx.x;
  double md = -1e300;
  for (int e = tid; e < n * n; e += 256) {
    const int r = e / n, c = e % n;
    if (c <= r) {
      const cplx v = A[r * ld + c];
      S[r * ldS + c] = v;
      if (c == r) md = fmax(md, v.x);
    }
  }
  md = block_max(md, red);
  if (P.shift_rel > 0.0 && md > 0.0) {
    const double sh = P.shift_rel * md;
    for (int i = tid; i < n; i += 256) S[i * ldS + i].x += sh;
    md += sh;
  }
  const double thresh = P.rel_tol * md;
  if (tid == 0) s_fail = (md > 0.0 && isfinite(md)) ? 0 : 1;
  __syncthreads();
  for (int c = 0; c < n && !s_fail; ++c) {
    const double d = S[c * ldS + c].x;
    if (!(d > thresh) || !isfinite(d)) {
      if (tid == 0) s_fail = c + 1;
      break;
    }
    const double sd = sqrt(d), inv = 1.0 / sd;
    for (int r = c + 1 + tid; r < n; r += 256) {
      const cplx v = S[r * ldS + c];
      S[r * ldS + c] = make_double2(v.x * inv, v.y * inv);
    }
    __syncthreads();
    if (tid == 0) S[c * ldS + c] = make_double2(sd, 0.0);
    for (int r = c + 1 + (tid >> 4); r < n; r += 16) {
      const cplx lr = S[r * ldS + c];
      for (int l = c + 1 + (tid & 15); l <= r; l += 16) {
        const cplx u = cmulc(lr, S[l * ldS + c]);
        S[r * ldS + l].x -= u.x;
        S[r * ldS + l].y -= u.y;
      }
    }
    __syncthreads();
  }
  __syncthreads();
  if (tid == 0 && P.info) *P.info = s_fail;
  if (s_fail) return;   // uniform
  if (P.write_l)
    for (int e = tid; e < n * n; e += 256) {
      const int r = e / n, c = e % n;
      A[r * ld + c] = c <= r ? S[r * ldS + c] : make_double2(0.0, 0.0);
    }
  for (int a = tid; a < n; a += 256) R[a] = cdiv(make_double2(1.0, 0.0), S[a * ldS + a]);
  __syncthreads();
  const int b = tid >> 2, sub = tid & 3, b0 = (tid >> 5) * 8;
  if (b0 < n) {
    if (sub == 0 && b < n)
      for (int a = 0; a < b; ++a) X[a * ldS + b] = make_double2(0.0, 0.0);
    __syncwarp();
    for (int a = b0; a < n; ++a) {
      const bool act = b < n && a >= b;
      double sr = 0.0, si = 0.0;
      if (act)
        for (int j = b + sub; j < a; j += 4) {
          const cplx u = cmul(S[a * ldS + j], X[j * ldS + b]);
          sr += u.x;
          si += u.y;
        }
      sr += __shfl_xor_sync(0xffffffffu, sr, 1);
      si += __shfl_xor_sync(0xffffffffu, si, 1);
      sr += __shfl_xor_sync(0xffffffffu, sr, 2);
      si += __shfl_xor_sync(0xffffffffu, si, 2);
      if (act && sub == 0) X[a * ldS + b] = cmul(make_double2((a == b ? 1.0 : 0.0) - sr, -si), R[a]);
      __syncwarp();
    }
  }
  __syncthreads();
  for (int e = tid; e < n * n; e += 256) {
    const int r = e / n, c = e % n;
    P.Linv[r * ld + c] = X[r * ldS + c];
  }
}

// one CTA per Gram: ||Li||_F^2 over the lower triangle and tr W, then the certificate
__global__ void __launch_bounds__(256) chol_certify(const CertProblem* __restrict__ probs) {
  TCBC_PDL_WAIT();
  const CertProblem P = probs[blockIdx.x];
  __shared__ double red[32];
  const int n = P.n;
  double s = 0.0, tr = 0.0;
  for (long long g = threadIdx.x; g < (long long)n * n; g += blockDim.x) {
    const int i = (int)(g / n), j = (int)(g % n);
    if (j <= i) {
      const cplx v = P.Li[g];
      s += v.x * v.x + v.y * v.y;
    }
  }
  for (int i = threadIdx.x; i < n; i += blockDim.x) tr += P.W[(size_t)i * n + i].x;
  for (int o = 16; o > 0; o >>= 1) {
    s += __shfl_xor_sync(0xffffffffu, s, o);
    tr += __shfl_xor_sync(0xffffffffu, tr, o);
  }
  if ((threadIdx.x & 31) == 0) {
    red[threadIdx.x >> 5] = s;
    red[16 + (threadIdx.x >> 5)] = tr;
  }
  __syncthreads();
  if (threadIdx.x == 0) {
    double S = 0.0, T = 0.0;
    for (int w = 0; w < (int)(blockDim.x >> 5); ++w) {
      S += red[w];
      T += red[16 + w];
    }
    const bool ok = *P.info == 0 && S > 0.0 && T > 0.0 && isfinite(S) && isfinite(T) && 1.0 / (S * T) >= P.thresh;
    *P.skip = ok ? 1 : 0;
  }
}

__global__ void exact_factor(const ExactFactorProblem* __restrict__ probs) {
  TCBC_PDL_WAIT();
  const ExactFactorProblem P = probs[blockIdx.y];
  if (!*P.skip) return;
  const double sc = (P.mode == 0 && P.exp2) ? ldexp(1.0, pow2_effective(*P.exp2)) : 1.0;
  const long long tot = (long long)P.rows * P.cols;
  for (long long g = blockIdx.x * (long long)blockDim.x + threadIdx.x; g < tot; g += (long long)gridDim.x * blockDim.x) {
    const int t = (int)(g / P.cols), c = (int)(g % P.cols);
    cplx v;
    if (P.mode == 0) {
      v = c >= t ? P.src[(size_t)c * P.cols + t] : make_double2(0.0, 0.0);
      v.x *= sc;
      v.y *= -sc;   // F = 2^e L^H
    } else {
      v = P.src[g];
    }
    P.F[g] = v;
  }
}

}  // namespace

void launch_chol_certify(CertProblem* h, int n, Stager& st, cudaStream_t s) {
  if (n == 0) return;
  const CertProblem* d = static_cast<const CertProblem*>(st.put(h, sizeof(CertProblem) * n));
  prof_begin(s);
  launch_k(chol_certify, n, 256, 0, s, d);
  prof_end(s, "potrf", 0.0, 0.0);
  count_launch();
}

void launch_exact_factor(ExactFactorProblem* h, int n, Stager& st, cudaStream_t s) {
  if (n == 0) return;
  long long mx = 1;
  for (int i = 0; i < n; ++i) mx = std::max<long long>(mx, (long long)h[i].rows * h[i].cols);
  const ExactFactorProblem* d = static_cast<const ExactFactorProblem*>(st.put(h, sizeof(ExactFactorProblem) * n));
  prof_begin(s);
  launch_k(exact_factor, dim3((unsigned)std::min<long long>((mx + 255) / 256, 64), n), 256, 0, s, d);
  prof_end(s, "misc", 0.0, 32.0 * (double)mx * n);
  count_launch();
}

void launch_potri(PotriProblem* h, int n, Stager& st, cudaStream_t s) {
  if (n == 0) return;
  int mx = 1;
  for (int i = 0; i < n; ++i) mx = std::max(mx, h[i].n);
  if (mx > CH_SMALL) {   // blocked kernels, two launches
    std::vector<PotrfProblem> pf(n);
    std::vector<TrtriProblem> tr(n);
    for (int i = 0; i < n; ++i) {
      pf[i] = PotrfProblem{h[i].A, h[i].lda, h[i].n, 0, h[i].info, h[i].rel_tol, h[i].shift_rel};
      tr[i] = TrtriProblem{h[i].A, h[i].Linv, h[i].lda, h[i].n, 0};
    }
    launch_potrf(pf.data(), n, st, s);
    launch_trtri(tr.data(), n, st, s);
    return;
  }
  const PotriProblem* d = static_cast<const PotriProblem*>(st.put(h, sizeof(PotriProblem) * n));
  double fl = 0.0;
  for (int i = 0; i < n; ++i) fl += 8.0 * 2.0 * (double)h[i].n * h[i].n * h[i].n / 6.0;
  const size_t sm = (2 * (size_t)mx * (mx + 1) + mx) * sizeof(cplx);
  func_smem(potri_small, (2 * (size_t)CH_SMALL * (CH_SMALL + 1) + CH_SMALL) * sizeof(cplx));
  prof_begin(s);
  launch_k(potri_small, n, 256, sm, s, d);
  prof_end(s, "potrf", fl, 0.0);
  count_launch();
}

void launch_geqr_q(GeqrProblem* h, int n, Stager& st, cudaStream_t s) {
  if (n == 0) return;
  const GeqrProblem* d = static_cast<const GeqrProblem*>(st.put(h, sizeof(GeqrProblem) * n));
  double fl = 0.0;
  for (int i = 0; i < n; ++i) fl += 16.0 * (double)h[i].m * h[i].k * h[i].k;
  prof_begin(s);
  launch_k(geqr_q_grouped, n, 256, 0, s, d);
  prof_end(s, "geqr", fl, 0.0);
  count_launch();
}

void launch_potrf(PotrfProblem* h, int n, Stager& st, cudaStream_t s) {
  if (n == 0) return;
  const PotrfProblem* d = static_cast<const PotrfProblem*>(st.put(h, sizeof(PotrfProblem) * n));
  double fl = 0.0;
  for (int i = 0; i < n; ++i) fl += 8.0 * (double)h[i].n * h[i].n * h[i].n / 6.0;
  int mx = 1;
  for (int i = 0; i < n; ++i) mx = std::max(mx, h[i].n);
  const size_t smem = (size_t)mx * CH_NB * sizeof(cplx);
  if (mx > CH_SMALL) func_smem(potrf_grouped, std::max<size_t>(smem, 48 << 10));
  prof_begin(s);
  if (mx <= CH_SMALL) {
    const size_t sm = (size_t)mx * (mx + 1) * sizeof(cplx);
    func_smem(potrf_small, (size_t)CH_SMALL * (CH_SMALL + 1) * sizeof(cplx));
    launch_k(potrf_small, n, 256, sm, s, d);
  } else {
    launch_k(potrf_grouped, n, CH_THREADS, smem, s, d);
  }
  prof_end(s, "potrf", fl, 0.0);
  count_launch();
}

void launch_trtri(TrtriProblem* h, int n, Stager& st, cudaStream_t s) {
  if (n == 0) return;
  const TrtriProblem* d = static_cast<const TrtriProblem*>(st.put(h, sizeof(TrtriProblem) * n));
  double fl = 0.0;
  for (int i = 0; i < n; ++i) fl += 8.0 * (double)h[i].n * h[i].n * h[i].n / 6.0;
  int mx = 1;
  for (int i = 0; i < n; ++i) mx = std::max(mx, h[i].n);
  const size_t smem = (size_t)mx * CH_NB * sizeof(cplx);
  if (mx > CH_SMALL) func_smem(trtri_grouped, std::max<size_t>(smem, 48 << 10));
  prof_begin(s);
  if (mx <= CH_SMALL) {
    const size_t sm = (2 * (size_t)mx * (mx + 1) + mx) * sizeof(cplx);
    func_smem(trtri_small, (2 * (size_t)CH_SMALL * (CH_SMALL + 1) + CH_SMALL) * sizeof(cplx));
    launch_k(trtri_small, n, 4 * CH_SMALL, sm, s, d);
  } else {
    launch_k(trtri_grouped, n, CH_THREADS, smem, s, d);
  }
  prof_end(s, "trtri", fl, 0.0);
  count_launch();
}

}  // namespace tcbc
