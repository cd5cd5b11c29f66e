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
#include <cmath>

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

__global__ void __launch_bounds__(256) potrf_grouped(const PotrfProblem* __restrict__ probs) {
  const PotrfProblem P = probs[blockIdx.x];
  const int n = P.n;
  const long long ld = P.lda;
  cplx* A = P.A;
  __shared__ double red[32];
  __shared__ int s_fail;
  double md = -1e300;
  for (int i = threadIdx.x; i < n; i += blockDim.x) md = fmax(md, A[i * ld + i].x);
  md = block_max(md, red);
  if (P.shift_rel > 0.0 && md > 0.0) {
    const double sh = P.shift_rel * md;
    for (int i = threadIdx.x; i < n; i += blockDim.x) A[i * ld + i].x += sh;
    md += sh;
    __syncthreads();
  }
  const double thresh = P.rel_tol * md;
  if (threadIdx.x == 0) s_fail = (md > 0.0 && isfinite(md)) ? 0 : 1;
  __syncthreads();
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5, nw = blockDim.x >> 5;
  for (int j = 0; j < n && !s_fail; ++j) {
    if (threadIdx.x == 0) {
      double ajj = A[j * ld + j].x;
      if (!(ajj > thresh) || !isfinite(ajj)) s_fail = j + 1;
      else A[j * ld + j] = make_double2(sqrt(ajj), 0.0);
    }
    __syncthreads();
    if (s_fail) break;
    const double inv = 1.0 / A[j * ld + j].x;
    for (int i = j + 1 + threadIdx.x; i < n; i += blockDim.x) {
      cplx v = A[i * ld + j];
      A[i * ld + j] = make_double2(v.x * inv, v.y * inv);
    }
    __syncthreads();
    for (int i = j + 1 + warp; i < n; i += nw) {
      const cplx lij = A[i * ld + j];
      for (int l = j + 1 + lane; l <= i; l += 32) {
        cplx llj = A[l * ld + j];
        cplx u = cmulc(lij, llj);
        cplx a = A[i * ld + l];
        A[i * ld + l] = make_double2(a.x - u.x, a.y - u.y);
      }
    }
    __syncthreads();
  }
  __syncthreads();
  if (!s_fail) {
    for (long long e = threadIdx.x; e < (long long)n * n; e += blockDim.x) {
      int i = (int)(e / n), l = (int)(e % n);
      if (l > i) A[i * ld + l] = make_double2(0.0, 0.0);
    }
  }
  if (threadIdx.x == 0 && P.info) *P.info = s_fail;
}

__global__ void __launch_bounds__(256) trtri_grouped(const TrtriProblem* __restrict__ probs) {
  const TrtriProblem P = probs[blockIdx.x];
  const int n = P.n;
  const long long ld = P.ld;
  for (int c = threadIdx.x; c < n; c += blockDim.x) {
    for (int i = 0; i < c; ++i) P.Linv[i * ld + c] = make_double2(0.0, 0.0);
    for (int i = c; i < n; ++i) {
      cplx s = make_double2(i == c ? 1.0 : 0.0, 0.0);
      for (int j = c; j < i; ++j) {
        cplx u = cmul(P.L[i * ld + j], P.Linv[j * ld + c]);
        s.x -= u.x;
        s.y -= u.y;
      }
      P.Linv[i * ld + c] = cdiv(s, P.L[i * ld + i]);
    }
  }
}

// Householder QR (zgeqr2) of a tall m x k matrix A (row-major, ld k; destroyed) and the
// thin Q = H_0 ... H_{k-1} [I; 0] written to Q (ld k).  Used for the S of Eq. 13 when
// CholeskyQR2 flags a rank-deficient S (circuit layers, zero states): Householder gives an
// isometry Q spanning range(S) for any rank, as the oracle's LAPACK QR does.
__global__ void __launch_bounds__(256) geqr_q_grouped(const GeqrProblem* __restrict__ probs) {
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

}  // namespace

void launch_geqr_q(GeqrProblem* h, int n, Stager& st, cudaStream_t s) {
  if (n == 0) return;
  const GeqrProblem* d = static_cast<const GeqrProblem*>(st.put(h, sizeof(GeqrProblem) * n));
  double fl = 0.0;
  for (int i = 0; i < n; ++i) fl += 16.0 * (double)h[i].m * h[i].k * h[i].k;
  prof_begin(s);
  geqr_q_grouped<<<n, 256, 0, s>>>(d);
  prof_end(s, "geqr", fl, 0.0);
  count_launch();
}

void launch_potrf(PotrfProblem* h, int n, Stager& st, cudaStream_t s) {
  if (n == 0) return;
  const PotrfProblem* d = static_cast<const PotrfProblem*>(st.put(h, sizeof(PotrfProblem) * n));
  double fl = 0.0;
  for (int i = 0; i < n; ++i) fl += 8.0 * (double)h[i].n * h[i].n * h[i].n / 6.0;
  prof_begin(s);
  potrf_grouped<<<n, 256, 0, s>>>(d);
  prof_end(s, "potrf", fl, 0.0);
  count_launch();
}

void launch_trtri(TrtriProblem* h, int n, Stager& st, cudaStream_t s) {
  if (n == 0) return;
  const TrtriProblem* d = static_cast<const TrtriProblem*>(st.put(h, sizeof(TrtriProblem) * n));
  double fl = 0.0;
  for (int i = 0; i < n; ++i) fl += 8.0 * (double)h[i].n * h[i].n * h[i].n / 6.0;
  prof_begin(s);
  trtri_grouped<<<n, 256, 0, s>>>(d);
  prof_end(s, "trtri", fl, 0.0);
  count_launch();
}

}  // namespace tcbc
