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

}  // namespace

void launch_potrf(PotrfProblem* h, int n, Stager& st, cudaStream_t s) {
  if (n == 0) return;
  const PotrfProblem* d = static_cast<const PotrfProblem*>(st.put(h, sizeof(PotrfProblem) * n));
  potrf_grouped<<<n, 256, 0, s>>>(d);
  count_launch();
}

void launch_trtri(TrtriProblem* h, int n, Stager& st, cudaStream_t s) {
  if (n == 0) return;
  const TrtriProblem* d = static_cast<const TrtriProblem*>(st.put(h, sizeof(TrtriProblem) * n));
  trtri_grouped<<<n, 256, 0, s>>>(d);
  count_launch();
}

}  // namespace tcbc
