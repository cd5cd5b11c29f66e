// Batched Hermitian eigensolver with truncation (B:5 (c); "compressed down to
// the desired new bond dimension D-bar, for example via singular value decomposition";
// P:362 tolerance).  For a compress input X (m x n) the GPU forms the smaller Gram
// (X^H X or X X^H, whose eigenpairs are the squared singular values and singular vectors of X;
// reading A1/A2 in DESIGN.md) and needs only its top-kmax eigenpairs.
//
// One CTA (8 warps) per matrix, all matrices of a sweep level in one launch:
//  1. Householder tridiagonalisation Q^H A Q = T (real symmetric tridiagonal; the complex
//     reflector makes every off-diagonal real), unblocked, full storage kept Hermitian.
//  2. Top-kmax eigenvalues of T by warp-parallel multisection of Sturm counts
//     (32 shifts per step: ~10 steps to machine precision).
//  3. Eigenvectors of T by inverse iteration (tridiagonal LU with partial pivoting), with
//     modified Gram-Schmidt inside clusters of close eigenvalues (gap < 1e-3 ||T||), as in
//     LAPACK's dstein.
//  4. Back-transform V = Q Z by the stored reflectors (warp per eigenvector).
//  5. Truncation decision k = min(max_bond, #{lam > tol^2 lam_1}, #{lam > floor lam_1}) >= 1
//     and discarded weight w = trace(A) - sum_{t<k} lam_t.
#include "kernels.h"
#include "prof.h"
#include <cfloat>
#include <cmath>

namespace tcbc {

namespace {

constexpr int HEEV_THREADS = 256;
constexpr int HEEV_WARPS = HEEV_THREADS / 32;
constexpr int HEEV_MAX_N = 2048;

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

// number of eigenvalues of T (d, e2 = e^2) strictly below x (LAPACK dlaebz recurrence)
__device__ __forceinline__ int sturm_count(const double* __restrict__ d, const double* __restrict__ e2,
                                           int n, double x, double pivmin) {
  int cnt = 0;
  double q = d[0] - x;
  if (q <= pivmin) { ++cnt; q = fmin(q, -pivmin); }
  for (int i = 1; i < n; ++i) {
    q = d[i] - x - e2[i - 1] / q;
    if (q <= pivmin) { ++cnt; q = fmin(q, -pivmin); }
  }
  return cnt;
}

__global__ void __launch_bounds__(HEEV_THREADS) heev_grouped(const HeevProblem* __restrict__ probs) {
  const HeevProblem P = probs[blockIdx.x];
  const int n = P.n, kmax = P.kmax;
  cplx* A = P.A;
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;

  extern __shared__ __align__(16) unsigned char smem_raw[];
  cplx* sv = reinterpret_cast<cplx*>(smem_raw);       // reflector v (n)
  cplx* sp = sv + n;                                   // p / w (n)
  double* sd = reinterpret_cast<double*>(sp + n);      // diag of T (n)
  double* se2 = sd + n;                                // e^2 (n)
  int* cstart = reinterpret_cast<int*>(se2 + n);       // cluster starts (kmax + 1)
  __shared__ double2 red[HEEV_WARPS + 1];
  __shared__ int s_ncl;

  double* dvec = P.work;            // n
  double* evec = P.work + n;        // n
  double* Z = P.work + 2 * n;       // kmax x n (eigenvectors of T)
  double* wscr = Z + (size_t)kmax * n + (size_t)warp * 6 * n;   // per-warp: DL D DU DU2 ipiv y

  // ---- trace of A (sum of the real diagonal)
  double tr = 0.0;
  for (int i = tid; i < n; i += HEEV_THREADS) tr += A[(size_t)i * n + i].x;
  const double trace = block_sum2(tr, 0.0, red).x;

  // ---- 1. tridiagonalisation (zhetd2, lower, full storage)
  for (int j = 0; j < n - 1; ++j) {
    const int len = n - j - 1;
    const cplx* col = A + (size_t)(j + 1) * n + j;      // x_i = col[i * n]
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
      const cplx den = make_double2(alpha.x - beta, alpha.y);          // 1 / (alpha - beta)
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
      A[(size_t)j * n + j + 1 + i] = v;                  // keep v_j in row j (unused from now on)
    }
    if (tid == 0) {
      evec[j] = beta;
      dvec[j] = A[(size_t)j * n + j].x;
      P.tau[j] = tau;
    }
    __syncthreads();
    if (tau.x == 0.0 && tau.y == 0.0) continue;
    cplx* A22 = A + (size_t)(j + 1) * n + (j + 1);
    // p = tau * A22 v
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
    // alpha2 = -1/2 tau (p^H v)
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
    // A22 -= v w^H + w v^H
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

  // ---- 2. eigenvalues (top kmax) by multisection
  double gl = 1e300, gu = -1e300, em = 0.0;
  for (int i = tid; i < n; i += HEEV_THREADS) {
    double di = dvec[i], ei = (i < n - 1) ? evec[i] : 0.0, ep = (i > 0) ? evec[i - 1] : 0.0;
    sd[i] = di;
    se2[i] = ei * ei;
    double rad = fabs(ei) + fabs(ep);
    gl = fmin(gl, di - rad);
    gu = fmax(gu, di + rad);
    em = fmax(em, ei * ei);
  }
  {  // block min / max via the sum helper on negated / positive maxima
    for (int o = 16; o > 0; o >>= 1) {
      gl = fmin(gl, __shfl_xor_sync(0xffffffffu, gl, o));
      gu = fmax(gu, __shfl_xor_sync(0xffffffffu, gu, o));
      em = fmax(em, __shfl_xor_sync(0xffffffffu, em, o));
    }
    __shared__ double mm[3][HEEV_WARPS];
    if (lane == 0) { mm[0][warp] = gl; mm[1][warp] = gu; mm[2][warp] = em; }
    __syncthreads();
    gl = mm[0][0]; gu = mm[1][0]; em = mm[2][0];
    for (int w = 1; w < HEEV_WARPS; ++w) { gl = fmin(gl, mm[0][w]); gu = fmax(gu, mm[1][w]); em = fmax(em, mm[2][w]); }
    __syncthreads();
  }
  const double tnorm = fmax(fabs(gl), fabs(gu));
  const double pivmin = DBL_MIN * fmax(1.0, em);
  gl -= 2.0 * DBL_EPSILON * tnorm * n + 2.0 * pivmin;
  gu += 2.0 * DBL_EPSILON * tnorm * n + 2.0 * pivmin;
  const double atol = 4.0 * DBL_EPSILON * tnorm;
  for (int t = warp; t < kmax; t += HEEV_WARPS) {
    const int idx = n - 1 - t;                 // ascending index of the t-th largest
    double lo = gl, hi = gu;
    for (int it = 0; it < 64; ++it) {
      if (hi - lo <= fmax(atol, 2.0 * DBL_EPSILON * fmax(fabs(lo), fabs(hi))) + pivmin) break;
      const double x = lo + (hi - lo) * (double)(lane + 1) / 33.0;
      const int c = sturm_count(sd, se2, n, x, pivmin);
      const unsigned m = __ballot_sync(0xffffffffu, c > idx);
      if (m == 0u) {
        lo = __shfl_sync(0xffffffffu, x, 31);
      } else {
        const int f = __ffs(m) - 1;
        const double xf = __shfl_sync(0xffffffffu, x, f);
        const double xp = __shfl_sync(0xffffffffu, x, f > 0 ? f - 1 : 0);
        if (f > 0) lo = xp;
        hi = xf;
      }
    }
    if (lane == 0) P.lam[t] = 0.5 * (lo + hi);
  }
  __syncthreads();

  // ---- clusters of close eigenvalues (descending order)
  if (tid == 0) {
    const double ortol = 1e-3 * tnorm;
    int nc = 0;
    cstart[nc++] = 0;
    for (int t = 1; t < kmax; ++t)
      if (P.lam[t - 1] - P.lam[t] > ortol) cstart[nc++] = t;
    cstart[nc] = kmax;
    s_ncl = nc;
  }
  __syncthreads();
  const int ncl = s_ncl;

  // ---- 3. inverse iteration, warp per cluster
  {
    double* DL = wscr;
    double* Dg = wscr + n;
    double* DU = wscr + 2 * n;
    double* DU2 = wscr + 3 * n;
    double* piv = wscr + 4 * n;
    double* y = wscr + 5 * n;
    const double pert = DBL_EPSILON * fmax(tnorm, DBL_MIN);
    for (int cl = warp; cl < ncl; cl += HEEV_WARPS) {
      for (int t = cstart[cl]; t < cstart[cl + 1]; ++t) {
        const double lam = P.lam[t];
        if (lane == 0) {  // LU with partial pivoting of T - lam I (dgttrf)
          for (int i = 0; i < n; ++i) {
            Dg[i] = sd[i] - lam;
            if (i < n - 1) { DL[i] = evec[i]; DU[i] = evec[i]; }
            DU2[i] = 0.0;
            piv[i] = 0.0;
          }
          for (int i = 0; i < n - 1; ++i) {
            if (fabs(Dg[i]) >= fabs(DL[i])) {
              if (Dg[i] == 0.0) Dg[i] = pert;
              const double f = DL[i] / Dg[i];
              DL[i] = f;
              Dg[i + 1] -= f * DU[i];
            } else {
              const double f = Dg[i] / DL[i];
              Dg[i] = DL[i];
              DL[i] = f;
              const double tmp = DU[i];
              DU[i] = Dg[i + 1];
              Dg[i + 1] = tmp - f * Dg[i + 1];
              if (i < n - 2) {
                DU2[i] = DU[i + 1];
                DU[i + 1] = -f * DU[i + 1];
              }
              piv[i] = 1.0;
            }
          }
          for (int i = 0; i < n; ++i)
            if (fabs(Dg[i]) < pert) Dg[i] = copysign(pert, Dg[i] == 0.0 ? 1.0 : Dg[i]);
        }
        // random start vector
        for (int i = lane; i < n; i += 32)
          y[i] = (double)(hash32((unsigned)(t * 7919 + i * 104729 + 12345)) & 0xffffff) / 16777216.0 - 0.5;
        __syncwarp();
        for (int it = 0; it < 3; ++it) {
          if (lane == 0) {  // solve (dgttrs)
            for (int i = 0; i < n - 1; ++i) {
              if (piv[i] == 0.0) y[i + 1] -= DL[i] * y[i];
              else {
                const double tmp = y[i];
                y[i] = y[i + 1];
                y[i + 1] = tmp - DL[i] * y[i];
              }
            }
            y[n - 1] /= Dg[n - 1];
            if (n > 1) y[n - 2] = (y[n - 2] - DU[n - 2] * y[n - 1]) / Dg[n - 2];
            for (int i = n - 3; i >= 0; --i) y[i] = (y[i] - DU[i] * y[i + 1] - DU2[i] * y[i + 2]) / Dg[i];
          }
          __syncwarp();
          // rescale to avoid overflow before orthogonalisation
          double mx = 0.0;
          for (int i = lane; i < n; i += 32) mx = fmax(mx, fabs(y[i]));
          for (int o = 16; o > 0; o >>= 1) mx = fmax(mx, __shfl_xor_sync(0xffffffffu, mx, o));
          const double inv = mx > 0.0 ? 1.0 / mx : 1.0;
          for (int i = lane; i < n; i += 32) y[i] *= inv;
          __syncwarp();
          for (int q = cstart[cl]; q < t; ++q) {  // MGS inside the cluster
            const double* zq = Z + (size_t)q * n;
            double dt = 0.0;
            for (int i = lane; i < n; i += 32) dt += y[i] * zq[i];
            dt = warp_sum(dt);
            for (int i = lane; i < n; i += 32) y[i] -= dt * zq[i];
            __syncwarp();
          }
          double nr = 0.0;
          for (int i = lane; i < n; i += 32) nr += y[i] * y[i];
          nr = warp_sum(nr);
          const double s = nr > 0.0 ? 1.0 / sqrt(nr) : 0.0;
          for (int i = lane; i < n; i += 32) y[i] *= s;
          __syncwarp();
        }
        double* zt = Z + (size_t)t * n;
        for (int i = lane; i < n; i += 32) zt[i] = y[i];
        __syncwarp();
      }
    }
  }
  __syncthreads();

  // ---- 4. back-transform Vt[t] = (Q z_t)^T, warp per eigenvector
  for (int t = warp; t < kmax; t += HEEV_WARPS) {
    cplx* vt = P.Vt + (size_t)t * n;
    const double* zt = Z + (size_t)t * n;
    for (int i = lane; i < n; i += 32) vt[i] = make_double2(zt[i], 0.0);
    __syncwarp();
    for (int j = n - 2; j >= 0; --j) {
      const cplx tau = P.tau[j];
      if (tau.x == 0.0 && tau.y == 0.0) continue;
      const int len = n - j - 1;
      const cplx* v = A + (size_t)j * n + j + 1;
      cplx* yy = vt + j + 1;
      double sr = 0.0, si = 0.0;   // s = v^H y
      for (int i = lane; i < len; i += 32) {
        cplx a = v[i], b = yy[i];
        sr += a.x * b.x + a.y * b.y;
        si += a.x * b.y - a.y * b.x;
      }
      sr = warp_sum(sr);
      si = warp_sum(si);
      const cplx ts = make_double2(tau.x * sr - tau.y * si, tau.x * si + tau.y * sr);
      for (int i = lane; i < len; i += 32) {
        cplx a = v[i], b = yy[i];
        b.x -= ts.x * a.x - ts.y * a.y;
        b.y -= ts.x * a.y + ts.y * a.x;
        yy[i] = b;
      }
      __syncwarp();
    }
  }

  // ---- 5. truncation decision
  if (tid == 0) {
    const double l1 = P.lam[0];
    int k = 1;
    double kept = 0.0;
    if (trace > 0.0 && l1 > 0.0) {
      int cnt = 0;
      for (int t = 0; t < kmax; ++t)
        if (P.lam[t] > P.tol2 * l1 && P.lam[t] > P.floor_rel * l1) ++cnt;
      k = cnt < 1 ? 1 : (cnt > P.max_bond ? P.max_bond : cnt);
      for (int t = 0; t < k; ++t) kept += P.lam[t];
    } else {
      for (int t = 0; t < kmax; ++t) P.lam[t] = 0.0;
    }
    if (P.k_out) *P.k_out = k;
    if (P.w_out) *P.w_out = fmax(trace - kept, 0.0);
  }
}

}  // namespace

size_t heev_work_doubles(int n, int kmax) {
  return (size_t)2 * n + (size_t)n * kmax + (size_t)HEEV_WARPS * 6 * n;
}

size_t heev_smem_bytes(int n, int kmax) {
  return (size_t)n * 16 * 2 + (size_t)n * 8 * 2 + (size_t)(kmax + 1) * 4 + 16;
}

int heev_max_n() { return HEEV_MAX_N; }

void launch_heev(HeevProblem* h, int n, Stager& st, cudaStream_t s) {
  if (n == 0) return;
  size_t smem = 0;
  for (int i = 0; i < n; ++i) smem = smem > heev_smem_bytes(h[i].n, h[i].kmax) ? smem : heev_smem_bytes(h[i].n, h[i].kmax);
  static bool attr = false;
  if (!attr) {
    cudaFuncSetAttribute(heev_grouped, cudaFuncAttributeMaxDynamicSharedMemorySize,
                         (int)heev_smem_bytes(HEEV_MAX_N, HEEV_MAX_N));
    attr = true;
  }
  const HeevProblem* d = static_cast<const HeevProblem*>(st.put(h, sizeof(HeevProblem) * n));
  double fl = 0.0, by = 0.0;
  for (int i = 0; i < n; ++i) {
    const double nn = h[i].n;
    fl += 8.0 * ((4.0 / 3.0) * nn * nn * nn + 2.0 * nn * nn * h[i].kmax);
    by += 16.0 * nn * nn;
  }
  prof_begin(s);
  heev_grouped<<<n, HEEV_THREADS, smem, s>>>(d);
  prof_end(s, "heev", fl, by);
  count_launch();
}

}  // namespace tcbc
