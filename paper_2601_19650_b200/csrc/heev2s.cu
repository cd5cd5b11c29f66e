// Two-stage Hermitian tridiagonalisation for the batched eigensolver of the compress step
// (B:5 (c); PAPER.md P:119 truncation "for example via singular value decomposition"
// "the SVD ... makes CBC less GPU-friendly").
//
// The one-stage Householder reduction (heev.cu heev_tridiag, zhetd2) streams the whole trailing
// matrix through the SM once per column: for config 3's 192 x 192 Grams that is 190 dependent
// passes over a matrix that does not fit one SM, so it runs latency-bound at ~20% of the FP64
// pipe.  Here the reduction is split (the two-stage scheme of SBR / PLASMA / MAGMA, re-derived
// for one CTA per Gram):
//
//  S1 heev_he2hb  dense -> Hermitian band of lower bandwidth NB = 16.  Per panel of NB columns:
//                 Householder QR of the m x NB panel below the band (rows in registers, two
//                 block reductions per column), compact WY T (zlarft), then the two-sided update
//                 of the m x m trailing matrix on the FP64 tensor cores (DMMA m8n8k4):
//                   X = A22 V T,  W = X - 1/2 V (T^H V^H X),  A22 -= V W^H + W V^H
//                 (lower 8 x 8 tiles + mirror).  The trailing matrix is read twice and written
//                 once per PANEL instead of once per column.
//  S2 heev_hb2st  band -> real symmetric tridiagonal by bulge chasing, the band (2 NB
//                 diagonals: band + bulge) in shared memory.  Sweep s annihilates column s
//                 below the subdiagonal (task t = 0) and chases the bulge down (tasks t >= 1:
//                 right-apply the previous reflector to the block below it, annihilate the
//                 first column of the bulge, two-sided update of the next diagonal block).
//                 Sweeps run concurrently one warp each, sweep s doing task T - 3s at lockstep
//                 step T (tasks three apart touch disjoint rows / columns).  Every subdiagonal
//                 comes out of a zlarfg beta, hence real.
//  K5 heev_bt2s   eigenvectors V = Q1 Q2 Z: the S2 reflectors in reverse order (warp-private
//                 columns, no barriers), then the S1 panels in reverse order (V^H Y, T, Y -= V W
//                 on DMMA).
//
// Outputs are exactly those of the one-stage K1 / K5 (d, e, trace and Gershgorin statistics in
// the work array; Vt rows), so bisection, inverse iteration and the truncation stages are shared.
// tools/twostage_proto.py is the NumPy prototype of the same algebra and schedule.
#include "heev2s.h"
#include "prof.h"
#include <cfloat>
#include <cmath>
#include <cstdlib>
#include <atomic>

namespace tcbc {

namespace {

constexpr int NB = H2S_NB;
constexpr int S1_T = 256, S1_W = S1_T / 32;
constexpr int LDB = 2 * NB;          // band storage: column c holds rows c .. c + 2 NB - 1
constexpr int BT_W = 4;              // back-transform warps (8 eigenvector columns each)
constexpr int BT_KC = 8 * BT_W;      // eigenvector columns per back-transform CTA
constexpr int S2_MAXW = 12;          // >= ceil(ceil(255 / NB) / 3) concurrent sweeps
enum { SC_GL = 0, SC_GU, SC_TNORM, SC_PIVMIN, SC_TRACE, SC_ATOL };
static_assert(SC_TRACE == H2S_S_TRACE, "work scalar layout");

__device__ __forceinline__ cplx cz() { return make_double2(0.0, 0.0); }
__device__ __forceinline__ cplx cmul(cplx a, cplx b) { return make_double2(a.x * b.x - a.y * b.y, a.x * b.y + a.y * b.x); }
__device__ __forceinline__ cplx cmulc(cplx a, cplx b) {   // conj(a) * b
  return make_double2(a.x * b.x + a.y * b.y, a.x * b.y - a.y * b.x);
}
__device__ __forceinline__ cplx cconj(cplx a) { return make_double2(a.x, -a.y); }
__device__ __forceinline__ cplx csub(cplx a, cplx b) { return make_double2(a.x - b.x, a.y - b.y); }
__device__ __forceinline__ cplx cadd(cplx a, cplx b) { return make_double2(a.x + b.x, a.y + b.y); }
__device__ __forceinline__ double negd(double x) {
  return __hiloint2double(__double2hiint(x) ^ 0x80000000, __double2loint(x));
}
__device__ __forceinline__ double wsum(double v) {
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  return v;
}
__device__ __forceinline__ cplx shfl_c(cplx v, int src) {
  return make_double2(__shfl_sync(0xffffffffu, v.x, src), __shfl_sync(0xffffffffu, v.y, src));
}
__device__ __forceinline__ cplx shfl_xor_c(cplx v, int m) {
  return make_double2(__shfl_xor_sync(0xffffffffu, v.x, m), __shfl_xor_sync(0xffffffffu, v.y, m));
}

// SFU seeds + two Newton steps (~1 ulp): the compiler's IEEE sqrt / division sequences carry
// slow-path branches and sit on the critical path of every Householder step
__device__ __forceinline__ double frcp(double b) {
  double r;
  asm("rcp.approx.ftz.f64 %0, %1;" : "=d"(r) : "d"(b));
  r = r * fma(-b, r, 2.0);
  r = r * fma(-b, r, 2.0);
  return r;
}
__device__ __forceinline__ double frsqrt(double x) {
  double y;
  asm("rsqrt.approx.ftz.f64 %0, %1;" : "=d"(y) : "d"(x));
  const double h = 0.5 * x;
  y = y * fma(-h * y, y, 1.5);
  y = y * fma(-h * y, y, 1.5);
  return y;
}

// zlarfg: H^H [alpha; x] = [beta; 0], H = I - tau v v^H, v = [1; x * scale], beta real
// (beta = -sign(Re alpha) sqrt(|alpha|^2 + |x|^2); |alpha - beta| >= |beta| > 0)
__device__ __forceinline__ void zlarfg(cplx alpha, double xn2, double& beta, cplx& tau, cplx& scale) {
  if (xn2 == 0.0 && alpha.y == 0.0) {
    beta = alpha.x;
    tau = cz();
    scale = cz();
    return;
  }
  const double sq = alpha.x * alpha.x + alpha.y * alpha.y + xn2;
  const double r = frsqrt(sq);
  const double sg = alpha.x >= 0.0 ? 1.0 : -1.0;
  beta = -sg * sq * r;
  const double ib = -sg * r;   // 1 / beta
  tau = make_double2(fma(-alpha.x, ib, 1.0), -alpha.y * ib);
  const cplx den = make_double2(alpha.x - beta, alpha.y);
  const double idd = frcp(den.x * den.x + den.y * den.y);
  scale = make_double2(den.x * idd, -den.y * idd);
}

// ------------------------------------------------------------------ DMMA 8 x 8 complex tiles
__device__ __forceinline__ void dmma(double& c0, double& c1, double a, double b) {
  asm("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
      : "+d"(c0), "+d"(c1)
      : "d"(a), "d"(b));
}
// accumulator of one 8 x 8 complex tile: lane holds C[lane / 4][2 (lane % 4) + h]
struct ZT {
  double r0, r1, i0, i1;
};
__device__ __forceinline__ void zt_zero(ZT& c) { c.r0 = c.r1 = c.i0 = c.i1 = 0.0; }
// one k-step of 4: a = A[lane / 4][k0 + lane % 4], b = B[k0 + lane % 4][lane / 4] (4M rule)
__device__ __forceinline__ void zstep(ZT& c, cplx a, cplx b) {
  dmma(c.r0, c.r1, a.x, b.x);
  dmma(c.i0, c.i1, a.x, b.y);
  dmma(c.r0, c.r1, negd(a.y), b.y);
  dmma(c.i0, c.i1, a.y, b.x);
}
__device__ __forceinline__ cplx zt_get(const ZT& c, int h) { return h ? make_double2(c.r1, c.i1) : make_double2(c.r0, c.i0); }


// ------------------------------------------------------------------ S1: dense -> band
constexpr int NT = NB / 8;        // 8-wide column tiles of a panel
constexpr int LDP = NB + 1;       // panel row stride during the QR
constexpr int RG = S1_T / NB;     // row groups of the QR (threads per panel column)
static_assert(RG <= 32 && (RG & (RG - 1)) == 0, "a panel column's threads sit in one warp");
// shared memory: V [mmax][NB], panel [mmax][NB + 1] (later X [mmax][NB]), T, M, G [NB][NB]
__host__ __device__ inline size_t s1_smem_bytes(int n) {
  const int mmax = n - NB > 0 ? n - NB : 1;
  return sizeof(cplx) * ((size_t)mmax * NB + (size_t)mmax * LDP + 3 * NB * NB + (size_t)4 * S1_W * NB * NB);
}

// C (NT x NT tiles, ld NB) = op(A)^H-style small products of a warp: tile (ti, tj) of
// sum_k a(k, row) b(k, col) over k < K, loaders given as lambdas
template <class FA, class FB>
__device__ __forceinline__ void small_tile(cplx* C, int ti, int tj, int K, FA fa, FB fb) {
  const int lane = threadIdx.x & 31, fr = lane >> 2, fc = lane & 3;
  ZT g;
  zt_zero(g);
  for (int k0 = 0; k0 < K; k0 += 4) {
    const int k = k0 + fc;
    zstep(g, k < K ? fa(k, ti * 8 + fr) : cz(), k < K ? fb(k, tj * 8 + fr) : cz());
  }
#pragma unroll
  for (int h = 0; h < 2; ++h) C[(ti * 8 + fr) * NB + tj * 8 + 2 * fc + h] = zt_get(g, h);
}

__global__ void __launch_bounds__(S1_T, 2) heev_he2hb(const HeevProblem* __restrict__ probs) {
  TCBC_PDL_WAIT();
  const HeevProblem& P = probs[blockIdx.x];
  if (P.skip && *P.skip) return;
  const int n = P.n;
  cplx* __restrict__ A = P.A;
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5, fr = lane >> 2, fc = lane & 3;
  const int mmax = n - NB > 0 ? n - NB : 1;
  extern __shared__ __align__(16) unsigned char smem_raw[];
  cplx* Vs = reinterpret_cast<cplx*>(smem_raw);
  cplx* Ps = Vs + (size_t)mmax * NB;   // the panel during the QR ...
  cplx* Xs = Ps;                       // ... then X / W
  cplx* Ts = Ps + (size_t)mmax * LDP;
  cplx* Ms = Ts + NB * NB;
  cplx* Gs = Ms + NB * NB;
  cplx* Pp = Gs + NB * NB;             // per-warp partial G = V^H V  [S1_W][NB][NB]
  cplx* Mp = Pp + S1_W * NB * NB;      // per-warp partial V^H X0     [S1_W][NB][NB]
  cplx* Sw = Mp + S1_W * NB * NB;      // per-warp scratch            [S1_W][2][NB][NB]
  __shared__ cplx stau[NB];
  __shared__ double sbeta[NB];
  __shared__ double rn[S1_W];
  cplx* Tg = reinterpret_cast<cplx*>(P.work + heev_base_doubles(n, P.kmax));   // [panels][NB][NB]

  {   // trace (the discarded weight is trace - kept eigenvalues)
    double tr = 0.0;
    for (int i = tid; i < n; i += S1_T) tr += A[(size_t)i * n + i].x;
    tr = wsum(tr);
    if (lane == 0) rn[warp] = tr;
    __syncthreads();
    if (tid == 0) {
      double s = 0.0;
      for (int w = 0; w < S1_W; ++w) s += rn[w];
      P.work[2 * n + SC_TRACE] = s;
    }
    __syncthreads();
  }

  for (int p = 0;; ++p) {
    const int c0 = p * NB, r0 = c0 + NB, m = n - r0;
    if (m < 2) break;
    const int kq = min(m, NB);
    cplx* A22 = A + (size_t)r0 * n + r0;
    // ---- (1) panel A[r0:, c0:c0+NB] -> Ps; V starts as the unit diagonal
    for (int e = tid; e < m * NB; e += S1_T) {
      const int t = e / NB, c = e % NB;
      Ps[t * LDP + c] = A[(size_t)(r0 + t) * n + c0 + c];
      Vs[e] = t == c ? make_double2(1.0, 0.0) : cz();
    }
    if (tid < NB) {
      stau[tid] = cz();
      sbeta[tid] = 0.0;
    }
    __syncthreads();
    // ---- (2) Householder QR of the panel (zgeqr2).  Thread (column c = tid / RG, row group
    // rg = tid % RG).  Step j needs one reduction over the RG row groups (one warp or half):
    // |x|^2 of column j below the diagonal and g_c = sum_{t > j} conj(A[t][j]) A[t][c]; then
    // u_c = A[j][c] + conj(scale) g_c = (v^H A)[c] and A[t][c] -= conj(tau) v_t u_c.  Column j
    // itself is left in place (v goes to Vs, beta to sbeta), so one barrier per column.
    {
      const int c = tid / RG, rg = tid % RG;
      for (int j = 0; j < kq; ++j) {
        double gn = 0.0, gr = 0.0, gi = 0.0;
        for (int t = rg; t < m; t += RG) {
          if (t <= j) continue;
          const cplx x = Ps[t * LDP + j], y = Ps[t * LDP + c];
          gn = fma(x.x, x.x, fma(x.y, x.y, gn));
          gr = fma(x.x, y.x, fma(x.y, y.y, gr));
          gi = fma(x.x, y.y, fma(-x.y, y.x, gi));
        }
        const cplx ajc = Ps[j * LDP + c];   // read before any thread of this column updates row j
        const cplx alpha = Ps[j * LDP + j];
#pragma unroll
        for (int o = RG / 2; o >= 1; o >>= 1) {
          gn += __shfl_xor_sync(0xffffffffu, gn, o);
          gr += __shfl_xor_sync(0xffffffffu, gr, o);
          gi += __shfl_xor_sync(0xffffffffu, gi, o);
        }
        double beta;
        cplx tau, scale;
        zlarfg(alpha, gn, beta, tau, scale);
        if (c == j) {
          for (int t = rg; t < m; t += RG)
            if (t > j) Vs[t * NB + j] = cmul(Ps[t * LDP + j], scale);
          if (rg == 0) {
            stau[j] = tau;
            sbeta[j] = beta;
          }
        } else if (c > j) {
          const cplx u = make_double2(ajc.x + scale.x * gr + scale.y * gi, ajc.y + scale.x * gi - scale.y * gr);
          const cplx cu = cmul(cconj(tau), u);
          for (int t = rg; t < m; t += RG) {
            if (t < j) continue;
            const cplx v = t == j ? make_double2(1.0, 0.0) : cmul(Ps[t * LDP + j], scale);
            Ps[t * LDP + c] = csub(Ps[t * LDP + c], cmul(v, cu));
          }
        }
        __syncthreads();
      }
    }
    // ---- (3) R (upper, beta on the diagonal) and V (below) into the panel region of A; every
    // warp's partial G_w = V_w^H V_w over its 8-row strips
    for (int e = tid; e < m * NB; e += S1_T) {
      const int t = e / NB, c = e % NB;
      A[(size_t)(r0 + t) * n + c0 + c] = t < c ? Ps[t * LDP + c] : (t == c ? make_double2(sbeta[c], 0.0) : Vs[e]);
    }
    static_assert(NT == 1, "one column tile per panel below");
    const int nstrip = (m + 7) >> 3;
    {
      ZT g;
      zt_zero(g);
      for (int sI = warp; sI < nstrip; sI += S1_W) {
#pragma unroll
        for (int k0 = 0; k0 < 8; k0 += 4) {
          const int k = sI * 8 + k0 + fc;
          const cplx a = k < m ? cconj(Vs[k * NB + fr]) : cz();
          const cplx b = k < m ? Vs[k * NB + fr] : cz();
          zstep(g, a, b);
        }
      }
#pragma unroll
      for (int h = 0; h < 2; ++h) Pp[(warp * NB + fr) * NB + 2 * fc + h] = zt_get(g, h);
    }
    __syncthreads();
    // ---- (4) warp 0: G = sum_w G_w, T (zlarft, forward columnwise); meanwhile (5) warps 1..:
    // X0 = A22 V (two 8-row strips per warp iteration: independent DMMA chains, the A22 loads
    // of a k-block issued together) and their partial M_w = V_w^H X0_w
    if (warp == 0) {
      for (int e = lane; e < NB * NB; e += 32) {
        cplx acc = cz();
#pragma unroll
        for (int w = 0; w < S1_W; ++w) acc = cadd(acc, Pp[w * NB * NB + e]);
        Gs[e] = acc;
      }
      __syncwarp();
      for (int j = 0; j < NB; ++j) {
        const cplx tj = stau[j];
        cplx val = cz();
        if (lane < j) {
          for (int q = lane; q < j; ++q) {
            const cplx a = Ts[lane * NB + q], b = Gs[q * NB + j];
            val.x += a.x * b.x - a.y * b.y;
            val.y += a.x * b.y + a.y * b.x;
          }
          val = cmul(make_double2(-tj.x, -tj.y), val);
        }
        __syncwarp();
        if (lane < NB) Ts[lane * NB + j] = lane < j ? val : (lane == j ? tj : cz());
        __syncwarp();
      }
      for (int e = lane; e < NB * NB; e += 32) Tg[(size_t)p * NB * NB + e] = Ts[e];
      for (int e = lane; e < NB * NB; e += 32) Mp[e] = cz();   // M_0 = 0
    } else {
      ZT mw;
      zt_zero(mw);
      constexpr int XW = S1_W - 1;   // warps on X0
      for (int s0 = warp - 1; s0 < nstrip; s0 += 2 * XW) {
        ZT x0, x1;
        zt_zero(x0);
        zt_zero(x1);
        const int s1 = s0 + XW;
        const int rowa = s0 * 8 + fr, rowb = s1 * 8 + fr;
        const bool va = rowa < m, vb = rowb < m;
        const cplx* pa = A22 + (size_t)(va ? rowa : 0) * n;
        const cplx* pb = A22 + (size_t)(vb ? rowb : 0) * n;
        for (int kb = 0; kb < m; kb += 32) {
          cplx a0[8], a1[8];
#pragma unroll
          for (int u = 0; u < 8; ++u) {
            const int k = min(kb + 4 * u + fc, m - 1);
            a0[u] = pa[k];
            a1[u] = pb[k];
          }
#pragma unroll
          for (int u = 0; u < 8; ++u) {
            const int k = kb + 4 * u + fc;
            const bool kv = k < m;
            const cplx b = kv ? Vs[k * NB + fr] : cz();
            zstep(x0, (va && kv) ? a0[u] : cz(), b);
            zstep(x1, (vb && kv) ? a1[u] : cz(), b);
          }
        }
#pragma unroll
        for (int h = 0; h < 2; ++h) {
          if (va) Xs[rowa * NB + 2 * fc + h] = zt_get(x0, h);
          if (vb) Xs[rowb * NB + 2 * fc + h] = zt_get(x1, h);
        }
        __syncwarp();
#pragma unroll
        for (int u = 0; u < 2; ++u) {   // M_w += V_strip^H X0_strip
          const int sI = u ? s1 : s0;
#pragma unroll
          for (int k0 = 0; k0 < 8; k0 += 4) {
            const int k = sI * 8 + k0 + fc;
            const cplx a = k < m ? cconj(Vs[k * NB + fr]) : cz();
            const cplx b = k < m ? Xs[k * NB + fr] : cz();
            zstep(mw, a, b);
          }
        }
      }
#pragma unroll
      for (int h = 0; h < 2; ++h) Mp[(warp * NB + fr) * NB + 2 * fc + h] = zt_get(mw, h);
    }
    __syncthreads();
    // ---- (6) every warp (no barrier): M0 = sum_w M_w, M = M0 T, Y2 = T^H M in its own scratch
    cplx* Sq = Sw + (size_t)warp * 2 * NB * NB;   // [M0 / Y2][M]
    for (int e = lane; e < NB * NB; e += 32) {
      cplx acc = cz();
#pragma unroll
      for (int w = 0; w < S1_W; ++w) acc = cadd(acc, Mp[w * NB * NB + e]);
      Sq[e] = acc;
    }
    __syncwarp();
    small_tile(Sq + NB * NB, 0, 0, NB, [&](int k, int r) { return Sq[r * NB + k]; }, [&](int k, int c) { return Ts[k * NB + c]; });
    __syncwarp();
    small_tile(Sq, 0, 0, NB, [&](int k, int r) { return cconj(Ts[k * NB + r]); }, [&](int k, int c) { return Sq[NB * NB + k * NB + c]; });
    __syncwarp();
    const cplx* Y2 = Sq;
    // ---- (8) W = X0 T - 1/2 V Y2 (in Xs, strip-private)
    for (int sI = warp; sI < nstrip; sI += S1_W) {
      const int row = sI * 8 + fr;
      const bool rv = row < m;
      ZT x, y;
      zt_zero(x);
      zt_zero(y);
#pragma unroll
      for (int k0 = 0; k0 < NB; k0 += 4) {
        const int k = k0 + fc;
        zstep(x, rv ? Xs[row * NB + k] : cz(), Ts[k * NB + fr]);
        zstep(y, rv ? Vs[row * NB + k] : cz(), Y2[k * NB + fr]);
      }
      __syncwarp();
      if (rv) {
#pragma unroll
        for (int h = 0; h < 2; ++h) {
          const cplx a = zt_get(x, h), b = zt_get(y, h);
          Xs[row * NB + 2 * fc + h] = make_double2(a.x - 0.5 * b.x, a.y - 0.5 * b.y);
        }
      }
    }
    __syncthreads();
    // ---- (9) A22 -= V W^H + W V^H = [V W] [W V]^H: lower 8 x 8 tiles (two per warp
    // iteration, their A22 entries loaded before the products), mirrored
    const int ntile = nstrip * (nstrip + 1) / 2;
    int ci = 0, cj = warp;   // lower-triangle tile (ci, cj) of linear index t0, advanced by steps
    while (cj > ci) {
      cj -= ci + 1;
      ++ci;
    }
    for (int t0 = warp; t0 < ntile; t0 += 2 * S1_W) {
      ZT c[2];
      int bi[2], bj[2];
      cplx old[2][2];
#pragma unroll
      for (int u = 0; u < 2; ++u) {
        bi[u] = ci;
        bj[u] = cj;
        cj += S1_W;
        while (cj > ci) {
          cj -= ci + 1;
          ++ci;
        }
        if (bi[u] >= nstrip) {   // past the last tile: a valid dummy (its store is skipped)
          bi[u] = nstrip - 1;
          bj[u] = 0;
        }
        zt_zero(c[u]);
        const int row = min(bi[u] * 8 + fr, m - 1);
#pragma unroll
        for (int h = 0; h < 2; ++h) old[u][h] = A22[(size_t)row * n + min(bj[u] * 8 + 2 * fc + h, m - 1)];
      }
#pragma unroll
      for (int k0 = 0; k0 < 2 * NB; k0 += 4) {
        const int k = k0 + fc;
#pragma unroll
        for (int u = 0; u < 2; ++u) {
          const int ra = bi[u] * 8 + fr, cb = bj[u] * 8 + fr;
          cplx a, b;
          if (k0 < NB) {
            a = ra < m ? Vs[ra * NB + k] : cz();
            b = cb < m ? cconj(Xs[cb * NB + k]) : cz();
          } else {
            a = ra < m ? Xs[ra * NB + k - NB] : cz();
            b = cb < m ? cconj(Vs[cb * NB + k - NB]) : cz();
          }
          zstep(c[u], a, b);
        }
      }
#pragma unroll
      for (int u = 0; u < 2; ++u) {
        if (t0 + u * S1_W >= ntile) continue;
        const int row = bi[u] * 8 + fr;
#pragma unroll
        for (int h = 0; h < 2; ++h) {
          const int col = bj[u] * 8 + 2 * fc + h;
          if (row < m && col < m) {
            const cplx nv = csub(old[u][h], zt_get(c[u], h));
            A22[(size_t)row * n + col] = nv;
            if (bi[u] != bj[u]) A22[(size_t)col * n + row] = cconj(nv);
          }
        }
      }
    }
    __syncthreads();
  }
}

// ------------------------------------------------------------------ S2: band -> tridiagonal
// One warp per active sweep; a task's 8 x 8 blocks sit one row and two columns per lane:
// lane = 8 cq + i holds rows i, columns 2 cq, 2 cq + 1 (row sums: xor 8, 16; column sums:
// xor 1, 2, 4).
static_assert(NB == 8, "the bulge-chasing lane layout is written for 8 x 8 blocks");
__host__ __device__ inline int s2_warps(int n) {
  const int w = (h2s_ntask(n, 0) + 2) / 3;
  return w < 1 ? 1 : (w > S2_MAXW ? S2_MAXW : w);
}
__host__ __device__ inline size_t s2_smem_bytes(int n) { return sizeof(cplx) * (size_t)n * LDB; }

__device__ __forceinline__ cplx rowsum(cplx v) {   // over the 4 lanes of a row
  v.x += __shfl_xor_sync(0xffffffffu, v.x, 8);
  v.y += __shfl_xor_sync(0xffffffffu, v.y, 8);
  v.x += __shfl_xor_sync(0xffffffffu, v.x, 16);
  v.y += __shfl_xor_sync(0xffffffffu, v.y, 16);
  return v;
}
__device__ __forceinline__ cplx colsum(cplx v) {   // over the 8 lanes (rows) of a column group
  for (int o = 1; o <= 4; o <<= 1) {
    v.x += __shfl_xor_sync(0xffffffffu, v.x, o);
    v.y += __shfl_xor_sync(0xffffffffu, v.y, o);
  }
  return v;
}

__global__ void __launch_bounds__(S2_MAXW * 32) heev_hb2st(const HeevProblem* __restrict__ probs) {
  TCBC_PDL_WAIT();
  const HeevProblem& P = probs[blockIdx.x];
  if (P.skip && *P.skip) return;
  const int n = P.n;
  const cplx* __restrict__ A = P.A;
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5, nthr = blockDim.x;
  const int ri = lane & 7, cq = lane >> 3;   // row, column pair (2 cq, 2 cq + 1)
  extern __shared__ __align__(16) unsigned char smem_raw[];
  cplx* Bd = reinterpret_cast<cplx*>(smem_raw);   // Bd[c * LDB + d] = A[c + d][c]
  __shared__ cplx vbuf[16][NB];
  __shared__ cplx tbuf[16];
  __shared__ int prog[H2S_MAX_N];   // tasks finished per sweep
  const size_t base2 = heev_base_doubles(n, P.kmax) + 2 * (size_t)h2s_panels(n) * NB * NB;
  cplx* R2v = reinterpret_cast<cplx*>(P.work + base2);
  cplx* R2t = R2v + (size_t)h2s_ref_base(n, n - 1) * NB;

  for (int e = tid; e < n * LDB; e += nthr) {
    const int c = e / LDB, dd = e % LDB;
    Bd[e] = (dd <= NB && c + dd < n) ? A[(size_t)(c + dd) * n + c] : cz();
  }
  for (int i = tid; i < n; i += nthr) prog[i] = 0;
  __syncthreads();

  // Sweeps are dealt round-robin to the warps; task (s, t) waits until sweep s - 1 has finished
  // task t + 2 (the lockstep order "sweep s does task T - 3s at step T" of tools/twostage_proto.py,
  // whose concurrent tasks touch disjoint rows / columns), signalled by per-sweep counters
  volatile int* vprog = prog;
  const int nw = nthr >> 5;
  for (int s = warp; s <= n - 2; s += nw) {
    const int nts = h2s_ntask(n, s);
    const int slot = s & 15;
    for (int t = 0; t < nts; ++t) {
      if (s > 0) {
        const int need = min(t + 3, h2s_ntask(n, s - 1));
        if (lane == 0)
          while (vprog[s - 1] < need) __nanosleep(32);   // polling would steal issue slots
        __syncwarp();
        __threadfence_block();
      }
      int j0, L;
      double beta;
      cplx tau, scale, vi;   // vi: v of this lane's row
      if (t == 0) {
        j0 = s + 1;
        L = min(NB, n - 1 - s);
        const cplx x = ri < L ? Bd[s * LDB + 1 + ri] : cz();
        cplx nq = make_double2((ri >= 1 && ri < L) ? x.x * x.x + x.y * x.y : 0.0, 0.0);
        nq = colsum(nq);
        const cplx alpha = shfl_c(x, 0);
        zlarfg(alpha, nq.x, beta, tau, scale);
        vi = ri == 0 ? make_double2(1.0, 0.0) : (ri < L ? cmul(x, scale) : cz());
        __syncwarp();
        if (cq == 0) {
          vbuf[slot][ri] = vi;
          if (ri < L) Bd[s * LDB + 1 + ri] = ri == 0 ? make_double2(beta, 0.0) : cz();
        }
        if (lane == 0) tbuf[slot] = tau;
      } else {
        const int jp = s + 1 + (t - 1) * NB, Lp = min(NB, n - jp);
        j0 = jp + NB;
        L = min(NB, n - j0);
        const cplx taup = tbuf[slot];
        cplx ev[2], vpj[2];
#pragma unroll
        for (int q = 0; q < 2; ++q) {
          const int j = 2 * cq + q;
          vpj[q] = vbuf[slot][j];
          ev[q] = (ri < L && j < Lp) ? Bd[(jp + j) * LDB + NB + ri - j] : cz();
        }
        // y = E v_prev (row sums), E -= tau_p y v_p^H
        cplx y = cadd(cmul(ev[0], vpj[0]), cmul(ev[1], vpj[1]));
        y = rowsum(y);
        const cplx ty = cmul(taup, y);
#pragma unroll
        for (int q = 0; q < 2; ++q) ev[q] = csub(ev[q], cmul(ty, cconj(vpj[q])));
        // new reflector from the bulge's first column (lanes cq == 0, q == 0)
        const cplx x = shfl_c(ev[0], ri);   // E[ri][0] from lane ri
        cplx nq = make_double2((ri >= 1 && ri < L) ? x.x * x.x + x.y * x.y : 0.0, 0.0);
        nq = colsum(nq);
        const cplx alpha = shfl_c(ev[0], 0);
        zlarfg(alpha, nq.x, beta, tau, scale);
        vi = ri == 0 ? make_double2(1.0, 0.0) : (ri < L ? cmul(x, scale) : cz());
        if (cq == 0) ev[0] = ri == 0 ? make_double2(beta, 0.0) : cz();
        // E[:, j >= 1] <- H^H E:  u_j = sum_i conj(v_i) E[i][j]
        const cplx ctau = cconj(tau);
#pragma unroll
        for (int q = 0; q < 2; ++q) {
          const int j = 2 * cq + q;
          const cplx u = colsum(cmulc(vi, ev[q]));
          if (j >= 1) ev[q] = csub(ev[q], cmul(vi, cmul(ctau, u)));
        }
#pragma unroll
        for (int q = 0; q < 2; ++q) {
          const int j = 2 * cq + q;
          if (ri < L && j < Lp) Bd[(jp + j) * LDB + NB + ri - j] = ev[q];
        }
        __syncwarp();
        if (cq == 0) vbuf[slot][ri] = vi;
        if (lane == 0) tbuf[slot] = tau;
      }
      {   // the reflector for the back-transform
        const int ridx = h2s_ref_base(n, s) + t;
        if (cq == 0) R2v[(size_t)ridx * NB + ri] = vi;
        if (lane == 0) R2t[ridx] = tau;
      }
      // two-sided update of the diagonal block D = A[j0 .. j0 + L)^2: D <- H^H D H
      cplx dv[2], vj[2];
#pragma unroll
      for (int q = 0; q < 2; ++q) {
        const int j = 2 * cq + q;
        vj[q] = shfl_c(vi, j);   // v_j from lane j (row j, cq = 0)
        cplx d = cz();
        if (ri < L && j < L) d = ri >= j ? Bd[(j0 + j) * LDB + ri - j] : cconj(Bd[(j0 + ri) * LDB + j - ri]);
        dv[q] = d;
      }
      cplx y = rowsum(cadd(cmul(dv[0], vj[0]), cmul(dv[1], vj[1])));   // y_i = (D v)_i
      cplx g = cq == 0 ? cmulc(vi, y) : cz();                           // gamma = v^H D v (real)
      g = colsum(g);
      const double gam = __shfl_sync(0xffffffffu, g.x, 0);
      const double t2 = tau.x * tau.x + tau.y * tau.y;
      const cplx ty = cmul(tau, y);
      const cplx w = make_double2(ty.x - 0.5 * t2 * gam * vi.x, ty.y - 0.5 * t2 * gam * vi.y);   // w_i
#pragma unroll
      for (int q = 0; q < 2; ++q) {
        const int j = 2 * cq + q;
        const cplx wj = shfl_c(w, j);
        const cplx a = cmul(w, cconj(vj[q])), b = cmul(vi, cconj(wj));
        dv[q].x -= a.x + b.x;
        dv[q].y -= a.y + b.y;
        if (ri >= j && ri < L && j < L) Bd[(j0 + j) * LDB + ri - j] = ri == j ? make_double2(dv[q].x, 0.0) : dv[q];
      }
      __syncwarp();
      __threadfence_block();
      if (lane == 0) vprog[s] = t + 1;
    }
  }
  __syncthreads();

  // d, e and the Gershgorin / pivmin statistics (as heev.cu tridiag_stats)
  double* dvec = P.work;
  double* evec = P.work + n;
  for (int i = tid; i < n; i += nthr) {
    dvec[i] = Bd[i * LDB].x;
    evec[i] = i < n - 1 ? Bd[i * LDB + 1].x : 0.0;
  }
  __syncthreads();
  double gl = 1e300, gu = -1e300, em = 0.0;
  for (int i = tid; i < n; i += nthr) {
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
  __shared__ double mm[3][S2_MAXW];
  if (lane == 0) {
    mm[0][warp] = gl;
    mm[1][warp] = gu;
    mm[2][warp] = em;
  }
  __syncthreads();
  if (tid == 0) {
    gl = mm[0][0];
    gu = mm[1][0];
    em = mm[2][0];
    for (int w = 1; w < (nthr >> 5); ++w) {
      gl = fmin(gl, mm[0][w]);
      gu = fmax(gu, mm[1][w]);
      em = fmax(em, mm[2][w]);
    }
    double* sc = P.work + 2 * n;
    const double tnorm = fmax(fabs(gl), fabs(gu));
    const double pivmin = DBL_MIN * fmax(1.0, em);
    sc[SC_GL] = gl - 2.0 * DBL_EPSILON * tnorm * n - 2.0 * pivmin;
    sc[SC_GU] = gu + 2.0 * DBL_EPSILON * tnorm * n + 2.0 * pivmin;
    sc[SC_TNORM] = tnorm;
    sc[SC_PIVMIN] = pivmin;
    sc[SC_ATOL] = 4.0 * DBL_EPSILON * tnorm;
  }
}

// ------------------------------------------------------------------ K5: V = Q1 Q2 Z
// One CTA of BT_W warps per (Gram, BT_KC = 32 eigenvector columns); Y in shared memory.
// Q2: warp w owns columns 8w .. 8w + 7, lane = 8 rq + c holds rows 2 rq, 2 rq + 1 of the 8-row
// reflector for column 8 w + c (dot: two local terms + xor 8, 16).  The reflectors are staged
// through a small buffer a chunk of whole sweeps at a time; Q1 reads V from the panel region of
// A directly (L2) and runs on DMMA.
constexpr int BT_STAGE = 96;   // reflectors per staging chunk
__host__ __device__ inline size_t bt_buf_cplx() {
  const size_t q2 = (size_t)BT_STAGE * (NB + 1), q1 = (size_t)2 * NB * BT_KC + NB * NB;
  return q2 > q1 ? q2 : q1;
}
__host__ __device__ inline size_t bt_smem_bytes(int n) { return sizeof(cplx) * ((size_t)n * BT_KC + bt_buf_cplx()); }

__device__ __forceinline__ int bt_find(const HeevProblem* p, int n, int b) {
  int lo = 0, hi = n - 1;
  while (lo < hi) {
    const int mid = (lo + hi + 1) >> 1;
    if (p[mid].bstart <= b) lo = mid; else hi = mid - 1;
  }
  return lo;
}

// y <- (I - tau v v^H) y on rows [j, j + 8) of column cc, all eight rows in this lane; rec =
// the staged reflector (v[0..8), tau in rec[8]: records of 9 complex keep the four reflectors a
// load instruction touches in distinct banks)
__device__ __forceinline__ void bt_refl(cplx* Ys, int n, int j, int cc, const cplx* rec) {
  cplx y[NB];
  cplx d = cz();
#pragma unroll
  for (int i = 0; i < NB; ++i) {
    y[i] = j + i < n ? Ys[(size_t)(j + i) * BT_KC + cc] : cz();
    const cplx p = cmulc(rec[i], y[i]);
    d.x += p.x;
    d.y += p.y;
  }
  const cplx td = cmul(rec[NB], d);
#pragma unroll
  for (int i = 0; i < NB; ++i)
    if (j + i < n) Ys[(size_t)(j + i) * BT_KC + cc] = csub(y[i], cmul(rec[i], td));
}

__global__ void __launch_bounds__(BT_W * 32) heev_bt2s(const HeevProblem* __restrict__ probs, int nprob) {
  TCBC_PDL_WAIT();
  const HeevProblem& P = probs[bt_find(probs, nprob, blockIdx.x)];
  if (P.skip && *P.skip) return;
  const int n = P.n, kmax = P.kmax;
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5, fr = lane >> 2, fc = lane & 3;
  constexpr int NTH = BT_W * 32;
  const int c0 = (blockIdx.x - P.bstart) * BT_KC;
  const int k = P.k_out ? *P.k_out : kmax;
  if (c0 >= k) {   // every vector of this block is dropped
    for (int e = tid; e < BT_KC * n; e += NTH) {
      const int c = c0 + e / n;
      if (c < kmax) P.Vt[(size_t)c * n + e % n] = cz();
    }
    return;
  }
  extern __shared__ __align__(16) unsigned char smem_raw[];
  cplx* Ys = reinterpret_cast<cplx*>(smem_raw);   // [n][BT_KC]
  cplx* buf = Ys + (size_t)n * BT_KC;
  const double* Z = P.work + 2 * n + 8;
  const cplx* Tg = reinterpret_cast<const cplx*>(P.work + heev_base_doubles(n, kmax));
  const cplx* R2v = Tg + (size_t)h2s_panels(n) * NB * NB;
  const cplx* R2t = R2v + (size_t)h2s_ref_base(n, n - 1) * NB;
#pragma unroll 4
  for (int e = tid; e < n * BT_KC; e += NTH) {
    const int i = e / BT_KC, c = e % BT_KC;
    Ys[e] = make_double2((c0 + c < k) ? Z[(size_t)i * kmax + c0 + c] : 0.0, 0.0);
  }
  // ---- Q2: reflectors of S2 in reverse order; those of one sweep act on disjoint rows and
  // are applied four at a time
  {
    // lane = 8 q + c: column 8 w + c, reflectors t = q, q + 4, ... of each sweep (disjoint rows;
    // a lane applies a whole 8-row reflector to its column, no shuffles).  The next chunk's
    // reflectors are loaded into registers while this chunk is applied.
    constexpr int REC = NB + 1, PRE = (BT_STAGE * REC + NTH - 1) / NTH;
    const int q = lane >> 3, cc = 8 * warp + (lane & 7);
    cplx* Rv = buf;
    auto chunk = [&](int shi, int& slo, int& cnt) {
      slo = shi;
      cnt = h2s_ntask(n, shi);
      while (slo > 0 && cnt + h2s_ntask(n, slo - 1) <= BT_STAGE) {
        --slo;
        cnt += h2s_ntask(n, slo);
      }
    };
    cplx pre[PRE];
    auto prefetch = [&](int lo, int cnt) {
#pragma unroll
      for (int u = 0; u < PRE; ++u) {
        const int e = tid + u * NTH, r = e / REC, i = e % REC;
        pre[u] = e < cnt * REC ? (i < NB ? R2v[(size_t)(lo + r) * NB + i] : R2t[lo + r]) : cz();
      }
    };
    int s = n - 2, slo, cnt;
    chunk(s, slo, cnt);
    prefetch(h2s_ref_base(n, slo), cnt);
    while (s >= 0) {
      const int lo = h2s_ref_base(n, slo);
      __syncthreads();
#pragma unroll
      for (int u = 0; u < PRE; ++u)
        if (tid + u * NTH < cnt * REC) Rv[tid + u * NTH] = pre[u];
      __syncthreads();
      const int s2 = slo - 1;
      int slo2 = 0, cnt2 = 0;
      if (s2 >= 0) {
        chunk(s2, slo2, cnt2);
        prefetch(h2s_ref_base(n, slo2), cnt2);
      }
      for (int ss = s; ss >= slo; --ss) {
        const int nt = h2s_ntask(n, ss), rb = h2s_ref_base(n, ss) - lo;
        int t = q;
        for (; t + 4 < nt; t += 8) {
          bt_refl(Ys, n, ss + 1 + t * NB, cc, Rv + (rb + t) * REC);
          bt_refl(Ys, n, ss + 1 + (t + 4) * NB, cc, Rv + (rb + t + 4) * REC);
        }
        if (t < nt) bt_refl(Ys, n, ss + 1 + t * NB, cc, Rv + (rb + t) * REC);
        __syncwarp();
      }
      s = s2;
      slo = slo2;
      cnt = cnt2;
    }
  }
  // ---- Q1: panels in reverse order, Y[r0:] -= V (T (V^H Y[r0:])), V from the panel region
  const cplx* A = P.A;
  cplx* Ws = buf;                  // [NB][BT_KC]
  cplx* W2 = Ws + NB * BT_KC;      // [NB][BT_KC]
  cplx* Tp = W2 + NB * BT_KC;      // [NB][NB]
  static_assert(BT_KC == 32 && BT_W == 4, "W: four 8-column tiles (one per warp)");
  for (int p = h2s_panels(n) - 1; p >= 0; --p) {
    const int pc0 = p * NB, r0 = pc0 + NB, m = n - r0;
    const cplx* Vg = A + (size_t)r0 * n + pc0;   // V[t][c] = Vg[t * n + c] for t > c
    __syncthreads();
    for (int e = tid; e < NB * NB; e += NTH) Tp[e] = Tg[(size_t)p * NB * NB + e];
    if (warp < 4) {   // W = V^H Y[r0:]  (NB x KC): warp w -> column tile w
      ZT g;
      zt_zero(g);
      cplx vv[8], vn[8];
#pragma unroll
      for (int u = 0; u < 8; ++u) vv[u] = Vg[(size_t)min(4 * u + fc, m - 1) * n + fr];
      for (int kb = 0; kb < m; kb += 32) {
#pragma unroll
        for (int u = 0; u < 8; ++u) vn[u] = Vg[(size_t)min(kb + 32 + 4 * u + fc, m - 1) * n + fr];
#pragma unroll
        for (int u = 0; u < 8; ++u) {
          const int kk = kb + 4 * u + fc;
          const cplx a = kk < m ? (kk > fr ? cconj(vv[u]) : (kk == fr ? make_double2(1.0, 0.0) : cz())) : cz();
          const cplx b = kk < m ? Ys[(size_t)(r0 + kk) * BT_KC + warp * 8 + fr] : cz();
          zstep(g, a, b);
        }
#pragma unroll
        for (int u = 0; u < 8; ++u) vv[u] = vn[u];
      }
#pragma unroll
      for (int h = 0; h < 2; ++h) Ws[fr * BT_KC + warp * 8 + 2 * fc + h] = zt_get(g, h);
    }
    __syncthreads();
    if (warp < 4) {   // W2 = T W
      ZT g;
      zt_zero(g);
#pragma unroll
      for (int k0 = 0; k0 < NB; k0 += 4) {
        const int kk = k0 + fc;
        zstep(g, Tp[fr * NB + kk], Ws[kk * BT_KC + warp * 8 + fr]);
      }
#pragma unroll
      for (int h = 0; h < 2; ++h) W2[fr * BT_KC + warp * 8 + 2 * fc + h] = zt_get(g, h);
    }
    __syncthreads();
    const int nstrip = (m + 7) >> 3;
    for (int sI = warp; sI < nstrip; sI += BT_W) {   // Y[r0:] -= V W2
      const int row = sI * 8 + fr;
      const bool rv = row < m;
      ZT y[BT_KC / 8];
#pragma unroll
      for (int q = 0; q < BT_KC / 8; ++q) zt_zero(y[q]);
      cplx vr[NB / 4];
#pragma unroll
      for (int u = 0; u < NB / 4; ++u) vr[u] = Vg[(size_t)min(row, m - 1) * n + 4 * u + fc];
#pragma unroll
      for (int k0 = 0; k0 < NB; k0 += 4) {
        const int kk = k0 + fc;
        const cplx a = rv ? (row > kk ? vr[k0 / 4] : (row == kk ? make_double2(1.0, 0.0) : cz())) : cz();
#pragma unroll
        for (int q = 0; q < BT_KC / 8; ++q) zstep(y[q], a, W2[kk * BT_KC + q * 8 + fr]);
      }
      if (rv) {
#pragma unroll
        for (int q = 0; q < BT_KC / 8; ++q)
#pragma unroll
          for (int h = 0; h < 2; ++h) {
            cplx& q0 = Ys[(size_t)(r0 + row) * BT_KC + q * 8 + 2 * fc + h];
            q0 = csub(q0, zt_get(y[q], h));
          }
      }
    }
  }
  __syncthreads();
  for (int e = tid; e < BT_KC * n; e += NTH) {
    const int c = e / n, i = e % n;
    if (c0 + c < kmax) P.Vt[(size_t)(c0 + c) * n + i] = (c0 + c < k) ? Ys[(size_t)i * BT_KC + c] : cz();
  }
}

std::atomic<int> g_route{0};

}  // namespace

void heev2s_set_route(int route) { g_route.store(route); }
int heev2s_route() { return g_route.load(); }

bool heev2s_use(int n, int count) {
  static const int env = [] {
    const char* e = getenv("TTN_HEEV_2S");
    return e ? atoi(e) : -1;
  }();
  const int r = g_route.load();
  if (r == 1 || env == 0) return false;
  if (n < H2S_MIN_N || n > H2S_MAX_N) return false;
  if (r == 2 || env == 1) return true;
  // measured on config 3 (ncu launch lists, profiles/): order 192 (896 Grams per step) 10.4 ->
  // 8.8 ms with the two-stage path, order 128 (1280 Grams) 5.4 -> 5.9 ms; config 5 neutral
  (void)count;
  return n >= H2S_ROUTE_N;
}

void launch_heev2s_reduce(const HeevProblem* d, int nprob, int maxn, cudaStream_t s) {
  if (nprob == 0) return;
  const size_t sm1 = s1_smem_bytes(maxn), sm2 = s2_smem_bytes(maxn);
  func_smem(heev_he2hb, s1_smem_bytes(H2S_MAX_N));
  func_smem(heev_hb2st, s2_smem_bytes(H2S_MAX_N));
  launch_k(heev_he2hb, nprob, S1_T, sm1, s, d);
  count_launch();
  launch_k(heev_hb2st, nprob, s2_warps(maxn) * 32, sm2, s, d);
  count_launch();
}

void heev2s_assign_blocks(HeevProblem* h, int nprob, int& nblocks) {
  nblocks = 0;
  for (int i = 0; i < nprob; ++i) {
    h[i].bstart = nblocks;
    nblocks += (h[i].kmax + BT_KC - 1) / BT_KC;
  }
}

void launch_heev2s_backtr(const HeevProblem* d, int nprob, int nblocks, int maxn, cudaStream_t s) {
  if (nprob == 0 || nblocks == 0) return;
  func_smem(heev_bt2s, bt_smem_bytes(H2S_MAX_N));
  launch_k(heev_bt2s, nblocks, BT_W * 32, bt_smem_bytes(maxn), s, d, nprob);
  count_launch();
}

}  // namespace tcbc
