// Grouped complex-FP64 GEMM on the B200 FP64 tensor path (DMMA).
//
// Every contraction of the CBC hot path (Eqs. 10-12 and 14; the Grams
// G = X^H X of B:5 (a); S = Z L^T; R = Q^H Z; factors U^H X) is lowered to
//   C = alpha * op(A) op(B) + beta * C
// over many independent problems of different shapes in one launch.
//
// sm_100a has no tcgen05 kind::f64: FP64 tensor-core math is the warp-level
// mma.sync.m8n8k4.f64 (SASS DMMA.8x8x4).  Measured peak on this B200 pool: 37.1 TF/s
// (profiles/fp64_peaks_r01.json).  One DMMA = 256 FMAs, so the SM issues one DMMA per
// ~4 clocks: the kernel needs register blocking (32x32 complex warp tiles = 64 DMMA per
// 8 LDS.128) rather than shared-memory bandwidth.
// Complex product by the 4M rule on separate re/im accumulators:
//   Cr += Ar Br - Ai Bi,  Ci += Ar Bi + Ai Br.
// Operands are staged in shared memory by a 3-stage cp.async (16 B per complex) pipeline.
#include "kernels.h"
#include "prof.h"
#include <cstdio>
#include <vector>
#include <algorithm>

namespace tcbc {

namespace {

constexpr int BM = 64, BN = 64, BK = 8, STAGES = 3, THREADS = 128;
constexpr int PADK = BK + 4;   // m-major / n-major rows: 12 complex = 192 B (conflict-free frags)

template <bool TA, bool TB>
struct Smem {
  static constexpr int A_ELEMS = TA ? BK * BM : BM * PADK;
  static constexpr int B_ELEMS = TB ? BN * PADK : BK * BN;
  static constexpr int BYTES = STAGES * (A_ELEMS + B_ELEMS) * 16;
};

__device__ __forceinline__ void cp_async16(void* smem, const void* gmem, bool valid) {
  unsigned saddr = static_cast<unsigned>(__cvta_generic_to_shared(smem));
  int sz = valid ? 16 : 0;
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16, %2;\n" ::"r"(saddr), "l"(gmem), "r"(sz));
}
__device__ __forceinline__ void cp_async_commit() { asm volatile("cp.async.commit_group;\n" ::); }
template <int N>
__device__ __forceinline__ void cp_async_wait() { asm volatile("cp.async.wait_group %0;\n" ::"n"(N)); }

__device__ __forceinline__ void dmma(double& c0, double& c1, double a, double b) {
  asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
               : "+d"(c0), "+d"(c1)
               : "d"(a), "d"(b));
}

__device__ __forceinline__ int find_problem(const GemmProblem* p, int n, int tile) {
  int lo = 0, hi = n - 1;
  while (lo < hi) {
    int mid = (lo + hi + 1) >> 1;
    if (p[mid].tile_start <= tile) lo = mid; else hi = mid - 1;
  }
  return lo;
}

template <bool TA, bool TB>
__global__ void __launch_bounds__(THREADS) zgemm_grouped(const GemmProblem* __restrict__ probs, int nprob) {
  extern __shared__ __align__(16) unsigned char smem_raw[];
  cplx* As = reinterpret_cast<cplx*>(smem_raw);
  cplx* Bs = As + STAGES * Smem<TA, TB>::A_ELEMS;

  const int pi = find_problem(probs, nprob, blockIdx.x);
  const GemmProblem P = probs[pi];
  const int t = blockIdx.x - P.tile_start;
  const int m0 = (t / P.tiles_n) * BM, n0 = (t % P.tiles_n) * BN;
  const int M = P.M, N = P.N, K = P.K;
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int wm = (warp >> 1) * 32, wn = (warp & 1) * 32;
  const bool conjA = (P.opA & 2) != 0, conjB = (P.opB & 2) != 0;

  auto load_stage = [&](int stage, int k0) {
    cplx* as = As + stage * Smem<TA, TB>::A_ELEMS;
    cplx* bs = Bs + stage * Smem<TA, TB>::B_ELEMS;
#pragma unroll
    for (int r = 0; r < (BM * BK) / THREADS; ++r) {
      int idx = tid + r * THREADS;
      if (!TA) {
        int m = idx / BK, k = idx % BK;
        bool v = (m0 + m < M) && (k0 + k < K);
        const cplx* src = v ? P.A + (long long)(m0 + m) * P.lda + (k0 + k) : P.A;
        cp_async16(as + m * PADK + k, src, v);
      } else {
        int k = idx / BM, m = idx % BM;
        bool v = (m0 + m < M) && (k0 + k < K);
        const cplx* src = v ? P.A + (long long)(k0 + k) * P.lda + (m0 + m) : P.A;
        cp_async16(as + k * BM + m, src, v);
      }
    }
#pragma unroll
    for (int r = 0; r < (BN * BK) / THREADS; ++r) {
      int idx = tid + r * THREADS;
      if (!TB) {
        int k = idx / BN, n = idx % BN;
        bool v = (n0 + n < N) && (k0 + k < K);
        const cplx* src = v ? P.B + (long long)(k0 + k) * P.ldb + (n0 + n) : P.B;
        cp_async16(bs + k * BN + n, src, v);
      } else {
        int n = idx / BK, k = idx % BK;
        bool v = (n0 + n < N) && (k0 + k < K);
        const cplx* src = v ? P.B + (long long)(n0 + n) * P.ldb + (k0 + k) : P.B;
        cp_async16(bs + n * PADK + k, src, v);
      }
    }
  };

  double acc_re[4][4][2], acc_im[4][4][2];
#pragma unroll
  for (int i = 0; i < 4; ++i)
#pragma unroll
    for (int j = 0; j < 4; ++j) {
      acc_re[i][j][0] = acc_re[i][j][1] = 0.0;
      acc_im[i][j][0] = acc_im[i][j][1] = 0.0;
    }

  const int ktiles = (K + BK - 1) / BK;
#pragma unroll
  for (int s = 0; s < STAGES - 1; ++s) {
    if (s < ktiles) load_stage(s, s * BK);
    cp_async_commit();
  }

  const int fr = lane >> 2, fc = lane & 3;   // fragment row / col within 8x4 / 4x8
  for (int kt = 0; kt < ktiles; ++kt) {
    cp_async_wait<STAGES - 2>();
    __syncthreads();
    {  // prefetch stage kt + STAGES - 1 (its buffer was consumed at iteration kt - 1)
      int kn = kt + STAGES - 1;
      if (kn < ktiles) load_stage(kn % STAGES, kn * BK);
      cp_async_commit();
    }
    const cplx* as = As + (kt % STAGES) * Smem<TA, TB>::A_ELEMS;
    const cplx* bs = Bs + (kt % STAGES) * Smem<TA, TB>::B_ELEMS;
#pragma unroll
    for (int kk = 0; kk < BK; kk += 4) {
      double ar[4], ai[4], nai[4], br[4], bi[4];
#pragma unroll
      for (int i = 0; i < 4; ++i) {
        int m = wm + i * 8 + fr, k = kk + fc;
        cplx a = TA ? as[k * BM + m] : as[m * PADK + k];
        ar[i] = a.x;
        ai[i] = conjA ? -a.y : a.y;
        nai[i] = -ai[i];
      }
#pragma unroll
      for (int j = 0; j < 4; ++j) {
        int n = wn + j * 8 + fr, k = kk + fc;
        cplx b = TB ? bs[n * PADK + k] : bs[k * BN + n];
        br[j] = b.x;
        bi[j] = conjB ? -b.y : b.y;
      }
#pragma unroll
      for (int i = 0; i < 4; ++i)
#pragma unroll
        for (int j = 0; j < 4; ++j) {
          dmma(acc_re[i][j][0], acc_re[i][j][1], ar[i], br[j]);
          dmma(acc_im[i][j][0], acc_im[i][j][1], ar[i], bi[j]);
          dmma(acc_re[i][j][0], acc_re[i][j][1], nai[i], bi[j]);
          dmma(acc_im[i][j][0], acc_im[i][j][1], ai[i], br[j]);
        }
    }
  }
  cp_async_wait<0>();

  // epilogue: C = alpha * acc + beta * C
  const cplx al = P.alpha, be = P.beta;
  const bool use_beta = (be.x != 0.0 || be.y != 0.0);
#pragma unroll
  for (int i = 0; i < 4; ++i) {
    int m = m0 + wm + i * 8 + fr;
    if (m >= M) continue;
#pragma unroll
    for (int j = 0; j < 4; ++j) {
#pragma unroll
      for (int h = 0; h < 2; ++h) {
        int n = n0 + wn + j * 8 + fc * 2 + h;
        if (n >= N) continue;
        double re = acc_re[i][j][h], im = acc_im[i][j][h];
        cplx out;
        out.x = al.x * re - al.y * im;
        out.y = al.x * im + al.y * re;
        cplx* cp = P.C + (long long)m * P.ldc + n;
        if (use_beta) {
          cplx c = *cp;
          out.x += be.x * c.x - be.y * c.y;
          out.y += be.x * c.y + be.y * c.x;
        }
        *cp = out;
      }
    }
  }
}

template <bool TA, bool TB>
void launch_variant(GemmProblem* h, int n, Stager& st, cudaStream_t s) {
  int tiles = 0;
  for (int i = 0; i < n; ++i) {
    int tm = (h[i].M + BM - 1) / BM, tn = (h[i].N + BN - 1) / BN;
    h[i].tile_start = tiles;
    h[i].tiles_n = std::max(tn, 1);
    tiles += tm * tn;
  }
  if (tiles == 0) return;
  const GemmProblem* d = static_cast<const GemmProblem*>(st.put(h, sizeof(GemmProblem) * n));
  static bool attr_done = false;
  if (!attr_done) {
    cudaFuncSetAttribute(zgemm_grouped<TA, TB>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                         Smem<TA, TB>::BYTES);
    attr_done = true;
  }
  double flops = 0.0, bytes = 0.0;
  for (int i = 0; i < n; ++i) {
    flops += 8.0 * (double)h[i].M * h[i].N * h[i].K;
    bytes += 16.0 * ((double)h[i].M * h[i].K + (double)h[i].K * h[i].N + (double)h[i].M * h[i].N);
  }
  prof_begin(s);
  zgemm_grouped<TA, TB><<<tiles, THREADS, Smem<TA, TB>::BYTES, s>>>(d, n);
  prof_end(s, "zgemm", flops, bytes);
  count_launch();
}

}  // namespace

void launch_gemm(GemmProblem* h, int n, Stager& st, cudaStream_t s) {
  // split by storage layout (transpose bits); conjugation is a runtime flag
  std::vector<GemmProblem> g[4];
  for (int i = 0; i < n; ++i) {
    if (h[i].M <= 0 || h[i].N <= 0) continue;
    g[(h[i].opA & 1) * 2 + (h[i].opB & 1)].push_back(h[i]);
  }
  if (!g[0].empty()) launch_variant<false, false>(g[0].data(), (int)g[0].size(), st, s);
  if (!g[1].empty()) launch_variant<false, true>(g[1].data(), (int)g[1].size(), st, s);
  if (!g[2].empty()) launch_variant<true, false>(g[2].data(), (int)g[2].size(), st, s);
  if (!g[3].empty()) launch_variant<true, true>(g[3].data(), (int)g[3].size(), st, s);
}

}  // namespace tcbc
