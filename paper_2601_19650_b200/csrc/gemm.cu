// Grouped complex-FP64 tensor-contraction GEMM on the B200 FP64 tensor path (DMMA).
//
// Every contraction of the CBC hot path (Eqs. 10-12 and 14; the Grams
// G = X^H X of B:5 (a); S = Z L^T; R = Q^H Z; factors U^H X) is lowered to
//   C[m, n] = alpha * sum_k opA(A)[m, k] opB(B)[k, n] + beta * C[m, n]
// where m, n, k are MULTI-indices (up to 6 legs each) addressed through arbitrary strides:
// the leg permutations of the tensor network are fused into the operand loads and the
// output store, so no transpose kernel ever runs between contraction steps.
//
// sm_100a has no tcgen05 kind::f64: FP64 tensor-core math is the warp-level
// mma.sync.m8n8k4.f64 (SASS DMMA.8x8x4).  Measured peak on this pool: 37.1 TF/s
// (profiles/fp64_peaks_r01.json) = one DMMA per 16 clocks per SM sub-partition; the same
// microbenchmark shows that 2 warps per sub-partition with 8 independent accumulator chains
// each saturate it.  So the kernel is organised around (i) independent DMMA chains: a warp
// tile of 4x4 (or 4x2) 8x8 tiles, and the four real products of the complex 4M rule
//   Cr += Ar Br - Ai Bi,  Ci += Ar Bi + Ai Br
// issued pass by pass (each accumulator is touched once per 16/32 DMMAs, never back to back),
// (ii) fragments of both k-steps of a stage read from shared memory before the first DMMA,
// (iii) no integer division in the k loop: the multi-index -> offset decode of the k legs is
// done one stage ahead by 2*BK threads into a small shared-memory ring (rows / columns are
// decoded once per CTA).  Operands are staged by a 3-stage cp.async (16 B = one complex)
// pipeline; shared-memory layouts are chosen per problem (k-contiguous or m/n-contiguous legs)
// so the global loads coalesce whenever one leg of the operand has unit stride.
#include "kernels.h"
#include "prof.h"
#include <algorithm>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <stdexcept>
#include <string>
#include <vector>

namespace tcbc {

namespace {

constexpr int BK = 8, STAGES = 3, THREADS = 128;
#ifndef TCBC_SKINNY_ST
#define TCBC_SKINNY_ST 2
#endif
#ifndef TCBC_SKINNY_MINB
#define TCBC_SKINNY_MINB 3
#endif
constexpr int PADK = BK + 4;   // m-major / n-major rows: 12 complex = 192 B (conflict-free frags)

// k-major rows (As[k][m], Bs[k][n]) are padded by 2 complex (32 B): the 4 k-rows a fragment
// load touches then start in different bank quarters (no 4-way conflicts)
template <int BM, int BN, bool AKM, bool BNM, int ST>
struct Cfg {
  static constexpr int LDAK = BM + 2, LDBK = BN + 2;
  static constexpr int A_ELEMS = AKM ? BK * LDAK : BM * PADK;
  static constexpr int B_ELEMS = BNM ? BN * PADK : BK * LDBK;
  static constexpr int TAB = (2 * (3 * BM + 3 * BN) + 2 * ST * BK) * 8;
  static constexpr int BYTES = ST * (A_ELEMS + B_ELEMS) * 16 + TAB + 2 * (int)sizeof(GemmProblem) + 64;
};

__device__ __forceinline__ void cp_async16(void* smem, const void* gmem, bool valid) {
  unsigned saddr = static_cast<unsigned>(__cvta_generic_to_shared(smem));
  int sz = valid ? 16 : 0;
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16, %2;\n" ::"r"(saddr), "l"(gmem), "r"(sz));
}
__device__ __forceinline__ void cp_async_commit() { asm volatile("cp.async.commit_group;\n" ::); }
template <int N>
__device__ __forceinline__ void cp_async_wait() { asm volatile("cp.async.wait_group %0;\n" ::"n"(N)); }

// Not volatile: the accumulator operands carry the dependencies, so ptxas may interleave the
// fragment loads of the next k-step with these.
__device__ __forceinline__ void dmma(double& c0, double& c1, double a, double b) {
  asm("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
      : "+d"(c0), "+d"(c1)
      : "d"(a), "d"(b));
}

// sign flip on the integer pipe (keeps the FP64 pipe out of the inner loop)
__device__ __forceinline__ double neg_if(double x, bool neg) {
  return neg ? __hiloint2double(__double2hiint(x) ^ 0x80000000, __double2loint(x)) : x;
}

// binary exponent of a double from its bit pattern (zero / denormal: "no data")
__device__ __forceinline__ int bexp(double x) {
  const int be = (__double2hiint(x) >> 20) & 0x7ff;
  return be ? be - 1023 : -2147483000;
}

// offset of multi-index x in a group of n legs (row-major: last leg fastest); the outermost
// leg needs no division
__device__ __forceinline__ long long goff(int x, int n, const int* d, const long long* s) {
  long long off = 0;
#pragma unroll 1
  for (int i = n - 1; i >= 1; --i) {
    int q = x / d[i];
    off += (long long)(x - q * d[i]) * s[i];
    x = q;
  }
  return off + (long long)x * s[0];
}

__device__ __forceinline__ int find_problem(const GemmProblem* p, int n, int tile) {
  int lo = 0, hi = n - 1;
  while (lo < hi) {
    int mid = (lo + hi + 1) >> 1;
    if (p[mid].tile_start <= tile) lo = mid; else hi = mid - 1;
  }
  return lo;
}

// Persistent: CTA c takes tiles c, c + gridDim.x, ...  Each tile's operand tables (row / column
// offsets, problem descriptor) are double-buffered in shared memory, so the next tile is set up
// and its first STAGES-1 operand stages are in flight (cp.async) while this tile's epilogue
// stores its accumulators: the prologue latency of short-K tiles (config 3's K = 32 steps)
// hides behind the epilogue instead of idling the tensor pipe.
template <int BM, int BN, int WGM, int WGN, bool AKM, bool BNM, int ST, int MINB>
__global__ void __launch_bounds__(THREADS, MINB) zgemm_grouped(const GemmProblem* __restrict__ probs, int nprob,
                                                            int total_tiles) {
  TCBC_PDL_WAIT();
  using C_ = Cfg<BM, BN, AKM, BNM, ST>;
  constexpr int WTM = BM / WGM, WTN = BN / WGN;     // warp tile
  constexpr int TM = WTM / 8, TN = WTN / 8;         // DMMA tiles per warp
  constexpr int TABN = 3 * BM + 3 * BN;             // offsets per table buffer
  constexpr int PWORDS = (int)(sizeof(GemmProblem) / 8);
  static_assert(sizeof(GemmProblem) % 8 == 0, "descriptor copy");
  static_assert(WGM * WGN == THREADS / 32, "warp grid");
  static_assert((BM * BK) % THREADS == 0 && (BN * BK) % THREADS == 0, "load mapping");
  extern __shared__ __align__(16) unsigned char smem_raw[];
  cplx* As = reinterpret_cast<cplx*>(smem_raw);
  cplx* Bs = As + ST * C_::A_ELEMS;
  long long* tab = reinterpret_cast<long long*>(Bs + ST * C_::B_ELEMS);   // [2][TABN]
  long long* kA = tab + 2 * TABN;            // [ST][BK] k-leg offsets into A (-1: k >= K)
  long long* kB = kA + ST * BK;          // [ST][BK] k-leg offsets into B
  GemmProblem* sP = reinterpret_cast<GemmProblem*>(kB + ST * BK);   // [2]
  int* sPi = reinterpret_cast<int*>(sP + 2);                            // [2] problem index

  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int wm = (warp / WGN) * WTM, wn = (warp % WGN) * WTN;
  const int fr = lane >> 2, fc = lane & 3;   // fragment row / col within 8x4 / 4x8

  struct Tile { int m0, n0, sp, kbeg, K, ktiles; bool mirror; };
  // descriptor + tables + first k-ring entries of `tile` into buffer `buf` (all threads)
  auto prepare = [&](int tile, int buf, int prev) -> Tile {
    if (tid == 0) {
      int pi = -1;
      if (prev >= 0) {   // consecutive tiles mostly belong to the same problem
        const GemmProblem& Q = sP[prev];
        if (tile >= Q.tile_start && tile < Q.tile_start + Q.tiles_mn * Q.ksplit) pi = sPi[prev];
      }
      sPi[buf] = pi >= 0 ? pi : find_problem(probs, nprob, tile);
    }
    __syncthreads();
    {
      const long long* src = reinterpret_cast<const long long*>(probs + sPi[buf]);
      long long* dst = reinterpret_cast<long long*>(sP + buf);
      for (int i = tid; i < PWORDS; i += THREADS) dst[i] = src[i];
    }
    __syncthreads();
    const GemmProblem& P = sP[buf];
    const int t0 = tile - P.tile_start;
    const int sp = t0 / P.tiles_mn, t = t0 % P.tiles_mn;   // k split, output tile
    int bi, bj;
    if (P.sym) {   // lower-triangular tile index
      bi = (int)((sqrtf(8.0f * t + 1.0f) - 1.0f) * 0.5f);
      while (bi * (bi + 1) / 2 > t) --bi;
      while ((bi + 1) * (bi + 2) / 2 <= t) ++bi;
      bj = t - bi * (bi + 1) / 2;
    } else {
      bi = t / P.tiles_n;
      bj = t % P.tiles_n;
    }
    Tile T;
    T.m0 = bi * BM;
    T.n0 = bj * BN;
    T.sp = sp;
    T.mirror = P.sym && bi != bj;
    T.kbeg = sp * P.kchunk;
    T.K = min(P.K, T.kbeg + P.kchunk);   // this tile's k range [kbeg, K)
    T.ktiles = (T.K - T.kbeg + BK - 1) / BK;
    long long* rowA = tab + buf * TABN;
    long long* colB = rowA + BM;
    long long* rowC = colB + BN;
    long long* colC = rowC + BM;
    long long* colCm = colC + BN;
    long long* rowCn = colCm + BM;
    for (int i = tid; i < BM; i += THREADS) {
      const int m = T.m0 + i;
      rowA[i] = m < P.M ? goff(m, P.nm, P.md, P.am) : -1;
      rowC[i] = m < P.M ? goff(m, P.nm, P.md, P.cm) : -1;
      if (T.mirror) colCm[i] = m < P.M ? goff(m, P.nn, P.nd, P.cn) : -1;
    }
    for (int i = tid; i < BN; i += THREADS) {
      const int n = T.n0 + i;
      colB[i] = n < P.N ? goff(n, P.nn, P.nd, P.bn) : -1;
      colC[i] = n < P.N ? goff(n, P.nn, P.nd, P.cn) : -1;
      if (T.mirror) rowCn[i] = n < P.N ? goff(n, P.nm, P.md, P.cm) : -1;
    }
    if (P.nk != 1)
      for (int j = tid; j < 2 * BK * ST; j += THREADS) {
        const int Tk = j / (2 * BK), jj = j % (2 * BK);
        if (Tk < T.ktiles) {
          const int kl = jj % BK, k = T.kbeg + Tk * BK + kl;
          if (jj < BK) kA[(Tk % ST) * BK + kl] = k < T.K ? goff(k, P.nk, P.kd, P.ak) : -1;
          else kB[(Tk % ST) * BK + kl] = k < T.K ? goff(k, P.nk, P.kd, P.bk) : -1;
        }
      }
    __syncthreads();
    return T;
  };

  // operand stage Tk of tile T (buffer buf) into ring slot Tk % ST
  auto load_stage = [&](const Tile& T, int buf, int Tk) {
    const GemmProblem& P = sP[buf];
    const long long* rowA = tab + buf * TABN;
    const long long* colB = rowA + BM;
    const bool k1 = P.nk == 1;
    const long long ak0 = P.ak[0], bk0 = P.bk[0];
    auto kofs = [&](const long long* ring, long long st0, int kl) -> long long {
      if (k1) {
        const int k = T.kbeg + Tk * BK + kl;
        return k < T.K ? (long long)k * st0 : -1;
      }
      return ring[(Tk % ST) * BK + kl];
    };
    const cplx* __restrict__ Ag = P.A;
    const cplx* __restrict__ Bg = P.B;
    const int stage = Tk % ST;
    cplx* as = As + stage * C_::A_ELEMS;
    cplx* bs = Bs + stage * C_::B_ELEMS;
    if (!AKM) {   // As[m][k]: k fixed per thread
      const int k = tid % BK;
      const long long ko = kofs(kA, ak0, k);
#pragma unroll
      for (int r = 0; r < (BM * BK) / THREADS; ++r) {
        const int m = tid / BK + r * (THREADS / BK);
        const long long ro = rowA[m];
        const bool v = ko >= 0 && ro >= 0;
        cp_async16(as + m * PADK + k, v ? Ag + ro + ko : Ag, v);
      }
    } else {      // As[k][m]
#pragma unroll
      for (int r = 0; r < (BM * BK) / THREADS; ++r) {
        const int idx = tid + r * THREADS;
        const int k = idx / BM, m = idx % BM;
        const long long ro = rowA[m], ko = kofs(kA, ak0, k);
        const bool v = ko >= 0 && ro >= 0;
        cp_async16(as + k * C_::LDAK + m, v ? Ag + ro + ko : Ag, v);
      }
    }
    if (BNM) {    // Bs[n][k]: k fixed per thread
      const int k = tid % BK;
      const long long ko = kofs(kB, bk0, k);
#pragma unroll
      for (int r = 0; r < (BN * BK) / THREADS; ++r) {
        const int n = tid / BK + r * (THREADS / BK);
        const long long co = colB[n];
        const bool v = ko >= 0 && co >= 0;
        cp_async16(bs + n * PADK + k, v ? Bg + co + ko : Bg, v);
      }
    } else {      // Bs[k][n]
#pragma unroll
      for (int r = 0; r < (BN * BK) / THREADS; ++r) {
        const int idx = tid + r * THREADS;
        const int k = idx / BN, n = idx % BN;
        const long long co = colB[n], ko = kofs(kB, bk0, k);
        const bool v = ko >= 0 && co >= 0;
        cp_async16(bs + k * C_::LDBK + n, v ? Bg + co + ko : Bg, v);
      }
    }
  };
  auto prologue = [&](const Tile& T, int buf) {
#pragma unroll
    for (int s = 0; s < ST - 1; ++s) {
      if (s < T.ktiles) load_stage(T, buf, s);
      cp_async_commit();
    }
  };

  int tile = blockIdx.x;
  if (tile >= total_tiles) return;
  int buf = 0;
  Tile T = prepare(tile, 0, -1);
  prologue(T, 0);
  while (true) {
    const GemmProblem& P = sP[buf];
    const bool conjA = P.conjA != 0, conjB = P.conjB != 0;
    double acc_re[TM][TN][2], acc_im[TM][TN][2];
#pragma unroll
    for (int i = 0; i < TM; ++i)
#pragma unroll
      for (int j = 0; j < TN; ++j) {
        acc_re[i][j][0] = acc_re[i][j][1] = 0.0;
        acc_im[i][j][0] = acc_im[i][j][1] = 0.0;
      }
    for (int kt = 0; kt < T.ktiles; ++kt) {
      cp_async_wait<ST - 2>();
      __syncthreads();
      // decode the k legs of tile kt + ST (slot kt % ST: its last reader, the load of
      // tile kt, was issued before this barrier); visible to the loads after the next barrier
      if (P.nk != 1 && tid < 2 * BK && kt + ST < T.ktiles) {
        const int Tk = kt + ST, kl = tid % BK, k = T.kbeg + Tk * BK + kl;
        if (tid < BK) kA[(Tk % ST) * BK + kl] = k < T.K ? goff(k, P.nk, P.kd, P.ak) : -1;
        else kB[(Tk % ST) * BK + kl] = k < T.K ? goff(k, P.nk, P.kd, P.bk) : -1;
      }
      {
        const int kn = kt + ST - 1;
        if (kn < T.ktiles) load_stage(T, buf, kn);
        cp_async_commit();
      }
      const cplx* as = As + (kt % ST) * C_::A_ELEMS;
      const cplx* bs = Bs + (kt % ST) * C_::B_ELEMS;
      double ar[BK / 4][TM], ai[BK / 4][TM], nai[BK / 4][TM], br[BK / 4][TN], bi[BK / 4][TN];
#pragma unroll
      for (int q = 0; q < BK / 4; ++q) {
        const int k = q * 4 + fc;
#pragma unroll
        for (int i = 0; i < TM; ++i) {
          const int m = wm + i * 8 + fr;
          const cplx a = AKM ? as[k * C_::LDAK + m] : as[m * PADK + k];
          ar[q][i] = a.x;
          ai[q][i] = neg_if(a.y, conjA);
          nai[q][i] = neg_if(a.y, !conjA);
        }
#pragma unroll
        for (int j = 0; j < TN; ++j) {
          const int n = wn + j * 8 + fr;
          const cplx b = BNM ? bs[n * PADK + k] : bs[k * C_::LDBK + n];
          br[q][j] = b.x;
          bi[q][j] = neg_if(b.y, conjB);
        }
      }
#pragma unroll
      for (int q = 0; q < BK / 4; ++q) {
#pragma unroll
        for (int i = 0; i < TM; ++i)
#pragma unroll
          for (int j = 0; j < TN; ++j) dmma(acc_re[i][j][0], acc_re[i][j][1], ar[q][i], br[q][j]);
#pragma unroll
        for (int i = 0; i < TM; ++i)
#pragma unroll
          for (int j = 0; j < TN; ++j) dmma(acc_im[i][j][0], acc_im[i][j][1], ar[q][i], bi[q][j]);
#pragma unroll
        for (int i = 0; i < TM; ++i)
#pragma unroll
          for (int j = 0; j < TN; ++j) dmma(acc_re[i][j][0], acc_re[i][j][1], nai[q][i], bi[q][j]);
#pragma unroll
        for (int i = 0; i < TM; ++i)
#pragma unroll
          for (int j = 0; j < TN; ++j) dmma(acc_im[i][j][0], acc_im[i][j][1], ai[q][i], br[q][j]);
      }
    }
    // every warp is done with this tile's stages and k ring: set up the next tile and start
    // its loads, then store this one
    const int next = tile + gridDim.x;
    const bool more = next < total_tiles;
    __syncthreads();
    Tile Tn{};
    if (more) {
      Tn = prepare(next, buf ^ 1, buf);
      prologue(Tn, buf ^ 1);
    }

    // epilogue: C = alpha * acc + beta * C (strided store: the output permutation is fused here);
    // split-k partials go raw to the workspace; Hermitian products also write the mirror tile
    {
      const long long* rowC = tab + buf * TABN + BM + BN;
      const long long* colC = rowC + BM;
      const long long* colCm = colC + BN;
      const long long* rowCn = colCm + BM;
      const int M = P.M, N = P.N;
      const cplx al = P.alpha, be = P.beta;
      const bool use_beta = (be.x != 0.0 || be.y != 0.0);
      cplx* __restrict__ Cg = P.C;
      int emax = -2147483000;
      if (P.ksplit > 1) {
        cplx* W = P.ws + (size_t)T.sp * M * N;
#pragma unroll
        for (int i = 0; i < TM; ++i) {
          const int m = T.m0 + wm + i * 8 + fr;
          if (m >= M) continue;
#pragma unroll
          for (int j = 0; j < TN; ++j)
#pragma unroll
            for (int h = 0; h < 2; ++h) {
              const int n = T.n0 + wn + j * 8 + fc * 2 + h;
              if (n < N) W[(size_t)m * N + n] = make_double2(acc_re[i][j][h], acc_im[i][j][h]);
            }
        }
      } else if (T.m0 + BM <= M && T.n0 + BN <= N && al.x == 1.0 && al.y == 0.0 && !use_beta && !T.mirror) {
        // common case (uniform branch): full tile, C = A B -- no bounds, scaling or mirror work
        const bool ex = P.exp_out != nullptr;
        long long co[TN][2];
#pragma unroll
        for (int j = 0; j < TN; ++j)
#pragma unroll
          for (int h = 0; h < 2; ++h) co[j][h] = colC[wn + j * 8 + fc * 2 + h];
#pragma unroll
        for (int i = 0; i < TM; ++i) {
          cplx* crow = Cg + rowC[wm + i * 8 + fr];
#pragma unroll
          for (int j = 0; j < TN; ++j)
#pragma unroll
            for (int h = 0; h < 2; ++h) {
              const double re = acc_re[i][j][h], im = acc_im[i][j][h];
              crow[co[j][h]] = make_double2(re, im);
              if (ex) emax = max(emax, max(bexp(re), bexp(im)));
            }
        }
        if (ex) {
          for (int o = 16; o > 0; o >>= 1) emax = max(emax, __shfl_xor_sync(0xffffffffu, emax, o));
          if (lane == 0 && emax > -2147483000) atomicMax(P.exp_out, emax);
        }
      } else {
#pragma unroll
        for (int i = 0; i < TM; ++i) {
          const int il = wm + i * 8 + fr;
          const long long ro = rowC[il];
          if (ro < 0) continue;
#pragma unroll
          for (int j = 0; j < TN; ++j) {
#pragma unroll
            for (int h = 0; h < 2; ++h) {
              const int jl = wn + j * 8 + fc * 2 + h;
              const long long co = colC[jl];
              if (co < 0) continue;
              const double re = acc_re[i][j][h], im = acc_im[i][j][h];
              cplx out;
              out.x = al.x * re - al.y * im;
              out.y = al.x * im + al.y * re;
              cplx* cp = Cg + ro + co;
              if (use_beta) {
                const cplx c = *cp;
                out.x += be.x * c.x - be.y * c.y;
                out.y += be.x * c.y + be.y * c.x;
              }
              *cp = out;
              if (T.mirror) Cg[rowCn[jl] + colCm[il]] = make_double2(out.x, -out.y);
              if (P.exp_out) emax = max(emax, max(bexp(out.x), bexp(out.y)));
            }
          }
        }
        if (P.exp_out) {   // the tile's largest binary exponent (uniform branch)
          for (int o = 16; o > 0; o >>= 1) emax = max(emax, __shfl_xor_sync(0xffffffffu, emax, o));
          if (lane == 0 && emax > -2147483000) atomicMax(P.exp_out, emax);
        }
      }
    }
    if (!more) break;
    tile = next;
    buf ^= 1;
    T = Tn;
  }
  cp_async_wait<0>();
}

// split-k reduction: C = alpha * sum_s W_s + beta * C (C through its strided legs)
__global__ void zgemm_splitk_reduce(const GemmProblem* __restrict__ probs, int nprob) {
  TCBC_PDL_WAIT();
  const GemmProblem& P = probs[blockIdx.y];
  const long long MN = (long long)P.M * P.N;
  const cplx al = P.alpha, be = P.beta;
  const bool use_beta = (be.x != 0.0 || be.y != 0.0);
  for (long long e = blockIdx.x * (long long)blockDim.x + threadIdx.x; e < MN; e += (long long)gridDim.x * blockDim.x) {
    double re = 0.0, im = 0.0;
    for (int s = 0; s < P.ksplit; ++s) {
      const cplx w = P.ws[s * MN + e];
      re += w.x;
      im += w.y;
    }
    const int m = (int)(e / P.N), n = (int)(e % P.N);
    if (P.sym && (m >> 6) < (n >> 6)) {   // upper tile of a Hermitian product: mirror of (n, m)
      re = 0.0;
      im = 0.0;
      for (int s = 0; s < P.ksplit; ++s) {
        const cplx w = P.ws[s * MN + (long long)n * P.N + m];
        re += w.x;
        im -= w.y;
      }
    }
    cplx* cp = P.C + goff(m, P.nm, P.md, P.cm) + goff(n, P.nn, P.nd, P.cn);
    cplx out = make_double2(al.x * re - al.y * im, al.x * im + al.y * re);
    if (use_beta) {
      const cplx c = *cp;
      out.x += be.x * c.x - be.y * c.y;
      out.y += be.x * c.y + be.y * c.x;
    }
    *cp = out;
    if (P.exp_out) {
      const int e = max(bexp(out.x), bexp(out.y));
      if (e > -2147483000) atomicMax(P.exp_out, e);
    }
  }
}

// tile bookkeeping of one variant's problems (tile_start, tiles_n, tiles_mn); returns the tiles
template <int BM, int BN>
int assign_tiles(GemmProblem* h, int n, double& flops, double& bytes) {
  int tiles = 0;
  for (int i = 0; i < n; ++i) {
    GemmProblem& p = h[i];
    const int tm = (p.M + BM - 1) / BM, tn = (p.N + BN - 1) / BN;
    p.tile_start = tiles;
    p.tiles_n = std::max(tn, 1);
    p.tiles_mn = p.sym ? tm * (tm + 1) / 2 : tm * tn;
    tiles += p.tiles_mn * std::max(p.ksplit, 1);
    flops += p.sym ? 8.0 * 0.5 * (double)p.M * (p.M + 1) * p.K : 8.0 * (double)p.M * p.N * p.K;
    bytes += 16.0 * ((double)p.M * p.K + (double)p.K * p.N + (double)p.M * p.N);
  }
  return tiles;
}

// stages / resident CTAs per SM: the 16-wide skinny tiles are latency-bound (short k loops, few
// warps), so they trade a pipeline stage for a third resident CTA
template <int BM, int BN> struct Occ { static constexpr int ST = (BM == 16 || BN == 16) ? TCBC_SKINNY_ST : STAGES, MINB = (BM == 16 || BN == 16) ? TCBC_SKINNY_MINB : 2; };

template <int BM, int BN, int WGM, int WGN, bool AKM, bool BNM>
void launch_variant(const GemmProblem* d, int n, int tiles, cudaStream_t s) {
  if (n == 0 || tiles == 0) return;
  constexpr int ST = Occ<BM, BN>::ST, MINB = Occ<BM, BN>::MINB;
  using C_ = Cfg<BM, BN, AKM, BNM, ST>;
  static_assert(MINB * C_::BYTES <= 227 * 1024, "shared memory for the resident CTAs");
  func_smem(zgemm_grouped<BM, BN, WGM, WGN, AKM, BNM, ST, MINB>, C_::BYTES);
  const int grid = std::min(tiles, MINB * 148);   // persistent: MINB resident CTAs per SM
  launch_k(zgemm_grouped<BM, BN, WGM, WGN, AKM, BNM, ST, MINB>, grid, THREADS, C_::BYTES, s, d, n, tiles);
  count_launch();
}

// CTA tile shapes (BM x BN); warp tiles 32x32 except the 16-wide skinny shapes (32x16, 16x32)
struct TileShape { int bm, bn; double eff; };
constexpr TileShape kShapes[] = {{64, 64, 1.0}, {128, 32, 1.0}, {32, 128, 1.0}, {128, 16, 0.8}, {16, 128, 0.8}};
constexpr int kNumShapes = 5;

// estimated cost of a problem on a tile shape: padded DMMA work / relative warp-tile efficiency
double shape_cost(const GemmProblem& p, const TileShape& t) {
  const double mp = (double)((p.M + t.bm - 1) / t.bm) * t.bm;
  const double np = (double)((p.N + t.bn - 1) / t.bn) * t.bn;
  const double kp = (double)((p.K + BK - 1) / BK) * BK;
  return mp * np * kp / t.eff;
}

}  // namespace

void gemm_from_ops(GemmProblem& g, int opA, long long lda, int opB, long long ldb, long long ldc) {
  g.nm = g.nn = g.nk = 1;
  g.md[0] = g.M;
  g.nd[0] = g.N;
  g.kd[0] = g.K;
  if (opA & 1) { g.am[0] = 1; g.ak[0] = lda; } else { g.am[0] = lda; g.ak[0] = 1; }
  if (opB & 1) { g.bn[0] = ldb; g.bk[0] = 1; } else { g.bk[0] = ldb; g.bn[0] = 1; }
  g.cm[0] = ldc;
  g.cn[0] = 1;
  g.conjA = (opA & 2) ? 1 : 0;
  g.conjB = (opB & 2) ? 1 : 0;
}


// ---------------------------------------------------------------- forked variant streams
constexpr int kAux = 3;
struct AuxStreams {
  int device = -1;
  cudaStream_t s[kAux] = {};
  cudaEvent_t fork = nullptr;
  cudaEvent_t join[kAux] = {};
};
#define TTN_GEMM_CHECK(x)                                                                   \
  do {                                                                                      \
    cudaError_t e__ = (x);                                                                  \
    if (e__ != cudaSuccess) throw std::runtime_error(std::string(#x) + ": " + cudaGetErrorString(e__)); \
  } while (0)
// per host thread and device (worker contexts run on their own threads)
AuxStreams& aux_streams() {
  thread_local std::vector<AuxStreams> per_dev;
  int dev = 0;
  cudaGetDevice(&dev);
  for (auto& a : per_dev)
    if (a.device == dev) return a;
  per_dev.emplace_back();
  AuxStreams& a = per_dev.back();
  a.device = dev;
  for (int i = 0; i < kAux; ++i) {
    TTN_GEMM_CHECK(cudaStreamCreateWithFlags(&a.s[i], cudaStreamNonBlocking));
    TTN_GEMM_CHECK(cudaEventCreateWithFlags(&a.join[i], cudaEventDisableTiming));
  }
  TTN_GEMM_CHECK(cudaEventCreateWithFlags(&a.fork, cudaEventDisableTiming));
  return a;
}
bool getenv_fork() {
  static const bool off = getenv("TTN_GEMM_NO_FORK") != nullptr;
  return !off;
}

void launch_gemm(GemmProblem* h, int n, Stager& st, cudaStream_t s, Scratch* ws, const char* family) {
  HostScope hs_("launch_gemm");
  // group by tile shape (least padded work) and shared-memory layouts; Hermitian products take
  // the square tile (lower-triangle tiles only); problems that cannot fill the GPU with output
  // tiles get their k range split (deterministic: partials reduced in a second kernel).  All
  // groups go to the device in one staging copy and are timed as one zgemm launch set.
  constexpr int NV = kNumShapes * 4;
  thread_local std::vector<unsigned char> grp;
  grp.assign(n, 255);
  int cnt[NV] = {0};
  int nsplit = 0, total = 0;
  int memo_m = -1, memo_n = -1, memo_k = -1, memo_best = 0;
  for (int i = 0; i < n; ++i) {
    GemmProblem& p = h[i];
    if (p.M <= 0 || p.N <= 0) continue;
    if (p.sym && !(p.M == p.N && p.alpha.y == 0.0 && p.beta.x == 0.0 && p.beta.y == 0.0)) p.sym = 0;
    // A: k-major smem when the innermost m leg is unit-stride and the innermost k leg is not
    const bool akm = (p.ak[p.nk - 1] != 1) && (p.am[p.nm - 1] == 1);
    // B: n-major smem when the innermost k leg is unit-stride and the innermost n leg is not
    const bool bnm = (p.bn[p.nn - 1] != 1) && (p.bk[p.nk - 1] == 1);
    const int v = (akm ? 2 : 0) + (bnm ? 1 : 0);
    int best = 0;
    if (!p.sym) {   // consecutive problems mostly share a shape (one plan step over the batch)
      if (p.M == memo_m && p.N == memo_n && p.K == memo_k) {
        best = memo_best;
      } else {
        double bc = shape_cost(p, kShapes[0]);
        for (int t = 1; t < kNumShapes; ++t) {
          const double c = shape_cost(p, kShapes[t]);
          if (c < bc * 0.999) { bc = c; best = t; }
        }
        memo_m = p.M;
        memo_n = p.N;
        memo_k = p.K;
        memo_best = best;
      }
    }
    p.ksplit = 1;
    p.kchunk = std::max(p.K, 1);
    p.ws = nullptr;
    if (ws) {
      const long long tm = (p.M + kShapes[best].bm - 1) / kShapes[best].bm;
      const long long tiles = p.sym ? tm * (tm + 1) / 2 : tm * ((p.N + kShapes[best].bn - 1) / kShapes[best].bn);
      if (tiles < 148 && p.K >= 1024) {
        int S = (int)std::min<long long>((296 + tiles - 1) / tiles, std::min(16, p.K / 512));
        if (S > 1) {
          int chunk = (p.K + S - 1) / S;
          chunk = (chunk + BK - 1) / BK * BK;
          S = (p.K + chunk - 1) / chunk;
          p.ksplit = S;
          p.kchunk = chunk;
          p.ws = static_cast<cplx*>(ws->get(sizeof(cplx) * (size_t)S * p.M * p.N));
          ++nsplit;
        }
      }
    }
    const int g = best * 4 + v;
    ++cnt[g];
    grp[i] = (unsigned char)g;
    ++total;
  }
  if (total == 0) return;
  // grouped order straight into the staging buffer, then the split-k problems again for the
  // reduction kernel
  int off[NV + 1];
  off[0] = 0;
  for (int g = 0; g < NV; ++g) off[g + 1] = off[g] + cnt[g];
  const size_t stage_bytes = sizeof(GemmProblem) * ((size_t)total + nsplit);
  GemmProblem* ord = static_cast<GemmProblem*>(st.reserve(stage_bytes));
  {
    int pos[NV];
    for (int g = 0; g < NV; ++g) pos[g] = off[g];
    int sp = total;
    for (int i = 0; i < n; ++i) {
      if (grp[i] == 255) continue;
      std::memcpy(&ord[pos[grp[i]]++], &h[i], sizeof(GemmProblem));
      if (h[i].ksplit > 1) std::memcpy(&ord[sp++], &h[i], sizeof(GemmProblem));
    }
  }
  double flops = 0.0, bytes = 0.0;
  int tiles[NV];
  for (int g = 0; g < NV; ++g) {
    GemmProblem* q = ord + off[g];
    switch (g / 4) {
      case 0: tiles[g] = assign_tiles<64, 64>(q, cnt[g], flops, bytes); break;
      case 1: tiles[g] = assign_tiles<128, 32>(q, cnt[g], flops, bytes); break;
      case 2: tiles[g] = assign_tiles<32, 128>(q, cnt[g], flops, bytes); break;
      case 3: tiles[g] = assign_tiles<128, 16>(q, cnt[g], flops, bytes); break;
      default: tiles[g] = assign_tiles<16, 128>(q, cnt[g], flops, bytes); break;
    }
  }
  const GemmProblem* d = static_cast<const GemmProblem*>(st.commit(ord, stage_bytes));
  // Variant kernels of one launch set are independent (distinct outputs); when several are
  // non-empty they run on forked streams so one persistent kernel's tail overlaps the next
  // kernel instead of idling SMs (fork / join by events: also valid inside a graph capture).
  int nv = 0;
  for (int g = 0; g < NV; ++g) nv += (cnt[g] > 0 && tiles[g] > 0) ? 1 : 0;
  AuxStreams& aux = aux_streams();
  const bool fork = nv > 1 && getenv_fork();
  if (fork) TTN_GEMM_CHECK(cudaEventRecord(aux.fork, s));
  int used = 0;
  auto pick = [&](int g) -> cudaStream_t {
    if (!fork || cnt[g] == 0 || tiles[g] == 0) return s;
    if (used == 0) {   // the first non-empty variant stays on s
      ++used;
      return s;
    }
    cudaStream_t a = aux.s[(used - 1) % kAux];
    if (used <= kAux) TTN_GEMM_CHECK(cudaStreamWaitEvent(a, aux.fork, 0));
    ++used;
    return a;
  };
#define TCBC_LV(G, BM, BN, WM, WN)                                                                      \
  launch_variant<BM, BN, WM, WN, false, false>(d + off[G + 0], cnt[G + 0], tiles[G + 0], pick(G + 0)); \
  launch_variant<BM, BN, WM, WN, false, true>(d + off[G + 1], cnt[G + 1], tiles[G + 1], pick(G + 1));  \
  launch_variant<BM, BN, WM, WN, true, false>(d + off[G + 2], cnt[G + 2], tiles[G + 2], pick(G + 2));  \
  launch_variant<BM, BN, WM, WN, true, true>(d + off[G + 3], cnt[G + 3], tiles[G + 3], pick(G + 3));
  prof_begin(s);
  TCBC_LV(0, 64, 64, 2, 2)
  TCBC_LV(4, 128, 32, 4, 1)
  TCBC_LV(8, 32, 128, 1, 4)
  TCBC_LV(12, 128, 16, 4, 1)
  TCBC_LV(16, 16, 128, 1, 4)
#undef TCBC_LV
  if (fork)   // join: s waits for every aux stream used
    for (int a = 0; a < std::min(used - 1, kAux); ++a) {
      TTN_GEMM_CHECK(cudaEventRecord(aux.join[a], aux.s[a]));
      TTN_GEMM_CHECK(cudaStreamWaitEvent(s, aux.join[a], 0));
    }
  prof_end(s, family, flops, bytes);
  if (nsplit > 0) {
    long long mx = 0;
    for (int i = total; i < total + nsplit; ++i) mx = std::max<long long>(mx, (long long)ord[i].M * ord[i].N);
    const int gx = (int)std::min<long long>((mx + 255) / 256, 1024);
    prof_begin(s);
    launch_k(zgemm_splitk_reduce, dim3(gx, (unsigned)nsplit), 256, 0, s, d + total, nsplit);
    prof_end(s, "zgemm_reduce", 0.0, 0.0);
    count_launch();
  }
}

}  // namespace tcbc
