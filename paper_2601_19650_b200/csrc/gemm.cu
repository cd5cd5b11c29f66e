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
#include <cuda.h>
#include <algorithm>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <stdexcept>
#include <string>
#include <unordered_map>
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
//
// TMA variant (TMA = true; problems whose operands fold to tensor-map boxes, tma_fold): every
// stage is BK = 8 complex = 128 B along the operand's unit-stride leg, loaded with the 128-byte
// swizzle (16-byte chunk c of 128-byte row r lands at c ^ (r & 7)), unpadded:
//   unit leg = the row leg (m of A, n of B): [row/8][k][8] -- BM/8 boxes of 8 rows x 8 k
//   unit leg = k:                            [row][8]      -- one box of BM rows x 8 k
// Fragments take k = 2*fc + q in k-step q (A and B alike), which makes every quarter-warp's
// eight 16-byte fragment loads hit eight distinct chunks in both layouts.
template <int BM, int BN, bool AKM, bool BNM, int ST, bool TMA = false>
struct Cfg {
  static constexpr int LDAK = BM + 2, LDBK = BN + 2;
  static constexpr int A_ELEMS = TMA ? BM * BK : (AKM ? BK * LDAK : BM * PADK);
  static constexpr int B_ELEMS = TMA ? BN * BK : (BNM ? BN * PADK : BK * LDBK);
  static constexpr int TAB = (2 * (3 * BM + 3 * BN) + 2 * ST * BK) * 8;
  static constexpr int TMAB = TMA ? (2 * ST * 8 + 1024) : 0;   // stage barriers, alignment
  static constexpr int BYTES = ST * (A_ELEMS + B_ELEMS) * 16 + TAB + 2 * (int)sizeof(GemmProblem) + 64 + TMAB;
};

__device__ __forceinline__ void cp_async16(void* smem, const void* gmem, bool valid) {
  unsigned saddr = static_cast<unsigned>(__cvta_generic_to_shared(smem));
  int sz = valid ? 16 : 0;
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16, %2;\n" ::"r"(saddr), "l"(gmem), "r"(sz));
}
__device__ __forceinline__ void cp_async_commit() { asm volatile("cp.async.commit_group;\n" ::); }
template <int N>
__device__ __forceinline__ void cp_async_wait() { asm volatile("cp.async.wait_group %0;\n" ::"n"(N)); }

// ---- TMA (cp.async.bulk.tensor) staging with mbarrier completion
__device__ __forceinline__ unsigned smem_u32(const void* p) { return static_cast<unsigned>(__cvta_generic_to_shared(p)); }
__device__ __forceinline__ void mbar_init(unsigned bar, unsigned count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(bar), "r"(count) : "memory");
}
__device__ __forceinline__ void mbar_arrive(unsigned bar) {
  asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(bar) : "memory");
}
__device__ __forceinline__ void mbar_expect_tx(unsigned bar, unsigned bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(bar), "r"(bytes) : "memory");
}
__device__ __forceinline__ void mbar_wait(unsigned bar, unsigned parity) {
  unsigned ok = 0;
  do {
    asm volatile(
        "{ .reg .pred p; mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2; selp.u32 %0, 1, 0, p; }"
        : "=r"(ok)
        : "r"(bar), "r"(parity)
        : "memory");
  } while (!ok);
}
// one box of a 5-d tensor map (every map is padded to rank 5) into shared memory; completion
// counted on `bar`
__device__ __forceinline__ void tma_load5(unsigned dst, const void* map, unsigned bar, const int* c) {
  asm volatile("cp.async.bulk.tensor.5d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%3, %4, %5, %6, %7}], [%2];"
               ::"r"(dst), "l"(map), "r"(bar), "r"(c[0]), "r"(c[1]), "r"(c[2]), "r"(c[3]), "r"(c[4]) : "memory");
}
// exact-rank form (TTN_TMA_RANK5=0)
__device__ __forceinline__ void tma_load_r(unsigned dst, const void* map, unsigned bar, const int* c, int rank) {
  switch (rank) {
    case 1:
      asm volatile("cp.async.bulk.tensor.1d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%3}], [%2];"
                   ::"r"(dst), "l"(map), "r"(bar), "r"(c[0]) : "memory");
      break;
    case 2:
      asm volatile("cp.async.bulk.tensor.2d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%3, %4}], [%2];"
                   ::"r"(dst), "l"(map), "r"(bar), "r"(c[0]), "r"(c[1]) : "memory");
      break;
    case 3:
      asm volatile("cp.async.bulk.tensor.3d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%3, %4, %5}], [%2];"
                   ::"r"(dst), "l"(map), "r"(bar), "r"(c[0]), "r"(c[1]), "r"(c[2]) : "memory");
      break;
    case 4:
      asm volatile("cp.async.bulk.tensor.4d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%3, %4, %5, %6}], [%2];"
                   ::"r"(dst), "l"(map), "r"(bar), "r"(c[0]), "r"(c[1]), "r"(c[2]), "r"(c[3]) : "memory");
      break;
    default:
      tma_load5(dst, map, bar, c);
  }
}
// coordinate of map dim d for a box at row x / contraction index k (TmaDims rule)
__device__ __forceinline__ int tma_coord(const TmaDims& D, int d, int x) {
  int v = x / D.div[d];
  if (D.mod[d]) v %= D.mod[d];
  return d == 0 ? 2 * v : v;
}

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

// Output tile `tile` of problem P: its origin, k split, k range and k stages
struct TileG { int m0, n0, sp, kbeg, K, ktiles; bool mirror; };
template <int BM, int BN>
__device__ __forceinline__ TileG tile_geom(const GemmProblem& P, int tile) {
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
  TileG T;
  T.m0 = bi * BM;
  T.n0 = bj * BN;
  T.sp = sp;
  T.mirror = P.sym && bi != bj;
  T.kbeg = sp * P.kchunk;
  T.K = min(P.K, T.kbeg + P.kchunk);   // this tile's k range [kbeg, K)
  T.ktiles = (T.K - T.kbeg + BK - 1) / BK;
  return T;
}

// TMA producer (the first warp of the kernel's producer warpgroup): walks the CTA's tiles in the
// consumers' order and fills stage g into slot g % ST once the consumer warps have released it
// (empty barrier), completion counted on the full barrier.  Lanes 0-4 / 5-9 compute the box
// coordinates of A / B (one runtime division pair each, in parallel); lane 0 issues.
template <int BM, int BN, int ST>
__device__ __forceinline__ void tma_producer(const GemmProblem* __restrict__ probs, int nprob, int total_tiles,
                                             const CUtensorMap* __restrict__ maps, unsigned as0, unsigned bs0,
                                             unsigned full0, unsigned empty0, int lane) {
  constexpr unsigned ABYTES = BM * BK * 16, BBYTES = BN * BK * 16;
  unsigned g = 0;
  int pi = -1;
  const CUtensorMap* last = nullptr;
  for (int tile = blockIdx.x; tile < total_tiles; tile += gridDim.x) {
    if (pi < 0 || tile < probs[pi].tile_start || tile >= probs[pi].tile_start + probs[pi].tiles_mn * probs[pi].ksplit)
      pi = find_problem(probs, nprob, tile);
    const GemmProblem& P = probs[pi];
    const TileG T = tile_geom<BM, BN>(P, tile);
    const TmaDims& D = lane < 5 ? P.ta : P.tb;
    const int dd = lane % 5;
    const bool kdim = (D.kmask >> dd) & 1;
    const int div = D.div[dd], mod = D.mod[dd];
    const int rowc = lane < 10 && !kdim ? tma_coord(D, dd, lane < 5 ? T.m0 : T.n0) : 0;
    const int ra = P.ta.rank, rb = P.tb.rank;
    const CUtensorMap* mA = maps + 2 * P.tma;
    if (lane == 0 && mA != last) {
      // the maps were copied into the (reused) descriptor ring by an H2D copy -- a write the
      // tensormap proxy must be ordered after, or the TMA unit may still hold a descriptor an
      // earlier launch staged at the same address
      asm volatile("fence.proxy.tensormap::generic.acquire.sys [%0], 128;" ::"l"(mA) : "memory");
      asm volatile("fence.proxy.tensormap::generic.acquire.sys [%0], 128;" ::"l"(mA + 1) : "memory");
      asm volatile("prefetch.tensormap [%0];" ::"l"(mA) : "memory");
      asm volatile("prefetch.tensormap [%0];" ::"l"(mA + 1) : "memory");
      last = mA;
    }
    for (int Tk = 0; Tk < T.ktiles; ++Tk, ++g) {
      const unsigned slot = g % ST;
      int v = rowc;
      if (lane < 10 && kdim) {
        v = (T.kbeg + Tk * BK) / div;
        if (mod) v %= mod;
        if (dd == 0) v *= 2;
      }
      int c[10];
#pragma unroll
      for (int j = 0; j < 10; ++j) c[j] = __shfl_sync(0xffffffffu, v, j);
      if (lane == 0) {
        mbar_wait(empty0 + 8 * slot, ((g / ST) & 1u) ^ 1u);
        const unsigned bar = full0 + 8 * slot;
        mbar_expect_tx(bar, ABYTES + BBYTES);
        tma_load_r(as0 + slot * ABYTES, mA, bar, c, ra);
        tma_load_r(bs0 + slot * BBYTES, mA + 1, bar, c + 5, rb);
      }
      __syncwarp();
    }
  }
}

// Persistent: CTA c takes tiles c, c + gridDim.x, ...  Each tile's operand tables (row / column
// offsets, problem descriptor) are double-buffered in shared memory, so the next tile is set up
// and its first STAGES-1 operand stages are in flight (cp.async) while this tile's epilogue
// stores its accumulators: the prologue latency of short-K tiles (config 3's K = 32 steps)
// hides behind the epilogue instead of idling the tensor pipe.
template <int BM, int BN, int WGM, int WGN, bool AKM, bool BNM, int ST, int MINB, bool TMA>
__global__ void __launch_bounds__(TMA ? 2 * THREADS : THREADS, MINB) zgemm_grouped(const GemmProblem* __restrict__ probs, int nprob,
                                                            int total_tiles, const CUtensorMap* __restrict__ maps) {
  TCBC_PDL_WAIT();
  using C_ = Cfg<BM, BN, AKM, BNM, ST, TMA>;
  constexpr int WTM = BM / WGM, WTN = BN / WGN;     // warp tile
  constexpr int TM = WTM / 8, TN = WTN / 8;         // DMMA tiles per warp
  constexpr int TABN = 3 * BM + 3 * BN;             // offsets per table buffer
  constexpr int PWORDS = (int)(sizeof(GemmProblem) / 8);
  static_assert(sizeof(GemmProblem) % 8 == 0, "descriptor copy");
  static_assert(WGM * WGN == THREADS / 32, "warp grid");
  static_assert((BM * BK) % THREADS == 0 && (BN * BK) % THREADS == 0, "load mapping");
  extern __shared__ __align__(16) unsigned char smem_raw[];
  // TMA boxes land 1024-byte aligned (the 128-byte swizzle pattern repeats every 1 KB)
  unsigned char* sbase = smem_raw + (TMA ? ((1024u - (smem_u32(smem_raw) & 1023u)) & 1023u) : 0u);
  cplx* As = reinterpret_cast<cplx*>(sbase);
  cplx* Bs = As + ST * C_::A_ELEMS;
  long long* tab = reinterpret_cast<long long*>(Bs + ST * C_::B_ELEMS);   // [2][TABN]
  long long* kA = tab + 2 * TABN;            // [ST][BK] k-leg offsets into A (-1: k >= K)
  long long* kB = kA + ST * BK;          // [ST][BK] k-leg offsets into B
  GemmProblem* sP = reinterpret_cast<GemmProblem*>(kB + ST * BK);   // [2]
  unsigned long long* fullb = reinterpret_cast<unsigned long long*>(sP + 2);   // [ST] TMA: stage loaded
  unsigned long long* emptyb = fullb + ST;                                      // [ST] TMA: stage released
  int* sPi = reinterpret_cast<int*>(fullb + (TMA ? 2 * ST : 0));      // [2] problem index
  if constexpr (TMA) {
    if (threadIdx.x == 0) {
      for (int s = 0; s < ST; ++s) {
        mbar_init(smem_u32(&fullb[s]), 1);
        mbar_init(smem_u32(&emptyb[s]), THREADS / 32);
      }
      asm volatile("fence.mbarrier_init.release.cluster;\n\tfence.proxy.async.shared::cta;" ::: "memory");
    }
    __syncthreads();
    // warpgroup 1 produces (one lane issues TMA), warpgroup 0 consumes: the producers hand their
    // registers to the consumers (per sub-partition: 2 CTAs x (216 + 40) x 32 = 16384)
    static_assert(MINB == 2, "the setmaxnreg split assumes two resident CTAs");
    if (threadIdx.x >= THREADS) {
      asm volatile("setmaxnreg.dec.sync.aligned.u32 40;" ::: "memory");
      if (threadIdx.x < THREADS + 32 && blockIdx.x < total_tiles)
        tma_producer<BM, BN, ST>(probs, nprob, total_tiles, maps, smem_u32(As), smem_u32(Bs), smem_u32(fullb),
                                 smem_u32(emptyb), threadIdx.x & 31);
      return;
    }
    asm volatile("setmaxnreg.inc.sync.aligned.u32 216;" ::: "memory");
  }
  // barrier of the THREADS consumer threads (the TMA variant's producer warp never joins)
  auto csync = [&]() {
    if constexpr (TMA) asm volatile("bar.sync 1, %0;" ::"n"(THREADS) : "memory");
    else __syncthreads();
  };
  unsigned gc = 0;   // TMA: stages consumed so far (slot gc % ST, full-barrier parity (gc / ST) & 1)

  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int wm = (warp / WGN) * WTM, wn = (warp % WGN) * WTN;
  const int fr = lane >> 2, fc = lane & 3;   // fragment row / col within 8x4 / 4x8

  using Tile = TileG;
  // descriptor + tables + first k-ring entries of `tile` into buffer `buf` (consumer threads)
  auto prepare = [&](int tile, int buf, int prev) -> Tile {
    if (tid == 0) {
      int pi = -1;
      if (prev >= 0) {   // consecutive tiles mostly belong to the same problem
        const GemmProblem& Q = sP[prev];
        if (tile >= Q.tile_start && tile < Q.tile_start + Q.tiles_mn * Q.ksplit) pi = sPi[prev];
      }
      sPi[buf] = pi >= 0 ? pi : find_problem(probs, nprob, tile);
    }
    csync();
    {
      const long long* src = reinterpret_cast<const long long*>(probs + sPi[buf]);
      long long* dst = reinterpret_cast<long long*>(sP + buf);
      for (int i = tid; i < PWORDS; i += THREADS) dst[i] = src[i];
    }
    csync();
    const GemmProblem& P = sP[buf];
    const Tile T = tile_geom<BM, BN>(P, tile);
    long long* rowA = tab + buf * TABN;
    long long* colB = rowA + BM;
    long long* rowC = colB + BN;
    long long* colC = rowC + BM;
    long long* colCm = colC + BN;
    long long* rowCn = colCm + BM;
    for (int i = tid; i < BM; i += THREADS) {
      const int m = T.m0 + i;
      if (!TMA) rowA[i] = m < P.M ? goff(m, P.nm, P.md, P.am) : -1;
      rowC[i] = m < P.M ? goff(m, P.nm, P.md, P.cm) : -1;
      if (T.mirror) colCm[i] = m < P.M ? goff(m, P.nn, P.nd, P.cn) : -1;
    }
    for (int i = tid; i < BN; i += THREADS) {
      const int n = T.n0 + i;
      if (!TMA) colB[i] = n < P.N ? goff(n, P.nn, P.nd, P.bn) : -1;
      colC[i] = n < P.N ? goff(n, P.nn, P.nd, P.cn) : -1;
      if (T.mirror) rowCn[i] = n < P.N ? goff(n, P.nm, P.md, P.cm) : -1;
    }
    if (!TMA && P.nk != 1)
      for (int j = tid; j < 2 * BK * ST; j += THREADS) {
        const int Tk = j / (2 * BK), jj = j % (2 * BK);
        if (Tk < T.ktiles) {
          const int kl = jj % BK, k = T.kbeg + Tk * BK + kl;
          if (jj < BK) kA[(Tk % ST) * BK + kl] = k < T.K ? goff(k, P.nk, P.kd, P.ak) : -1;
          else kB[(Tk % ST) * BK + kl] = k < T.K ? goff(k, P.nk, P.kd, P.bk) : -1;
        }
      }
    csync();
    return T;
  };

  // operand stage Tk of tile T (buffer buf) into ring slot Tk % ST
  auto load_stage = [&](const Tile& T, int buf, int Tk) {
    const GemmProblem& P = sP[buf];
    if constexpr (TMA) return;   // the producer warp stages TMA problems
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
      if (!TMA) cp_async_commit();
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
      const int slot = TMA ? (int)(gc % ST) : kt % ST;
      if constexpr (TMA) {
        mbar_wait(smem_u32(&fullb[slot]), (gc / ST) & 1u);
      } else {
        cp_async_wait<ST - 2>();
        __syncthreads();
      }
      // decode the k legs of tile kt + ST (slot kt % ST: its last reader, the load of
      // tile kt, was issued before this barrier); visible to the loads after the next barrier
      if (!TMA && P.nk != 1 && tid < 2 * BK && kt + ST < T.ktiles) {
        const int Tk = kt + ST, kl = tid % BK, k = T.kbeg + Tk * BK + kl;
        if (tid < BK) kA[(Tk % ST) * BK + kl] = k < T.K ? goff(k, P.nk, P.kd, P.ak) : -1;
        else kB[(Tk % ST) * BK + kl] = k < T.K ? goff(k, P.nk, P.kd, P.bk) : -1;
      }
      if (!TMA) {
        const int kn = kt + ST - 1;
        if (kn < T.ktiles) load_stage(T, buf, kn);
        cp_async_commit();
      }
      const cplx* as = As + slot * C_::A_ELEMS;
      const cplx* bs = Bs + slot * C_::B_ELEMS;
      double ar[BK / 4][TM], ai[BK / 4][TM], nai[BK / 4][TM], br[BK / 4][TN], bi[BK / 4][TN];
#pragma unroll
      for (int q = 0; q < BK / 4; ++q) {
        const int k = TMA ? 2 * fc + q : q * 4 + fc;
        const int sw = k ^ fr;   // TMA: swizzled chunk of (row fr, k) in both layouts
#pragma unroll
        for (int i = 0; i < TM; ++i) {
          const int m = wm + i * 8 + fr;
          const cplx a = TMA ? (AKM ? as[((wm >> 3) + i) * 64 + k * 8 + sw] : as[m * 8 + sw])
                             : (AKM ? as[k * C_::LDAK + m] : as[m * PADK + k]);
          ar[q][i] = a.x;
          ai[q][i] = neg_if(a.y, conjA);
          nai[q][i] = neg_if(a.y, !conjA);
        }
#pragma unroll
        for (int j = 0; j < TN; ++j) {
          const int n = wn + j * 8 + fr;
          const cplx b = TMA ? (BNM ? bs[n * 8 + sw] : bs[((wn >> 3) + j) * 64 + k * 8 + sw])
                             : (BNM ? bs[n * PADK + k] : bs[k * C_::LDBK + n]);
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
      if constexpr (TMA) {   // the DMMAs have consumed the fragments (so their shared loads are
                             // complete): release the slot to the producer
        // the slot's next writer is the async proxy (TMA): order this thread's generic-proxy
        // reads of it first (without the fence config 3 showed corrupted stages)
        asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
        __syncwarp();
        if (lane == 0) mbar_arrive(smem_u32(&emptyb[slot]));
        ++gc;
      }
    }
    // every warp is done with this tile's stages and k ring: set up the next tile and start
    // its loads, then store this one
    const int next = tile + gridDim.x;
    const bool more = next < total_tiles;
    csync();
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
  if (!TMA) cp_async_wait<0>();
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
// TMA variants: two CTAs of (consumer + producer warpgroup) per SM -- the register split of
// setmaxnreg is sized for two -- and a deeper ring (the producer runs ahead on its own warp)
#ifndef TCBC_TMA_ST
#define TCBC_TMA_ST 4
#endif
template <int BM, int BN, bool TMA = false> struct Occ {
  static constexpr bool SK = BM == 16 || BN == 16;
  static constexpr int ST = TMA ? TCBC_TMA_ST : (SK ? TCBC_SKINNY_ST : STAGES), MINB = TMA ? 2 : (SK ? TCBC_SKINNY_MINB : 2);
};

template <int BM, int BN, int WGM, int WGN, bool AKM, bool BNM, bool TMA>
void launch_variant(const GemmProblem* d, int n, int tiles, cudaStream_t s, const CUtensorMap* maps) {
  if (n == 0 || tiles == 0) return;
  constexpr int ST = Occ<BM, BN, TMA>::ST, MINB = Occ<BM, BN, TMA>::MINB;
  using C_ = Cfg<BM, BN, AKM, BNM, ST, TMA>;
  static_assert(MINB * C_::BYTES <= 227 * 1024, "shared memory for the resident CTAs");
  func_smem(zgemm_grouped<BM, BN, WGM, WGN, AKM, BNM, ST, MINB, TMA>, C_::BYTES);
  const int grid = std::min(tiles, MINB * 148);   // persistent: MINB resident CTAs per SM
  launch_k(zgemm_grouped<BM, BN, WGM, WGN, AKM, BNM, ST, MINB, TMA>, grid, TMA ? 2 * THREADS : THREADS, C_::BYTES, s, d,
           n, tiles, maps);
  count_launch();
}

// ---------------------------------------------------------------- TMA tensor maps
// A leg of a multi-index: extent and element stride.
struct Leg { long long ext, stride; };
// legs innermost first, extent-1 legs dropped, adjacent legs that address one affine range merged
int norm_legs(int n, const int* d, const long long* st, Leg* out) {
  int c = 0;
  for (int i = n - 1; i >= 0; --i) {
    if (d[i] == 1) continue;
    if (c > 0 && st[i] == out[c - 1].ext * out[c - 1].stride) {
      out[c - 1].ext *= d[i];
      continue;
    }
    out[c++] = {d[i], st[i]};
  }
  if (c == 0) out[c++] = {1, 1};
  return c;
}
// box extents over legs (innermost first) such that every T-aligned block of the multi-index is
// one box: a leg either holds the rest of the block (its extent a multiple of it) or is covered
// whole; the outermost leg may end ragged (out-of-range coordinates are zero-filled by TMA)
bool fold_block(const Leg* L, int n, int T, int* box) {
  long long rem = T;
  for (int j = 0; j < n; ++j) {
    if (rem == 1) { box[j] = 1; continue; }
    if (j == n - 1 || L[j].ext % rem == 0) { box[j] = (int)rem; rem = 1; continue; }
    if (rem % L[j].ext != 0) return false;
    box[j] = (int)L[j].ext;
    rem /= L[j].ext;
  }
  return rem == 1;
}

typedef CUresult (*EncodeTiledFn)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*, const cuuint64_t*,
                                  const cuuint64_t*, const cuuint32_t*, const cuuint32_t*, CUtensorMapInterleave,
                                  CUtensorMapSwizzle, CUtensorMapL2promotion, CUtensorMapFloatOOBfill);
EncodeTiledFn encode_fn() {
  static EncodeTiledFn fn = [] {
    void* f = nullptr;
    cudaDriverEntryPointQueryResult q{};
    if (cudaGetDriverEntryPointByVersion("cuTensorMapEncodeTiled", &f, 12000, cudaEnableDefault, &q) != cudaSuccess ||
        q != cudaDriverEntryPointSuccess)
      f = nullptr;
    return reinterpret_cast<EncodeTiledFn>(f);
  }();
  return fn;
}
bool tma_enabled() {
  static const bool on = [] {
    const char* e = getenv("TTN_GEMM_TMA");
    return (e == nullptr || atoi(e) != 0) && encode_fn() != nullptr;
  }();
  return on;
}

// Problems below this many complex MACs, or with K below TTN_TMA_MIN_K, stay on the cp.async
// kernels (A/B knobs, default 0: every problem whose operands fold).  Measured: any threshold
// that moves config-3 / config-2 problems off TMA costs 2-7% there; config 5's run-to-run
// spread (host-bound, 800-2400 applies/s with and without TMA) hides any effect.
double tma_min_mnk() {
  static const double v = [] { const char* e = getenv("TTN_TMA_MIN_MNK"); return e ? atof(e) : 0.0; }();
  return v;
}

int tma_min_k() {
  static const int v = [] { const char* e = getenv("TTN_TMA_MIN_K"); return e ? atoi(e) : 0; }();
  return v;
}

CUtensorMapL2promotion l2prom() {
  static const int v = [] { const char* e = getenv("TTN_TMA_L2"); return e ? atoi(e) : 2; }();
  return v == 0 ? CU_TENSOR_MAP_L2_PROMOTION_NONE : v == 1 ? CU_TENSOR_MAP_L2_PROMOTION_L2_128B : CU_TENSOR_MAP_L2_PROMOTION_L2_256B;
}
// Encoded maps are cached by their full description (the arenas hand out the same addresses
// apply after apply, so steady-state launches encode nothing).
struct MapKey {
  const void* base;
  int rank, pad_;
  unsigned long long dim[5], stride[5];
  unsigned box[5];
  bool operator==(const MapKey& o) const { return std::memcmp(this, &o, sizeof(MapKey)) == 0; }
};
struct MapKeyHash {
  size_t operator()(const MapKey& k) const {
    const unsigned char* p = reinterpret_cast<const unsigned char*>(&k);
    unsigned long long h = 1469598103934665603ull;
    for (size_t i = 0; i < sizeof(MapKey); ++i) h = (h ^ p[i]) * 1099511628211ull;
    return (size_t)h;
  }
};

// Tensor map of one operand: `rows` = its m (A) or n (B) legs, `ks` its k legs, `row_unit`
// whether the unit-stride leg is the innermost row leg (boxes of 8 rows x 8 k) or the innermost
// k leg (one box of TR rows x 8 k).  Fails (-> cp.async path) when a block does not fold.
bool tma_operand(const cplx* base, const Leg* rows, int nr, const Leg* ks, int nk, bool row_unit, int TR,
                 TmaDims& D, CUtensorMap& map) {
  if (nr + nk > 5) return false;
  MapKey key;
  std::memset(&key, 0, sizeof(key));
  key.base = base;
  int boxk[5], boxr[5];
  const Leg* u = row_unit ? rows : ks;   // the unit leg -> dim 0
  const int nu = row_unit ? nr : nk;
  if (u[0].stride != 1 || (nu > 1 && u[0].ext % BK != 0)) return false;
  // the other multi-index folds as a block (8 k values, or TR rows); the unit multi-index's
  // outer legs get box 1
  if (row_unit ? !fold_block(ks, nk, BK, boxk) : !fold_block(rows, nr, TR, boxr)) return false;
  int d = 0;
  long long pu = 1, po = 1;
  D.kmask = 0;
  D.chunks = 1;
  // row-unit operand whose unit leg is a multiple of 8: dims (8 rows | k legs | rows / 8 |
  // outer row legs), so one box of 8 x 8 x TR/8 is the whole stage, laid out [row/8][k][8]
  Leg hi[GEMM_MAXD];
  int boxh[GEMM_MAXD];
  static const bool nosplit = getenv("TTN_TMA_NOSPLIT") != nullptr;
  const bool split = !nosplit && row_unit && u[0].ext % BK == 0 && nr + nk + 1 <= 5;
  if (split) {
    hi[0] = {u[0].ext / BK, u[0].stride * BK};
    for (int j = 1; j < nu; ++j) hi[j] = u[j];
    if (!fold_block(hi, nu, TR / BK, boxh)) return false;
  } else if (row_unit) {
    return false;   // a ragged unit row leg would need one 1-KB box per 8 rows: measured far slower
  }
  auto add = [&](const Leg& L, int box, bool is_k, long long div, bool outer) {
    key.dim[d] = d == 0 ? 2ull * L.ext : (unsigned long long)L.ext;
    key.stride[d] = (unsigned long long)L.stride * 16ull;
    key.box[d] = d == 0 ? 2u * box : (unsigned)box;
    D.div[d] = (int)div;
    D.mod[d] = outer ? 0 : (int)L.ext;
    if (is_k) D.kmask |= 1 << d;
    ++d;
  };
  if (split) add(Leg{BK, 1}, BK, false, 1, false);
  else add(u[0], BK, !row_unit, 1, nu == 1);
  pu = u[0].ext;
  const Leg* o = row_unit ? ks : rows;
  const int no = row_unit ? nk : nr;
  const int* bo = row_unit ? boxk : boxr;
  for (int j = 0; j < no; ++j) {
    add(o[j], bo[j], row_unit, po, j == no - 1);
    po *= o[j].ext;
  }
  if (split) {
    long long ph = BK;
    for (int j = 0; j < nu; ++j) {
      add(hi[j], boxh[j], false, ph, j == nu - 1);
      ph *= hi[j].ext;
    }
  } else {
    for (int j = 1; j < nu; ++j) {
      add(u[j], 1, !row_unit, pu, j == nu - 1);
      pu *= u[j].ext;
    }
  }
  for (int j = 0; j < d; ++j)
    if (key.box[j] > 256 || key.dim[j] >= (1ull << 32) || key.stride[j] >= (1ull << 40)) return false;
  // pad to rank 5 (one TMA instruction form): extent-1 dims at coordinate 0 ((x / 1) % 1)
  static const bool pad5 = [] { const char* e = getenv("TTN_TMA_RANK5"); return e != nullptr && atoi(e) != 0; }();
  unsigned long long smax = 16;
  for (int j = 1; j < d; ++j) smax = std::max(smax, key.stride[j]);
  D.rank = d;
  for (; d < 5; ++d) {
    D.div[d] = 1;
    D.mod[d] = 1;
    if (!pad5) continue;
    key.dim[d] = 1;
    key.stride[d] = smax;
    key.box[d] = 1;
  }
  if (!pad5) d = D.rank;
  D.rank = d;   // the instruction form the producer issues
  key.rank = d;
  thread_local std::unordered_map<MapKey, CUtensorMap, MapKeyHash> cache;
  auto it = cache.find(key);
  if (it != cache.end()) {
    map = it->second;
    return true;
  }
  cuuint64_t gdim[5], gstr[4];
  cuuint32_t box[5], est[5];
  for (int j = 0; j < d; ++j) {
    gdim[j] = key.dim[j];
    box[j] = key.box[j];
    est[j] = 1;
    if (j > 0) gstr[j - 1] = key.stride[j];
  }
  auto encode = [&](CUtensorMap& out) {
    HostScope hs_("tma_encode");
    return encode_fn()(&out, CU_TENSOR_MAP_DATA_TYPE_FLOAT64, (cuuint32_t)d, const_cast<cplx*>(base), gdim, gstr, box,
                       est, CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B, l2prom(),
                       CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) == CUDA_SUCCESS;
  };
  if (!encode(map)) return false;
  if (cache.size() > (1u << 16)) cache.clear();
  cache.emplace(key, map);
  return true;
}

// both operand maps of a problem for tile rows TM (A) / TN (B), or false
bool tma_problem(GemmProblem& p, bool akm, bool bnm, int tm, int tn, CUtensorMap* maps2) {
  Leg m[GEMM_MAXD], n[GEMM_MAXD], ka[GEMM_MAXD], kb[GEMM_MAXD];
  const int nm = norm_legs(p.nm, p.md, p.am, m);
  const int nka = norm_legs(p.nk, p.kd, p.ak, ka);
  const int nn = norm_legs(p.nn, p.nd, p.bn, n);
  const int nkb = norm_legs(p.nk, p.kd, p.bk, kb);
  const bool okA = tma_operand(p.A, m, nm, ka, nka, akm, tm, p.ta, maps2[0]);
  const bool okB = okA && tma_operand(p.B, n, nn, kb, nkb, !bnm, tn, p.tb, maps2[1]);
  static const bool dbg = getenv("TTN_DEBUG_TMA") != nullptr;
  if (dbg && !okB) {   // the folds that fail, once per shape
    thread_local std::unordered_map<std::string, int> seen;
    auto legs = [](const Leg* L, int c) {
      std::string o;
      for (int j = 0; j < c; ++j) o += std::to_string(L[j].ext) + ":" + std::to_string(L[j].stride) + " ";
      return o;
    };
    const std::string k = std::string(okA ? "B" : "A") + " tile " + std::to_string(tm) + "x" + std::to_string(tn) +
                          (okA ? " n[" + legs(n, nn) + "] k[" + legs(kb, nkb) + "] row_unit=" + std::to_string(!bnm)
                               : " m[" + legs(m, nm) + "] k[" + legs(ka, nka) + "] row_unit=" + std::to_string(akm));
    if (seen[k]++ == 0)
      fprintf(stderr, "[tma-fail] %s MNK %dx%dx%d\n", k.c_str(), p.M, p.N, p.K);
  }
  return okB;
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
  constexpr int NV = kNumShapes * 8;   // (shape, A layout, B layout, TMA)
  thread_local std::vector<unsigned char> grp;
  thread_local std::vector<CUtensorMap> tmaps;
  grp.assign(n, 255);
  tmaps.clear();
  const bool use_tma = tma_enabled();
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
    p.tma = -1;
    if (use_tma && p.K >= tma_min_k() && (double)p.M * p.N * p.K >= tma_min_mnk()) {
      CUtensorMap m2[2];
      if (tma_problem(p, akm, bnm, kShapes[best].bm, kShapes[best].bn, m2)) {
        p.tma = (int)(tmaps.size() / 2);
        tmaps.push_back(m2[0]);
        tmaps.push_back(m2[1]);
      }
    }
    const int g = (best * 4 + v) * 2 + (p.tma >= 0 ? 1 : 0);
    ++cnt[g];
    grp[i] = (unsigned char)g;
    ++total;
  }
  if (total == 0) return;
  static const bool dbg = getenv("TTN_DEBUG_GEMM") != nullptr;
  if (dbg) {
    double ft = 0.0, fa = 0.0;
    for (int i = 0; i < n; ++i) {
      if (grp[i] == 255) continue;
      const double f = (double)h[i].M * h[i].N * h[i].K;
      fa += f;
      if (h[i].tma >= 0) ft += f;
    }
    fprintf(stderr, "[gemm-tma] %zu of %d problems, %.3f of the MNK on TMA\n", tmaps.size() / 2, total, fa > 0 ? ft / fa : 0.0);
  }
  // grouped order straight into the staging buffer, then the split-k problems again for the
  // reduction kernel
  int off[NV + 1];
  off[0] = 0;
  for (int g = 0; g < NV; ++g) off[g + 1] = off[g] + cnt[g];
  // problems, then the tensor maps (128-byte aligned) in the same staged block
  const size_t prob_bytes = sizeof(GemmProblem) * ((size_t)total + nsplit);
  const size_t map_off = (prob_bytes + 127) & ~size_t(127);
  const size_t stage_bytes = tmaps.empty() ? prob_bytes : map_off + sizeof(CUtensorMap) * tmaps.size();
  GemmProblem* ord = static_cast<GemmProblem*>(st.reserve(stage_bytes));
  if (!tmaps.empty()) std::memcpy(reinterpret_cast<char*>(ord) + map_off, tmaps.data(), sizeof(CUtensorMap) * tmaps.size());
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
    switch (g / 8) {
      case 0: tiles[g] = assign_tiles<64, 64>(q, cnt[g], flops, bytes); break;
      case 1: tiles[g] = assign_tiles<128, 32>(q, cnt[g], flops, bytes); break;
      case 2: tiles[g] = assign_tiles<32, 128>(q, cnt[g], flops, bytes); break;
      case 3: tiles[g] = assign_tiles<128, 16>(q, cnt[g], flops, bytes); break;
      default: tiles[g] = assign_tiles<16, 128>(q, cnt[g], flops, bytes); break;
    }
  }
  const GemmProblem* d = static_cast<const GemmProblem*>(st.commit(ord, stage_bytes));
  const CUtensorMap* dmaps = tmaps.empty() ? nullptr : reinterpret_cast<const CUtensorMap*>(reinterpret_cast<const char*>(d) + map_off);
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
#define TCBC_LV1(G, BM, BN, WM, WN, AK, BN_, T) \
  launch_variant<BM, BN, WM, WN, AK, BN_, T>(d + off[G], cnt[G], tiles[G], pick(G), dmaps);
#define TCBC_LV(G, BM, BN, WM, WN)                 \
  TCBC_LV1(G + 0, BM, BN, WM, WN, false, false, false) \
  TCBC_LV1(G + 1, BM, BN, WM, WN, false, false, true)  \
  TCBC_LV1(G + 2, BM, BN, WM, WN, false, true, false)  \
  TCBC_LV1(G + 3, BM, BN, WM, WN, false, true, true)   \
  TCBC_LV1(G + 4, BM, BN, WM, WN, true, false, false)  \
  TCBC_LV1(G + 5, BM, BN, WM, WN, true, false, true)   \
  TCBC_LV1(G + 6, BM, BN, WM, WN, true, true, false)   \
  TCBC_LV1(G + 7, BM, BN, WM, WN, true, true, true)
  prof_begin(s);
  TCBC_LV(0, 64, 64, 2, 2)
  TCBC_LV(8, 128, 32, 4, 1)
  TCBC_LV(16, 32, 128, 1, 4)
  TCBC_LV(24, 128, 16, 4, 1)
  TCBC_LV(32, 16, 128, 1, 4)
#undef TCBC_LV
#undef TCBC_LV1
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
