// Top-k eigenpairs of LARGE compress Grams (n > kLargeN, e.g. BASELINE config 4's junction
// Grams, n = 2048, k = 128) by Chebyshev-filtered subspace iteration with Rayleigh-Ritz.
//
// Why not the tridiagonal pipeline of heev.cu: a one-stage Householder tridiagonalisation is
// BLAS-2 -- it streams the trailing matrix once per column, n^3/3 complex reads (46 GB for
// n = 2048) through L2/HBM, seconds per matrix.  CBC only needs the top-k eigenspace of the
// Gram (reading A1/A2: the same kept subspace as the truncated SVD), and here k << n, so
// the work is re-expressed as dense complex GEMMs on the DMMA path (gemm.cu), where B200's
// FP64 throughput lives:
//   V <- orth(random n x p),  p = kmax + oversampling
//   repeat:  Rayleigh-Ritz  W = G V, H = V^H W = Z Theta Z^H (heev.cu, p <= 512), V <- V Z,
//            residuals r_t = ||W z_t - theta_t V z_t|| for the wanted t < kmax;
//            stop when every wanted r_t <= kResTol * theta_1;
//            otherwise filter V <- p_m(G) V D with the scaled three-term Chebyshev recurrence
//            (Zhou & Saad) damping [0, theta_p] (the unwanted end of the spectrum of a PSD
//            Gram), D = diag(1 / p_m(theta_j)) keeping the columns O(1), then CholeskyQR2.
// Every Chebyshev degree is ONE grouped GEMM over all matrices of the level:
//   Y_{j+1} = a_j (G - c I) Y_j - b_j Y_{j-1}   (in place over Y_{j-1}: C = alpha A B + beta C).
// The result is written in heev.cu's HeevProblem contract (lam descending, Vt rows = eigenvectors,
// k = min(max_bond, #{lam > tol^2 lam_1}, #{lam > floor lam_1}) >= 1, w = trace - sum_{t<k} lam_t),
// so the factor formation downstream is shared.  Accuracy: the kept subspace is accurate to
// ~ r / gap (Davis-Kahan); r <= 1e-12 lambda_1 is far inside the parity budget (1 - cos <= 1e-10).
#include "chfsi.h"
#include "prof.h"

#include <algorithm>
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <string>

namespace tcbc {

namespace {

// converged: ||G v - theta v|| <= kResTol * theta_1 for every wanted pair.  The kept subspace
// is then accurate to ~kResTol theta_1 / gap (Davis-Kahan); with the gaps of random Grams
// (>= 1e-3 theta_1 at the cut) that is <= 1e-7 in angle, i.e. 1 - cos <= 1e-14.
constexpr double kResTol = 1e-10;
// per filter pass: amplification of the slowest wanted direction over the damped interval.
// Bounded because a Ritz vector's contamination by the top directions grows by the same
// kind of factor: 1e8 from the first (random) Ritz basis, 1e10 once residuals are small.
constexpr double kAmpFirst = 1e8, kAmpLater = 1e10, kCondMax = 1e10;
constexpr int kMaxIter = 12;

__device__ __forceinline__ unsigned hash32(unsigned x) {
  x ^= x >> 16; x *= 0x7feb352dU; x ^= x >> 15; x *= 0x846ca68bU; x ^= x >> 16;
  return x;
}

struct LargeDev {
  const cplx* G;    // n x n (full Hermitian)
  cplx* Gs;         // n x n shifted copy
  cplx* V;          // n x p
  double* dscale;   // p column scales
  double shift;
  int n, p;
};

__global__ void random_fill(LargeDev* P) {
  TCBC_PDL_WAIT();
  const LargeDev& L = P[blockIdx.y];
  const long long tot = (long long)L.n * L.p;
  for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < tot; i += (long long)gridDim.x * blockDim.x) {
    const unsigned h1 = hash32((unsigned)(i * 2 + 1) ^ 0x9e3779b9u), h2 = hash32((unsigned)(i * 2 + 2) ^ 0x7f4a7c15u);
    L.V[i] = make_double2((h1 & 0xffffff) / 16777216.0 - 0.5, (h2 & 0xffffff) / 16777216.0 - 0.5);
  }
}

__global__ void shift_copy(LargeDev* P) {
  TCBC_PDL_WAIT();
  const LargeDev& L = P[blockIdx.y];
  const long long tot = (long long)L.n * L.n;
  for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < tot; i += (long long)gridDim.x * blockDim.x) {
    cplx v = L.G[i];
    if (i / L.n == i % L.n) v.x -= L.shift;
    L.Gs[i] = v;
  }
}

__global__ void col_scale(LargeDev* P) {
  TCBC_PDL_WAIT();
  const LargeDev& L = P[blockIdx.y];
  const long long tot = (long long)L.n * L.p;
  for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < tot; i += (long long)gridDim.x * blockDim.x) {
    const double s = L.dscale[i % L.p];
    L.V[i].x *= s;
    L.V[i].y *= s;
  }
}

struct ResDev {
  const cplx* V;     // n x p Ritz vectors
  const cplx* W;     // n x p  G V
  const double* theta;
  double* res;       // kmax
  int n, p, kmax;
};

// one warp per (matrix, wanted Ritz pair): r_t = || W[:, t] - theta_t V[:, t] ||
__global__ void ritz_residual(const ResDev* P, int nprob, int maxk) {
  TCBC_PDL_WAIT();
  const int gw = (blockIdx.x * blockDim.x + threadIdx.x) >> 5, lane = threadIdx.x & 31;
  const int b = gw / maxk, t = gw % maxk;
  if (b >= nprob) return;
  const ResDev& R = P[b];
  if (t >= R.kmax) return;
  const double th = R.theta[t];
  double s = 0.0;
  for (int i = lane; i < R.n; i += 32) {
    const cplx w = R.W[(long long)i * R.p + t], v = R.V[(long long)i * R.p + t];
    const double dx = w.x - th * v.x, dy = w.y - th * v.y;
    s += dx * dx + dy * dy;
  }
  for (int o = 16; o > 0; o >>= 1) s += __shfl_xor_sync(0xffffffffu, s, o);
  if (lane == 0) R.res[t] = sqrt(s);
}

struct FinDev {
  const cplx* G;
  const cplx* V;     // n x p
  const double* theta;
  HeevProblem hp;    // destination (lam, Vt, k_out, w_out, tol2, floor_rel, max_bond)
  int p;
};

// trace, truncation decision and discarded weight (one thread per matrix), then Vt = V^T rows
__global__ void large_finish(FinDev* P, int nprob) {
  TCBC_PDL_WAIT();
  const int b = blockIdx.y;
  if (b >= nprob) return;
  const FinDev& F = P[b];
  const HeevProblem& H = F.hp;
  const int n = H.n, kmax = H.kmax;
  __shared__ double red[32];
  double tr = 0.0;
  for (int i = threadIdx.x; i < n; i += blockDim.x) tr += F.G[(long long)i * n + i].x;
  for (int o = 16; o > 0; o >>= 1) tr += __shfl_xor_sync(0xffffffffu, tr, o);
  if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = tr;
  __syncthreads();
  if (threadIdx.x == 0 && blockIdx.x == 0) {
    double trace = 0.0;
    for (int w = 0; w < (int)(blockDim.x >> 5); ++w) trace += red[w];
    const double l1 = F.theta[0];
    int k = 1;
    double kept = 0.0;
    if (trace > 0.0 && l1 > 0.0) {
      int cnt = 0;
      for (int t = 0; t < kmax; ++t)
        if (F.theta[t] > H.tol2 * l1 && F.theta[t] > H.floor_rel * l1) ++cnt;
      k = cnt < 1 ? 1 : (cnt > H.max_bond ? H.max_bond : cnt);
      for (int t = 0; t < k; ++t) kept += F.theta[t];
    }
    const int e2 = H.exp2 ? 2 * pow2_effective(*H.exp2) : 0;   // back to the unscaled Gram
    for (int t = 0; t < kmax; ++t) H.lam[t] = (t < k && trace > 0.0 && l1 > 0.0) ? ldexp(F.theta[t], e2) : 0.0;
    if (H.k_out) *H.k_out = k;
    if (H.w_out) *H.w_out = ldexp(fmax(trace - kept, 0.0), e2);
  }
  for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < (long long)kmax * n;
       i += (long long)gridDim.x * blockDim.x) {
    const int t = (int)(i / n), r = (int)(i % n);
    H.Vt[i] = F.V[(long long)r * F.p + t];
  }
}

// scaled Chebyshev filter value p_m(x) on [lo, cut] normalised at top (host scalar recurrence,
// identical to the one applied to the vectors)
double cheb_value(double x, int m, double lo, double cut, double top) {
  const double e = 0.5 * (cut - lo), c = 0.5 * (cut + lo);
  const double s1 = e / (top - c);
  double sigma = s1;
  double y0 = 1.0, y1 = (x - c) * s1 / e;
  for (int j = 2; j <= m; ++j) {
    const double sn = 1.0 / (2.0 / s1 - sigma);
    const double y2 = 2.0 * sn / e * (x - c) * y1 - sigma * sn * y0;
    y0 = y1;
    y1 = y2;
    sigma = sn;
  }
  return y1;
}

struct Job {
  HeevProblem* hp;
  int n, p, kmax;
  cplx *Gs, *V, *Y, *W, *V2, *W2, *H, *Zt, *Wg, *Li, *Q1, *tau;
  double *theta, *res, *dscale, *hwork, *thr;
  cplx* Vr;               // Ritz basis before the last filter pass (restored if that pass breaks down)
  double prev_worst = 1e300, prev_top = 0.0;
  int c = 0;              // locked (converged) leading Ritz vectors: not filtered any more
  int* info;
  bool done = false;
};

}  // namespace

bool chfsi_applicable(int n, int kmax) {
  const int p = chfsi_block(n, kmax);
  static const int lo = [] { const char* e = getenv("TTN_CHFSI_MIN_N"); return e ? atoi(e) : kLargeN; }();
  return n > lo && p <= 512 && 2 * p <= n;
}

int chfsi_block(int n, int kmax) {
  int p = kmax + std::max(32, kmax / 2);
  p = (p + 15) / 16 * 16;
  return std::min(p, n);
}

void chfsi_heev(ttn_ctx_s* ctx, std::vector<HeevProblem*>& probs, ExecStats& st) {
  if (probs.empty()) return;
  cudaStream_t s = ctx->stream;
  const int nb = (int)probs.size();
  std::vector<Job> J(nb);
  auto A = [&](size_t elems) { return static_cast<cplx*>(ctx->scratch.alloc(sizeof(cplx) * std::max<size_t>(elems, 1))); };
  auto Ad = [&](size_t elems) { return static_cast<double*>(ctx->scratch.alloc(sizeof(double) * std::max<size_t>(elems, 1))); };
  int maxk = 0;
  for (int b = 0; b < nb; ++b) {
    Job& j = J[b];
    j.hp = probs[b];
    j.n = j.hp->n;
    j.kmax = j.hp->kmax;
    j.p = chfsi_block(j.n, j.kmax);
    const size_t n = j.n, p = j.p;
    j.Gs = A(n * n);
    j.V = A(n * p); j.Y = A(n * p); j.W = A(n * p); j.V2 = A(n * p); j.W2 = A(n * p); j.Q1 = A(n * p);
    j.H = A(p * p); j.Zt = A(p * p); j.Wg = A(p * p); j.Li = A(p * p);
    j.tau = A(std::max(n, p));
    j.theta = Ad(p); j.res = Ad(j.kmax); j.dscale = Ad(p); j.thr = Ad(p); j.Vr = A(n * p);
    j.hwork = Ad(heev_work_doubles((int)p, (int)p));
    j.info = static_cast<int*>(ctx->scratch.alloc(sizeof(int) * 2));
    maxk = std::max(maxk, j.kmax);
  }
  auto large_launch = [&](void (*kern)(LargeDev*), std::vector<Job*>& act, std::vector<double>* shifts, bool scale) {
    std::vector<LargeDev> L;
    for (size_t q = 0; q < act.size(); ++q) {
      Job& j = *act[q];
      L.push_back(LargeDev{j.hp->A, j.Gs, j.V, j.dscale, shifts ? (*shifts)[q] : 0.0, j.n, j.p});
    }
    LargeDev* d = static_cast<LargeDev*>(ctx->stager->put(L.data(), sizeof(LargeDev) * L.size()));
    (void)scale;
    launch_k(kern, dim3(296, (unsigned)L.size()), 256, 0, s, d);
    count_launch();
  };
  // orthonormalise the unlocked tail V[:, c:p] of every active job in place: projected twice
  // against the locked (already orthonormal) columns V[:, 0:c], then shifted CholeskyQR3
  // (Fukaya et al.): a first Cholesky pass of Y^H Y + s I (s ~ 1e-13 max diag) brings any block
  // with cond <= ~1e13 to cond <= ~1e7, then CholeskyQR2 finishes; the span is kept throughout.
  auto orth = [&](std::vector<Job*>& act) {
    for (int rep = 0; rep < 2; ++rep) {   // Y -= V_L (V_L^H Y)
      std::vector<GemmProblem> gp1, gp2;
      for (Job* jp : act) {
        Job& j = *jp;
        if (j.c == 0) continue;
        const int64_t n = j.n, p = j.p, c = j.c, w = p - c;
        gp1.push_back(mk_gemm(j.V, OP_C, p, j.V + c, OP_N, p, j.Wg, w, c, w, n));
        GemmProblem g2 = mk_gemm(j.V, OP_N, p, j.Wg, OP_N, w, j.V + c, p, n, w, c);
        g2.alpha = make_double2(-1.0, 0.0);
        g2.beta = make_double2(1.0, 0.0);
        gp2.push_back(g2);
      }
      gemm_batch(ctx, gp1, st, "heev");
      gemm_batch(ctx, gp2, st, "heev");
    }
    for (int pass = 0; pass < 3; ++pass) {
      std::vector<GemmProblem> g1, g2;
      std::vector<PotrfProblem> p1;
      std::vector<TrtriProblem> t1;
      for (Job* jp : act) {
        Job& j = *jp;
        const int64_t n = j.n, p = j.p, c = j.c, w = p - c;
        g1.push_back(mk_gemm(j.V + c, OP_C, p, j.V + c, OP_N, p, j.Wg, w, w, w, n));
        g1.back().sym = 1;
        PotrfProblem pp{j.Wg, w, (int)w, 0, j.info + (pass == 2 ? 1 : 0), 1e-15};
        pp.shift_rel = pass == 0 ? 1e-13 : 0.0;
        p1.push_back(pp);
        t1.push_back(TrtriProblem{j.Wg, j.Li, w, (int)w, 0});
        g2.push_back(mk_gemm(j.V + c, OP_N, p, j.Li, OP_C, w, j.Q1 + c, p, n, w, w));
      }
      gemm_batch(ctx, g1, st, "heev");
      launch_potrf(p1.data(), (int)p1.size(), *ctx->stager, s);
      launch_trtri(t1.data(), (int)t1.size(), *ctx->stager, s);
      gemm_batch(ctx, g2, st, "heev");
      for (Job* jp : act) {
        Job& j = *jp;
        const size_t w = (size_t)(j.p - j.c);
        TTN_CUDA(cudaMemcpy2DAsync(j.V + j.c, sizeof(cplx) * j.p, j.Q1 + j.c, sizeof(cplx) * j.p, sizeof(cplx) * w,
                                   (size_t)j.n, cudaMemcpyDeviceToDevice, s));
      }
    }
  };
  // Rayleigh-Ritz of every active job: theta, V <- V Z (W <- G V Z), residuals of wanted pairs
  auto rayleigh_ritz = [&](std::vector<Job*>& act) {
    std::vector<GemmProblem> gw, gh, gv;
    std::vector<HeevProblem> hh;
    std::vector<ResDev> rd;
    for (Job* jp : act) {
      Job& j = *jp;
      const int64_t n = j.n, p = j.p;
      gw.push_back(mk_gemm(j.hp->A, OP_N, n, j.V, OP_N, p, j.W, p, n, p, n));     // W = G V
      gh.push_back(mk_gemm(j.V, OP_C, p, j.W, OP_N, p, j.H, p, p, p, n));         // H = V^H W
      HeevProblem h{};
      h.A = j.H; h.n = (int)p; h.kmax = (int)p; h.lam = j.theta; h.Vt = j.Zt; h.k_out = nullptr; h.w_out = nullptr;
      h.work = j.hwork; h.tau = j.tau; h.tol2 = 0.0; h.floor_rel = -1e300; h.max_bond = (int)p;
      hh.push_back(h);
      gv.push_back(mk_gemm(j.V, OP_N, p, j.Zt, OP_T, p, j.V2, p, n, p, p));       // V2 = V Z
      gv.push_back(mk_gemm(j.W, OP_N, p, j.Zt, OP_T, p, j.W2, p, n, p, p));       // W2 = W Z
      rd.push_back(ResDev{j.V2, j.W2, j.theta, j.res, (int)n, (int)p, j.kmax});
    }
    gemm_batch(ctx, gw, st, "heev");
    gemm_batch(ctx, gh, st, "heev");
    launch_heev(hh.data(), (int)hh.size(), *ctx->stager, s);
    gemm_batch(ctx, gv, st, "heev");
    const ResDev* d = static_cast<const ResDev*>(ctx->stager->put(rd.data(), sizeof(ResDev) * rd.size()));
    const long long warps = (long long)rd.size() * maxk;
    launch_k(ritz_residual, (unsigned)((warps * 32 + 255) / 256), 256, 0, s, d, (int)rd.size(), maxk);
    count_launch();
    for (Job* jp : act) {
      std::swap(jp->V, jp->V2);
      std::swap(jp->W, jp->W2);
    }
  };

  std::vector<Job*> act;
  for (auto& j : J) act.push_back(&j);
  large_launch(random_fill, act, nullptr, false);
  orth(act);
  rayleigh_ritz(act);
  int maxp = 0;
  for (auto& j : J) maxp = std::max(maxp, j.p);
  ctx->ensure_small(sizeof(double) * (size_t)nb * (maxp + maxk) + sizeof(int) * 2 * nb + 64);
  double* hbuf = reinterpret_cast<double*>(ctx->hbuf);
  int* hinfo = reinterpret_cast<int*>(hbuf + (size_t)nb * (maxp + maxk));
  int iter = 0;
  for (;; ++iter) {
    for (int b = 0; b < nb; ++b) {
      if (J[b].done) continue;
      TTN_CUDA(cudaMemcpyAsync(hbuf + (size_t)b * (maxp + maxk), J[b].theta, sizeof(double) * J[b].p,
                               cudaMemcpyDeviceToHost, s));
      TTN_CUDA(cudaMemcpyAsync(hbuf + (size_t)b * (maxp + maxk) + maxp, J[b].res, sizeof(double) * J[b].kmax,
                               cudaMemcpyDeviceToHost, s));
      TTN_CUDA(cudaMemcpyAsync(hinfo + 2 * b, J[b].info, sizeof(int) * 2, cudaMemcpyDeviceToHost, s));
    }
    ctx->sync();
    act.clear();
    std::vector<double> shifts;
    std::vector<std::vector<double>> coefs;
    for (int b = 0; b < nb; ++b) {
      Job& j = J[b];
      if (j.done) continue;
      const double* th = hbuf + (size_t)b * (maxp + maxk);
      const double* rs = th + maxp;
      const double top = th[0];
      static const bool dbgi = getenv("TTN_DEBUG_CHFSI") != nullptr;
      if (dbgi) {
        double wr = 0.0;
        for (int t = 0; t < j.kmax; ++t) wr = std::max(wr, rs[t]);
        fprintf(stderr, "[chfsi] iter %d job %d: theta0=%.6e theta_k=%.6e theta_p=%.6e maxres/theta0=%.3e info=%d,%d locked=%d\n",
                iter, b, th[0], th[j.kmax - 1], th[j.p - 1], wr / top, hinfo[2 * b], hinfo[2 * b + 1], j.c);
      }
      if (hinfo[2 * b] != 0 || hinfo[2 * b + 1] != 0) {
        // the last filter pass collapsed the block (contamination by the top directions grew
        // past double precision): fall back to the Ritz basis it started from if that one was
        // already accurate, else give up loudly
        if (j.prev_worst <= 1e-8 * j.prev_top) {
          TTN_CUDA(cudaMemcpyAsync(j.V, j.Vr, sizeof(cplx) * (size_t)j.n * j.p, cudaMemcpyDeviceToDevice, s));
          TTN_CUDA(cudaMemcpyAsync(j.theta, j.thr, sizeof(double) * j.p, cudaMemcpyDeviceToDevice, s));
          j.done = true;
          continue;
        }
        throw Error(TTN_ERR_NUMERIC, "large-Gram eigensolver: CholeskyQR of the filtered block flagged rank deficiency");
      }
      bool conv = true;
      double worst = 0.0;
      int lock = -1;   // first unconverged wanted pair: the leading ones are locked
      for (int t = 0; t < j.kmax; ++t) {
        if (!std::isfinite(th[t]) || !std::isfinite(rs[t])) throw Error(TTN_ERR_NUMERIC, "non-finite Ritz pair (non-finite input?)");
        if (th[t] <= 1e-13 * top) break;   // numerically-zero directions are never kept (reading A4)
        worst = std::max(worst, rs[t]);
        if (rs[t] > kResTol * top) {
          conv = false;
          if (lock < 0) lock = t;
        }
      }
      if (!(top > 0.0)) conv = true;   // zero Gram: nothing to resolve
      if (conv) { j.done = true; continue; }
      j.prev_worst = worst;
      j.prev_top = top;
      TTN_CUDA(cudaMemcpyAsync(j.Vr, j.V, sizeof(cplx) * (size_t)j.n * j.p, cudaMemcpyDeviceToDevice, s));
      TTN_CUDA(cudaMemcpyAsync(j.thr, j.theta, sizeof(double) * j.p, cudaMemcpyDeviceToDevice, s));
      if (iter >= kMaxIter) {
        if (worst <= 1e-9 * top) { j.done = true; continue; }
        throw Error(TTN_ERR_NUMERIC, "large-Gram eigensolver did not converge (residual " + std::to_string(worst / top) + ")");
      }
      // damp [lo, cut]: cut = smallest Ritz value (>= a tiny fraction of top), lo just below 0
      const double cut = std::max(th[j.p - 1], 1e-6 * top), lo = -1e-12 * top;
      // degree: amplify the slowest wanted direction by up to kAmp per pass, but keep the growth
      // of every Ritz vector's contamination by the top directions (~ eps * p(theta_1)/p(cut),
      // eps = current relative residual) below kCondMax so the block stays orthonormalisable
      const double kAmp = iter == 0 ? kAmpFirst : kAmpLater;
      const double eps = std::max(worst / top, 1e-16);
      const double xk = th[std::min(j.kmax, j.p) - 1];
      j.c = std::max(lock, 0);   // locked columns are projected out explicitly, so only the
      const double tu = th[j.c];  // largest UNLOCKED Ritz value bounds the contamination growth
      auto amp = [&](double x, int mm) { return std::fabs(cheb_value(x, mm, lo, cut, top) / cheb_value(cut, mm, lo, cut, top)); };
      int m = 4;
      while (m < 48 && amp(xk, m) < kAmp && eps * amp(tu, m + 2) <= kCondMax) m += 2;
      std::vector<double> cf;   // m, lo, cut, top
      cf.push_back(m); cf.push_back(lo); cf.push_back(cut); cf.push_back(top);
      coefs.push_back(cf);
      // column pre-scaling D = diag(1 / p_m(theta_j))
      std::vector<double> dsc(j.p);
      for (int t = 0; t < j.p; ++t) {
        const double v = cheb_value(th[t], m, lo, cut, top);
        dsc[t] = t < j.c ? 1.0 : (std::fabs(v) > 1e-12) ? 1.0 / v : (v < 0 ? -1e12 : 1e12);   // cap the dynamic range
      }
      TTN_CUDA(cudaMemcpyAsync(j.dscale, ctx->stager->put(dsc.data(), sizeof(double) * j.p), sizeof(double) * j.p,
                               cudaMemcpyDeviceToDevice, s));
      shifts.push_back(0.5 * (cut + lo));
      act.push_back(&j);
    }
    if (act.empty()) break;
    large_launch(shift_copy, act, &shifts, false);
    large_launch(col_scale, act, nullptr, true);
    // filter: Y = p_m(G) V, recurrence over (X, Y) with X = V, in place
    int mmax = 0;
    for (auto& cf : coefs) mmax = std::max(mmax, (int)cf[0]);
    std::vector<double> sigma(act.size()), s1(act.size());
    std::vector<cplx*> xb(act.size()), yb(act.size());   // recurrence buffers (tails of V and Y)
    {
      std::vector<GemmProblem> g;
      for (size_t q = 0; q < act.size(); ++q) {
        Job& j = *act[q];
        const double lo = coefs[q][1], cut = coefs[q][2], top = coefs[q][3];
        const double e = 0.5 * (cut - lo), c = 0.5 * (cut + lo);
        s1[q] = e / (top - c);
        sigma[q] = s1[q];
        GemmProblem gp = mk_gemm(j.Gs, OP_N, j.n, j.V + j.c, OP_N, j.p, j.Y + j.c, j.p, j.n, j.p - j.c, j.n);
        gp.alpha = make_double2(s1[q] / e, 0.0);
        g.push_back(gp);
        xb[q] = j.V + j.c;
        yb[q] = j.Y + j.c;
      }
      gemm_batch(ctx, g, st, "heev");
    }
    for (int deg = 2; deg <= mmax; ++deg) {
      std::vector<GemmProblem> g;
      for (size_t q = 0; q < act.size(); ++q) {
        Job& j = *act[q];
        if (deg > (int)coefs[q][0]) continue;
        const double lo = coefs[q][1], cut = coefs[q][2];
        const double e = 0.5 * (cut - lo);
        const double sn = 1.0 / (2.0 / s1[q] - sigma[q]);
        // X <- (2 sn / e) Gs Y - sigma sn X, then swap roles
        GemmProblem gp = mk_gemm(j.Gs, OP_N, j.n, yb[q], OP_N, j.p, xb[q], j.p, j.n, j.p - j.c, j.n);
        gp.alpha = make_double2(2.0 * sn / e, 0.0);
        gp.beta = make_double2(-sigma[q] * sn, 0.0);
        g.push_back(gp);
        sigma[q] = sn;
        std::swap(xb[q], yb[q]);
      }
      gemm_batch(ctx, g, st, "heev");
    }
    // the newest filtered tail is yb; the locked columns live in V[:, 0:c]: bring it there
    for (size_t q = 0; q < act.size(); ++q) {
      Job& j = *act[q];
      if (yb[q] != j.V + j.c)
        TTN_CUDA(cudaMemcpy2DAsync(j.V + j.c, sizeof(cplx) * j.p, yb[q], sizeof(cplx) * j.p,
                                   sizeof(cplx) * (size_t)(j.p - j.c), (size_t)j.n, cudaMemcpyDeviceToDevice, s));
    }
    orth(act);
    rayleigh_ritz(act);
  }
  // results in the HeevProblem contract
  std::vector<FinDev> F;
  for (auto& j : J) F.push_back(FinDev{j.hp->A, j.V, j.theta, *j.hp, j.p});
  FinDev* d = static_cast<FinDev*>(ctx->stager->put(F.data(), sizeof(FinDev) * F.size()));
  launch_k(large_finish, dim3(64, nb), 256, 0, s, d, nb);
  count_launch();
  static const bool dbg = getenv("TTN_DEBUG_CHFSI") != nullptr;
  if (dbg) fprintf(stderr, "[chfsi] %d matrices, n=%d p=%d kmax=%d: %d outer iterations\n", nb, J[0].n, J[0].p, J[0].kmax, iter);
}

}  // namespace tcbc
