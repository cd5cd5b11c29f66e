// CBC driver: the level-synchronous schedule of PAPER.md §III.B over a batch of
// independent instances (same parent array), every stage one set of grouped launches.
//
//   up-sweep    (Eq. 10)  deepest level first; X = T O prod_c L^{[c]}
//   down-sweep  (Eq. 11)  root level first;    Y = T O L^{[(p,i)]} prod_{c!=k} L^{[c]}
//   compress       Gram (X^H X or X X^H) -> top-k eigenpairs -> factor
//   final sweep (Eqs. 12-14) deepest first: Z = T O prod_c R^{[c]};
//               S = Z L^{[(p,i)]T}; Q = CholeskyQR2(S); T' = Q; R^{[i]} = Q^H Z
//   assembly          T'_root = Z_root
// Host synchronisation: once per compress level (data-dependent ranks) and once per final
// level (Cholesky pivot flags).
#include "chfsi.h"
#include "contract.h"
#include "runtime.h"
#include "prof.h"

#include <algorithm>
#include <chrono>
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <functional>
#include <map>
#include <memory>
#include <set>

namespace tcbc {

namespace {

struct Fac {
  cplx* p = nullptr;   // [k, b, a] row-major (fac_ba(), the default; TTN_FAC_BA=0: [k, a, b])
  int64_t k = 0, a = 0, b = 0;
};

constexpr double kRankFloor = 1e-13;   // reading A4: lambda_j <= 1e-13 lambda_1 is numerically zero
constexpr double kCholTol = 1e-13;     // relative pivot threshold of CholeskyQR (rank flag)
// exact-factor shortcut: certified lambda_min / lambda_1 lower bound; 100x
// above the rank floor, so the eigensolver route would keep every direction too (and so would
// the oracle's 1e-14 sigma floor, reading A4)
constexpr double kExactCert = 1e-11;

// labels of a node contraction
constexpr int L_SIG = 0, L_SIGP = 1, L_A = 10, L_B = 30, L_F = 50;

struct CompressJob {
  const cplx* X;
  int64_t m, n;
  Fac* dst;
  int64_t a, b;      // column legs of X (n = a*b)
  int inst;
  int* exp = nullptr;   // max binary exponent of X, written by the producing GEMM (or null)
  cplx* G_pre = nullptr;   // row-split compress: the (already range-scaled) Gram X^H X; G route only
};

struct LevelScratch : Scratch {   // the ctx's per-level arena as launcher workspace
  Arena& a;
  explicit LevelScratch(Arena& ar) : a(ar) {}
  void* get(size_t bytes) override { return a.alloc(bytes); }
};

struct QRJob {
  const cplx* S;     // m x kd
  int64_t m, kd;
  cplx* Q;           // m x r output, r = min(m, kd)
  int inst;
  int* exp = nullptr;   // max binary exponent of S, written by the producing GEMM
};

// Per-instance flop counts (8 per complex MAC).  `all` is the report's flops_algorithmic;
// `nongemm` the eigensolver / Cholesky proxies inside it; cx_exec / cx_min the node
// contractions as executed / at the cheapest pairwise order (the roofline's algorithmic work).
struct FlopAcc {
  double all = 0.0, nongemm = 0.0, cx_exec = 0.0, cx_min = 0.0;
  FlopAcc& operator+=(double v) {   // a GEMM issued as is (Gram, factor, S, QR, R)
    all += v;
    return *this;
  }
  void add_nongemm(double v) {
    all += v;
    nongemm += v;
  }
  void add_contract(double exec, double mn) {
    all += exec;
    cx_exec += exec;
    cx_min += mn;
  }
  double gemm_exec() const { return all - nongemm; }
  double gemm_min() const { return all - nongemm - (cx_exec - cx_min); }
};

// Device side of a speculative apply (no host synchronisation inside the sweeps): the host
// plans every compress with k = kmax and every QR as full rank; the device accumulates the
// discarded weights / exact-factor counts per instance and raises `flag` when a rank differs
// (1), a weight is not finite (2) or a CholeskyQR pivot fails (4) -- the caller then discards
// the result and re-runs the apply with synchronised ranks.
struct SpecDev {
  double* wacc;   // [nb]
  int* xacc;      // [nb]
  int* flag;
  bool* host_synced;   // set when a stage had to synchronise anyway (Chebyshev solver)
};

bool fac_ba() {
  static const bool v = [] { const char* e = getenv("TTN_FAC_BA"); return e == nullptr || atoi(e) != 0; }();
  return v;
}

Task node_task(const ttn_s* st, const ttn_s* op, int i, const std::map<int, const Fac*>& facs, int open_leg,
               cplx* out) {
  Task t;
  Operand T;
  T.ptr = st->node(i);
  T.dims = st->shape[i];
  T.labels.push_back(L_SIG);
  for (size_t l = 0; l + 1 < T.dims.size(); ++l) T.labels.push_back(L_A + (int)l);
  Operand O;
  O.ptr = op->node(i);
  O.dims = op->shape[i];
  O.labels.push_back(L_SIGP);
  O.labels.push_back(L_SIG);
  for (size_t l = 0; l + 2 < O.dims.size(); ++l) O.labels.push_back(L_B + (int)l);
  t.ops.push_back(T);
  t.ops.push_back(O);
  t.out_labels.push_back(L_SIGP);
  // factors (and the contraction outputs whose Grams make them) order each edge's legs
  // (operator bond, state bond) -- [k][b][a] -- when fac_ba(): the state bond is then the
  // unit-stride leg a contraction over it reads, and the kept legs (k, b) merge into one, so
  // the GEMM operands fold into TMA boxes (the (a, b) order leaves the operator bond
  // innermost, split from k by the contracted leg)
  const bool ba = fac_ba();
  for (auto& kv : facs) {
    Operand F;
    F.ptr = kv.second->p;
    if (ba) {
      F.dims = {kv.second->k, kv.second->b, kv.second->a};
      F.labels = {L_F + kv.first, L_B + kv.first, L_A + kv.first};
    } else {
      F.dims = {kv.second->k, kv.second->a, kv.second->b};
      F.labels = {L_F + kv.first, L_A + kv.first, L_B + kv.first};
    }
    t.ops.push_back(F);
    t.out_labels.push_back(L_F + kv.first);
  }
  t.out_labels.push_back((ba ? L_B : L_A) + open_leg);
  t.out_labels.push_back((ba ? L_A : L_B) + open_leg);
  t.out = out;
  return t;
}

void check_heev_size(int64_t nn) {
  if (nn > heev_max_n())
    throw Error(TTN_ERR_UNSUPPORTED, "compress Gram of order " + std::to_string(nn) + " exceeds the eigensolver limit " +
                                         std::to_string(heev_max_n()));
}

// Gram -> eigenpairs -> factor, for every job; synchronises once to read the ranks.
void compress_batch(ttn_ctx_s* ctx, std::vector<CompressJob>& jobs, int64_t max_bond, double tol,
                    ExecStats& st, std::vector<double>& w_inst, std::vector<FlopAcc>& flops_inst,
                    std::vector<int>& exact_inst, const SpecDev* spec, Comm* shard = nullptr) {
  if (jobs.empty()) return;
  HostScope hs_("compress_batch");
  const int nj = (int)jobs.size();
  // sharded (replicated top of a partitioned apply): job j's Gram, eigensolve and
  // factor run on rank j % world only; the factor rows, rank, discarded weight and shortcut
  // flag are then broadcast from that rank
  const bool sharded = shard && shard->world > 1 && !spec;
  auto mine = [&](int j) { return !sharded || j % shard->world == shard->rank; };
  std::vector<GemmProblem> grams, fgemm;
  std::vector<HeevProblem> hp(nj);
  std::vector<ScaleRowsProblem> sr;
  int* d_k = static_cast<int*>(ctx->scratch.alloc(sizeof(int) * nj));
  double* d_w = static_cast<double*>(ctx->scratch.alloc(sizeof(double) * nj));
  int* d_e = static_cast<int*>(ctx->scratch.alloc(sizeof(int) * nj));   // pow2 range exponents
  std::vector<Pow2Problem> p2(nj);
  std::vector<int64_t> kmaxs(nj);
  // exact-factor shortcut candidates: untruncated (tol = 0, max_bond >= min(m, n)) compresses
  // of the tridiagonal-solver range.  W = copy of the Gram, Cholesky, L^{-1}, certificate; the
  // eigensolver skips a certified job and its factor becomes L^H (G route) or X (K route).
  int* d_skip = static_cast<int*>(ctx->scratch.alloc(sizeof(int) * nj));
  int* d_cinfo = static_cast<int*>(ctx->scratch.alloc(sizeof(int) * nj));
  TTN_CUDA(cudaMemsetAsync(d_skip, 0, sizeof(int) * nj, ctx->stream));
  std::vector<PermProblem> ccopy;
  std::vector<PotriProblem> cpot;
  std::vector<CertProblem> ccert;
  std::vector<ExactFactorProblem> cfac;
  for (int j = 0; j < nj; ++j) {
    CompressJob& J = jobs[j];
    const int64_t m = J.m, n = J.n, nn = std::min(m, n);
    const int64_t kmax = std::min<int64_t>(max_bond, nn);
    if (!chfsi_applicable((int)std::min<int64_t>(nn, INT32_MAX), (int)kmax)) check_heev_size(nn);
    kmaxs[j] = kmax;
    cplx* G = J.G_pre;
    if (!G) {
      G = static_cast<cplx*>(ctx->scratch.alloc(sizeof(cplx) * nn * nn));
      GemmProblem g = (m >= n) ? mk_gemm(J.X, OP_C, n, J.X, OP_N, n, G, nn, n, n, m)     // G = X^H X
                               : mk_gemm(J.X, OP_N, n, J.X, OP_C, n, G, nn, m, m, n);    // K = X X^H
      g.sym = 1;   // Hermitian: lower tiles + mirror (HERK)
      if (mine(j)) grams.push_back(g);
      flops_inst[J.inst] += gemm_flops(g);
    } else if (m < n) {
      throw Error(TTN_ERR_ARG, "row-split compress needs the G route (m >= n)");
    }
    HeevProblem& h = hp[j];
    h.A = G;
    h.n = (int)nn;
    h.kmax = (int)kmax;
    h.lam = static_cast<double*>(ctx->scratch.alloc(sizeof(double) * kmax));
    h.Vt = static_cast<cplx*>(ctx->scratch.alloc(sizeof(cplx) * kmax * nn));
    h.k_out = d_k + j;
    h.w_out = d_w + j;
    h.work = static_cast<double*>(ctx->scratch.alloc(sizeof(double) * heev_work_doubles((int)nn, (int)kmax)));
    h.tau = static_cast<cplx*>(ctx->scratch.alloc(sizeof(cplx) * nn));
    h.tol2 = tol * tol;
    h.floor_rel = kRankFloor;
    int* ej = J.exp ? J.exp : d_e + j;
    h.exp2 = ej;
    p2[j] = Pow2Problem{const_cast<cplx*>(J.X), m * n, ej};
    h.max_bond = (int)std::min<int64_t>(max_bond, INT32_MAX);
    flops_inst[J.inst].add_nongemm(8.0 * ((4.0 / 3.0) * nn * nn * nn + 2.0 * nn * nn * kmax));
    // factor storage (kmax rows; the first k are the factor)
    J.dst->p = static_cast<cplx*>(ctx->env.alloc(sizeof(cplx) * kmax * n));
    J.dst->a = J.a;
    J.dst->b = J.b;
    if (m >= n) {
      ScaleRowsProblem s{};
      s.Vt = h.Vt; s.lam = h.lam; s.F = J.dst->p; s.kmax = (int)kmax; s.n = (int)n;
      if (mine(j)) sr.push_back(s);
    } else {   // F = conj(Vt) X  (U_k^H X)
      if (mine(j)) fgemm.push_back(mk_gemm(h.Vt, OP_R, m, J.X, OP_N, n, J.dst->p, n, kmax, n, m));
      flops_inst[J.inst] += 8.0 * (double)kmax * n * m;
    }
    st.peak_entries = std::max(st.peak_entries, nn * nn);
    // (below order 32 the eigensolver is launch-latency bound: the shortcut's extra launches
    // would cost more than the stages it skips)
    if (mine(j) && tol == 0.0 && kmax == nn && nn > std::max(32, heev_small_n()) && !chfsi_applicable((int)nn, (int)kmax) && (m >= n || J.X)) {
      cplx* Wc = static_cast<cplx*>(ctx->scratch.alloc(sizeof(cplx) * nn * nn));
      cplx* Li = static_cast<cplx*>(ctx->scratch.alloc(sizeof(cplx) * nn * nn));
      PermProblem pp{};
      pp.src = G; pp.dst = Wc; pp.rank = 1; pp.dims[0] = nn * nn; pp.sstride[0] = 1; pp.total = nn * nn;
      ccopy.push_back(pp);
      cpot.push_back(PotriProblem{Wc, nn, (int)nn, 1, d_cinfo + j, 0.0, 0.0, Li});
      ccert.push_back(CertProblem{G, Li, d_cinfo + j, d_skip + j, (int)nn, 0, kExactCert});
      h.skip = d_skip + j;
      ExactFactorProblem ef{};
      ef.skip = d_skip + j;
      if (m >= n) {
        ef.src = Wc; ef.mode = 0; ef.rows = (int)n; ef.cols = (int)n; ef.exp2 = ej;
      } else {
        ef.src = J.X; ef.mode = 1; ef.rows = (int)m; ef.cols = (int)n;
      }
      ef.F = J.dst->p;
      cfac.push_back(ef);
    }
  }
  {   // the Gram squares X: exponents from the producing GEMM's epilogue where available
    std::vector<Pow2Problem> have, need, back;
    for (int j = 0; j < nj; ++j) {
      if (jobs[j].G_pre || !mine(j)) continue;   // row-split: X was scaled before its partial Grams
      (jobs[j].exp ? have : need).push_back(p2[j]);
      back.push_back(p2[j]);
    }
    launch_pow2_apply(have.data(), (int)have.size(), *ctx->stager, ctx->stream);
    launch_pow2_normalize(need.data(), (int)need.size(), *ctx->stager, ctx->stream);
    gemm_batch(ctx, grams, st);
    launch_pow2_restore(back.data(), (int)back.size(), *ctx->stager, ctx->stream);   // the K-route factor reads X
  }
  if (!ccert.empty()) {   // exact-factor shortcut: Cholesky of a copy of each candidate's Gram
    launch_permute(ccopy.data(), (int)ccopy.size(), *ctx->stager, ctx->stream);
    launch_potri(cpot.data(), (int)cpot.size(), *ctx->stager, ctx->stream);
    launch_chol_certify(ccert.data(), (int)ccert.size(), *ctx->stager, ctx->stream);
  }
  if (spec) {   // speculative: k = kmax, checked on the device (no host read, no sync)
    {
      std::vector<HeevProblem> small;
      std::vector<HeevProblem*> large;
      for (auto& h : hp) {
        if (chfsi_applicable(h.n, h.kmax)) large.push_back(&h);
        else small.push_back(h);
      }
      LevelScratch lws(ctx->scratch);
      if (!small.empty()) launch_heev(small.data(), (int)small.size(), *ctx->stager, ctx->stream, {}, &lws);
      if (!large.empty()) {
        *spec->host_synced = true;
        chfsi_heev(ctx, large, st);
      }
    }
    if (!sr.empty()) launch_scale_rows(sr.data(), (int)sr.size(), *ctx->stager, ctx->stream);
    gemm_batch(ctx, fgemm, st);
    launch_exact_factor(cfac.data(), (int)cfac.size(), *ctx->stager, ctx->stream);
    std::vector<SpecCheck> sc(nj);
    for (int j = 0; j < nj; ++j) {
      sc[j] = SpecCheck{d_k + j, d_w + j, d_skip + j, (int)kmaxs[j], jobs[j].inst};
      jobs[j].dst->k = kmaxs[j];
    }
    launch_spec_check(sc.data(), nj, spec->wacc, spec->xacc, spec->flag, *ctx->stager, ctx->stream);
    return;
  }
  // ranks and discarded weights go to the host as soon as the eigenvalue stages have fixed them:
  // the host waits on that point only, and builds the next level while the eigenvector stages
  // and the factor kernels still run (the next level's launches queue behind them)
  // pinned layout: ranks (padded to 8 bytes), discarded weights, shortcut flags
  const size_t small_bytes = sizeof(int) * ((nj + 1) & ~1) + sizeof(double) * nj + sizeof(int) * nj;
  ctx->ensure_small(small_bytes);
  int* hk = reinterpret_cast<int*>(ctx->hbuf);
  double* hw = reinterpret_cast<double*>(ctx->hbuf + sizeof(int) * ((nj + 1) & ~1));
  int* hs = reinterpret_cast<int*>(hw + nj);
  auto read_ranks = [&]() {
    TTN_CUDA(cudaMemcpyAsync(hk, d_k, sizeof(int) * nj, cudaMemcpyDeviceToHost, ctx->stream));
    TTN_CUDA(cudaMemcpyAsync(hw, d_w, sizeof(double) * nj, cudaMemcpyDeviceToHost, ctx->stream));
    TTN_CUDA(cudaMemcpyAsync(hs, d_skip, sizeof(int) * nj, cudaMemcpyDeviceToHost, ctx->stream));
  };
  bool early = false;
  {   // small Grams: tridiagonal pipeline (heev.cu); large ones: Chebyshev subspace (chfsi.cu)
    std::vector<HeevProblem> small;
    std::vector<HeevProblem*> large;
    for (int j = 0; j < nj; ++j) {
      if (!mine(j)) continue;
      HeevProblem& h = hp[j];
      if (chfsi_applicable(h.n, h.kmax)) large.push_back(&h);
      else small.push_back(h);
    }
    std::function<void()> ready;
    if (large.empty() && !sharded)
      ready = [&]() {
        read_ranks();
        ctx->mark_ranks();
        early = true;
      };
    LevelScratch lws(ctx->scratch);
    if (!small.empty()) launch_heev(small.data(), (int)small.size(), *ctx->stager, ctx->stream, ready, &lws);
    else if (ready) ready();
    chfsi_heev(ctx, large, st);
  }
  if (!sr.empty()) launch_scale_rows(sr.data(), (int)sr.size(), *ctx->stager, ctx->stream);
  gemm_batch(ctx, fgemm, st);
  launch_exact_factor(cfac.data(), (int)cfac.size(), *ctx->stager, ctx->stream);   // certified jobs
  if (sharded) {   // results from each job's rank
    shard->group_start();
    for (int j = 0; j < nj; ++j) {
      const int owner = j % shard->world;
      shard->bcast(jobs[j].dst->p, sizeof(cplx) * kmaxs[j] * jobs[j].n, owner, ctx->stream);
      shard->bcast(d_k + j, sizeof(int), owner, ctx->stream);
      shard->bcast(d_w + j, sizeof(double), owner, ctx->stream);
      shard->bcast(d_skip + j, sizeof(int), owner, ctx->stream);
    }
    shard->group_end();
  }
  if (early) {
    ctx->wait_ranks();
  } else {
    // the Chebyshev solver may have grown (reallocated) the small pinned buffer: re-derive
    ctx->ensure_small(small_bytes);
    hk = reinterpret_cast<int*>(ctx->hbuf);
    hw = reinterpret_cast<double*>(ctx->hbuf + sizeof(int) * ((nj + 1) & ~1));
    hs = reinterpret_cast<int*>(hw + nj);
    read_ranks();
    ctx->sync();
  }
  for (int j = 0; j < nj; ++j) {
    if (hk[j] < 1 || hk[j] > kmaxs[j]) throw Error(TTN_ERR_NUMERIC, "eigensolver returned an invalid rank");
    if (!std::isfinite(hw[j])) throw Error(TTN_ERR_NUMERIC, "non-finite discarded weight (non-finite input?)");
    jobs[j].dst->k = hk[j];
    w_inst[jobs[j].inst] += hw[j];
    exact_inst[jobs[j].inst] += hs[j] ? 1 : 0;
  }
}

// CholeskyQR2 of every S (m > kd); Q = I for m <= kd.  Synchronises once for pivot flags.
int qr_batch(ttn_ctx_s* ctx, std::vector<QRJob>& jobs, ExecStats& st, std::vector<FlopAcc>& flops_inst,
             std::vector<int>& fb_inst, const SpecDev* spec) {
  if (jobs.empty()) return 0;
  HostScope hs_("qr_batch");
  std::vector<EyeProblem> eyes;
  std::vector<GemmProblem> g1, g2, g3, g4;
  std::vector<PotriProblem> p1, p2;
  std::vector<int> tall;
  int* d_info = static_cast<int*>(ctx->scratch.alloc(sizeof(int) * 2 * jobs.size()));
  TTN_CUDA(cudaMemsetAsync(d_info, 0, sizeof(int) * 2 * jobs.size(), ctx->stream));   // Q = I jobs stay 0
  for (size_t j = 0; j < jobs.size(); ++j) {
    QRJob& J = jobs[j];
    if (J.m <= J.kd) {
      eyes.push_back(EyeProblem{J.Q, (int)J.m, (int)J.m, 0});
      continue;
    }
    tall.push_back((int)j);
    const int64_t m = J.m, k = J.kd;
    cplx* W = static_cast<cplx*>(ctx->scratch.alloc(sizeof(cplx) * k * k));
    cplx* Li = static_cast<cplx*>(ctx->scratch.alloc(sizeof(cplx) * k * k));
    cplx* Q1 = static_cast<cplx*>(ctx->scratch.alloc(sizeof(cplx) * m * k));
    cplx* W2 = static_cast<cplx*>(ctx->scratch.alloc(sizeof(cplx) * k * k));
    cplx* Li2 = static_cast<cplx*>(ctx->scratch.alloc(sizeof(cplx) * k * k));
    auto gp = [&](const cplx* A, int opA, long long lda, const cplx* B, int opB, long long ldb, cplx* C, int64_t M,
                  int64_t N, int64_t K) {
      GemmProblem g = mk_gemm(A, opA, lda, B, opB, ldb, C, N, M, N, K);
      flops_inst[J.inst] += 8.0 * (double)M * N * K;
      return g;
    };
    g1.push_back(gp(J.S, OP_C, k, J.S, OP_N, k, W, k, k, m));        // W = S^H S
    g1.back().sym = 1;
    p1.push_back(PotriProblem{W, k, (int)k, 0, d_info + 2 * j, kCholTol, 0.0, Li});
    g2.push_back(gp(J.S, OP_N, k, Li, OP_C, k, Q1, m, k, k));        // Q1 = S L^{-H}
    g3.push_back(gp(Q1, OP_C, k, Q1, OP_N, k, W2, k, k, m));         // W2 = Q1^H Q1
    g3.back().sym = 1;
    p2.push_back(PotriProblem{W2, k, (int)k, 0, d_info + 2 * j + 1, kCholTol * 1e-2, 0.0, Li2});
    g4.push_back(gp(Q1, OP_N, k, Li2, OP_C, k, J.Q, m, k, k));       // Q = Q1 L2^{-H}
    flops_inst[J.inst].add_nongemm(8.0 * 2.0 * (k * k * k / 3.0));
  }
  if (!eyes.empty()) launch_eye(eyes.data(), (int)eyes.size(), *ctx->stager, ctx->stream);
  if (tall.empty()) return 0;
  {   // W = S^H S squares S: bring S into range first (Q is invariant under S -> c S, c > 0)
    int* d_e = static_cast<int*>(ctx->scratch.alloc(sizeof(int) * tall.size()));
    std::vector<Pow2Problem> have, need;
    for (size_t q = 0; q < tall.size(); ++q) {
      QRJob& J = jobs[tall[q]];
      if (J.exp) have.push_back(Pow2Problem{const_cast<cplx*>(J.S), J.m * J.kd, J.exp});
      else need.push_back(Pow2Problem{const_cast<cplx*>(J.S), J.m * J.kd, d_e + q});
    }
    launch_pow2_apply(have.data(), (int)have.size(), *ctx->stager, ctx->stream);
    launch_pow2_normalize(need.data(), (int)need.size(), *ctx->stager, ctx->stream);
  }
  gemm_batch(ctx, g1, st);
  launch_potri(p1.data(), (int)p1.size(), *ctx->stager, ctx->stream);
  gemm_batch(ctx, g2, st);
  gemm_batch(ctx, g3, st);
  launch_potri(p2.data(), (int)p2.size(), *ctx->stager, ctx->stream);
  gemm_batch(ctx, g4, st);
  if (spec) {   // speculative: a pivot failure (rank-deficient S) invalidates the apply
    launch_flag_nonzero(d_info, 2 * (int)jobs.size(), spec->flag, 4, ctx->stream);
    return 0;
  }
  ctx->ensure_small(sizeof(int) * 2 * jobs.size());
  int* hi = reinterpret_cast<int*>(ctx->hbuf);
  TTN_CUDA(cudaMemcpyAsync(hi, d_info, sizeof(int) * 2 * jobs.size(), cudaMemcpyDeviceToHost, ctx->stream));
  ctx->sync();
  // rank-deficient (or too ill-conditioned) S: Householder QR fallback, stream-ordered
  std::vector<GeqrProblem> fb;
  for (int j : tall)
    if (hi[2 * j] != 0 || hi[2 * j + 1] != 0) {
      QRJob& J = jobs[j];
      cplx* tau = static_cast<cplx*>(ctx->scratch.alloc(sizeof(cplx) * J.kd));
      fb.push_back(GeqrProblem{const_cast<cplx*>(J.S), J.Q, tau, (int)J.m, (int)J.kd});
      flops_inst[J.inst].add_nongemm(8.0 * 2.0 * (double)J.m * J.kd * J.kd);
      fb_inst[J.inst] += 1;
    }
  if (!fb.empty()) launch_geqr_q(fb.data(), (int)fb.size(), *ctx->stager, ctx->stream);
  return (int)fb.size();
}

}  // namespace

// Subtree partition of a multi-GPU apply (ttn_ctx_set_comm; SURVEY §8(e) mechanism 2).
// group[i] = -1: node of the replicated top (always the root); else the subtree group.
struct Partition {
  bool on = false;
  int world = 1, rank = 0;
  std::vector<int> group;
  std::vector<int> cuts;     // subtree roots (their parent is a top node)
  bool top(int i) const { return group[i] < 0; }
  bool mine(int i) const { return group[i] < 0 || group[i] % world == rank; }
  int owner(int i) const { return group[i] % world; }
};

// subtree groups of a `parts`-way partition (host-only; also exported as ttn_partition_plan)
std::vector<int> partition_groups(const ttn_s* ref, int parts, std::vector<int>* cuts_out) {
  const int n = ref->n;
  std::vector<int> group(n, -1);
  if (parts <= 1) return group;
  const auto& ch = ref->children;
  // subtree sizes (nodes in post-order: deepest first)
  std::vector<int> order(n), size(n, 1);
  for (int i = 0; i < n; ++i) order[i] = i;
  std::sort(order.begin(), order.end(), [&](int x, int y) { return ref->depth[x] > ref->depth[y]; });
  for (int i : order)
    if (ref->parent[i] >= 0) size[ref->parent[i]] += size[i];
  std::vector<int> units(ch[ref->root].begin(), ch[ref->root].end());
  while ((int)units.size() < parts) {   // expand the largest subtree that branches (>= 2 children)
    int best = -1;
    for (size_t u = 0; u < units.size(); ++u)
      if (ch[units[u]].size() >= 2 && (best < 0 || size[units[u]] > size[units[best]] ||
                                    (size[units[u]] == size[units[best]] && units[u] < units[best])))
        best = (int)u;
    if (best < 0) break;
    const int x = units[best];
    units.erase(units.begin() + best);
    units.insert(units.end(), ch[x].begin(), ch[x].end());
  }
  std::sort(units.begin(), units.end(), [&](int x, int y) { return size[x] != size[y] ? size[x] > size[y] : x < y; });
  std::vector<long long> load(parts, 0);
  for (int u : units) {
    const int g = (int)(std::min_element(load.begin(), load.end()) - load.begin());
    load[g] += size[u];
    std::vector<int> st{u};
    while (!st.empty()) {
      const int x = st.back();
      st.pop_back();
      group[x] = g;
      for (int c : ch[x]) st.push_back(c);
    }
  }
  if (cuts_out) {
    *cuts_out = units;
    std::sort(cuts_out->begin(), cuts_out->end());
  }
  return group;
}

Partition make_partition(const ttn_s* ref, const ttn_ctx_s* ctx) {
  Partition P;
  P.group.assign(ref->n, -1);
  if (!ctx->comm || ctx->parts <= 1) return P;
  P.on = true;
  P.world = ctx->comm->world;
  P.rank = ctx->comm->rank;
  P.group = partition_groups(ref, ctx->parts, &P.cuts);
  return P;
}

namespace {

enum class Mode { Sync, Spec, Capture };

// Control block of one pass of the schedule.  Sync: ranks read by the host per level (the
// general path).  Spec / Capture: speculative ranks, no host synchronisation; the per-instance
// results (norms, discarded weights, exact-factor counts, the flag) are copied into
// `host_res` at the end (layout of SpecRes) and the caller synchronises and checks them.
struct CoreCtl {
  Mode mode = Mode::Sync;
  char* host_res = nullptr;                     // pinned, SpecRes::bytes(nb)
  std::function<cplx*(int64_t)> out_alloc;      // Capture: outputs in the graph's buffer
  bool host_synced = false;                     // a stage synchronised anyway (no capture)
  int64_t out_elems = 0;                        // entries of all outputs
  // host-side per-instance results (known from shapes alone in the speculative modes)
  std::vector<FlopAcc> flops;
  std::vector<int64_t> maxb;
  int64_t peak = 0;
};

// layout of the speculative result block (device: env arena; host: pinned)
struct SpecRes {
  static size_t bytes(int nb) { return sizeof(double) * 2 * nb + sizeof(int) * (nb + 1); }
  static double* sq(char* p, int nb) { (void)nb; return reinterpret_cast<double*>(p); }
  static double* w(char* p, int nb) { return reinterpret_cast<double*>(p) + nb; }
  static int* x(char* p, int nb) { return reinterpret_cast<int*>(reinterpret_cast<double*>(p) + 2 * nb); }
  static int* flag(char* p, int nb) { return x(p, nb) + nb; }
};

void apply_core(ttn_ctx_s* ctx, int nb, const ttn_s* const* ops, const ttn_s* const* sts, int64_t max_bond,
                double tol, ttn_s** outs, ttn_cbc_report* reps, CoreCtl& cc) {
  auto t0 = std::chrono::steady_clock::now();
  const bool specm = cc.mode != Mode::Sync;
  if (nb <= 0) throw Error(TTN_ERR_ARG, "batch size must be >= 1");
  if (max_bond < 1) throw Error(TTN_ERR_ARG, "max_bond must be >= 1");
  if (!(tol >= 0.0 && tol < 1.0)) throw Error(TTN_ERR_ARG, "tol must be in [0, 1)");
  const ttn_s* ref = sts[0];
  for (int b = 0; b < nb; ++b) {
    if (!ops[b] || !sts[b]) throw Error(TTN_ERR_ARG, "NULL handle");
    if (ops[b]->kind != TTN_OPERATOR || sts[b]->kind != TTN_STATE)
      throw Error(TTN_ERR_ARG, "cbc_apply expects (operator, state) handles");
    if (ops[b]->n != ref->n || sts[b]->n != ref->n || ops[b]->parent != ref->parent || sts[b]->parent != ref->parent)
      throw Error(TTN_ERR_TOPOLOGY, "topology mismatch: parent arrays differ");
    if (ops[b]->phys != ref->phys || sts[b]->phys != ref->phys)
      throw Error(TTN_ERR_SHAPE, "leg mismatch: physical dimensions differ");
  }
  const int n = ref->n;
  const int root = ref->root;
  const auto& ch = ref->children;
  int maxd = 0;
  for (int i = 0; i < n; ++i) maxd = std::max(maxd, ref->depth[i]);
  // A9: up-factors that are read
  std::vector<char> used(n, 0);
  {
    std::vector<int> order(n);
    for (int i = 0; i < n; ++i) order[i] = i;
    std::sort(order.begin(), order.end(), [&](int x, int y) { return ref->depth[x] < ref->depth[y]; });
    for (int i : order) {
      int p = ref->parent[i];
      if (p < 0) continue;
      used[i] = (ch[p].size() >= 2) || used[p];
    }
  }
  const Partition part = make_partition(ref, ctx);
  Comm* comm = part.on ? ctx->comm : nullptr;
  ctx->env.reset();
  ctx->scratch.reset();
  ctx->host_syncs = 0;
  ctx->sync_wait_s = 0.0;
  ExecStats st;
  // speculative modes: device accumulators and the result block (zeroed in stream order)
  char* d_res = nullptr;
  SpecDev sdev{};
  if (specm) {
    d_res = static_cast<char*>(ctx->env.alloc(SpecRes::bytes(nb)));
    TTN_CUDA(cudaMemsetAsync(d_res, 0, SpecRes::bytes(nb), ctx->stream));
    sdev = SpecDev{SpecRes::w(d_res, nb), SpecRes::x(d_res, nb), SpecRes::flag(d_res, nb), &cc.host_synced};
  }
  const SpecDev* spec = specm ? &sdev : nullptr;
  // per-instance accumulators: replicated top work counted on every rank, subtree work only
  // on its owner (summed over ranks at the end)
  std::vector<double> w_inst(nb, 0.0), w_sub(nb, 0.0);
  std::vector<FlopAcc> flops_inst(nb), flops_sub(nb);
  std::vector<int> fb_inst(nb, 0), fb_sub(nb, 0), split_inst(nb, 0), exact_inst(nb, 0), exact_sub(nb, 0);
  std::vector<Fac> up((size_t)nb * n), down((size_t)nb * n), R((size_t)nb * n);
  // trivial factor L^{[(-,r)]} = 1 (extent-1 legs)
  cplx* one = static_cast<cplx*>(ctx->env.alloc(sizeof(cplx)));
  launch_fill(one, 1, make_double2(1.0, 0.0), ctx->stream);
  for (int b = 0; b < nb; ++b) down[(size_t)b * n + root] = Fac{one, 1, 1, 1};

  auto acc_w = [&](bool sub) -> std::vector<double>& { return sub ? w_sub : w_inst; };
  auto acc_f = [&](bool sub) -> std::vector<FlopAcc>& { return sub ? flops_sub : flops_inst; };
  auto acc_x = [&](bool sub) -> std::vector<int>& { return sub ? exact_sub : exact_inst; };

  // ---------------- row split of the replicated top's heavy compresses (partitioned apply):
  // a G-route compress of X (rows m >= cols n) whose widest factor leg has extent k is cut into
  // S >= world slices along that leg; each rank contracts its slices X_s (the factor operand
  // is a contiguous sub-block), forms sum_s X_s^H X_s, and the partial Grams are summed over
  // ranks (ncclAllReduce) -- G = X^H X exactly, at 1/world of the contraction and Gram work.
  // The eigensolve and the factor (Lambda^1/2 V^H needs only G) then run replicated.
  // TTN_PARTITION_SLICES (tests) forces more slices than ranks on one GPU.
  const char* slices_env = getenv("TTN_PARTITION_SLICES");
  const int nslices = part.on ? std::max(part.world, slices_env ? atoi(slices_env) : 0) : 1;
  const int64_t split_min = slices_env ? 0 : (int64_t(1) << 22);   // entries of X worth splitting
  auto split_rows = [&](std::vector<Task>& tasks, std::vector<CompressJob>& jobs) {
    if (nslices < 2) return;
    std::vector<Task> keep_t, sl_t;
    std::vector<CompressJob> keep_j, sp_j;
    std::vector<int> sl_job, sl_s;
    for (size_t j = 0; j < tasks.size(); ++j) {
      Task& t = tasks[j];
      CompressJob& J = jobs[j];
      const int64_t n = J.a * J.b;
      int64_t m = t.ops[1].dims[0];   // sigma'
      for (size_t o = 2; o < t.ops.size(); ++o) m *= t.ops[o].dims[0];
      size_t fo = 0;   // slice the factor with the widest compressed leg
      for (size_t o = 2; o < t.ops.size(); ++o)
        if (!fo || t.ops[o].dims[0] > t.ops[fo].dims[0]) fo = o;
      const int64_t k = fo ? t.ops[fo].dims[0] : 1;
      if (m < n || k < nslices || m * n < split_min) {   // K route, too thin, or small: replicated
        keep_t.push_back(t);
        keep_j.push_back(J);
        continue;
      }
      for (int sl = 0; sl < nslices; ++sl) {
        if (sl % part.world != part.rank) continue;
        const int64_t k0 = k * sl / nslices, k1 = k * (sl + 1) / nslices;
        Task ts = t;
        Operand& F = ts.ops[fo];
        F.ptr += k0 * F.dims[1] * F.dims[2];
        F.dims[0] = k1 - k0;
        ts.out = nullptr;
        sl_t.push_back(ts);
        sl_job.push_back((int)sp_j.size());
        sl_s.push_back(sl);
      }
      J.m = m;
      J.n = n;
      ++split_inst[J.inst];
      sp_j.push_back(J);
    }
    tasks.swap(keep_t);
    jobs.swap(keep_j);
    if (sp_j.empty()) return;
    // shared range exponent per job (max over slices and ranks), then the partial Grams
    const int ns = (int)sp_j.size();
    int* d_e = static_cast<int*>(ctx->env.alloc(sizeof(int) * ns));
    pow2_reset(d_e, ns, ctx->stream);
    for (size_t q = 0; q < sl_t.size(); ++q) sl_t[q].out_exp = d_e + sl_job[q];
    ExecStats cs;
    if (!sl_t.empty()) contract_batch(ctx, sl_t, cs);
    for (size_t q = 0; q < sl_t.size(); ++q) flops_sub[sp_j[sl_job[q]].inst].add_contract(sl_t[q].flops, sl_t[q].flops_min);
    st.flops += cs.flops;
    st.peak_entries = std::max(st.peak_entries, cs.peak_entries);
    comm->allreduce_max(d_e, ns, ctx->stream);
    std::vector<Pow2Problem> p2;
    for (size_t q = 0; q < sl_t.size(); ++q) {
      int64_t tot = 1;
      for (auto d : sl_t[q].out_dims) tot *= d;
      p2.push_back(Pow2Problem{sl_t[q].out, tot, d_e + sl_job[q]});
    }
    launch_pow2_apply(p2.data(), (int)p2.size(), *ctx->stager, ctx->stream);
    std::vector<cplx*> G(ns);
    for (int q = 0; q < ns; ++q) {
      const int64_t n = sp_j[q].n;
      G[q] = static_cast<cplx*>(ctx->env.alloc(sizeof(cplx) * n * n));
      TTN_CUDA(cudaMemsetAsync(G[q], 0, sizeof(cplx) * n * n, ctx->stream));
    }
    // rounds of one slice per job (beta = 1 accumulation keeps the rounds stream-ordered)
    for (int round = 0;; ++round) {
      std::vector<GemmProblem> g;
      std::vector<int> seen(ns, 0);
      for (size_t q = 0; q < sl_t.size(); ++q) {
        const int jq = sl_job[q];
        if (seen[jq]++ != round) continue;
        const int64_t n = sp_j[jq].n;
        int64_t tot = 1;
        for (auto d : sl_t[q].out_dims) tot *= d;
        GemmProblem gp = mk_gemm(sl_t[q].out, OP_C, n, sl_t[q].out, OP_N, n, G[jq], n, n, n, tot / n);
        gp.beta = make_double2(1.0, 0.0);
        flops_sub[sp_j[jq].inst] += gemm_flops(gp);
        g.push_back(gp);
      }
      if (g.empty()) break;
      gemm_batch(ctx, g, st);
    }
    for (int q = 0; q < ns; ++q) comm->allreduce_sum(reinterpret_cast<double*>(G[q]), 2 * (size_t)sp_j[q].n * sp_j[q].n, ctx->stream);
    for (int q = 0; q < ns; ++q) {
      sp_j[q].G_pre = G[q];
      sp_j[q].exp = d_e + q;
      sp_j[q].X = nullptr;
    }
    compress_batch(ctx, sp_j, max_bond, tol, st, w_inst, flops_inst, exact_inst, spec, comm);
  };

  // ---------------- 1. up-sweep (Eq. 10) over the nodes selected by `sel`, deepest level first
  auto up_sweep = [&](auto sel, bool sub) {
    HostScope hs_("up_sweep");
    for (int L = maxd; L >= 1; --L) {
      HostScope hb_("build_tasks");
      std::vector<Task> tasks;
      std::vector<CompressJob> jobs;
      for (int b = 0; b < nb; ++b)
        for (int i = 0; i < n; ++i) {
          if (ref->depth[i] != L || !used[i] || !sel(i)) continue;
          std::map<int, const Fac*> f;
          for (size_t l = 0; l < ch[i].size(); ++l) f[1 + (int)l] = &up[(size_t)b * n + ch[i][l]];
          tasks.push_back(node_task(sts[b], ops[b], i, f, 0, nullptr));
          jobs.push_back(CompressJob{nullptr, 0, 0, &up[(size_t)b * n + i], sts[b]->shape[i][1], ops[b]->shape[i][2], b});
        }
      if (tasks.empty()) continue;
      if (!sub && part.on) split_rows(tasks, jobs);   // heavy replicated G-route compresses
      if (tasks.empty()) { ctx->scratch.reset(); continue; }
      int* d_e = static_cast<int*>(ctx->scratch.alloc(sizeof(int) * tasks.size()));
      pow2_reset(d_e, (int)tasks.size(), ctx->stream);
      for (size_t j = 0; j < tasks.size(); ++j) {
        tasks[j].out_exp = d_e + j;
        jobs[j].exp = d_e + j;
      }
      ExecStats cs;
      contract_batch(ctx, tasks, cs);
      for (size_t j = 0; j < tasks.size(); ++j) {
        int64_t tot = 1;
        for (auto d : tasks[j].out_dims) tot *= d;
        jobs[j].X = tasks[j].out;
        jobs[j].n = jobs[j].a * jobs[j].b;
        jobs[j].m = tot / jobs[j].n;
      }
      st.peak_entries = std::max(st.peak_entries, cs.peak_entries);
      for (size_t j = 0; j < jobs.size(); ++j) acc_f(sub)[jobs[j].inst].add_contract(tasks[j].flops, tasks[j].flops_min);
      st.flops += cs.flops;
      compress_batch(ctx, jobs, max_bond, tol, st, acc_w(sub), acc_f(sub), acc_x(sub), spec,
                     sub ? nullptr : comm);   // the replicated top's compresses: sharded
      ctx->scratch.reset();
    }
  };
  // ---------------- 2. down-sweep (Eq. 11): nodes selected by `sel` give their children factors
  auto down_sweep = [&](auto sel, bool sub) {
    HostScope hs_("down_sweep");
    for (int L = 0; L < maxd; ++L) {
      std::vector<Task> tasks;
      std::vector<CompressJob> jobs;
      for (int b = 0; b < nb; ++b)
        for (int i = 0; i < n; ++i) {
          if (ref->depth[i] != L || !sel(i)) continue;
          for (size_t lk = 0; lk < ch[i].size(); ++lk) {
            int k = ch[i][lk];
            std::map<int, const Fac*> f;
            f[0] = &down[(size_t)b * n + i];
            for (size_t l = 0; l < ch[i].size(); ++l)
              if (l != lk) f[1 + (int)l] = &up[(size_t)b * n + ch[i][l]];
            tasks.push_back(node_task(sts[b], ops[b], i, f, 1 + (int)lk, nullptr));
            jobs.push_back(CompressJob{nullptr, 0, 0, &down[(size_t)b * n + k], sts[b]->shape[k][1], ops[b]->shape[k][2], b});
          }
        }
      if (tasks.empty()) continue;
      if (!sub && part.on) split_rows(tasks, jobs);   // heavy replicated G-route compresses
      if (tasks.empty()) { ctx->scratch.reset(); continue; }
      int* d_e = static_cast<int*>(ctx->scratch.alloc(sizeof(int) * tasks.size()));
      pow2_reset(d_e, (int)tasks.size(), ctx->stream);
      for (size_t j = 0; j < tasks.size(); ++j) {
        tasks[j].out_exp = d_e + j;
        jobs[j].exp = d_e + j;
      }
      ExecStats cs;
      contract_batch(ctx, tasks, cs);
      for (size_t j = 0; j < tasks.size(); ++j) {
        int64_t tot = 1;
        for (auto d : tasks[j].out_dims) tot *= d;
        jobs[j].X = tasks[j].out;
        jobs[j].n = jobs[j].a * jobs[j].b;
        jobs[j].m = tot / jobs[j].n;
      }
      st.peak_entries = std::max(st.peak_entries, cs.peak_entries);
      for (size_t j = 0; j < jobs.size(); ++j) acc_f(sub)[jobs[j].inst].add_contract(tasks[j].flops, tasks[j].flops_min);
      st.flops += cs.flops;
      compress_batch(ctx, jobs, max_bond, tol, st, acc_w(sub), acc_f(sub), acc_x(sub), spec,
                     sub ? nullptr : comm);   // the replicated top's compresses: sharded
      ctx->scratch.reset();
    }
  };
  // rank-owned integers (factor ranks) made global: owners fill, zeros elsewhere, sum
  auto share_ints = [&](std::vector<int>& v) {
    if (!comm || v.empty()) return;
    int* d = static_cast<int*>(ctx->scratch.alloc(sizeof(int) * v.size()));
    TTN_CUDA(cudaMemcpyAsync(d, v.data(), sizeof(int) * v.size(), cudaMemcpyHostToDevice, ctx->stream));
    comm->allreduce_sum(d, v.size(), ctx->stream);
    TTN_CUDA(cudaMemcpyAsync(v.data(), d, sizeof(int) * v.size(), cudaMemcpyDeviceToHost, ctx->stream));
    ctx->sync();
  };
  // broadcast factors `F[b*n + u]` of the cut nodes from their owners (ranks k shared first)
  auto share_factors = [&](std::vector<Fac>& F, bool only_used) {
    if (!part.on) return;
    std::vector<int> ks;
    for (int b = 0; b < nb; ++b)
      for (int u : part.cuts) {
        if (only_used && !used[u]) continue;
        const Fac& f = F[(size_t)b * n + u];
        ks.push_back(part.owner(u) == part.rank ? (int)f.k : 0);
      }
    share_ints(ks);
    size_t q = 0;
    comm->group_start();
    for (int b = 0; b < nb; ++b)
      for (int u : part.cuts) {
        if (only_used && !used[u]) continue;
        Fac& f = F[(size_t)b * n + u];
        const int k = ks[q++];
        if (part.owner(u) != part.rank) {
          f.k = k;
          f.a = sts[b]->shape[u][1];
          f.b = ops[b]->shape[u][2];
          f.p = static_cast<cplx*>(ctx->env.alloc(sizeof(cplx) * std::max<int64_t>(f.k * f.a * f.b, 1)));
        }
        comm->bcast(f.p, sizeof(cplx) * f.k * f.a * f.b, part.owner(u), ctx->stream);
      }
    comm->group_end();
  };

  auto in_sub = [&](int i) { return !part.top(i) && part.mine(i); };
  auto in_top = [&](int i) { return part.top(i); };
  // up-sweep: subtrees (rank-local), boundary environments, replicated top
  if (part.on) {
    up_sweep(in_sub, true);
    share_factors(up, true);
  }
  up_sweep(in_top, false);
  // down-sweep: replicated top (gives the subtree roots their down factors), then subtrees
  down_sweep(in_top, false);
  if (part.on) down_sweep(in_sub, true);

  // ---------------- output shapes: r_i = min(d_i prod_c r_c, kd_i); root 1
  if (part.on) {   // subtree nodes' down ranks (kd) from their owners
    std::vector<int> kd;
    for (int b = 0; b < nb; ++b)
      for (int i = 0; i < n; ++i)
        if (!part.top(i) && i != root) kd.push_back(part.mine(i) ? (int)down[(size_t)b * n + i].k : 0);
    share_ints(kd);
    size_t q = 0;
    for (int b = 0; b < nb; ++b)
      for (int i = 0; i < n; ++i)
        if (!part.top(i) && i != root) down[(size_t)b * n + i].k = kd[q++];
  }
  std::vector<std::vector<int64_t>> rb(nb, std::vector<int64_t>(n, 1));
  {
    std::vector<int> order(n);
    for (int i = 0; i < n; ++i) order[i] = i;
    std::sort(order.begin(), order.end(), [&](int x, int y) { return ref->depth[x] > ref->depth[y]; });
    for (int b = 0; b < nb; ++b)
      for (int i : order) {
        if (i == root) { rb[b][i] = 1; continue; }
        int64_t ms = ref->phys[i];
        for (int c : ch[i]) ms *= rb[b][c];
        rb[b][i] = std::min<int64_t>(ms, down[(size_t)b * n + i].k);
      }
  }
  for (int b = 0; b < nb; ++b) {
    outs[b] = new_ttn_like(ctx, ref, TTN_STATE, rb[b], cc.out_alloc);
    cc.out_elems += outs[b]->total;
  }

  // ---------------- row split of the replicated top's heavy final-sweep nodes (partitioned
  // apply, SURVEY §8(e) "Junction CholeskyQR2 row-split"): Z_i is cut along its widest child
  // factor leg into slices (rank r contracts slices s = r mod world); then, with the partial
  // sums all-reduced over the ranks,
  //   S_s = Z_s L^T,  W = sum_s S_s^H S_s = L1 L1^H,  Q1_s = S_s L1^-H,
  //   W2 = sum_s Q1_s^H Q1_s = L2 L2^H,  Q_s = Q1_s L2^-H          (CholeskyQR2, Eq. 13)
  //   R_i = sum_s Q_s^H Z_s                                          (Eq. 14 with Q*)
  // and every rank scatters its slices' rows of Q into the (zeroed) new tensor T'_i, which an
  // all-reduce completes on every rank.  Exact up to the order of the row sums.
  auto final_split = [&](int b, int i, const Task& t) {
    HostScope hs_("final_split");
    const Fac& fd = down[(size_t)b * n + i];
    const int64_t nz = fd.a * fd.b, kd = fd.k, r = rb[b][i], d = ref->phys[i];
    size_t fo = 2;   // the widest child factor
    for (size_t o = 3; o < t.ops.size(); ++o)
      if (t.ops[o].dims[0] > t.ops[fo].dims[0]) fo = o;
    const int cpos = (int)fo - 2;   // child position of the sliced leg
    const int64_t kfull = t.ops[fo].dims[0];
    std::vector<int64_t> rc;        // child factor ranks (leg order)
    for (size_t o = 2; o < t.ops.size(); ++o) rc.push_back(t.ops[o].dims[0]);
    int64_t ms = d;
    for (auto x : rc) ms *= x;
    std::vector<Task> sl;
    std::vector<int64_t> k0s, k1s;
    for (int s = 0; s < nslices; ++s) {
      if (s % part.world != part.rank) continue;
      const int64_t k0 = kfull * s / nslices, k1 = kfull * (s + 1) / nslices;
      if (k1 <= k0) continue;
      Task ts = t;
      ts.ops[fo].ptr += k0 * ts.ops[fo].dims[1] * ts.ops[fo].dims[2];
      ts.ops[fo].dims[0] = k1 - k0;
      ts.out = nullptr;
      sl.push_back(ts);
      k0s.push_back(k0);
      k1s.push_back(k1);
    }
    const int nsl = (int)sl.size();
    ExecStats cs;
    if (nsl) contract_batch(ctx, sl, cs);
    st.peak_entries = std::max(st.peak_entries, cs.peak_entries);
    for (auto& x : sl) flops_sub[b].add_contract(x.flops, x.flops_min);
    int* d_e = static_cast<int*>(ctx->scratch.alloc(sizeof(int) * 2 + sizeof(int) * 2));
    int* d_info = d_e + 2;
    pow2_reset(d_e, 1, ctx->stream);
    std::vector<cplx*> S(nsl), Q1(nsl), Q(nsl);
    std::vector<int64_t> mss(nsl);
    std::vector<GemmProblem> g;
    for (int q = 0; q < nsl; ++q) {
      mss[q] = ms / kfull * (k1s[q] - k0s[q]);
      S[q] = static_cast<cplx*>(ctx->scratch.alloc(sizeof(cplx) * mss[q] * kd));
      g.push_back(mk_gemm(sl[q].out, OP_N, nz, fd.p, OP_T, nz, S[q], kd, mss[q], kd, nz));   // S_s = Z_s L^T
      g.back().exp_out = d_e;
      flops_sub[b] += gemm_flops(g.back());
    }
    gemm_batch(ctx, g, st);
    comm->allreduce_max(d_e, 1, ctx->stream);   // one range exponent for all of S
    {
      std::vector<Pow2Problem> p2;
      for (int q = 0; q < nsl; ++q) p2.push_back(Pow2Problem{S[q], mss[q] * kd, d_e});
      launch_pow2_apply(p2.data(), (int)p2.size(), *ctx->stager, ctx->stream);
    }
    cplx* W = static_cast<cplx*>(ctx->scratch.alloc(sizeof(cplx) * kd * kd));
    cplx* Li = static_cast<cplx*>(ctx->scratch.alloc(sizeof(cplx) * kd * kd));
    auto gram_sum = [&](const std::vector<cplx*>& X) {   // W = sum over all ranks' slices of X^H X
      TTN_CUDA(cudaMemsetAsync(W, 0, sizeof(cplx) * kd * kd, ctx->stream));
      for (int q = 0; q < nsl; ++q) {
        std::vector<GemmProblem> gg{mk_gemm(X[q], OP_C, kd, X[q], OP_N, kd, W, kd, kd, kd, mss[q])};
        gg[0].beta = make_double2(1.0, 0.0);
        flops_sub[b] += gemm_flops(gg[0]);
        gemm_batch(ctx, gg, st);
      }
      comm->allreduce_sum(reinterpret_cast<double*>(W), 2 * (size_t)kd * kd, ctx->stream);
    };
    auto solve = [&](const std::vector<cplx*>& X, std::vector<cplx*>& Y, int* info, double tol_rel) {
      gram_sum(X);
      PotriProblem pp{W, kd, (int)kd, 0, info, tol_rel, 0.0, Li};
      launch_potri(&pp, 1, *ctx->stager, ctx->stream);
      flops_inst[b].add_nongemm(8.0 * 2.0 * (kd * kd * kd / 3.0));
      std::vector<GemmProblem> gg;
      for (int q = 0; q < nsl; ++q) {
        Y[q] = static_cast<cplx*>(ctx->scratch.alloc(sizeof(cplx) * mss[q] * kd));
        gg.push_back(mk_gemm(X[q], OP_N, kd, Li, OP_C, kd, Y[q], kd, mss[q], kd, kd));   // X L^-H
        flops_sub[b] += gemm_flops(gg.back());
      }
      gemm_batch(ctx, gg, st);
    };
    solve(S, Q1, d_info, kCholTol);
    solve(Q1, Q, d_info + 1, kCholTol * 1e-2);
    ctx->ensure_small(sizeof(int) * 2);
    int* hi = reinterpret_cast<int*>(ctx->hbuf);
    TTN_CUDA(cudaMemcpyAsync(hi, d_info, sizeof(int) * 2, cudaMemcpyDeviceToHost, ctx->stream));
    ctx->sync();
    if (hi[0] != 0 || hi[1] != 0)
      throw Error(TTN_ERR_NUMERIC, "rank-deficient S in a row-split final sweep (CholeskyQR2 pivot)");
    if (r != kd) throw Error(TTN_ERR_UNSUPPORTED, "row-split final sweep expects r = kd");
    // T'_i: scatter my slices' rows of Q into the zeroed tensor [d, r, rc...], then all-reduce
    cplx* T = outs[b]->node(i);
    int64_t te = d * r;
    for (auto x : rc) te *= x;
    TTN_CUDA(cudaMemsetAsync(T, 0, sizeof(cplx) * te, ctx->stream));
    std::vector<PermProblem> pq;
    std::vector<long long> dst(2 + rc.size());   // strides of T' [d, r, rc...]
    {
      long long s = 1;
      for (int l = (int)rc.size() - 1; l >= 0; --l) {
        dst[2 + l] = s;
        s *= rc[l];
      }
      dst[1] = s;
      dst[0] = s * r;
    }
    for (int q = 0; q < nsl; ++q) {
      std::vector<int64_t> rcs = rc;
      rcs[cpos] = k1s[q] - k0s[q];
      PermProblem pp{};
      pp.src = Q[q];
      pp.dst = T + k0s[q] * dst[2 + cpos];
      pp.rank = 2 + (int)rc.size();
      if (pp.rank > 8) throw Error(TTN_ERR_UNSUPPORTED, "row split: too many legs");
      pp.dims[0] = d;
      pp.dims[1] = r;
      long long srow = r;   // Q_s rows (d, rcs...), columns r
      for (int l = (int)rcs.size() - 1; l >= 0; --l) {
        pp.dims[2 + l] = rcs[l];
        pp.sstride[2 + l] = srow;
        srow *= rcs[l];
      }
      pp.sstride[0] = srow;
      pp.sstride[1] = 1;
      pp.dst_strided = 1;
      pp.total = 1;
      for (int x = 0; x < pp.rank; ++x) {
        pp.dstride[x] = dst[x];
        pp.total *= pp.dims[x];
      }
      pq.push_back(pp);
    }
    if (!pq.empty()) launch_permute(pq.data(), (int)pq.size(), *ctx->stager, ctx->stream);
    comm->allreduce_sum(reinterpret_cast<double*>(T), 2 * (size_t)te, ctx->stream);
    // R_i = sum_s Q_s^H Z_s
    Fac& Ri = R[(size_t)b * n + i];
    Ri.p = static_cast<cplx*>(ctx->env.alloc(sizeof(cplx) * r * nz));
    Ri.k = r;
    Ri.a = fd.a;
    Ri.b = fd.b;
    TTN_CUDA(cudaMemsetAsync(Ri.p, 0, sizeof(cplx) * r * nz, ctx->stream));
    for (int q = 0; q < nsl; ++q) {
      std::vector<GemmProblem> gg{mk_gemm(Q[q], OP_C, r, sl[q].out, OP_N, nz, Ri.p, nz, r, nz, mss[q])};
      gg[0].beta = make_double2(1.0, 0.0);
      flops_sub[b] += gemm_flops(gg[0]);
      gemm_batch(ctx, gg, st);
    }
    comm->allreduce_sum(reinterpret_cast<double*>(Ri.p), 2 * (size_t)r * nz, ctx->stream);
    ++split_inst[b];
  };

  // ---------------- 3. final sweep (Eqs. 12-14) and 4. assembly, over the nodes selected
  auto final_sweep = [&](auto sel, bool sub) {
    HostScope hs_("final_sweep");
    for (int L = maxd; L >= 0; --L) {
      std::vector<Task> tasks;
      std::vector<std::pair<int, int>> who;
      for (int b = 0; b < nb; ++b)
        for (int i = 0; i < n; ++i) {
          if (ref->depth[i] != L || !sel(i)) continue;
          std::map<int, const Fac*> f;
          for (size_t l = 0; l < ch[i].size(); ++l) f[1 + (int)l] = &R[(size_t)b * n + ch[i][l]];
          cplx* out = (i == root) ? outs[b]->node(i) : nullptr;   // assembly: T'_root = Z_root
          Task t = node_task(sts[b], ops[b], i, f, 0, out);
          if (!sub && part.on && nslices >= 2 && i != root && !ch[i].empty()) {
            int64_t ms = ref->phys[i], kw = 0;
            for (size_t o = 2; o < t.ops.size(); ++o) {
              ms *= t.ops[o].dims[0];
              kw = std::max<int64_t>(kw, t.ops[o].dims[0]);
            }
            const Fac& fd = down[(size_t)b * n + i];
            if (ms > fd.k && kw >= nslices && ms * fd.a * fd.b >= split_min && rb[b][i] == fd.k) {
              final_split(b, i, t);   // heavy replicated node: rows split over the ranks
              continue;
            }
          }
          tasks.push_back(t);
          who.push_back({b, i});
        }
      if (tasks.empty()) { ctx->scratch.reset(); continue; }
      ExecStats cs;
      contract_batch(ctx, tasks, cs);
      st.peak_entries = std::max(st.peak_entries, cs.peak_entries);
      for (size_t j = 0; j < who.size(); ++j) acc_f(sub)[who[j].first].add_contract(tasks[j].flops, tasks[j].flops_min);
      st.flops += cs.flops;
      std::vector<GemmProblem> sg, rg;
      std::vector<QRJob> qj;
      std::vector<PermProblem> pq;
      int* s_exp = static_cast<int*>(ctx->scratch.alloc(sizeof(int) * tasks.size()));   // max exponents of S
      pow2_reset(s_exp, (int)tasks.size(), ctx->stream);
      for (size_t j = 0; j < tasks.size(); ++j) {
        const int b = who[j].first, i = who[j].second;
        if (i == root) continue;
        const Fac& fd = down[(size_t)b * n + i];
        const int64_t nz = fd.a * fd.b;
        int64_t tot = 1;
        for (auto d : tasks[j].out_dims) tot *= d;
        const int64_t ms = tot / nz, kd = fd.k, r = rb[b][i];
        cplx* S = static_cast<cplx*>(ctx->scratch.alloc(sizeof(cplx) * ms * kd));
        int* se = s_exp + j;
        sg.push_back(mk_gemm(tasks[j].out, OP_N, nz, fd.p, OP_T, nz, S, kd, ms, kd, nz));   // S = Z Fd^T (Eq. 12 via Z)
        sg.back().exp_out = se;
        acc_f(sub)[b] += 8.0 * (double)ms * kd * nz;
        cplx* Q = static_cast<cplx*>(ctx->scratch.alloc(sizeof(cplx) * ms * r));
        qj.push_back(QRJob{S, ms, kd, Q, b, se});
        // T'_i = Q in ABI order [d, r, r_c...]: Q viewed as [d, Rc, r] -> [d, r, Rc]
        const int64_t d = ref->phys[i], Rc = ms / d;
        PermProblem pp{};
        pp.src = Q; pp.dst = outs[b]->node(i); pp.rank = 3; pp.conj = 0;
        pp.dims[0] = d; pp.dims[1] = r; pp.dims[2] = Rc;
        pp.sstride[0] = Rc * r; pp.sstride[1] = 1; pp.sstride[2] = r;
        pp.total = d * r * Rc;
        pq.push_back(pp);
        // R_i = Q^H Z  (Eq. 14 with Q*, reading A6)
        Fac& Ri = R[(size_t)b * n + i];
        Ri.p = static_cast<cplx*>(ctx->env.alloc(sizeof(cplx) * r * nz));
        Ri.k = r; Ri.a = fd.a; Ri.b = fd.b;
        rg.push_back(mk_gemm(Q, OP_C, r, tasks[j].out, OP_N, nz, Ri.p, nz, r, nz, ms));
        acc_f(sub)[b] += 8.0 * (double)r * nz * ms;
      }
      gemm_batch(ctx, sg, st);
      qr_batch(ctx, qj, st, acc_f(sub), sub ? fb_sub : fb_inst, spec);
      if (!pq.empty()) launch_permute(pq.data(), (int)pq.size(), *ctx->stager, ctx->stream);
      gemm_batch(ctx, rg, st);
      ctx->scratch.reset();
    }
  };
  if (part.on) {
    final_sweep(in_sub, true);
    share_factors(R, false);   // subtree roots' R^{[u]} (Eq. 14) for the top's final sweep
    comm->group_start();       // every subtree's new tensors to every rank
    for (int b = 0; b < nb; ++b)
      for (int i = 0; i < n; ++i)
        if (!part.top(i)) {
          int64_t e = 1;
          for (auto d : outs[b]->shape[i]) e *= d;
          comm->bcast(outs[b]->node(i), sizeof(cplx) * e, part.owner(i), ctx->stream);
        }
    comm->group_end();
  }
  final_sweep(in_top, false);

  // ---------------- report: ||phi|| = ||T'_root||_F; subtree totals summed over ranks
  std::vector<SumsqProblem> sq(nb);
  double* d_sq = static_cast<double*>(ctx->scratch.alloc(sizeof(double) * nb * 8));
  for (int b = 0; b < nb; ++b) {
    sq[b].x = outs[b]->node(root);
    sq[b].len = 1;
    for (auto d : outs[b]->shape[root]) sq[b].len *= d;
    sq[b].out = d_sq + b;
  }
  launch_sumsq(sq.data(), nb, *ctx->stager, ctx->stream);
  if (specm) {   // results to the caller's pinned block; the caller synchronises and checks
    TTN_CUDA(cudaMemcpyAsync(d_res, d_sq, sizeof(double) * nb, cudaMemcpyDeviceToDevice, ctx->stream));
    TTN_CUDA(cudaMemcpyAsync(cc.host_res, d_res, SpecRes::bytes(nb), cudaMemcpyDeviceToHost, ctx->stream));
    cc.flops = flops_inst;
    cc.maxb.assign(nb, 1);
    for (int b = 0; b < nb; ++b)
      for (int i = 0; i < n; ++i) cc.maxb[b] = std::max<int64_t>(cc.maxb[b], rb[b][i]);
    cc.peak = st.peak_entries;
    return;
  }
  if (part.on) {
    constexpr int NF = 7;
    std::vector<double> h(NF * (size_t)nb);
    for (int b = 0; b < nb; ++b) {
      h[b] = w_sub[b];
      h[nb + b] = flops_sub[b].all;
      h[2 * nb + b] = fb_sub[b];
      h[3 * nb + b] = exact_sub[b];
      h[4 * nb + b] = flops_sub[b].nongemm;
      h[5 * nb + b] = flops_sub[b].cx_exec;
      h[6 * nb + b] = flops_sub[b].cx_min;
    }
    TTN_CUDA(cudaMemcpyAsync(d_sq + nb, h.data(), sizeof(double) * NF * nb, cudaMemcpyHostToDevice, ctx->stream));
    comm->allreduce_sum(d_sq + nb, NF * (size_t)nb, ctx->stream);
    TTN_CUDA(cudaMemcpyAsync(h.data(), d_sq + nb, sizeof(double) * NF * nb, cudaMemcpyDeviceToHost, ctx->stream));
    ctx->sync();
    for (int b = 0; b < nb; ++b) {
      w_inst[b] += h[b];
      flops_inst[b].all += h[nb + b];
      fb_inst[b] += (int)std::lround(h[2 * nb + b]);
      exact_inst[b] += (int)std::lround(h[3 * nb + b]);
      flops_inst[b].nongemm += h[4 * nb + b];
      flops_inst[b].cx_exec += h[5 * nb + b];
      flops_inst[b].cx_min += h[6 * nb + b];
    }
  }
  ctx->ensure_small(sizeof(double) * nb);
  double* hs = reinterpret_cast<double*>(ctx->hbuf);
  TTN_CUDA(cudaMemcpyAsync(hs, d_sq, sizeof(double) * nb, cudaMemcpyDeviceToHost, ctx->stream));
  ctx->sync();
  TTN_CUDA(cudaGetLastError());
  ctx->scratch.reset();
  ctx->env.reset();
  for (int b = 0; b < nb; ++b)
    if (!std::isfinite(hs[b])) throw Error(TTN_ERR_NUMERIC, "non-finite result (non-finite input?)");
  double secs = std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count();
  static const bool hprof = getenv("TTN_HOST_PROF") != nullptr;
  if (hprof) {
    fprintf(stderr, "[host] apply %.3f ms: blocked in %d syncs %.3f ms, host work %.3f ms\n", secs * 1e3,
            ctx->host_syncs, ctx->sync_wait_s * 1e3, (secs - ctx->sync_wait_s) * 1e3);
    host_prof_add("sync_wait", ctx->sync_wait_s);
    host_prof_dump();
  }
  if (reps) {
    for (int b = 0; b < nb; ++b) {
      ttn_cbc_report& r = reps[b];
      r.norm = std::sqrt(hs[b]);
      r.discarded_weight_sum = w_inst[b];
      r.max_bond = 1;
      for (int i = 0; i < n; ++i) r.max_bond = std::max<int64_t>(r.max_bond, rb[b][i]);
      r.peak_entries = st.peak_entries;
      r.seconds = secs;
      r.flops_algorithmic = flops_inst[b].all;
      r.flops_gemm_exec = flops_inst[b].gemm_exec();
      r.flops_gemm_min = flops_inst[b].gemm_min();
      r.rank_fallbacks = fb_inst[b];
      r.host_syncs = ctx->host_syncs;
      r.split_compresses = split_inst[b];
      r.exact_factors = exact_inst[b];
    }
  }
}

// ---------------------------------------------------------------- speculative schedule + graphs
// "captures CUDA graphs when ranks are static".  With tol = 0 the ranks of a
// generic apply are min(max_bond, m, n), known from the shapes alone; the schedule is planned
// with those ranks and checked on the device (SpecDev), so an apply needs ONE host
// synchronisation (its results) instead of one per level.  A speculative apply that succeeded
// is captured as a CUDA graph (keyed by shapes) against graph-owned copies of its inputs;
// later applies of the same shapes copy their inputs into those buffers (device to device,
// stream ordered) and replay it: no host planning, one graph launch -- also for inputs created
// afresh for every apply (the end-to-end path: ttn_create from host buffers).  A failed check (rank-deficient
// or tolerance-truncated data) discards the result and re-runs the synchronised schedule;
// those shapes are then never speculated again on this ctx.
struct GraphEntry {
  cudaGraph_t g = nullptr;
  cudaGraphExec_t ex = nullptr;
  char* desc = nullptr;           // device descriptors of every launch (uploaded once)
  cplx* outbuf = nullptr;         // the outputs, copied to fresh handles after each replay
  cplx* inbuf = nullptr;          // graph-owned inputs (the caller's are copied in per replay)
  std::vector<ttn_s*> in_ops, in_sts;   // clones of the capture's inputs; data points into inbuf
  char* host = nullptr;           // pinned result block (SpecRes)
  std::vector<ttn_s*> tmpl;       // output shapes; data points into outbuf (not owned)
  std::vector<FlopAcc> flops;
  std::vector<int64_t> maxb;
  int64_t peak = 0;
  long long launches = 0;         // kernels per replay
  ProfSink sink;
  uint64_t last_use = 0;
};

}  // namespace

struct GraphCache {
  std::map<std::vector<int64_t>, std::unique_ptr<GraphEntry>> map;
  std::set<std::vector<int64_t>> failed;    // trees whose speculation failed: always synchronised
  std::set<std::vector<int64_t>> nograph;   // keys whose capture failed
  std::set<std::vector<int64_t>> seen;      // keys with one successful speculative apply
  uint64_t tick = 0;
};

namespace {

void destroy_entry(ttn_ctx_s* ctx, GraphEntry* e) {
  if (e->ex) cudaGraphExecDestroy(e->ex);
  if (e->g) cudaGraphDestroy(e->g);
  if (e->desc) cudaFree(e->desc);
  if (e->outbuf) ctx->put(e->outbuf);
  if (e->inbuf) ctx->put(e->inbuf);
  for (auto* t : e->in_ops) delete t;   // data belongs to inbuf
  for (auto* t : e->in_sts) delete t;
  e->in_ops.clear();
  e->in_sts.clear();
  if (e->host) cudaFreeHost(e->host);
  for (auto* t : e->tmpl) delete t;   // data belongs to outbuf
  e->tmpl.clear();
}

GraphCache& graphs_of(ttn_ctx_s* ctx) {
  if (!ctx->gr) ctx->gr = new GraphCache();
  return *ctx->gr;
}

std::vector<int64_t> shape_key(int nb, const ttn_s* const* ops, const ttn_s* const* sts, int64_t max_bond) {
  const ttn_s* ref = sts[0];
  std::vector<int64_t> k{nb, max_bond, ref->n};
  for (int i = 0; i < ref->n; ++i) {
    k.push_back(ref->parent[i]);
    k.push_back(ref->phys[i]);
  }
  for (int b = 0; b < nb; ++b)
    for (int i = 0; i < ref->n; ++i) {
      k.push_back(sts[b]->bond[i]);
      k.push_back(ops[b]->bond[i]);
    }
  return k;
}

void fill_reports(ttn_cbc_report* reps, int nb, char* host, const std::vector<FlopAcc>& flops,
                  const std::vector<int64_t>& maxb, int64_t peak, double secs, int syncs) {
  if (!reps) return;
  for (int b = 0; b < nb; ++b) {
    ttn_cbc_report& r = reps[b];
    r.norm = std::sqrt(SpecRes::sq(host, nb)[b]);
    r.discarded_weight_sum = SpecRes::w(host, nb)[b];
    r.max_bond = maxb[b];
    r.peak_entries = peak;
    r.seconds = secs;
    r.flops_algorithmic = flops[b].all;
    r.flops_gemm_exec = flops[b].gemm_exec();
    r.flops_gemm_min = flops[b].gemm_min();
    r.rank_fallbacks = 0;
    r.host_syncs = syncs;
    r.split_compresses = 0;
    r.exact_factors = SpecRes::x(host, nb)[b];
  }
}

bool spec_ok(char* host, int nb) {
  if (*SpecRes::flag(host, nb) != 0) return false;
  for (int b = 0; b < nb; ++b)
    if (!std::isfinite(SpecRes::sq(host, nb)[b])) return false;
  return true;
}

// Capture the speculative schedule as a graph (after a successful uncaptured run that sized
// the descriptor and output buffers).  Returns null if the capture is not possible.
std::unique_ptr<GraphEntry> capture(ttn_ctx_s* ctx, int nb, const ttn_s* const* ops, const ttn_s* const* sts,
                                    int64_t max_bond, size_t desc_bytes, int64_t out_elems) {
  std::unique_ptr<GraphEntry> e(new GraphEntry());
  const size_t cap = desc_bytes + (1u << 16);
  if (cudaMalloc(&e->desc, cap) != cudaSuccess) {
    cudaGetLastError();
    e->desc = nullptr;
    return nullptr;
  }
  if (cudaMallocHost(&e->host, SpecRes::bytes(nb)) != cudaSuccess) {
    cudaGetLastError();
    e->host = nullptr;
    destroy_entry(ctx, e.get());
    return nullptr;
  }
  int64_t in_elems = 0;
  for (int b = 0; b < nb; ++b) in_elems += ops[b]->total + sts[b]->total;
  try {
    e->outbuf = static_cast<cplx*>(ctx->get(sizeof(cplx) * std::max<int64_t>(out_elems, 1)));
    e->inbuf = static_cast<cplx*>(ctx->get(sizeof(cplx) * std::max<int64_t>(in_elems, 1)));
  } catch (...) {
    destroy_entry(ctx, e.get());
    return nullptr;
  }
  {   // the graph reads its own copies of the inputs
    int64_t off = 0;
    auto clone = [&](const ttn_s* t) {
      ttn_s* c = new ttn_s(*t);
      c->data = e->inbuf + off;
      off += t->total;
      TTN_CUDA(cudaMemcpyAsync(c->data, t->data, sizeof(cplx) * t->total, cudaMemcpyDeviceToDevice, ctx->stream));
      return c;
    };
    for (int b = 0; b < nb; ++b) {
      e->in_ops.push_back(clone(ops[b]));
      e->in_sts.push_back(clone(sts[b]));
    }
  }
  TTN_CUDA(cudaStreamSynchronize(ctx->stream));   // outbuf / inbuf ready before capture
  CaptureStager cs(e->desc, cap);
  int64_t used = 0;
  CoreCtl cc;
  cc.mode = Mode::Capture;
  cc.host_res = e->host;
  cc.out_alloc = [&](int64_t elems) -> cplx* {
    if (used + elems > out_elems) throw Error(TTN_ERR_UNSUPPORTED, "graph output buffer too small");
    cplx* p = e->outbuf + used;
    used += elems;
    return p;
  };
  std::vector<ttn_s*> outs(nb, nullptr);
  const long long lc0 = launch_count();
  ctx->stager = &cs;
  ctx->scratch.frozen = ctx->env.frozen = true;
  ctx->capturing = true;
  const bool prof = prof_on();
  if (prof) prof_set_sink(&e->sink);
  bool ok = cudaStreamBeginCapture(ctx->stream, cudaStreamCaptureModeThreadLocal) == cudaSuccess;
  if (ok) {
    try {
      std::vector<const ttn_s*> co(e->in_ops.begin(), e->in_ops.end()), cs_(e->in_sts.begin(), e->in_sts.end());
      apply_core(ctx, nb, co.data(), cs_.data(), max_bond, 0.0, outs.data(), nullptr, cc);
    } catch (...) {
      ok = false;
    }
    cudaGraph_t g = nullptr;
    const bool ended = cudaStreamEndCapture(ctx->stream, &g) == cudaSuccess;
    ok = ok && ended && g && !cc.host_synced;
    if (g && !ok) cudaGraphDestroy(g);
    if (ok) e->g = g;
  }
  cudaGetLastError();
  if (prof) prof_set_sink(nullptr);
  ctx->capturing = false;
  ctx->scratch.frozen = ctx->env.frozen = false;
  ctx->stager = ctx->ring;
  e->launches = launch_count() - lc0;
  add_launches(-e->launches);   // captured, not launched
  e->tmpl = outs;
  if (!ok) {
    destroy_entry(ctx, e.get());
    return nullptr;
  }
  TTN_CUDA(cudaMemcpy(e->desc, cs.shadow.data(), cs.shadow.size(), cudaMemcpyHostToDevice));
  if (cudaGraphInstantiate(&e->ex, e->g, 0) != cudaSuccess) {
    cudaGetLastError();
    e->ex = nullptr;
    destroy_entry(ctx, e.get());
    return nullptr;
  }
  e->flops = cc.flops;
  e->maxb = cc.maxb;
  e->peak = cc.peak;
  return e;
}

// one replay; false when the device check failed (outputs discarded)
bool replay(ttn_ctx_s* ctx, GraphEntry* e, int nb, const ttn_s* const* ops, const ttn_s* const* sts, ttn_s** outs,
            ttn_cbc_report* reps) {
  auto t0 = std::chrono::steady_clock::now();
  ctx->host_syncs = 0;
  for (int b = 0; b < nb; ++b) {   // this apply's inputs into the graph's buffers
    TTN_CUDA(cudaMemcpyAsync(e->in_ops[b]->data, ops[b]->data, sizeof(cplx) * ops[b]->total, cudaMemcpyDeviceToDevice,
                             ctx->stream));
    TTN_CUDA(cudaMemcpyAsync(e->in_sts[b]->data, sts[b]->data, sizeof(cplx) * sts[b]->total, cudaMemcpyDeviceToDevice,
                             ctx->stream));
  }
  const ttn_s* ref = sts[0];
  TTN_CUDA(cudaGraphLaunch(e->ex, ctx->stream));
  add_launches(e->launches);
  for (int b = 0; b < nb; ++b) {
    outs[b] = new_ttn_like(ctx, ref, TTN_STATE, e->tmpl[b]->bond);
    TTN_CUDA(cudaMemcpyAsync(outs[b]->data, e->tmpl[b]->data, sizeof(cplx) * e->tmpl[b]->total,
                             cudaMemcpyDeviceToDevice, ctx->stream));
  }
  ctx->sync();
  prof_replay(e->sink);
  if (!spec_ok(e->host, nb)) {
    for (int b = 0; b < nb; ++b) {
      free_ttn(outs[b]);
      outs[b] = nullptr;
    }
    return false;
  }
  const double secs = std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count();
  fill_reports(reps, nb, e->host, e->flops, e->maxb, e->peak, secs, ctx->host_syncs);
  return true;
}

}  // namespace

void graphs_release(ttn_ctx_s* ctx) {
  if (!ctx->gr) return;
  cudaStreamSynchronize(ctx->stream);
  for (auto& kv : ctx->gr->map) destroy_entry(ctx, kv.second.get());
  delete ctx->gr;
  ctx->gr = nullptr;
}

void cbc_apply_impl(ttn_ctx_s* ctx, int nb, const ttn_s* const* ops, const ttn_s* const* sts, int64_t max_bond,
                    double tol, ttn_s** outs, ttn_cbc_report* reps) {
  CoreCtl sync_cc;
  const bool part_on = ctx->comm && ctx->parts > 1;
  if (!ctx->speculate || tol != 0.0 || part_on || nb <= 0 || !ops || !sts || !ops[0] || !sts[0]) {
    apply_core(ctx, nb, ops, sts, max_bond, tol, outs, reps, sync_cc);
    return;
  }
  for (int b = 0; b < nb; ++b)
    if (!ops[b] || !sts[b]) throw Error(TTN_ERR_ARG, "NULL handle");
  auto& G = graphs_of(ctx);
  const std::vector<int64_t> skey = shape_key(nb, ops, sts, max_bond);
  // a failed speculation marks the tree (topology, dimensions, max_bond), not just these bonds:
  // workloads whose ranks are data dependent (circuits) change bonds every apply
  const std::vector<int64_t> tkey(skey.begin(), skey.begin() + 3 + 2 * sts[0]->n);
  if (G.failed.count(tkey)) {
    apply_core(ctx, nb, ops, sts, max_bond, tol, outs, reps, sync_cc);
    return;
  }
  const std::vector<int64_t>& gkey = skey;
  if (ctx->graphs) {
    auto it = G.map.find(gkey);
    if (it != G.map.end()) {
      it->second->last_use = ++G.tick;
      if (replay(ctx, it->second.get(), nb, ops, sts, outs, reps)) return;
      destroy_entry(ctx, it->second.get());
      G.map.erase(it);
      G.failed.insert(tkey);
      apply_core(ctx, nb, ops, sts, max_bond, tol, outs, reps, sync_cc);
      return;
    }
  }
  // speculative run (uncaptured)
  const size_t rb = SpecRes::bytes(nb);
  if (ctx->spec_host_size < rb) {
    if (ctx->spec_host) cudaFreeHost(ctx->spec_host);
    ctx->spec_host = nullptr;
    ctx->spec_host_size = 0;
    TTN_CUDA(cudaMallocHost(&ctx->spec_host, rb));
    ctx->spec_host_size = rb;
  }
  auto t0 = std::chrono::steady_clock::now();
  CoreCtl cc;
  cc.mode = Mode::Spec;
  cc.host_res = ctx->spec_host;
  ctx->ring->staged = 0;
  apply_core(ctx, nb, ops, sts, max_bond, tol, outs, nullptr, cc);
  const size_t staged = ctx->ring->staged;
  ctx->sync();
  TTN_CUDA(cudaGetLastError());
  if (!spec_ok(ctx->spec_host, nb)) {
    for (int b = 0; b < nb; ++b) {
      free_ttn(outs[b]);
      outs[b] = nullptr;
    }
    G.failed.insert(tkey);
    apply_core(ctx, nb, ops, sts, max_bond, tol, outs, reps, sync_cc);
    return;
  }
  const double secs = std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count();
  fill_reports(reps, nb, ctx->spec_host, cc.flops, cc.maxb, cc.peak, secs, ctx->host_syncs);
  // capture on the second successful speculative apply of the same shapes (a one-off apply
  // never pays for a capture)
  if (ctx->graphs && !cc.host_synced && !G.nograph.count(gkey) && !G.seen.count(gkey)) {
    if (G.seen.size() >= 256) G.seen.clear();
    G.seen.insert(gkey);
    return;
  }
  if (ctx->graphs && !cc.host_synced && !G.nograph.count(gkey)) {
    G.seen.erase(gkey);
    std::unique_ptr<GraphEntry> e = capture(ctx, nb, ops, sts, max_bond, staged, cc.out_elems);
    if (!e) {
      G.nograph.insert(gkey);
      return;
    }
    e->last_use = ++G.tick;
    if (G.map.size() >= 8) {   // least recently used entry goes
      auto old = G.map.begin();
      for (auto it = G.map.begin(); it != G.map.end(); ++it)
        if (it->second->last_use < old->second->last_use) old = it;
      destroy_entry(ctx, old->second.get());
      G.map.erase(old);
    }
    G.map[gkey] = std::move(e);
  }
}

void overlap_impl(ttn_ctx_s* ctx, int nb, const ttn_s* const* a, const ttn_s* const* bb, cplx* out) {
  const ttn_s* ref = a[0];
  for (int j = 0; j < nb; ++j) {
    if (!a[j] || !bb[j]) throw Error(TTN_ERR_ARG, "NULL handle");
    if (a[j]->kind != TTN_STATE || bb[j]->kind != TTN_STATE) throw Error(TTN_ERR_ARG, "ttn_overlap expects states");
    if (a[j]->parent != ref->parent || bb[j]->parent != ref->parent) throw Error(TTN_ERR_TOPOLOGY, "topology mismatch");
    if (a[j]->phys != ref->phys || bb[j]->phys != ref->phys) throw Error(TTN_ERR_SHAPE, "leg mismatch: physical dimensions");
  }
  const int n = ref->n;
  int maxd = 0;
  for (int i = 0; i < n; ++i) maxd = std::max(maxd, ref->depth[i]);
  ctx->scratch.reset();
  ctx->env.reset();
  std::vector<Fac> E((size_t)nb * n);
  ExecStats st;
  for (int L = maxd; L >= 0; --L) {
    std::vector<Task> tasks;
    std::vector<Fac*> dst;
    for (int j = 0; j < nb; ++j)
      for (int i = 0; i < n; ++i) {
        if (ref->depth[i] != L) continue;
        Task t;
        Operand A, B;
        A.ptr = a[j]->node(i); A.dims = a[j]->shape[i]; A.conj = true;
        B.ptr = bb[j]->node(i); B.dims = bb[j]->shape[i];
        A.labels.push_back(L_SIG);
        B.labels.push_back(L_SIG);
        for (size_t l = 0; l + 1 < A.dims.size(); ++l) {
          A.labels.push_back(L_A + (int)l);
          B.labels.push_back(L_B + (int)l);
        }
        t.ops.push_back(A);
        t.ops.push_back(B);
        for (size_t l = 0; l < ref->children[i].size(); ++l) {
          const Fac& ec = E[(size_t)j * n + ref->children[i][l]];
          Operand F;
          F.ptr = ec.p;
          F.dims = {ec.a, ec.b};
          F.labels = {L_A + 1 + (int)l, L_B + 1 + (int)l};
          t.ops.push_back(F);
        }
        t.out_labels = {L_A, L_B};
        Fac& e = E[(size_t)j * n + i];
        e.a = A.dims[1];
        e.b = B.dims[1];
        e.k = 1;
        e.p = static_cast<cplx*>(ctx->env.alloc(sizeof(cplx) * e.a * e.b));
        t.out = e.p;
        tasks.push_back(t);
      }
    contract_batch(ctx, tasks, st);
    ctx->scratch.reset();
  }
  ctx->ensure_small(sizeof(cplx) * nb);
  cplx* h = reinterpret_cast<cplx*>(ctx->hbuf);
  for (int j = 0; j < nb; ++j)
    TTN_CUDA(cudaMemcpyAsync(h + j, E[(size_t)j * n + ref->root].p, sizeof(cplx), cudaMemcpyDeviceToHost, ctx->stream));
  ctx->sync();
  TTN_CUDA(cudaGetLastError());
  for (int j = 0; j < nb; ++j) out[j] = h[j];
  ctx->env.reset();
}

// <bra| O_1 ... O_m |ket> by one leaves-to-root environment sweep: every node contracts its
// layer tensors (conj(bra), the operators, ket) with the children's environments (one leg
// per layer) into its parent-edge environment, through the same batched contraction engine.
// An operator layer with `dagger` enters as conj(O) with its physical legs swapped (O^dagger).
// Used for <phi|O|psi> (the projection identity P2 at full size) and ||O psi||^2 =
// <psi|O^dagger O|psi> (the truncation error eps^2 = 1 - ||phi||^2 / ||O psi||^2, A19).
void sweep_impl(ttn_ctx_s* ctx, int nb, const std::vector<SweepLayer>& layers, cplx* out) {
  const int nl = (int)layers.size();
  if (nl < 2 || layers.front().op || layers.back().op) throw Error(TTN_ERR_ARG, "sweep: bra and ket must be states");
  const ttn_s* ref = layers[0].h[0];
  for (int j = 0; j < nb; ++j)
    for (const auto& Ly : layers) {
      const ttn_s* t = Ly.h[j];
      if (!t) throw Error(TTN_ERR_ARG, "NULL handle");
      if ((t->kind == TTN_OPERATOR) != Ly.op) throw Error(TTN_ERR_ARG, "sweep: operator / state handle expected");
      if (t->parent != ref->parent) throw Error(TTN_ERR_TOPOLOGY, "topology mismatch");
      if (t->phys != ref->phys) throw Error(TTN_ERR_SHAPE, "leg mismatch: physical dimensions");
    }
  const int n = ref->n;
  int maxd = 0;
  for (int i = 0; i < n; ++i) maxd = std::max(maxd, ref->depth[i]);
  ctx->scratch.reset();
  ctx->env.reset();
  // environment of node i: one leg per layer (that layer's parent-edge bond)
  std::vector<cplx*> E((size_t)nb * n, nullptr);
  std::vector<std::vector<int64_t>> Edims((size_t)nb * n);
  ExecStats st;
  auto PHY = [](int k) { return 1 + k; };              // physical label between layers k-1 and k
  auto VIR = [](int k, int leg) { return 100 * (k + 1) + leg; };
  for (int L = maxd; L >= 0; --L) {
    std::vector<Task> tasks;
    for (int j = 0; j < nb; ++j)
      for (int i = 0; i < n; ++i) {
        if (ref->depth[i] != L) continue;
        Task t;
        int pk = 0;   // physical label index above the current layer
        for (int k = 0; k < nl; ++k) {
          const SweepLayer& Ly = layers[k];
          const ttn_s* h = Ly.h[j];
          Operand X;
          X.ptr = h->node(i);
          X.dims = h->shape[i];
          X.conj = Ly.conj;
          size_t v0;
          if (!Ly.op) {
            X.labels.push_back(PHY(pk));
            v0 = 1;
          } else {
            // O[out, in, ...]: plain O maps the label below (pk+1) to the one above (pk);
            // O^dagger = conj(O) with out / in swapped
            X.labels.push_back(Ly.dagger ? PHY(pk + 1) : PHY(pk));
            X.labels.push_back(Ly.dagger ? PHY(pk) : PHY(pk + 1));
            ++pk;
            v0 = 2;
          }
          for (size_t l = v0; l < X.dims.size(); ++l) X.labels.push_back(VIR(k, (int)(l - v0)));
          t.ops.push_back(X);
        }
        for (size_t c = 0; c < ref->children[i].size(); ++c) {
          const size_t ci = (size_t)j * n + ref->children[i][c];
          Operand F;
          F.ptr = E[ci];
          F.dims = Edims[ci];
          for (int k = 0; k < nl; ++k) F.labels.push_back(VIR(k, 1 + (int)c));
          t.ops.push_back(F);
        }
        std::vector<int64_t> od;
        int64_t tot = 1;
        for (int k = 0; k < nl; ++k) {
          t.out_labels.push_back(VIR(k, 0));
          const int64_t e = layers[k].h[j]->shape[i][layers[k].op ? 2 : 1];
          od.push_back(e);
          tot *= e;
        }
        const size_t me = (size_t)j * n + i;
        E[me] = static_cast<cplx*>(ctx->env.alloc(sizeof(cplx) * std::max<int64_t>(tot, 1)));
        Edims[me] = od;
        t.out = E[me];
        tasks.push_back(t);
      }
    contract_batch(ctx, tasks, st);
    ctx->scratch.reset();
  }
  ctx->ensure_small(sizeof(cplx) * nb);
  cplx* h = reinterpret_cast<cplx*>(ctx->hbuf);
  for (int j = 0; j < nb; ++j)
    TTN_CUDA(cudaMemcpyAsync(h + j, E[(size_t)j * n + ref->root], sizeof(cplx), cudaMemcpyDeviceToHost, ctx->stream));
  ctx->sync();
  TTN_CUDA(cudaGetLastError());
  for (int j = 0; j < nb; ++j) out[j] = h[j];
  ctx->env.reset();
}

}  // namespace tcbc
