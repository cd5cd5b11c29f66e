// Contraction planner / executor (see contract.h).
//
// Plans are cached per (operand labels, extents, conjugation, output order): the 64
// identical-shape instances of a batch share one plan.  A plan is a list of pairwise steps,
// each a ready-made strided GemmProblem template (the leg permutations live in the strides),
// so executing a batch is: bump-allocate the intermediates, patch pointers, and issue one
// grouped GEMM launch per step round.
#include "contract.h"
#include "prof.h"

#include <algorithm>
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <functional>
#include <map>
#include <memory>
#include <mutex>
#include <sstream>
#include <unordered_map>

namespace tcbc {

namespace {

struct StepT {
  int a = -1, b = -1;          // operand slots
  GemmProblem g{};             // legs / strides filled; A, B, C pointers patched at run time
  int64_t res_elems = 0;
  bool to_out = false;
};

struct PlanT {
  int nin = 0;
  std::vector<StepT> steps;
  double flops = 0.0;
  double flops_min = 0.0;      // the minimum over all pairwise orders (algorithmic work)
  int64_t peak = 0;
  bool permute_only = false;   // single operand: plain permutation into the output
};

std::vector<int64_t> rm_strides(const std::vector<int64_t>& dims) {
  std::vector<int64_t> s(dims.size(), 1);
  for (int i = (int)dims.size() - 2; i >= 0; --i) s[i] = s[i + 1] * dims[i + 1];
  return s;
}

int index_of(const std::vector<int>& L, int l) {
  return (int)(std::find(L.begin(), L.end(), l) - L.begin());
}

// One leg group (M, N or K) with the strides it has in two operands; adjacent legs that are
// contiguous in both operands are folded into one.
void fill_group(const std::vector<int>& labels, const std::map<int, int64_t>& dim,
                const std::vector<int>& L1, const std::vector<int64_t>& s1,
                const std::vector<int>& L2, const std::vector<int64_t>& s2,
                int& n, int* d, long long* st1, long long* st2) {
  std::vector<int64_t> dd, x1, x2;
  for (int l : labels) {
    const int64_t e = dim.at(l);
    if (e == 1) continue;   // extent-1 legs carry no index
    dd.push_back(e);
    x1.push_back(s1[index_of(L1, l)]);
    x2.push_back(s2[index_of(L2, l)]);
  }
  // fold: leg i followed by leg i+1 is one leg when s[i] == s[i+1] * d[i+1] in both
  std::vector<int64_t> fd, f1, f2;
  for (size_t i = 0; i < dd.size(); ++i) {
    if (!fd.empty() && f1.back() == x1[i] * dd[i] && f2.back() == x2[i] * dd[i]) {
      fd.back() *= dd[i];
      f1.back() = x1[i];
      f2.back() = x2[i];
    } else {
      fd.push_back(dd[i]);
      f1.push_back(x1[i]);
      f2.push_back(x2[i]);
    }
  }
  if (fd.empty()) {
    fd.push_back(1);
    f1.push_back(0);
    f2.push_back(0);
  }
  if ((int)fd.size() > GEMM_MAXD) throw Error(TTN_ERR_UNSUPPORTED, "contraction step with more than 6 folded legs");
  n = (int)fd.size();
  for (int i = 0; i < n; ++i) {
    if (fd[i] > INT32_MAX) throw Error(TTN_ERR_UNSUPPORTED, "leg extent exceeds 2^31");
    d[i] = (int)fd[i];
    st1[i] = f1[i];
    st2[i] = f2[i];
  }
}

PlanT make_plan(const Task& t) {
  const int n = (int)t.ops.size();
  std::map<int, int64_t> dim;
  for (auto& o : t.ops)
    for (size_t i = 0; i < o.labels.size(); ++i) dim[o.labels[i]] = o.dims[i];
  PlanT P;
  P.nin = n;
  if (n == 1) {
    P.permute_only = true;
    return P;
  }
  const int full = (1 << n) - 1;
  std::vector<std::vector<int>> freel(1 << n);
  for (int m = 1; m <= full; ++m) {
    std::map<int, int> cnt;
    std::vector<int> order;
    for (int i = 0; i < n; ++i)
      if (m & (1 << i))
        for (int l : t.ops[i].labels) {
          if (!cnt.count(l)) order.push_back(l);
          cnt[l] += 1;
        }
    for (int l : order)
      if (cnt[l] == 1) freel[m].push_back(l);
  }
  auto prod = [&](const std::vector<int>& L) {
    double p = 1.0;
    for (int l : L) p *= (double)dim[l];
    return p;
  };
  // cost of a pairwise step: time at the FP64 roofline (37 TF/s, 6.5 TB/s), the DMMA rate
  // derated for short contractions: a tile's fixed prologue / epilogue costs about 24 k-steps
  // (measured, tools/gemm_bench: 19 TF/s at K = 32, 29 at K = 128, 34 at K = 4096)
  static const double k0 = getenv("TTN_PLAN_K0") ? atof(getenv("TTN_PLAN_K0")) : 24.0;
  auto step_cost = [&](int sa, int sb, int sm) {
    std::vector<int> un = freel[sa];
    for (int l : freel[sb])
      if (std::find(un.begin(), un.end(), l) == un.end()) un.push_back(l);
    const double kk = prod(un) / std::max(1.0, prod(freel[sm]));   // contracted extent
    const double fl = 8.0 * prod(un) * (1.0 + k0 / std::max(1.0, kk));
    const double by = 16.0 * (prod(freel[sa]) + prod(freel[sb]) + prod(freel[sm]));
    return std::max(fl / 37e12, by / 6.5e12) + 2e-7;
  };
  // algorithmic work: the fewest flops of any pairwise order (what the roofline counts); the
  // executed order below may spend more flops where that is faster on the device
  {
    std::vector<double> fmin(1 << n, 0.0);
    for (int m = 1; m <= full; ++m) {
      if ((m & (m - 1)) == 0) continue;
      fmin[m] = 1e300;
      for (int sub = (m - 1) & m; sub > 0; sub = (sub - 1) & m) {
        const int rest = m ^ sub;
        if (sub < rest) continue;
        std::vector<int> un = freel[sub];
        for (int l : freel[rest])
          if (std::find(un.begin(), un.end(), l) == un.end()) un.push_back(l);
        fmin[m] = std::min(fmin[m], fmin[sub] + fmin[rest] + 8.0 * prod(un));
      }
    }
    P.flops_min = fmin[full];
  }
  std::vector<double> best(1 << n, 0.0), peak(1 << n, 0.0);
  std::vector<int> split(1 << n, 0);
  for (int m = 1; m <= full; ++m) {
    if ((m & (m - 1)) == 0) continue;
    best[m] = 1e300;
    for (int sub = (m - 1) & m; sub > 0; sub = (sub - 1) & m) {
      const int rest = m ^ sub;
      if (sub < rest) continue;
      const double c = best[sub] + best[rest] + step_cost(sub, rest, m);
      const double pk = std::max({peak[sub], peak[rest], prod(freel[m])});
      if (c < best[m] * (1 - 1e-9) || (c <= best[m] * (1 + 1e-9) && pk < peak[m])) {
        best[m] = c;
        peak[m] = pk;
        split[m] = sub;
      }
    }
  }
  std::vector<std::vector<int>> slab;
  std::vector<std::vector<int64_t>> sdim;
  for (auto& o : t.ops) {
    slab.push_back(o.labels);
    sdim.push_back(o.dims);
  }
  // Intermediate layouts, top-down: an intermediate's legs are ordered [legs its consumer
  // keeps, in the consumer's output order] ++ [legs the consumer contracts, in the order of the
  // sibling operand when that is an input].  The consumer then reads it as a plain row-major
  // operand with the contraction innermost (coalesced, folded legs), instead of gathering it.
  std::vector<std::vector<int>> layout(1 << n);
  static const bool natural = getenv("TTN_PLAN_NATURAL") != nullptr;
  if (!natural) {
    std::function<void(int)> assign = [&](int m) {
      if ((m & (m - 1)) == 0) return;   // input operand: fixed layout
      const int sub = split[m], rest = m ^ sub;
      const int ma = (sub & -sub) < (rest & -rest) ? sub : rest;
      const int mb = m ^ ma;
      const std::vector<int>& Lm = (m == full) ? t.out_labels : layout[m];
      auto has = [](const std::vector<int>& L, int l) { return std::find(L.begin(), L.end(), l) != L.end(); };
      for (int c : {ma, mb}) {
        if ((c & (c - 1)) == 0) continue;
        const int sib = m ^ c;
        std::vector<int> L;
        for (int l : Lm)
          if (has(freel[c], l)) L.push_back(l);
        // contracted legs: the sibling input's order; between two intermediates one common
        // order (the A side's), so the consumer's k legs fold in both operands
        const std::vector<int>& ko = ((sib & (sib - 1)) == 0) ? t.ops[__builtin_ctz(sib)].labels : freel[ma];
        for (int l : ko)
          if (has(freel[c], l) && has(freel[sib], l) && !has(L, l)) L.push_back(l);
        for (int l : freel[c])   // safety: every leg exactly once
          if (!has(L, l)) L.push_back(l);
        layout[c] = L;
      }
      assign(ma);
      assign(mb);
    };
    assign(full);
  }
  std::vector<int> slot_of_mask(1 << n, -1);
  for (int i = 0; i < n; ++i) slot_of_mask[1 << i] = i;
  std::function<int(int)> emit = [&](int m) -> int {
    if (slot_of_mask[m] >= 0) return slot_of_mask[m];
    const int sub = split[m], rest = m ^ sub;
    const int ma = (sub & -sub) < (rest & -rest) ? sub : rest;   // A: part with the lowest operand
    const int mb = m ^ ma;
    const int a = emit(ma), b = emit(mb);
    const std::vector<int>& LA = slab[a];
    const std::vector<int>& LB = slab[b];
    std::vector<int> K, FA, FB;
    for (int l : LA) (std::find(LB.begin(), LB.end(), l) != LB.end() ? K : FA).push_back(l);
    for (int l : LB)
      if (std::find(LA.begin(), LA.end(), l) == LA.end()) FB.push_back(l);
    const bool last = (m == full);
    std::vector<int> LC;
    if (last) LC = t.out_labels;
    else if (!layout[m].empty()) LC = layout[m];
    else {
      LC = FA;
      LC.insert(LC.end(), FB.begin(), FB.end());
    }
    std::vector<int64_t> dC;
    for (int l : LC) dC.push_back(dim[l]);
    const auto sA = rm_strides(sdim[a]), sB = rm_strides(sdim[b]), sC = rm_strides(dC);
    StepT s;
    s.a = a;
    s.b = b;
    s.to_out = last;
    GemmProblem& g = s.g;
    int64_t M = 1, N = 1, KK = 1;
    for (int l : FA) M *= dim[l];
    for (int l : FB) N *= dim[l];
    for (int l : K) KK *= dim[l];
    if (M > INT32_MAX || N > INT32_MAX || KK > INT32_MAX) throw Error(TTN_ERR_UNSUPPORTED, "GEMM extent exceeds 2^31");
    g.M = (int)M;
    g.N = (int)N;
    g.K = (int)KK;
    fill_group(FA, dim, LA, sA, LC, sC, g.nm, g.md, g.am, g.cm);
    fill_group(FB, dim, LB, sB, LC, sC, g.nn, g.nd, g.bn, g.cn);
    fill_group(K, dim, LA, sA, LB, sB, g.nk, g.kd, g.ak, g.bk);
    g.alpha = make_double2(1.0, 0.0);
    g.beta = make_double2(0.0, 0.0);
    g.conjA = (a < n && t.ops[a].conj) ? 1 : 0;
    g.conjB = (b < n && t.ops[b].conj) ? 1 : 0;
    s.res_elems = M * N;
    P.flops += 8.0 * (double)M * N * KK;
    P.peak = std::max<int64_t>(P.peak, M * N);
    P.steps.push_back(s);
    slab.push_back(LC);
    sdim.push_back(dC);
    slot_of_mask[m] = (int)slab.size() - 1;
    return slot_of_mask[m];
  };
  emit(full);
  return P;
}

// plan key: the integer signature of the task (per operand: conj flag, labels, extents;
// then the output labels), hashed without building strings (this lookup runs for every node
// of every instance at every level: ~1e5 times per config-5 step)
struct KeyHash {
  size_t operator()(const std::vector<int64_t>& v) const {
    uint64_t h = 1469598103934665603ull;
    for (int64_t x : v) {
      h ^= (uint64_t)x + 0x9e3779b97f4a7c15ull + (h << 6) + (h >> 2);
      h *= 1099511628211ull;
    }
    return (size_t)h;
  }
};

void plan_key(const Task& t, std::vector<int64_t>& k) {
  k.clear();
  for (auto& o : t.ops) {
    k.push_back(o.conj ? -2 : -3);
    for (size_t i = 0; i < o.labels.size(); ++i) {
      k.push_back(o.labels[i]);
      k.push_back(o.dims[i]);
    }
  }
  k.push_back(-4);
  for (int l : t.out_labels) k.push_back(l);
}

// Plans are shared: a batch (and other worker threads) keep the plans they use alive while
// the cache evicts, so bounding the cache never frees a plan in use.
using PlanPtr = std::shared_ptr<const PlanT>;
std::mutex g_plan_mu;
std::unordered_map<std::vector<int64_t>, PlanPtr, KeyHash>& plan_cache() {
  static std::unordered_map<std::vector<int64_t>, PlanPtr, KeyHash> c;
  return c;
}

PlanPtr get_plan(const Task& t) {
  thread_local std::vector<int64_t> key;
  plan_key(t, key);
  {
    std::lock_guard<std::mutex> lk(g_plan_mu);
    auto& c = plan_cache();
    auto it = c.find(key);
    if (it != c.end()) return it->second;
  }
  PlanPtr p = std::make_shared<const PlanT>(make_plan(t));   // planned outside the lock
  std::lock_guard<std::mutex> lk(g_plan_mu);
  auto& c = plan_cache();
  if (c.size() > 200000) c.clear();   // in-use plans survive through their shared owners
  return c.emplace(key, p).first->second;
}

}  // namespace

namespace {
struct ArenaScratch : Scratch {
  Arena& a;
  explicit ArenaScratch(Arena& ar) : a(ar) {}
  void* get(size_t bytes) override { return a.alloc(bytes); }
};
}  // namespace

double gemm_flops(const GemmProblem& g) {
  return g.sym ? 4.0 * (double)g.M * (g.M + 1) * g.K : 8.0 * (double)g.M * g.N * g.K;
}

void gemm_batch(ttn_ctx_s* ctx, std::vector<GemmProblem>& probs, ExecStats& st, const char* family) {
  HostScope hs_("gemm_batch");
  for (auto& g : probs) st.flops += gemm_flops(g);
  static const bool dbg = getenv("TTN_DEBUG_GEMM") != nullptr;
  if (dbg && !probs.empty()) {
    std::map<std::string, int> shapes;
    for (auto& g : probs) {
      std::ostringstream o;
      o << g.M << "x" << g.N << "x" << g.K << " legs" << g.nm << g.nn << g.nk << " c" << g.conjA << g.conjB;
      if ((double)g.M * g.N * g.K > 5e7) {
        o << " [m";
        for (int q = 0; q < g.nm; ++q) o << " " << g.md[q] << ":" << g.am[q] << "/" << g.cm[q];
        o << " n";
        for (int q = 0; q < g.nn; ++q) o << " " << g.nd[q] << ":" << g.bn[q] << "/" << g.cn[q];
        o << " k";
        for (int q = 0; q < g.nk; ++q) o << " " << g.kd[q] << ":" << g.ak[q] << "/" << g.bk[q];
        o << "]";
      }
      shapes[o.str()] += 1;
    }
    fprintf(stderr, "[gemm] %zu problems:", probs.size());
    for (auto& kv : shapes) fprintf(stderr, " %s*%d", kv.first.c_str(), kv.second);
    fprintf(stderr, "\n");
  }
  ArenaScratch ws(ctx->scratch);
  if (!probs.empty()) launch_gemm(probs.data(), (int)probs.size(), *ctx->stager, ctx->stream, &ws, family);
}

GemmProblem mk_gemm(const cplx* A, int opA, long long lda, const cplx* B, int opB, long long ldb, cplx* C,
                    long long ldc, int64_t M, int64_t N, int64_t K) {
  GemmProblem g{};
  g.A = A;
  g.B = B;
  g.C = C;
  g.M = (int)M;
  g.N = (int)N;
  g.K = (int)K;
  gemm_from_ops(g, opA, lda, opB, ldb, ldc);
  g.alpha = make_double2(1.0, 0.0);
  g.beta = make_double2(0.0, 0.0);
  return g;
}

void contract_batch(ttn_ctx_s* ctx, std::vector<Task>& tasks, ExecStats& st) {
  HostScope hs_("contract_batch");
  if (tasks.empty()) return;
  std::vector<PlanPtr> plans(tasks.size());
  size_t max_steps = 0;
  std::vector<PermProblem> perms;
  for (size_t i = 0; i < tasks.size(); ++i) {
    Task& t = tasks[i];
    plans[i] = get_plan(t);
    t.out_dims.clear();
    int64_t tot = 1;
    for (int l : t.out_labels) {   // extent of each output label (first operand carrying it)
      int64_t e = -1;
      for (auto& o : t.ops) {
        for (size_t j = 0; j < o.labels.size(); ++j)
          if (o.labels[j] == l) { e = o.dims[j]; break; }
        if (e >= 0) break;
      }
      if (e < 0) throw Error(TTN_ERR_ARG, "output label not carried by any operand");
      t.out_dims.push_back(e);
      tot *= e;
    }
    if (!t.out) t.out = static_cast<cplx*>(ctx->scratch.alloc(sizeof(cplx) * std::max<int64_t>(tot, 1)));
    st.peak_entries = std::max(st.peak_entries, std::max(tot, plans[i]->peak));
    t.flops = plans[i]->flops;
    t.flops_min = plans[i]->flops_min;
    max_steps = std::max(max_steps, plans[i]->steps.size());
    if (plans[i]->permute_only) {   // single operand: permutation into the output
      const Operand& o = t.ops[0];
      PermProblem pp{};
      pp.src = o.ptr;
      pp.dst = t.out;
      pp.rank = (int)t.out_labels.size();
      if (pp.rank > 8) throw Error(TTN_ERR_UNSUPPORTED, "rank > 8 permutation");
      auto s = rm_strides(o.dims);
      pp.total = tot;
      for (int r = 0; r < pp.rank; ++r) {
        const int j = index_of(o.labels, t.out_labels[r]);
        pp.dims[r] = o.dims[j];
        pp.sstride[r] = s[j];
      }
      pp.conj = o.conj ? 1 : 0;
      perms.push_back(pp);
    }
  }
  if (!perms.empty()) launch_permute(perms.data(), (int)perms.size(), *ctx->stager, ctx->stream);
  // slot pointers per task
  std::vector<std::vector<const cplx*>> slot(tasks.size());
  for (size_t i = 0; i < tasks.size(); ++i) {
    slot[i].resize(plans[i]->nin + plans[i]->steps.size());
    for (int j = 0; j < plans[i]->nin; ++j) slot[i][j] = tasks[i].ops[j].ptr;
  }
  std::vector<GemmProblem> round;
  for (size_t r = 0; r < max_steps; ++r) {
    round.clear();
    for (size_t i = 0; i < tasks.size(); ++i) {
      const PlanT& P = *plans[i];
      if (r >= P.steps.size()) continue;
      const StepT& s = P.steps[r];
      GemmProblem g = s.g;
      g.A = slot[i][s.a];
      g.B = slot[i][s.b];
      cplx* C = s.to_out ? tasks[i].out
                         : static_cast<cplx*>(ctx->scratch.alloc(sizeof(cplx) * std::max<int64_t>(s.res_elems, 1)));
      g.C = C;
      if (s.to_out) g.exp_out = tasks[i].out_exp;
      slot[i][P.nin + r] = C;
      round.push_back(g);
    }
    gemm_batch(ctx, round, st);
  }
}

}  // namespace tcbc
