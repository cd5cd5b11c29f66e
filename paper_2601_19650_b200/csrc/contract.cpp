// Contraction planner / executor (see contract.h).
#include "contract.h"

#include <algorithm>
#include <functional>
#include <map>
#include <numeric>
#include <sstream>

namespace tcbc {

namespace {

struct Step {
  int a = -1, b = -1;
  bool permA = false, permB = false;
  std::vector<int> newA, newB;        // stored label order after permutation
  bool tA = false, tB = false;        // stored transposed
  std::vector<int> labC;
};

struct Plan {
  std::vector<Step> steps;
  std::vector<std::vector<int>> slot_labels;   // inputs then step results
  bool final_perm = false;
  std::string sig;
};

bool is_prefix(const std::vector<int>& L, const std::vector<int>& K) {
  if (K.size() > L.size()) return false;
  for (size_t i = 0; i < K.size(); ++i)
    if (std::find(K.begin(), K.end(), L[i]) == K.end()) return false;
  return true;
}
bool is_suffix(const std::vector<int>& L, const std::vector<int>& K) {
  if (K.size() > L.size()) return false;
  size_t off = L.size() - K.size();
  for (size_t i = 0; i < K.size(); ++i)
    if (std::find(K.begin(), K.end(), L[off + i]) == K.end()) return false;
  return true;
}
std::vector<int> ordered_subset(const std::vector<int>& L, const std::vector<int>& S) {
  std::vector<int> out;
  for (int l : L)
    if (std::find(S.begin(), S.end(), l) != S.end()) out.push_back(l);
  return out;
}
std::vector<int> minus(const std::vector<int>& L, const std::vector<int>& S) {
  std::vector<int> out;
  for (int l : L)
    if (std::find(S.begin(), S.end(), l) == S.end()) out.push_back(l);
  return out;
}

// Decide the GEMM layout of one pairwise contraction.
void layout_step(Step& s, const std::vector<int>& LA, const std::vector<int>& LB,
                 const std::map<int, int64_t>& dim) {
  std::vector<int> K = ordered_subset(LA, LB);
  std::vector<int> FA = minus(LA, K), FB = minus(LB, K);
  auto size_of = [&](const std::vector<int>& L) {
    int64_t p = 1;
    for (int l : L) p *= dim.at(l);
    return p;
  };
  bool sufA = is_suffix(LA, K), preA = is_prefix(LA, K);
  bool preB = is_prefix(LB, K), sufB = is_suffix(LB, K);
  std::vector<int> KA, KB;
  if (sufA) KA = std::vector<int>(LA.end() - K.size(), LA.end());
  else if (preA) KA = std::vector<int>(LA.begin(), LA.begin() + K.size());
  if (preB) KB = std::vector<int>(LB.begin(), LB.begin() + K.size());
  else if (sufB) KB = std::vector<int>(LB.end() - K.size(), LB.end());
  bool okA = sufA || preA, okB = preB || sufB;
  s.permA = s.permB = false;
  std::vector<int> Kord;
  if (okA && okB && KA == KB) {
    Kord = KA;
  } else if (okA && okB) {
    if (size_of(LA) <= size_of(LB)) { Kord = KB; s.permA = true; }
    else { Kord = KA; s.permB = true; }
  } else if (okA) {
    Kord = KA; s.permB = true;
  } else if (okB) {
    Kord = KB; s.permA = true;
  } else {
    Kord = K; s.permA = s.permB = true;
  }
  if (s.permA) {
    s.newA = FA;
    s.newA.insert(s.newA.end(), Kord.begin(), Kord.end());
    s.tA = false;
  } else {
    s.newA = LA;
    s.tA = !sufA;                    // stored [K, FA] -> transposed
  }
  if (s.permB) {
    s.newB = Kord;
    s.newB.insert(s.newB.end(), FB.begin(), FB.end());
    s.tB = false;
  } else {
    s.newB = LB;
    s.tB = !preB;                    // stored [FB, K] -> transposed
  }
  s.labC = FA;
  s.labC.insert(s.labC.end(), FB.begin(), FB.end());
}

Plan make_plan(const Task& t) {
  const int n = (int)t.ops.size();
  std::map<int, int64_t> dim;
  std::map<int, int> total_count;
  for (auto& o : t.ops)
    for (size_t i = 0; i < o.labels.size(); ++i) {
      dim[o.labels[i]] = o.dims[i];
      total_count[o.labels[i]] += 1;
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
  std::vector<double> best(1 << n, 0.0), peak(1 << n, 0.0);
  std::vector<int> split(1 << n, 0);
  for (int m = 1; m <= full; ++m) {
    if ((m & (m - 1)) == 0) { best[m] = 0; peak[m] = 0; continue; }
    best[m] = 1e300;
    for (int sub = (m - 1) & m; sub > 0; sub = (sub - 1) & m) {
      int rest = m ^ sub;
      if (sub < rest) continue;
      std::vector<int> un = freel[sub];
      for (int l : freel[rest])
        if (std::find(un.begin(), un.end(), l) == un.end()) un.push_back(l);
      double c = best[sub] + best[rest] + prod(un);
      double pk = std::max({peak[sub], peak[rest], prod(freel[m])});
      if (c < best[m] * (1 - 1e-12) || (c <= best[m] * (1 + 1e-12) && pk < peak[m])) {
        best[m] = c;
        peak[m] = pk;
        split[m] = sub;
      }
    }
  }
  Plan p;
  for (auto& o : t.ops) p.slot_labels.push_back(o.labels);
  std::vector<int> slot_of_mask(1 << n, -1);
  for (int i = 0; i < n; ++i) slot_of_mask[1 << i] = i;
  // emit in post-order
  std::function<int(int)> emit = [&](int m) -> int {
    if (slot_of_mask[m] >= 0) return slot_of_mask[m];
    int sub = split[m], rest = m ^ sub;
    // A side: the part that holds the lowest-index operand (the state tensor is operand 0)
    int ma = (sub & -sub) < (rest & -rest) ? sub : rest;
    int mb = m ^ ma;
    int a = emit(ma), b = emit(mb);
    Step s;
    s.a = a;
    s.b = b;
    layout_step(s, p.slot_labels[a], p.slot_labels[b], dim);
    p.steps.push_back(s);
    p.slot_labels.push_back(s.labC);
    slot_of_mask[m] = (int)p.slot_labels.size() - 1;
    return slot_of_mask[m];
  };
  int last = emit(full);
  p.final_perm = (p.slot_labels[last] != t.out_labels);
  // signature: structure with labels replaced by positions
  std::ostringstream os;
  os << n << ":";
  for (auto& o : t.ops) os << o.labels.size() << (o.conj ? "c" : "") << ",";
  auto pos = [](const std::vector<int>& L, const std::vector<int>& newL) {
    std::ostringstream q;
    for (int l : newL) q << (int)(std::find(L.begin(), L.end(), l) - L.begin()) << ".";
    return q.str();
  };
  for (auto& s : p.steps) {
    os << "|" << s.a << "," << s.b << "," << s.tA << s.tB << s.permA << s.permB << ","
       << pos(p.slot_labels[s.a], s.newA) << "," << pos(p.slot_labels[s.b], s.newB);
  }
  os << "|F" << p.final_perm << pos(p.slot_labels[last], t.out_labels);
  // labels of the inputs also fixed (positions refer to them): include them
  for (auto& o : t.ops) {
    os << "/";
    for (int l : o.labels) os << l << ".";
  }
  p.sig = os.str();
  return p;
}

std::vector<int64_t> strides_of(const std::vector<int64_t>& dims) {
  std::vector<int64_t> s(dims.size(), 1);
  for (int i = (int)dims.size() - 2; i >= 0; --i) s[i] = s[i + 1] * dims[i + 1];
  return s;
}

PermProblem make_perm(const cplx* src, cplx* dst, const std::vector<int>& L, const std::vector<int64_t>& dims,
                      const std::vector<int>& newL) {
  PermProblem pp{};
  pp.src = src;
  pp.dst = dst;
  auto st = strides_of(dims);
  pp.rank = (int)newL.size();
  if (pp.rank > 8) throw Error(TTN_ERR_UNSUPPORTED, "tensor rank > 8 in a contraction step");
  pp.total = 1;
  for (int r = 0; r < pp.rank; ++r) {
    int i = (int)(std::find(L.begin(), L.end(), newL[r]) - L.begin());
    pp.dims[r] = dims[i];
    pp.sstride[r] = st[i];
    pp.total *= dims[i];
  }
  pp.conj = 0;
  return pp;
}

}  // namespace

void gemm_batch(ttn_ctx_s* ctx, std::vector<GemmProblem>& probs, ExecStats& st) {
  for (auto& g : probs) st.flops += 8.0 * (double)g.M * g.N * g.K;
  if (!probs.empty()) launch_gemm(probs.data(), (int)probs.size(), *ctx->stager, ctx->stream);
}

void contract_batch(ttn_ctx_s* ctx, std::vector<Task>& tasks, ExecStats& st) {
  if (tasks.empty()) return;
  std::vector<Plan> plans(tasks.size());
  std::map<std::string, std::vector<int>> groups;
  for (size_t i = 0; i < tasks.size(); ++i) {
    plans[i] = make_plan(tasks[i]);
    groups[plans[i].sig].push_back((int)i);
    // output dims
    std::map<int, int64_t> dim;
    for (auto& o : tasks[i].ops)
      for (size_t j = 0; j < o.labels.size(); ++j) dim[o.labels[j]] = o.dims[j];
    tasks[i].out_dims.clear();
    int64_t tot = 1;
    for (int l : tasks[i].out_labels) {
      tasks[i].out_dims.push_back(dim.at(l));
      tot *= dim.at(l);
    }
    if (!tasks[i].out) tasks[i].out = static_cast<cplx*>(ctx->scratch.alloc(sizeof(cplx) * std::max<int64_t>(tot, 1)));
    st.peak_entries = std::max(st.peak_entries, tot);
  }
  for (auto& kv : groups) {
    const std::vector<int>& idx = kv.second;
    const Plan& P0 = plans[idx[0]];
    const int nin = (int)tasks[idx[0]].ops.size();
    const int nslots = nin + (int)P0.steps.size();
    // per task slot state
    std::vector<std::vector<const cplx*>> sptr(idx.size(), std::vector<const cplx*>(nslots, nullptr));
    std::vector<std::vector<std::vector<int64_t>>> sdims(idx.size(), std::vector<std::vector<int64_t>>(nslots));
    std::vector<std::map<int, int64_t>> dims(idx.size());
    for (size_t g = 0; g < idx.size(); ++g) {
      Task& t = tasks[idx[g]];
      for (int i = 0; i < nin; ++i) {
        sptr[g][i] = t.ops[i].ptr;
        sdims[g][i] = t.ops[i].dims;
        for (size_t j = 0; j < t.ops[i].labels.size(); ++j) dims[g][t.ops[i].labels[j]] = t.ops[i].dims[j];
      }
    }
    if (P0.steps.empty()) {  // single operand: permute into out
      std::vector<PermProblem> pp;
      for (size_t g = 0; g < idx.size(); ++g) {
        Task& t = tasks[idx[g]];
        PermProblem q = make_perm(t.ops[0].ptr, t.out, t.ops[0].labels, t.ops[0].dims, t.out_labels);
        q.conj = t.ops[0].conj ? 1 : 0;
        pp.push_back(q);
      }
      launch_permute(pp.data(), (int)pp.size(), *ctx->stager, ctx->stream);
      continue;
    }
    for (size_t si = 0; si < P0.steps.size(); ++si) {
      const Step& S = P0.steps[si];
      const bool last = (si + 1 == P0.steps.size());
      std::vector<PermProblem> perms;
      std::vector<GemmProblem> gemms;
      for (size_t g = 0; g < idx.size(); ++g) {
        Task& t = tasks[idx[g]];
        const Plan& Pg = plans[idx[g]];
        const std::vector<int>& LA = Pg.slot_labels[S.a];
        const std::vector<int>& LB = Pg.slot_labels[S.b];
        auto dl = [&](const std::vector<int>& L) {
          std::vector<int64_t> d;
          for (int l : L) d.push_back(dims[g].at(l));
          return d;
        };
        std::vector<int64_t> dA = dl(LA), dB = dl(LB);
        const cplx* pA = sptr[g][S.a];
        const cplx* pB = sptr[g][S.b];
        bool cA = S.a < nin && t.ops[S.a].conj, cB = S.b < nin && t.ops[S.b].conj;
        int64_t sizeA = 1, sizeB = 1;
        for (auto x : dA) sizeA *= x;
        for (auto x : dB) sizeB *= x;
        if (S.permA) {
          cplx* tmp = static_cast<cplx*>(ctx->scratch.alloc(sizeof(cplx) * std::max<int64_t>(sizeA, 1)));
          perms.push_back(make_perm(pA, tmp, LA, dA, S.newA));
          pA = tmp;
        }
        if (S.permB) {
          cplx* tmp = static_cast<cplx*>(ctx->scratch.alloc(sizeof(cplx) * std::max<int64_t>(sizeB, 1)));
          perms.push_back(make_perm(pB, tmp, LB, dB, S.newB));
          pB = tmp;
        }
        // M, N, K
        std::vector<int> K = ordered_subset(S.newA, S.newB);
        int64_t M = 1, N = 1, KK = 1;
        for (int l : S.newA)
          if (std::find(K.begin(), K.end(), l) == K.end()) M *= dims[g].at(l);
        for (int l : S.newB)
          if (std::find(K.begin(), K.end(), l) == K.end()) N *= dims[g].at(l);
        for (int l : K) KK *= dims[g].at(l);
        cplx* C;
        if (last && !Pg.final_perm) C = t.out;
        else C = static_cast<cplx*>(ctx->scratch.alloc(sizeof(cplx) * std::max<int64_t>(M * N, 1)));
        st.peak_entries = std::max(st.peak_entries, M * N);
        if (M > INT32_MAX || N > INT32_MAX || KK > INT32_MAX)
          throw Error(TTN_ERR_UNSUPPORTED, "GEMM dimension exceeds 2^31");
        GemmProblem gp{};
        gp.A = pA;
        gp.B = pB;
        gp.C = C;
        gp.M = (int)M;
        gp.N = (int)N;
        gp.K = (int)KK;
        gp.opA = (S.tA ? OP_T : OP_N) | (cA ? 2 : 0);
        gp.opB = (S.tB ? OP_T : OP_N) | (cB ? 2 : 0);
        gp.lda = S.tA ? M : KK;
        gp.ldb = S.tB ? KK : N;
        gp.ldc = N;
        gp.alpha = make_double2(1.0, 0.0);
        gp.beta = make_double2(0.0, 0.0);
        gemms.push_back(gp);
        sptr[g][nin + si] = C;
      }
      if (!perms.empty()) launch_permute(perms.data(), (int)perms.size(), *ctx->stager, ctx->stream);
      gemm_batch(ctx, gemms, st);
    }
    if (P0.final_perm) {
      std::vector<PermProblem> perms;
      for (size_t g = 0; g < idx.size(); ++g) {
        Task& t = tasks[idx[g]];
        const Plan& Pg = plans[idx[g]];
        int lastslot = nslots - 1;
        const std::vector<int>& L = Pg.slot_labels[lastslot];
        std::vector<int64_t> d;
        for (int l : L) d.push_back(dims[g].at(l));
        perms.push_back(make_perm(sptr[g][lastslot], t.out, L, d, t.out_labels));
      }
      launch_permute(perms.data(), (int)perms.size(), *ctx->stager, ctx->stream);
    }
  }
}

}  // namespace tcbc
