// Batched tensor-network contraction engine: every node contraction of the CBC sweeps
// (Eqs. 10, 11, 12 and 14) and of the overlap sweep is a small network
// (state tensor, operator tensor, up to three environment factors).  The host plans the
// cheapest pairwise order (exhaustive over subsets, cost = complex MACs, tie-break on the
// largest intermediate), lowers each pair to one GEMM (operand legs permuted only when they
// are not already a contiguous prefix / suffix in matching order), groups tasks whose plans
// have the same structure, and issues one grouped permute + one grouped GEMM launch per step.
#pragma once
#include "runtime.h"

#include <string>
#include <vector>

namespace tcbc {

struct Operand {
  const cplx* ptr = nullptr;
  std::vector<int> labels;
  std::vector<int64_t> dims;
  bool conj = false;
};

struct Task {
  std::vector<Operand> ops;
  std::vector<int> out_labels;
  cplx* out = nullptr;                 // destination; allocated from ctx->scratch when null
  int* out_exp = nullptr;              // optional: max binary exponent of the output (GEMM epilogue)
  std::vector<int64_t> out_dims;       // filled by contract_batch
  double flops = 0.0;                  // filled by contract_batch (8 * complex MACs)
  double flops_min = 0.0;              // filled by contract_batch: the cheapest order's flops
};

struct ExecStats {
  double flops = 0.0;                  // 8 * complex MACs issued to the GEMM core
  int64_t peak_entries = 0;            // largest single intermediate / output (complex entries)
};

void contract_batch(ttn_ctx_s* ctx, std::vector<Task>& tasks, ExecStats& st);

// Convenience: grouped GEMM with host bookkeeping of flops.  `family` is the profiler family the
// launch is timed under (the eigensolver's own GEMMs go under "heev", not the contraction's "zgemm").
void gemm_batch(ttn_ctx_s* ctx, std::vector<GemmProblem>& probs, ExecStats& st, const char* family = "zgemm");

// Algorithmic flops of one problem (8 per complex MAC; Hermitian products count the lower half).
double gemm_flops(const GemmProblem& g);

// Plain matrix product problem from BLAS-style op flags (OP_N/T/R/C) and leading dimensions.
GemmProblem mk_gemm(const cplx* A, int opA, long long lda, const cplx* B, int opB, long long ldb, cplx* C,
                    long long ldc, int64_t M, int64_t N, int64_t K);

}  // namespace tcbc
