// Large-Gram top-k eigensolver (Chebyshev-filtered subspace iteration on the DMMA GEMM path);
// see chfsi.cu.  Writes results in the HeevProblem contract of kernels.h.
#pragma once
#include "contract.h"

#include <vector>

namespace tcbc {

constexpr int kLargeN = 512;   // Grams above this order go to chfsi_heev when applicable

int chfsi_block(int n, int kmax);            // subspace width p = kmax + oversampling
bool chfsi_applicable(int n, int kmax);      // n > kLargeN, p <= 512, 2p <= n
// Top-kmax eigenpairs of every problem's A (not modified); host-driven, synchronises once per
// outer iteration.  Throws Error(TTN_ERR_NUMERIC) on non-finite data or non-convergence.
void chfsi_heev(ttn_ctx_s* ctx, std::vector<HeevProblem*>& probs, ExecStats& st);

}  // namespace tcbc
