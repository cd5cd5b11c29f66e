// Device-kernel launchers of libttncbc (grouped / batched problems, complex128).
// Every launcher takes a host copy of the problem array (for scheduling) and a device copy
// (what the kernel reads); both describe the same problems.
#pragma once
#include <functional>
#include <utility>
#include <vector>
#include <cuda_runtime.h>
#include <cstdint>

namespace tcbc {

// Programmatic dependent launch (sm_90+): every kernel of the library begins with
// griddepcontrol.wait (it returns once the preceding grid of the stream has completed and its
// writes are visible; immediately when there is none), so launching with
// cudaLaunchAttributeProgrammaticStreamSerialization only lets a kernel's launch and prologue
// overlap the tail of the previous one.  No kernel triggers its dependents early (a persistent
// GEMM must keep every SM).  Opt-in (TTN_PDL=1): measured neutral to slightly negative on
// configs 1, 2, 3 and 5 (the small kernels' own duration, not the launch gap, dominates).
#define TCBC_PDL_WAIT() asm volatile("griddepcontrol.wait;" ::: "memory")
bool pdl_enabled();
template <typename... KArgs, typename... Args>
inline void launch_k(void (*kern)(KArgs...), dim3 grid, dim3 block, size_t smem, cudaStream_t s, Args&&... args) {
  cudaLaunchConfig_t cfg{};
  cfg.gridDim = grid;
  cfg.blockDim = block;
  cfg.dynamicSmemBytes = smem;
  cfg.stream = s;
  cudaLaunchAttribute at[1];
  at[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  at[0].val.programmaticStreamSerializationAllowed = pdl_enabled() ? 1 : 0;
  cfg.attrs = at;
  cfg.numAttrs = 1;
  cudaLaunchKernelEx(&cfg, kern, std::forward<Args>(args)...);
}

typedef double2 cplx;   // (x = re, y = im), 16-byte aligned

// op bits: bit0 = transpose, bit1 = conjugate
enum { OP_N = 0, OP_T = 1, OP_R = 2 /*conj, no transpose*/, OP_C = 3 /*conj transpose*/ };

// Strided tensor-contraction GEMM:
//   C[m, n] = alpha * sum_k opA(A)[m, k] * opB(B)[k, n] + beta * C[m, n]
// m, n, k are multi-indices over nm / nn / nk legs (extents md / nd / kd, row-major: the last
// leg fastest); element offsets are sum_leg index * stride with per-operand strides
// (am, ak for A; bk, bn for B; cm, cn for C).  conjA / conjB conjugate the operand.
constexpr int GEMM_MAXD = 6;
// Coordinate rule of one operand's TMA tensor map (gemm.cu, tma_fold): dim d of the map is a
// leg of the operand's row multi-index (m for A, n for B) or of its k multi-index (bit d of
// kmask); for a box starting at row x / contraction index k its coordinate is
// (x_or_k / div[d]) % mod[d] (mod 0: none), doubled for dim 0 (counted in doubles).
struct TmaDims {
  int rank, kmask;
  int chunks;   // boxes per stage: 1, or one per 8 rows (row leg ragged), each 1 KB further on
  int pad_;
  int div[5], mod[5];
};
struct GemmProblem {
  const cplx* A;
  const cplx* B;
  cplx* C;
  int M, N, K;
  int conjA, conjB;
  int nm, nn, nk;
  int md[GEMM_MAXD], nd[GEMM_MAXD], kd[GEMM_MAXD];
  long long am[GEMM_MAXD], ak[GEMM_MAXD], bk[GEMM_MAXD], bn[GEMM_MAXD], cm[GEMM_MAXD], cn[GEMM_MAXD];
  int tile_start;      // filled by the launcher
  int tiles_n;         // filled by the launcher
  cplx alpha, beta;
  int sym;             // Hermitian product (C = A^H A or A A^H, alpha real, beta 0): only the
                       // lower tiles are computed, each off-diagonal tile also writes its mirror
  int ksplit;          // filled by the launcher: k-range splits (partials reduced in ws)
  int kchunk;          // filled by the launcher
  int tiles_mn;        // filled by the launcher: output tiles per split
  cplx* ws;            // filled by the launcher: ksplit x M x N partial products
  int* exp_out;        // may be null: atomicMax of the binary exponents of the written C
                       // entries (the producer side of pow2 range control)
  // TMA staging (filled by the launcher): tma >= 0 is the index of this problem's operand
  // tensor maps in the launch's map array (A at 2*tma, B at 2*tma + 1); -1 = cp.async path
  int tma;
  int tma_pad_;
  TmaDims ta, tb;
};
// Device scratch for the launchers (stream-ordered bump memory owned by the caller).
struct Scratch {
  virtual void* get(size_t bytes) = 0;
  virtual ~Scratch() {}
};
// Fill the leg descriptors of a plain matrix product from BLAS-style op flags
// (bit0 transpose: A stored K x M / B stored N x K; bit1 conjugate) and leading dimensions.
void gemm_from_ops(GemmProblem& g, int opA, long long lda, int opB, long long ldb, long long ldc);

// dst[i] = (conj?) src[offset(i)], dst contiguous with dims[0..rank) (row-major);
// sstride[r] is the source stride of destination axis r.
struct PermProblem {
  const cplx* src;
  cplx* dst;
  long long total;
  long long start;     // filled by the launcher (prefix of totals)
  int rank;
  int conj;
  long long dims[8];
  long long sstride[8];
  int dst_strided;     // 0: dst contiguous; 1: dst offset = sum_r index_r * dstride[r] (a scatter)
  int pad_;
  long long dstride[8];
};

// Top-kmax eigenpairs of an n x n Hermitian matrix A (full storage, row-major, lda = n;
// destroyed).  Writes lam[0..kmax) descending, Vt[t*n + i] = i-th entry of eigenvector t,
// and the truncation decision k = min(max_bond, #{lam > tol^2 lam_1}, #{lam > floor lam_1}) >= 1,
// discarded weight w = trace - sum_{t<k} lam_t, trace, and zero-matrix flag.
struct HeevProblem {
  cplx* A;
  int n;
  int kmax;
  double* lam;
  cplx* Vt;
  int* k_out;          // may be null
  double* w_out;       // may be null
  double* work;        // real workspace, heev_work_doubles(n, kmax) entries
  cplx* tau;           // n entries
  double tol2;         // tol^2
  double floor_rel;    // rank floor on lam / lam_1
  int max_bond;
  int estart;          // filled by the launcher: prefix sum of kmax (eigenpair task index)
  int bstart;          // filled by the launcher: first back-transform block of this problem
  const int* exp2;     // may be null: A was formed from data scaled by 2^-e (pow2_normalize);
                       // the returned eigenvalues and discarded weight are scaled by 2^(2e)
  const int* skip;     // may be null: *skip != 0 (set on the device by chol_certify) = the
                       // exact-factor shortcut took this compress: every stage skips it, and
                       // k = kmax, w = 0 are written (lam / Vt are left unset)
};
size_t heev_work_doubles(int n, int kmax);
size_t heev_smem_bytes(int n, int kmax);
int heev_max_n();
int heev_small_n();   // Grams up to this order take the one-launch Jacobi kernel

// In-place lower Cholesky A + s I = L L^H of an n x n Hermitian matrix (full storage, ld = lda;
// s = shift_rel * max diag, 0 by default: the shifted first pass of CholeskyQR3);
// the strict upper triangle is zeroed.  info = 0 or j+1 at the first pivot <= rel_tol * max diag.
struct PotrfProblem {
  cplx* A;
  long long lda;
  int n;
  int pad_;
  int* info;
  double rel_tol;
  double shift_rel;
};

// potrf then trtri of the same matrix (Linv = L^{-1} of A + s I = L L^H); one fused launch for
// orders <= 64 (the factor stays in shared memory), the blocked pair otherwise.  A receives L
// when write_l (always for the blocked pair).  Linv is unspecified when info != 0.
struct PotriProblem {
  cplx* A;
  long long lda;
  int n;
  int write_l;
  int* info;
  double rel_tol;
  double shift_rel;
  cplx* Linv;
};

// Linv = L^{-1} (n x n lower, full storage, upper zeroed).
struct TrtriProblem {
  const cplx* L;
  cplx* Linv;
  long long ld;
  int n;
  int pad_;
};

// Exact-factor shortcut of an untruncated compress ("G = M^dagger M,
// which is a Cholesky decomposition of G"): with L L^H = W (potrf of a copy of the Gram W) and
// Li = L^{-1} (trtri), lambda_min(W) >= 1 / ||Li||_F^2 and lambda_1(W) <= tr W, so
// 1 / (||Li||_F^2 tr W) >= thresh certifies that every eigenvalue passes the rank floor and
// the eigensolver would keep all of them.  *skip = (info == 0 && certified).
struct CertProblem {
  const cplx* W;       // the Gram (n x n, ld n; its diagonal is read)
  const cplx* Li;      // L^{-1} (n x n lower, ld n)
  const int* info;     // potrf status of the copy
  int* skip;
  int n;
  int pad_;
  double thresh;
};
// Factor of a certified compress, written over the eigensolver route's output when *skip:
//   mode 0 (G route, W = X^H X = L L^H):  F = L^H  (n x n upper; F^H F = W exactly);
//   mode 1 (K route, m <= max_bond):      F = X    (m x n; F^H F = X^H X trivially).
struct ExactFactorProblem {
  const cplx* src;     // mode 0: L (n x n lower, ld cols); mode 1: X (rows x cols)
  cplx* F;             // rows x cols
  const int* skip;
  const int* exp2;     // mode 0, may be null: W was formed from X scaled by 2^-e, F is scaled by 2^e
  int rows, cols;
  int mode;
  int pad_;
};

// G-route factor F[t*ldf + c] = sqrt(max(lam_t,0)) * conj(Vt[t*n + c]), t < kmax, c < n.
struct ScaleRowsProblem {
  const cplx* Vt;
  const double* lam;
  cplx* F;
  int kmax;
  int n;
  long long start;
};

// Copies a host array to device memory, stream-ordered before the next launch; the returned
// device pointer stays valid until the owner's next host synchronisation.
struct Stager {
  virtual void* put(const void* host, size_t bytes) = 0;
  // Two-phase staging without an intermediate host copy: reserve() returns a host buffer of
  // `bytes` to fill, commit() enqueues its copy and returns the device pointer.  The default
  // goes through put().
  virtual void* reserve(size_t bytes) {
    tmp_.resize(bytes);
    return tmp_.data();
  }
  virtual void* commit(void* host, size_t bytes) { return put(host, bytes); }
  virtual void epoch() {}   // after a full stream synchronisation
  virtual ~Stager() {}
 private:
  std::vector<char> tmp_;
};

// Launchers fill the scheduling fields of the host problems, stage them, and launch.
// family: the ttn_profile family the launch set is timed under
void launch_gemm(GemmProblem* h, int n, Stager& st, cudaStream_t s, Scratch* ws = nullptr, const char* family = "zgemm");
void launch_permute(PermProblem* h, int n, Stager& st, cudaStream_t s);
// values_ready (optional) is called once the ranks (k_out) and discarded weights (w_out) are
// final in stream order -- before the eigenvector stages are enqueued -- so a caller can start
// reading them while the vectors are still being computed.
// ws (optional): workspace for the blocked (WY) back-transform on the GEMM kernel
void launch_heev(HeevProblem* h, int n, Stager& st, cudaStream_t s,
                 const std::function<void()>& values_ready = std::function<void()>(), Scratch* ws = nullptr);
void launch_potrf(PotrfProblem* h, int n, Stager& st, cudaStream_t s);
struct PotriProblem;
void launch_potri(PotriProblem* h, int n, Stager& st, cudaStream_t s);
void launch_chol_certify(CertProblem* h, int n, Stager& st, cudaStream_t s);
void launch_exact_factor(ExactFactorProblem* h, int n, Stager& st, cudaStream_t s);
void launch_trtri(TrtriProblem* h, int n, Stager& st, cudaStream_t s);
void launch_scale_rows(ScaleRowsProblem* h, int n, Stager& st, cudaStream_t s);
// out[j] = sum_i |x_j[i]|^2 of n device vectors
struct SumsqProblem { const cplx* x; long long len; double* out; };
void launch_sumsq(SumsqProblem* h, int n, Stager& st, cudaStream_t s);
void launch_fill(cplx* p, long long n, cplx v, cudaStream_t s);
// Householder QR of a tall m x k matrix A (ld k, destroyed) -> thin Q (m x k, ld k).
struct GeqrProblem { cplx* A; cplx* Q; cplx* tau; int m; int k; };
void launch_geqr_q(GeqrProblem* h, int n, Stager& st, cudaStream_t s);
// P[i*ld + j] = (i == j) for i < m, j < ncols, grouped
struct EyeProblem { cplx* p; int m; int ncols; long long start; };
void launch_eye(EyeProblem* h, int n, Stager& st, cudaStream_t s);

// Exact power-of-two range control (PAPER.md's CBC is scale covariant, pin P12): Grams and
// CholeskyQR square their inputs, so data whose largest entry is beyond 2^+-200 (positive-bias
// random networks reach 1e80) is scaled by 2^-e before the square and back after.
// e is the largest binary exponent of the problem's entries, kept in *exp (device);
// pow2_effective(e) = 0 when no scaling is needed (then the data is untouched).
struct Pow2Problem { cplx* x; long long len; int* exp; };
void launch_pow2_normalize(Pow2Problem* h, int n, Stager& st, cudaStream_t s);   // x *= 2^-e
void launch_pow2_restore(Pow2Problem* h, int n, Stager& st, cudaStream_t s);     // x *= 2^+e
// x *= 2^-e with *exp already holding the maximum exponent (the producing GEMM's exp_out)
void launch_pow2_apply(Pow2Problem* h, int n, Stager& st, cudaStream_t s);
// *exp = "no data yet" for n contiguous exponents
void pow2_reset(int* exp, int n, cudaStream_t s);
__host__ __device__ inline int pow2_effective(int e) { return (e < -2000 || (e > -100 && e < 100)) ? 0 : e; }

// cudaFuncSetAttribute on the CURRENT device, once per (device, function, attribute) and only
// ever raising the value (thread-safe): a kernel attribute is per device, and contexts on
// several devices or worker threads may launch the same kernel.
void func_attr(const void* func, cudaFuncAttribute attr, int value);
template <typename F>
inline void func_smem(F* func, size_t bytes) {
  func_attr(reinterpret_cast<const void*>(func), cudaFuncAttributeMaxDynamicSharedMemorySize, (int)bytes);
}

// Speculative ranks (cbc.cpp): the host plans with k = kmax and checks on the device.
// One thread per compress: flag |= 1 if the eigensolver's rank differs from kmax, |= 2 if the
// discarded weight is not finite; wacc[inst] += w, xacc[inst] += skip (exact-factor count).
struct SpecCheck { const int* k; const double* w; const int* skip; int kmax; int inst; };
void launch_spec_check(SpecCheck* h, int n, double* wacc, int* xacc, int* flag, Stager& st, cudaStream_t s);
// flag |= bit if any of info[0..n) is non-zero (CholeskyQR pivot failures)
void launch_flag_nonzero(const int* info, int n, int* flag, int bit, cudaStream_t s);

// Counters of kernel launches issued by this library (for the bench's gpu_launches claim).
long long launch_count();
void count_launch();
void add_launches(long long delta);   // graph replays (+ nodes) and captures (- recorded launches)

}  // namespace tcbc
