// Microbenchmark + check of the grouped DMMA zgemm (libttncbc's csrc/gemm.cu) against cuBLAS
// zgemm on the GEMM shapes that dominate BASELINE configs 3 and 4.  Tool, not product code.
//   nvcc ... tools/gemm_bench.cu paper_2601_19650_b200/build/{gemm,prof,misc}.o -lcublas
#include <cublas_v2.h>
#include <cuda_runtime.h>
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <vector>
#include "../paper_2601_19650_b200/csrc/kernels.h"

using namespace tcbc;

struct SimpleStager : Stager {
  char* d = nullptr;
  size_t off = 0, cap = 64 << 20;
  cudaStream_t s;
  explicit SimpleStager(cudaStream_t st) : s(st) { cudaMalloc(&d, cap); }
  void* put(const void* h, size_t b) override {
    if (off + b > cap) off = 0;
    void* p = d + off;
    cudaMemcpyAsync(p, h, b, cudaMemcpyHostToDevice, s);
    cudaStreamSynchronize(s);
    off += (b + 255) & ~size_t(255);
    return p;
  }
};

struct Case { const char* name; int M, N, K, batch, opA, opB; int sym = 0; };
struct DevScratch : Scratch {   // stream-ordered reuse of one buffer (launches are serialised)
  char* buf = nullptr;
  size_t cap = 512ull << 20, off = 0;
  DevScratch() { cudaMalloc(&buf, cap); }
  ~DevScratch() { cudaFree(buf); }
  void* get(size_t b) override { if (off + b > cap) off = 0; void* p = buf + off; off += (b + 255) & ~size_t(255); return p; }
  void release() { off = 0; }
};

int main(int argc, char** argv) {
  cudaStream_t s;
  cudaStreamCreate(&s);
  cublasHandle_t hb;
  cublasCreate(&hb);
  cublasSetStream(hb, s);
  SimpleStager st(s);
  // opA/opB: 0 N, 3 conj-transpose, 1 transpose  (A stored M x K row-major for N)
  std::vector<Case> cases = {
      {"cfg3 contraction 12288x32x192 x64", 12288, 32, 192, 64, 0, 0},
      {"cfg3 contraction 3072x32x192 x64", 3072, 32, 192, 64, 0, 0},
      {"cfg3 gram 192x192x2048 (X^H X) x64", 192, 192, 2048, 64, 3, 0},
      {"cfg3 2048x192x32 x64", 2048, 192, 32, 64, 0, 0},
      {"cfg3 S 2048x32x192 x64", 2048, 32, 192, 64, 0, 1},
      {"cfg3 R 32x192x2048 x64", 32, 192, 2048, 64, 3, 0},
      {"cfg2 128x512x64", 128, 512, 64, 1, 0, 0},
      {"cfg4 2048x2048x16384", 2048, 2048, 16384, 1, 0, 0},
      {"cfg4 gram 2048x2048x16384 (X^H X)", 2048, 2048, 16384, 1, 3, 0},
      {"cfg4 16384x2048x128", 16384, 2048, 128, 1, 0, 0},
      {"cfg4 128x2048x16384 (Q^H Z)", 128, 2048, 16384, 1, 3, 0},
      {"square 4096", 4096, 4096, 4096, 1, 0, 0},
      {"herk cfg4 gram 2048x2048x16384 sym", 2048, 2048, 16384, 1, 3, 0, 1},
      {"herk cfg3 gram 192x192x2048 sym x64", 192, 192, 2048, 64, 3, 0, 1},
      {"herk chfsi 192x192x2048 sym x4", 192, 192, 2048, 4, 3, 0, 1},
  };
  int reps = argc > 1 ? atoi(argv[1]) : 5;
  printf("[");
  bool first = true;
  const char* filt = argc > 2 ? argv[2] : nullptr;
  for (auto& c : cases) {
    if (filt && !strstr(c.name, filt)) continue;
    const size_t szA = (size_t)c.M * c.K, szB = (size_t)c.K * c.N, szC = (size_t)c.M * c.N;
    cplx *A, *B, *C, *Cref;
    cudaMalloc(&A, szA * 16 * c.batch);
    cudaMalloc(&B, szB * 16 * c.batch);
    cudaMalloc(&C, szC * 16 * c.batch);
    cudaMalloc(&Cref, szC * 16 * c.batch);
    {
      std::vector<cplx> h(std::max(szA, szB) * c.batch);
      srand(1);
      for (auto& v : h) { v.x = rand() / (double)RAND_MAX - 0.5; v.y = rand() / (double)RAND_MAX - 0.5; }
      cudaMemcpy(A, h.data(), szA * 16 * c.batch, cudaMemcpyHostToDevice);
      cudaMemcpy(B, h.data(), szB * 16 * c.batch, cudaMemcpyHostToDevice);
    }
    std::vector<GemmProblem> probs(c.batch);
    for (int b = 0; b < c.batch; ++b) {
      GemmProblem& g = probs[b];
      g = GemmProblem{};
      g.A = A + szA * b; g.B = B + szB * b; g.C = C + szC * b;
      g.M = c.M; g.N = c.N; g.K = c.K;
      const long long lda = (c.opA & 1) ? c.M : c.K, ldb = (c.opB & 1) ? c.K : c.N;
      gemm_from_ops(g, c.opA, lda, c.opB, ldb, c.N);
      g.alpha = make_double2(1, 0);
      g.beta = make_double2(0, 0);
      g.sym = c.sym;
    }
    DevScratch scr;
    // reference: row-major C = op(A) op(B)  <=>  col-major C^T = op(B)^T op(A)^T
    auto cop = [](int op) { return op == 0 ? CUBLAS_OP_N : op == 1 ? CUBLAS_OP_T : CUBLAS_OP_C; };
    cuDoubleComplex one = make_cuDoubleComplex(1, 0), zero = make_cuDoubleComplex(0, 0);
    auto ref = [&]() {
      for (int b = 0; b < c.batch; ++b)
        cublasZgemm(hb, cop(c.opB), cop(c.opA), c.N, c.M, c.K, &one,
                    (const cuDoubleComplex*)(B + szB * b), (c.opB & 1) ? c.K : c.N,
                    (const cuDoubleComplex*)(A + szA * b), (c.opA & 1) ? c.M : c.K, &zero,
                    (cuDoubleComplex*)(Cref + szC * b), c.N);
    };
    ref();
    std::vector<GemmProblem> tmp = probs;
    launch_gemm(tmp.data(), c.batch, st, s, &scr);
    cudaStreamSynchronize(s);
    std::vector<cplx> h1(szC * c.batch), h2(szC * c.batch);
    cudaMemcpy(h1.data(), C, szC * 16 * c.batch, cudaMemcpyDeviceToHost);
    cudaMemcpy(h2.data(), Cref, szC * 16 * c.batch, cudaMemcpyDeviceToHost);
    double num = 0, den = 0;
    for (size_t i = 0; i < h1.size(); ++i) {
      const double dx = h1[i].x - h2[i].x, dy = h1[i].y - h2[i].y;
      num += dx * dx + dy * dy;
      den += h2[i].x * h2[i].x + h2[i].y * h2[i].y;
    }
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0);
    cudaEventCreate(&e1);
    float ms = 0, msr = 0;
    for (int w = 0; w < 2; ++w) { tmp = probs; launch_gemm(tmp.data(), c.batch, st, s, &scr); }
    cudaEventRecord(e0, s);
    for (int r = 0; r < reps; ++r) { tmp = probs; launch_gemm(tmp.data(), c.batch, st, s, &scr); }
    cudaEventRecord(e1, s);
    cudaEventSynchronize(e1);
    cudaEventElapsedTime(&ms, e0, e1);
    ref();
    cudaEventRecord(e0, s);
    for (int r = 0; r < reps; ++r) ref();
    cudaEventRecord(e1, s);
    cudaEventSynchronize(e1);
    cudaEventElapsedTime(&msr, e0, e1);
    const double fl = (c.sym ? 4.0 * c.M * (c.M + 1.0) : 8.0 * c.M * c.N) * (double)c.K * c.batch;
    cudaDeviceSynchronize();
    scr.release();
    printf("%s\n {\"case\": \"%s\", \"rel_err\": %.3e, \"ms\": %.4f, \"tflops\": %.2f, \"cublas_ms\": %.4f, "
           "\"cublas_tflops\": %.2f}",
           first ? "" : ",", c.name, std::sqrt(num / den), ms / reps, fl / (ms / reps) / 1e9, msr / reps,
           fl / (msr / reps) / 1e9);
    first = false;
    cudaFree(A); cudaFree(B); cudaFree(C); cudaFree(Cref);
  }
  printf("\n]\n");
  printf("err: %s\n", cudaGetErrorString(cudaGetLastError()));
  return 0;
}
