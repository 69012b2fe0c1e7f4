// gemm_bench.cu — back-to-back timing of the DMMA tiles (k_dense.cu) at the solver's shapes,
// CUDA events around R launches (no per-call synchronisation), TF/s against the 37 TF DMMA peak.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -I. -o /tmp/gemm_bench tools/gemm_bench.cu
#include <cstdarg>
#include <cstdlib>
#include <cstdio>
#include <vector>

#include "../paper_2510_23215_b200/csrc/k_dense.cu"

namespace scsf {
void set_error(const char* fmt, ...) {
  va_list ap;
  va_start(ap, fmt);
  vfprintf(stderr, fmt, ap);
  va_end(ap);
  fprintf(stderr, "\n");
}
void count_launch(int) {}
void set_capturing(bool) {}
bool debug_sync() { return false; }
}  // namespace scsf

using namespace scsf;

int main() {
  const int64_t n = getenv("GB_N") ? atoll(getenv("GB_N")) : 10000;
  const int64_t ld = (n + 31) / 32 * 32;
  const int R = 50;
  double *X, *Y, *M, *C, *P, *O;
  cudaMalloc(&X, ld * 400 * 8);
  cudaMalloc(&Y, ld * 400 * 8);
  cudaMalloc(&O, ld * 400 * 8);
  const int BIG = getenv("GB_B") ? atoi(getenv("GB_B")) : 0;
  cudaMalloc(&M, 400 * 400 * 8);
  cudaMalloc(&C, 400 * 800 * 8);
  cudaMalloc(&P, tn_partial_doubles(n, 400, 400) * 8 + 1024);
  cudaMemset(X, 0, ld * 400 * 8);
  cudaMemset(Y, 0, ld * 400 * 8);
  cudaMemset(M, 0, 400 * 400 * 8);
  cudaStream_t s;
  cudaStreamCreate(&s);
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  struct Case { const char* what; int b1, b2, kind; };   // kind 0 NN, 1 NN tri, 2 TN upper, 3 TN full, 4 TN dual
  std::vector<Case> cases = {{"NN  n x 120 . 120 x 120", 120, 120, 0}, {"NN  tri 120", 120, 120, 1},
                             {"NN  n x 80 . 80 x 40 (BCGS)", 80, 40, 0}, {"TN  upper 120", 120, 120, 2},
                             {"TN  80 x 40 (BCGS)", 80, 40, 3}, {"TN  dual 120", 120, 120, 4},
                             {"NN  n x 56 . 56 x 56", 56, 56, 0}, {"TN  upper 56", 56, 56, 2}};
  if (BIG) cases = {{"NN  n x B . B x B", BIG, BIG, 0}, {"NN  tri B", BIG, BIG, 1}, {"TN  upper B", BIG, BIG, 2},
                    {"TN  dual B", BIG, BIG, 4}};
  for (auto& c : cases) {
    double flops = 2.0 * n * c.b1 * c.b2;
    if (c.kind == 1 || c.kind == 2) flops *= 0.5;
    for (int rep = 0; rep < 2; ++rep) {
      cudaEventRecord(e0, s);
      for (int r = 0; r < R; ++r) {
        if (c.kind <= 1) gemm_nn_ex(X, ld, n, c.b1, M, c.b1, c.b2, 1.0, 0.0, O, ld, c.kind, s);
        else if (c.kind <= 3) gemm_tn(X, ld, c.b1, Y, ld, c.b2, n, 1.0, c.kind == 2, C, c.b1, P, s);
        else gemm_tn_dual(X, ld, X, Y, ld, c.b1, n, C, c.b1, P, s);
      }
      cudaEventRecord(e1, s);
      cudaEventSynchronize(e1);
      float ms;
      cudaEventElapsedTime(&ms, e0, e1);
      const double us = 1000.0 * ms / R;
      if (c.kind == 4) flops = 2.0 * n * c.b1 * c.b2;   // two upper products
      if (rep) printf("%-32s %8.2f us  %6.2f TF/s\n", c.what, us, flops / us / 1e6);
    }
  }
  printf("%s\n", cudaGetErrorString(cudaGetLastError()));
  return 0;
}
