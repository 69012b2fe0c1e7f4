// solver.cuh — workspace layout and driver entry shared by api.cu and solver.cu.
#pragma once
#include "common.cuh"

namespace scsf {

struct SolveWS {
  int64_t n = 0, ldv = 0;
  int b = 0;
  double *V = nullptr, *W = nullptr, *T1 = nullptr, *T2 = nullptr;   // n x b blocks (ld ldv)
  double *S = nullptr, *Rinv = nullptr, *Zs = nullptr, *Zwork = nullptr, *Gwork = nullptr;  // b x b
  double *C = nullptr, *P = nullptr;                                   // projections, split-K partials
  double *theta = nullptr, *theta_sorted = nullptr, *res = nullptr, *wn = nullptr, *rel = nullptr;
  double* fp = nullptr;                                                // filter (lambda, c, e)
  int* perm = nullptr;
  Ctrl* ctrl = nullptr;
  unsigned long long* gersh = nullptr;
};

size_t solve_ws_bytes(const scsf_ops* ops, int L, int nex);
int carve_solve_ws(const scsf_ops* ops, int L, int nex, void* ws, size_t ws_bytes, SolveWS& w);
int solve_core(const scsf_ops* ops, int op, int L, int nex, int degree, double tol, int max_iter,
               bool warm, bool orthonormalize, uint64_t seed, SolveWS& w, scsf_stats* st, cudaStream_t s);

}  // namespace scsf
