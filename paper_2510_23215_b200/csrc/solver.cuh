// solver.cuh — workspace layout and driver entry shared by api.cu and solver.cu.
#pragma once
#include "common.cuh"

namespace scsf {

struct Comm;

// Row partition of one operator over ranks: this rank owns
// grid rows [y0, y1) of a 2-D operator; comm carries the exchanges.
struct DistCtx {
  Comm* comm = nullptr;
  int y0 = 0, y1 = 0;
};

struct SolveWS {
  int64_t n = 0, ldv = 0;
  int64_t n_glob = 0, goff = 0;                                        // global size, global index of local row 0
  Comm* comm = nullptr;                                                // non-null: row-partitioned solve
  int nx = 0;
  double *send_lo = nullptr, *send_hi = nullptr, *recv_lo = nullptr, *recv_hi = nullptr;  // [b][nx] halos
  double *colbuf = nullptr, *colgath = nullptr;                        // sign convention (3 b, world 3 b)
  double* coef_buf = nullptr;                                          // this operator's arrays (graph replay)
  int* deg = nullptr;                                                  // per-column filter degree
  int* deg_on = nullptr;                                               // == deg when the adaptive degree is on
  int mdeg = 20;
  int cap_on = 1;       // k_lock applies the degree cap (R28); 0 for the RR of a random start
  int b = 0;
  double *V = nullptr, *W = nullptr, *T1 = nullptr, *T2 = nullptr;   // n x b blocks (ld ldv)
  double *S = nullptr, *Rinv = nullptr, *Zs = nullptr, *Zwork = nullptr, *Gwork = nullptr;  // b x b
  double *C = nullptr, *P = nullptr;                                   // projections, split-K partials
  double *C2 = nullptr, *Tb = nullptr, *Mb = nullptr;                  // [S2 | H] (b x 2b), b x b products
  double *theta = nullptr, *theta_sorted = nullptr, *res = nullptr, *wn = nullptr, *rel = nullptr;
  double* fp = nullptr;                                                // filter (lambda, c, e)
  int* perm = nullptr;
  Ctrl* ctrl = nullptr;
  unsigned long long* gersh = nullptr;
};

size_t solve_ws_bytes(const scsf_ops* ops, int L, int nex, const DistCtx* dist = nullptr);
int carve_solve_ws(const scsf_ops* ops, int L, int nex, void* ws, size_t ws_bytes, SolveWS& w,
                   const DistCtx* dist = nullptr);
int solve_core(const scsf_ops* ops, int op, int L, int nex, int degree, double tol, int max_iter,
               bool warm, bool orthonormalize, uint64_t seed, SolveWS& w, scsf_stats* st, cudaStream_t s);

}  // namespace scsf
