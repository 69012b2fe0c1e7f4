// solver.cu — ChFSI driver, Alg. 3, and the SCSF chain
// (Fig. 2 d1-d3; warm start P:270-277).
//
// Block layout: V, W = AV, T1, T2 are n x b column-major blocks (ld = n
// rounded up to 32).  Columns [0, kL) of V are locked Ritz vectors (ascending
// Ritz values), columns [kL, b) are active.  Per outer iteration:
//   1. filter   Y_m = C_m(V_act)             Alg. 1, m stencil steps
//   2. BCGS2    Y <- Y - V_L (V_L^T Y), x2   orthogonality to locked (R14)
//   3. CholQR2  Y = Q R, two passes          l. 4 (R13)
//   4. RR       W = AQ, G = Q^T W, G = Z T Z^T, V_act <- QZ, W <- WZ   ll. 5-6
//   5. resid    ||W_j - t_j V_j|| / ||W_j||
//   6. lock     contiguous run from kL (R15); next (lambda, c, e) (R9)
// The host reads the device control block once per iteration (kL drives the
// launch shapes of the next iteration).
#include "solver.cuh"
#include "comm.cuh"

#include <algorithm>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <memory>
#include <mutex>
#include <unordered_map>
#include <utility>
#include <vector>

namespace scsf {

// kernels (k_*.cu)
int stencil_impl(const scsf_ops* ops, int op, const double* X, const double* Xp, double* Out,
                 int64_t ldv, int ncols, const double* fp, int step, cudaStream_t s, const int* deg = nullptr);
bool stencil_v4_ok(const scsf_ops* ops, int64_t ldv);
bool filter_resident_ok(const scsf_ops* ops);
int filter_resident_impl(const scsf_ops* ops, int op, const double* X, double* Out, int64_t ldv, int ncols,
                         const double* fp, int m, cudaStream_t s, const int* deg = nullptr);
int stencil_resid_impl(const scsf_ops* ops, int op, const double* V, int64_t ldv, int ncols, const double* theta,
                       double* res, double* wn, double* P, cudaStream_t s, bool* done);
int resid_impl(const double* V, const double* W, int64_t ldv, int64_t n, int ncols,
               const double* theta, double* res, double* wn, cudaStream_t s);
int gershgorin_impl(const scsf_ops* ops, int op, unsigned long long* out, cudaStream_t s);
int gemm_tn(const double* X, int64_t ldx, int b1, const double* Y, int64_t ldy, int b2, int64_t n,
            double alpha, int sym, double* C, int64_t ldc, double* P, cudaStream_t s);
int gemm_nn(const double* X, int64_t ldx, int64_t n, int b1, const double* M, int64_t ldm, int b2,
            double alpha, double beta, double* Out, int64_t ldo, cudaStream_t s);
int gemm_nn_ex(const double* X, int64_t ldx, int64_t n, int b1, const double* M, int64_t ldm, int b2,
               double alpha, double beta, double* Out, int64_t ldo, int tri, cudaStream_t s);
size_t tn_partial_doubles(int64_t n, int b1, int b2);
size_t resid_partial_doubles(int64_t ldv, int ncols);
int gemm_tn_dual(const double* X, int64_t ldx, const double* Y1, const double* Y2, int64_t ldy, int b, int64_t n,
                 double* C, int64_t ldc, double* P, cudaStream_t s);
int symm_upper_impl(double* A, int b, int64_t ld, cudaStream_t s);
size_t small_scratch_doubles(int b);
int chol_inv_impl(const double* S, int64_t lds, int b, int64_t nrows, double* Rinv, double* scratch,
                  Ctrl* ctrl, cudaStream_t s);
int jacobi_impl(const double* G, int64_t ldg, int b, double* scratchG, double* Z, double* theta,
                double* Zout, Ctrl* ctrl, cudaStream_t s);
int lock_impl(const double* theta, const double* res, const double* wn, double* rel, int b, int L,
              double tol, Ctrl* ctrl, double* fp, int* deg, int mdeg, int cap_on, cudaStream_t s);
int ctrl_init_impl(Ctrl* ctrl, const unsigned long long* gersh, cudaStream_t s);
int bounds_from_theta_impl(const double* theta_sorted, int b, Ctrl* ctrl, double* fp, int mdeg, cudaStream_t s);
int step_table_impl(double* fp, int m, cudaStream_t s);
int rand_block_impl(double* V, int64_t ldv, int64_t n, int ncols, uint64_t seed, int64_t goff, cudaStream_t s);
int pack_rows_impl(const double* X, int64_t ldv, int64_t n_loc, int nx, int ncols, double* send_lo,
                   double* send_hi, cudaStream_t s);
int stencil_slab_impl(const scsf_ops* ops, int op, int64_t goff, int64_t n_loc, const double* X, const double* Xp,
                      double* Out, int64_t ldv, int ncols, const double* ghost_lo, const double* ghost_hi,
                      const double* fp, int step, cudaStream_t s, int part = 0, const int* deg = nullptr);
int colmax_local_impl(const double* V, int64_t ldv, int64_t n, const int* perm, int b, int64_t goff, double* colbuf,
                      cudaStream_t s);
int sort_theta_impl(const double* theta, const double* rel, int b, int L, int* perm, double* theta_sorted,
                    Ctrl* ctrl, cudaStream_t s);
int sign_apply_impl(const double* V, int64_t ldv, int64_t n, const int* perm, const double* gath, int world, int b,
                    double* Out, int64_t ldo, cudaStream_t s);
int finalize_impl(const double* theta, const double* rel, int b, int L, int* perm, double* theta_sorted,
                  const double* V, int64_t ldv, int64_t n, double* Out, int64_t ldo, Ctrl* ctrl,
                  cudaStream_t s);

static void carve(Arena& a, SolveWS& w, const scsf_ops* ops, int b, const DistCtx* dist) {
  const int64_t n_glob = (int64_t)ops->nx * ops->ny * ops->nz;
  int64_t n = n_glob;
  w.n_glob = n_glob;
  w.goff = 0;
  w.comm = nullptr;
  w.nx = ops->nx;
  if (dist && dist->comm) {
    n = (int64_t)ops->nx * (dist->y1 - dist->y0);
    w.goff = (int64_t)ops->nx * dist->y0;
    w.comm = dist->comm;
  }
  w.n = n;
  w.b = b;
  w.ldv = round_up(n, 32);
  w.V = a.take<double>(w.ldv * b);
  w.W = a.take<double>(w.ldv * b);
  w.T1 = a.take<double>(w.ldv * b);
  w.T2 = a.take<double>(w.ldv * b);
  const int64_t bb = (int64_t)b * b;
  w.S = a.take<double>(bb);
  w.Rinv = a.take<double>(bb);
  w.Zs = a.take<double>(bb);
  w.Zwork = a.take<double>(bb);
  w.Gwork = a.take<double>((int64_t)small_scratch_doubles(b));
  w.C = a.take<double>(bb);
  w.C2 = a.take<double>(2 * bb);
  w.Tb = a.take<double>(bb);
  w.Mb = a.take<double>(bb);
  // split-K partials of the TN products, and the fused residual pass's per-CTA partials
  w.P = a.take<double>((int64_t)std::max(tn_partial_doubles(n, b, b), resid_partial_doubles(w.ldv, b)));
  w.theta = a.take<double>(b);
  w.theta_sorted = a.take<double>(b);
  w.res = a.take<double>(b);
  w.wn = a.take<double>(b);
  w.rel = a.take<double>(b);
  w.fp = a.take<double>(FP_DOUBLES);
  w.perm = a.take<int>(b);
  w.ctrl = a.take<Ctrl>(1);
  w.gersh = a.take<unsigned long long>(1);
  w.coef_buf = a.take<double>((int64_t)ncoef(ops) * ops->ld);
  w.deg = a.take<int>(b);
  if (dist && dist->comm) {
    const int64_t hb = (int64_t)b * ops->nx;
    w.send_lo = a.take<double>(hb);
    w.send_hi = a.take<double>(hb);
    w.recv_lo = a.take<double>(hb);
    w.recv_hi = a.take<double>(hb);
    w.colbuf = a.take<double>(3 * (int64_t)b);
    w.colgath = a.take<double>(3 * (int64_t)b * dist->comm->world);
  }
}

size_t solve_ws_bytes(const scsf_ops* ops, int L, int nex, const DistCtx* dist) {
  Arena a(nullptr, 0);
  SolveWS w;
  carve(a, w, ops, L + nex, dist);
  return a.off;
}

int carve_solve_ws(const scsf_ops* ops, int L, int nex, void* ws, size_t ws_bytes, SolveWS& w,
                   const DistCtx* dist) {
  Arena a(ws, ws_bytes);
  carve(a, w, ops, L + nex, dist);
  if (a.overflow || ws == nullptr) {
    set_error("workspace too small: need %zu bytes, got %zu", a.off, ws_bytes);
    return SCSF_ERR_WORKSPACE;
  }
  return SCSF_OK;
}

// ---- optional DGEMM timers (scsf_set_timing): CUDA events around every tall-skinny DGEMM
// tile launch of an iteration, summed after the iteration's control-block read; the flops are
// the algorithmic ones of the product (upper-triangle Grams count their unique entries)
static int g_timing = 0;
// kinds: 0 Gram (gram(): BCGS V_L^T F, CholQR Y^T Y), 1 triangular R^{-1} apply, 2 rotation (V Z, W Z),
// 3 dual Gram [Q1^T Q1 | Q1^T W1], 4 V <- Q1 M, 5 BCGS update F -= V_L C
constexpr int GT_KINDS = 6;
struct GemmTiming {
  std::vector<cudaEvent_t> ev;     // pairs (begin, end), reused
  std::vector<double> flops;
  std::vector<int> kind;
  size_t used = 0;
  double ms = 0.0, total_flops = 0.0;
  double kind_ms[GT_KINDS] = {0}, kind_flops[GT_KINDS] = {0};
};
static thread_local GemmTiming* t_gt = nullptr;
static int gt_begin(cudaStream_t s) {
  GemmTiming* g = t_gt;
  if (!g) return SCSF_OK;
  if (g->used + 2 > g->ev.size()) {
    for (int i = 0; i < 2; ++i) {
      cudaEvent_t e;
      SCSF_CUDA_CHECK(cudaEventCreate(&e));
      g->ev.push_back(e);
    }
  }
  SCSF_CUDA_CHECK(cudaEventRecord(g->ev[g->used], s));
  return SCSF_OK;
}
static int gt_end(cudaStream_t s, double flops, int kind) {
  GemmTiming* g = t_gt;
  if (!g) return SCSF_OK;
  SCSF_CUDA_CHECK(cudaEventRecord(g->ev[g->used + 1], s));
  if (g->flops.size() < g->ev.size() / 2) {
    g->flops.resize(g->ev.size() / 2);
    g->kind.resize(g->ev.size() / 2);
  }
  g->flops[g->used / 2] = flops;
  g->kind[g->used / 2] = kind;
  g->used += 2;
  return SCSF_OK;
}
// after a synchronisation that follows every recorded pair
static int gt_collect() {
  GemmTiming* g = t_gt;
  if (!g) return SCSF_OK;
  for (size_t i = 0; i < g->used; i += 2) {
    float ms = 0.f;
    SCSF_CUDA_CHECK(cudaEventElapsedTime(&ms, g->ev[i], g->ev[i + 1]));
    g->ms += ms;
    g->total_flops += g->flops[i / 2];
    g->kind_ms[g->kind[i / 2]] += ms;
    g->kind_flops[g->kind[i / 2]] += g->flops[i / 2];
  }
  g->used = 0;
  return SCSF_OK;
}

// ---- the exchange points of the row-partitioned solve (no-ops on one GPU) ----
// C = X^T Y summed over ranks (Gram / projection blocks, Alg. 3 ll. 4-5)
static int gram(SolveWS& w, const double* X, int b1, const double* Y, int b2, int sym, double* C,
                cudaStream_t s) {
  SCSF_TRY(gt_begin(s));
  SCSF_TRY(gemm_tn(X, w.ldv, b1, Y, w.ldv, b2, w.n, 1.0, sym, C, b1, w.P, s));
  SCSF_TRY(gt_end(s, sym ? (double)w.n * b1 * (b1 + 1) : 2.0 * w.n * b1 * b2, 0));
  if (w.comm) SCSF_TRY(w.comm->allreduce_sum(C, (size_t)b1 * b2, s));
  return SCSF_OK;
}

// One stencil application (filter step `step`, or A X when step < 0) on ncols columns.
// Row partition: the slab's boundary rows are packed and exchanged with the neighbours on a side
// stream while the interior rows (which need no ghost row) compute on the solver's stream; the
// first and last rows follow once the ghosts have landed (fork / join by events, capturable).
struct HaloStreams {
  cudaStream_t side = nullptr;
  cudaEvent_t packed = nullptr, landed = nullptr;
};
static int halo_streams(HaloStreams*& hs) {
  static thread_local HaloStreams t;
  if (!t.side) {
    SCSF_CUDA_CHECK(cudaStreamCreateWithFlags(&t.side, cudaStreamNonBlocking));
    SCSF_CUDA_CHECK(cudaEventCreateWithFlags(&t.packed, cudaEventDisableTiming));
    SCSF_CUDA_CHECK(cudaEventCreateWithFlags(&t.landed, cudaEventDisableTiming));
  }
  hs = &t;
  return SCSF_OK;
}
static bool halo_overlap() {                       // SCSF_HALO_OVERLAP=0: exchange, then one stencil launch
  static const int v = [] {            // thread-safe one-time read (chain worker threads)
    int v;
    const char* e = getenv("SCSF_HALO_OVERLAP");
    v = (e && e[0] == '0') ? 0 : 1;
    return v;
  }();
  return v == 1;
}
static int spmm(const scsf_ops* ops, int op, SolveWS& w, const double* X, const double* Xp, double* Out, int ncols,
                int step, cudaStream_t s, const int* deg = nullptr) {
  if (!w.comm) return stencil_impl(ops, op, X, Xp, Out, w.ldv, ncols, w.fp, step, s, deg);
  const double* glo = w.comm->rank > 0 ? w.recv_lo : nullptr;
  const double* ghi = w.comm->rank + 1 < w.comm->world ? w.recv_hi : nullptr;
  if (w.comm->world == 1)                          // one slab: no neighbour, no exchange
    return stencil_slab_impl(ops, op, w.goff, w.n, X, Xp, Out, w.ldv, ncols, glo, ghi, w.fp, step, s, 0, deg);
  SCSF_TRY(pack_rows_impl(X, w.ldv, w.n, w.nx, ncols, w.send_lo, w.send_hi, s));
  if (!halo_overlap()) {
    SCSF_TRY(w.comm->halo(w.send_lo, w.send_hi, w.recv_lo, w.recv_hi, (size_t)ncols * w.nx, s));
    return stencil_slab_impl(ops, op, w.goff, w.n, X, Xp, Out, w.ldv, ncols, glo, ghi, w.fp, step, s, 0, deg);
  }
  HaloStreams* hs;
  SCSF_TRY(halo_streams(hs));
  SCSF_CUDA_CHECK(cudaEventRecord(hs->packed, s));
  SCSF_CUDA_CHECK(cudaStreamWaitEvent(hs->side, hs->packed, 0));
  SCSF_TRY(w.comm->halo(w.send_lo, w.send_hi, w.recv_lo, w.recv_hi, (size_t)ncols * w.nx, hs->side));
  SCSF_CUDA_CHECK(cudaEventRecord(hs->landed, hs->side));
  SCSF_TRY(stencil_slab_impl(ops, op, w.goff, w.n, X, Xp, Out, w.ldv, ncols, glo, ghi, w.fp, step, s, 1, deg));
  SCSF_CUDA_CHECK(cudaStreamWaitEvent(s, hs->landed, 0));
  return stencil_slab_impl(ops, op, w.goff, w.n, X, Xp, Out, w.ldv, ncols, glo, ghi, w.fp, step, s, 2, deg);
}

// Q = CholQR pass on columns [0, ncols) of Y (in place, or into Out when Out != Y).
static int cholqr_pass(SolveWS& w, double* Y, double* Out, int ncols, cudaStream_t s) {
  SCSF_TRY(gram(w, Y, ncols, Y, ncols, 1, w.S, s));
  SCSF_TRY(chol_inv_impl(w.S, ncols, ncols, w.n_glob, w.Rinv, w.Gwork, w.ctrl, s));
  SCSF_TRY(gt_begin(s));
  SCSF_TRY(gemm_nn_ex(Y, w.ldv, w.n, ncols, w.Rinv, ncols, ncols, 1.0, 0.0, Out, w.ldv, 1, s));
  SCSF_TRY(gt_end(s, (double)w.n * ncols * (ncols + 1), 1));                  // triangular R^{-1}
  return SCSF_OK;
}

// Rayleigh-Ritz on block columns [k0, b): W = AV, G = V^T W, rotate V and W,
// residual norms, locking.
static int rayleigh_ritz(const scsf_ops* ops, int op, SolveWS& w, int k0, int L, double tol,
                         int64_t& spmm_cols, cudaStream_t s) {
  const int ba = w.b - k0;
  double* Va = w.V + (int64_t)k0 * w.ldv;
  double* Wa = w.W + (int64_t)k0 * w.ldv;
  SCSF_TRY(spmm(ops, op, w, Va, nullptr, Wa, ba, -1, s));
  spmm_cols += ba;
  SCSF_TRY(gram(w, Va, ba, Wa, ba, 1, w.S, s));
  SCSF_TRY(jacobi_impl(w.S, ba, ba, w.Gwork, w.Zwork, w.theta + k0, w.Zs, w.ctrl, s));
  SCSF_TRY(gt_begin(s));
  SCSF_TRY(gemm_nn(Va, w.ldv, w.n, ba, w.Zs, ba, ba, 1.0, 0.0, Va, w.ldv, s));
  SCSF_TRY(gemm_nn(Wa, w.ldv, w.n, ba, w.Zs, ba, ba, 1.0, 0.0, Wa, w.ldv, s));
  SCSF_TRY(gt_end(s, 4.0 * w.n * ba * ba, 2));
  SCSF_TRY(resid_impl(Va, Wa, w.ldv, w.n, ba, w.theta + k0, w.res + k0, w.wn + k0, s));
  if (w.comm) {
    SCSF_TRY(w.comm->allreduce_sum(w.res + k0, ba, s));
    SCSF_TRY(w.comm->allreduce_sum(w.wn + k0, ba, s));
  }
  SCSF_TRY(lock_impl(w.theta, w.res, w.wn, w.rel, w.b, L, tol, w.ctrl, w.fp, w.deg_on, w.mdeg, w.cap_on, s));
  return SCSF_OK;
}

// Rayleigh-Ritz with CholQR's second pass folded in.  On entry V[:, k0:b) holds
// Q1 = F R1^{-1} (first CholQR pass).  With W1 = A Q1, one pass over Q1 gives
// S2 = Q1^T Q1 and H = Q1^T W1; then R2 = chol(S2), G = R2^{-T} H R2^{-1}
// (the Rayleigh quotient of Q2 = Q1 R2^{-1}), G = Z Theta Z^T, M = R2^{-1} Z and
// V <- Q1 M, W <- W1 M (= A V).  Same result as CholQR2 followed by the
// Rayleigh-Ritz step (Q2 Z = Q1 (R2^{-1} Z)); it saves one n x b pass (the
// second triangular apply) and fuses two Gram passes into one.  The b x b
// products are replicated (identical on every rank of a row partition).
static bool fused_resid() {                         // SCSF_FUSED_RESID=0: W = A V then k_resid
  static const int v = [] {            // thread-safe one-time read (chain worker threads)
    int v;
    const char* e = getenv("SCSF_FUSED_RESID");
    v = (e && e[0] == '0') ? 0 : 1;
    return v;
  }();
  return v == 1;
}

static int rayleigh_ritz_q1(const scsf_ops* ops, int op, SolveWS& w, int k0, int L, double tol, cudaStream_t s) {
  const int ba = w.b - k0;
  const int64_t bb = (int64_t)ba * ba;
  double* Va = w.V + (int64_t)k0 * w.ldv;
  double* Wa = w.W + (int64_t)k0 * w.ldv;
  SCSF_TRY(spmm(ops, op, w, Va, nullptr, Wa, ba, -1, s));
  SCSF_TRY(gt_begin(s));
  SCSF_TRY(gemm_tn_dual(Va, w.ldv, Va, Wa, w.ldv, ba, w.n, w.C2, ba, w.P, s));
  SCSF_TRY(gt_end(s, 2.0 * w.n * ba * (ba + 1), 3));                            // two upper Grams
  if (w.comm) SCSF_TRY(w.comm->allreduce_sum(w.C2, (size_t)2 * bb, s));
  const double* S2 = w.C2;
  double* H = w.C2 + bb;
  SCSF_TRY(symm_upper_impl(H, ba, ba, s));                                                 // H = Q1^T A Q1 (symmetric)
  SCSF_TRY(chol_inv_impl(S2, ba, ba, w.n_glob, w.Rinv, w.Gwork, w.ctrl, s));
  SCSF_TRY(gemm_nn_ex(H, ba, ba, ba, w.Rinv, ba, ba, 1.0, 0.0, w.Tb, ba, 1, s));         // T = H R2^{-1}
  SCSF_TRY(gemm_tn(w.Rinv, ba, ba, w.Tb, ba, ba, ba, 1.0, 1, w.S, ba, w.P, s));           // G = R2^{-T} T (upper)
  SCSF_TRY(jacobi_impl(w.S, ba, ba, w.Gwork, w.Zwork, w.theta + k0, w.Zs, w.ctrl, s));
  SCSF_TRY(gemm_nn_ex(w.Rinv, ba, ba, ba, w.Zs, ba, ba, 1.0, 0.0, w.Mb, ba, 0, s));        // M = R2^{-1} Z
  SCSF_TRY(gt_begin(s));
  SCSF_TRY(gemm_nn(Va, w.ldv, w.n, ba, w.Mb, ba, ba, 1.0, 0.0, Va, w.ldv, s));
  SCSF_TRY(gt_end(s, 2.0 * w.n * ba * ba, 4));
  // residuals of A V by one stencil pass (cheaper than the n x b x b product W1 M); without a row
  // partition the pass is fused with the norms and W is not written (only the residuals use it)
  bool fused = false;
  if ((!w.comm || w.comm->world == 1) && fused_resid())   // (one slab: the whole operator, goff = 0)
    SCSF_TRY(stencil_resid_impl(ops, op, Va, w.ldv, ba, w.theta + k0, w.res + k0, w.wn + k0, w.P, s, &fused));
  if (!fused) {
    SCSF_TRY(spmm(ops, op, w, Va, nullptr, Wa, ba, -1, s));
    SCSF_TRY(resid_impl(Va, Wa, w.ldv, w.n, ba, w.theta + k0, w.res + k0, w.wn + k0, s));
  }
  if (w.comm) {
    SCSF_TRY(w.comm->allreduce_sum(w.res + k0, ba, s));
    SCSF_TRY(w.comm->allreduce_sum(w.wn + k0, ba, s));
  }
  SCSF_TRY(lock_impl(w.theta, w.res, w.wn, w.rel, w.b, L, tol, w.ctrl, w.fp, w.deg_on, w.mdeg, w.cap_on, s));
  return SCSF_OK;
}

// Warm solves start filtering with the previous operator's Ritz values (the paper's
// P:193-194 / P:297, reading R11); SCSF_INHERIT_BOUNDS=0 restores the extra Rayleigh-Ritz of
// the new operator before the first filter.
static bool inherit_bounds() {
  static const int v = [] {            // thread-safe one-time read (chain worker threads)
    int v;
    const char* e = getenv("SCSF_INHERIT_BOUNDS");
    v = (e && e[0] == '0') ? 0 : 1;
    return v;
  }();
  return v == 1;
}

// SCSF_TRACE=1: one stderr line per outer iteration (diagnostics for tools/; host reads only)
static bool trace_enabled() {
  static const int v = [] {            // thread-safe one-time read (chain worker threads)
    int v;
    const char* e = getenv("SCSF_TRACE");
    v = (e && e[0] == '1') ? 1 : 0;
    return v;
  }();
  return v == 1;
}

int fill_int_impl(int* p, int n, int v, cudaStream_t s);

// ---- optional phase timers (scsf_set_timing) ----
int set_timing(int on) {
  int old = g_timing;
  g_timing = on ? 1 : 0;
  return old;
}

static thread_local cudaEvent_t t_phase_ev[4] = {nullptr, nullptr, nullptr, nullptr};

struct PhaseTimer {
  cudaEvent_t* ev = t_phase_ev;      // created once per host thread, reused by every operator
  bool on = false;
  double filter = 0, ortho = 0, rr = 0;
  int init() {
    on = g_timing != 0;
    if (!on) return SCSF_OK;
    for (int i = 0; i < 4; ++i)
      if (!ev[i]) SCSF_CUDA_CHECK(cudaEventCreate(&ev[i]));
    return SCSF_OK;
  }
  int mark(int i, cudaStream_t s) {
    if (on) SCSF_CUDA_CHECK(cudaEventRecord(ev[i], s));
    return SCSF_OK;
  }
  // call after a stream sync that follows mark(3)
  int accumulate() {
    if (!on) return SCSF_OK;
    float a = 0, b = 0, c = 0;
    SCSF_CUDA_CHECK(cudaEventElapsedTime(&a, ev[0], ev[1]));
    SCSF_CUDA_CHECK(cudaEventElapsedTime(&b, ev[1], ev[2]));
    SCSF_CUDA_CHECK(cudaEventElapsedTime(&c, ev[2], ev[3]));
    filter += a;
    ortho += b;
    rr += c;
    return SCSF_OK;
  }
};

// Per-iteration host read of the control block.  The wait is a blocking-sync
// event (the host thread sleeps instead of spinning), so many concurrent chain
// threads do not compete for host cores.
static thread_local cudaEvent_t t_ev = nullptr;
static thread_local Ctrl* t_pinned = nullptr;
static int read_ctrl(const SolveWS& w, Ctrl& h, cudaStream_t s) {
  if (!t_ev) {
    SCSF_CUDA_CHECK(cudaEventCreateWithFlags(&t_ev, cudaEventBlockingSync | cudaEventDisableTiming));
    SCSF_CUDA_CHECK(cudaMallocHost(&t_pinned, sizeof(Ctrl)));
  }
  SCSF_CUDA_CHECK(cudaMemcpyAsync(t_pinned, w.ctrl, sizeof(Ctrl), cudaMemcpyDeviceToHost, s));
  SCSF_CUDA_CHECK(cudaEventRecord(t_ev, s));
  SCSF_CUDA_CHECK(cudaEventSynchronize(t_ev));
  h = *t_pinned;
  return SCSF_OK;
}

static int clear_chol_flag(SolveWS& w, cudaStream_t s) {
  SCSF_CUDA_CHECK(cudaMemsetAsync(&w.ctrl->chol_fail, 0, sizeof(int32_t), s));
  return SCSF_OK;
}

// ---- CUDA graphs of the outer iteration ----
// The ~25 launches of one iteration are captured once per (workspace, operator
// arrays, shape, kL) and replayed with one cudaGraphLaunch: with many chains
// the host launch rate, not the GPU, bounds throughput otherwise.  The
// operator's coefficient pointer is part of the key (a new operator of the
// batch is a new graph; its arrays live in the caller's batch).  Disabled by
// SCSF_GRAPHS=0, under SCSF_DEBUG_SYNC=1 and for the row-partitioned solve
// (its loopback collectives synchronise on the host).
struct GraphKey {
  // every device pointer an iteration's launches capture, and every shape / kernel choice:
  // a cached graph is replayed only on the exact buffers and operator kind it was captured for
  const void *V, *W, *T1, *T2, *P, *ctrl, *fp, *coef, *comm;
  int64_t n, ldv, ld, dims, goff;
  int b, kL, degree, L, timing, stencil, ncoef, deg_on;
  double tol;
  bool operator==(const GraphKey& o) const { return memcmp(this, &o, sizeof(GraphKey)) == 0; }
};
struct GraphKeyHash {
  size_t operator()(const GraphKey& k) const {
    const unsigned char* p = reinterpret_cast<const unsigned char*>(&k);
    size_t h = 1469598103934665603ull;
    for (size_t i = 0; i < sizeof(GraphKey); ++i) h = (h ^ p[i]) * 1099511628211ull;
    return h;
  }
};
// The exec is destroyed when the last holder lets go: the cache on eviction, or a thread that
// looked it up just before the eviction, after its cudaGraphLaunch (an in-flight executable
// graph is freed asynchronously on completion).
struct GraphExec {
  cudaGraphExec_t exec = nullptr;
  int kernels = 0;
  ~GraphExec() {
    if (exec) cudaGraphExecDestroy(exec);
  }
};
static std::mutex g_graph_mu;
static std::unordered_map<GraphKey, std::shared_ptr<GraphExec>, GraphKeyHash>* g_graphs = nullptr;
constexpr size_t GRAPH_CACHE_MAX = 20000;

static bool graphs_enabled() {
  static const int v = [] {            // thread-safe one-time read (chain worker threads)
    int v;
    const char* e = getenv("SCSF_GRAPHS");
    v = (e && e[0] == '0') ? 0 : 1;
    return v;
  }();
  return v == 1 && !debug_sync();
}

template <class F>
static int graph_run(const GraphKey& key, F&& body, cudaStream_t s) {
  std::shared_ptr<GraphExec> e;
  {
    std::lock_guard<std::mutex> lk(g_graph_mu);
    if (!g_graphs) g_graphs = new std::unordered_map<GraphKey, std::shared_ptr<GraphExec>, GraphKeyHash>();
    auto it = g_graphs->find(key);
    if (it != g_graphs->end()) e = it->second;
  }
  if (!e) {
    e = std::make_shared<GraphExec>();
    SCSF_CUDA_CHECK(cudaStreamBeginCapture(s, cudaStreamCaptureModeThreadLocal));
    set_capturing(true);
    take_cond_kernels();
    const int r = body();
    set_capturing(false);
    cudaGraph_t g = nullptr;
    const cudaError_t ce = cudaStreamEndCapture(s, &g);
    if (r != SCSF_OK) {
      if (g) cudaGraphDestroy(g);
      return r;
    }
    if (ce != cudaSuccess) {
      set_error("graph capture failed: %s", cudaGetErrorString(ce));
      return SCSF_ERR_DEVICE;
    }
    size_t nn = 0;
    SCSF_CUDA_CHECK(cudaGraphGetNodes(g, nullptr, &nn));
    std::vector<cudaGraphNode_t> nodes(nn);
    if (nn) SCSF_CUDA_CHECK(cudaGraphGetNodes(g, nodes.data(), &nn));
    for (auto nd : nodes) {
      cudaGraphNodeType t;
      // (the runtime reports an error, not a type, for a conditional node: it is not a kernel)
      if (cudaGraphNodeGetType(nd, &t) != cudaSuccess) {
        cudaGetLastError();
        continue;
      }
      e->kernels += (t == cudaGraphNodeTypeKernel);
    }
    e->kernels += take_cond_kernels();                 // a conditional body counts once per replay
    const cudaError_t ie = cudaGraphInstantiate(&e->exec, g, 0);
    cudaGraphDestroy(g);
    SCSF_CUDA_CHECK(ie);
    std::lock_guard<std::mutex> lk(g_graph_mu);
    if (g_graphs->size() >= GRAPH_CACHE_MAX) g_graphs->clear();   // bound the cache; execs freed by their holders
    g_graphs->emplace(key, e);
  }
  SCSF_CUDA_CHECK(cudaGraphLaunch(e->exec, s));
  count_launch(e->kernels);
  return SCSF_OK;
}

// Solve operator `op`.  warm: V already holds the initial b-block (orthonormal).
// On return w.V holds the final block sorted ascending with the sign convention,
// w.theta_sorted the Ritz values.
int solve_core(const scsf_ops* ops_in, int op_in, int L, int nex, int degree_arg, double tol, int max_iter,
               bool warm, bool orthonormalize, uint64_t seed, SolveWS& w, scsf_stats* st, cudaStream_t s) {
  const int b = L + nex;
  // degree_arg > 0: uniform degree m for every active column (reading R8); degree_arg < 0: per-column
  // degrees (Alg. 1 l. 5's staggered update) chosen by k_lock, capped at |degree_arg|
  const bool adaptive = degree_arg < 0;
  const int degree = adaptive ? -degree_arg : degree_arg;
  // (row partition: only a communicator whose collectives are stream-ordered device work (NCCL) can be
  // captured; the loopback backend meets at host barriers)
  const bool graphs = graphs_enabled() && (!w.comm || w.comm->capturable()) && s != nullptr && !g_timing;
  // With graphs, the operator's arrays are first copied into the chain's own
  // buffer, so every captured iteration is independent of the operator index.
  scsf_ops opl = *ops_in;
  int op = op_in;
  if (graphs) {
    const size_t per = (size_t)ncoef(ops_in) * ops_in->ld;
    SCSF_CUDA_CHECK(cudaMemcpyAsync(w.coef_buf, ops_in->coef + (int64_t)op_in * per, per * sizeof(double),
                                    cudaMemcpyDeviceToDevice, s));
    opl.coef = w.coef_buf;
    opl.n_ops = 1;
    op = 0;
  }
  const scsf_ops* ops = &opl;
  int64_t spmm_cols = 0;
  int filter_steps = 0, iters = 0;
  double filter_bytes = 0.0;
  const double coef_bytes = 8.0 * ncoef(ops) * (double)w.n;
  PhaseTimer tm;
  SCSF_TRY(tm.init());
  static thread_local GemmTiming t_gt_store;
  t_gt_store.ms = 0.0;
  t_gt_store.total_flops = 0.0;
  for (int k = 0; k < GT_KINDS; ++k) t_gt_store.kind_ms[k] = t_gt_store.kind_flops[k] = 0.0;
  t_gt_store.used = 0;
  t_gt = tm.on ? &t_gt_store : nullptr;
  Ctrl h{};
  SCSF_TRY(gershgorin_impl(ops, op, w.gersh, s));
  SCSF_TRY(ctrl_init_impl(w.ctrl, w.gersh, s));
  w.mdeg = degree;
  // per-column degrees where the filter kernel honours them: the resident filters, the vectorised
  // streaming step and (row partition, always nx % 4 == 0) the slab step; the degrees come from
  // k_lock on all-reduced residuals, so every rank of a partition picks the same ones
  w.deg_on = (adaptive && (w.comm || filter_resident_ok(ops) || stencil_v4_ok(ops, w.ldv))) ? w.deg : nullptr;
  if (w.deg_on) SCSF_TRY(fill_int_impl(w.deg, b, degree, s));
  if (!warm) SCSF_TRY(rand_block_impl(w.V, w.ldv, w.n, b, seed, w.goff, s));
  if (!warm || orthonormalize) {
    SCSF_TRY(cholqr_pass(w, w.V, w.V, b, s));
    SCSF_TRY(cholqr_pass(w, w.V, w.V, b, s));
  }
  w.cap_on = warm ? 1 : 0;
  if (warm && !orthonormalize && inherit_bounds()) {
    // P:193-194, P:297 read literally: the first filter of a warm solve uses the previous
    // operator's Ritz values (lambda = theta_1, alpha = theta_b) and this operator's beta
    SCSF_TRY(bounds_from_theta_impl(w.theta_sorted, b, w.ctrl, w.fp, degree, s));
    SCSF_TRY(read_ctrl(w, h, s));
  } else {
    // one Rayleigh-Ritz of the new operator on the initial block (R11)
    SCSF_TRY(rayleigh_ritz(ops, op, w, 0, L, tol, spmm_cols, s));
    SCSF_TRY(read_ctrl(w, h, s));
  }
  w.cap_on = 1;
  int kL = h.kL;
  int fallbacks = 0;
  // degree the next filter runs: m, or the conditioning cap k_lock / k_bounds_from_theta wrote
  // (ctrl->pad[2], = fp[3]; the kernels apply it on the device, the host only counts with it)
  auto filter_degree = [&](const Ctrl& c) { return (c.pad[2] > 0 && c.pad[2] < degree) ? (int)c.pad[2] : degree; };
  int64_t next_colsteps = (int64_t)filter_degree(h) * (b - kL);   // per-column degrees start at m
  // One outer iteration (steps 1-6) as device work only; replayed from a CUDA graph
  // keyed by kL (every pointer and shape of the iteration is a function of kL).
  auto iteration = [&](int kLc) -> int {
    const int ba = b - kLc;
    double* y[3] = {w.V + (int64_t)kLc * w.ldv, w.T1 + (int64_t)kLc * w.ldv, w.T2 + (int64_t)kLc * w.ldv};
    // 1. Chebyshev filter (Alg. 1) on the active block
    SCSF_TRY(tm.mark(0, s));
    double* F;
    if (!w.comm && filter_resident_ok(ops)) {
      SCSF_TRY(filter_resident_impl(ops, op, y[0], y[1], w.ldv, ba, w.fp, degree, s,
                                    w.deg_on ? w.deg_on + kLc : nullptr));
      F = y[1];
    } else {
      SCSF_TRY(step_table_impl(w.fp, degree, s));
      // per-column degrees (f2): columns past their degree are skipped in place; k_lock rounds every
      // degree to = m (mod 3), so each column's last output lands in y[m % 3] as well
      const int* dg = w.deg_on ? w.deg_on + kLc : nullptr;
      SCSF_TRY(spmm(ops, op, w, y[0], nullptr, y[1], ba, 0, s, dg));
      for (int st_i = 1; st_i < degree; ++st_i)
        SCSF_TRY(spmm(ops, op, w, y[st_i % 3], y[(st_i - 1) % 3], y[(st_i + 1) % 3], ba, st_i, s, dg));
      F = y[degree % 3];
    }
    SCSF_TRY(tm.mark(1, s));
    // 2. block classical Gram-Schmidt, twice, against the locked vectors
    if (kLc > 0) {
      for (int rep = 0; rep < 2; ++rep) {
        SCSF_TRY(gram(w, w.V, kLc, F, ba, 0, w.C, s));
        SCSF_TRY(gt_begin(s));
        SCSF_TRY(gemm_nn(w.V, w.ldv, w.n, kLc, w.C, kLc, ba, -1.0, 1.0, F, w.ldv, s));
        SCSF_TRY(gt_end(s, 2.0 * w.n * kLc * ba, 5));
      }
    }
    // 3. CholQR, first pass (lands the block in V's active columns)
    SCSF_TRY(clear_chol_flag(w, s));
    SCSF_TRY(cholqr_pass(w, F, y[0], ba, s));
    SCSF_TRY(tm.mark(2, s));
    // 4.-6. CholQR's second pass folded into Rayleigh-Ritz, residuals, locking
    SCSF_TRY(rayleigh_ritz_q1(ops, op, w, kLc, L, tol, s));
    SCSF_TRY(tm.mark(3, s));
    return SCSF_OK;
  };
  while (kL < L && iters < max_iter && !(h.nonfinite & 1)) {
    ++iters;
    const int ba = b - kL;
    if (graphs) {                       // b > 128: the block-Jacobi sweeps are a conditional WHILE node
      GraphKey key;
      memset(&key, 0, sizeof(key));                    // padding bytes take part in the hash / compare
      key.V = w.V;
      key.W = w.W;
      key.T1 = w.T1;
      key.T2 = w.T2;
      key.P = w.P;
      key.ctrl = w.ctrl;
      key.fp = w.fp;
      key.coef = ops->coef + (int64_t)op * ncoef(ops) * ops->ld;
      key.comm = w.comm;
      key.goff = w.goff;
      key.n = w.n;
      key.ldv = w.ldv;
      key.ld = ops->ld;
      key.b = b;
      key.kL = kL;
      key.degree = degree;
      key.L = L;
      key.timing = tm.on ? 1 : 0;
      key.stencil = ops->stencil;
      key.ncoef = ncoef(ops);
      key.deg_on = w.deg_on ? 1 : 0;
      key.dims = ops->nx + 65536LL * (ops->ny + 65536LL * (ops->nz + 65536LL * ops->dim));
      key.tol = tol;
      SCSF_TRY(graph_run(key, [&]() { return iteration(kL); }, s));
    } else {
      SCSF_TRY(iteration(kL));
    }
    // algorithmic bytes: first step reads Y0 + writes Y1, later steps read Y_s, Y_{s-1}
    // and write Y_{s+1}; one pass over the coefficient arrays per step
    // column-steps of this filter: m b_act, or the sum of the per-column degrees (f2)
    const int m_it = filter_degree(h);
    const int64_t colsteps = w.deg_on ? next_colsteps : (int64_t)m_it * ba;
    filter_bytes += 16.0 * w.n * ba + 24.0 * w.n * (double)(colsteps - ba) + coef_bytes * m_it;
    filter_steps += m_it;
    spmm_cols += colsteps + 2 * ba;
    SCSF_TRY(read_ctrl(w, h, s));
    SCSF_TRY(tm.accumulate());
    SCSF_TRY(gt_collect());
    next_colsteps = h.pad[1];
    if (trace_enabled())
      fprintf(stderr, "[scsf trace] op %d warm %d it %d m %d kL %d lambda %.6e alpha %.6e beta %.6e next_m %d "
              "chol_fail %d nonfinite %d max_rel %.3e\n", op_in, warm ? 1 : 0, iters, m_it, h.kL, h.lambda, h.alpha,
              h.beta, filter_degree(h), h.chol_fail, h.nonfinite, h.max_rel);
    if (h.chol_fail) {
      // shifted CholQR was needed: one more CholQR pass, then redo the RR step
      ++fallbacks;
      SCSF_CUDA_CHECK(cudaMemcpyAsync(&w.ctrl->kL, &kL, sizeof(int32_t), cudaMemcpyHostToDevice, s));
      SCSF_TRY(clear_chol_flag(w, s));
      SCSF_TRY(cholqr_pass(w, w.V + (int64_t)kL * w.ldv, w.V + (int64_t)kL * w.ldv, ba, s));
      SCSF_TRY(rayleigh_ritz(ops, op, w, kL, L, tol, spmm_cols, s));
      SCSF_TRY(read_ctrl(w, h, s));
    }
    kL = h.kL;
  }
  // final ascending order + sign convention into T1, then swap so V holds it
  if (w.comm) {
    SCSF_TRY(sort_theta_impl(w.theta, w.rel, b, L, w.perm, w.theta_sorted, w.ctrl, s));
    SCSF_TRY(colmax_local_impl(w.V, w.ldv, w.n, w.perm, b, w.goff, w.colbuf, s));
    SCSF_TRY(w.comm->allgather(w.colbuf, w.colgath, 3 * (size_t)b, s));
    SCSF_TRY(sign_apply_impl(w.V, w.ldv, w.n, w.perm, w.colgath, w.comm->world, b, w.T1, w.ldv, s));
  } else {
    SCSF_TRY(finalize_impl(w.theta, w.rel, b, L, w.perm, w.theta_sorted, w.V, w.ldv, w.n, w.T1, w.ldv,
                           w.ctrl, s));
  }
  std::swap(w.V, w.T1);
  SCSF_TRY(read_ctrl(w, h, s));
  SCSF_TRY(gt_collect());
  int status = SCSF_OK;
  if (kL < L || (h.nonfinite & 1)) status = SCSF_ERR_NUMERICAL;
  if (st) {
    st->status = status;
    st->iterations = iters;
    st->filter_steps = filter_steps;
    st->cholqr_fallbacks = fallbacks;
    st->n_locked = kL;
    st->warm = warm ? 1 : 0;
    st->spmm_columns = spmm_cols;
    st->max_rel_resid = h.max_rel;
    st->beta = h.beta;
    st->t_filter_ms = tm.filter;
    st->t_ortho_ms = tm.ortho;
    st->t_rr_ms = tm.rr;
    st->filter_bytes = filter_bytes;
    st->jacobi_sweeps = h.pad[0];
    SCSF_TRY(gt_collect());
    st->t_gemm_ms = t_gt ? t_gt->ms : 0.0;
    st->gemm_flops = t_gt ? t_gt->total_flops : 0.0;
    if (t_gt && getenv("SCSF_GEMM_PROFILE")) {          // per-kind DGEMM times (tools/; stderr)
      fprintf(stderr, "scsf_gemm_profile n=%lld b=%d", (long long)w.n, b);
      for (int k = 0; k < GT_KINDS; ++k)
        fprintf(stderr, " k%d=%.4f/%.6e", k, t_gt->kind_ms[k], t_gt->kind_flops[k]);
      fprintf(stderr, "\n");
    }
  }
  if (status != SCSF_OK)
    set_error("operator %d: %d of %d pairs converged after %d iterations (worst rel. residual %.3e)", op_in,
              kL, L, iters, h.max_rel);
  return status;
}

}  // namespace scsf
