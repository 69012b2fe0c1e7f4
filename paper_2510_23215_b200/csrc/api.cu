// api.cu — the extern "C" entry points declared in include/scsf.h:
// argument validation, workspace carving, error strings.  All arithmetic is
// in the k_*.cu kernels; this file only sequences them.
#include "common.cuh"

#include <atomic>
#include <cstdarg>
#include <cstdlib>
#include <cstring>
#include <mutex>
#include <string>
#include <thread>
#include <vector>

namespace scsf {

static thread_local char g_err[512] = "";
static std::atomic<int64_t> g_launches{0};

void set_error(const char* fmt, ...) {
  va_list ap;
  va_start(ap, fmt);
  vsnprintf(g_err, sizeof(g_err), fmt, ap);
  va_end(ap);
}
static thread_local bool t_capturing = false;
void set_capturing(bool on) { t_capturing = on; }
void count_launch(int n) {
  if (!t_capturing) g_launches += n;
}
bool debug_sync() {
  if (t_capturing) return false;
  static const int v = [] {            // thread-safe one-time read (chain worker threads)
    int v;
    const char* e = getenv("SCSF_DEBUG_SYNC");
    v = (e && e[0] == '1') ? 1 : 0;
    return v;
  }();
  return v == 1;
}

// k_sort.cu
size_t sort_ws_bytes(int N, int dim, int p, int F, int p0);
int signatures_impl(const double* params, int N, int dim, int p, int F, int p0, double2* sig, Arena& a,
                    cudaStream_t s);
int sort_impl(const double* params, int N, int dim, int p, int F, int p0, int start, int* perm,
              double* d2_best, double* d2_second, Arena& a, cudaStream_t s);
// k_dense.cu / k_small.cu primitives
size_t tn_partial_doubles(int64_t n, int b1, int b2);
size_t small_scratch_doubles(int b);
int gemm_tn(const double* X, int64_t ldx, int b1, const double* Y, int64_t ldy, int b2, int64_t n,
            double alpha, int sym, double* C, int64_t ldc, double* P, cudaStream_t s);
int gemm_nn(const double* X, int64_t ldx, int64_t n, int b1, const double* M, int64_t ldm, int b2,
            double alpha, double beta, double* Out, int64_t ldo, cudaStream_t s);
int chol_inv_impl(const double* S, int64_t lds, int b, int64_t nrows, double* Rinv, double* scratch,
                  Ctrl* ctrl, cudaStream_t s);
int jacobi_impl(const double* G, int64_t ldg, int b, double* scratchG, double* Z, double* theta,
                double* Zout, Ctrl* ctrl, cudaStream_t s);
// solver.cu
int set_timing(int on);
// k_small.cu / k_dense.cu: one-time kernel attributes (set before any worker thread starts)
int set_small_attrs();
int dense_init_attrs();
int stencil_init_attrs();
static int init_kernel_attrs() {
  static std::mutex mu;                    // API calls from several user threads: one initialiser at a time
  std::lock_guard<std::mutex> lk(mu);
  SCSF_TRY(set_small_attrs());
  SCSF_TRY(dense_init_attrs());
  SCSF_TRY(stencil_init_attrs());
  return SCSF_OK;
}
// k_grf.cu
size_t grf_ws_doubles(int nx, int K);
int grf_impl(int dim, int nx, int K, double s, double sigma, double vscale, int family, int n_ops,
             const double* xi, double* fx, double* fy, double* fz, double* c, double* params, double* tab,
             cudaStream_t st);
// k_stencil.cu
int assemble_vib_impl(const scsf_ops* ops, double h, const double* D, const double* rho, int64_t fstride,
                      double* coef, cudaStream_t s);
int step_table_impl(double* fp, int m, cudaStream_t s);
int assemble_impl(const scsf_ops* ops, double h, const double* fx, const double* fy, const double* fz,
                  const double* c, double* coef, cudaStream_t s);
int stencil_impl(const scsf_ops* ops, int op, const double* X, const double* Xp, double* Out, int64_t ldv,
                 int ncols, const double* fp, int step, cudaStream_t s, const int* deg = nullptr);
bool filter_resident_ok(const scsf_ops* ops);
int filter_kind(const scsf_ops* ops);
int filter_resident_impl(const scsf_ops* ops, int op, const double* X, double* Out, int64_t ldv, int ncols,
                         const double* fp, int m, cudaStream_t s, const int* deg = nullptr);

}  // namespace scsf

#include "solver.cuh"
#include "comm.cuh"

using namespace scsf;

static int check_ops(const scsf_ops* ops) {
  SCSF_ARG_CHECK(ops != nullptr, "ops is NULL");
  SCSF_ARG_CHECK(ops->dim == 2 || ops->dim == 3, "dim must be 2 or 3 (got %d)", ops->dim);
  SCSF_ARG_CHECK(ops->nx >= 1 && ops->ny >= 1 && ops->nz >= 1, "grid sizes must be >= 1");
  SCSF_ARG_CHECK(ops->dim == 3 || ops->nz == 1, "nz must be 1 when dim == 2");
  SCSF_ARG_CHECK(ops->n_ops >= 1, "n_ops must be >= 1");
  int64_t n = (int64_t)ops->nx * ops->ny * ops->nz;
  SCSF_ARG_CHECK(ops->ld >= n && ops->ld % 32 == 0, "ld must be >= n and a multiple of 32");
  SCSF_ARG_CHECK(ops->coef != nullptr, "coef is NULL");
  SCSF_ARG_CHECK(ops->stencil == SCSF_STENCIL_FLUX || ops->stencil == SCSF_STENCIL_VIB13,
                 "unknown stencil kind %d", ops->stencil);
  SCSF_ARG_CHECK(ops->stencil == SCSF_STENCIL_FLUX || ops->dim == 2, "the 13-point vibration stencil is 2-D");
  SCSF_ARG_CHECK(ops->stencil == SCSF_STENCIL_FLUX || (ops->nx >= 3 && ops->ny >= 3),
                 "the 13-point vibration stencil needs nx, ny >= 3");
  return SCSF_OK;
}

static int check_solve_args(const scsf_ops* ops, int L, int nex, int degree, double tol, int max_iter) {
  SCSF_TRY(check_ops(ops));
  int64_t n = (int64_t)ops->nx * ops->ny * ops->nz;
  SCSF_ARG_CHECK(L >= 1, "L must be >= 1");
  SCSF_ARG_CHECK(nex >= 0, "nex must be >= 0");
  SCSF_ARG_CHECK(L + nex <= n, "L + nex must be <= n");
  SCSF_ARG_CHECK(L + nex <= 368, "L + nex must be <= 368 in this build");
  SCSF_ARG_CHECK((degree >= 1 && degree <= FP_MAX_DEGREE) || (degree <= -4 && degree >= -FP_MAX_DEGREE),
                 "degree must be in [1, %d] (uniform) or [-%d, -4] (per-column adaptive, cap |degree|)",
                 FP_MAX_DEGREE, FP_MAX_DEGREE);
  SCSF_ARG_CHECK(tol > 0.0, "tol must be > 0");
  SCSF_ARG_CHECK(max_iter >= 0, "max_iter must be >= 0");
  return SCSF_OK;
}

extern "C" {

const char* scsf_last_error(void) { return g_err; }
int scsf_abi_version(void) { return SCSF_ABI_VERSION; }
int64_t scsf_launch_count(void) { return g_launches.load(); }
int scsf_set_timing(int32_t on) { return set_timing(on); }
int scsf_filter_kind(const scsf_ops* ops) {
  if (check_ops(ops) != SCSF_OK) return -1;
  return filter_kind(ops);
}

size_t scsf_sort_workspace_bytes(int32_t N, int32_t dim, int32_t p, int32_t F, int32_t p0) {
  if (N < 1 || (dim != 2 && dim != 3) || p < 1 || F < 1 || p0 < 1) return 0;
  return sort_ws_bytes(N, dim, p, F, p0);
}

static int check_sort(int32_t N, int32_t dim, int32_t p, int32_t F, int32_t p0) {
  SCSF_ARG_CHECK(N >= 1, "N must be >= 1");
  SCSF_ARG_CHECK(dim == 2 || dim == 3, "dim must be 2 or 3");
  SCSF_ARG_CHECK(p >= 1 && F >= 1, "p and F must be >= 1");
  SCSF_ARG_CHECK(p0 >= 2 && p0 % 2 == 0 && p0 <= p, "p0 must be even with 2 <= p0 <= p");
  return SCSF_OK;
}

int scsf_signatures(const double* params, int32_t N, int32_t dim, int32_t p, int32_t F, int32_t p0,
                    double* sig, void* ws, size_t ws_bytes, void* stream) {
  SCSF_TRY(check_sort(N, dim, p, F, p0));
  SCSF_ARG_CHECK(params && sig, "params / sig is NULL");
  cudaStream_t s = (cudaStream_t)stream;
  Arena a(ws, ws_bytes);
  if (!ws) {
    set_error("workspace is NULL");
    return SCSF_ERR_WORKSPACE;
  }
  int r = signatures_impl(params, N, dim, p, F, p0, (double2*)sig, a, s);
  if (r == SCSF_ERR_WORKSPACE) set_error("workspace too small");
  if (r != SCSF_OK) return r;
  SCSF_CUDA_CHECK(cudaStreamSynchronize(s));
  return SCSF_OK;
}

int scsf_sort(const double* params, int32_t N, int32_t dim, int32_t p, int32_t F, int32_t p0, int32_t start,
              int32_t* perm, double* d2_best, double* d2_second, void* ws, size_t ws_bytes, void* stream) {
  SCSF_TRY(check_sort(N, dim, p, F, p0));
  SCSF_ARG_CHECK(params && perm, "params / perm is NULL");
  SCSF_ARG_CHECK(start >= 0 && start < N, "start out of range");
  if (!ws || ws_bytes < sort_ws_bytes(N, dim, p, F, p0)) {
    set_error("workspace too small: need %zu bytes", sort_ws_bytes(N, dim, p, F, p0));
    return SCSF_ERR_WORKSPACE;
  }
  Arena a(ws, ws_bytes);
  return sort_impl(params, N, dim, p, F, p0, start, perm, d2_best, d2_second, a, (cudaStream_t)stream);
}

int scsf_assemble(const scsf_ops* ops, double h, const double* faces_x, const double* faces_y,
                  const double* faces_z, const double* c, double* coef_out, void* stream) {
  SCSF_ARG_CHECK(ops != nullptr, "ops is NULL");
  scsf_ops o = *ops;
  o.coef = coef_out;
  SCSF_TRY(check_ops(&o));
  SCSF_ARG_CHECK(ops->stencil == SCSF_STENCIL_FLUX, "scsf_assemble builds flux-form stencils (stencil = 0)");
  SCSF_ARG_CHECK(faces_x && faces_y && (ops->dim == 2 || faces_z), "face arrays missing");
  SCSF_ARG_CHECK(h > 0.0, "h must be > 0");
  cudaStream_t s = (cudaStream_t)stream;
  SCSF_TRY(assemble_impl(&o, h, faces_x, faces_y, faces_z, c, coef_out, s));
  SCSF_CUDA_CHECK(cudaStreamSynchronize(s));
  return SCSF_OK;
}

int scsf_assemble_vibration(const scsf_ops* ops, double h, const double* D, const double* rho,
                            int64_t field_stride, double* coef_out, void* stream) {
  SCSF_ARG_CHECK(ops != nullptr, "ops is NULL");
  scsf_ops o = *ops;
  o.coef = coef_out;
  SCSF_TRY(check_ops(&o));
  SCSF_ARG_CHECK(o.stencil == SCSF_STENCIL_VIB13, "ops->stencil must be SCSF_STENCIL_VIB13");
  SCSF_ARG_CHECK(D && rho, "D / rho NULL");
  SCSF_ARG_CHECK(field_stride >= (int64_t)o.nx * o.ny, "field_stride must be >= n");
  SCSF_ARG_CHECK(h > 0.0, "h must be > 0");
  cudaStream_t s = (cudaStream_t)stream;
  SCSF_TRY(assemble_vib_impl(&o, h, D, rho, field_stride, coef_out, s));
  SCSF_CUDA_CHECK(cudaStreamSynchronize(s));
  return SCSF_OK;
}

size_t scsf_grf_workspace_bytes(int32_t nx, int32_t K) {
  if (nx < 1 || K < 1) return 0;
  return grf_ws_doubles(nx, K) * sizeof(double);
}

int scsf_grf_fields(int32_t dim, int32_t nx, int32_t K, double s, double sigma, double vscale, int32_t family,
                    int32_t n_ops, const double* xi, double* faces_x, double* faces_y, double* faces_z, double* c,
                    double* params, void* ws, size_t ws_bytes, void* stream) {
  SCSF_ARG_CHECK(dim == 2 || dim == 3, "dim must be 2 or 3");
  SCSF_ARG_CHECK(nx >= 1 && n_ops >= 0, "nx >= 1 and n_ops >= 0 required");
  SCSF_ARG_CHECK(K >= 1 && (dim == 2 ? K <= 32 : K * K * K <= 1024), "K out of range (2-D: <= 32, 3-D: K^3 <= 1024)");
  SCSF_ARG_CHECK(dim == 2 || nx + 1 <= 64, "3-D fields need nx <= 63");
  SCSF_ARG_CHECK(family >= 0 && family <= 3, "family must be 0 (diva), 1 (lapv), 2 (divac) or 3 (vib)");
  SCSF_ARG_CHECK(s >= 0.0 && vscale > 0.0, "s >= 0 and vscale > 0 required");
  if (n_ops == 0) return SCSF_OK;
  SCSF_ARG_CHECK(xi && params && (family == 3 || (faces_x && faces_y && (dim == 2 || faces_z) && c)),
                 "NULL array");
  if (!ws || ws_bytes < grf_ws_doubles(nx, K) * sizeof(double)) {
    set_error("workspace too small: need %zu bytes", grf_ws_doubles(nx, K) * sizeof(double));
    return SCSF_ERR_WORKSPACE;
  }
  cudaStream_t st = (cudaStream_t)stream;
  SCSF_TRY(grf_impl(dim, nx, K, s, sigma, vscale, family, n_ops, xi, faces_x, faces_y, faces_z, c, params,
                    (double*)ws, st));
  SCSF_CUDA_CHECK(cudaStreamSynchronize(st));
  return SCSF_OK;
}

size_t scsf_filter_workspace_bytes(const scsf_ops* ops, int32_t k, int64_t ldy) {
  if (!ops || k < 1) return 0;
  Arena a(nullptr, 0);
  a.take<double>(2 * ldy * k);
  a.take<double>(FP_DOUBLES);
  return a.off;
}

int scsf_cheb_filter(const scsf_ops* ops, int32_t op_index, const double* Y0, int64_t ldy, int32_t k,
                     int32_t degree, double lambda, double c, double e, double* Ym, void* ws, size_t ws_bytes,
                     void* stream) {
  SCSF_TRY(check_ops(ops));
  int64_t n = (int64_t)ops->nx * ops->ny * ops->nz;
  SCSF_ARG_CHECK(op_index >= 0 && op_index < ops->n_ops, "op_index out of range");
  SCSF_ARG_CHECK(Y0 && Ym && Y0 != Ym, "Y0 / Ym NULL or aliased");
  SCSF_ARG_CHECK(k >= 1 && ldy >= n, "k >= 1 and ldy >= n required");
  SCSF_ARG_CHECK(degree >= 1 && degree <= FP_MAX_DEGREE, "degree must be in [1, %d]", FP_MAX_DEGREE);
  SCSF_ARG_CHECK(e > 0.0 && lambda != c, "need e > 0 and lambda != c");
  Arena a(ws, ws_bytes);
  double* B1 = a.take<double>(ldy * k);
  double* B2 = a.take<double>(ldy * k);
  double* fp = a.take<double>(FP_DOUBLES);
  if (a.overflow || !ws) {
    set_error("workspace too small");
    return SCSF_ERR_WORKSPACE;
  }
  cudaStream_t s = (cudaStream_t)stream;
  double hfp[4] = {lambda, c, e, 0.0};
  SCSF_CUDA_CHECK(cudaMemcpyAsync(fp, hfp, sizeof(hfp), cudaMemcpyHostToDevice, s));
  if (filter_resident_ok(ops) && !(getenv("SCSF_FILTER_STREAMING") && getenv("SCSF_FILTER_STREAMING")[0] == '1')) {
    SCSF_TRY(filter_resident_impl(ops, op_index, Y0, Ym, ldy, k, fp, degree, s));
    SCSF_CUDA_CHECK(cudaStreamSynchronize(s));
    return SCSF_OK;
  }
  SCSF_TRY(step_table_impl(fp, degree, s));
  // rotate over {Y0 (read-only), B1, B2, Ym}: Y_{s+1} never overwrites Y_s or Y_{s-1}
  const double* prev = nullptr;
  const double* cur = Y0;
  double* bufs[3] = {B1, B2, Ym};
  int bi = 0;
  for (int st = 0; st < degree; ++st) {
    double* out;
    if (st == degree - 1) {
      out = Ym;
    } else {
      out = bufs[bi % 2];   // B1 / B2 alternate
      ++bi;
    }
    SCSF_TRY(stencil_impl(ops, op_index, cur, prev, out, ldy, k, fp, st, s));
    prev = cur;
    cur = out;
  }
  SCSF_CUDA_CHECK(cudaStreamSynchronize(s));
  return SCSF_OK;
}

size_t scsf_solve_workspace_bytes(const scsf_ops* ops, int32_t L, int32_t nex) {
  if (!ops || L < 1 || nex < 0) return 0;
  return solve_ws_bytes(ops, L, nex);
}

int scsf_solve_one(const scsf_ops* ops, int32_t op_index, int32_t L, int32_t nex, int32_t degree, double tol,
                   int32_t max_iter, const double* warm_vecs, uint64_t seed, double* evals, double* evecs,
                   int64_t ld_vec, scsf_stats* st, void* ws, size_t ws_bytes, void* stream) {
  SCSF_TRY(check_solve_args(ops, L, nex, degree, tol, max_iter));
  int64_t n = (int64_t)ops->nx * ops->ny * ops->nz;
  SCSF_ARG_CHECK(op_index >= 0 && op_index < ops->n_ops, "op_index out of range");
  SCSF_ARG_CHECK(evals && evecs, "evals / evecs NULL");
  SCSF_ARG_CHECK(ld_vec >= n, "ld_vec must be >= n");
  cudaStream_t s = (cudaStream_t)stream;
  SolveWS w;
  SCSF_TRY(carve_solve_ws(ops, L, nex, ws, ws_bytes, w));
  const int b = L + nex;
  if (warm_vecs) {
    SCSF_CUDA_CHECK(cudaMemcpy2DAsync(w.V, w.ldv * sizeof(double), warm_vecs, ld_vec * sizeof(double),
                                      n * sizeof(double), b, cudaMemcpyDeviceToDevice, s));
    if (w.ldv > n)
      SCSF_CUDA_CHECK(cudaMemset2DAsync(w.V + n, w.ldv * sizeof(double), 0, (w.ldv - n) * sizeof(double), b, s));
  }
  int r = solve_core(ops, op_index, L, nex, degree, tol, max_iter, warm_vecs != nullptr, true,
                     seed + (uint64_t)op_index, w, st, s);
  if (r != SCSF_OK && r != SCSF_ERR_NUMERICAL) return r;
  SCSF_CUDA_CHECK(cudaMemcpyAsync(evals, w.theta_sorted, b * sizeof(double), cudaMemcpyDeviceToDevice, s));
  SCSF_CUDA_CHECK(cudaMemcpy2DAsync(evecs, ld_vec * sizeof(double), w.V, w.ldv * sizeof(double),
                                    n * sizeof(double), b, cudaMemcpyDeviceToDevice, s));
  SCSF_CUDA_CHECK(cudaStreamSynchronize(s));
  return r;
}

// One warm-start chain on one stream: chain[0] cold, every later operator warm
// from the previous final block.  Outputs by chain position.
// Host outputs streamed while the chain runs (SURVEY f4 "streaming eigenpair writer"): each
// operator's L pairs are staged on the device (double buffer) and copied to pinned host memory
// on a second stream, overlapping the next operator's solve.
struct HostSink {
  double* evals = nullptr;     // host [n_chain][L]
  double* evecs = nullptr;     // host [n_chain][L][ld] or NULL
  int64_t ld = 0;
  double* stage[2] = {nullptr, nullptr};      // device L x ldv each
  double* stage_ev[2] = {nullptr, nullptr};   // device L each
};

static int run_chain(const scsf_ops* ops, const int32_t* chain, int32_t n_chain, int32_t L, int32_t nex,
                     int32_t degree, double tol, int32_t max_iter, uint64_t seed, double* evals, double* evecs,
                     int64_t ld_vec, scsf_stats* st, SolveWS& w, cudaStream_t s, HostSink* sink = nullptr,
                     const double* state_in = nullptr, double* state_out = nullptr) {
  const int bb = L + nex;
  if (state_in) {   // resume: the block and Ritz values of the operator solved before chain[0]
    SCSF_CUDA_CHECK(cudaMemcpyAsync(w.theta_sorted, state_in, bb * sizeof(double), cudaMemcpyDeviceToDevice, s));
    SCSF_CUDA_CHECK(cudaMemcpy2DAsync(w.V, w.ldv * sizeof(double), state_in + bb, w.n * sizeof(double),
                                      w.n * sizeof(double), bb, cudaMemcpyDeviceToDevice, s));
    if (w.ldv > w.n)
      SCSF_CUDA_CHECK(cudaMemset2DAsync(w.V + w.n, w.ldv * sizeof(double), 0, (w.ldv - w.n) * sizeof(double), bb, s));
  }
  cudaStream_t cs = nullptr;
  cudaEvent_t ready[2] = {nullptr, nullptr}, done[2] = {nullptr, nullptr};
  if (sink) {
    SCSF_CUDA_CHECK(cudaStreamCreateWithFlags(&cs, cudaStreamNonBlocking));
    for (int i = 0; i < 2; ++i) {
      SCSF_CUDA_CHECK(cudaEventCreateWithFlags(&ready[i], cudaEventDisableTiming));
      SCSF_CUDA_CHECK(cudaEventCreateWithFlags(&done[i], cudaEventDisableTiming));
    }
  }
  auto cleanup = [&]() {
    if (!sink) return;
    cudaStreamSynchronize(cs);
    cudaStreamDestroy(cs);
    for (int i = 0; i < 2; ++i) {
      cudaEventDestroy(ready[i]);
      cudaEventDestroy(done[i]);
    }
  };
  const int r = [&]() -> int {
  int worst = SCSF_OK;
  bool prev_ok = state_in != nullptr;      // a warm start needs a converged block to start from
  for (int k = 0; k < n_chain; ++k) {
    scsf_stats local{};
    const bool warm = k > 0 ? prev_ok : state_in != nullptr;
    int r = solve_core(ops, chain[k], L, nex, degree, tol, max_iter, warm, false, seed + (uint64_t)chain[k], w,
                       &local, s);
    if (r == SCSF_ERR_NUMERICAL && warm) {
      // R29: a warm start that broke down (a queue neighbour too dissimilar for the inherited
      // bounds, or a degree past the stability ceiling) is solved again from a random block, and
      // the chain goes on from that result; the statistics count both attempts
      scsf_stats again{};
      r = solve_core(ops, chain[k], L, nex, degree, tol, max_iter, false, false, seed + (uint64_t)chain[k], w,
                     &again, s);
      again.iterations += local.iterations;
      again.filter_steps += local.filter_steps;
      again.cholqr_fallbacks += local.cholqr_fallbacks;
      again.spmm_columns += local.spmm_columns;
      again.t_filter_ms += local.t_filter_ms;
      again.t_ortho_ms += local.t_ortho_ms;
      again.t_rr_ms += local.t_rr_ms;
      again.filter_bytes += local.filter_bytes;
      again.jacobi_sweeps += local.jacobi_sweeps;
      again.t_gemm_ms += local.t_gemm_ms;
      again.gemm_flops += local.gemm_flops;
      again.cold_retry = 1;
      local = again;
    }
    if (r != SCSF_OK && r != SCSF_ERR_NUMERICAL) return r;
    prev_ok = (r == SCSF_OK);
    if (r > worst) worst = r;
    if (st) st[k] = local;
    if (evals)
      SCSF_CUDA_CHECK(cudaMemcpyAsync(evals + (int64_t)k * L, w.theta_sorted, L * sizeof(double),
                                      cudaMemcpyDeviceToDevice, s));
    if (evecs)
      SCSF_CUDA_CHECK(cudaMemcpy2DAsync(evecs + (int64_t)k * L * ld_vec, ld_vec * sizeof(double), w.V,
                                        w.ldv * sizeof(double), w.n * sizeof(double), L, cudaMemcpyDeviceToDevice,
                                        s));
    if (sink) {
      const int b = k & 1;
      if (k >= 2) SCSF_CUDA_CHECK(cudaStreamWaitEvent(s, done[b], 0));   // staging b is free again
      SCSF_CUDA_CHECK(cudaMemcpyAsync(sink->stage_ev[b], w.theta_sorted, L * sizeof(double),
                                      cudaMemcpyDeviceToDevice, s));
      if (sink->evecs)
        SCSF_CUDA_CHECK(cudaMemcpy2DAsync(sink->stage[b], w.ldv * sizeof(double), w.V, w.ldv * sizeof(double),
                                          w.n * sizeof(double), L, cudaMemcpyDeviceToDevice, s));
      SCSF_CUDA_CHECK(cudaEventRecord(ready[b], s));
      SCSF_CUDA_CHECK(cudaStreamWaitEvent(cs, ready[b], 0));
      SCSF_CUDA_CHECK(cudaMemcpyAsync(sink->evals + (int64_t)k * L, sink->stage_ev[b], L * sizeof(double),
                                      cudaMemcpyDeviceToHost, cs));
      if (sink->evecs)
        SCSF_CUDA_CHECK(cudaMemcpy2DAsync(sink->evecs + (int64_t)k * L * sink->ld, sink->ld * sizeof(double),
                                          sink->stage[b], w.ldv * sizeof(double), w.n * sizeof(double), L,
                                          cudaMemcpyDeviceToHost, cs));
      SCSF_CUDA_CHECK(cudaEventRecord(done[b], cs));
    }
  }
  if (state_out && n_chain > 0) {
    SCSF_CUDA_CHECK(cudaMemcpyAsync(state_out, w.theta_sorted, bb * sizeof(double), cudaMemcpyDeviceToDevice, s));
    SCSF_CUDA_CHECK(cudaMemcpy2DAsync(state_out + bb, w.n * sizeof(double), w.V, w.ldv * sizeof(double),
                                      w.n * sizeof(double), bb, cudaMemcpyDeviceToDevice, s));
  }
  SCSF_CUDA_CHECK(cudaStreamSynchronize(s));
  return worst;
  }();
  cleanup();
  return r;
}

static int check_queue(const scsf_ops* ops, const int32_t* queue, int32_t len, double* evals, double* evecs,
                       int64_t ld_vec) {
  int64_t n = (int64_t)ops->nx * ops->ny * ops->nz;
  SCSF_ARG_CHECK(len >= 0, "chain length must be >= 0");
  SCSF_ARG_CHECK(len == 0 || queue != nullptr, "chain is NULL");
  SCSF_ARG_CHECK(len == 0 || evals != nullptr, "evals is NULL");
  SCSF_ARG_CHECK(evecs == nullptr || ld_vec >= n, "ld_vec must be >= n");
  for (int k = 0; k < len; ++k)
    SCSF_ARG_CHECK(queue[k] >= 0 && queue[k] < ops->n_ops, "chain[%d]=%d out of range", k, queue[k]);
  return SCSF_OK;
}

int scsf_solve_queue(const scsf_ops* ops, const int32_t* chain, int32_t n_chain, int32_t L, int32_t nex,
                     int32_t degree, double tol, int32_t max_iter, uint64_t seed, double* evals, double* evecs,
                     int64_t ld_vec, scsf_stats* st, void* ws, size_t ws_bytes, void* stream) {
  SCSF_TRY(check_solve_args(ops, L, nex, degree, tol, max_iter));
  SCSF_TRY(check_queue(ops, chain, n_chain, evals, evecs, ld_vec));
  if (n_chain == 0) return SCSF_OK;
  SCSF_TRY(init_kernel_attrs());
  SolveWS w;
  SCSF_TRY(carve_solve_ws(ops, L, nex, ws, ws_bytes, w));
  cudaStream_t s = (cudaStream_t)stream;
  if (s != nullptr) return run_chain(ops, chain, n_chain, L, nex, degree, tol, max_iter, seed, evals, evecs, ld_vec, st, w, s);
  // the legacy default stream cannot be captured into a graph: run on a private stream
  SCSF_CUDA_CHECK(cudaStreamSynchronize(nullptr));
  cudaStream_t ps = nullptr;
  SCSF_CUDA_CHECK(cudaStreamCreateWithFlags(&ps, cudaStreamNonBlocking));
  const int r = run_chain(ops, chain, n_chain, L, nex, degree, tol, max_iter, seed, evals, evecs, ld_vec, st, w, ps);
  cudaStreamSynchronize(ps);
  cudaStreamDestroy(ps);
  return r;
}

static int64_t state_doubles(const scsf_ops* ops, int L, int nex) {
  return (int64_t)(L + nex) * (1 + (int64_t)ops->nx * ops->ny * ops->nz);
}

static int solve_chains_impl(const scsf_ops* ops, const int32_t* queue, const int32_t* chain_start,
                             int32_t n_chains, int32_t L, int32_t nex, int32_t degree, double tol, int32_t max_iter,
                             uint64_t seed, double* evals, double* evecs, int64_t ld_vec, scsf_stats* st, void* ws,
                             size_t ws_bytes, void* stream, double* evals_host, double* evecs_host,
                             int64_t ld_host, const double* state_in = nullptr, double* state_out = nullptr);

int64_t scsf_chain_state_doubles(const scsf_ops* ops, int32_t L, int32_t nex) {
  if (!ops || L < 1 || nex < 0) return 0;
  return state_doubles(ops, L, nex);
}

int scsf_solve_chains_resume(const scsf_ops* ops, const int32_t* queue, const int32_t* chain_start,
                             int32_t n_chains, int32_t L, int32_t nex, int32_t degree, double tol, int32_t max_iter,
                             uint64_t seed, const double* state_in, double* state_out, double* evals, double* evecs,
                             int64_t ld_vec, scsf_stats* st, void* ws, size_t ws_bytes, void* stream) {
  SCSF_ARG_CHECK(state_out != nullptr, "state_out is NULL");
  SCSF_ARG_CHECK(state_in != state_out, "state_in and state_out must not alias");
  return solve_chains_impl(ops, queue, chain_start, n_chains, L, nex, degree, tol, max_iter, seed, evals, evecs,
                           ld_vec, st, ws, ws_bytes, stream, nullptr, nullptr, 0, state_in, state_out);
}

static size_t sink_bytes(const scsf_ops* ops, int L) {
  const int64_t ldv = round_up((int64_t)ops->nx * ops->ny * ops->nz, 32);
  return (size_t)round_up(2 * ldv * L * (int64_t)sizeof(double), 256) + (size_t)round_up(2 * L * 8, 256);
}

size_t scsf_solve_chains_host_workspace_bytes(const scsf_ops* ops, int32_t L, int32_t nex) {
  if (!ops) return 0;
  return solve_ws_bytes(ops, L, nex) + sink_bytes(ops, L);
}

int scsf_solve_chains_host(const scsf_ops* ops, const int32_t* queue, const int32_t* chain_start,
                           int32_t n_chains, int32_t L, int32_t nex, int32_t degree, double tol, int32_t max_iter,
                           uint64_t seed, double* evals_host, double* evecs_host, int64_t ld_host, scsf_stats* st,
                           void* ws, size_t ws_bytes, void* stream) {
  SCSF_ARG_CHECK(evals_host != nullptr, "evals_host is NULL");
  SCSF_ARG_CHECK(ops == nullptr || evecs_host == nullptr || ld_host >= (int64_t)ops->nx * ops->ny * ops->nz,
                 "ld_host must be >= n");
  return solve_chains_impl(ops, queue, chain_start, n_chains, L, nex, degree, tol, max_iter, seed, nullptr, nullptr,
                           0, st, ws, ws_bytes, stream, evals_host, evecs_host, ld_host);
}

int scsf_solve_chains(const scsf_ops* ops, const int32_t* queue, const int32_t* chain_start, int32_t n_chains,
                      int32_t L, int32_t nex, int32_t degree, double tol, int32_t max_iter, uint64_t seed,
                      double* evals, double* evecs, int64_t ld_vec, scsf_stats* st, void* ws, size_t ws_bytes,
                      void* stream) {
  return solve_chains_impl(ops, queue, chain_start, n_chains, L, nex, degree, tol, max_iter, seed, evals, evecs,
                           ld_vec, st, ws, ws_bytes, stream, nullptr, nullptr, 0);
}

static int solve_chains_impl(const scsf_ops* ops, const int32_t* queue, const int32_t* chain_start,
                             int32_t n_chains, int32_t L, int32_t nex, int32_t degree, double tol, int32_t max_iter,
                             uint64_t seed, double* evals, double* evecs, int64_t ld_vec, scsf_stats* st, void* ws,
                             size_t ws_bytes, void* stream, double* evals_host, double* evecs_host,
                             int64_t ld_host, const double* state_in, double* state_out) {
  const bool to_host = evals_host != nullptr;
  SCSF_TRY(check_solve_args(ops, L, nex, degree, tol, max_iter));
  SCSF_ARG_CHECK(n_chains >= 1 && chain_start != nullptr, "n_chains >= 1 and chain_start required");
  SCSF_ARG_CHECK(chain_start[0] == 0, "chain_start[0] must be 0");
  for (int c = 0; c < n_chains; ++c)
    SCSF_ARG_CHECK(chain_start[c + 1] >= chain_start[c], "chain_start must be non-decreasing");
  const int32_t len = chain_start[n_chains];
  SCSF_TRY(check_queue(ops, queue, len, to_host ? evals_host : evals, evecs, ld_vec));
  if (len == 0 && !state_out) return SCSF_OK;
  const size_t per_solve = solve_ws_bytes(ops, L, nex);
  const size_t per = per_solve + (to_host ? sink_bytes(ops, L) : 0);
  if (!ws || ws_bytes < per * (size_t)n_chains) {
    set_error("workspace too small: need %zu bytes (%d chains), got %zu", per * (size_t)n_chains, n_chains,
              ws_bytes);
    return SCSF_ERR_WORKSPACE;
  }
  cudaStream_t caller = (cudaStream_t)stream;
  SCSF_TRY(init_kernel_attrs());
  SCSF_CUDA_CHECK(cudaStreamSynchronize(caller));   // inputs produced on the caller's stream are ready
  int dev = 0;
  SCSF_CUDA_CHECK(cudaGetDevice(&dev));
  std::vector<int> status(n_chains, SCSF_OK);
  std::vector<std::string> msg(n_chains);
  auto worker = [&](int c) {
    cudaSetDevice(dev);
    cudaStream_t s = nullptr;
    if (cudaStreamCreateWithFlags(&s, cudaStreamNonBlocking) != cudaSuccess) {
      status[c] = SCSF_ERR_DEVICE;
      msg[c] = "cudaStreamCreate failed";
      return;
    }
    SolveWS w;
    char* base = (char*)ws + per * (size_t)c;
    int r = carve_solve_ws(ops, L, nex, base, per_solve, w);
    const int32_t b0 = chain_start[c], cnt = chain_start[c + 1] - chain_start[c];
    HostSink sink;
    if (to_host) {
      Arena a(base + per_solve, per - per_solve);
      double* st2 = a.take<double>(2 * w.ldv * L);
      double* se2 = a.take<double>(2 * L);
      sink.stage[0] = st2;
      sink.stage[1] = st2 + w.ldv * L;
      sink.stage_ev[0] = se2;
      sink.stage_ev[1] = se2 + L;
      sink.evals = evals_host + (int64_t)b0 * L;
      sink.evecs = evecs_host ? evecs_host + (int64_t)b0 * L * ld_host : nullptr;
      sink.ld = ld_host;
    }
    const int64_t sd = state_doubles(ops, L, nex);
    const double* sin_c = state_in ? state_in + sd * c : nullptr;
    double* sout_c = state_out ? state_out + sd * c : nullptr;
    if (r == SCSF_OK && cnt > 0)
      r = run_chain(ops, queue + b0, cnt, L, nex, degree, tol, max_iter, seed,
                    evals ? evals + (int64_t)b0 * L : nullptr, evecs ? evecs + (int64_t)b0 * L * ld_vec : nullptr,
                    ld_vec, st ? st + b0 : nullptr, w, s, to_host ? &sink : nullptr, sin_c, sout_c);
    else if (r == SCSF_OK && sout_c && sout_c != sin_c) {   // an empty slice carries its state through
      cudaError_t e = sin_c ? cudaMemcpyAsync(sout_c, sin_c, sd * sizeof(double), cudaMemcpyDeviceToDevice, s)
                            : cudaMemsetAsync(sout_c, 0xff, sd * sizeof(double), s);   // NaN: no state
      if (e != cudaSuccess) {
        r = SCSF_ERR_DEVICE;
        set_error("state copy: %s", cudaGetErrorString(e));
      }
    }
    status[c] = r;
    if (r != SCSF_OK) msg[c] = scsf_last_error();
    cudaStreamSynchronize(s);
    cudaStreamDestroy(s);
  };
  std::vector<std::thread> th;
  th.reserve(n_chains);
  for (int c = 0; c < n_chains; ++c) th.emplace_back(worker, c);
  for (auto& t : th) t.join();
  int worst = SCSF_OK;
  for (int c = 0; c < n_chains; ++c) {
    const int r = status[c];
    if (r != SCSF_OK && r != SCSF_ERR_NUMERICAL) {
      set_error("chain %d: %s", c, msg[c].c_str());
      return r;
    }
    if (r > worst) {
      worst = r;
      set_error("chain %d: %s", c, msg[c].c_str());
    }
  }
  return worst;
}

size_t scsf_dev_workspace_bytes(int64_t n, int32_t b1, int32_t b2) {
  Arena a(nullptr, 0);
  const int bm = b1 > b2 ? b1 : b2;
  a.take<double>((int64_t)tn_partial_doubles(n, b1, b2));
  a.take<double>(3 * (int64_t)bm * bm + 2);
  a.take<double>((int64_t)small_scratch_doubles(bm));
  a.take<Ctrl>(1);
  return a.off;
}

int scsf_gemm_tn(const double* X, int64_t ldx, int32_t b1, const double* Y, int64_t ldy, int32_t b2, int64_t n,
                 double alpha, int32_t upper, double* C, int64_t ldc, void* ws, size_t ws_bytes, void* stream) {
  SCSF_ARG_CHECK(X && Y && C && b1 >= 1 && b2 >= 1 && n >= 1, "bad gemm_tn arguments");
  SCSF_ARG_CHECK(ldx >= n && ldy >= n && ldc >= b1, "bad leading dimensions");
  SCSF_ARG_CHECK(!upper || b1 == b2, "upper requires b1 == b2");
  Arena a(ws, ws_bytes);
  double* P = a.take<double>((int64_t)tn_partial_doubles(n, b1, b2));
  if (a.overflow || !ws) {
    set_error("workspace too small");
    return SCSF_ERR_WORKSPACE;
  }
  SCSF_TRY(init_kernel_attrs());
  cudaStream_t s = (cudaStream_t)stream;
  SCSF_TRY(gemm_tn(X, ldx, b1, Y, ldy, b2, n, alpha, upper, C, ldc, P, s));
  SCSF_CUDA_CHECK(cudaStreamSynchronize(s));
  return SCSF_OK;
}

int scsf_gemm_nn(const double* X, int64_t ldx, int64_t n, int32_t b1, const double* M, int64_t ldm, int32_t b2,
                 double alpha, double beta, double* Out, int64_t ldo, void* stream) {
  SCSF_ARG_CHECK(X && M && Out && b1 >= 1 && b2 >= 1 && n >= 1, "bad gemm_nn arguments");
  SCSF_ARG_CHECK(ldx >= n && ldo >= n && ldm >= b1, "bad leading dimensions");
  SCSF_ARG_CHECK(Out != X || ldo == ldx, "in-place needs ldo == ldx");
  SCSF_TRY(init_kernel_attrs());
  cudaStream_t s = (cudaStream_t)stream;
  SCSF_TRY(gemm_nn(X, ldx, n, b1, M, ldm, b2, alpha, beta, Out, ldo, s));
  SCSF_CUDA_CHECK(cudaStreamSynchronize(s));
  return SCSF_OK;
}

int scsf_chol_inv(const double* S, int64_t lds, int32_t b, int64_t nrows, double* Rinv, void* ws, size_t ws_bytes,
                  void* stream) {
  SCSF_ARG_CHECK(S && Rinv && b >= 1 && b <= 384 && lds >= b, "bad chol_inv arguments");
  Arena a(ws, ws_bytes);
  double* scratch = a.take<double>((int64_t)small_scratch_doubles(b));
  Ctrl* ctrl = a.take<Ctrl>(1);
  if (a.overflow || !ws) {
    set_error("workspace too small");
    return SCSF_ERR_WORKSPACE;
  }
  SCSF_TRY(init_kernel_attrs());
  cudaStream_t s = (cudaStream_t)stream;
  SCSF_CUDA_CHECK(cudaMemsetAsync(ctrl, 0, sizeof(Ctrl), s));
  SCSF_TRY(chol_inv_impl(S, lds, b, nrows, Rinv, scratch, ctrl, s));
  Ctrl h{};
  SCSF_CUDA_CHECK(cudaMemcpyAsync(&h, ctrl, sizeof(Ctrl), cudaMemcpyDeviceToHost, s));
  SCSF_CUDA_CHECK(cudaStreamSynchronize(s));
  if (h.chol_fail) {
    set_error("Gram matrix not numerically SPD: shifted factor returned");
    return SCSF_ERR_NUMERICAL;
  }
  return SCSF_OK;
}

int scsf_syev_small(const double* G, int64_t ldg, int32_t b, double* theta, double* Z, int32_t* sweeps, void* ws,
                    size_t ws_bytes, void* stream) {
  SCSF_ARG_CHECK(G && theta && Z && b >= 1 && b <= 384 && ldg >= b, "bad syev_small arguments");
  Arena a(ws, ws_bytes);
  double* g = a.take<double>((int64_t)small_scratch_doubles(b));
  double* zw = a.take<double>((int64_t)b * b);
  Ctrl* ctrl = a.take<Ctrl>(1);
  if (a.overflow || !ws) {
    set_error("workspace too small");
    return SCSF_ERR_WORKSPACE;
  }
  SCSF_TRY(init_kernel_attrs());
  cudaStream_t s = (cudaStream_t)stream;
  SCSF_CUDA_CHECK(cudaMemsetAsync(ctrl, 0, sizeof(Ctrl), s));
  SCSF_TRY(jacobi_impl(G, ldg, b, g, zw, theta, Z, ctrl, s));
  Ctrl h{};
  SCSF_CUDA_CHECK(cudaMemcpyAsync(&h, ctrl, sizeof(Ctrl), cudaMemcpyDeviceToHost, s));
  SCSF_CUDA_CHECK(cudaStreamSynchronize(s));
  if (sweeps) *sweeps = h.pad[0];
  if (h.nonfinite & 2) {
    set_error("Jacobi did not converge within the sweep cap");
    return SCSF_ERR_NUMERICAL;
  }
  return SCSF_OK;
}


/* ---------------------------------------------- row-partitioned solve ---- */
struct scsf_comm;   // opaque: a scsf::Comm

int scsf_comm_unique_id(void* id128) {
  SCSF_ARG_CHECK(id128 != nullptr, "id128 is NULL");
  return comm_unique_id(id128);
}

int scsf_comm_create(int32_t rank, int32_t world, const void* id128, scsf_comm** out) {
  SCSF_ARG_CHECK(out && id128, "NULL argument");
  SCSF_ARG_CHECK(world >= 1 && rank >= 0 && rank < world, "bad rank / world");
  Comm* c = nullptr;
  SCSF_TRY(comm_create_nccl(rank, world, id128, &c));
  *out = reinterpret_cast<scsf_comm*>(c);
  return SCSF_OK;
}

int scsf_comm_create_loopback(int32_t world, scsf_comm** out) {
  SCSF_ARG_CHECK(out && world >= 1, "bad loopback arguments");
  std::vector<Comm*> cs(world, nullptr);
  SCSF_TRY(comm_create_loopback(world, cs.data()));
  for (int r = 0; r < world; ++r) out[r] = reinterpret_cast<scsf_comm*>(cs[r]);
  return SCSF_OK;
}

int scsf_comm_destroy(scsf_comm* c) {
  delete reinterpret_cast<Comm*>(c);
  return SCSF_OK;
}

int scsf_comm_rank(const scsf_comm* c, int32_t* rank, int32_t* world) {
  SCSF_ARG_CHECK(c != nullptr, "comm is NULL");
  const Comm* cc = reinterpret_cast<const Comm*>(c);
  if (rank) *rank = cc->rank;
  if (world) *world = cc->world;
  return SCSF_OK;
}

void scsf_slab_rows(int32_t ny, int32_t world, int32_t rank, int32_t* y0, int32_t* y1) {
  if (y0) *y0 = (int32_t)(((int64_t)rank * ny) / world);
  if (y1) *y1 = (int32_t)(((int64_t)(rank + 1) * ny) / world);
}

static int check_dist(const scsf_ops* ops, int32_t y0, int32_t y1, const scsf_comm* comm) {
  SCSF_ARG_CHECK(comm != nullptr, "comm is NULL");
  if (ops->stencil != SCSF_STENCIL_FLUX) {
    set_error("the row-partitioned solve supports the flux-form stencil only");
    return SCSF_ERR_NOT_IMPLEMENTED;
  }
  SCSF_ARG_CHECK(ops->dim == 2, "the row-partitioned solve is 2-D (got dim %d)", ops->dim);
  SCSF_ARG_CHECK(ops->nx % 4 == 0, "the row-partitioned solve needs nx %% 4 == 0 (got %d)", ops->nx);
  SCSF_ARG_CHECK(0 <= y0 && y0 < y1 && y1 <= ops->ny, "slab rows [%d, %d) invalid for ny = %d", y0, y1, ops->ny);
  const Comm* c = reinterpret_cast<const Comm*>(comm);
  int32_t e0, e1;
  scsf_slab_rows(ops->ny, c->world, c->rank, &e0, &e1);
  SCSF_ARG_CHECK(e0 == y0 && e1 == y1, "slab rows [%d, %d) differ from scsf_slab_rows [%d, %d)", y0, y1, e0, e1);
  return SCSF_OK;
}

size_t scsf_solve_dist_workspace_bytes(const scsf_ops* ops, int32_t y0, int32_t y1, int32_t L, int32_t nex,
                                       int32_t world) {
  if (!ops || world < 1 || y1 <= y0) return 0;
  struct FakeComm final : Comm {
    int allreduce_sum(double*, size_t, cudaStream_t) override { return 0; }
    int allreduce_max_u64(unsigned long long*, size_t, cudaStream_t) override { return 0; }
    int allgather(const double*, double*, size_t, cudaStream_t) override { return 0; }
    int halo(const double*, const double*, double*, double*, size_t, cudaStream_t) override { return 0; }
  } fake;
  fake.world = world;
  DistCtx d;
  d.comm = &fake;
  d.y0 = y0;
  d.y1 = y1;
  return solve_ws_bytes(ops, L, nex, &d);
}

int scsf_solve_queue_dist(const scsf_ops* ops, int32_t y0, int32_t y1, const int32_t* chain, int32_t n_chain,
                          int32_t L, int32_t nex, int32_t degree, double tol, int32_t max_iter, uint64_t seed,
                          double* evals, double* evecs_local, int64_t ld_vec, scsf_stats* st, scsf_comm* comm,
                          void* ws, size_t ws_bytes, void* stream) {
  SCSF_TRY(check_solve_args(ops, L, nex, degree, tol, max_iter));
  SCSF_TRY(check_dist(ops, y0, y1, comm));
  SCSF_TRY(check_queue(ops, chain, n_chain, evals, nullptr, ld_vec));
  const int64_t n_loc = (int64_t)ops->nx * (y1 - y0);
  SCSF_ARG_CHECK(evecs_local == nullptr || ld_vec >= n_loc, "ld_vec must be >= the slab's rows x nx");
  if (n_chain == 0) return SCSF_OK;
  SCSF_TRY(init_kernel_attrs());
  DistCtx d;
  d.comm = reinterpret_cast<Comm*>(comm);
  d.y0 = y0;
  d.y1 = y1;
  SolveWS w;
  SCSF_TRY(carve_solve_ws(ops, L, nex, ws, ws_bytes, w, &d));
  return run_chain(ops, chain, n_chain, L, nex, degree, tol, max_iter, seed, evals, evecs_local, ld_vec, st, w,
                   (cudaStream_t)stream);
}

}  // extern "C"
