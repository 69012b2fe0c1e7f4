/*
 * scsf.h — C ABI of libscsf.so, the sm_100a hot path of SCSF
 * (Sorting Chebyshev Subspace Filter, arXiv 2510.23215).
 *
 * Citations "P:n" are lines of the paper text /root/reference/PAPER.md
 * (section / algorithm named alongside); DESIGN.md lists every reading taken
 * where the paper is silent (R1..R24).
 *
 * Conventions shared by every entry point
 *  - Plain C types only.  `stream` is a cudaStream_t passed as void* (NULL =
 *    legacy default stream).  Every call is synchronous on return: it
 *    enqueues its kernels on `stream` and synchronises that stream.
 *  - Device pointers ("dev") are caller-owned (the Python side allocates them
 *    with torch); host pointers ("host") are plain CPU memory.  The library
 *    never allocates or frees device memory; scratch space comes from the
 *    caller's `ws` (device, 256-byte aligned, at least the size reported by
 *    the matching *_workspace_bytes query).
 *  - Vector blocks are fp64, column-major: column j of an n-row block starts
 *    at ptr + j*ld, with ld >= n.  Unknowns are ordered x fastest:
 *    k = ix + nx*(iy + ny*iz)  (row-major grid order, Eq. 2).
 *  - Return value: scsf_status.  On failure scsf_last_error() returns a
 *    thread-local message.  No exception or abort crosses the ABI.
 *  - Not re-entrant on one stream; distinct streams/devices are independent.
 */
#ifndef SCSF_H_
#define SCSF_H_

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define SCSF_ABI_VERSION 2

typedef enum {
  SCSF_OK = 0,
  SCSF_ERR_ARG = 1,             /* invalid argument (shape, range, NULL)            */
  SCSF_ERR_NUMERICAL = 2,       /* not converged in max_iter / QR breakdown          */
  SCSF_ERR_DEVICE = 3,          /* CUDA error (launch, memcpy, sync)                 */
  SCSF_ERR_NOT_IMPLEMENTED = 4, /* configuration not supported by this build         */
  SCSF_ERR_WORKSPACE = 5        /* ws NULL or ws_bytes below the queried size        */
} scsf_status;

/*
 * A batch of discretised operators A^(i), i = 0..n_ops-1 (Eq. 3),
 * each a real symmetric 5-point (dim 2) or 7-point (dim 3) stencil, stored
 * as symmetric DIA arrays in device memory:
 *   coef[(i*(1+dim) + 0)*ld + k] = A(k, k)           (diag)
 *   coef[(i*(1+dim) + 1)*ld + k] = A(k, k+1)         (cx; 0 when ix = nx-1)
 *   coef[(i*(1+dim) + 2)*ld + k] = A(k, k+nx)        (cy; 0 when iy = ny-1)
 *   coef[(i*(1+dim) + 3)*ld + k] = A(k, k+nx*ny)     (cz; dim 3; 0 when iz = nz-1)
 * ld >= n = nx*ny*nz, multiple of 32.  Produced by scsf_assemble() or by the
 * caller.  The matrix must be symmetric positive definite for the solve
 * (R20: flux form); eigenvalues are returned ascending, which is
 * the |lambda| order of P:150 for SPD operators.
 */
typedef struct {
  int32_t dim;          /* 2 or 3                                        */
  int32_t nx, ny, nz;   /* interior grid size (nz = 1 when dim == 2)     */
  int32_t n_ops;        /* operators in the batch                        */
  int32_t stencil;      /* SCSF_STENCIL_FLUX (0) or SCSF_STENCIL_VIB13 (1) */
  int64_t ld;           /* stride between coefficient arrays (doubles)   */
  const double* coef;   /* dev [n_ops][scsf_ncoef][ld]                   */
} scsf_ops;

/*
 * Stencil kinds.  SCSF_STENCIL_FLUX: the layout above, 1 + dim arrays.
 * SCSF_STENCIL_VIB13 (dim 2 only): the standard form B of the thin-plate
 * vibration pencil (reading R25; scsf_assemble_vibration), a
 * symmetric 13-point stencil in 7 arrays, k = ix + nx*iy:
 *   coef[(i*7 + 0)*ld + k] = B(k, k)
 *   coef[(i*7 + 1)*ld + k] = B(k, k+1)       (0 when ix = nx-1)
 *   coef[(i*7 + 2)*ld + k] = B(k, k+2)       (0 when ix >= nx-2)
 *   coef[(i*7 + 3)*ld + k] = B(k, k+nx-1)    (0 when ix = 0 or iy = ny-1)
 *   coef[(i*7 + 4)*ld + k] = B(k, k+nx)      (0 when iy = ny-1)
 *   coef[(i*7 + 5)*ld + k] = B(k, k+nx+1)    (0 when ix = nx-1 or iy = ny-1)
 *   coef[(i*7 + 6)*ld + k] = B(k, k+2nx)     (0 when iy >= ny-2)
 * The filter runs the per-step streaming stencil for this kind, and the
 * row-partitioned solve (scsf_solve_queue_dist) does not support it.
 */
enum { SCSF_STENCIL_FLUX = 0, SCSF_STENCIL_VIB13 = 1 };

/* Per-operator statistics (SPEC S:384-388 SolveRecord fields; P:463-479 Tab. sort1). */
typedef struct {
  int32_t status;            /* scsf_status of this operator                          */
  int32_t iterations;        /* outer ChFSI iterations (Alg. 3 repeat loop)    */
  int32_t filter_steps;      /* Chebyshev three-term steps applied (sum over iters)   */
  int32_t cholqr_fallbacks;  /* shifted-CholQR fallbacks taken                        */
  int32_t n_locked;          /* converged pairs locked at exit (>= L on success)      */
  int32_t warm;              /* 1 if started from the previous operator's block       */
  int64_t spmm_columns;      /* stencil applications x columns (filter + RR)          */
  double max_rel_resid;      /* max over returned pairs of ||Av - lv|| / ||Av|| */
  double beta;               /* spectral upper bound used by the filter (Gershgorin)  */
  /* phase timers, CUDA events on the launching stream (0 unless scsf_set_timing(1)) */
  double t_filter_ms;        /* Chebyshev filter steps (Alg. 1)                       */
  double t_ortho_ms;         /* BCGS2 against locked + CholQR2 (Alg. 3 l. 4)          */
  double t_rr_ms;            /* Rayleigh-Ritz + residuals + locking (ll. 5-7)          */
  double filter_bytes;       /* algorithmic HBM bytes of the filter steps */
  int32_t jacobi_sweeps;     /* reduced-eigensolver sweeps, summed over RR steps      */
  int32_t cold_retry;        /* 1 if a warm start broke down and the operator was     */
                             /* solved again from a random block (R29); the counts    */
                             /* above include both attempts                           */
  double t_gemm_ms;          /* tall-skinny DGEMM tiles (Gram / projection / rotation),
                                CUDA events around each launch (0 unless timing is on)  */
  double gemm_flops;         /* their algorithmic flops (upper-triangle Grams: unique
                                entries; triangular R^-1: half) (0 unless timing is on) */
} scsf_stats;

/* ---------------------------------------------------------------- sort ---- */

/* Workspace for scsf_sort / scsf_signatures (bytes). */
size_t scsf_sort_workspace_bytes(int32_t N, int32_t dim, int32_t p, int32_t F, int32_t p0);

/*
 * Truncated-FFT greedy ordering, Alg. 2.
 *  params  dev [N][F][p^dim] fp64, x fastest: the parameter matrices P^(i)
 *          (nodal coefficient values, R7), F fields per problem (R6).
 *  p0      truncation: modes k in [-p0/2, p0/2-1]^dim are kept (R1);
 *          even, 2 <= p0 <= p.
 *  start   first problem ("i_0 = 1", 0-based here).
 *  perm    host [N] out: solve order seq_mat, a permutation of 0..N-1.
 *  d2_best host [N-1] out or NULL: squared Frobenius distance of each greedy step.
 *  d2_second host [N-1] out or NULL: runner-up squared distance (inf if none).
 * Distances are compared squared (R5); ties go to the lowest index (strict `<`,
 * P:243, R4); `dis = 1000` is read as +inf (R3).
 * Errors: SCSF_ERR_ARG (N < 1, dim not 2/3, p0 odd or > p, start out of range).
 */
int scsf_sort(const double* params, int32_t N, int32_t dim, int32_t p, int32_t F,
              int32_t p0, int32_t start, int32_t* perm, double* d2_best,
              double* d2_second, void* ws, size_t ws_bytes, void* stream);

/*
 * Alg. 2 ll. 3-5 only: sig dev [N][F*p0^dim] complex128 (interleaved re, im),
 * C order [f][kz][ky][kx], k from -p0/2: the unnormalised DFT
 * S[k] = sum_x P[x] exp(-2 pi i <k,x>/p) at the kept modes (R1, R2).
 */
int scsf_signatures(const double* params, int32_t N, int32_t dim, int32_t p, int32_t F,
                    int32_t p0, double* sig, void* ws, size_t ws_bytes, void* stream);

/* ------------------------------------------------------------ operators ---- */

/*
 * Thin-plate vibration operators ("Lap(D Lap u) =
 * lambda rho u", reading R25):  B = diag(rho)^-1/2 Lh diag(D) Lh diag(rho)^-1/2,
 * Lh the 5-point Dirichlet -Lap_h (4 u_k - neighbours)/h^2, so per entry
 *   h^4 sqrt(rho_k rho_l) B(k,l) = 16 D_k + sum of D over k's in-grid x/y neighbours   (l = k)
 *                              = -4 (D_k + D_l)                 (l = k+1 or k+nx, same row / column)
 *                              = D_m                            (l = k+2 or k+2nx, m the point between)
 *                              = D of the two common neighbours (l = k+nx+-1, diagonal)
 * ops->stencil must be SCSF_STENCIL_VIB13, ops->dim 2.
 *  D, rho  dev, operator i's nodal fields at D + i*field_stride, rho + i*field_stride
 *          (x fastest; field_stride >= n; both > 0 — e.g. params [N][2][n] with
 *          rho = params + n and field_stride = 2n)
 *  coef_out dev [n_ops][7][ld]; pads k >= n with 0.
 */
int scsf_assemble_vibration(const scsf_ops* ops, double h, const double* D, const double* rho,
                            int64_t field_stride, double* coef_out, void* stream);

/*
 * Coefficient fields of a batch on the device (Fig. 1 steps 1-2,
 * P:49; the paper gives no GRF recipe, P:759/789/807 — this is DESIGN.md §3's):
 *   g(x) = sum_{k in {1..K}^dim} xi_k (1 + |k|^2)^(-s) prod_d sin(pi k_d x_d),
 *   g <- g * sigma / s_K when sigma > 0, s_K = sqrt(sum_k (1+|k|^2)^(-2s) / 2^dim),
 * at nodes x_i = (i+1) h and face midpoints (i+1/2) h, h = 1/(nx+1); then
 *   family 0 (diva,  -div(a grad u)):         faces = vscale e^g, c = 0, P0 = vscale e^g(nodes)
 *   family 1 (lapv,  -Lap u + V u):           faces = 1, c = P0 = vscale e^g(nodes)
 *   family 2 (divac, -div(a grad u) + c u):   faces = e^{g_a}, P0 = e^{g_a}, c = P1 = e^{g_c}
 *   family 3 (vib, Lap(D Lap u) = l rho u):   P0 = D = e^{g_0}, P1 = rho = e^{g_1}; faces, c unused
 *                                             (may be NULL; feed P to scsf_assemble_vibration)
 *  xi       dev [n_ops][F][K^dim] standard normal draws (F = 2 for divac / vib, else 1),
 *           C order [kx][ky](kz) — drawn by the caller, so a batch is reproducible
 *  faces_*  dev out, layouts as scsf_assemble's inputs; c dev [n_ops][n] out;
 *  params   dev [n_ops][F][n] out (scsf_sort's parameter matrices)
 *  ws       dev >= scsf_grf_workspace_bytes(nx, K) (basis tables)
 * Limits: dim 2: K <= 32; dim 3: K^3 <= 1024 and nx <= 63.
 * Errors: SCSF_ERR_ARG, SCSF_ERR_WORKSPACE, SCSF_ERR_DEVICE.  Synchronises the stream.
 */
size_t scsf_grf_workspace_bytes(int32_t nx, int32_t K);
int scsf_grf_fields(int32_t dim, int32_t nx, int32_t K, double s, double sigma, double vscale,
                    int32_t family, int32_t n_ops, const double* xi, double* faces_x,
                    double* faces_y, double* faces_z, double* c, double* params, void* ws,
                    size_t ws_bytes, void* stream);

/*
 * Flux-form FD assembly (App. B; reading R20):
 *   A(k,k) = sum of the 2*dim face coefficients around node k / h^2 + c[k],
 *   A(k,k+s_d) = -a(face between k and k+s_d) / h^2.
 * faces_x dev [n_ops][nz][ny][nx+1], faces_y dev [n_ops][nz][ny+1][nx],
 * faces_z dev [n_ops][nz+1][ny][nx] (dim 3, else NULL), c dev [n_ops][n]
 * (NULL = 0); h = 1/(nx+1).  Writes ops->coef (cast away const: the caller
 * owns it) for all n_ops operators; pads k >= n with 0.
 */
int scsf_assemble(const scsf_ops* ops, double h, const double* faces_x,
                  const double* faces_y, const double* faces_z, const double* c,
                  double* coef_out, void* stream);

/* ------------------------------------------------------------- filter ---- */

/*
 * Chebyshev filter, Alg. 1 with uniform degree (R8):
 *   A~ = (A - cI)/e, sigma_1 = e/(lambda - c), Y_1 = sigma_1 A~ Y_0,
 *   sigma_{i+1} = 1/(2/sigma_1 - sigma_i),
 *   Y_{i+1} = 2 sigma_{i+1} A~ Y_i - sigma_{i+1} sigma_i Y_{i-1}.
 * Y0 dev [k][ldy] in; Ym dev [k][ldy] out (may not alias Y0).  ws: 2 blocks.
 * Errors: SCSF_ERR_ARG (degree < 1, e <= 0, lambda == c, ldy < n).
 */
size_t scsf_filter_workspace_bytes(const scsf_ops* ops, int32_t k, int64_t ldy);
int scsf_cheb_filter(const scsf_ops* ops, int32_t op_index, const double* Y0, int64_t ldy,
                     int32_t k, int32_t degree, double lambda, double c, double e,
                     double* Ym, void* ws, size_t ws_bytes, void* stream);

/* --------------------------------------------------------------- solve ---- */

/*
 * Workspace for scsf_solve_one / scsf_solve_queue with block b = L + nex.
 */
size_t scsf_solve_workspace_bytes(const scsf_ops* ops, int32_t L, int32_t nex);

/*
 * ChFSI for one operator, Alg. 3: the L smallest eigenpairs of
 * A^(op_index) to relative residual ||Av - lv||/||Av|| <= tol.
 *  nex       extra (inherited) subspace columns: block b = L + nex (R12)
 *  degree    Chebyshev filter degree m (default 20).  m in [1, 256]: every active
 *            column is filtered with degree m (reading R8).  m in [-256, -4]: per-column
 *            degrees (Alg. 1 l. 5's staggered update, the ChASE-style
 *            variant the paper cites): after each Rayleigh-Ritz step column j gets
 *            the degree its residual and Ritz value need to reach 0.1 tol, clamped to
 *            [4, |m|]; finished columns are left untouched by the remaining steps.
 *            Honoured by the resident filters, the vectorised streaming step
 *            (5-/7-point operators, nx % 4 == 0) and the row partition's slab step
 *            (scsf_solve_queue_dist); elsewhere (13-point family, scalar streaming
 *            step) it falls back to the uniform degree |m|.
 *            Conditioning guard (R28): each filter runs at most the degree
 *            for which C_m(t_lambda) = cosh(m acosh|(lambda - c)/e|) <= 1e8 (rounded
 *            down to = m mod 3, >= 4), so a degree past CholQR's stability ceiling
 *            is lowered on the device instead of breaking the orthonormalisation;
 *            below that ceiling m is used as given.  stats->filter_steps counts
 *            the steps actually run.
 *  max_iter  outer-iteration cap (R24; 200)
 *  warm_vecs dev [b][ld_vec] or NULL: initial block V~_0 ("V~_0 = V^(i-1)");
 *            NULL = seeded Gaussian start (R17), seed + op_index.
 *  evals     dev [b] out: Ritz values ascending; the first L are converged.
 *  evecs     dev [b][ld_vec] out: orthonormal Ritz vectors (sign: largest |.|
 *            entry positive, R21); may alias warm_vecs.
 *  ld_vec    leading dimension of warm_vecs / evecs (>= n).
 *  st        host out (may be NULL).
 * Errors: SCSF_ERR_ARG (L < 1, nex < 0, L + nex > n, degree outside [1, 256] and
 * [-256, -4], tol <= 0),
 * SCSF_ERR_WORKSPACE, SCSF_ERR_NUMERICAL (not converged; outputs hold the
 * best pairs found and st->max_rel_resid the worst residual).
 */
int scsf_solve_one(const scsf_ops* ops, int32_t op_index, int32_t L, int32_t nex,
                   int32_t degree, double tol, int32_t max_iter, const double* warm_vecs,
                   uint64_t seed, double* evals, double* evecs, int64_t ld_vec,
                   scsf_stats* st, void* ws, size_t ws_bytes, void* stream);

/*
 * SCSF sequential solve along a sorted chain (Fig. 2 d1-d3):
 * operator chain[0] starts from a seeded random block, every later one from
 * the previous operator's final b-block (warm start).  Reading R11 (P:193-194,
 * P:297 "Lambda~_0 = Lambda^(i-1)"): the first filter of a warm solve uses the
 * previous operator's Ritz values as its bounds (lambda = theta_1, alpha =
 * theta_b) with the new operator's Gershgorin beta; the first Rayleigh-Ritz
 * follows that filter.  The process-wide switch SCSF_INHERIT_BOUNDS=0 restores
 * one Rayleigh-Ritz of the new operator before the first filter.
 *  chain   host [n_chain]: operator indices in solve order (a slice of scsf_sort's perm)
 *  evals   dev [n_chain][L] out, by chain position
 *  evecs   dev [n_chain][L][ld_vec] out or NULL
 *  st      host [n_chain] out or NULL
 * A non-converged operator is recorded in st[k].status and the chain
 * continues; the return value is the worst status.
 */
int scsf_solve_queue(const scsf_ops* ops, const int32_t* chain, int32_t n_chain, int32_t L,
                     int32_t nex, int32_t degree, double tol, int32_t max_iter, uint64_t seed,
                     double* evals, double* evecs, int64_t ld_vec, scsf_stats* st,
                     void* ws, size_t ws_bytes, void* stream);

/*
 * Several warm-start chains of one queue solved concurrently on one GPU — the
 * paper's "N problems partitioned into M independent chunks, M instances of
 * SCSF in parallel" with a chunk per chain.  Chain c is
 * queue[chain_start[c] .. chain_start[c+1]) (contiguous slices of the sorted
 * order); each runs on its own host thread and CUDA stream with its own
 * workspace slice, so latency-bound kernels of different chains overlap.
 *  queue        host [chain_start[n_chains]]: operator indices
 *  chain_start  host [n_chains + 1], chain_start[0] = 0, non-decreasing
 *  evals / evecs / st  indexed by queue position (as scsf_solve_queue)
 *  ws_bytes     >= n_chains * scsf_solve_workspace_bytes(ops, L, nex)
 * The caller's stream is synchronised before the chains start; the call
 * returns when every chain has finished.  Return value: worst status.
 */
int scsf_solve_chains(const scsf_ops* ops, const int32_t* queue, const int32_t* chain_start,
                      int32_t n_chains, int32_t L, int32_t nex, int32_t degree, double tol,
                      int32_t max_iter, uint64_t seed, double* evals, double* evecs, int64_t ld_vec,
                      scsf_stats* st, void* ws, size_t ws_bytes, void* stream);

/*
 * scsf_solve_chains with the results streamed to pinned host memory while the
 * chains run ("streaming eigenpair writer"; Fig. 1 steps 5-6,
 * P:49): after each operator its L Ritz pairs are staged on the device
 * (double buffer per chain) and copied to the host on a second stream, so the
 * device-to-host traffic overlaps the next operator's solve.
 *  evals_host  host [len][L] (pinned), by queue position
 *  evecs_host  host [len][L][ld_host] (pinned) or NULL; ld_host >= n
 *  ws_bytes    >= n_chains * scsf_solve_chains_host_workspace_bytes(ops, L, nex)
 * Returns when every chain's copies have landed.  Errors as scsf_solve_chains.
 */
size_t scsf_solve_chains_host_workspace_bytes(const scsf_ops* ops, int32_t L, int32_t nex);
int scsf_solve_chains_host(const scsf_ops* ops, const int32_t* queue, const int32_t* chain_start,
                           int32_t n_chains, int32_t L, int32_t nex, int32_t degree, double tol,
                           int32_t max_iter, uint64_t seed, double* evals_host, double* evecs_host,
                           int64_t ld_host, scsf_stats* st, void* ws, size_t ws_bytes, void* stream);

/*
 * Resumable chains ("per-chain cursor plus the last Ritz block
 * persisted, so a chain resumes from its last solved operator as a warm start";
 * warm start P:270-277, "V~_0 = V^(i-1)").  A chain's state after an
 * operator is what the next operator's warm start reads:
 *   state = [ theta (b doubles, Ritz values ascending) | V (b x n, column-major, ld = n) ]
 * scsf_chain_state_doubles returns b * (n + 1) (0 on bad arguments).
 * scsf_solve_chains_resume is scsf_solve_chains where
 *  state_in   dev [n_chains][state] or NULL.  Non-NULL: chain c's first operator
 *             warm-starts from state_in[c] exactly as if it followed, in one call,
 *             the operator that produced it (inherited bounds included), so a
 *             queue solved in segments gives bit-identical pairs to one pass.
 *             NULL: every chain starts cold (seeded random block).
 *  state_out  dev [n_chains][state] out (required; must not alias state_in): the
 *             state after each chain's last operator of this call.  A chain with an
 *             empty slice copies state_in[c] (or writes NaNs when state_in is NULL).
 * Errors as scsf_solve_chains; SCSF_ERR_ARG when state_out is NULL or aliases state_in.
 */
int64_t scsf_chain_state_doubles(const scsf_ops* ops, int32_t L, int32_t nex);
int scsf_solve_chains_resume(const scsf_ops* ops, const int32_t* queue, const int32_t* chain_start,
                             int32_t n_chains, int32_t L, int32_t nex, int32_t degree, double tol,
                             int32_t max_iter, uint64_t seed, const double* state_in, double* state_out,
                             double* evals, double* evecs, int64_t ld_vec, scsf_stats* st, void* ws,
                             size_t ws_bytes, void* stream);

/* ------------------------------------------- row-partitioned solve ---- */
/*
 * One operator too large for one GPU's share of the work (BASELINE.json
 * configs[4]): the grid rows of a 2-D operator are
 * split into contiguous slabs, one per rank; every n x b block of Alg. 3
 * holds only the rank's rows.  The exchange steps:
 *  - before every stencil application (filter step, Alg. 1; W = AQ,
 *    P:302): the slab's first / last grid row of every column goes to the
 *    lower / upper neighbour (halo);
 *  - every Gram / projection block X^T Y (CholQR l. 4 P:301, BCGS against the
 *    locked vectors, G = Q^T A Q l. 5 P:302) and the residual norms (l. 7,
 *    P:304, metric P:844) are summed over ranks;
 *  - the b x b factorisation / eigensolve (ll. 4-6) runs replicated on every
 *    rank on the identical all-reduced input, so every rank takes the same
 *    locking decision;
 *  - the sign convention of the returned vectors uses the global largest |.|
 *    entry (all-gather of per-rank candidates).
 * Operator arrays stay global (replicated: 8 (1 + dim) n bytes per operator,
 * small next to the b-column blocks); the chain-head random block is the
 * same global block on any partition (counter-based, global row index).
 *
 * scsf_comm: NCCL over NVLink/NVSwitch (one process per GPU; libnccl is
 * resolved at run time from the process, i.e. the copy torch loaded) or an
 * in-process loopback of `world` virtual ranks on one device (each driven
 * by its own host thread; collectives meet at a host barrier, no kernel
 * waits on another rank).  The loopback allocates its own tiny device
 * scratch (pointer tables), the one exception to "the library never
 * allocates device memory".
 *
 * scsf_comm_unique_id   128 B NCCL id (rank 0; the caller broadcasts it)
 * scsf_comm_create      NCCL communicator for (rank, world); collective over
 *                       all ranks (ncclCommInitRank)
 * scsf_comm_create_loopback  out[world]: communicators of `world` virtual ranks
 * scsf_slab_rows        rows [y0, y1) of `rank`: y0 = floor(rank ny / world)
 * scsf_solve_queue_dist scsf_solve_queue on this rank's slab.  ops: the global
 *                       operator batch (dim 2, nx % 4 == 0); [y0, y1) must be
 *                       scsf_slab_rows(ny, world, rank).  evals dev
 *                       [n_chain][L] (identical on every rank); evecs_local
 *                       dev [n_chain][L][ld_vec] or NULL, the slab's rows
 *                       (ld_vec >= nx (y1 - y0)).  Every rank must call it
 *                       with the same chain and parameters.
 * Errors as scsf_solve_queue; SCSF_ERR_NOT_IMPLEMENTED when NCCL cannot be
 * loaded; SCSF_ERR_ARG for dim 3, nx % 4 != 0 or a slab that does not match.
 */
typedef struct scsf_comm scsf_comm;
int scsf_comm_unique_id(void* id128);
int scsf_comm_create(int32_t rank, int32_t world, const void* id128, scsf_comm** out);
int scsf_comm_create_loopback(int32_t world, scsf_comm** out);
int scsf_comm_destroy(scsf_comm* comm);
int scsf_comm_rank(const scsf_comm* comm, int32_t* rank, int32_t* world);
void scsf_slab_rows(int32_t ny, int32_t world, int32_t rank, int32_t* y0, int32_t* y1);
size_t scsf_solve_dist_workspace_bytes(const scsf_ops* ops, int32_t y0, int32_t y1, int32_t L,
                                       int32_t nex, int32_t world);
int scsf_solve_queue_dist(const scsf_ops* ops, int32_t y0, int32_t y1, const int32_t* chain,
                          int32_t n_chain, int32_t L, int32_t nex, int32_t degree, double tol,
                          int32_t max_iter, uint64_t seed, double* evals, double* evecs_local,
                          int64_t ld_vec, scsf_stats* st, scsf_comm* comm, void* ws,
                          size_t ws_bytes, void* stream);

/* ------------------------------------------- component entry points ---- */
/*
 * Single steps of Alg. 3 exposed for parity tests and microbenchmarks.  Same
 * conventions as above; all pointers device; synchronous; ws from the query.
 *
 * scsf_gemm_tn:  C (b1 x b2, ldc) = alpha X^T Y, X n x b1 (ldx), Y n x b2 (ldy):
 *   the Gram / Rayleigh-quotient contraction (Alg. 3 ll. 4-5).
 *   upper != 0: only the upper triangle (i <= j, b1 == b2) is defined on return.
 * scsf_gemm_nn:  Out (n x b2, ldo) = alpha X M + beta Out, X n x b1, M b1 x b2
 *   (ldm): the basis rotation / triangular apply (ll. 4 and 6).
 *   Out may alias X (in-place) when ldo == ldx.
 * scsf_chol_inv: S (b x b, upper triangle used) = R^T R; writes R^{-1} (b x b,
 *   upper, ld b): CholQR's small factor (l. 4, reading R13).  Returns
 *   SCSF_ERR_NUMERICAL if S needed the shifted fallback.
 * scsf_syev_small: G (b x b, upper triangle used) = Z diag(theta) Z^T, theta
 *   ascending (b), Z (b x b, ld b): the reduced eigenproblem (l. 6).
 *   SCSF_ERR_NUMERICAL if the sweep cap was hit.
 */
size_t scsf_dev_workspace_bytes(int64_t n, int32_t b1, int32_t b2);
int scsf_gemm_tn(const double* X, int64_t ldx, int32_t b1, const double* Y, int64_t ldy, int32_t b2,
                 int64_t n, double alpha, int32_t upper, double* C, int64_t ldc, void* ws,
                 size_t ws_bytes, void* stream);
int scsf_gemm_nn(const double* X, int64_t ldx, int64_t n, int32_t b1, const double* M, int64_t ldm,
                 int32_t b2, double alpha, double beta, double* Out, int64_t ldo, void* stream);
int scsf_chol_inv(const double* S, int64_t lds, int32_t b, int64_t nrows, double* Rinv, void* ws,
                  size_t ws_bytes, void* stream);
int scsf_syev_small(const double* G, int64_t ldg, int32_t b, double* theta, double* Z,
                    int32_t* sweeps /* host out or NULL */, void* ws, size_t ws_bytes, void* stream);

/* ------------------------------------------------------------- helpers ---- */

const char* scsf_last_error(void);   /* thread-local message for the last non-OK status */
int scsf_abi_version(void);          /* SCSF_ABI_VERSION                                */
int64_t scsf_launch_count(void);     /* kernels launched by this process so far         */
int scsf_set_timing(int32_t on);     /* enable per-phase CUDA-event timers; returns the old state */
/* which Alg. 1 kernel the solver uses for these operators: 3 = register-patch
 * cluster-resident whole filter (k_filter_rp), 2 = cluster-resident whole filter
 * (k_filter_cl), 1 = single-CTA resident (k_filter_res2d), 0 = one streaming
 * launch per step (k_stencil_v4 / k_stencil / k_stencil_vib_t); -1 = invalid ops */
int scsf_filter_kind(const scsf_ops* ops);

#ifdef __cplusplus
}
#endif
#endif /* SCSF_H_ */
