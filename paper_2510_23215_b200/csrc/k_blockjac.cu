// k_blockjac.cu — the reduced eigenproblem of Alg. 3 l. 6 for
// blocks wider than one CTA's Jacobi (b > 128: configs[2] b = 240, configs[4]
// b = 360).  Two-sided *block* Jacobi (the method is unstated by the paper;
// reading R10-adjacent): the index set is cut into nb = 2P blocks
// of width w <= 64; each round pairs the blocks (round-robin tournament) into
// P sub-problems of size 2w <= 128 that are diagonalised exactly by the
// one-CTA Jacobi kernels (batched, one CTA per sub-problem), and the whole
// matrix is rotated with the block-diagonal Q:  G <- Q^T G Q,  Z <- Z Q.
// G is kept in the round's block order (each sub-problem is a contiguous
// diagonal block); between rounds a block permutation re-arranges G and Z.
// Padded indices (b rounded up to nb w) are exactly decoupled (zero rows and
// columns) and dropped at the end.  Sweeps stop when every off-diagonal
// |g_ij| <= 1e-14 sqrt|g_ii g_jj| (as the one-CTA Jacobi).
#include "common.cuh"

#include <cstdlib>
#include <mutex>
#include <vector>

namespace scsf {

int jacobi_batched_impl(const double* G, int64_t ldg, int bs, int batch, int64_t gstride, double* scratch,
                        double* theta, double* Q, Ctrl* ctrl, cudaStream_t s, const int* skip);

// Every kernel of a sweep takes `run` (the loop flag): inside a captured, unrolled sweep sequence
// a sweep after convergence (*run == 0) returns at once.
__device__ __forceinline__ bool bj_skip(const int* run) { return run && *(volatile const int*)run == 0; }

// Gershgorin bound max_i sum_j |g_ij| of the upper-stored G (one CTA)
__global__ void __launch_bounds__(512) k_bj_bound(const double* __restrict__ G, int64_t ldg, int b,
                                                  double* __restrict__ out) {
  double m = 0.0;
  for (int i = threadIdx.x; i < b; i += 512) {
    double r = 0.0;
    for (int j = 0; j < b; ++j) r += fabs(i <= j ? G[i + (int64_t)j * ldg] : G[j + (int64_t)i * ldg]);
    m = fmax(m, r);
  }
  __shared__ double red[16];
  m = warp_max(m);
  if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = m;
  __syncthreads();
  if (threadIdx.x == 0) {
    double v = 0.0;
    for (int k = 0; k < 16; ++k) v = fmax(v, red[k]);
    *out = v;
  }
}

// Gp (n x n, full) from the upper triangle of G (b x b, ldg).  Padding indices are decoupled
// (zero off-diagonal) with a diagonal above the whole spectrum (2 x the Gershgorin bound + 1),
// so every sorted sub-solve keeps them last, i.e. at their own positions.
__global__ void k_bj_load(const double* __restrict__ G, int64_t ldg, int b, int n, const double* __restrict__ bound,
                          double* __restrict__ Gp, double* __restrict__ Zp, int* __restrict__ counter) {
  const int i = blockIdx.x * blockDim.x + threadIdx.x, j = blockIdx.y;
  if (i == 0 && j == 0) {
    counter[0] = 0;                                   // sweeps of this solve
    counter[-1] = 1;                                  // the loop flag: run the first sweep
  }
  if (i >= n) return;
  double v = 0.0;
  if (i < b && j < b) v = (i <= j) ? G[i + (int64_t)j * ldg] : G[j + (int64_t)i * ldg];
  else if (i == j) v = 2.0 * (*bound) + 1.0;
  Gp[i + (int64_t)j * n] = v;
  Zp[i + (int64_t)j * n] = (i == j) ? 1.0 : 0.0;
}

// Out[r, q m + c] = sum_k op(X)[r, q m + k] Q_q[k, c],  op(X) = X or X^T (X n x n, ld n),
// Q_q = Q + q m^2 (m x m, ld m).  CTA: 32 rows x the m columns of one block q.
constexpr int BJ_R = 32;
__global__ void __launch_bounds__(256) k_bj_blkmm(const double* __restrict__ X, int n, int transX,
                                                  const double* __restrict__ Q, int m, double* __restrict__ Out,
                                                  const int* run) {
  if (bj_skip(run)) return;
  extern __shared__ double sm[];
  double* xs = sm;                           // [m][BJ_R + 1]: xs[k][r]
  double* qs = sm + m * (BJ_R + 1);          // [m][m]: qs[k + c m]
  const int r0 = blockIdx.x * BJ_R, q = blockIdx.y, tid = threadIdx.x;
  const double* Qq = Q + (int64_t)q * m * m;
  for (int i = tid; i < m * m; i += 256) qs[i] = Qq[i];
  for (int i = tid; i < m * BJ_R; i += 256) {
    int k, r;
    if (transX) { r = i / m; k = i % m; } else { k = i / BJ_R; r = i % BJ_R; }
    const int row = r0 + r, col = q * m + k;
    double v = 0.0;
    if (row < n) v = transX ? X[col + (int64_t)row * n] : X[row + (int64_t)col * n];
    xs[k * (BJ_R + 1) + r] = v;
  }
  __syncthreads();
  // thread: row r = tid % 32, columns c = tid / 32 + 8 t
  const int r = tid & 31, c0 = tid >> 5;
  double acc[16];
#pragma unroll
  for (int t = 0; t < 16; ++t) acc[t] = 0.0;
  for (int k = 0; k < m; ++k) {
    const double xv = xs[k * (BJ_R + 1) + r];
#pragma unroll
    for (int t = 0; t < 16; ++t) {
      const int c = c0 + 8 * t;
      if (c < m) acc[t] = fma(xv, qs[k + c * m], acc[t]);
    }
  }
  const int row = r0 + r;
  if (row < n)
#pragma unroll
    for (int t = 0; t < 16; ++t) {
      const int c = c0 + 8 * t;
      if (c < m) Out[row + (int64_t)(q * m + c) * n] = acc[t];
    }
}

struct BjPerm {
  int src[8];
};
// dst = src, n*n doubles (an SM copy: inside the captured sweep body a memcpy node would go to a
// copy engine shared by every chain)
__global__ void k_bj_copy(const double* __restrict__ src, double* __restrict__ dst, int64_t count, const int* run) {
  if (bj_skip(run)) return;
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < count; i += (int64_t)gridDim.x * blockDim.x)
    dst[i] = src[i];
}

__global__ void k_bj_perm(const double* __restrict__ Gin, const double* __restrict__ Zin, int n, int w, BjPerm p,
                          double* __restrict__ Gout, double* __restrict__ Zout, const int* run) {
  if (bj_skip(run)) return;
  const int i = blockIdx.x * blockDim.x + threadIdx.x, j = blockIdx.y;
  if (i >= n) return;
  const int oi = p.src[i / w] * w + i % w, oj = p.src[j / w] * w + j % w;
  Gout[i + (int64_t)j * n] = Gin[oi + (int64_t)oj * n];
  Zout[i + (int64_t)j * n] = Zin[i + (int64_t)oj * n];          // Z: columns only
}

// Block permutation: new position block pb holds old block src[pb] (w indices each).
// Original index held at position i when position block i / w holds original block arr[i / w]
// (-1 for padding).
__device__ __forceinline__ int bj_orig(const BjPerm& arr, int i, int w, int b) {
  const int o = arr.src[i / w] * w + i % w;
  return o < b ? o : -1;
}

// One sweep's convergence test: max_{i<j} |g_ij| / sqrt|g_ii g_jj| over real indices, against tol.
// Continues the sweep loop (DevLoop) while above tol and fewer than max_sweeps sweeps ran; a loop
// that stops on the cap flags ctrl->nonfinite bit 2 (informational: the Rayleigh-Ritz rotation is
// then exact but G not fully diagonal, so the residual test of l. 7 simply locks less).
// COND: the kernel may set the WHILE node's condition (only the conditional-node mode needs that;
// ncu does not profile, and the graph treats specially, kernels that can set a conditional handle)
template <bool COND>
__global__ void __launch_bounds__(1024) k_bj_offmax(const double* __restrict__ Gp, int n, BjPerm arr, int w, int b,
                                                    double tol, int* __restrict__ counter, int max_sweeps,
                                                    Ctrl* ctrl, DevLoop loop) {
  if (bj_skip(loop.flag)) return;                      // (unrolled sweeps after convergence)
  double mx = 0.0, dmax = 0.0;
  for (int i = threadIdx.x; i < n; i += 1024) dmax = fmax(dmax, fabs(Gp[i + (int64_t)i * n]));
  __shared__ double red[32];
  dmax = warp_max(dmax);
  if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = dmax;
  __syncthreads();
  if (threadIdx.x == 0) {
    double v = 0.0;
    for (int k = 0; k < 32; ++k) v = fmax(v, red[k]);
    red[0] = v;
  }
  __syncthreads();
  // rounding floor of the block updates (two n-long dot products per entry): entries below it are noise
  const double gfloor = 8.0 * n * 2.220446049250313e-16 * red[0];   // (padding diagonals included: ~2 ||G||)
  __syncthreads();
  for (int64_t idx = threadIdx.x; idx < (int64_t)n * n; idx += 1024) {
    const int i = (int)(idx % n), j = (int)(idx / n);
    if (i >= j || bj_orig(arr, i, w, b) < 0 || bj_orig(arr, j, w, b) < 0) continue;
    const double g = fabs(Gp[idx]);
    if (g > gfloor) mx = fmax(mx, g / fmax(sqrt(fabs(Gp[i + (int64_t)i * n] * Gp[j + (int64_t)j * n])), 1e-300));
  }
  mx = warp_max(mx);
  if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = mx;
  __syncthreads();
  if (threadIdx.x == 0) {
    double v = 0.0;
    for (int k = 0; k < 32; ++k) v = fmax(v, red[k]);
    const int cnt = ++(*counter);
    const bool above = v > tol;
    if (ctrl) ctrl->pad[0] += 1;                   // cumulative sweeps (stats)
    if (above && cnt >= max_sweeps && ctrl) atomicOr(&ctrl->nonfinite, 2);
    if (COND)
      dev_loop_continue(loop, above && cnt < max_sweeps);
    else
      *loop.flag = (above && cnt < max_sweeps) ? 1 : 0;
  }
}

// theta ascending over the real indices, Zout[:, rank] = Zp[orig rows, position] (b x b, ld b)
__global__ void __launch_bounds__(512) k_bj_final(const double* __restrict__ Gp, const double* __restrict__ Zp, int n,
                                                  BjPerm arr, int w, int b, double* __restrict__ theta,
                                                  double* __restrict__ Zout) {
  __shared__ int rank_s[512];
  for (int pos = threadIdx.x; pos < n; pos += 512) {
    int rk = -1;
    const int op = bj_orig(arr, pos, w, b);
    if (op >= 0) {
      const double v = Gp[pos + (int64_t)pos * n];
      rk = 0;
      for (int q = 0; q < n; ++q) {
        const int oq = bj_orig(arr, q, w, b);
        if (oq < 0) continue;
        const double u = Gp[q + (int64_t)q * n];
        rk += (u < v) || (u == v && oq < op);
      }
      theta[rk] = v;
    }
    rank_s[pos] = rk;
  }
  __syncthreads();
  // Zp rows are original indices (Z <- Z Q acts on columns); column pos -> output column rank
  for (int64_t idx = threadIdx.x; idx < (int64_t)n * n; idx += 512) {
    const int row = (int)(idx % n), pos = (int)(idx / n);
    const int rk = rank_s[pos];
    if (rk < 0 || row >= b) continue;
    Zout[row + (int64_t)rk * b] = Zp[row + (int64_t)pos * n];
  }
}

// SCSF_BJ_UNROLL=k (default 6): inside a CUDA-graph capture, run k unrolled sweeps whose kernels
// return at once after convergence; 0: a WHILE conditional node instead.  Measured on C3 (64
// operators, 32 chains, tools/graph_ab.py): m = 60: unrolled 2.10-2.14 s, eager with a host
// synchronisation per sweep 2.31 s, conditional node 2.57 s (device-launched bodies of the 32
// chains' graphs do not overlap as well); m = 120: unroll 4 / 5 / 6 / 8: 1.71 / 1.72 / 1.71 / 1.73 s,
// and 6 sweeps never truncated a solve (3.58 sweeps per iteration, as the unbounded loop)
static int bj_unroll() {
  static const int v = [] {            // thread-safe one-time read (chain worker threads)
    int v;
    const char* e = getenv("SCSF_BJ_UNROLL");
    v = e ? atoi(e) : 6;
    if (v < 0) v = 0;
    return v;
  }();
  return v;
}

size_t blockjac_scratch_doubles(int b) {
  const int nb = 2 * ((b + 127) / 128), w = (b + nb - 1) / nb, n = nb * w;
  return (size_t)4 * n * n + (size_t)(nb / 2) * 128 * 128 + (size_t)n + 4096;
}

// G (b x b, upper, ldg) = Z diag(theta) Z^T, theta ascending (b), Z (b x b, ld b).
// scratch: blockjac_scratch_doubles(b) doubles; jscratch: the batched one-CTA Jacobi scratch.
//
// The round-robin schedule is fixed, so the host computes every round's block permutation
// up front; the blocks are first arranged as in the last round of a sweep, which makes all
// sweeps identical.  The sweeps run as a device-decided loop (device_while): inside a
// CUDA-graph capture a WHILE conditional node, so a b > 128 outer iteration replays from
// one graph with no host synchronisation.
int blockjac_impl(const double* G, int64_t ldg, int b, double* scratch, double* jscratch, double* theta,
                  double* Zout, Ctrl* ctrl, cudaStream_t s) {
  const int nb = 2 * ((b + 127) / 128), P = nb / 2;
  const int w = (b + nb - 1) / nb, m = 2 * w, n = nb * w;
  if (nb > 8) {
    set_error("block Jacobi: b = %d too large", b);
    return SCSF_ERR_NOT_IMPLEMENTED;
  }
  double* Gp = scratch;
  double* Zp = Gp + (size_t)n * n;
  double* T = Zp + (size_t)n * n;
  double* T2 = T + (size_t)n * n;
  double* Q = T2 + (size_t)n * n;
  double* th = Q + (size_t)P * 128 * 128;
  int* aux_d = reinterpret_cast<int*>(th + n);      // [0] loop flag, [1] sweep counter
  int* flag_d = aux_d;
  int* counter_d = aux_d + 1;
  static thread_local int* t_flag = nullptr;
  if (!t_flag) SCSF_CUDA_CHECK(cudaMallocHost(&t_flag, sizeof(int)));
  const size_t smm = (size_t)(m * (BJ_R + 1) + m * m) * sizeof(double);
  static std::once_flag attr_once;
  static cudaError_t attr_err = cudaSuccess;
  std::call_once(attr_once, [] {
    attr_err = cudaFuncSetAttribute(k_bj_blkmm, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                    (int)((128 * (BJ_R + 1) + 128 * 128) * sizeof(double)));
  });
  SCSF_CUDA_CHECK(attr_err);
  double* bound_d = reinterpret_cast<double*>(aux_d + 16);
  k_bj_bound<<<1, 512, 0, s>>>(G, ldg, b, bound_d);
  SCSF_LAUNCH_CHECK();
  k_bj_load<<<dim3(ceil_div(n, 128), n), 128, 0, s>>>(G, ldg, b, n, bound_d, Gp, Zp, counter_d);
  SCSF_LAUNCH_CHECK();
  // tournament (circle method): c[0] fixed, c[1..nb-1] rotate; pairs (c[i], c[nb-1-i]) -> positions (2i, 2i+1).
  // After nb - 1 rounds the circle is back where it started, so every sweep has the same arrangements.
  std::vector<BjPerm> arr(nb - 1);
  std::vector<int> c(nb);
  for (int i = 0; i < nb; ++i) c[i] = i;
  for (int r = 0; r < nb - 1; ++r) {
    for (int i = 0; i < P; ++i) {
      arr[r].src[2 * i] = c[i];
      arr[r].src[2 * i + 1] = c[nb - 1 - i];
    }
    const int last = c[nb - 1];
    for (int i = nb - 1; i > 1; --i) c[i] = c[i - 1];
    c[1] = last;
  }
  // permutation taking arrangement `from` (position -> original block) to `to`
  auto perm_between = [&](const BjPerm& from, const BjPerm& to, BjPerm& pm) {
    bool ident = true;
    for (int pb = 0; pb < nb; ++pb) {
      int at = 0;
      while (from.src[at] != to.src[pb]) ++at;
      pm.src[pb] = at;
      ident = ident && (at == pb);
    }
    return ident;
  };
  BjPerm idn{};
  for (int i = 0; i < nb; ++i) idn.src[i] = i;
  const BjPerm& A_last = arr[nb - 2];
  // bring the identity arrangement into the last round's (the loop's invariant at each sweep start)
  BjPerm pm0;
  if (!perm_between(idn, A_last, pm0)) {
    k_bj_perm<<<dim3(ceil_div(n, 128), n), 128, 0, s>>>(Gp, Zp, n, w, pm0, T, T2, nullptr);
    SCSF_LAUNCH_CHECK();
    k_bj_copy<<<ceil_div((int64_t)n * n, 1024), 256, 0, s>>>(T, Gp, (int64_t)n * n, nullptr);
    SCSF_LAUNCH_CHECK();
    k_bj_copy<<<ceil_div((int64_t)n * n, 1024), 256, 0, s>>>(T2, Zp, (int64_t)n * n, nullptr);
    SCSF_LAUNCH_CHECK();
  }
  std::vector<BjPerm> pms(nb - 1);
  std::vector<bool> ident(nb - 1);
  for (int r = 0; r < nb - 1; ++r) ident[r] = perm_between(r == 0 ? A_last : arr[r - 1], arr[r], pms[r]);
  const int max_sweeps = 30;
  // One sweep.  Every round ends with G and Z back in (Gp, Zp): a permutation or Z <- Z Q that
  // lands in T / T2 is copied back, so the captured body is position-independent.
  // unrolled mode (captured): a fixed number of sweeps whose kernels return at once after convergence
  const int unroll = stream_capturing(s) ? bj_unroll() : 0;
  const int cap = unroll > 0 ? unroll : max_sweeps;
  auto sweep = [&](cudaStream_t bs, const DevLoop& loop) -> int {
    const int* run = loop.flag;
    for (int r = 0; r < nb - 1; ++r) {
      if (!ident[r]) {
        k_bj_perm<<<dim3(ceil_div(n, 128), n), 128, 0, bs>>>(Gp, Zp, n, w, pms[r], T, T2, run);
        SCSF_LAUNCH_CHECK();
      }
      const double* Gr = ident[r] ? Gp : T;
      const double* Zr = ident[r] ? Zp : T2;
      // P sub-problems on the diagonal blocks of width m, one CTA each
      SCSF_TRY(jacobi_batched_impl(Gr, n, m, P, (int64_t)m * (n + 1), jscratch, th, Q, ctrl, bs, run));
      // G <- Q^T G Q  (X = G Q, G = X^T Q by symmetry),  Z <- Z Q
      if (!ident[r]) {                                   // G' in T, Z' in T2; Gp, Zp are free
        k_bj_blkmm<<<dim3(ceil_div(n, BJ_R), P), 256, smm, bs>>>(Gr, n, 0, Q, m, Gp, run);     // Gp = (T) Q
        SCSF_LAUNCH_CHECK();
        k_bj_blkmm<<<dim3(ceil_div(n, BJ_R), P), 256, smm, bs>>>(Gp, n, 1, Q, m, T, run);      // T = Gp^T Q
        SCSF_LAUNCH_CHECK();
        k_bj_blkmm<<<dim3(ceil_div(n, BJ_R), P), 256, smm, bs>>>(Zr, n, 0, Q, m, Zp, run);     // Zp = T2 Q
        SCSF_LAUNCH_CHECK();
        k_bj_copy<<<ceil_div((int64_t)n * n, 1024), 256, 0, bs>>>(T, Gp, (int64_t)n * n, run);
        SCSF_LAUNCH_CHECK();
      } else {
        k_bj_blkmm<<<dim3(ceil_div(n, BJ_R), P), 256, smm, bs>>>(Gp, n, 0, Q, m, T, run);      // T = Gp Q
        SCSF_LAUNCH_CHECK();
        k_bj_blkmm<<<dim3(ceil_div(n, BJ_R), P), 256, smm, bs>>>(T, n, 1, Q, m, Gp, run);      // Gp = T^T Q
        SCSF_LAUNCH_CHECK();
        k_bj_blkmm<<<dim3(ceil_div(n, BJ_R), P), 256, smm, bs>>>(Zp, n, 0, Q, m, T2, run);     // T2 = Zp Q
        SCSF_LAUNCH_CHECK();
        k_bj_copy<<<ceil_div((int64_t)n * n, 1024), 256, 0, bs>>>(T2, Zp, (int64_t)n * n, run);
        SCSF_LAUNCH_CHECK();
      }
    }
    if (loop.in_graph)
      k_bj_offmax<true><<<1, 1024, 0, bs>>>(Gp, n, A_last, w, b, 1e-14, counter_d, cap, ctrl, loop);
    else
      k_bj_offmax<false><<<1, 1024, 0, bs>>>(Gp, n, A_last, w, b, 1e-14, counter_d, cap, ctrl, loop);
    SCSF_LAUNCH_CHECK();
    return SCSF_OK;
  };
  if (unroll > 0) {
    DevLoop flag_only;
    flag_only.flag = flag_d;
    for (int k = 0; k < unroll; ++k) SCSF_TRY(sweep(s, flag_only));
  } else {
    SCSF_TRY(device_while(s, flag_d, t_flag, max_sweeps, sweep));
  }
  k_bj_final<<<1, 512, 0, s>>>(Gp, Zp, n, A_last, w, b, theta, Zout);
  SCSF_LAUNCH_CHECK();
  return SCSF_OK;
}

}  // namespace scsf
