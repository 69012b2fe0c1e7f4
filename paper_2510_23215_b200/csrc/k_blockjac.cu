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

#include <vector>

namespace scsf {

int jacobi_batched_impl(const double* G, int64_t ldg, int bs, int batch, int64_t gstride, double* scratch,
                        double* theta, double* Q, Ctrl* ctrl, cudaStream_t s);

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
                          double* __restrict__ Gp, double* __restrict__ Zp) {
  const int i = blockIdx.x * blockDim.x + threadIdx.x, j = blockIdx.y;
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
                                                  const double* __restrict__ Q, int m, double* __restrict__ Out) {
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

// Block permutation: new position block pb holds old block src[pb] (w indices each).
struct BjPerm {
  int src[8];
};
__global__ void k_bj_perm(const double* __restrict__ Gin, const double* __restrict__ Zin, int n, int w, BjPerm p,
                          double* __restrict__ Gout, double* __restrict__ Zout) {
  const int i = blockIdx.x * blockDim.x + threadIdx.x, j = blockIdx.y;
  if (i >= n) return;
  const int oi = p.src[i / w] * w + i % w, oj = p.src[j / w] * w + j % w;
  Gout[i + (int64_t)j * n] = Gin[oi + (int64_t)oj * n];
  Zout[i + (int64_t)j * n] = Zin[i + (int64_t)oj * n];          // Z: columns only
}

// max_{i<j} |g_ij| / sqrt|g_ii g_jj| over real indices (orig >= 0); flag = (max > tol)
__global__ void __launch_bounds__(1024) k_bj_offmax(const double* __restrict__ Gp, int n, const int* __restrict__ orig,
                                                    double tol, int* __restrict__ flag) {
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
    if (i >= j || orig[i] < 0 || orig[j] < 0) continue;
    const double g = fabs(Gp[idx]);
    if (g > gfloor) mx = fmax(mx, g / fmax(sqrt(fabs(Gp[i + (int64_t)i * n] * Gp[j + (int64_t)j * n])), 1e-300));
  }
  mx = warp_max(mx);
  if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = mx;
  __syncthreads();
  if (threadIdx.x == 0) {
    double v = 0.0;
    for (int k = 0; k < 32; ++k) v = fmax(v, red[k]);
    *flag = v > tol ? 1 : 0;
  }
}

// theta ascending over the real indices, Zout[:, rank] = Zp[orig rows, position] (b x b, ld b)
__global__ void __launch_bounds__(512) k_bj_final(const double* __restrict__ Gp, const double* __restrict__ Zp, int n,
                                                  const int* __restrict__ orig, int b, double* __restrict__ theta,
                                                  double* __restrict__ Zout) {
  __shared__ int rank_s[512];
  for (int pos = threadIdx.x; pos < n; pos += 512) {
    int rk = -1;
    if (orig[pos] >= 0) {
      const double v = Gp[pos + (int64_t)pos * n];
      rk = 0;
      for (int q = 0; q < n; ++q) {
        if (orig[q] < 0) continue;
        const double u = Gp[q + (int64_t)q * n];
        rk += (u < v) || (u == v && orig[q] < orig[pos]);
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

__global__ void k_bj_flag(Ctrl* ctrl) { atomicOr(&ctrl->nonfinite, 2); }

size_t blockjac_scratch_doubles(int b) {
  const int nb = 2 * ((b + 127) / 128), w = (b + nb - 1) / nb, n = nb * w;
  return (size_t)4 * n * n + (size_t)(nb / 2) * 128 * 128 + (size_t)n + 4096;
}

// G (b x b, upper, ldg) = Z diag(theta) Z^T, theta ascending (b), Z (b x b, ld b).
// scratch: blockjac_scratch_doubles(b) doubles; jscratch: the batched one-CTA Jacobi scratch.
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
  int* orig_d = reinterpret_cast<int*>(th + n);
  int* flag_d = orig_d + 512;
  int* flag_h = nullptr;
  static thread_local int* t_flag = nullptr;
  static thread_local cudaEvent_t t_ev = nullptr;
  if (!t_flag) {
    SCSF_CUDA_CHECK(cudaMallocHost(&t_flag, sizeof(int)));
    SCSF_CUDA_CHECK(cudaEventCreateWithFlags(&t_ev, cudaEventBlockingSync | cudaEventDisableTiming));
  }
  flag_h = t_flag;
  const size_t smm = (size_t)(m * (BJ_R + 1) + m * m) * sizeof(double);
  static bool attr = false;
  if (!attr) {
    SCSF_CUDA_CHECK(cudaFuncSetAttribute(k_bj_blkmm, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                         (int)((128 * (BJ_R + 1) + 128 * 128) * sizeof(double))));
    attr = true;
  }
  double* bound_d = reinterpret_cast<double*>(flag_d + 16);
  k_bj_bound<<<1, 512, 0, s>>>(G, ldg, b, bound_d);
  SCSF_LAUNCH_CHECK();
  k_bj_load<<<dim3(ceil_div(n, 128), n), 128, 0, s>>>(G, ldg, b, n, bound_d, Gp, Zp);
  SCSF_LAUNCH_CHECK();
  // tournament (circle method): c[0] fixed, c[1..nb-1] rotate; pairs (c[i], c[nb-1-i]) -> positions (2i, 2i+1)
  std::vector<int> c(nb), arr(nb), cur(nb);
  for (int i = 0; i < nb; ++i) c[i] = i, cur[i] = i;
  std::vector<int> orig(n);
  for (int i = 0; i < n; ++i) orig[i] = (i < b) ? i : -1;
  const int max_sweeps = 30;
  int sweep = 0;
  for (; sweep < max_sweeps; ++sweep) {
    for (int r = 0; r < nb - 1; ++r) {
      for (int i = 0; i < P; ++i) {
        arr[2 * i] = c[i];
        arr[2 * i + 1] = c[nb - 1 - i];
      }
      // bring the arrangement `arr` into place: new position pb holds the block now at position of arr[pb]
      BjPerm pm{};
      bool ident = true;
      for (int pb = 0; pb < nb; ++pb) {
        int at = 0;
        while (cur[at] != arr[pb]) ++at;
        pm.src[pb] = at;
        ident = ident && (at == pb);
      }
      if (!ident) {
        k_bj_perm<<<dim3(ceil_div(n, 128), n), 128, 0, s>>>(Gp, Zp, n, w, pm, T, T2);
        SCSF_LAUNCH_CHECK();
        std::swap(Gp, T);
        std::swap(Zp, T2);
        std::vector<int> no(n);
        for (int i = 0; i < n; ++i) no[i] = orig[pm.src[i / w] * w + i % w];
        orig.swap(no);
        cur = arr;
      }
      // P sub-problems on the diagonal blocks of width m, one CTA each
      SCSF_TRY(jacobi_batched_impl(Gp, n, m, P, (int64_t)m * (n + 1), jscratch, th, Q, ctrl, s));
      // G <- Q^T G Q  (T = G Q, G = T^T Q by symmetry),  Z <- Z Q
      k_bj_blkmm<<<dim3(ceil_div(n, BJ_R), P), 256, smm, s>>>(Gp, n, 0, Q, m, T);
      SCSF_LAUNCH_CHECK();
      k_bj_blkmm<<<dim3(ceil_div(n, BJ_R), P), 256, smm, s>>>(T, n, 1, Q, m, Gp);
      SCSF_LAUNCH_CHECK();
      k_bj_blkmm<<<dim3(ceil_div(n, BJ_R), P), 256, smm, s>>>(Zp, n, 0, Q, m, T);
      SCSF_LAUNCH_CHECK();
      std::swap(Zp, T);
      // rotate the circle
      const int last = c[nb - 1];
      for (int i = nb - 1; i > 1; --i) c[i] = c[i - 1];
      c[1] = last;
    }
    SCSF_CUDA_CHECK(cudaMemcpyAsync(orig_d, orig.data(), n * sizeof(int), cudaMemcpyHostToDevice, s));
    k_bj_offmax<<<1, 1024, 0, s>>>(Gp, n, orig_d, 1e-14, flag_d);
    SCSF_LAUNCH_CHECK();
    SCSF_CUDA_CHECK(cudaMemcpyAsync(flag_h, flag_d, sizeof(int), cudaMemcpyDeviceToHost, s));
    SCSF_CUDA_CHECK(cudaEventRecord(t_ev, s));
    SCSF_CUDA_CHECK(cudaEventSynchronize(t_ev));
    if (*flag_h == 0) break;
  }
  if (sweep >= max_sweeps && ctrl) {
    k_bj_flag<<<1, 1, 0, s>>>(ctrl);
    SCSF_LAUNCH_CHECK();
  }
  SCSF_CUDA_CHECK(cudaMemcpyAsync(orig_d, orig.data(), n * sizeof(int), cudaMemcpyHostToDevice, s));
  k_bj_final<<<1, 512, 0, s>>>(Gp, Zp, n, orig_d, b, theta, Zout);
  SCSF_LAUNCH_CHECK();
  return SCSF_OK;
}

}  // namespace scsf
